/*
 * sale.h -- C ABI of libsale, the B200-native SALE hot path.
 *
 * What it computes: the per-cycle staggered-grid hydro update of the SALE
 * scheme that ScalSALE (arXiv 2209.01983) is built on -- P:133 ("3D
 * multi-material hydrodynamic scheme ... based on ... SALE"), P:158 ("apply the
 * ideal gas equation-of-state"), P:181 (Table I: "Lagrangian rezoning, Eulerian
 * rezoning, Advection") -- on a structured 3D hexahedral mesh, for the
 * Sedov-Taylor blast wave (Fig. 2b "3D Eulerian Sedov-Taylor").
 * The paper gives no discrete equations; the operators are SURVEY.md §8(c)
 * c.1-c.6 with the readings listed in DESIGN.md §3 (round 2: the viscous hourglass
 * damping HG and the viscous signal speed in the time step DT-Q).  One cycle is:
 *   Lagrangian phase  S1-S7  (geometry, EoS, viscosity, CFL dt, corner forces with
 *                             hourglass damping, kinematics + reflecting BC,
 *                             compatible pdV energy)
 *   Eulerian remap    R1-R5  (rezone = SALE_EULER only: swept volumes,
 *                             donor-cell fluxes of mass/energy/momentum, reset)
 *   X1 halo exchange, X2 dt min-reduction   (z-slabs over ranks)
 *
 * Data layout, not visible through this ABI: SoA fp64 arrays in HBM, x fastest,
 * then y, then z planes; one z-slab per rank plus ghost planes.
 *
 * Ownership: the caller owns the device workspace, the CUDA stream and the
 * process group; the library owns the context, its NCCL communicator, a few
 * bytes of pinned host memory and, on single-rank contexts, a private stream plus
 * up to two CUDA graphs (a captured pair of cycles, replayed by sale_step on the
 * caller's stream; SALE_GRAPHS=0 in the environment disables them).  A context is
 * not thread-safe.  create / step / destroy are collective over the ranks of one
 * job.
 *
 * Error behaviour: every entry point returns a status code (SALE_OK = 0).  A
 * numerical error in sale_step (ETANGLED, EDTCOLLAPSE, ENEGMASS) or a CUDA /
 * NCCL failure poisons the context: later calls return SALE_EPOISONED, except
 * get_field / get_clock / last_error / destroy.  No entry point aborts or
 * prints.
 */
#ifndef SALE_H
#define SALE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SALE_ABI_VERSION 4
#define SALE_MAX_MAT 4       /* materials per cell (multi-material mode)            */

/* status codes */
#define SALE_OK 0
#define SALE_EINVAL 1        /* invalid argument / params / field / count           */
#define SALE_ENOMEM 2        /* workspace too small or NULL                         */
#define SALE_ECUDA 3         /* CUDA runtime error (detail in sale_last_error)      */
#define SALE_ENCCL 4         /* NCCL error                                          */
#define SALE_ETANGLED 5      /* some cell's new volume V' is not > 0 (c.3 step 7)   */
#define SALE_EDTCOLLAPSE 6   /* dt_u not > 0, or < 1e-14 * t_end (c.5; without an
                                end time: < 1e-14 * t, reading DT-C)                 */
#define SALE_ENEGMASS 7      /* remapped mass m'' not > 0 (c.4 step 3)              */
#define SALE_EPOISONED 8     /* context unusable after an earlier error             */
#define SALE_EREPLICA 9      /* replicated interface node planes differ (self-check) */

/* halo exchange modes (sale_params.halo) */
#define SALE_HALO_COPY 0     /* X1 as messages: grouped ncclSend/ncclRecv of whole ghost
                                planes between ranks, device copies between emulated slabs */
#define SALE_HALO_PEER 1     /* X1 fused into the kernels: the kernels that produce the planes
                                a neighbour needs also store them straight into its ghost
                                planes (the neighbour rank's workspace mapped over NVLink
                                with CUDA IPC, or the neighbouring emulated slab), then
                                signal it with one system-scope counter per cycle          */

/* rezone modes */
#define SALE_LAGRANGE 0
#define SALE_EULER 1

/* field ids; node fields 0..6, cell fields 7..13 (and the material fields 16..27 below) */
#define SALE_F_X 0
#define SALE_F_Y 1
#define SALE_F_Z 2
#define SALE_F_UX 3
#define SALE_F_UY 4
#define SALE_F_UZ 5
#define SALE_F_NODE_MASS 6   /* derived: M = 0.125 * sum of adjacent cell masses */
#define SALE_F_MASS 7
#define SALE_F_E 8           /* specific internal energy                          */
#define SALE_F_RHO 9         /* derived: m / V                                    */
#define SALE_F_VOL 10        /* derived: V from the 8 nodes (c.2)                 */
#define SALE_F_P 11          /* derived: (gamma-1) rho e, not floored             */
#define SALE_F_Q 12          /* derived: artificial viscosity at the current state */
#define SALE_F_CS 13         /* derived: sqrt(gamma max(p,0) / rho)               */
/* material fields (nmat >= 1; material m in [0, nmat)); cell fields, read and write */
#define SALE_F_MAT_F(m) (16 + (m))  /* volume fraction f_m                          */
#define SALE_F_MAT_M(m) (20 + (m))  /* material mass m_m; writing it re-sums MASS    */
#define SALE_F_MAT_E(m) (24 + (m))  /* material specific internal energy e_m         */

typedef struct sale_params {
    int32_t abi_version;      /* = SALE_ABI_VERSION                                */
    int32_t nx, ny, nz;       /* GLOBAL cells per axis, each >= 1                  */
    double lx, ly, lz;        /* domain [0,lx]x[0,ly]x[0,lz]; X_i = (lx*i)/nx      */
    double gamma;             /* ideal-gas gamma > 1                               */
    double q_lin, q_quad;     /* viscosity c1 (linear), c2 (quadratic), >= 0       */
    double cfl;               /* > 0                                               */
    double dt_growth;         /* dt <= dt_growth * dt_prev, > 0                    */
    double t_end;             /* <= 0: no end time; else stop when t >= t_end     */
    int32_t rezone;           /* SALE_LAGRANGE or SALE_EULER                       */
    uint32_t reflect_mask;    /* bit f set: face f of {-x,+x,-y,+y,-z,+z} reflects
                                 (normal velocity zeroed); clear: free surface.
                                 Sedov octant = 0x15                               */
    double rho0;              /* Sedov ambient density > 0                         */
    double e_background;      /* Sedov background specific energy                  */
    double e_deposit;         /* Sedov energy E0 placed in global cell (0,0,0)    */
    int32_t rank, nranks;     /* this process's rank in [0,nranks)                 */
    const void* nccl_unique_id; /* 128-byte ncclUniqueId from rank 0 (see
                                   sale_nccl_unique_id); required when nranks > 1.
                                   With nranks == 1 it is optional: a 1-rank NCCL
                                   communicator then carries the dt allreduce (used
                                   to exercise the NCCL path on a single GPU). */
    void* stream;             /* cudaStream_t to enqueue on (NULL = legacy stream) */
    void* workspace;          /* device memory, >= sale_workspace_bytes(), 256-B
                                 aligned, owned by the caller, not freed by us     */
    uint64_t workspace_bytes;
    int32_t device;           /* CUDA device ordinal this context runs on          */
    int32_t overlap;          /* boundary-first cycles (P:372-375
                                 non-blocking exchange): the kernels that produce the
                                 planes the halo exchange sends run first on those
                                 planes, the exchange then runs on a side stream while
                                 they finish the interior.  0 = automatic (on with more
                                 than one rank), 1 = on (also for local_slabs > 1),
                                 -1 = off.  Results are identical either way.        */
    int32_t local_slabs;      /* >= 1.  With nranks == 1, split the mesh into this
                                 many z-slabs on the same device exchanging halos
                                 by device copies (emulated ranks, used to prove
                                 decomposition bit-exactness on one GPU).  Must be
                                 1 when nranks > 1.                                */
    int32_t nmat;             /* multi-material cells (DESIGN.md
                                 §10d readings MM0-MM7; P:133, P:183, P:403 name them,
                                 SPEC S:255-263 the closure).  0: single material
                                 (gamma above).  1..SALE_MAX_MAT: every cell carries
                                 per material a volume fraction, mass and specific
                                 energy (fields SALE_F_MAT_*), material m has the
                                 ideal-gas gamma mat_gamma[m] (> 1); the Sedov init puts
                                 the whole cell in material 0; the cell pressure is the
                                 volume-fraction-weighted sum of the material
                                 pressures; the remap moves each material's mass,
                                 volume and energy from the donor cell.  MASS and E
                                 are then read-only (MASS = sum of material masses,
                                 E = mass-weighted mixture energy).  The cycle
                                 kernels carry the material count as a compile-time
                                 parameter; nmat = 1 gives the single-material
                                 results bit for bit.                              */
    double mat_gamma[SALE_MAX_MAT];
    double hg;                /* hourglass viscosity coefficient >= 0 (reading HG,
                                 DESIGN.md §3; 0 = none, the Sedov configs use 0.5):
                                 per cell nu = min((hg (m c)) / (Lsum / 3), (m / 64) / dt)
                                 with Lsum the sum of its three face-centroid
                                 separations; the corner force -nu sum_m Gamma_m g_m
                                 damps the four hourglass modes g_m of u^n, its work
                                 heats the cell (total energy is conserved).       */
    int32_t halo;             /* SALE_HALO_COPY (0) or SALE_HALO_PEER (1): how the ghost
                                 planes of the new state reach the neighbours every
                                 cycle (the paper's per-cycle
                                 exchange).  PEER with nranks > 1
                                 needs every rank's workspace in one cudaMalloc'd
                                 allocation (CUDA IPC) and peer access between the
                                 devices (NVLink / NVSwitch); the exchange at the start
                                 of each sale_step call (and of the first cycle) stays
                                 a copy exchange.  Results are identical either way.
                                 Boundary-first cycles (overlap) apply to COPY only.  */
} sale_params;

typedef struct sale_ctx sale_ctx;

/* Device bytes this rank needs (state ping-pong buffers + ghosts + scratch).
 * Returns 0 if the parameters are invalid (same checks as sale_create). */
uint64_t sale_workspace_bytes(const sale_params* p);

/* Writes a fresh 128-byte NCCL unique id into id_out (call on rank 0, then
 * broadcast it).  One id initialises one communicator: every context (every
 * sale_create of a job) needs its own.  SALE_ENCCL on failure. */
int32_t sale_nccl_unique_id(void* id_out_128);

/* Validate; carve the workspace; NCCL init when nranks > 1; Sedov initial state
 * (c.6: x = x^T, u = 0, m = rho0 V, e = e_bg, e_000 = E0/m_000); sync.
 * On error *out is NULL and nothing leaks. */
int32_t sale_create(const sale_params* p, sale_ctx** out);

/* Enqueue up to ncycles cycles on the stream, then synchronise once.  Each
 * step call starts with a halo exchange and a cell-state + dt-candidate pass, so
 * state set with sale_set_field / sale_set_clock is always honoured.  Stops early (status
 * OK, *cycles_done < ncycles) when t >= t_end.  On a numerical error returns its
 * code, sets *cycles_done to the number of good cycles, poisons the context. */
int32_t sale_step(sale_ctx* c, int32_t ncycles, int32_t* cycles_done);

/* Enqueue only (no synchronisation, no status read-back): for timing loops.
 * The next sale_step / sale_sync reports errors that happened meanwhile. */
int32_t sale_step_async(sale_ctx* c, int32_t ncycles);
/* Synchronise the stream, read back status; *cycles_done = good cycles since the
 * last sale_sync / sale_step. */
int32_t sale_sync(sale_ctx* c, int32_t* cycles_done);

/* Copy this rank's owned slab of a field.  Node fields cover global z node
 * planes [k0, k1] (the interface plane is replicated on both owners), cell
 * fields cover cell planes [k0, k1); with local_slabs > 1 the whole mesh is
 * assembled (replicated planes are checked bit-equal, else SALE_EREPLICA).
 * count must equal the slab size: (nx+1)(ny+1)(k1-k0+1) or nx*ny*(k1-k0),
 * else SALE_EINVAL.  Material fields are cell fields (SALE_EINVAL for a material
 * >= nmat); with nmat >= 1, E reads the mixture's (sum_k m_k e_k) / m and P, CS, Q
 * the mixed closure.  dst_on_device != 0: dst is device memory on this device.
 * Layout of dst: x fastest, then y, then z. */
int32_t sale_get_field(sale_ctx* c, int32_t field, double* dst, uint64_t count,
                       int32_t dst_on_device);

/* Overwrite a state field (X, Y, Z in Lagrange mode only; UX, UY, UZ; MASS and E
 * with nmat = 0; SALE_F_MAT_* with nmat >= 1, a MAT_M write re-summing MASS) on this
 * rank's owned slab (same shape and layout as get_field).  Replicated interface
 * planes must be identical on both owners. */
int32_t sale_set_field(sale_ctx* c, int32_t field, const double* src, uint64_t count,
                       int32_t src_on_device);

/* clock: t, dt of the last completed cycle (< 0: none yet), completed cycles,
 * finished = (t_end > 0 && t >= t_end) */
int32_t sale_get_clock(sale_ctx* c, double* t, double* dt_last, int64_t* cycle,
                       int32_t* finished);
int32_t sale_set_clock(sale_ctx* c, double t, double dt_last, int64_t cycle);

/* owned global cell planes [k0, k1) of this rank (remainder planes go to the
 * lowest ranks); with local_slabs > 1 the union [0, nz). */
int32_t sale_get_layout(sale_ctx* c, int32_t* k0, int32_t* k1);

/* kernels launched so far by this context (all of them are libsale's own) */
int64_t sale_kernel_launches(const sale_ctx* c);

/* Kernel-class timing: while enabled, every launch group of a class is
 * bracketed by cudaEventRecord on the context's stream; the elapsed times are
 * accumulated at the next synchronisation (sale_step / sale_sync).  Enabling
 * resets the accumulators.  Classes: */
#define SALE_K_BEGIN 0     /* dt finalisation + clock commit (one thread)          */
#define SALE_K_PROLOGUE 1  /* per-call halo exchange + cell-state / dt-candidate pass */
#define SALE_K_LAGRANGE 2  /* Lagrangian phase S1-S7 (+ the cell state and dt
                              candidate: Lagrange of the new state, Euler of the
                              cycle-start state)                                    */
#define SALE_K_REMAP 3     /* Eulerian remap R1-R5                                 */
#define SALE_K_HALO 4      /* per-cycle halo exchange + dt/error allreduce         */
#define SALE_K_NCLASS 5
int32_t sale_profile_enable(sale_ctx* c, int32_t on);
/* total device milliseconds and number of timed launch groups of a class */
int32_t sale_profile_read(sale_ctx* c, int32_t kclass, double* total_ms, int64_t* count);

/* ---- halo plan (host-only, no GPU): what X1 exchanges between ranks --------
 * Local arrays of a rank hold global planes [k0-g, k1+g) (cells) / [k0-g, k1+g]
 * (nodes), plane-major (x fastest), g = 1 (LAGRANGE) or 3 (EULER); see
 * sale_local_layout.  One message = one contiguous run of whole planes of one
 * state field.  sale_step executes exactly this plan with ncclSend/ncclRecv in
 * one group per cycle (full = 0), and once with full = 1 at the start of every
 * sale_step call (adds MASS in LAGRANGE mode, where m is otherwise constant). */
typedef struct sale_halo_msg {
    int32_t peer;    /* rank sent to / received from                          */
    int32_t send;    /* 1 = send, 0 = receive                                 */
    int32_t field;   /* SALE_F_X..SALE_F_UZ, SALE_F_MASS or SALE_F_E           */
    int32_t first_plane; /* global plane index of the first plane moved       */
    int64_t offset;  /* element offset into this rank's local array of field  */
    int64_t count;   /* elements (whole planes)                               */
} sale_halo_msg;
/* Writes up to cap messages; returns their number, or -1 if p is invalid. */
int32_t sale_halo_plan(const sale_params* p, int32_t full, sale_halo_msg* out, int32_t cap);
/* Local slab geometry of rank p->rank: owned cell planes [k0,k1), ghost depth,
 * allocated local node / cell planes.  SALE_EINVAL if p is invalid. */
int32_t sale_local_layout(const sale_params* p, int32_t* k0, int32_t* k1, int32_t* ghost,
                          int32_t* node_planes, int32_t* cell_planes);

/* ---- Steinberg shear modulus and yield stress --------
 * The paper's own extension example (Fig. 6b): for every owned cell of
 * the current state,
 *   eta   = rho0 / rho                      rho = m / V   (as get_field RHO)
 *   shear = (G0 + (GP * p) * eta^(1/3)) + GT * (T - T0)     p as get_field P
 *   yield = min(Y0 * (1 + beta * eps_p)^n, Ymax) * (shear / G0)
 * with the readings of DESIGN.md §10c: T = e / cv (ideal gas), uniform reference
 * density rho0 and initial temperature T0.  eta^(1/3) is cbrt(eta) here and the
 * paper's eta**(1d0/3) = pow(eta, 1/3) in the oracle; neither cbrt nor pow is
 * correctly rounded, so results agree with the oracle to a few ulp (tests: 1e-14
 * relative), not bitwise. */
typedef struct sale_steinberg_params {
    double G0, GP, GT;        /* shear modulus at reference; pressure / temperature slopes */
    double Y0, Ymax, beta, n; /* yield: Y0 (1 + beta eps_p)^n capped at Ymax             */
    double cv, rho0, T0;      /* T = e / cv; eta = rho0 / rho; T - T0                     */
} sale_steinberg_params;
/* eps_p: plastic strain per owned cell, or NULL for zero; shear, yield: outputs.
 * All three are DEVICE pointers with the layout and count of get_field's cell
 * fields (count = owned cells; emulated slabs concatenated in plane order).
 * With a material axis (nmat >= 1) sp points to nmat parameter sets and shear /
 * yield hold nmat * count values, material m's at offset m * count (Fig. 6b's
 * shear(m,i,j,k): every material's constants applied to the cell's rho, p and
 * mixture energy, as get_field RHO / P / E).  Asynchronous on the context's stream
 * (synchronises first with pending cycles); the call launches one kernel per slab.
 * SALE_EINVAL on NULL / count mismatch, SALE_EPOISONED on a poisoned context. */
int32_t sale_steinberg(sale_ctx* c, const sale_steinberg_params* sp, const double* eps_p, double* shear,
                       double* yield, uint64_t count);

/* human-readable detail of the last error: code, cycle, cell, CUDA/NCCL text */
const char* sale_last_error(const sale_ctx* c);

/* NULL-safe.  Destroys the NCCL communicator; never frees workspace or stream. */
void sale_destroy(sale_ctx* c);

#ifdef __cplusplus
}
#endif
#endif /* SALE_H */
