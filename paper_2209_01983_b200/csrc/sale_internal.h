// sale_internal.h -- structures shared by the libsale host code and kernels.
// Not part of the ABI (include/sale.h is).
#pragma once
#include <cstdint>

namespace sale {

constexpr unsigned long long KEY_NONE = 0xFFFFFFFFFFFFFFFFull;
constexpr int MAX_MAT = 4;

// Physics and mesh parameters (validated copy of sale_params), by value into kernels.
struct Phys {
    double lx, ly, lz;
    double gamma, c1, c2, cfl, growth, t_end;
    double rho0, e_bg, e_dep;
    double hg;                // hourglass viscosity coefficient (reading HG)
    int nx, ny, nz;           // global cells
    unsigned reflect;         // bit f: face f of {-x,+x,-y,+y,-z,+z} reflects
    int rezone;               // 0 Lagrange, 1 Euler
    int diag_areas;           // Euler: every target face area vector is axis-aligned (off-diagonal
                              // components exactly zero, diagonal non-zero; checked at create), so
                              // a corner vector (c.2) is exactly (+-Ax.x, +-Ay.y, +-Az.z)
    int diag_jumps;           // Euler: every axis-jump separation d of the target mesh lies on its
                              // axis (off-axis components exactly zero; checked at create)
};

// Device-resident clock and status (one per context; all local slabs share it).
struct DevState {
    double t;                 // time of the current state
    double dt_prev;           // dt of the last committed cycle (< 0: none)
    double dt;                // dt of the cycle in flight
    long long cycle;          // committed cycles
    unsigned long long cand_key;  // min over cells of key(dt_K) for the next cycle
    unsigned long long err_key;   // min over failing cells of (order << 48 | cell)
    int status;               // sticky SALE_* code, 0 = OK
    int active;               // 1 while a cycle is in flight
    int finished;             // t_end reached
    int good;                 // committed cycles since the last host read
    long long err_cycle;      // cycle in which status became non-zero
    long long err_cell;       // global linear cell index (-1 if none)
    // peer-store halo between ranks (sale_params.halo = SALE_HALO_PEER): halo_in[side] counts
    // the cycles whose planes the lower (0) / upper (1) neighbour has stored into this
    // rank's ghost planes (the neighbour adds 1 at system scope after its producers);
    // halo_seen[side] the ones this rank has consumed
    unsigned long long halo_in[2];
    unsigned long long halo_seen[2];
};

// Peer-store halo (sale_params.halo = SALE_HALO_PEER, the paper's
// halo exchange P:372-375 fused into the kernels that produce the planes): the arrays
// of the lower (side 0) and upper (side 1) neighbour slab -- another rank's workspace
// mapped over NVLink (CUDA IPC), or the neighbouring emulated slab on this device --
// into whose ghost planes the producer kernels store the planes the copy exchange
// would send.  Null pointers: no neighbour on that side (or the field does not exist).
// Device-resident (one per slab, in the workspace); Slab::hp points to it.
struct HaloPeer {
    double* x[2][2][3];       // [side][buffer][axis]: node positions (Lagrange)
    double* u[2][2][3];       // node velocities
    double* m[2][2];          // cell mass (Euler)
    double* e[2][2];          // specific internal energy
    double* mf[2][2];         // material fractions / masses (Euler) and energies, material k
    double* mm[2][2];         //   at + k * mstride[side] (the neighbour's material stride)
    double* me[2][2];
    long long mstride[2];
    int kb[2];                // the neighbour's local plane base (its global plane k is
                              // local plane k - kb)
    unsigned long long* flag[2];  // ranks: the neighbour's DevState::halo_in entry for this
                                  // rank (lower neighbour: its [1], upper: its [0]); else null
};

// One z-slab of the mesh with its ghost planes, by value into kernels.
// Global cell planes [k0,k1) are owned; local plane 0 is global plane kb = k0-g.
struct Slab {
    int k0, k1, g, kb;
    int nzc, nzn;             // allocated local cell / node planes
    long long pn, pc;         // node / cell plane sizes (nx+1)(ny+1), nx*ny
    double* x[2][3];          // Lagrange node positions (ping-pong); unused in Euler
    double* u[2][3];          // node velocities (ping-pong)
    double* m[2];             // cell mass (Euler ping-pong; Lagrange uses m[0])
    double* e[2];             // specific internal energy (ping-pong)
    double* sig;              // cell state of the cycle start: sigma = 0.25 (pf + q) (c.3 step 3) and
    double* hnu;              // the uncapped hourglass coefficient nu_u (reading HG), written by the
                              // state passes (Lagrange: the energy kernel of the previous cycle for
                              // the new state, the prologue and the ghost pass; Euler: ke_state)
    double* x1[3];            // unused (null): x' is formed from u' where it is staged (Euler)
    double* u1[3];            // Euler scratch: u'
    double* e1;               // Euler scratch: e'
    double* V1;               // Euler scratch: V'
    double* dm;               // Euler scratch: Delta m (multi-material cycle: k_mat_flux -> kn_update;
    double* dP[3];            //   Delta P           the single-material kr_tail keeps them on chip)
    double* dV[3];            // Euler scratch: swept volume of the -x/-y/-z face of each cell (kr_sweep)
    double* rD;               // Euler scratch: donor density m/V' of each cell (kr_sweep)
    double* UD[3];            // Euler scratch: donor velocity (8-node mean of u') of each cell (kr_sweep)
    double* der;              // derive / staging scratch (node-plane sized)
    double* VT;               // Euler: target cell volume V^T (constant; set at create)
    double* sT[3];            // Euler: s of the target x/y/z face anchored at each cell (-a faces)
    // Euler: geometry of the fixed target mesh x^T at t^n (constant; computed once at
    // create by k_target_tables with the same c.2 primitives the kernels would apply
    // to x^T every cycle, so the values are the same bits).  x^T is a tensor
    // product of the 1-D tables below, so each face family's area vector depends on
    // two indices only, and a cell's centroid separation d / |d| along axis a (c.3
    // step 2) on one:
    double* TAx[3];           // A of x-faces, index (k-kb)*ny + j  (independent of i)
    double* TAy[3];           // A of y-faces, index (k-kb)*nx + i  (independent of j)
    double* TAz[3];           // A of z-faces, index j*nx + i       (independent of k)
    double* sF[3];            // Euler scratch: s' (c.2 s of the moved face) of the x-, y-, z-face
                              // anchored at node (i,j,k), node-indexed; written by kc_energy
                              // (which needs them for V'), read by kr_sweep's swept volumes
    double* TDx;              // cells i: cfl * sqrt(edge length^2 along x) of the target mesh (c.5);
    double* TDy;              //   the dt numerator cfl*sqrt(min(lx,ly,lz)) = min of these (sqrt and
    double* TDz;              //   the positive scaling are monotone, so the same bits)
    double* TJx;              // cells i: d.x d.y d.z L at TJx[4*i + c] (x-axis jump)
    double* TJy;              // cells j (y-axis)
    double* TJz;              // cells at local plane k-kb (z-axis)
    double* Xt;               // target node coordinates X_i, i in [0,nx]
    double* Yt;               // Y_j, j in [0,ny]
    double* Zt;               // Z_k for local node planes (index = k - kb)
    // multi-material cells (Phys::nmat >= 1): material k's cell array
    // starts at k * pc * nzc (a material-major Data4d).  Lagrange mode: f and m_k are
    // constant (index [0]), e_k ping-pongs; Euler mode: all three ping-pong.
    double* mf[2];            // volume fraction f_k
    double* mm[2];            // material mass m_k (m above holds the sum over k)
    double* me[2];            // material specific energy e_k
    double* sgm;              // each material's stress 0.25 (pf_k + q) at the cycle start (MM4; state passes)
    double* e1m;              // Euler scratch: e'_k
    double* rDm;              // Euler scratch: donor material density m_k / V' of each cell (kr_sweep<NM>)
    double mg[MAX_MAT];       // gamma of each material (here rather than in Phys: growing Phys
    int nmat;                 //   perturbed the single-material kernels' code generation)
                              // nmat: 0 single material; 1..MAX_MAT the material axis (§10d)
    DevState* st;
    const HaloPeer* hp;       // peer-store halo: the neighbours' arrays (null: copy exchange)
};

// Steinberg model parameters (copy of sale_steinberg_params, by value into the kernel)
struct SteinbergP {
    double G0, GP, GT, Y0, Ymax, beta, n, cv, rho0, T0;
};
// one parameter set per material (n = nmat, or 1 without a material axis)
struct SteinbergSet {
    SteinbergP m[MAX_MAT];
    int n;
};

// status codes mirrored from include/sale.h (kept in sync by a static_assert in host code)
enum { S_OK = 0, S_EINVAL = 1, S_ENOMEM = 2, S_ECUDA = 3, S_ENCCL = 4, S_ETANGLED = 5,
       S_EDTCOLLAPSE = 6, S_ENEGMASS = 7, S_EPOISONED = 8, S_EREPLICA = 9 };

// kernel-side error ordering inside a cycle: tangling (Lagrangian phase) first
constexpr unsigned long long ERR_ORDER_TANGLED = 1, ERR_ORDER_NEGMASS = 2;

// ---- launchers (kernels_*.cu) ----------------------------------------------
// every launcher returns the number of kernels it launched
typedef struct CUstream_st* Stream;

// every launcher calls note_launch() right after each kernel launch: it keeps the
// first launch error of this host thread (a later runtime call may clear the
// runtime's own last-error slot); the host's launch check takes it
void note_launch();
int take_launch_error();  // a cudaError_t, 0 if none; resets

int launch_init_tables(const Slab& s, const Phys& p, Stream st);
int launch_sedov_init(const Slab& s, const Phys& p, Stream st);
int launch_target_tables(const Slab& s, const Phys& p, Stream st);
int launch_prep(DevState* d, Stream st);
int launch_begin(DevState* d, const Phys& p, Stream st);
int launch_commit(DevState* d, const Phys& p, Stream st);
int launch_reset_good(DevState* d, Stream st);
int launch_derive(const Slab& s, const Phys& p, int cur, int field, Stream st);
// Steinberg shear / yield of the owned cells (include/sale.h); outputs at sh / y (device)
int launch_steinberg(const Slab& s, const Phys& p, int cur, const SteinbergSet& set, const double* eps, double* sh,
                     double* y, long long mstride, Stream st);

// ---- the cycle (kernels_lag.cu, kernels_remap.cu, kernels_mat.cu) ------------
// the cell state (sigma, nu_u, material stresses) and the c.5 dt candidate of the
// cycle-start state in buffer `cur`, before the cycle's k_begin (gate = 0 for the
// first cycle of a sale_step call, when DevState.active is still 0): every cell the
// force gather reads (Lagrange: [k0-1, k1]; Euler: the remap's ghost region too)
int launch_state(const Slab& s, const Phys& p, int cur, int gate, Stream st);
// S5-S6: corner forces (pressure, viscosity, hourglass) gathered in the fixed order,
// kinematics + BC.  Lagrange: x', u' into buffer cur^1; Euler: u' into Slab::u1.
int launch_force(const Slab& s, const Phys& p, int cur, Stream st);
// S7: V', tangle check, compatible energy with the hourglass work.  Lagrange: e' into
// buffer cur^1; Euler: e' (e'_k), V', and the moved-face s' the sweep reads.
// [ka, kb): a sub-range of the cell planes (boundary-first cycles); -1: all of them
int launch_energy(const Slab& s, const Phys& p, int cur, Stream st, int ka = -1, int kb = -1);
// R1-R4 (kernels_remap.cu; materials: kernels_mat.cu); nodes = 0: the caller launches
// the node part by node-plane ranges, boundary first (single material: R1 only, then
// launch_rtail = R2-R4; materials: R1-R3, then launch_kn_update = R4)
int launch_remap(const Slab& s, const Phys& p, int cur, Stream st, int nodes = 1);
int launch_remap_mat(const Slab& s, const Phys& p, int cur, Stream st, int nodes = 1);
int launch_sweep(const Slab& s, const Phys& p, int cur, Stream st);
// single material: R2-R4 (fluxes, cell update, node momentum) over the owned node
// planes, or the sub-range [ka, kb] (cells stored: planes [ka, kb] n [k0, k1))
int launch_rtail(const Slab& s, const Phys& p, int cur, Stream st, int ka = -1, int kb = -1);
// R4 over the owned node planes, or the sub-range [ka, kb]
int launch_kn_update(const Slab& s, const Phys& p, int cur, Stream st, int ka = -1, int kb = -1);
int launch_mat_init(const Slab& s, const Phys& p, Stream st);
// peer-store halo between ranks: signal the neighbours that this cycle's planes are
// stored (after the cycle's producer kernels); wait for theirs before the next cycle
// reads the ghost planes (first = 1: the first cycle of a sale_step call, whose ghost
// planes come from the copy exchange: absorb, no wait)
int launch_halo_signal(DevState* d, const HaloPeer* hp_dev, Stream st);
int launch_halo_wait(DevState* d, int first, int sides, Stream st);  // sides: bit 0 lower, 1 upper
int launch_mat_total(const Slab& s, const Phys& p, int cur, Stream st);

}  // namespace sale
