/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, single-threaded CPU oracle of the SALE hot path
 * (arXiv 2209.01983, "ScalSALE").  It exists to check the
 * CUDA path; nothing in the product package may include, link or call it.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load liboracle.so.
 *
 * It shares no code with paper_2209_01983_b200/ (no headers, helpers, tables).
 * Its ABI mirrors the product ABI (include/sale.h) with the prefix `oracle_`,
 * host pointers only and a single rank.
 *
 * The paper never writes the discrete scheme (only the Steinberg
 * loop P:442-459 and the efficiency formula P:509-516 are formulas).  Every
 * operator here follows SURVEY §8(c) c.1-c.6 step by step, in its order and
 * notation, with the readings Q1-Q23 listed in DESIGN.md §3.
 *
 * Build: gcc -O2 -ffp-contract=off -std=c11 (never -ffast-math): every + - * /
 * sqrt is one correctly rounded IEEE binary64 operation in the written order.
 */
#ifndef SALE_ORACLE_H
#define SALE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORACLE_ABI_VERSION 3
#define ORACLE_MAX_MAT 4

/* Same fields and meaning as sale_params (include/sale.h), minus the device /
 * communication members.  SURVEY §8(b). */
typedef struct oracle_params {
    int32_t abi_version;          /* must be ORACLE_ABI_VERSION                */
    int32_t nx, ny, nz;           /* cells per axis (global)                   */
    double lx, ly, lz;            /* domain extents; node X_i = (lx*i)/nx      */
    double gamma;                 /* ideal-gas gamma (> 1)                     */
    double q_lin, q_quad;         /* viscosity c1 (linear), c2 (quadratic)     */
    double cfl;                   /* CFL number                                */
    double dt_growth;             /* dt_u <= dt_growth * dt_prev               */
    double t_end;                 /* <= 0: no end time                         */
    int32_t rezone;               /* 0 = LAGRANGE, 1 = EULER                   */
    uint32_t reflect_mask;        /* bit f: face f in {-x,+x,-y,+y,-z,+z} reflects */
    double rho0;                  /* Sedov ambient density                     */
    double e_background;          /* Sedov background specific energy          */
    double e_deposit;             /* Sedov energy E0 put in cell (0,0,0)       */
    /* multi-material cells (readings MM1-MM7 in DESIGN.md
     * §10d).  nmat = 0: the single-material scheme above.  nmat in [1,4]: every
     * cell carries per material m a volume fraction f_m, a mass m_m and a specific
     * energy e_m, each material its own ideal-gas gamma mat_gamma[m] (> 1); the
     * initial state puts the whole Sedov cell in material 0.  With nmat = 1 the
     * material path reproduces the single-material scheme bit for bit. */
    int32_t nmat;
    int32_t pad0;
    double mat_gamma[ORACLE_MAX_MAT];
    /* hourglass viscosity coefficient (reading HG): the cell's
     * viscous hourglass coefficient is nu = min((hg*(m*c))/(Lsum/3), (m/64)/dt)
     * (Lsum: the sum of its three face-centroid separations); hg = 0 switches it
     * off.  ABI version 3. */
    double hg;
} oracle_params;

typedef struct oracle_ctx oracle_ctx;

/* status codes (same numbering as the product) */
enum {
    ORACLE_OK = 0, ORACLE_EINVAL = 1, ORACLE_ENOMEM = 2,
    ORACLE_ETANGLED = 5, ORACLE_EDTCOLLAPSE = 6, ORACLE_ENEGMASS = 7,
    ORACLE_EPOISONED = 8
};

/* field ids (same numbering as the product) */
enum {
    ORACLE_F_X = 0, ORACLE_F_Y, ORACLE_F_Z, ORACLE_F_UX, ORACLE_F_UY, ORACLE_F_UZ,
    ORACLE_F_NODE_MASS,                                   /* node fields 0..6  */
    ORACLE_F_MASS = 7, ORACLE_F_E, ORACLE_F_RHO, ORACLE_F_VOL, ORACLE_F_P,
    ORACLE_F_Q, ORACLE_F_CS,                              /* cell fields 7..13 */
    /* material fields (nmat >= 1), material m in [0, nmat): */
    ORACLE_F_MAT_F = 16,   /* + m: volume fraction f_m                           */
    ORACLE_F_MAT_M = 20,   /* + m: material mass m_m (MASS = sum over m)          */
    ORACLE_F_MAT_E = 24    /* + m: material specific internal energy e_m          */
};

int32_t oracle_create(const oracle_params* p, oracle_ctx** out);
int32_t oracle_step(oracle_ctx* c, int32_t ncycles, int32_t* cycles_done);
int32_t oracle_get_field(oracle_ctx* c, int32_t field, double* dst, uint64_t count);
int32_t oracle_set_field(oracle_ctx* c, int32_t field, const double* src, uint64_t count);
int32_t oracle_get_clock(oracle_ctx* c, double* t, double* dt_last, int64_t* cycle,
                         int32_t* finished);
int32_t oracle_set_clock(oracle_ctx* c, double t, double dt_last, int64_t cycle);
/* error detail: "<code name> cycle=<n> cell=<i,j,k>" of the last failure */
const char* oracle_last_error(const oracle_ctx* c);
/* linear cell index of the last ETANGLED/ENEGMASS cell, -1 if none */
int64_t oracle_last_error_cell(const oracle_ctx* c);
/* dt the next cycle would use (c.5), without advancing; <0 if finished. */
int32_t oracle_next_dt(oracle_ctx* c, double* dt);
void oracle_destroy(oracle_ctx* c);

/* ---- unit entry points (the same primitives the cycle uses), for pins ---- */
/* c.2: face from 4 points (P[4][3]) -> A[3], Xbar[3], s */
void oracle_face(const double* P, double* A, double* Xbar, double* s);
/* c.2: volume of the hex whose local node (a,b,c) is N[((c*2+b)*2+a)*3 + comp] */
double oracle_hex_volume(const double* N);
/* c.3 step 1: p, pf, c from (gamma, rho, e) */
void oracle_eos(double gamma, double rho, double e, double* p, double* pf, double* cs);
/* MM1: mixed-cell closure of nmat materials (gamma[m], f[m], m_m[m], e[m]) in a
 * cell of volume V and density rho: p = sum f_m p_m, P = sum f_m max(p_m, 0),
 * cs = sqrt(sum f_m gamma_m max(p_m,0) / rho) */
void oracle_mix_eos(int32_t nmat, const double* gamma, const double* f, const double* mm, const double* e,
                    double V, double rho, double* p, double* P, double* cs);
/* c.3 step 2 last line: q from rho, c, du */
double oracle_q_of_du(double rho, double cs, double du, double c1, double c2);
/* c.5 with reading DT-Q: per-cell candidate from l2 = min edge^2, v2 = max node
 * speed^2, c and the compressive jump du (c.3 step 2; du >= 0: no viscous term):
 * (cfl*sqrt(l2)) / (((c + sqrt(v2)) + cq) + 1e-30), cq = 2*((c1*c) + (c2*(-du))) */
double oracle_dt_cell(double cfl, double l2, double v2, double cs, double du, double c1, double c2);
/* reading HG: hourglass mode amplitudes g[m*3+comp] = sum_h Gamma_m(h) U[h*3+comp]
 * (m = xi*eta, eta*zeta, zeta*xi, xi*eta*zeta; xi = 2a-1 on hex-local (a,b,c)) */
void oracle_hg_modes(const double* U, double* g);
/* reading HG: corner force f[3] = -(nu * sum_m Gamma_m(h) g_m) of hex corner h */
void oracle_hg_corner(const double* g, double nu, int32_t h, double* f);
/* reading HG: nu = min((hg*(m*c))/(Lsum/3), (m/64)/dt), Lsum = ((Lx+Ly)+Lz) */
double oracle_hg_nu(double hg, double m, double cs, double Lsum, double dt);
/* c.4 step 1: swept volume between target face PT[4][3] and moved face PL[4][3] */
double oracle_swept_volume(const double* PT, const double* PL);
/* c.3 step 7 for one cell: N0 = nodes at t^n in hex order, U0/U1 = node
 * velocities u / u' in hex order, nu = the cell's hourglass coefficient (HG; 0:
 * none); returns e' = e - ((((sigma*W) + W_hg)*dt)/m). */
double oracle_cell_energy(const double* N0, const double* U0, const double* U1,
                          double sigma, double nu, double m, double e, double dt);

/* ---- Steinberg shear modulus and yield stress --------
 * The paper's extension example, Fig. 6b, per cell:
 *   eta = rho0 / rho
 *   shear = (G0 + (GP * p) * eta^(1/3)) + GT * (T - T0)
 *   yield = min(Y0 * (1 + beta * eps_p)^n, Ymax) * (shear / G0)
 * with p the cell pressure of the EoS and rho = m / V of the current state; the
 * readings: temperature T = e / cv (ideal gas), a uniform
 * reference density rho0 and initial temperature T0, eta^(1/3) = pow(eta, 1/3) as
 * the paper's eta**(1d0/3). */
typedef struct oracle_steinberg_params {
    double G0, GP, GT;        /* shear modulus at reference; pressure, temperature slopes */
    double Y0, Ymax, beta, n; /* yield: Y0 (1 + beta eps_p)^n capped at Ymax             */
    double cv, rho0, T0;      /* T = e / cv; eta = rho0 / rho; T - T0                     */
} oracle_steinberg_params;
/* one cell from its (p, rho, e, eps_p) */
void oracle_steinberg_point(const oracle_steinberg_params* sp, double p, double rho, double e, double eps_p,
                            double* shear, double* yield);
/* every cell of the current state; eps_p: cell array or NULL (all zero); shear,
 * yield: cell arrays (count = nx*ny*nz).  With nmat >= 1 materials: sp holds nmat
 * parameter sets and shear / yield nmat * count values, material m's at m * count
 * (Fig. 6b's loop over materials; rho, p and the mixture energy of the cell as
 * oracle_get_field RHO / P / E). */
int32_t oracle_steinberg(oracle_ctx* c, const oracle_steinberg_params* sp, const double* eps_p, double* shear,
                         double* yield, uint64_t count);

#ifdef __cplusplus
}
#endif
#endif
