/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain single-threaded fp64 CPU oracle of the SALE per-cycle update
 * (arXiv 2209.01983; the scheme as written down in SURVEY.md §8(c), because
 * the paper itself names the steps -- P:133 "SALE", "ideal gas EoS",
 * P:181 "Lagrangian rezoning / Eulerian rezoning / Advection"
 * "Calculate_density" -- but prints no discrete equation).  Each function
 * below cites the §8(c) item it follows.  Loops are whole-mesh, one step at a
 * time, in the order c.3 / c.4 lists them; no blocking or fusion.
 *
 * Parity status of each part: see DESIGN.md §4 (pins).  "Parity unpinned" there:
 * the absolute discretisation error beyond the Sedov radius / symmetry checks and
 * the exact-solution comparisons of the Sod / Noh problems; the value hg = 0.5 of
 * the hourglass coefficient (reading HG: any value in [0.2, 1] runs C1); the
 * Lagrangian Sedov peak density (about 12 against the strong-shock bound 6).
 * The readings of round 2 (HG, DT-Q, DT-C) are pinned by tests/test_oracle_readings_r2.py.
 *
 * Compile: gcc -O2 -ffp-contract=off (no FMA contraction, no fast-math).
 * The whole-mesh loops carry OpenMP work-sharing pragmas that only a -fopenmp
 * build honours (scripts/oracle_digests.py, for the full-size golden digests):
 * every iteration writes its own cell or node, the dt min is order-free and the
 * failure reports take the lowest failing cell index, so the results are the
 * single-threaded ones bit for bit.  The default build (tests, bench) is serial.
 */
#include "oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* context                                                                    */
/* ------------------------------------------------------------------------- */
struct oracle_ctx {
    oracle_params p;
    int64_t nx, ny, nz;          /* cells */
    int64_t NX, NY, NZ;          /* nodes = cells + 1 */
    int64_t ncell, nnode;
    /* state (c.1): node position and velocity, cell mass and specific energy */
    double *x[3], *u[3];
    double *m, *e;
    /* target (initial) mesh x^T, node-wise (c.1, c.4 step 5) */
    double *xT[3];
    /* cycle scratch */
    double *sig;                 /* sigma_K (c.3 step 3)              */
    double *hnu, *hgm;           /* HG: nu_K and the mode amplitudes g_K (4 x 3 per cell) */
    double *x1[3], *u1[3];       /* x', u' (c.3 step 6)               */
    double *e1, *V1;             /* e', V' (c.3 step 7)               */
    double *dm, *dE, *dP[3], *m2; /* Delta m, Delta E, Delta P, m'' (c.4 step 3) */
    /* multi-material cells (nmat >= 1, readings MM1-MM7): per
     * material m the volume fraction f_m, mass m_m, specific energy e_m; m above
     * then holds the cell total sum_m m_m and e is unused */
    int32_t nmat;
    double *mf[ORACLE_MAX_MAT], *mmat[ORACLE_MAX_MAT], *me[ORACLE_MAX_MAT];
    double *qv, *pfm[ORACLE_MAX_MAT];   /* MM3/MM4 scratch: q and pf_m of the cycle start */
    double *e1m[ORACLE_MAX_MAT];        /* e'_m (MM4)                                      */
    double *dmm[ORACLE_MAX_MAT], *dEm[ORACLE_MAX_MAT], *vm2[ORACLE_MAX_MAT]; /* MM6         */
    /* clock (c.3 step 8, c.5) */
    double t, dt_prev;
    int64_t cycle;
    int32_t finished, poisoned;
    int64_t err_cell;
    char err[256];
};

#ifdef _OPENMP
#define OMP_FOR _Pragma("omp parallel for schedule(static)")
#define OMP_FOR_MIN_BAD _Pragma("omp parallel for schedule(static) reduction(min:bad)")
#else
#define OMP_FOR
#define OMP_FOR_MIN_BAD
#endif

static inline int64_t nid(const oracle_ctx* c, int64_t i, int64_t j, int64_t k)
{
    return i + c->NX * (j + c->NY * k);
}
static inline int64_t cid(const oracle_ctx* c, int64_t i, int64_t j, int64_t k)
{
    return i + c->nx * (j + c->ny * k);
}

/* ------------------------------------------------------------------------- */
/* c.2 geometry primitives                                                    */
/* ------------------------------------------------------------------------- */
typedef struct { double A[3], Xb[3], s; } face_t;

/* c.2: d1 = P2-P0, d2 = P3-P1; A = 0.5*(d1 x d2); Xbar = 0.25*(((P0+P1)+P2)+P3);
 * s = (Xbx*Ax + Xby*Ay) + Xbz*Az. */
static void face_geom(const double P0[3], const double P1[3], const double P2[3],
                      const double P3[3], face_t* f)
{
    double d1[3], d2[3];
    for (int a = 0; a < 3; ++a) {
        d1[a] = P2[a] - P0[a];
        d2[a] = P3[a] - P1[a];
    }
    f->A[0] = 0.5 * (d1[1] * d2[2] - d1[2] * d2[1]);
    f->A[1] = 0.5 * (d1[2] * d2[0] - d1[0] * d2[2]);
    f->A[2] = 0.5 * (d1[0] * d2[1] - d1[1] * d2[0]);
    for (int a = 0; a < 3; ++a)
        f->Xb[a] = 0.25 * (((P0[a] + P1[a]) + P2[a]) + P3[a]);
    f->s = (f->Xb[0] * f->A[0] + f->Xb[1] * f->A[1]) + f->Xb[2] * f->A[2];
}

/* Hex-local node (a,b,c) has index (c*2+b)*2+a.  Faces in the order
 * X0, X1, Y0, Y1, Z0, Z1, each with its canonical P0..P3 (c.2):
 *   X(a): (a,0,0) (a,1,0) (a,1,1) (a,0,1)
 *   Y(b): (0,b,0) (0,b,1) (1,b,1) (1,b,0)
 *   Z(c): (0,0,c) (1,0,c) (1,1,c) (0,1,c)                                    */
static const int FACE_NODES[6][4] = {
    {0, 2, 6, 4}, {1, 3, 7, 5},   /* X0, X1 */
    {0, 4, 5, 1}, {2, 6, 7, 3},   /* Y0, Y1 */
    {0, 1, 3, 2}, {4, 5, 7, 6},   /* Z0, Z1 */
};

static void hex_faces(const double N[8][3], face_t F[6])
{
    for (int f = 0; f < 6; ++f)
        face_geom(N[FACE_NODES[f][0]], N[FACE_NODES[f][1]], N[FACE_NODES[f][2]],
                  N[FACE_NODES[f][3]], &F[f]);
}

/* c.2: V = (((((s(F+x) - s(F-x)) + s(F+y)) - s(F-y)) + s(F+z)) - s(F-z)) / 3.0 */
static double hex_volume_from_faces(const face_t F[6])
{
    return (((((F[1].s - F[0].s) + F[3].s) - F[2].s) + F[5].s) - F[4].s) / 3.0;
}

/* c.2: corner vector of hex corner (a,b,c): C = ((A_x(a) + A_y(b)) + A_z(c)),
 * A_x(1) = A(F+x), A_x(0) = -A(F-x), likewise y, z. */
static void corner_vector(const face_t F[6], int a, int b, int c, double C[3])
{
    for (int q = 0; q < 3; ++q) {
        double ax = a ? F[1].A[q] : -F[0].A[q];
        double ay = b ? F[3].A[q] : -F[2].A[q];
        double az = c ? F[5].A[q] : -F[4].A[q];
        C[q] = (ax + ay) + az;
    }
}

/* gather the 8 node positions of cell (i,j,k) from arrays X[3] */
static void cell_nodes(const oracle_ctx* c, double* const X[3], int64_t i, int64_t j,
                       int64_t k, double N[8][3])
{
    for (int cc = 0; cc < 2; ++cc)
        for (int b = 0; b < 2; ++b)
            for (int a = 0; a < 2; ++a) {
                int64_t n = nid(c, i + a, j + b, k + cc);
                int h = (cc * 2 + b) * 2 + a;
                for (int q = 0; q < 3; ++q) N[h][q] = X[q][n];
            }
}

/* ------------------------------------------------------------------------- */
/* c.3 step 1: EoS                                                            */
/* ------------------------------------------------------------------------- */
static void eos(double gamma, double rho, double e, double* p, double* pf, double* cs)
{
    *p = ((gamma - 1.0) * rho) * e;
    *pf = (*p > 0.0) ? *p : 0.0;
    *cs = sqrt((gamma * *pf) / rho);
}

/* c.3 step 2, last line */
static double q_of_du(double rho, double cs, double du, double c1, double c2)
{
    return (du < 0.0) ? rho * ((c2 * (du * du)) + ((c1 * cs) * (-du))) : 0.0;
}

/* MM1 (multi-material closure; "mixed_cell_pressure"):
 * each present material (f_m > 0) at its own density rho_m = m_m / (f_m V) and the
 * ideal-gas EoS of c.3 step 1, p_m = ((gamma_m - 1) rho_m) e_m, pf_m = max(p_m, 0);
 * the cell pressure is the volume-fraction-weighted sum p = sum_m f_m p_m (floored:
 * P = sum_m f_m pf_m), the sound speed c = sqrt((sum_m f_m (gamma_m pf_m)) / rho)
 * with rho = m / V of the whole cell.  Sums run m = 0, 1, ... left to right from
 * the first present material.  With one material and f_0 = 1 every line reduces to
 * eos() bit for bit (1.0 * a = a, m / (1.0 * V) = m / V).  pf[m] = 0 for absent
 * materials. */
static void mix_eos(int nmat, const double* gam, const double* f, const double* mm, const double* e,
                    double V, double rho, double* p, double* P, double* cs, double* pf)
{
    double ps = 0.0, Ps = 0.0, G = 0.0;
    int first = 1;
    for (int k = 0; k < nmat; ++k) {
        pf[k] = 0.0;
        if (!(f[k] > 0.0)) continue;
        double rk = mm[k] / (f[k] * V);
        double pk = ((gam[k] - 1.0) * rk) * e[k];
        double pfk = (pk > 0.0) ? pk : 0.0;
        pf[k] = pfk;
        double a = f[k] * pk, b = f[k] * pfk, g = f[k] * (gam[k] * pfk);
        if (first) { ps = a; Ps = b; G = g; first = 0; }
        else { ps = ps + a; Ps = Ps + b; G = G + g; }
    }
    *p = ps;
    *P = Ps;
    *cs = sqrt(G / rho);
}

static inline double dmin(double a, double b) { return (b < a) ? b : a; }
static inline double dmax(double a, double b) { return (b > a) ? b : a; }

/* c.3 step 2: per logical axis, face-centroid separation d, face-average
 * velocity jump w, delta_a = (w . d)/|d|; du = min over axes.  Also returns
 * Lsum = ((L_x + L_y) + L_z), the sum of the separations |d| (reading HG). */
static double cell_jumps(const face_t F[6], const double U[8][3], double* Lsum)
{
    double delta[3], Ls[3];
    for (int ax = 0; ax < 3; ++ax) {
        const face_t* fm = &F[2 * ax];
        const face_t* fp = &F[2 * ax + 1];
        const int* nm = FACE_NODES[2 * ax];
        const int* np = FACE_NODES[2 * ax + 1];
        double d[3], w[3];
        for (int q = 0; q < 3; ++q) {
            double Um = 0.25 * (((U[nm[0]][q] + U[nm[1]][q]) + U[nm[2]][q]) + U[nm[3]][q]);
            double Up = 0.25 * (((U[np[0]][q] + U[np[1]][q]) + U[np[2]][q]) + U[np[3]][q]);
            d[q] = fp->Xb[q] - fm->Xb[q];
            w[q] = Up - Um;
        }
        double L = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
        delta[ax] = ((w[0] * d[0] + w[1] * d[1]) + w[2] * d[2]) / L;
        Ls[ax] = L;
    }
    if (Lsum) *Lsum = (Ls[0] + Ls[1]) + Ls[2];
    return dmin(dmin(delta[0], delta[1]), delta[2]);
}

/* c.3 step 2: q of the cell */
static double cell_q(const face_t F[6], const double U[8][3], double rho, double cs,
                     double c1, double c2)
{
    return q_of_du(rho, cs, cell_jumps(F, U, NULL), c1, c2);
}

/* the 12 edges of a hex as pairs of hex-local node indices */
static const int EDGES[12][2] = {
    {0, 1}, {2, 3}, {4, 5}, {6, 7},   /* along a */
    {0, 2}, {1, 3}, {4, 6}, {5, 7},   /* along b */
    {0, 4}, {1, 5}, {2, 6}, {3, 7},   /* along c */
};

/* reading DT-Q: the viscous signal speed of a compressing cell
 * (du < 0, c.3 step 2), cq = 2*((c1*c) + (c2*(-du))), else 0 */
static double visc_speed(double cs, double du, double c1, double c2)
{
    return (du < 0.0) ? 2.0 * ((c1 * cs) + (c2 * (-du))) : 0.0;
}

/* c.5 with reading DT-Q: the signal speed adds cq:
 * dt_K = (cfl*sqrt(l2)) / (((c + sqrt(v2)) + cq) + 1e-30) */
static double dt_cell(double cfl, double l2, double v2, double cs, double du, double c1,
                      double c2)
{
    double cq = visc_speed(cs, du, c1, c2);
    return (cfl * sqrt(l2)) / (((cs + sqrt(v2)) + cq) + 1e-30);
}

/* ------------------------------------------------------------------------- */
/* reading HG: viscous hourglass damping                      */
/* ------------------------------------------------------------------------- */
/* Gamma_m(h) on hex-local node h = (c*2+b)*2+a with xi = 2a-1, eta = 2b-1,
 * zeta = 2c-1: m = 0 xi*eta, 1 eta*zeta, 2 zeta*xi, 3 xi*eta*zeta (all +-1). */
static double hg_gamma(int m, int h)
{
    double xi = (h & 1) ? 1.0 : -1.0, eta = (h & 2) ? 1.0 : -1.0, zeta = (h & 4) ? 1.0 : -1.0;
    switch (m) {
    case 0: return xi * eta;
    case 1: return eta * zeta;
    case 2: return zeta * xi;
    default: return (xi * eta) * zeta;
    }
}

/* g_m = sum over h = 0..7 (left to right) of Gamma_m(h) * U_h, componentwise */
static void hg_modes(const double U[8][3], double g[4][3])
{
    for (int m = 0; m < 4; ++m)
        for (int q = 0; q < 3; ++q) {
            double s = hg_gamma(m, 0) * U[0][q];
            for (int h = 1; h < 8; ++h) s = s + hg_gamma(m, h) * U[h][q];
            g[m][q] = s;
        }
}

/* corner force of hex corner h: f = -(nu * (((G0 g0 + G1 g1) + G2 g2) + G3 g3)) */
static void hg_corner(const double g[4][3], double nu, int h, double f[3])
{
    for (int q = 0; q < 3; ++q) {
        double s = ((hg_gamma(0, h) * g[0][q] + hg_gamma(1, h) * g[1][q]) + hg_gamma(2, h) * g[2][q])
                   + hg_gamma(3, h) * g[3][q];
        f[q] = -(nu * s);
    }
}

/* uncapped coefficient nu_u = (hg*(m*c)) / lbar, lbar = Lsum/3 the mean of the
 * cell's three face-centroid separations (c.3 step 2) */
static double hg_nu(double hg, double m, double cs, double Lsum)
{
    return (hg * (m * cs)) / (Lsum / 3.0);
}

/* nu = min(nu_u, (m/64)/dt): the cap keeps the explicit damping of a mesh-wide
 * checkerboard (64 nu dt / M per cycle) at most 1 */
static double hg_cap(double nu_u, double m, double dt)
{
    return dmin(nu_u, (m / 64.0) / dt);
}

/* c.5 per-cell l2 = min over the 12 edges of the squared edge length */
static double min_edge2(const double N[8][3])
{
    double l2 = 0.0;
    for (int ed = 0; ed < 12; ++ed) {
        const double* A = N[EDGES[ed][0]];
        const double* B = N[EDGES[ed][1]];
        double d0 = B[0] - A[0], d1 = B[1] - A[1], d2 = B[2] - A[2];
        double len2 = (d0 * d0 + d1 * d1) + d2 * d2;
        l2 = (ed == 0) ? len2 : dmin(l2, len2);
    }
    return l2;
}



/* ------------------------------------------------------------------------- */
/* errors                                                                     */
/* ------------------------------------------------------------------------- */
static const char* code_name(int32_t code)
{
    switch (code) {
    case ORACLE_OK: return "OK";
    case ORACLE_EINVAL: return "EINVAL";
    case ORACLE_ENOMEM: return "ENOMEM";
    case ORACLE_ETANGLED: return "ETANGLED";
    case ORACLE_EDTCOLLAPSE: return "EDTCOLLAPSE";
    case ORACLE_ENEGMASS: return "ENEGMASS";
    case ORACLE_EPOISONED: return "EPOISONED";
    default: return "E?";
    }
}

static int32_t fail(oracle_ctx* c, int32_t code, int64_t cell)
{
    c->poisoned = 1;
    c->err_cell = cell;
    if (cell >= 0) {
        int64_t i = cell % c->nx, j = (cell / c->nx) % c->ny, k = cell / (c->nx * c->ny);
        snprintf(c->err, sizeof c->err, "%s cycle=%lld cell=%lld,%lld,%lld", code_name(code),
                 (long long)c->cycle, (long long)i, (long long)j, (long long)k);
    } else {
        snprintf(c->err, sizeof c->err, "%s cycle=%lld", code_name(code), (long long)c->cycle);
    }
    return code;
}

/* ------------------------------------------------------------------------- */
/* c.1 mesh, c.6 Sedov init                                                   */
/* ------------------------------------------------------------------------- */
static int params_valid(const oracle_params* p)
{
    if (!p || p->abi_version != ORACLE_ABI_VERSION) return 0;
    if (p->nx < 1 || p->ny < 1 || p->nz < 1) return 0;
    if (!(p->lx > 0.0) || !(p->ly > 0.0) || !(p->lz > 0.0)) return 0;
    if (!(p->gamma > 1.0) || !(p->cfl > 0.0) || !(p->dt_growth > 0.0)) return 0;
    if (!(p->q_lin >= 0.0) || !(p->q_quad >= 0.0)) return 0;
    if (p->rezone != 0 && p->rezone != 1) return 0;
    if (p->reflect_mask > 0x3Fu) return 0;
    if (!(p->rho0 > 0.0)) return 0;
    if (!(p->hg >= 0.0)) return 0;
    if (p->nmat < 0 || p->nmat > ORACLE_MAX_MAT) return 0;
    for (int k = 0; k < p->nmat; ++k)
        if (!(p->mat_gamma[k] > 1.0)) return 0;
    return 1;
}

static double* alloc_d(int64_t n, int* ok)
{
    double* v = (double*)calloc((size_t)n, sizeof(double));
    if (!v) *ok = 0;
    return v;
}

int32_t oracle_create(const oracle_params* p, oracle_ctx** out)
{
    if (!out) return ORACLE_EINVAL;
    *out = NULL;
    if (!params_valid(p)) return ORACLE_EINVAL;
    oracle_ctx* c = (oracle_ctx*)calloc(1, sizeof *c);
    if (!c) return ORACLE_ENOMEM;
    c->p = *p;
    c->nx = p->nx; c->ny = p->ny; c->nz = p->nz;
    c->NX = c->nx + 1; c->NY = c->ny + 1; c->NZ = c->nz + 1;
    c->ncell = c->nx * c->ny * c->nz;
    c->nnode = c->NX * c->NY * c->NZ;
    int ok = 1;
    for (int q = 0; q < 3; ++q) {
        c->x[q] = alloc_d(c->nnode, &ok);
        c->u[q] = alloc_d(c->nnode, &ok);
        c->xT[q] = alloc_d(c->nnode, &ok);
        c->x1[q] = alloc_d(c->nnode, &ok);
        c->u1[q] = alloc_d(c->nnode, &ok);
        c->dP[q] = alloc_d(c->ncell, &ok);
    }
    c->m = alloc_d(c->ncell, &ok);
    c->e = alloc_d(c->ncell, &ok);
    c->sig = alloc_d(c->ncell, &ok);
    c->hnu = alloc_d(c->ncell, &ok);
    c->hgm = alloc_d(12 * c->ncell, &ok);
    c->e1 = alloc_d(c->ncell, &ok);
    c->V1 = alloc_d(c->ncell, &ok);
    c->dm = alloc_d(c->ncell, &ok);
    c->dE = alloc_d(c->ncell, &ok);
    c->m2 = alloc_d(c->ncell, &ok);
    c->nmat = p->nmat;
    if (c->nmat > 0) c->qv = alloc_d(c->ncell, &ok);
    for (int k = 0; k < c->nmat; ++k) {
        c->mf[k] = alloc_d(c->ncell, &ok);
        c->mmat[k] = alloc_d(c->ncell, &ok);
        c->me[k] = alloc_d(c->ncell, &ok);
        c->pfm[k] = alloc_d(c->ncell, &ok);
        c->e1m[k] = alloc_d(c->ncell, &ok);
        c->dmm[k] = alloc_d(c->ncell, &ok);
        c->dEm[k] = alloc_d(c->ncell, &ok);
        c->vm2[k] = alloc_d(c->ncell, &ok);
    }
    if (!ok) {
        oracle_destroy(c);
        return ORACLE_ENOMEM;
    }
    /* c.1: X_i = (lx*i)/nx, Y_j = (ly*j)/ny, Z_k = (lz*k)/nz */
    for (int64_t k = 0; k < c->NZ; ++k)
        for (int64_t j = 0; j < c->NY; ++j)
            for (int64_t i = 0; i < c->NX; ++i) {
                int64_t n = nid(c, i, j, k);
                c->xT[0][n] = (p->lx * (double)i) / (double)p->nx;
                c->xT[1][n] = (p->ly * (double)j) / (double)p->ny;
                c->xT[2][n] = (p->lz * (double)k) / (double)p->nz;
                for (int q = 0; q < 3; ++q) {
                    c->x[q][n] = c->xT[q][n];
                    c->u[q][n] = 0.0;
                }
            }
    /* c.6: m_K = rho0 * V_K(x^T); e = e_bg except e_000 = E0 / m_000 */
    for (int64_t k = 0; k < c->nz; ++k)
        for (int64_t j = 0; j < c->ny; ++j)
            for (int64_t i = 0; i < c->nx; ++i) {
                double N[8][3];
                face_t F[6];
                cell_nodes(c, c->x, i, j, k, N);
                hex_faces(N, F);
                int64_t K = cid(c, i, j, k);
                c->m[K] = p->rho0 * hex_volume_from_faces(F);
                c->e[K] = p->e_background;
            }
    c->e[0] = p->e_deposit / c->m[0];
    /* MM7: the whole Sedov cell is material 0 (f_0 = 1, m_0 = m, e_0 = e); the
     * other materials are absent (f = m = e = 0) until set through the fields */
    if (c->nmat > 0)
        for (int64_t K = 0; K < c->ncell; ++K) {
            c->mf[0][K] = 1.0;
            c->mmat[0][K] = c->m[K];
            c->me[0][K] = c->e[K];
        }
    c->t = 0.0;
    c->dt_prev = -1.0;
    c->cycle = 0;
    c->err_cell = -1;
    snprintf(c->err, sizeof c->err, "OK");
    *out = c;
    return ORACLE_OK;
}

void oracle_destroy(oracle_ctx* c)
{
    if (!c) return;
    for (int q = 0; q < 3; ++q) {
        free(c->x[q]); free(c->u[q]); free(c->xT[q]);
        free(c->x1[q]); free(c->u1[q]); free(c->dP[q]);
    }
    free(c->hnu); free(c->hgm);
    free(c->m); free(c->e); free(c->sig); free(c->e1); free(c->V1);
    free(c->dm); free(c->dE); free(c->m2);
    free(c->qv);
    for (int k = 0; k < c->nmat; ++k) {
        free(c->mf[k]); free(c->mmat[k]); free(c->me[k]); free(c->pfm[k]);
        free(c->e1m[k]); free(c->dmm[k]); free(c->dEm[k]); free(c->vm2[k]);
    }
    free(c);
}

/* MM1 for cell K of the current state at volume V (rho = m / V of the cell) */
static void cell_mix(const oracle_ctx* c, int64_t K, double V, double rho, double* p, double* P,
                     double* cs, double* pf)
{
    double f[ORACLE_MAX_MAT], mm[ORACLE_MAX_MAT], e[ORACLE_MAX_MAT];
    for (int k = 0; k < c->nmat; ++k) {
        f[k] = c->mf[k][K];
        mm[k] = c->mmat[k][K];
        e[k] = c->me[k][K];
    }
    mix_eos(c->nmat, c->p.mat_gamma, f, mm, e, V, rho, p, P, cs, pf);
}

/* ------------------------------------------------------------------------- */
/* c.5 time step                                                              */
/* ------------------------------------------------------------------------- */
/* dt_cfl = min over cells of dt_K, from the state (x, u, m, e) */
static double dt_cfl_of_state(oracle_ctx* c)
{
    const oracle_params* p = &c->p;
    double best = INFINITY;
    int any_nan = 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) reduction(min : best) reduction(| : any_nan)
#endif
    for (int64_t k = 0; k < c->nz; ++k)
        for (int64_t j = 0; j < c->ny; ++j)
            for (int64_t i = 0; i < c->nx; ++i) {
                double N[8][3], U[8][3];
                face_t F[6];
                cell_nodes(c, c->x, i, j, k, N);
                cell_nodes(c, c->u, i, j, k, U);
                hex_faces(N, F);
                int64_t K = cid(c, i, j, k);
                double V = hex_volume_from_faces(F);
                double rho = c->m[K] / V, pr, pf, cs;
                if (c->nmat > 0) {
                    double pfk[ORACLE_MAX_MAT];
                    cell_mix(c, K, V, rho, &pr, &pf, &cs, pfk);
                } else {
                    eos(p->gamma, rho, c->e[K], &pr, &pf, &cs);
                }
                double du = cell_jumps(F, U, NULL);
                double l2 = min_edge2(N);
                double v2 = 0.0;
                for (int h = 0; h < 8; ++h) {
                    double s2 = (U[h][0] * U[h][0] + U[h][1] * U[h][1]) + U[h][2] * U[h][2];
                    v2 = (h == 0) ? s2 : dmax(v2, s2);
                }
                double dtK = dt_cell(p->cfl, l2, v2, cs, du, p->q_lin, p->q_quad);
                if (dtK != dtK) any_nan = 1;
                else best = dmin(best, dtK);
            }
    /* a NaN candidate anywhere makes dt_cfl NaN (order-free), which trips the
     * !(dt_u > 0) collapse check (reading Q21). */
    return any_nan ? NAN : best;
}

/* c.5: returns 0 and *dt, or an error code. */
static int32_t next_dt(oracle_ctx* c, double* dt)
{
    const oracle_params* p = &c->p;
    double dt_cfl = dt_cfl_of_state(c);
    double dt_u = (c->dt_prev < 0.0) ? dt_cfl : dmin(dt_cfl, p->dt_growth * c->dt_prev);
    /* collapse: relative to t_end, or without an end time to the time
     * reached so far (reading DT-C) */
    double tref = (p->t_end > 0.0) ? p->t_end : c->t;
    if (!(dt_u > 0.0) || dt_u < 1e-14 * tref)
        return ORACLE_EDTCOLLAPSE;
    double d = dt_u;
    if (p->t_end > 0.0) d = dmin(dt_u, p->t_end - c->t);
    *dt = d;
    return ORACLE_OK;
}

/* ------------------------------------------------------------------------- */
/* c.3 Lagrangian phase                                                       */
/* ------------------------------------------------------------------------- */
static void reflect(const oracle_ctx* c, int64_t i, int64_t j, int64_t k, double v[3])
{
    uint32_t r = c->p.reflect_mask;
    if (((r & 1u) && i == 0) || ((r & 2u) && i == c->nx)) v[0] = 0.0;
    if (((r & 4u) && j == 0) || ((r & 8u) && j == c->ny)) v[1] = 0.0;
    if (((r & 16u) && k == 0) || ((r & 32u) && k == c->nz)) v[2] = 0.0;
}

static int cell_exists(const oracle_ctx* c, int64_t i, int64_t j, int64_t k)
{
    return i >= 0 && i < c->nx && j >= 0 && j < c->ny && k >= 0 && k < c->nz;
}

/* Steps 1-3: per cell rho, p, pf, c, q, sigma = 0.25*(pf+q); reading HG: the
 * cell's hourglass coefficient nu and mode amplitudes g of u^n */
static void lagrange_sigma(oracle_ctx* c, double dt)
{
    const oracle_params* p = &c->p;
    OMP_FOR
    for (int64_t k = 0; k < c->nz; ++k)
        for (int64_t j = 0; j < c->ny; ++j)
            for (int64_t i = 0; i < c->nx; ++i) {
                double N[8][3], U[8][3];
                face_t F[6];
                cell_nodes(c, c->x, i, j, k, N);
                cell_nodes(c, c->u, i, j, k, U);
                hex_faces(N, F);
                int64_t K = cid(c, i, j, k);
                double V = hex_volume_from_faces(F);
                double rho = c->m[K] / V, pr, pf, cs;
                if (c->nmat > 0) {
                    /* MM2-MM3: q from the cell density and the mixed sound speed;
                     * sigma from the mixed floored pressure P (pf here) */
                    double pfk[ORACLE_MAX_MAT];
                    cell_mix(c, K, V, rho, &pr, &pf, &cs, pfk);
                    for (int m = 0; m < c->nmat; ++m) c->pfm[m][K] = pfk[m];
                } else {
                    eos(p->gamma, rho, c->e[K], &pr, &pf, &cs);
                }
                double Lsum;
                double du = cell_jumps(F, U, &Lsum);
                double q = q_of_du(rho, cs, du, p->q_lin, p->q_quad);
                if (c->nmat > 0) c->qv[K] = q;
                c->sig[K] = 0.25 * (pf + q);
                double g[4][3];
                hg_modes(U, g);
                c->hnu[K] = hg_cap(hg_nu(p->hg, c->m[K], cs, Lsum), c->m[K], dt);
                for (int m = 0; m < 4; ++m)
                    for (int q3 = 0; q3 < 3; ++q3) c->hgm[12 * K + 3 * m + q3] = g[m][q3];
            }
}

static void cell_hg_modes(const oracle_ctx* c, int64_t K, double g[4][3])
{
    for (int m = 0; m < 4; ++m)
        for (int q = 0; q < 3; ++q) g[m][q] = c->hgm[12 * K + 3 * m + q];
}

/* Steps 4-6: nodal force and mass by gather, kinematics, BC, move.  Reading HG:
 * cell K's contribution to node n is (sigma_K C_K,n) + f_K,h (h = n's corner). */
static void lagrange_nodes(oracle_ctx* c, double dt)
{
    OMP_FOR
    for (int64_t k = 0; k < c->NZ; ++k)
        for (int64_t j = 0; j < c->NY; ++j)
            for (int64_t i = 0; i < c->NX; ++i) {
                double F[3] = {0.0, 0.0, 0.0}, M = 0.0;
                int first = 1;
                /* gather order: cells (i-1+a', j-1+b', k-1+c'), a' fastest */
                for (int cp = 0; cp < 2; ++cp)
                    for (int bp = 0; bp < 2; ++bp)
                        for (int ap = 0; ap < 2; ++ap) {
                            int64_t ci = i - 1 + ap, cj = j - 1 + bp, ck = k - 1 + cp;
                            if (!cell_exists(c, ci, cj, ck)) continue;
                            double N[8][3], C[3];
                            face_t Fc[6];
                            cell_nodes(c, c->x, ci, cj, ck, N);
                            hex_faces(N, Fc);
                            corner_vector(Fc, 1 - ap, 1 - bp, 1 - cp, C);
                            int64_t K = cid(c, ci, cj, ck);
                            double s = c->sig[K], g[4][3], fh[3];
                            cell_hg_modes(c, K, g);
                            hg_corner(g, c->hnu[K], ((1 - cp) * 2 + (1 - bp)) * 2 + (1 - ap), fh);
                            if (first) {
                                for (int q = 0; q < 3; ++q) F[q] = (s * C[q]) + fh[q];
                                M = c->m[K];
                                first = 0;
                            } else {
                                for (int q = 0; q < 3; ++q) F[q] = F[q] + ((s * C[q]) + fh[q]);
                                M = M + c->m[K];
                            }
                        }
                M = 0.125 * M;
                int64_t n = nid(c, i, j, k);
                double un[3];
                for (int q = 0; q < 3; ++q) un[q] = c->u[q][n] + ((F[q] / M) * dt);
                reflect(c, i, j, k, un);
                for (int q = 0; q < 3; ++q) {
                    c->u1[q][n] = un[q];
                    c->x1[q][n] = c->x[q][n] + (un[q] * dt);
                }
            }
}

/* c.3 step 7: W = sum over corners of C_h(x^n) . (u_h + u'_h)/2 */
static double cell_work(const double N0[8][3], const double U0[8][3], const double U1[8][3])
{
    face_t F[6];
    hex_faces(N0, F);
    double W = 0.0;
    for (int cc = 0; cc < 2; ++cc)
        for (int b = 0; b < 2; ++b)
            for (int a = 0; a < 2; ++a) {
                int h = (cc * 2 + b) * 2 + a;
                double C[3], ub[3];
                corner_vector(F, a, b, cc, C);
                for (int q = 0; q < 3; ++q) ub[q] = 0.5 * (U0[h][q] + U1[h][q]);
                double term = (C[0] * ub[0] + C[1] * ub[1]) + C[2] * ub[2];
                W = (h == 0) ? term : W + term;
            }
    return W;
}

/* reading HG: W_hg = sum over corners of f_h . (u_h + u'_h)/2, f_h the cell's
 * hourglass corner force (from u^n) */
static double cell_hg_work(const double g[4][3], double nu, const double U0[8][3],
                           const double U1[8][3])
{
    double W = 0.0;
    for (int h = 0; h < 8; ++h) {
        double f[3], ub[3];
        hg_corner(g, nu, h, f);
        for (int q = 0; q < 3; ++q) ub[q] = 0.5 * (U0[h][q] + U1[h][q]);
        double term = (f[0] * ub[0] + f[1] * ub[1]) + f[2] * ub[2];
        W = (h == 0) ? term : W + term;
    }
    return W;
}

/* c.3 step 7 for one cell (shared with the exported unit entry point), with the
 * hourglass work of reading HG: e' = e - ((((sigma W) + W_hg) dt) / m) */
static double energy_update(const double N0[8][3], const double U0[8][3],
                            const double U1[8][3], double sigma, double nu, double m,
                            double e, double dt)
{
    double W = cell_work(N0, U0, U1);
    double g[4][3];
    hg_modes(U0, g);
    double Wh = cell_hg_work(g, nu, U0, U1);
    return e - ((((sigma * W) + Wh) * dt) / m);
}

/* Step 7: V' (tangle check), compatible pdV energy update */
static int32_t lagrange_energy(oracle_ctx* c, double dt)
{
    int64_t bad = INT64_MAX;   /* lowest tangled cell (the serial scan's first) */
    OMP_FOR_MIN_BAD
    for (int64_t k = 0; k < c->nz; ++k)
        for (int64_t j = 0; j < c->ny; ++j)
            for (int64_t i = 0; i < c->nx; ++i) {
                double N0[8][3], N1[8][3], U0[8][3], U1[8][3];
                face_t F1[6];
                cell_nodes(c, c->x, i, j, k, N0);
                cell_nodes(c, c->x1, i, j, k, N1);
                cell_nodes(c, c->u, i, j, k, U0);
                cell_nodes(c, c->u1, i, j, k, U1);
                hex_faces(N1, F1);
                int64_t K = cid(c, i, j, k);
                double V1 = hex_volume_from_faces(F1);
                if (!(V1 > 0.0)) {
                    bad = (K < bad) ? K : bad;
                    continue;
                }
                c->V1[K] = V1;
                if (c->nmat > 0) {
                    /* MM4: each present material does the cell's work with its own
                     * stress sigma_m = 0.25 (pf_m + q) on its volume share f_m (shared
                     * strain: f_m is constant through the Lagrangian phase) */
                    double W = cell_work(N0, U0, U1), g[4][3];
                    cell_hg_modes(c, K, g);
                    double Wh = cell_hg_work(g, c->hnu[K], U0, U1);
                    for (int m = 0; m < c->nmat; ++m) {
                        double f = c->mf[m][K], mm = c->mmat[m][K], em = c->me[m][K];
                        if (f > 0.0 && mm > 0.0) {
                            /* HG: the hourglass heat is shared by volume fraction */
                            double sm = 0.25 * (c->pfm[m][K] + c->qv[K]);
                            c->e1m[m][K] = em - (((((sm * W) + Wh) * dt) * f) / mm);
                        } else {
                            c->e1m[m][K] = em;
                        }
                    }
                } else {
                    double W = cell_work(N0, U0, U1), g[4][3];
                    cell_hg_modes(c, K, g);
                    double Wh = cell_hg_work(g, c->hnu[K], U0, U1);
                    c->e1[K] = c->e[K] - ((((c->sig[K] * W) + Wh) * dt) / c->m[K]);
                }
            }
    if (bad != INT64_MAX) return fail(c, ORACLE_ETANGLED, bad);
    return ORACLE_OK;
}

/* ------------------------------------------------------------------------- */
/* c.4 Eulerian remap                                                         */
/* ------------------------------------------------------------------------- */
/* c.4 step 1: hex (0,0,0)=P0^T (1,0,0)=P1^T (1,1,0)=P2^T (0,1,0)=P3^T,
 *                 (0,0,1)=P0'  (1,0,1)=P1'  (1,1,1)=P2'  (0,1,1)=P3'        */
static double swept_volume(const double PT[4][3], const double PL[4][3])
{
    double N[8][3];
    static const int map[4][2] = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
    for (int v = 0; v < 4; ++v) {
        int a = map[v][0], b = map[v][1];
        for (int q = 0; q < 3; ++q) {
            N[(0 * 2 + b) * 2 + a][q] = PT[v][q];
            N[(1 * 2 + b) * 2 + a][q] = PL[v][q];
        }
    }
    face_t F[6];
    hex_faces(N, F);
    return hex_volume_from_faces(F);
}

/* canonical P0..P3 of the physical face of axis `ax` at lower cell (i,j,k)'s
 * +ax side, i.e. node plane (i+1 | j+1 | k+1), as global node indices. */
static void face_node_ids(const oracle_ctx* c, int ax, int64_t i, int64_t j, int64_t k,
                          int64_t ids[4])
{
    if (ax == 0) {        /* X-face at node plane i+1: (i',j,k)(i',j+1,k)(i',j+1,k+1)(i',j,k+1) */
        int64_t I = i + 1;
        ids[0] = nid(c, I, j, k); ids[1] = nid(c, I, j + 1, k);
        ids[2] = nid(c, I, j + 1, k + 1); ids[3] = nid(c, I, j, k + 1);
    } else if (ax == 1) { /* Y-face at node plane j+1: (i,j',k)(i,j',k+1)(i+1,j',k+1)(i+1,j',k) */
        int64_t J = j + 1;
        ids[0] = nid(c, i, J, k); ids[1] = nid(c, i, J, k + 1);
        ids[2] = nid(c, i + 1, J, k + 1); ids[3] = nid(c, i + 1, J, k);
    } else {              /* Z-face at node plane k+1: (i,j,k')(i+1,j,k')(i+1,j+1,k')(i,j+1,k') */
        int64_t Kp = k + 1;
        ids[0] = nid(c, i, j, Kp); ids[1] = nid(c, i + 1, j, Kp);
        ids[2] = nid(c, i + 1, j + 1, Kp); ids[3] = nid(c, i, j + 1, Kp);
    }
}

/* c.4 steps 1-2 for the interior face between cell L=(i,j,k) and its +ax
 * neighbour U: the swept volume dV, the donor cell D and its mean velocity Ub. */
static void face_donor(oracle_ctx* c, int ax, int64_t i, int64_t j, int64_t k, double* dVout,
                       int64_t* Dout, double Ub[3])
{
    int64_t ids[4];
    face_node_ids(c, ax, i, j, k, ids);
    double PT[4][3], PL[4][3];
    for (int v = 0; v < 4; ++v)
        for (int q = 0; q < 3; ++q) {
            PT[v][q] = c->xT[q][ids[v]];
            PL[v][q] = c->x1[q][ids[v]];
        }
    double dV = swept_volume(PT, PL);
    int64_t di = i, dj = j, dk = k;             /* donor: lower if dV > 0 */
    if (!(dV > 0.0)) {
        if (ax == 0) di = i + 1; else if (ax == 1) dj = j + 1; else dk = k + 1;
    }
    int64_t D = cid(c, di, dj, dk);
    double U[8][3];
    cell_nodes(c, c->u1, di, dj, dk, U);
    for (int q = 0; q < 3; ++q) {
        double s = U[0][q];
        for (int h = 1; h < 8; ++h) s = s + U[h][q];
        Ub[q] = 0.125 * s;
    }
    *dVout = dV;
    *Dout = D;
}

/* c.4 steps 1-2: mu, eps, pi[3] through the face (positive = toward +ax). */
static void face_flux(oracle_ctx* c, int ax, int64_t i, int64_t j, int64_t k, double* mu,
                      double* eps, double pi[3])
{
    double dV, Ub[3];
    int64_t D;
    face_donor(c, ax, i, j, k, &dV, &D, Ub);
    *mu = (c->m[D] / c->V1[D]) * dV;
    *eps = *mu * c->e1[D];
    for (int q = 0; q < 3; ++q) pi[q] = *mu * Ub[q];
}

/* c.4 steps 1-3: per cell, fluxes through its six faces (boundary faces carry
 * +0.0), Delta m/E/P, m'' = m + Delta m (ENEGMASS if !(m'' > 0)). */
static int32_t euler_cells(oracle_ctx* c)
{
    const int64_t nmax[3] = {c->nx, c->ny, c->nz};
    int64_t bad = INT64_MAX;   /* lowest cell with m'' !> 0 (the serial scan's first) */
    OMP_FOR_MIN_BAD
    for (int64_t k = 0; k < c->nz; ++k)
        for (int64_t j = 0; j < c->ny; ++j)
            for (int64_t i = 0; i < c->nx; ++i) {
                double mu[6], ep[6], pi[6][3];   /* order -x,+x,-y,+y,-z,+z */
                const int64_t ijk[3] = {i, j, k};
                for (int ax = 0; ax < 3; ++ax) {
                    if (ijk[ax] > 0) {           /* -ax face: lower cell ijk - e_ax */
                        int64_t l[3] = {i, j, k};
                        l[ax] -= 1;
                        face_flux(c, ax, l[0], l[1], l[2], &mu[2 * ax], &ep[2 * ax], pi[2 * ax]);
                    } else {
                        mu[2 * ax] = 0.0; ep[2 * ax] = 0.0;
                        pi[2 * ax][0] = pi[2 * ax][1] = pi[2 * ax][2] = 0.0;
                    }
                    if (ijk[ax] < nmax[ax] - 1) { /* +ax face: lower cell is ijk */
                        face_flux(c, ax, i, j, k, &mu[2 * ax + 1], &ep[2 * ax + 1], pi[2 * ax + 1]);
                    } else {
                        mu[2 * ax + 1] = 0.0; ep[2 * ax + 1] = 0.0;
                        pi[2 * ax + 1][0] = pi[2 * ax + 1][1] = pi[2 * ax + 1][2] = 0.0;
                    }
                }
                int64_t K = cid(c, i, j, k);
                double dm = ((((mu[0] - mu[1]) + mu[2]) - mu[3]) + mu[4]) - mu[5];
                double dE = ((((ep[0] - ep[1]) + ep[2]) - ep[3]) + ep[4]) - ep[5];
                for (int q = 0; q < 3; ++q)
                    c->dP[q][K] = ((((pi[0][q] - pi[1][q]) + pi[2][q]) - pi[3][q]) + pi[4][q]) - pi[5][q];
                double m2 = c->m[K] + dm;
                if (!(m2 > 0.0)) {
                    bad = (K < bad) ? K : bad;
                    continue;
                }
                c->dm[K] = dm;
                c->dE[K] = dE;
                c->m2[K] = m2;
            }
    if (bad != INT64_MAX) return fail(c, ORACLE_ENEGMASS, bad);
    return ORACLE_OK;
}

/* MM5: per material m through the face: mass mu_m = (m_m,D / V'_D) dV (the
 * donor's material mass per unit cell volume), volume phi_m = f_m,D dV, energy
 * eps_m = mu_m e'_m,D; the face total mu = sum_m mu_m carries the momentum
 * pi = mu Ub.  With one material, mu = mu_0 = (m_D / V'_D) dV as in c.4. */
typedef struct { double mu, pi[3], mum[ORACLE_MAX_MAT], phim[ORACLE_MAX_MAT], epm[ORACLE_MAX_MAT]; } mflux_t;

static void face_flux_mm(oracle_ctx* c, int ax, int64_t i, int64_t j, int64_t k, mflux_t* o)
{
    double dV, Ub[3];
    int64_t D;
    face_donor(c, ax, i, j, k, &dV, &D, Ub);
    for (int m = 0; m < c->nmat; ++m) {
        o->mum[m] = (c->mmat[m][D] / c->V1[D]) * dV;
        o->phim[m] = c->mf[m][D] * dV;
        o->epm[m] = o->mum[m] * c->e1m[m][D];
        o->mu = (m == 0) ? o->mum[0] : o->mu + o->mum[m];
    }
    for (int q = 0; q < 3; ++q) o->pi[q] = o->mu * Ub[q];
}

static void mflux_zero(mflux_t* o)
{
    memset(o, 0, sizeof *o);   /* boundary faces carry +0.0 */
}

/* c.4 steps 1-3 with materials (MM6): six-face sums (order -x +x -y +y -z +z, as
 * c.4 step 3) per material of mu_m, eps_m, phi_m, and of the totals mu and pi;
 * m''_m = m_m + Dm_m, V''_m = (f_m V') + Dphi_m, m'' = sum_m m''_m.  ENEGMASS if
 * !(m'' > 0), or any m''_m < 0 or V''_m < 0, or !(sum_m V''_m > 0). */
static int32_t euler_cells_mm(oracle_ctx* c)
{
    const int64_t nmax[3] = {c->nx, c->ny, c->nz};
    int64_t bad = INT64_MAX;   /* lowest failing cell (the serial scan's first) */
    OMP_FOR_MIN_BAD
    for (int64_t k = 0; k < c->nz; ++k)
        for (int64_t j = 0; j < c->ny; ++j)
            for (int64_t i = 0; i < c->nx; ++i) {
                mflux_t F[6];
                const int64_t ijk[3] = {i, j, k};
                for (int ax = 0; ax < 3; ++ax) {
                    if (ijk[ax] > 0) {
                        int64_t l[3] = {i, j, k};
                        l[ax] -= 1;
                        face_flux_mm(c, ax, l[0], l[1], l[2], &F[2 * ax]);
                    } else {
                        mflux_zero(&F[2 * ax]);
                    }
                    if (ijk[ax] < nmax[ax] - 1) face_flux_mm(c, ax, i, j, k, &F[2 * ax + 1]);
                    else mflux_zero(&F[2 * ax + 1]);
                }
                int64_t K = cid(c, i, j, k);
                c->dm[K] = ((((F[0].mu - F[1].mu) + F[2].mu) - F[3].mu) + F[4].mu) - F[5].mu;
                for (int q = 0; q < 3; ++q)
                    c->dP[q][K] = ((((F[0].pi[q] - F[1].pi[q]) + F[2].pi[q]) - F[3].pi[q]) + F[4].pi[q]) - F[5].pi[q];
                double m2 = 0.0, VV = 0.0;
                int neg = 0;
                for (int m = 0; m < c->nmat; ++m) {
                    double dmm = ((((F[0].mum[m] - F[1].mum[m]) + F[2].mum[m]) - F[3].mum[m]) + F[4].mum[m]) - F[5].mum[m];
                    double dEm = ((((F[0].epm[m] - F[1].epm[m]) + F[2].epm[m]) - F[3].epm[m]) + F[4].epm[m]) - F[5].epm[m];
                    double dph = ((((F[0].phim[m] - F[1].phim[m]) + F[2].phim[m]) - F[3].phim[m]) + F[4].phim[m]) - F[5].phim[m];
                    double mm2 = c->mmat[m][K] + dmm;
                    double vm2 = (c->mf[m][K] * c->V1[K]) + dph;
                    if (mm2 < 0.0 || vm2 < 0.0) neg = 1;
                    c->dmm[m][K] = dmm;
                    c->dEm[m][K] = dEm;
                    c->vm2[m][K] = vm2;
                    m2 = (m == 0) ? mm2 : m2 + mm2;
                    VV = (m == 0) ? vm2 : VV + vm2;
                }
                if (neg || !(m2 > 0.0) || !(VV > 0.0)) {
                    bad = (K < bad) ? K : bad;
                    continue;
                }
                c->m2[K] = m2;
            }
    if (bad != INT64_MAX) return fail(c, ORACLE_ENEGMASS, bad);
    return ORACLE_OK;
}

static void euler_nodes(oracle_ctx* c);

/* MM6 commit: e''_m = e'_m + ((DE_m - e'_m Dm_m) / m''_m) (c.4 step 3 per material;
 * 0 for a material whose mass is 0), f''_m = V''_m / sum_k V''_k, m_m := m''_m;
 * then the node update and x := x^T as c.4 steps 4-5 with the cell totals. */
static void euler_commit_mm(oracle_ctx* c)
{
    OMP_FOR
    for (int64_t K = 0; K < c->ncell; ++K) {
        double VV = 0.0;
        for (int m = 0; m < c->nmat; ++m) VV = (m == 0) ? c->vm2[0][K] : VV + c->vm2[m][K];
        for (int m = 0; m < c->nmat; ++m) {
            double mm2 = c->mmat[m][K] + c->dmm[m][K];
            double e1 = c->e1m[m][K];
            c->me[m][K] = (mm2 > 0.0) ? e1 + ((c->dEm[m][K] - (e1 * c->dmm[m][K])) / mm2) : 0.0;
            c->mf[m][K] = c->vm2[m][K] / VV;
            c->mmat[m][K] = mm2;
        }
    }
    euler_nodes(c);
}

/* c.4 step 3 (e''), step 4 (node momentum, BC), step 5 (x := x^T) */
static void euler_commit(oracle_ctx* c)
{
    OMP_FOR
    for (int64_t K = 0; K < c->ncell; ++K) {
        double e1 = c->e1[K];
        c->e[K] = e1 + ((c->dE[K] - (e1 * c->dm[K])) / c->m2[K]);
    }
    euler_nodes(c);
}

/* c.4 step 4 (node momentum from the gathered Dm, DP, m''; BC), step 5 (x := x^T), m := m'' */
static void euler_nodes(oracle_ctx* c)
{
    OMP_FOR
    for (int64_t k = 0; k < c->NZ; ++k)
        for (int64_t j = 0; j < c->NY; ++j)
            for (int64_t i = 0; i < c->NX; ++i) {
                double Dm = 0.0, DP[3] = {0.0, 0.0, 0.0}, M2 = 0.0;
                int first = 1;
                for (int cp = 0; cp < 2; ++cp)
                    for (int bp = 0; bp < 2; ++bp)
                        for (int ap = 0; ap < 2; ++ap) {
                            int64_t ci = i - 1 + ap, cj = j - 1 + bp, ck = k - 1 + cp;
                            if (!cell_exists(c, ci, cj, ck)) continue;
                            int64_t K = cid(c, ci, cj, ck);
                            if (first) {
                                Dm = c->dm[K];
                                for (int q = 0; q < 3; ++q) DP[q] = c->dP[q][K];
                                M2 = c->m2[K];
                                first = 0;
                            } else {
                                Dm = Dm + c->dm[K];
                                for (int q = 0; q < 3; ++q) DP[q] = DP[q] + c->dP[q][K];
                                M2 = M2 + c->m2[K];
                            }
                        }
                Dm = 0.125 * Dm;
                for (int q = 0; q < 3; ++q) DP[q] = 0.125 * DP[q];
                M2 = 0.125 * M2;
                int64_t n = nid(c, i, j, k);
                double un[3];
                for (int q = 0; q < 3; ++q) {
                    double u1 = c->u1[q][n];
                    un[q] = u1 + ((DP[q] - (u1 * Dm)) / M2);
                }
                reflect(c, i, j, k, un);
                for (int q = 0; q < 3; ++q) {
                    c->u[q][n] = un[q];
                    c->x[q][n] = c->xT[q][n];
                }
            }
    for (int64_t K = 0; K < c->ncell; ++K) c->m[K] = c->m2[K];
}

/* ------------------------------------------------------------------------- */
/* one cycle (c.3, then c.4 in EULER mode), clock (c.3 step 8)                */
/* ------------------------------------------------------------------------- */
static int32_t cycle_once(oracle_ctx* c, double dt)
{
    lagrange_sigma(c, dt);
    lagrange_nodes(c, dt);
    int32_t rc = lagrange_energy(c, dt);
    if (rc) return rc;
    if (c->p.rezone == 1 && c->nmat > 0) {
        rc = euler_cells_mm(c);
        if (rc) return rc;
        euler_commit_mm(c);
    } else if (c->p.rezone == 1) {
        rc = euler_cells(c);
        if (rc) return rc;
        euler_commit(c);
    } else {
        for (int q = 0; q < 3; ++q) {
            double* t;
            t = c->x[q]; c->x[q] = c->x1[q]; c->x1[q] = t;
            t = c->u[q]; c->u[q] = c->u1[q]; c->u1[q] = t;
        }
        double* t = c->e; c->e = c->e1; c->e1 = t;
        for (int m = 0; m < c->nmat; ++m) {
            t = c->me[m]; c->me[m] = c->e1m[m]; c->e1m[m] = t;
        }
    }
    c->t = c->t + dt;
    c->cycle = c->cycle + 1;
    c->dt_prev = dt;
    return ORACLE_OK;
}

int32_t oracle_step(oracle_ctx* c, int32_t ncycles, int32_t* cycles_done)
{
    if (cycles_done) *cycles_done = 0;
    if (!c || ncycles < 0) return ORACLE_EINVAL;
    if (c->poisoned) return ORACLE_EPOISONED;
    int32_t done = 0;
    for (int32_t n = 0; n < ncycles; ++n) {
        if (c->p.t_end > 0.0 && c->t >= c->p.t_end) {   /* c.5 last line */
            c->finished = 1;
            break;
        }
        double dt;
        int32_t rc = next_dt(c, &dt);
        if (rc) {
            if (cycles_done) *cycles_done = done;
            return fail(c, rc, -1);
        }
        rc = cycle_once(c, dt);
        if (rc) {
            if (cycles_done) *cycles_done = done;
            return rc;
        }
        ++done;
    }
    if (c->p.t_end > 0.0 && c->t >= c->p.t_end) c->finished = 1;
    if (cycles_done) *cycles_done = done;
    return ORACLE_OK;
}

int32_t oracle_next_dt(oracle_ctx* c, double* dt)
{
    if (!c || !dt) return ORACLE_EINVAL;
    if (c->p.t_end > 0.0 && c->t >= c->p.t_end) { *dt = -1.0; return ORACLE_OK; }
    return next_dt(c, dt);
}

/* ------------------------------------------------------------------------- */
/* fields (SURVEY §8(b) sale_get_field / sale_set_field)                      */
/* ------------------------------------------------------------------------- */
static int is_node_field(int32_t f) { return f >= ORACLE_F_X && f <= ORACLE_F_NODE_MASS; }
static int is_cell_field(int32_t f) { return f >= ORACLE_F_MASS && f <= ORACLE_F_CS; }
/* material field -> (kind 0 f / 1 m / 2 e, material), or -1 */
static int mat_field(const oracle_ctx* c, int32_t f, int* mat)
{
    if (f < ORACLE_F_MAT_F || f >= ORACLE_F_MAT_E + ORACLE_MAX_MAT) return -1;
    int kind = (f - ORACLE_F_MAT_F) / ORACLE_MAX_MAT;
    *mat = (f - ORACLE_F_MAT_F) % ORACLE_MAX_MAT;
    return (*mat < c->nmat) ? kind : -1;
}
static double* mat_array(oracle_ctx* c, int kind, int mat)
{
    return kind == 0 ? c->mf[mat] : (kind == 1 ? c->mmat[mat] : c->me[mat]);
}

int32_t oracle_get_field(oracle_ctx* c, int32_t field, double* dst, uint64_t count)
{
    if (!c || !dst) return ORACLE_EINVAL;
    if (is_node_field(field)) {
        if (count != (uint64_t)c->nnode) return ORACLE_EINVAL;
        if (field <= ORACLE_F_Z) {
            memcpy(dst, c->x[field - ORACLE_F_X], sizeof(double) * (size_t)c->nnode);
        } else if (field <= ORACLE_F_UZ) {
            memcpy(dst, c->u[field - ORACLE_F_UX], sizeof(double) * (size_t)c->nnode);
        } else { /* NODE_MASS: c.3 step 5 */
            for (int64_t k = 0; k < c->NZ; ++k)
                for (int64_t j = 0; j < c->NY; ++j)
                    for (int64_t i = 0; i < c->NX; ++i) {
                        double M = 0.0;
                        int first = 1;
                        for (int cp = 0; cp < 2; ++cp)
                            for (int bp = 0; bp < 2; ++bp)
                                for (int ap = 0; ap < 2; ++ap) {
                                    int64_t ci = i - 1 + ap, cj = j - 1 + bp, ck = k - 1 + cp;
                                    if (!cell_exists(c, ci, cj, ck)) continue;
                                    double mk = c->m[cid(c, ci, cj, ck)];
                                    M = first ? mk : M + mk;
                                    first = 0;
                                }
                        dst[nid(c, i, j, k)] = 0.125 * M;
                    }
        }
        return ORACLE_OK;
    }
    int mat, kind = mat_field(c, field, &mat);
    if (!is_cell_field(field) && kind < 0) return ORACLE_EINVAL;
    if (count != (uint64_t)c->ncell) return ORACLE_EINVAL;
    if (kind >= 0) { memcpy(dst, mat_array(c, kind, mat), sizeof(double) * (size_t)c->ncell); return 0; }
    if (field == ORACLE_F_MASS) { memcpy(dst, c->m, sizeof(double) * (size_t)c->ncell); return 0; }
    if (field == ORACLE_F_E && c->nmat > 0) {
        /* mixture specific energy (sum_m m_m e_m) / m */
        for (int64_t K = 0; K < c->ncell; ++K) {
            double s = 0.0;
            for (int m = 0; m < c->nmat; ++m) {
                double t = c->mmat[m][K] * c->me[m][K];
                s = (m == 0) ? t : s + t;
            }
            dst[K] = s / c->m[K];
        }
        return 0;
    }
    if (field == ORACLE_F_E) { memcpy(dst, c->e, sizeof(double) * (size_t)c->ncell); return 0; }
    for (int64_t k = 0; k < c->nz; ++k)
        for (int64_t j = 0; j < c->ny; ++j)
            for (int64_t i = 0; i < c->nx; ++i) {
                double N[8][3], U[8][3];
                face_t F[6];
                cell_nodes(c, c->x, i, j, k, N);
                hex_faces(N, F);
                int64_t K = cid(c, i, j, k);
                double V = hex_volume_from_faces(F);
                double rho = c->m[K] / V, pr, pf, cs;
                if (c->nmat > 0) {
                    double pfk[ORACLE_MAX_MAT];
                    cell_mix(c, K, V, rho, &pr, &pf, &cs, pfk);
                } else {
                    eos(c->p.gamma, rho, c->e[K], &pr, &pf, &cs);
                }
                double v;
                switch (field) {
                case ORACLE_F_RHO: v = rho; break;
                case ORACLE_F_VOL: v = V; break;
                case ORACLE_F_P: v = pr; break;
                case ORACLE_F_CS: v = cs; break;
                default: /* Q */
                    cell_nodes(c, c->u, i, j, k, U);
                    v = cell_q(F, U, rho, cs, c->p.q_lin, c->p.q_quad);
                    break;
                }
                dst[K] = v;
            }
    return ORACLE_OK;
}

int32_t oracle_set_field(oracle_ctx* c, int32_t field, const double* src, uint64_t count)
{
    if (!c || !src) return ORACLE_EINVAL;
    if (c->poisoned) return ORACLE_EPOISONED;
    double* dst = NULL;
    uint64_t need = 0;
    int mat, kind = mat_field(c, field, &mat);
    if (kind >= 0) {
        if (count != (uint64_t)c->ncell) return ORACLE_EINVAL;
        memcpy(mat_array(c, kind, mat), src, sizeof(double) * (size_t)c->ncell);
        if (kind == 1)   /* the cell mass is the sum of the material masses */
            for (int64_t K = 0; K < c->ncell; ++K) {
                double s = 0.0;
                for (int m = 0; m < c->nmat; ++m) s = (m == 0) ? c->mmat[0][K] : s + c->mmat[m][K];
                c->m[K] = s;
            }
        return ORACLE_OK;
    }
    if (c->nmat > 0 && (field == ORACLE_F_MASS || field == ORACLE_F_E)) return ORACLE_EINVAL;
    if (field >= ORACLE_F_X && field <= ORACLE_F_Z) {
        if (c->p.rezone == 1) return ORACLE_EINVAL;     /* Euler: x = x^T */
        dst = c->x[field - ORACLE_F_X]; need = (uint64_t)c->nnode;
    } else if (field >= ORACLE_F_UX && field <= ORACLE_F_UZ) {
        dst = c->u[field - ORACLE_F_UX]; need = (uint64_t)c->nnode;
    } else if (field == ORACLE_F_MASS) {
        dst = c->m; need = (uint64_t)c->ncell;
    } else if (field == ORACLE_F_E) {
        dst = c->e; need = (uint64_t)c->ncell;
    } else {
        return ORACLE_EINVAL;
    }
    if (count != need) return ORACLE_EINVAL;
    memcpy(dst, src, sizeof(double) * (size_t)need);
    return ORACLE_OK;
}

int32_t oracle_get_clock(oracle_ctx* c, double* t, double* dt_last, int64_t* cycle,
                         int32_t* finished)
{
    if (!c) return ORACLE_EINVAL;
    if (t) *t = c->t;
    if (dt_last) *dt_last = c->dt_prev;
    if (cycle) *cycle = c->cycle;
    if (finished) *finished = (c->p.t_end > 0.0 && c->t >= c->p.t_end) ? 1 : 0;
    return ORACLE_OK;
}

int32_t oracle_set_clock(oracle_ctx* c, double t, double dt_last, int64_t cycle)
{
    if (!c || cycle < 0) return ORACLE_EINVAL;
    if (c->poisoned) return ORACLE_EPOISONED;
    c->t = t;
    c->dt_prev = dt_last;
    c->cycle = cycle;
    c->finished = 0;
    return ORACLE_OK;
}

const char* oracle_last_error(const oracle_ctx* c) { return c ? c->err : "null context"; }
int64_t oracle_last_error_cell(const oracle_ctx* c) { return c ? c->err_cell : -1; }

/* ------------------------------------------------------------------------- */
/* unit entry points for the pins                                             */
/* ------------------------------------------------------------------------- */
void oracle_face(const double* P, double* A, double* Xbar, double* s)
{
    face_t f;
    face_geom(P, P + 3, P + 6, P + 9, &f);
    for (int q = 0; q < 3; ++q) { A[q] = f.A[q]; Xbar[q] = f.Xb[q]; }
    *s = f.s;
}

double oracle_hex_volume(const double* Nflat)
{
    double N[8][3];
    face_t F[6];
    for (int h = 0; h < 8; ++h)
        for (int q = 0; q < 3; ++q) N[h][q] = Nflat[h * 3 + q];
    hex_faces(N, F);
    return hex_volume_from_faces(F);
}

void oracle_eos(double gamma, double rho, double e, double* p, double* pf, double* cs)
{
    eos(gamma, rho, e, p, pf, cs);
}

void oracle_mix_eos(int32_t nmat, const double* gamma, const double* f, const double* mm, const double* e,
                    double V, double rho, double* p, double* P, double* cs)
{
    double pf[ORACLE_MAX_MAT];
    if (nmat < 1 || nmat > ORACLE_MAX_MAT) return;
    mix_eos(nmat, gamma, f, mm, e, V, rho, p, P, cs, pf);
}

double oracle_q_of_du(double rho, double cs, double du, double c1, double c2)
{
    return q_of_du(rho, cs, du, c1, c2);
}

double oracle_dt_cell(double cfl, double l2, double v2, double cs, double du, double c1, double c2)
{
    return dt_cell(cfl, l2, v2, cs, du, c1, c2);
}

void oracle_hg_modes(const double* Uf, double* gf)
{
    double U[8][3], g[4][3];
    for (int h = 0; h < 8; ++h)
        for (int q = 0; q < 3; ++q) U[h][q] = Uf[h * 3 + q];
    hg_modes(U, g);
    for (int m = 0; m < 4; ++m)
        for (int q = 0; q < 3; ++q) gf[m * 3 + q] = g[m][q];
}

void oracle_hg_corner(const double* gf, double nu, int32_t h, double* f)
{
    double g[4][3];
    for (int m = 0; m < 4; ++m)
        for (int q = 0; q < 3; ++q) g[m][q] = gf[m * 3 + q];
    hg_corner(g, nu, (int)h, f);
}

double oracle_hg_nu(double hg, double m, double cs, double Lsum, double dt)
{
    return hg_cap(hg_nu(hg, m, cs, Lsum), m, dt);
}

double oracle_swept_volume(const double* PTf, const double* PLf)
{
    double PT[4][3], PL[4][3];
    for (int v = 0; v < 4; ++v)
        for (int q = 0; q < 3; ++q) { PT[v][q] = PTf[v * 3 + q]; PL[v][q] = PLf[v * 3 + q]; }
    return swept_volume(PT, PL);
}

double oracle_cell_energy(const double* N0f, const double* U0f, const double* U1f,
                          double sigma, double nu, double m, double e, double dt)
{
    double N0[8][3], U0[8][3], U1[8][3];
    for (int h = 0; h < 8; ++h)
        for (int q = 0; q < 3; ++q) {
            N0[h][q] = N0f[h * 3 + q]; U0[h][q] = U0f[h * 3 + q]; U1[h][q] = U1f[h * 3 + q];
        }
    return energy_update(N0, U0, U1, sigma, nu, m, e, dt);
}

/* ---- Steinberg (Fig. 6b) ------------------------ */
void oracle_steinberg_point(const oracle_steinberg_params* sp, double p, double rho, double e, double eps_p,
                            double* shear, double* yield)
{
    const double eta = sp->rho0 / rho;
    const double T = e / sp->cv;
    const double G = (sp->G0 + (sp->GP * p) * pow(eta, 1.0 / 3.0)) + sp->GT * (T - sp->T0);
    const double h = sp->Y0 * pow(1.0 + sp->beta * eps_p, sp->n);
    *shear = G;
    *yield = ((h < sp->Ymax) ? h : sp->Ymax) * (G / sp->G0);
}

int32_t oracle_steinberg(oracle_ctx* c, const oracle_steinberg_params* sp, const double* eps_p, double* shear,
                         double* yield, uint64_t count)
{
    if (!c || !sp || !shear || !yield || count != (uint64_t)c->ncell) return ORACLE_EINVAL;
    double* rho = (double*)malloc(sizeof(double) * (size_t)c->ncell);
    double* pr = (double*)malloc(sizeof(double) * (size_t)c->ncell);
    double* e = (double*)malloc(sizeof(double) * (size_t)c->ncell);
    if (!rho || !pr || !e) {
        free(rho);
        free(pr);
        free(e);
        return ORACLE_EINVAL;
    }
    int32_t rc = oracle_get_field(c, ORACLE_F_RHO, rho, count);
    if (!rc) rc = oracle_get_field(c, ORACLE_F_P, pr, count);
    if (!rc) rc = oracle_get_field(c, ORACLE_F_E, e, count);
    /* Fig. 6b: do m = 1, nmats -- every material's constants on the cell quantities */
    const int nm = c->nmat > 0 ? c->nmat : 1;
    for (int m = 0; !rc && m < nm; ++m)
        for (int64_t K = 0; K < c->ncell; ++K)
            oracle_steinberg_point(&sp[m], pr[K], rho[K], e[K], eps_p ? eps_p[K] : 0.0,
                                   &shear[(int64_t)m * c->ncell + K], &yield[(int64_t)m * c->ncell + K]);
    free(rho);
    free(pr);
    free(e);
    return rc;
}

