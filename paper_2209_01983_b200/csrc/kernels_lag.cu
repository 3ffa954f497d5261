// kernels_lag.cu -- the Lagrangian phase of the SALE cycle (SURVEY §8(a) rows S1-S7,
// §8(c) c.3 and c.5, with the readings HG and DT-Q of DESIGN.md §3) for both
// rezoning modes, as z-marching kernels.
//
//   kl_state / ke_state (before the cycle's k_begin): per cell of the cycle-start
//              state the cell state -- sigma = 0.25 (pf + q), the uncapped hourglass
//              coefficient nu_u, each material's stress -- and the c.5 dt candidate
//              (DT-Q signal speed); Lagrange from x, Euler from the target tables.
//   kc_force   : S1 face area vectors at t^n (Lagrange; Euler: target tables), the
//              hourglass mode amplitudes of u^n, per cell the eight corner forces
//              (sigma C_h + f_h) staged in shared memory, the nodal force and mass
//              gather in the fixed order of c.2, kinematics + BC (S5, S6).
//   kc_energy  : S7 geometry at t^{n+1} (V', tangle check), the compatible energy
//              update with the hourglass work.
//
// The node gather is split across z-steps: cell plane k contributes to node plane k
// (its corners c = 0) and starts node plane k+1 (corners c = 1); the running sums
// carry in registers, so one cell plane of corner forces is resident at a time and
// the association stays the oracle's left-to-right gather order (cells a' fastest,
// then b', then c').  Every expression tree is the oracle's, compiled with
// -fmad=false and IEEE div / sqrt, so results are bit-identical.
#include <cuda_runtime.h>

#include <map>
#include <mutex>

#include "sale_mesh.cuh"

// resident CTAs per SM the register budgets are sized for (compile-time tuning knobs)
#ifndef SALE_MB_ENERGY_L
#define SALE_MB_ENERGY_L 2
#endif
#ifndef SALE_MB_FORCE
#define SALE_MB_FORCE 2
#endif
#ifndef SALE_MB_STATE
#define SALE_MB_STATE 2
#endif
#ifndef SALE_MB_STATE_E
#define SALE_MB_STATE_E 4
#endif
#ifndef SALE_FORCE_XROW  // kc_force: one node row staged beyond the thread rows
#define SALE_FORCE_XROW 1
#endif
#ifndef SALE_MB_FORCE_E
#define SALE_MB_FORCE_E 2
#endif
#ifndef SALE_MB_ENERGY_E
#define SALE_MB_ENERGY_E 2
#endif

namespace sale {

namespace {

constexpr int FW = 32;       // columns per warp row
constexpr int PAD = FW + 1;  // smem window padding (neighbour reads never clamp)
constexpr int ZCHUNK = 32;   // z-planes per CTA on large meshes

inline int cdiv(int a, int b) { return (a + b - 1) / b; }
inline int imin_h(int a, int b) { return a < b ? a : b; }
inline int imax_h(int a, int b) { return a > b ? a : b; }

__device__ __forceinline__ D3 ld3s(const double* b, int o0, int stride)
{
    return D3{b[o0], b[o0 + stride], b[o0 + 2 * stride]};
}
__device__ __forceinline__ void st3s(double* b, int o0, int stride, D3 v)
{
    b[o0] = v.x;
    b[o0 + stride] = v.y;
    b[o0 + 2 * stride] = v.z;
}
__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }


// opt a kernel into `bytes` of dynamic shared memory, once per kernel (a process-wide
// registry keyed by the kernel's address: instantiations of one launch lambda share
// its function-local statics, so those cannot carry the flag)
template <typename K>
void set_smem(K kernel, size_t bytes)
{
    static std::mutex mu;
    static std::map<const void*, size_t> done;
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = done[(const void*)kernel];
    if (have < bytes) {
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        have = bytes;
    }
}

template <int N>
struct IC {
    static constexpr int value = N;
};
template <class F>
void by_nmat(int nmat, F&& f)
{
    switch (nmat) {
    case 0: f(IC<0>{}); break;
    case 1: f(IC<1>{}); break;
    case 2: f(IC<2>{}); break;
    case 3: f(IC<3>{}); break;
    default: f(IC<4>{}); break;
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// the cell state of c.3 steps 1-3 and reading HG for one cell: from its mass m,
// energy e (NM > 0: the material operands), volume V, compressive jump du and
// separation sum Lsum.  sig = 0.25 (pf + q) (materials: P of MM1; sg[k] = 0.25
// (pf_k + q)), nu_u = (hg (m c)) / (Lsum / 3), cq = the DT-Q viscous speed.
// ---------------------------------------------------------------------------
template <int NM>
__device__ __forceinline__ void cell_state(const Slab& s, const Phys& p, double m, double e, const double* f,
                                           const double* mm, const double* em, double V, double du, double Lsum,
                                           double& sig, double& nu_u, double& cs, double& cq, double sg[MAX_MAT])
{
    const double rho = ddiv(m, V);
    double pr, pf, pfk[MAX_MAT];
    if constexpr (NM > 0) mix_eos_r<NM>(s, f, mm, em, V, rho, pr, pf, cs, pfk);
    else eos(p.gamma, rho, e, pr, pf, cs);
    const double q = q_of_du(rho, cs, du, p.c1, p.c2);
    sig = 0.25 * (pf + q);
#pragma unroll
    for (int a = 0; a < NM; ++a) sg[a] = 0.25 * (pfk[a] + q);
    nu_u = hg_nu(p.hg, m, cs, Lsum);
    cq = visc_speed(cs, du, p.c1, p.c2);
}

// ============================================================================
// kl_state (Lagrange): z-march over cell planes [kc0, kc1) of the state in buffer
// `cur` (x, u, m, e).  Per column the x- and y-faces anchored there (centroid,
// face-average velocity, s) and the z-face of the next node plane, the x' edge
// lengths; per cell V (c.2), the EoS, the axis jumps (c.3 step 2), q, sigma, nu_u,
// and for owned cells the c.5 dt candidate with the DT-Q signal speed.  A 32 x NW
// tile yields 31 x (NW-1) cells.
// ============================================================================
template <int NW, int NM>
struct StateLagCTA {
    static constexpr int PL = NW * FW, TX = FW - 1, TY = NW - 1;
    __host__ __device__ static constexpr int oN(int par, int c) { return (par * 7 + c) * PL; }  // x(3) u(3) |u|^2
    static constexpr int OXB = 14 * PL;   // Xbar of the x-face (3), y-face (3)
    static constexpr int OUB = 20 * PL;   // Ubar of the x-face (3), y-face (3)
    static constexpr int OS = 26 * PL;    // s of the x-face, y-face
    static constexpr int OED = 28 * PL;   // edge^2 minima: x-edges (2 planes), y-edges, z-edge
    static constexpr int WORDS = 31 * PL + 2 * PAD;

    const Slab& s;
    const Phys& p;
    const int cur;
    double* me;
    int i, j, za, zb;
    long long nbc, cbc, cb;
    bool out_cell;
    D3 px, pu;
    double pm, pe;
    double pmf[NM > 0 ? NM : 1], pmm[NM > 0 ? NM : 1], pme[NM > 0 ? NM : 1];
    D3 zXb, zUb;          // z-face at node plane kz: centroid, face-average u
    double zs, zex, zey;  // its s and the x / y edges at (i, j) of that plane
    unsigned long long key;

    __device__ __forceinline__ StateLagCTA(const Slab& s_, const Phys& p_, int cur_, double* smem, int kc0, int kc1,
                                           int zchunk)
        : s(s_), p(p_), cur(cur_)
    {
        const int ix = threadIdx.x, iy = threadIdx.y;
        me = smem + PAD + iy * FW + ix;
        i = blockIdx.x * TX + ix;
        j = blockIdx.y * TY + iy;
        za = kc0 + zchunk_base(zchunk);
        zb = za + zchunk - 1 < kc1 - 1 ? za + zchunk - 1 : kc1 - 1;
        const int in = i < p.nx ? i : p.nx, jn = j < p.ny ? j : p.ny;
        const int ic = i < p.nx ? i : p.nx - 1, jc = j < p.ny ? j : p.ny - 1;
        nbc = (long long)in + (long long)(p.nx + 1) * (jn - (long long)(p.ny + 1) * s.kb);
        cbc = (long long)ic + (long long)p.nx * (jc - (long long)p.ny * s.kb);
        cb = (long long)i + (long long)p.nx * (j - (long long)p.ny * s.kb);
        out_cell = i < p.nx && j < p.ny && ix < TX && iy < TY;
        key = KEY_NONE;
    }
    __device__ __forceinline__ void fetch(int k)  // node plane k, cell plane k-1
    {
        const int kn = clampi(k, s.kb, s.kb + s.nzn - 1);
        const long long n = nbc + (long long)kn * s.pn;
        px = ld3(s.x[cur], n);
        pu = ld3(s.u[cur], n);
        const int kc = clampi(k - 1, s.kb, s.kb + s.nzc - 1);
        const long long c = cbc + (long long)kc * s.pc;
        pm = s.m[0][c];
        pe = s.e[cur][c];
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            pmf[a] = s.mf[0][c + a * mat_stride(s)];
            pmm[a] = s.mm[0][c + a * mat_stride(s)];
            pme[a] = s.me[cur][c + a * mat_stride(s)];
        }
    }
    template <int PAR>
    __device__ __forceinline__ void put()
    {
        st3s(me, oN(PAR, 0), PL, px);
        st3s(me, oN(PAR, 3), PL, pu);
        me[oN(PAR, 6)] = speed2(pu);
    }
    template <int PAR>
    __device__ __forceinline__ D3 X(int off) const { return ld3s(me + off, oN(PAR, 0), PL); }
    template <int PAR>
    __device__ __forceinline__ D3 U(int off) const { return ld3s(me + off, oN(PAR, 3), PL); }
    template <int PAR>
    __device__ __forceinline__ double V2(int off) const { return me[off + oN(PAR, 6)]; }
    // the z-face at this column of node plane B: (i,j) (i+1,j) (i+1,j+1) (i,j+1)
    template <int B>
    __device__ __forceinline__ void zface(D3& Xb, D3& Ub, double& sz, double& ex, double& ey) const
    {
        const D3 T0 = X<B>(0), T1 = X<B>(1), T2 = X<B>(FW + 1), T3 = X<B>(FW);
        Xb = avg4(T0, T1, T2, T3);
        sz = face_s(Xb, face_area(T0, T1, T2, T3));
        Ub = avg4(U<B>(0), U<B>(1), U<B>(FW + 1), U<B>(FW));
        ex = len2(T0, T1);
        ey = len2(T0, T3);
    }

    template <int B0>
    __device__ __forceinline__ void step(int kz)
    {
        constexpr int B1 = B0 ^ 1;
        put<B1>();
        const double m = pm, e = pe;
        double cmf[NM > 0 ? NM : 1], cmm[NM > 0 ? NM : 1], cme[NM > 0 ? NM : 1];
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            cmf[a] = pmf[a];
            cmm[a] = pmm[a];
            cme[a] = pme[a];
        }
        if (kz < zb) fetch(kz + 2);
        __syncthreads();
        // ---- the faces anchored at this column
        D3 zXbn, zUbn;
        double zsn, zexn, zeyn;
        zface<B1>(zXbn, zUbn, zsn, zexn, zeyn);
        {
            // x-face at node plane i: (i,j,kz) (i,j+1,kz) (i,j+1,kz+1) (i,j,kz+1)
            const D3 Q0 = X<B0>(0), Q1 = X<B0>(FW), Q2 = X<B1>(FW), Q3 = X<B1>(0);
            const D3 Xbx = avg4(Q0, Q1, Q2, Q3);
            me[OS] = face_s(Xbx, face_area(Q0, Q1, Q2, Q3));
            st3s(me, OXB, PL, Xbx);
            st3s(me, OUB, PL, avg4(U<B0>(0), U<B0>(FW), U<B1>(FW), U<B1>(0)));
            // y-face at node plane j: (i,j,kz) (i,j,kz+1) (i+1,j,kz+1) (i+1,j,kz)
            const D3 R2 = X<B1>(1), R3 = X<B0>(1);
            const D3 Xby = avg4(Q0, Q3, R2, R3);
            me[OS + PL] = face_s(Xby, face_area(Q0, Q3, R2, R3));
            st3s(me, OXB + 3 * PL, PL, Xby);
            st3s(me, OUB + 3 * PL, PL, avg4(U<B0>(0), U<B1>(0), U<B1>(1), U<B0>(1)));
            me[OED] = dmin(zex, zexn);        // x-edges (i,j) on planes kz, kz+1
            me[OED + PL] = dmin(zey, zeyn);   // y-edges
            me[OED + 2 * PL] = len2(Q0, Q3);  // z-edge (i,j): kz -> kz+1
        }
        double v2 = V2<B0>(0);  // max node speed^2 in corner order (before the barrier)
        v2 = dmax(v2, V2<B0>(1));
        v2 = dmax(v2, V2<B0>(FW));
        v2 = dmax(v2, V2<B0>(FW + 1));
        v2 = dmax(v2, V2<B1>(0));
        v2 = dmax(v2, V2<B1>(1));
        v2 = dmax(v2, V2<B1>(FW));
        v2 = dmax(v2, V2<B1>(FW + 1));
        __syncthreads();
        // ---- cell (i,j,kz)
        if (out_cell && kz >= 0 && kz < p.nz) {
            double sv[6] = {me[OS], me[1 + OS], me[OS + PL], me[FW + OS + PL], zs, zsn};
            const double V = vol_from_s(sv);
            double Lx, Ly, Lz;
            const double dx =
                axis_jump_L(ld3s(me, OXB, PL), ld3s(me + 1, OXB, PL), ld3s(me, OUB, PL), ld3s(me + 1, OUB, PL), Lx);
            const double dy = axis_jump_L(ld3s(me, OXB + 3 * PL, PL), ld3s(me + FW, OXB + 3 * PL, PL),
                                          ld3s(me, OUB + 3 * PL, PL), ld3s(me + FW, OUB + 3 * PL, PL), Ly);
            const double dz = axis_jump_L(zXb, zXbn, zUb, zUbn, Lz);
            const double du = dmin(dmin(dx, dy), dz);
            double sig, nu_u, cs, cq, sg[MAX_MAT];
            cell_state<NM>(s, p, m, e, cmf, cmm, cme, V, du, (Lx + Ly) + Lz, sig, nu_u, cs, cq, sg);
            const long long c = cb + (long long)kz * s.pc;
            s.sig[c] = sig;
            s.hnu[c] = nu_u;
#pragma unroll
            for (int a = 0; a < NM; ++a) s.sgm[c + a * mat_stride(s)] = sg[a];
            if (kz >= s.k0 && kz < s.k1) {
                double l2 = dmin(dmin(me[OED], me[FW + OED]), dmin(me[OED + PL], me[1 + OED + PL]));
                l2 = dmin(l2, dmin(dmin(me[OED + 2 * PL], me[1 + OED + 2 * PL]),
                                   dmin(me[FW + OED + 2 * PL], me[FW + 1 + OED + 2 * PL])));
                const unsigned long long kk = dt_key(dt_cell(p.cfl, l2, v2, cs, cq));
                key = kk < key ? kk : key;
            }
        }
        zXb = zXbn;
        zUb = zUbn;
        zs = zsn;
        zex = zexn;
        zey = zeyn;
        __syncthreads();
    }

    __device__ __forceinline__ void run()
    {
        fetch(za);
        if (za & 1) put<1>();
        else put<0>();
        fetch(za + 1);
        __syncthreads();
        if (za & 1) zface<1>(zXb, zUb, zs, zex, zey);
        else zface<0>(zXb, zUb, zs, zex, zey);
        for (int kz = za; kz <= zb; ++kz) {
            if (kz & 1) step<1>(kz);
            else step<0>(kz);
        }
        block_min_atomic(key, &s.st->cand_key);
    }
};

// gate = 0 for the first cycle of a sale_step call (DevState.active is still 0 there)
template <int NW, int NM>
__global__ void __launch_bounds__(FW * NW, SALE_MB_STATE) kl_state(Slab s, Phys p, int cur, int kc0, int kc1, int zchunk, int gate)
{
    if (gate && !s.st->active) return;
    extern __shared__ double smem[];
    StateLagCTA<NW, NM> c(s, p, cur, smem, kc0, kc1, zchunk);
    c.run();
}

// ============================================================================
// ke_state (Euler): z-march over cell planes [kc0, kc1) of the cycle-start state.
// Face-average velocities of the three faces anchored at a column, then the cell
// state and (owned cells) the dt candidate.  The target mesh is a tensor product
// of X_i, Y_j, Z_k, so every axis-jump separation d lies on its axis (checked at
// create, Phys::diag_jumps): w . d = w_a d_a exactly whenever it is non-zero, and a
// zero jump's sign never reaches q, cq or the state -- only the a-component of the
// face-average velocity on axis a is formed.  A 32 x NW tile yields 31 x (NW-1) cells.
// ============================================================================
template <int NW, int NM>
struct StateEulerCTA {
    static constexpr int PL = NW * FW, TX = FW - 1, TY = NW - 1;
    // node u in a ring of 3 slots filled by cp.async two planes ahead
    __host__ __device__ static constexpr int oU(int par, int c) { return (par * 3 + c) * PL; }  // node u
    __host__ __device__ static constexpr int oW(int xy) { return 9 * PL + xy * PL; }            // x/y face Ubar_a
    static constexpr int WORDS = 11 * PL + 2 * PAD;

    const Slab& s;
    const Phys& p;
    const int cur;
    double* me;
    int i, j, za, zb, ic, jc;
    long long nbn, cb, cbc;
    bool out_cell;
    double pm, pe, pv;
    double pmf[NM > 0 ? NM : 1], pmm[NM > 0 ? NM : 1], pme[NM > 0 ? NM : 1];
    double zprev;  // Ubar_z of the z-face at node plane kz (the -z face of cell kz)
    unsigned long long key;

    __device__ __forceinline__ StateEulerCTA(const Slab& s_, const Phys& p_, int cur_, double* smem, int kc0, int kc1,
                                             int zchunk)
        : s(s_), p(p_), cur(cur_)
    {
        const int ix = threadIdx.x, iy = threadIdx.y;
        me = smem + PAD + iy * FW + ix;
        i = blockIdx.x * TX + ix;
        j = blockIdx.y * TY + iy;
        ic = i < p.nx ? i : p.nx - 1;
        jc = j < p.ny ? j : p.ny - 1;
        za = kc0 + zchunk_base(zchunk);
        zb = imin(za + zchunk - 1, kc1 - 1);
        const int in = i < p.nx ? i : p.nx, jn = j < p.ny ? j : p.ny;
        nbn = (long long)in + (long long)(p.nx + 1) * (jn - (long long)(p.ny + 1) * s.kb);
        cb = (long long)i + (long long)p.nx * (j - (long long)p.ny * s.kb);
        cbc = (long long)ic + (long long)p.nx * (jc - (long long)p.ny * s.kb);
        out_cell = i < p.nx && j < p.ny && ix < TX && iy < TY;
        key = KEY_NONE;
    }
    __device__ __forceinline__ static int imin(int a, int b) { return a < b ? a : b; }
    // node plane k (u of this column, clamped always-valid address) into slot SL
    template <int SL>
    __device__ __forceinline__ void stage(int k)
    {
        const int kn = clampi(k, s.kb, s.kb + s.nzn - 1);
        cpa3(me + oU(SL, 0), PL, s.u[cur], nbn + (long long)kn * s.pn);
        cpa_commit();
    }
    __device__ __forceinline__ void fetch(int k)  // cell plane k-1 (m, e, V^T)
    {
        const int kc = clampi(k - 1, s.kb, s.kb + s.nzc - 1);
        const long long c = cbc + (long long)kc * s.pc;
        pm = s.m[cur][c];
        pe = s.e[cur][c];
        pv = s.VT[c];
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            pmf[a] = s.mf[cur][c + a * mat_stride(s)];
            pmm[a] = s.mm[cur][c + a * mat_stride(s)];
            pme[a] = s.me[cur][c + a * mat_stride(s)];
        }
    }
    template <int PAR>
    __device__ __forceinline__ D3 U(int off) const { return ld3s(me + off, oU(PAR, 0), PL); }

    // B0, B1, B2: the slots of node planes kz, kz+1, kz+2
    template <int B0, int B1, int B2>
    __device__ __forceinline__ void step(int kz)
    {
        cpa_wait_all();
        __syncthreads();  // node plane kz+1 landed; slot B2 (plane kz-1) free
        const double m = pm, e = pe, V = pv;
        double cmf[NM > 0 ? NM : 1], cmm[NM > 0 ? NM : 1], cme[NM > 0 ? NM : 1];
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            cmf[a] = pmf[a];
            cmm[a] = pmm[a];
            cme[a] = pme[a];
        }
        if (kz < zb) {
            stage<B2>(kz + 2);
            fetch(kz + 2);
        }
        // the a-component of the face-average velocity of the faces anchored here
        const double* Ux0 = me + oU(B0, 0);
        const double* Ux1 = me + oU(B1, 0);
        const double* Uy0 = me + oU(B0, 1);
        const double* Uy1 = me + oU(B1, 1);
        const double* Uz1 = me + oU(B1, 2);
        const double ux = 0.25 * (((Ux0[0] + Ux0[FW]) + Ux1[FW]) + Ux1[0]);  // x-face (i,j,k)(i,j+1,k)(i,j+1,k+1)(i,j,k+1)
        const double uy = 0.25 * (((Uy0[0] + Uy1[0]) + Uy1[1]) + Uy0[1]);    // y-face (i,j,k)(i,j,k+1)(i+1,j,k+1)(i+1,j,k)
        const double uz = 0.25 * (((Uz1[0] + Uz1[1]) + Uz1[FW + 1]) + Uz1[FW]);  // z-face at node plane k+1
        me[oW(0)] = ux;
        me[oW(1)] = uy;
        // max node speed^2 of the cell in corner order
        double v2 = speed2(U<B0>(0));
        v2 = dmax(v2, speed2(U<B0>(1)));
        v2 = dmax(v2, speed2(U<B0>(FW)));
        v2 = dmax(v2, speed2(U<B0>(FW + 1)));
        v2 = dmax(v2, speed2(U<B1>(0)));
        v2 = dmax(v2, speed2(U<B1>(1)));
        v2 = dmax(v2, speed2(U<B1>(FW)));
        v2 = dmax(v2, speed2(U<B1>(FW + 1)));
        const int kl = kz - s.kb;
        const double* TJx = s.TJx + 4 * ic;
        const double* TJy = s.TJy + 4 * jc;
        const double* TJz = s.TJz + 4 * kl;
        const double dxx = TJx[0], Lx = TJx[3], dyy = TJy[1], Ly = TJy[3], dzz = TJz[2], Lz = TJz[3];
        __syncthreads();
        if (out_cell && kz >= 0 && kz < p.nz) {
            const double dx = ddiv((me[1 + oW(0)] - ux) * dxx, Lx);
            const double dy = ddiv((me[FW + oW(1)] - uy) * dyy, Ly);
            const double dz = ddiv((uz - zprev) * dzz, Lz);
            const double du = dmin(dmin(dx, dy), dz);
            const double Lsum = (Lx + Ly) + Lz;
            double sig, nu_u, cs, cq, sg[MAX_MAT];
            cell_state<NM>(s, p, m, e, cmf, cmm, cme, V, du, Lsum, sig, nu_u, cs, cq, sg);
            const long long c = cb + (long long)kz * s.pc;
            s.sig[c] = sig;
            s.hnu[c] = nu_u;
#pragma unroll
            for (int a = 0; a < NM; ++a) s.sgm[c + a * mat_stride(s)] = sg[a];
            if (kz >= s.k0 && kz < s.k1) {
                // c.5 on the target mesh: cfl * sqrt(min edge^2) = the min of the per-axis
                // tabled factors (monotone maps: the same bits)
                const double num = dmin(dmin(s.TDx[ic], s.TDy[jc]), s.TDz[kl]);
                const unsigned long long kk = dt_key(dt_cell_num(num, v2, cs, cq));
                key = kk < key ? kk : key;
            }
        }
        zprev = uz;
    }

    __device__ __forceinline__ void run()
    {
        // slot of node plane k: (k - za) mod 3
        stage<0>(za);
        stage<1>(za + 1);
        fetch(za + 1);
        cpa_wait_all();
        __syncthreads();
        {
            const double* Uz = me + oU(0, 2);
            zprev = 0.25 * (((Uz[0] + Uz[1]) + Uz[FW + 1]) + Uz[FW]);
        }
        for (int kz = za; kz <= zb; ++kz) {
            switch ((kz - za) % 3) {
            case 0: step<0, 1, 2>(kz); break;
            case 1: step<1, 2, 0>(kz); break;
            default: step<2, 0, 1>(kz); break;
            }
        }
        block_min_atomic(key, &s.st->cand_key);
    }
};

// gate = 0 for the first cycle of a sale_step call (DevState.active is still 0 there)
template <int NW, int NM>
__global__ void __launch_bounds__(FW * NW, SALE_MB_STATE_E) ke_state(Slab s, Phys p, int cur, int kc0, int kc1, int zchunk, int gate)
{
    if (gate && !s.st->active) return;
    extern __shared__ double smem[];
    StateEulerCTA<NW, NM> c(s, p, cur, smem, kc0, kc1, zchunk);
    c.run();
}

// ============================================================================
// kc_force: node planes [kn0, kn1] in z-chunks.  Thread (ix, iy) owns column
// (i, j) = (bx*TX - 1 + ix, by*TY - 1 + iy): it stages nodes (i, j), computes
// the faces anchored there (Lagrange), cell (i, j) when ix <= FW-2, iy <= NW-2
// (it needs the +x / +y nodes), and node (i, j) when 1 <= ix <= FW-2, 1 <= iy <=
// NW-2 (it needs the -x / -y cells).
// ============================================================================
template <bool EULER, int NW>
struct ForceCTA {
    // XR: node rows staged beyond the NW thread rows (row NW, by the first warp row), so
    // every warp row computes cells (NW rows) and NW-1 rows gather nodes
    static constexpr int XR = SALE_FORCE_XROW;
    static constexpr int PL = NW * FW, PLN = (NW + XR) * FW, TX = FW - 2, TY = NW - 2 + XR;
    static constexpr int NNW = EULER ? 3 : 6;  // staged words per node: (x,) u
    // node planes in a ring of 3 slots filled by cp.async two planes ahead
    __host__ __device__ static constexpr int oN(int par, int c) { return (par * NNW + c) * PLN; }
    static constexpr int OT = 3 * NNW * PLN;                 // cell: corner forces t_h (24), m
    __host__ __device__ static constexpr int oT(int h, int c) { return OT + (h * 3 + c) * PL; }
    static constexpr int OM = OT + 24 * PL;
    static constexpr int WORDS = OM + PL + 2 * PAD;

    const Slab& s;
    const Phys& p;
    const int cur;
    double* me;
    int i, j, za, zb, ic, jc;
    long long nbc, cbc, nb, nbx;  // nbx: the extra staged row's node (i, j + NW), clamped
    double dt;
    bool node_thr, cell_thr, col_in, cellcol_in;
    bool pxm, pxp, pym, pyp;
    // prefetch registers (clamped, always-valid addresses)
    double psig, pnu, pm, pax, pay;
    double az;    // Euler: z-face area (x-y cross-section) of this column, constant in z
    D3 zprevA;    // Lagrange: A of the z-face at node plane kz
    D3 Fp;        // running node force of node plane kz+1 (cells of plane kz with c' = 0)
    double Mp;
    bool have;

    __device__ __forceinline__ ForceCTA(const Slab& s_, const Phys& p_, int cur_, double* smem, int kn0, int kn1,
                                        int zchunk)
        : s(s_), p(p_), cur(cur_)
    {
        const int ix = threadIdx.x, iy = threadIdx.y;
        me = smem + PAD + iy * FW + ix;
        i = blockIdx.x * TX - 1 + ix;
        j = blockIdx.y * TY - 1 + iy;
        za = kn0 + zchunk_base(zchunk);
        zb = za + zchunk - 1 < kn1 ? za + zchunk - 1 : kn1;
        const int in = clampi(i, 0, p.nx), jn = clampi(j, 0, p.ny);
        ic = clampi(i, 0, p.nx - 1);
        jc = clampi(j, 0, p.ny - 1);
        nbc = (long long)in + (long long)(p.nx + 1) * (jn - (long long)(p.ny + 1) * s.kb);
        cbc = (long long)ic + (long long)p.nx * (jc - (long long)p.ny * s.kb);
        nb = (long long)i + (long long)(p.nx + 1) * (j - (long long)(p.ny + 1) * s.kb);
        dt = s.st->dt;
        col_in = i >= 0 && i <= p.nx && j >= 0 && j <= p.ny;
        cellcol_in = i >= 0 && i < p.nx && j >= 0 && j < p.ny;
        node_thr = col_in && ix >= 1 && ix <= TX && iy >= 1 && iy <= TY;
        cell_thr = cellcol_in && ix <= FW - 2 && iy <= NW - 2 + XR;
        {
            const int jx = clampi(j + NW, 0, p.ny);
            nbx = (long long)in + (long long)(p.nx + 1) * (jx - (long long)(p.ny + 1) * s.kb);
        }
        pxm = i >= 1;    // cell i-1 exists (for a node column inside the mesh)
        pxp = i < p.nx;  // cell i exists
        pym = j >= 1;
        pyp = j < p.ny;
        if (EULER) az = s.TAz[2][(long long)jc * p.nx + ic];
    }

    // node plane k (x, u of this column, clamped always-valid addresses) into slot SL by
    // cp.async
    template <int SL>
    __device__ __forceinline__ void stage(int k)
    {
        const int kn = clampi(k, s.kb, s.kb + s.nzn - 1);
        const long long n = nbc + (long long)kn * s.pn;
        if (!EULER) cpa3(me + oN(SL, 0), PLN, s.x[cur], n);
        cpa3(me + oN(SL, EULER ? 0 : 3), PLN, s.u[cur], n);
        if (XR && threadIdx.y == 0) {
            const long long nx_ = nbx + (long long)kn * s.pn;
            if (!EULER) cpa3(me + NW * FW + oN(SL, 0), PLN, s.x[cur], nx_);
            cpa3(me + NW * FW + oN(SL, EULER ? 0 : 3), PLN, s.u[cur], nx_);
        }
        cpa_commit();
    }
    // cell plane k-1 (sigma, nu_u, m; Euler: table areas) into registers
    __device__ __forceinline__ void fetch(int k)
    {
        const int kc = clampi(k - 1, s.kb, s.kb + s.nzc - 1);
        const long long c = cbc + (long long)kc * s.pc;
        psig = s.sig[c];
        pnu = s.hnu[c];
        pm = mass_cur(s, p, cur)[c];
        if (EULER) {
            const int kl = kc - s.kb;
            pax = s.TAx[0][(long long)kl * p.ny + jc];
            pay = s.TAy[1][(long long)kl * p.nx + ic];
        }
    }
    template <int PAR>
    __device__ __forceinline__ D3 X(int off) const { return ld3s(me + off, oN(PAR, 0), PLN); }
    template <int PAR>
    __device__ __forceinline__ D3 U(int off) const { return ld3s(me + off, oN(PAR, EULER ? 0 : 3), PLN); }
    template <int PAR>
    __device__ __forceinline__ D3 zface() const
    {
        return face_area(X<PAR>(0), X<PAR>(1), X<PAR>(FW + 1), X<PAR>(FW));
    }

    // corner force of cell (offset dx, dy in the tile) at corner H
    template <int H>
    __device__ __forceinline__ D3 T(int off) const { return ld3s(me + off, oT(H, 0), PL); }

    // accumulate the four cells of the staged plane at corners c = CZ (H = a + 2b + 4 CZ
    // with a = 1 - a', b = 1 - b'), in gather order a' fastest, from the running sums
    template <int CZ>
    __device__ __forceinline__ void gather4(D3& F, double& M, bool& hv, bool pz) const
    {
        if (pz && pxm && pxp && pym && pyp) {  // all four present (interior): no selects
            const D3 t0 = T<3 + 4 * CZ>(-1 - FW), t1 = T<2 + 4 * CZ>(-FW), t2 = T<1 + 4 * CZ>(-1), t3 = T<0 + 4 * CZ>(0);
            const double m0 = me[-1 - FW + OM], m1 = me[-FW + OM], m2 = me[-1 + OM], m3 = me[OM];
            if (hv) {
                F = add(add(add(add(F, t0), t1), t2), t3);
                M = (((M + m0) + m1) + m2) + m3;
            } else {
                F = add(add(add(t0, t1), t2), t3);
                M = ((m0 + m1) + m2) + m3;
            }
            hv = true;
            return;
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const int ap = g & 1, bp = g >> 1;
            const int off = (ap ? 0 : -1) + (bp ? 0 : -FW);
            const bool pres = pz && (ap ? pxp : pxm) && (bp ? pyp : pym);
            D3 t;
            switch (g) {  // H = (1-ap) + 2(1-bp) + 4 CZ
            case 0: t = T<3 + 4 * CZ>(off); break;
            case 1: t = T<2 + 4 * CZ>(off); break;
            case 2: t = T<1 + 4 * CZ>(off); break;
            default: t = T<0 + 4 * CZ>(off); break;
            }
            const double mk = me[off + OM];
            if (pres) {
                F = hv ? add(F, t) : t;
                M = hv ? M + mk : mk;
                hv = true;
            }
        }
    }

    // B0, B1, B2: the slots of node planes kz, kz+1, kz+2
    template <int B0, int B1, int B2>
    __device__ __forceinline__ void step(int kz)
    {
        // ---- P1: node plane kz+1 landed (its copies were issued a step ago); the cell
        // operands of plane kz; node plane kz+2 into the slot plane kz-1 left
        cpa_wait_all();
        __syncthreads();
        const double sig = psig, nu_u = pnu, m = pm, ax = pax, ay = pay;
        if (kz < zb) {
            stage<B2>(kz + 2);
            fetch(kz + 2);
        }
        // ---- P2 (Lagrange): the z-face area of node plane kz+1 at this column (t^n);
        // the cell's x- and y-faces are formed in P3 by the thread itself (its own and
        // the +x / +y neighbours' anchored faces: two faces computed twice instead of a
        // barrier and a shared-memory round trip)
        D3 Azn;
        if constexpr (!EULER) Azn = zface<B1>();
        // ---- P3: cell (i,j,kz): hourglass modes, the eight corner forces
        if (cell_thr && kz >= 0 && kz < p.nz) {
            D3 g[4];
            {
                const D3 Uc[8] = {U<B0>(0), U<B0>(1), U<B0>(FW), U<B0>(FW + 1),
                                  U<B1>(0), U<B1>(1), U<B1>(FW), U<B1>(FW + 1)};
                hg_modes(Uc, g);
            }
            const double nu = hg_cap(nu_u, m, dt);
            if constexpr (EULER) {
                // axis-aligned target areas (Phys::diag_areas): the corner vector of corner
                // (a,b,c) is exactly (+-ax, +-ay, +-az), and sigma (-a) = -(sigma a)
                const double sa = sig * ax, sb = sig * ay, sc = sig * az;
#define SALE_TE(H)                                                                                  \
    {                                                                                               \
        const D3 f = hg_corner<H>(g, nu);                                                           \
        st3s(me, oT(H, 0), PL,                                                                      \
             D3{((H)&1 ? sa : -sa) + f.x, ((H)&2 ? sb : -sb) + f.y, ((H)&4 ? sc : -sc) + f.z});     \
    }
                SALE_TE(0) SALE_TE(1) SALE_TE(2) SALE_TE(3) SALE_TE(4) SALE_TE(5) SALE_TE(6) SALE_TE(7)
#undef SALE_TE
            } else {
                // x-faces at node planes i, i+1: (i,j,kz) (i,j+1,kz) (i,j+1,kz+1) (i,j,kz+1);
                // y-faces at node planes j, j+1: (i,j,kz) (i,j,kz+1) (i+1,j,kz+1) (i+1,j,kz)
                const D3 A[6] = {face_area(X<B0>(0), X<B0>(FW), X<B1>(FW), X<B1>(0)),
                                 face_area(X<B0>(1), X<B0>(FW + 1), X<B1>(FW + 1), X<B1>(1)),
                                 face_area(X<B0>(0), X<B1>(0), X<B1>(1), X<B0>(1)),
                                 face_area(X<B0>(FW), X<B1>(FW), X<B1>(FW + 1), X<B0>(FW + 1)), zprevA, Azn};
#define SALE_TL(H)                                                                                  \
    {                                                                                               \
        const D3 C = corner_vec(A, (H)&1, ((H) >> 1) & 1, (H) >> 2);                                \
        const D3 f = hg_corner<H>(g, nu);                                                           \
        st3s(me, oT(H, 0), PL, D3{(sig * C.x) + f.x, (sig * C.y) + f.y, (sig * C.z) + f.z});      \
    }
                SALE_TL(0) SALE_TL(1) SALE_TL(2) SALE_TL(3) SALE_TL(4) SALE_TL(5) SALE_TL(6) SALE_TL(7)
#undef SALE_TL
            }
            me[OM] = m;
        }
        if constexpr (!EULER) zprevA = Azn;
        __syncthreads();
        // ---- P4: node (i,j,kz) from the running sums and cell plane kz; then start
        // node plane kz+1 from cell plane kz
        if (node_thr) {
            const bool pz = kz >= 0 && kz < p.nz;  // cell plane kz exists
            if (kz >= za) {
                D3 F = Fp;
                double M = Mp;
                bool hv = have;
                gather4<0>(F, M, hv, pz);
                M = 0.125 * M;
                const D3 u = U<B0>(0);
                D3 un = d3(u.x + (ddiv(F.x, M) * dt), u.y + (ddiv(F.y, M) * dt), u.z + (ddiv(F.z, M) * dt));
                un = reflect(p, i, j, kz, un);
                const long long n = nb + (long long)kz * s.pn;
                if constexpr (EULER) {
                    st3(s.u1, n, un);
                } else {
                    const D3 x = X<B0>(0);
                    const D3 xn = d3(x.x + (un.x * dt), x.y + (un.y * dt), x.z + (un.z * dt));
                    st3(s.x[cur ^ 1], n, xn);
                    st3(s.u[cur ^ 1], n, un);
                    if (s.hp) {  // peer-store halo: the neighbours' ghost node planes
                        const long long q = (long long)i + (long long)(p.nx + 1) * j;
                        halo_node3(s, s.hp->x, cur ^ 1, kz, q, xn);
                        halo_node3(s, s.hp->u, cur ^ 1, kz, q, un);
                    }
                }
            }
            have = false;
            Fp = D3{0.0, 0.0, 0.0};
            Mp = 0.0;
            if (kz < zb) gather4<1>(Fp, Mp, have, pz);
        }
    }

    __device__ __forceinline__ void run()
    {
        // prologue: node planes za-1 (and its z-face) and za, the operands of cell plane
        // za-1; slot of node plane k: (k - za + 1) mod 3
        stage<0>(za - 1);
        stage<1>(za);
        fetch(za);
        have = false;
        Fp = D3{0.0, 0.0, 0.0};
        Mp = 0.0;
        cpa_wait_all();
        __syncthreads();
        if constexpr (!EULER) zprevA = zface<0>();
        for (int kz = za - 1; kz <= zb; ++kz) {
            switch ((kz - za + 1) % 3) {
            case 0: step<0, 1, 2>(kz); break;
            case 1: step<1, 2, 0>(kz); break;
            default: step<2, 0, 1>(kz); break;
            }
        }
    }
};

template <bool EULER, int NW>
__global__ void __launch_bounds__(FW * NW, EULER ? SALE_MB_FORCE_E : SALE_MB_FORCE) kc_force(Slab s, Phys p, int cur, int kn0, int kn1, int zchunk)
{
    if (!s.st->active) return;
    extern __shared__ double smem[];
    ForceCTA<EULER, NW> c(s, p, cur, smem, kn0, kn1, zchunk);
    c.run();
}

// ============================================================================
// kc_energy: cell planes [kc0, kc1) in z-chunks; thread (ix, iy) owns column
// (i, j) = (bx*TX + ix, by*TY + iy) and its cell when ix < FW-1, iy < NW-1.
//   Lagrange: stages x^n, x', u^n, u'; per column the t^n face areas and the moved
//   faces' s'; per cell W, the hourglass work, e', V' and the tangle check.
//   Euler: stages x' (formed from u'), u^n and ubar; areas from the tables; also
//   writes V' and the moved-face s' the sweep reads.
// ============================================================================
template <bool EULER, int NW, int NM>
struct EnergyCTA {
    static constexpr int PL = NW * FW, TX = FW - 1, TY = NW - 1;
    // node words: Lagrange x^n(3) x'(3) u^n(3) u'(3) (u' replaced by ubar once landed);
    // Euler x'(3) u^n(3) ubar(3)
    static constexpr int NNW = EULER ? 9 : 12;
    // node-plane slots: Euler 2 (register prefetch, staged one plane ahead: x' and ubar
    // are formed when staged); Lagrange a ring of 3 filled by cp.async two planes ahead
    // (the raw x^n, x', u^n, u' never pass through registers)
    static constexpr int NSL = EULER ? 2 : 3;
    __host__ __device__ static constexpr int oN(int par, int c) { return (par * NNW + c) * PL; }
    static constexpr int OS = NSL * NNW * PL;  // s' of the x-face, y-face
    static constexpr int OAN = OS + 2 * PL;   // Lagrange: A^n of the x-face (3), y-face (3)
    static constexpr int WORDS = OAN + (EULER ? 0 : 6) * PL + 2 * PAD;

    const Slab& s;
    const Phys& p;
    const int cur;
    double* me;
    int i, j, za, zb, ic, jc;
    long long nbc, cbc, nb, cb;
    double dt;
    bool col_in, cell_thr, own_col;
    // prefetch registers
    D3 fx, fx1, fu, fu1;
    double fm, fe, fsig, fnu, fz, fax, fay;
    double rf[NM > 0 ? NM : 1], rm[NM > 0 ? NM : 1], re[NM > 0 ? NM : 1], rs[NM > 0 ? NM : 1];
    double xcol, ycol, az;
    // carried z-face of node plane kz: t^n area (Lagrange), s' of the moved face
    D3 zA;
    double zs;

    __device__ __forceinline__ EnergyCTA(const Slab& s_, const Phys& p_, int cur_, double* smem, int kc0, int kc1,
                                         int zchunk)
        : s(s_), p(p_), cur(cur_)
    {
        const int ix = threadIdx.x, iy = threadIdx.y;
        me = smem + PAD + iy * FW + ix;
        i = blockIdx.x * TX + ix;
        j = blockIdx.y * TY + iy;
        za = kc0 + zchunk_base(zchunk);
        zb = za + zchunk - 1 < kc1 - 1 ? za + zchunk - 1 : kc1 - 1;
        const int in = i < p.nx ? i : p.nx, jn = j < p.ny ? j : p.ny;
        ic = i < p.nx ? i : p.nx - 1;
        jc = j < p.ny ? j : p.ny - 1;
        nbc = (long long)in + (long long)(p.nx + 1) * (jn - (long long)(p.ny + 1) * s.kb);
        cbc = (long long)ic + (long long)p.nx * (jc - (long long)p.ny * s.kb);
        nb = (long long)i + (long long)(p.nx + 1) * (j - (long long)(p.ny + 1) * s.kb);
        cb = (long long)i + (long long)p.nx * (j - (long long)p.ny * s.kb);
        dt = s.st->dt;
        col_in = i <= p.nx && j <= p.ny;
        cell_thr = i < p.nx && j < p.ny && ix < TX && iy < TY;
        own_col = col_in && ix < TX && iy < TY;
        if (EULER) {
            xcol = s.Xt[in];
            ycol = s.Yt[jn];
            az = s.TAz[2][(long long)jc * p.nx + ic];
        }
    }

    // Lagrange: cp.async of node plane k (x^n, x', u^n, u' of this column, clamped
    // always-valid addresses) into slot SL
    template <int SL>
    __device__ __forceinline__ void stage(int k)
    {
        const int kn = clampi(k, s.kb, s.kb + s.nzn - 1);
        const long long n = nbc + (long long)kn * s.pn;
        cpa3(me + oN(SL, 0), PL, s.x[cur], n);
        cpa3(me + oN(SL, 3), PL, s.x[cur ^ 1], n);
        cpa3(me + oN(SL, 6), PL, s.u[cur], n);
        cpa3(me + oN(SL, 9), PL, s.u[cur ^ 1], n);
        cpa_commit();
    }
    __device__ __forceinline__ void fetch(int k)  // node plane k (Euler), cell plane k-1
    {
        const int kn = clampi(k, s.kb, s.kb + s.nzn - 1);
        const long long n = nbc + (long long)kn * s.pn;
        if constexpr (EULER) {
            fu = ld3(s.u[cur], n);
            fu1 = ld3(s.u1, n);
            fz = s.Zt[kn - s.kb];
        }
        const int kc = clampi(k - 1, s.kb, s.kb + s.nzc - 1);
        const long long c = cbc + (long long)kc * s.pc;
        fm = mass_cur(s, p, cur)[c];
        fe = s.e[cur][c];
        fsig = s.sig[c];
        fnu = s.hnu[c];
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            const long long ca = c + a * mat_stride(s);
            rf[a] = mat_f(s, p, cur)[ca];
            rm[a] = mat_m(s, p, cur)[ca];
            re[a] = s.me[cur][ca];
            rs[a] = s.sgm[ca];
        }
        if (EULER) {
            const int kl = kc - s.kb;
            fax = s.TAx[0][(long long)kl * p.ny + jc];
            fay = s.TAy[1][(long long)kl * p.nx + ic];
        }
    }
    template <int PAR>
    __device__ __forceinline__ void put()
    {
        if constexpr (EULER) {
            // x' = x^T + u' dt (kc_force's expression, c.3 step 6), formed when staged
            st3s(me, oN(PAR, 0), PL, D3{xcol + (fu1.x * dt), ycol + (fu1.y * dt), fz + (fu1.z * dt)});
            st3s(me, oN(PAR, 3), PL, fu);
            st3s(me, oN(PAR, 6), PL, scl(0.5, add(fu, fu1)));
        } else {
            st3s(me, oN(PAR, 0), PL, fx);
            st3s(me, oN(PAR, 3), PL, fx1);
            st3s(me, oN(PAR, 6), PL, fu);
            st3s(me, oN(PAR, 9), PL, fu1);
        }
    }
    template <int PAR>
    __device__ __forceinline__ D3 Xn(int off) const { return ld3s(me + off, oN(PAR, 0), PL); }
    template <int PAR>
    __device__ __forceinline__ D3 X1(int off) const { return ld3s(me + off, oN(PAR, EULER ? 0 : 3), PL); }
    template <int PAR>
    __device__ __forceinline__ D3 Un(int off) const { return ld3s(me + off, oN(PAR, EULER ? 3 : 6), PL); }
    template <int PAR>
    __device__ __forceinline__ D3 Ub(int off) const  // ubar = 0.5 (u + u')
    {
        return ld3s(me + off, oN(PAR, EULER ? 6 : 9), PL);
    }
    // Lagrange: once node plane PAR has landed, the column's own thread replaces u' by
    // ubar = 0.5 (u + u') (the only use of u' here), once per node instead of once per
    // cell corner
    template <int PAR>
    __device__ __forceinline__ void put_ubar()
    {
        st3s(me, oN(PAR, 9), PL, scl(0.5, add(Un<PAR>(0), ld3s(me, oN(PAR, 9), PL))));
    }

    // the z-face at this column of node plane B: s' of the moved face, t^n area (Lagrange)
    template <int B>
    __device__ __forceinline__ void zstate(D3& A, double& sz) const
    {
        const D3 T0 = X1<B>(0), T1 = X1<B>(1), T2 = X1<B>(FW + 1), T3 = X1<B>(FW);
        sz = face_s(avg4(T0, T1, T2, T3), face_area(T0, T1, T2, T3));
        if constexpr (!EULER) A = face_area(Xn<B>(0), Xn<B>(1), Xn<B>(FW + 1), Xn<B>(FW));
    }

    // B0, B1: the slots of node planes kz, kz+1; B2 (Lagrange): the slot plane kz+2 goes to
    template <int B0, int B1, int B2>
    __device__ __forceinline__ void step(int kz)
    {
        // ---- P1: stage node plane kz+1 (Lagrange: wait for its copies); this cell's
        // operands; prefetch
        if constexpr (EULER) {
            put<B1>();
        } else {
            cpa_wait_all();
            __syncthreads();  // plane kz+1 visible; slot B2 (plane kz-1) free
            put_ubar<B1>();   // read by the cells after the P2 / P3 barrier
        }
        const double m = fm, e = fe, sig = fsig, nu_u = fnu, ax = fax, ay = fay;
        double cf[NM > 0 ? NM : 1], cm[NM > 0 ? NM : 1], ce[NM > 0 ? NM : 1], cs_[NM > 0 ? NM : 1];
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            cf[a] = rf[a];
            cm[a] = rm[a];
            ce[a] = re[a];
            cs_[a] = rs[a];
        }
        if (kz < zb) {
            if constexpr (!EULER) stage<B2>(kz + 2);
            fetch(kz + 2);
        }
        if constexpr (EULER) __syncthreads();
        // ---- P2: faces anchored at this column
        D3 zAn;
        double zsn;
        zstate<B1>(zAn, zsn);
        {
            // moved x-face at node plane i: (i,j,kz) (i,j+1,kz) (i,j+1,kz+1) (i,j,kz+1)
            const D3 Q0 = X1<B0>(0), Q1 = X1<B0>(FW), Q2 = X1<B1>(FW), Q3 = X1<B1>(0);
            me[OS] = face_s(avg4(Q0, Q1, Q2, Q3), face_area(Q0, Q1, Q2, Q3));
            // moved y-face at node plane j: (i,j,kz) (i,j,kz+1) (i+1,j,kz+1) (i+1,j,kz)
            const D3 R2 = X1<B1>(1), R3 = X1<B0>(1);
            me[OS + PL] = face_s(avg4(Q0, Q3, R2, R3), face_area(Q0, Q3, R2, R3));
            if constexpr (!EULER) {
                st3s(me, OAN, PL, face_area(Xn<B0>(0), Xn<B0>(FW), Xn<B1>(FW), Xn<B1>(0)));
                st3s(me, OAN + 3 * PL, PL, face_area(Xn<B0>(0), Xn<B1>(0), Xn<B1>(1), Xn<B0>(1)));
            } else if (own_col) {
                // s' of the faces anchored at node (i,j,kz), for the sweep's swept volumes
                const long long n = nb + (long long)kz * s.pn;
                s.sF[0][n] = me[OS];
                s.sF[1][n] = me[OS + PL];
                s.sF[2][n] = zs;
            }
        }
        __syncthreads();
        // ---- P3: cell (i,j,kz)
        if (cell_thr && kz >= 0 && kz < p.nz) {
            const long long cc = cb + (long long)kz * s.pc;
            double sv[6] = {me[OS], me[1 + OS], me[OS + PL], me[FW + OS + PL], zs, zsn};
            const double V1 = vol_from_s(sv);
            if (kz >= s.k0 && kz < s.k1 && !(V1 > 0.0))
                atomicMin(&s.st->err_key, (ERR_ORDER_TANGLED << 48) | (unsigned long long)gcell(p, i, j, kz));
            double W = 0.0, Wh = 0.0;
            if constexpr (EULER) {
            // hourglass modes of u^n and the capped coefficient
            D3 g[4];
            {
                const D3 Uc[8] = {Un<B0>(0), Un<B0>(1), Un<B0>(FW), Un<B0>(FW + 1),
                                  Un<B1>(0), Un<B1>(1), Un<B1>(FW), Un<B1>(FW + 1)};
                hg_modes(Uc, g);
            }
            const double nu = hg_cap(nu_u, m, dt);
            // W = sum_h C_h . ubar_h and W_hg = sum_h f_h . ubar_h in corner order
            {
                D3 A[6];
                if constexpr (!EULER)
                    A[0] = ld3s(me, OAN, PL), A[1] = ld3s(me + 1, OAN, PL), A[2] = ld3s(me, OAN + 3 * PL, PL),
                    A[3] = ld3s(me + FW, OAN + 3 * PL, PL), A[4] = zA, A[5] = zAn;
#define SALE_WH(H)                                                                                 \
    {                                                                                              \
        constexpr int a = (H)&1, b = ((H) >> 1) & 1, c = (H) >> 2;                                  \
        const D3 ub = c ? Ub<B1>(a + b * FW) : Ub<B0>(a + b * FW);                                 \
        D3 C;                                                                                      \
        if constexpr (EULER) C = D3{a ? ax : -ax, b ? ay : -ay, c ? az : -az};                    \
        else C = corner_vec(A, a, b, c);                                                           \
        const double tw = dot(C, ub);                                                              \
        const double th = dot(hg_corner<H>(g, nu), ub);                                            \
        W = (H) == 0 ? tw : W + tw;                                                                \
        Wh = (H) == 0 ? th : Wh + th;                                                              \
    }
                SALE_WH(0) SALE_WH(1) SALE_WH(2) SALE_WH(3) SALE_WH(4) SALE_WH(5) SALE_WH(6) SALE_WH(7)
#undef SALE_WH
            }
            } else {  // Lagrange: W first, then the modes (the face areas and the modes are
                      // never live together: 2 CTAs per SM fit with a smaller spill)
            // W = sum_h C_h . ubar_h in corner order (the face areas live only here) ...
            {
                D3 A[6];
                if constexpr (!EULER)
                    A[0] = ld3s(me, OAN, PL), A[1] = ld3s(me + 1, OAN, PL), A[2] = ld3s(me, OAN + 3 * PL, PL),
                    A[3] = ld3s(me + FW, OAN + 3 * PL, PL), A[4] = zA, A[5] = zAn;
#define SALE_W(H)                                                                                  \
    {                                                                                              \
        constexpr int a = (H)&1, b = ((H) >> 1) & 1, c = (H) >> 2;                                  \
        const D3 ub = c ? Ub<B1>(a + b * FW) : Ub<B0>(a + b * FW);                                 \
        D3 C;                                                                                      \
        if constexpr (EULER) C = D3{a ? ax : -ax, b ? ay : -ay, c ? az : -az};                    \
        else C = corner_vec(A, a, b, c);                                                           \
        const double tw = dot(C, ub);                                                              \
        W = (H) == 0 ? tw : W + tw;                                                                \
    }
                SALE_W(0) SALE_W(1) SALE_W(2) SALE_W(3) SALE_W(4) SALE_W(5) SALE_W(6) SALE_W(7)
#undef SALE_W
            }
            // ... then the hourglass modes of u^n, the capped coefficient and W_hg =
            // sum_h f_h . ubar_h (the modes live only here: fewer registers at the peak)
            {
                D3 g[4];
                {
                    const D3 Uc[8] = {Un<B0>(0), Un<B0>(1), Un<B0>(FW), Un<B0>(FW + 1),
                                      Un<B1>(0), Un<B1>(1), Un<B1>(FW), Un<B1>(FW + 1)};
                    hg_modes(Uc, g);
                }
                const double nu = hg_cap(nu_u, m, dt);
#define SALE_WHG(H)                                                                                \
    {                                                                                              \
        constexpr int a = (H)&1, b = ((H) >> 1) & 1, c = (H) >> 2;                                  \
        const D3 ub = c ? Ub<B1>(a + b * FW) : Ub<B0>(a + b * FW);                                 \
        const double th = dot(hg_corner<H>(g, nu), ub);                                            \
        Wh = (H) == 0 ? th : Wh + th;                                                              \
    }
                SALE_WHG(0) SALE_WHG(1) SALE_WHG(2) SALE_WHG(3) SALE_WHG(4) SALE_WHG(5) SALE_WHG(6) SALE_WHG(7)
#undef SALE_WHG
            }
            }
            // compatible energy with the hourglass work (HG); materials: MM4 share + HG heat
            if constexpr (NM > 0) {
#pragma unroll
                for (int a = 0; a < NM; ++a) {
                    const double e1k = (cf[a] > 0.0 && cm[a] > 0.0)
                                           ? ce[a] - ddiv((((cs_[a] * W) + Wh) * dt) * cf[a], cm[a])
                                           : ce[a];
                    if (EULER) {
                        s.e1m[cc + a * mat_stride(s)] = e1k;
                    } else {
                        s.me[cur ^ 1][cc + a * mat_stride(s)] = e1k;
                        if (s.hp) halo_cell(s, s.hp->me, cur ^ 1, a, kz, (long long)i + (long long)p.nx * j, e1k);
                    }
                }
            } else {
                const double e1 = e - ddiv(((sig * W) + Wh) * dt, m);
                if (EULER) {
                    s.e1[cc] = e1;
                } else {
                    s.e[cur ^ 1][cc] = e1;
                    if (s.hp) halo_cell(s, s.hp->e, cur ^ 1, 0, kz, (long long)i + (long long)p.nx * j, e1);
                }
            }
            if (EULER) s.V1[cc] = V1;
        }
        zA = zAn;
        zs = zsn;
        if constexpr (EULER) __syncthreads();
    }

    __device__ __forceinline__ void run()
    {
        if constexpr (EULER) {
            fetch(za);
            if (za & 1) put<1>();
            else put<0>();
            fetch(za + 1);
            __syncthreads();
            if (za & 1) zstate<1>(zA, zs);
            else zstate<0>(zA, zs);
            for (int kz = za; kz <= zb; ++kz) {
                if (kz & 1) step<1, 0, 0>(kz);
                else step<0, 1, 0>(kz);
            }
        } else {
            // slot of node plane k: (k - za) mod 3
            stage<0>(za);
            stage<1>(za + 1);
            fetch(za + 1);
            cpa_wait_all();
            __syncthreads();
            put_ubar<0>();
            zstate<0>(zA, zs);
            for (int kz = za; kz <= zb; ++kz) {
                switch ((kz - za) % 3) {
                case 0: step<0, 1, 2>(kz); break;
                case 1: step<1, 2, 0>(kz); break;
                default: step<2, 0, 1>(kz); break;
                }
            }
        }
    }
};

#ifndef SALE_MB_ENERGY_L_MAT  // Lagrange with >= SALE_NM_ENERGY_L_MAT materials: one CTA per SM
#define SALE_MB_ENERGY_L_MAT 1    // (their operands spill at two: C3 4 materials 9.47 -> 8.64 ms)
#endif
#ifndef SALE_NM_ENERGY_L_MAT
#define SALE_NM_ENERGY_L_MAT 3
#endif
template <bool EULER, int NW, int NM>
__global__ void __launch_bounds__(FW * NW, EULER ? SALE_MB_ENERGY_E : (NM >= SALE_NM_ENERGY_L_MAT ? SALE_MB_ENERGY_L_MAT : SALE_MB_ENERGY_L)) kc_energy(Slab s, Phys p, int cur, int kc0, int kc1, int zchunk)
{
    if (!s.st->active) return;
    extern __shared__ double smem[];
    EnergyCTA<EULER, NW, NM> c(s, p, cur, smem, kc0, kc1, zchunk);
    c.run();
}

// ============================================================================
// launchers
// ============================================================================
namespace {
// warp rows per CTA (compile-time tuning knobs; scripts/build_probe.sh -D... for A/B runs)
#ifndef SALE_NW_STATE
#define SALE_NW_STATE 8
#endif
#ifndef SALE_NW_FORCE
#define SALE_NW_FORCE 8
#endif
#ifndef SALE_NW_ENERGY
#define SALE_NW_ENERGY 8
#endif
constexpr int NW_STATE = SALE_NW_STATE, NW_FORCE = SALE_NW_FORCE, NW_ENERGY = SALE_NW_ENERGY;

// Euler: node planes the Lagrangian phase updates (owned + the ghost region the remap
// reads), and the cell planes whose state the force gather needs
inline void euler_ranges(const Slab& s, const Phys& p, int& kn0, int& kn1)
{
    kn0 = imax_h(s.k0 - 2, 0);
    kn1 = imin_h(s.k1 + 2, p.nz);
}
}  // namespace

int launch_state(const Slab& s, const Phys& p, int cur, int gate, Stream st)
{
    int kc0, kc1;
    if (p.rezone) {
        int kn0, kn1;
        euler_ranges(s, p, kn0, kn1);
        kc0 = imax_h(kn0 - 1, 0);
        kc1 = imin_h(kn1 + 1, p.nz);
    } else {  // the cells around the owned node planes [k0, k1]
        kc0 = imax_h(s.k0 - 1, 0);
        kc1 = imin_h(s.k1 + 1, p.nz);
    }
    by_nmat(s.nmat, [&](auto nm) {
        constexpr int NM = decltype(nm)::value;
        auto go = [&](auto kern, size_t words) {
            const size_t sm = sizeof(double) * words;
            set_smem(kern, sm);
            const long long xy = (long long)cdiv(p.nx, FW - 1) * cdiv(p.ny, NW_STATE - 1);
            const int zc = zchunk_for(xy, kc1 - kc0, ZCHUNK);
            dim3 grid(cdiv(p.nx, FW - 1), cdiv(p.ny, NW_STATE - 1), cdiv(kc1 - kc0, zc));
            kern<<<grid, dim3(FW, NW_STATE), sm, (cudaStream_t)st>>>(s, p, cur, kc0, kc1, zorder(zc), gate);
            note_launch();
        };
        if (p.rezone) go(ke_state<NW_STATE, NM>, StateEulerCTA<NW_STATE, NM>::WORDS);
        else go(kl_state<NW_STATE, NM>, StateLagCTA<NW_STATE, NM>::WORDS);
    });
    return 1;
}

int launch_force(const Slab& s, const Phys& p, int cur, Stream st)
{
    int kn0 = s.k0, kn1 = s.k1;
    if (p.rezone) euler_ranges(s, p, kn0, kn1);
    auto go = [&](auto kern, size_t words) {
        const size_t sm = sizeof(double) * words;
        set_smem(kern, sm);
        constexpr int TY = NW_FORCE - 2 + SALE_FORCE_XROW;
        const long long xy = (long long)cdiv(p.nx + 1, FW - 2) * cdiv(p.ny + 1, TY);
        const int zc = zchunk_for(xy, kn1 - kn0 + 1, ZCHUNK);
        dim3 grid(cdiv(p.nx + 1, FW - 2), cdiv(p.ny + 1, TY), cdiv(kn1 - kn0 + 1, zc));
        kern<<<grid, dim3(FW, NW_FORCE), sm, (cudaStream_t)st>>>(s, p, cur, kn0, kn1, zorder(zc));
        note_launch();
    };
    if (p.rezone) go(kc_force<true, NW_FORCE>, ForceCTA<true, NW_FORCE>::WORDS);
    else go(kc_force<false, NW_FORCE>, ForceCTA<false, NW_FORCE>::WORDS);
    return 1;
}

int launch_energy(const Slab& s, const Phys& p, int cur, Stream st, int ka, int kb)
{
    int kc0 = s.k0, kc1 = s.k1;
    if (p.rezone) euler_ranges(s, p, kc0, kc1);
    if (ka >= 0) {  // a sub-range of the cell planes (boundary-first cycles)
        kc0 = ka > kc0 ? ka : kc0;
        kc1 = kb < kc1 ? kb : kc1;
    }
    if (kc1 <= kc0) return 0;
    auto go = [&](auto kern, size_t words) {
        const size_t sm = sizeof(double) * words;
        set_smem(kern, sm);
        const long long xy = (long long)cdiv(p.nx, FW - 1) * cdiv(p.ny, NW_ENERGY - 1);
        const int zc = zchunk_for(xy, kc1 - kc0, ZCHUNK);
        dim3 grid(cdiv(p.nx, FW - 1), cdiv(p.ny, NW_ENERGY - 1), cdiv(kc1 - kc0, zc));
        kern<<<grid, dim3(FW, NW_ENERGY), sm, (cudaStream_t)st>>>(s, p, cur, kc0, kc1, zorder(zc));
        note_launch();
    };
    by_nmat(s.nmat, [&](auto nm) {
        constexpr int NM = decltype(nm)::value;
        if (p.rezone) go(kc_energy<true, NW_ENERGY, NM>, EnergyCTA<true, NW_ENERGY, NM>::WORDS);
        else go(kc_energy<false, NW_ENERGY, NM>, EnergyCTA<false, NW_ENERGY, NM>::WORDS);
    });
    return 1;
}

}  // namespace sale
