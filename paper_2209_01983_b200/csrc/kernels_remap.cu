// kernels_remap.cu -- the Eulerian remap:
//
//   kr_sweep  : z-march; R1 swept volumes of the -x/-y/-z faces of every cell (the
//               ribbons between the target and the moved faces shared between
//               neighbouring faces; the moved faces' s' from kc_energy) and the
//               R2 donor data m/V' (per material: m_k/V') and the 8-node mean u'.
//   kr_tail   : z-march; R2 donor-cell fluxes and R3 cell update per cell, R4 node
//               momentum from the gathered Delta m, Delta P, m'' (fixed gather order,
//               through shared memory) + reflecting BC; R5 (x := x^T) is implicit.
//   kn_update : one thread per node, R4 alone: the multi-material cycle's node update
//               after k_mat_flux (kernels_mat.cu), which hands Delta m, Delta P, m''
//               through HBM.
//
// Same expression trees and association as the oracle, so the results are
// bit-identical.  Shared-memory access pattern: compile-time plane parity,
// per-thread base + immediate.
#include <cuda_runtime.h>


#include "sale_mesh.cuh"

#ifndef SALE_MB_SWEEP
#define SALE_MB_SWEEP 2
#endif
#ifndef SALE_MB_TAIL
#define SALE_MB_TAIL 2
#endif
#ifndef SALE_TAIL_PF  // kr_tail: L2 prefetch distance in planes (0: none)
#define SALE_TAIL_PF 2
#endif
#ifndef SALE_NW_TAIL
#define SALE_NW_TAIL 8
#endif

namespace sale {

namespace {

constexpr int RW = 32;
constexpr int RPAD = RW + 1;

__device__ __forceinline__ D3 ld3r(const double* b, int o0, int stride) { return D3{b[o0], b[o0 + stride], b[o0 + 2 * stride]}; }
__device__ __forceinline__ void st3r(double* b, int o0, int stride, D3 v)
{
    b[o0] = v.x;
    b[o0 + stride] = v.y;
    b[o0 + 2 * stride] = v.z;
}

}  // namespace

// ============================================================================
// kn_update: R4 as a barrier-free kernel (one thread per node, operands through
// L1; high occupancy).
// ============================================================================
// grid: x = ceil((nx+1)(ny+1) / 256) (flattened node plane: no idle lanes), y = planes
template <bool TILE>  // TILE: 32 x 8 node tiles (grid x = x-tiles * y-tiles) instead of flattened rows
// (8 CTAs per SM at 32 registers: more warps for the latency-bound gather)
__global__ void __launch_bounds__(256, 8) kn_update(Slab s, Phys p, int cur, int kbase)
{
    if (!s.st->active) return;
    int i, j, t;
    if (TILE) {
        const int tx = (p.nx + 32) / 32;
        i = (blockIdx.x % tx) * 32 + (threadIdx.x & 31);
        j = (blockIdx.x / tx) * 8 + (threadIdx.x >> 5);
        if (i > p.nx || j > p.ny) return;
        t = i + (p.nx + 1) * j;
    } else {
        t = blockIdx.x * 256 + threadIdx.x;
        if (t >= (int)s.pn) return;
        i = t % (p.nx + 1);
        j = t / (p.nx + 1);
    }
    const int k = kbase + blockIdx.y;
    const bool pxm = i >= 1, pxp = i < p.nx, pym = j >= 1, pyp = j < p.ny, pzm = k >= 1, pzp = k < p.nz;
    const int c00 = i + p.nx * (j + p.ny * (k - s.kb));  // 32-bit: a slab holds < 2^31 cells
    const int sx = 1, sy = p.nx, sz = p.nx * p.ny;
    const double* __restrict__ dm = s.dm + c00;
    const double* __restrict__ m2 = s.m[cur ^ 1] + c00;
    const double* __restrict__ p0 = s.dP[0] + c00;
    const double* __restrict__ p1 = s.dP[1] + c00;
    const double* __restrict__ p2 = s.dP[2] + c00;
    double Dm = 0.0, M2 = 0.0;
    D3 DP = D3{0.0, 0.0, 0.0};
    const bool all = pxm && pxp && pym && pyp && pzm && pzp;
    bool first = true;
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        const int ap = g & 1, bp = (g >> 1) & 1, cp = g >> 2;
        const int off = (ap - 1) * sx + (bp - 1) * sy + (cp - 1) * sz;
        if (all) {
            const double d = __ldg(dm + off), mm = __ldg(m2 + off);
            const D3 dp = D3{__ldg(p0 + off), __ldg(p1 + off), __ldg(p2 + off)};
            Dm = g == 0 ? d : Dm + d;
            DP = g == 0 ? dp : add(DP, dp);
            M2 = g == 0 ? mm : M2 + mm;
        } else {
            const bool pres = (ap ? pxp : pxm) && (bp ? pyp : pym) && (cp ? pzp : pzm);
            if (!pres) continue;
            const double d = __ldg(dm + off), mm = __ldg(m2 + off);
            const D3 dp = D3{__ldg(p0 + off), __ldg(p1 + off), __ldg(p2 + off)};
            Dm = first ? d : Dm + d;
            DP = first ? dp : add(DP, dp);
            M2 = first ? mm : M2 + mm;
            first = false;
        }
    }
    Dm = 0.125 * Dm;
    DP = scl(0.125, DP);
    M2 = 0.125 * M2;
    const long long n = (long long)t + s.pn * (long long)(k - s.kb);
    const D3 u1 = ld3(s.u1, n);
    D3 un = d3(u1.x + ddiv(DP.x - (u1.x * Dm), M2), u1.y + ddiv(DP.y - (u1.y * Dm), M2),
               u1.z + ddiv(DP.z - (u1.z * Dm), M2));
    un = reflect(p, i, j, k, un);
    st3(s.u[cur ^ 1], n, un);
    if (s.hp) halo_node3(s, s.hp->u, cur ^ 1, k, t, un);
}

// ============================================================================
// kr_sweep: z-march over cell planes; stages x', u' node planes; per column and
// plane the six ribbons and three moved faces of c.4 step 1 (ribbons shared with
// the neighbouring faces), the swept volumes dV of the cell's -x/-y/-z faces, and
// the donor data r = m/V', Ubar = 8-node mean of u' (c.4 step 2).  Writes Slab::dV,
// rD, UD (read by kr_tail).  Dependencies reach only the +x / +y neighbours, so a
// 32 x NW tile yields 31 x (NW-1) columns.  Same expressions, operands and
// association as the oracle.
// ============================================================================
// NM > 0: multi-material cells: the donor data per material,
// m_k / V' (Slab::rDm, MM5), instead of r = m / V'
template <int NW, int NM = 0>
struct SweepCTA {
    static constexpr int PL = NW * RW, TX = RW - 1, TY = NW - 1;
    __host__ __device__ static constexpr int oN(int par, int c) { return (par * 6 + c) * PL; }  // x'(3) u'(3)
    __host__ __device__ static constexpr int oR(int c) { return 12 * PL + c * PL; }           // Rxz Ryz Rzy Rzx
    static constexpr int WORDS = 16 * PL + 2 * RPAD;

    const Slab& s;
    const Phys& p;
    const int cur;
    double* me;
    int i, j, ix, iy, ta, tb, kr0, kr1;
    long long nb, cb, nbc, cbc;  // nbc / cbc: the column clamped into the cells (always-valid addresses)
    long long nbn;               // the column clamped into the nodes
    bool col_in, out_col;
    double tx0, tx1, ty0, ty1;
    D3 qu1;             // prefetch: node plane (unconditional loads, selected at use)
    double xcol, ycol, dt;  // target X, Y of the (clamped) node column; the cycle's dt
    double qm, qv;      // prefetch: cell m, V' of the plane before
    double qmm[NM > 0 ? NM : 1];  // prefetch: material masses
    double qz;          // prefetch: Z of node plane k
    double zprev;       // Z of node plane t
    bool qnok;
    double rxy_t, ryx_t;  // ribbons Rxy, Ryx of node plane t (own column)

    __device__ __forceinline__ SweepCTA(const Slab& s_, const Phys& p_, int cur_, double* smem, int kr0_, int kr1_,
                                        int zchunk)
        : s(s_), p(p_), cur(cur_)
    {
        ix = threadIdx.x;
        iy = threadIdx.y;
        me = smem + RPAD + iy * RW + ix;
        i = blockIdx.x * TX + ix;
        j = blockIdx.y * TY + iy;
        kr0 = kr0_;
        kr1 = kr1_;
        const int t0 = kr0 - 1 > 0 ? kr0 - 1 : 0, t1 = kr1 < p.nz - 1 ? kr1 : p.nz - 1;  // cell planes [t0, t1]
        ta = t0 + zchunk_base(zchunk);
        tb = ta + zchunk - 1 < t1 ? ta + zchunk - 1 : t1;
        nb = (long long)i + (long long)(p.nx + 1) * (j - (long long)(p.ny + 1) * s.kb);
        cb = (long long)i + (long long)p.nx * (j - (long long)p.ny * s.kb);
        col_in = i <= p.nx && j <= p.ny;
        out_col = i < p.nx && j < p.ny && ix < TX && iy < TY;
        {
            const int ic = i < p.nx ? i : p.nx - 1, jc = j < p.ny ? j : p.ny - 1;
            nbc = (long long)ic + (long long)(p.nx + 1) * (jc - (long long)(p.ny + 1) * s.kb);
            cbc = (long long)ic + (long long)p.nx * (jc - (long long)p.ny * s.kb);
            const int in = i > p.nx ? p.nx : i, jn = j > p.ny ? p.ny : j;
            nbn = (long long)in + (long long)(p.nx + 1) * (jn - (long long)(p.ny + 1) * s.kb);
            xcol = s.Xt[in];
            ycol = s.Yt[jn];
        }
        dt = s.st->dt;
        tx0 = col_in ? s.Xt[i] : 0.0;
        tx1 = (col_in && i + 1 <= p.nx) ? s.Xt[i + 1] : 0.0;
        ty0 = col_in ? s.Yt[j] : 0.0;
        ty1 = (col_in && j + 1 <= p.ny) ? s.Yt[j + 1] : 0.0;
    }

    __device__ __forceinline__ static double fs(D3 Q0, D3 Q1, D3 Q2, D3 Q3)
    {
        return face_s(avg4(Q0, Q1, Q2, Q3), face_area(Q0, Q1, Q2, Q3));
    }
    __device__ __forceinline__ void fetch(int k)  // node plane k, cell plane k-1
    {
        qnok = col_in && k >= 0 && k <= p.nz;
        const int kn = k < s.kb ? s.kb : (k > s.kb + s.nzn - 1 ? s.kb + s.nzn - 1 : k);
        const long long n = nbn + (long long)kn * s.pn;
        qu1 = ld3(s.u1, n);
        int kc = k - 1;
        kc = kc < s.kb ? s.kb : (kc > s.kb + s.nzc - 1 ? s.kb + s.nzc - 1 : kc);
        const long long c = cbc + (long long)kc * s.pc;
        qm = s.m[cur][c];
        qv = s.V1[c];
#pragma unroll
        for (int a = 0; a < NM; ++a) qmm[a] = s.mm[cur][c + a * mat_stride(s)];
        qz = s.Zt[kn - s.kb];
    }
    template <int PAR>
    __device__ __forceinline__ void put()
    {
        const D3 z = D3{0.0, 0.0, 0.0};
        // x' = x^T + u' dt, kc_force's expression (c.3 step 6), formed when staged
        const D3 x1 = D3{xcol + (qu1.x * dt), ycol + (qu1.y * dt), qz + (qu1.z * dt)};
        st3r(me, oN(PAR, 0), PL, qnok ? x1 : z);
        st3r(me, oN(PAR, 3), PL, qnok ? qu1 : z);
    }
    template <int PAR>
    __device__ __forceinline__ D3 XL(int off) const { return ld3r(me + off, oN(PAR, 0), PL); }
    template <int PAR>
    __device__ __forceinline__ D3 UL(int off) const { return ld3r(me + off, oN(PAR, 3), PL); }
    // Rxy / Ryx of node plane k (parity PAR), own column
    template <int PAR>
    __device__ __forceinline__ void rib_xy(int k, double z, double& rxy, double& ryx) const
    {
        rxy = 0.0;
        ryx = 0.0;
        if (col_in && k >= 0 && k <= p.nz) {
            const D3 T = D3{tx0, ty0, z}, L = XL<PAR>(0);
            if (j + 1 <= p.ny) rxy = fs(T, L, XL<PAR>(RW), D3{tx0, ty1, z});
            if (i + 1 <= p.nx) ryx = fs(T, D3{tx1, ty0, z}, XL<PAR>(1), L);
        }
    }

    template <int B0>
    __device__ __forceinline__ void step(int t)
    {
        constexpr int B1 = B0 ^ 1;
        // ---- P1: stage node plane t+1 (its cell-plane t operands come with it); prefetch t+2
        put<B1>();
        const double m = qm, V1 = qv, z0 = zprev, z1 = qz;
        double cmm[NM > 0 ? NM : 1];
#pragma unroll
        for (int a = 0; a < NM; ++a) cmm[a] = qmm[a];
        if (t < tb) fetch(t + 2);
        __syncthreads();
        // ---- P2: ribbons of this column, moved faces, donor data of cell (i,j,t)
        // (the s' / s^T operands of P3 are loaded first, from always-valid addresses,
        // so their latency hides behind the ribbons)
        const long long c = cb + (long long)t * s.pc;
        const long long nL = nbc + (long long)t * s.pn, cL = cbc + (long long)t * s.pc;
        const double sx = s.sF[0][nL], sy = s.sF[1][nL], sz = s.sF[2][nL];
        const double sTx = s.sT[0][cL], sTy = s.sT[1][cL], sTz = s.sT[2][cL];
        double rxy_n, ryx_n;
        rib_xy<B1>(t + 1, z1, rxy_n, ryx_n);
        double rxz = 0.0, ryz = 0.0, rzy = 0.0, rzx = 0.0;
        if (col_in) {
            const D3 T0 = D3{tx0, ty0, z0}, T1 = D3{tx0, ty0, z1}, L0 = XL<B0>(0), L1 = XL<B1>(0);
            rxz = fs(T0, T1, L1, L0);
            ryz = fs(T0, L0, L1, T1);
            if (j + 1 <= p.ny) rzy = fs(T0, D3{tx0, ty1, z0}, XL<B0>(RW), L0);
            if (i + 1 <= p.nx) rzx = fs(T0, L0, XL<B0>(1), D3{tx1, ty0, z0});
        }
        me[oR(0)] = rxz;
        me[oR(1)] = ryz;
        me[oR(2)] = rzy;
        me[oR(3)] = rzx;
        if (out_col) {  // c.4 step 2 donor data: r = m / V', Ubar = 0.125 * (sum of u' in corner order)
            D3 sum = UL<B0>(0);
            sum = add(sum, UL<B0>(1));
            sum = add(sum, UL<B0>(RW));
            sum = add(sum, UL<B0>(RW + 1));
            sum = add(sum, UL<B1>(0));
            sum = add(sum, UL<B1>(1));
            sum = add(sum, UL<B1>(RW));
            sum = add(sum, UL<B1>(RW + 1));
            st3(s.UD, c, scl(0.125, sum));
            if constexpr (NM > 0) {
#pragma unroll
                for (int a = 0; a < NM; ++a) s.rDm[c + a * mat_stride(s)] = ddiv(cmm[a], V1);
            } else {
                s.rD[c] = ddiv(m, V1);
            }
        }
        __syncthreads();
        // ---- P3: swept volumes of the cell's -x, -y, -z faces (interior faces only)
        if (out_col && t >= kr0 && t <= kr1) {
            if (t < kr1 && i >= 1) {
                const double dV = ddiv(((((me[RW + oR(0)] - me[oR(0)]) + rxy_n) - rxy_t) + sx) - sTx, 3.0);
                s.dV[0][c] = dV;
            }
            if (t < kr1 && j >= 1) {
                const double dV = ddiv(((((ryx_n - ryx_t) + me[1 + oR(1)]) - me[oR(1)]) + sy) - sTy, 3.0);
                s.dV[1][c] = dV;
            }
            if (t >= 1) {
                const double dV = ddiv(((((me[1 + oR(2)] - me[oR(2)]) + me[RW + oR(3)]) - me[oR(3)]) + sz) - sTz, 3.0);
                s.dV[2][c] = dV;
            }
        }
        rxy_t = rxy_n;
        ryx_t = ryx_n;
        zprev = z1;
    }

    __device__ __forceinline__ void run()
    {
        fetch(ta);
        if (ta & 1) put<1>();
        else put<0>();
        zprev = qz;
        fetch(ta + 1);
        __syncthreads();
        if (ta & 1) rib_xy<1>(ta, zprev, rxy_t, ryx_t);
        else rib_xy<0>(ta, zprev, rxy_t, ryx_t);
        for (int t = ta; t <= tb; ++t) {
            if (t & 1) step<1>(t);
            else step<0>(t);
        }
    }
};

template <int NW, int MB, int NM = 0>
__global__ void __launch_bounds__(RW * NW, MB) kr_sweep(Slab s, Phys p, int cur, int kr0, int kr1, int zchunk)
{
    if (!s.st->active) return;
    extern __shared__ double smem[];
    SweepCTA<NW, NM> c(s, p, cur, smem, kr0, kr1, zchunk);
    c.run();
}

// ============================================================================
// kr_tail: R2 fluxes + R3 cell update and R4 node momentum in one z-march (the
// round-2 kr_flux + kn_update pair, whose Delta m, Delta P and m'' went through HBM).
// Thread (ix, iy) of a 32 x NW tile owns node (i, j) = (bx*TX + ix, by*TY + iy) and
// the cell (i-1, j-1) below-left of it: per cell plane t it forms that cell's six face
// fluxes from the swept volumes and the donor data of kr_sweep (c.4 step 2, every
// operand loaded before the donor sign test, so the loads overlap), the cell update
// (c.4 step 3) -- m'', e'' stored for the owned cells -- and puts Delta m, Delta P, m''
// into shared memory (double-buffered by plane parity: one barrier per plane); then
// node (i, j) of plane t is finished from the running sums (cells of plane t-1, c' = 0)
// and the four cells of plane t (c' = 1), and node plane t+1 started from the same four
// cells -- kn_update's fixed gather order, cells a' fastest, then b', then c'.  A tile
// yields (32-1) x (NW-1) nodes; node planes [ka, kb] (cell planes [ka-1, kb]).
// ============================================================================
struct Donor {
    double r, e;
    D3 u;
};
__device__ __forceinline__ Donor donor_at(const Slab& s, long long d)
{
    return Donor{s.rD[d], s.e1[d], ld3(s.UD, d)};
}
// c.4 steps 2-3 for cell (i, j, t): Delta m, Delta P and m''; stores m'', e'' (and the
// ENEGMASS check) when `own`
__device__ __forceinline__ void flux_cell(const Slab& s, const Phys& p, int cur, int i, int j, int t, bool own,
                                          double& dm, D3& dP, double& m2)
{
    const long long c = (long long)i + (long long)p.nx * ((long long)j + (long long)p.ny * (t - s.kb));
    const long long sa[3] = {1, p.nx, s.pc};
    const int ia[3] = {i, j, t}, na[3] = {p.nx, p.ny, p.nz};
    const Donor own_d = donor_at(s, c);
    // faces in the order of c.4 step 3: -x +x -y +y -z +z; boundary faces carry no flux
    double mu[6], ep[6];
    D3 pi[6];
#pragma unroll
    for (int f = 0; f < 6; ++f) {
        const int a = f >> 1;
        const bool plus = f & 1;
        const bool inner = plus ? ia[a] + 1 <= na[a] - 1 : ia[a] >= 1;  // a cell on both sides
        const long long nbr = inner ? (plus ? c + sa[a] : c - sa[a]) : c;
        const double dV = inner ? s.dV[a][plus ? nbr : c] : 0.0;  // the face is the -a face of the upper cell
        const Donor other = donor_at(s, nbr);
        // donor: the lower cell if the face moved toward +a (c.4 step 2)
        const Donor& D = (dV > 0.0) == plus ? own_d : other;
        mu[f] = inner ? D.r * dV : 0.0;
        ep[f] = inner ? mu[f] * D.e : 0.0;
        pi[f] = inner ? scl(mu[f], D.u) : D3{0.0, 0.0, 0.0};
    }
    dm = ((((mu[0] - mu[1]) + mu[2]) - mu[3]) + mu[4]) - mu[5];
    const double dE = ((((ep[0] - ep[1]) + ep[2]) - ep[3]) + ep[4]) - ep[5];
    dP = sub(add(sub(add(sub(pi[0], pi[1]), pi[2]), pi[3]), pi[4]), pi[5]);
    const double m = s.m[cur][c], e1 = own_d.e;
    m2 = m + dm;
    if (own) {
        if (t >= s.k0 && t < s.k1 && !(m2 > 0.0))
            atomicMin(&s.st->err_key, (ERR_ORDER_NEGMASS << 48) | (unsigned long long)gcell(p, i, j, t));
        const double e2 = e1 + ddiv(dE - (e1 * dm), m2);
        s.e[cur ^ 1][c] = e2;
        s.m[cur ^ 1][c] = m2;
        if (s.hp) {  // peer-store halo: the neighbours' ghost cell planes
            const long long q = (long long)i + (long long)p.nx * j;
            halo_cell(s, s.hp->e, cur ^ 1, 0, t, q, e2);
            halo_cell(s, s.hp->m, cur ^ 1, 0, t, q, m2);
        }
    }
}

template <int NW>
struct TailCTA {
    static constexpr int PL = NW * RW, TX = RW - 1, TY = NW - 1;
    __host__ __device__ static constexpr int oC(int par, int c) { return (par * 5 + c) * PL; }  // dm, dP(3), m''
    static constexpr int WORDS = 10 * PL;

    const Slab& s;
    const Phys& p;
    const int cur;
    double* me;
    int i, j, ka, kb, za, zb;
    long long nb;
    bool node_thr, cell_col, own_col;
    bool pxm, pxp, pym, pyp;
    D3 Fp;  // running sums of node plane t+1 (cells of plane t, c' = 0)
    double Dp, Mp;
    bool have;

    __device__ __forceinline__ TailCTA(const Slab& s_, const Phys& p_, int cur_, double* smem, int ka_, int kb_,
                                       int zchunk)
        : s(s_), p(p_), cur(cur_)
    {
        const int ix = threadIdx.x, iy = threadIdx.y;
        me = smem + iy * RW + ix;
        i = blockIdx.x * TX + ix;
        j = blockIdx.y * TY + iy;
        ka = ka_;
        kb = kb_;
        za = ka + zchunk_base(zchunk);
        zb = za + zchunk - 1 < kb ? za + zchunk - 1 : kb;
        nb = (long long)i + (long long)(p.nx + 1) * (j - (long long)(p.ny + 1) * s.kb);
        node_thr = ix < TX && iy < TY && i <= p.nx && j <= p.ny;
        cell_col = i >= 1 && i <= p.nx && j >= 1 && j <= p.ny;  // cell (i-1, j-1) exists
        own_col = cell_col && ix >= 1 && iy >= 1;                // ... and this tile stores it
        pxm = i >= 1;
        pxp = i < p.nx;
        pym = j >= 1;
        pyp = j < p.ny;
    }

    // the four cells of the plane in buffer PAR at corners c' = CZ of node (i, j), in
    // gather order a' fastest (cell (i-1+a', j-1+b') sits at me + a' + b' RW)
    template <int PAR>
    __device__ __forceinline__ void gather4(double& Dm, D3& DP, double& M2, bool& hv, bool pz) const
    {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const int ap = g & 1, bp = g >> 1;
            const int off = ap + bp * RW;
            const bool pres = pz && (ap ? pxp : pxm) && (bp ? pyp : pym);
            if (pres) {
                const double d = me[off + oC(PAR, 0)], mm = me[off + oC(PAR, 4)];
                const D3 dp = D3{me[off + oC(PAR, 1)], me[off + oC(PAR, 2)], me[off + oC(PAR, 3)]};
                Dm = hv ? Dm + d : d;
                DP = hv ? add(DP, dp) : dp;
                M2 = hv ? M2 + mm : mm;
                hv = true;
            }
        }
    }

    template <int PAR>
    __device__ __forceinline__ void step(int t)
    {
        const bool fin = node_thr && t >= za;  // node plane t is finished in this step
        const long long n = nb + (long long)t * s.pn;
        D3 u1 = D3{0.0, 0.0, 0.0};
        if (fin) u1 = ld3(s.u1, n);
        const bool pz = t >= 0 && t < p.nz;  // cell plane t exists
#if SALE_TAIL_PF
        // the operands of plane t + PF into L2 (no registers held): the loads of a
        // z-march step are exposed once per plane, an L2 hit shortens them
        if (cell_col && t + SALE_TAIL_PF < p.nz && t + SALE_TAIL_PF <= zb) {
            constexpr int PF = SALE_TAIL_PF;
            const int tp = t + PF;
            const long long c = (long long)(i - 1) + (long long)p.nx * ((long long)(j - 1) + (long long)p.ny * (tp - s.kb));
            const double* a[9] = {s.rD, s.e1, s.UD[0], s.UD[1], s.UD[2], s.dV[0], s.dV[1], s.dV[2], s.m[cur]};
#pragma unroll
            for (int q = 0; q < 9; ++q) asm volatile("prefetch.global.L2 [%0];" ::"l"(a[q] + c));
            if (node_thr) {
                const long long np = nb + (long long)tp * s.pn;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(s.u1[0] + np));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(s.u1[1] + np));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(s.u1[2] + np));
            }
        }
#endif
        if (cell_col && pz) {
            double dm, m2;
            D3 dP;
            flux_cell(s, p, cur, i - 1, j - 1, t, own_col && t >= ka && t <= kb && t < s.k1, dm, dP, m2);
            me[oC(PAR, 0)] = dm;
            me[oC(PAR, 1)] = dP.x;
            me[oC(PAR, 2)] = dP.y;
            me[oC(PAR, 3)] = dP.z;
            me[oC(PAR, 4)] = m2;
        }
        __syncthreads();
        if (!node_thr) return;
        if (fin) {
            double Dm = Dp, M2 = Mp;
            D3 DP = Fp;
            bool hv = have;
            gather4<PAR>(Dm, DP, M2, hv, pz);
            Dm = 0.125 * Dm;
            DP = scl(0.125, DP);
            M2 = 0.125 * M2;
            D3 un = d3(u1.x + ddiv(DP.x - (u1.x * Dm), M2), u1.y + ddiv(DP.y - (u1.y * Dm), M2),
                       u1.z + ddiv(DP.z - (u1.z * Dm), M2));
            un = reflect(p, i, j, t, un);
            st3(s.u[cur ^ 1], n, un);
            if (s.hp) halo_node3(s, s.hp->u, cur ^ 1, t, (long long)i + (long long)(p.nx + 1) * j, un);
        }
        have = false;
        Dp = 0.0;
        Mp = 0.0;
        Fp = D3{0.0, 0.0, 0.0};
        if (t < zb) gather4<PAR>(Dp, Fp, Mp, have, pz);
    }

    __device__ __forceinline__ void run()
    {
        have = false;
        Dp = 0.0;
        Mp = 0.0;
        Fp = D3{0.0, 0.0, 0.0};
        for (int t = za - 1; t <= zb; ++t) {
            if (t & 1) step<1>(t);
            else step<0>(t);
        }
    }
};

// grid: x = ceil((nx+1) / 31), y = ceil((ny+1) / (NW-1)), z = z-chunks of node planes [ka, kb]
template <int NW>
__global__ void __launch_bounds__(RW * NW, SALE_MB_TAIL) kr_tail(Slab s, Phys p, int cur, int ka, int kb, int zchunk)
{
    if (!s.st->active) return;
    extern __shared__ double smem[];
    TailCTA<NW> c(s, p, cur, smem, ka, kb, zchunk);
    c.run();
}

// ============================================================================
namespace {
inline int cdivr(int a, int b) { return (a + b - 1) / b; }
constexpr int RZ = 32;
}  // namespace

template <int NW, int NM>
static void sweep_launch(const Slab& s, const Phys& p, int cur, int kr0, int kr1, cudaStream_t cs)
{
    auto kern = kr_sweep<NW, SALE_MB_SWEEP, NM>;
    const size_t sm = sizeof(double) * SweepCTA<NW, NM>::WORDS;
    static bool init = false;
    if (!init) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        init = true;
    }
    const int t0 = kr0 - 1 > 0 ? kr0 - 1 : 0, t1 = kr1 < p.nz - 1 ? kr1 : p.nz - 1;
    const int zc = zchunk_for((long long)cdivr(p.nx, RW - 1) * cdivr(p.ny, NW - 1), t1 - t0 + 1, RZ);
    dim3 grid(cdivr(p.nx, RW - 1), cdivr(p.ny, NW - 1), cdivr(t1 - t0 + 1, zc));
    kern<<<grid, dim3(RW, NW), sm, cs>>>(s, p, cur, kr0, kr1, zorder(zc));
    note_launch();
}

// R1 swept volumes and the donor data (multi-material cells: per material)
int launch_sweep(const Slab& s, const Phys& p, int cur, Stream st)
{
    const int kr0 = s.k0 - 1 > 0 ? s.k0 - 1 : 0, kr1 = s.k1 + 1 < p.nz ? s.k1 + 1 : p.nz;
    cudaStream_t cs = (cudaStream_t)st;
    switch (s.nmat) {
    case 0: sweep_launch<8, 0>(s, p, cur, kr0, kr1, cs); break;
    case 1: sweep_launch<8, 1>(s, p, cur, kr0, kr1, cs); break;
    case 2: sweep_launch<8, 2>(s, p, cur, kr0, kr1, cs); break;
    case 3: sweep_launch<8, 3>(s, p, cur, kr0, kr1, cs); break;
    default: sweep_launch<8, 4>(s, p, cur, kr0, kr1, cs); break;
    }
    return 1;
}

// R4 node momentum update on the cell totals (32 x 8 node tiles: the gathered cell
// values are reused inside a block through L1)
int launch_kn_update(const Slab& s, const Phys& p, int cur, Stream st, int ka, int kb)
{
    int k0 = s.k0, k1 = s.k1;  // node planes [k0, k1]
    if (ka >= 0) {             // a sub-range [ka, kb] (boundary-first cycles)
        k0 = ka > k0 ? ka : k0;
        k1 = kb < k1 ? kb : k1;
    }
    if (k1 < k0) return 0;
    kn_update<true><<<dim3(cdivr(p.nx + 1, 32) * cdivr(p.ny + 1, 8), k1 - k0 + 1), 256, 0, (cudaStream_t)st>>>(
        s, p, cur, k0);
    note_launch();
    return 1;
}

// R2-R4 of the single-material scheme over node planes [ka, kb] (default: the owned
// planes [k0, k1]); the cells of planes [ka-1, kb] are formed, those in [ka, kb] n
// [k0, k1) stored (so boundary-first sub-ranges split the owned cells disjointly)
int launch_rtail(const Slab& s, const Phys& p, int cur, Stream st, int ka, int kb)
{
    int k0 = s.k0, k1 = s.k1;
    if (ka >= 0) {
        k0 = ka > k0 ? ka : k0;
        k1 = kb < k1 ? kb : k1;
    }
    if (k1 < k0) return 0;
    constexpr int NW = SALE_NW_TAIL;
    auto kern = kr_tail<NW>;
    const size_t sm = sizeof(double) * TailCTA<NW>::WORDS;
    static bool init = false;
    if (!init) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        init = true;
    }
    const long long xy = (long long)cdivr(p.nx + 1, RW - 1) * cdivr(p.ny + 1, NW - 1);
    const int zc = zchunk_for(xy, k1 - k0 + 1, RZ);
    dim3 grid(cdivr(p.nx + 1, RW - 1), cdivr(p.ny + 1, NW - 1), cdivr(k1 - k0 + 1, zc));
    kern<<<grid, dim3(RW, NW), sm, (cudaStream_t)st>>>(s, p, cur, k0, k1, zorder(zc));
    note_launch();
    return 1;
}

// R1-R4 of the single-material scheme: kr_sweep and (nodes = 1) kr_tail over every
// owned node plane (the next cycle's ke_state forms the dt candidate of the remapped
// state); nodes = 0 leaves R2-R4 to the caller (boundary-first cycles: launch_rtail by
// node-plane ranges)
int launch_remap(const Slab& s, const Phys& p, int cur, Stream st, int nodes)
{
    launch_sweep(s, p, cur, st);
    if (!nodes) return 1;
    return 1 + launch_rtail(s, p, cur, st);
}

}  // namespace sale
