// kernels_remap.cu -- the fused Eulerian remap
// as two z-marching kernels:
//
//   kr_cells : R1 swept volume of the three faces anchored at each column (each
//              physical face computed once per CTA), R2 donor-cell fluxes with
//              the donor data (m/V', e', 8-node mean u') staged in shared
//              memory, R3 cell update m'', e'', Delta m, Delta P.
//   kr_nodes : R4 node momentum update u'' from the gathered Delta m, Delta P,
//              m'' (fixed gather order) + reflecting BC; R5 (x := x^T) is
//              implicit; then the next cycle's dt candidate (c.5) on the target
//              mesh with a running min, warp-shuffle + block min, one atomicMin.
//
// Same expression trees and association as the oracle / v0 kernels, so the
// results are bit-identical.  Shared-memory access pattern as in
// kernels_fused.cu: compile-time plane parity, per-thread base + immediate.
#include <cuda_runtime.h>

#include <cstdlib>

#include "sale_mesh.cuh"

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

struct Flux {
    double mu, eps;
    D3 pi;
};

}  // namespace

// ============================================================================
// kr_cells: cell planes [kr0, kr1) (global), z-chunked.  Columns i = i0-1+ix.
// ============================================================================
template <int NW>
struct RemapCellsCTA {
    static constexpr int PL = NW * RW, TX = RW - 3, TY = NW - 3;
    __host__ __device__ static constexpr int oN(int par, int c) { return (par * 6 + c) * PL; }  // x'(3), u'(3)
    __host__ __device__ static constexpr int oC(int c) { return 12 * PL + c * PL; }            // donor r, e', Ubar(3)
    __host__ __device__ static constexpr int oF(int par, int xy, int c) { return 17 * PL + ((par * 2 + xy) * 5 + c) * PL; }
    __host__ __device__ static constexpr int oR(int c) { return 37 * PL + c * PL; }  // ribbons Rxz Ryz Rzy Rzx
    static constexpr int WORDS = 41 * PL + 2 * RPAD;

    const Slab& s;
    const Phys& p;
    const int cur;
    double* me;
    int i, j, ix, iy, za, zb, kr0, kr1;
    long long nb, cb;
    bool col_in, cell_col, xface_on, yface_on, zface_on, upd_on;
    D3 qx1, qu1;            // prefetch: node x', u'
    double qm, qe, qv;      // prefetch: cell m, e', V'
    double qs0, qs1, qs2;   // prefetch: s^T of the cell's -x/-y/-z target faces
    double qz;              // prefetch: Z of node plane k
    double tx0, tx1, ty0, ty1;  // this column's X_i, X_{i+1}, Y_j, Y_{j+1}
    double tz0, tz1;        // Z of node planes kz, kz+1
    // own column, previous cell plane (kz-1): donor data and pre-remap state
    double r_prev, e_prev, m_prev;
    D3 ub_prev;
    Flux fz_prev;           // z-face flux at node plane kz-1... carried one step
    double rxy_prev, ryx_prev;  // ribbons Rxy, Ryx of node plane kz (computed at step kz-1)
    bool rib_on;

    __device__ __forceinline__ RemapCellsCTA(const Slab& s_, const Phys& p_, int cur_, double* smem, int kr0_, int kr1_,
                                             int zchunk)
        : s(s_), p(p_), cur(cur_)
    {
        ix = threadIdx.x;
        iy = threadIdx.y;
        me = smem + RPAD + iy * RW + ix;
        i = blockIdx.x * TX - 1 + ix;
        j = blockIdx.y * TY - 1 + iy;
        kr0 = kr0_;
        kr1 = kr1_;
        za = kr0 + blockIdx.z * zchunk;
        zb = za + zchunk - 1 < kr1 - 1 ? za + zchunk - 1 : kr1 - 1;
        nb = (long long)i + (long long)(p.nx + 1) * (j - (long long)(p.ny + 1) * s.kb);
        cb = (long long)i + (long long)p.nx * (j - (long long)p.ny * s.kb);
        col_in = i >= 0 && i <= p.nx && j >= 0 && j <= p.ny;
        cell_col = i >= 0 && i < p.nx && j >= 0 && j < p.ny;
        const bool in_x = ix >= 1 && ix <= TX, in_y = iy >= 1 && iy <= TY;
        // x-faces at node planes [i0, i0+TX] of cell rows [j0, j0+TY); interior iff 1 <= i <= nx-1
        xface_on = ix >= 1 && ix <= TX + 1 && in_y && i >= 1 && i <= p.nx - 1 && j >= 0 && j < p.ny;
        yface_on = in_x && iy >= 1 && iy <= TY + 1 && j >= 1 && j <= p.ny - 1 && i >= 0 && i < p.nx;
        zface_on = in_x && in_y && cell_col;
        upd_on = in_x && in_y && cell_col;
        rib_on = col_in && ix >= 1 && iy >= 1 && iy <= TY + 1;
        tx0 = col_in ? s.Xt[i] : 0.0;
        tx1 = (col_in && i + 1 <= p.nx) ? s.Xt[i + 1] : 0.0;
        ty0 = col_in ? s.Yt[j] : 0.0;
        ty1 = (col_in && j + 1 <= p.ny) ? s.Yt[j + 1] : 0.0;
        tz0 = tz1 = 0.0;
    }

    // s of a ribbon / face from its 4 points in canonical order (c.2)
    __device__ __forceinline__ static double fs(D3 Q0, D3 Q1, D3 Q2, D3 Q3)
    {
        return face_s(avg4(Q0, Q1, Q2, Q3), face_area(Q0, Q1, Q2, Q3));
    }

    __device__ __forceinline__ void fetch(int k)  // node plane k, cell plane k-1
    {
        qx1 = D3{0.0, 0.0, 0.0};
        qu1 = qx1;
        if (col_in && k >= 0 && k <= p.nz) {
            long long n = nb + (long long)k * s.pn;
            qx1 = ld3(s.x1, n);
            qu1 = ld3(s.u1, n);
        }
        qm = 0.0;
        qe = 0.0;
        qv = 1.0;
        qs0 = qs1 = qs2 = 0.0;
        qz = (k - s.kb >= 0 && k - s.kb < s.nzn) ? s.Zt[k - s.kb] : 0.0;
        const int kc = k - 1;
        if (cell_col && kc >= 0 && kc < p.nz) {
            long long c = cb + (long long)kc * s.pc;
            qm = s.m[cur][c];
            qe = s.e1[c];
            qv = s.V1[c];
            qs0 = s.sT[0][c];
            qs1 = s.sT[1][c];
            qs2 = s.sT[2][c];
        }
    }
    template <int PAR>
    __device__ __forceinline__ void put()
    {
        st3r(me, oN(PAR, 0), PL, qx1);
        st3r(me, oN(PAR, 3), PL, qu1);
    }
    template <int PAR>
    __device__ __forceinline__ D3 XL(int off) const { return ld3r(me + off, oN(PAR, 0), PL); }
    template <int PAR>
    __device__ __forceinline__ D3 UL(int off) const { return ld3r(me + off, oN(PAR, 3), PL); }
    // target node position from the per-thread table registers (dk = 0: plane kz, 1: kz+1)
    __device__ __forceinline__ D3 XT(int di, int dj, int dk) const
    {
        return D3{di ? tx1 : tx0, dj ? ty1 : ty0, dk ? tz1 : tz0};
    }

    // donor-cell flux through a face with swept volume dV, donors lower (L) / upper (U)
    __device__ __forceinline__ static Flux flux(double dV, double rL, double eL, D3 uL, double rU, double eU, D3 uU)
    {
        const bool low = dV > 0.0;
        Flux f;
        f.mu = (low ? rL : rU) * dV;
        f.eps = f.mu * (low ? eL : eU);
        f.pi = scl(f.mu, low ? uL : uU);
        return f;
    }

    template <int B0>
    __device__ __forceinline__ void step(int kz)
    {
        constexpr int B1 = B0 ^ 1;
        // ---- P1: stage node plane kz+1, cell (i,j,kz); prefetch next
        put<B1>();
        const double m = qm, e1 = qe, V1 = qv, sT0 = qs0, sT1 = qs1, sT2 = qs2;
        tz0 = tz1;
        tz1 = qz;
        if (kz < zb + 1) fetch(kz + 2);
        __syncthreads();
        // ---- P2: donor data of cell (i,j,kz); swept volumes of the anchored faces
        const bool cell_ok = cell_col && kz >= 0 && kz < p.nz;
        D3 ub = D3{0.0, 0.0, 0.0};
        double r = 0.0;
        if (cell_ok) {
            // Ubar = 0.125 * (sum of u' over the 8 corners, corner order)
            D3 sum = UL<B0>(0);
            sum = add(sum, UL<B0>(1));
            sum = add(sum, UL<B0>(RW));
            sum = add(sum, UL<B0>(RW + 1));
            sum = add(sum, UL<B1>(0));
            sum = add(sum, UL<B1>(1));
            sum = add(sum, UL<B1>(RW));
            sum = add(sum, UL<B1>(RW + 1));
            ub = scl(0.125, sum);
            r = ddiv(m, V1);
        }
        me[oC(0)] = r;
        me[oC(1)] = e1;
        st3r(me, oC(2), PL, ub);
        // c.4 step 1 with shared ribbons.  The swept hex of a face has the target
        // face as bottom (Z0, constant: s^T precomputed), the moved face as top
        // (Z1), and four lateral ribbons between a target edge and its moved
        // edge.  Same-family neighbouring faces see the same ribbon with the same
        // canonical node sequence, so it is computed once (bit-identical):
        //   x-face (i,j,k): X0 Rxz(i,j)  X1 Rxz(i,j+1)  Y0 Rxy(k)  Y1 Rxy(k+1)
        //   y-face (i,j,k): X0 Ryx(k)    X1 Ryx(k+1)    Y0 Ryz(i,j) Y1 Ryz(i+1,j)
        //   z-face (i,j,k): X0 Rzy(i,j)  X1 Rzy(i+1,j)  Y0 Rzx(i,j) Y1 Rzx(i,j+1)
        double rxy_next = 0.0, ryx_next = 0.0;
        {
            double rxz = 0.0, ryz = 0.0, rzy = 0.0, rzx = 0.0;
            if (rib_on && kz + 1 >= 0 && kz + 1 <= p.nz) {  // edges in node plane kz+1
                const D3 T1 = XT(0, 0, 1), L1 = XL<B1>(0);
                if (j + 1 <= p.ny) rxy_next = fs(T1, L1, XL<B1>(RW), XT(0, 1, 1));  // Rxy(i,j,kz+1)
                if (i + 1 <= p.nx) ryx_next = fs(T1, XT(1, 0, 1), XL<B1>(1), L1);  // Ryx(i,j,kz+1)
            }
            if (rib_on && kz >= 0 && kz < p.nz) {  // z-edge kz -> kz+1 and edges in plane kz
                const D3 T0 = XT(0, 0, 0), T1 = XT(0, 0, 1), L0 = XL<B0>(0), L1 = XL<B1>(0);
                rxz = fs(T0, T1, L1, L0);
                ryz = fs(T0, L0, L1, T1);
                if (j + 1 <= p.ny) rzy = fs(T0, XT(0, 1, 0), XL<B0>(RW), L0);  // Rzy(i,j,kz)
                if (i + 1 <= p.nx) rzx = fs(T0, L0, XL<B0>(1), XT(1, 0, 0));  // Rzx(i,j,kz)
            }
            me[oR(0)] = rxz;
            me[oR(1)] = ryz;
            me[oR(2)] = rzy;
            me[oR(3)] = rzx;
        }
        const bool do_x = xface_on && kz >= 0 && kz < p.nz && kz >= za && kz <= zb;
        const bool do_y = yface_on && kz >= 0 && kz < p.nz && kz >= za && kz <= zb;
        const bool do_z = zface_on && kz >= 1 && kz <= p.nz - 1 && kz >= za;
        __syncthreads();
        // ---- P3: swept volumes and donor-cell fluxes (boundary faces: +0.0)
        Flux fx = Flux{0.0, 0.0, D3{0.0, 0.0, 0.0}}, fy = fx, fz = fx;
        if (do_x) {
            // moved x-face at node plane i: (i,j,kz) (i,j+1,kz) (i,j+1,kz+1) (i,j,kz+1)
            const double sL = fs(XL<B0>(0), XL<B0>(RW), XL<B1>(RW), XL<B1>(0));
            const double sT = sT0;
            const double dV = ddiv(((((me[RW + oR(0)] - me[oR(0)]) + rxy_next) - rxy_prev) + sL) - sT, 3.0);
            const double* L = me - 1;
            fx = flux(dV, L[oC(0)], L[oC(1)], ld3r(L, oC(2), PL), r, e1, ub);
        }
        if (do_y) {
            // moved y-face at node plane j: (i,j,kz) (i,j,kz+1) (i+1,j,kz+1) (i+1,j,kz)
            const double sL = fs(XL<B0>(0), XL<B1>(0), XL<B1>(1), XL<B0>(1));
            const double sT = sT1;
            const double dV = ddiv(((((ryx_next - ryx_prev) + me[1 + oR(1)]) - me[oR(1)]) + sL) - sT, 3.0);
            const double* L = me - RW;
            fy = flux(dV, L[oC(0)], L[oC(1)], ld3r(L, oC(2), PL), r, e1, ub);
        }
        if (do_z) {
            // moved z-face at node plane kz: (i,j,kz) (i+1,j,kz) (i+1,j+1,kz) (i,j+1,kz)
            const double sL = fs(XL<B0>(0), XL<B0>(1), XL<B0>(RW + 1), XL<B0>(RW));
            const double sT = sT2;
            const double dV = ddiv(((((me[1 + oR(2)] - me[oR(2)]) + me[RW + oR(3)]) - me[oR(3)]) + sL) - sT, 3.0);
            fz = flux(dV, r_prev, e_prev, ub_prev, r, e1, ub);
        }
        me[oF(B0, 0, 0)] = fx.mu;
        me[oF(B0, 0, 1)] = fx.eps;
        st3r(me, oF(B0, 0, 2), PL, fx.pi);
        me[oF(B0, 1, 0)] = fy.mu;
        me[oF(B0, 1, 1)] = fy.eps;
        st3r(me, oF(B0, 1, 2), PL, fy.pi);
        __syncthreads();
        // ---- P4: cell update for cell plane kz-1
        const int kc = kz - 1;
        if (upd_on && kc >= za && kc >= 0 && kc < p.nz) {
            const double* own = me;
            const double* xp = me + 1;
            const double* yp = me + RW;
            const double mu[6] = {own[oF(B1, 0, 0)], xp[oF(B1, 0, 0)], own[oF(B1, 1, 0)], yp[oF(B1, 1, 0)],
                                  fz_prev.mu, fz.mu};
            const double ep[6] = {own[oF(B1, 0, 1)], xp[oF(B1, 0, 1)], own[oF(B1, 1, 1)], yp[oF(B1, 1, 1)],
                                  fz_prev.eps, fz.eps};
            const D3 pi[6] = {ld3r(own, oF(B1, 0, 2), PL), ld3r(xp, oF(B1, 0, 2), PL), ld3r(own, oF(B1, 1, 2), PL),
                              ld3r(yp, oF(B1, 1, 2), PL), fz_prev.pi, fz.pi};
            const double dm = ((((mu[0] - mu[1]) + mu[2]) - mu[3]) + mu[4]) - mu[5];
            const double dE = ((((ep[0] - ep[1]) + ep[2]) - ep[3]) + ep[4]) - ep[5];
            const D3 dP = sub(add(sub(add(sub(pi[0], pi[1]), pi[2]), pi[3]), pi[4]), pi[5]);
            const double m2 = m_prev + dm;
            if (kc >= s.k0 && kc < s.k1 && !(m2 > 0.0))
                atomicMin(&s.st->err_key, (ERR_ORDER_NEGMASS << 48) | (unsigned long long)gcell(p, i, j, kc));
            const long long c = cb + (long long)kc * s.pc;
            s.e[cur ^ 1][c] = e_prev + ddiv(dE - (e_prev * dm), m2);
            s.m[cur ^ 1][c] = m2;
            s.dm[c] = dm;
            st3(s.dP, c, dP);
        }
        r_prev = r;
        e_prev = e1;
        m_prev = m;
        ub_prev = ub;
        fz_prev = fz;
        rxy_prev = rxy_next;
        ryx_prev = ryx_next;
    }

    __device__ __forceinline__ void run()
    {
        // prologue: node plane za-1 staged, prefetch node plane za + cell za-1
        fetch(za - 1);
        if ((za - 1) & 1) put<1>();
        else put<0>();
        tz1 = qz;  // Z of node plane za-1 (becomes tz0 at the first step)
        fetch(za);
        __syncthreads();
        fz_prev = Flux{0.0, 0.0, D3{0.0, 0.0, 0.0}};
        r_prev = 0.0;
        e_prev = 0.0;
        m_prev = 0.0;
        ub_prev = D3{0.0, 0.0, 0.0};
        rxy_prev = 0.0;
        ryx_prev = 0.0;
        // step kz computes donor data / fluxes of plane kz and updates plane kz-1
        for (int kz = za - 1; kz <= zb + 1; ++kz) {
            if (kz & 1) step<1>(kz);
            else step<0>(kz);
        }
    }
};

template <int NW>
__global__ void __launch_bounds__(RW * NW, 2) kr_cells(Slab s, Phys p, int cur, int kr0, int kr1, int zchunk)
{
    if (!s.st->active) return;
    extern __shared__ double smem[];
    RemapCellsCTA<NW> c(s, p, cur, smem, kr0, kr1, zchunk);
    c.run();
}

// ============================================================================
// kr_cells_p: the same computation as kr_cells, software-pipelined along z so
// that one __syncthreads per z-step suffices.  Step t runs, back to back,
//   B(t)   swept volumes + fluxes of plane t      (reads A(t) outputs),
//   C(t-1) cell update of plane t-1               (reads B(t-1) fluxes),
//   A(t+1) donor data, ribbons, moved-face s' of plane t+1 (reads node planes t+1, t+2),
//   put node plane t+3, prefetch node plane t+4 / cell plane t+2,
// with every cross-thread hand-off double-buffered (node planes: ring of 3).
// ============================================================================
template <int NW>
struct RemapCellsP {
    static constexpr int PL = NW * RW, TX = RW - 3, TY = NW - 3;
    __host__ __device__ static constexpr int oN(int slot, int c) { return (slot * 6 + c) * PL; }     // x'(3) u'(3)
    __host__ __device__ static constexpr int oC(int par, int c) { return 18 * PL + (par * 5 + c) * PL; }  // r e' Ubar
    __host__ __device__ static constexpr int oR(int par, int c) { return 28 * PL + (par * 4 + c) * PL; }  // Rxz Ryz Rzy Rzx
    __host__ __device__ static constexpr int oF(int par, int xy, int c) { return 36 * PL + ((par * 2 + xy) * 5 + c) * PL; }
    static constexpr int WORDS = 56 * PL + 2 * RPAD;

    struct Cell {
        double r, e1;
        D3 ub;
    };

    const Slab& s;
    const Phys& p;
    const int cur;
    double* me;
    int i, j, ix, iy, za, zb;
    long long nb, cb;
    bool col_in, cell_col, xface_on, yface_on, zface_on, upd_on, rib_on;
    double tx0, tx1, ty0, ty1;
    // prefetch registers: node plane, cell plane
    D3 qx1, qu1;
    double qm, qe, qv, qs0, qs1, qs2;
    // carried state
    Cell c_tm1, c_t;            // own donor data of planes t-1, t
    double rxy_t, rxy_t1, ryx_t, ryx_t1;  // Rxy/Ryx of node planes t, t+1
    double sLx, sLy, sLz;       // moved-face s of plane t (from A(t))
    double sTx, sTy, sTz;       // target-face s of plane t
    double m_t, e_t, m_tm1, e_tm1;  // pre-remap m, e' of cells t, t-1
    double sTx_n, sTy_n, sTz_n, m_n, e_n;  // the same for plane t+1 (from A(t+1))
    Flux fz_tm1;                // z-face flux at node plane t-1

    __device__ __forceinline__ RemapCellsP(const Slab& s_, const Phys& p_, int cur_, double* smem, int kr0, int kr1,
                                           int zchunk)
        : s(s_), p(p_), cur(cur_)
    {
        ix = threadIdx.x;
        iy = threadIdx.y;
        me = smem + RPAD + iy * RW + ix;
        i = blockIdx.x * TX - 1 + ix;
        j = blockIdx.y * TY - 1 + iy;
        za = kr0 + blockIdx.z * zchunk;
        zb = za + zchunk - 1 < kr1 - 1 ? za + zchunk - 1 : kr1 - 1;
        nb = (long long)i + (long long)(p.nx + 1) * (j - (long long)(p.ny + 1) * s.kb);
        cb = (long long)i + (long long)p.nx * (j - (long long)p.ny * s.kb);
        col_in = i >= 0 && i <= p.nx && j >= 0 && j <= p.ny;
        cell_col = i >= 0 && i < p.nx && j >= 0 && j < p.ny;
        const bool in_x = ix >= 1 && ix <= TX, in_y = iy >= 1 && iy <= TY;
        xface_on = ix >= 1 && ix <= TX + 1 && in_y && i >= 1 && i <= p.nx - 1 && j >= 0 && j < p.ny;
        yface_on = in_x && iy >= 1 && iy <= TY + 1 && j >= 1 && j <= p.ny - 1 && i >= 0 && i < p.nx;
        zface_on = in_x && in_y && cell_col;
        upd_on = in_x && in_y && cell_col;
        rib_on = col_in && ix >= 1 && iy >= 1 && iy <= TY + 1;
        tx0 = col_in ? s.Xt[i] : 0.0;
        tx1 = (col_in && i + 1 <= p.nx) ? s.Xt[i + 1] : 0.0;
        ty0 = col_in ? s.Yt[j] : 0.0;
        ty1 = (col_in && j + 1 <= p.ny) ? s.Yt[j + 1] : 0.0;
    }

    __device__ __forceinline__ static double fs(D3 Q0, D3 Q1, D3 Q2, D3 Q3)
    {
        return face_s(avg4(Q0, Q1, Q2, Q3), face_area(Q0, Q1, Q2, Q3));
    }
    __device__ __forceinline__ static Flux flux(double dV, const Cell& L, const Cell& U)
    {
        const bool low = dV > 0.0;
        Flux f;
        f.mu = (low ? L.r : U.r) * dV;
        f.eps = f.mu * (low ? L.e1 : U.e1);
        f.pi = scl(f.mu, low ? L.ub : U.ub);
        return f;
    }
    __device__ __forceinline__ double zt(int k) const
    {
        return (k - s.kb >= 0 && k - s.kb < s.nzn) ? s.Zt[k - s.kb] : 0.0;
    }
    __device__ __forceinline__ void fetch_node(int k)
    {
        qx1 = D3{0.0, 0.0, 0.0};
        qu1 = qx1;
        if (col_in && k >= 0 && k <= p.nz) {
            long long n = nb + (long long)k * s.pn;
            qx1 = ld3(s.x1, n);
            qu1 = ld3(s.u1, n);
        }
    }
    __device__ __forceinline__ void fetch_cell(int k)
    {
        qm = 0.0;
        qe = 0.0;
        qv = 1.0;
        qs0 = qs1 = qs2 = 0.0;
        if (cell_col && k >= 0 && k < p.nz) {
            long long c = cb + (long long)k * s.pc;
            qm = s.m[cur][c];
            qe = s.e1[c];
            qv = s.V1[c];
            qs0 = s.sT[0][c];
            qs1 = s.sT[1][c];
            qs2 = s.sT[2][c];
        }
    }
    __device__ __forceinline__ void put(int k)
    {
        const int slot = ((k % 3) + 3) % 3;
        double* b = me + oN(slot, 0);
        b[0] = qx1.x;
        b[PL] = qx1.y;
        b[2 * PL] = qx1.z;
        b[3 * PL] = qu1.x;
        b[4 * PL] = qu1.y;
        b[5 * PL] = qu1.z;
    }

    // A(tau): donor data, ribbons, moved-face s of plane tau (node planes tau, tau+1)
    template <int PAR>
    __device__ __forceinline__ void stageA(int tau, int slot0, int slot1, Cell& cell, double& rxy_n, double& ryx_n,
                                           double& sx, double& sy, double& sz)
    {
        const double* N0 = me + oN(slot0, 0);
        const double* N1 = me + oN(slot1, 0);
        auto XL0 = [&](int off) { return ld3r(N0 + off, 0, PL); };
        auto XL1 = [&](int off) { return ld3r(N1 + off, 0, PL); };
        auto UL0 = [&](int off) { return ld3r(N0 + off, 3 * PL, PL); };
        auto UL1 = [&](int off) { return ld3r(N1 + off, 3 * PL, PL); };
        // donor data of cell (i,j,tau)
        cell = Cell{0.0, qe, D3{0.0, 0.0, 0.0}};
        if (cell_col && tau >= 0 && tau < p.nz) {
            D3 sum = UL0(0);
            sum = add(sum, UL0(1));
            sum = add(sum, UL0(RW));
            sum = add(sum, UL0(RW + 1));
            sum = add(sum, UL1(0));
            sum = add(sum, UL1(1));
            sum = add(sum, UL1(RW));
            sum = add(sum, UL1(RW + 1));
            cell.ub = scl(0.125, sum);
            cell.r = ddiv(qm, qv);
        }
        me[oC(PAR, 0)] = cell.r;
        me[oC(PAR, 1)] = cell.e1;
        st3r(me, oC(PAR, 2), PL, cell.ub);
        // ribbons (see kr_cells for the sharing rule) and moved faces
        const double z0 = zt(tau), z1 = zt(tau + 1);
        const D3 T0 = D3{tx0, ty0, z0}, T1 = D3{tx0, ty0, z1};
        double rxz = 0.0, ryz = 0.0, rzy = 0.0, rzx = 0.0;
        rxy_n = 0.0;
        ryx_n = 0.0;
        sx = sy = sz = 0.0;
        if (rib_on && tau + 1 >= 0 && tau + 1 <= p.nz) {
            const D3 L1 = XL1(0);
            if (j + 1 <= p.ny) rxy_n = fs(T1, L1, XL1(RW), D3{tx0, ty1, z1});   // Rxy(i,j,tau+1)
            if (i + 1 <= p.nx) ryx_n = fs(T1, D3{tx1, ty0, z1}, XL1(1), L1);    // Ryx(i,j,tau+1)
        }
        if (rib_on && tau >= 0 && tau < p.nz) {
            const D3 L0 = XL0(0), L1 = XL1(0);
            rxz = fs(T0, T1, L1, L0);
            ryz = fs(T0, L0, L1, T1);
            if (j + 1 <= p.ny) {
                rzy = fs(T0, D3{tx0, ty1, z0}, XL0(RW), L0);  // Rzy(i,j,tau)
                sx = fs(L0, XL0(RW), XL1(RW), L1);             // moved x-face
            }
            if (i + 1 <= p.nx) {
                rzx = fs(T0, L0, XL0(1), D3{tx1, ty0, z0});   // Rzx(i,j,tau)
                sy = fs(L0, L1, XL1(1), XL0(1));               // moved y-face
            }
            if (i + 1 <= p.nx && j + 1 <= p.ny) sz = fs(L0, XL0(1), XL0(RW + 1), XL0(RW));  // moved z-face
        }
        me[oR(PAR, 0)] = rxz;
        me[oR(PAR, 1)] = ryz;
        me[oR(PAR, 2)] = rzy;
        me[oR(PAR, 3)] = rzx;
    }

    // B(t): swept volumes and fluxes of plane t (reads A(t) data of parity PAR)
    template <int PAR>
    __device__ __forceinline__ void stageB(int t, Flux& fzt)
    {
        Flux fx = Flux{0.0, 0.0, D3{0.0, 0.0, 0.0}}, fy = fx;
        fzt = fx;
        const bool do_x = xface_on && t >= 0 && t < p.nz && t >= za && t <= zb;
        const bool do_y = yface_on && t >= 0 && t < p.nz && t >= za && t <= zb;
        const bool do_z = zface_on && t >= 1 && t <= p.nz - 1 && t >= za;
        if (do_x) {
            const double dV = ddiv(((((me[RW + oR(PAR, 0)] - me[oR(PAR, 0)]) + rxy_t1) - rxy_t) + sLx) - sTx, 3.0);
            const double* L = me - 1;
            fx = flux(dV, Cell{L[oC(PAR, 0)], L[oC(PAR, 1)], ld3r(L, oC(PAR, 2), PL)}, c_t);
        }
        if (do_y) {
            const double dV = ddiv(((((ryx_t1 - ryx_t) + me[1 + oR(PAR, 1)]) - me[oR(PAR, 1)]) + sLy) - sTy, 3.0);
            const double* L = me - RW;
            fy = flux(dV, Cell{L[oC(PAR, 0)], L[oC(PAR, 1)], ld3r(L, oC(PAR, 2), PL)}, c_t);
        }
        if (do_z) {
            const double dV =
                ddiv(((((me[1 + oR(PAR, 2)] - me[oR(PAR, 2)]) + me[RW + oR(PAR, 3)]) - me[oR(PAR, 3)]) + sLz) - sTz, 3.0);
            fzt = flux(dV, c_tm1, c_t);
        }
        me[oF(PAR, 0, 0)] = fx.mu;
        me[oF(PAR, 0, 1)] = fx.eps;
        st3r(me, oF(PAR, 0, 2), PL, fx.pi);
        me[oF(PAR, 1, 0)] = fy.mu;
        me[oF(PAR, 1, 1)] = fy.eps;
        st3r(me, oF(PAR, 1, 2), PL, fy.pi);
    }

    // C(kc): cell update of plane kc = t-1 (reads B(t-1) fluxes of parity PAR)
    template <int PAR>
    __device__ __forceinline__ void stageC(int kc, const Flux& fz_lo, const Flux& fz_hi)
    {
        if (!(upd_on && kc >= za && kc <= zb && kc >= 0 && kc < p.nz)) return;
        const double* own = me;
        const double* xp = me + 1;
        const double* yp = me + RW;
        const double mu[6] = {own[oF(PAR, 0, 0)], xp[oF(PAR, 0, 0)], own[oF(PAR, 1, 0)], yp[oF(PAR, 1, 0)], fz_lo.mu,
                              fz_hi.mu};
        const double ep[6] = {own[oF(PAR, 0, 1)], xp[oF(PAR, 0, 1)], own[oF(PAR, 1, 1)], yp[oF(PAR, 1, 1)], fz_lo.eps,
                              fz_hi.eps};
        const D3 pi[6] = {ld3r(own, oF(PAR, 0, 2), PL), ld3r(xp, oF(PAR, 0, 2), PL), ld3r(own, oF(PAR, 1, 2), PL),
                          ld3r(yp, oF(PAR, 1, 2), PL), fz_lo.pi, fz_hi.pi};
        const double dm = ((((mu[0] - mu[1]) + mu[2]) - mu[3]) + mu[4]) - mu[5];
        const double dE = ((((ep[0] - ep[1]) + ep[2]) - ep[3]) + ep[4]) - ep[5];
        const D3 dP = sub(add(sub(add(sub(pi[0], pi[1]), pi[2]), pi[3]), pi[4]), pi[5]);
        const double m2 = m_tm1 + dm;
        if (kc >= s.k0 && kc < s.k1 && !(m2 > 0.0))
            atomicMin(&s.st->err_key, (ERR_ORDER_NEGMASS << 48) | (unsigned long long)gcell(p, i, j, kc));
        const long long c = cb + (long long)kc * s.pc;
        s.e[cur ^ 1][c] = e_tm1 + ddiv(dE - (e_tm1 * dm), m2);
        s.m[cur ^ 1][c] = m2;
        s.dm[c] = dm;
        st3(s.dP, c, dP);
    }

    template <int PT>  // PT = t & 1
    __device__ __forceinline__ void step(int t)
    {
        constexpr int PN = PT ^ 1;
        Flux fz_t;
        stageB<PT>(t, fz_t);
        stageC<PN>(t - 1, fz_tm1, fz_t);
        // A(t+1): consume the cell prefetch of plane t+1
        Cell cn;
        double rxy_n, ryx_n, sx, sy, sz;
        const int s1 = (((t + 1) % 3) + 3) % 3, s2 = (((t + 2) % 3) + 3) % 3;
        stageA<PN>(t + 1, s1, s2, cn, rxy_n, ryx_n, sx, sy, sz);
        const double nsT0 = qs0, nsT1 = qs1, nsT2 = qs2, nm = qm, ne = qe;
        put(t + 3);
        fetch_node(t + 4);
        fetch_cell(t + 2);
        // rotate carried state: plane t -> t-1, t+1 -> t
        fz_tm1 = fz_t;
        m_tm1 = m_t;
        e_tm1 = e_t;
        m_t = nm;
        e_t = ne;
        c_tm1 = c_t;
        c_t = cn;
        rxy_t = rxy_t1;
        ryx_t = ryx_t1;
        rxy_t1 = rxy_n;
        ryx_t1 = ryx_n;
        sLx = sx;
        sLy = sy;
        sLz = sz;
        sTx = nsT0;
        sTy = nsT1;
        sTz = nsT2;
        __syncthreads();
    }

    __device__ __forceinline__ void run()
    {
        // prologue: node planes za-1, za staged; cell za-1 and node plane za+1 prefetched
        fetch_node(za - 1);
        put(za - 1);
        fetch_node(za);
        put(za);
        fetch_cell(za - 1);
        fetch_node(za + 1);
        __syncthreads();
        // A(za-1) (step za-2 would also run B(za-2), C(za-3): nothing to do there)
        {
            Cell cn;
            double rxy_n, ryx_n, sx, sy, sz;
            const int s0 = (((za - 1) % 3) + 3) % 3, s1 = ((za % 3) + 3) % 3;
            if ((za - 1) & 1) stageA<1>(za - 1, s0, s1, cn, rxy_n, ryx_n, sx, sy, sz);
            else stageA<0>(za - 1, s0, s1, cn, rxy_n, ryx_n, sx, sy, sz);
            c_t = cn;
            c_tm1 = Cell{0.0, 0.0, D3{0.0, 0.0, 0.0}};
            m_t = qm;
            e_t = qe;
            m_tm1 = e_tm1 = 0.0;
            sTx = qs0;
            sTy = qs1;
            sTz = qs2;
            rxy_t = ryx_t = 0.0;
            rxy_t1 = rxy_n;
            ryx_t1 = ryx_n;
            sLx = sx;
            sLy = sy;
            sLz = sz;
            fz_tm1 = Flux{0.0, 0.0, D3{0.0, 0.0, 0.0}};
            put(za + 1);
            fetch_node(za + 2);
            fetch_cell(za);
            __syncthreads();
        }
        // steps t = za-1 .. zb+1 (carried state now describes plane t = za-1)
        for (int t = za - 1; t <= zb + 1; ++t) {
            if (t & 1) step<1>(t);
            else step<0>(t);
        }
    }
};

template <int NW, int MB>
__global__ void __launch_bounds__(RW * NW, MB) kr_cells_p(Slab s, Phys p, int cur, int kr0, int kr1, int zchunk)
{
    if (!s.st->active) return;
    extern __shared__ double smem[];
    RemapCellsP<NW> c(s, p, cur, smem, kr0, kr1, zchunk);
    c.run();
}

// ============================================================================
// kr_nodes: node planes [k0, k1] + dt candidate of cells [k0, k1).  Columns i = i0-1+ix.
// ============================================================================
template <int NW>
struct RemapNodesCTA {
    static constexpr int PL = NW * RW, TX = RW - 2, TY = NW - 2;
    __host__ __device__ static constexpr int oU(int par, int c) { return (par * 5 + c) * PL; }  // dm, dP(3), m''
    __host__ __device__ static constexpr int oV(int par) { return 10 * PL + par * PL; }         // |u''|^2
    static constexpr int WORDS = 12 * PL + 2 * RPAD;

    const Slab& s;
    const Phys& p;
    const int cur;
    double* me;
    int i, j, za, zb, zlast;
    long long nb, cb;
    bool col_in, cell_col, node_calc, node_out, dt_col, pxm, pxp, pym, pyp;
    unsigned long long key;
    double qdm, qm2, qe2, qvt;
    D3 qdp, qu1;
    double l2;

    __device__ __forceinline__ RemapNodesCTA(const Slab& s_, const Phys& p_, int cur_, double* smem, int zchunk)
        : s(s_), p(p_), cur(cur_)
    {
        const int ix = threadIdx.x, iy = threadIdx.y;
        me = smem + RPAD + iy * RW + ix;
        i = blockIdx.x * TX - 1 + ix;
        j = blockIdx.y * TY - 1 + iy;
        za = s.k0 + blockIdx.z * zchunk;
        zb = za + zchunk - 1 < s.k1 ? za + zchunk - 1 : s.k1;   // node planes written [za, zb]
        zlast = zb + 1 <= s.k1 ? zb + 1 : s.k1;                  // node planes computed [za, zlast]
        nb = (long long)i + (long long)(p.nx + 1) * (j - (long long)(p.ny + 1) * s.kb);
        cb = (long long)i + (long long)p.nx * (j - (long long)p.ny * s.kb);
        col_in = i >= 0 && i <= p.nx && j >= 0 && j <= p.ny;
        cell_col = i >= 0 && i < p.nx && j >= 0 && j < p.ny;
        const bool in_x = ix >= 1 && ix <= TX, in_y = iy >= 1 && iy <= TY;
        node_calc = col_in && ix >= 1 && iy >= 1;   // nodes [i0, i0+TX] (the last is the neighbour's)
        node_out = node_calc && in_x && in_y;        // nodes owned by this CTA
        dt_col = cell_col && in_x && in_y;
        pxm = i >= 1 && i <= p.nx;
        pxp = i >= 0 && i < p.nx;
        pym = j >= 1 && j <= p.ny;
        pyp = j >= 0 && j < p.ny;
        key = KEY_NONE;
        // c.5 on the target mesh: every edge of cell (i,j) along a is (X_{i+1}-X_i, 0, 0) etc.
        l2 = 0.0;
        if (dt_col) {
            D3 a = D3{s.Xt[i], s.Yt[j], 0.0}, b = D3{s.Xt[i + 1], s.Yt[j + 1], 0.0};
            const double lx = len2(D3{a.x, 0.0, 0.0}, D3{b.x, 0.0, 0.0});
            const double ly = len2(D3{0.0, a.y, 0.0}, D3{0.0, b.y, 0.0});
            l2 = dmin(lx, ly);
        }
    }

    __device__ __forceinline__ void fetch(int k)  // cell plane k (Delta m, Delta P, m''), node plane k (u'), cell k-1 (e'', V^T)
    {
        qdm = 0.0;
        qm2 = 0.0;
        qdp = D3{0.0, 0.0, 0.0};
        if (cell_col && k >= 0 && k < p.nz) {
            long long c = cb + (long long)k * s.pc;
            qdm = s.dm[c];
            qdp = ld3(s.dP, c);
            qm2 = s.m[cur ^ 1][c];
        }
        qu1 = D3{0.0, 0.0, 0.0};
        if (col_in && k >= 0 && k <= p.nz) qu1 = ld3(s.u1, nb + (long long)k * s.pn);
        qe2 = 0.0;
        qvt = 1.0;
        const int kc = k - 1;
        if (dt_col && kc >= 0 && kc < p.nz) {
            long long c = cb + (long long)kc * s.pc;
            qe2 = s.e[cur ^ 1][c];
            qvt = s.VT[c];
        }
    }

    // c.4 step 4: D_m, D_P, M'' sums over the present cells in gather order
    template <int B0, bool ALL>
    __device__ __forceinline__ void gather(double& Dm, D3& DP, double& M2, bool pzm, bool pzp, bool) const
    {
        constexpr int B1 = B0 ^ 1;
        Dm = 0.0;
        M2 = 0.0;
        DP = D3{0.0, 0.0, 0.0};
        bool first = true;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const int ap = g & 1, bp = (g >> 1) & 1, cp = g >> 2;
            const int off = (ap ? 0 : -1) + (bp ? 0 : -RW);
            const int PAR = cp ? B0 : B1;
            const double dm = me[off + oU(PAR, 0)];
            const D3 dp = ld3r(me + off, oU(PAR, 1), PL);
            const double mm = me[off + oU(PAR, 4)];
            if (ALL) {
                Dm = g == 0 ? dm : Dm + dm;
                DP = g == 0 ? dp : add(DP, dp);
                M2 = g == 0 ? mm : M2 + mm;
            } else {
                const bool pres = (ap ? pxp : pxm) && (bp ? pyp : pym) && (cp ? pzp : pzm);
                if (pres) {
                    Dm = first ? dm : Dm + dm;
                    DP = first ? dp : add(DP, dp);
                    M2 = first ? mm : M2 + mm;
                    first = false;
                }
            }
        }
    }

    template <int B0>
    __device__ __forceinline__ void step(int kz)
    {
        constexpr int B1 = B0 ^ 1;
        // ---- P1: stage cell plane kz
        me[oU(B0, 0)] = qdm;
        st3r(me, oU(B0, 1), PL, qdp);
        me[oU(B0, 4)] = qm2;
        const D3 u1 = qu1;
        const double e2 = qe2, vt = qvt;
        if (kz < zlast) fetch(kz + 1);
        __syncthreads();
        // ---- P2: node (i,j,kz)
        if (node_calc && kz >= za) {
            const bool pzm = kz >= 1, pzp = kz < p.nz;
            double Dm, M2;
            D3 DP;
            if (pxm && pxp && pym && pyp && pzm && pzp) gather<B0, true>(Dm, DP, M2, true, true, true);
            else gather<B0, false>(Dm, DP, M2, pzm, pzp, false);
            Dm = 0.125 * Dm;
            DP = scl(0.125, DP);
            M2 = 0.125 * M2;
            D3 un = d3(u1.x + ddiv(DP.x - (u1.x * Dm), M2), u1.y + ddiv(DP.y - (u1.y * Dm), M2),
                       u1.z + ddiv(DP.z - (u1.z * Dm), M2));
            un = reflect(p, i, j, kz, un);
            if (node_out && kz <= zb) st3(s.u[cur ^ 1], nb + (long long)kz * s.pn, un);
            me[oV(B0)] = speed2(un);
        }
        __syncthreads();
        // ---- P3: dt candidate of cell (i,j,kz-1) on the target mesh
        const int kc = kz - 1;
        if (dt_col && kc >= za && kc <= zb && kc < s.k1) {
            double v2 = me[oV(B1)];
            v2 = dmax(v2, me[1 + oV(B1)]);
            v2 = dmax(v2, me[RW + oV(B1)]);
            v2 = dmax(v2, me[RW + 1 + oV(B1)]);
            v2 = dmax(v2, me[oV(B0)]);
            v2 = dmax(v2, me[1 + oV(B0)]);
            v2 = dmax(v2, me[RW + oV(B0)]);
            v2 = dmax(v2, me[RW + 1 + oV(B0)]);
            const double lz = len2(D3{0.0, 0.0, s.Zt[kc - s.kb]}, D3{0.0, 0.0, s.Zt[kc + 1 - s.kb]});
            const double m2 = me[oU(B1, 4)];
            double rho = ddiv(m2, vt), pr, pf, cs;
            eos(p.gamma, rho, e2, pr, pf, cs);
            const unsigned long long kk = dt_key(dt_cell(p.cfl, dmin(l2, lz), v2, cs));
            key = kk < key ? kk : key;
        }
        __syncthreads();
    }

    __device__ __forceinline__ void run()
    {
        fetch(za - 1);
        // stage cell plane za-1 directly (B parity of za-1)
        if ((za - 1) & 1) {
            me[oU(1, 0)] = qdm;
            st3r(me, oU(1, 1), PL, qdp);
            me[oU(1, 4)] = qm2;
        } else {
            me[oU(0, 0)] = qdm;
            st3r(me, oU(0, 1), PL, qdp);
            me[oU(0, 4)] = qm2;
        }
        fetch(za);
        for (int kz = za; kz <= zlast; ++kz) {
            if (kz & 1) step<1>(kz);
            else step<0>(kz);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
            key = other < key ? other : key;
        }
        __shared__ unsigned long long red[32];
        if (threadIdx.x == 0) red[threadIdx.y] = key;
        __syncthreads();
        if (threadIdx.y == 0) {
            key = threadIdx.x < NW ? red[threadIdx.x] : KEY_NONE;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
                key = other < key ? other : key;
            }
            if (threadIdx.x == 0 && key != KEY_NONE) atomicMin(&s.st->cand_key, key);
        }
    }
};

template <int NW>
__global__ void __launch_bounds__(RW * NW, 2) kr_nodes(Slab s, Phys p, int cur, int zchunk)
{
    if (!s.st->active) return;
    extern __shared__ double smem[];
    RemapNodesCTA<NW> c(s, p, cur, smem, zchunk);
    c.run();
}

// ============================================================================
// kn_update / kn_dt: R4 and the Euler dt candidate as two barrier-free kernels
// (one thread per node / per cell, operands through L1; high occupancy).
// ============================================================================
// grid: x = ceil((nx+1)(ny+1) / 256) (flattened node plane: no idle lanes), y = planes
template <bool TILE>  // TILE: 32 x 8 node tiles (grid x = x-tiles * y-tiles) instead of flattened rows
// spd = 1: also store |u''|^2 per node for kn_dt (only when kn_dt runs)
// (8 CTAs per SM at 32 registers, as kn_force_e: more warps for the latency-bound gather)
__global__ void __launch_bounds__(256, 8) kn_update(Slab s, Phys p, int cur, int spd)
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
    const int k = s.k0 + blockIdx.y;
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
    if (spd) s.x1[0][n] = speed2(un);  // |u''|^2 (x' scratch is free after the remap's cell kernels)
}

// grid: x = ceil(nx*ny / 256) (flattened cell plane), y = owned cell planes
__global__ void __launch_bounds__(256) kn_dt(Slab s, Phys p, int cur)
{
    if (!s.st->active) return;
    const int t = blockIdx.x * 256 + threadIdx.x, k = s.k0 + blockIdx.y;
    unsigned long long key = KEY_NONE;
    if (t < (int)s.pc) {
        const int i = t % p.nx, j = t / p.nx;
        const long long n0 = (long long)i + (long long)(p.nx + 1) * ((long long)j + (long long)(p.ny + 1) * (k - s.kb));
        const int pn = (p.nx + 1) * (p.ny + 1), rw = p.nx + 1;
        const double* __restrict__ v = s.x1[0] + n0;
        double v2 = __ldg(v);
        v2 = dmax(v2, __ldg(v + 1));
        v2 = dmax(v2, __ldg(v + rw));
        v2 = dmax(v2, __ldg(v + rw + 1));
        v2 = dmax(v2, __ldg(v + pn));
        v2 = dmax(v2, __ldg(v + pn + 1));
        v2 = dmax(v2, __ldg(v + pn + rw));
        v2 = dmax(v2, __ldg(v + pn + rw + 1));
        const long long c = (long long)t + s.pc * (long long)(k - s.kb);
        double rho = ddiv(s.m[cur ^ 1][c], s.VT[c]), pr, pf, cs;
        eos(p.gamma, rho, s.e[cur ^ 1][c], pr, pf, cs);
        // c.5 on the target mesh: cfl * sqrt(min of the 12 axis-aligned edges^2) as the
        // min of the per-axis tabled factors (monotone maps: same bits)
        const double num = dmin(dmin(s.TDx[i], s.TDy[j]), s.TDz[k - s.kb]);
        key = dt_key(ddiv(num, (cs + dsqrt(v2)) + 1e-30));
    }
    block_min_atomic(key, &s.st->cand_key);
}

// ============================================================================
// kr_sweep + kr_flux: the remap as two lean kernels (the alternative to the
// pipelined kr_cells_p, whose carried state spills).
//
//   kr_sweep : z-march over cell planes; stages x', u' node planes; per column
//              and plane the six ribbons and three moved faces of c.4 step 1
//              (ribbons shared with the neighbouring faces as in kr_cells), the
//              swept volumes dV of the cell's -x/-y/-z faces, and the donor data
//              r = m/V', Ubar = 8-node mean of u' (c.4 step 2).  Writes
//              Slab::dV, rD, UD.  Dependencies reach only the +x / +y neighbours,
//              so a 32 x NW tile yields 31 x (NW-1) columns.
//   kr_flux  : one thread per cell: the six face fluxes from dV and the donor
//              data (c.4 step 2), the cell update (c.4 step 3).
// Same expressions, operands and association as kr_cells / the oracle.
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
        ta = t0 + blockIdx.z * zchunk;
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
        // x' = x^T + u' dt, kn_force_e's expression (c.3 step 6), formed when staged
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

// grid: x = ceil(nx / 32), y = ceil(ny / 8), z = cell planes [kr0, kr1)
// All loads are independent of the swept volumes' signs (both candidate donors of
// every face are loaded, the donor is selected afterwards), so they overlap.
#ifndef KR_FLUX_MB
#define KR_FLUX_MB 3
#endif
struct Donor {
    double r, e;
    D3 u;
};
__device__ __forceinline__ Donor donor_at(const Slab& s, long long d)
{
    return Donor{s.rD[d], s.e1[d], ld3(s.UD, d)};
}
__global__ void __launch_bounds__(256, KR_FLUX_MB) kr_flux(Slab s, Phys p, int cur, int kr0)
{
    if (!s.st->active) return;
    const int i = blockIdx.x * 32 + threadIdx.x, j = blockIdx.y * 8 + threadIdx.y, t = kr0 + blockIdx.z;
    if (i >= p.nx || j >= p.ny) return;
    const long long c = (long long)i + (long long)p.nx * ((long long)j + (long long)p.ny * (t - s.kb));
    const long long sa[3] = {1, p.nx, s.pc};
    const int ia[3] = {i, j, t}, na[3] = {p.nx, p.ny, p.nz};
    const Donor own = donor_at(s, c);
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
        const Donor& D = (dV > 0.0) == plus ? own : other;
        mu[f] = inner ? D.r * dV : 0.0;
        ep[f] = inner ? mu[f] * D.e : 0.0;
        pi[f] = inner ? scl(mu[f], D.u) : D3{0.0, 0.0, 0.0};
    }
    const double dm = ((((mu[0] - mu[1]) + mu[2]) - mu[3]) + mu[4]) - mu[5];
    const double dE = ((((ep[0] - ep[1]) + ep[2]) - ep[3]) + ep[4]) - ep[5];
    const D3 dP = sub(add(sub(add(sub(pi[0], pi[1]), pi[2]), pi[3]), pi[4]), pi[5]);
    const double m = s.m[cur][c], e1 = own.e;
    const double m2 = m + dm;
    if (t >= s.k0 && t < s.k1 && !(m2 > 0.0))
        atomicMin(&s.st->err_key, (ERR_ORDER_NEGMASS << 48) | (unsigned long long)gcell(p, i, j, t));
    s.e[cur ^ 1][c] = e1 + ddiv(dE - (e1 * dm), m2);
    s.m[cur ^ 1][c] = m2;
    s.dm[c] = dm;
    st3(s.dP, c, dP);
}

// ============================================================================
namespace {
inline int cdivr(int a, int b) { return (a + b - 1) / b; }
constexpr int NW_RC = 8, NW_RN = 8, RZ = 32;
}  // namespace

template <int NW, int MB>
static void cells_p_launch(const Slab& s, const Phys& p, int cur, int kr0, int kr1, cudaStream_t cs)
{
    const size_t sm = sizeof(double) * RemapCellsP<NW>::WORDS;
    static bool init = false;
    if (!init) {
        cudaFuncSetAttribute(kr_cells_p<NW, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        init = true;
    }
    const int zc = zchunk_for((long long)cdivr(p.nx, RW - 3) * cdivr(p.ny, NW - 3), kr1 - kr0, RZ);

    dim3 grid(cdivr(p.nx, RW - 3), cdivr(p.ny, NW - 3), cdivr(kr1 - kr0, zc));
    kr_cells_p<NW, MB><<<grid, dim3(RW, NW), sm, cs>>>(s, p, cur, kr0, kr1, zc);
}

// multi-material cells: kr_sweep with the per-material donor densities (Slab::rDm)
int launch_sweep_mat(const Slab& s, const Phys& p, int cur, Stream st)
{
    const int kr0 = s.k0 - 1 > 0 ? s.k0 - 1 : 0, kr1 = s.k1 + 1 < p.nz ? s.k1 + 1 : p.nz;
    auto sweep = [&](auto kern) {
        static bool init = false;
        const size_t words = SweepCTA<8>::WORDS;
        if (!init) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(double) * words));
            init = true;
        }
        const int t0 = kr0 - 1 > 0 ? kr0 - 1 : 0, t1 = kr1 < p.nz - 1 ? kr1 : p.nz - 1;
        const int zc = zchunk_for((long long)cdivr(p.nx, RW - 1) * cdivr(p.ny, 8 - 1), t1 - t0 + 1, RZ);
        dim3 grid(cdivr(p.nx, RW - 1), cdivr(p.ny, 8 - 1), cdivr(t1 - t0 + 1, zc));
        kern<<<grid, dim3(RW, 8), sizeof(double) * words, (cudaStream_t)st>>>(s, p, cur, kr0, kr1, zc);
    };
    switch (s.nmat) {
    case 1: sweep(kr_sweep<8, 2, 1>); break;
    case 2: sweep(kr_sweep<8, 2, 2>); break;
    case 3: sweep(kr_sweep<8, 2, 3>); break;
    default: sweep(kr_sweep<8, 2, 4>); break;
    }
    return 1;
}

// R4 node momentum update on the cell totals (the material path reuses it)
int launch_kn_update(const Slab& s, const Phys& p, int cur, Stream st)
{
    kn_update<true><<<dim3(cdivr(p.nx + 1, 32) * cdivr(p.ny + 1, 8), s.k1 - s.k0 + 1), 256, 0, (cudaStream_t)st>>>(
        s, p, cur, 0);
    return 1;
}

int launch_remap_fused(const Slab& s, const Phys& p, int cur, Stream st)
{
    cudaStream_t cs = (cudaStream_t)st;
    const int kr0 = s.k0 - 1 > 0 ? s.k0 - 1 : 0, kr1 = s.k1 + 1 < p.nz ? s.k1 + 1 : p.nz;
    static const int variant = [] {
        const char* v = getenv("SALE_REMAP");
        return v ? atoi(v) : 7;
    }();
    if (variant == 0) {
        constexpr int NW = NW_RC;
        const size_t sm = sizeof(double) * RemapCellsCTA<NW>::WORDS;
        static bool init = false;
        if (!init) {
            cudaFuncSetAttribute(kr_cells<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            init = true;
        }
        const int zc = zchunk_for((long long)cdivr(p.nx, RW - 3) * cdivr(p.ny, NW - 3), kr1 - kr0, RZ);

        dim3 grid(cdivr(p.nx, RW - 3), cdivr(p.ny, NW - 3), cdivr(kr1 - kr0, zc));
        kr_cells<NW><<<grid, dim3(RW, NW), sm, cs>>>(s, p, cur, kr0, kr1, zc);
    } else if (variant == 7) {  // default: kr_sweep + kr_flux
        auto sweep = [&](auto kern, int nw, size_t words) {
            static bool init = false;
            if (!init) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(double) * words));
                init = true;
            }
            const int t0 = kr0 - 1 > 0 ? kr0 - 1 : 0, t1 = kr1 < p.nz - 1 ? kr1 : p.nz - 1;
            const int zc = zchunk_for((long long)cdivr(p.nx, RW - 1) * cdivr(p.ny, nw - 1), t1 - t0 + 1, RZ);

            dim3 grid(cdivr(p.nx, RW - 1), cdivr(p.ny, nw - 1), cdivr(t1 - t0 + 1, zc));
            kern<<<grid, dim3(RW, nw), sizeof(double) * words, cs>>>(s, p, cur, kr0, kr1, zc);
        };
        // (with kx_energy_sweep the swept volumes and donor data came with the energy kernel)
        if (euler_esweep_variant() == 0) sweep(kr_sweep<8, 2>, 8, SweepCTA<8>::WORDS);
        kr_flux<<<dim3(cdivr(p.nx, 32), cdivr(p.ny, 8), kr1 - kr0), dim3(32, 8), 0, cs>>>(s, p, cur, kr0);
    } else {  // SALE_REMAP=6: the one-kernel software-pipelined remap
        cells_p_launch<15, 1>(s, p, cur, kr0, kr1, cs);
    }
    static const int nvariant = [] {
        const char* v = getenv("SALE_RNODES");
        return v ? atoi(v) : 1;
    }();
    if (nvariant == 0) {
        constexpr int NW = NW_RN;
        const size_t sm = sizeof(double) * RemapNodesCTA<NW>::WORDS;
        static bool init = false;
        if (!init) {
            cudaFuncSetAttribute(kr_nodes<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            init = true;
        }
        const int zc = zchunk_for((long long)cdivr(p.nx + 1, RW - 2) * cdivr(p.ny + 1, NW - 2), s.k1 - s.k0 + 1, RZ);

        dim3 grid(cdivr(p.nx + 1, RW - 2), cdivr(p.ny + 1, NW - 2), cdivr(s.k1 - s.k0 + 1, zc));
        kr_nodes<NW><<<grid, dim3(RW, NW), sm, cs>>>(s, p, cur, zc);
    } else {
        // 32 x 8 node tiles: the gathered cell values are reused inside a block through L1
        // (measured faster than full-lane flattened rows despite the ragged last tile)
        kn_update<true><<<dim3(cdivr(p.nx + 1, 32) * cdivr(p.ny + 1, 8), s.k1 - s.k0 + 1), 256, 0, cs>>>(
            s, p, cur, euler_pre_sigma() ? 0 : 1);
        if (euler_pre_sigma()) return 3;  // the next cycle's kf_sigma_e evaluates the dt candidate
        kn_dt<<<dim3(cdivr((int)s.pc, 256), s.k1 - s.k0), 256, 0, cs>>>(s, p, cur);
        return 4;
    }
    return 2;
}

}  // namespace sale
