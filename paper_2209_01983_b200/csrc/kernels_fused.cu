// kernels_fused.cu -- the fused Lagrangian phase as two z-marching kernels.
//
// Each CTA owns an x-y tile of columns and marches along z (2.5D): node planes
// are loaded once from HBM (coalesced, one warp per x-row of 32 columns; the
// loads for plane k+1 are issued one step ahead into registers), staged in
// shared memory, and every face quantity is computed ONCE per CTA and shared
// by the cells / nodes that use it:
//
//   kf_force  : S1 geometry at t^n (three faces anchored at each column), S2
//               EoS, S3 viscosity -> sigma; S5 corner forces gathered in the
//               fixed order of c.2; S6 kinematics + reflecting BC.  Writes u',
//               x' (Euler: u', x' to scratch) and sigma.
//   kf_energy : S7 geometry at t^{n+1} (V', tangle check), compatible pdV
//               energy, and (Lagrange) the next cycle's dt candidate: running
//               min per thread, warp-shuffle + block min, one atomicMin per CTA.
//
// The arithmetic of every quantity is the expression tree of SURVEY §8(c)
// with the association of the oracle and the v0 kernels, so results are
// bit-identical; only the operand sources (registers / shared memory instead
// of recomputation) differ.
//
// Performance structure: the plane parity is a template parameter of the step
// function, so every shared-memory access is a per-thread base pointer plus an
// immediate offset (no integer index arithmetic in the inner loop); the smem
// window is padded by one row+column on both sides so neighbour reads never
// need clamping; cell presence in the node gather is a predicate, not a branch.
#include <cuda_runtime.h>

#include <type_traits>

#include <cstdio>
#include <cstdlib>

#include "sale_mesh.cuh"

namespace sale {

bool fused_available() { return true; }

namespace {

constexpr int FW = 32;   // columns per warp row
constexpr int MINB = 2;  // resident CTAs per SM the register budget is sized for
constexpr int PAD = FW + 1;

inline int imin_h(int a, int b) { return a < b ? a : b; }
inline int imax_h(int a, int b) { return a > b ? a : b; }

struct FaceQ {
    D3 A, Xb, Ub;
    double s;
};
__device__ __forceinline__ FaceQ faceq(D3 P0, D3 P1, D3 P2, D3 P3, D3 U0, D3 U1, D3 U2, D3 U3)
{
    FaceQ f;
    f.A = face_area(P0, P1, P2, P3);
    f.Xb = avg4(P0, P1, P2, P3);
    f.s = face_s(f.Xb, f.A);
    f.Ub = avg4(U0, U1, U2, U3);
    return f;
}

__device__ __forceinline__ D3 ld3s(const double* b, int o0, int stride) { return D3{b[o0], b[o0 + stride], b[o0 + 2 * stride]}; }
__device__ __forceinline__ void st3s(double* b, int o0, int stride, D3 v)
{
    b[o0] = v.x;
    b[o0 + stride] = v.y;
    b[o0 + 2 * stride] = v.z;
}

}  // namespace

// Euler: does any active kernel load x' from memory?  The default path forms it from
// u' (kf_energy_e, kr_sweep); SALE_ESWEEP=1 (kx_energy_sweep), SALE_REMAP != 7
// (kr_cells / kr_cells_p) and SALE_MAT_V0=1 (k_mat_energy / k_mat_sweep) load it.
bool euler_x1_stored()
{
    static const bool v = [] {
        auto env = [](const char* n, int d) {
            const char* e = getenv(n);
            return e ? atoi(e) : d;
        };
        return env("SALE_ESWEEP", 0) > 0 || env("SALE_REMAP", 7) != 7 || env("SALE_MAT_V0", 0) == 1;
    }();
    return v;
}

// ============================================================================
// kf_force
// ============================================================================
// NM > 0 (Lagrange, multi-material cells): sigma from the mixed
// closure MM1 of the NM materials (always from V; the single-material EoS cache does
// not apply), and q is stored for the materials' energy update (k_mat_energy)
template <bool EULER, int NW, int NM = 0>
struct ForceCTA {
    static constexpr int PL = NW * FW, TX = FW - 2, TY = NW - 2;
    // shared-memory words (doubles) relative to the per-thread base pointer
    __host__ __device__ static constexpr int oN(int par, int c) { return (par * 6 + c) * PL; }          // node x,y,z,ux,uy,uz
    __host__ __device__ static constexpr int oQ(int xy, int c) { return 12 * PL + (xy * 7 + c) * PL; }  // face s, Xb, Ub
    __host__ __device__ static constexpr int oA(int par, int xy) { return 26 * PL + (par * 2 + xy) * 3 * PL; }  // x/y face A
    __host__ __device__ static constexpr int oZ(int par) { return 38 * PL + par * 3 * PL; }            // z-face A
    __host__ __device__ static constexpr int oS(int par, int c) { return 44 * PL + (par * 2 + c) * PL; }  // sigma, m
    static constexpr int WORDS = 48 * PL + 2 * PAD;

    const Slab& s;
    const Phys& p;
    const int cur;
    double* me;
    int i, j, za, zb, kn0, kn1;
    int swlo, sw1;     // this CTA writes sigma of cell planes [swlo, sw1)
    long long nb, cb;  // node / cell index of (i,j) at local plane 0
    double dt;
    bool col_in, cellcol_in, node_out, sig_col;
    bool pxm, pxp, pym, pyp;
    D3 px, pu;  // prefetch registers
    double pm, pe, prho, pcs;  // prefetch: cell m, e and (owned planes) the EoS cache
    double pmf[NM > 0 ? NM : 1], pmm[NM > 0 ? NM : 1], pme[NM > 0 ? NM : 1];  // prefetch: materials
    FaceQ zprev;

    // sigma is written for cell planes [sw0, sw1) (kf_force's launch range: [kn0, kn1);
    // a split range also writes the cell just outside it, launch_lagrange_fused_part):
    // each cell by the z-chunk that owns it, the first chunk also owning cell kn0-1
    __device__ __forceinline__ ForceCTA(const Slab& s_, const Phys& p_, int cur_, double* smem, int kn0_, int kn1_,
                                        int zchunk, int sw0_, int sw1_)
        : s(s_), p(p_), cur(cur_)
    {
        const int ix = threadIdx.x, iy = threadIdx.y;
        me = smem + PAD + iy * FW + ix;
        i = blockIdx.x * TX - 1 + ix;
        j = blockIdx.y * TY - 1 + iy;
        kn0 = kn0_;
        kn1 = kn1_;
        za = kn0 + blockIdx.z * zchunk;
        zb = za + zchunk - 1 < kn1 ? za + zchunk - 1 : kn1;
        swlo = (za == kn0) ? sw0_ : (za > sw0_ ? za : sw0_);
        sw1 = sw1_;
        nb = (long long)i + (long long)(p.nx + 1) * (j - (long long)(p.ny + 1) * s.kb);
        cb = (long long)i + (long long)p.nx * (j - (long long)p.ny * s.kb);
        dt = s.st->dt;
        col_in = i >= 0 && i <= p.nx && j >= 0 && j <= p.ny;
        cellcol_in = i >= 0 && i < p.nx && j >= 0 && j < p.ny;
        node_out = col_in && ix >= 1 && ix <= TX && iy >= 1 && iy <= TY;
        sig_col = cellcol_in && ix >= 1 && ix <= TX && iy >= 1 && iy <= TY;
        pxm = i >= 1 && i <= p.nx;  // cell i-1 exists
        pxp = i >= 0 && i < p.nx;   // cell i exists
        pym = j >= 1 && j <= p.ny;
        pyp = j >= 0 && j < p.ny;
    }

    // global loads of node plane k and cell (i,j,k-1) into registers
    __device__ __forceinline__ void fetch(int k)
    {
        px = D3{0.0, 0.0, 0.0};
        pu = px;
        if (col_in && k >= 0 && k <= p.nz) {
            long long n = nb + (long long)k * s.pn;
            if (EULER) px = D3{s.Xt[i], s.Yt[j], s.Zt[k - s.kb]};
            else px = ld3(s.x[cur], n);
            pu = ld3(s.u[cur], n);
        }
        pm = 0.0;
        pe = 0.0;
        const int kc = k - 1;
        if (cellcol_in && kc >= 0 && kc < p.nz) {
            long long c = cb + (long long)kc * s.pc;
            pm = mass_cur(s, p, cur)[c];
            pe = s.e[cur][c];
            if (NM == 0 && kc >= s.k0 && kc < s.k1) {
                prho = s.rhoc[c];
                pcs = s.csc[c];
            }
#pragma unroll
            for (int a = 0; a < NM; ++a) {
                pmf[a] = mat_f(s, p, cur)[c + a * mat_stride(s)];
                pmm[a] = mat_m(s, p, cur)[c + a * mat_stride(s)];
                pme[a] = s.me[cur][c + a * mat_stride(s)];
            }
        }
    }
    template <int PAR>
    __device__ __forceinline__ void put()
    {
        st3s(me, oN(PAR, 0), PL, px);
        st3s(me, oN(PAR, 3), PL, pu);
    }
    template <int PAR>
    __device__ __forceinline__ D3 X(int off) const { return ld3s(me + off, oN(PAR, 0), PL); }
    template <int PAR>
    __device__ __forceinline__ D3 U(int off) const { return ld3s(me + off, oN(PAR, 3), PL); }

    template <int PAR>
    __device__ __forceinline__ FaceQ zface() const
    {
        return faceq(X<PAR>(0), X<PAR>(1), X<PAR>(FW + 1), X<PAR>(FW), U<PAR>(0), U<PAR>(1), U<PAR>(FW + 1),
                     U<PAR>(FW));
    }

    // c.3 steps 4-5: F = sum over present cells (gather order) of sigma_K C_K,n; M = sum m_K
    template <int B0, bool ALL>
    __device__ __forceinline__ void gather(D3& F, double& M, bool pxm_, bool pxp_, bool pym_, bool pyp_, bool pzm,
                                           bool pzp) const
    {
        constexpr int B1 = B0 ^ 1;
        F = D3{0.0, 0.0, 0.0};
        M = 0.0;
        bool first = true;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const int ap = g & 1, bp = (g >> 1) & 1, cp = g >> 2;
            const int dx = ap ? 0 : -1, dy = bp ? 0 : -FW;
            const int PAR = cp ? B0 : B1;  // plane parity of cell kz-1+cp
            const D3 Ax = ld3s(me + dy, oA(PAR, 0), PL);   // x-face at node plane i, row j-1+bp
            const D3 Ay = ld3s(me + dx, oA(PAR, 1), PL);   // y-face at node plane j, col i-1+ap
            const D3 Az = ld3s(me + dx + dy, oZ(B0), PL);  // z-face at node plane kz
            const D3 C = add(add(ap ? neg(Ax) : Ax, bp ? neg(Ay) : Ay), cp ? neg(Az) : Az);
            const double sg = me[dx + dy + oS(PAR, 0)];
            const double mk = me[dx + dy + oS(PAR, 1)];
            const D3 term = scl(sg, C);
            if (ALL) {
                F = g == 0 ? term : add(F, term);
                M = g == 0 ? mk : M + mk;
            } else {
                const bool pres = (ap ? pxp_ : pxm_) && (bp ? pyp_ : pym_) && (cp ? pzp : pzm);
                if (pres) {
                    F = first ? term : add(F, term);
                    M = first ? mk : M + mk;
                    first = false;
                }
            }
        }
    }

    template <int B0>
    __device__ __forceinline__ void step(int kz)
    {
        constexpr int B1 = B0 ^ 1;
        // ---- P1: stage node plane kz+1 and cell (i,j,kz); prefetch the next
        put<B1>();
        const double m = pm, e = pe, crho = prho, ccs = pcs;
        double cmf[NM > 0 ? NM : 1], cmm[NM > 0 ? NM : 1], cme[NM > 0 ? NM : 1], pfk[MAX_MAT];
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            cmf[a] = pmf[a];
            cmm[a] = pmm[a];
            cme[a] = pme[a];
        }
        if (kz < zb) fetch(kz + 2);
        __syncthreads();
        // ---- P2: the three faces anchored at this column
        // x-face at node plane i: (i,j,kz) (i,j+1,kz) (i,j+1,kz+1) (i,j,kz+1)
        const FaceQ fx = faceq(X<B0>(0), X<B0>(FW), X<B1>(FW), X<B1>(0), U<B0>(0), U<B0>(FW), U<B1>(FW), U<B1>(0));
        // y-face at node plane j: (i,j,kz) (i,j,kz+1) (i+1,j,kz+1) (i+1,j,kz)
        const FaceQ fy = faceq(X<B0>(0), X<B1>(0), X<B1>(1), X<B0>(1), U<B0>(0), U<B1>(0), U<B1>(1), U<B0>(1));
        // z-face at node plane kz+1
        const FaceQ zn = zface<B1>();
        me[oQ(0, 0)] = fx.s;
        st3s(me, oQ(0, 1), PL, fx.Xb);
        st3s(me, oQ(0, 4), PL, fx.Ub);
        me[oQ(1, 0)] = fy.s;
        st3s(me, oQ(1, 1), PL, fy.Xb);
        st3s(me, oQ(1, 4), PL, fy.Ub);
        st3s(me, oA(B0, 0), PL, fx.A);
        st3s(me, oA(B0, 1), PL, fy.A);
        st3s(me, oZ(B1), PL, zn.A);
        __syncthreads();
        // ---- P3: cell (i,j,kz): V, rho, EoS, q, sigma
        {
            double sig = 0.0;
            if (cellcol_in && kz >= 0 && kz < p.nz) {
                const double* qx = me + 1;   // +x face (anchored at i+1)
                const double* qy = me + FW;  // +y face (anchored at j+1)
                double rho, pf, cs;
                if constexpr (NM > 0) {
                    double sv[6] = {fx.s, qx[oQ(0, 0)], fy.s, qy[oQ(1, 0)], zprev.s, zn.s};
                    double V = vol_from_s(sv), pr;
                    rho = ddiv(m, V);
                    mix_eos_r<NM>(s, cmf, cmm, cme, V, rho, pr, pf, cs, pfk);
                } else if (kz >= s.k0 && kz < s.k1) {  // owned: rho, c from the EoS cache (c.5 pass, same state)
                    rho = crho;
                    cs = ccs;
                    const double pr = ((p.gamma - 1.0) * rho) * e;
                    pf = (pr > 0.0) ? pr : 0.0;
                } else {
                    double sv[6] = {fx.s, qx[oQ(0, 0)], fy.s, qy[oQ(1, 0)], zprev.s, zn.s};
                    double V = vol_from_s(sv), pr;
                    rho = ddiv(m, V);
                    eos(p.gamma, rho, e, pr, pf, cs);
                }
                double dx = axis_jump(fx.Xb, ld3s(qx, oQ(0, 1), PL), fx.Ub, ld3s(qx, oQ(0, 4), PL));
                double dy = axis_jump(fy.Xb, ld3s(qy, oQ(1, 1), PL), fy.Ub, ld3s(qy, oQ(1, 4), PL));
                double dz = axis_jump(zprev.Xb, zn.Xb, zprev.Ub, zn.Ub);
                double du = dmin(dmin(dx, dy), dz);
                double q = q_of_du(rho, cs, du, p.c1, p.c2);
                sig = 0.25 * (pf + q);
                if (sig_col && kz >= swlo && kz < sw1) {
                    s.sig[cb + (long long)kz * s.pc] = sig;
#pragma unroll
                    for (int a = 0; a < NM; ++a)  // each material's stress (MM4)
                        s.sgm[cb + (long long)kz * s.pc + a * mat_stride(s)] = 0.25 * (pfk[a] + q);
                }
            }
            me[oS(B0, 0)] = sig;
            me[oS(B0, 1)] = m;
        }
        zprev = zn;
        __syncthreads();
        // ---- P4: node (i,j,kz): force + mass gather, kinematics, BC, move
        if (node_out && kz >= za) {
            const bool pzm = kz >= 1, pzp = kz < p.nz;
            D3 F;
            double M;
            // interior nodes (all 8 cells present, the common case) take the
            // select-free path; both paths sum in the same gather order
            if (pxm && pxp && pym && pyp && pzm && pzp) gather<B0, true>(F, M, true, true, true, true, true, true);
            else gather<B0, false>(F, M, pxm, pxp, pym, pyp, pzm, pzp);
            M = 0.125 * M;
            const D3 u = U<B0>(0), x = X<B0>(0);
            D3 un = d3(u.x + (ddiv(F.x, M) * dt), u.y + (ddiv(F.y, M) * dt), u.z + (ddiv(F.z, M) * dt));
            un = reflect(p, i, j, kz, un);
            const D3 xn = d3(x.x + (un.x * dt), x.y + (un.y * dt), x.z + (un.z * dt));
            const long long n = nb + (long long)kz * s.pn;
            if (EULER) {
                st3(s.u1, n, un);
                st3(s.x1, n, xn);
            } else {
                st3(s.x[cur ^ 1], n, xn);
                st3(s.u[cur ^ 1], n, un);
            }
        }
    }

    __device__ __forceinline__ void run()
    {
        // prologue: node plane za-1 and its z-faces (the -z faces of cell plane za-1)
        fetch(za - 1);
        if ((za - 1) & 1) put<1>();
        else put<0>();
        fetch(za);
        __syncthreads();
        zprev = ((za - 1) & 1) ? zface<1>() : zface<0>();
        for (int kz = za - 1; kz <= zb; ++kz) {
            if (kz & 1) step<1>(kz);
            else step<0>(kz);
        }
    }
};

template <bool EULER, int NW, int NM = 0>
__global__ void __launch_bounds__(FW * NW, NW >= 12 ? 1 : MINB)
    kf_force(Slab s, Phys p, int cur, int kn0, int kn1, int zchunk, int sw0, int sw1)
{
    if (!s.st->active) return;
    extern __shared__ double smem[];
    ForceCTA<EULER, NW, NM> c(s, p, cur, smem, kn0, kn1, zchunk, sw0, sw1);
    c.run();
}

// ============================================================================
// kf_force, Euler mode: the same computation with the t^n geometry of the fixed
// target mesh taken from the tables built at create (Slab::TAx..TJz, V^T) instead
// of being re-evaluated from x^T every cycle: face area vectors (corner forces),
// cell volume, and the centroid separations of the viscosity (same bits).  Only
// velocities are staged; per column and step the work is the three face-average
// velocities, EoS + q + sigma of one cell, and the force gather of one node.
// ============================================================================
template <int NW>
struct ForceEulerCTA {
    static constexpr int PL = NW * FW, TX = FW - 2, TY = NW - 2;
    __host__ __device__ static constexpr int oU(int par, int c) { return (par * 3 + c) * PL; }         // node u
    __host__ __device__ static constexpr int oW(int xy, int c) { return 6 * PL + (xy * 3 + c) * PL; }    // x/y face Ubar
    __host__ __device__ static constexpr int oA(int par, int xy) { return 12 * PL + (par * 2 + xy) * 3 * PL; }  // x/y face A
    __host__ __device__ static constexpr int oZ() { return 24 * PL; }                                    // z-face A
    __host__ __device__ static constexpr int oS(int par, int c) { return 27 * PL + (par * 2 + c) * PL; }  // sigma, m
    static constexpr int WORDS = 31 * PL + 2 * PAD;

    const Slab& s;
    const Phys& p;
    const int cur;
    double* me;
    int i, j, za, zb, kn0, kn1, ic, jc;  // ic, jc: i, j clamped into the cell range (table indices)
    long long nb, cb, nbc, cbc;  // nbc / cbc: the column clamped into the mesh (always-valid loads)
    double dt;
    bool col_in, cellcol_in, node_out, sig_col;
    bool pxm, pxp, pym, pyp;
    // prefetch registers.  Loads are unconditional (clamped addresses) and the
    // out-of-mesh zero is selected where the value is consumed: a predicated load
    // followed by a default write would make the write wait for the load.
    D3 pu;  // node u of plane k
    double pm, pe, pv;  // cell m, e, V^T of plane k-1
    double pz;          // Z of node plane k
    double xi, yj;      // X_i, Y_j of this column (clamped)
    bool pnok, pcok;
    D3 pax, pay;        // prefetch: x- / y-face area vectors of cell plane k-1 (tables)
    D3 zprev;  // Ubar of the z-face at node plane kz (the -z face of cell kz)
    double zc;  // Z of node plane kz

    __device__ __forceinline__ ForceEulerCTA(const Slab& s_, const Phys& p_, int cur_, double* smem, int kn0_, int kn1_,
                                             int zchunk)
        : s(s_), p(p_), cur(cur_)
    {
        const int ix = threadIdx.x, iy = threadIdx.y;
        me = smem + PAD + iy * FW + ix;
        i = blockIdx.x * TX - 1 + ix;
        j = blockIdx.y * TY - 1 + iy;
        ic = i < 0 ? 0 : (i >= p.nx ? p.nx - 1 : i);
        jc = j < 0 ? 0 : (j >= p.ny ? p.ny - 1 : j);
        kn0 = kn0_;
        kn1 = kn1_;
        za = kn0 + blockIdx.z * zchunk;
        zb = za + zchunk - 1 < kn1 ? za + zchunk - 1 : kn1;
        nb = (long long)i + (long long)(p.nx + 1) * (j - (long long)(p.ny + 1) * s.kb);
        cb = (long long)i + (long long)p.nx * (j - (long long)p.ny * s.kb);
        {
            const int in = i < 0 ? 0 : (i > p.nx ? p.nx : i), jn = j < 0 ? 0 : (j > p.ny ? p.ny : j);
            nbc = (long long)in + (long long)(p.nx + 1) * (jn - (long long)(p.ny + 1) * s.kb);
            cbc = (long long)ic + (long long)p.nx * (jc - (long long)p.ny * s.kb);
        }
        dt = s.st->dt;
        col_in = i >= 0 && i <= p.nx && j >= 0 && j <= p.ny;
        cellcol_in = i >= 0 && i < p.nx && j >= 0 && j < p.ny;
        node_out = col_in && ix >= 1 && ix <= TX && iy >= 1 && iy <= TY;
        xi = s.Xt[i < 0 ? 0 : (i > p.nx ? p.nx : i)];
        yj = s.Yt[j < 0 ? 0 : (j > p.ny ? p.ny : j)];
        sig_col = cellcol_in && ix >= 1 && ix <= TX && iy >= 1 && iy <= TY;
        pxm = i >= 1 && i <= p.nx;
        pxp = i >= 0 && i < p.nx;
        pym = j >= 1 && j <= p.ny;
        pyp = j >= 0 && j < p.ny;
        // the z-face area vectors do not depend on the plane: staged once
        const long long tz = (long long)jc * p.nx + ic;
        st3s(me, oZ(), PL, D3{s.TAz[0][tz], s.TAz[1][tz], s.TAz[2][tz]});
    }

    __device__ __forceinline__ void fetch(int k)  // node plane k, cell plane k-1
    {
        pnok = col_in && k >= 0 && k <= p.nz;
        const int kn = k < s.kb ? s.kb : (k > s.kb + s.nzn - 1 ? s.kb + s.nzn - 1 : k);
        pu = ld3(s.u[cur], nbc + (long long)kn * s.pn);
        pz = s.Zt[kn - s.kb];
        const int kc = k - 1;
        pcok = cellcol_in && kc >= 0 && kc < p.nz;
        int kl = kc - s.kb;  // cell / table plane clamped into the slab (values unused outside)
        kl = kl < 0 ? 0 : (kl >= s.nzc ? s.nzc - 1 : kl);
        const long long c = cbc + (long long)(kl + s.kb) * s.pc;
        pm = s.m[cur][c];
        pe = s.e[cur][c];
        pv = s.VT[c];
        const long long tx = (long long)kl * p.ny + jc, ty = (long long)kl * p.nx + ic;
        pax = D3{s.TAx[0][tx], s.TAx[1][tx], s.TAx[2][tx]};
        pay = D3{s.TAy[0][ty], s.TAy[1][ty], s.TAy[2][ty]};
    }
    template <int PAR>
    __device__ __forceinline__ D3 U(int off) const { return ld3s(me + off, oU(PAR, 0), PL); }

    template <int B0, bool ALL>
    __device__ __forceinline__ void gather(D3& F, double& M, bool pzm, bool pzp) const
    {
        constexpr int B1 = B0 ^ 1;
        F = D3{0.0, 0.0, 0.0};
        M = 0.0;
        bool first = true;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const int ap = g & 1, bp = (g >> 1) & 1, cp = g >> 2;
            const int dx = ap ? 0 : -1, dy = bp ? 0 : -FW;
            const int PAR = cp ? B0 : B1;
            const D3 Ax = ld3s(me + dy, oA(PAR, 0), PL);
            const D3 Ay = ld3s(me + dx, oA(PAR, 1), PL);
            const D3 Az = ld3s(me + dx + dy, oZ(), PL);
            const D3 C = add(add(ap ? neg(Ax) : Ax, bp ? neg(Ay) : Ay), cp ? neg(Az) : Az);
            const double sg = me[dx + dy + oS(PAR, 0)];
            const double mk = me[dx + dy + oS(PAR, 1)];
            const D3 term = scl(sg, C);
            if (ALL) {
                F = g == 0 ? term : add(F, term);
                M = g == 0 ? mk : M + mk;
            } else {
                const bool pres = (ap ? pxp : pxm) && (bp ? pyp : pym) && (cp ? pzp : pzm);
                if (pres) {
                    F = first ? term : add(F, term);
                    M = first ? mk : M + mk;
                    first = false;
                }
            }
        }
    }

    // c.3 step 2 on one axis with the table's d and L
    __device__ __forceinline__ static double jump(const double* T, D3 Um, D3 Up)
    {
        const D3 w = sub(Up, Um);
        return ddiv((w.x * T[0] + w.y * T[1]) + w.z * T[2], T[3]);
    }

    template <int B0>
    __device__ __forceinline__ void step(int kz)
    {
        constexpr int B1 = B0 ^ 1;
        // ---- P1: stage node plane kz+1 (u), cell (i,j,kz); prefetch the next
        st3s(me, oU(B1, 0), PL, pnok ? pu : D3{0.0, 0.0, 0.0});
        const double m = pcok ? pm : 0.0, e = pcok ? pe : 0.0, V = pcok ? pv : 1.0;
        const double z1 = pz;  // Z of node plane kz+1
        const D3 ax = pax, ay = pay;
        if (kz < zb) fetch(kz + 2);
        __syncthreads();
        // ---- P2: face-average velocities of the three faces anchored here; A from the tables
        const D3 ux = avg4(U<B0>(0), U<B0>(FW), U<B1>(FW), U<B1>(0));
        const D3 uy = avg4(U<B0>(0), U<B1>(0), U<B1>(1), U<B0>(1));
        const D3 uz = avg4(U<B1>(0), U<B1>(1), U<B1>(FW + 1), U<B1>(FW));
        st3s(me, oW(0, 0), PL, ux);
        st3s(me, oW(1, 0), PL, uy);
        const int kl = kz - s.kb;
        st3s(me, oA(B0, 0), PL, ax);
        st3s(me, oA(B0, 1), PL, ay);
        // the axis-jump constants of P3, loaded before the barrier
        const double* TJ[3] = {s.TJx + 4 * ic, s.TJy + 4 * jc, s.TJz + 4 * kl};
        double tj[3][4];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) tj[a][c] = TJ[a][c];
        __syncthreads();
        // ---- P3: cell (i,j,kz): rho, EoS, q, sigma
        {
            double sig = 0.0;
            if (cellcol_in && kz >= 0 && kz < p.nz) {
                double rho = ddiv(m, V), pr, pf, cs;
                eos(p.gamma, rho, e, pr, pf, cs);
                const double dx = jump(tj[0], ux, ld3s(me + 1, oW(0, 0), PL));
                const double dy = jump(tj[1], uy, ld3s(me + FW, oW(1, 0), PL));
                const double dz = jump(tj[2], zprev, uz);
                const double du = dmin(dmin(dx, dy), dz);
                const double q = q_of_du(rho, cs, du, p.c1, p.c2);
                sig = 0.25 * (pf + q);
                if (sig_col && kz >= za && kz >= kn0 && kz < kn1) s.sig[cb + (long long)kz * s.pc] = sig;
            }
            me[oS(B0, 0)] = sig;
            me[oS(B0, 1)] = m;
        }
        zprev = uz;
        const double zcur = zc;  // Z of node plane kz (P4)
        zc = z1;
        __syncthreads();
        // ---- P4: node (i,j,kz): force + mass gather, kinematics, BC, move
        if (node_out && kz >= za) {
            const bool pzm = kz >= 1, pzp = kz < p.nz;
            D3 F;
            double M;
            if (pxm && pxp && pym && pyp && pzm && pzp) gather<B0, true>(F, M, true, true);
            else gather<B0, false>(F, M, pzm, pzp);
            M = 0.125 * M;
            const D3 u = U<B0>(0), x = D3{xi, yj, zcur};
            D3 un = d3(u.x + (ddiv(F.x, M) * dt), u.y + (ddiv(F.y, M) * dt), u.z + (ddiv(F.z, M) * dt));
            un = reflect(p, i, j, kz, un);
            const D3 xn = d3(x.x + (un.x * dt), x.y + (un.y * dt), x.z + (un.z * dt));
            const long long n = nb + (long long)kz * s.pn;
            st3(s.u1, n, un);
            st3(s.x1, n, xn);
        }
    }

    __device__ __forceinline__ void run()
    {
        fetch(za - 1);
        if ((za - 1) & 1) st3s(me, oU(1, 0), PL, pnok ? pu : D3{0.0, 0.0, 0.0});
        else st3s(me, oU(0, 0), PL, pnok ? pu : D3{0.0, 0.0, 0.0});
        zc = pz;
        fetch(za);
        __syncthreads();
        zprev = ((za - 1) & 1) ? avg4(U<1>(0), U<1>(1), U<1>(FW + 1), U<1>(FW))
                               : avg4(U<0>(0), U<0>(1), U<0>(FW + 1), U<0>(FW));
        for (int kz = za - 1; kz <= zb; ++kz) {
            if (kz & 1) step<1>(kz);
            else step<0>(kz);
        }
    }
};

template <int NW, int MB>
__global__ void __launch_bounds__(FW * NW, MB) kf_force_e(Slab s, Phys p, int cur, int kn0, int kn1, int zchunk)
{
    if (!s.st->active) return;
    extern __shared__ double smem[];
    ForceEulerCTA<NW> c(s, p, cur, smem, kn0, kn1, zchunk);
    c.run();
}

// ============================================================================
// Euler mode, split form of kf_force_e (SALE_FORCE_E=9):
//   kf_sigma_e : z-march; face-average velocities of the three faces anchored at a
//                column, then EoS + q + sigma of the cell (S2, S3).  Dependencies
//                reach only the +x / +y neighbours: a 32 x NW tile yields
//                31 x (NW-1) cells.  Writes sigma.
//   kn_force_e : one thread per node: the corner-force and mass gather in the
//                fixed order of c.2 with the target face areas from the tables,
//                kinematics + reflecting BC (S5, S6).  Writes u', x'.
// ============================================================================
// DIAG: the target mesh's axis-jump separations lie on their axes (Phys::diag_jumps).
// Then w . d = (w_a d_a + w_b * 0) + w_c * 0 equals w_a d_a whenever that is non-zero,
// and when it is zero the jump is a zero of some sign, which q ignores (q depends on
// du only through du < 0 and, when negative, its value): sigma is the same bits with
// only the a-component of the face-average velocity on axis a.
// NM > 0: multi-material cells: the mixed closure MM1, and each
// material's stress 0.25 (pf_k + q) stored for the energy kernel (Slab::sgm)
template <int NW, bool DIAG, int NM = 0>
struct SigmaEulerCTA {
    static constexpr int PL = NW * FW, TX = FW - 1, TY = NW - 1;
    __host__ __device__ static constexpr int oU(int par, int c) { return (par * 3 + c) * PL; }       // node u
    __host__ __device__ static constexpr int oW(int xy, int c) { return 6 * PL + (xy * 3 + c) * PL; }  // x/y face Ubar
    static constexpr int WORDS = 12 * PL + 2 * PAD;

    const Slab& s;
    const Phys& p;
    const int cur;
    double* me;
    int i, j, za, zb, kc0, kc1, ic, jc;
    long long nbn, cb, cbc;
    bool col_in, out_cell;
    D3 pu;
    double pm, pe, pv;
    double pmf[NM > 0 ? NM : 1], pmm[NM > 0 ? NM : 1], pme[NM > 0 ? NM : 1];  // prefetch: materials
    bool pnok;
    D3 zprev;
    unsigned long long key;  // running min of the owned cells' dt keys (c.5)

    __device__ __forceinline__ SigmaEulerCTA(const Slab& s_, const Phys& p_, int cur_, double* smem, int kc0_, int kc1_,
                                             int zchunk)
        : s(s_), p(p_), cur(cur_)
    {
        const int ix = threadIdx.x, iy = threadIdx.y;
        me = smem + PAD + iy * FW + ix;
        i = blockIdx.x * TX + ix;
        j = blockIdx.y * TY + iy;
        ic = i < p.nx ? i : p.nx - 1;
        jc = j < p.ny ? j : p.ny - 1;
        kc0 = kc0_;
        kc1 = kc1_;
        za = kc0 + blockIdx.z * zchunk;
        zb = za + zchunk - 1 < kc1 - 1 ? za + zchunk - 1 : kc1 - 1;
        const int in = i < p.nx ? i : p.nx, jn = j < p.ny ? j : p.ny;
        nbn = (long long)in + (long long)(p.nx + 1) * (jn - (long long)(p.ny + 1) * s.kb);
        cb = (long long)i + (long long)p.nx * (j - (long long)p.ny * s.kb);
        cbc = (long long)ic + (long long)p.nx * (jc - (long long)p.ny * s.kb);
        col_in = i <= p.nx && j <= p.ny;
        out_cell = i < p.nx && j < p.ny && ix < TX && iy < TY;
        key = KEY_NONE;
    }
    __device__ __forceinline__ void fetch(int k)  // node plane k (u), cell plane k-1 (m, e, V^T)
    {
        pnok = col_in && k >= 0 && k <= p.nz;
        const int kn = k < s.kb ? s.kb : (k > s.kb + s.nzn - 1 ? s.kb + s.nzn - 1 : k);
        pu = ld3(s.u[cur], nbn + (long long)kn * s.pn);
        int kc = k - 1;
        kc = kc < s.kb ? s.kb : (kc > s.kb + s.nzc - 1 ? s.kb + s.nzc - 1 : kc);
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
    __device__ __forceinline__ static double jump(const double* T, D3 Um, D3 Up)
    {
        const D3 w = sub(Up, Um);
        return ddiv((w.x * T[0] + w.y * T[1]) + w.z * T[2], T[3]);
    }

    template <int B0>
    __device__ __forceinline__ void step(int kz)
    {
        constexpr int B1 = B0 ^ 1;
        st3s(me, oU(B1, 0), PL, pnok ? pu : D3{0.0, 0.0, 0.0});
        const double m = pm, e = pe, V = pv;
        double cmf[NM > 0 ? NM : 1], cmm[NM > 0 ? NM : 1], cme[NM > 0 ? NM : 1];
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            cmf[a] = pmf[a];
            cmm[a] = pmm[a];
            cme[a] = pme[a];
        }
        if (kz < zb) fetch(kz + 2);
        __syncthreads();
        D3 ux, uy, uz;
        if constexpr (DIAG) {  // the a-component of the face average on axis a only (c.3 step 2)
            const double* Ux0 = me + oU(B0, 0);
            const double* Ux1 = me + oU(B1, 0);
            const double* Uy0 = me + oU(B0, 1);
            const double* Uy1 = me + oU(B1, 1);
            const double* Uz1 = me + oU(B1, 2);
            ux.x = 0.25 * (((Ux0[0] + Ux0[FW]) + Ux1[FW]) + Ux1[0]);
            uy.y = 0.25 * (((Uy0[0] + Uy1[0]) + Uy1[1]) + Uy0[1]);
            uz.z = 0.25 * (((Uz1[0] + Uz1[1]) + Uz1[FW + 1]) + Uz1[FW]);
            me[oW(0, 0)] = ux.x;
            me[oW(1, 0)] = uy.y;
        } else {
            ux = avg4(U<B0>(0), U<B0>(FW), U<B1>(FW), U<B1>(0));
            uy = avg4(U<B0>(0), U<B1>(0), U<B1>(1), U<B0>(1));
            uz = avg4(U<B1>(0), U<B1>(1), U<B1>(FW + 1), U<B1>(FW));
            st3s(me, oW(0, 0), PL, ux);
            st3s(me, oW(1, 0), PL, uy);
        }
        // max node speed^2 of the cell in corner order (read here, before the barrier:
        // the next step's P1 overwrites the plane-kz slot)
        double v2 = speed2(U<B0>(0));
        v2 = dmax(v2, speed2(U<B0>(1)));
        v2 = dmax(v2, speed2(U<B0>(FW)));
        v2 = dmax(v2, speed2(U<B0>(FW + 1)));
        v2 = dmax(v2, speed2(U<B1>(0)));
        v2 = dmax(v2, speed2(U<B1>(1)));
        v2 = dmax(v2, speed2(U<B1>(FW)));
        v2 = dmax(v2, speed2(U<B1>(FW + 1)));
        const int kl = kz - s.kb;
        const double* TJ[3] = {s.TJx + 4 * ic, s.TJy + 4 * jc, s.TJz + 4 * kl};
        double tj[3][4];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) tj[a][c] = TJ[a][c];
        __syncthreads();
        if (out_cell && kz >= 0 && kz < p.nz) {
            double rho = ddiv(m, V), pr, pf, cs, pfk[MAX_MAT];
            if constexpr (NM > 0) mix_eos_r<NM>(s, cmf, cmm, cme, V, rho, pr, pf, cs, pfk);
            else eos(p.gamma, rho, e, pr, pf, cs);
            double dx, dy, dz;
            if constexpr (DIAG) {
                dx = ddiv((me[1 + oW(0, 0)] - ux.x) * tj[0][0], tj[0][3]);
                dy = ddiv((me[FW + oW(1, 0)] - uy.y) * tj[1][1], tj[1][3]);
                dz = ddiv((uz.z - zprev.z) * tj[2][2], tj[2][3]);
            } else {
                dx = jump(tj[0], ux, ld3s(me + 1, oW(0, 0), PL));
                dy = jump(tj[1], uy, ld3s(me + FW, oW(1, 0), PL));
                dz = jump(tj[2], zprev, uz);
            }
            const double du = dmin(dmin(dx, dy), dz);
            const double q = q_of_du(rho, cs, du, p.c1, p.c2);
            s.sig[cb + (long long)kz * s.pc] = 0.25 * (pf + q);
#pragma unroll
            for (int a = 0; a < NM; ++a) s.sgm[cb + (long long)kz * s.pc + a * mat_stride(s)] = 0.25 * (pfk[a] + q);
            if (kz >= s.k0 && kz < s.k1) {
                // c.5 dt candidate of this (cycle-start) state: v2 (P2), cfl * sqrt(min
                // edge^2) from the per-axis tables (as kn_dt)
                const double num = dmin(dmin(s.TDx[ic], s.TDy[jc]), s.TDz[kl]);
                const unsigned long long kk = dt_key(ddiv(num, (cs + dsqrt(v2)) + 1e-30));
                key = kk < key ? kk : key;
            }
        }
        zprev = uz;
    }

    __device__ __forceinline__ void run()
    {
        fetch(za);
        if (za & 1) st3s(me, oU(1, 0), PL, pnok ? pu : D3{0.0, 0.0, 0.0});
        else st3s(me, oU(0, 0), PL, pnok ? pu : D3{0.0, 0.0, 0.0});
        fetch(za + 1);
        __syncthreads();
        zprev = (za & 1) ? avg4(U<1>(0), U<1>(1), U<1>(FW + 1), U<1>(FW)) : avg4(U<0>(0), U<0>(1), U<0>(FW + 1), U<0>(FW));
        if constexpr (DIAG) zprev = D3{0.0, 0.0, zprev.z};
        for (int kz = za; kz <= zb; ++kz) {
            if (kz & 1) step<1>(kz);
            else step<0>(kz);
        }
        block_min_atomic(key, &s.st->cand_key);
    }
};

// gate = 0 for the first cycle of a sale_step call (DevState.active is still 0 there)
template <int NW, int MB, bool DIAG, int NM = 0>
__global__ void __launch_bounds__(FW * NW, MB) kf_sigma_e(Slab s, Phys p, int cur, int kc0, int kc1, int zchunk, int gate)
{
    if (gate && !s.st->active) return;
    extern __shared__ double smem[];
    SigmaEulerCTA<NW, DIAG, NM> c(s, p, cur, smem, kc0, kc1, zchunk);
    c.run();
}

// grid: x = ceil((nx+1)(ny+1) / 256) (flattened node plane), y = node planes [kn0, kn1]
// (32-bit index arithmetic: a slab holds < 2^31 cells)
// wx1 = 0: x' is not stored -- its consumers on the default path (kf_energy_e,
// kr_sweep) form x' = x^T + u' dt from u' and the target tables when they stage a
// node plane (the same expression, the same bits); the alternative kernels that load
// x' need wx1 = 1 (euler_x1_stored)
// (8 CTAs per SM at 32 registers: a small spill, but a latency-bound gather gains more
// from the warps -- measured C4 3.077 -> 3.003 ms with kn_update's bound)
__global__ void __launch_bounds__(256, 8) kn_force_e(Slab s, Phys p, int cur, int kn0, int wx1)
{
    if (!s.st->active) return;
    const int t = blockIdx.x * 256 + threadIdx.x;
    if (t >= (int)s.pn) return;
    const int nx = p.nx, ny = p.ny, pc = (int)s.pc;
    const int i = t % (nx + 1), j = t / (nx + 1), k = kn0 + blockIdx.y, kl = k - s.kb;
    const bool pxm = i >= 1, pxp = i < nx, pym = j >= 1, pyp = j < ny, pzm = k >= 1, pzp = k < p.nz;
    const int c11 = i + nx * (j + ny * kl);
    const double dt = s.st->dt;
    D3 F = D3{0.0, 0.0, 0.0};
    double M = 0.0;
    bool first = true;
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        const int ap = g & 1, bp = (g >> 1) & 1, cp = g >> 2;
        const bool pres = (ap ? pxp : pxm) && (bp ? pyp : pym) && (cp ? pzp : pzm);
        if (!pres) continue;
        const int ci = i - 1 + ap, cj = j - 1 + bp, ckl = kl - 1 + cp;
        const int ox = ckl * ny + cj, oy = ckl * nx + ci, oz = cj * nx + ci;
        // cell (i-1+ap, j-1+bp, k-1+cp): the node is its corner (1-ap, 1-bp, 1-cp)
        D3 C;
        if (p.diag_areas) {  // axis-aligned areas: ((+-a, 0, 0) + (0, +-b, 0)) + (0, 0, +-c) exactly
            const double ax = __ldg(s.TAx[0] + ox), ay = __ldg(s.TAy[1] + oy), az = __ldg(s.TAz[2] + oz);
            C = D3{ap ? -ax : ax, bp ? -ay : ay, cp ? -az : az};
        } else {
            const D3 Ax = D3{__ldg(s.TAx[0] + ox), __ldg(s.TAx[1] + ox), __ldg(s.TAx[2] + ox)};
            const D3 Ay = D3{__ldg(s.TAy[0] + oy), __ldg(s.TAy[1] + oy), __ldg(s.TAy[2] + oy)};
            const D3 Az = D3{__ldg(s.TAz[0] + oz), __ldg(s.TAz[1] + oz), __ldg(s.TAz[2] + oz)};
            C = add(add(ap ? neg(Ax) : Ax, bp ? neg(Ay) : Ay), cp ? neg(Az) : Az);
        }
        const int c = c11 + (ap - 1) + nx * (bp - 1) + pc * (cp - 1);
        const D3 term = scl(__ldg(s.sig + c), C);
        const double mk = __ldg(s.m[cur] + c);
        F = first ? term : add(F, term);
        M = first ? mk : M + mk;
        first = false;
    }
    M = 0.125 * M;
    const long long n = (long long)t + s.pn * (long long)kl;
    const D3 u = ld3(s.u[cur], n), x = D3{s.Xt[i], s.Yt[j], s.Zt[kl]};
    D3 un = d3(u.x + (ddiv(F.x, M) * dt), u.y + (ddiv(F.y, M) * dt), u.z + (ddiv(F.z, M) * dt));
    un = reflect(p, i, j, k, un);
    st3(s.u1, n, un);
    if (wx1) st3(s.x1, n, d3(x.x + (un.x * dt), x.y + (un.y * dt), x.z + (un.z * dt)));
}

// ============================================================================
// kf_energy
// ============================================================================
// NM > 0 (Lagrange, multi-material cells): MM4 per material from the
// stresses kf_force stored (Slab::sgm), and the dt candidate from the mixed closure
template <bool EULER, int NW, int NM = 0>
struct EnergyCTA : MatRegs<NM> {
    static constexpr int PL = NW * FW, TX = FW - 1, TY = NW - 1;
    __host__ __device__ static constexpr int oP(int par, int c) { return (par * 10 + c) * PL; }  // x^n(3) x'(3) ubar(3) |u'|^2
    __host__ __device__ static constexpr int oF(int xy, int c) { return 20 * PL + (xy * 4 + c) * PL; }  // A^n(3), s'
    __host__ __device__ static constexpr int oE(int c) { return 28 * PL + c * PL; }                 // edge^2 minima
    static constexpr int WORDS = 31 * PL + 2 * PAD;

    const Slab& s;
    const Phys& p;
    const int cur;
    double* me;
    int i, j, za, zb;
    long long nb, cb;
    double dt;
    bool col_in, cell_col;
    unsigned long long key;
    D3 fx, fu, fu1, fx1;  // prefetch registers
    double fm, fe, fs;
    D3 zA_prev;
    double zs_prev, ex_prev, ey_prev;

    __device__ __forceinline__ EnergyCTA(const Slab& s_, const Phys& p_, int cur_, double* smem, int kc0, int kc1,
                                         int zchunk)
        : s(s_), p(p_), cur(cur_)
    {
        const int ix = threadIdx.x, iy = threadIdx.y;
        me = smem + PAD + iy * FW + ix;
        i = blockIdx.x * TX + ix;
        j = blockIdx.y * TY + iy;
        za = kc0 + blockIdx.z * zchunk;
        zb = za + zchunk - 1 < kc1 - 1 ? za + zchunk - 1 : kc1 - 1;
        nb = (long long)i + (long long)(p.nx + 1) * (j - (long long)(p.ny + 1) * s.kb);
        cb = (long long)i + (long long)p.nx * (j - (long long)p.ny * s.kb);
        dt = s.st->dt;
        col_in = i <= p.nx && j <= p.ny;
        cell_col = i < p.nx && j < p.ny && ix < TX && iy < TY;
        key = KEY_NONE;
    }

    __device__ __forceinline__ void fetch(int k)  // node plane k, cell plane k-1
    {
        fx = D3{0.0, 0.0, 0.0};
        fu = fx;
        fu1 = fx;
        fx1 = fx;
        if (col_in && k >= 0 && k <= p.nz) {
            long long n = nb + (long long)k * s.pn;
            if (EULER) fx = D3{s.Xt[i], s.Yt[j], s.Zt[k - s.kb]};
            else fx = ld3(s.x[cur], n);
            fu = ld3(s.u[cur], n);
            fu1 = EULER ? ld3(s.u1, n) : ld3(s.u[cur ^ 1], n);
            fx1 = EULER ? ld3(s.x1, n) : ld3(s.x[cur ^ 1], n);
        }
        fm = 0.0;
        fe = 0.0;
        fs = 0.0;
        const int kc = k - 1;
        if (cell_col && kc >= 0 && kc < p.nz) {
            long long c = cb + (long long)kc * s.pc;
            fm = mass_cur(s, p, cur)[c];
            fe = s.e[cur][c];
            fs = s.sig[c];
            if constexpr (NM > 0) {
#pragma unroll
                for (int a = 0; a < NM; ++a) {
                    const long long ca = c + a * mat_stride(s);
                    this->rf[a] = mat_f(s, p, cur)[ca];
                    this->rm[a] = mat_m(s, p, cur)[ca];
                    this->re[a] = s.me[cur][ca];
                    this->rs[a] = s.sgm[ca];
                }
            }
        }
    }
    template <int PAR>
    __device__ __forceinline__ void put()
    {
        const D3 ub = scl(0.5, add(fu, fu1));
        st3s(me, oP(PAR, 0), PL, fx);
        st3s(me, oP(PAR, 3), PL, fx1);
        st3s(me, oP(PAR, 6), PL, ub);
        me[oP(PAR, 9)] = speed2(fu1);
    }
    template <int PAR>
    __device__ __forceinline__ D3 Xn(int off) const { return ld3s(me + off, oP(PAR, 0), PL); }
    template <int PAR>
    __device__ __forceinline__ D3 X1(int off) const { return ld3s(me + off, oP(PAR, 3), PL); }
    template <int PAR>
    __device__ __forceinline__ D3 Ub(int off) const { return ld3s(me + off, oP(PAR, 6), PL); }
    template <int PAR>
    __device__ __forceinline__ double V2(int off) const { return me[off + oP(PAR, 9)]; }

    template <int B>
    __device__ __forceinline__ void zstate(D3& zA, double& zs, double& ex, double& ey) const
    {
        zA = face_area(Xn<B>(0), Xn<B>(1), Xn<B>(FW + 1), Xn<B>(FW));
        const D3 T0 = X1<B>(0), T1 = X1<B>(1), T2 = X1<B>(FW + 1), T3 = X1<B>(FW);
        zs = face_s(avg4(T0, T1, T2, T3), face_area(T0, T1, T2, T3));
        ex = len2(T0, T1);
        ey = len2(T0, T3);
    }

    template <int B0>
    __device__ __forceinline__ void step(int kz)
    {
        constexpr int B1 = B0 ^ 1;
        // ---- P1
        put<B1>();
        const double m = fm, e = fe, sig = fs;
        const MatRegs<NM> cmat = *this;  // this plane's material operands (the prefetch moves on)
        if (kz < zb) fetch(kz + 2);
        __syncthreads();
        // ---- P2: faces anchored at this column (A at t^n, s' at t^{n+1}); x' edges
        D3 zA_next;
        double zs_next, ex_next, ey_next;
        {
            // x-face at node plane i: (i,j,kz) (i,j+1,kz) (i,j+1,kz+1) (i,j,kz+1)
            const D3 Ax = face_area(Xn<B0>(0), Xn<B0>(FW), Xn<B1>(FW), Xn<B1>(0));
            const D3 Q0 = X1<B0>(0), Q1 = X1<B0>(FW), Q2 = X1<B1>(FW), Q3 = X1<B1>(0);
            const double sx = face_s(avg4(Q0, Q1, Q2, Q3), face_area(Q0, Q1, Q2, Q3));
            // y-face at node plane j: (i,j,kz) (i,j,kz+1) (i+1,j,kz+1) (i+1,j,kz)
            const D3 Ay = face_area(Xn<B0>(0), Xn<B1>(0), Xn<B1>(1), Xn<B0>(1));
            const D3 R0 = Q0, R1 = Q3, R2 = X1<B1>(1), R3 = X1<B0>(1);
            const double sy = face_s(avg4(R0, R1, R2, R3), face_area(R0, R1, R2, R3));
            zstate<B1>(zA_next, zs_next, ex_next, ey_next);
            const double ez = len2(Q0, Q3);  // z-edge (i,j): kz -> kz+1
            st3s(me, oF(0, 0), PL, Ax);
            me[oF(0, 3)] = sx;
            st3s(me, oF(1, 0), PL, Ay);
            me[oF(1, 3)] = sy;
            me[oE(0)] = dmin(ex_prev, ex_next);
            me[oE(1)] = dmin(ey_prev, ey_next);
            me[oE(2)] = ez;
        }
        __syncthreads();
        // ---- P3: cell (i,j,kz)
        if (cell_col && kz < p.nz) {
            double sv[6] = {me[oF(0, 3)], me[1 + oF(0, 3)], me[oF(1, 3)], me[FW + oF(1, 3)], zs_prev, zs_next};
            const double V1 = vol_from_s(sv);
            const bool owned = kz >= s.k0 && kz < s.k1;
            if (owned && !(V1 > 0.0))
                atomicMin(&s.st->err_key, (ERR_ORDER_TANGLED << 48) | (unsigned long long)gcell(p, i, j, kz));
            const D3 A[6] = {ld3s(me, oF(0, 0), PL),      ld3s(me + 1, oF(0, 0), PL), ld3s(me, oF(1, 0), PL),
                             ld3s(me + FW, oF(1, 0), PL), zA_prev,                    zA_next};
            double W = 0.0;
#pragma unroll
            for (int h = 0; h < 8; ++h) {
                const int a = h & 1, b = (h >> 1) & 1, c = h >> 2;
                const D3 C = corner_vec(A, a, b, c);
                const D3 ub = c ? Ub<B1>(a + b * FW) : Ub<B0>(a + b * FW);
                const double term = dot(C, ub);
                W = (h == 0) ? term : W + term;
            }
            const long long cc = cb + (long long)kz * s.pc;
            double e1k[NM > 0 ? NM : 1];
            if constexpr (NM > 0) {  // MM4: each present material's share of the work
#pragma unroll
                for (int a = 0; a < NM; ++a) {
                    e1k[a] = (cmat.rf[a] > 0.0 && cmat.rm[a] > 0.0)
                                 ? cmat.re[a] - ddiv(((cmat.rs[a] * W) * dt) * cmat.rf[a], cmat.rm[a])
                                 : cmat.re[a];
                    s.me[cur ^ 1][cc + a * mat_stride(s)] = e1k[a];
                }
            }
            const double e1 = NM > 0 ? 0.0 : e - ddiv((sig * W) * dt, m);
            if (EULER) {
                s.e1[cc] = e1;
                s.V1[cc] = V1;
            } else {
                if (NM == 0) s.e[cur ^ 1][cc] = e1;
                if (owned) {
                    double rho = ddiv(m, V1), pr, pf, cs;
                    if constexpr (NM > 0) {
                        double pfk[MAX_MAT];
                        mix_eos_r<NM>(s, cmat.rf, cmat.rm, e1k, V1, rho, pr, pf, cs, pfk);
                    } else {
                        eos(p.gamma, rho, e1, pr, pf, cs);
                    }
                    s.rhoc[cc] = rho;
                    s.csc[cc] = cs;
                    double l2 = dmin(dmin(me[oE(0)], me[FW + oE(0)]), dmin(me[oE(1)], me[1 + oE(1)]));
                    l2 = dmin(l2, dmin(dmin(me[oE(2)], me[1 + oE(2)]), dmin(me[FW + oE(2)], me[FW + 1 + oE(2)])));
                    double v2 = V2<B0>(0);
                    v2 = dmax(v2, V2<B0>(1));
                    v2 = dmax(v2, V2<B0>(FW));
                    v2 = dmax(v2, V2<B0>(FW + 1));
                    v2 = dmax(v2, V2<B1>(0));
                    v2 = dmax(v2, V2<B1>(1));
                    v2 = dmax(v2, V2<B1>(FW));
                    v2 = dmax(v2, V2<B1>(FW + 1));
                    const unsigned long long kk = dt_key(dt_cell(p.cfl, l2, v2, cs));
                    key = kk < key ? kk : key;  // running min over this column's planes
                }
            }
        }
        zA_prev = zA_next;
        zs_prev = zs_next;
        ex_prev = ex_next;
        ey_prev = ey_next;
        __syncthreads();
    }

    __device__ __forceinline__ void run()
    {
        fetch(za);
        if (za & 1) put<1>();
        else put<0>();
        fetch(za + 1);
        __syncthreads();
        if (za & 1) zstate<1>(zA_prev, zs_prev, ex_prev, ey_prev);
        else zstate<0>(zA_prev, zs_prev, ex_prev, ey_prev);
        for (int kz = za; kz <= zb; ++kz) {
            if (kz & 1) step<1>(kz);
            else step<0>(kz);
        }
        if (!EULER) {
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
    }
};

template <bool EULER, int NW, int MB, int NM = 0>
__global__ void __launch_bounds__(FW * NW, MB)
    kf_energy(Slab s, Phys p, int cur, int kc0, int kc1, int zchunk)
{
    if (!s.st->active) return;
    extern __shared__ double smem[];
    EnergyCTA<EULER, NW, NM> c(s, p, cur, smem, kc0, kc1, zchunk);
    c.run();
}

// ============================================================================
// kf_energy, Euler mode: A^n from the target tables (as kf_force_e); stages only
// x' and ubar = (u + u')/2.  Writes e' and V' (the remap's inputs).
// ============================================================================
// NM > 0: multi-material cells: MM4 per material (e'_k into
// Slab::e1m) from the stresses kf_sigma_e stored, instead of e'
template <int NW, int NM = 0>
struct EnergyEulerCTA : MatRegs<NM> {
    static constexpr int PL = NW * FW, TX = FW - 1, TY = NW - 1;
    __host__ __device__ static constexpr int oP(int par, int c) { return (par * 6 + c) * PL; }        // x'(3) ubar(3)
    __host__ __device__ static constexpr int oF(int xy, int c) { return 12 * PL + (xy * 4 + c) * PL; }  // A^n(3), s'
    __host__ __device__ static constexpr int oZ() { return 20 * PL; }                                 // z-face A^n
    static constexpr int WORDS = 23 * PL + 2 * PAD;

    const Slab& s;
    const Phys& p;
    double* me;
    int i, j, za, zb, ic, jc;
    long long nb, cb, nbc, cbc;  // column clamped into the mesh (always-valid loads)
    double dt;
    bool col_in, cell_col, own_col;
    D3 fu, fu1;       // prefetch registers (unconditional loads, selected at use)
    double fz;        // prefetch: target Z of the node plane
    double xcol, ycol;  // target X, Y of the (clamped) node column
    double fm, fe, fs;
    D3 fax, fay;      // prefetch: table A of the x- / y-face of cell plane k-1
    bool fnok, fcok;
    double zs_prev;

    __device__ __forceinline__ EnergyEulerCTA(const Slab& s_, const Phys& p_, double* smem, int kc0, int kc1, int zchunk)
        : s(s_), p(p_)
    {
        const int ix = threadIdx.x, iy = threadIdx.y;
        me = smem + PAD + iy * FW + ix;
        i = blockIdx.x * TX + ix;
        j = blockIdx.y * TY + iy;
        ic = i >= p.nx ? p.nx - 1 : i;
        jc = j >= p.ny ? p.ny - 1 : j;
        za = kc0 + blockIdx.z * zchunk;
        zb = za + zchunk - 1 < kc1 - 1 ? za + zchunk - 1 : kc1 - 1;
        nb = (long long)i + (long long)(p.nx + 1) * (j - (long long)(p.ny + 1) * s.kb);
        cb = (long long)i + (long long)p.nx * (j - (long long)p.ny * s.kb);
        {
            const int in = i > p.nx ? p.nx : i, jn = j > p.ny ? p.ny : j;
            nbc = (long long)in + (long long)(p.nx + 1) * (jn - (long long)(p.ny + 1) * s.kb);
            cbc = (long long)ic + (long long)p.nx * (jc - (long long)p.ny * s.kb);
            xcol = s.Xt[in];
            ycol = s.Yt[jn];
        }
        dt = s.st->dt;
        col_in = i <= p.nx && j <= p.ny;
        cell_col = i < p.nx && j < p.ny && ix < TX && iy < TY;
        own_col = col_in && ix < TX && iy < TY;
        const long long tz = (long long)jc * p.nx + ic;
        st3s(me, oZ(), PL, D3{s.TAz[0][tz], s.TAz[1][tz], s.TAz[2][tz]});
    }

    __device__ __forceinline__ void fetch(int k, int cur)  // node plane k, cell plane k-1
    {
        fnok = col_in && k >= 0 && k <= p.nz;
        const int kn = k < s.kb ? s.kb : (k > s.kb + s.nzn - 1 ? s.kb + s.nzn - 1 : k);
        const long long n = nbc + (long long)kn * s.pn;
        fu = ld3(s.u[cur], n);
        fu1 = ld3(s.u1, n);
        fz = s.Zt[kn - s.kb];
        const int kc = k - 1;
        fcok = cell_col && kc >= 0 && kc < p.nz;
        int kl = kc - s.kb;
        kl = kl < 0 ? 0 : (kl >= s.nzc ? s.nzc - 1 : kl);
        const long long c = cbc + (long long)(kl + s.kb) * s.pc;
        fm = s.m[cur][c];
        fe = s.e[cur][c];
        fs = s.sig[c];
        if constexpr (NM > 0) {
#pragma unroll
            for (int a = 0; a < NM; ++a) {
                const long long ca = c + a * mat_stride(s);
                this->rf[a] = s.mf[cur][ca];
                this->rm[a] = s.mm[cur][ca];
                this->re[a] = s.me[cur][ca];
                this->rs[a] = s.sgm[ca];
            }
        }
        const long long tx = (long long)kl * p.ny + jc, ty = (long long)kl * p.nx + ic;
        fax = D3{s.TAx[0][tx], s.TAx[1][tx], s.TAx[2][tx]};
        fay = D3{s.TAy[0][ty], s.TAy[1][ty], s.TAy[2][ty]};
    }
    template <int PAR>
    __device__ __forceinline__ void put()
    {
        const D3 z = D3{0.0, 0.0, 0.0};
        // x' = x^T + u' dt, kn_force_e's expression (c.3 step 6), formed when staged
        const D3 x1 = D3{xcol + (fu1.x * dt), ycol + (fu1.y * dt), fz + (fu1.z * dt)};
        st3s(me, oP(PAR, 0), PL, fnok ? x1 : z);
        st3s(me, oP(PAR, 3), PL, scl(0.5, add(fnok ? fu : z, fnok ? fu1 : z)));
    }
    template <int PAR>
    __device__ __forceinline__ D3 X1(int off) const { return ld3s(me + off, oP(PAR, 0), PL); }
    template <int PAR>
    __device__ __forceinline__ D3 Ub(int off) const { return ld3s(me + off, oP(PAR, 3), PL); }
    template <int B>
    __device__ __forceinline__ double zs() const  // s' of the moved z-face at this column, plane parity B
    {
        const D3 T0 = X1<B>(0), T1 = X1<B>(1), T2 = X1<B>(FW + 1), T3 = X1<B>(FW);
        return face_s(avg4(T0, T1, T2, T3), face_area(T0, T1, T2, T3));
    }

    template <int B0>
    __device__ __forceinline__ void step(int kz, int cur)
    {
        constexpr int B1 = B0 ^ 1;
        put<B1>();
        const double m = fcok ? fm : 0.0, e = fcok ? fe : 0.0, sig = fcok ? fs : 0.0;
        const MatRegs<NM> cmat = *this;  // this plane's material operands (the prefetch moves on)
        const D3 ax = fax, ay = fay;
        if (kz < zb) fetch(kz + 2, cur);
        __syncthreads();
        // ---- P2: s' of the moved x- and y-faces anchored here, A^n from the tables
        const D3 Q0 = X1<B0>(0), Q1 = X1<B0>(FW), Q2 = X1<B1>(FW), Q3 = X1<B1>(0);
        const double sx = face_s(avg4(Q0, Q1, Q2, Q3), face_area(Q0, Q1, Q2, Q3));
        const D3 R2 = X1<B1>(1), R3 = X1<B0>(1);
        const double sy = face_s(avg4(Q0, Q3, R2, R3), face_area(Q0, Q3, R2, R3));
        const double zs_next = zs<B1>();
        st3s(me, oF(0, 0), PL, ax);
        me[oF(0, 3)] = sx;
        st3s(me, oF(1, 0), PL, ay);
        me[oF(1, 3)] = sy;
        if (own_col) {  // s' of the faces anchored at node (i,j,kz), for kr_sweep's swept volumes
            const long long n = nb + (long long)kz * s.pn;
            s.sF[0][n] = sx;
            s.sF[1][n] = sy;
            s.sF[2][n] = zs_prev;
        }
        __syncthreads();
        // ---- P3: cell (i,j,kz)
        if (cell_col && kz < p.nz) {
            double sv[6] = {me[oF(0, 3)], me[1 + oF(0, 3)], me[oF(1, 3)], me[FW + oF(1, 3)], zs_prev, zs_next};
            const double V1 = vol_from_s(sv);
            if (kz >= s.k0 && kz < s.k1 && !(V1 > 0.0))
                atomicMin(&s.st->err_key, (ERR_ORDER_TANGLED << 48) | (unsigned long long)gcell(p, i, j, kz));
            const D3 Az = ld3s(me, oZ(), PL);
            const D3 A[6] = {ld3s(me, oF(0, 0), PL),      ld3s(me + 1, oF(0, 0), PL), ld3s(me, oF(1, 0), PL),
                             ld3s(me + FW, oF(1, 0), PL), Az,                         Az};
            double W = 0.0;
            const bool dg = p.diag_areas;
#pragma unroll
            for (int h = 0; h < 8; ++h) {
                const int a = h & 1, b = (h >> 1) & 1, c = h >> 2;
                // axis-aligned areas: the corner vector is exactly (+-Ax.x, +-Ay.y, +-Az.z)
                const D3 C = dg ? D3{a ? A[1].x : -A[0].x, b ? A[3].y : -A[2].y, c ? A[5].z : -A[4].z}
                                : corner_vec(A, a, b, c);
                const D3 ub = c ? Ub<B1>(a + b * FW) : Ub<B0>(a + b * FW);
                const double term = dot(C, ub);
                W = (h == 0) ? term : W + term;
            }
            const long long cc = cb + (long long)kz * s.pc;
            if constexpr (NM > 0) {  // MM4: each present material's share of the work
#pragma unroll
                for (int a = 0; a < NM; ++a)
                    s.e1m[cc + a * mat_stride(s)] =
                        (cmat.rf[a] > 0.0 && cmat.rm[a] > 0.0)
                            ? cmat.re[a] - ddiv(((cmat.rs[a] * W) * dt) * cmat.rf[a], cmat.rm[a])
                            : cmat.re[a];
            } else {
                s.e1[cc] = e - ddiv((sig * W) * dt, m);
            }
            s.V1[cc] = V1;
        }
        zs_prev = zs_next;
        __syncthreads();
    }

    __device__ __forceinline__ void run(int cur)
    {
        fetch(za, cur);
        if (za & 1) put<1>();
        else put<0>();
        fetch(za + 1, cur);
        __syncthreads();
        zs_prev = (za & 1) ? zs<1>() : zs<0>();
        for (int kz = za; kz <= zb; ++kz) {
            if (kz & 1) step<1>(kz, cur);
            else step<0>(kz, cur);
        }
    }
};

// ============================================================================
// kx_energy_sweep (Euler): kf_energy_e and the remap's kr_sweep in one z-march.
// Both read the same moved nodes x' and depend only on +x / +y neighbour columns;
// fused, the moved-face s' (V' and the swept-hex tops) and V' (V' and the donor
// density) stay on chip.  Per column and cell plane t:
//   P2: s' of the x-, y-faces anchored here and of the z-face at t+1; the six
//       ribbons of c.4 step 1 (shared as in kr_sweep); the 8-node mean of u'
//   P3: V' (tangle check), W and e' (S7); the swept volumes of the -x/-y/-z faces;
//       the donor data r = m/V', Ubar (R2)
// Writes e', dV, rD, UD (kr_flux's inputs).
// ============================================================================
template <int NW>
struct EnergySweepCTA {
    static constexpr int PL = NW * FW, TX = FW - 1, TY = NW - 1;
    __host__ __device__ static constexpr int oP(int par, int c) { return (par * 9 + c) * PL; }  // x'(3) ubar(3) u'(3)
    __host__ __device__ static constexpr int oF(int xy, int c) { return 18 * PL + (xy * 4 + c) * PL; }  // A^n(3), s'
    __host__ __device__ static constexpr int oZ() { return 26 * PL; }                                 // z-face A^n
    __host__ __device__ static constexpr int oR(int c) { return 29 * PL + c * PL; }                   // Rxz Ryz Rzy Rzx
    static constexpr int WORDS = 33 * PL + 2 * PAD;

    const Slab& s;
    const Phys& p;
    double* me;
    int i, j, za, zb, ic, jc, kr0, kr1;
    long long nb, cb, nbc, cbc;
    double dt, tx0, tx1, ty0, ty1;
    bool col_in, cell_col;
    D3 fu, fu1, fx1;  // prefetch: node plane k (unconditional loads, selected at use)
    double fm, fe, fs, fsx, fsy, fsz, fz;  // prefetch: cell plane k-1 (m, e, sigma, s^T x3), Z_k
    D3 fax, fay;
    bool fnok, fcok;
    double zs_prev, rxy_t, ryx_t, zprev;

    __device__ __forceinline__ EnergySweepCTA(const Slab& s_, const Phys& p_, double* smem, int kc0, int kc1, int kr0_,
                                              int kr1_, int zchunk)
        : s(s_), p(p_)
    {
        const int ix = threadIdx.x, iy = threadIdx.y;
        me = smem + PAD + iy * FW + ix;
        i = blockIdx.x * TX + ix;
        j = blockIdx.y * TY + iy;
        ic = i >= p.nx ? p.nx - 1 : i;
        jc = j >= p.ny ? p.ny - 1 : j;
        kr0 = kr0_;
        kr1 = kr1_;
        za = kc0 + blockIdx.z * zchunk;
        zb = za + zchunk - 1 < kc1 - 1 ? za + zchunk - 1 : kc1 - 1;
        nb = (long long)i + (long long)(p.nx + 1) * (j - (long long)(p.ny + 1) * s.kb);
        cb = (long long)i + (long long)p.nx * (j - (long long)p.ny * s.kb);
        {
            const int in = i > p.nx ? p.nx : i, jn = j > p.ny ? p.ny : j;
            nbc = (long long)in + (long long)(p.nx + 1) * (jn - (long long)(p.ny + 1) * s.kb);
            cbc = (long long)ic + (long long)p.nx * (jc - (long long)p.ny * s.kb);
        }
        dt = s.st->dt;
        col_in = i <= p.nx && j <= p.ny;
        cell_col = i < p.nx && j < p.ny && ix < TX && iy < TY;
        tx0 = col_in ? s.Xt[i] : 0.0;
        tx1 = (col_in && i + 1 <= p.nx) ? s.Xt[i + 1] : 0.0;
        ty0 = col_in ? s.Yt[j] : 0.0;
        ty1 = (col_in && j + 1 <= p.ny) ? s.Yt[j + 1] : 0.0;
        const long long tz = (long long)jc * p.nx + ic;
        st3s(me, oZ(), PL, D3{s.TAz[0][tz], s.TAz[1][tz], s.TAz[2][tz]});
    }

    __device__ __forceinline__ static double fs4(D3 Q0, D3 Q1, D3 Q2, D3 Q3)
    {
        return face_s(avg4(Q0, Q1, Q2, Q3), face_area(Q0, Q1, Q2, Q3));
    }
    __device__ __forceinline__ void fetch(int k, int cur)  // node plane k, cell plane k-1
    {
        fnok = col_in && k >= 0 && k <= p.nz;
        const int kn = k < s.kb ? s.kb : (k > s.kb + s.nzn - 1 ? s.kb + s.nzn - 1 : k);
        const long long n = nbc + (long long)kn * s.pn;
        fu = ld3(s.u[cur], n);
        fu1 = ld3(s.u1, n);
        fx1 = ld3(s.x1, n);
        fz = s.Zt[kn - s.kb];
        const int kc = k - 1;
        fcok = cell_col && kc >= 0 && kc < p.nz;
        int kl = kc - s.kb;
        kl = kl < 0 ? 0 : (kl >= s.nzc ? s.nzc - 1 : kl);
        const long long c = cbc + (long long)(kl + s.kb) * s.pc;
        fm = s.m[cur][c];
        fe = s.e[cur][c];
        fs = s.sig[c];
        fsx = s.sT[0][c];
        fsy = s.sT[1][c];
        fsz = s.sT[2][c];
        const long long tx = (long long)kl * p.ny + jc, ty = (long long)kl * p.nx + ic;
        fax = D3{s.TAx[0][tx], s.TAx[1][tx], s.TAx[2][tx]};
        fay = D3{s.TAy[0][ty], s.TAy[1][ty], s.TAy[2][ty]};
    }
    template <int PAR>
    __device__ __forceinline__ void put()
    {
        const D3 z = D3{0.0, 0.0, 0.0};
        const D3 u0 = fnok ? fu : z, u1 = fnok ? fu1 : z;
        st3s(me, oP(PAR, 0), PL, fnok ? fx1 : z);
        st3s(me, oP(PAR, 3), PL, scl(0.5, add(u0, u1)));
        st3s(me, oP(PAR, 6), PL, u1);
    }
    template <int PAR>
    __device__ __forceinline__ D3 X1(int off) const { return ld3s(me + off, oP(PAR, 0), PL); }
    template <int PAR>
    __device__ __forceinline__ D3 Ub(int off) const { return ld3s(me + off, oP(PAR, 3), PL); }
    template <int PAR>
    __device__ __forceinline__ D3 U1(int off) const { return ld3s(me + off, oP(PAR, 6), PL); }
    template <int B>
    __device__ __forceinline__ double zs() const
    {
        return fs4(X1<B>(0), X1<B>(1), X1<B>(FW + 1), X1<B>(FW));
    }
    // ribbons Rxy, Ryx of node plane k (parity PAR), own column, Z of that plane z
    template <int PAR>
    __device__ __forceinline__ void rib_xy(int k, double z, double& rxy, double& ryx) const
    {
        rxy = 0.0;
        ryx = 0.0;
        if (col_in && k >= 0 && k <= p.nz) {
            const D3 T = D3{tx0, ty0, z}, L = X1<PAR>(0);
            if (j + 1 <= p.ny) rxy = fs4(T, L, X1<PAR>(FW), D3{tx0, ty1, z});
            if (i + 1 <= p.nx) ryx = fs4(T, D3{tx1, ty0, z}, X1<PAR>(1), L);
        }
    }

    template <int B0>
    __device__ __forceinline__ void step(int t, int cur)
    {
        constexpr int B1 = B0 ^ 1;
        put<B1>();
        const double m = fcok ? fm : 0.0, e = fcok ? fe : 0.0, sig = fcok ? fs : 0.0;
        const double sTx = fsx, sTy = fsy, sTz = fsz, z0 = zprev, z1 = fz;
        const D3 ax = fax, ay = fay;
        if (t < zb) fetch(t + 2, cur);
        __syncthreads();
        // ---- P2: moved faces (s'), ribbons, A^n from the tables, Ubar of u'
        const D3 L0 = X1<B0>(0), L1 = X1<B1>(0);
        const double sx = fs4(L0, X1<B0>(FW), X1<B1>(FW), L1);
        const double sy = fs4(L0, L1, X1<B1>(1), X1<B0>(1));
        const double zs_next = zs<B1>();
        st3s(me, oF(0, 0), PL, ax);
        me[oF(0, 3)] = sx;
        st3s(me, oF(1, 0), PL, ay);
        me[oF(1, 3)] = sy;
        double rxy_n, ryx_n;
        rib_xy<B1>(t + 1, z1, rxy_n, ryx_n);
        double rxz = 0.0, ryz = 0.0, rzy = 0.0, rzx = 0.0;
        if (col_in) {
            const D3 T0 = D3{tx0, ty0, z0}, T1 = D3{tx0, ty0, z1};
            rxz = fs4(T0, T1, L1, L0);
            ryz = fs4(T0, L0, L1, T1);
            if (j + 1 <= p.ny) rzy = fs4(T0, D3{tx0, ty1, z0}, X1<B0>(FW), L0);
            if (i + 1 <= p.nx) rzx = fs4(T0, L0, X1<B0>(1), D3{tx1, ty0, z0});
        }
        me[oR(0)] = rxz;
        me[oR(1)] = ryz;
        me[oR(2)] = rzy;
        me[oR(3)] = rzx;
        D3 ubar = D3{0.0, 0.0, 0.0};
        if (cell_col) {
            D3 sum = U1<B0>(0);
            sum = add(sum, U1<B0>(1));
            sum = add(sum, U1<B0>(FW));
            sum = add(sum, U1<B0>(FW + 1));
            sum = add(sum, U1<B1>(0));
            sum = add(sum, U1<B1>(1));
            sum = add(sum, U1<B1>(FW));
            sum = add(sum, U1<B1>(FW + 1));
            ubar = scl(0.125, sum);
        }
        __syncthreads();
        // ---- P3: cell (i,j,t): V', W, e' (S7); swept volumes, donor data (R1, R2)
        if (cell_col && t < p.nz) {
            double sv[6] = {sx, me[1 + oF(0, 3)], sy, me[FW + oF(1, 3)], zs_prev, zs_next};
            const double V1 = vol_from_s(sv);
            if (t >= s.k0 && t < s.k1 && !(V1 > 0.0))
                atomicMin(&s.st->err_key, (ERR_ORDER_TANGLED << 48) | (unsigned long long)gcell(p, i, j, t));
            const D3 Az = ld3s(me, oZ(), PL);
            const D3 A[6] = {ax, ld3s(me + 1, oF(0, 0), PL), ay, ld3s(me + FW, oF(1, 0), PL), Az, Az};
            double W = 0.0;
            const bool dg = p.diag_areas;
#pragma unroll
            for (int h = 0; h < 8; ++h) {
                const int a = h & 1, b = (h >> 1) & 1, c = h >> 2;
                // axis-aligned areas: the corner vector is exactly (+-Ax.x, +-Ay.y, +-Az.z)
                const D3 C = dg ? D3{a ? A[1].x : -A[0].x, b ? A[3].y : -A[2].y, c ? A[5].z : -A[4].z}
                                : corner_vec(A, a, b, c);
                const D3 ub = c ? Ub<B1>(a + b * FW) : Ub<B0>(a + b * FW);
                const double term = dot(C, ub);
                W = (h == 0) ? term : W + term;
            }
            const long long cc = cb + (long long)t * s.pc;
            s.e1[cc] = e - ddiv((sig * W) * dt, m);
            st3(s.UD, cc, ubar);
            s.rD[cc] = ddiv(m, V1);
            if (t >= kr0 && t <= kr1) {
                if (t < kr1 && i >= 1)
                    s.dV[0][cc] = ddiv(((((me[FW + oR(0)] - me[oR(0)]) + rxy_n) - rxy_t) + sx) - sTx, 3.0);
                if (t < kr1 && j >= 1)
                    s.dV[1][cc] = ddiv(((((ryx_n - ryx_t) + me[1 + oR(1)]) - me[oR(1)]) + sy) - sTy, 3.0);
                if (t >= 1)
                    s.dV[2][cc] = ddiv(((((me[1 + oR(2)] - me[oR(2)]) + me[FW + oR(3)]) - me[oR(3)]) + zs_prev) - sTz, 3.0);
            }
        }
        zs_prev = zs_next;
        rxy_t = rxy_n;
        ryx_t = ryx_n;
        zprev = z1;
        __syncthreads();
    }

    __device__ __forceinline__ void run(int cur)
    {
        fetch(za, cur);
        if (za & 1) put<1>();
        else put<0>();
        zprev = fz;
        fetch(za + 1, cur);
        __syncthreads();
        zs_prev = (za & 1) ? zs<1>() : zs<0>();
        if (za & 1) rib_xy<1>(za, zprev, rxy_t, ryx_t);
        else rib_xy<0>(za, zprev, rxy_t, ryx_t);
        for (int t = za; t <= zb; ++t) {
            if (t & 1) step<1>(t, cur);
            else step<0>(t, cur);
        }
    }
};

template <int NW, int MB>
__global__ void __launch_bounds__(FW * NW, MB)
    kx_energy_sweep(Slab s, Phys p, int cur, int kc0, int kc1, int kr0, int kr1, int zchunk)
{
    if (!s.st->active) return;
    extern __shared__ double smem[];
    EnergySweepCTA<NW> c(s, p, smem, kc0, kc1, kr0, kr1, zchunk);
    c.run(cur);
}

template <int NW, int MB, int NM = 0>
__global__ void __launch_bounds__(FW * NW, MB) kf_energy_e(Slab s, Phys p, int cur, int kc0, int kc1, int zchunk)
{
    if (!s.st->active) return;
    extern __shared__ double smem[];
    EnergyEulerCTA<NW, NM> c(s, p, smem, kc0, kc1, zchunk);
    c.run(cur);
}

// ============================================================================
// launchers
// ============================================================================
namespace {
constexpr int NW_FORCE = 8;
constexpr int NW_ENERGY = 8;
constexpr int ZCHUNK = 32;

template <typename K>
void set_smem(K kernel, size_t bytes)
{
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

inline int cdiv(int a, int b) { return (a + b - 1) / b; }
}  // namespace

template <bool EULER, int NW, int NM = 0>
static void force_launch(const Slab& s, const Phys& p, int cur, int kn0, int kn1, int zc, cudaStream_t cs,
                         int sw0 = -1, int sw1 = -1)
{
    if (sw0 < 0) {  // sigma of the launch's own cell planes [kn0, kn1)
        sw0 = kn0;
        sw1 = kn1;
    }
    const size_t sm = sizeof(double) * ForceCTA<EULER, NW, NM>::WORDS;
    static bool init = false;
    if (!init) {
        set_smem(kf_force<EULER, NW, NM>, sm);
        init = true;
    }
    zc = zchunk_for((long long)cdiv(p.nx + 1, FW - 2) * cdiv(p.ny + 1, NW - 2), kn1 - kn0 + 1, zc);
    dim3 grid(cdiv(p.nx + 1, FW - 2), cdiv(p.ny + 1, NW - 2), cdiv(kn1 - kn0 + 1, zc));
    kf_force<EULER, NW, NM><<<grid, dim3(FW, NW), sm, cs>>>(s, p, cur, kn0, kn1, zc, sw0, sw1);
}
template <bool EULER, int NW, int MB, int NM = 0>
static void energy_launch(const Slab& s, const Phys& p, int cur, int kc0, int kc1, int zc, cudaStream_t cs)
{
    const size_t sm = sizeof(double) * EnergyCTA<EULER, NW, NM>::WORDS;
    static bool init = false;
    if (!init) {
        set_smem(kf_energy<EULER, NW, MB, NM>, sm);
        init = true;
    }
    zc = zchunk_for((long long)cdiv(p.nx, FW - 1) * cdiv(p.ny, NW - 1), kc1 - kc0, zc);
    dim3 grid(cdiv(p.nx, FW - 1), cdiv(p.ny, NW - 1), cdiv(kc1 - kc0, zc));
    kf_energy<EULER, NW, MB, NM><<<grid, dim3(FW, NW), sm, cs>>>(s, p, cur, kc0, kc1, zc);
}

// z-chunk length of the z-marching grids (SALE_ZCHUNK overrides, for tuning runs)
struct Tune {
    int zc = ZCHUNK;
    Tune()
    {
        if (const char* t = getenv("SALE_ZCHUNK")) zc = atoi(t);
        if (zc < 4) zc = 4;
    }
};

template <int NW, int MB>
static void force_e_launch(const Slab& s, const Phys& p, int cur, int kn0, int kn1, int zc, cudaStream_t cs)
{
    const size_t sm = sizeof(double) * ForceEulerCTA<NW>::WORDS;
    static bool init = false;
    if (!init) {
        set_smem(kf_force_e<NW, MB>, sm);
        init = true;
    }
    zc = zchunk_for((long long)cdiv(p.nx + 1, FW - 2) * cdiv(p.ny + 1, NW - 2), kn1 - kn0 + 1, zc);
    dim3 grid(cdiv(p.nx + 1, FW - 2), cdiv(p.ny + 1, NW - 2), cdiv(kn1 - kn0 + 1, zc));
    kf_force_e<NW, MB><<<grid, dim3(FW, NW), sm, cs>>>(s, p, cur, kn0, kn1, zc);
}

template <int NW, int MB, int NM = 0>
static void energy_e_launch(const Slab& s, const Phys& p, int cur, int kc0, int kc1, int zc, cudaStream_t cs)
{
    const size_t sm = sizeof(double) * EnergyEulerCTA<NW, NM>::WORDS;
    static bool init = false;
    if (!init) {
        set_smem(kf_energy_e<NW, MB, NM>, sm);
        init = true;
    }
    zc = zchunk_for((long long)cdiv(p.nx, FW - 1) * cdiv(p.ny, NW - 1), kc1 - kc0, zc);
    dim3 grid(cdiv(p.nx, FW - 1), cdiv(p.ny, NW - 1), cdiv(kc1 - kc0, zc));
    kf_energy_e<NW, MB, NM><<<grid, dim3(FW, NW), sm, cs>>>(s, p, cur, kc0, kc1, zc);
}

template <int NW, int MB, bool DIAG, int NM = 0>
static void sigma_e_launch(const Slab& s, const Phys& p, int cur, int kc0, int kc1, int zc, int gate, cudaStream_t cs)
{
    const size_t sm = sizeof(double) * SigmaEulerCTA<NW, DIAG, NM>::WORDS;
    static bool init = false;
    if (!init) {
        set_smem(kf_sigma_e<NW, MB, DIAG, NM>, sm);
        init = true;
    }
    zc = zchunk_for((long long)cdiv(p.nx, FW - 1) * cdiv(p.ny, NW - 1), kc1 - kc0, zc);
    dim3 grid(cdiv(p.nx, FW - 1), cdiv(p.ny, NW - 1), cdiv(kc1 - kc0, zc));
    kf_sigma_e<NW, MB, DIAG, NM><<<grid, dim3(FW, NW), sm, cs>>>(s, p, cur, kc0, kc1, zc, gate);
}

template <int NW, int MB>
static void esweep_launch(const Slab& s, const Phys& p, int cur, int kc0, int kc1, int zc, cudaStream_t cs)
{
    const size_t sm = sizeof(double) * EnergySweepCTA<NW>::WORDS;
    static bool init = false;
    if (!init) {
        set_smem(kx_energy_sweep<NW, MB>, sm);
        init = true;
    }
    const int kr0 = s.k0 - 1 > 0 ? s.k0 - 1 : 0, kr1 = s.k1 + 1 < p.nz ? s.k1 + 1 : p.nz;
    zc = zchunk_for((long long)cdiv(p.nx, FW - 1) * cdiv(p.ny, NW - 1), kc1 - kc0, zc);
    dim3 grid(cdiv(p.nx, FW - 1), cdiv(p.ny, NW - 1), cdiv(kc1 - kc0, zc));
    kx_energy_sweep<NW, MB><<<grid, dim3(FW, NW), sm, cs>>>(s, p, cur, kc0, kc1, kr0, kr1, zc);
}

// Euler: kf_energy_e + kr_sweep as one kernel (SALE_ESWEEP=1).  Measured 2% slower
// than the two kernels on C4 (210 registers: 12 warps/SM), so off by default.
int euler_esweep_variant()
{
    static const int v = [] {
        const char* e = getenv("SALE_ESWEEP");
        return e ? atoi(e) : 0;
    }();
    return v;
}

template <bool EULER>
static int lagrange_fused(const Slab& s, const Phys& p, int cur, Stream st)
{
    static const Tune tune;
    cudaStream_t cs = (cudaStream_t)st;
    if constexpr (EULER) {
        // node planes updated / cell planes energised, plus the ghost region the remap needs
        const int kn0 = imax_h(s.k0 - 2, 0), kn1 = imin_h(s.k1 + 2, p.nz);
        if (euler_pre_sigma())  // split form: kf_sigma_e ran before the cycle's k_begin
            kn_force_e<<<dim3(cdiv((int)s.pn, 256), kn1 - kn0 + 1), 256, 0, cs>>>(s, p, cur, kn0,
                                                                                  euler_x1_stored() ? 1 : 0);
        else  // SALE_FORCE_E=1: the one-kernel form
            force_e_launch<8, 2>(s, p, cur, kn0, kn1, tune.zc, cs);
        // kf_energy_e also writes the moved-face s' kr_sweep reads (Slab::sF)
        if (euler_esweep_variant() > 0) esweep_launch<12, 1>(s, p, cur, kn0, kn1, tune.zc, cs);
        else energy_e_launch<8, 2>(s, p, cur, kn0, kn1, tune.zc, cs);
    } else {
        force_launch<false, NW_FORCE>(s, p, cur, s.k0, s.k1, tune.zc, cs);
        energy_launch<false, NW_ENERGY, MINB>(s, p, cur, s.k0, s.k1, tune.zc, cs);
    }
    return 2;
}

// Euler, split force: sigma (and the cycle-start dt candidate, which replaces the
// remap's kn_dt pass) of cell planes [kn0-1, kn1], launched before k_begin
bool euler_pre_sigma()
{
    static const int fe = [] {
        const char* v = getenv("SALE_FORCE_E");
        return v ? atoi(v) : 0;
    }();
    return fe != 1;
}
int launch_euler_pre(const Slab& s, const Phys& p, int cur, int gate, Stream st)
{
    static const Tune tune;
    const int kn0 = imax_h(s.k0 - 2, 0), kn1 = imin_h(s.k1 + 2, p.nz);
    const int sc0 = kn0 - 1 > 0 ? kn0 - 1 : 0, sc1 = kn1 + 1 < p.nz ? kn1 + 1 : p.nz;
    if (p.diag_jumps) sigma_e_launch<8, 2, true>(s, p, cur, sc0, sc1, tune.zc, gate, (cudaStream_t)st);
    else sigma_e_launch<8, 2, false>(s, p, cur, sc0, sc1, tune.zc, gate, (cudaStream_t)st);
    return 1;
}

// Euler, multi-material cells: kf_sigma_e with the mixed closure (sigma, the materials'
// stresses, the dt candidate), before the cycle's k_begin, over launch_euler_pre's planes
int launch_sigma_e_mat(const Slab& s, const Phys& p, int cur, int gate, Stream st)
{
    static const Tune tune;
    const int kn0 = imax_h(s.k0 - 2, 0), kn1 = imin_h(s.k1 + 2, p.nz);
    const int sc0 = kn0 - 1 > 0 ? kn0 - 1 : 0, sc1 = kn1 + 1 < p.nz ? kn1 + 1 : p.nz;
    cudaStream_t cs = (cudaStream_t)st;
    auto go = [&](auto dg) {
        constexpr bool DG = decltype(dg)::value;
        switch (s.nmat) {
        case 1: sigma_e_launch<8, 2, DG, 1>(s, p, cur, sc0, sc1, tune.zc, gate, cs); break;
        case 2: sigma_e_launch<8, 2, DG, 2>(s, p, cur, sc0, sc1, tune.zc, gate, cs); break;
        case 3: sigma_e_launch<8, 2, DG, 3>(s, p, cur, sc0, sc1, tune.zc, gate, cs); break;
        default: sigma_e_launch<8, 2, DG, 4>(s, p, cur, sc0, sc1, tune.zc, gate, cs); break;
        }
    };
    if (p.diag_jumps) go(std::true_type{});
    else go(std::false_type{});
    return 1;
}

// Lagrange, multi-material cells: S1-S6 in one z-march with the mixed closure (kf_force
// with NM materials; writes sigma, the materials' stresses, x', u'), then S7 per
// material + the dt candidate (kf_energy with NM materials)
int launch_force_mat(const Slab& s, const Phys& p, int cur, Stream st)
{
    static const Tune tune;
    cudaStream_t cs = (cudaStream_t)st;
    // (energy: two 8-warp CTAs per SM at 128 registers for 1-2 materials, measured
    // faster despite the spill; one CTA for 3-4, whose larger spill made it slower)
    switch (s.nmat) {
    case 1:
        force_launch<false, NW_FORCE, 1>(s, p, cur, s.k0, s.k1, tune.zc, cs);
        energy_launch<false, NW_ENERGY, 2, 1>(s, p, cur, s.k0, s.k1, tune.zc, cs);
        break;
    case 2:
        force_launch<false, NW_FORCE, 2>(s, p, cur, s.k0, s.k1, tune.zc, cs);
        energy_launch<false, NW_ENERGY, 2, 2>(s, p, cur, s.k0, s.k1, tune.zc, cs);
        break;
    case 3:
        force_launch<false, NW_FORCE, 3>(s, p, cur, s.k0, s.k1, tune.zc, cs);
        energy_launch<false, NW_ENERGY, 1, 3>(s, p, cur, s.k0, s.k1, tune.zc, cs);
        break;
    default:
        force_launch<false, NW_FORCE, 4>(s, p, cur, s.k0, s.k1, tune.zc, cs);
        energy_launch<false, NW_ENERGY, 1, 4>(s, p, cur, s.k0, s.k1, tune.zc, cs);
        break;
    }
    return 2;
}

// Euler, multi-material cells: S7 per material (kf_energy_e with NM materials; writes
// e'_k, V', and the moved-face s' kr_sweep reads), over lagrange_fused's planes
int launch_energy_e_mat(const Slab& s, const Phys& p, int cur, Stream st)
{
    static const Tune tune;
    const int kn0 = imax_h(s.k0 - 2, 0), kn1 = imin_h(s.k1 + 2, p.nz);
    cudaStream_t cs = (cudaStream_t)st;
    switch (s.nmat) {
    case 1: energy_e_launch<8, 2, 1>(s, p, cur, kn0, kn1, tune.zc, cs); break;
    case 2: energy_e_launch<8, 2, 2>(s, p, cur, kn0, kn1, tune.zc, cs); break;
    case 3: energy_e_launch<8, 2, 3>(s, p, cur, kn0, kn1, tune.zc, cs); break;
    default: energy_e_launch<8, 2, 4>(s, p, cur, kn0, kn1, tune.zc, cs); break;
    }
    return 1;
}

// Euler S5-S6 node gather on sigma and the cell totals (the material path reuses it)
int launch_kn_force_e(const Slab& s, const Phys& p, int cur, Stream st)
{
    const int kn0 = imax_h(s.k0 - 2, 0), kn1 = imin_h(s.k1 + 2, p.nz);
    kn_force_e<<<dim3(cdiv((int)s.pn, 256), kn1 - kn0 + 1), 256, 0, (cudaStream_t)st>>>(s, p, cur, kn0,
                                                                                         euler_x1_stored() ? 1 : 0);
    return 1;
}

// Lagrange, boundary-first: part 0 = what the halo exchange sends
// (node planes [k0, k0+g] and [k1-g, k1] with their cells [k0, k0+g) and [k1-g, k1)),
// part 1 = the interior (node planes (k0+g, k1-g), cells [k0+g, k1-g)).  The two parts
// are exactly the work of launch_lagrange_fused; the exchange can start after part 0.
// A slab too thin to have an interior runs whole as part 0.
int launch_lagrange_fused_part(const Slab& s, const Phys& p, int cur, int part, Stream st)
{
    static const Tune tune;
    cudaStream_t cs = (cudaStream_t)st;
    const int g = s.g, k0 = s.k0, k1 = s.k1;
    if (k1 - k0 < 2 * g + 2) return part == 0 ? lagrange_fused<false>(s, p, cur, st) : 0;
    // sigma write ranges: the cell next to each split is written by both neighbouring
    // launches (same bits, stream order), so every energy range finds its sigma
    if (part == 0) {
        force_launch<false, NW_FORCE>(s, p, cur, k0, k0 + g, tune.zc, cs, k0, k0 + g + 1);
        energy_launch<false, NW_ENERGY, MINB>(s, p, cur, k0, k0 + g, tune.zc, cs);
        force_launch<false, NW_FORCE>(s, p, cur, k1 - g, k1, tune.zc, cs, k1 - g - 1, k1);
        energy_launch<false, NW_ENERGY, MINB>(s, p, cur, k1 - g, k1, tune.zc, cs);
        return 4;
    }
    force_launch<false, NW_FORCE>(s, p, cur, k0 + g + 1, k1 - g - 1, tune.zc, cs, k0 + g, k1 - g);
    energy_launch<false, NW_ENERGY, MINB>(s, p, cur, k0 + g, k1 - g, tune.zc, cs);
    return 2;
}

int launch_lagrange_fused(const Slab& s, const Phys& p, int cur, Stream st)
{
    return p.rezone ? lagrange_fused<true>(s, p, cur, st) : lagrange_fused<false>(s, p, cur, st);
}


}  // namespace sale
