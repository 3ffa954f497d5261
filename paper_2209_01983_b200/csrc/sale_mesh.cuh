// sale_mesh.cuh -- slab indexing and state loaders shared by the kernels.
#pragma once
#include "sale_geom.cuh"

namespace sale {

// local linear node / cell index of GLOBAL (i, j, k)
__device__ __forceinline__ long long nidx(const Slab& s, const Phys& p, int i, int j, int k)
{
    return (long long)i + (long long)(p.nx + 1) * ((long long)j + (long long)(p.ny + 1) * (k - s.kb));
}
__device__ __forceinline__ long long cidx(const Slab& s, const Phys& p, int i, int j, int k)
{
    return (long long)i + (long long)p.nx * ((long long)j + (long long)p.ny * (k - s.kb));
}
// global linear cell index (for error reports)
__device__ __forceinline__ long long gcell(const Phys& p, int i, int j, int k)
{
    return (long long)i + (long long)p.nx * ((long long)j + (long long)p.ny * k);
}
__device__ __forceinline__ bool cell_in(const Phys& p, int i, int j, int k)
{
    return i >= 0 && i < p.nx && j >= 0 && j < p.ny && k >= 0 && k < p.nz;
}

// node position at the start of the cycle: Lagrange from x[b], Euler x^T
template <bool EULER>
__device__ __forceinline__ D3 pos(const Slab& s, const Phys& p, int b, int i, int j, int k)
{
    if (EULER) return D3{s.Xt[i], s.Yt[j], s.Zt[k - s.kb]};
    long long n = nidx(s, p, i, j, k);
    return D3{s.x[b][0][n], s.x[b][1][n], s.x[b][2][n]};
}
__device__ __forceinline__ D3 tpos(const Slab& s, int i, int j, int k)
{
    return D3{s.Xt[i], s.Yt[j], s.Zt[k - s.kb]};
}
__device__ __forceinline__ D3 ld3(double* const a[3], long long n)
{
    return D3{a[0][n], a[1][n], a[2][n]};
}
__device__ __forceinline__ void st3(double* const a[3], long long n, D3 v)
{
    a[0][n] = v.x;
    a[1][n] = v.y;
    a[2][n] = v.z;
}

// ---- peer-store halo (HaloPeer, sale_internal.h) --------------------------------
// The neighbour sides that receive global node plane k (bit 0: lower, its ghost
// planes [k0+1, k0+g]; bit 1: upper, [k1-g, k1-1]) and cell plane k ([k0, k0+g) /
// [k1-g, k1)): the planes the copy exchange sends (build_plan).
__device__ __forceinline__ int halo_sides_node(const Slab& s, int k)
{
    return ((k >= s.k0 + 1 && k <= s.k0 + s.g) ? 1 : 0) | ((k >= s.k1 - s.g && k <= s.k1 - 1) ? 2 : 0);
}
__device__ __forceinline__ int halo_sides_cell(const Slab& s, int k)
{
    return ((k >= s.k0 && k < s.k0 + s.g) ? 1 : 0) | ((k >= s.k1 - s.g && k < s.k1) ? 2 : 0);
}
// store node value v (three components of arrays a[side][b]) of global plane k,
// in-plane index q, into the neighbours' ghost planes
__device__ __forceinline__ void halo_node3(const Slab& s, double* const (*a)[2][3], int b, int k, long long q,
                                           D3 v)
{
    const int sides = halo_sides_node(s, k);
#pragma unroll
    for (int side = 0; side < 2; ++side) {
        if (!((sides >> side) & 1)) continue;
        double* const* d = a[side][b];
        double* const d0 = d[0];
        if (!d0) continue;
        const long long o = (long long)(k - s.hp->kb[side]) * s.pn + q;
        d0[o] = v.x;
        d[1][o] = v.y;
        d[2][o] = v.z;
    }
}
// cell value v of array a[side][b] (+ material k's offset), global plane k, in-plane q
__device__ __forceinline__ void halo_cell(const Slab& s, double* const (*a)[2], int b, int mat, int k, long long q,
                                          double v)
{
    const int sides = halo_sides_cell(s, k);
#pragma unroll
    for (int side = 0; side < 2; ++side) {
        if (!((sides >> side) & 1)) continue;
        double* const d = a[side][b];
        if (!d) continue;
        d[(long long)(k - s.hp->kb[side]) * s.pc + q + mat * s.hp->mstride[side]] = v;
    }
}

// the first plane offset of this CTA's z-chunk.  A launch passes zchunk < 0 to run its
// chunks in reverse order (consecutive kernels alternate, so each starts on the planes
// the previous one finished last, whose data are still in L2); zchunk is made positive.
// The order of the chunks never changes a result (each CTA's work is independent).
__device__ __forceinline__ int zchunk_base(int& zchunk)
{
    const bool rev = zchunk < 0;
    if (rev) zchunk = -zchunk;
    return (int)(rev ? gridDim.z - 1 - blockIdx.z : blockIdx.z) * zchunk;
}

// asynchronous global -> shared copies (cp.async, 8 B): a node plane is staged
// without passing through registers (no prefetch registers held across a step)
__device__ __forceinline__ void cpa8(double* sdst, const double* gsrc)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cpa3(double* sdst, int stride, double* const a[3], long long n)
{
    cpa8(sdst, a[0] + n);
    cpa8(sdst + stride, a[1] + n);
    cpa8(sdst + 2 * stride, a[2] + n);
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// the 8 nodes of cell (i,j,k) in hex order (c*2+b)*2+a
template <bool EULER>
__device__ __forceinline__ void load_hex_pos(const Slab& s, const Phys& p, int b, int i, int j,
                                             int k, D3 N[8])
{
#pragma unroll
    for (int h = 0; h < 8; ++h) N[h] = pos<EULER>(s, p, b, i + (h & 1), j + ((h >> 1) & 1), k + (h >> 2));
}
__device__ __forceinline__ void load_hex3(const Slab& s, const Phys& p, double* const a[3], int i,
                                          int j, int k, D3 N[8])
{
#pragma unroll
    for (int h = 0; h < 8; ++h)
        N[h] = ld3(a, nidx(s, p, i + (h & 1), j + ((h >> 1) & 1), k + (h >> 2)));
}

// reflecting boundary: zero the normal component on reflecting planes (c.3 step 6)
__device__ __forceinline__ D3 reflect(const Phys& p, int i, int j, int k, D3 v)
{
    unsigned r = p.reflect;
    if (((r & 1u) && i == 0) || ((r & 2u) && i == p.nx)) v.x = 0.0;
    if (((r & 4u) && j == 0) || ((r & 8u) && j == p.ny)) v.y = 0.0;
    if (((r & 16u) && k == 0) || ((r & 32u) && k == p.nz)) v.z = 0.0;
    return v;
}

__device__ __forceinline__ double* mass_cur(const Slab& s, const Phys& p, int cur)
{
    return p.rezone ? s.m[cur] : s.m[0];
}

// ---- multi-material cells (Phys::nmat >= 1) -----------------
__device__ __forceinline__ long long mat_stride(const Slab& s) { return s.pc * (long long)s.nzc; }
// the material arrays of the state in buffer b (Lagrange: f_k and m_k never change)
__device__ __forceinline__ const double* mat_f(const Slab& s, const Phys& p, int b)
{
    return p.rezone ? s.mf[b] : s.mf[0];
}
__device__ __forceinline__ const double* mat_m(const Slab& s, const Phys& p, int b)
{
    return p.rezone ? s.mm[b] : s.mm[0];
}

// per-cell material operands a z-march kernel prefetches into registers: volume
// fraction, mass, specific energy, stress (NM = 0: an empty base, so the single-material
// instantiations keep their original layout and code)
template <int NM>
struct MatRegs {
    double rf[NM], rm[NM], re[NM], rs[NM];
};
template <>
struct MatRegs<0> {
};

// MM1: the mixed-cell closure of cell c (material k at c + k*stride) at volume V and
// cell density rho: each present material (f_k > 0) at rho_k = m_k / (f_k V) through
// the c.3 step 1 EoS with its own gamma; pr = sum f_k p_k, P = sum f_k pf_k,
// cs = sqrt((sum f_k (gamma_k pf_k)) / rho); sums left to right from the first present
// material.  pf[k] = 0 for absent materials.  One material with f_0 = 1 gives eos()'s
// bits (1.0 * a = a).  NM > 0: the material count as a compile-time constant (the
// loop unrolls, pf stays in registers); NM = 0: p.nmat.
template <int NM>
__device__ __forceinline__ void mix_eos_r(const Slab& s, const double* f, const double* mm, const double* e, double V,
                                          double rho, double& pr, double& P, double& cs, double pf[MAX_MAT])
{
    double ps = 0.0, Ps = 0.0, G = 0.0;
    bool first = true;
#pragma unroll
    for (int k = 0; k < (NM ? NM : s.nmat); ++k) {
        pf[k] = 0.0;
        const double fk = f[k];
        if (!(fk > 0.0)) continue;
        const double rk = ddiv(mm[k], fk * V);
        const double pk = ((s.mg[k] - 1.0) * rk) * e[k];
        const double pfk = (pk > 0.0) ? pk : 0.0;
        pf[k] = pfk;
        const double a = fk * pk, b = fk * pfk, g = fk * (s.mg[k] * pfk);
        if (first) {
            ps = a;
            Ps = b;
            G = g;
            first = false;
        } else {
            ps = ps + a;
            Ps = Ps + b;
            G = G + g;
        }
    }
    pr = ps;
    P = Ps;
    cs = dsqrt(ddiv(G, rho));
}
// the same from the material arrays of cell c (material k at c + k*stride)
template <int NM>
__device__ __forceinline__ void mix_eos_t(const Slab& s, const double* f, const double* mm, const double* e,
                                          long long c, long long stride, double V, double rho, double& pr,
                                          double& P, double& cs, double pf[MAX_MAT])
{
    double fr[MAX_MAT], mr[MAX_MAT], er[MAX_MAT];
#pragma unroll
    for (int k = 0; k < (NM ? NM : s.nmat); ++k) {
        fr[k] = f[c + k * stride];
        mr[k] = mm[c + k * stride];
        er[k] = e[c + k * stride];
    }
    mix_eos_r<NM>(s, fr, mr, er, V, rho, pr, P, cs, pf);
}
__device__ __forceinline__ void mix_eos(const Slab& s, const double* f, const double* mm, const double* e,
                                        long long c, long long stride, double V, double rho, double& pr,
                                        double& P, double& cs, double pf[MAX_MAT])
{
    mix_eos_t<0>(s, f, mm, e, c, stride, V, rho, pr, P, cs, pf);
}

// host: z-chunk length of a z-marching grid.  Large meshes use zc0 planes per CTA;
// small ones shorter chunks (down to 4) so the grid still covers the 148 SMs twice
// (a z-march is a chain of dependent plane steps; its length is the small-mesh time).
// Chunking changes only which CTA computes a plane, never the arithmetic.
#ifndef SALE_ZALT
#define SALE_ZALT 1
#endif
// host: the zchunk argument of the next z-march launch, its chunk order alternating
// from launch to launch (zchunk_base; performance only)
inline int zorder(int zc)
{
    static thread_local unsigned n = 0;
    return (SALE_ZALT && (n++ & 1u)) ? -zc : zc;
}
inline int zchunk_for(long long ctas_xy, int planes, int zc0)
{
    int zc = zc0;
    while (zc > 4 && ctas_xy * ((planes + zc - 1) / zc) < 2 * 148) zc /= 2;
    return zc;
}



}  // namespace sale
