// sale_geom.cuh -- device primitives of the SALE cycle.
//
// All arithmetic is fp64 with the association written in SURVEY §8(c); the
// library is compiled with -fmad=false so no a*b+c is contracted into DFMA, and
// with IEEE div/sqrt (nvcc defaults), so every value is bit-identical to any
// other correctly rounded evaluation of the same expression tree.
#pragma once
#include <cstdint>

#include "sale_internal.h"

namespace sale {

struct D3 {
    double x, y, z;
};

__device__ __forceinline__ D3 d3(double x, double y, double z) { return D3{x, y, z}; }
__device__ __forceinline__ D3 sub(D3 a, D3 b) { return D3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ D3 add(D3 a, D3 b) { return D3{a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ D3 neg(D3 a) { return D3{-a.x, -a.y, -a.z}; }
__device__ __forceinline__ D3 scl(double s, D3 a) { return D3{s * a.x, s * a.y, s * a.z}; }
// (a.x*b.x + a.y*b.y) + a.z*b.z
__device__ __forceinline__ double dot(D3 a, D3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }

// IEEE a / b (round to nearest).  A zero numerator over a finite non-zero
// divisor returns a * b -- the same signed zero the division produces -- without
// entering the division's out-of-line slow path, which CUDA's fp64 division takes
// for zero operands.  Zero numerators are the common case in the quiescent part
// of the Sedov domain (zero velocity jumps, forces, fluxes), so this is a large
// saving there; results are bit-identical to a / b for every input.
__device__ __forceinline__ double ddiv(double a, double b)
{
    if (a == 0.0 && b != 0.0 && fabs(b) < __longlong_as_double(0x7FF0000000000000ll)) return a * b;
    return a / b;
}
// IEEE sqrt; sqrt(+-0) = +-0 without the slow path
__device__ __forceinline__ double dsqrt(double x)
{
    if (x == 0.0) return x;
    return sqrt(x);
}

// min / max with the exact semantics of the written "(b < a) ? b : a"
__device__ __forceinline__ double dmin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double dmax(double a, double b) { return (b > a) ? b : a; }

// c.2 face area vector A = 0.5 * ((P2-P0) x (P3-P1))
__device__ __forceinline__ D3 face_area(D3 P0, D3 P1, D3 P2, D3 P3)
{
    D3 d1 = sub(P2, P0), d2 = sub(P3, P1);
    return D3{0.5 * (d1.y * d2.z - d1.z * d2.y), 0.5 * (d1.z * d2.x - d1.x * d2.z),
              0.5 * (d1.x * d2.y - d1.y * d2.x)};
}
// c.2 face centroid 0.25 * (((P0+P1)+P2)+P3)  (also the face-average velocity)
__device__ __forceinline__ D3 avg4(D3 P0, D3 P1, D3 P2, D3 P3)
{
    return scl(0.25, add(add(add(P0, P1), P2), P3));
}
// c.2 s = (Xb.x*A.x + Xb.y*A.y) + Xb.z*A.z
__device__ __forceinline__ double face_s(D3 Xb, D3 A) { return dot(Xb, A); }

// Hex-local node (a,b,c) -> index (c*2+b)*2+a.  Canonical face node lists
// (X(a), Y(b), Z(c) as in c.2):
//   X0 {0,2,6,4}  X1 {1,3,7,5}  Y0 {0,4,5,1}  Y1 {2,6,7,3}  Z0 {0,1,3,2}  Z1 {4,5,7,6}
__device__ __forceinline__ void hex_face_nodes(int f, int& a, int& b, int& c, int& d)
{
    switch (f) {
    case 0: a = 0; b = 2; c = 6; d = 4; break;
    case 1: a = 1; b = 3; c = 7; d = 5; break;
    case 2: a = 0; b = 4; c = 5; d = 1; break;
    case 3: a = 2; b = 6; c = 7; d = 3; break;
    case 4: a = 0; b = 1; c = 3; d = 2; break;
    default: a = 4; b = 5; c = 7; d = 6; break;
    }
}

// c.2 volume from the six face s-values, order X0 X1 Y0 Y1 Z0 Z1:
// (((((s1 - s0) + s3) - s2) + s5) - s4) / 3.0
__device__ __forceinline__ double vol_from_s(const double s[6])
{
    return ddiv((((((s[1] - s[0]) + s[3]) - s[2]) + s[5]) - s[4]), 3.0);
}

// full hex: areas, centroids, s of the six faces
__device__ __forceinline__ void hex_faces(const D3 N[8], D3 A[6], D3 Xb[6], double s[6])
{
#pragma unroll
    for (int f = 0; f < 6; ++f) {
        int a, b, c, d;
        hex_face_nodes(f, a, b, c, d);
        A[f] = face_area(N[a], N[b], N[c], N[d]);
        Xb[f] = avg4(N[a], N[b], N[c], N[d]);
        s[f] = face_s(Xb[f], A[f]);
    }
}

__device__ __forceinline__ double hex_volume(const D3 N[8])
{
    D3 A[6], Xb[6];
    double s[6];
    hex_faces(N, A, Xb, s);
    return vol_from_s(s);
}

// c.2 corner vector of hex corner (a,b,c): ((Ax(a) + Ay(b)) + Az(c)),
// Ax(1) = A[X1], Ax(0) = -A[X0], likewise y, z
__device__ __forceinline__ D3 corner_vec(const D3 A[6], int a, int b, int c)
{
    D3 ax = a ? A[1] : neg(A[0]);
    D3 ay = b ? A[3] : neg(A[2]);
    D3 az = c ? A[5] : neg(A[4]);
    return add(add(ax, ay), az);
}

// c.3 step 1: p = ((g-1)*rho)*e; pf = p > 0 ? p : 0; c = sqrt((g*pf)/rho)
__device__ __forceinline__ void eos(double g, double rho, double e, double& p, double& pf,
                                    double& cs)
{
    p = ((g - 1.0) * rho) * e;
    pf = (p > 0.0) ? p : 0.0;
    cs = dsqrt(ddiv(g * pf, rho));
}

// c.3 step 2 (per axis): delta = (w . d) / sqrt(d . d)
__device__ __forceinline__ double axis_jump(D3 Xm, D3 Xp, D3 Um, D3 Up)
{
    D3 d = sub(Xp, Xm);
    D3 w = sub(Up, Um);
    double L = dsqrt((d.x * d.x + d.y * d.y) + d.z * d.z);
    return ddiv((w.x * d.x + w.y * d.y) + w.z * d.z, L);
}

// c.3 step 2 last line
__device__ __forceinline__ double q_of_du(double rho, double cs, double du, double c1, double c2)
{
    return (du < 0.0) ? rho * ((c2 * (du * du)) + ((c1 * cs) * (-du))) : 0.0;
}

// c.3 step 2 (per axis) also returning the separation L = sqrt(d . d) (reading HG)
__device__ __forceinline__ double axis_jump_L(D3 Xm, D3 Xp, D3 Um, D3 Up, double& L)
{
    D3 d = sub(Xp, Xm);
    D3 w = sub(Up, Um);
    L = dsqrt((d.x * d.x + d.y * d.y) + d.z * d.z);
    return ddiv((w.x * d.x + w.y * d.y) + w.z * d.z, L);
}

// c.3 step 2 for a hex: face-average velocities over the canonical face nodes;
// du = min over the axes, Lsum = ((Lx + Ly) + Lz)
__device__ __forceinline__ double hex_du(const D3 Xb[6], const D3 U[8], double& Lsum)
{
    double dl[3], L[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        int a, b, c, d;
        hex_face_nodes(2 * ax, a, b, c, d);
        D3 Um = avg4(U[a], U[b], U[c], U[d]);
        hex_face_nodes(2 * ax + 1, a, b, c, d);
        D3 Up = avg4(U[a], U[b], U[c], U[d]);
        dl[ax] = axis_jump_L(Xb[2 * ax], Xb[2 * ax + 1], Um, Up, L[ax]);
    }
    Lsum = (L[0] + L[1]) + L[2];
    return dmin(dmin(dl[0], dl[1]), dl[2]);
}
__device__ __forceinline__ double hex_q(const D3 Xb[6], const D3 U[8], double rho, double cs,
                                        double c1, double c2)
{
    double Lsum;
    return q_of_du(rho, cs, hex_du(Xb, U, Lsum), c1, c2);
}

// reading DT-Q: viscous signal speed of a compressing cell,
// cq = 2*((c1*c) + (c2*(-du))) for du < 0, else 0
__device__ __forceinline__ double visc_speed(double cs, double du, double c1, double c2)
{
    return (du < 0.0) ? 2.0 * ((c1 * cs) + (c2 * (-du))) : 0.0;
}

// c.5 with DT-Q: dt_K = (cfl*sqrt(l2)) / (((c + sqrt(v2)) + cq) + 1e-30)
__device__ __forceinline__ double dt_cell(double cfl, double l2, double v2, double cs, double cq)
{
    return ddiv(cfl * dsqrt(l2), ((cs + dsqrt(v2)) + cq) + 1e-30);
}
// the same with the numerator cfl*sqrt(l2) given (tabled on the Euler target mesh)
__device__ __forceinline__ double dt_cell_num(double num, double v2, double cs, double cq)
{
    return ddiv(num, ((cs + dsqrt(v2)) + cq) + 1e-30);
}

// ---- reading HG: viscous hourglass damping ---------------------
// Gamma_m(h) on hex corner h = (c*2+b)*2+a, xi = 2a-1, eta = 2b-1, zeta = 2c-1:
// m = 0 xi*eta, 1 eta*zeta, 2 zeta*xi, 3 xi*eta*zeta.  Returns +1 / -1.
__host__ __device__ constexpr int hg_gamma(int m, int h)
{
    return (m == 0)   ? (((h & 1) ? 1 : -1) * ((h & 2) ? 1 : -1))
           : (m == 1) ? (((h & 2) ? 1 : -1) * ((h & 4) ? 1 : -1))
           : (m == 2) ? (((h & 4) ? 1 : -1) * ((h & 1) ? 1 : -1))
                      : (((h & 1) ? 1 : -1) * ((h & 2) ? 1 : -1) * ((h & 4) ? 1 : -1));
}
// a + G*b for G = +-1 (exact: the product is a sign flip)
__device__ __forceinline__ D3 addsg(D3 a, D3 b, int G) { return G > 0 ? add(a, b) : sub(a, b); }
__device__ __forceinline__ double addsg(double a, double b, int G) { return G > 0 ? a + b : a - b; }
// g_m = sum over h = 0..7, left to right, of Gamma_m(h) U_h (componentwise)
template <int M>
__device__ __forceinline__ D3 hg_mode(const D3 U[8])
{
    D3 s = hg_gamma(M, 0) > 0 ? U[0] : neg(U[0]);
#pragma unroll
    for (int h = 1; h < 8; ++h) s = addsg(s, U[h], hg_gamma(M, h));
    return s;
}
__device__ __forceinline__ void hg_modes(const D3 U[8], D3 g[4])
{
    g[0] = hg_mode<0>(U);
    g[1] = hg_mode<1>(U);
    g[2] = hg_mode<2>(U);
    g[3] = hg_mode<3>(U);
}
// corner force of corner H: f = -(nu * (((G0 g0 + G1 g1) + G2 g2) + G3 g3))
template <int H>
__device__ __forceinline__ D3 hg_corner(const D3 g[4], double nu)
{
    D3 t = hg_gamma(0, H) > 0 ? g[0] : neg(g[0]);
    t = addsg(t, g[1], hg_gamma(1, H));
    t = addsg(t, g[2], hg_gamma(2, H));
    t = addsg(t, g[3], hg_gamma(3, H));
    return D3{-(nu * t.x), -(nu * t.y), -(nu * t.z)};
}
__device__ __forceinline__ D3 hg_corner_rt(const D3 g[4], double nu, int h)
{
    switch (h) {
    case 0: return hg_corner<0>(g, nu);
    case 1: return hg_corner<1>(g, nu);
    case 2: return hg_corner<2>(g, nu);
    case 3: return hg_corner<3>(g, nu);
    case 4: return hg_corner<4>(g, nu);
    case 5: return hg_corner<5>(g, nu);
    case 6: return hg_corner<6>(g, nu);
    default: return hg_corner<7>(g, nu);
    }
}
// uncapped coefficient nu_u = (hg*(m*c)) / (Lsum/3), Lsum = ((Lx+Ly)+Lz)
__device__ __forceinline__ double hg_nu(double hg, double m, double cs, double Lsum)
{
    return ddiv(hg * (m * cs), ddiv(Lsum, 3.0));
}
// nu = min(nu_u, (m/64)/dt)
__device__ __forceinline__ double hg_cap(double nu_u, double m, double dt)
{
    return dmin(nu_u, ddiv(ddiv(m, 64.0), dt));
}

__device__ __forceinline__ double len2(D3 a, D3 b)
{
    D3 d = sub(b, a);
    return (d.x * d.x + d.y * d.y) + d.z * d.z;
}

// c.5 per-cell l2 = min over the 12 edges, v2 = max over the 8 nodes
__device__ __forceinline__ double hex_min_edge2(const D3 N[8])
{
    double l = len2(N[0], N[1]);
    l = dmin(l, len2(N[2], N[3]));
    l = dmin(l, len2(N[4], N[5]));
    l = dmin(l, len2(N[6], N[7]));
    l = dmin(l, len2(N[0], N[2]));
    l = dmin(l, len2(N[1], N[3]));
    l = dmin(l, len2(N[4], N[6]));
    l = dmin(l, len2(N[5], N[7]));
    l = dmin(l, len2(N[0], N[4]));
    l = dmin(l, len2(N[1], N[5]));
    l = dmin(l, len2(N[2], N[6]));
    l = dmin(l, len2(N[3], N[7]));
    return l;
}
__device__ __forceinline__ double speed2(D3 u) { return (u.x * u.x + u.y * u.y) + u.z * u.z; }
__device__ __forceinline__ double hex_max_speed2(const D3 U[8])
{
    double v = speed2(U[0]);
#pragma unroll
    for (int h = 1; h < 8; ++h) v = dmax(v, speed2(U[h]));
    return v;
}

// order-free encoding of a dt candidate (>= +0 or NaN) for an unsigned min:
// NaN -> 0 (wins the min, propagates), else bits + 1 (monotone for x >= +0)
__device__ __forceinline__ unsigned long long dt_key(double dt)
{
    if (dt != dt) return 0ull;
    return (unsigned long long)__double_as_longlong(dt) + 1ull;
}
__device__ __forceinline__ double dt_unkey(unsigned long long k)
{
    if (k == 0ull) return __longlong_as_double(0x7FF8000000000000ll);
    if (k == KEY_NONE) return __longlong_as_double(0x7FF0000000000000ll);
    return __longlong_as_double((long long)(k - 1ull));
}

// c.4 step 1: swept volume of the hex (0,0,0)=PT0 (1,0,0)=PT1 (1,1,0)=PT2
// (0,1,0)=PT3, (0,0,1)=PL0 (1,0,1)=PL1 (1,1,1)=PL2 (0,1,1)=PL3
__device__ __forceinline__ double swept_volume(D3 T0, D3 T1, D3 T2, D3 T3, D3 L0, D3 L1, D3 L2,
                                               D3 L3)
{
    D3 N[8] = {T0, T1, T3, T2, L0, L1, L3, L2};
    return hex_volume(N);
}

// warp + block min of an unsigned 64-bit key, then one atomicMin per block
// (any block shape whose size is a multiple of 32; all threads must call it)
__device__ __forceinline__ void block_min_atomic(unsigned long long key, unsigned long long* dst)
{
    __shared__ unsigned long long red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
        key = other < key ? other : key;
    }
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int lane = tid & 31, wid = tid >> 5;
    const int nw = (blockDim.x * blockDim.y * blockDim.z + 31) >> 5;
    if (lane == 0) red[wid] = key;
    __syncthreads();
    if (wid == 0) {
        key = lane < nw ? red[lane] : KEY_NONE;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
            key = other < key ? other : key;
        }
        if (lane == 0 && key != KEY_NONE) atomicMin(dst, key);
    }
}

}  // namespace sale
