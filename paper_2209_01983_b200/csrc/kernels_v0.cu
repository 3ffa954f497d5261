// kernels_v0.cu -- the unfused bring-up path: one kernel per step of the cycle,
// one thread per cell or node, every operand straight from global memory.
// SURVEY §8(a) rows S1-S7, R1-R5; operator definitions SURVEY §8(c) c.3-c.5.
// Kept as the cross-check for the fused kernels (kernels_fused.cu).
#include <cuda_runtime.h>

#include "sale_mesh.cuh"

namespace sale {

static inline unsigned grid_for(long long n, int bs)
{
    long long g = (n + bs - 1) / bs;
    return (unsigned)(g > 0 ? g : 1);
}

// S1-S3: geometry at t^n, EoS, viscosity; sigma = 0.25 (pf + q)
template <bool EULER>
__global__ void k0_sigma(Slab s, Phys p, int cur, int ka0, int ka1)
{
    if (!s.st->active) return;
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= s.pc * (ka1 - ka0)) return;
    int k = ka0 + (int)(t / s.pc);
    long long r = t % s.pc;
    int j = (int)(r / p.nx), i = (int)(r % p.nx);
    D3 N[8], U[8], A[6], Xb[6];
    double sv[6];
    load_hex_pos<EULER>(s, p, cur, i, j, k, N);
    load_hex3(s, p, s.u[cur], i, j, k, U);
    hex_faces(N, A, Xb, sv);
    long long c = cidx(s, p, i, j, k);
    double V = vol_from_s(sv);
    double rho = ddiv(mass_cur(s, p, cur)[c], V), pr, pf, cs;
    eos(p.gamma, rho, s.e[cur][c], pr, pf, cs);
    double q = hex_q(Xb, U, rho, cs, p.c1, p.c2);
    s.sig[c] = 0.25 * (pf + q);
}

// S5-S6: nodal force and mass by gather (fixed order), kinematics, BC, move
template <bool EULER>
__global__ void k0_nodes(Slab s, Phys p, int cur, int kb0, int kb1)
{
    if (!s.st->active) return;
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= s.pn * (kb1 - kb0 + 1)) return;
    int k = kb0 + (int)(t / s.pn);
    long long r = t % s.pn;
    int j = (int)(r / (p.nx + 1)), i = (int)(r % (p.nx + 1));
    const double* m = mass_cur(s, p, cur);
    D3 F = d3(0.0, 0.0, 0.0);
    double M = 0.0;
    bool first = true;
    for (int g = 0; g < 8; ++g) {
        int ap = g & 1, bp = (g >> 1) & 1, cp = g >> 2;
        int ci = i - 1 + ap, cj = j - 1 + bp, ck = k - 1 + cp;
        if (!cell_in(p, ci, cj, ck)) continue;
        D3 N[8], A[6], Xb[6];
        double sv[6];
        load_hex_pos<EULER>(s, p, cur, ci, cj, ck, N);
        hex_faces(N, A, Xb, sv);
        D3 C = corner_vec(A, 1 - ap, 1 - bp, 1 - cp);
        long long c = cidx(s, p, ci, cj, ck);
        D3 term = scl(s.sig[c], C);
        if (first) {
            F = term;
            M = m[c];
            first = false;
        } else {
            F = add(F, term);
            M = M + m[c];
        }
    }
    M = 0.125 * M;
    double dt = s.st->dt;
    long long n = nidx(s, p, i, j, k);
    D3 u = ld3(s.u[cur], n);
    D3 un = d3(u.x + (ddiv(F.x, M) * dt), u.y + (ddiv(F.y, M) * dt), u.z + (ddiv(F.z, M) * dt));
    un = reflect(p, i, j, k, un);
    D3 x = pos<EULER>(s, p, cur, i, j, k);
    D3 xn = d3(x.x + (un.x * dt), x.y + (un.y * dt), x.z + (un.z * dt));
    if (EULER) {
        st3(s.x1, n, xn);
        st3(s.u1, n, un);
    } else {
        st3(s.x[cur ^ 1], n, xn);
        st3(s.u[cur ^ 1], n, un);
    }
}

// S7: V' + tangle check, compatible pdV energy; Lagrange: next dt candidate
template <bool EULER>
__global__ void k0_energy(Slab s, Phys p, int cur, int kc0, int kc1)
{
    if (!s.st->active) return;
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long key = KEY_NONE;
    if (t < s.pc * (kc1 - kc0)) {
        int k = kc0 + (int)(t / s.pc);
        long long r = t % s.pc;
        int j = (int)(r / p.nx), i = (int)(r % p.nx);
        bool owned = k >= s.k0 && k < s.k1;
        D3 N0[8], N1[8], U0[8], U1[8], A[6], Xb[6];
        double sv[6];
        load_hex_pos<EULER>(s, p, cur, i, j, k, N0);
        load_hex3(s, p, s.u[cur], i, j, k, U0);
        if (EULER) {
            load_hex3(s, p, s.x1, i, j, k, N1);
            load_hex3(s, p, s.u1, i, j, k, U1);
        } else {
            load_hex3(s, p, s.x[cur ^ 1], i, j, k, N1);
            load_hex3(s, p, s.u[cur ^ 1], i, j, k, U1);
        }
        double V1 = hex_volume(N1);
        if (owned && !(V1 > 0.0))
            atomicMin(&s.st->err_key, (ERR_ORDER_TANGLED << 48) | (unsigned long long)gcell(p, i, j, k));
        hex_faces(N0, A, Xb, sv);
        double W = 0.0;
#pragma unroll
        for (int h = 0; h < 8; ++h) {
            D3 C = corner_vec(A, h & 1, (h >> 1) & 1, h >> 2);
            D3 ub = scl(0.5, add(U0[h], U1[h]));
            double term = dot(C, ub);
            W = (h == 0) ? term : W + term;
        }
        long long c = cidx(s, p, i, j, k);
        double m = mass_cur(s, p, cur)[c];
        double e1 = s.e[cur][c] - ddiv((s.sig[c] * W) * s.st->dt, m);
        if (EULER) {
            s.e1[c] = e1;
            s.V1[c] = V1;
        } else {
            s.e[cur ^ 1][c] = e1;
            if (owned) {
                double rho = ddiv(m, V1), pr, pf, cs;
                eos(p.gamma, rho, e1, pr, pf, cs);
                key = dt_key(dt_cell(p.cfl, hex_min_edge2(N1), hex_max_speed2(U1), cs));
            }
        }
    }
    if (!EULER) block_min_atomic(key, &s.st->cand_key);
}

// R1-R2 for the interior face on the +ax side of lower cell (li,lj,lk)
__device__ __forceinline__ void face_flux(const Slab& s, const Phys& p, int cur, int ax, int li,
                                          int lj, int lk, double& mu, double& eps, D3& pi)
{
    int I[4], J[4], K[4];
    if (ax == 0) {
        int X = li + 1;
        I[0] = X; J[0] = lj;     K[0] = lk;
        I[1] = X; J[1] = lj + 1; K[1] = lk;
        I[2] = X; J[2] = lj + 1; K[2] = lk + 1;
        I[3] = X; J[3] = lj;     K[3] = lk + 1;
    } else if (ax == 1) {
        int Y = lj + 1;
        I[0] = li;     J[0] = Y; K[0] = lk;
        I[1] = li;     J[1] = Y; K[1] = lk + 1;
        I[2] = li + 1; J[2] = Y; K[2] = lk + 1;
        I[3] = li + 1; J[3] = Y; K[3] = lk;
    } else {
        int Z = lk + 1;
        I[0] = li;     J[0] = lj;     K[0] = Z;
        I[1] = li + 1; J[1] = lj;     K[1] = Z;
        I[2] = li + 1; J[2] = lj + 1; K[2] = Z;
        I[3] = li;     J[3] = lj + 1; K[3] = Z;
    }
    D3 T[4], L[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        T[v] = tpos(s, I[v], J[v], K[v]);
        L[v] = ld3(s.x1, nidx(s, p, I[v], J[v], K[v]));
    }
    double dV = swept_volume(T[0], T[1], T[2], T[3], L[0], L[1], L[2], L[3]);
    int di = li, dj = lj, dk = lk;
    if (!(dV > 0.0)) {
        if (ax == 0) di = li + 1;
        else if (ax == 1) dj = lj + 1;
        else dk = lk + 1;
    }
    D3 U[8];
    load_hex3(s, p, s.u1, di, dj, dk, U);
    D3 sum = U[0];
#pragma unroll
    for (int h = 1; h < 8; ++h) sum = add(sum, U[h]);
    D3 Ub = scl(0.125, sum);
    long long D = cidx(s, p, di, dj, dk);
    mu = ddiv(s.m[cur][D], s.V1[D]) * dV;
    eps = mu * s.e1[D];
    pi = scl(mu, Ub);
}

// R3: per cell Delta m / E / P, m'', e''
__global__ void k0_remap_cells(Slab s, Phys p, int cur, int kr0, int kr1)
{
    if (!s.st->active) return;
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= s.pc * (kr1 - kr0)) return;
    int k = kr0 + (int)(t / s.pc);
    long long r = t % s.pc;
    int j = (int)(r / p.nx), i = (int)(r % p.nx);
    int ijk[3] = {i, j, k};
    int nmax[3] = {p.nx, p.ny, p.nz};
    double mu[6], ep[6];
    D3 pi[6];
    for (int ax = 0; ax < 3; ++ax) {
        if (ijk[ax] > 0) {
            int l[3] = {i, j, k};
            l[ax] -= 1;
            face_flux(s, p, cur, ax, l[0], l[1], l[2], mu[2 * ax], ep[2 * ax], pi[2 * ax]);
        } else {
            mu[2 * ax] = 0.0;
            ep[2 * ax] = 0.0;
            pi[2 * ax] = d3(0.0, 0.0, 0.0);
        }
        if (ijk[ax] < nmax[ax] - 1) {
            face_flux(s, p, cur, ax, i, j, k, mu[2 * ax + 1], ep[2 * ax + 1], pi[2 * ax + 1]);
        } else {
            mu[2 * ax + 1] = 0.0;
            ep[2 * ax + 1] = 0.0;
            pi[2 * ax + 1] = d3(0.0, 0.0, 0.0);
        }
    }
    double dm = ((((mu[0] - mu[1]) + mu[2]) - mu[3]) + mu[4]) - mu[5];
    double dE = ((((ep[0] - ep[1]) + ep[2]) - ep[3]) + ep[4]) - ep[5];
    D3 dP = sub(add(sub(add(sub(pi[0], pi[1]), pi[2]), pi[3]), pi[4]), pi[5]);
    long long c = cidx(s, p, i, j, k);
    double m2 = s.m[cur][c] + dm;
    if (k >= s.k0 && k < s.k1 && !(m2 > 0.0))
        atomicMin(&s.st->err_key, (ERR_ORDER_NEGMASS << 48) | (unsigned long long)gcell(p, i, j, k));
    double e1 = s.e1[c];
    s.e[cur ^ 1][c] = e1 + ddiv(dE - (e1 * dm), m2);
    s.m[cur ^ 1][c] = m2;
    s.dm[c] = dm;
    st3(s.dP, c, dP);
}

// R4-R5: node momentum update from gathered Delta m, Delta P, m''; BC
__global__ void k0_remap_nodes(Slab s, Phys p, int cur)
{
    if (!s.st->active) return;
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= s.pn * (s.k1 - s.k0 + 1)) return;
    int k = s.k0 + (int)(t / s.pn);
    long long r = t % s.pn;
    int j = (int)(r / (p.nx + 1)), i = (int)(r % (p.nx + 1));
    double Dm = 0.0, M2 = 0.0;
    D3 DP = d3(0.0, 0.0, 0.0);
    bool first = true;
    for (int g = 0; g < 8; ++g) {
        int ci = i - 1 + (g & 1), cj = j - 1 + ((g >> 1) & 1), ck = k - 1 + (g >> 2);
        if (!cell_in(p, ci, cj, ck)) continue;
        long long c = cidx(s, p, ci, cj, ck);
        D3 dp = ld3(s.dP, c);
        if (first) {
            Dm = s.dm[c];
            DP = dp;
            M2 = s.m[cur ^ 1][c];
            first = false;
        } else {
            Dm = Dm + s.dm[c];
            DP = add(DP, dp);
            M2 = M2 + s.m[cur ^ 1][c];
        }
    }
    Dm = 0.125 * Dm;
    DP = scl(0.125, DP);
    M2 = 0.125 * M2;
    long long n = nidx(s, p, i, j, k);
    D3 u1 = ld3(s.u1, n);
    D3 un = d3(u1.x + ddiv(DP.x - (u1.x * Dm), M2), u1.y + ddiv(DP.y - (u1.y * Dm), M2),
               u1.z + ddiv(DP.z - (u1.z * Dm), M2));
    st3(s.u[cur ^ 1], n, reflect(p, i, j, k, un));
}

int launch_dt_candidate_gated(const Slab& s, const Phys& p, int cur, Stream st);


int launch_lagrange_v0(const Slab& s, const Phys& p, int cur, Stream st)
{
    cudaStream_t cs = (cudaStream_t)st;
    const int bs = 128;
    if (!p.rezone) {
        int ka0 = s.k0 > 0 ? s.k0 - 1 : 0, ka1 = s.k1 < p.nz ? s.k1 + 1 : p.nz;
        k0_sigma<false><<<grid_for(s.pc * (ka1 - ka0), bs), bs, 0, cs>>>(s, p, cur, ka0, ka1);
        k0_nodes<false><<<grid_for(s.pn * (s.k1 - s.k0 + 1), bs), bs, 0, cs>>>(s, p, cur, s.k0, s.k1);
        k0_energy<false><<<grid_for(s.pc * (s.k1 - s.k0), bs), bs, 0, cs>>>(s, p, cur, s.k0, s.k1);
        return 3;
    }
    // Euler: the Lagrangian phase also runs on the ghost region the remap needs
    int ka0 = s.k0 - 3 > 0 ? s.k0 - 3 : 0, ka1 = s.k1 + 3 < p.nz ? s.k1 + 3 : p.nz;
    int kb0 = s.k0 - 2 > 0 ? s.k0 - 2 : 0, kb1 = s.k1 + 2 < p.nz ? s.k1 + 2 : p.nz;
    k0_sigma<true><<<grid_for(s.pc * (ka1 - ka0), bs), bs, 0, cs>>>(s, p, cur, ka0, ka1);
    k0_nodes<true><<<grid_for(s.pn * (kb1 - kb0 + 1), bs), bs, 0, cs>>>(s, p, cur, kb0, kb1);
    k0_energy<true><<<grid_for(s.pc * (kb1 - kb0), bs), bs, 0, cs>>>(s, p, cur, kb0, kb1);
    return 3;
}

int launch_remap_v0(const Slab& s, const Phys& p, int cur, Stream st)
{
    cudaStream_t cs = (cudaStream_t)st;
    const int bs = 128;
    int kr0 = s.k0 - 1 > 0 ? s.k0 - 1 : 0, kr1 = s.k1 + 1 < p.nz ? s.k1 + 1 : p.nz;
    k0_remap_cells<<<grid_for(s.pc * (kr1 - kr0), bs), bs, 0, cs>>>(s, p, cur, kr0, kr1);
    k0_remap_nodes<<<grid_for(s.pn * (s.k1 - s.k0 + 1), bs), bs, 0, cs>>>(s, p, cur);
    return 2 + launch_dt_candidate_gated(s, p, cur ^ 1, st);
}

}  // namespace sale
