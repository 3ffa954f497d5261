// kernels_common.cu -- initialisation, target-mesh tables, clock / dt
// finalisation, derived fields, the Steinberg cell kernel.  SURVEY §8(c) c.1, c.5,
// c.6; the dt candidates come with the cell-state passes (kernels_lag.cu).
#include <cuda_runtime.h>

#include "sale_mesh.cuh"

namespace sale {

static thread_local cudaError_t g_launch_err = cudaSuccess;
void note_launch()
{
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess && g_launch_err == cudaSuccess) g_launch_err = e;
}
int take_launch_error()
{
    const cudaError_t e = g_launch_err;
    g_launch_err = cudaSuccess;
    return (int)e;
}

static inline unsigned grid_for(long long n, int bs)
{
    long long g = (n + bs - 1) / bs;
    return (unsigned)(g > 0 ? g : 1);
}

// c.1: X_i = (lx*i)/nx etc.; Z over the slab's local node planes
__global__ void k_init_tables(Slab s, Phys p)
{
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t <= p.nx) s.Xt[t] = (p.lx * (double)t) / (double)p.nx;
    if (t <= p.ny) s.Yt[t] = (p.ly * (double)t) / (double)p.ny;
    if (t < s.nzn) s.Zt[t] = (p.lz * (double)(s.kb + t)) / (double)p.nz;
}

// c.6 Sedov: x = x^T, u = 0 on every local node plane inside the domain
__global__ void k_sedov_nodes(Slab s, Phys p)
{
    long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long total = s.pn * s.nzn;
    if (n >= total) return;
    int l = (int)(n / s.pn);
    int k = s.kb + l;
    if (k < 0 || k > p.nz) return;
    long long r = n % s.pn;
    int j = (int)(r / (p.nx + 1)), i = (int)(r % (p.nx + 1));
    if (!p.rezone) {
        s.x[0][0][n] = s.Xt[i];
        s.x[0][1][n] = s.Yt[j];
        s.x[0][2][n] = s.Zt[l];
    }
    s.u[0][0][n] = 0.0;
    s.u[0][1][n] = 0.0;
    s.u[0][2][n] = 0.0;
}

// c.6 Sedov: m = rho0 * V(x^T); e = e_bg; e_000 = E0 / m_000
__global__ void k_sedov_cells(Slab s, Phys p)
{
    long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long total = s.pc * s.nzc;
    if (c >= total) return;
    int k = s.kb + (int)(c / s.pc);
    if (k < 0 || k >= p.nz) return;
    long long r = c % s.pc;
    int j = (int)(r / p.nx), i = (int)(r % p.nx);
    D3 N[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) N[h] = tpos(s, i + (h & 1), j + ((h >> 1) & 1), k + (h >> 2));
    D3 A[6], Xb[6];
    double sv[6];
    hex_faces(N, A, Xb, sv);
    const double V = vol_from_s(sv);
    double m = p.rho0 * V;
    s.m[0][c] = m;
    if (p.rezone) {  // constants of the fixed Euler mesh: V^T and s of the -x/-y/-z target faces
        s.VT[c] = V;
        s.sT[0][c] = sv[0];
        s.sT[1][c] = sv[2];
        s.sT[2][c] = sv[4];
    }
    s.e[0][c] = (i == 0 && j == 0 && k == 0) ? p.e_dep / m : p.e_bg;
}

int launch_init_tables(const Slab& s, const Phys& p, Stream st)
{
    int n = p.nx > p.ny ? p.nx : p.ny;
    n = n > s.nzn ? n : s.nzn;
    k_init_tables<<<grid_for(n + 1, 256), 256, 0, (cudaStream_t)st>>>(s, p);
    note_launch();
    return 1;
}

int launch_sedov_init(const Slab& s, const Phys& p, Stream st)
{
    k_sedov_nodes<<<grid_for(s.pn * s.nzn, 256), 256, 0, (cudaStream_t)st>>>(s, p);
    note_launch();
    k_sedov_cells<<<grid_for(s.pc * s.nzc, 256), 256, 0, (cudaStream_t)st>>>(s, p);
    note_launch();
    return 2;
}

// Euler target-mesh tables (Slab::TAx..TJz): the c.2 face area vectors and the
// c.3 step 2 centroid separations of x^T, evaluated with the same primitives and
// canonical node orders as every per-cycle evaluation, at a representative index
// of the coordinates they do not depend on (x^T is a tensor product of X_i, Y_j,
// Z_k, and every difference of equal coordinates is exactly +0).
__global__ void k_target_tables(Slab s, Phys p)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int nx = p.nx, ny = p.ny, nzc = s.nzc, kb = s.kb;
    // x-faces (j, k): nodes (i,j,k) (i,j+1,k) (i,j+1,k+1) (i,j,k+1) at i = 0
    if (t < ny * nzc) {
        const int j = t % ny, k = kb + t / ny;
        const D3 A = face_area(tpos(s, 0, j, k), tpos(s, 0, j + 1, k), tpos(s, 0, j + 1, k + 1), tpos(s, 0, j, k + 1));
        s.TAx[0][t] = A.x;
        s.TAx[1][t] = A.y;
        s.TAx[2][t] = A.z;
    }
    // y-faces (i, k): nodes (i,j,k) (i,j,k+1) (i+1,j,k+1) (i+1,j,k) at j = 0
    if (t < nx * nzc) {
        const int i = t % nx, k = kb + t / nx;
        const D3 A = face_area(tpos(s, i, 0, k), tpos(s, i, 0, k + 1), tpos(s, i + 1, 0, k + 1), tpos(s, i + 1, 0, k));
        s.TAy[0][t] = A.x;
        s.TAy[1][t] = A.y;
        s.TAy[2][t] = A.z;
    }
    // z-faces (i, j): nodes (i,j,k) (i+1,j,k) (i+1,j+1,k) (i,j+1,k) at local plane 0
    if (t < nx * ny) {
        const int i = t % nx, j = t / nx;
        const D3 A = face_area(tpos(s, i, j, kb), tpos(s, i + 1, j, kb), tpos(s, i + 1, j + 1, kb), tpos(s, i, j + 1, kb));
        s.TAz[0][t] = A.x;
        s.TAz[1][t] = A.y;
        s.TAz[2][t] = A.z;
    }
    // axis-jump constants: d = Xbar(+a face) - Xbar(-a face), L = sqrt(d.d) (c.3 step 2)
    auto jump = [](D3 Xm, D3 Xp, double* out) {
        const D3 d = sub(Xp, Xm);
        out[0] = d.x;
        out[1] = d.y;
        out[2] = d.z;
        out[3] = dsqrt((d.x * d.x + d.y * d.y) + d.z * d.z);
    };
    // dt numerator factors (c.5 on the target mesh: the edges of a cell are axis-aligned)
    if (t < nx) s.TDx[t] = p.cfl * dsqrt(len2(D3{s.Xt[t], 0.0, 0.0}, D3{s.Xt[t + 1], 0.0, 0.0}));
    if (t < ny) s.TDy[t] = p.cfl * dsqrt(len2(D3{0.0, s.Yt[t], 0.0}, D3{0.0, s.Yt[t + 1], 0.0}));
    if (t < nzc) s.TDz[t] = p.cfl * dsqrt(len2(D3{0.0, 0.0, s.Zt[t]}, D3{0.0, 0.0, s.Zt[t + 1]}));
    const int k0 = kb;
    if (t < nx) {
        const int i = t;
        const D3 Xm = avg4(tpos(s, i, 0, k0), tpos(s, i, 1, k0), tpos(s, i, 1, k0 + 1), tpos(s, i, 0, k0 + 1));
        const D3 Xp = avg4(tpos(s, i + 1, 0, k0), tpos(s, i + 1, 1, k0), tpos(s, i + 1, 1, k0 + 1), tpos(s, i + 1, 0, k0 + 1));
        jump(Xm, Xp, s.TJx + 4 * i);
    }
    if (t < ny) {
        const int j = t;
        const D3 Xm = avg4(tpos(s, 0, j, k0), tpos(s, 0, j, k0 + 1), tpos(s, 1, j, k0 + 1), tpos(s, 1, j, k0));
        const D3 Xp = avg4(tpos(s, 0, j + 1, k0), tpos(s, 0, j + 1, k0 + 1), tpos(s, 1, j + 1, k0 + 1), tpos(s, 1, j + 1, k0));
        jump(Xm, Xp, s.TJy + 4 * j);
    }
    if (t < nzc) {
        const int k = kb + t;
        const D3 Xm = avg4(tpos(s, 0, 0, k), tpos(s, 1, 0, k), tpos(s, 1, 1, k), tpos(s, 0, 1, k));
        const D3 Xp = avg4(tpos(s, 0, 0, k + 1), tpos(s, 1, 0, k + 1), tpos(s, 1, 1, k + 1), tpos(s, 0, 1, k + 1));
        jump(Xm, Xp, s.TJz + 4 * t);
    }
}

int launch_target_tables(const Slab& s, const Phys& p, Stream st)
{
    long long n = (long long)p.ny * s.nzc;
    n = n > (long long)p.nx * s.nzc ? n : (long long)p.nx * s.nzc;
    n = n > (long long)p.nx * p.ny ? n : (long long)p.nx * p.ny;
    k_target_tables<<<grid_for(n, 256), 256, 0, (cudaStream_t)st>>>(s, p);
    note_launch();
    return 1;
}

// ---------------------------------------------------------------- clock
__global__ void k_prep(DevState* d)
{
    d->cand_key = KEY_NONE;
    d->err_key = KEY_NONE;
    d->active = 0;
}

__device__ __forceinline__ void commit(DevState* d)
{
    if (!d->active) return;
    d->active = 0;
    if (d->err_key != KEY_NONE) {
        unsigned long long order = d->err_key >> 48;
        d->status = (order == ERR_ORDER_TANGLED) ? S_ETANGLED : S_ENEGMASS;
        d->err_cycle = d->cycle;
        d->err_cell = (long long)(d->err_key & 0xFFFFFFFFFFFFull);
        return;
    }
    d->t = d->t + d->dt;
    d->cycle = d->cycle + 1;
    d->dt_prev = d->dt;
    d->good = d->good + 1;
}

// commit the cycle in flight, then c.5: finalise dt from the reduced candidate
__global__ void k_begin(DevState* d, Phys p)
{
    commit(d);
    if (d->status) return;
    if (p.t_end > 0.0 && d->t >= p.t_end) {
        d->finished = 1;
        return;
    }
    double dt_cfl = dt_unkey(d->cand_key);
    double dt_u = (d->dt_prev < 0.0) ? dt_cfl : dmin(dt_cfl, p.growth * d->dt_prev);
    // collapse: relative to t_end, without an end time to the time reached (DT-C)
    const double tref = (p.t_end > 0.0) ? p.t_end : d->t;
    if (!(dt_u > 0.0) || dt_u < 1e-14 * tref) {
        d->status = S_EDTCOLLAPSE;
        d->err_cycle = d->cycle;
        d->err_cell = -1;
        return;
    }
    d->dt = (p.t_end > 0.0) ? dmin(dt_u, p.t_end - d->t) : dt_u;
    d->cand_key = KEY_NONE;
    d->err_key = KEY_NONE;
    d->active = 1;
}

__global__ void k_commit(DevState* d, Phys p)
{
    commit(d);
    if (!d->status && p.t_end > 0.0 && d->t >= p.t_end) d->finished = 1;
}

__global__ void k_reset_good(DevState* d) { d->good = 0; }

// ---------------------------------------------------------------- peer-store halo
// (ranks).  After a cycle's producer kernels stored their planes into the
// neighbours' ghost planes: one increment of each neighbour's arrival counter at system
// scope (the producers are complete and their NVLink stores performed when this kernel
// runs: stream order).  Before the next cycle's state pass reads the ghost planes:
// wait until every neighbour's count reaches the cycles consumed + 1.  A cycle that is
// not in flight (finished / failed: the same on every rank, dt and the error key being
// all-reduced) neither signals nor waits.  The wait gives up after 60 s (a lost peer)
// with SALE_ENCCL instead of hanging the device.
__global__ void k_halo_signal(DevState* d, const HaloPeer* hp)
{
    if (!d->active) return;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
        unsigned long long* f = hp->flag[side];
        if (f) {
            __threadfence_system();
            atomicAdd_system(f, 1ull);
        }
    }
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* a)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long global_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_halo_wait(DevState* d, int first, int sides)
{
    if (first) {  // the copy exchange filled the ghost planes: absorb earlier arrivals
        d->halo_seen[0] = ld_acquire_sys(&d->halo_in[0]);
        d->halo_seen[1] = ld_acquire_sys(&d->halo_in[1]);
        return;
    }
    if (!d->active) return;
    const unsigned long long t0 = global_ns();
    for (int side = 0; side < 2; ++side) {
        if (!((sides >> side) & 1)) continue;  // no neighbour on this side
        const unsigned long long want = d->halo_seen[side] + 1;
        while (ld_acquire_sys(&d->halo_in[side]) < want) {
            if (global_ns() - t0 > 60000000000ull) {
                d->status = S_ENCCL;
                d->err_cycle = d->cycle;
                d->err_cell = -1;
                d->active = 0;
                return;
            }
            __nanosleep(200);
        }
        d->halo_seen[side] = want;
    }
}

int launch_prep(DevState* d, Stream st)
{
    k_prep<<<1, 1, 0, (cudaStream_t)st>>>(d);
    note_launch();
    return 1;
}
int launch_begin(DevState* d, const Phys& p, Stream st)
{
    k_begin<<<1, 1, 0, (cudaStream_t)st>>>(d, p);
    note_launch();
    return 1;
}
int launch_commit(DevState* d, const Phys& p, Stream st)
{
    k_commit<<<1, 1, 0, (cudaStream_t)st>>>(d, p);
    note_launch();
    return 1;
}
int launch_halo_signal(DevState* d, const HaloPeer* hp_dev, Stream st)
{
    k_halo_signal<<<1, 1, 0, (cudaStream_t)st>>>(d, hp_dev);
    note_launch();
    return 1;
}
int launch_halo_wait(DevState* d, int first, int sides, Stream st)
{
    k_halo_wait<<<1, 1, 0, (cudaStream_t)st>>>(d, first, sides);
    note_launch();
    return 1;
}
int launch_reset_good(DevState* d, Stream st)
{
    k_reset_good<<<1, 1, 0, (cudaStream_t)st>>>(d);
    note_launch();
    return 1;
}

// ------------------------------------------------------- derived fields
// Writes the owned slab of a derived field into s.der, compact (plane k-k0).
// field ids as in include/sale.h.
template <bool EULER>
__global__ void k_derive_cells(Slab s, Phys p, int cur, int field)
{
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long total = s.pc * (s.k1 - s.k0);
    if (t >= total) return;
    int k = s.k0 + (int)(t / s.pc);
    long long r = t % s.pc;
    int j = (int)(r / p.nx), i = (int)(r % p.nx);
    D3 N[8], A[6], Xb[6];
    double sv[6];
    load_hex_pos<EULER>(s, p, cur, i, j, k, N);
    hex_faces(N, A, Xb, sv);
    long long c = cidx(s, p, i, j, k);
    double V = vol_from_s(sv);
    double rho = ddiv(mass_cur(s, p, cur)[c], V), pr, pf, cs;
    if (s.nmat) {
        double pfk[MAX_MAT];
        mix_eos(s, mat_f(s, p, cur), mat_m(s, p, cur), s.me[cur], c, mat_stride(s), V, rho, pr, pf, cs, pfk);
    } else {
        eos(p.gamma, rho, s.e[cur][c], pr, pf, cs);
    }
    double v;
    switch (field) {
    case 8: {  // materials: the mixture's specific energy (sum_k m_k e_k) / m
        const double* mk = mat_m(s, p, cur);
        double sum = 0.0;
        for (int a = 0; a < s.nmat; ++a) {
            const double t = mk[c + a * mat_stride(s)] * s.me[cur][c + a * mat_stride(s)];
            sum = (a == 0) ? t : sum + t;
        }
        v = ddiv(sum, mass_cur(s, p, cur)[c]);
        break;
    }
    case 9: v = rho; break;
    case 10: v = V; break;
    case 11: v = pr; break;
    case 13: v = cs; break;
    default: {
        D3 U[8];
        load_hex3(s, p, s.u[cur], i, j, k, U);
        v = hex_q(Xb, U, rho, cs, p.c1, p.c2);
    }
    }
    s.der[t] = v;
}

// NODE_MASS (c.3 step 5) and, in Euler mode, X/Y/Z = x^T
__global__ void k_derive_nodes(Slab s, Phys p, int cur, int field)
{
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long total = s.pn * (s.k1 - s.k0 + 1);
    if (t >= total) return;
    int k = s.k0 + (int)(t / s.pn);
    long long r = t % s.pn;
    int j = (int)(r / (p.nx + 1)), i = (int)(r % (p.nx + 1));
    double v;
    if (field <= 2) {
        D3 X = tpos(s, i, j, k);
        v = field == 0 ? X.x : (field == 1 ? X.y : X.z);
    } else {
        const double* m = mass_cur(s, p, cur);
        double M = 0.0;
        bool first = true;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            int ci = i - 1 + (g & 1), cj = j - 1 + ((g >> 1) & 1), ck = k - 1 + (g >> 2);
            if (!cell_in(p, ci, cj, ck)) continue;
            double mk = m[cidx(s, p, ci, cj, ck)];
            M = first ? mk : M + mk;
            first = false;
        }
        v = 0.125 * M;
    }
    s.der[t] = v;
}

int launch_derive(const Slab& s, const Phys& p, int cur, int field, Stream st)
{
    if (field <= 6) {
        long long n = s.pn * (s.k1 - s.k0 + 1);
        k_derive_nodes<<<grid_for(n, 256), 256, 0, (cudaStream_t)st>>>(s, p, cur, field);
        note_launch();
    } else {
        long long n = s.pc * (s.k1 - s.k0);
        if (p.rezone)
            k_derive_cells<true><<<grid_for(n, 256), 256, 0, (cudaStream_t)st>>>(s, p, cur, field);
        else
            k_derive_cells<false><<<grid_for(n, 256), 256, 0, (cudaStream_t)st>>>(s, p, cur, field);
        note_launch();
    }
    return 1;
}

// ------------------------------------------------ Steinberg (Fig. 6b)
// One thread per owned cell: rho = m / V, p and e exactly as get_field's RHO / P / E,
// then the paper's shear / yield loop body (association as written there) once per
// material with that material's constants (Fig. 6b's "do m=1, nmats"; one set when
// the context has no material axis).  Material m's outputs at sh / y + m * mstride.
// the Steinberg formulas of owned cell t (local index c) with volume V
template <int NM>
__device__ __forceinline__ void steinberg_tail(const Slab& s, const Phys& p, int cur, const SteinbergSet& set,
                                               const double* eps, double* sh, double* y, long long mstride,
                                               long long t, long long c, double V, const double* hconst)
{
    const double m = mass_cur(s, p, cur)[c];
    double rho = ddiv(m, V), pr, pf, cs, e;
    if constexpr (NM > 0) {  // the mixed closure and the mixture's specific energy (as get_field P / E)
        double pfk[MAX_MAT];
        mix_eos_t<NM>(s, mat_f(s, p, cur), mat_m(s, p, cur), s.me[cur], c, mat_stride(s), V, rho, pr, pf, cs, pfk);
        const double* mk = mat_m(s, p, cur);
        double sum = 0.0;
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            const double tt = mk[c + a * mat_stride(s)] * s.me[cur][c + a * mat_stride(s)];
            sum = (a == 0) ? tt : sum + tt;
        }
        e = ddiv(sum, m);
    } else {
        e = s.e[cur][c];
        eos(p.gamma, rho, e, pr, pf, cs);
    }
    const double ep = eps ? eps[t] : 0.0;
#pragma unroll
    for (int a = 0; a < (NM > 0 ? NM : 1); ++a) {
        const SteinbergP& sp = set.m[a];
        const double eta = sp.rho0 / rho;
        const double T = e / sp.cv;
        // eta^(1/3): cbrt (within an ulp of the paper's pow(eta, 1/3), at a fraction of its cost)
        const double G = (sp.G0 + (sp.GP * pr) * cbrt(eta)) + sp.GT * (T - sp.T0);
        const double h = eps ? sp.Y0 * pow(1.0 + sp.beta * ep, sp.n) : hconst[a];
        sh[t + a * mstride] = G;
        y[t + a * mstride] = ((h < sp.Ymax) ? h : sp.Ymax) * (G / sp.G0);
    }
}
template <bool EULER, int NM>  // NM: materials (0: no material axis, one parameter set)
__device__ __forceinline__ void steinberg_cells(const Slab& s, const Phys& p, int cur, const SteinbergSet& set,
                                                const double* eps, double* sh, double* y, long long mstride)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long total = s.pc * (s.k1 - s.k0);
    // without a plastic strain field the hardening factor Y0 (1 + beta 0)^n is the same for
    // every cell: formed once per block (the same expression, the same bits) instead of one
    // pow per cell
    __shared__ double hconst[MAX_MAT];
    if (!eps) {
        if (threadIdx.x < (NM > 0 ? NM : 1)) {
            const SteinbergP& sp = set.m[threadIdx.x];
            hconst[threadIdx.x] = sp.Y0 * pow(1.0 + sp.beta * 0.0, sp.n);
        }
        __syncthreads();
    }
    if (t >= total) return;
    const int k = s.k0 + (int)(t / s.pc);
    const long long r = t % s.pc;
    const int j = (int)(r / p.nx), i = (int)(r % p.nx);
    const long long c = cidx(s, p, i, j, k);
    static_assert(EULER, "Lagrange runs k_steinberg_zl");
    const double V = s.VT[c];  // the fixed mesh's volume (same formula, evaluated at create)
    steinberg_tail<NM>(s, p, cur, set, eps, sh, y, mstride, t, c, V, hconst);
}

// Euler: V from the target tables (light)
template <int NM>
__global__ void __launch_bounds__(256) k_steinberg_e(Slab s, Phys p, int cur, SteinbergSet set, const double* eps,
                                                     double* sh, double* y, long long mstride)
{
    steinberg_cells<true, NM>(s, p, cur, set, eps, sh, y, mstride);
}
// Lagrange as a z-march (kl_state's face sharing): a 32 x 8 CTA stages node planes of
// x in shared memory and forms the s of the x- / y-face anchored at each column once per
// plane (the z-face carried in a register), so a cell's V = vol_from_s of its six faces
// costs three face evaluations instead of six, and its nodes are loaded once per column
// instead of eight times per cell.  The faces' node order and expressions are
// hex_faces' (c.2), so V is the same bits as the thread-per-cell kernel's.
template <int NM>
__global__ void __launch_bounds__(256) k_steinberg_zl(Slab s, Phys p, int cur, SteinbergSet set, const double* eps,
                                                      double* sh, double* y, long long mstride, int zchunk)
{
    constexpr int FWS = 32, NWS = 8, PLS = NWS * FWS, PADS = FWS + 1, TXS = FWS - 1, TYS = NWS - 1;
    constexpr int OSS = 6 * PLS;  // node slots: x (3) of 2 planes; then s of the x-face, y-face
    __shared__ double sm[OSS + 2 * PLS + 2 * PADS];
    __shared__ double hconst[MAX_MAT];
    if (!eps) {
        if (threadIdx.y == 0 && threadIdx.x < (NM > 0 ? NM : 1)) {
            const SteinbergP& sp = set.m[threadIdx.x];
            hconst[threadIdx.x] = sp.Y0 * pow(1.0 + sp.beta * 0.0, sp.n);
        }
    }
    const int ix = threadIdx.x, iy = threadIdx.y;
    double* me = sm + PADS + iy * FWS + ix;
    const int i = blockIdx.x * TXS + ix, j = blockIdx.y * TYS + iy;
    const int za = s.k0 + zchunk_base(zchunk);
    const int zb = za + zchunk - 1 < s.k1 - 1 ? za + zchunk - 1 : s.k1 - 1;
    const int in = i < p.nx ? i : p.nx, jn = j < p.ny ? j : p.ny;
    const long long nbc = (long long)in + (long long)(p.nx + 1) * (jn - (long long)(p.ny + 1) * s.kb);
    const bool out_cell = i < p.nx && j < p.ny && ix < TXS && iy < TYS;
    auto fetch = [&](int k) { return ld3(s.x[cur], nbc + (long long)k * s.pn); };  // node planes [za, zb+1] exist
    auto put = [&](int par, D3 v) {
        double* q = me + par * 3 * PLS;
        q[0] = v.x;
        q[PLS] = v.y;
        q[2 * PLS] = v.z;
    };
    auto X = [&](int par, int off) {
        const double* q = me + off + par * 3 * PLS;
        return D3{q[0], q[PLS], q[2 * PLS]};
    };
    auto zs_of = [&](int par) {  // s of the z-face at this column: (i,j) (i+1,j) (i+1,j+1) (i,j+1)
        const D3 T0 = X(par, 0), T1 = X(par, 1), T2 = X(par, FWS + 1), T3 = X(par, FWS);
        return face_s(avg4(T0, T1, T2, T3), face_area(T0, T1, T2, T3));
    };
    D3 px = fetch(za);
    put(za & 1, px);
    px = fetch(za + 1);
    __syncthreads();
    double zs = zs_of(za & 1);
    for (int kz = za; kz <= zb; ++kz) {
        const int b0 = kz & 1, b1 = b0 ^ 1;
        put(b1, px);  // node plane kz+1
        if (kz < zb) px = fetch(kz + 2);
        __syncthreads();
        const double zsn = zs_of(b1);
        {
            // x-face at node plane i: (i,j,kz) (i,j+1,kz) (i,j+1,kz+1) (i,j,kz+1)
            const D3 Q0 = X(b0, 0), Q1 = X(b0, FWS), Q2 = X(b1, FWS), Q3 = X(b1, 0);
            me[OSS] = face_s(avg4(Q0, Q1, Q2, Q3), face_area(Q0, Q1, Q2, Q3));
            // y-face at node plane j: (i,j,kz) (i,j,kz+1) (i+1,j,kz+1) (i+1,j,kz)
            const D3 R2 = X(b1, 1), R3 = X(b0, 1);
            me[OSS + PLS] = face_s(avg4(Q0, Q3, R2, R3), face_area(Q0, Q3, R2, R3));
        }
        __syncthreads();
        if (out_cell) {
            const double sv[6] = {me[OSS], me[1 + OSS], me[OSS + PLS], me[FWS + OSS + PLS], zs, zsn};
            const long long t = (long long)(kz - s.k0) * s.pc + (long long)j * p.nx + i;
            steinberg_tail<NM>(s, p, cur, set, eps, sh, y, mstride, t, cidx(s, p, i, j, kz), vol_from_s(sv), hconst);
        }
        zs = zsn;
        __syncthreads();
    }
}

int launch_steinberg(const Slab& s, const Phys& p, int cur, const SteinbergSet& set, const double* eps, double* sh,
                     double* y, long long mstride, Stream st)
{
    const long long n = s.pc * (s.k1 - s.k0);
    auto go = [&](auto kern) { kern<<<grid_for(n, 256), 256, 0, (cudaStream_t)st>>>(s, p, cur, set, eps, sh, y, mstride); note_launch(); };
    if (!p.rezone) {  // Lagrange: the z-march kernel
        const int planes = s.k1 - s.k0;
        const long long xy = (long long)((p.nx + 30) / 31) * ((p.ny + 6) / 7);
        const int zc = zchunk_for(xy, planes, 32);
        const dim3 grid((p.nx + 30) / 31, (p.ny + 6) / 7, (planes + zc - 1) / zc);
        auto gz = [&](auto kern) {
            kern<<<grid, dim3(32, 8), 0, (cudaStream_t)st>>>(s, p, cur, set, eps, sh, y, mstride, zorder(zc));
            note_launch();
        };
        switch (s.nmat) {
        case 0: gz(k_steinberg_zl<0>); break;
        case 1: gz(k_steinberg_zl<1>); break;
        case 2: gz(k_steinberg_zl<2>); break;
        case 3: gz(k_steinberg_zl<3>); break;
        default: gz(k_steinberg_zl<4>); break;
        }
        return 1;
    }
    switch (s.nmat) {  // Euler: one thread per cell (V from the target tables)
    case 0: go(k_steinberg_e<0>); break;
    case 1: go(k_steinberg_e<1>); break;
    case 2: go(k_steinberg_e<2>); break;
    case 3: go(k_steinberg_e<3>); break;
    default: go(k_steinberg_e<4>); break;
    }
    return 1;
}

}  // namespace sale
