// kernels_mat.cu -- multi-material cells (readings MM0-MM7 in
// DESIGN.md §10d; the paper's multi-material ScalSALE, with the
// closure of SPEC S:255-263).  The cell carries f_k, m_k, e_k of up to MAX_MAT materials
// (material-major arrays, Slab::mf/mm/me); the EoS is the mixed closure (mix_eos_*,
// sale_mesh.cuh), each material does its share of the cell's pdV work, and the remap
// moves each material's mass, volume and energy from the donor cell.
//
// The cycle runs on the z-march kernels with a material axis (kernels_fused.cu
// kf_force / kf_energy / kf_sigma_e / kf_energy_e and kernels_remap.cu kr_sweep, each
// with NM materials as a template parameter) and the single-material node kernels
// (kn_force_e, kn_update: they read sigma and the cell totals only).  This file holds
// the launch sequences, the per-material flux + cell update (k_mat_flux), init / mass
// re-summing, and the one-thread-per-cell Euler kernels k_mat_sigma / k_mat_energy /
// k_mat_sweep (SALE_MAT_V0=1: the first cut of the path, kept as a cross-check).
#include <cuda_runtime.h>

#include <cstdlib>

#include "sale_mesh.cuh"

namespace sale {

static inline unsigned grid_for(long long n, int bs)
{
    long long g = (n + bs - 1) / bs;
    return (unsigned)(g > 0 ? g : 1);
}

// SALE_MAT_V0=1: the Euler material path on its one-thread-per-cell kernels
// (k_mat_sigma, k_mat_energy, k_mat_sweep) instead of the z-march kernels with the
// material axis (kf_sigma_e, kf_energy_e, kr_sweep) -- a cross-check, same bits
static bool mat_v0()
{
    static const int v = [] {
        const char* e = getenv("SALE_MAT_V0");
        return e ? atoi(e) : 0;
    }();
    return v == 1;
}

// call f(std::integral_constant<int, nmat>) -- the kernels are instantiated per
// material count so the material loops unroll into registers
template <int N>
struct IC {
    static constexpr int value = N;
};
template <class F>
static void by_nmat(int nmat, F&& f)
{
    switch (nmat) {
    case 1: f(IC<1>{}); break;
    case 2: f(IC<2>{}); break;
    case 3: f(IC<3>{}); break;
    default: f(IC<4>{}); break;
    }
}


// MM1-MM3: geometry at t^n, mixed EoS, q from the cell density and mixed sound speed;
// sigma = 0.25 (P + q); q is kept for the materials' stresses (MM4).  Euler: launched
// before the cycle's k_begin (gate = 0 for the first cycle of a sale_step call, when
// DevState.active is still 0), it also forms the c.5 dt candidate of the owned cells
// from the same mixed sound speed (the fixed target mesh's edges: as k_dt_candidate)
template <bool EULER, int NM>
__global__ void k_mat_sigma(Slab s, Phys p, int cur, int ka0, int ka1, int gate)
{
    if (gate && !s.st->active) return;
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long key = KEY_NONE;
    if (t < s.pc * (ka1 - ka0)) {
        int k = ka0 + (int)(t / s.pc);
        long long r = t % s.pc;
        int j = (int)(r / p.nx), i = (int)(r % p.nx);
        D3 N[8], U[8], A[6], Xb[6];
        double sv[6], pf[MAX_MAT];
        load_hex_pos<EULER>(s, p, cur, i, j, k, N);
        load_hex3(s, p, s.u[cur], i, j, k, U);
        hex_faces(N, A, Xb, sv);
        long long c = cidx(s, p, i, j, k);
        double V = vol_from_s(sv);
        double rho = ddiv(mass_cur(s, p, cur)[c], V), pr, P, cs;
        mix_eos_t<NM>(s, mat_f(s, p, cur), mat_m(s, p, cur), s.me[cur], c, mat_stride(s), V, rho, pr, P, cs, pf);
        double q = hex_q(Xb, U, rho, cs, p.c1, p.c2);
        s.sig[c] = 0.25 * (P + q);
#pragma unroll
        for (int a = 0; a < NM; ++a) s.sgm[c + a * mat_stride(s)] = 0.25 * (pf[a] + q);
        if (EULER && k >= s.k0 && k < s.k1) {
            const double lx = len2(D3{s.Xt[i], 0.0, 0.0}, D3{s.Xt[i + 1], 0.0, 0.0});
            const double ly = len2(D3{0.0, s.Yt[j], 0.0}, D3{0.0, s.Yt[j + 1], 0.0});
            const double lz = len2(D3{0.0, 0.0, s.Zt[k - s.kb]}, D3{0.0, 0.0, s.Zt[k + 1 - s.kb]});
            key = dt_key(dt_cell(p.cfl, dmin(dmin(lx, ly), lz), hex_max_speed2(U), cs));
        }
    }
    if (EULER) block_min_atomic(key, &s.st->cand_key);
}

// MM4: V' + tangle check; each present material's e'_k from its stress
// sigma_k = 0.25 (pf_k + q) on its share f_k of the cell's work W (c.3 step 7);
// Lagrange: the next dt candidate from the mixed EoS of the new state
template <bool EULER, int NM>
__global__ void k_mat_energy(Slab s, Phys p, int cur, int kc0, int kc1)
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
        double sv[6], pf[MAX_MAT];
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
        const long long c = cidx(s, p, i, j, k), st = mat_stride(s);
        const double m = mass_cur(s, p, cur)[c];
        const double* f = mat_f(s, p, cur);
        const double* mk = mat_m(s, p, cur);
        const double dt = s.st->dt;
        double* e1 = EULER ? s.e1m : s.me[cur ^ 1];
#pragma unroll
    for (int a = 0; a < NM; ++a) {
            const long long ca = c + a * st;
            const double fa = f[ca], ma = mk[ca], ea = s.me[cur][ca];
            if (fa > 0.0 && ma > 0.0) {
                const double sa = s.sgm[ca];  // 0.25 (pf_k + q), from the sigma pass
                e1[ca] = ea - ddiv(((sa * W) * dt) * fa, ma);
            } else {
                e1[ca] = ea;
            }
        }
        if (EULER) {
            s.V1[c] = V1;
        } else if (owned) {
            double pr, P, cs;
            mix_eos_t<NM>(s, f, mk, s.me[cur ^ 1], c, st, V1, ddiv(m, V1), pr, P, cs, pf);
            key = dt_key(dt_cell(p.cfl, hex_min_edge2(N1), hex_max_speed2(U1), cs));
        }
    }
    if (!EULER) block_min_atomic(key, &s.st->cand_key);
}

// c.4 steps 1-2, per cell c: the swept volumes of its -x / -y / -z faces (interior
// faces only; stored at the upper cell, as kr_sweep does), and the cell's donor data:
// mean node velocity Ub = 0.125 * sum of u' and, per material, m_k / V' (MM5)
template <int NM>
__global__ void k_mat_sweep(Slab s, Phys p, int cur, int ks0, int ks1)
{
    if (!s.st->active) return;
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= s.pc * (ks1 - ks0)) return;
    const int k = ks0 + (int)(t / s.pc);
    const long long r = t % s.pc;
    const int j = (int)(r / p.nx), i = (int)(r % p.nx);
    const long long c = cidx(s, p, i, j, k);
    D3 U[8];
    load_hex3(s, p, s.u1, i, j, k, U);
    D3 sum = U[0];
#pragma unroll
    for (int h = 1; h < 8; ++h) sum = add(sum, U[h]);
    st3(s.UD, c, scl(0.125, sum));
    const double V1 = s.V1[c];
    const long long st = mat_stride(s);
    for (int a = 0; a < NM; ++a) s.rDm[c + a * st] = ddiv(s.mm[cur][c + a * st], V1);
    // faces at node planes i / j / k, their lower cell at -1 on that axis; canonical
    // P0..P3 as c.4 step 1 / face_node_ids
    const int lo[3] = {i, j, k};
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        if (lo[ax] < 1) continue;
        int I[4], J[4], K[4];
        if (ax == 0) {
            I[0] = i; J[0] = j;     K[0] = k;
            I[1] = i; J[1] = j + 1; K[1] = k;
            I[2] = i; J[2] = j + 1; K[2] = k + 1;
            I[3] = i; J[3] = j;     K[3] = k + 1;
        } else if (ax == 1) {
            I[0] = i;     J[0] = j; K[0] = k;
            I[1] = i;     J[1] = j; K[1] = k + 1;
            I[2] = i + 1; J[2] = j; K[2] = k + 1;
            I[3] = i + 1; J[3] = j; K[3] = k;
        } else {
            I[0] = i;     J[0] = j;     K[0] = k;
            I[1] = i + 1; J[1] = j;     K[1] = k;
            I[2] = i + 1; J[2] = j + 1; K[2] = k;
            I[3] = i;     J[3] = j + 1; K[3] = k;
        }
        D3 T[4], L[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            T[v] = tpos(s, I[v], J[v], K[v]);
            L[v] = ld3(s.x1, nidx(s, p, I[v], J[v], K[v]));
        }
        s.dV[ax][c] = swept_volume(T[0], T[1], T[2], T[3], L[0], L[1], L[2], L[3]);
    }
}

// six-face sum in c.4 step 3's order, built face by face:
// ((((v0 - v1) + v2) - v3) + v4) - v5
__device__ __forceinline__ double acc6(int f, double acc, double v)
{
    return f == 0 ? v : ((f & 1) ? acc - v : acc + v);
}

// MM5-MM6: per cell, the materials' fluxes through its six faces (boundary faces carry
// +0.0), m''_k, V''_k, e''_k, f''_k, the totals Delta m, Delta P, m'' for the node update
template <int NM>
__global__ void k_mat_flux(Slab s, Phys p, int cur, int kr0, int kr1)
{
    if (!s.st->active) return;
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= s.pc * (kr1 - kr0)) return;
    const int k = kr0 + (int)(t / s.pc);
    const long long r = t % s.pc;
    const int j = (int)(r / p.nx), i = (int)(r % p.nx);
    const int ijk[3] = {i, j, k};
    const int nmax[3] = {p.nx, p.ny, p.nz};
    const long long c = cidx(s, p, i, j, k), sa[3] = {1, p.nx, s.pc};
    const long long st = mat_stride(s);
    double dmk[MAX_MAT] = {0.0}, dEk[MAX_MAT] = {0.0}, dphk[MAX_MAT] = {0.0};
    double dm = 0.0;
    D3 dP = d3(0.0, 0.0, 0.0);
    // the six swept volumes first (independent loads), then every face's donor loads
    double dVf[6];
    long long Df[6];
    bool inf[6];
#pragma unroll
    for (int f = 0; f < 6; ++f) {
        const int ax = f >> 1;
        const bool plus = f & 1;
        inf[f] = plus ? ijk[ax] < nmax[ax] - 1 : ijk[ax] > 0;
        const long long nbr = inf[f] ? (plus ? c + sa[ax] : c - sa[ax]) : c;
        dVf[f] = inf[f] ? s.dV[ax][plus ? nbr : c] : 0.0;  // the face is the -ax face of the upper cell
        Df[f] = (dVf[f] > 0.0) == plus ? c : nbr;          // donor: the lower cell if the face moved toward +ax
    }
#pragma unroll
    for (int f = 0; f < 6; ++f) {
        const bool inner = inf[f];
        const double dV = dVf[f];
        const long long D = Df[f];
        double mu = 0.0;
        D3 pi = d3(0.0, 0.0, 0.0);
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            double mua = 0.0, pha = 0.0, epa = 0.0;
            if (inner) {
                const long long Da = D + a * st;
                mua = s.rDm[Da] * dV;
                pha = s.mf[cur][Da] * dV;
                epa = mua * s.e1m[Da];
                mu = (a == 0) ? mua : mu + mua;
            }
            dmk[a] = acc6(f, dmk[a], mua);
            dEk[a] = acc6(f, dEk[a], epa);
            dphk[a] = acc6(f, dphk[a], pha);
        }
        if (inner) pi = scl(mu, ld3(s.UD, D));
        dm = acc6(f, dm, mu);
        dP = d3(acc6(f, dP.x, pi.x), acc6(f, dP.y, pi.y), acc6(f, dP.z, pi.z));
    }
    double m2 = 0.0, VV = 0.0, vm2[MAX_MAT];
    bool bad = false;
#pragma unroll
    for (int a = 0; a < NM; ++a) {
        const long long ca = c + a * st;
        const double mm2 = s.mm[cur][ca] + dmk[a];
        vm2[a] = (s.mf[cur][ca] * s.V1[c]) + dphk[a];
        if (mm2 < 0.0 || vm2[a] < 0.0) bad = true;
        m2 = (a == 0) ? mm2 : m2 + mm2;
        VV = (a == 0) ? vm2[a] : VV + vm2[a];
    }
    if (k >= s.k0 && k < s.k1 && (bad || !(m2 > 0.0) || !(VV > 0.0)))
        atomicMin(&s.st->err_key, (ERR_ORDER_NEGMASS << 48) | (unsigned long long)gcell(p, i, j, k));
#pragma unroll
    for (int a = 0; a < NM; ++a) {
        const long long ca = c + a * st;
        const double mm2 = s.mm[cur][ca] + dmk[a];
        const double e1 = s.e1m[ca];
        s.me[cur ^ 1][ca] = (mm2 > 0.0) ? e1 + ddiv(dEk[a] - (e1 * dmk[a]), mm2) : 0.0;
        s.mf[cur ^ 1][ca] = ddiv(vm2[a], VV);
        s.mm[cur ^ 1][ca] = mm2;
    }
    s.m[cur ^ 1][c] = m2;
    s.dm[c] = dm;
    st3(s.dP, c, dP);
}

// MM7: the Sedov cell is material 0; the others are absent.  Every local cell plane
// (ghost planes outside the mesh: all zero).
__global__ void k_mat_init(Slab s, Phys p)
{
    long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= mat_stride(s)) return;
    const int k = s.kb + (int)(c / s.pc);
    const bool in = k >= 0 && k < p.nz;
    const long long st = mat_stride(s);
    for (int a = 0; a < s.nmat; ++a) {
        const long long ca = c + a * st;
        s.mf[0][ca] = (in && a == 0) ? 1.0 : 0.0;
        s.mm[0][ca] = (in && a == 0) ? s.m[0][c] : 0.0;
        s.me[0][ca] = (in && a == 0) ? s.e[0][c] : 0.0;
    }
}

// the cell mass is the sum of the material masses (after set_field of MAT_M)
__global__ void k_mat_total(Slab s, Phys p, int cur)
{
    long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= mat_stride(s)) return;
    const double* mk = mat_m(s, p, cur);
    const long long st = mat_stride(s);
    double m = 0.0;
    for (int a = 0; a < s.nmat; ++a) m = (a == 0) ? mk[c] : m + mk[c + a * st];
    (p.rezone ? s.m[cur] : s.m[0])[c] = m;
}

// Lagrange: the v0 schedule on the material kernels.  Euler: sigma and the dt
// candidate ran before k_begin (launch_mat_pre); the node gather is the fused
// kn_force_e (it reads sigma and the cell totals only).
int launch_lagrange_mat(const Slab& s, const Phys& p, int cur, Stream st)
{
    cudaStream_t cs = (cudaStream_t)st;
    const int bs = 128;
    if (!p.rezone) {
        // the fused z-march kernels with the material axis (kernels_fused.cu)
        return launch_force_mat(s, p, cur, st);
    }
    int kb0 = s.k0 - 2 > 0 ? s.k0 - 2 : 0, kb1 = s.k1 + 2 < p.nz ? s.k1 + 2 : p.nz;
    launch_kn_force_e(s, p, cur, st);
    if (!mat_v0()) return 1 + launch_energy_e_mat(s, p, cur, st);
    by_nmat(s.nmat, [&](auto nm) {
        constexpr int NM = decltype(nm)::value;
        k_mat_energy<true, NM><<<grid_for(s.pc * (kb1 - kb0), bs), bs, 0, cs>>>(s, p, cur, kb0, kb1);
    });
    return 2;
}

// Euler: sigma of cell planes [k0-3, k1+3) (the node gather's reach) and the dt
// candidate of the owned cells, before the cycle's k_begin
int launch_mat_pre(const Slab& s, const Phys& p, int cur, int gate, Stream st)
{
    if (!mat_v0()) return launch_sigma_e_mat(s, p, cur, gate, st);
    int ka0 = s.k0 - 3 > 0 ? s.k0 - 3 : 0, ka1 = s.k1 + 3 < p.nz ? s.k1 + 3 : p.nz;
    by_nmat(s.nmat, [&](auto nm) {
        constexpr int NM = decltype(nm)::value;
        k_mat_sigma<true, NM><<<grid_for(s.pc * (ka1 - ka0), 128), 128, 0, (cudaStream_t)st>>>(s, p, cur, ka0, ka1,
                                                                                               gate);
    });
    return 1;
}

// R1-R4: swept volumes and donor data, the material fluxes and cell update, the fused
// node momentum update (kn_update) on the totals; no dt pass (the next cycle's
// k_mat_sigma forms the candidate)
int launch_remap_mat(const Slab& s, const Phys& p, int cur, Stream st)
{
    cudaStream_t cs = (cudaStream_t)st;
    const int bs = 128;
    int kr0 = s.k0 - 1 > 0 ? s.k0 - 1 : 0, kr1 = s.k1 + 1 < p.nz ? s.k1 + 1 : p.nz;
    int ks0 = kr0 - 1 > 0 ? kr0 - 1 : 0, ks1 = kr1 + 1 < p.nz ? kr1 + 1 : p.nz;
    const bool v0 = mat_v0();
    if (!v0) launch_sweep_mat(s, p, cur, st);
    by_nmat(s.nmat, [&](auto nm) {
        constexpr int NM = decltype(nm)::value;
        if (v0) k_mat_sweep<NM><<<grid_for(s.pc * (ks1 - ks0), bs), bs, 0, cs>>>(s, p, cur, ks0, ks1);
        k_mat_flux<NM><<<grid_for(s.pc * (kr1 - kr0), bs), bs, 0, cs>>>(s, p, cur, kr0, kr1);
    });
    launch_kn_update(s, p, cur, st);
    return 3;
}

int launch_mat_init(const Slab& s, const Phys& p, Stream st)
{
    k_mat_init<<<grid_for(s.pc * s.nzc, 256), 256, 0, (cudaStream_t)st>>>(s, p);
    return 1;
}

int launch_mat_total(const Slab& s, const Phys& p, int cur, Stream st)
{
    k_mat_total<<<grid_for(s.pc * s.nzc, 256), 256, 0, (cudaStream_t)st>>>(s, p, cur);
    return 1;
}

}  // namespace sale
