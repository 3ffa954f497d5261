// kernels_mat.cu -- multi-material cells (readings MM0-MM7 in
// DESIGN.md §10d; the paper's multi-material ScalSALE, with the
// closure of SPEC S:255-263).  The cell carries f_k, m_k, e_k of up to MAX_MAT materials
// (material-major arrays, Slab::mf/mm/me); the EoS is the mixed closure (mix_eos_*,
// sale_mesh.cuh), each material does its share of the cell's pdV work, and the remap
// moves each material's mass, volume and energy from the donor cell.
//
// The cycle runs on the z-march kernels with a material axis (kernels_lag.cu
// kl_state / ke_state / kc_energy and kernels_remap.cu kr_sweep, each with NM
// materials as a template parameter) and the single-material kernels that read
// sigma and the cell totals only (kc_force, kn_update).  This file holds the remap
// sequence, the per-material flux + cell update (k_mat_flux) and init / mass
// re-summing.
#include <cuda_runtime.h>


#include "sale_mesh.cuh"

namespace sale {

static inline unsigned grid_for(long long n, int bs)
{
    long long g = (n + bs - 1) / bs;
    return (unsigned)(g > 0 ? g : 1);
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
    // the material state of the owned cells (the ghost cells' come from the exchange);
    // the cell total m'' of every cell (kn_update gathers the ghost cells' too)
    const bool own = k >= s.k0 && k < s.k1;
    const long long q = (long long)i + (long long)p.nx * j;
#pragma unroll
    for (int a = 0; a < NM; ++a) {
        if (!own) break;
        const long long ca = c + a * st;
        const double mm2 = s.mm[cur][ca] + dmk[a];
        const double e1 = s.e1m[ca];
        const double me2 = (mm2 > 0.0) ? e1 + ddiv(dEk[a] - (e1 * dmk[a]), mm2) : 0.0;
        const double mf2 = ddiv(vm2[a], VV);
        s.me[cur ^ 1][ca] = me2;
        s.mf[cur ^ 1][ca] = mf2;
        s.mm[cur ^ 1][ca] = mm2;
        if (s.hp) {  // peer-store halo: the neighbours' ghost cell planes
            halo_cell(s, s.hp->me, cur ^ 1, a, k, q, me2);
            halo_cell(s, s.hp->mf, cur ^ 1, a, k, q, mf2);
            halo_cell(s, s.hp->mm, cur ^ 1, a, k, q, mm2);
        }
    }
    s.m[cur ^ 1][c] = m2;
    // (an owned cell's m'' is also a neighbour's ghost cell: bit-identical to the value
    // the neighbour forms for it itself, so the two stores never disagree)
    if (s.hp && own) halo_cell(s, s.hp->m, cur ^ 1, 0, k, q, m2);
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

// R1-R4 with the material axis: the swept volumes and per-material donor data
// (kr_sweep with NM materials), the material fluxes and cell update (k_mat_flux),
// the node momentum update on the totals (kn_update)
int launch_remap_mat(const Slab& s, const Phys& p, int cur, Stream st, int nodes)
{
    cudaStream_t cs = (cudaStream_t)st;
    const int bs = 128;
    const int kr0 = s.k0 - 1 > 0 ? s.k0 - 1 : 0, kr1 = s.k1 + 1 < p.nz ? s.k1 + 1 : p.nz;
    launch_sweep(s, p, cur, st);
    by_nmat(s.nmat, [&](auto nm) {
        constexpr int NM = decltype(nm)::value;
        k_mat_flux<NM><<<grid_for(s.pc * (kr1 - kr0), bs), bs, 0, cs>>>(s, p, cur, kr0, kr1);
        note_launch();
    });
    if (!nodes) return 2;
    launch_kn_update(s, p, cur, st);
    return 3;
}

int launch_mat_init(const Slab& s, const Phys& p, Stream st)
{
    k_mat_init<<<grid_for(s.pc * s.nzc, 256), 256, 0, (cudaStream_t)st>>>(s, p);
    note_launch();
    return 1;
}

int launch_mat_total(const Slab& s, const Phys& p, int cur, Stream st)
{
    k_mat_total<<<grid_for(s.pc * s.nzc, 256), 256, 0, (cudaStream_t)st>>>(s, p, cur);
    note_launch();
    return 1;
}

}  // namespace sale
