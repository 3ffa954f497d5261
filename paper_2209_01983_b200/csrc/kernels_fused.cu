// kernels_fused.cu -- the fused Lagrangian phase as two z-marching kernels.
//
// Each CTA owns an x-y tile of columns and marches along z (2.5D): node planes
// are loaded once from HBM (coalesced, one warp per x-row of 32 columns),
// staged in shared memory, and every face quantity is computed ONCE per CTA and
// shared by the cells / nodes that use it:
//
//   kf_force  : S1 geometry at t^n (faces anchored at each column), S2 EoS,
//               S3 viscosity, sigma; S5 corner forces gathered in the fixed
//               order of c.2; S6 kinematics + reflecting BC.  Writes u', x'
//               (Lagrange) or u' (Euler), and sigma.
//   kf_energy : S7 geometry at t^{n+1} (V', tangle check), compatible pdV
//               energy, and (Lagrange) the next cycle's dt candidate with a
//               warp-shuffle + block min and one atomicMin per CTA (S4).
//
// The arithmetic of every quantity is the expression tree of SURVEY §8(c),
// evaluated with the same association as the v0 kernels and the oracle, so
// results are bit-identical; only where operands come from (registers / shared
// memory instead of recomputation) differs.  Tiles: 32 columns per warp row in
// x (one halo column each side), NW warp rows in y.
#include <cuda_runtime.h>

#include "sale_mesh.cuh"

namespace sale {

bool fused_available() { return true; }

namespace {

constexpr int FW = 32;  // columns per warp row
constexpr int MINB = 2; // resident CTAs per SM the register budget is sized for

// shared-memory 2D plane helper: [NW][32] doubles
template <int NW>
struct Plane {
    double* p;
    __device__ __forceinline__ double& at(int y, int x) const { return p[y * FW + x]; }
};

__device__ __forceinline__ int imin(int a, int b) { return a < b ? a : b; }
__device__ __forceinline__ int imax(int a, int b) { return a > b ? a : b; }
inline int imin_h(int a, int b) { return a < b ? a : b; }
inline int imax_h(int a, int b) { return a > b ? a : b; }
__device__ __forceinline__ bool cell_in_dom(const Phys& p, int i, int j, int k) { return cell_in(p, i, j, k); }

// face from 4 points: A, centroid Xb, s, and (optionally) the face-average velocity
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

}  // namespace

// ============================================================================
// kf_force: node planes [kn0, kn1] (global, inclusive), z-chunked by blockIdx.z
// ============================================================================
template <bool EULER, int NW>
__global__ void __launch_bounds__(FW * NW, MINB)
    kf_force(Slab s, Phys p, int cur, int kn0, int kn1, int zchunk)
{
    if (!s.st->active) return;
    constexpr int TX = FW - 2, TY = NW - 2;
    extern __shared__ double smem[];
    constexpr int PL = NW * FW;  // doubles per plane array
    // layout
    double* sN = smem;                  // [2 parity][6][PL]  x,y,z,ux,uy,uz of node planes
    double* sQ = sN + 2 * 6 * PL;       // [2 x|y][7][PL]     s, Xb(3), Ub(3) of x/y faces of cell plane kz
    double* sA = sQ + 2 * 7 * PL;       // [2 parity][2 x|y][3][PL]  A of x/y faces per cell plane
    double* sZ = sA + 2 * 2 * 3 * PL;   // [2 parity][3][PL]  A of z-faces per node plane
    double* sS = sZ + 2 * 3 * PL;       // [2 parity][2][PL]  sigma, m per cell plane

    const int ix = threadIdx.x, iy = threadIdx.y;
    const int tid = iy * FW + ix;
    const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
    const int i = i0 - 1 + ix, j = j0 - 1 + iy;
    const int za = kn0 + blockIdx.z * zchunk;
    const int zb = imin(kn1, za + zchunk - 1);
    const double dt = s.st->dt;
    const bool col_in = i >= 0 && i <= p.nx && j >= 0 && j <= p.ny;
    const int ixp = imin(ix + 1, FW - 1), iyp = imin(iy + 1, NW - 1);
    const int ixm = imax(ix - 1, 0), iym = imax(iy - 1, 0);

    auto NODE = [&](int par, int comp, int y, int x) -> double& { return sN[(par * 6 + comp) * PL + y * FW + x]; };
    auto node_pos = [&](int par, int y, int x) { return D3{NODE(par, 0, y, x), NODE(par, 1, y, x), NODE(par, 2, y, x)}; };
    auto node_vel = [&](int par, int y, int x) { return D3{NODE(par, 3, y, x), NODE(par, 4, y, x), NODE(par, 5, y, x)}; };

    // Register prefetch, one plane ahead: the global loads for node plane k+1
    // and cell (i,j,k) are issued at step k-1 and land in shared memory at step
    // k, so their DRAM latency overlaps a whole step of arithmetic.
    D3 px = D3{0.0, 0.0, 0.0}, pu = px;
    double pm = 0.0, pe = 0.0;
    auto fetch = [&](int k) {  // node plane k, cell plane k-1
        px = D3{0.0, 0.0, 0.0};
        pu = px;
        if (col_in && k >= 0 && k <= p.nz) {
            long long n = nidx(s, p, i, j, k);
            px = pos<EULER>(s, p, cur, i, j, k);
            pu = ld3(s.u[cur], n);
        }
        pm = 0.0;
        pe = 0.0;
        const int kc = k - 1;
        if (i >= 0 && i < p.nx && j >= 0 && j < p.ny && kc >= 0 && kc < p.nz) {
            long long c = cidx(s, p, i, j, kc);
            pm = mass_cur(s, p, cur)[c];
            pe = s.e[cur][c];
        }
    };
    auto put = [&](int k) {
        int par = k & 1;
        NODE(par, 0, iy, ix) = px.x;
        NODE(par, 1, iy, ix) = px.y;
        NODE(par, 2, iy, ix) = px.z;
        NODE(par, 3, iy, ix) = pu.x;
        NODE(par, 4, iy, ix) = pu.y;
        NODE(par, 5, iy, ix) = pu.z;
    };
    // z-face at node plane k anchored at this column: nodes (i,j),(i+1,j),(i+1,j+1),(i,j+1)
    auto zface = [&](int k) {
        int par = k & 1;
        return faceq(node_pos(par, iy, ix), node_pos(par, iy, ixp), node_pos(par, iyp, ixp), node_pos(par, iyp, ix),
                     node_vel(par, iy, ix), node_vel(par, iy, ixp), node_vel(par, iyp, ixp), node_vel(par, iyp, ix));
    };

    // prologue: node plane za-1 and its z-faces (the -z faces of cell plane za-1)
    fetch(za - 1);
    put(za - 1);
    fetch(za);
    __syncthreads();
    FaceQ zprev = zface(za - 1);

    for (int kz = za - 1; kz <= zb; ++kz) {
        const int b0 = kz & 1, b1 = (kz + 1) & 1;
        // ---- P1: node plane kz+1 and cell (i,j,kz) from the prefetch registers; prefetch the next
        put(kz + 1);
        const bool cell_in = i >= 0 && i < p.nx && j >= 0 && j < p.ny && kz >= 0 && kz < p.nz;
        const double m = pm, e = pe;
        if (kz < zb) fetch(kz + 2);
        __syncthreads();
        // ---- P2: faces of cell plane kz anchored at this column
        // x-face at node plane i: (i,j,kz) (i,j+1,kz) (i,j+1,kz+1) (i,j,kz+1)
        FaceQ fx = faceq(node_pos(b0, iy, ix), node_pos(b0, iyp, ix), node_pos(b1, iyp, ix), node_pos(b1, iy, ix),
                         node_vel(b0, iy, ix), node_vel(b0, iyp, ix), node_vel(b1, iyp, ix), node_vel(b1, iy, ix));
        // y-face at node plane j: (i,j,kz) (i,j,kz+1) (i+1,j,kz+1) (i+1,j,kz)
        FaceQ fy = faceq(node_pos(b0, iy, ix), node_pos(b1, iy, ix), node_pos(b1, iy, ixp), node_pos(b0, iy, ixp),
                         node_vel(b0, iy, ix), node_vel(b1, iy, ix), node_vel(b1, iy, ixp), node_vel(b0, iy, ixp));
        FaceQ znext = zface(kz + 1);
        {
            double* q0 = sQ;            // x-face
            double* q1 = sQ + 7 * PL;   // y-face
            q0[0 * PL + tid] = fx.s;
            q0[1 * PL + tid] = fx.Xb.x; q0[2 * PL + tid] = fx.Xb.y; q0[3 * PL + tid] = fx.Xb.z;
            q0[4 * PL + tid] = fx.Ub.x; q0[5 * PL + tid] = fx.Ub.y; q0[6 * PL + tid] = fx.Ub.z;
            q1[0 * PL + tid] = fy.s;
            q1[1 * PL + tid] = fy.Xb.x; q1[2 * PL + tid] = fy.Xb.y; q1[3 * PL + tid] = fy.Xb.z;
            q1[4 * PL + tid] = fy.Ub.x; q1[5 * PL + tid] = fy.Ub.y; q1[6 * PL + tid] = fy.Ub.z;
            double* ax = sA + ((b0 * 2 + 0) * 3) * PL;
            double* ay = sA + ((b0 * 2 + 1) * 3) * PL;
            ax[0 * PL + tid] = fx.A.x; ax[1 * PL + tid] = fx.A.y; ax[2 * PL + tid] = fx.A.z;
            ay[0 * PL + tid] = fy.A.x; ay[1 * PL + tid] = fy.A.y; ay[2 * PL + tid] = fy.A.z;
            double* az = sZ + (b1 * 3) * PL;
            az[0 * PL + tid] = znext.A.x; az[1 * PL + tid] = znext.A.y; az[2 * PL + tid] = znext.A.z;
        }
        __syncthreads();
        // ---- P3: cell (i,j,kz): V, rho, EoS, q, sigma
        {
            double sig = 0.0;
            if (cell_in) {
                const double* q0 = sQ;
                const double* q1 = sQ + 7 * PL;
                const int tx = iy * FW + ixp, ty = iyp * FW + ix;
                double sxp = q0[tx], syp = q1[ty];
                double sv[6] = {fx.s, sxp, fy.s, syp, zprev.s, znext.s};
                double V = vol_from_s(sv);
                double rho = m / V, pr, pf, cs;
                eos(p.gamma, rho, e, pr, pf, cs);
                D3 Xxp = D3{q0[1 * PL + tx], q0[2 * PL + tx], q0[3 * PL + tx]};
                D3 Uxp = D3{q0[4 * PL + tx], q0[5 * PL + tx], q0[6 * PL + tx]};
                D3 Xyp = D3{q1[1 * PL + ty], q1[2 * PL + ty], q1[3 * PL + ty]};
                D3 Uyp = D3{q1[4 * PL + ty], q1[5 * PL + ty], q1[6 * PL + ty]};
                double dx = axis_jump(fx.Xb, Xxp, fx.Ub, Uxp);
                double dy = axis_jump(fy.Xb, Xyp, fy.Ub, Uyp);
                double dz = axis_jump(zprev.Xb, znext.Xb, zprev.Ub, znext.Ub);
                double du = dmin(dmin(dx, dy), dz);
                double q = q_of_du(rho, cs, du, p.c1, p.c2);
                sig = 0.25 * (pf + q);
                if (kz >= za && kz >= kn0 && kz < kn1 && ix >= 1 && ix <= TX && iy >= 1 && iy <= TY)
                    s.sig[cidx(s, p, i, j, kz)] = sig;
            }
            sS[(b0 * 2 + 0) * PL + tid] = sig;
            sS[(b0 * 2 + 1) * PL + tid] = m;
        }
        zprev = znext;
        __syncthreads();
        // ---- P4: node (i,j,kz): force + mass gather, kinematics, BC, move
        if (kz >= za && ix >= 1 && ix <= TX && iy >= 1 && iy <= TY && col_in) {
            D3 F = D3{0.0, 0.0, 0.0};
            double M = 0.0;
            bool first = true;
            const int bz = kz & 1;
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                const int ap = g & 1, bp = (g >> 1) & 1, cp = g >> 2;
                const int ci = i - 1 + ap, cj = j - 1 + bp, ck = kz - 1 + cp;
                if (!cell_in_dom(p, ci, cj, ck)) continue;
                const int pc = ck & 1;
                const int cx = ix - 1 + ap, cy = iy - 1 + bp;
                const double* ax = sA + ((pc * 2 + 0) * 3) * PL + cy * FW + ix;   // x-face at plane i, row cj
                const double* ay = sA + ((pc * 2 + 1) * 3) * PL + iy * FW + cx;   // y-face at plane j, col ci
                const double* az = sZ + (bz * 3) * PL + cy * FW + cx;             // z-face at plane kz, (ci,cj)
                D3 Ax = D3{ax[0], ax[PL], ax[2 * PL]};
                D3 Ay = D3{ay[0], ay[PL], ay[2 * PL]};
                D3 Az = D3{az[0], az[PL], az[2 * PL]};
                D3 C = add(add(ap ? neg(Ax) : Ax, bp ? neg(Ay) : Ay), cp ? neg(Az) : Az);
                const double sg = sS[(pc * 2 + 0) * PL + cy * FW + cx];
                const double mk = sS[(pc * 2 + 1) * PL + cy * FW + cx];
                D3 term = scl(sg, C);
                if (first) {
                    F = term;
                    M = mk;
                    first = false;
                } else {
                    F = add(F, term);
                    M = M + mk;
                }
            }
            M = 0.125 * M;
            D3 u = node_vel(bz, iy, ix);
            D3 x = node_pos(bz, iy, ix);
            D3 un = d3(u.x + ((F.x / M) * dt), u.y + ((F.y / M) * dt), u.z + ((F.z / M) * dt));
            un = reflect(p, i, j, kz, un);
            D3 xn = d3(x.x + (un.x * dt), x.y + (un.y * dt), x.z + (un.z * dt));
            long long n = nidx(s, p, i, j, kz);
            if (EULER) {
                st3(s.u1, n, un);
                st3(s.x1, n, xn);
            } else {
                st3(s.x[cur ^ 1], n, xn);
                st3(s.u[cur ^ 1], n, un);
            }
        }
    }
}

// ============================================================================
// kf_energy: cell planes [kc0, kc1), z-chunked.  Columns i = i0 + ix (no lower halo).
// ============================================================================
template <bool EULER, int NW>
__global__ void __launch_bounds__(FW * NW, MINB)
    kf_energy(Slab s, Phys p, int cur, int kc0, int kc1, int zchunk)
{
    if (!s.st->active) return;
    constexpr int TX = FW - 1, TY = NW - 1;
    extern __shared__ double smem[];
    constexpr int PL = NW * FW;
    double* sP = smem;                  // [2 parity][10][PL] x^n(3), x'(3), ubar(3), |u'|^2 of node planes
    double* sF = sP + 2 * 10 * PL;      // [2 x|y][4][PL]      A^n(3), s' of x/y faces of cell plane kz
    double* sE = sF + 2 * 4 * PL;       // [3][PL]             edge^2 minima: x-edges, y-edges (2 planes), z-edge

    const int ix = threadIdx.x, iy = threadIdx.y;
    const int tid = iy * FW + ix;
    const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
    const int i = i0 + ix, j = j0 + iy;
    const int za = kc0 + blockIdx.z * zchunk;
    const int zb = imin(kc1 - 1, za + zchunk - 1);
    const double dt = s.st->dt;
    const bool col_in = i <= p.nx && j <= p.ny;
    const int ixp = imin(ix + 1, FW - 1), iyp = imin(iy + 1, NW - 1);
    unsigned long long key = KEY_NONE;

    auto P = [&](int par, int comp, int y, int x) -> double& { return sP[(par * 10 + comp) * PL + y * FW + x]; };
    auto xn_at = [&](int par, int y, int x) { return D3{P(par, 0, y, x), P(par, 1, y, x), P(par, 2, y, x)}; };
    auto x1_at = [&](int par, int y, int x) { return D3{P(par, 3, y, x), P(par, 4, y, x), P(par, 5, y, x)}; };
    auto ub_at = [&](int par, int y, int x) { return D3{P(par, 6, y, x), P(par, 7, y, x), P(par, 8, y, x)}; };

    // stage node plane k: x^n, x', ubar = 0.5 (u + u'), |u'|^2.  The raw loads
    // are issued one step ahead into registers (fetch) and staged next step (put).
    D3 fx = D3{0.0, 0.0, 0.0}, fu = fx, fu1 = fx, fx1 = fx;
    double fm = 0.0, fe = 0.0, fs = 0.0;
    auto fetch = [&](int k) {  // node plane k, cell plane k-1
        fx = D3{0.0, 0.0, 0.0};
        fu = fx; fu1 = fx; fx1 = fx;
        if (col_in && k >= 0 && k <= p.nz) {
            long long n = nidx(s, p, i, j, k);
            fx = pos<EULER>(s, p, cur, i, j, k);
            fu = ld3(s.u[cur], n);
            fu1 = EULER ? ld3(s.u1, n) : ld3(s.u[cur ^ 1], n);
            fx1 = EULER ? ld3(s.x1, n) : ld3(s.x[cur ^ 1], n);
        }
        fm = 0.0; fe = 0.0; fs = 0.0;
        const int kc = k - 1;
        if (i < p.nx && j < p.ny && kc >= 0 && kc < p.nz && ix < TX && iy < TY) {
            long long c = cidx(s, p, i, j, kc);
            fm = mass_cur(s, p, cur)[c];
            fe = s.e[cur][c];
            fs = s.sig[c];
        }
    };
    auto put = [&](int k) {
        int par = k & 1;
        D3 ub = scl(0.5, add(fu, fu1));
        double v2 = speed2(fu1);
        P(par, 0, iy, ix) = fx.x; P(par, 1, iy, ix) = fx.y; P(par, 2, iy, ix) = fx.z;
        P(par, 3, iy, ix) = fx1.x; P(par, 4, iy, ix) = fx1.y; P(par, 5, iy, ix) = fx1.z;
        P(par, 6, iy, ix) = ub.x; P(par, 7, iy, ix) = ub.y; P(par, 8, iy, ix) = ub.z;
        P(par, 9, iy, ix) = v2;
    };

    // prologue: node plane za; its z-face (A^n, s') and in-plane edges of x'
    fetch(za);
    put(za);
    fetch(za + 1);
    __syncthreads();
    D3 zA_prev;
    double zs_prev, ex_prev, ey_prev;
    {
        const int b = za & 1;
        zA_prev = face_area(xn_at(b, iy, ix), xn_at(b, iy, ixp), xn_at(b, iyp, ixp), xn_at(b, iyp, ix));
        D3 P0 = x1_at(b, iy, ix), P1 = x1_at(b, iy, ixp), P2 = x1_at(b, iyp, ixp), P3 = x1_at(b, iyp, ix);
        zs_prev = face_s(avg4(P0, P1, P2, P3), face_area(P0, P1, P2, P3));
        ex_prev = len2(P0, P1);
        ey_prev = len2(P0, P3);
    }

    for (int kz = za; kz <= zb; ++kz) {
        const int b0 = kz & 1, b1 = (kz + 1) & 1;
        // ---- P1: stage node plane kz+1 / cell kz from the prefetch registers, prefetch the next
        put(kz + 1);
        const bool cell_in = i < p.nx && j < p.ny && kz < p.nz;
        const double m = fm, e = fe, sig = fs;
        if (kz < zb) fetch(kz + 2);
        __syncthreads();
        // ---- P2: faces anchored at this column (A at t^n, s' at t^{n+1}); x' edges
        D3 zA_next;
        double zs_next, ex_next, ey_next;
        {
            // x-face at node plane i: (i,j,kz) (i,j+1,kz) (i,j+1,kz+1) (i,j,kz+1)
            D3 Ax = face_area(xn_at(b0, iy, ix), xn_at(b0, iyp, ix), xn_at(b1, iyp, ix), xn_at(b1, iy, ix));
            D3 Q0 = x1_at(b0, iy, ix), Q1 = x1_at(b0, iyp, ix), Q2 = x1_at(b1, iyp, ix), Q3 = x1_at(b1, iy, ix);
            double sx = face_s(avg4(Q0, Q1, Q2, Q3), face_area(Q0, Q1, Q2, Q3));
            // y-face at node plane j: (i,j,kz) (i,j,kz+1) (i+1,j,kz+1) (i+1,j,kz)
            D3 Ay = face_area(xn_at(b0, iy, ix), xn_at(b1, iy, ix), xn_at(b1, iy, ixp), xn_at(b0, iy, ixp));
            D3 R0 = x1_at(b0, iy, ix), R1 = x1_at(b1, iy, ix), R2 = x1_at(b1, iy, ixp), R3 = x1_at(b0, iy, ixp);
            double sy = face_s(avg4(R0, R1, R2, R3), face_area(R0, R1, R2, R3));
            // z-face at node plane kz+1
            zA_next = face_area(xn_at(b1, iy, ix), xn_at(b1, iy, ixp), xn_at(b1, iyp, ixp), xn_at(b1, iyp, ix));
            D3 T0 = x1_at(b1, iy, ix), T1 = x1_at(b1, iy, ixp), T2 = x1_at(b1, iyp, ixp), T3 = x1_at(b1, iyp, ix);
            zs_next = face_s(avg4(T0, T1, T2, T3), face_area(T0, T1, T2, T3));
            ex_next = len2(T0, T1);
            ey_next = len2(T0, T3);
            double ez = len2(Q0, Q3);  // z-edge (i,j): kz -> kz+1
            double* f0 = sF;
            double* f1 = sF + 4 * PL;
            f0[0 * PL + tid] = Ax.x; f0[1 * PL + tid] = Ax.y; f0[2 * PL + tid] = Ax.z; f0[3 * PL + tid] = sx;
            f1[0 * PL + tid] = Ay.x; f1[1 * PL + tid] = Ay.y; f1[2 * PL + tid] = Ay.z; f1[3 * PL + tid] = sy;
            sE[0 * PL + tid] = dmin(ex_prev, ex_next);
            sE[1 * PL + tid] = dmin(ey_prev, ey_next);
            sE[2 * PL + tid] = ez;
        }
        __syncthreads();
        // ---- P3: cell (i,j,kz)
        if (cell_in && ix < TX && iy < TY) {
            const int tx = iy * FW + ixp, ty = iyp * FW + ix;
            const double* f0 = sF;
            const double* f1 = sF + 4 * PL;
            double sv[6] = {f0[3 * PL + tid], f0[3 * PL + tx], f1[3 * PL + tid], f1[3 * PL + ty], zs_prev, zs_next};
            double V1 = vol_from_s(sv);
            const bool owned = kz >= s.k0 && kz < s.k1;
            if (owned && !(V1 > 0.0))
                atomicMin(&s.st->err_key, (ERR_ORDER_TANGLED << 48) | (unsigned long long)gcell(p, i, j, kz));
            D3 A[6] = {D3{f0[tid], f0[PL + tid], f0[2 * PL + tid]}, D3{f0[tx], f0[PL + tx], f0[2 * PL + tx]},
                       D3{f1[tid], f1[PL + tid], f1[2 * PL + tid]}, D3{f1[ty], f1[PL + ty], f1[2 * PL + ty]},
                       zA_prev, zA_next};
            double W = 0.0;
#pragma unroll
            for (int h = 0; h < 8; ++h) {
                const int a = h & 1, b = (h >> 1) & 1, c = h >> 2;
                D3 C = corner_vec(A, a, b, c);
                D3 ub = ub_at(c ? b1 : b0, iy + b, ix + a);
                double term = dot(C, ub);
                W = (h == 0) ? term : W + term;
            }
            long long cc = cidx(s, p, i, j, kz);
            double e1 = e - (((sig * W) * dt) / m);
            if (EULER) {
                s.e1[cc] = e1;
                s.V1[cc] = V1;
            } else {
                s.e[cur ^ 1][cc] = e1;
                if (owned) {
                    double rho = m / V1, pr, pf, cs;
                    eos(p.gamma, rho, e1, pr, pf, cs);
                    double l2 = dmin(dmin(sE[tid], sE[ty]), dmin(sE[PL + tid], sE[PL + tx]));
                    l2 = dmin(l2, dmin(dmin(sE[2 * PL + tid], sE[2 * PL + tx]),
                                       dmin(sE[2 * PL + ty], sE[2 * PL + iyp * FW + ixp])));
                    double v2 = P(b0, 9, iy, ix);
                    v2 = dmax(v2, P(b0, 9, iy, ix + 1));
                    v2 = dmax(v2, P(b0, 9, iy + 1, ix));
                    v2 = dmax(v2, P(b0, 9, iy + 1, ix + 1));
                    v2 = dmax(v2, P(b1, 9, iy, ix));
                    v2 = dmax(v2, P(b1, 9, iy, ix + 1));
                    v2 = dmax(v2, P(b1, 9, iy + 1, ix));
                    v2 = dmax(v2, P(b1, 9, iy + 1, ix + 1));
                    unsigned long long kk = dt_key(dt_cell(p.cfl, l2, v2, cs));
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
    if (!EULER) {
        // warp + block min, then one atomicMin per CTA
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
            key = other < key ? other : key;
        }
        __shared__ unsigned long long red[32];
        if (ix == 0) red[iy] = key;
        __syncthreads();
        if (iy == 0) {
            key = ix < NW ? red[ix] : KEY_NONE;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
                key = other < key ? other : key;
            }
            if (ix == 0 && key != KEY_NONE) atomicMin(&s.st->cand_key, key);
        }
    }
}

// ============================================================================
// launchers
// ============================================================================
namespace {
constexpr int NW_FORCE = 8;
constexpr int NW_ENERGY = 8;
constexpr int ZCHUNK = 32;

constexpr size_t force_smem(int nw) { return sizeof(double) * (size_t)nw * FW * (2 * 6 + 2 * 7 + 2 * 2 * 3 + 2 * 3 + 2 * 2); }
constexpr size_t energy_smem(int nw) { return sizeof(double) * (size_t)nw * FW * (2 * 10 + 2 * 4 + 3); }

template <typename K>
void set_smem(K kernel, size_t bytes)
{
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

inline int cdiv(int a, int b) { return (a + b - 1) / b; }
}  // namespace

template <bool EULER>
static int lagrange_fused(const Slab& s, const Phys& p, int cur, Stream st)
{
    cudaStream_t cs = (cudaStream_t)st;
    // node planes updated / cell planes energised (Euler: plus the ghost region the remap needs)
    int kn0, kn1, kc0, kc1;
    if (!EULER) {
        kn0 = s.k0; kn1 = s.k1; kc0 = s.k0; kc1 = s.k1;
    } else {
        kn0 = imax_h(s.k0 - 2, 0); kn1 = imin_h(s.k1 + 2, p.nz);
        kc0 = kn0; kc1 = kn1;
    }
    {
        constexpr int NW = NW_FORCE;
        size_t sm = force_smem(NW);
        static bool init = false;
        if (!init) {
            set_smem(kf_force<EULER, NW>, sm);
            init = true;
        }
        dim3 grid(cdiv(p.nx + 1, FW - 2), cdiv(p.ny + 1, NW - 2), cdiv(kn1 - kn0 + 1, ZCHUNK));
        kf_force<EULER, NW><<<grid, dim3(FW, NW), sm, cs>>>(s, p, cur, kn0, kn1, ZCHUNK);
    }
    {
        constexpr int NW = NW_ENERGY;
        size_t sm = energy_smem(NW);
        static bool init = false;
        if (!init) {
            set_smem(kf_energy<EULER, NW>, sm);
            init = true;
        }
        dim3 grid(cdiv(p.nx, FW - 1), cdiv(p.ny, NW - 1), cdiv(kc1 - kc0, ZCHUNK));
        kf_energy<EULER, NW><<<grid, dim3(FW, NW), sm, cs>>>(s, p, cur, kc0, kc1, ZCHUNK);
    }
    return 2;
}

int launch_lagrange_fused(const Slab& s, const Phys& p, int cur, Stream st)
{
    return p.rezone ? lagrange_fused<true>(s, p, cur, st) : lagrange_fused<false>(s, p, cur, st);
}

// remap: the v0 kernels for now (they read x1/u1/e1/V1 written above)
int launch_remap_fused(const Slab& s, const Phys& p, int cur, Stream st) { return launch_remap_v0(s, p, cur, st); }

}  // namespace sale
