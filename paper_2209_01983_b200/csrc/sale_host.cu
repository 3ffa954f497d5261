// sale_host.cu -- the C ABI of libsale (include/sale.h): parameter validation,
// workspace carving, z-slab layout, cycle enqueueing, halo exchange (device
// copies between local slabs, NCCL send/recv between ranks), dt / error
// min-reduction (NCCL allreduce), field access.
//
// Paper context: ScalSALE's kernel layer owns the data structures
// (Data3d with ghost frames) and the Communication / CommParams
// classes doing blocking and non-blocking ghost exchange
// (P:372-375).  Here that becomes: SoA fp64 slabs with ghost z-planes,
// one grouped NCCL exchange + one 16-byte allreduce-min per cycle, all enqueued
// on the caller's stream with no host synchronisation inside sale_step's loop.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstddef>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "sale.h"
#include "sale_internal.h"

static_assert(SALE_OK == sale::S_OK && SALE_ETANGLED == sale::S_ETANGLED &&
                  SALE_EDTCOLLAPSE == sale::S_EDTCOLLAPSE && SALE_ENEGMASS == sale::S_ENEGMASS &&
                  SALE_EREPLICA == sale::S_EREPLICA,
              "status codes out of sync");
static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
static_assert(SALE_MAX_MAT == sale::MAX_MAT, "material count out of sync");
static_assert(offsetof(sale::DevState, err_key) == offsetof(sale::DevState, cand_key) + 8,
              "cand_key / err_key must be adjacent for the 2-element allreduce");

using sale::DevState;
using sale::Phys;
using sale::Slab;

struct sale_ctx {
    sale_params prm;
    Phys phys;
    int g = 1;                       // ghost depth
    std::vector<Slab> slabs;
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;
    DevState* dstate = nullptr;      // device
    DevState* hstate = nullptr;      // pinned host mirror
    int cur = 0;                     // parity of the current state at the last sync
    int cur_enq = 0;                 // parity the next enqueued cycle reads
    bool poisoned = false;
    long long launches = 0;
    std::string err = "OK";
    // kernel-class timing (sale_profile_enable)
    struct Pending {
        int cls;
        cudaEvent_t a, b;
    };
    bool prof_on = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<Pending> pending;
    double prof_ms[SALE_K_NCLASS] = {0};
    long long prof_cnt[SALE_K_NCLASS] = {0};
    // captured two-cycle CUDA graphs by starting buffer parity, and their kernel count
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    long long glaunches[2] = {0, 0};
    cudaStream_t cap_stream = nullptr;  // private stream the graphs are captured on
    // boundary-first cycles: the halo exchange runs on `side` while the interior
    // finishes; evB = boundary planes done, evX = exchange done
    cudaStream_t side = nullptr;
    cudaEvent_t evB = nullptr, evX = nullptr;
    // peer-store halo (sale_params.halo = SALE_HALO_PEER): per slab its device table of
    // the neighbours' arrays; ranks: the neighbours' workspaces mapped by CUDA IPC, and
    // which neighbours exist (bit 0 lower, bit 1 upper)
    std::vector<sale::HaloPeer*> hp_dev;
    void* ipc[2] = {nullptr, nullptr};
    int peer_sides = 0;
};

namespace {

const char* code_name(int c)
{
    switch (c) {
    case SALE_OK: return "OK";
    case SALE_EINVAL: return "EINVAL";
    case SALE_ENOMEM: return "ENOMEM";
    case SALE_ECUDA: return "ECUDA";
    case SALE_ENCCL: return "ENCCL";
    case SALE_ETANGLED: return "ETANGLED";
    case SALE_EDTCOLLAPSE: return "EDTCOLLAPSE";
    case SALE_ENEGMASS: return "ENEGMASS";
    case SALE_EPOISONED: return "EPOISONED";
    case SALE_EREPLICA: return "EREPLICA";
    default: return "E?";
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard()
    {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

int ghost_depth(const sale_params* p) { return p->rezone == SALE_EULER ? 3 : 1; }

bool params_ok(const sale_params* p)
{
    if (!p || p->abi_version != SALE_ABI_VERSION) return false;
    if (p->nx < 1 || p->ny < 1 || p->nz < 1) return false;
    if (!(p->lx > 0.0) || !(p->ly > 0.0) || !(p->lz > 0.0)) return false;
    if (!(p->gamma > 1.0) || !(p->cfl > 0.0) || !(p->dt_growth > 0.0)) return false;
    if (!(p->q_lin >= 0.0) || !(p->q_quad >= 0.0)) return false;
    if (p->rezone != SALE_LAGRANGE && p->rezone != SALE_EULER) return false;
    if (p->reflect_mask > 0x3Fu) return false;
    if (!(p->rho0 > 0.0)) return false;
    if (p->nranks < 1 || p->rank < 0 || p->rank >= p->nranks) return false;
    if (p->nranks > 1 && p->nccl_unique_id == nullptr) return false;  // nranks == 1 + id: 1-rank NCCL comm
    if (p->local_slabs < 1 || (p->nranks > 1 && p->local_slabs != 1)) return false;
    if (!(p->hg >= 0.0)) return false;
    if (p->overlap < -1 || p->overlap > 1) return false;
    if (p->halo != SALE_HALO_COPY && p->halo != SALE_HALO_PEER) return false;
    int T = p->nranks * p->local_slabs;
    if (p->nz < T) return false;
    if (T > 1 && p->nz / T < ghost_depth(p)) return false;  // every slab owns >= g planes
    if ((long long)(p->nx + 1) * (p->ny + 1) > (1ll << 40)) return false;
    if (p->nmat < 0 || p->nmat > SALE_MAX_MAT) return false;
    for (int k = 0; k < p->nmat; ++k)
        if (!(p->mat_gamma[k] > 1.0)) return false;
    return true;
}

// parameter checks for the host-only planning entry points (no NCCL id needed)
bool params_ok_layout(const sale_params* p)
{
    if (!p) return false;
    sale_params q = *p;
    q.nccl_unique_id = q.nranks > 1 ? (const void*)p : nullptr;
    return params_ok(&q);
}

// slab s of T: remainder planes go to the lowest slabs
void slab_range(int nz, int T, int s, int& k0, int& k1)
{
    int base = nz / T, rem = nz % T;
    k0 = s * base + (s < rem ? s : rem);
    k1 = k0 + base + (s < rem ? 1 : 0);
}

const size_t ALIGN = 256;
size_t align_up(size_t v) { return (v + ALIGN - 1) / ALIGN * ALIGN; }

// carve one slab's arrays from base (nullptr: size only); returns bytes used
size_t carve_slab(const sale_params* p, Slab& s, char* base)
{
    size_t off = 0;
    auto take = [&](long long ndouble) -> double* {
        double* ptr = base ? reinterpret_cast<double*>(base + off) : nullptr;
        off += align_up(sizeof(double) * (size_t)ndouble);
        return ptr;
    };
    long long nn = s.pn * s.nzn, nc = s.pc * s.nzc;
    bool euler = p->rezone == SALE_EULER;
    for (int b = 0; b < 2; ++b)
        for (int a = 0; a < 3; ++a) {
            s.x[b][a] = euler ? nullptr : take(nn);
            s.u[b][a] = take(nn);
        }
    s.m[0] = take(nc);
    s.m[1] = euler ? take(nc) : nullptr;
    s.e[0] = take(nc);
    s.e[1] = take(nc);
    s.sig = take(nc);
    s.hnu = take(nc);
    for (int a = 0; a < 3; ++a) {
        s.x1[a] = nullptr;  // x' is formed from u' where needed (Euler)
        s.u1[a] = euler ? take(nn) : nullptr;
        s.dP[a] = euler ? take(nc) : nullptr;
    }
    s.e1 = euler ? take(nc) : nullptr;
    s.V1 = euler ? take(nc) : nullptr;
    s.dm = euler ? take(nc) : nullptr;
    for (int a = 0; a < 3; ++a) {
        s.dV[a] = euler ? take(nc) : nullptr;
        s.UD[a] = euler ? take(nc) : nullptr;
    }
    s.rD = euler ? take(nc) : nullptr;
    s.der = take(s.pn * (long long)(s.k1 - s.k0 + 1));
    s.VT = euler ? take(nc) : nullptr;
    for (int a = 0; a < 3; ++a) s.sT[a] = euler ? take(nc) : nullptr;
    for (int a = 0; a < 3; ++a) {
        s.TAx[a] = euler ? take((long long)p->ny * s.nzc) : nullptr;
        s.TAy[a] = euler ? take((long long)p->nx * s.nzc) : nullptr;
        s.TAz[a] = euler ? take((long long)p->nx * p->ny) : nullptr;
    }
    for (int a = 0; a < 3; ++a) s.sF[a] = euler ? take(nn) : nullptr;
    s.TDx = euler ? take(p->nx) : nullptr;
    s.TDy = euler ? take(p->ny) : nullptr;
    s.TDz = euler ? take(s.nzc) : nullptr;
    s.TJx = euler ? take(4LL * p->nx) : nullptr;
    s.TJy = euler ? take(4LL * p->ny) : nullptr;
    s.TJz = euler ? take(4LL * s.nzc) : nullptr;
    s.Xt = take(p->nx + 1);
    s.Yt = take(p->ny + 1);
    s.Zt = take(s.nzn);
    const long long M = p->nmat;
    for (int b = 0; b < 2; ++b) {  // Lagrange: f_k and m_k never change (index [0] only)
        s.mf[b] = M && (b == 0 || euler) ? take(M * nc) : nullptr;
        s.mm[b] = M && (b == 0 || euler) ? take(M * nc) : nullptr;
        s.me[b] = M ? take(M * nc) : nullptr;
    }
    s.sgm = M ? take(M * nc) : nullptr;
    s.e1m = M && euler ? take(M * nc) : nullptr;
    s.rDm = M && euler ? take(M * nc) : nullptr;
    return off;
}

void layout_slabs(const sale_params* p, std::vector<Slab>& out)
{
    int g = ghost_depth(p);
    int T = p->nranks * p->local_slabs;
    out.clear();
    for (int l = 0; l < p->local_slabs; ++l) {
        Slab s;
        std::memset(&s, 0, sizeof s);
        int sid = p->rank * p->local_slabs + l;
        slab_range(p->nz, T, sid, s.k0, s.k1);
        s.g = g;
        s.kb = s.k0 - g;
        s.nzc = (s.k1 - s.k0) + 2 * g;
        s.nzn = s.nzc + 1;
        s.pn = (long long)(p->nx + 1) * (p->ny + 1);
        s.pc = (long long)p->nx * p->ny;
        s.nmat = p->nmat;
        for (int k = 0; k < sale::MAX_MAT; ++k) s.mg[k] = k < p->nmat ? p->mat_gamma[k] : 0.0;
        out.push_back(s);
    }
}

size_t total_bytes(const sale_params* p)
{
    std::vector<Slab> v;
    layout_slabs(p, v);
    size_t total = align_up(sizeof(DevState));
    for (auto& s : v) total += carve_slab(p, s, nullptr);
    if (p->halo == SALE_HALO_PEER) total += v.size() * align_up(sizeof(sale::HaloPeer));  // peer tables
    return total;
}

int set_err(sale_ctx* c, int code, const std::string& msg)
{
    if (c) {
        c->err = std::string(code_name(code)) + ": " + msg;
        if (code != SALE_EINVAL && code != SALE_ENOMEM) c->poisoned = true;
    }
    return code;
}

int cuda_check(sale_ctx* c, cudaError_t e, const char* what)
{
    if (e == cudaSuccess) return SALE_OK;
    return set_err(c, SALE_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int nccl_check(sale_ctx* c, ncclResult_t r, const char* what)
{
    if (r == ncclSuccess) return SALE_OK;
    return set_err(c, SALE_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

int launch_check(sale_ctx* c)
{
    cudaError_t e = cudaGetLastError();
    const cudaError_t noted = (cudaError_t)sale::take_launch_error();
    return cuda_check(c, noted != cudaSuccess ? noted : e, "kernel launch");
}

cudaEvent_t take_event(sale_ctx* c)
{
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// bracket a launch group of class cls with events (no-op unless profiling)
int prof_open(sale_ctx* c, int cls)
{
    if (!c->prof_on) return -1;
    sale_ctx::Pending p{cls, take_event(c), take_event(c)};
    cudaEventRecord(p.a, c->stream);
    c->pending.push_back(p);
    return (int)c->pending.size() - 1;
}
void prof_close(sale_ctx* c, int idx)
{
    if (idx >= 0) cudaEventRecord(c->pending[idx].b, c->stream);
}
// after a stream sync: accumulate and recycle
void prof_collect(sale_ctx* c)
{
    for (auto& p : c->pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
            c->prof_ms[p.cls] += ms;
            c->prof_cnt[p.cls] += 1;
        }
        c->ev_pool.push_back(p.a);
        c->ev_pool.push_back(p.b);
    }
    c->pending.clear();
}

void state_arrays(const sale_ctx* c, const Slab& s, int b, bool include_mass,
                  std::vector<double*>& nodes, std::vector<double*>& cells)
{
    nodes.clear();
    cells.clear();
    bool euler = c->prm.rezone == SALE_EULER;
    if (!euler)
        for (int a = 0; a < 3; ++a) nodes.push_back(s.x[b][a]);
    for (int a = 0; a < 3; ++a) nodes.push_back(s.u[b][a]);
    if (euler)
        cells.push_back(s.m[b]);
    else if (include_mass)
        cells.push_back(s.m[0]);
    cells.push_back(s.e[b]);
    // material axis: one cell array per material and quantity (the same field order
    // as plan_fields)
    const long long nc = s.pc * (long long)s.nzc;
    if (euler || include_mass)
        for (int k = 0; k < c->prm.nmat; ++k) {
            cells.push_back(s.mf[euler ? b : 0] + k * nc);
            cells.push_back(s.mm[euler ? b : 0] + k * nc);
        }
    for (int k = 0; k < c->prm.nmat; ++k) cells.push_back(s.me[b] + k * nc);
}

// the state fields a halo exchange moves, in plan order
void plan_fields(const sale_params* p, int full, std::vector<int>& node_f, std::vector<int>& cell_f)
{
    node_f.clear();
    cell_f.clear();
    bool euler = p->rezone == SALE_EULER;
    if (!euler) {
        node_f.push_back(SALE_F_X);
        node_f.push_back(SALE_F_Y);
        node_f.push_back(SALE_F_Z);
    }
    node_f.push_back(SALE_F_UX);
    node_f.push_back(SALE_F_UY);
    node_f.push_back(SALE_F_UZ);
    if (euler || full) cell_f.push_back(SALE_F_MASS);
    cell_f.push_back(SALE_F_E);
    if (euler || full)
        for (int k = 0; k < p->nmat; ++k) {
            cell_f.push_back(SALE_F_MAT_F(k));
            cell_f.push_back(SALE_F_MAT_M(k));
        }
    for (int k = 0; k < p->nmat; ++k) cell_f.push_back(SALE_F_MAT_E(k));
}

// X1 plan of rank p->rank (one slab per rank): for every field, to / from r-1
// then r+1; node planes [k0+1, k0+g] / [k1-g, k1-1] go out, ghosts [k0-g, k0-1] /
// [k1+1, k1+g] come in; cell planes [k0, k0+g) / [k1-g, k1) out, [k0-g, k0) /
// [k1, k1+g) in.  Offsets are into the local arrays (local plane = k - (k0-g)).
void build_plan(const sale_params* p, int full, std::vector<sale_halo_msg>& out)
{
    out.clear();
    if (p->nranks <= 1) return;
    std::vector<Slab> v;
    layout_slabs(p, v);
    const Slab& S = v[0];
    const int g = S.g, r = p->rank, n = p->nranks;
    std::vector<int> nf, cf;
    plan_fields(p, full, nf, cf);
    auto push = [&](int peer, int send, int field, int k_first, long long plane, int kb) {
        sale_halo_msg m;
        m.peer = peer;
        m.send = send;
        m.field = field;
        m.first_plane = k_first;
        m.offset = (int64_t)(k_first - kb) * plane;
        m.count = (int64_t)g * plane;
        out.push_back(m);
    };
    for (int f : nf) {
        if (r > 0) {
            push(r - 1, 1, f, S.k0 + 1, S.pn, S.kb);
            push(r - 1, 0, f, S.k0 - g, S.pn, S.kb);
        }
        if (r < n - 1) {
            push(r + 1, 1, f, S.k1 - g, S.pn, S.kb);
            push(r + 1, 0, f, S.k1 + 1, S.pn, S.kb);
        }
    }
    for (int f : cf) {
        if (r > 0) {
            push(r - 1, 1, f, S.k0, S.pc, S.kb);
            push(r - 1, 0, f, S.k0 - g, S.pc, S.kb);
        }
        if (r < n - 1) {
            push(r + 1, 1, f, S.k1 - g, S.pc, S.kb);
            push(r + 1, 0, f, S.k1, S.pc, S.kb);
        }
    }
}

// material field -> 0 (f) / 1 (m) / 2 (e) and the material, or -1
int mat_kind(int nmat, int field, int* mat)
{
    if (field < SALE_F_MAT_F(0) || field >= SALE_F_MAT_E(SALE_MAX_MAT)) return -1;
    *mat = (field - SALE_F_MAT_F(0)) % SALE_MAX_MAT;
    return *mat < nmat ? (field - SALE_F_MAT_F(0)) / SALE_MAX_MAT : -1;
}

// the (local, whole-slab) array of material field `field` in buffer b
double* mat_array(const sale_ctx* c, const Slab& s, int b, int field)
{
    int mat, kind = mat_kind(c->prm.nmat, field, &mat);
    if (kind < 0) return nullptr;
    const bool euler = c->prm.rezone == SALE_EULER;
    const long long off = (long long)mat * s.pc * s.nzc;
    if (kind == 2) return s.me[b] + off;
    return (kind == 0 ? s.mf[euler ? b : 0] : s.mm[euler ? b : 0]) + off;
}

double* field_array(const sale_ctx* c, const Slab& s, int b, int field)
{
    bool euler = c->prm.rezone == SALE_EULER;
    if (field >= SALE_F_MAT_F(0)) return mat_array(c, s, b, field);
    if (field <= SALE_F_Z) return s.x[b][field];
    if (field <= SALE_F_UZ) return s.u[b][field - SALE_F_UX];
    if (field == SALE_F_MASS) return euler ? s.m[b] : s.m[0];
    return s.e[b];
}

// X1: ghost planes between neighbouring slabs, buffer b, on stream `on` (default: the
// context's stream)
int exchange(sale_ctx* c, int b, bool include_mass, cudaStream_t on = nullptr)
{
    const cudaStream_t stream_ = on ? on : c->stream;
    const int g = c->g;
    const size_t pn = (size_t)c->slabs[0].pn, pc = (size_t)c->slabs[0].pc;
    std::vector<double*> nL, cL, nU, cU;
    // local slab pairs: device-to-device copies
    for (size_t l = 0; l + 1 < c->slabs.size(); ++l) {
        const Slab& L = c->slabs[l];
        const Slab& U = c->slabs[l + 1];
        int kI = L.k1;
        state_arrays(c, L, b, include_mass, nL, cL);
        state_arrays(c, U, b, include_mass, nU, cU);
        for (size_t f = 0; f < nL.size(); ++f) {
            // U ghost nodes [kI-g, kI-1] <- L ; L ghost nodes [kI+1, kI+g] <- U
            size_t bytes = sizeof(double) * pn * g;
            cudaMemcpyAsync(nU[f] + (size_t)(kI - g - U.kb) * pn, nL[f] + (size_t)(kI - g - L.kb) * pn,
                            bytes, cudaMemcpyDeviceToDevice, stream_);
            cudaMemcpyAsync(nL[f] + (size_t)(kI + 1 - L.kb) * pn, nU[f] + (size_t)(kI + 1 - U.kb) * pn,
                            bytes, cudaMemcpyDeviceToDevice, stream_);
        }
        for (size_t f = 0; f < cL.size(); ++f) {
            size_t bytes = sizeof(double) * pc * g;
            cudaMemcpyAsync(cU[f] + (size_t)(kI - g - U.kb) * pc, cL[f] + (size_t)(kI - g - L.kb) * pc,
                            bytes, cudaMemcpyDeviceToDevice, stream_);
            cudaMemcpyAsync(cL[f] + (size_t)(kI - L.kb) * pc, cU[f] + (size_t)(kI - U.kb) * pc,
                            bytes, cudaMemcpyDeviceToDevice, stream_);
        }
    }
    int rc = cuda_check(c, cudaGetLastError(), "halo copy");
    if (rc) return rc;
    if (c->prm.nranks == 1) return SALE_OK;  // (a 1-rank communicator has no halo messages)
    // ranks: one grouped NCCL exchange with r-1 and r+1, exactly the messages of
    // the host-side plan (sale_halo_plan, tested on CPU with gloo)
    const Slab& S = c->slabs[0];
    std::vector<sale_halo_msg> plan;
    build_plan(&c->prm, include_mass ? 1 : 0, plan);
    ncclGroupStart();
    for (const sale_halo_msg& m : plan) {
        double* a = field_array(c, S, b, m.field);
        if (m.send)
            ncclSend(a + m.offset, (size_t)m.count, ncclFloat64, m.peer, c->comm, stream_);
        else
            ncclRecv(a + m.offset, (size_t)m.count, ncclFloat64, m.peer, c->comm, stream_);
    }
    return nccl_check(c, ncclGroupEnd(), "halo exchange");
}

// X2: min over ranks of (dt candidate key, error key)
int reduce_keys(sale_ctx* c)
{
    if (!c->comm) return SALE_OK;
    return nccl_check(c,
                      ncclAllReduce(&c->dstate->cand_key, &c->dstate->cand_key, 2, ncclUint64, ncclMin,
                                    c->comm, c->stream),
                      "dt allreduce");
}

bool overlap_on(const sale_ctx* c)
{
    if (c->prm.halo == SALE_HALO_PEER) return false;  // no exchange to overlap
    const int o = c->prm.overlap;
    const bool multi = c->prm.nranks > 1 || c->prm.local_slabs > 1;
    return multi && (o > 0 || (o == 0 && c->prm.nranks > 1));
}

int overlap_resources(sale_ctx* c)
{
    int rc = SALE_OK;
    if (!c->side) rc = cuda_check(c, cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking), "side stream");
    if (!rc && !c->evB) rc = cuda_check(c, cudaEventCreateWithFlags(&c->evB, cudaEventDisableTiming), "event");
    if (!rc && !c->evX) rc = cuda_check(c, cudaEventCreateWithFlags(&c->evX, cudaEventDisableTiming), "event");
    return rc;
}

// ---- peer-store halo (SALE_HALO_PEER) ----------------------------------------
// side 0 / 1 of table h: the arrays of neighbour slab P (in its owner's address space as
// mapped here) that receive the planes of the per-cycle exchange (plan_fields, full = 0)
void fill_side(const sale_ctx* c, const Slab& P, int side, sale::HaloPeer& h)
{
    const bool euler = c->prm.rezone == SALE_EULER;
    const bool mat = c->prm.nmat > 0;
    for (int b = 0; b < 2; ++b) {
        for (int a = 0; a < 3; ++a) {
            h.x[side][b][a] = euler ? nullptr : P.x[b][a];
            h.u[side][b][a] = P.u[b][a];
        }
        h.m[side][b] = euler ? P.m[b] : nullptr;
        h.e[side][b] = P.e[b];
        h.mf[side][b] = mat && euler ? P.mf[b] : nullptr;
        h.mm[side][b] = mat && euler ? P.mm[b] : nullptr;
        h.me[side][b] = mat ? P.me[b] : nullptr;
    }
    h.mstride[side] = P.pc * (long long)P.nzc;
    h.kb[side] = P.kb;
}

// ranks: map the neighbours' workspaces (CUDA IPC handles of the allocations holding
// them, exchanged with one ncclAllGather) and fill the rank's table from their layout
int ipc_neighbours(sale_ctx* c, sale::HaloPeer& h)
{
    typedef int (*RangeFn)(unsigned long long*, size_t*, unsigned long long);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
        q != cudaDriverEntryPointSuccess)
        return set_err(c, SALE_ECUDA, "peer halo: cuMemGetAddressRange unavailable");
    unsigned long long abase = 0;
    size_t asz = 0;
    if (((RangeFn)fn)(&abase, &asz, (unsigned long long)(uintptr_t)c->prm.workspace) != 0)
        return set_err(c, SALE_ECUDA, "peer halo: workspace allocation range");
    struct Rec {
        cudaIpcMemHandle_t h;
        unsigned long long off;
        char pad[128 - sizeof(cudaIpcMemHandle_t) - 8];
    };
    static_assert(sizeof(Rec) == 128, "IPC record");
    Rec mine;
    std::memset(&mine, 0, sizeof mine);
    int rc = cuda_check(c, cudaIpcGetMemHandle(&mine.h, (void*)(uintptr_t)abase),
                        "peer halo: cudaIpcGetMemHandle (the workspace must be cudaMalloc memory)");
    if (rc) return rc;
    mine.off = (unsigned long long)((uintptr_t)c->prm.workspace - abase);
    const int n = c->prm.nranks, r = c->prm.rank;
    char* dbuf = nullptr;
    if ((rc = cuda_check(c, cudaMalloc((void**)&dbuf, sizeof(Rec) * (n + 1)), "peer halo: scratch"))) return rc;
    std::vector<Rec> all(n);
    rc = cuda_check(c, cudaMemcpy(dbuf, &mine, sizeof mine, cudaMemcpyHostToDevice), "peer halo: copy");
    if (!rc)
        rc = nccl_check(c, ncclAllGather(dbuf, dbuf + sizeof(Rec), sizeof(Rec), ncclUint8, c->comm, c->stream),
                        "peer halo: handle allgather");
    if (!rc) rc = cuda_check(c, cudaStreamSynchronize(c->stream), "peer halo: sync");
    if (!rc)
        rc = cuda_check(c, cudaMemcpy(all.data(), dbuf + sizeof(Rec), sizeof(Rec) * n, cudaMemcpyDeviceToHost),
                        "peer halo: copy");
    cudaFree(dbuf);
    if (rc) return rc;
    for (int side = 0; side < 2; ++side) {
        const int peer = r + (side ? 1 : -1);
        if (peer < 0 || peer >= n) continue;
        void* mp = nullptr;
        rc = cuda_check(c, cudaIpcOpenMemHandle(&mp, all[peer].h, cudaIpcMemLazyEnablePeerAccess),
                        "peer halo: cudaIpcOpenMemHandle");
        if (rc) return rc;
        c->ipc[side] = mp;
        char* pws = static_cast<char*>(mp) + all[peer].off;
        sale_params qp = c->prm;
        qp.rank = peer;
        std::vector<Slab> v;
        layout_slabs(&qp, v);
        Slab P = v[0];
        carve_slab(&qp, P, pws + align_up(sizeof(DevState)));
        fill_side(c, P, side, h);
        // we are our lower neighbour's upper neighbour: its halo_in[1], and vice versa
        h.flag[side] = &reinterpret_cast<DevState*>(pws)->halo_in[1 - side];
        c->peer_sides |= 1 << side;
    }
    return SALE_OK;
}

// build every slab's table (emulated slabs: the neighbouring slabs of this context;
// ranks: the mapped neighbours) and point the slabs at them
int peer_tables(sale_ctx* c)
{
    const size_t L = c->slabs.size();
    std::vector<sale::HaloPeer> h(L);
    for (auto& t : h) std::memset(&t, 0, sizeof t);
    for (size_t l = 0; l < L; ++l) {
        if (l > 0) fill_side(c, c->slabs[l - 1], 0, h[l]);
        if (l + 1 < L) fill_side(c, c->slabs[l + 1], 1, h[l]);
    }
    int rc = SALE_OK;
    if (c->prm.nranks > 1 && (rc = ipc_neighbours(c, h[0]))) return rc;
    for (size_t l = 0; l < L; ++l) {
        rc = cuda_check(c, cudaMemcpy(c->hp_dev[l], &h[l], sizeof h[l], cudaMemcpyHostToDevice), "peer table");
        if (rc) return rc;
        c->slabs[l].hp = c->hp_dev[l];
    }
    return SALE_OK;
}

// The planes of a slab the exchange sends and the slab's last kernel writes:
// Lagrange cell planes [k0, k0+g) and [k1-g, k1) (e'; x', u' come from kc_force, which
// runs whole before); Euler node planes [k0, k0+g] and [k1-g, k1] (u''; single
// material: kr_tail forms and stores m'', e'' of cell planes [k0, k0+g] and [k1-g, k1)
// in the same launches; materials: k_mat_flux runs whole before).  part 0 = those, part 1 = the rest.
// A slab too thin to have an interior runs whole as part 0.
int launch_tail(sale_ctx* c, const Slab& s, int b, int part, sale::Stream st)
{
    const bool euler = c->prm.rezone == SALE_EULER;
    const int g = s.g, k0 = s.k0, k1 = s.k1;
    const bool thin = k1 - k0 < 2 * g + 2;
    if (part == 1 && thin) return 0;
    int n = 0;
    if (euler) {
        // single material: kr_tail (R2-R4, the cells of the range stored by it);
        // materials: kn_update (R4; k_mat_flux ran whole before)
        auto nodes = c->prm.nmat ? sale::launch_kn_update : sale::launch_rtail;
        if (part == 0 && thin) return nodes(s, c->phys, b, st, -1, -1);
        if (part == 0) {
            n += nodes(s, c->phys, b, st, k0, k0 + g);
            n += nodes(s, c->phys, b, st, k1 - g, k1);
        } else {
            n += nodes(s, c->phys, b, st, k0 + g + 1, k1 - g - 1);
        }
    } else {
        if (part == 0 && thin) return sale::launch_energy(s, c->phys, b, st);
        if (part == 0) {
            n += sale::launch_energy(s, c->phys, b, st, k0, k0 + g);
            n += sale::launch_energy(s, c->phys, b, st, k1 - g, k1);
        } else {
            n += sale::launch_energy(s, c->phys, b, st, k0 + g, k1 - g);
        }
    }
    return n;
}

// one cycle reading buffers [b]; first = the first cycle of a sale_step call (its
// state pass runs ungated, DevState.active being still 0 then).  Both modes:
//   kl_state / ke_state (cell state + dt candidate of the cycle-start state) -> dt /
//   error allreduce -> k_begin (commit the previous cycle, finalise dt) -> kc_force
//   -> kc_energy -> [Euler: remap] -> halo exchange of the new state
// Boundary-first (overlap_on): the last kernel of the cycle (Lagrange kc_energy, Euler
// kn_update) runs first on the planes the exchange sends (launch_tail part 0 on every
// slab), the exchange starts on the side stream, the interior (part 1) runs on the
// context's stream meanwhile, and the stream joins the exchange before the next
// cycle.  The interior writes owned planes of b^1 only, the exchange ghost planes of
// b^1 only; it reads owned planes the boundary part finished.
int enqueue_one_cycle(sale_ctx* c, int b, bool first)
{
    int rc;
    sale::Stream st = (sale::Stream)c->stream;
    const bool euler = c->prm.rezone == SALE_EULER;
    const bool ov = overlap_on(c);
    if (ov && (rc = overlap_resources(c))) return rc;
    const bool peer = c->prm.halo == SALE_HALO_PEER;
    int pr;
    if (peer && c->peer_sides) {  // ranks: the neighbours' planes of the previous cycle landed
        pr = prof_open(c, SALE_K_HALO);
        c->launches += sale::launch_halo_wait(c->dstate, first ? 1 : 0, c->peer_sides, st);
        prof_close(c, pr);
    }
    pr = prof_open(c, SALE_K_LAGRANGE);
    for (auto& s : c->slabs) c->launches += sale::launch_state(s, c->phys, b, first ? 0 : 1, st);
    prof_close(c, pr);
    pr = prof_open(c, SALE_K_HALO);
    if ((rc = reduce_keys(c))) return rc;
    prof_close(c, pr);
    pr = prof_open(c, SALE_K_BEGIN);
    c->launches += sale::launch_begin(c->dstate, c->phys, st);
    prof_close(c, pr);
    for (auto& s : c->slabs) {
        pr = prof_open(c, SALE_K_LAGRANGE);
        c->launches += sale::launch_force(s, c->phys, b, st);
        if (euler || !ov) c->launches += sale::launch_energy(s, c->phys, b, st);
        else c->launches += launch_tail(c, s, b, 0, st);
        prof_close(c, pr);
        if (euler) {
            pr = prof_open(c, SALE_K_REMAP);
            const int nodes = ov ? 0 : 1;
            c->launches += c->prm.nmat ? sale::launch_remap_mat(s, c->phys, b, st, nodes)
                                       : sale::launch_remap(s, c->phys, b, st, nodes);
            if (ov) c->launches += launch_tail(c, s, b, 0, st);
            prof_close(c, pr);
        }
    }
    if ((rc = launch_check(c))) return rc;
    if (!ov && peer) {  // the producers stored the ghost planes; ranks: signal the neighbours
        if (c->peer_sides) {
            pr = prof_open(c, SALE_K_HALO);
            c->launches += sale::launch_halo_signal(c->dstate, c->hp_dev[0], st);
            prof_close(c, pr);
        }
        return launch_check(c);
    }
    if (!ov) {
        pr = prof_open(c, SALE_K_HALO);
        if ((rc = exchange(c, b ^ 1, false))) return rc;
        prof_close(c, pr);
        return launch_check(c);
    }
    if ((rc = cuda_check(c, cudaEventRecord(c->evB, c->stream), "event record"))) return rc;
    if ((rc = cuda_check(c, cudaStreamWaitEvent(c->side, c->evB, 0), "stream wait"))) return rc;
    if ((rc = exchange(c, b ^ 1, false, c->side))) return rc;
    if ((rc = cuda_check(c, cudaEventRecord(c->evX, c->side), "event record"))) return rc;
    pr = prof_open(c, euler ? SALE_K_REMAP : SALE_K_LAGRANGE);
    for (auto& s : c->slabs) c->launches += launch_tail(c, s, b, 1, st);
    prof_close(c, pr);
    if ((rc = launch_check(c))) return rc;
    return cuda_check(c, cudaStreamWaitEvent(c->stream, c->evX, 0), "stream wait");
}

// CUDA graph of two consecutive cycles starting from buffer parity b (they return to
// b), captured once per context and parity, then replayed: a cycle is 4-8 kernel
// launches plus copies, which dominate small meshes.  The NCCL send/recv group and
// the allreduce of a multi-rank cycle are captured with the kernels (NCCL >= 2.9
// supports stream capture).  Never while profiling; SALE_GRAPHS=0 disables them.
bool graphs_enabled(const sale_ctx* c)
{
    static const int on = [] {
        const char* v = getenv("SALE_GRAPHS");
        return v ? atoi(v) : 1;
    }();
    return on && !c->prof_on;
}

int graph_for(sale_ctx* c, int b, cudaGraphExec_t* out)
{
    if (c->gexec[b]) {
        *out = c->gexec[b];
        return SALE_OK;
    }
    const long long before = c->launches;
    cudaGraph_t g = nullptr;
    // capture on a private stream (the caller's may be the legacy default stream,
    // which cannot capture); the graph is then launched on the caller's stream
    int rc = SALE_OK;
    if (!c->cap_stream)
        rc = cuda_check(c, cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking), "capture stream");
    if (rc) return rc;
    cudaStream_t user = c->stream;
    c->stream = c->cap_stream;
    rc = cuda_check(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), "graph capture");
    if (rc) {
        c->stream = user;
        return rc;
    }
    int rc1 = enqueue_one_cycle(c, b, false);
    if (!rc1) rc1 = enqueue_one_cycle(c, b ^ 1, false);
    rc = cuda_check(c, cudaStreamEndCapture(c->stream, &g), "graph capture end");
    c->stream = user;
    if (rc1 || rc) {
        if (g) cudaGraphDestroy(g);
        c->launches = before;
        return rc1 ? rc1 : rc;
    }
    rc = cuda_check(c, cudaGraphInstantiate(&c->gexec[b], g, 0), "graph instantiate");
    cudaGraphDestroy(g);
    c->glaunches[b] = c->launches - before;
    c->launches = before;
    if (rc) return rc;
    *out = c->gexec[b];
    return SALE_OK;
}

int enqueue_cycles(sale_ctx* c, int ncycles)
{
    int rc;
    int b = c->cur_enq;
    sale::Stream st = (sale::Stream)c->stream;
    // prologue: the ghost planes of the current state (set_field / resume honoured);
    // each cycle's state pass then forms the cell state and the dt candidate
    int pr = prof_open(c, SALE_K_PROLOGUE);
    c->launches += sale::launch_prep(c->dstate, st);
    if ((rc = exchange(c, b, true))) return rc;
    prof_close(c, pr);
    int n = 0;
    if (ncycles > 0) {  // the first cycle on the plain path (ungated state pass)
        if ((rc = enqueue_one_cycle(c, b, true))) return rc;
        b ^= 1;
        n = 1;
    }
    if (graphs_enabled(c) && ncycles - n >= 2) {
        cudaGraphExec_t ge = nullptr;
        if ((rc = graph_for(c, b, &ge))) return rc;
        for (; n + 2 <= ncycles; n += 2) {
            if ((rc = cuda_check(c, cudaGraphLaunch(ge, c->stream), "graph launch"))) return rc;
            c->launches += c->glaunches[b];
        }
    }
    for (; n < ncycles; ++n) {
        if ((rc = enqueue_one_cycle(c, b, false))) return rc;
        b ^= 1;
    }
    if (ncycles > 0 && (rc = reduce_keys(c))) return rc;  // the last cycle's error key
    c->launches += sale::launch_commit(c->dstate, c->phys, (sale::Stream)c->stream);
    c->cur_enq = b;
    return launch_check(c);
}

// synchronise, read the device state, fix the parity from the committed cycles
int sync_state(sale_ctx* c, int* good_out)
{
    int rc = cuda_check(c, cudaMemcpyAsync(c->hstate, c->dstate, sizeof(DevState), cudaMemcpyDeviceToHost,
                                           c->stream),
                        "state read");
    if (rc) return rc;
    if ((rc = cuda_check(c, cudaStreamSynchronize(c->stream), "stream sync"))) return rc;
    prof_collect(c);
    if (c->comm) {
        ncclResult_t ar;
        if (ncclCommGetAsyncError(c->comm, &ar) == ncclSuccess && ar != ncclSuccess)
            return nccl_check(c, ar, "async");
    }
    int good = c->hstate->good;
    c->cur = (c->cur + good) & 1;
    c->cur_enq = c->cur;
    if (good_out) *good_out = good;
    if (good) {
        c->launches += sale::launch_reset_good(c->dstate, (sale::Stream)c->stream);
        c->hstate->good = 0;
    }
    int st = c->hstate->status;
    if (st != SALE_OK && !c->poisoned) {
        char buf[160];
        long long cell = c->hstate->err_cell;
        if (cell >= 0) {
            long long nx = c->prm.nx, ny = c->prm.ny;
            std::snprintf(buf, sizeof buf, "cycle=%lld cell=%lld,%lld,%lld", c->hstate->err_cycle, cell % nx,
                          (cell / nx) % ny, cell / (nx * ny));
        } else {
            std::snprintf(buf, sizeof buf, "cycle=%lld", c->hstate->err_cycle);
        }
        set_err(c, st, buf);
    }
    return st;
}

bool is_node_field(int f) { return f >= SALE_F_X && f <= SALE_F_NODE_MASS; }
bool is_cell_field(int f) { return f >= SALE_F_MASS && f <= SALE_F_CS; }
bool is_cell_field(const sale_ctx* c, int f)
{
    int mat;
    return is_cell_field(f) || mat_kind(c->prm.nmat, f, &mat) >= 0;
}

uint64_t owned_count(const sale_ctx* c, const Slab& s, int field)
{
    return is_node_field(field) ? (uint64_t)s.pn * (uint64_t)(s.k1 - s.k0 + 1)
                                : (uint64_t)s.pc * (uint64_t)(s.k1 - s.k0);
}

uint64_t expected_count(const sale_ctx* c, int field)
{
    if (c->prm.local_slabs == 1) return owned_count(c, c->slabs[0], field);
    const Slab& s = c->slabs[0];
    return is_node_field(field) ? (uint64_t)s.pn * (uint64_t)(c->prm.nz + 1)
                                : (uint64_t)s.pc * (uint64_t)c->prm.nz;
}

// device pointer to the owned data of `field` of slab s (after deriving if needed)
const double* field_src(sale_ctx* c, const Slab& s, int field)
{
    int b = c->cur;
    bool euler = c->prm.rezone == SALE_EULER;
    size_t on = (size_t)(s.k0 - s.kb) * s.pn, oc = (size_t)(s.k0 - s.kb) * s.pc;
    switch (field) {
    case SALE_F_X:
    case SALE_F_Y:
    case SALE_F_Z:
        if (!euler) return s.x[b][field] + on;
        break;
    case SALE_F_UX:
    case SALE_F_UY:
    case SALE_F_UZ: return s.u[b][field - SALE_F_UX] + on;
    case SALE_F_MASS: return (euler ? s.m[b] : s.m[0]) + oc;
    case SALE_F_E:
        if (c->prm.nmat == 0) return s.e[b] + oc;
        break;  // the mixture's (sum_k m_k e_k) / m, derived
    default:
        if (double* a = mat_array(c, s, b, field)) return a + oc;
        break;
    }
    c->launches += sale::launch_derive(s, c->phys, b, field, (sale::Stream)c->stream);
    return s.der;
}


// Euler: read the target face-area tables back once and set Phys::diag_areas when
// every x-face area is (a, 0, 0), y-face (0, b, 0), z-face (0, 0, c) with a, b, c
// non-zero and the zeros exact (true for the tensor-product target mesh): the
// kernels then form corner vectors from the diagonal components only (same bits).
int check_diag_areas(sale_ctx* c)
{
    bool diag = true;
    std::vector<double> h;
    for (auto& s : c->slabs) {
        const long long n[3] = {(long long)c->phys.ny * s.nzc, (long long)c->phys.nx * s.nzc,
                                (long long)c->phys.nx * c->phys.ny};
        double* const* T[3] = {s.TAx, s.TAy, s.TAz};
        for (int f = 0; f < 3 && diag; ++f)
            for (int comp = 0; comp < 3 && diag; ++comp) {
                h.resize((size_t)n[f]);
                int rc = cuda_check(c, cudaMemcpy(h.data(), T[f][comp], sizeof(double) * (size_t)n[f],
                                                  cudaMemcpyDeviceToHost),
                                    "area tables");
                if (rc) return rc;
                for (double v : h)
                    if ((comp == f) ? !(v != 0.0) : v != 0.0) {
                        diag = false;
                        break;
                    }
            }
    }
    c->phys.diag_areas = diag ? 1 : 0;
    // axis-jump separations: d = (dx, 0, 0) on x, (0, dy, 0) on y, (0, 0, dz) on z
    bool dj = true;
    for (auto& s : c->slabs) {
        const long long n[3] = {c->phys.nx, c->phys.ny, s.nzc};
        const double* T[3] = {s.TJx, s.TJy, s.TJz};
        for (int a = 0; a < 3 && dj; ++a) {
            h.resize((size_t)(4 * n[a]));
            int rc = cuda_check(c, cudaMemcpy(h.data(), T[a], sizeof(double) * (size_t)(4 * n[a]), cudaMemcpyDeviceToHost),
                                "jump tables");
            if (rc) return rc;
            for (long long t = 0; t < n[a] && dj; ++t)
                for (int comp = 0; comp < 3; ++comp)
                    if (comp != a && h[(size_t)(4 * t + comp)] != 0.0) dj = false;
        }
    }
    c->phys.diag_jumps = dj ? 1 : 0;
    return SALE_OK;
}

}  // namespace

extern "C" {

uint64_t sale_workspace_bytes(const sale_params* p)
{
    if (!params_ok(p)) return 0;
    return (uint64_t)total_bytes(p);
}

int32_t sale_nccl_unique_id(void* id_out_128)
{
    if (!id_out_128) return SALE_EINVAL;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return SALE_ENCCL;
    std::memcpy(id_out_128, &id, sizeof id);
    return SALE_OK;
}

int32_t sale_create(const sale_params* p, sale_ctx** out)
{
    if (!out) return SALE_EINVAL;
    *out = nullptr;
    if (!params_ok(p)) return SALE_EINVAL;
    size_t need = total_bytes(p);
    if (!p->workspace || p->workspace_bytes < need || (reinterpret_cast<uintptr_t>(p->workspace) % ALIGN))
        return SALE_ENOMEM;
    DeviceGuard guard(p->device);
    sale_ctx* c = new sale_ctx();
    c->prm = *p;
    c->g = ghost_depth(p);
    c->stream = (cudaStream_t)p->stream;
    Phys& ph = c->phys;
    ph.lx = p->lx; ph.ly = p->ly; ph.lz = p->lz;
    ph.gamma = p->gamma; ph.c1 = p->q_lin; ph.c2 = p->q_quad; ph.cfl = p->cfl;
    ph.growth = p->dt_growth; ph.t_end = p->t_end;
    ph.rho0 = p->rho0; ph.e_bg = p->e_background; ph.e_dep = p->e_deposit;
    ph.hg = p->hg;
    ph.nx = p->nx; ph.ny = p->ny; ph.nz = p->nz;
    ph.reflect = p->reflect_mask; ph.rezone = p->rezone;
    layout_slabs(p, c->slabs);
    char* base = static_cast<char*>(p->workspace);
    c->dstate = reinterpret_cast<DevState*>(base);
    size_t off = align_up(sizeof(DevState));
    for (auto& s : c->slabs) {
        s.st = c->dstate;
        s.hp = nullptr;
        off += carve_slab(p, s, base + off);
    }
    if (p->halo == SALE_HALO_PEER)
        for (size_t l = 0; l < c->slabs.size(); ++l) {
            c->hp_dev.push_back(reinterpret_cast<sale::HaloPeer*>(base + off));
            off += align_up(sizeof(sale::HaloPeer));
        }
    int rc = cuda_check(c, cudaHostAlloc((void**)&c->hstate, sizeof(DevState), cudaHostAllocDefault),
                        "cudaHostAlloc");
    if (rc) {
        delete c;
        return rc;
    }
    std::memset(c->hstate, 0, sizeof(DevState));
    c->hstate->t = 0.0;
    c->hstate->dt_prev = -1.0;
    c->hstate->cand_key = sale::KEY_NONE;
    c->hstate->err_key = sale::KEY_NONE;
    c->hstate->err_cell = -1;
    if (p->nccl_unique_id) {
        ncclUniqueId id;
        std::memcpy(&id, p->nccl_unique_id, sizeof id);
        rc = nccl_check(c, ncclCommInitRank(&c->comm, p->nranks, id, p->rank), "ncclCommInitRank");
        if (rc) {
            cudaFreeHost(c->hstate);
            delete c;
            return rc;
        }
    }
    rc = cuda_check(c, cudaMemcpyAsync(c->dstate, c->hstate, sizeof(DevState), cudaMemcpyHostToDevice, c->stream),
                    "state init");
    if (!rc && p->halo == SALE_HALO_PEER) rc = peer_tables(c);
    for (auto& s : c->slabs) {
        if (rc) break;
        c->launches += sale::launch_init_tables(s, ph, (sale::Stream)c->stream);
        c->launches += sale::launch_sedov_init(s, ph, (sale::Stream)c->stream);
        if (s.nmat) c->launches += sale::launch_mat_init(s, ph, (sale::Stream)c->stream);
        if (ph.rezone) c->launches += sale::launch_target_tables(s, ph, (sale::Stream)c->stream);
        rc = launch_check(c);
    }
    if (!rc) rc = cuda_check(c, cudaStreamSynchronize(c->stream), "create sync");
    if (!rc && ph.rezone) rc = check_diag_areas(c);
    // the Euler kernels form corner vectors and axis jumps from the diagonal table
    // components (a tensor-product target mesh always has them)
    if (!rc && ph.rezone && !(ph.diag_areas && ph.diag_jumps))
        rc = set_err(c, SALE_EINVAL, "target mesh tables are not axis-aligned");
    if (rc) {
        for (auto m : c->ipc)
            if (m) cudaIpcCloseMemHandle(m);
        if (c->comm) ncclCommDestroy(c->comm);
        cudaFreeHost(c->hstate);
        delete c;
        return rc;
    }
    *out = c;
    return SALE_OK;
}

int32_t sale_step_async(sale_ctx* c, int32_t ncycles)
{
    if (!c || ncycles < 0) return SALE_EINVAL;
    if (c->poisoned) return SALE_EPOISONED;
    DeviceGuard guard(c->prm.device);
    return enqueue_cycles(c, ncycles);
}

int32_t sale_sync(sale_ctx* c, int32_t* cycles_done)
{
    if (cycles_done) *cycles_done = 0;
    if (!c) return SALE_EINVAL;
    DeviceGuard guard(c->prm.device);
    int good = 0;
    int rc = sync_state(c, &good);
    if (cycles_done) *cycles_done = good;
    return rc;
}

int32_t sale_step(sale_ctx* c, int32_t ncycles, int32_t* cycles_done)
{
    if (cycles_done) *cycles_done = 0;
    if (!c || ncycles < 0) return SALE_EINVAL;
    if (c->poisoned) return SALE_EPOISONED;
    DeviceGuard guard(c->prm.device);
    int rc = enqueue_cycles(c, ncycles);
    if (rc) return rc;
    return sale_sync(c, cycles_done);
}

int32_t sale_steinberg(sale_ctx* c, const sale_steinberg_params* sp, const double* eps_p, double* shear,
                       double* yield, uint64_t count)
{
    if (!c || !sp || !shear || !yield) return SALE_EINVAL;
    if (count != expected_count(c, SALE_F_MASS)) return SALE_EINVAL;
    if (c->poisoned) return SALE_EPOISONED;
    DeviceGuard guard(c->prm.device);
    int rc = sync_state(c, nullptr);
    if (rc) return rc;
    sale::SteinbergSet set{};
    set.n = c->prm.nmat > 0 ? c->prm.nmat : 1;
    for (int a = 0; a < set.n; ++a) {
        const sale_steinberg_params& q = sp[a];
        set.m[a] = sale::SteinbergP{q.G0, q.GP, q.GT, q.Y0, q.Ymax, q.beta, q.n, q.cv, q.rho0, q.T0};
    }
    const size_t plane = (size_t)c->slabs[0].pc;
    for (auto& s : c->slabs) {
        const size_t off = c->prm.local_slabs > 1 ? (size_t)s.k0 * plane : 0;
        c->launches += sale::launch_steinberg(s, c->phys, c->cur, set, eps_p ? eps_p + off : nullptr, shear + off,
                                              yield + off, (long long)count, (sale::Stream)c->stream);
    }
    return launch_check(c);
}

int32_t sale_get_field(sale_ctx* c, int32_t field, double* dst, uint64_t count, int32_t dst_on_device)
{
    if (!c || !dst || !(is_node_field(field) || is_cell_field(c, field))) return SALE_EINVAL;
    if (count != expected_count(c, field)) return SALE_EINVAL;
    DeviceGuard guard(c->prm.device);
    int rc = sync_state(c, nullptr);
    if (rc && rc != c->hstate->status) return rc;  // CUDA/NCCL failure; numerical status still readable
    cudaMemcpyKind kind = dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    bool node = is_node_field(field);
    size_t plane = node ? (size_t)c->slabs[0].pn : (size_t)c->slabs[0].pc;
    std::vector<double> rep_a, rep_b;
    for (size_t l = 0; l < c->slabs.size(); ++l) {
        const Slab& s = c->slabs[l];
        const double* src = field_src(c, s, field);
        size_t n = (size_t)owned_count(c, s, field);
        size_t dst_off = c->prm.local_slabs > 1 ? (size_t)s.k0 * plane : 0;
        if (node && l > 0) {
            // replicated interface plane k0: compare with what the lower slab wrote
            rep_a.resize(plane);
            rep_b.resize(plane);
            rc = cuda_check(c, cudaMemcpyAsync(rep_b.data(), src, plane * sizeof(double), cudaMemcpyDeviceToHost,
                                               c->stream),
                            "replica read");
            if (rc) return rc;
            rc = cuda_check(c, cudaMemcpyAsync(rep_a.data(), dst + dst_off, plane * sizeof(double),
                                               dst_on_device ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost,
                                               c->stream),
                            "replica read");
            if (rc) return rc;
            if ((rc = cuda_check(c, cudaStreamSynchronize(c->stream), "replica sync"))) return rc;
            if (std::memcmp(rep_a.data(), rep_b.data(), plane * sizeof(double)) != 0) {
                c->err = "EREPLICA: interface node plane differs between slabs";
                return SALE_EREPLICA;
            }
        }
        rc = cuda_check(c, cudaMemcpyAsync(dst + dst_off, src, n * sizeof(double), kind, c->stream), "field copy");
        if (rc) return rc;
        // der is reused per slab: finish this copy before the next derive
        if ((rc = cuda_check(c, cudaStreamSynchronize(c->stream), "field sync"))) return rc;
    }
    return SALE_OK;
}

int32_t sale_set_field(sale_ctx* c, int32_t field, const double* src, uint64_t count, int32_t src_on_device)
{
    if (!c || !src) return SALE_EINVAL;
    if (c->poisoned) return SALE_EPOISONED;
    bool euler = c->prm.rezone == SALE_EULER;
    int mat;
    const bool matf = mat_kind(c->prm.nmat, field, &mat) >= 0;
    bool ok = (field >= SALE_F_UX && field <= SALE_F_UZ) ||
              (c->prm.nmat == 0 && (field == SALE_F_MASS || field == SALE_F_E)) || matf ||
              (!euler && field >= SALE_F_X && field <= SALE_F_Z);
    if (!ok || count != expected_count(c, field)) return SALE_EINVAL;
    DeviceGuard guard(c->prm.device);
    int rc = sync_state(c, nullptr);
    if (rc) return rc;
    bool node = is_node_field(field);
    size_t plane = node ? (size_t)c->slabs[0].pn : (size_t)c->slabs[0].pc;
    int b = c->cur;
    cudaMemcpyKind kind = src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    for (auto& s : c->slabs) {
        double* arr;
        if (matf) arr = mat_array(c, s, b, field);
        else if (field <= SALE_F_Z) arr = s.x[b][field];
        else if (field <= SALE_F_UZ) arr = s.u[b][field - SALE_F_UX];
        else if (field == SALE_F_MASS) arr = euler ? s.m[b] : s.m[0];
        else arr = s.e[b];
        size_t off = (size_t)(s.k0 - s.kb) * plane;
        size_t src_off = c->prm.local_slabs > 1 ? (size_t)s.k0 * plane : 0;
        size_t n = (size_t)owned_count(c, s, field);
        rc = cuda_check(c, cudaMemcpyAsync(arr + off, src + src_off, n * sizeof(double), kind, c->stream),
                        "set_field copy");
        if (rc) return rc;
        // the cell mass is the sum of the material masses (MM0)
        if (matf && field >= SALE_F_MAT_M(0) && field < SALE_F_MAT_E(0))
            c->launches += sale::launch_mat_total(s, c->phys, b, (sale::Stream)c->stream);
    }
    return cuda_check(c, cudaStreamSynchronize(c->stream), "set_field sync");
}

int32_t sale_get_clock(sale_ctx* c, double* t, double* dt_last, int64_t* cycle, int32_t* finished)
{
    if (!c) return SALE_EINVAL;
    DeviceGuard guard(c->prm.device);
    int rc = sync_state(c, nullptr);
    if (rc && rc != c->hstate->status) return rc;
    if (t) *t = c->hstate->t;
    if (dt_last) *dt_last = c->hstate->dt_prev;
    if (cycle) *cycle = c->hstate->cycle;
    if (finished) *finished = (c->prm.t_end > 0.0 && c->hstate->t >= c->prm.t_end) ? 1 : 0;
    return SALE_OK;
}

int32_t sale_set_clock(sale_ctx* c, double t, double dt_last, int64_t cycle)
{
    if (!c || cycle < 0) return SALE_EINVAL;
    if (c->poisoned) return SALE_EPOISONED;
    DeviceGuard guard(c->prm.device);
    int rc = sync_state(c, nullptr);
    if (rc) return rc;
    c->hstate->t = t;
    c->hstate->dt_prev = dt_last;
    c->hstate->cycle = cycle;
    c->hstate->finished = (c->prm.t_end > 0.0 && t >= c->prm.t_end) ? 1 : 0;
    // (the clock and status only: the peer-store halo counters stay the device's)
    rc = cuda_check(c, cudaMemcpyAsync(c->dstate, c->hstate, offsetof(DevState, halo_in), cudaMemcpyHostToDevice,
                                       c->stream),
                    "set_clock");
    if (rc) return rc;
    return cuda_check(c, cudaStreamSynchronize(c->stream), "set_clock sync");
}

int32_t sale_get_layout(sale_ctx* c, int32_t* k0, int32_t* k1)
{
    if (!c) return SALE_EINVAL;
    if (k0) *k0 = c->slabs.front().k0;
    if (k1) *k1 = c->slabs.back().k1;
    return SALE_OK;
}

int64_t sale_kernel_launches(const sale_ctx* c) { return c ? c->launches : 0; }

int32_t sale_halo_plan(const sale_params* p, int32_t full, sale_halo_msg* out, int32_t cap)
{
    if (!params_ok_layout(p)) return -1;
    std::vector<sale_halo_msg> plan;
    build_plan(p, full, plan);
    int32_t n = (int32_t)plan.size();
    for (int32_t k = 0; k < n && k < cap && out; ++k) out[k] = plan[k];
    return n;
}

int32_t sale_local_layout(const sale_params* p, int32_t* k0, int32_t* k1, int32_t* ghost, int32_t* node_planes,
                          int32_t* cell_planes)
{
    if (!params_ok_layout(p)) return SALE_EINVAL;
    std::vector<Slab> v;
    layout_slabs(p, v);
    if (k0) *k0 = v.front().k0;
    if (k1) *k1 = v.back().k1;
    if (ghost) *ghost = v[0].g;
    if (node_planes) *node_planes = v[0].nzn;
    if (cell_planes) *cell_planes = v[0].nzc;
    return SALE_OK;
}

int32_t sale_profile_enable(sale_ctx* c, int32_t on)
{
    if (!c) return SALE_EINVAL;
    c->prof_on = on != 0;
    if (c->prof_on)
        for (int k = 0; k < SALE_K_NCLASS; ++k) {
            c->prof_ms[k] = 0.0;
            c->prof_cnt[k] = 0;
        }
    return SALE_OK;
}

int32_t sale_profile_read(sale_ctx* c, int32_t kclass, double* total_ms, int64_t* count)
{
    if (!c || kclass < 0 || kclass >= SALE_K_NCLASS) return SALE_EINVAL;
    if (total_ms) *total_ms = c->prof_ms[kclass];
    if (count) *count = c->prof_cnt[kclass];
    return SALE_OK;
}

const char* sale_last_error(const sale_ctx* c) { return c ? c->err.c_str() : "null context"; }

void sale_destroy(sale_ctx* c)
{
    if (!c) return;
    DeviceGuard guard(c->prm.device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (auto m : c->ipc)
        if (m) cudaIpcCloseMemHandle(m);
    if (c->comm) ncclCommDestroy(c->comm);
    if (c->hstate) cudaFreeHost(c->hstate);
    for (auto& p : c->pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    for (auto ge : c->gexec)
        if (ge) cudaGraphExecDestroy(ge);
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->evB) cudaEventDestroy(c->evB);
    if (c->evX) cudaEventDestroy(c->evX);
    delete c;
}

}  // extern "C"
