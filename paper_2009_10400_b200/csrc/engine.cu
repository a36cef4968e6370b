// engine.cu — the device engine behind the C ABI of include/tvegpu.h.
//
// Replaces tve::Engine (engine.hpp:83-143).  The constructor's work
// (engine.hpp:85-87) plus precompute() (mesh.hpp:81-83) happens once in
// tvegpu_create: validation, the compressed precompute, Morton/first-touch
// reordering and (nranks > 1) the RCB partition run on the host (plan.cpp),
// then everything is uploaded and stays resident in HBM.  Engine::step()
// (engine.hpp:89-90) becomes K1..K5 on one stream, replayed as CUDA graphs of
// `steps_per_graph` steps; time, step counter, BC ramps and the finite check
// live on the device so a graph replay needs no host work.  The only per-call
// host work is the regional-source refresh when the active-source mask changes
// (engine.hpp:119, 140), predicted from the same fp64 time sequence.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include "kernels.cuh"
#include "plan.hpp"

using namespace tvegpu;

namespace {

thread_local std::string g_create_error;

#define CU(x)                                                                                      \
    do {                                                                                           \
        cudaError_t _e = (x);                                                                      \
        if (_e != cudaSuccess)                                                                     \
            throw Error(TVEGPU_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e));           \
    } while (0)

// ---------------------------------------------------------------- NCCL, loaded lazily (multi-GPU only)
struct NcclApi {
    void* lib = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    if (!api.lib) {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) throw Error(TVEGPU_E_NCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
        auto sym = [&](const char* n) {
            void* p = dlsym(h, n);
            if (!p) throw Error(TVEGPU_E_NCCL, std::string("libnccl.so.2 lacks ") + n);
            return p;
        };
        api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
        api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
        api.Send = (decltype(api.Send))sym("ncclSend");
        api.Recv = (decltype(api.Recv))sym("ncclRecv");
        api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
        api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
        api.lib = h;
    }
    return api;
}

#define NC(x)                                                                                      \
    do {                                                                                           \
        ncclResult_t _r = (x);                                                                     \
        if (_r != ncclSuccess) throw Error(TVEGPU_E_NCCL, std::string(#x) + ": " + nccl().GetErrorString(_r)); \
    } while (0)

template <class T>
T* dalloc(std::vector<void*>& owned, size_t n) {
    if (n == 0) n = 1;
    void* p = nullptr;
    CU(cudaMalloc(&p, n * sizeof(T)));
    owned.push_back(p);
    return static_cast<T*>(p);
}
// Host -> device upload of setup arrays.  A pageable cudaMemcpy is staged by the driver
// through a single-threaded copy (~6 GB/s); large arrays instead go through a
// process-wide double-buffered pinned ring (2 x 32 MB, allocated once): the host threads
// fill one buffer (parallel memcpy) while the other is in flight at link speed.
// Returns after the source may be reused (like a pageable cudaMemcpyAsync).
void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    constexpr size_t kSmall = (size_t)4 << 20, kBuf = (size_t)32 << 20;
    if (bytes <= kSmall) {
        CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    static std::mutex mu;
    static char* buf[2] = {nullptr, nullptr};
    static cudaEvent_t done[2] = {nullptr, nullptr};
    std::lock_guard<std::mutex> lock(mu);
    if (!buf[0])
        for (int k = 0; k < 2; ++k) {
            CU(cudaMallocHost(&buf[k], kBuf));
            CU(cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming));
            CU(cudaEventRecord(done[k], s));
        }
    const char* in = static_cast<const char*>(src);
    char* out = static_cast<char*>(dst);
    int k = 0;
    for (size_t off = 0; off < bytes; off += kBuf, k ^= 1) {
        const size_t n = std::min(kBuf, bytes - off);
        CU(cudaEventSynchronize(done[k]));  // this buffer's previous copy has left
        const int pieces = (int)((n + ((size_t)1 << 20) - 1) >> 20);
#pragma omp parallel for schedule(static)
        for (int q = 0; q < pieces; ++q) {
            const size_t a = (size_t)q << 20, b = std::min(n, a + ((size_t)1 << 20));
            std::memcpy(buf[k] + a, in + off + a, b - a);
        }
        CU(cudaMemcpyAsync(out + off, buf[k], n, cudaMemcpyHostToDevice, s));
        CU(cudaEventRecord(done[k], s));
    }
}

template <class T, class Al>
T* dupload(std::vector<void*>& owned, const std::vector<T, Al>& v, cudaStream_t s) {
    T* p = dalloc<T>(owned, v.size());
    if (!v.empty()) h2d(p, v.data(), v.size() * sizeof(T), s);
    return p;
}

// Temporary device buffers of one setup stage, freed on scope exit (the caller
// synchronises the stream first).
struct DeviceScratch {
    std::vector<void*> p;
    template <class T>
    T* get(size_t n) {
        void* q = nullptr;
        CU(cudaMalloc(&q, std::max<size_t>(1, n) * sizeof(T)));
        p.push_back(q);
        return static_cast<T*>(q);
    }
    ~DeviceScratch() {
        for (void* q : p) cudaFree(q);
    }
};

// Setup kernels: node records / coordinates / lumped constants in local order from the
// original-order inputs; the chunks' fixed-stride staging entries; the chunks'
// coordinate blocks in shared-slot order.
__global__ void k_init_nodes(const int32_t* __restrict__ node_orig, const double* __restrict__ xyz,
                             const double* __restrict__ mass_o, const double* __restrict__ vn_o, double T0, int N,
                             double4* rec0, double4* rec1, double4* X, double* mass, double* vn) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const size_t o = (size_t)node_orig[i];
    rec0[i] = rec1[i] = make_double4(0.0, 0.0, 0.0, T0);
    X[i] = make_double4(xyz[3 * o], xyz[3 * o + 1], xyz[3 * o + 2], 0.0);
    mass[i] = mass_o[o];
    vn[i] = vn_o[o];
}
// out[c] = 1 iff flag[e] for every element e of chunk c
__global__ void k_chunk_all(const int32_t* __restrict__ chunk_start, const uint8_t* __restrict__ flag,
                            uint8_t* __restrict__ out) {
    const int c = blockIdx.x;
    int ok = 1;
    for (int e = chunk_start[c] + threadIdx.x; e < chunk_start[c + 1]; e += blockDim.x) ok &= flag[e];
    ok = __syncthreads_and(ok);
    if (threadIdx.x == 0) out[c] = (uint8_t)ok;
}
__global__ void k_stage_entries(const int32_t* __restrict__ off, const int32_t* __restrict__ nodes,
                                const uint16_t* __restrict__ slot, int st, int2* __restrict__ ent) {
    const int c = blockIdx.x;
    const int u0 = off[c], u1 = off[c + 1];
    for (int k = threadIdx.x; k < st; k += blockDim.x) {
        const int u = u0 + k;
        ent[(size_t)c * st + k] = u < u1 ? make_int2(nodes[u], (int)slot[u]) : make_int2(-1, 0);
    }
}
__global__ void k_chunk_coords(const int32_t* __restrict__ off, const int32_t* __restrict__ nodes,
                               const uint16_t* __restrict__ slot, const int32_t* __restrict__ xs,
                               const double4* __restrict__ X, int xstride, double* __restrict__ cx) {
    const int c = blockIdx.x;
    const int S = xs[c];
    double* b = cx + (size_t)c * xstride;
    for (int u = off[c] + threadIdx.x; u < off[c + 1]; u += blockDim.x) {
        const double4 x = X[nodes[u]];
        const int sl = slot[u];
        b[sl] = x.x;
        b[S + sl] = x.y;
        b[2 * S + sl] = x.z;
    }
}

struct Region {
    double q_r, t_start, t_end;
    std::vector<int32_t> nodes;  // nn per element, original ids
    std::vector<double> vol;
    bool active_at(double t) const { return t >= t_start && t < t_end; }
};

}  // namespace

namespace tvegpu {
void set_create_error(const std::string& m) { g_create_error = m; }
}  // namespace tvegpu

namespace {
// Halo transport between the partitions of one step.  The step code
// (enqueue_partitioned_step) is the same for every transport: boundary elements,
// pack + ev_pack on the compute stream, exchange() on the comm streams ending in
// ev_comm, interior elements, node kernel after ev_comm.
//   NcclTransport      one partition per process and GPU: grouped ncclSend/ncclRecv.
//   LoopbackTransport  all partitions in this process on one device (tvegpu_group):
//                      device copies of each neighbour's packed segment, ordered by
//                      the same events — so only the two NCCL calls differ.
struct Transport {
    virtual ~Transport() = default;
    // Called once every part has packed its send segment of this phase and recorded
    // ev_pack on its compute stream; fills each part's receive area on its comm stream
    // and records ev_comm there.
    // t0 (profiling, may be null): recorded on parts[0]'s comm stream once the transfer may start.
    virtual void exchange(const std::vector<tvegpu_engine*>& parts, bool mech, cudaEvent_t t0 = nullptr) = 0;
    // In-place element-wise all-reduce (max or min) of n unsigned 64-bit words,
    // buf[k] on parts[k], ordered after each part's compute stream; on return the
    // result is enqueued on (and complete before later work of) every compute stream.
    virtual void allreduce_u64(const std::vector<tvegpu_engine*>& parts, const std::vector<unsigned long long*>& buf,
                               size_t n, bool max) = 0;
};

// The partitions one process steps together, and their CUDA-graph cache: a single
// engine is a one-part set; tvegpu_group holds all partitions of a mesh.
struct Stepper {
    std::vector<tvegpu_engine*> parts;
    std::map<std::pair<int, int>, cudaGraphExec_t> graphs;  // (parity, nsteps)
    int steps_per_graph = 64;
    bool warmed = false;  // a plain (un-captured) step has run
    cudaEvent_t ev_fork = nullptr;  // multi-part sets: origin stream -> part streams
};
}  // namespace

struct tvegpu_engine {
    int device = 0, nn = 4, kind = 0, mode = 0, N_global = 0, E_global = 0, P = 0;
    double dt = 0;
    RankPlan plan;
    DevParams prm{};
    DevPtrs ptr{};
    std::vector<void*> owned;
    cudaStream_t s = nullptr, sc = nullptr;
    cudaEvent_t ev_pack = nullptr, ev_comm = nullptr;
    cudaEvent_t ev_src = nullptr, ev_T = nullptr;  // tvegpu_step_io: sources landed / T final
    double* d_pw = nullptr;                        // tvegpu_step_io: uploaded source powers
    int cur = 0;
    double host_time = 0;
    long long host_step = 0;
    bool halted = false;
    // sources
    std::vector<Region> regions;
    std::vector<char> active;
    bool sources_init = false, source_override = false;
    double* qr_host = nullptr;  // pinned staging of the nodal source vector (local order)
    // multi-GPU
    ncclComm_t comm = nullptr;
    Transport* tx = nullptr;                // halo transport (nranks > 1): own NCCL one or the group's loopback
    std::unique_ptr<Transport> own_tx;
    double* send_th = nullptr;
    double* send_m = nullptr;
    const int32_t* d_send_slot = nullptr;  // element-major slot ids of the send lists
    cudaEvent_t ev_join = nullptr;          // multi-part sets: part stream -> origin stream
    Stepper solo;                           // this engine as a one-part step set (graph cache)
    bool pdl = false;     // programmatic dependent launch of the step kernels (single partition)
    bool pair = false;    // node kernels with two threads per node (long CSR gather lists: T4)
    int n_affine_chunks = 0;  // H8 chunks whose elements are all affine (K3 skips their c_al rows)
    bool slot32 = false;      // tvegpu_options.slot_fp32: contributions stored as fp32, summed in fp64
    size_t slot_bytes() const { return slot32 ? sizeof(float) : sizeof(double); }
    // peer-memory halo (kernels.cuh peer_send / peer_signal / peer_wait)
    int halo_transport = TVEGPU_HALO_PEER;  // tvegpu_options.halo_transport
    bool peer = false;                      // attached: the boundary element kernels deliver the halo
    std::vector<void*> ipc_open;            // neighbours' allocations mapped by cudaIpcOpenMemHandle
    // errors
    std::string err;
    long long err_step = -1;
    int err_node = -1;
    tvegpu_status last_status = TVEGPU_OK;
    // a failure in a partitioned step leaves the partitions at different steps (the
    // failing one halts, the others ran on with stale halo values): the state is
    // unusable until set_state / load_checkpoint (every partition reports the same error)
    bool state_invalid = false;
    bool pending = false;  // steps enqueued whose finite check has not been read back
    long long pend_step = 0;
    int pend_cur = 0;
    double pend_time = 0;
    cudaEvent_t ev_entry = nullptr;  // tvegpu_step_io: work already on s before the side-stream upload
    // tvegpu_step_io read-back slices: K4 of the last step runs over local nodes
    // [io_cut[k], io_cut[k+1]); once slice k is done every node of original id < io_done[k]
    // is final, so u[io_done[k-1], io_done[k]) is copied while the next slices compute
    std::vector<int> io_cut, io_done;
    std::vector<cudaEvent_t> ev_u;
    unsigned long long* h_words = nullptr;  // pinned: clock (3 words) + err_inst + err_elem
    double4* stage = nullptr;               // pinned readback staging (N records)
    double* d_io = nullptr;                 // device I/O buffer in original numbering (4N doubles)
    int32_t* d_conn = nullptr;              // local connectivity (run-level outputs only, lazily)
    double* d_part = nullptr;               // per-block partials of the run-level reductions
    double* h_part = nullptr;               // pinned: reduced run-level outputs
    double* d_ef = nullptr;                 // element fields in original order (2E, lazily)
    const uint8_t* d_owned = nullptr;       // plan.node_owned on the device (state gathers, lazily)
    // MechBCs::motion_override (mechanics.hpp:43-46): a host callback, so a slow path —
    // per step the host evaluates it at t + dt for the candidate nodes into pinned
    // memory, uploads it and K4 applies the pins last (no graph replay while active)
    tvegpu_motion_fn motion_fn = nullptr;
    void* motion_user = nullptr;
    std::vector<int32_t> motion_orig;       // candidate rows: original node ids
    double4* motion_host = nullptr;         // pinned [rows]
};

namespace {

int blocks(int n, int t) { return (n + t - 1) / t; }

// NVTX range per C-ABI call (header-only NVTX 3: free unless a tool attaches), so
// ncu --nvtx / Nsight timelines show which API call enqueued which kernels.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
#define TVEGPU_RANGE() NvtxRange nvtx_range_(__func__)

void refresh_sources_if_needed(tvegpu_engine* h, double t) {
    if (h->source_override) return;
    bool changed = !h->sources_init;
    for (size_t r = 0; r < h->regions.size(); ++r) {
        const char a = h->regions[r].active_at(t) ? 1 : 0;
        if (a != h->active[r]) changed = true;
        h->active[r] = a;
    }
    h->sources_init = true;
    if (!changed) return;
    // accumulate_nodal_sources (bioheat.hpp:65-69): region order, element order, local order
    std::vector<double> q(h->N_global, 0.0);
    for (size_t r = 0; r < h->regions.size(); ++r) {
        if (!h->active[r]) continue;
        const Region& g = h->regions[r];
        for (size_t e = 0; e < g.vol.size(); ++e)
            for (int a = 0; a < h->nn; ++a) q[g.nodes[e * h->nn + a]] += g.q_r * g.vol[e] / h->nn;
    }
#pragma omp parallel for schedule(static)
    for (int li = 0; li < h->plan.N; ++li) h->qr_host[li] = q[h->plan.node_orig[li]];
    CU(cudaMemcpyAsync(const_cast<double*>(h->ptr.qr), h->qr_host, (size_t)h->plan.N * 8,
                       cudaMemcpyHostToDevice, h->s));
    CU(cudaStreamSynchronize(h->s));  // qr_host is reused
}

bool sources_stable(tvegpu_engine* h, double t) {
    if (h->source_override) return true;
    for (size_t r = 0; r < h->regions.size(); ++r)
        if ((h->regions[r].active_at(t) ? 1 : 0) != h->active[r]) return false;
    return true;
}

// ---------------------------------------------------------------- halo transports
// Halo exchange of interface contributions: each part packs its
// boundary elements' contributions (k_pack) on the compute stream and records
// ev_pack; the transport delivers every part's receive area (appended to its slot
// buffer; the gather lists index it) on the comm stream and records ev_comm; the
// interior elements run meanwhile and the node kernel waits on ev_comm.
void pack_halo(tvegpu_engine* h, bool mech) {
    const int ns = h->plan.send_off.back();
    double* slots = mech ? h->ptr.slot_m : h->ptr.slot_th;
    double* out = mech ? h->send_m : h->send_th;
    if (ns > 0 && h->slot32)
        k_pack<float><<<blocks(ns, 256), 256, 0, h->s>>>(reinterpret_cast<const float*>(slots), h->d_send_slot, ns,
                                                         mech ? kMW : 1, reinterpret_cast<float*>(out));
    else if (ns > 0)
        k_pack<double><<<blocks(ns, 256), 256, 0, h->s>>>(slots, h->d_send_slot, ns, mech ? kMW : 1, out);
    CU(cudaEventRecord(h->ev_pack, h->s));
}

// element offset in the slot buffer's own type (fp64 or fp32 slots) -> pointer
double* slot_ptr(const tvegpu_engine* h, bool mech, size_t entries) {
    const int width = mech ? kMW : 1;
    return reinterpret_cast<double*>(reinterpret_cast<char*>(mech ? h->ptr.slot_m : h->ptr.slot_th) +
                                     entries * width * h->slot_bytes());
}
double* recv_area(tvegpu_engine* h, bool mech) { return slot_ptr(h, mech, (size_t)h->plan.E * h->plan.nn); }
// entries of a packed send buffer
const double* send_ptr(const tvegpu_engine* h, bool mech, size_t entries) {
    const int width = mech ? kMW : 1;
    return reinterpret_cast<const double*>(reinterpret_cast<const char*>(mech ? h->send_m : h->send_th) +
                                           entries * width * h->slot_bytes());
}

struct NcclTransport final : Transport {
    ncclComm_t comm = nullptr;
    void exchange(const std::vector<tvegpu_engine*>& parts, bool mech, cudaEvent_t t0) override {
        tvegpu_engine* h = parts[0];  // one partition per process and GPU
        const RankPlan& pl = h->plan;
        const int width = mech ? kMW : 1;
        const ncclDataType_t type = h->slot32 ? ncclFloat32 : ncclFloat64;
        CU(cudaStreamWaitEvent(h->sc, h->ev_pack, 0));
        if (t0) CU(cudaEventRecord(t0, h->sc));
        auto& api = nccl();
        NC(api.GroupStart());
        for (size_t j = 0; j < pl.neighbors.size(); ++j) {
            const int peer = pl.neighbors[j];
            const size_t so = pl.send_off[j], sn = pl.send_off[j + 1] - so;
            const size_t ro = pl.recv_off[j], rn = pl.recv_off[j + 1] - ro;
            if (sn) NC(api.Send(send_ptr(h, mech, so), sn * width, type, peer, comm, h->sc));
            if (rn) NC(api.Recv(slot_ptr(h, mech, (size_t)pl.E * pl.nn + ro), rn * width, type, peer, comm, h->sc));
        }
        NC(api.GroupEnd());
        CU(cudaEventRecord(h->ev_comm, h->sc));
    }
    void allreduce_u64(const std::vector<tvegpu_engine*>& parts, const std::vector<unsigned long long*>& buf, size_t n,
                       bool max) override {
        tvegpu_engine* h = parts[0];
        NC(nccl().AllReduce(buf[0], buf[0], n, ncclUint64, max ? ncclMax : ncclMin, comm, h->s));
    }
};

__global__ void k_combine_u64(unsigned long long* __restrict__ acc, const unsigned long long* __restrict__ v, size_t n,
                              int max) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x)
        acc[k] = max ? (acc[k] > v[k] ? acc[k] : v[k]) : (acc[k] < v[k] ? acc[k] : v[k]);
}

struct LoopbackTransport final : Transport {
    void exchange(const std::vector<tvegpu_engine*>& parts, bool mech, cudaEvent_t t0) override {
        const int width = mech ? kMW : 1;
        for (tvegpu_engine* r : parts) {
            const RankPlan& pr = r->plan;
            // the receive area is rewritten only after this part's node kernel of the
            // previous step read it (ordered before r's own ev_pack)
            CU(cudaStreamWaitEvent(r->sc, r->ev_pack, 0));
            if (t0 && r == parts[0])
                for (const tvegpu_engine* q : parts) CU(cudaStreamWaitEvent(r->sc, q->ev_pack, 0));
            if (t0 && r == parts[0]) CU(cudaEventRecord(t0, r->sc));
            for (size_t j = 0; j < pr.neighbors.size(); ++j) {
                const tvegpu_engine* q = parts.at(pr.neighbors[j]);
                const RankPlan& ps = q->plan;
                const size_t jj = std::find(ps.neighbors.begin(), ps.neighbors.end(), pr.rank) - ps.neighbors.begin();
                if (jj == ps.neighbors.size()) throw Error(TVEGPU_E_ARG, "internal: asymmetric halo");
                const size_t n = (size_t)(ps.send_off[jj + 1] - ps.send_off[jj]);
                if (n != (size_t)(pr.recv_off[j + 1] - pr.recv_off[j])) throw Error(TVEGPU_E_ARG, "internal: halo size");
                if (!n) continue;
                CU(cudaStreamWaitEvent(r->sc, q->ev_pack, 0));  // the neighbour's packed segment (ncclRecv)
                CU(cudaMemcpyAsync(slot_ptr(r, mech, (size_t)pr.E * pr.nn + pr.recv_off[j]),
                                   send_ptr(q, mech, ps.send_off[jj]), n * width * r->slot_bytes(),
                                   cudaMemcpyDeviceToDevice, r->sc));
            }
            CU(cudaEventRecord(r->ev_comm, r->sc));
        }
    }
    void allreduce_u64(const std::vector<tvegpu_engine*>& parts, const std::vector<unsigned long long*>& buf, size_t n,
                       bool max) override {
        tvegpu_engine* h0 = parts[0];
        for (size_t k = 1; k < parts.size(); ++k) {
            CU(cudaEventRecord(parts[k]->ev_join, parts[k]->s));
            CU(cudaStreamWaitEvent(h0->s, parts[k]->ev_join, 0));
        }
        const int nb = (int)std::min<size_t>(1184, (n + 255) / 256);
        for (size_t k = 1; k < parts.size() && n; ++k)
            k_combine_u64<<<nb, 256, 0, h0->s>>>(buf[0], buf[k], n, max ? 1 : 0);
        for (size_t k = 1; k < parts.size() && n; ++k)
            CU(cudaMemcpyAsync(buf[k], buf[0], n * 8, cudaMemcpyDeviceToDevice, h0->s));
        CU(cudaGetLastError());
        CU(cudaEventRecord(h0->ev_join, h0->s));
        for (size_t k = 1; k < parts.size(); ++k) CU(cudaStreamWaitEvent(parts[k]->s, h0->ev_join, 0));
    }
};

// One partition stepped alone (tvegpu_peer_attach_solo: a measurement hook): no peers,
// no collective — the partition's own error words are the verdict.
struct SoloTransport final : Transport {
    void exchange(const std::vector<tvegpu_engine*>&, bool, cudaEvent_t) override {
        throw Error(TVEGPU_E_ARG, "partition without NCCL: attach the peer-memory halo first");
    }
    void allreduce_u64(const std::vector<tvegpu_engine*>&, const std::vector<unsigned long long*>&, size_t,
                       bool) override {}
};

// ---------------------------------------------------------------- peer-memory halo setup
// What a partition publishes to its neighbours: where its receive areas and inbox are
// (pointers valid in the attaching process) and its receive segments per neighbour.
struct PeerDesc {
    int rank = -1;
    double* th = nullptr;                    // thermal receive area
    double* m = nullptr;                     // mechanical receive area (kMW doubles per entry)
    unsigned long long* inbox = nullptr;     // per neighbour (its order) a flag word, then an ack word
    std::vector<int32_t> nbr, recv_off;      // its neighbour ranks; receive segment offsets (nbr + 1)
};

PeerDesc peer_desc(const tvegpu_engine* h) {
    PeerDesc d;
    d.rank = h->plan.rank;
    d.th = recv_area(const_cast<tvegpu_engine*>(h), false);
    d.m = recv_area(const_cast<tvegpu_engine*>(h), true);
    d.inbox = h->ptr.inbox;
    d.nbr = h->plan.neighbors;
    d.recv_off = h->plan.recv_off;
    return d;
}

// Builds this partition's destination table from its neighbours' descriptors: each
// send-list entry k of neighbour j (a boundary slot, canonical order) goes to index
// recv_off'[j'] + (k - send_off[j]) of that neighbour's receive area, j' = this
// partition's position in the neighbour's list — exactly where the NCCL transport's
// ncclRecv would have put it, so the gathers (and results) are unchanged.
void peer_attach(tvegpu_engine* h, const std::vector<PeerDesc>& by_rank) {
    const RankPlan& pl = h->plan;
    const int np = (int)pl.neighbors.size();
    if (np > 63) throw Error(TVEGPU_E_ARG, "peer-memory halo: more than 63 neighbouring partitions");
    const int nb = pl.Eb * pl.nn;
    std::vector<double*> pth(np), pm(np);
    std::vector<unsigned long long*> pf(np), pa(np);
    std::vector<int32_t> start(np), off((size_t)nb + 1, 0);
    for (int j = 0; j < np; ++j) {
        const int r = pl.neighbors[j];
        if (r < 0 || r >= (int)by_rank.size() || by_rank[r].rank != r)
            throw Error(TVEGPU_E_ARG, "peer-memory halo: no descriptor of partition " + std::to_string(r));
        const PeerDesc& d = by_rank[r];
        const auto it = std::find(d.nbr.begin(), d.nbr.end(), pl.rank);
        if (it == d.nbr.end()) throw Error(TVEGPU_E_ARG, "internal: asymmetric halo");
        const size_t jj = (size_t)(it - d.nbr.begin());
        if (d.recv_off.size() != d.nbr.size() + 1 ||
            d.recv_off[jj + 1] - d.recv_off[jj] != pl.send_off[j + 1] - pl.send_off[j])
            throw Error(TVEGPU_E_ARG, "internal: halo size");
        pth[j] = d.th;
        pm[j] = d.m;
        pf[j] = d.inbox + jj;
        pa[j] = d.inbox + d.nbr.size() + jj;
        start[j] = d.recv_off[jj];
        for (int k = pl.send_off[j]; k < pl.send_off[j + 1]; ++k) {
            const int32_t sl = pl.send_slot[k];
            if (sl < 0 || sl >= nb) throw Error(TVEGPU_E_ARG, "internal: send slot outside the boundary elements");
            off[(size_t)sl + 1]++;
        }
    }
    for (int k = 0; k < nb; ++k) off[(size_t)k + 1] += off[k];
    std::vector<uint32_t> ent(off[nb]);
    std::vector<int32_t> fill(off.begin(), off.end() - 1);
    for (int j = 0; j < np; ++j)
        for (int k = pl.send_off[j]; k < pl.send_off[j + 1]; ++k) {
            const int64_t dst = (int64_t)start[j] + (k - pl.send_off[j]);
            if (dst >= (1 << 26)) throw Error(TVEGPU_E_ARG, "peer-memory halo: receive area above 2^26 entries");
            ent[fill[pl.send_slot[k]]++] = (uint32_t)j << 26 | (uint32_t)dst;
        }
    cudaStream_t s = h->s;
    auto& own = h->owned;
    h->ptr.pd_off = dupload(own, off, s);
    h->ptr.pd_ent = dupload(own, ent, s);
    h->ptr.peer_th = dupload(own, pth, s);
    h->ptr.peer_m = dupload(own, pm, s);
    h->ptr.peer_flag = dupload(own, pf, s);
    h->ptr.peer_ack = dupload(own, pa, s);
    CU(cudaStreamSynchronize(s));
    h->prm.npeers = np;
    h->prm.ack = h->mode == TVEGPU_COUPLED ? 0 : 1;
    h->prm.nb_chunks = pl.nchunks_boundary;
    {  // nodes that gather received contributions: boundary elements' nodes, numbered first
        const int32_t local = pl.E * pl.nn;
        int hi = 0;
#pragma omp parallel for schedule(static) reduction(max : hi)
        for (int i = 0; i < pl.N; ++i)
            for (int k = pl.csr_off[i]; k < pl.csr_off[i + 1]; ++k)
                if (pl.csr_slot[k] >= local) hi = std::max(hi, i + 1);
        h->prm.halo_hi = hi;
    }
    // programmatic dependent launch between the step kernels, as for one partition: every
    // peer-path kernel waits for its predecessor grid before touching its outputs
    h->pdl = !std::getenv("TVEGPU_NO_PDL");
    for (auto& kv : h->solo.graphs) CU(cudaGraphExecDestroy(kv.second));
    h->solo.graphs.clear();
    {
        const char* t = std::getenv("TVEGPU_HALO_TIMEOUT_MS");
        const double ms = t ? std::atof(t) : 20000.0;
        h->prm.halo_timeout_ns = (unsigned long long)(std::max(1.0, ms) * 1e6);
        const char* d = std::getenv("TVEGPU_HALO_DROP_RANK");  // fault injection (tests)
        h->prm.drop_signal = (d && std::atoi(d) == pl.rank) ? 1 : 0;
    }
    h->peer = true;
}

// Cross-process form of PeerDesc (tvegpu_peer_export / tvegpu_peer_attach): CUDA IPC
// handles of the two slot buffers and the inbox, then the neighbour ranks and offsets.
struct PeerBlobHead {
    uint32_t magic;
    int32_t rank, nnbr, abi;
    cudaIpcMemHandle_t th, m, inbox;
    uint64_t off_th, off_m;
};
constexpr uint32_t kPeerMagic = 0x54564550u;  // "PEVT"

// element-kernel dynamic shared memory: mbarrier, the chunk's element rows (TMA),
// the staged node planes (ux,uy), (uz,T)
size_t elem_smem(const tvegpu_engine* h, int rows) {
    return kRowsOffset + (size_t)rows * kChunkThreads * sizeof(double) + 2 * (size_t)h->prm.max_chunk_nodes * sizeof(double2);
}
size_t k1_smem(const tvegpu_engine* h) {
    const bool xst = h->nn == 8 ? k1_xstage<8>() : k1_xstage<4>();
    const int rows = kTmaK1 ? (h->nn == 8 ? k1_rows<8>() : k1_rows<4>()).total() : 0;
    return elem_smem(h, rows) + (xst ? (size_t)h->prm.xstride * sizeof(double) : 0);
}
size_t k3_smem(const tvegpu_engine* h) {
    const int exp = h->prm.exp_kind < 0 ? 0 : (h->prm.exp_kind == 0 ? 1 : 2);
    const RowPlan r = h->nn == 8 ? (exp == 2 ? k3_rows<8, 2>(h->prm) : k3_rows<8, 0>(h->prm))
                                 : (exp == 2 ? k3_rows<4, 2>(h->prm) : k3_rows<4, 0>(h->prm));
    const bool xst = h->nn == 8 ? k3_xstage<8>() : k3_xstage<4>();
    return elem_smem(h, kTmaK3 ? r.total() : 0) + (xst ? (size_t)h->prm.xstride * sizeof(double) : 0);
}

// Launches a step kernel on the compute stream, with programmatic stream
// serialization when h->pdl (kernels.cuh pdl_wait / pdl_trigger).
template <typename... KArgs, typename... Args>
void launch_step_kernel(tvegpu_engine* h, void (*kern)(KArgs...), int grid, int block, size_t smem, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = h->s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = h->pdl ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
    if (e != cudaSuccess) {
        char buf[160];
        std::snprintf(buf, sizeof buf, " (grid %d, block %d, dynamic shared memory %zu B, pdl %d)", grid, block, smem,
                      (int)h->pdl);
        throw Error(TVEGPU_E_CUDA, std::string("cudaLaunchKernelEx: ") + cudaGetErrorString(e) + buf);
    }
}

using NodeKernel = void (*)(const DevParams, const DevPtrs, int, int, double*);
NodeKernel thermal_node_kernel(const tvegpu_engine* h) {
    if (h->slot32)
        return h->pair ? k_thermal_node<2, float> : (h->prm.ell > 1 ? k_thermal_node<1, float> : k_thermal_node<0, float>);
    return h->pair ? k_thermal_node<2> : (h->prm.ell > 1 ? k_thermal_node<1> : k_thermal_node<0>);
}

// Element kernels run one CTA per 128-element chunk over chunk range [c0, c1).
template <int NN, typename ST>
void launch_mech_element(tvegpu_engine* h, int c0, int c1) {
    if (c1 <= c0) return;
    const size_t sm = k3_smem(h);
    switch (h->prm.exp_kind < 0 ? 0 : (h->prm.exp_kind == 0 ? 1 : 2)) {
        case 0: launch_step_kernel(h, k_mech_element<NN, 0, ST>, c1 - c0, kChunkThreads, sm, h->prm, h->ptr, h->cur, c0, c1); break;
        case 1: launch_step_kernel(h, k_mech_element<NN, 1, ST>, c1 - c0, kChunkThreads, sm, h->prm, h->ptr, h->cur, c0, c1); break;
        default: launch_step_kernel(h, k_mech_element<NN, 2, ST>, c1 - c0, kChunkThreads, sm, h->prm, h->ptr, h->cur, c0, c1); break;
    }
}

template <int NN, typename ST>
void launch_thermal_element(tvegpu_engine* h, int c0, int c1) {
    if (c1 <= c0) return;
    launch_step_kernel(h, k_thermal_element<NN, ST>, c1 - c0, kChunkThreads, k1_smem(h), h->prm, h->ptr, h->cur, c0, c1);
}
void launch_thermal_elements(tvegpu_engine* h, int c0, int c1) {
    if (h->slot32) h->nn == 4 ? launch_thermal_element<4, float>(h, c0, c1) : launch_thermal_element<8, float>(h, c0, c1);
    else h->nn == 4 ? launch_thermal_element<4, double>(h, c0, c1) : launch_thermal_element<8, double>(h, c0, c1);
}
void launch_mech_elements(tvegpu_engine* h, int c0, int c1) {
    if (h->slot32) h->nn == 4 ? launch_mech_element<4, float>(h, c0, c1) : launch_mech_element<8, float>(h, c0, c1);
    else h->nn == 4 ? launch_mech_element<4, double>(h, c0, c1) : launch_mech_element<8, double>(h, c0, c1);
}
void launch_thermal_node(tvegpu_engine* h, double* t_out) {
    const int N = h->plan.N;
    launch_step_kernel(h, thermal_node_kernel(h), blocks(h->pair ? 2 * N : N, kNodeThreads), kNodeThreads, 0, h->prm,
                       h->ptr, h->cur, (int)(h->mode == TVEGPU_THERMAL_ONLY), t_out);
}
void launch_mech_node(tvegpu_engine* h, double* u_out, int n0 = 0, int n1 = -1, int closes = 1) {
    if (n1 < 0) n1 = h->plan.N;
    const int n = std::max(0, n1 - n0);
    const int nb = std::max(1, blocks(h->pair ? 2 * n : n, kNodeThreads));
    auto k = h->slot32 ? (h->pair ? k_mech_node<true, float> : k_mech_node<false, float>)
                       : (h->pair ? k_mech_node<true> : k_mech_node<false>);
    launch_step_kernel(h, k, nb, kNodeThreads, 0, h->prm, h->ptr, h->cur, closes, u_out, n0, n1);
}

template <class ST, class F>
void for_each_element_kernel_t(F&& f) {
    f((const void*)k_thermal_element<4, ST>);
    f((const void*)k_thermal_element<8, ST>);
    f((const void*)k_mech_element<4, 0, ST>);
    f((const void*)k_mech_element<4, 1, ST>);
    f((const void*)k_mech_element<4, 2, ST>);
    f((const void*)k_mech_element<8, 0, ST>);
    f((const void*)k_mech_element<8, 1, ST>);
    f((const void*)k_mech_element<8, 2, ST>);
}
template <class F>
void for_each_element_kernel(F&& f) {
    for_each_element_kernel_t<double>(f);
    for_each_element_kernel_t<float>(f);
}

void set_smem_limits(tvegpu_engine* h) {
    const int sm = (int)std::max(k1_smem(h), k3_smem(h));
    // TVEGPU_CARVEOUT=<percent>: one shared-memory carve-out for all four step kernels
    // (an SM runs blocks of two kernels side by side only under the same L1/shared split)
    if (const char* cv = std::getenv("TVEGPU_CARVEOUT")) {
        const int pct = std::atoi(cv);
        auto co = [&](const void* f) { CU(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, pct)); };
        for_each_element_kernel(co);
        co((const void*)k_thermal_node<0>);
        co((const void*)k_thermal_node<1>);
        co((const void*)k_thermal_node<2>);
        co((const void*)k_mech_node<false>);
        co((const void*)k_mech_node<true>);
        co((const void*)k_thermal_node<0, float>);
        co((const void*)k_thermal_node<1, float>);
        co((const void*)k_thermal_node<2, float>);
        co((const void*)k_mech_node<false, float>);
        co((const void*)k_mech_node<true, float>);
    }
    // the limit is a per-function attribute shared by every engine of the process: only
    // ever raise it (a later, smaller engine must not undercut an earlier one's launches)
    static std::mutex mu;
    static int set_to = 48 * 1024;
    std::lock_guard<std::mutex> lock(mu);
    if (sm <= set_to) return;
    set_to = sm;
    auto attr = [&](const void* f) { CU(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, sm)); };
    for_each_element_kernel(attr);
}

// One Engine::step() (engine.hpp:70-82) of a single-partition engine: K1 K2 [K3 K4]
// back to back on one stream (programmatic dependent launch between them).
// evs: profiling events around each kernel; wait_src: event K2 waits on (sources
// uploaded on another stream); t_final: event recorded once this step's temperatures
// are final (after K2); t_out / u_out: original-numbering copies of the new T / u
// written by K2 / K4.
void enqueue_one_step(tvegpu_engine* h, cudaEvent_t* evs = nullptr, cudaEvent_t wait_src = nullptr,
                      cudaEvent_t t_final = nullptr, double* t_out = nullptr, double* u_out = nullptr) {
    const int nc = (int)h->plan.chunk_start.size() - 1;
    int ev = 0;
    auto mark = [&]() {
        if (evs) CU(cudaEventRecord(evs[ev++], h->s));
    };
    mark();
    if (h->mode != TVEGPU_MECHANICAL_ONLY) {
        launch_thermal_elements(h, 0, nc);
        mark();
        if (wait_src) CU(cudaStreamWaitEvent(h->s, wait_src, 0));
        launch_thermal_node(h, t_out);
        mark();
    } else if (wait_src) {
        CU(cudaStreamWaitEvent(h->s, wait_src, 0));
    }
    if (t_final) CU(cudaEventRecord(t_final, h->s));
    if (h->mode != TVEGPU_THERMAL_ONLY) {
        launch_mech_elements(h, 0, nc);
        mark();
        const int ns = (int)h->io_cut.size() - 1;
        if (u_out && ns > 1) {  // tvegpu_step_io: K4 in node slices, each read back once complete
            for (int k = 0; k < ns; ++k) {
                launch_mech_node(h, u_out, h->io_cut[k], h->io_cut[k + 1], k == ns - 1 ? 1 : 0);
                CU(cudaEventRecord(h->ev_u[k], h->s));
            }
        } else {
            launch_mech_node(h, u_out);
        }
        mark();
        h->cur ^= 1;
    }
    // the closing node kernel (K2 in ThermalOnly, else K4) ends the step: verdict, t += dt, step++
    CU(cudaGetLastError());
}

// Peer-memory form (every part attached, peer_attach): per phase one launch of the
// element kernel — the boundary chunks first (element math + stores into the neighbours'
// receive areas + flags), then the interior chunks — and the node kernel, whose blocks
// holding interface nodes wait for the neighbours' flags on the device.  No pack kernel, no comm stream, no NCCL call.  Parts sharing one device
// (a group) additionally order each node kernel after its neighbours' element launches
// with events, so a waiting kernel never occupies the SMs a sender still needs; in
// single-physics steps (no other phase in between) each element launch also follows its
// neighbours' previous node kernels (DevParams::ack; a group: events as well).
// xev (profiling, one-part sets): zero-length (start, end) pairs: the transfer is in-kernel.
void enqueue_peer_step(Stepper& S, cudaEvent_t* evs, cudaEvent_t* xev) {
    const std::vector<tvegpu_engine*>& parts = S.parts;
    tvegpu_engine* h0 = parts[0];
    const bool shared_device = parts.size() > 1;
    int ev = 0;
    auto mark = [&]() {
        if (evs) CU(cudaEventRecord(evs[ev++], h0->s));
    };
    auto phase = [&](bool mech, cudaEvent_t* x) {
        for (tvegpu_engine* h : parts) {
            const int nc = (int)h->plan.chunk_start.size() - 1;
            // one launch: the boundary chunks first (they forward + signal), then the interior
            (mech ? launch_mech_elements : launch_thermal_elements)(h, 0, nc);
            if (x && h == h0) {  // the transfer is inside the element kernel: nothing separate to time
                CU(cudaEventRecord(x[0], h->s));
                CU(cudaEventRecord(x[1], h->s));
            }
            if (shared_device) CU(cudaEventRecord(h->ev_pack, h->s));
        }
        mark();
        for (tvegpu_engine* h : parts) {
            if (shared_device)
                for (int r : h->plan.neighbors) CU(cudaStreamWaitEvent(h->s, parts.at(r)->ev_pack, 0));
            if (mech) {
                launch_mech_node(h, nullptr);
                h->cur ^= 1;
            } else {
                launch_thermal_node(h, nullptr);
            }
        }
        if (shared_device && h0->prm.ack) {  // single physics: next element launch after the neighbours' node kernels
            for (tvegpu_engine* h : parts) CU(cudaEventRecord(h->ev_comm, h->s));
            for (tvegpu_engine* h : parts)
                for (int r : h->plan.neighbors) CU(cudaStreamWaitEvent(h->s, parts.at(r)->ev_comm, 0));
        }
        mark();
    };
    mark();
    if (h0->mode != TVEGPU_MECHANICAL_ONLY) phase(false, xev);
    if (h0->mode != TVEGPU_THERMAL_ONLY) phase(true, xev ? xev + 2 : nullptr);
    CU(cudaGetLastError());
}

// One step of a partitioned set (every part an RCB partition), phase by
// phase over the parts so the transport sees every part's packed segment:
//   boundary elements + pack (ev_pack) | exchange (ev_comm) | interior elements,
//   wait ev_comm, node kernel.
// The same code drives one NCCL rank (parts = {h}) and a loopback group.
// evs (one-part sets only): profiling marks at the phase boundaries.
// xev (profiling, one-part sets): per phase a (start, end) pair on the comm stream
// around the halo transfer itself.
void enqueue_partitioned_step(Stepper& S, cudaEvent_t* evs = nullptr, cudaEvent_t* xev = nullptr) {
    const std::vector<tvegpu_engine*>& parts = S.parts;
    tvegpu_engine* h0 = parts[0];
    if (h0->peer) {
        enqueue_peer_step(S, evs, xev);
        return;
    }
    int ev = 0;
    auto mark = [&]() {
        if (evs) CU(cudaEventRecord(evs[ev++], h0->s));
    };
    auto nchunks = [](const tvegpu_engine* h) { return (int)h->plan.chunk_start.size() - 1; };
    mark();
    if (h0->mode != TVEGPU_MECHANICAL_ONLY) {
        for (tvegpu_engine* h : parts) {
            launch_thermal_elements(h, 0, h->plan.nchunks_boundary);
            pack_halo(h, false);
        }
        h0->tx->exchange(parts, false, xev ? xev[0] : nullptr);
        if (xev) CU(cudaEventRecord(xev[1], h0->sc));
        for (tvegpu_engine* h : parts) launch_thermal_elements(h, h->plan.nchunks_boundary, nchunks(h));
        mark();
        for (tvegpu_engine* h : parts) {
            CU(cudaStreamWaitEvent(h->s, h->ev_comm, 0));
            launch_thermal_node(h, nullptr);
        }
        mark();
    }
    if (h0->mode != TVEGPU_THERMAL_ONLY) {
        for (tvegpu_engine* h : parts) {
            launch_mech_elements(h, 0, h->plan.nchunks_boundary);
            pack_halo(h, true);
        }
        h0->tx->exchange(parts, true, xev ? xev[2] : nullptr);
        if (xev) CU(cudaEventRecord(xev[3], h0->sc));
        for (tvegpu_engine* h : parts) launch_mech_elements(h, h->plan.nchunks_boundary, nchunks(h));
        mark();
        for (tvegpu_engine* h : parts) {
            CU(cudaStreamWaitEvent(h->s, h->ev_comm, 0));
            launch_mech_node(h, nullptr);
            h->cur ^= 1;
        }
        mark();
    }
    CU(cudaGetLastError());
}

bool partitioned(const Stepper& S) { return S.parts.size() > 1 || S.parts[0]->plan.nranks > 1; }

void enqueue_set_step(Stepper& S) {
    if (partitioned(S)) enqueue_partitioned_step(S);
    else enqueue_one_step(S.parts[0]);
}

// Multi-part sets: the parts' compute streams follow the origin stream (parts[0]->s)
// after work enqueued on it (fork), and the origin follows every part (join).
void fork_parts(Stepper& S) {
    if (S.parts.size() < 2) return;
    CU(cudaEventRecord(S.ev_fork, S.parts[0]->s));
    for (size_t k = 1; k < S.parts.size(); ++k) CU(cudaStreamWaitEvent(S.parts[k]->s, S.ev_fork, 0));
}
void join_parts(Stepper& S) {
    for (size_t k = 1; k < S.parts.size(); ++k) {
        CU(cudaEventRecord(S.parts[k]->ev_join, S.parts[k]->s));
        CU(cudaStreamWaitEvent(S.parts[0]->s, S.parts[k]->ev_join, 0));
    }
}

cudaGraphExec_t get_graph(Stepper& S, int nsteps) {
    auto key = std::make_pair(S.parts[0]->cur, nsteps);
    auto it = S.graphs.find(key);
    if (it != S.graphs.end()) return it->second;
    std::vector<int> cur0;
    for (tvegpu_engine* h : S.parts) cur0.push_back(h->cur);
    auto restore = [&] {
        for (size_t k = 0; k < S.parts.size(); ++k) S.parts[k]->cur = cur0[k];
    };
    cudaStream_t o = S.parts[0]->s;
    cudaGraph_t g;
    CU(cudaStreamBeginCapture(o, cudaStreamCaptureModeThreadLocal));
    try {
        fork_parts(S);  // the other parts' streams join the capture
        for (int k = 0; k < nsteps; ++k) enqueue_set_step(S);
        join_parts(S);
    } catch (...) {
        cudaStreamEndCapture(o, &g);
        restore();
        throw;
    }
    CU(cudaStreamEndCapture(o, &g));
    restore();
    cudaGraphExec_t ex;
    CU(cudaGraphInstantiate(&ex, g, 0));
    CU(cudaGraphDestroy(g));
    S.graphs[key] = ex;
    return ex;
}

bool flips(const tvegpu_engine* h) { return h->mode != TVEGPU_THERMAL_ONLY; }

void begin_pending(tvegpu_engine* h) {
    if (!h->pending) {
        h->pending = true;
        h->pend_step = h->host_step;
        h->pend_cur = h->cur;
        h->pend_time = h->host_time;
    }
}

// motion_override slow path: the pins of the step starting at h->host_time
// (value at t + dt, like the prescribed ramps, mechanics.hpp:89) for K4 to apply.
void upload_motion(tvegpu_engine* h) {
    const size_t rows = h->motion_orig.size();
    if (!rows) return;
    CU(cudaStreamSynchronize(h->s));  // the pinned rows of the previous step are uploaded
    const double t = h->host_time + h->dt;
    for (size_t r = 0; r < rows; ++r) {
        double d[3] = {0.0, 0.0, 0.0};
        const int pin = h->motion_fn(h->motion_user, h->motion_orig[r], t, d);
        h->motion_host[r] = make_double4(d[0], d[1], d[2], pin ? 1.0 : 0.0);
    }
    CU(cudaMemcpyAsync(const_cast<double4*>(h->ptr.motion_val), h->motion_host, rows * sizeof(double4),
                       cudaMemcpyHostToDevice, h->s));
}

// Enqueue nsteps: graph chunks, split where the active-source mask changes.
void enqueue_steps(Stepper& S, long long nsteps) {
    tvegpu_engine* h0 = S.parts[0];
    if (h0->halted) return;
    for (tvegpu_engine* h : S.parts) begin_pending(h);
    if (h0->prm.motion) {  // host callback every step: plain launches
        for (long long k = 0; k < nsteps; ++k) {
            for (tvegpu_engine* h : S.parts) {
                refresh_sources_if_needed(h, h->host_time);
                upload_motion(h);
            }
            enqueue_set_step(S);
            S.warmed = true;
            for (tvegpu_engine* h : S.parts) {
                h->host_time += h->dt;
                h->host_step += 1;
            }
        }
        return;
    }
    long long done = 0;
    while (done < nsteps) {
        for (tvegpu_engine* h : S.parts) refresh_sources_if_needed(h, h->host_time);
        // how many steps keep the same source mask? (every part holds the same schedule)
        long long k = 0;
        double t = h0->host_time;
        const long long cap = std::min<long long>(nsteps - done, S.steps_per_graph);
        while (k < cap) {
            if (k > 0 && !sources_stable(h0, t)) break;
            t += h0->dt;
            ++k;
        }
        // Graph replays once the set has run one plain step (NCCL sets up its
        // peer connections lazily on first use, which must not happen in capture).
        if (k == S.steps_per_graph && S.warmed) {
            cudaGraphExec_t ex = get_graph(S, (int)k);
            join_parts(S);
            CU(cudaGraphLaunch(ex, h0->s));
            fork_parts(S);
            if (flips(h0) && (k & 1))
                for (tvegpu_engine* h : S.parts) h->cur ^= 1;
        } else {
            for (long long j = 0; j < k; ++j) enqueue_set_step(S);
            S.warmed = true;
        }
        for (tvegpu_engine* h : S.parts) {
            h->host_time = t;
            h->host_step += k;
        }
        done += k;
    }
}

// Enqueues the 40-byte status read (clock + error words) on the main stream.
void enqueue_status_read(tvegpu_engine* h) {
    CU(cudaMemcpyAsync(h->h_words, h->ptr.clock, 6 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->s));
}

// Ends a pending window: waits for every part, agrees on the first failure across
// the partitions (all-reduce of the packed error words through the transport) and
// applies one verdict to every part.  status_enqueued: the caller already enqueued
// enqueue_status_read after the last step (single-partition sets).
tvegpu_status sync_and_check(Stepper& S, bool status_enqueued = false) {
    const bool multi = partitioned(S);
    for (tvegpu_engine* h : S.parts)
        if (!status_enqueued || multi) enqueue_status_read(h);
    for (tvegpu_engine* h : S.parts) {
        CU(cudaStreamSynchronize(h->s));
        h->pending = false;
    }
    bool any_halt = false;
    for (tvegpu_engine* h : S.parts) {
        Clock c;
        std::memcpy(&c, h->h_words, sizeof(Clock));
        any_halt |= c.halted != 0;
    }
    unsigned long long wi = S.parts[0]->h_words[3], we = S.parts[0]->h_words[4], wh = S.parts[0]->h_words[5];
    if (multi) {
        // agree on the first failure: min over the partitions of (err_inst, err_elem, err_halo)
        std::vector<unsigned long long*> w;
        for (tvegpu_engine* h : S.parts) w.push_back(reinterpret_cast<unsigned long long*>(h->ptr.err_inst));
        S.parts[0]->tx->allreduce_u64(S.parts, w, 3, /*max=*/false);
        for (tvegpu_engine* h : S.parts) {
            CU(cudaMemcpyAsync(h->h_words + 3, h->ptr.err_inst, 24, cudaMemcpyDeviceToHost, h->s));
            CU(cudaStreamSynchronize(h->s));
        }
        wi = S.parts[0]->h_words[3];
        we = S.parts[0]->h_words[4];
        wh = S.parts[0]->h_words[5];
    }
    if (wh != ~0ULL) {  // a peer-memory halo wait timed out: no verdict on the physics is possible
        char buf[200];
        std::snprintf(buf, sizeof buf,
                      "halo exchange: a neighbouring partition's contributions did not arrive in time (step %llu)", wh);
        for (tvegpu_engine* h : S.parts) {
            h->halted = true;
            h->err_step = (long long)wh;
            h->err_node = -1;
            h->err = buf;
            h->state_invalid = true;
        }
        return TVEGPU_E_NCCL;
    }
    if (!any_halt && wi == ~0ULL && we == ~0ULL) {
        for (tvegpu_engine* h : S.parts) {
            Clock c;
            std::memcpy(&c, h->h_words, sizeof(Clock));
            if (c.step != h->host_step) throw Error(TVEGPU_E_CUDA, "internal: device/host step mismatch");
            h->host_time = c.time;
        }
        return TVEGPU_OK;
    }
    // A step failed.  One partition: the device halted right after it (state = the
    // reference's state when step() throws: that step applied, time/step not advanced).
    tvegpu_status status;
    long long err_step;
    int err_id;
    char buf[320];
    if (we != ~0ULL && (wi == ~0ULL || (long long)(we >> 32) <= (long long)(wi >> 33))) {
        err_step = (long long)(we >> 32);
        err_id = (int)(we & 0xffffffffu);
        std::snprintf(buf, sizeof buf, "non-SPD C or singular F in element %d at step %lld", err_id, err_step);
        status = TVEGPU_E_VALIDATION;
    } else {
        err_step = (long long)(wi >> 33);
        err_id = (int)(wi & 0xffffffffu);
        std::snprintf(buf, sizeof buf, "non-finite %s at step %lld, node %d", ((wi >> 32) & 1) ? "displacement" : "temperature",
                      err_step, err_id);
        status = TVEGPU_E_INSTABILITY;
    }
    for (tvegpu_engine* h : S.parts) {
        Clock c;
        std::memcpy(&c, h->h_words, sizeof(Clock));
        h->halted = true;
        h->err_step = err_step;
        h->err_node = err_id;
        h->err = buf;
        if (!multi) {
            h->host_time = c.time;
            const long long executed = c.step - h->pend_step + (c.halted ? 1 : 0);
            h->host_step = c.step;
            h->cur = flips(h) ? (h->pend_cur ^ (int)(executed & 1)) : h->pend_cur;
        } else {
            // Partitioned: the failing partition halted after err_step; the others ran on
            // (their halo held stale contributions).  Every partition reports the same
            // failure at the same step and time; the state must be reset before use.
            double t = h->pend_time;
            for (long long k = h->pend_step; k < err_step; ++k) t += h->dt;
            h->host_time = t;
            h->host_step = err_step;
            h->state_invalid = true;
            h->err += " (partitioned run: the partitions' state is invalid; reset it with set_state or load_checkpoint)";
        }
    }
    return status;
}

void check_state_valid(const tvegpu_engine* h) {
    if (h->state_invalid)
        throw Error(TVEGPU_E_INSTABILITY, "state invalid after a failure in a partitioned step (step " +
                                              std::to_string(h->err_step) + "); reset it with set_state or load_checkpoint");
}

// loopback: a partition driven by a tvegpu_group on one device (halo copied by the
// group driver instead of NCCL) — single-GPU validation of the multi-GPU data path.
void build_engine(tvegpu_engine* h, const tvegpu_problem& p, const tvegpu_options& o, bool loopback = false) {
    if (o.device >= 0) CU(cudaSetDevice(o.device));
    CU(cudaGetDevice(&h->device));
    const int nranks = o.nranks > 0 ? o.nranks : 1;
    GlobalMesh g = build_global(p);  // validates first: the dt check dereferences element indices
    if (!p.allow_unstable_dt) {
        double th, me;
        critical_timestep_from_edge(p, g.min_edge, &th, &me);
        if (p.dt > std::min(th, me)) {
            char buf[200];
            std::snprintf(buf, sizeof buf, "dt %.6g above critical timestep (thermal %.6g, mechanical %.6g)", p.dt, th, me);
            throw Error(TVEGPU_E_VALIDATION, buf);
        }
    }
    h->plan = build_rank_plan(p, g, nranks, o.rank, o.reorder);
    StageTimer tm_dev("device tables + uploads");
    LapTimer lap;
    const RankPlan& pl = h->plan;
    h->nn = g.nn;
    h->kind = p.kind;
    h->mode = p.mode;
    h->dt = p.dt;
    h->N_global = g.N;
    h->E_global = g.E;
    h->P = p.prony_count;
    if (o.steps_per_graph > 0) h->solo.steps_per_graph = o.steps_per_graph;
    const int nn = g.nn, E = pl.E, N = pl.N, P = p.prony_count;
    // ---- params
    DevParams& m = h->prm;
    m.nn = nn;
    m.E = E;
    m.es = ((E + 1) + 15) / 16 * 16;  // per-element row stride: 128-byte aligned rows, one pad element
    m.N = N;
    m.P = P;
    m.mode = p.mode;
    m.td = p.temperature_dependent ? 1 : 0;
    m.dt = p.dt;
    m.mu = p.mu;
    m.kappa = p.kappa;
    m.eta_a = p.eta_a;
    m.kh = p.hourglass_stiffness * p.mu;
    m.rho = p.density;
    m.wbcb = p.perfusion_rate * p.blood_specific_heat;
    m.Ta = p.arterial_temperature;
    m.Qm = p.metabolic_rate;
    m.gamma = p.damping_gamma;
    m.inv_2dt = 1.0 / (2.0 * p.dt);
    m.inv_dt2 = 1.0 / (p.dt * p.dt);
    m.c_len = p.c_table_len;
    m.k_len = p.k_table_len;
    for (int i = 0; i < std::min(p.c_table_len, kMaxTable); ++i) {
        m.cT[i] = p.c_table_T[i];
        m.cV[i] = p.c_table_value[i];
    }
    for (int i = 0; i < std::min(p.k_table_len, kMaxTable); ++i) {
        m.kT[i] = p.k_table_T[i];
        for (int q = 0; q < 9; ++q) m.kK[i][q] = p.k_table_tensor[9 * i + q];
    }
    // every table and Prony coefficient in one device array (read there when longer than
    // the launch-parameter copies): cT | cV | kT | kK (9 per entry) | pa | pb
    std::vector<double> tabs;
    {
        auto put = [&](const double* v, size_t n) {
            const int off = (int)tabs.size();
            tabs.insert(tabs.end(), v, v + n);
            return off;
        };
        m.tab_cT = put(p.c_table_T, p.c_table_len);
        m.tab_cV = put(p.c_table_value, p.c_table_len);
        m.tab_kT = put(p.k_table_T, p.k_table_len);
        m.tab_kK = put(p.k_table_tensor, (size_t)9 * p.k_table_len);
        std::vector<double> pa(P), pb(P);
        for (int i = 0; i < P; ++i) {
            const double phi = p.prony_phi[i], tau = p.prony_tau[i];
            pa[i] = p.dt * phi / (p.dt + tau);
            pb[i] = tau / (p.dt + tau);
            if (i < kMaxProny) {
                m.pa[i] = pa[i];
                m.pb[i] = pb[i];
            }
        }
        m.tab_pa = put(pa.data(), P);
        m.tab_pb = put(pb.data(), P);
    }
    // fixed-property temperature 37 degC (engine.hpp:141)
    {
        auto interp = [&](const double* Ts, const double* Vs, int n, double T) {
            if (n == 1 || T <= Ts[0]) return Vs[0];
            if (T >= Ts[n - 1]) return Vs[n - 1];
            int j = 0;
            while (j + 2 < n && T >= Ts[j + 1]) ++j;
            const double w = (T - Ts[j]) / (Ts[j + 1] - Ts[j]);
            return Vs[j] + (Vs[j + 1] - Vs[j]) * w;
        };
        m.c_fixed = interp(p.c_table_T, p.c_table_value, m.c_len, 37.0);
        std::vector<double> col(m.k_len);
        for (int q = 0; q < 9; ++q) {
            for (int i = 0; i < m.k_len; ++i) col[i] = p.k_table_tensor[9 * i + q];
            m.k_fixed[q] = interp(p.k_table_T, col.data(), m.k_len, 37.0);
        }
    }
    const bool expansion = p.mode == TVEGPU_COUPLED && p.expansion_enabled && p.has_expansion;
    m.exp_kind = expansion ? p.expansion_kind : -1;
    m.alpha_i = p.alpha_i;
    m.alpha_m = p.alpha_m;
    m.alpha_n = p.alpha_n;
    m.Tref = p.reference_temperature;
    for (int k = 0; k < 3; ++k) {
        m.axis_m[k] = p.axis_m[k];
        m.axis_n[k] = p.axis_n[k];
        m.fiber[k] = p.fiber[k];
    }
    m.axes_per_elem = p.expansion_axes ? 1 : 0;
    m.fiber_mode = p.eta_a > 0 ? (p.fiber_dirs ? 2 : 1) : 0;
    m.diag = o.diagnostics ? 1 : 0;
    // ---- streams
    CU(cudaStreamCreateWithFlags(&h->s, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&h->sc, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&h->ev_pack, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&h->ev_comm, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&h->ev_src, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&h->ev_T, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&h->ev_entry, cudaEventDisableTiming));
    h->solo.parts = {h};
    CU(cudaMallocHost(&h->h_words, 8 * sizeof(unsigned long long)));
    cudaStream_t s = h->s;
    auto& own = h->owned;
    // ---- node arrays, built on the device from the original-order inputs (no host
    // loops over N, and only the inputs cross the link)
    h->ptr.node_orig = dupload(own, pl.node_orig, s);
    h->ptr.rec0 = dalloc<double4>(own, N);
    h->ptr.rec1 = dalloc<double4>(own, N);
    h->ptr.X = dalloc<double4>(own, N);
    h->ptr.mass = dalloc<double>(own, N);
    h->ptr.vnode = dalloc<double>(own, N);
    {
        const size_t Ng = (size_t)g.N;
        DeviceScratch tmp;
        double* xyz = tmp.get<double>(3 * Ng);
        double* mo = tmp.get<double>(Ng);
        double* vo = tmp.get<double>(Ng);
        h2d(xyz, p.nodes, 3 * Ng * 8, s);
        h2d(mo, g.mass.data(), Ng * 8, s);
        h2d(vo, g.vnode.data(), Ng * 8, s);
        if (N > 0)
            k_init_nodes<<<blocks(N, 256), 256, 0, s>>>(h->ptr.node_orig, xyz, mo, vo, p.initial_temperature, N,
                                                        h->ptr.rec0, h->ptr.rec1, const_cast<double4*>(h->ptr.X),
                                                        const_cast<double*>(h->ptr.mass),
                                                        const_cast<double*>(h->ptr.vnode));
        CU(cudaGetLastError());
        CU(cudaStreamSynchronize(s));  // before the scratch is freed
    }
    lap("node arrays");
    // ---- element arrays: the chunked connectivity (per chunk its unique node list as
    // fixed-stride {node, slot} staging entries, per element 16-bit indices into the staged
    // planes), built on the device from the per-chunk lists
    h->ptr.chunk_start = dupload(own, pl.chunk_start, s);
    h->ptr.chunk_node_off = dupload(own, pl.chunk_node_off, s);
    h->ptr.chunk_nodes = dupload(own, pl.chunk_nodes, s);
    h->ptr.chunk_node_slot = dupload(own, pl.chunk_node_slot, s);
    h->ptr.lconn = dupload(own, pl.lconn, s);
    m.max_chunk_nodes = std::max(1, pl.max_chunk_nodes);
    {
        const int nc = (int)pl.chunk_start.size() - 1;
        int st = 1;
#pragma omp parallel for schedule(static) reduction(max : st)
        for (int c = 0; c < nc; ++c) st = std::max(st, pl.chunk_node_off[c + 1] - pl.chunk_node_off[c]);
        int2* ent = dalloc<int2>(own, (size_t)nc * st);
        if (nc > 0)
            k_stage_entries<<<nc, 128, 0, s>>>(h->ptr.chunk_node_off, h->ptr.chunk_nodes, h->ptr.chunk_node_slot, st,
                                               ent);
        CU(cudaGetLastError());
        h->ptr.stage_ent = ent;
        m.stage_stride = st;
        // element-kernel coordinate blocks (k1_xstage / k3_xstage): per chunk its nodes'
        // reference coordinates in shared-slot order, x[S] y[S] z[S] with S = slots used
        // (even), one bulk copy each
        const int ms2 = (m.max_chunk_nodes + 1) & ~1;
        m.xstride = 3 * ms2;
        if (pl.nn == 8 ? (k3_xstage<8>() || k1_xstage<8>()) : (k3_xstage<4>() || k1_xstage<4>())) {
            std::vector<int32_t> cs(std::max(1, nc), 2);
#pragma omp parallel for schedule(static)
            for (int c = 0; c < nc; ++c) {
                int S = 0;
                for (int u = pl.chunk_node_off[c]; u < pl.chunk_node_off[c + 1]; ++u)
                    S = std::max(S, (int)pl.chunk_node_slot[u] + 1);
                cs[c] = std::max(2, (S + 1) & ~1);
            }
            h->ptr.chunk_xs = dupload(own, cs, s);
            double* cx = dalloc<double>(own, (size_t)std::max(1, nc) * m.xstride);
            CU(cudaMemsetAsync(cx, 0, (size_t)std::max(1, nc) * m.xstride * 8, s));
            if (nc > 0)
                k_chunk_coords<<<nc, 128, 0, s>>>(h->ptr.chunk_node_off, h->ptr.chunk_nodes, h->ptr.chunk_node_slot,
                                                  h->ptr.chunk_xs, h->ptr.X, m.xstride, cx);
            CU(cudaGetLastError());
            h->ptr.chunk_x = cx;
        }
    }
    set_smem_limits(h);
    // PDL only where the four step kernels follow each other directly on one stream
    h->pdl = !loopback && pl.nranks == 1 && !std::getenv("TVEGPU_NO_PDL");
    h->ptr.elem_orig = dupload(own, pl.elem_orig, s);
    const size_t es = (size_t)m.es;
    h->ptr.theta = dalloc<double>(own, (size_t)6 * P * es);
    h->ptr.tabs = dupload(own, tabs, h->s);
    CU(cudaMemsetAsync(h->ptr.theta, 0, std::max<size_t>(1, (size_t)6 * P * es) * 8, s));
    if (p.fiber_dirs && m.fiber_mode == 2) {
        fvec<double> f((size_t)3 * es);
#pragma omp parallel for schedule(static)
        for (size_t e = 0; e < es; ++e)
            for (int k = 0; k < 3; ++k)
                f[(size_t)k * es + e] = e < (size_t)E ? p.fiber_dirs[3 * (size_t)pl.elem_orig[e] + k] : 0.0;
        h->ptr.fiber = dupload(own, f, s);
    }
    if (p.expansion_axes && expansion) {
        fvec<double> f((size_t)6 * es);
#pragma omp parallel for schedule(static)
        for (size_t e = 0; e < es; ++e)
            for (int k = 0; k < 6; ++k)
                f[(size_t)k * es + e] = e < (size_t)E ? p.expansion_axes[6 * (size_t)pl.elem_orig[e] + k] : 0.0;
        h->ptr.axes = dupload(own, f, s);
    }
    lap("chunks, element rows");
    {  // per-element reference geometry, once (k_geometry): read by the element kernels
       // (TMA rows) and the run-level energy reduction
        if (!h->d_conn) h->d_conn = dupload(own, pl.conn, s);
        // A, V (10 rows) for K1 and the run-level energy; + the H8 hourglass vectors when K3
        // reads them instead of rebuilding them from the chunk coordinates (k3_xstage)
        const int grows = (nn == 8 && !k3_xstage<8>()) ? kGeoRows : 10;
        double* geo = dalloc<double>(own, (size_t)grows * es);
        CU(cudaMemsetAsync(geo, 0, (size_t)grows * es * 8, s));  // the pad columns feed whole-chunk bulk copies
        // affine H8 elements (parallelepipeds): k_geometry stores their hourglass geometry as
        // exact zeros and flags them; per chunk whether all are, and whether the whole
        // partition is — then K3 stages only the 10 A / V rows (TVEGPU_NO_AFFINE: off)
        const bool detect = nn == 8 && grows == kGeoRows && pl.E > 0 && !std::getenv("TVEGPU_NO_AFFINE");
        DeviceScratch tmp;
        uint8_t* aff = detect ? tmp.get<uint8_t>(pl.E) : nullptr;
        if (pl.E > 0) {
            if (nn == 8) k_geometry<8><<<blocks(pl.E, 256), 256, 0, s>>>(h->ptr.X, h->d_conn, pl.E, m.es, grows, geo, aff);
            else k_geometry<4><<<blocks(pl.E, 256), 256, 0, s>>>(h->ptr.X, h->d_conn, pl.E, m.es, grows, geo, nullptr);
            CU(cudaGetLastError());
        }
        h->ptr.geo = geo;
        if (detect) {
            const int nc = (int)pl.chunk_start.size() - 1;
            uint8_t* caff = dalloc<uint8_t>(own, nc);
            k_chunk_all<<<nc, 128, 0, s>>>(h->ptr.chunk_start, aff, caff);
            CU(cudaGetLastError());
            std::vector<uint8_t> hc(nc);
            CU(cudaMemcpyAsync(hc.data(), caff, nc, cudaMemcpyDeviceToHost, s));
            CU(cudaStreamSynchronize(s));
            int all = 1;
            for (uint8_t v : hc) all &= v;
            h->ptr.chunk_affine = caff;
            m.affine_all = all;
            h->n_affine_chunks = 0;
            for (uint8_t v : hc) h->n_affine_chunks += v;
        }
    }
    CU(cudaMallocHost(&h->qr_host, std::max(1, N) * sizeof(double)));
    std::memset(h->qr_host, 0, std::max(1, N) * sizeof(double));
    h->ptr.qr = dalloc<double>(own, N);
    CU(cudaMemsetAsync(const_cast<double*>(h->ptr.qr), 0, std::max(1, N) * sizeof(double), s));
    lap("geometry kernel");
    // ---- boundary conditions (mechanics.hpp:37-47, bioheat.hpp:32-35)
    {
        fvec<int32_t> local(g.N);
#pragma omp parallel for schedule(static)
        for (int i = 0; i < g.N; ++i) local[i] = -1;
#pragma omp parallel for schedule(static)
        for (int i = 0; i < N; ++i) local[pl.node_orig[i]] = i;
        fvec<uint8_t> mask(N);
        fvec<int32_t> row(N);
#pragma omp parallel for schedule(static)
        for (int i = 0; i < N; ++i) mask[i] = 0, row[i] = -1;
        std::vector<int32_t> presc;  // [nbc][3]
        std::vector<double> tfix;
        auto get_row = [&](int li) {
            if (row[li] < 0) {
                row[li] = (int32_t)tfix.size();
                tfix.push_back(0.0);
                presc.insert(presc.end(), {-1, -1, -1});
            }
            return row[li];
        };
        for (int k = 0; k < p.num_fixed_nodes; ++k) {
            const int li = local[p.fixed_nodes[k]];
            if (li >= 0) mask[li] |= BC_FIXED;
        }
        std::vector<double> tg(std::max(1, p.num_prescribed)), rt(std::max(1, p.num_prescribed));
        for (int q = 0; q < p.num_prescribed; ++q) {
            const auto& d = p.prescribed[q];
            tg[q] = d.target;
            rt[q] = d.ramp_time;
            for (int k = 0; k < d.num_nodes; ++k) {
                const int li = local[d.nodes[k]];
                if (li < 0) continue;
                mask[li] |= (uint8_t)(BC_PX << d.component);
                presc[3 * get_row(li) + d.component] = q;  // list order: last wins (C9)
            }
        }
        for (int k = 0; k < p.num_fixed_temperatures; ++k) {
            const int li = local[p.fixed_temperature_nodes[k]];
            if (li < 0) continue;
            mask[li] |= BC_TFIX;
            tfix[get_row(li)] = p.fixed_temperature_values[k];  // last wins
        }
#pragma omp parallel for schedule(static)
        for (int i = 0; i < N; ++i)
            if (row[i] < 0) row[i] = 0;
        if (tfix.empty()) {
            tfix.push_back(0.0);
            presc.insert(presc.end(), {-1, -1, -1});
        }
        h->ptr.mask = dupload(own, mask, s);
        h->ptr.bc_index = dupload(own, row, s);
        h->ptr.bc_presc = dupload(own, presc, s);
        h->ptr.bc_tfix = dupload(own, tfix, s);
        h->ptr.presc_target = dupload(own, tg, s);
        h->ptr.presc_ramp = dupload(own, rt, s);
        CU(cudaStreamSynchronize(s));
        // external + body force R (engine.hpp:139)
        bool anyR = p.body_force[0] != 0 || p.body_force[1] != 0 || p.body_force[2] != 0;
        if (p.external_force)
            for (int64_t k = 0; k < 3 * (int64_t)g.N && !anyR; ++k) anyR = p.external_force[k] != 0;
        m.has_R = anyR ? 1 : 0;
        if (anyR) {
            std::vector<double> R((size_t)3 * N);
            for (int i = 0; i < N; ++i)
                for (int c = 0; c < 3; ++c) {
                    const int oi = pl.node_orig[i];
                    const double ext = p.external_force ? p.external_force[3 * (size_t)oi + c] : 0.0;
                    R[(size_t)3 * i + c] = ext + p.body_force[c] * g.vnode[oi];
                }
            h->ptr.R = dupload(own, R, s);
            CU(cudaStreamSynchronize(s));
        }
    }
    lap("boundary conditions");
    // ---- gather CSR and slot buffers
    h->ptr.csr_off = dupload(own, pl.csr_off, s);
    h->ptr.csr_slot = dupload(own, pl.csr_slot, s);
    const size_t nrecv = pl.recv_off.empty() ? 0 : pl.recv_off.back();
    const size_t nslots = (size_t)nn * E + nrecv;
    m.nslots = (int)nslots;
    // + one sentinel slot (index nslots) that nothing writes: the ELL padding target
    h->slot32 = o.slot_fp32 != 0;
    const size_t sb = h->slot_bytes();  // (fp32 slots: half the doubles allocated, rounded up)
    h->ptr.slot_th = dalloc<double>(own, ((nslots + 1) * sb + 7) / 8);
    h->ptr.slot_m = dalloc<double>(own, (kMW * (nslots + 1) * sb + 7) / 8);
    CU(cudaMemsetAsync(h->ptr.slot_th, 0, (nslots + 1) * sb, s));
    CU(cudaMemsetAsync(h->ptr.slot_m, 0, kMW * (nslots + 1) * sb, s));
    {
        StageTimer tm("gather tables (ELL, valence)");
        // Node-kernel summation trees must not depend on the partition (bit-identity at any
        // rank count): two threads per node (halves of the canonical list, then their sum)
        // iff some node of the GLOBAL mesh has > 8 contributions (T4); otherwise one thread
        // sums an ELL row of 8 ids in order (H8).
        {
            int gmax = 0;  // the global mesh's largest valence
#pragma omp parallel for schedule(static) reduction(max : gmax)
            for (int i = 0; i < g.N; ++i) gmax = std::max(gmax, g.adj_off[i + 1] - g.adj_off[i]);
            h->pair = gmax > 8 && !std::getenv("TVEGPU_NO_PAIR");
        }
        int maxc = 0;
#pragma omp parallel for schedule(static) reduction(max : maxc)
        for (int i = 0; i < pl.N; ++i) maxc = std::max(maxc, pl.csr_off[i + 1] - pl.csr_off[i]);
        // ELL rows of 8 G ids (G = ceil(max contributions / 8), up to 64 contributions);
        // the pair kernels read the CSR lists instead
        const int G = (std::max(1, maxc) + 7) / 8;
        m.ell = (!h->pair && G <= 8 && !std::getenv("TVEGPU_NO_ELL")) ? G : 0;
        if (m.ell) {
            const size_t W = (size_t)8 * G;
            fvec<int32_t> ell(W * pl.N);
#pragma omp parallel for schedule(static)
            for (int i = 0; i < pl.N; ++i) {
                const int k0 = pl.csr_off[i], d = pl.csr_off[i + 1] - k0;
                for (int k = 0; k < (int)W; ++k) ell[W * i + k] = k < d ? pl.csr_slot[k0 + k] : (int32_t)nslots;
            }
            h->ptr.ell = reinterpret_cast<const int4*>(dupload(own, ell, s));
        }
    }
    lap("gather lists, slot buffers");
    // ---- clock and error words
    // clock + the three error words contiguous: the end-of-call check is one 48-byte read
    static_assert(sizeof(Clock) == 24, "status block layout");
    {
        unsigned long long* st = dalloc<unsigned long long>(own, 7);
        h->ptr.clock = reinterpret_cast<Clock*>(st);
        h->ptr.err_inst = st + 3;
        h->ptr.err_elem = st + 4;
        h->ptr.err_halo = st + 5;
        h->ptr.epoch = st + 6;  // never reset (peer-memory halo sequence base)
    }
    {
        Clock c{0.0, 0, 0, 0};
        CU(cudaMemcpyAsync(h->ptr.clock, &c, sizeof c, cudaMemcpyHostToDevice, s));
        CU(cudaMemsetAsync(h->ptr.err_inst, 0xff, 24, s));
        CU(cudaMemsetAsync(h->ptr.epoch, 0, 8, s));
        CU(cudaStreamSynchronize(s));
    }
    if (m.diag) {
        h->ptr.diag_F = dalloc<double>(own, (size_t)9 * E);
        h->ptr.diag_S = dalloc<double>(own, (size_t)9 * E);
        h->ptr.diag_f = dalloc<double>(own, (size_t)3 * N);
        CU(cudaMemsetAsync(h->ptr.diag_F, 0, (size_t)9 * E * 8, s));
        CU(cudaMemsetAsync(h->ptr.diag_S, 0, (size_t)9 * E * 8, s));
        CU(cudaMemsetAsync(h->ptr.diag_f, 0, (size_t)3 * N * 8, s));
    }
    // ---- sources
    for (int r = 0; r < p.num_sources; ++r) {
        Region reg;
        reg.q_r = p.sources[r].q_r;
        reg.t_start = p.sources[r].t_start;
        reg.t_end = p.sources[r].t_end;
        for (int k = 0; k < p.sources[r].num_elements; ++k) {
            const int e = p.sources[r].elements[k];
            for (int a = 0; a < nn; ++a) reg.nodes.push_back(p.elements[(size_t)e * nn + a]);
            reg.vol.push_back(g.vol[e]);
        }
        h->regions.push_back(std::move(reg));
    }
    h->active.assign(h->regions.size(), 0);
    // ---- tvegpu_step_io read-back slices (single partition)
    if (pl.nranks == 1 && N == g.N && N > 0) {
        const char* env = std::getenv("TVEGPU_IO_SLICES");
        const int ns = std::max(1, std::min(16, env ? std::atoi(env) : 4));
        fvec<int32_t> suf((size_t)N + 1);  // min original id over local nodes [i, N)
        suf[N] = g.N;
        for (int i = N - 1; i >= 0; --i) suf[i] = std::min(suf[i + 1], pl.node_orig[i]);
        for (int k = 0; k <= ns; ++k) h->io_cut.push_back((int)((int64_t)N * k / ns));
        for (int k = 0; k < ns; ++k) h->io_done.push_back(suf[h->io_cut[k + 1]]);
        h->ev_u.resize(ns);
        for (auto& ev : h->ev_u) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    // ---- multi-GPU halo
    if (nranks > 1) {
        if (!loopback && !o.nccl_unique_id) {  // only for tvegpu_peer_attach_solo (measurement hook)
            if (o.halo_transport != TVEGPU_HALO_PEER)
                throw Error(TVEGPU_E_ARG, "nranks > 1 needs options.nccl_unique_id");
            auto t = std::make_unique<SoloTransport>();
            h->tx = t.get();
            h->own_tx = std::move(t);
        } else if (!loopback) {  // one partition per process and GPU: the NCCL transport
            ncclUniqueId id;
            std::memcpy(&id, o.nccl_unique_id, sizeof id);
            NC(nccl().CommInitRank(&h->comm, nranks, id, o.rank));
            auto t = std::make_unique<NcclTransport>();
            t->comm = h->comm;
            h->tx = t.get();
            h->own_tx = std::move(t);
        }  // loopback: the group installs its transport
        const size_t ns = pl.send_off.back();
        h->d_send_slot = dupload(own, pl.send_slot, s);
        h->send_th = dalloc<double>(own, ns);
        h->send_m = dalloc<double>(own, kMW * ns);
        // peer-memory halo: the inbox the neighbours raise their flags in, the send-kernel CTA counters
        h->halo_transport = o.halo_transport;
        // [0, np): the neighbours' phase flags; [np, 2 np): their end-of-step acks (single physics)
        const size_t np = std::max<size_t>(1, pl.neighbors.size());
        h->ptr.inbox = dalloc<unsigned long long>(own, 2 * np);
        h->ptr.ack_inbox = h->ptr.inbox + pl.neighbors.size();
        CU(cudaMemsetAsync(h->ptr.inbox, 0, 2 * np * 8, s));
        h->ptr.send_cnt = dalloc<unsigned>(own, 2);
        CU(cudaMemsetAsync(h->ptr.send_cnt, 0, 8, s));
        CU(cudaStreamSynchronize(s));
    }
    CU(cudaStreamSynchronize(s));
}


template <class F>
tvegpu_status guard(tvegpu_engine* h, F&& f) {
    try {
        return f();
    } catch (const Error& e) {
        if (h) {
            h->err = e.what();
            h->last_status = e.status;
        }
        return e.status;
    } catch (const std::exception& e) {
        if (h) h->err = e.what();
        return TVEGPU_E_ARG;
    }
}

void to_local_rec(tvegpu_engine* h, std::vector<double4>& r0, std::vector<double4>& r1) {
    const int N = h->plan.N;
    r0.resize(N);
    r1.resize(N);
    CU(cudaMemcpyAsync(r0.data(), h->ptr.rec0, N * sizeof(double4), cudaMemcpyDeviceToHost, h->s));
    CU(cudaMemcpyAsync(r1.data(), h->ptr.rec1, N * sizeof(double4), cudaMemcpyDeviceToHost, h->s));
    CU(cudaStreamSynchronize(h->s));
}

// One D2H copy of the current node record (u, T) into pinned staging, scattered to
// original numbering; the previous record is copied only when u_prev is wanted.
// Device-side renumbering for host I/O: the local (Morton/first-touch) order is
// scattered to the caller's original numbering on the GPU, so the host transfer is
// one contiguous copy straight into the caller's buffer (pinned buffers give the
// full link bandwidth) and no host loop touches the data.
__global__ void k_fields_to_orig(const double4* __restrict__ rec, const int32_t* __restrict__ node_orig, int N,
                                 double* __restrict__ T, double* __restrict__ u) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const double4 r = rec[i];
    const size_t o = (size_t)node_orig[i];
    if (T) T[o] = r.w;
    if (u) {
        u[3 * o] = r.x;
        u[3 * o + 1] = r.y;
        u[3 * o + 2] = r.z;
    }
}
__global__ void k_orig_to_local(const double* __restrict__ v, const int32_t* __restrict__ node_orig, int N,
                                double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N) out[i] = v[node_orig[i]];
}

double* io_buffer(tvegpu_engine* h) {
    if (!h->d_io) h->d_io = dalloc<double>(h->owned, 4 * (size_t)h->plan.N);
    return h->d_io;
}

void read_fields(tvegpu_engine* h, double* T, double* u, double* up) {
    check_state_valid(h);
    const int N = h->plan.N;
    if (h->plan.nranks == 1 && N == h->N_global) {  // one partition covers every node
        double* dT = io_buffer(h);
        double* du = dT + N;
        const double4* rc = h->cur ? h->ptr.rec1 : h->ptr.rec0;
        const double4* rp = h->cur ? h->ptr.rec0 : h->ptr.rec1;
        k_fields_to_orig<<<blocks(N, 256), 256, 0, h->s>>>(rc, h->ptr.node_orig, N, T ? dT : nullptr,
                                                           u ? du : nullptr);
        if (T) CU(cudaMemcpyAsync(T, dT, (size_t)N * 8, cudaMemcpyDeviceToHost, h->s));
        if (u) CU(cudaMemcpyAsync(u, du, (size_t)3 * N * 8, cudaMemcpyDeviceToHost, h->s));
        if (up) {
            CU(cudaStreamSynchronize(h->s));  // du is reused
            k_fields_to_orig<<<blocks(N, 256), 256, 0, h->s>>>(rp, h->ptr.node_orig, N, nullptr, du);
            CU(cudaMemcpyAsync(up, du, (size_t)3 * N * 8, cudaMemcpyDeviceToHost, h->s));
        }
        CU(cudaStreamSynchronize(h->s));
        return;
    }
    if (!h->stage) CU(cudaMallocHost(&h->stage, (size_t)N * sizeof(double4)));
    const double4* rc = h->cur ? h->ptr.rec1 : h->ptr.rec0;
    const double4* rp = h->cur ? h->ptr.rec0 : h->ptr.rec1;
    CU(cudaMemcpyAsync(h->stage, rc, N * sizeof(double4), cudaMemcpyDeviceToHost, h->s));
    CU(cudaStreamSynchronize(h->s));
    // partitions: this rank's nodes scattered into the caller's arrays (host threads)
    const int32_t* no = h->plan.node_orig.data();
#pragma omp parallel for schedule(static)
    for (int i = 0; i < N; ++i) {
        const double4 r = h->stage[i];
        const size_t o = (size_t)no[i];
        if (T) T[o] = r.w;
        if (u) {
            u[3 * o] = r.x;
            u[3 * o + 1] = r.y;
            u[3 * o + 2] = r.z;
        }
    }
    if (up) {
        CU(cudaMemcpyAsync(h->stage, rp, N * sizeof(double4), cudaMemcpyDeviceToHost, h->s));
        CU(cudaStreamSynchronize(h->s));
#pragma omp parallel for schedule(static)
        for (int i = 0; i < N; ++i) {
            const size_t o = 3 * (size_t)no[i];
            up[o] = h->stage[i].x;
            up[o + 1] = h->stage[i].y;
            up[o + 2] = h->stage[i].z;
        }
    }
}

// ------------------------------------------------------------------ run-level outputs
// Deterministic two-pass reductions: fixed per-block trees, then one block over the
// block partials in index order, so repeated calls return identical bits.
constexpr int kRedThreads = 256, kRedMaxBlocks = 2048;

// Block tree of NV doubles per thread under op (0 sum, 1 max, 2 min), written by thread 0.
template <int NV>
__device__ void block_reduce(double (&v)[NV], const int (&op)[NV], double* out) {
    __shared__ double sh[NV][kRedThreads];
#pragma unroll
    for (int q = 0; q < NV; ++q) sh[q][threadIdx.x] = v[q];
    __syncthreads();
    for (int s = kRedThreads / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s)
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                const double a = sh[q][threadIdx.x], b = sh[q][threadIdx.x + s];
                sh[q][threadIdx.x] = op[q] == 0 ? a + b : op[q] == 1 ? fmax(a, b) : fmin(a, b);
            }
        __syncthreads();
    }
    if (threadIdx.x == 0)
#pragma unroll
        for (int q = 0; q < NV; ++q) out[q] = sh[q][0];
}

// Second pass: one block folds the nb partial rows (stride NV) in index order.
template <int NV>
__global__ void k_reduce_rows(const double* __restrict__ part, int nb, int o0, int o1, int o2, int o3, int o4,
                              int o5, int o6, double* __restrict__ out) {
    const int opsv[7] = {o0, o1, o2, o3, o4, o5, o6};
    int op[NV];
    double v[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        op[q] = opsv[q];
        v[q] = op[q] == 0 ? 0.0 : op[q] == 1 ? -INFINITY : INFINITY;
    }
    for (int b = threadIdx.x; b < nb; b += kRedThreads)
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const double x = part[(size_t)b * NV + q];
            v[q] = op[q] == 0 ? v[q] + x : op[q] == 1 ? fmax(v[q], x) : fmin(v[q], x);
        }
    block_reduce<NV>(v, op, out);
}

// RunSummary node extrema (engine.hpp:57-66): max T, per-component min and max of u.
__global__ void __launch_bounds__(kRedThreads) k_summary(const double4* __restrict__ rec, int N, double* part) {
    const int op[7] = {1, 2, 2, 2, 1, 1, 1};
    double v[7] = {-INFINITY, INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    for (int i = blockIdx.x * kRedThreads + threadIdx.x; i < N; i += gridDim.x * kRedThreads) {
        const double4 r = rec[i];
        v[0] = fmax(v[0], r.w);
        v[1] = fmin(v[1], r.x), v[2] = fmin(v[2], r.y), v[3] = fmin(v[3], r.z);
        v[4] = fmax(v[4], r.x), v[5] = fmax(v[5], r.y), v[6] = fmax(v[6], r.z);
    }
    block_reduce<7>(v, op, part + (size_t)blockIdx.x * 7);
}

// Volume fraction of a tetrahedron above thr (oracle tet_fraction_above).
__device__ double tet_fraction_above(const double (&T)[4], double thr) {
    int up[4], dn[4], nu = 0, nd = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (T[i] >= thr) up[nu++] = i;
        else dn[nd++] = i;
    }
    auto t = [&](int i, int j) { return (T[i] - thr) / (T[i] - T[j]); };
    if (nu == 0) return 0.0;
    if (nu == 4) return 1.0;
    if (nu == 1) return t(up[0], dn[0]) * t(up[0], dn[1]) * t(up[0], dn[2]);
    if (nu == 3) {
        const int d = dn[0];
        auto sd = [&](int j) { return (thr - T[d]) / (T[j] - T[d]); };
        return 1.0 - sd(up[0]) * sd(up[1]) * sd(up[2]);
    }
    const int a = up[0], b = up[1], c = dn[0], d = dn[1];
    const double tac = t(a, c), tad = t(a, d), tbc = t(b, c), tbd = t(b, d);
    return tac * tad * (1.0 - tbd) + tac * tbd * (1.0 - tbc) + tbc * tbd;
}

__constant__ int c_hex_tets[6][4] = {{0, 1, 2, 6}, {0, 2, 3, 6}, {0, 3, 7, 6}, {0, 7, 4, 6}, {0, 4, 5, 6}, {0, 5, 1, 6}};

// ablation_volume: per element the clipped volume of its
// tetrahedra (H8: 6 around the 0-6 diagonal) at X (+ u when deformed); partial rows
// {volume, #elements with a non-zero clipped volume}.
template <int NN>
__global__ void __launch_bounds__(kRedThreads) k_ablation(const int32_t* __restrict__ conn, const double4* __restrict__ X,
                                                     const double4* __restrict__ rec, int E, double thr, int deformed,
                                                     double* part) {
    double v[2] = {0.0, 0.0};
    const int op[2] = {0, 0};
    for (int e = blockIdx.x * kRedThreads + threadIdx.x; e < E; e += gridDim.x * kRedThreads) {
        double px[NN][3], Tn[NN];
#pragma unroll
        for (int a = 0; a < NN; ++a) {
            const int i = conn[(size_t)e * NN + a];
            const double4 x = X[i], r = rec[i];
            px[a][0] = x.x + (deformed ? r.x : 0.0);
            px[a][1] = x.y + (deformed ? r.y : 0.0);
            px[a][2] = x.z + (deformed ? r.z : 0.0);
            Tn[a] = r.w;
        }
        double ve = 0.0;
        for (int k = 0; k < (NN == 4 ? 1 : 6); ++k) {
            int id[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) id[q] = NN == 4 ? q : c_hex_tets[k][q];
            const double Tq[4] = {Tn[id[0]], Tn[id[1]], Tn[id[2]], Tn[id[3]]};
            const double f = tet_fraction_above(Tq, thr);
            if (f == 0.0) continue;
            double M[3][3];
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int q = 0; q < 3; ++q) M[c][q] = px[id[q + 1]][c] - px[id[0]][c];
            const double dt = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
                              M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                              M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
            ve += f * fabs(dt) / 6.0;
        }
        if (ve > 0.0) {
            v[0] += ve;
            v[1] += 1.0;
        }
    }
    block_reduce<2>(v, op, part + (size_t)blockIdx.x * 2);
}

// total_energy (engine.hpp:108): kinetic 1/2 m |(u - u_prev)/dt|^2 per node plus the
// hyperelastic energy V det(F_th) Psi(C_el) per element (the oracle's definition, with
// F_th from the current element-mean temperature, i.e. the last mechanics phase's).
// Psi = mu/2 (J^-2/3 tr C - 3) + kappa/2 (J - 1)^2 [+ eta/2 (J^-2/3 a.Ca - 1)^2].
template <int NN>
__global__ void __launch_bounds__(kRedThreads) k_energy(const DevParams P, const DevPtrs D, const int32_t* __restrict__ conn,
                                                   const double4* __restrict__ rc, const double4* __restrict__ rp,
                                                   double* part) {
    double v[2] = {0.0, 0.0};
    const int op[2] = {0, 0};
    const int E = P.E, N = P.N;
    for (int i = blockIdx.x * kRedThreads + threadIdx.x; i < N; i += gridDim.x * kRedThreads) {
        const double4 a = rc[i], b = rp[i];
        const double vx = (a.x - b.x) / P.dt, vy = (a.y - b.y) / P.dt, vz = (a.z - b.z) / P.dt;
        v[0] += 0.5 * D.mass[i] * (vx * vx + vy * vy + vz * vz);
    }
    for (int e = blockIdx.x * kRedThreads + threadIdx.x; e < E; e += gridDim.x * kRedThreads) {
        double H[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, Ts = 0.0;
        double u[NN][3];
        for (int q = 0; q < NN; ++q) {
            const double4 r = rc[conn[(size_t)e * NN + q]];
            u[q][0] = r.x, u[q][1] = r.y, u[q][2] = r.z;
            Ts += r.w;
        }
        if (NN == 4) {
            for (int q = 1; q < 4; ++q)
                for (int i = 0; i < 3; ++i) H[i * 3 + q - 1] = u[q][i] - u[0][i];
        } else {
            for (int q = 0; q < 8; ++q)
                for (int j = 0; j < 3; ++j)
                    for (int i = 0; i < 3; ++i) H[i * 3 + j] += h8s(q, j) * u[q][i];
        }
        double A[9];
        for (int q = 0; q < 9; ++q) A[q] = D.geo[(size_t)q * P.es + e];
        const double V = D.geo[(size_t)9 * P.es + e];
        double F[9];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                F[i * 3 + j] = (i == j ? 1.0 : 0.0) + H[i * 3 + 0] * A[j * 3 + 0] + H[i * 3 + 1] * A[j * 3 + 1] +
                               H[i * 3 + 2] * A[j * 3 + 2];
        double Fth[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
        if (P.exp_kind >= 0) {
            const double dT = Ts / NN - P.Tref;
            double m[3], n[3];
            for (int k = 0; k < 3; ++k) {
                m[k] = P.axes_per_elem ? D.axes[(size_t)k * P.es + e] : P.axis_m[k];
                n[k] = P.axes_per_elem ? D.axes[(size_t)(3 + k) * P.es + e] : P.axis_n[k];
            }
            const double ei = P.alpha_i * dT;
            const double dm = P.exp_kind >= 1 ? P.alpha_m * dT - ei : 0.0;
            const double dn = P.exp_kind == 2 ? P.alpha_n * dT - ei : 0.0;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j)
                    Fth[i * 3 + j] = (i == j ? 1.0 + ei : 0.0) + dm * m[i] * m[j] + dn * n[i] * n[j];
        }
        double Ad[9];
        const double dth = adj3(Fth, Ad);
        double Fel[9];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                Fel[i * 3 + j] = (F[i * 3 + 0] * Ad[0 * 3 + j] + F[i * 3 + 1] * Ad[1 * 3 + j] + F[i * 3 + 2] * Ad[2 * 3 + j]) / dth;
        double Cm[9];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                Cm[i * 3 + j] = Fel[0 * 3 + i] * Fel[0 * 3 + j] + Fel[1 * 3 + i] * Fel[1 * 3 + j] + Fel[2 * 3 + i] * Fel[2 * 3 + j];
        double Ac[9];
        const double J = sqrt(adj3(Cm, Ac));
        const double Jm23 = pow(J, -2.0 / 3.0);
        double psi = 0.5 * P.mu * (Jm23 * (Cm[0] + Cm[4] + Cm[8]) - 3.0) + 0.5 * P.kappa * (J - 1.0) * (J - 1.0);
        if (P.eta_a > 0 && P.fiber_mode) {
            double fa[3];
            for (int k = 0; k < 3; ++k) fa[k] = P.fiber_mode == 2 ? D.fiber[(size_t)k * P.es + e] : P.fiber[k];
            double aCa = 0;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) aCa += fa[i] * Cm[i * 3 + j] * fa[j];
            const double I4 = Jm23 * aCa;
            psi += 0.5 * P.eta_a * (I4 - 1.0) * (I4 - 1.0);
        }
        v[1] += V * dth * psi;
    }
    block_reduce<2>(v, op, part + (size_t)blockIdx.x * 2);
}

// det F and the largest eigenvalue of S_tilde (PK2) per element, original order,
// from the diagnostics of the last mechanics phase (Snapshot det_f /
// max_principal_stress, engine.hpp:47-55).
__global__ void k_element_fields(const double* __restrict__ F, const double* __restrict__ S,
                                 const int32_t* __restrict__ elem_orig, int E, double* detf, double* smax) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    const double* f = F + (size_t)e * 9;
    const double* m = S + (size_t)e * 9;
    const int o = elem_orig[e];
    if (detf)
        detf[o] = f[0] * (f[4] * f[8] - f[5] * f[7]) - f[1] * (f[3] * f[8] - f[5] * f[6]) +
                  f[2] * (f[3] * f[7] - f[4] * f[6]);
    if (smax) {
        // symmetric 3x3 eigenvalues, trigonometric form
        const double a = m[0], b = m[4], c = m[8], d = m[1], ee = m[5], ff = m[2];
        const double p1 = d * d + ee * ee + ff * ff;
        const double q = (a + b + c) / 3.0;
        double lmax;
        if (p1 == 0.0) {
            lmax = fmax(a, fmax(b, c));
        } else {
            const double p2 = (a - q) * (a - q) + (b - q) * (b - q) + (c - q) * (c - q) + 2.0 * p1;
            const double p = sqrt(p2 / 6.0);
            const double ip = 1.0 / p;
            const double B0 = (a - q) * ip, B1 = (b - q) * ip, B2 = (c - q) * ip, B3 = d * ip, B4 = ee * ip,
                         B5 = ff * ip;
            const double r = 0.5 * (B0 * (B1 * B2 - B4 * B4) - B3 * (B3 * B2 - B4 * B5) + B5 * (B3 * B4 - B1 * B5));
            const double phi = r <= -1.0 ? M_PI / 3.0 : r >= 1.0 ? 0.0 : acos(r) / 3.0;
            lmax = q + 2.0 * p * cos(phi);
        }
        smax[o] = lmax;
    }
}

// Runs one two-pass reduction (kernel writes nb rows of NV) and returns the NV
// values in h->h_part; for nranks > 1 the values are all-reduced across ranks.
template <int NV, class Launch>
void reduce_to_host(tvegpu_engine* h, int nb, const int (&op)[NV], Launch&& launch) {
    check_state_valid(h);
    if (!h->d_part) h->d_part = dalloc<double>(h->owned, (size_t)kRedMaxBlocks * 8 + 8);
    if (!h->h_part) CU(cudaMallocHost(&h->h_part, 8 * sizeof(double)));
    double* fin = h->d_part + (size_t)kRedMaxBlocks * 8;
    launch(h->d_part);
    int o[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int q = 0; q < NV; ++q) o[q] = op[q];
    k_reduce_rows<NV><<<1, kRedThreads, 0, h->s>>>(h->d_part, nb, o[0], o[1], o[2], o[3], o[4], o[5], o[6], fin);
    CU(cudaGetLastError());
    if (h->comm) {
        NcclApi& api = nccl();
        // group the ops by kind: sums, maxima, minima (one all-reduce per value, tiny)
        for (int q = 0; q < NV; ++q)
            NC(api.AllReduce(fin + q, fin + q, 1, ncclFloat64, op[q] == 0 ? ncclSum : op[q] == 1 ? ncclMax : ncclMin,
                             h->comm, h->s));
    }
    CU(cudaMemcpyAsync(h->h_part, fin, NV * sizeof(double), cudaMemcpyDeviceToHost, h->s));
    CU(cudaStreamSynchronize(h->s));
}

int red_blocks(int n) { return std::max(1, std::min(kRedMaxBlocks, (n + kRedThreads - 1) / kRedThreads)); }

}  // namespace

// =====================================================================================
extern "C" {

int32_t tvegpu_abi_version(void) { return TVEGPU_ABI_VERSION; }

const char* tvegpu_status_string(tvegpu_status s) {
    switch (s) {
        case TVEGPU_OK: return "ok";
        case TVEGPU_E_PARSE: return "ParseError";
        case TVEGPU_E_VALIDATION: return "ValidationError";
        case TVEGPU_E_INSTABILITY: return "InstabilityError";
        case TVEGPU_E_IO: return "IoError";
        case TVEGPU_E_CUDA: return "CudaError";
        case TVEGPU_E_NCCL: return "NcclError";
        case TVEGPU_E_ARG: return "ArgumentError";
    }
    return "unknown";
}

const char* tvegpu_create_error(void) { return g_create_error.c_str(); }

void tvegpu_default_options(tvegpu_options* o) {
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->device = -1;
    o->nranks = 1;
    o->rank = 0;
    o->reorder = 1;
    o->steps_per_graph = 64;
    o->halo_transport = TVEGPU_HALO_PEER;
}

tvegpu_status tvegpu_create(const tvegpu_problem* p, const tvegpu_options* o, tvegpu_engine** out) {
    TVEGPU_RANGE();
    if (!p || !out) {
        g_create_error = "NULL argument";
        return TVEGPU_E_ARG;
    }
    *out = nullptr;
    tvegpu_options def;
    tvegpu_default_options(&def);
    if (!o) o = &def;
    auto* h = new tvegpu_engine();
    try {
        build_engine(h, *p, *o);
    } catch (const Error& e) {
        g_create_error = e.what();
        tvegpu_destroy(h);
        return e.status;
    } catch (const std::exception& e) {
        g_create_error = e.what();
        tvegpu_destroy(h);
        return TVEGPU_E_ARG;
    }
    g_create_error.clear();
    *out = h;
    return TVEGPU_OK;
}

void tvegpu_destroy(tvegpu_engine* h) {
    if (!h) return;
    for (auto& kv : h->solo.graphs) cudaGraphExecDestroy(kv.second);
    if (h->s) cudaStreamSynchronize(h->s);
    if (h->sc) cudaStreamSynchronize(h->sc);
    if (h->comm) nccl().CommDestroy(h->comm);
    for (void* p : h->ipc_open) cudaIpcCloseMemHandle(p);
    for (void* p : h->owned) cudaFree(p);
    if (h->h_words) cudaFreeHost(h->h_words);
    if (h->stage) cudaFreeHost(h->stage);
    if (h->qr_host) cudaFreeHost(h->qr_host);
    if (h->motion_host) cudaFreeHost(h->motion_host);
    if (h->ev_pack) cudaEventDestroy(h->ev_pack);
    if (h->ev_src) cudaEventDestroy(h->ev_src);
    if (h->h_part) cudaFreeHost(h->h_part);
    if (h->ev_T) cudaEventDestroy(h->ev_T);
    if (h->ev_comm) cudaEventDestroy(h->ev_comm);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    if (h->ev_entry) cudaEventDestroy(h->ev_entry);
    for (cudaEvent_t ev : h->ev_u) cudaEventDestroy(ev);
    if (h->s) cudaStreamDestroy(h->s);
    if (h->sc) cudaStreamDestroy(h->sc);
    delete h;
}

tvegpu_status tvegpu_enqueue_steps(tvegpu_engine* h, int64_t n) {
    TVEGPU_RANGE();
    if (!h || n < 0) return TVEGPU_E_ARG;
    return guard(h, [&] {
        enqueue_steps(h->solo, n);
        return TVEGPU_OK;
    });
}

tvegpu_status tvegpu_sync(tvegpu_engine* h) {
    TVEGPU_RANGE();
    if (!h) return TVEGPU_E_ARG;
    return guard(h, [&] {
        if (h->halted) return h->last_status;
        if (!h->pending) {
            CU(cudaStreamSynchronize(h->s));
            return TVEGPU_OK;
        }
        h->last_status = sync_and_check(h->solo);
        return h->last_status;
    });
}

tvegpu_status tvegpu_step(tvegpu_engine* h, int64_t n) {
    TVEGPU_RANGE();
    if (!h || n < 0) return TVEGPU_E_ARG;
    return guard(h, [&] {
        if (h->halted) {
            h->err = "engine halted by an earlier failure; reset the state with tvegpu_set_state";
            return h->last_status;
        }
        enqueue_steps(h->solo, n);
        h->last_status = sync_and_check(h->solo);
        return h->last_status;
    });
}

double tvegpu_time(const tvegpu_engine* h) { return h ? h->host_time : 0.0; }
int64_t tvegpu_step_count(const tvegpu_engine* h) { return h ? h->host_step : 0; }

tvegpu_status tvegpu_get_temperatures(tvegpu_engine* h, double* T) {
    if (!h || !T) return TVEGPU_E_ARG;
    return guard(h, [&] {
        read_fields(h, T, nullptr, nullptr);
        return TVEGPU_OK;
    });
}

tvegpu_status tvegpu_get_displacements(tvegpu_engine* h, double* u, double* up) {
    if (!h || !u) return TVEGPU_E_ARG;
    return guard(h, [&] {
        read_fields(h, nullptr, u, up);
        return TVEGPU_OK;
    });
}

tvegpu_status tvegpu_make_snapshot(tvegpu_engine* h, double* T, double* u) {
    TVEGPU_RANGE();
    if (!h || (!T && !u)) return TVEGPU_E_ARG;
    return guard(h, [&] {
        read_fields(h, T, u, nullptr);
        return TVEGPU_OK;
    });
}

tvegpu_status tvegpu_get_viscous(tvegpu_engine* h, double* v) {
    if (!h || !v) return TVEGPU_E_ARG;
    return guard(h, [&] {
        check_state_valid(h);
        const int E = h->plan.E, P = h->P;
        const size_t es = (size_t)h->prm.es;
        std::vector<double> th((size_t)6 * P * es);
        if (!th.empty()) {
            CU(cudaMemcpyAsync(th.data(), h->ptr.theta, th.size() * 8, cudaMemcpyDeviceToHost, h->s));
            CU(cudaStreamSynchronize(h->s));
        }
        static const int map9[9] = {0, 3, 5, 3, 1, 4, 5, 4, 2};
        for (int e = 0; e < E; ++e)
            for (int p = 0; p < P; ++p) {
                double* o = v + ((size_t)h->plan.elem_orig[e] * P + p) * 9;
                for (int q = 0; q < 9; ++q) o[q] = th[((size_t)p * 6 + map9[q]) * es + e];
            }
        return TVEGPU_OK;
    });
}

tvegpu_status tvegpu_set_state(tvegpu_engine* h, const double* T, const double* u, const double* up,
                               const double* viscous, double time, int64_t step) {
    TVEGPU_RANGE();
    if (!h) return TVEGPU_E_ARG;
    return guard(h, [&] {
        std::vector<double4> r0, r1;
        to_local_rec(h, r0, r1);
        auto& rc = h->cur ? r1 : r0;
        auto& rp = h->cur ? r0 : r1;
        for (int i = 0; i < h->plan.N; ++i) {
            const size_t o = (size_t)h->plan.node_orig[i];
            if (T) rc[i].w = rp[i].w = T[o];
            if (u) rc[i] = make_double4(u[3 * o], u[3 * o + 1], u[3 * o + 2], rc[i].w);
            if (up) rp[i] = make_double4(up[3 * o], up[3 * o + 1], up[3 * o + 2], rp[i].w);
        }
        const int N = h->plan.N;
        CU(cudaMemcpyAsync(h->ptr.rec0, r0.data(), N * sizeof(double4), cudaMemcpyHostToDevice, h->s));
        CU(cudaMemcpyAsync(h->ptr.rec1, r1.data(), N * sizeof(double4), cudaMemcpyHostToDevice, h->s));
        if (viscous && h->P) {
            const int E = h->plan.E, P = h->P;
            const size_t es = (size_t)h->prm.es;
            std::vector<double> th((size_t)6 * P * es, 0.0);
            static const int pick[6] = {0, 4, 8, 1, 5, 2};  // xx yy zz xy yz xz from row-major 3x3
            for (int e = 0; e < E; ++e)
                for (int p = 0; p < P; ++p) {
                    const double* iv = viscous + ((size_t)h->plan.elem_orig[e] * P + p) * 9;
                    for (int q = 0; q < 6; ++q) th[((size_t)p * 6 + q) * es + e] = iv[pick[q]];
                }
            CU(cudaMemcpyAsync(h->ptr.theta, th.data(), th.size() * 8, cudaMemcpyHostToDevice, h->s));
            CU(cudaStreamSynchronize(h->s));
        }
        Clock c{time, (long long)step, 0, 0};
        CU(cudaMemcpyAsync(h->ptr.clock, &c, sizeof c, cudaMemcpyHostToDevice, h->s));
        CU(cudaMemsetAsync(h->ptr.err_inst, 0xff, 24, h->s));
        CU(cudaStreamSynchronize(h->s));
        h->host_time = time;
        h->host_step = step;
        h->halted = false;
        h->state_invalid = false;
        h->last_status = TVEGPU_OK;
        return TVEGPU_OK;
    });
}

tvegpu_status tvegpu_set_nodal_sources(tvegpu_engine* h, const double* power) {
    if (!h) return TVEGPU_E_ARG;
    return guard(h, [&] {
        if (!power) {
            h->source_override = false;
            h->sources_init = false;
            return TVEGPU_OK;
        }
        h->source_override = true;
        if (h->plan.nranks == 1 && h->plan.N == h->N_global) {  // upload as given, renumber on the device
            double* d = io_buffer(h);
            CU(cudaMemcpyAsync(d, power, (size_t)h->N_global * 8, cudaMemcpyHostToDevice, h->s));
            k_orig_to_local<<<blocks(h->plan.N, 256), 256, 0, h->s>>>(d, h->ptr.node_orig, h->plan.N,
                                                                     const_cast<double*>(h->ptr.qr));
            CU(cudaGetLastError());
            CU(cudaStreamSynchronize(h->s));  // the caller may reuse `power` on return
            return TVEGPU_OK;
        }
#pragma omp parallel for schedule(static)
        for (int li = 0; li < h->plan.N; ++li) h->qr_host[li] = power[h->plan.node_orig[li]];
        CU(cudaMemcpyAsync(const_cast<double*>(h->ptr.qr), h->qr_host, (size_t)h->plan.N * 8,
                           cudaMemcpyHostToDevice, h->s));
        CU(cudaStreamSynchronize(h->s));
        return TVEGPU_OK;
    });
}

// MechBCs::motion_override (mechanics.hpp:43-46).  nodes (original ids) limits the
// callback to those candidates; NULL = every node, as the reference evaluates it.
tvegpu_status tvegpu_set_motion_override(tvegpu_engine* h, tvegpu_motion_fn fn, void* user, int32_t num_nodes,
                                         const int32_t* nodes) {
    TVEGPU_RANGE();
    if (!h || num_nodes < 0 || (num_nodes > 0 && !nodes)) return TVEGPU_E_ARG;
    return guard(h, [&] {
        CU(cudaStreamSynchronize(h->s));
        for (auto& kv : h->solo.graphs) cudaGraphExecDestroy(kv.second);  // captured with the old parameters
        h->solo.graphs.clear();
        h->motion_fn = fn;
        h->motion_user = user;
        h->motion_orig.clear();
        h->prm.motion = 0;
        if (!fn) return TVEGPU_OK;
        const int N = h->plan.N;
        std::vector<int32_t> local(h->N_global, -1);
        for (int i = 0; i < N; ++i) local[h->plan.node_orig[i]] = i;
        std::vector<int32_t> row(N, -1);
        auto add = [&](int32_t o) {
            if (o < 0 || o >= h->N_global) throw Error(TVEGPU_E_ARG, "motion_override node out of range");
            const int li = local[o];
            if (li < 0 || row[li] >= 0) return;  // another partition's node, or listed twice
            row[li] = (int32_t)h->motion_orig.size();
            h->motion_orig.push_back(o);
        };
        if (nodes)
            for (int k = 0; k < num_nodes; ++k) add(nodes[k]);
        else
            for (int o = 0; o < h->N_global; ++o) add(o);
        const size_t rows = std::max<size_t>(1, h->motion_orig.size());
        if (h->motion_host) CU(cudaFreeHost(h->motion_host));
        h->motion_host = nullptr;
        CU(cudaMallocHost(&h->motion_host, rows * sizeof(double4)));
        h->ptr.motion_row = dupload(h->owned, row, h->s);
        double4* val = dalloc<double4>(h->owned, rows);
        CU(cudaMemsetAsync(val, 0, rows * sizeof(double4), h->s));
        h->ptr.motion_val = val;
        CU(cudaStreamSynchronize(h->s));
        h->prm.motion = 1;
        return TVEGPU_OK;
    });
}

// Closed-loop iteration with the host copies overlapped with the step (single
// partition): the source upload runs on the side stream while K1 computes (only K2
// reads the sources), and the temperature read-back runs there while K3/K4 compute
// (T is final after K2).  Only the displacement read-back follows the step.
tvegpu_status tvegpu_step_io(tvegpu_engine* h, const double* power, int64_t n, double* T, double* u) {
    TVEGPU_RANGE();
    if (!h || n < 1) return TVEGPU_E_ARG;
    if (h->plan.nranks != 1 || h->plan.N != h->N_global || h->prm.motion) {  // no overlap: partitions, motion pins
        tvegpu_status st = power ? tvegpu_set_nodal_sources(h, power) : TVEGPU_OK;
        if (st == TVEGPU_OK) st = tvegpu_step(h, n);
        if (st == TVEGPU_OK && (T || u)) st = tvegpu_make_snapshot(h, T, u);
        return st;
    }
    return guard(h, [&] {
        if (h->halted) {
            h->err = "engine halted by an earlier failure; reset the state with tvegpu_set_state";
            return h->last_status;
        }
        const int N = h->plan.N;
        if (power) {
            if (!h->d_pw) h->d_pw = dalloc<double>(h->owned, (size_t)N);
            h->source_override = true;
            // steps still queued from tvegpu_enqueue_steps read the old sources: the
            // side stream rewrites them only after the work already on the main stream
            CU(cudaEventRecord(h->ev_entry, h->s));
            CU(cudaStreamWaitEvent(h->sc, h->ev_entry, 0));
            CU(cudaMemcpyAsync(h->d_pw, power, (size_t)N * 8, cudaMemcpyHostToDevice, h->sc));
            k_orig_to_local<<<blocks(N, 256), 256, 0, h->sc>>>(h->d_pw, h->ptr.node_orig, N,
                                                                const_cast<double*>(h->ptr.qr));
            CU(cudaEventRecord(h->ev_src, h->sc));
        }
        begin_pending(h);
        // K2 / K4 of the last step write T / u straight into the I/O buffer in original
        // numbering (no renumbering kernel on the tail); modes without that kernel
        // renumber the unchanged field from the records instead
        double* dT = io_buffer(h);
        double* du = dT + N;
        const bool thermal = h->mode != TVEGPU_MECHANICAL_ONLY, mech = h->mode != TVEGPU_THERMAL_ONLY;
        auto one = [&](bool first, bool last) {
            refresh_sources_if_needed(h, h->host_time);
            enqueue_one_step(h, nullptr, first && power ? h->ev_src : nullptr, last && T ? h->ev_T : nullptr,
                             last && T && thermal ? dT : nullptr, last && u && mech ? du : nullptr);
            h->host_time += h->dt;
            h->host_step += 1;
        };
        one(true, n == 1);
        if (n > 2) enqueue_steps(h->solo, n - 2);
        if (n > 1) one(false, true);
        const bool early_status = h->plan.nranks == 1;
        if (early_status) enqueue_status_read(h);  // before the u read-back: no extra tail
        if (T) {
            CU(cudaStreamWaitEvent(h->sc, h->ev_T, 0));  // recorded after K2 (T final)
            if (!thermal) {
                const double4* rc = h->cur ? h->ptr.rec1 : h->ptr.rec0;
                k_fields_to_orig<<<blocks(N, 256), 256, 0, h->sc>>>(rc, h->ptr.node_orig, N, dT, nullptr);
            }
            CU(cudaMemcpyAsync(T, dT, (size_t)N * 8, cudaMemcpyDeviceToHost, h->sc));
        }
        if (u && mech && h->io_cut.size() > 2) {
            // each K4 slice's completion releases the original-id prefix it finished: the
            // read-back of u overlaps the remaining slices (same side stream as T, in order)
            int done = 0;
            for (size_t k = 0; k + 1 < h->io_cut.size(); ++k) {
                const int upto = h->io_done[k];
                if (upto <= done) continue;
                CU(cudaStreamWaitEvent(h->sc, h->ev_u[k], 0));
                CU(cudaMemcpyAsync(u + 3 * (size_t)done, du + 3 * (size_t)done, (size_t)3 * (upto - done) * 8,
                                   cudaMemcpyDeviceToHost, h->sc));
                done = upto;
            }
        } else if (u) {
            if (!mech) {
                const double4* rc = h->cur ? h->ptr.rec1 : h->ptr.rec0;
                k_fields_to_orig<<<blocks(N, 256), 256, 0, h->s>>>(rc, h->ptr.node_orig, N, nullptr, du);
            }
            CU(cudaMemcpyAsync(u, du, (size_t)3 * N * 8, cudaMemcpyDeviceToHost, h->s));
        }
        CU(cudaGetLastError());
        CU(cudaStreamSynchronize(h->sc));
        h->last_status = sync_and_check(h->solo, early_status);
        return h->last_status;
    });
}

// ---- checkpoint / restart (engine.hpp:110-111) ----
// Layout (little-endian, documented in DESIGN.md): header, then T[N], u[3N],
// u_prev[3N], viscous[E][P][9] (row-major 3x3), and power[N] when a nodal-source
// override is active — all in original numbering, so a checkpoint written by one
// partitioning loads into any other.
namespace {
struct CkptHeader {
    char magic[8];  // "TVEGPUCK"
    int32_t version, kind, N, E, P, has_sources;
    int64_t step;
    double time;
};
uint64_t ckpt_bytes(const tvegpu_engine* h) {
    const uint64_t N = h->N_global, E = h->E_global, P = h->P;
    return sizeof(CkptHeader) + 8 * (N + 3 * N + 3 * N + 9 * P * E + (h->source_override ? N : 0));
}
}  // namespace

tvegpu_status tvegpu_checkpoint_size(tvegpu_engine* h, uint64_t* bytes) {
    if (!h || !bytes) return TVEGPU_E_ARG;
    *bytes = ckpt_bytes(h);
    return TVEGPU_OK;
}

namespace {
// State image of a partitioned set in original numbering, assembled on the device:
// every part writes the raw bits of the nodes it owns (the lowest rank touching a
// node; replicas are bit-identical anyway) and of its elements' viscous history into
// a zeroed global-size word buffer; an all-reduce(max) over u64 through the set's
// transport (NCCL, or the loopback group) then leaves the full image on every part
// (each word has exactly one writer or is 0).  Layout (words):
//   T[Ng] u[3 Ng] u_prev[3 Ng] power[Ng] theta[Eg][P][6]
__global__ void k_image_nodes(const double4* __restrict__ rc, const double4* __restrict__ rp,
                              const double* __restrict__ qr, const int32_t* __restrict__ node_orig,
                              const uint8_t* __restrict__ owned, int N, size_t Ng, unsigned long long* __restrict__ img) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N || !owned[i]) return;
    const size_t o = (size_t)node_orig[i];
    const double4 a = rc[i], b = rp[i];
    auto w = [](double v) { return (unsigned long long)__double_as_longlong(v); };
    img[o] = w(a.w);
    img[Ng + 3 * o] = w(a.x), img[Ng + 3 * o + 1] = w(a.y), img[Ng + 3 * o + 2] = w(a.z);
    img[4 * Ng + 3 * o] = w(b.x), img[4 * Ng + 3 * o + 1] = w(b.y), img[4 * Ng + 3 * o + 2] = w(b.z);
    img[7 * Ng + o] = w(qr[i]);
}
__global__ void k_image_elems(const double* __restrict__ theta, const int32_t* __restrict__ elem_orig, int E, int es,
                              int P, unsigned long long* __restrict__ img_th) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    const size_t o = (size_t)elem_orig[e];
    for (int p = 0; p < P; ++p)
        for (int c = 0; c < 6; ++c)
            img_th[(o * P + p) * 6 + c] = (unsigned long long)__double_as_longlong(theta[((size_t)p * 6 + c) * es + e]);
}

// Fills the host image of a partitioned set (every part's buffer holds it after the
// all-reduce; parts[0]'s is read back).  Collective over the NCCL ranks.
void gather_state_image(Stepper& S, std::vector<unsigned long long>& out) {
    tvegpu_engine* h0 = S.parts[0];
    const size_t Ng = h0->N_global, Eg = h0->E_global, P = h0->P;
    // nodes: T, u, u_prev, power (8 words/node) first, then theta (6 P / element)
    const size_t nwords = 8 * Ng + 6 * P * Eg;
    std::vector<unsigned long long*> bufs;
    try {
        for (tvegpu_engine* h : S.parts) {
            check_state_valid(h);
            void* d = nullptr;
            CU(cudaMalloc(&d, nwords * 8));
            bufs.push_back(static_cast<unsigned long long*>(d));
            CU(cudaMemsetAsync(d, 0, nwords * 8, h->s));
            const double4* rc = h->cur ? h->ptr.rec1 : h->ptr.rec0;
            const double4* rp = h->cur ? h->ptr.rec0 : h->ptr.rec1;
            if (!h->d_owned) h->d_owned = dupload(h->owned, h->plan.node_owned, h->s);
            if (h->plan.N)
                k_image_nodes<<<blocks(h->plan.N, 256), 256, 0, h->s>>>(rc, rp, h->ptr.qr, h->ptr.node_orig, h->d_owned,
                                                                        h->plan.N, Ng, bufs.back());
            if (P && h->plan.E)
                k_image_elems<<<blocks(h->plan.E, 256), 256, 0, h->s>>>(h->ptr.theta, h->ptr.elem_orig, h->plan.E,
                                                                        h->prm.es, (int)P,
                                                                        bufs.back() + 8 * Ng);
            CU(cudaGetLastError());
        }
        h0->tx->allreduce_u64(S.parts, bufs, nwords, /*max=*/true);
        out.resize(nwords);
        CU(cudaMemcpyAsync(out.data(), bufs[0], nwords * 8, cudaMemcpyDeviceToHost, h0->s));
        for (tvegpu_engine* h : S.parts) CU(cudaStreamSynchronize(h->s));
    } catch (...) {
        for (auto* b : bufs) cudaFree(b);
        throw;
    }
    for (auto* b : bufs) cudaFree(b);
}

// Writes the checkpoint (header + T, u, u_prev, viscous[E][P][9], power) of a set.
void write_checkpoint(Stepper& S, void* buf) {
    tvegpu_engine* h = S.parts[0];
    const size_t N = h->N_global, E = h->E_global, P = h->P;
    CkptHeader hd{};
    std::memcpy(hd.magic, "TVEGPUCK", 8);
    hd.version = 1, hd.kind = h->kind, hd.N = (int32_t)N, hd.E = (int32_t)E, hd.P = (int32_t)P;
    hd.has_sources = h->source_override ? 1 : 0;
    hd.step = h->host_step;
    hd.time = h->host_time;
    char* o = static_cast<char*>(buf);
    std::memcpy(o, &hd, sizeof hd);
    double* T = reinterpret_cast<double*>(o + sizeof hd);
    double* u = T + N;
    double* up = u + 3 * N;
    double* vis = up + 3 * N;
    double* pw = vis + 9 * P * E;
    if (!partitioned(S)) {
        read_fields(h, T, u, up);
        if (P) {
            const tvegpu_status st = tvegpu_get_viscous(h, vis);
            if (st != TVEGPU_OK) throw Error(st, h->err);
        }
        if (h->source_override) {
            std::vector<double> q(N);
            CU(cudaMemcpyAsync(q.data(), h->ptr.qr, N * 8, cudaMemcpyDeviceToHost, h->s));
            CU(cudaStreamSynchronize(h->s));
            for (size_t i = 0; i < N; ++i) pw[h->plan.node_orig[i]] = q[i];
        }
        return;
    }
    std::vector<unsigned long long> img;
    gather_state_image(S, img);
    std::memcpy(T, img.data(), 7 * N * 8);  // T, u, u_prev are contiguous in both layouts
    static const int map9[9] = {0, 3, 5, 3, 1, 4, 5, 4, 2};
    const unsigned long long* th = img.data() + 8 * N;
#pragma omp parallel for schedule(static)
    for (size_t e = 0; e < E; ++e)
        for (size_t p = 0; p < P; ++p)
            for (int q = 0; q < 9; ++q) std::memcpy(vis + (e * P + p) * 9 + q, th + (e * P + p) * 6 + map9[q], 8);
    if (h->source_override) std::memcpy(pw, img.data() + 7 * N, N * 8);
}
}  // namespace

// Single-partition engines read their state directly; a partitioned engine (one NCCL
// rank) gathers the image over NCCL — collective: every rank calls it and every rank
// receives the same image.
tvegpu_status tvegpu_save_checkpoint(tvegpu_engine* h, void* buf, uint64_t bytes) {
    TVEGPU_RANGE();
    if (!h || !buf) return TVEGPU_E_ARG;
    if (bytes < ckpt_bytes(h)) {
        h->err = "checkpoint buffer too small (tvegpu_checkpoint_size)";
        return TVEGPU_E_ARG;
    }
    return guard(h, [&] {
        write_checkpoint(h->solo, buf);
        return TVEGPU_OK;
    });
}

namespace {
// Validates a checkpoint image against an engine's problem; fills the field pointers.
tvegpu_status parse_checkpoint(tvegpu_engine* h, const void* buf, uint64_t bytes, CkptHeader& hd,
                               const double*& T, const double*& vis) {
    if (bytes < sizeof hd) {
        h->err = "checkpoint truncated";
        return TVEGPU_E_IO;
    }
    std::memcpy(&hd, buf, sizeof hd);
    if (std::memcmp(hd.magic, "TVEGPUCK", 8) != 0 || hd.version != 1) {
        h->err = "not a version-1 tvegpu checkpoint";
        return TVEGPU_E_IO;
    }
    if (hd.kind != h->kind || hd.N != h->N_global || hd.E != h->E_global || hd.P != h->P) {
        h->err = "checkpoint does not match this problem (element kind, node/element/Prony counts)";
        return TVEGPU_E_IO;
    }
    const uint64_t N = hd.N, E = hd.E, P = hd.P;
    const uint64_t need = sizeof hd + 8 * (7 * N + 9 * P * E + (hd.has_sources ? N : 0));
    if (bytes < need) {
        h->err = "checkpoint truncated";
        return TVEGPU_E_IO;
    }
    T = reinterpret_cast<const double*>(static_cast<const char*>(buf) + sizeof hd);
    vis = T + 7 * N;
    return TVEGPU_OK;
}
}  // namespace

// Loads into any partitioning: each partition takes its nodes and elements from the
// original-numbering image (tvegpu_set_state).
tvegpu_status tvegpu_load_checkpoint(tvegpu_engine* h, const void* buf, uint64_t bytes) {
    TVEGPU_RANGE();
    if (!h || !buf) return TVEGPU_E_ARG;
    CkptHeader hd;
    const double *T = nullptr, *vis = nullptr;
    tvegpu_status st = parse_checkpoint(h, buf, bytes, hd, T, vis);
    if (st != TVEGPU_OK) return st;
    const uint64_t N = hd.N, E = hd.E, P = hd.P;
    st = tvegpu_set_state(h, T, T + N, T + 4 * N, P ? vis : nullptr, hd.time, hd.step);
    if (st == TVEGPU_OK) st = tvegpu_set_nodal_sources(h, hd.has_sources ? vis + 9 * P * E : nullptr);
    return st;
}

tvegpu_status tvegpu_get_summary(tvegpu_engine* h, tvegpu_summary* out) {
    TVEGPU_RANGE();
    if (!h || !out) return TVEGPU_E_ARG;
    return guard(h, [&] {
        const int nb = red_blocks(h->plan.N);
        const int op[7] = {1, 2, 2, 2, 1, 1, 1};
        const double4* rc = h->cur ? h->ptr.rec1 : h->ptr.rec0;
        reduce_to_host<7>(h, nb, op, [&](double* part) {
            k_summary<<<nb, kRedThreads, 0, h->s>>>(rc, h->plan.N, part);
        });
        out->steps = h->host_step;
        out->time = h->host_time;
        out->max_temperature = h->h_part[0];
        for (int c = 0; c < 3; ++c) {
            out->min_disp[c] = h->h_part[1 + c];
            out->max_disp[c] = h->h_part[4 + c];
        }
        return TVEGPU_OK;
    });
}

tvegpu_status tvegpu_ablation_volume(tvegpu_engine* h, double threshold, int32_t deformed, double* volume,
                                     int64_t* elements_above) {
    TVEGPU_RANGE();
    if (!h || !volume || !std::isfinite(threshold)) return TVEGPU_E_ARG;
    return guard(h, [&] {
        if (!h->d_conn) {
            h->d_conn = dalloc<int32_t>(h->owned, h->plan.conn.size());
            CU(cudaMemcpyAsync(h->d_conn, h->plan.conn.data(), h->plan.conn.size() * 4, cudaMemcpyHostToDevice, h->s));
        }
        const int E = h->plan.E, nb = red_blocks(E);
        const int op[2] = {0, 0};
        const double4* rc = h->cur ? h->ptr.rec1 : h->ptr.rec0;
        reduce_to_host<2>(h, nb, op, [&](double* part) {
            if (h->nn == 8)
                k_ablation<8><<<nb, kRedThreads, 0, h->s>>>(h->d_conn, h->ptr.X, rc, E, threshold, deformed ? 1 : 0, part);
            else
                k_ablation<4><<<nb, kRedThreads, 0, h->s>>>(h->d_conn, h->ptr.X, rc, E, threshold, deformed ? 1 : 0, part);
        });
        *volume = h->h_part[0];
        if (elements_above) *elements_above = (int64_t)llround(h->h_part[1]);
        return TVEGPU_OK;
    });
}

tvegpu_status tvegpu_total_energy(tvegpu_engine* h, double* kinetic, double* strain) {
    TVEGPU_RANGE();
    if (!h || (!kinetic && !strain)) return TVEGPU_E_ARG;
    return guard(h, [&] {
        if (!h->d_conn) {
            h->d_conn = dalloc<int32_t>(h->owned, h->plan.conn.size());
            CU(cudaMemcpyAsync(h->d_conn, h->plan.conn.data(), h->plan.conn.size() * 4, cudaMemcpyHostToDevice, h->s));
        }
        const int nb = red_blocks(std::max(h->plan.E, h->plan.N));
        const int op[2] = {0, 0};
        const double4* rc = h->cur ? h->ptr.rec1 : h->ptr.rec0;
        const double4* rp = h->cur ? h->ptr.rec0 : h->ptr.rec1;
        reduce_to_host<2>(h, nb, op, [&](double* part) {
            if (h->nn == 8) k_energy<8><<<nb, kRedThreads, 0, h->s>>>(h->prm, h->ptr, h->d_conn, rc, rp, part);
            else k_energy<4><<<nb, kRedThreads, 0, h->s>>>(h->prm, h->ptr, h->d_conn, rc, rp, part);
        });
        if (kinetic) *kinetic = h->h_part[0];
        if (strain) *strain = h->h_part[1];
        return TVEGPU_OK;
    });
}

tvegpu_status tvegpu_element_fields(tvegpu_engine* h, double* det_f, double* max_principal_stress) {
    TVEGPU_RANGE();
    if (!h || (!det_f && !max_principal_stress)) return TVEGPU_E_ARG;
    if (!h->prm.diag) {
        h->err = "element fields need options.diagnostics = 1 (F and S of the last mechanics phase)";
        return TVEGPU_E_ARG;
    }
    if (h->plan.nranks != 1 || h->plan.E != h->E_global) {
        h->err = "element fields are read on single-partition engines";
        return TVEGPU_E_ARG;
    }
    return guard(h, [&] {
        const int E = h->plan.E;
        if (!h->d_ef) h->d_ef = dalloc<double>(h->owned, (size_t)2 * E);
        double* d = h->d_ef;
        k_element_fields<<<blocks(E, 256), 256, 0, h->s>>>(h->ptr.diag_F, h->ptr.diag_S, h->ptr.elem_orig, E,
                                                             det_f ? d : nullptr, max_principal_stress ? d + E : nullptr);
        CU(cudaGetLastError());
        if (det_f) CU(cudaMemcpyAsync(det_f, d, (size_t)E * 8, cudaMemcpyDeviceToHost, h->s));
        if (max_principal_stress)
            CU(cudaMemcpyAsync(max_principal_stress, d + E, (size_t)E * 8, cudaMemcpyDeviceToHost, h->s));
        CU(cudaStreamSynchronize(h->s));
        return TVEGPU_OK;
    });
}

tvegpu_status tvegpu_get_diagnostics(tvegpu_engine* h, double* f_int, double* F, double* S) {
    if (!h) return TVEGPU_E_ARG;
    if (!h->prm.diag) {
        h->err = "diagnostics need options.diagnostics = 1";
        return TVEGPU_E_ARG;
    }
    return guard(h, [&] {
        const int E = h->plan.E, N = h->plan.N;
        std::vector<double> buf((size_t)9 * std::max(E, N));
        // on the engine stream: steps enqueued by tvegpu_enqueue_steps may still write these
        auto copy = [&](const double* src, size_t n) {
            CU(cudaMemcpyAsync(buf.data(), src, n * 8, cudaMemcpyDeviceToHost, h->s));
            CU(cudaStreamSynchronize(h->s));
        };
        if (f_int) {
            copy(h->ptr.diag_f, (size_t)3 * N);
            for (int i = 0; i < N; ++i)
                for (int c = 0; c < 3; ++c) f_int[3 * (size_t)h->plan.node_orig[i] + c] = buf[3 * (size_t)i + c];
        }
        for (int k = 0; k < 2; ++k) {
            double* dst = k == 0 ? F : S;
            if (!dst) continue;
            copy(k == 0 ? h->ptr.diag_F : h->ptr.diag_S, (size_t)9 * E);
            for (int e = 0; e < E; ++e)
                for (int q = 0; q < 9; ++q) dst[9 * (size_t)h->plan.elem_orig[e] + q] = buf[9 * (size_t)e + q];
        }
        return TVEGPU_OK;
    });
}

tvegpu_status tvegpu_last_error(const tvegpu_engine* h, char* msg, size_t cap, int64_t* step, int32_t* node) {
    if (!h) return TVEGPU_E_ARG;
    if (msg && cap) {
        std::strncpy(msg, h->err.c_str(), cap - 1);
        msg[cap - 1] = 0;
    }
    if (step) *step = h->err_step;
    if (node) *node = h->err_node;
    return h->last_status;
}

tvegpu_status tvegpu_critical_timestep(const tvegpu_problem* p, double* thermal, double* mechanical) {
    if (!p || !thermal || !mechanical) return TVEGPU_E_ARG;
    try {
        validate_problem(*p);
        critical_timestep(*p, thermal, mechanical);
    } catch (const Error& e) {
        g_create_error = e.what();
        return e.status;
    }
    return TVEGPU_OK;
}

// ---------------------------------------------------------------- plan (host only)
struct tvegpu_plan {
    RankPlan r;
};

tvegpu_status tvegpu_plan_create(const tvegpu_problem* p, int32_t nranks, int32_t rank, int32_t reorder,
                                 tvegpu_plan** out) {
    if (!p || !out) return TVEGPU_E_ARG;
    try {
        GlobalMesh g = build_global(*p);
        auto* pl = new tvegpu_plan();
        pl->r = build_rank_plan(*p, g, nranks, rank, reorder);
        *out = pl;
    } catch (const Error& e) {
        g_create_error = e.what();
        return e.status;
    } catch (const std::exception& e) {
        g_create_error = e.what();
        return TVEGPU_E_ARG;
    }
    return TVEGPU_OK;
}

tvegpu_status tvegpu_plan_get(const tvegpu_plan* pl, tvegpu_plan_view* v) {
    if (!pl || !v) return TVEGPU_E_ARG;
    const RankPlan& r = pl->r;
    v->nranks = r.nranks;
    v->rank = r.rank;
    v->nn = r.nn;
    v->num_elements = r.E;
    v->num_boundary_elements = r.Eb;
    v->num_nodes = r.N;
    v->element_orig = r.elem_orig.data();
    v->node_orig = r.node_orig.data();
    v->conn = r.conn.data();
    v->csr_offsets = r.csr_off.data();
    v->csr_slots = r.csr_slot.data();
    v->num_neighbors = (int32_t)r.neighbors.size();
    v->neighbor_ranks = r.neighbors.data();
    v->send_offsets = r.send_off.data();
    v->send_slots = r.send_slot.data();
    v->recv_offsets = r.recv_off.data();
    v->element_owner = r.owner.data();
    v->num_elements_global = (int32_t)r.owner.size();
    v->num_chunks = (int32_t)r.chunk_start.size() - 1;
    v->chunk_start = r.chunk_start.data();
    v->chunk_node_off = r.chunk_node_off.data();
    v->chunk_nodes = r.chunk_nodes.data();
    v->chunk_node_slot = r.chunk_node_slot.data();
    v->chunk_conn = r.lconn.data();
    v->max_chunk_slots = r.max_chunk_nodes;
    return TVEGPU_OK;
}

void tvegpu_plan_destroy(tvegpu_plan* p) { delete p; }

tvegpu_status tvegpu_nccl_unique_id(void* out128) {
    if (!out128) return TVEGPU_E_ARG;
    try {
        ncclUniqueId id;
        NC(nccl().GetUniqueId(&id));
        std::memcpy(out128, &id, sizeof id);
    } catch (const Error& e) {
        g_create_error = e.what();
        return e.status;
    }
    return TVEGPU_OK;
}

tvegpu_status tvegpu_peer_export(tvegpu_engine* h, void* blob, size_t cap, size_t* len) {
    if (!h || !len) return TVEGPU_E_ARG;
    return guard(h, [&] {
        const RankPlan& pl = h->plan;
        if (pl.nranks < 2) throw Error(TVEGPU_E_ARG, "tvegpu_peer_export: not a partitioned engine (nranks == 1)");
        const size_t nn = pl.neighbors.size();
        const size_t need = sizeof(PeerBlobHead) + (2 * nn + 1) * sizeof(int32_t);
        *len = need;
        if (!blob) return TVEGPU_OK;  // size query
        if (cap < need) throw Error(TVEGPU_E_ARG, "tvegpu_peer_export: buffer too small");
        PeerBlobHead hd{};
        hd.magic = kPeerMagic;
        hd.rank = pl.rank;
        hd.nnbr = (int32_t)nn;
        hd.abi = TVEGPU_ABI_VERSION;
        CU(cudaIpcGetMemHandle(&hd.th, h->ptr.slot_th));
        CU(cudaIpcGetMemHandle(&hd.m, h->ptr.slot_m));
        CU(cudaIpcGetMemHandle(&hd.inbox, h->ptr.inbox));
        hd.off_th = (uint64_t)((char*)recv_area(h, false) - (char*)h->ptr.slot_th);
        hd.off_m = (uint64_t)((char*)recv_area(h, true) - (char*)h->ptr.slot_m);
        char* b = static_cast<char*>(blob);
        std::memcpy(b, &hd, sizeof hd);
        std::memcpy(b + sizeof hd, pl.neighbors.data(), nn * sizeof(int32_t));
        std::memcpy(b + sizeof hd + nn * sizeof(int32_t), pl.recv_off.data(), (nn + 1) * sizeof(int32_t));
        return TVEGPU_OK;
    });
}

tvegpu_status tvegpu_peer_attach(tvegpu_engine* h, const void* const* blobs, const size_t* lens, int32_t nranks) {
    if (!h || !blobs || !lens) return TVEGPU_E_ARG;
    return guard(h, [&] {
        const RankPlan& pl = h->plan;
        if (nranks != pl.nranks) throw Error(TVEGPU_E_ARG, "tvegpu_peer_attach: one descriptor per rank expected");
        if (h->peer) throw Error(TVEGPU_E_ARG, "tvegpu_peer_attach: already attached");
        if (h->pending) {
            const tvegpu_status st = sync_and_check(h->solo);
            if (st != TVEGPU_OK) return st;
        }
        std::vector<PeerDesc> by_rank(nranks);
        for (int r : pl.neighbors) {  // only the neighbours' buffers are mapped
            if (!blobs[r] || lens[r] < sizeof(PeerBlobHead)) throw Error(TVEGPU_E_ARG, "tvegpu_peer_attach: short descriptor");
            PeerBlobHead hd;
            std::memcpy(&hd, blobs[r], sizeof hd);
            const size_t nn = hd.nnbr < 0 ? 0 : (size_t)hd.nnbr;
            if (hd.magic != kPeerMagic || hd.rank != r || hd.abi != TVEGPU_ABI_VERSION ||
                lens[r] < sizeof hd + (2 * nn + 1) * sizeof(int32_t))
                throw Error(TVEGPU_E_ARG, "tvegpu_peer_attach: bad descriptor of rank " + std::to_string(r));
            PeerDesc& d = by_rank[r];
            d.rank = r;
            const char* b = static_cast<const char*>(blobs[r]);
            d.nbr.assign(reinterpret_cast<const int32_t*>(b + sizeof hd), reinterpret_cast<const int32_t*>(b + sizeof hd) + nn);
            const int32_t* ro = reinterpret_cast<const int32_t*>(b + sizeof hd + nn * sizeof(int32_t));
            d.recv_off.assign(ro, ro + nn + 1);
            void *pth = nullptr, *pm = nullptr, *pin = nullptr;
            CU(cudaIpcOpenMemHandle(&pth, hd.th, cudaIpcMemLazyEnablePeerAccess));
            h->ipc_open.push_back(pth);
            CU(cudaIpcOpenMemHandle(&pm, hd.m, cudaIpcMemLazyEnablePeerAccess));
            h->ipc_open.push_back(pm);
            CU(cudaIpcOpenMemHandle(&pin, hd.inbox, cudaIpcMemLazyEnablePeerAccess));
            h->ipc_open.push_back(pin);
            d.th = reinterpret_cast<double*>(static_cast<char*>(pth) + hd.off_th);
            d.m = reinterpret_cast<double*>(static_cast<char*>(pm) + hd.off_m);
            d.inbox = static_cast<unsigned long long*>(pin);
        }
        peer_attach(h, by_rank);
        return TVEGPU_OK;
    });
}

int32_t tvegpu_halo_peer(const tvegpu_engine* h) { return h && h->peer ? 1 : 0; }

tvegpu_status tvegpu_peer_attach_solo(tvegpu_engine* h) {
    if (!h) return TVEGPU_E_ARG;
    return guard(h, [&] {
        const RankPlan& pl = h->plan;
        if (pl.nranks < 2 || h->peer) throw Error(TVEGPU_E_ARG, "tvegpu_peer_attach_solo: unattached partition expected");
        if (!dynamic_cast<SoloTransport*>(h->tx))
            throw Error(TVEGPU_E_ARG, "tvegpu_peer_attach_solo: create the partition without an NCCL id");
        // every neighbour is a scratch area on this device; the partition's own waits pass at once
        int32_t most = 1;
        for (size_t j = 0; j + 1 < pl.send_off.size(); ++j) most = std::max(most, pl.send_off[j + 1] - pl.send_off[j]);
        double* sth = dalloc<double>(h->owned, most);
        double* sm = dalloc<double>(h->owned, (size_t)kMW * most);
        unsigned long long* sin = dalloc<unsigned long long>(h->owned, 2);
        std::vector<PeerDesc> by_rank(pl.nranks);
        for (size_t j = 0; j < pl.neighbors.size(); ++j) {
            PeerDesc& d = by_rank[pl.neighbors[j]];
            d.rank = pl.neighbors[j];
            d.th = sth;
            d.m = sm;
            d.inbox = sin;
            d.nbr = {pl.rank};
            d.recv_off = {0, pl.send_off[j + 1] - pl.send_off[j]};
        }
        peer_attach(h, by_rank);
        if (std::getenv("TVEGPU_SOLO_NOFWD")) h->prm.nb_chunks = 0;  // (measurement: the ordering alone)
        CU(cudaMemsetAsync(h->ptr.inbox, 0xff, 2 * std::max<size_t>(1, pl.neighbors.size()) * 8, h->s));
        CU(cudaStreamSynchronize(h->s));
        return TVEGPU_OK;
    });
}

tvegpu_status tvegpu_peer_detach(tvegpu_engine* h) {
    if (!h) return TVEGPU_E_ARG;
    return guard(h, [&] {
        if (h->pending) {
            const tvegpu_status st = sync_and_check(h->solo);
            if (st != TVEGPU_OK) return st;
        }
        CU(cudaStreamSynchronize(h->s));
        for (auto& kv : h->solo.graphs) CU(cudaGraphExecDestroy(kv.second));  // captured with the peer path
        h->solo.graphs.clear();
        for (void* p : h->ipc_open) CU(cudaIpcCloseMemHandle(p));
        h->ipc_open.clear();
        h->peer = false;
        h->prm.npeers = 0;
        h->prm.ack = 0;
        h->prm.nb_chunks = 0;
        h->pdl = false;  // the NCCL path's pack kernel is not PDL-aware
        return TVEGPU_OK;
    });
}

void* tvegpu_stream(tvegpu_engine* h) { return h ? (void*)h->s : nullptr; }

tvegpu_status tvegpu_halo_info(const tvegpu_engine* h, int32_t* neighbors, int64_t* send_bytes, int64_t* recv_bytes) {
    if (!h) return TVEGPU_E_ARG;
    const RankPlan& pl = h->plan;
    const int64_t ns = pl.send_off.empty() ? 0 : pl.send_off.back(), nr = pl.recv_off.empty() ? 0 : pl.recv_off.back();
    int64_t per = 0;  // values per contribution and step: 1 thermal + kMW mechanical, per coupled phase
    if (h->mode != TVEGPU_MECHANICAL_ONLY) per += 1;
    if (h->mode != TVEGPU_THERMAL_ONLY) per += kMW;
    if (neighbors) *neighbors = (int32_t)pl.neighbors.size();
    if (send_bytes) *send_bytes = (int64_t)h->slot_bytes() * per * ns;
    if (recv_bytes) *recv_bytes = (int64_t)h->slot_bytes() * per * nr;
    return TVEGPU_OK;
}

int32_t tvegpu_affine_chunks(const tvegpu_engine* h) { return h ? h->n_affine_chunks : 0; }

int32_t tvegpu_kernels_per_step(const tvegpu_engine* h) {
    if (!h) return 0;
    const bool multi = h->plan.nranks > 1;
    // per phase: element kernel + node kernel; partitioned: boundary and interior element
    // launches, plus the halo pack with the NCCL transport (peer memory: none)
    const int per = multi ? (h->peer ? 2 : 4) : 2;
    int k = 0;
    if (h->mode != TVEGPU_MECHANICAL_ONLY) k += per;
    if (h->mode != TVEGPU_THERMAL_ONLY) k += per;
    return k;
}

tvegpu_status tvegpu_profile_kernels(tvegpu_engine* h, int32_t nsteps, double* ms, int32_t* count, char* names,
                                     size_t cap) {
    if (!h || nsteps <= 0 || !ms || !count) return TVEGPU_E_ARG;
    return guard(h, [&] {
        if (h->halted) return h->last_status;
        if (h->pending) {
            h->last_status = sync_and_check(h->solo);
            if (h->last_status != TVEGPU_OK) return h->last_status;
        }
        std::vector<std::string> nm;
        if (h->mode != TVEGPU_MECHANICAL_ONLY) {
            nm.push_back(h->nn == 4 ? "k_thermal_element<4>" : "k_thermal_element<8>");
            nm.push_back("k_thermal_node");
        }
        if (h->mode != TVEGPU_THERMAL_ONLY) {
            nm.push_back(h->nn == 4 ? "k_mech_element<4>" : "k_mech_element<8>");
            nm.push_back("k_mech_node");
        }
        // (the end-of-step verdict runs inside the last node kernel)
        const int nk = (int)nm.size();
        const bool part = partitioned(h->solo);
        std::vector<cudaEvent_t> ev((size_t)(nk + 1) * nsteps), xev(part ? (size_t)4 * nsteps : 0);
        for (auto& e : ev) CU(cudaEventCreate(&e));
        for (auto& e : xev) CU(cudaEventCreate(&e));
        // partitioned engines: the marks bracket the phases (element kernels + pack +
        // exchange enqueue, then the wait for the halo + node kernel)
        begin_pending(h);
        for (int k = 0; k < nsteps; ++k) {
            refresh_sources_if_needed(h, h->host_time);
            if (h->prm.motion) upload_motion(h);
            if (part)
                enqueue_partitioned_step(h->solo, ev.data() + (size_t)k * (nk + 1), xev.data() + (size_t)4 * k);
            else enqueue_one_step(h, ev.data() + (size_t)k * (nk + 1));
            h->host_time += h->dt;
            h->host_step += 1;
        }
        tvegpu_status st = sync_and_check(h->solo);
        std::vector<double> acc(nk, 0.0);
        for (int k = 0; k < nsteps; ++k)
            for (int j = 0; j < nk; ++j) {
                float t = 0;
                CU(cudaEventElapsedTime(&t, ev[(size_t)k * (nk + 1) + j], ev[(size_t)k * (nk + 1) + j + 1]));
                acc[j] += t;
            }
        // partitioned: the halo transfers (thermal, mechanical) on the comm stream
        double xacc[2] = {0.0, 0.0};
        const bool th = h->mode != TVEGPU_MECHANICAL_ONLY, me = h->mode != TVEGPU_THERMAL_ONLY;
        for (int k = 0; k < nsteps && part; ++k)
            for (int q = 0; q < 2; ++q) {
                if ((q == 0 && !th) || (q == 1 && !me)) continue;
                float t = 0;
                CU(cudaEventElapsedTime(&t, xev[(size_t)4 * k + 2 * q], xev[(size_t)4 * k + 2 * q + 1]));
                xacc[q] += t;
            }
        for (auto& e : ev) cudaEventDestroy(e);
        for (auto& e : xev) cudaEventDestroy(e);
        std::string all;
        for (int j = 0; j < nk; ++j) {
            ms[j] = acc[j] / nsteps;
            all += (j ? ";" : "") + nm[j];
        }
        int cnt = nk;
        if (part) {
            if (th) ms[cnt++] = xacc[0] / nsteps, all += ";halo_exchange_thermal";
            if (me) ms[cnt++] = xacc[1] / nsteps, all += ";halo_exchange_mech";
        }
        *count = cnt;
        if (names && cap) {
            std::strncpy(names, all.c_str(), cap - 1);
            names[cap - 1] = 0;
        }
        return st;
    });
}

}  // extern "C"

// ---------------------------------------------------------------- partition group (loopback transport)
// P RCB partitions of one problem, each a full partition engine with its own compute
// and comm streams, stepped by the same code as one NCCL rank per GPU
// (enqueue_partitioned_step, CUDA-graph capture, verdict agreement, state gather);
// only the transport differs: device copies of each neighbour's packed send segment
// into the receive area, ordered by the same ev_pack / ev_comm events, in place of
// ncclSend / ncclRecv.  Results are bit-identical to a single partition.
struct tvegpu_group {
    std::vector<tvegpu_engine*> parts;
    Stepper st;
    LoopbackTransport tx;
    std::string err;
    tvegpu_status last_status = TVEGPU_OK;
};

namespace {
template <class F>
tvegpu_status group_guard(tvegpu_group* G, F&& f) {
    try {
        const tvegpu_status st = f();
        if (st != TVEGPU_OK) {
            G->last_status = st;
            for (tvegpu_engine* h : G->parts)
                if (!h->err.empty()) {
                    G->err = h->err;
                    break;
                }
        }
        return st;
    } catch (const Error& e) {
        G->err = e.what();
        G->last_status = e.status;
        return e.status;
    } catch (const std::exception& e) {
        G->err = e.what();
        return TVEGPU_E_ARG;
    }
}
tvegpu_status each_part(tvegpu_group* G, const std::function<tvegpu_status(tvegpu_engine*)>& f) {
    for (tvegpu_engine* h : G->parts) {
        const tvegpu_status st = f(h);
        if (st != TVEGPU_OK) {
            G->err = h->err;
            return st;
        }
    }
    return TVEGPU_OK;
}
}  // namespace

extern "C" {

tvegpu_status tvegpu_group_create(const tvegpu_problem* p, int32_t nparts, const tvegpu_options* o,
                                  tvegpu_group** out) {
    if (!p || !out || nparts < 2) return TVEGPU_E_ARG;
    *out = nullptr;
    tvegpu_options def;
    tvegpu_default_options(&def);
    if (!o) o = &def;
    auto* G = new tvegpu_group();
    try {
        for (int r = 0; r < nparts; ++r) {
            tvegpu_options oo = *o;
            oo.nranks = nparts;
            oo.rank = r;
            oo.reorder = 1;
            auto* h = new tvegpu_engine();
            G->parts.push_back(h);
            build_engine(h, *p, oo, /*loopback=*/true);
            h->tx = &G->tx;
        }
        if (o->halo_transport == TVEGPU_HALO_PEER) {  // the parts' buffers are on this device: plain pointers
            std::vector<PeerDesc> d;
            for (tvegpu_engine* h : G->parts) d.push_back(peer_desc(h));
            for (tvegpu_engine* h : G->parts) peer_attach(h, d);
        }
        G->st.parts = G->parts;
        G->st.steps_per_graph = o->steps_per_graph > 0 ? o->steps_per_graph : 64;
        CU(cudaEventCreateWithFlags(&G->st.ev_fork, cudaEventDisableTiming));
    } catch (const std::exception& e) {
        g_create_error = e.what();
        tvegpu_group_destroy(G);
        return dynamic_cast<const Error*>(&e) ? static_cast<const Error&>(e).status : TVEGPU_E_ARG;
    }
    *out = G;
    return TVEGPU_OK;
}

void tvegpu_group_destroy(tvegpu_group* G) {
    if (!G) return;
    for (tvegpu_engine* h : G->parts)
        if (h->s) cudaStreamSynchronize(h->s);
    for (auto& kv : G->st.graphs) cudaGraphExecDestroy(kv.second);
    if (G->st.ev_fork) cudaEventDestroy(G->st.ev_fork);
    for (tvegpu_engine* h : G->parts) tvegpu_destroy(h);
    delete G;
}

tvegpu_status tvegpu_group_step(tvegpu_group* G, int64_t n) {
    TVEGPU_RANGE();
    if (!G || n < 0) return TVEGPU_E_ARG;
    return group_guard(G, [&] {
        if (G->parts[0]->halted) return G->last_status;
        enqueue_steps(G->st, n);
        return sync_and_check(G->st);
    });
}

tvegpu_status tvegpu_group_get_state(tvegpu_group* G, double* T, double* disp, double* disp_prev, double* viscous) {
    if (!G) return TVEGPU_E_ARG;
    return group_guard(G, [&] {
        return each_part(G, [&](tvegpu_engine* h) {
            if (T || disp || disp_prev) {
                check_state_valid(h);
                read_fields(h, T, disp, disp_prev);
            }
            return viscous && h->P ? tvegpu_get_viscous(h, viscous) : TVEGPU_OK;
        });
    });
}

tvegpu_status tvegpu_group_get_fields(tvegpu_group* G, double* T, double* disp, double* viscous) {
    return tvegpu_group_get_state(G, T, disp, nullptr, viscous);
}

tvegpu_status tvegpu_group_set_state(tvegpu_group* G, const double* T, const double* disp, const double* disp_prev,
                                     const double* viscous, double time, int64_t step) {
    if (!G) return TVEGPU_E_ARG;
    return group_guard(G, [&] {
        const tvegpu_status st =
            each_part(G, [&](tvegpu_engine* h) { return tvegpu_set_state(h, T, disp, disp_prev, viscous, time, step); });
        if (st == TVEGPU_OK) G->last_status = TVEGPU_OK;
        return st;
    });
}

tvegpu_status tvegpu_group_set_nodal_sources(tvegpu_group* G, const double* power) {
    if (!G) return TVEGPU_E_ARG;
    return group_guard(G, [&] { return each_part(G, [&](tvegpu_engine* h) { return tvegpu_set_nodal_sources(h, power); }); });
}

// The partitioned form of tvegpu_step_io (what one NCCL rank runs): sources, n steps,
// snapshot of T and u in original numbering.
tvegpu_status tvegpu_group_step_io(tvegpu_group* G, const double* power, int64_t n, double* T, double* disp) {
    if (!G || n < 1) return TVEGPU_E_ARG;
    tvegpu_status st = power ? tvegpu_group_set_nodal_sources(G, power) : TVEGPU_OK;
    if (st == TVEGPU_OK) st = tvegpu_group_step(G, n);
    if (st == TVEGPU_OK && (T || disp)) st = tvegpu_group_get_state(G, T, disp, nullptr, nullptr);
    return st;
}

double tvegpu_group_time(const tvegpu_group* G) { return G ? G->parts[0]->host_time : 0.0; }
int64_t tvegpu_group_step_count(const tvegpu_group* G) { return G ? G->parts[0]->host_step : 0; }

tvegpu_status tvegpu_group_last_error(const tvegpu_group* G, char* msg, size_t cap, int64_t* step, int32_t* node) {
    if (!G) return TVEGPU_E_ARG;
    if (msg && cap) {
        std::strncpy(msg, G->err.c_str(), cap - 1);
        msg[cap - 1] = 0;
    }
    if (step) *step = G->parts[0]->err_step;
    if (node) *node = G->parts[0]->err_node;
    return G->last_status;
}

tvegpu_status tvegpu_group_checkpoint_size(tvegpu_group* G, uint64_t* bytes) {
    return G ? tvegpu_checkpoint_size(G->parts[0], bytes) : TVEGPU_E_ARG;
}

tvegpu_status tvegpu_group_save_checkpoint(tvegpu_group* G, void* buf, uint64_t bytes) {
    TVEGPU_RANGE();
    if (!G || !buf) return TVEGPU_E_ARG;
    if (bytes < ckpt_bytes(G->parts[0])) {
        G->err = "checkpoint buffer too small (tvegpu_group_checkpoint_size)";
        return TVEGPU_E_ARG;
    }
    return group_guard(G, [&] {
        write_checkpoint(G->st, buf);
        return TVEGPU_OK;
    });
}

tvegpu_status tvegpu_group_load_checkpoint(tvegpu_group* G, const void* buf, uint64_t bytes) {
    TVEGPU_RANGE();
    if (!G || !buf) return TVEGPU_E_ARG;
    return group_guard(G, [&] {
        const tvegpu_status st =
            each_part(G, [&](tvegpu_engine* h) { return tvegpu_load_checkpoint(h, buf, bytes); });
        if (st == TVEGPU_OK) G->last_status = TVEGPU_OK;
        return st;
    });
}

}  // extern "C"
