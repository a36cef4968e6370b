// plan.hpp — host-side setup for the B200 TLED step: validation, the
// compressed precompute, element/node reordering, the deterministic gather CSR
// and (for nranks > 1) the RCB partition with its halo lists.
//
// Replaces the reference's precompute() (mesh.hpp:81-83) for the device path.
// Unlike the reference layout (3 x nn gradients per element, stored 4 x 8
// hourglass basis), the device keeps only A_e (G_e = A_e Xi, 9 doubles) and V_e
// per element; per-node sums (lumped mass, volume) are
// accumulated once on the GLOBAL mesh in canonical adjacency order (ascending
// original element, then local index; mesh.hpp:58-61) so every partition sees
// bit-identical node constants.
#pragma once

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "../../include/tvegpu.h"

namespace tvegpu {

// Setup-stage timing to stderr when TVEGPU_TIMING is set.
struct StageTimer {
    const char* name;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit StageTimer(const char* n) : name(n) {}
    ~StageTimer() {
        static const bool on = std::getenv("TVEGPU_TIMING") != nullptr;
        if (on)
            std::fprintf(stderr, "[tvegpu setup] %-28s %8.1f ms\n", name,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
};

// Lap timer inside one stage: lap("name") reports the time since the previous lap.
struct LapTimer {
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void operator()(const char* name) {
        static const bool on = std::getenv("TVEGPU_TIMING") != nullptr;
        const auto now = std::chrono::steady_clock::now();
        if (on)
            std::fprintf(stderr, "[tvegpu setup]   %-26s %8.1f ms\n", name,
                         std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

// std::vector whose resize leaves trivially constructible elements uninitialised, so
// large setup arrays are first touched by the parallel loops that fill them (a zeroing
// resize of a 128M-entry array is a serial memset of half a gigabyte).
template <class T, class A = std::allocator<T>>
struct default_init_allocator : A {
    using A::A;
    template <class U>
    struct rebind {
        using other = default_init_allocator<U, typename std::allocator_traits<A>::template rebind_alloc<U>>;
    };
    template <class U>
    void construct(U* p) noexcept(std::is_nothrow_default_constructible<U>::value) {
        ::new (static_cast<void*>(p)) U;
    }
    template <class U, class... Args>
    void construct(U* p, Args&&... args) {
        std::allocator_traits<A>::construct(static_cast<A&>(*this), p, std::forward<Args>(args)...);
    }
};
template <class T>
using fvec = std::vector<T, default_init_allocator<T>>;

struct Error : std::runtime_error {
    Error(tvegpu_status s, const std::string& m) : std::runtime_error(m), status(s) {}
    tvegpu_status status;
};

// Reference corner signs (H8 brick order) and T4 reference gradients.
extern const int kH8Sign[8][3];
extern const int kT4Xi[4][3];
extern const int kHg[4][8];

struct GlobalMesh {
    int kind = TVEGPU_T4, nn = 4, N = 0, E = 0;
    fvec<double> vol;              // per element (T4: V; H8: 8 det J0)
    fvec<double> centroid;         // 3 per element
    fvec<double> mass;             // per node: sum rho V_e / nn (canonical order)
    fvec<double> vnode;            // per node: sum V_e / nn (canonical order)
    fvec<int32_t> adj_off;         // node -> (element, local): canonical CSR over original ids
    fvec<int32_t> adj_elem, adj_local;
    double lo[3], hi[3];           // bounding box of element centroids
    double min_edge = 0;           // smallest element edge length (Morton lattice spacing)
};

// Validates the problem (the reference's ValidationError cases) and builds the
// global compressed precompute.  Throws Error.
void validate_problem(const tvegpu_problem& p);
GlobalMesh build_global(const tvegpu_problem& p);

// Morton key of a centroid: round((c - lo) * scale) per axis, 21 bits each;
// scale = 1 / (smallest element edge), capped so the extent fits 21 bits.
uint64_t morton_key(const double* c, const double* lo, double scale);
double morton_scale(const GlobalMesh& g);

// Deterministic recursive coordinate bisection of element centroids into nranks parts.
std::vector<int32_t> rcb_partition(const GlobalMesh& g, int nranks);

struct RankPlan {
    int nranks = 1, rank = 0, nn = 4;
    int E = 0, Eb = 0, N = 0;
    std::vector<int32_t> elem_orig;   // local -> original element
    std::vector<int32_t> node_orig;   // local -> original node
    fvec<int32_t> conn;               // nn * E, element-major, local node ids
    fvec<int32_t> csr_off;            // N + 1
    fvec<int32_t> csr_slot;           // local slot (e*nn + a) or nn*E + receive index
    std::vector<int32_t> neighbors;
    std::vector<int32_t> send_off, send_slot, recv_off;
    std::vector<int32_t> owner;       // global element -> rank
    std::vector<uint8_t> node_owned;  // N: 1 if this rank is the lowest one touching the node
    // Element chunks (one CTA each): <= kChunk consecutive local elements, never
    // straddling the boundary/interior split; each chunk's unique nodes are
    // staged in shared memory and elements address them by a 16-bit index.
    std::vector<int32_t> chunk_start;     // nchunks + 1
    std::vector<int32_t> chunk_node_off;  // nchunks + 1
    std::vector<int32_t> chunk_nodes;     // unique local node ids per chunk, ascending
    std::vector<uint16_t> chunk_node_slot;  // shared-memory slot of each chunk_nodes entry
    fvec<uint16_t> lconn;                 // E * nn, element-major: slot of node (e, a) in its chunk
    int nchunks_boundary = 0;             // chunks [0, nchunks_boundary) cover [0, Eb)
    int max_chunk_nodes = 0;              // max shared-memory slots (incl. colour padding) of a chunk
};

#ifndef TVEGPU_CHUNK
#define TVEGPU_CHUNK 128  // elements per chunk = threads per element-kernel CTA (kernels.cuh kChunkThreads)
#endif
constexpr int kChunk = TVEGPU_CHUNK;

// Fills the chunk fields of a plan (called by build_rank_plan).
void build_chunks(RankPlan& r);

// Builds one rank's plan.  reorder = 0 keeps the original element and node order
// (single rank only); otherwise Morton element order (boundary elements first)
// and first-touch node order.
RankPlan build_rank_plan(const tvegpu_problem& p, const GlobalMesh& g, int nranks, int rank, int reorder);

// Critical timestep (mesh.hpp:92-97).  The problem must be validated
// first (element indices are dereferenced unchecked).
void critical_timestep(const tvegpu_problem& p, double* thermal, double* mechanical);
// The same from the smallest element edge L (GlobalMesh::min_edge, same arithmetic).
void critical_timestep_from_edge(const tvegpu_problem& p, double L, double* thermal, double* mechanical);

}  // namespace tvegpu
