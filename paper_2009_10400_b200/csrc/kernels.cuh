// kernels.cuh — the sm_100a kernels of one TLED step.
//
//   K1 k_thermal_element<NN>   F from u^n, element-mean T^n -> D(T), conduction load
//                              V det F B^T D B T_e (Eqs. 16/18/19; bioheat.hpp:37-47)
//   K2 k_thermal_node          deterministic CSR gather + Eq. 20 (bioheat.hpp:49-63)
//   K3 k_mech_element<NN,EXP>  F_ther (Eq. 11), total PK2 (Eqs. 8-10), Prony (Eq. 28),
//                              f = V F S~ G plus closed-form H8 hourglass
//                              (materials.hpp:99-127; mechanics.hpp:55-84)
//   K4 k_mech_node             CSR gather + Eq. 22 central difference + BCs
//                              (mechanics.hpp:86-97)
//   The last node kernel of the step also closes it: the last block to finish
//   applies the finite-check verdict and advances t and the step counter
//   (engine.hpp:89-90, 120), so a step is 4 launches.
//
// fp64 throughout (north_star parity <= 1e-10).  One thread per element / node.
// Node state is a packed 32-byte record (ux, uy, uz, T), so an element gathers one
// sector per node.  The element geometry (A_e with G_e = A_e Xi, V_e and the H8
// hourglass vectors c_al = X h_al) is computed once by k_geometry and stored SoA
// with the other per-element rows (Prony history, fibres, axes); an element kernel
// pulls its chunk's rows into shared memory with TMA bulk copies.
// Assembly is a gather in canonical (original element, local) order — one
// thread per node in order (H8), or two threads each summing one half and then
// their sum (T4, > 8 contributions per node) — with a tree chosen from the
// global mesh: no float atomics, results bit-identical at any partition count.
// The only atomics are integer atomicMin on the error words and the end-of-step
// ticket.
#pragma once

#include <cassert>
#include <cstdint>
#include <cuda_runtime.h>

namespace tvegpu {

constexpr int kMaxTable = 16;  // table entries held in the launch parameters (longer tables: D.tabs)
constexpr int kMaxProny = 4;   // Prony terms with coefficients in the launch parameters and staged history rows
#ifndef TVEGPU_CHUNK
#define TVEGPU_CHUNK 128
#endif
constexpr int kChunkThreads = TVEGPU_CHUNK;  // element kernels: one thread per element of a chunk (plan.hpp kChunk)
// Mechanical slot record: packed (fx, fy, fz), 24 bytes.  An element's NN records are
// 32-byte aligned as a block (96 / 192 bytes): T4 writes them with three 256-bit
// stores, H8 with one 256-bit + one 128-bit store per corner pair; a node reads a
// record as one 16-byte + one 8-byte load.  25 % fewer slot bytes than padded 32-byte
// records (one 256-bit store / load each): K3 -11 %, K4 -9 % on cfg4.
// TVEGPU_MW=4 builds the padded layout.
#ifndef TVEGPU_MW
#define TVEGPU_MW 3
#endif
constexpr int kMW = TVEGPU_MW;

#ifndef TVEGPU_TMA_ROWS
#define TVEGPU_TMA_ROWS 3  // per-element rows into shared memory by cp.async.bulk: bit 0 K1, bit 1 K3 (else L1 prefetch)
#endif
constexpr bool kTmaK1 = (TVEGPU_TMA_ROWS & 1) != 0, kTmaK3 = (TVEGPU_TMA_ROWS & 2) != 0;
// K3 rebuilds A, V (and the H8 hourglass vectors) from a bulk-copied block of the chunk's
// node coordinates instead of reading the stored geometry rows: bit 0 T4, bit 1 H8.
// T4 chunks hold few nodes (~9 B of coordinates per element against 80 B of rows); H8
// chunks save more bytes but the rebuild's FP64 work and register pressure cost more
// than they save (K3 cfg4 120.6 vs 109.1 us, measured).
#ifndef TVEGPU_K3_XSTAGE
#define TVEGPU_K3_XSTAGE 1
#endif
template <int NN>
__host__ __device__ constexpr bool k3_xstage() { return kTmaK3 && (TVEGPU_K3_XSTAGE & (NN == 4 ? 1 : 2)) != 0; }
// The same choice for K1 (A and V only).
#ifndef TVEGPU_K1_XSTAGE
#define TVEGPU_K1_XSTAGE 1
#endif
template <int NN>
__host__ __device__ constexpr bool k1_xstage() { return kTmaK1 && (TVEGPU_K1_XSTAGE & (NN == 4 ? 1 : 2)) != 0; }

struct Clock {
    double time;
    long long step;
    int halted;
    unsigned ticket;  // end-of-step block counter of the closing node kernel
};

struct DevParams {
    int nn, E, N, P, mode, td, exp_kind, fiber_mode, axes_per_elem, has_R, diag, nslots;
    int max_chunk_nodes;  // shared-memory stride of the staged node records
    int stage_stride;     // entries per chunk in stage_ent (max unique nodes of a chunk)
    int ell;              // G > 0: ELL gathers with rows of 8 G slot ids (every node has <= 8 G contributions)
    int motion;           // MechBCs::motion_override active (host-evaluated pins, K4 reads motion_row/val)
    int npeers;           // peer-memory halo (nranks > 1): neighbours whose inbox flags the node kernels wait for
    int ack;              // ... single-physics mode: element kernels' boundary chunks also wait for the neighbours' end-of-step acks
    int drop_signal;      // fault injection (TVEGPU_HALO_DROP_RANK): this partition's boundary chunks raise no flags
    unsigned long long halo_timeout_ns;  // bound of every peer-memory wait (TVEGPU_HALO_TIMEOUT_MS, default 20 s)
    int es;               // row stride of the per-element SoA arrays (geo, theta, fiber, axes): >= E + 1, 16-aligned
    int xstride;          // doubles per chunk in chunk_x (3 * even max_chunk_nodes)
    double dt, mu, kappa, eta_a, kh, rho, wbcb, Ta, Qm, gamma;
    double inv_2dt, inv_dt2;  // 1/(2 dt), 1/dt^2 (Eq. 22 coefficients)
    double fiber[3];
    double c_fixed;
    double k_fixed[9];
    int c_len, k_len;
    double cT[kMaxTable], cV[kMaxTable], kT[kMaxTable], kK[kMaxTable][9];
    double alpha_i, alpha_m, alpha_n, Tref;
    double axis_m[3], axis_n[3];
    double pa[kMaxProny], pb[kMaxProny];
    // offsets into DevPtrs::tabs (every table and all Prony coefficients, any length); the
    // kernels read them from there only when c_len / k_len > kMaxTable or P > kMaxProny
    int tab_cT, tab_cV, tab_kT, tab_kK, tab_pa, tab_pb;
    int affine_all;       // H8: every element affine (hourglass geometry c_al = 0): K3 stages no c_al rows
    int nb_chunks;        // boundary chunks [0, nb_chunks): the element-kernel CTAs that forward and signal (0: no peers)
    int halo_hi;          // local nodes [0, halo_hi) hold every node that gathers received contributions
};

struct DevPtrs {
    const int32_t* chunk_start;     // [nchunks + 1] first local element of each 128-element chunk
    const int32_t* chunk_node_off;  // [nchunks + 1]
    const int32_t* chunk_nodes;     // unique local nodes of each chunk (ascending)
    const uint16_t* chunk_node_slot;  // their shared-memory slots
    const uint16_t* lconn;          // [E][nn] index of node (e, a) in its chunk's node list
    const int2* stage_ent;          // [nchunks][stage_stride] {local node, shared slot}, {-1, 0} padded
    const double* chunk_x;          // [nchunks][xstride] per chunk its nodes' coordinates by shared slot: x[S], y[S], z[S]
    const int32_t* chunk_xs;        // [nchunks] S: slots used (even)
    const double* geo;              // [kGeoRows][es] A (9, row-major), V, H8: c_al = X h_al (12)
    double* theta;             // [P][6][es]   (xx, yy, zz, xy, yz, xz)
    const double* fiber;       // [3][es] or null
    const double* axes;        // [6][es] or null
    const int32_t* elem_orig;  // [E]
    double4* rec0;             // node record (ux, uy, uz, T), two rotating buffers
    double4* rec1;
    const double4* X;          // [N] reference coordinates (x, y, z, 0)
    const double* mass;        // [N]
    const double* vnode;       // [N]
    const double* qr;          // [N] lumped nodal source power
    const uint8_t* mask;       // [N] bit0 fixed, bit1..3 prescribed x/y/z, bit4 fixed T
    const int32_t* bc_index;   // [N] -> row of the BC tables (masked nodes only)
    const int32_t* bc_presc;   // [nbc][3] prescribed entry id or -1
    const double* bc_tfix;     // [nbc]
    const double* presc_target;
    const double* presc_ramp;
    const double* R;           // [N][3] external + body force, or null
    const int32_t* csr_off;    // [N+1]
    const int32_t* csr_slot;   // gather list: element-major slot ids (e*nn + a, or receive area)
    const int4* ell;           // [N][8 G] the same lists padded with a zero sentinel slot (ell = G > 0)
    const int32_t* node_orig;  // [N]
    double* slot_th;           // [nslots]
    double* slot_m;            // [nslots][kMW] (fx, fy, fz[, pad])
    Clock* clock;
    unsigned long long* err_inst;  // (step << 33) | (field << 32) | orig node
    unsigned long long* err_elem;  // (step << 32) | orig element
    double* diag_F;            // [E][9] or null
    double* diag_S;            // [E][9] or null
    double* diag_f;            // [N][3] or null
    const int32_t* motion_row;  // [N] row of motion_val for override candidates, else -1 (motion only)
    const double4* motion_val;  // [rows] (x, y, z, pinned) of this step's motion_override(node, t + dt)
    const double* tabs;         // c(T), k(T) tables and Prony coefficients (DevParams::tab_*)
    const uint8_t* chunk_affine;  // H8: per chunk 1 if all its elements are affine (c_al rows not staged)
    // peer-memory halo (nranks > 1, DevParams::npeers > 0): see peer_forward / peer_signal / peer_wait
    const int32_t* pd_off;                 // [Eb nn + 1] per boundary slot (e nn + a) its destinations
    const uint32_t* pd_ent;                // (neighbour << 26) | index in that neighbour's receive area
    double* const* peer_th;                // [npeers] the neighbours' thermal receive areas
    double* const* peer_m;                 // [npeers] mechanical receive areas (kMW doubles per entry)
    unsigned long long* const* peer_flag;  // [npeers] this partition's flag word in each neighbour's inbox
    unsigned long long* inbox;             // [npeers] flags raised by the neighbours
    unsigned* send_cnt;                    // [2] boundary CTAs done in the running send kernel (per phase)
    unsigned long long* epoch;             // steps enqueued since creation (never reset): flag sequence base
    unsigned long long* err_halo;          // first step whose halo wait timed out, else ~0
    unsigned long long* ack_inbox;         // [npeers] neighbours' completed steps (DevParams::ack)
    unsigned long long* const* peer_ack;   // [npeers] this partition's word in each neighbour's ack_inbox
};

enum : uint8_t { BC_FIXED = 1, BC_PX = 2, BC_PY = 4, BC_PZ = 8, BC_TFIX = 16 };

// ------------------------------------------------------------------ small fp64 algebra
__device__ __forceinline__ double interp1(const double* Ts, const double* Vs, int n, double T) {
    if (n == 1 || T <= Ts[0]) return Vs[0];
    if (T >= Ts[n - 1]) return Vs[n - 1];
    int j = 0;
    while (j + 2 < n && T >= Ts[j + 1]) ++j;
    const double w = (T - Ts[j]) / (Ts[j + 1] - Ts[j]);
    return Vs[j] + (Vs[j + 1] - Vs[j]) * w;
}

// k(T) at the element-mean temperature from tables (T_j) and (K_j, 9 each)
__device__ __forceinline__ void conductivity_interp(const double* kT, const double* kK, int n, double T, double D[9]) {
    if (n == 1 || T <= kT[0]) {
#pragma unroll
        for (int q = 0; q < 9; ++q) D[q] = kK[q];
        return;
    }
    if (T >= kT[n - 1]) {
#pragma unroll
        for (int q = 0; q < 9; ++q) D[q] = kK[9 * (n - 1) + q];
        return;
    }
    int j = 0;
    while (j + 2 < n && T >= kT[j + 1]) ++j;
    const double w = (T - kT[j]) / (kT[j + 1] - kT[j]);
#pragma unroll
    for (int q = 0; q < 9; ++q) D[q] = kK[9 * j + q] + (kK[9 * (j + 1) + q] - kK[9 * j + q]) * w;
}
// ConductivityTable::at / ScalarTable::at (materials.hpp:39-65): short tables from the
// launch parameters, any longer one from device memory (same arithmetic)
__device__ __forceinline__ void conductivity_at(const DevParams& P, const DevPtrs& D, double T, double Dk[9]) {
    if (P.k_len <= kMaxTable) conductivity_interp(P.kT, &P.kK[0][0], P.k_len, T, Dk);
    else conductivity_interp(D.tabs + P.tab_kT, D.tabs + P.tab_kK, P.k_len, T, Dk);
}
__device__ __forceinline__ double heat_capacity_at(const DevParams& P, const DevPtrs& D, double T) {
    return P.c_len <= kMaxTable ? interp1(P.cT, P.cV, P.c_len, T)
                                : interp1(D.tabs + P.tab_cT, D.tabs + P.tab_cV, P.c_len, T);
}

// adjugate (transpose of cofactors) of a row-major 3x3, returns det
__device__ __forceinline__ double adj3(const double m[9], double a[9]) {
    a[0] = m[4] * m[8] - m[5] * m[7];
    a[1] = m[2] * m[7] - m[1] * m[8];
    a[2] = m[1] * m[5] - m[2] * m[4];
    a[3] = m[5] * m[6] - m[3] * m[8];
    a[4] = m[0] * m[8] - m[2] * m[6];
    a[5] = m[2] * m[3] - m[0] * m[5];
    a[6] = m[3] * m[7] - m[4] * m[6];
    a[7] = m[1] * m[6] - m[0] * m[7];
    a[8] = m[0] * m[4] - m[1] * m[3];
    return m[0] * a[0] + m[1] * a[3] + m[2] * a[6];
}

__device__ __forceinline__ unsigned long long pack_inst(long long step, int field, int node) {
    return ((unsigned long long)step << 33) | ((unsigned long long)field << 32) | (unsigned)node;
}
__device__ __forceinline__ unsigned long long pack_elem(long long step, int elem) {
    return ((unsigned long long)step << 32) | (unsigned)elem;
}

// One 256-bit read-only load (sm_100 LDG.E.256): a 32-byte node record in one
// request/sector instead of two 128-bit requests.
__device__ __forceinline__ double4 ldg4(const double4* p) {
    double4 v;
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
    return v;
}
// 256-bit coherent load (data written earlier in the same step by another kernel is fine
// with .nc too, but records this kernel itself writes must not use the read-only path)
__device__ __forceinline__ double4 ld4(const double4* p) {
    double4 v;
    asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void st4(double4* p, const double4& v) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w)
                 : "memory");
}

// H8 corner signs (standard brick order) and hourglass vectors.
__device__ __forceinline__ constexpr int h8s(int a, int j) {
    return ((j == 0) ? ((a == 1 || a == 2 || a == 5 || a == 6) ? 1 : -1)
                     : (j == 1) ? ((a == 2 || a == 3 || a == 6 || a == 7) ? 1 : -1) : (a >= 4 ? 1 : -1));
}
__device__ __forceinline__ constexpr int h8h(int al, int a) {
    // h1 = eta*zeta, h2 = zeta*xi, h3 = xi*eta, h4 = xi*eta*zeta
    return al == 0 ? h8s(a, 1) * h8s(a, 2)
                   : al == 1 ? h8s(a, 2) * h8s(a, 0) : al == 2 ? h8s(a, 0) * h8s(a, 1) : h8s(a, 0) * h8s(a, 1) * h8s(a, 2);
}

// A chunk's nodes staged in shared memory as two 16-byte planes, (ux, uy) and
// (uz, T), indexed by colour-assigned slot (plan.cpp colour_slots): each
// quarter-warp's 16-byte reads of node a hit 8 distinct bank groups.
struct NodeStage {
    double2* a;
    double2* b;
    __device__ __forceinline__ double4 rec(int n) const {
        const double2 p = a[n], q = b[n];
        return make_double4(p.x, p.y, q.x, q.y);
    }
};

// ------------------------------------------------------------------ per-element rows by TMA
// A chunk's per-element SoA rows (geometry, Prony history, per-element fibres / axes)
// are contiguous 128-element segments: row stride P.es (a multiple of 16 elements)
// and even chunk starts (plan.cpp) make each segment a 16-byte-aligned bulk copy.  At
// kernel start one warp issues one cp.async.bulk per row into shared memory (none of
// these rows is written by the predecessor kernel, so before the PDL wait), completing
// on one mbarrier; the element threads read their column after the node staging.
// This replaces per-thread L1 prefetches + global loads of every row.
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init_expect(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_row(double* dst, const double* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait0(unsigned long long* bar) {
    asm volatile(
        "{\n .reg .pred p;\n TMA_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        " @!p bra TMA_WAIT_%=;\n}" ::"r"(smem_addr(bar)) : "memory");
}

// Rows of one element kernel: [0, ngeo) geometry, then 6 P Prony history, then 3
// fibre and 6 expansion-axis rows when those are per element.
constexpr int kGeoRows = 22;  // A (9), V, H8 hourglass geometry c_al = X h_al (12)
struct RowPlan {
    int ngeo, ntheta, nfib, nax;
    __host__ __device__ __forceinline__ int total() const { return ngeo + ntheta + nfib + nax; }
    __host__ __device__ __forceinline__ int theta0() const { return ngeo; }
    __host__ __device__ __forceinline__ int fib0() const { return ngeo + ntheta; }
    __host__ __device__ __forceinline__ int ax0() const { return ngeo + ntheta + nfib; }
};

// The element rows of this thread's chunk: shared memory (TMA) or global (L1 prefetch).
template <bool TMA>
struct ElemRows {
    const double* s;  // [rows][kChunkThreads] (TMA)
    int t;            // element within the chunk
    // row r of the shared block, or element e of global row g
    __device__ __forceinline__ double get(int r, const double* g) const {
        if constexpr (TMA) return s[r * kChunkThreads + t];
        else return __ldg(g);
    }
};

// Warp 0: issue the chunk's row copies (or, without TMA, every thread prefetches its
// rows into L1).  e0 = first element of the chunk, ne = its element count.
// skip_hg: an affine H8 chunk — its hourglass rows [10, kGeoRows) are zero, not copied.
template <bool TMA>
__device__ __forceinline__ void load_elem_rows(const DevParams& P, const DevPtrs& D, const RowPlan& rp, int e0, int ne,
                                               double* rows, unsigned long long* bar, double* blob = nullptr,
                                               const double* blob_src = nullptr, unsigned blob_bytes = 0,
                                               bool skip_hg = false) {
    const int R = rp.total();
    const int hg0 = skip_hg && rp.ngeo == kGeoRows ? 10 : R, hg1 = skip_hg && rp.ngeo == kGeoRows ? kGeoRows : R;
    auto src = [&](int r) -> const double* {
        if (r < rp.theta0()) return D.geo + (size_t)r * P.es;
        if (r < rp.fib0()) return D.theta + (size_t)(r - rp.theta0()) * P.es;
        if (r < rp.ax0()) return D.fiber + (size_t)(r - rp.fib0()) * P.es;
        return D.axes + (size_t)(r - rp.ax0()) * P.es;
    };
    if constexpr (TMA) {
        if (threadIdx.x >= 32) return;
        const unsigned bytes = (unsigned)((ne + 1) & ~1) * 8u;  // even: 16-byte multiple (rows are padded)
        if (threadIdx.x == 0) mbar_init_expect(bar, bytes * (unsigned)(R - (hg1 - hg0)) + blob_bytes);
        __syncwarp();
        for (int r = threadIdx.x; r < R; r += 32)
            if (r < hg0 || r >= hg1) tma_row(rows + r * kChunkThreads, src(r) + e0, bytes, bar);
        if (blob_bytes && threadIdx.x == 31) tma_row(blob, blob_src, blob_bytes, bar);
    } else if ((int)threadIdx.x < ne) {
        for (int r = 0; r < R; ++r)
            if (r < hg0 || r >= hg1) asm volatile("prefetch.global.L1 [%0];" ::"l"(src(r) + e0 + threadIdx.x));
    }
}
template <bool TMA>
__device__ __forceinline__ void wait_elem_rows(unsigned long long* bar) {
    if constexpr (TMA) mbar_wait0(bar);
}

// Dynamic shared memory of an element kernel: [mbarrier | pad to 128 B][rows][2 staged planes].
constexpr int kRowsOffset = 128;

// Reference geometry from the element's corner coordinates, in exactly the
// arithmetic order of element_pass: J (T4: edge matrix; H8: X Xi^T / 8), A = J^-T
// (H8: / 8), V; and for H8 the hourglass geometry c_al = X h_al in corner order.
template <int NN>
__global__ void k_geometry(const double4* __restrict__ X, const int32_t* __restrict__ conn, int E, int es, int rows,
                           double* geo, uint8_t* __restrict__ affine) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    double J[9];
    if constexpr (NN == 4) {
        const double4 x0 = X[conn[(size_t)e * 4]];
#pragma unroll
        for (int a = 1; a < 4; ++a) {
            const double4 x = X[conn[(size_t)e * 4 + a]];
            J[0 * 3 + a - 1] = x.x - x0.x;
            J[1 * 3 + a - 1] = x.y - x0.y;
            J[2 * 3 + a - 1] = x.z - x0.z;
        }
    } else {
        double cX[4][3];
#pragma unroll
        for (int q = 0; q < 9; ++q) J[q] = 0.0;
#pragma unroll
        for (int al = 0; al < 4; ++al) cX[al][0] = cX[al][1] = cX[al][2] = 0.0;
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const double4 x = X[conn[(size_t)e * 8 + a]];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const double s = (double)h8s(a, j);
                J[0 * 3 + j] += s * x.x;
                J[1 * 3 + j] += s * x.y;
                J[2 * 3 + j] += s * x.z;
            }
#pragma unroll
            for (int al = 0; al < 4; ++al) {
                const double h = (double)h8h(al, a);
                cX[al][0] += h * x.x;
                cX[al][1] += h * x.y;
                cX[al][2] += h * x.z;
            }
        }
#pragma unroll
        for (int q = 0; q < 9; ++q) J[q] = J[q] / 8.0;
        if (rows > 10) {
            // affine element (parallelepiped: X h_al = 0 up to the rounding of the corner sums,
            // |c_al| <= 1e-12 of the element size): exact zeros, so K3 need not stage the rows
            const double L = cbrt(fabs(8.0 * (J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
                                             J[2] * (J[3] * J[7] - J[4] * J[6]))));
            double cm = 0.0;
#pragma unroll
            for (int al = 0; al < 4; ++al)
#pragma unroll
                for (int i = 0; i < 3; ++i) cm = fmax(cm, fabs(cX[al][i]));
            const bool aff = affine && cm <= 1e-12 * L;  // (affine == nullptr: no detection)
#pragma unroll
            for (int al = 0; al < 4; ++al)
#pragma unroll
                for (int i = 0; i < 3; ++i) geo[(size_t)(10 + al * 3 + i) * es + e] = aff ? 0.0 : cX[al][i];
            if (affine) affine[e] = aff ? 1 : 0;
        }
    }
    double Ad[9];
    const double dJ = adj3(J, Ad);
    const double s = (NN == 4 ? 1.0 : 0.125) / dJ;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) geo[(size_t)(i * 3 + j) * es + e] = Ad[j * 3 + i] * s;
    geo[(size_t)9 * es + e] = NN == 4 ? dJ * (1.0 / 6.0) : 8.0 * dJ;
}

// Element kinematics from one pass over the element's staged nodes:
//   H = U Xi^T (displacement sums), Ts = sum T, gT = Xi T_e (thermal only);
//   A (G_e = A Xi) and V from the geometry rows.
template <int NN, bool WANT_GT, bool TMA, bool SUMS_ONLY = false>
__device__ __forceinline__ void element_pass(const NodeStage& S, const int (&n)[NN], const DevParams& P,
                                             const DevPtrs& D, const ElemRows<TMA>& rows, int e, double H[9],
                                             double A[9], double& V, double& Ts, double gT[3]) {
    if constexpr (NN == 4) {
        const double4 r0 = S.rec(n[0]);
        Ts = r0.w;
#pragma unroll
        for (int a = 1; a < 4; ++a) {
            const double4 r = S.rec(n[a]);
            H[0 * 3 + a - 1] = r.x - r0.x;
            H[1 * 3 + a - 1] = r.y - r0.y;
            H[2 * 3 + a - 1] = r.z - r0.z;
            if constexpr (WANT_GT) gT[a - 1] = r.w - r0.w;
            Ts += r.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < 9; ++q) H[q] = 0.0;
        if constexpr (WANT_GT) gT[0] = gT[1] = gT[2] = 0.0;
        Ts = 0.0;
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const double4 r = S.rec(n[a]);
            Ts += r.w;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const double s = (double)h8s(a, j);
                H[0 * 3 + j] += s * r.x;
                H[1 * 3 + j] += s * r.y;
                H[2 * 3 + j] += s * r.z;
                if constexpr (WANT_GT) gT[j] += s * r.w;
            }
        }
    }
    if constexpr (SUMS_ONLY) return;
    // ptxas would hoist these shared-memory reads up into the record loads above and
    // spill (584 B at K3's 128 registers); a CTA-scope fence keeps them after the sums
    if constexpr (TMA) __threadfence_block();
#pragma unroll
    for (int q = 0; q < 9; ++q) A[q] = rows.get(q, D.geo + (size_t)q * P.es + e);
    V = rows.get(9, D.geo + (size_t)9 * P.es + e);
}

// The chunk's node coordinates in shared memory by slot (k3_xstage): x[S], y[S], z[S].
struct CoordStage {
    const double* x;
    const double* y;
    const double* z;
};
// A (G_e = A Xi) and V from the element's corner coordinates, in exactly k_geometry's
// arithmetic, so the result is bit-identical to the stored geometry rows.
template <int NN>
__device__ __forceinline__ void geometry_from_coords(const CoordStage& X, const int (&n)[NN], double A[9], double& V) {
    double J[9];
    if constexpr (NN == 4) {
        const double x0 = X.x[n[0]], y0 = X.y[n[0]], z0 = X.z[n[0]];
#pragma unroll
        for (int a = 1; a < 4; ++a) {
            J[0 * 3 + a - 1] = X.x[n[a]] - x0;
            J[1 * 3 + a - 1] = X.y[n[a]] - y0;
            J[2 * 3 + a - 1] = X.z[n[a]] - z0;
        }
    } else {
#pragma unroll
        for (int q = 0; q < 9; ++q) J[q] = 0.0;
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const double x = X.x[n[a]], y = X.y[n[a]], z = X.z[n[a]];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const double s = (double)h8s(a, j);
                J[0 * 3 + j] += s * x;
                J[1 * 3 + j] += s * y;
                J[2 * 3 + j] += s * z;
            }
        }
#pragma unroll
        for (int q = 0; q < 9; ++q) J[q] = J[q] / 8.0;
    }
    double Ad[9];
    const double dJ = adj3(J, Ad);
    const double s = (NN == 4 ? 1.0 : 0.125) / dJ;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) A[i * 3 + j] = Ad[j * 3 + i] * s;
    V = NN == 4 ? dJ * (1.0 / 6.0) : 8.0 * dJ;
}

// Programmatic dependent launch (single-partition graphs): a kernel issues the loads
// of data its immediate predecessor does not write (staging indices, coordinates,
// node constants), then waits for the predecessor grid; every kernel signals its
// dependents only after its own wait, so anything two launches back is complete
// when a kernel starts.  Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Stage one chunk: its unique nodes' (u, T) records go to shared memory once per chunk (each node is used by up to 8 of the chunk's elements),
// replacing 2*NN random 32-byte global gathers per element.  Returns this
// thread's element (or -1) and its nodes' shared-memory slots.
// The staging is latency-bound (a dependent index load, then the record loads),
// so every load is issued before any is consumed: the element's own slot indices,
// then up to kStageBatch node indices per thread, then all their records.
constexpr int kStageBatch = 3;
// L2 prefetch of the entry list a CTA about two resident waves later loads first (streamed
// from DRAM each step, at the head of the staging chain).  The same for the node kernels'
// ELL rows was slower (K2 +2 us, K4 +1 us on cfg4).
#ifndef TVEGPU_ENT_PREFETCH
#define TVEGPU_ENT_PREFETCH 1184  // element kernels: chunks ahead (0: off)
#endif
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
// The chunk's index loads, issued first thing in the kernel (before warp 0 issues the row
// copies, which wait for the chunk start): the first batch of staging entries — fixed
// stride, so its address needs no load — and this thread's element node slots.
template <int NN>
struct StageHead {
    int2 en[kStageBatch];
    uint4 w8;
    uint2 w4;
    int e;
};
template <int NN>
__device__ __forceinline__ StageHead<NN> stage_head(const DevPtrs& D, int c, const int st, int e0, int ne, int cend) {
    StageHead<NN> h;
    const int2* ent = D.stage_ent + (size_t)c * st;
    if constexpr (TVEGPU_ENT_PREFETCH > 0) {  // (cfg4 K3 -1 us, cfg5 T4 K1 / K3 -2 %)
        const int cn = c + TVEGPU_ENT_PREFETCH;
        if (cn < cend && (int)threadIdx.x < ((st * 8 + 127) >> 7)) prefetch_l2(D.stage_ent + (size_t)cn * st + threadIdx.x * 16);
    }
#pragma unroll
    for (int j = 0; j < kStageBatch; ++j) {
        const int k = j * kChunkThreads + threadIdx.x;
        h.en[j] = k < st ? __ldg(ent + k) : make_int2(-1, 0);
    }
    h.e = (int)threadIdx.x < ne ? e0 + (int)threadIdx.x : -1;
    h.w8 = make_uint4(0, 0, 0, 0);
    h.w4 = make_uint2(0, 0);
    if (h.e >= 0) {
        if constexpr (NN == 8) h.w8 = __ldg(reinterpret_cast<const uint4*>(D.lconn) + h.e);
        else h.w4 = __ldg(reinterpret_cast<const uint2*>(D.lconn) + h.e);
    }
    return h;
}
template <int NN>
__device__ __forceinline__ int stage_chunk(const DevPtrs& D, const double4* __restrict__ R, int c, const int st,
                                           const NodeStage& S, int (&n)[NN], const StageHead<NN>& h) {
    const int2* ent = D.stage_ent + (size_t)c * st;
    int2 en[kStageBatch];
#pragma unroll
    for (int j = 0; j < kStageBatch; ++j) en[j] = h.en[j];
    const int e = h.e;
    const uint4 w8 = h.w8;
    const uint2 w4 = h.w4;
    for (int k0 = 0; k0 < st; k0 += kStageBatch * kChunkThreads) {  // ascending node ids: coalesced loads
        int g[kStageBatch], s[kStageBatch];
#pragma unroll
        for (int j = 0; j < kStageBatch; ++j) {
            if (k0 > 0) {
                const int k = k0 + j * kChunkThreads + threadIdx.x;
                en[j] = k < st ? __ldg(ent + k) : make_int2(-1, 0);
            }
            g[j] = en[j].x;
            s[j] = en[j].y;
        }
        double4 r[kStageBatch];
        pdl_wait();  // the node records are the predecessor's output
#pragma unroll
        for (int j = 0; j < kStageBatch; ++j)
            if (g[j] >= 0) r[j] = ldg4(R + g[j]);
#pragma unroll
        for (int j = 0; j < kStageBatch; ++j)
            if (g[j] >= 0) {
                S.a[s[j]] = make_double2(r[j].x, r[j].y);
                S.b[s[j]] = make_double2(r[j].z, r[j].w);
            }
    }
    if constexpr (NN == 8) {
        n[0] = w8.x & 0xffff, n[1] = w8.x >> 16, n[2] = w8.y & 0xffff, n[3] = w8.y >> 16;
        n[4] = w8.z & 0xffff, n[5] = w8.z >> 16, n[6] = w8.w & 0xffff, n[7] = w8.w >> 16;
    } else {
        n[0] = w4.x & 0xffff, n[1] = w4.x >> 16, n[2] = w4.y & 0xffff, n[3] = w4.y >> 16;
    }
    __syncthreads();
    return e;
}

// ------------------------------------------------------------------ bounds-checking build
// TVEGPU_BOUNDS_CHECK=1 (csrc/Makefile `variant`, scripts/gpu_bounds_check.sh) asserts every
// index the step kernels dereference: chunk staging entries and element slots (K1/K3),
// gather lists (K2/K4).  compute-sanitizer is not available on the GPU pool; this build
// plus the parity suite stands in for memcheck.  Off: no code.
#ifndef TVEGPU_BOUNDS_CHECK
#define TVEGPU_BOUNDS_CHECK 0
#endif
template <int NN>
__device__ __forceinline__ void check_chunk(const DevParams& P, const DevPtrs& D, int c, int e, const int (&n)[NN]) {
    if constexpr (TVEGPU_BOUNDS_CHECK) {
        const int eb = D.chunk_start[c], ee = D.chunk_start[c + 1];
        assert(0 <= eb && eb <= ee && ee <= P.E && ee - eb <= kChunkThreads);
        assert(e < 0 || (eb <= e && e < ee));
        for (int k = threadIdx.x; k < P.stage_stride; k += kChunkThreads) {
            const int2 en = D.stage_ent[(size_t)c * P.stage_stride + k];
            assert(en.x >= -1 && en.x < P.N && en.y >= 0 && en.y < P.max_chunk_nodes);
        }
        if (e >= 0)
            for (int a = 0; a < NN; ++a) assert(n[a] >= 0 && n[a] < P.max_chunk_nodes);
    }
}
__device__ __forceinline__ void check_gather(const DevParams& P, const DevPtrs& D, int i) {
    if constexpr (TVEGPU_BOUNDS_CHECK) {
        const int k0 = D.csr_off[i], k1 = D.csr_off[i + 1];
        assert(0 <= k0 && k0 <= k1);
        for (int k = k0; k < k1; ++k) assert(D.csr_slot[k] >= 0 && D.csr_slot[k] < P.nslots);
        if (P.ell) {
            const int32_t* row = reinterpret_cast<const int32_t*>(D.ell) + (size_t)8 * P.ell * i;
            assert(k1 - k0 <= 8 * P.ell);
            for (int k = 0; k < 8 * P.ell; ++k)
                assert(k < k1 - k0 ? row[k] == D.csr_slot[k0 + k] : row[k] == P.nslots);
        }
    }
}

// ------------------------------------------------------------------ peer-memory halo
// In a partitioned step the boundary chunks of the element kernel forward every
// contribution another partition gathers, right after computing it, straight into that
// partition's receive area — NVLink peer memory of the
// other GPU (CUDA IPC mapping), or another partition's buffer in a group — so the
// element math and the halo transfer are one kernel (no pack kernel, no NCCL call).
// When the launch's last CTA is done it raises flag = 2 epoch + 1 + phase in each
// neighbour's inbox (release, system scope); the neighbours' node kernels wait for it
// (acquire) while the interior chunks still run.  Receive areas are reused safely
// without a second buffer: a partition's phase-p sends of step n follow its own node
// kernel of the other phase, which waited for its neighbours' sends that follow their
// reads of the receive areas (shared nodes make every halo relation symmetric).
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// the contributions (e, a) of a boundary element (W doubles each) to every partition that
// gathers them: read back from the thread's own slot stores (program order) and stored into
// the neighbours' receive areas.  Forwarding the stored bits, instead of sending from the
// element math, keeps that math — and its FMA contraction — identical to the kernel every
// other element and every single-GPU run uses: bit-identity across partitions needs it.
template <int NN, int W, typename ST>
__device__ __forceinline__ void peer_forward(const DevPtrs& D, const ST* slots, int e) {
    // every load issued up front (the element's destination offsets and its whole slot
    // block, just stored: L2 hits), then the destinations: a few dependent round trips
    // instead of a chain per corner — boundary CTAs must not stretch the launch's first wave
    int off[NN + 1];
#pragma unroll
    for (int a = 0; a <= NN; ++a) off[a] = __ldg(D.pd_off + (size_t)e * NN + a);
    ST v[NN * W];
#pragma unroll
    for (int q = 0; q < NN * W; ++q) v[q] = slots[(size_t)e * NN * W + q];  // coherent: written just above
    ST* const* base = reinterpret_cast<ST* const*>(W == 1 ? D.peer_th : D.peer_m);
#pragma unroll
    for (int a = 0; a < NN; ++a)
        for (int k = off[a]; k < off[a + 1]; ++k) {
            const uint32_t en = __ldg(D.pd_ent + k);
            ST* b = base[en >> 26] + (size_t)(en & 0x3ffffffu) * W;
#pragma unroll
            for (int q = 0; q < W; ++q) b[q] = v[a * W + q];
        }
}
// start of a boundary CTA in a single-physics partitioned step (DevParams::ack): the
// neighbours' node kernels of the previous step are done with the receive areas this
// launch overwrites.  (In coupled steps the other phase's flags already imply it.)
__device__ __forceinline__ void peer_wait_ack(const DevParams& P, const DevPtrs& D) {
    pdl_wait();  // the epoch is bumped by the predecessor (the closing node kernel)
    if (threadIdx.x == 0) {
        const unsigned long long ep = *(volatile unsigned long long*)D.epoch;
        const unsigned long long t0 = globaltimer_ns();
        for (int j = 0; j < P.npeers; ++j)
            while (ld_acquire_sys(D.ack_inbox + j) < ep) {
                if (globaltimer_ns() - t0 > P.halo_timeout_ns) {
                    atomicMin(D.err_halo, (unsigned long long)D.clock->step);
                    break;
                }
                __nanosleep(100);
            }
    }
    __syncthreads();
}
// end of a boundary CTA of an element kernel (every thread; halted partitions still signal so
// their neighbours never wait on them): the last boundary CTA raises the phase flag in each
// neighbour's inbox.  The interior chunks run in the same launch, after the boundary ones.
__device__ __forceinline__ void peer_signal(const DevParams& P, const DevPtrs& D, int phase, int c) {
    if (c >= P.nb_chunks) return;  // interior chunk of the launch (CTA-uniform)
    __syncthreads();               // the CTA's peer stores happen before thread 0's release
    if (threadIdx.x != 0) return;
    __threadfence_system();        // cumulative: orders them before the arrival and the flags
    const unsigned n = atomicAdd(D.send_cnt + phase, 1u);
    if (n != (unsigned)P.nb_chunks - 1) return;
    D.send_cnt[phase] = 0;
    __threadfence_system();
    const unsigned long long seq = 2 * *D.epoch + 1 + phase;
    if (P.drop_signal) return;
    for (int j = 0; j < P.npeers; ++j) st_release_sys(D.peer_flag[j], seq);
}
// start of a node kernel of a partitioned step: this phase's contributions from every
// neighbour have landed.  Bounded: after P.halo_timeout_ns the wait gives up and records
// the step in err_halo (the call's verdict reports it, collectively) instead of hanging.
__device__ __forceinline__ void peer_wait(const DevParams& P, const DevPtrs& D, int phase, int first_node) {
    if (P.npeers == 0 || first_node >= P.halo_hi) return;  // no received contributions in this block
    if (threadIdx.x == 0) {
        const unsigned long long seq = 2 * *(volatile unsigned long long*)D.epoch + 1 + phase;
        const unsigned long long t0 = globaltimer_ns();
        for (int j = 0; j < P.npeers; ++j)
            while (ld_acquire_sys(D.inbox + j) < seq) {
                if (globaltimer_ns() - t0 > P.halo_timeout_ns) {
                    atomicMin(D.err_halo, (unsigned long long)D.clock->step);
                    break;
                }
                __nanosleep(100);
            }
    }
    __syncthreads();
}

// ------------------------------------------------------------------ K1: thermal element
#ifdef TVEGPU_K1_MINBLOCKS
#define K1_BOUNDS __launch_bounds__(kChunkThreads, TVEGPU_K1_MINBLOCKS)
#else
#define K1_BOUNDS __launch_bounds__(kChunkThreads)
#endif
// K1 element body: element e of the staged chunk S (n = its node slots)
template <int NN, typename ST>
__device__ __forceinline__ void k1_body(const DevParams& P, const DevPtrs& D, const NodeStage& S,
                                        const ElemRows<kTmaK1>& rows, const CoordStage& xs, const int e,
                                        const int (&n)[NN]) {
    double H[9], A[9], gT[3], V, Ts;
    if constexpr (k1_xstage<NN>()) {
        element_pass<NN, true, kTmaK1, true>(S, n, P, D, rows, e, H, A, V, Ts, gT);
        __threadfence_block();  // keep the coordinate reads after the record sums (register pressure)
        geometry_from_coords<NN>(xs, n, A, V);
    } else {
        element_pass<NN, true, kTmaK1>(S, n, P, D, rows, e, H, A, V, Ts, gT);
    }
    // F = I + H A^T
    double F[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            F[i * 3 + j] = (i == j ? 1.0 : 0.0) + H[i * 3 + 0] * A[j * 3 + 0] + H[i * 3 + 1] * A[j * 3 + 1] +
                           H[i * 3 + 2] * A[j * 3 + 2];
    double Dk[9];
    if (P.td) conductivity_at(P, D, Ts / NN, Dk);
    else {
#pragma unroll
        for (int q = 0; q < 9; ++q) Dk[q] = P.k_fixed[q];
    }
    // g = G T_e = A (Xi T_e);  w = adj(F)^T g;  q = (V / det F) adj(F) D w;  f_a = xi_a . (A^T q)
    double g[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) g[i] = A[i * 3 + 0] * gT[0] + A[i * 3 + 1] * gT[1] + A[i * 3 + 2] * gT[2];
    double Ad[9];
    const double dF = adj3(F, Ad);
    double w[3], dw[3], q[3], r[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) w[i] = Ad[0 * 3 + i] * g[0] + Ad[1 * 3 + i] * g[1] + Ad[2 * 3 + i] * g[2];
#pragma unroll
    for (int i = 0; i < 3; ++i) dw[i] = Dk[i * 3 + 0] * w[0] + Dk[i * 3 + 1] * w[1] + Dk[i * 3 + 2] * w[2];
    const double sc = V / dF;
#pragma unroll
    for (int i = 0; i < 3; ++i) q[i] = sc * (Ad[i * 3 + 0] * dw[0] + Ad[i * 3 + 1] * dw[1] + Ad[i * 3 + 2] * dw[2]);
#pragma unroll
    for (int j = 0; j < 3; ++j) r[j] = A[0 * 3 + j] * q[0] + A[1 * 3 + j] * q[1] + A[2 * 3 + j] * q[2];
    // element-major slots: one contiguous 8*NN-byte write per element.  (A node-major
    // layout written through a position map made the node kernels ~25 % faster but
    // the scattered element writes cost more; measured.)
    if constexpr (sizeof(ST) == 4) {  // mixed precision: the element's NN contributions as fp32
        float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(D.slot_th) + (size_t)e * NN);
        if constexpr (NN == 4) {
            o[0] = make_float4((float)-(r[0] + r[1] + r[2]), (float)r[0], (float)r[1], (float)r[2]);
        } else {
            float f[8];
#pragma unroll
            for (int a = 0; a < 8; ++a) f[a] = (float)(h8s(a, 0) * r[0] + h8s(a, 1) * r[1] + h8s(a, 2) * r[2]);
            o[0] = make_float4(f[0], f[1], f[2], f[3]);
            o[1] = make_float4(f[4], f[5], f[6], f[7]);
        }
        if (dF == 0.0) atomicMin(D.err_elem, pack_elem(D.clock->step, D.elem_orig[e]));
        return;
    }
    double* out = D.slot_th + (size_t)e * NN;
    if constexpr (NN == 4) {
        const double f0 = -(r[0] + r[1] + r[2]);
        reinterpret_cast<double2*>(out)[0] = make_double2(f0, r[0]);
        reinterpret_cast<double2*>(out)[1] = make_double2(r[1], r[2]);
    } else {
        double f[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) f[a] = h8s(a, 0) * r[0] + h8s(a, 1) * r[1] + h8s(a, 2) * r[2];
#pragma unroll
        for (int a = 0; a < 8; a += 2) reinterpret_cast<double2*>(out)[a / 2] = make_double2(f[a], f[a + 1]);
    }
    if (dF == 0.0) atomicMin(D.err_elem, pack_elem(D.clock->step, D.elem_orig[e]));
}

// K1 rows: A (9) and V, unless rebuilt from the chunk coordinates
template <int NN>
__host__ __device__ __forceinline__ RowPlan k1_rows() { return RowPlan{k1_xstage<NN>() ? 0 : 10, 0, 0, 0}; }

// One kernel for every path: with the peer-memory halo attached (P.npeers > 0) its
// boundary chunks [0, P.nb_chunks) also forward their contributions and signal
// (peer_forward / peer_signal).  A separate "send" kernel would be compiled separately,
// and ptxas may contract its element math into FMAs differently: the partitions would
// then no longer match one GPU bit for bit (measured: 1e-15 drifts on T4).
template <int NN, typename ST = double>
__global__ void K1_BOUNDS k_thermal_element(const DevParams P, const DevPtrs D, int cur, int c0, int c1) {
    extern __shared__ __align__(128) unsigned char smem[];
    const RowPlan rp = k1_rows<NN>();
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem);
    double* rows = reinterpret_cast<double*>(smem + kRowsOffset);
    double* xblk = rows + (kTmaK1 ? rp.total() * kChunkThreads : 0);  // k1_xstage: the chunk's coordinates
    double2* planes = reinterpret_cast<double2*>(xblk + (k1_xstage<NN>() ? P.xstride : 0));
    const int ms = P.max_chunk_nodes;
    const NodeStage S{planes, planes + ms};
    const int c = c0 + blockIdx.x;
    CoordStage xs{nullptr, nullptr, nullptr};
    const int e0 = __ldg(D.chunk_start + c), ne = __ldg(D.chunk_start + c + 1) - e0;
    // H8: the index loads go out before the row copies (K3 104 -> 99 us, K1 54 -> 52 us on
    // cfg4); T4 chunks are slower that way (K3 305 -> 313 us on cfg5 n=100) and load them after
    StageHead<NN> hd;
    if constexpr (NN == 8) hd = stage_head<NN>(D, c, P.stage_stride, e0, ne, c1);
    {
        if constexpr (k1_xstage<NN>()) {
            const int Sx = __ldg(D.chunk_xs + c);
            xs = CoordStage{xblk, xblk + Sx, xblk + 2 * Sx};
            load_elem_rows<kTmaK1>(P, D, rp, e0, ne, rows, bar, xblk, D.chunk_x + (size_t)c * P.xstride, 24u * Sx);
        } else {
            load_elem_rows<kTmaK1>(P, D, rp, e0, ne, rows, bar);
        }
    }
    int n[NN];
    if constexpr (NN == 4) hd = stage_head<NN>(D, c, P.stage_stride, e0, ne, c1);
    const int e = stage_chunk<NN>(D, cur ? D.rec1 : D.rec0, c, P.stage_stride, S, n, hd);
    wait_elem_rows<kTmaK1>(bar);  // every thread: the CTA must not retire with bulk copies in flight
    const bool bnd = c < P.nb_chunks;  // a boundary chunk of a peer-memory partition (else false)
    if (P.ack && bnd) peer_wait_ack(P, D);
    if (!D.clock->halted && e >= 0) {  // halted: uniform across the grid (read after the wait)
        check_chunk<NN>(P, D, c, e, n);
        k1_body<NN, ST>(P, D, S, ElemRows<kTmaK1>{rows, (int)threadIdx.x}, xs, e, n);
        if (bnd) peer_forward<NN, 1>(D, reinterpret_cast<const ST*>(D.slot_th), e);
    }
    if (P.npeers) peer_signal(P, D, 0, c);  // every thread of a boundary CTA, halted or not
    pdl_trigger();  // after this block's work: the successor fills in behind the last wave
}

// ------------------------------------------------------------------ end of step (last block)
// Applies the finite-check verdict of the step and advances time/step
// (engine.hpp:89-90: the reference throws before advancing).  Called by every
// block of the closing node kernel after its body; the last block to arrive acts.
__device__ __forceinline__ void close_step(const DevParams& P, const DevPtrs& D, double dt) {
    __syncthreads();
    if (threadIdx.x != 0) return;
    __threadfence();
    const unsigned t = atomicAdd(&D.clock->ticket, 1u);
    if (t != gridDim.x - 1) return;
    __threadfence();
    Clock* c = D.clock;
    volatile unsigned long long* wi = D.err_inst;
    volatile unsigned long long* we = D.err_elem;
    if (!c->halted) {
        const unsigned long long s = (unsigned long long)c->step;
        const bool bad = (*we != ~0ULL && (*we >> 32) == s) || (*wi != ~0ULL && (*wi >> 33) == s);
        if (bad) c->halted = 1;
        else {
            c->time += dt;
            c->step += 1;
        }
    }
    c->ticket = 0;
    if (P.npeers) {  // peer-memory halo: every enqueued step, halted or not, so the ranks' sequences agree
        const unsigned long long ep = *D.epoch + 1;
        *D.epoch = ep;
        if (P.ack) {  // single-physics peer halo: this step's receive areas are consumed
            __threadfence_system();
            for (int j = 0; j < P.npeers; ++j)
                asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(D.peer_ack[j]), "l"(ep) : "memory");
        }
    }
    __threadfence();
}

// Slot values are fp64 (ST = double, the default and the parity path) or, in the
// mixed-precision mode (tvegpu_options.slot_fp32), fp32 contributions summed in fp64.
template <typename ST>
__device__ __forceinline__ double ldslot(const ST* p) { return (double)__ldg(p); }

// Sum of a node's contributions through its gather list, in canonical
// (original element, local) order.
template <typename ST>
__device__ __forceinline__ double gather1(const ST* __restrict__ slots, const int32_t* __restrict__ idx, int k0,
                                         int k1) {
    double s = 0.0;
    for (int k = k0; k < k1; ++k) s += ldslot(slots + __ldg(idx + k));
    return s;
}

// Packed 24-byte slot record: the 16-byte-aligned pair is (x, y) for even ids and
// (y, z) for odd ids; the remaining component is one 8-byte load.  (fp32: 12-byte
// records, three 4-byte loads from one or two sectors.)
template <typename ST>
__device__ __forceinline__ double3 ld_slot3(const ST* __restrict__ slots, int id) {
    if constexpr (sizeof(ST) == 4) {
        const ST* b = slots + 3 * (size_t)id;
        return make_double3((double)__ldg(b), (double)__ldg(b + 1), (double)__ldg(b + 2));
    } else {
        const int lo = id & 1;
        const double* b = slots + 3 * (size_t)id;
        const double2 v = __ldg(reinterpret_cast<const double2*>(b + lo));
        const double w = __ldg(b + (lo ? 0 : 2));
        return lo ? make_double3(w, v.x, v.y) : make_double3(v.x, v.y, w);
    }
}
template <typename ST>
__device__ __forceinline__ void gather3(const ST* __restrict__ slots, const int32_t* __restrict__ idx, int k0,
                                        int k1, double& f0, double& f1, double& f2) {
    f0 = f1 = f2 = 0.0;
    if constexpr (kMW == 3 || sizeof(ST) == 4) {
        for (int k = k0; k < k1; ++k) {
            const double3 s = ld_slot3(slots, __ldg(idx + k));
            f0 += s.x;
            f1 += s.y;
            f2 += s.z;
        }
        return;
    }
    for (int k = k0; k < k1; ++k) {
        const double4 s = ldg4(reinterpret_cast<const double4*>(slots) + __ldg(idx + k));
        f0 += s.x;
        f1 += s.y;
        f2 += s.z;
    }
}

// ELL-8 gathers: the node's 8 slot ids in one 32-byte row (two 16-byte loads, no
// offset load first), then all 8 contributions in flight at once.  Padding entries
// name a slot that is always +0.0 and sit after the real ones, so the canonical-
// order sum is unchanged bit for bit (s + 0.0 == s; s is never -0.0 from a +0.0 start).
// Rows wider than 8 (T4 meshes: ~24 contributions per node) go in groups of 8: the
// next group's ids load while the current group's contributions are in flight.
template <bool WIDE, typename ST>
__device__ __forceinline__ double gather1_ell(const ST* __restrict__ slots, const int4* __restrict__ row, int G,
                                             int4 a, int4 b) {
    double s = 0.0;
    if (!WIDE) {  // one group: straight line (H8 meshes)
        const double v0 = ldslot(slots + a.x), v1 = ldslot(slots + a.y), v2 = ldslot(slots + a.z), v3 = ldslot(slots + a.w);
        const double v4 = ldslot(slots + b.x), v5 = ldslot(slots + b.y), v6 = ldslot(slots + b.z), v7 = ldslot(slots + b.w);
        s += v0, s += v1, s += v2, s += v3, s += v4, s += v5, s += v6, s += v7;
        return s;
    }
    for (int g = 0; g < G; ++g) {
        int4 na = a, nb = b;
        if (g + 1 < G) na = __ldg(row + 2 * (g + 1)), nb = __ldg(row + 2 * (g + 1) + 1);
        const double v0 = ldslot(slots + a.x), v1 = ldslot(slots + a.y), v2 = ldslot(slots + a.z), v3 = ldslot(slots + a.w);
        const double v4 = ldslot(slots + b.x), v5 = ldslot(slots + b.y), v6 = ldslot(slots + b.z), v7 = ldslot(slots + b.w);
        s += v0, s += v1, s += v2, s += v3, s += v4, s += v5, s += v6, s += v7;
        a = na, b = nb;
    }
    return s;
}
// (the mechanical gather uses the ELL row only for single-group rows: with 3 groups of
// eight 32-byte loads the grouped loop measured slower than the CSR loop, T4 K4 +35 %)
template <typename ST>
__device__ __forceinline__ void gather3_ell(const ST* __restrict__ slots, const int4 a, const int4 b, double& f0,
                                            double& f1, double& f2) {
    const double4* S = reinterpret_cast<const double4*>(slots);
    const int id[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    if constexpr (kMW == 3 || sizeof(ST) == 4) {
        double3 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = ld_slot3(slots, id[k]);
        f0 = f1 = f2 = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            f0 += v[k].x;
            f1 += v[k].y;
            f2 += v[k].z;
        }
        return;
    }
    double4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = ldg4(S + id[k]);
    f0 = f1 = f2 = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        f0 += v[k].x;
        f1 += v[k].y;
        f2 += v[k].z;
    }
}

// ------------------------------------------------------------------ K2: thermal node
// t_out (tvegpu_step_io only): also write T^{n+1} in original numbering for the host read-back.
#ifndef TVEGPU_NODE_THREADS
#define TVEGPU_NODE_THREADS 256
#endif
constexpr int kNodeThreads = TVEGPU_NODE_THREADS;
// Node kernels walk their blocks in reverse: the element kernel before each wrote its
// contributions in element order, so the last-written ones — still in L2 — belong to the
// last nodes; taking those first turns part of the slot gather into L2 hits.  (Interface
// nodes, numbered first, are then also the last to need their neighbours' flags.)
#ifndef TVEGPU_NODE_REV
#define TVEGPU_NODE_REV 1
#endif
__device__ __forceinline__ int node_block() { return TVEGPU_NODE_REV ? (int)(gridDim.x - 1 - blockIdx.x) : (int)blockIdx.x; }
// Node kernels issue the loads of data their predecessor does not write (node record,
// sources, masks, masses) before the PDL wait, so only the slot gathers follow it:
// bit 0 K2, bit 1 K4.
#ifndef TVEGPU_NODE_HOIST
#define TVEGPU_NODE_HOIST 1
#endif
// (an explicit min-blocks of 1 lets ptxas give K4 114 registers: 96 vs 78 us)
#ifdef TVEGPU_NODE_MINBLOCKS
#define NODE_BOUNDS __launch_bounds__(kNodeThreads, TVEGPU_NODE_MINBLOCKS)
#else
#define NODE_BOUNDS __launch_bounds__(kNodeThreads)
#endif
// G: 0 = ELL rows of one group (H8) or CSR, 1 = ELL rows of several groups, 2 = two
// threads per node over the CSR list (T4; see k_mech_node<PAIR>)
// (the pair form is held to 6 blocks/SM: left free, ptxas picks 32 registers and spills)
template <int G, typename ST = double>
__global__ void __launch_bounds__(kNodeThreads, G == 2 ? 6 : 0) k_thermal_node(const DevParams P, const DevPtrs D, int cur, int closes,
                                           double* __restrict__ t_out) {
    constexpr bool PAIR = G == 2, WIDE = G == 1;
    const int b = node_block();
    const int t = b * blockDim.x + threadIdx.x;
    const int i = PAIR ? (t >> 1) : t;
    const bool lead = !PAIR || !(threadIdx.x & 1);
    int4 ia = make_int4(0, 0, 0, 0), ib = ia;
    double V = 0.0, T = 0.0, qr = 0.0;
    uint8_t m = 0;
    double4* R = cur ? D.rec1 : D.rec0;
    constexpr bool HOIST = (TVEGPU_NODE_HOIST & 1) != 0;
    if (i < P.N) {  // predecessor-independent loads first (index row, node volume)
        if (!PAIR && P.ell) ia = __ldg(D.ell + 2 * (size_t)P.ell * i), ib = __ldg(D.ell + 2 * (size_t)P.ell * i + 1);
        V = __ldg(D.vnode + i);
        if (HOIST && lead) {  // T^n: K4 of the previous step (two launches back) wrote it
            T = R[i].w;
            qr = __ldg(D.qr + i);
            m = __ldg(D.mask + i);
        }
    }
    pdl_wait();
    peer_wait(P, D, 0, PAIR ? (int)(b * blockDim.x) >> 1 : (int)(b * blockDim.x));
    const bool active = i < P.N && !D.clock->halted;  // the same for both threads of a pair
    double s = 0.0;
    if constexpr (PAIR) {
        if (active) {
            check_gather(P, D, i);
            const int k0 = __ldg(D.csr_off + i), k1 = __ldg(D.csr_off + i + 1), km = k0 + ((k1 - k0 + 1) >> 1);
            s = gather1(reinterpret_cast<const ST*>(D.slot_th), D.csr_slot, lead ? k0 : km, lead ? km : k1);
        }
        s += __shfl_down_sync(0xffffffffu, s, 1);
    }
    if (active && lead) {
        if constexpr (!PAIR) {
            check_gather(P, D, i);
            const ST* slot_th = reinterpret_cast<const ST*>(D.slot_th);
            s = P.ell ? gather1_ell<WIDE>(slot_th, D.ell + 2 * (size_t)P.ell * i, P.ell, ia, ib)
                      : gather1(slot_th, D.csr_slot, __ldg(D.csr_off + i), __ldg(D.csr_off + i + 1));
        }
        if constexpr (!HOIST) {
            T = R[i].w;
            qr = __ldg(D.qr + i);
            m = __ldg(D.mask + i);
        }
        const double c = P.td ? heat_capacity_at(P, D, T) : P.c_fixed;
        const double C = P.rho * c * V;
        double Tn = T + P.dt / C * (-s - P.wbcb * V * (T - P.Ta) + P.Qm * V + qr);
        if (m & BC_TFIX) Tn = __ldg(D.bc_tfix + __ldg(D.bc_index + i));
        if (!isfinite(Tn)) atomicMin(D.err_inst, pack_inst(D.clock->step, 0, D.node_orig[i]));
        R[i].w = Tn;
        if (t_out) t_out[__ldg(D.node_orig + i)] = Tn;
    }
    pdl_trigger();
    if (closes) close_step(P, D, P.dt);
}

// ------------------------------------------------------------------ K3: mechanical element
// EXP: 0 = F_ther = I, 1 = isotropic lambda I, 2 = general (transversely isotropic / orthotropic)
#ifndef TVEGPU_K3_WHT
#define TVEGPU_K3_WHT 1  // H8 corner-force synthesis as a 2x2x2 Walsh transform (0: direct sums)
#endif
#ifndef TVEGPU_K3_MINBLOCKS
#define TVEGPU_K3_MINBLOCKS 4  // H8: 128 registers, 16 warps/SM (168 unbounded -> 8 warps, latency-bound)
#endif
#ifndef TVEGPU_K3_MINBLOCKS_T4
#define TVEGPU_K3_MINBLOCKS_T4 5  // T4: 102 registers, 20 warps/SM (cfg5 T4 K3 -12 % vs 4)
#endif
// K3 element body: element e of the staged chunk st (n = its node slots)
// affine: the chunk's elements are all affine (c_al = 0, rows not staged)
template <int NN, int EXP, typename ST>
__device__ __forceinline__ void k3_body(const DevParams& P, const DevPtrs& D, const NodeStage& st,
                                        const ElemRows<kTmaK3>& rows, const RowPlan& rp, const CoordStage& xs,
                                        const int e, const int (&n)[NN], bool affine = false) {
    const size_t es = (size_t)P.es;
    // affine chunk (all its elements affine; CTA-uniform): K3 takes the short hourglass branch.
    // An affine element in a mixed chunk takes the general branch, which computes the same
    // values for c_al = 0 (exact zeros: A^T c_al = Hd c_al = 0, 1/(8 + 0) = 1/8), so the
    // result does not depend on which chunk — which partitioning — the element lands in.
    // (A per-element flag instead: +5 us on cfg4 with every node jittered, for its load.)
    const bool eaff = NN == 8 && affine;
    double Hd[9], A[9], V, Ts;
    {
        double H[9], gT[3];
        if constexpr (k3_xstage<NN>()) {
            element_pass<NN, false, kTmaK3, true>(st, n, P, D, rows, e, H, A, V, Ts, gT);
            __threadfence_block();  // keep the coordinate reads after the record sums (register pressure)
            geometry_from_coords<NN>(xs, n, A, V);
        } else {
            element_pass<NN, false, kTmaK3>(st, n, P, D, rows, e, H, A, V, Ts, gT);
        }
        // displacement gradient Hd = F - I = H A^T, kept separate from I (small-strain accuracy)
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j)
                Hd[i * 3 + j] = H[i * 3 + 0] * A[j * 3 + 0] + H[i * 3 + 1] * A[j * 3 + 1] + H[i * 3 + 2] * A[j * 3 + 2];
    }
    // ---- elastic part: F_el - I = (Hd - Delta) F_ther^-1, Delta = F_ther - I (Eqs. 8, 11)
    double Hel[9];
    double lam = 1.0, Fi[9], detFth = 1.0;
    if constexpr (EXP == 0) {
#pragma unroll
        for (int q = 0; q < 9; ++q) Hel[q] = Hd[q];
    } else if constexpr (EXP == 1) {
        const double e1v = P.alpha_i * (Ts / NN - P.Tref);
        lam = 1.0 + e1v;
        const double il = 1.0 / lam;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) Hel[i * 3 + j] = (Hd[i * 3 + j] - (i == j ? e1v : 0.0)) * il;
    } else {
        const double dT = Ts / NN - P.Tref;
        const double ei = P.alpha_i * dT;
        double m[3], nn_[3];
        if (P.axes_per_elem) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                m[k] = rows.get(rp.ax0() + k, D.axes + k * es + e);
                nn_[k] = rows.get(rp.ax0() + 3 + k, D.axes + (3 + k) * es + e);
            }
        } else {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                m[k] = P.axis_m[k];
                nn_[k] = P.axis_n[k];
            }
        }
        const double dm = P.alpha_m * dT - ei;
        const double dn = P.exp_kind == 2 ? P.alpha_n * dT - ei : 0.0;
        double Dl[9], Fth[9];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                Dl[i * 3 + j] = (i == j ? ei : 0.0) + dm * m[i] * m[j] + dn * nn_[i] * nn_[j];
                Fth[i * 3 + j] = (i == j ? 1.0 : 0.0) + Dl[i * 3 + j];
            }
        double Ad[9];
        detFth = adj3(Fth, Ad);
        const double idt = 1.0 / detFth;
#pragma unroll
        for (int q = 0; q < 9; ++q) Fi[q] = Ad[q] * idt;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j)
                Hel[i * 3 + j] = (Hd[i * 3 + 0] - Dl[i * 3 + 0]) * Fi[0 * 3 + j] +
                                 (Hd[i * 3 + 1] - Dl[i * 3 + 1]) * Fi[1 * 3 + j] +
                                 (Hd[i * 3 + 2] - Dl[i * 3 + 2]) * Fi[2 * 3 + j];
    }
    // ---- strain X = C_el - I = Hel + Hel^T + Hel^T Hel  (symmetric: 00 11 22 01 12 02)
    auto hh = [&](int i, int j) {
        return Hel[0 * 3 + i] * Hel[0 * 3 + j] + Hel[1 * 3 + i] * Hel[1 * 3 + j] + Hel[2 * 3 + i] * Hel[2 * 3 + j];
    };
    const double x00 = 2.0 * Hel[0] + hh(0, 0), x11 = 2.0 * Hel[4] + hh(1, 1), x22 = 2.0 * Hel[8] + hh(2, 2);
    const double x01 = Hel[1] + Hel[3] + hh(0, 1), x12 = Hel[5] + Hel[7] + hh(1, 2), x02 = Hel[2] + Hel[6] + hh(0, 2);
    // ---- S_int = 2 dPsi/dC from X without O(1) cancellation (identities in oracle pk2_from_strain):
    //   det C - 1 = i1 + i2 + det X;  I - I1/3 C^-1 = C^-1 dev X;  J - 1 = (det C - 1)/(J + 1);
    //   J^-2/3 - 1 = -(det C - 1)/(c (c^2 + c + 1)), c = cbrt(det C)
    const double i1 = x00 + x11 + x22;
    const double trX2 = x00 * x00 + x11 * x11 + x22 * x22 + 2.0 * (x01 * x01 + x12 * x12 + x02 * x02);
    const double detX = x00 * (x11 * x22 - x12 * x12) - x01 * (x01 * x22 - x12 * x02) + x02 * (x01 * x12 - x11 * x02);
    const double d1 = i1 + 0.5 * (i1 * i1 - trX2) + detX;
    if (!(d1 > -1.0)) atomicMin(D.err_elem, pack_elem(D.clock->step, D.elem_orig[e]));
    const double detC = 1.0 + d1;
    const double J = sqrt(detC);
    const double cb = cbrt(detC);
    // one reciprocal for 1/detC, 1/(J+1) and 1/(cb (cb^2 + cb + 1))
    const double qa = J + 1.0, qb = cb * (cb * cb + cb + 1.0);
    const double rq = 1.0 / (detC * qa * qb);
    const double idC = qa * qb * rq;
    const double Jm1 = d1 * (detC * qb * rq);
    const double Jm23m1 = -d1 * (detC * qa * rq);
    const double Jm23 = 1.0 + Jm23m1;
    const double c00 = 1.0 + x00, c11 = 1.0 + x11, c22 = 1.0 + x22;
    const double k00 = (c11 * c22 - x12 * x12) * idC, k11 = (c00 * c22 - x02 * x02) * idC,
                 k22 = (c00 * c11 - x01 * x01) * idC;  // C^-1
    const double k01 = (x02 * x12 - x01 * c22) * idC, k12 = (x01 * x02 - c00 * x12) * idC,
                 k02 = (x01 * x12 - x02 * c11) * idC;
    const double t3 = i1 * (1.0 / 3.0);
    const double v00 = x00 - t3, v11 = x11 - t3, v22 = x22 - t3;  // dev X
    const double iso = 0.5 * P.mu * Jm23;
    double S[6];  // mu J^-2/3 sym(C^-1 dev X)
    S[0] = iso * 2.0 * (k00 * v00 + k01 * x01 + k02 * x02);
    S[1] = iso * 2.0 * (k01 * x01 + k11 * v11 + k12 * x12);
    S[2] = iso * 2.0 * (k02 * x02 + k12 * x12 + k22 * v22);
    S[3] = iso * ((k00 * x01 + k01 * v11 + k02 * x12) + (k01 * v00 + k11 * x01 + k12 * x02));
    S[4] = iso * ((k01 * x02 + k11 * x12 + k12 * v22) + (k02 * x01 + k12 * v11 + k22 * x12));
    S[5] = iso * ((k00 * x02 + k01 * x12 + k02 * v22) + (k02 * v00 + k12 * x01 + k22 * x02));
    double ciw = P.kappa * J * Jm1;  // coefficient of C^-1
    if (P.fiber_mode) {
        double fa[3];
        if (P.fiber_mode == 2) {
#pragma unroll
            for (int k = 0; k < 3; ++k) fa[k] = rows.get(rp.fib0() + k, D.fiber + k * es + e);
        } else {
#pragma unroll
            for (int k = 0; k < 3; ++k) fa[k] = P.fiber[k];
        }
        const double Xa0 = x00 * fa[0] + x01 * fa[1] + x02 * fa[2];
        const double Xa1 = x01 * fa[0] + x11 * fa[1] + x12 * fa[2];
        const double Xa2 = x02 * fa[0] + x12 * fa[1] + x22 * fa[2];
        const double aa = fa[0] * fa[0] + fa[1] * fa[1] + fa[2] * fa[2];
        const double aXa = fa[0] * Xa0 + fa[1] * Xa1 + fa[2] * Xa2;
        const double I4 = aa + aXa;
        const double an = 2.0 * P.eta_a * (Jm23m1 + Jm23 * ((aa - 1.0) + aXa)) * Jm23;
        S[0] += an * fa[0] * fa[0];
        S[1] += an * fa[1] * fa[1];
        S[2] += an * fa[2] * fa[2];
        S[3] += an * fa[0] * fa[1];
        S[4] += an * fa[1] * fa[2];
        S[5] += an * fa[0] * fa[2];
        ciw -= an * (I4 / 3.0);
    }
    S[0] += ciw * k00;
    S[1] += ciw * k11;
    S[2] += ciw * k22;
    S[3] += ciw * k01;
    S[4] += ciw * k12;
    S[5] += ciw * k02;
    // ---- pull back to the reference configuration: det(F_th) F_th^-1 S F_th^-T
    if constexpr (EXP == 1) {
#pragma unroll
        for (int q = 0; q < 6; ++q) S[q] *= lam;
    } else if constexpr (EXP == 2) {
        const double Sm[9] = {S[0], S[3], S[5], S[3], S[1], S[4], S[5], S[4], S[2]};
        double T1[9];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j)
                T1[i * 3 + j] = Fi[i * 3 + 0] * Sm[0 * 3 + j] + Fi[i * 3 + 1] * Sm[1 * 3 + j] + Fi[i * 3 + 2] * Sm[2 * 3 + j];
        auto pb = [&](int i, int j) {
            return detFth * (T1[i * 3 + 0] * Fi[j * 3 + 0] + T1[i * 3 + 1] * Fi[j * 3 + 1] + T1[i * 3 + 2] * Fi[j * 3 + 2]);
        };
        S[0] = pb(0, 0);
        S[1] = pb(1, 1);
        S[2] = pb(2, 2);
        S[3] = pb(0, 1);
        S[4] = pb(1, 2);
        S[5] = pb(0, 2);
    }
    // ---- Prony recurrence (Eq. 28): theta_i <- a_i S + b_i theta_i ;  S~ = S - sum theta_i
    double St[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) St[q] = S[q];
#pragma unroll 1
    for (int p = 0; p < (P.P < kMaxProny ? P.P : kMaxProny); ++p) {  // staged history rows
        double* th = D.theta + (size_t)p * 6 * es + e;
        double t[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) t[q] = rows.get(rp.theta0() + p * 6 + q, th + q * es);
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            t[q] = P.pa[p] * S[q] + P.pb[p] * t[q];
            th[q * es] = t[q];
            St[q] -= t[q];
        }
    }
#pragma unroll 1
    for (int p = kMaxProny; p < P.P; ++p) {  // further terms: history and coefficients from device memory
        double* th = D.theta + (size_t)p * 6 * es + e;
        const double pa = D.tabs[P.tab_pa + p], pb = D.tabs[P.tab_pb + p];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            const double t = pa * S[q] + pb * th[q * es];
            th[q * es] = t;
            St[q] -= t;
        }
    }
    // ---- P = V F S~ = V (S~ + Hd S~) ;  Q = P A  (f_a = Q xi_a)
    const double Sm[9] = {St[0], St[3], St[5], St[3], St[1], St[4], St[5], St[4], St[2]};
    double Q[9];
    {
        double Pm[9];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j)
                Pm[i * 3 + j] = V * (Sm[i * 3 + j] + (Hd[i * 3 + 0] * Sm[0 * 3 + j] + Hd[i * 3 + 1] * Sm[1 * 3 + j] +
                                                      Hd[i * 3 + 2] * Sm[2 * 3 + j]));
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j)
                Q[i * 3 + j] = Pm[i * 3 + 0] * A[0 * 3 + j] + Pm[i * 3 + 1] * A[1 * 3 + j] + Pm[i * 3 + 2] * A[2 * 3 + j];
    }
    double4* out = reinterpret_cast<double4*>(D.slot_m) + (size_t)e * NN;
    double* out3 = D.slot_m + (size_t)e * NN * 3;  // kMW == 3: 32-byte aligned (96 / 192 bytes per element)
    float4* outf = reinterpret_cast<float4*>(reinterpret_cast<float*>(D.slot_m) + (size_t)e * NN * 3);  // fp32 slots
    if constexpr (NN == 4 && sizeof(ST) == 4) {
        outf[0] = make_float4((float)-(Q[0] + Q[1] + Q[2]), (float)-(Q[3] + Q[4] + Q[5]), (float)-(Q[6] + Q[7] + Q[8]),
                              (float)Q[0]);
        outf[1] = make_float4((float)Q[3], (float)Q[6], (float)Q[1], (float)Q[4]);
        outf[2] = make_float4((float)Q[7], (float)Q[2], (float)Q[5], (float)Q[8]);
    } else if constexpr (NN == 4 && kMW == 3) {
        double4* o = reinterpret_cast<double4*>(out3);
        st4(o + 0, make_double4(-(Q[0] + Q[1] + Q[2]), -(Q[3] + Q[4] + Q[5]), -(Q[6] + Q[7] + Q[8]), Q[0]));
        st4(o + 1, make_double4(Q[3], Q[6], Q[1], Q[4]));
        st4(o + 2, make_double4(Q[7], Q[2], Q[5], Q[8]));
    } else if constexpr (NN == 4) {
        st4(out + 0, make_double4(-(Q[0] + Q[1] + Q[2]), -(Q[3] + Q[4] + Q[5]), -(Q[6] + Q[7] + Q[8]), 0.0));
        st4(out + 1, make_double4(Q[0], Q[3], Q[6], 0.0));
        st4(out + 2, make_double4(Q[1], Q[4], Q[7], 0.0));
        st4(out + 3, make_double4(Q[2], Q[5], Q[8], 0.0));
    } else {
        // ---- closed-form hourglass, second pass over the element's nodes (L1-hot):
        //   U gamma_hat_al = U h_al - Hd c_al,  |gamma_hat_al|^2 = 8 + 8 |A^T c_al|^2,  c_al = X h_al
        //   f_hg[:, a] = k sum_al g_al gamma_hat_al[a] = k (sum_al h_al[a] g_al - W A xi_a),
        //   g_al = U gamma_hat_al / |gamma_hat_al|^2,  W A = sum_al g_al (A^T c_al)^T
        double Uh[4][3], cX[4][3];
#pragma unroll
        for (int al = 0; al < 4; ++al)
#pragma unroll
            for (int i = 0; i < 3; ++i) Uh[al][i] = 0.0;
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const double2 ra = st.a[n[a]], rb = st.b[n[a]];
#pragma unroll
            for (int al = 0; al < 4; ++al) {
                const double h = (double)h8h(al, a);
                Uh[al][0] += h * ra.x;
                Uh[al][1] += h * ra.y;
                Uh[al][2] += h * rb.x;
            }
        }
        if constexpr (k3_xstage<NN>()) {  // c_al = X h_al in corner order (k_geometry's arithmetic)
            __threadfence_block();  // (keeps ptxas from hoisting these reads into the Uh sums: spills)
#pragma unroll
            for (int al = 0; al < 4; ++al) cX[al][0] = cX[al][1] = cX[al][2] = 0.0;
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                const double x = xs.x[n[a]], y = xs.y[n[a]], z = xs.z[n[a]];
#pragma unroll
                for (int al = 0; al < 4; ++al) {
                    const double h = (double)h8h(al, a);
                    cX[al][0] += h * x;
                    cX[al][1] += h * y;
                    cX[al][2] += h * z;
                }
            }
        } else {
#pragma unroll
            for (int al = 0; al < 4; ++al)
#pragma unroll
                for (int i = 0; i < 3; ++i)
                    cX[al][i] = affine ? 0.0 : rows.get(10 + al * 3 + i, D.geo + (10 + al * 3 + i) * es + e);
        }
        const double k = P.kh * cbrt(V);
        if (eaff) {
            // affine element (c_al = 0): gamma_hat_al = h_al, |gamma_hat_al|^2 = 8 — g_al = U h_al / 8,
            // the general branch's value without its A^T c_al and Hd c_al products (zeros here)
#pragma unroll
            for (int al = 0; al < 4; ++al)
#pragma unroll
                for (int i = 0; i < 3; ++i) Uh[al][i] *= 0.125;
        } else {
#pragma unroll
        for (int al = 0; al < 4; ++al) {
            double atc[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) atc[j] = A[0 * 3 + j] * cX[al][0] + A[1 * 3 + j] * cX[al][1] + A[2 * 3 + j] * cX[al][2];
            const double in2 = 1.0 / (8.0 + 8.0 * (atc[0] * atc[0] + atc[1] * atc[1] + atc[2] * atc[2]));
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const double hc = Hd[i * 3 + 0] * cX[al][0] + Hd[i * 3 + 1] * cX[al][1] + Hd[i * 3 + 2] * cX[al][2];
                Uh[al][i] = (Uh[al][i] - hc) * in2;  // g_al, in place
            }
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j) Q[i * 3 + j] -= k * Uh[al][i] * atc[j];
        }
        }
#if TVEGPU_K3_WHT
        // corner forces f_a = Q xi_a + sum_al h_al[a] (k g_al): the eight corners are the
        // 2x2x2 Walsh transform of the mode coefficients (0, Q_i0, Q_i1, k g_3, Q_i2,
        // k g_2, k g_1, k g_4) in binary corner order — 24 adds per component instead of 48
        double fw[3][8];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            double c[8] = {0.0, Q[i * 3 + 0], Q[i * 3 + 1], k * Uh[2][i], Q[i * 3 + 2], k * Uh[1][i], k * Uh[0][i],
                           k * Uh[3][i]};
#pragma unroll
            for (int d = 1; d < 8; d <<= 1)
#pragma unroll
                for (int m = 0; m < 8; ++m)
                    if (!(m & d)) {
                        const double lo = c[m] - c[m | d], hi = c[m] + c[m | d];
                        c[m] = lo;
                        c[m | d] = hi;
                    }
#pragma unroll
            for (int b = 0; b < 8; ++b) fw[i][b] = c[b];
        }
        // brick corner a -> binary index (xi + 2 eta + 4 zeta, each bit set where the sign is +)
        auto corner = [&](int a, double f[3]) {
            const int b = (h8s(a, 0) > 0 ? 1 : 0) | (h8s(a, 1) > 0 ? 2 : 0) | (h8s(a, 2) > 0 ? 4 : 0);
#pragma unroll
            for (int i = 0; i < 3; ++i) f[i] = fw[i][b];
        };
#else
        auto corner = [&](int a, double f[3]) {
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const double v = h8s(a, 0) * Q[i * 3 + 0] + h8s(a, 1) * Q[i * 3 + 1] + h8s(a, 2) * Q[i * 3 + 2];
                const double hg =
                    h8h(0, a) * Uh[0][i] + h8h(1, a) * Uh[1][i] + h8h(2, a) * Uh[2][i] + h8h(3, a) * Uh[3][i];
                f[i] = v + k * hg;
            }
        };
#endif
        if constexpr (sizeof(ST) == 4) {  // fp32 slots: 8 x 12 bytes = six 16-byte stores
            float f[24];
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                double g[3];
                corner(a, g);
                f[3 * a] = (float)g[0], f[3 * a + 1] = (float)g[1], f[3 * a + 2] = (float)g[2];
            }
#pragma unroll
            for (int q = 0; q < 6; ++q) outf[q] = make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
        } else if constexpr (kMW == 3) {
            // corner pairs: 48 bytes = one 32-byte and one 16-byte store (pair 2p starts 32-byte aligned)
#pragma unroll
            for (int a = 0; a < 8; a += 2) {
                double f[3], g[3];
                corner(a, f);
                corner(a + 1, g);
                double* o = out3 + 3 * a;
                if ((a / 2) % 2 == 0) {
                    st4(reinterpret_cast<double4*>(o), make_double4(f[0], f[1], f[2], g[0]));
                    *reinterpret_cast<double2*>(o + 4) = make_double2(g[1], g[2]);
                } else {
                    *reinterpret_cast<double2*>(o) = make_double2(f[0], f[1]);
                    st4(reinterpret_cast<double4*>(o + 2), make_double4(f[2], g[0], g[1], g[2]));
                }
            }
        } else {
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                double f[3];
                corner(a, f);
                st4(out + a, make_double4(f[0], f[1], f[2], 0.0));
            }
        }
    }
    if (P.diag) {
#pragma unroll
        for (int q = 0; q < 9; ++q) D.diag_F[(size_t)e * 9 + q] = Hd[q] + ((q == 0 || q == 4 || q == 8) ? 1.0 : 0.0);
#pragma unroll
        for (int q = 0; q < 9; ++q) D.diag_S[(size_t)e * 9 + q] = Sm[q];
    }
}

// K3 rows: geometry (T4 10, H8 22 with the hourglass vectors), Prony history (the first
// kMaxProny terms; any further term is read in place), and the per-element fibres / expansion axes when the material has them
template <int NN, int EXP>
__host__ __device__ __forceinline__ RowPlan k3_rows(const DevParams& P) {
    return RowPlan{k3_xstage<NN>() ? 0 : (NN == 8 && !P.affine_all ? kGeoRows : 10), 6 * (P.P < kMaxProny ? P.P : kMaxProny), P.fiber_mode == 2 ? 3 : 0,
                   (EXP == 2 && P.axes_per_elem) ? 6 : 0};
}

template <int NN, int EXP, typename ST = double>
__global__ void __launch_bounds__(kChunkThreads, NN == 4 ? TVEGPU_K3_MINBLOCKS_T4 : TVEGPU_K3_MINBLOCKS)
    k_mech_element(const DevParams P, const DevPtrs D, int cur, int c0, int c1) {
    extern __shared__ __align__(128) unsigned char smem[];
    const RowPlan rp = k3_rows<NN, EXP>(P);
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem);
    double* rows = reinterpret_cast<double*>(smem + kRowsOffset);
    double* xblk = rows + (kTmaK3 ? rp.total() * kChunkThreads : 0);  // k3_xstage: the chunk's coordinates
    double2* planes = reinterpret_cast<double2*>(xblk + (k3_xstage<NN>() ? P.xstride : 0));
    const int ms = P.max_chunk_nodes;
    const NodeStage st{planes, planes + ms};
    const int c = c0 + blockIdx.x;
    CoordStage xs{nullptr, nullptr, nullptr};
    // affine H8 chunk: hourglass geometry c_al = 0, its rows neither staged nor read
    const bool affine = NN == 8 && !k3_xstage<NN>() && (P.affine_all || (D.chunk_affine && __ldg(D.chunk_affine + c)));
    const int e0 = __ldg(D.chunk_start + c), ne = __ldg(D.chunk_start + c + 1) - e0;
    StageHead<NN> hd;  // (see k_thermal_element)
    if constexpr (NN == 8) hd = stage_head<NN>(D, c, P.stage_stride, e0, ne, c1);
    {
        if constexpr (k3_xstage<NN>()) {
            const int S = __ldg(D.chunk_xs + c);
            xs = CoordStage{xblk, xblk + S, xblk + 2 * S};
            load_elem_rows<kTmaK3>(P, D, rp, e0, ne, rows, bar, xblk, D.chunk_x + (size_t)c * P.xstride, 24u * S);
        } else {
            load_elem_rows<kTmaK3>(P, D, rp, e0, ne, rows, bar, nullptr, nullptr, 0, affine);
        }
    }
    int n[NN];
    if constexpr (NN == 4) hd = stage_head<NN>(D, c, P.stage_stride, e0, ne, c1);
    const int e = stage_chunk<NN>(D, cur ? D.rec1 : D.rec0, c, P.stage_stride, st, n, hd);
    wait_elem_rows<kTmaK3>(bar);  // every thread: the CTA must not retire with bulk copies in flight
    const bool bnd = c < P.nb_chunks;  // (see k_thermal_element)
    if (P.ack && bnd) peer_wait_ack(P, D);
    if (!D.clock->halted && e >= 0) {
        check_chunk<NN>(P, D, c, e, n);
        k3_body<NN, EXP, ST>(P, D, st, ElemRows<kTmaK3>{rows, (int)threadIdx.x}, rp, xs, e, n, affine);
        if (bnd) peer_forward<NN, kMW>(D, reinterpret_cast<const ST*>(D.slot_m), e);
    }
    if (P.npeers) peer_signal(P, D, 1, c);
    pdl_trigger();
}

// ------------------------------------------------------------------ K4: mechanical node
// u_out (tvegpu_step_io only): also write u^{n+1} in original numbering for the host read-back.
// PAIR: two threads per node for long CSR lists (T4, ~24 contributions): each sums one
// half in canonical order, the first half's sum + the second's is the node's force (a
// fixed two-leaf tree: deterministic, partition-invariant).
// [n0, n1): the local node range of this launch (the whole partition, or one of the
// slices tvegpu_step_io reads back as they complete).
template <bool PAIR, typename ST = double>
__global__ void NODE_BOUNDS k_mech_node(const DevParams P, const DevPtrs D, int cur, int closes,
                                                   double* __restrict__ u_out, int n0, int n1) {
    const ST* slot_m = reinterpret_cast<const ST*>(D.slot_m);
    const int b = node_block();
    const int t = b * blockDim.x + threadIdx.x;
    const int i = n0 + (PAIR ? (t >> 1) : t);
    const bool lead = !PAIR || !(threadIdx.x & 1);
    int4 ia = make_int4(0, 0, 0, 0), ib = ia;
    if (!PAIR && i < n1 && P.ell == 1) ia = __ldg(D.ell + 2 * (size_t)i), ib = __ldg(D.ell + 2 * (size_t)i + 1);
    const double4* Rc = cur ? D.rec1 : D.rec0;
    double4* Rn = cur ? D.rec0 : D.rec1;  // holds u^{n-1}; receives u^{n+1}
    constexpr bool HOIST = (TVEGPU_NODE_HOIST & 2) != 0;
    double4 u = make_double4(0.0, 0.0, 0.0, 0.0), up = u;
    double m = 0.0;
    uint8_t msk = 0;
    if (HOIST && i < n1 && lead) {  // u^n, T^{n+1}, u^{n-1}: written two or more launches back
        u = ldg4(Rc + i);
        up = ld4(Rn + i);
        m = __ldg(D.mass + i);
        msk = __ldg(D.mask + i);
    }
    pdl_wait();
    peer_wait(P, D, 1, n0 + (PAIR ? (int)(b * blockDim.x) >> 1 : (int)(b * blockDim.x)));
    const bool active = i < n1 && !D.clock->halted;  // the same for both threads of a pair
    double f0 = 0.0, f1 = 0.0, f2 = 0.0;
    if constexpr (PAIR) {
        if (active) {
            check_gather(P, D, i);
            const int k0 = __ldg(D.csr_off + i), k1 = __ldg(D.csr_off + i + 1), km = k0 + ((k1 - k0 + 1) >> 1);
            gather3(slot_m, D.csr_slot, lead ? k0 : km, lead ? km : k1, f0, f1, f2);
        }
        f0 += __shfl_down_sync(0xffffffffu, f0, 1);
        f1 += __shfl_down_sync(0xffffffffu, f1, 1);
        f2 += __shfl_down_sync(0xffffffffu, f2, 1);
    }
    if (active && lead) {
        if constexpr (!PAIR) {
            check_gather(P, D, i);
            if (P.ell == 1) gather3_ell(slot_m, ia, ib, f0, f1, f2);
            else gather3(slot_m, D.csr_slot, __ldg(D.csr_off + i), __ldg(D.csr_off + i + 1), f0, f1, f2);
        }
        if constexpr (!HOIST) {
            u = ldg4(Rc + i);  // read-only in this kernel
            up = ld4(Rn + i);  // this thread overwrites it below
            m = __ldg(D.mass + i);
            msk = __ldg(D.mask + i);
        }
        const double Dm = P.gamma * m;
        const double a = Dm * P.inv_2dt, b = m * P.inv_dt2;
        const double iab = 1.0 / (a + b);
        double R0 = 0.0, R1 = 0.0, R2 = 0.0;
        if (P.has_R) {
            R0 = __ldg(D.R + 3 * (size_t)i);
            R1 = __ldg(D.R + 3 * (size_t)i + 1);
            R2 = __ldg(D.R + 3 * (size_t)i + 2);
        }
        double x = (R0 - f0 + 2.0 * b * u.x + (a - b) * up.x) * iab;
        double y = (R1 - f1 + 2.0 * b * u.y + (a - b) * up.y) * iab;
        double z = (R2 - f2 + 2.0 * b * u.z + (a - b) * up.z) * iab;
        if (msk & (BC_FIXED | BC_PX | BC_PY | BC_PZ)) {
            if (msk & BC_FIXED) x = y = z = 0.0;
            if (msk & (BC_PX | BC_PY | BC_PZ)) {
                const double tn = D.clock->time + P.dt;  // value_at(t + dt), mechanics.hpp:89
                const int row = __ldg(D.bc_index + i);
                auto value_at = [&](int q) {
                    const int id = __ldg(D.bc_presc + 3 * row + q);
                    const double tg = D.presc_target[id], rt = D.presc_ramp[id];
                    return rt <= 0.0 ? tg : tg * fmin(tn / rt, 1.0);
                };
                if (msk & BC_PX) x = value_at(0);
                if (msk & BC_PY) y = value_at(1);
                if (msk & BC_PZ) z = value_at(2);
            }
        }
        if (P.motion) {  // motion_override wins last (mechanics.hpp:43-46, C9)
            const int r = __ldg(D.motion_row + i);
            if (r >= 0) {
                const double4 v = D.motion_val[r];
                if (v.w != 0.0) x = v.x, y = v.y, z = v.z;
            }
        }
        if (!(isfinite(x) && isfinite(y) && isfinite(z)))
            atomicMin(D.err_inst, pack_inst(D.clock->step, 1, D.node_orig[i]));
        st4(Rn + i, make_double4(x, y, z, u.w));
        if (u_out) {
            double* o = u_out + 3 * (size_t)__ldg(D.node_orig + i);
            o[0] = x, o[1] = y, o[2] = z;
        }
        if (P.diag) {
            D.diag_f[3 * (size_t)i] = f0;
            D.diag_f[3 * (size_t)i + 1] = f1;
            D.diag_f[3 * (size_t)i + 2] = f2;
        }
    }
    pdl_trigger();
    if (closes) close_step(P, D, P.dt);
}

// ------------------------------------------------------------------ halo pack / unpack (nranks > 1)
// pack: send buffer k <- node-major slot send_pos[k];  unpack: slot recv_pos[r] <- receive buffer r
template <typename ST>
__global__ void k_pack(const ST* __restrict__ slots, const int32_t* __restrict__ idx, int n, int width,
                       ST* __restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int s = idx[k];
    for (int c = 0; c < width; ++c) out[(size_t)k * width + c] = slots[(size_t)s * width + c];
}
template <typename ST>
__global__ void k_unpack(ST* __restrict__ slots, const int32_t* __restrict__ idx, int n, int width,
                         const ST* __restrict__ in) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int s = idx[k];
    for (int c = 0; c < width; ++c) slots[(size_t)s * width + c] = in[(size_t)k * width + c];
}

}  // namespace tvegpu
