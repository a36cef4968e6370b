// plan.cpp — host setup for the device path (see plan.hpp).
#include "plan.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <numeric>
#include <parallel/algorithm>

#include <omp.h>

namespace tvegpu {



const int kH8Sign[8][3] = {{-1, -1, -1}, {1, -1, -1}, {1, 1, -1}, {-1, 1, -1},
                           {-1, -1, 1},  {1, -1, 1},  {1, 1, 1},  {-1, 1, 1}};
const int kT4Xi[4][3] = {{-1, -1, -1}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
const int kHg[4][8] = {{1, 1, -1, -1, -1, -1, 1, 1},
                       {1, -1, -1, 1, -1, 1, 1, -1},
                       {1, -1, 1, -1, 1, -1, 1, -1},
                       {-1, 1, -1, 1, 1, -1, 1, -1}};

namespace {

[[noreturn]] void invalid(const std::string& m) { throw Error(TVEGPU_E_VALIDATION, m); }

double det3(const double m[3][3]) {
    return m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) - m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
           m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
}

double sym_max_eig(const double* t) {
    double a[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) a[i][j] = 0.5 * (t[i * 3 + j] + t[j * 3 + i]);
    // closed-form eigenvalues of a symmetric 3x3 (trigonometric method)
    const double p1 = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
    if (p1 == 0) return std::max(a[0][0], std::max(a[1][1], a[2][2]));
    const double q = (a[0][0] + a[1][1] + a[2][2]) / 3;
    const double p2 = (a[0][0] - q) * (a[0][0] - q) + (a[1][1] - q) * (a[1][1] - q) + (a[2][2] - q) * (a[2][2] - q) +
                      2 * p1;
    const double p = std::sqrt(p2 / 6);
    double B[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) B[i][j] = (a[i][j] - (i == j ? q : 0)) / p;
    double r = det3(B) / 2;
    r = std::max(-1.0, std::min(1.0, r));
    const double phi = std::acos(r) / 3;
    return q + 2 * p * std::cos(phi);
}

uint64_t spread21(uint64_t v) {
    v &= 0x1fffff;
    v = (v | (v << 32)) & 0x1f00000000ffffULL;
    v = (v | (v << 16)) & 0x1f0000ff0000ffULL;
    v = (v | (v << 8)) & 0x100f00f00f00f00fULL;
    v = (v | (v << 4)) & 0x10c30c30c30c30c3ULL;
    v = (v | (v << 2)) & 0x1249249249249249ULL;
    return v;
}

}  // namespace

// Morton key of an element centroid on the "element lattice": coordinates are
// measured in units of the smallest element edge (isotropic scale, capped so the
// extent fits 21 bits) and rounded.  On structured meshes this maps centroids to
// their integer cell indices, so 8 consecutive keys are an aligned 2x2x2 block of
// cells — what the shared-memory colouring (colour_slots) relies on.
uint64_t morton_key(const double* c, const double* lo, double scale) {
    uint64_t q[3];
    for (int k = 0; k < 3; ++k) {
        double v = std::floor((c[k] - lo[k]) * scale + 0.5);
        v = std::min(2097151.0, std::max(0.0, v));
        q[k] = (uint64_t)v;
    }
    return spread21(q[0]) | (spread21(q[1]) << 1) | (spread21(q[2]) << 2);
}

double morton_scale(const GlobalMesh& g) {
    double ext = 0;
    for (int k = 0; k < 3; ++k) ext = std::max(ext, g.hi[k] - g.lo[k]);
    double s = g.min_edge > 0 ? 1.0 / g.min_edge : 0.0;
    if (ext > 0 && ext * s > 2097151.0) s = 2097151.0 / ext;
    return s;
}

void validate_problem(const tvegpu_problem& p) {
    if (p.kind != TVEGPU_T4 && p.kind != TVEGPU_H8) invalid("unknown element kind");
    if (p.num_nodes <= 0 || p.num_elements <= 0 || !p.nodes || !p.elements) invalid("empty mesh");
    const int nn = p.kind == TVEGPU_T4 ? 4 : 8;
    {
        const int64_t n = (int64_t)p.num_elements * nn;
        int64_t first = n;  // lowest offending entry (the message names its element)
#pragma omp parallel for schedule(static) reduction(min : first)
        for (int64_t k = 0; k < n; ++k) {
            const int v = p.elements[k];
            if ((v < 0 || v >= p.num_nodes) && k < first) first = k;
        }
        if (first < n)
            invalid("element " + std::to_string(first / nn + 1) + " references out-of-range node " +
                    std::to_string(p.elements[first] + 1));
    }
    if (!(p.mu > 0) || !(p.kappa > 0) || p.eta_a < 0) invalid("hyperelastic parameters need mu > 0, kappa > 0, eta_a >= 0");
    double sphi = 0;
    for (int i = 0; i < p.prony_count; ++i) {
        if (!(p.prony_phi[i] > 0) || !(p.prony_tau[i] > 0)) invalid("Prony terms need phi > 0 and tau > 0");
        sphi += p.prony_phi[i];
    }
    if (p.prony_count > 0 && !(sphi < 1.0)) invalid("Prony weights must sum to < 1");
    if (!(p.density > 0)) invalid("density must be > 0");
    if (p.c_table_len < 1 || p.k_table_len < 1) invalid("property tables need at least one entry");
    if (p.prony_count < 0) invalid("prony_count must be >= 0");
    for (int i = 0; i < p.c_table_len; ++i)
        if (!(p.c_table_value[i] > 0)) invalid("specific heat must be > 0");
    for (int i = 1; i < p.c_table_len; ++i)
        if (!(p.c_table_T[i] > p.c_table_T[i - 1])) invalid("specific heat table must be sorted by T");
    for (int i = 1; i < p.k_table_len; ++i)
        if (!(p.k_table_T[i] > p.k_table_T[i - 1])) invalid("conductivity table must be sorted by T");
    if (!(p.dt > 0)) invalid("dt must be > 0");
    if (p.mode < 0 || p.mode > 2) invalid("unknown coupling mode");
    if (p.eta_a > 0 && !p.has_fiber && !p.fiber_dirs) invalid("eta_a > 0 requires a fiber direction");
    auto unit = [](const double* v) { return std::fabs(v[0] * v[0] + v[1] * v[1] + v[2] * v[2] - 1.0) <= 1e-6; };
    if (p.has_expansion) {
        if (p.expansion_kind < 0 || p.expansion_kind > 2) invalid("unknown expansion kind");
        auto check_axes = [&](const double* m, const double* n) {
            if (p.expansion_kind >= TVEGPU_EXP_TRANSVERSELY_ISOTROPIC && !unit(m)) invalid("expansion axis m not unit");
            if (p.expansion_kind == TVEGPU_EXP_ORTHOTROPIC &&
                (!unit(n) || std::fabs(m[0] * n[0] + m[1] * n[1] + m[2] * n[2]) > 1e-6))
                invalid("expansion axes not orthonormal");
        };
        if (p.expansion_axes)
            for (int e = 0; e < p.num_elements; ++e) check_axes(p.expansion_axes + 6 * (size_t)e, p.expansion_axes + 6 * (size_t)e + 3);
        else
            check_axes(p.axis_m, p.axis_n);
    }
    for (int i = 0; i < p.num_prescribed; ++i) {
        const auto& q = p.prescribed[i];
        if (q.component < 0 || q.component > 2) invalid("prescribed component must be 0..2");
        for (int k = 0; k < q.num_nodes; ++k)
            if (q.nodes[k] < 0 || q.nodes[k] >= p.num_nodes) invalid("prescribed node out of range");
    }
    for (int i = 0; i < p.num_fixed_nodes; ++i)
        if (p.fixed_nodes[i] < 0 || p.fixed_nodes[i] >= p.num_nodes) invalid("fixed node out of range");
    for (int i = 0; i < p.num_fixed_temperatures; ++i)
        if (p.fixed_temperature_nodes[i] < 0 || p.fixed_temperature_nodes[i] >= p.num_nodes)
            invalid("fixed-temperature node out of range");
    for (int i = 0; i < p.num_sources; ++i)
        for (int k = 0; k < p.sources[i].num_elements; ++k)
            if (p.sources[i].elements[k] < 0 || p.sources[i].elements[k] >= p.num_elements)
                invalid("source element out of range");
}

// Node -> (element, local) lists in canonical order (ascending element, then local;
// mesh.hpp:58-61) as keys e * nn + a: a counting sort in which every thread owns a range
// of node ids and scans the whole connectivity for its own nodes — no atomics, and each
// node's list fills in ascending key order, i.e. already canonical.
static void build_adjacency(const int32_t* elements, int E, int N, int nn, fvec<int32_t>& off, fvec<int32_t>& key) {
    const int64_t n = (int64_t)E * nn;
    off.resize((size_t)N + 1);
    key.resize((size_t)n);
    fvec<int32_t> fill((size_t)N);
#pragma omp parallel
    {
        const int t = omp_get_thread_num(), nt = omp_get_num_threads();
        const int32_t n0 = (int32_t)((int64_t)N * t / nt), n1 = (int32_t)((int64_t)N * (t + 1) / nt);
        const uint32_t span = (uint32_t)(n1 - n0);
        for (int32_t i = n0; i < n1; ++i) fill[i] = 0;
        for (int64_t k = 0; k < n; ++k) {
            const uint32_t d = (uint32_t)(elements[k] - n0);
            if (d < span) fill[n0 + d]++;
        }
#pragma omp barrier
#pragma omp single
        {
            off[0] = 0;
            for (int i = 0; i < N; ++i) off[i + 1] = off[i] + fill[i];
        }
        for (int32_t i = n0; i < n1; ++i) fill[i] = off[i];
        for (int64_t k = 0; k < n; ++k) {
            const uint32_t d = (uint32_t)(elements[k] - n0);
            if (d < span) key[fill[n0 + d]++] = (int32_t)k;
        }
    }
}

GlobalMesh build_global(const tvegpu_problem& p) {
    StageTimer tm("build_global");
    LapTimer lap;
    validate_problem(p);
    lap("validate");
    GlobalMesh g;
    g.kind = p.kind;
    g.nn = p.kind == TVEGPU_T4 ? 4 : 8;
    g.N = p.num_nodes;
    g.E = p.num_elements;
    const int nn = g.nn, E = g.E, N = g.N;
    g.vol.resize(E);
    g.centroid.resize((size_t)3 * E);
    for (int k = 0; k < 3; ++k) {
        g.lo[k] = std::numeric_limits<double>::infinity();
        g.hi[k] = -std::numeric_limits<double>::infinity();
    }
    // one pass over the elements: volume (det J; its sign validates the element),
    // centroid, smallest edge, centroid bounding box
    static const int t4e[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    static const int h8e[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6},
                                   {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
    int bad = -1;
    double L = std::numeric_limits<double>::infinity();
#pragma omp parallel reduction(max : bad) reduction(min : L)
    {
        double lo[3], hi[3];
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::numeric_limits<double>::infinity();
            hi[k] = -std::numeric_limits<double>::infinity();
        }
#pragma omp for schedule(static) nowait
        for (int e = 0; e < E; ++e) {
            const int32_t* el = p.elements + (size_t)e * nn;
            double X[8][3];
            for (int a = 0; a < nn; ++a)
                for (int i = 0; i < 3; ++i) X[a][i] = p.nodes[3 * (size_t)el[a] + i];
            double J[3][3];
            if (nn == 4) {
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) J[i][j] = X[j + 1][i] - X[0][i];
            } else {
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) {
                        double s = 0;
                        for (int a = 0; a < 8; ++a) s += X[a][i] * kH8Sign[a][j];
                        J[i][j] = s / 8.0;
                    }
            }
            const double d = det3(J);
            const double V = nn == 4 ? d / 6.0 : 8.0 * d;
            if (!(V > 0)) {
                bad = std::max(bad, E - e);  // keep the LOWEST failing element
                continue;
            }
            g.vol[e] = V;
            for (int k = 0; k < 3; ++k) {
                double s = 0;
                for (int a = 0; a < nn; ++a) s += X[a][k];
                const double c = s / nn;
                g.centroid[(size_t)3 * e + k] = c;
                lo[k] = std::min(lo[k], c);
                hi[k] = std::max(hi[k], c);
            }
            for (int k = 0; k < (nn == 4 ? 6 : 12); ++k) {
                const int a = nn == 4 ? t4e[k][0] : h8e[k][0], b = nn == 4 ? t4e[k][1] : h8e[k][1];
                double d2 = 0;
                for (int i = 0; i < 3; ++i) {
                    const double dd = X[a][i] - X[b][i];
                    d2 += dd * dd;
                }
                L = std::min(L, std::sqrt(d2));
            }
        }
#pragma omp critical
        for (int k = 0; k < 3; ++k) {
            g.lo[k] = std::min(g.lo[k], lo[k]);
            g.hi[k] = std::max(g.hi[k], hi[k]);
        }
    }
    if (bad >= 0) invalid("degenerate or inverted element " + std::to_string(E - bad + 1));
    g.min_edge = L;
    lap("element geometry + bounds");
    // canonical adjacency over original ids
    fvec<int32_t> key;
    build_adjacency(p.elements, E, N, nn, g.adj_off, key);
    g.adj_elem.resize(key.size());
    g.adj_local.resize(key.size());
#pragma omp parallel for schedule(static)
    for (size_t k = 0; k < key.size(); ++k) {
        g.adj_elem[k] = key[k] / nn;
        g.adj_local[k] = key[k] % nn;
    }
    lap("adjacency");
    g.mass.resize(N);
    g.vnode.resize(N);
    int orphan = -1;
#pragma omp parallel for schedule(static) reduction(max : orphan)
    for (int i = 0; i < N; ++i) {
        if (g.adj_off[i] == g.adj_off[i + 1]) orphan = std::max(orphan, N - i);
        double m = 0, v = 0;
        for (int k = g.adj_off[i]; k < g.adj_off[i + 1]; ++k) {
            const double V = g.vol[g.adj_elem[k]];
            m += p.density * V / nn;
            v += V / nn;
        }
        g.mass[i] = m;
        g.vnode[i] = v;
    }
    if (orphan >= 0) invalid("node " + std::to_string(N - orphan) + " is not attached to any element (zero lumped mass)");
    lap("lumped node constants");
    return g;
}

// ---------------------------------------------------------------- RCB
static void rcb_rec(const GlobalMesh& g, std::vector<int32_t>& ids, size_t b, size_t e, int parts, int first,
                    std::vector<int32_t>& owner) {
    if (parts == 1) {
        for (size_t k = b; k < e; ++k) owner[ids[k]] = first;
        return;
    }
    double lo[3], hi[3];
    for (int k = 0; k < 3; ++k) {
        lo[k] = std::numeric_limits<double>::infinity();
        hi[k] = -lo[k];
    }
    for (size_t k = b; k < e; ++k)
        for (int c = 0; c < 3; ++c) {
            lo[c] = std::min(lo[c], g.centroid[(size_t)3 * ids[k] + c]);
            hi[c] = std::max(hi[c], g.centroid[(size_t)3 * ids[k] + c]);
        }
    int ax = 0;
    for (int c = 1; c < 3; ++c)
        if (hi[c] - lo[c] > hi[ax] - lo[ax]) ax = c;
    const int left_parts = parts / 2;
    const size_t n = e - b;
    const size_t nl = (size_t)((n * (uint64_t)left_parts) / parts);
    auto less = [&](int32_t x, int32_t y) {
        const double cx = g.centroid[(size_t)3 * x + ax], cy = g.centroid[(size_t)3 * y + ax];
        return cx < cy || (cx == cy && x < y);
    };
    std::nth_element(ids.begin() + b, ids.begin() + b + nl, ids.begin() + e, less);
    std::sort(ids.begin() + b, ids.begin() + b + nl);
    std::sort(ids.begin() + b + nl, ids.begin() + e);
    rcb_rec(g, ids, b, b + nl, left_parts, first, owner);
    rcb_rec(g, ids, b + nl, e, parts - left_parts, first + left_parts, owner);
}

std::vector<int32_t> rcb_partition(const GlobalMesh& g, int nranks) {
    std::vector<int32_t> owner(g.E, 0);
    if (nranks <= 1) return owner;
    std::vector<int32_t> ids(g.E);
    std::iota(ids.begin(), ids.end(), 0);
    rcb_rec(g, ids, 0, ids.size(), nranks, 0, owner);
    return owner;
}

// ---------------------------------------------------------------- parallel helpers
// Stable LSD radix sort of ids by key[id] (8-bit digits up to kmax's top bit): with the
// ids initially ascending, the result is the total order (key, id).
static void radix_sort_by_key(std::vector<int32_t>& ids, const uint64_t* key, uint64_t kmax) {
    const size_t n = ids.size();
    if (n < 2) return;
    int bits = 0;
    while (bits < 64 && (kmax >> bits)) ++bits;
    fvec<int32_t> tmp(n);
    int32_t* src = ids.data();
    int32_t* dst = tmp.data();
    const int T = std::max(1, omp_get_max_threads());
    std::vector<size_t> hist((size_t)T * 256);
    int passes = 0;
    for (int shift = 0; shift < bits; shift += 8, ++passes) {
#pragma omp parallel num_threads(T)
        {
            const int t = omp_get_thread_num(), nt = omp_get_num_threads();
            const size_t b0 = n * t / nt, b1 = n * (t + 1) / nt;
            size_t* h = hist.data() + (size_t)t * 256;
            std::fill(h, h + 256, 0);
            for (size_t q = b0; q < b1; ++q) h[(key[src[q]] >> shift) & 255]++;
#pragma omp barrier
#pragma omp single
            {
                size_t run = 0;  // digit-major, thread-minor: stable across the thread blocks
                for (int d = 0; d < 256; ++d)
                    for (int u = 0; u < nt; ++u) {
                        const size_t c = hist[(size_t)u * 256 + d];
                        hist[(size_t)u * 256 + d] = run;
                        run += c;
                    }
            }
            for (size_t q = b0; q < b1; ++q) dst[h[(key[src[q]] >> shift) & 255]++] = src[q];
        }
        std::swap(src, dst);
    }
    if (passes & 1) std::copy(tmp.begin(), tmp.end(), ids.begin());
}

// The non-negative entries of `at` in index order (parallel compaction).
static void compact_in_order(const fvec<int32_t>& at, std::vector<int32_t>& out) {
    const size_t n = at.size();
    const int T = std::max(1, omp_get_max_threads());
    std::vector<size_t> cnt((size_t)T + 1, 0);
#pragma omp parallel num_threads(T)
    {
        const int t = omp_get_thread_num(), nt = omp_get_num_threads();
        const size_t b0 = n * t / nt, b1 = n * (t + 1) / nt;
        size_t c = 0;
        for (size_t q = b0; q < b1; ++q) c += at[q] >= 0;
        cnt[t + 1] = c;
#pragma omp barrier
#pragma omp single
        {
            for (int u = 0; u < nt; ++u) cnt[u + 1] += cnt[u];
            out.resize(cnt[nt]);
        }
        size_t o = cnt[t];
        for (size_t q = b0; q < b1; ++q)
            if (at[q] >= 0) out[o++] = at[q];
    }
}

// ---------------------------------------------------------------- rank plan
RankPlan build_rank_plan(const tvegpu_problem& p, const GlobalMesh& g, int nranks, int rank, int reorder) {
    StageTimer tm("build_rank_plan (total)");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(TVEGPU_E_ARG, "bad rank / nranks");
    if (nranks > 1 && !reorder) throw Error(TVEGPU_E_ARG, "reorder = 0 needs nranks = 1");
    RankPlan r;
    r.nranks = nranks;
    r.rank = rank;
    r.nn = g.nn;
    const int nn = g.nn, N = g.N, E = g.E;
    LapTimer lap;
    r.owner = rcb_partition(g, nranks);
    lap("rcb partition");
    // sharers of each node: bitmask of ranks touching it (nranks <= 64), from its adjacency
    if (nranks > 64) throw Error(TVEGPU_E_ARG, "at most 64 ranks");
    fvec<uint64_t> touch((size_t)N);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < N; ++i) {
        uint64_t t = 0;
        for (int k = g.adj_off[i]; k < g.adj_off[i + 1]; ++k) t |= 1ULL << r.owner[g.adj_elem[k]];
        touch[i] = t;
    }
    const uint64_t me = 1ULL << rank;
    // owned elements, split into boundary (touches a shared node) and interior
    std::vector<int32_t> bnd, inr;
    if (nranks == 1) {
        inr.resize(E);
        std::iota(inr.begin(), inr.end(), 0);
    } else {
        fvec<uint8_t> cls((size_t)E);  // 0 other rank, 1 boundary, 2 interior
#pragma omp parallel for schedule(static)
        for (int e = 0; e < E; ++e) {
            if (r.owner[e] != rank) {
                cls[e] = 0;
                continue;
            }
            bool b = false;
            for (int a = 0; a < nn && !b; ++a) b = (touch[p.elements[(size_t)e * nn + a]] & ~me) != 0;
            cls[e] = b ? 1 : 2;
        }
        for (int e = 0; e < E; ++e)
            if (cls[e]) (cls[e] == 1 ? bnd : inr).push_back(e);
    }
    if (reorder) {
        fvec<uint64_t> key((size_t)E);
        const double mscale = morton_scale(g);
        // lattice origin: the partition's own lowest centroid (every partition's Morton blocks
        // start at its corner, not wherever the global lattice happens to cut it)
        double klo[3] = {g.lo[0], g.lo[1], g.lo[2]};
        if (nranks > 1) {
            double l0 = INFINITY, l1 = INFINITY, l2 = INFINITY;
            auto scan = [&](const std::vector<int32_t>& v) {
#pragma omp parallel for schedule(static) reduction(min : l0, l1, l2)
                for (size_t q = 0; q < v.size(); ++q) {
                    const double* c = &g.centroid[(size_t)3 * v[q]];
                    l0 = std::min(l0, c[0]), l1 = std::min(l1, c[1]), l2 = std::min(l2, c[2]);
                }
            };
            scan(bnd);
            scan(inr);
            if (l0 != INFINITY) klo[0] = l0, klo[1] = l1, klo[2] = l2;
        }
        auto sort_group = [&](std::vector<int32_t>& v) {
            uint64_t kmax = 0;
#pragma omp parallel for schedule(static) reduction(max : kmax)
            for (size_t q = 0; q < v.size(); ++q) {
                key[v[q]] = morton_key(&g.centroid[(size_t)3 * v[q]], klo, mscale);
                kmax = std::max(kmax, key[v[q]]);
            }
            // total order (key, id): a stable radix sort of the id-ordered list by key
            radix_sort_by_key(v, key.data(), kmax);
        };
        sort_group(bnd);
        sort_group(inr);
    }
    // chunks start at even elements (16-byte aligned per-element rows for the element
    // kernels' bulk copies): an odd boundary group takes the first interior element
    if (bnd.size() % 2 == 1 && !inr.empty()) {
        bnd.push_back(inr.front());
        inr.erase(inr.begin());
    }
    lap("boundary split + morton sort");
    r.Eb = (int)bnd.size();
    r.elem_orig.resize(bnd.size() + inr.size());
    std::copy(bnd.begin(), bnd.end(), r.elem_orig.begin());
    std::copy(inr.begin(), inr.end(), r.elem_orig.begin() + bnd.size());
    r.E = (int)r.elem_orig.size();
    fvec<int32_t> elem_local((size_t)E);
#pragma omp parallel for schedule(static)
    for (int e = 0; e < E; ++e) elem_local[e] = -1;
#pragma omp parallel for schedule(static)
    for (int le = 0; le < r.E; ++le) elem_local[r.elem_orig[le]] = le;
    // first-touch node numbering (identity when reorder = 0, nranks = 1): a node's number
    // is its rank by first local touch (local element, local index) — the minimum of
    // le * nn + a over its adjacency; those keys are distinct, so scattering the nodes to
    // their keys and compacting gives the numbering without a serial walk
    fvec<int32_t> local((size_t)N);
    if (reorder) {
        const int64_t nk = (int64_t)r.E * nn;
        fvec<int32_t> at((size_t)std::max<int64_t>(1, nk));
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < nk; ++k) at[k] = -1;
#pragma omp parallel for schedule(static)
        for (int i = 0; i < N; ++i) {
            int64_t first = INT64_MAX;
            for (int k = g.adj_off[i]; k < g.adj_off[i + 1]; ++k) {
                const int le = elem_local[g.adj_elem[k]];
                if (le >= 0) first = std::min(first, (int64_t)le * nn + g.adj_local[k]);
            }
            if (first != INT64_MAX) at[first] = i;
            local[i] = -1;
        }
        compact_in_order(at, r.node_orig);
#pragma omp parallel for schedule(static)
        for (size_t li = 0; li < r.node_orig.size(); ++li) local[r.node_orig[li]] = (int32_t)li;
    } else {
        r.node_orig.resize(N);
        std::iota(r.node_orig.begin(), r.node_orig.end(), 0);
        std::iota(local.begin(), local.end(), 0);
    }
    r.N = (int)r.node_orig.size();
    // node ownership for state gathers (checkpoint images): the lowest rank touching it
    r.node_owned.resize(r.N);
#pragma omp parallel for schedule(static)
    for (int li = 0; li < r.N; ++li) {
        const uint64_t t = touch[r.node_orig[li]];
        r.node_owned[li] = (uint8_t)((t & (~t + 1)) == me);
    }
    r.conn.resize((size_t)r.E * nn);
#pragma omp parallel for schedule(static)
    for (int le = 0; le < r.E; ++le) {
        for (int a = 0; a < nn; ++a) r.conn[(size_t)le * nn + a] = local[p.elements[(size_t)r.elem_orig[le] * nn + a]];
    }
    lap("node numbering + conn");
    // neighbours and halo lists: for each neighbour s, the (orig e, a) contributions of
    // elements owned by the SENDER to nodes shared with the receiver, canonical order.
    std::vector<std::vector<int32_t>> send(nranks), recv_keys(nranks);  // recv: global adjacency index k
    for (int i = 0; i < N; ++i) {
        const uint64_t t = touch[i];
        if (!(t & me) || (t & (t - 1)) == 0) continue;  // not local or not shared
        for (int k = g.adj_off[i]; k < g.adj_off[i + 1]; ++k) {
            const int e = g.adj_elem[k], a = g.adj_local[k];
            const int o = r.owner[e];
            if (o == rank) {
                for (int s = 0; s < nranks; ++s)
                    if (s != rank && (t >> s & 1)) send[s].push_back(elem_local[e] * nn + a);
            } else {
                recv_keys[o].push_back(k);
            }
        }
    }
    // send lists must be in canonical (orig e, a) order per neighbour: sort by (orig e, a)
    for (int s = 0; s < nranks; ++s) {
        auto& v = send[s];
        std::sort(v.begin(), v.end(), [&](int32_t x, int32_t y) {
            const int ex = r.elem_orig[x / nn], ey = r.elem_orig[y / nn];
            return ex < ey || (ex == ey && x % nn < y % nn);
        });
        v.erase(std::unique(v.begin(), v.end()), v.end());
        auto& w = recv_keys[s];
        std::sort(w.begin(), w.end(), [&](int32_t x, int32_t y) {
            return g.adj_elem[x] < g.adj_elem[y] || (g.adj_elem[x] == g.adj_elem[y] && g.adj_local[x] < g.adj_local[y]);
        });
        w.erase(std::unique(w.begin(), w.end(), [&](int32_t x, int32_t y) {
                    return g.adj_elem[x] == g.adj_elem[y] && g.adj_local[x] == g.adj_local[y];
                }), w.end());
    }
    r.send_off.push_back(0);
    r.recv_off.push_back(0);
    // receive index of global adjacency entry k (only for remote contributions)
    std::vector<std::pair<int64_t, int32_t>> recv_index;  // key = e*nn + a -> receive slot
    for (int s = 0; s < nranks; ++s) {
        if (s == rank || (send[s].empty() && recv_keys[s].empty())) continue;
        r.neighbors.push_back(s);
        r.send_slot.insert(r.send_slot.end(), send[s].begin(), send[s].end());
        r.send_off.push_back((int32_t)r.send_slot.size());
        for (size_t q = 0; q < recv_keys[s].size(); ++q) {
            const int32_t k = recv_keys[s][q];
            recv_index.push_back({(int64_t)g.adj_elem[k] * nn + g.adj_local[k], r.recv_off.back() + (int32_t)q});
        }
        r.recv_off.push_back(r.recv_off.back() + (int32_t)recv_keys[s].size());
    }
    std::sort(recv_index.begin(), recv_index.end());
    lap("halo lists");
    // CSR per local node in canonical order: local slots and receive slots interleaved
    r.csr_off.assign(r.N + 1, 0);
    for (int li = 0; li < r.N; ++li) {
        const int i = r.node_orig[li];
        r.csr_off[li + 1] = r.csr_off[li] + (g.adj_off[i + 1] - g.adj_off[i]);
    }
    r.csr_slot.resize(r.csr_off[r.N]);
    const int32_t base = r.E * nn;
    int halo_miss = 0;
#pragma omp parallel for schedule(static) reduction(| : halo_miss)
    for (int li = 0; li < r.N; ++li) {
        const int i = r.node_orig[li];
        int32_t pos = r.csr_off[li];
        for (int k = g.adj_off[i]; k < g.adj_off[i + 1]; ++k) {
            const int e = g.adj_elem[k], a = g.adj_local[k];
            if (r.owner[e] == rank) {
                r.csr_slot[pos++] = elem_local[e] * nn + a;
            } else {
                const int64_t key = (int64_t)e * nn + a;
                auto it = std::lower_bound(recv_index.begin(), recv_index.end(), std::make_pair(key, (int32_t)-1));
                if (it == recv_index.end() || it->first != key) {
                    halo_miss = 1;
                    r.csr_slot[pos++] = 0;
                } else {
                    r.csr_slot[pos++] = base + it->second;
                }
            }
        }
    }
    if (halo_miss) throw Error(TVEGPU_E_ARG, "internal: halo map");
    lap("gather CSR");
    // every element contribution and every received one is gathered exactly once
    {
        const size_t ns = base + (r.recv_off.empty() ? 0 : r.recv_off.back());
        fvec<uint8_t> placed(ns);
#pragma omp parallel for schedule(static)
        for (size_t k = 0; k < ns; ++k) placed[k] = 0;
        int twice = 0, unplaced = 0;
        const size_t nc = r.csr_slot.size();
#pragma omp parallel for schedule(static) reduction(| : twice)
        for (size_t k = 0; k < nc; ++k) {
            const int32_t sl = r.csr_slot[k];
            if (sl < 0 || (size_t)sl >= ns || __atomic_fetch_add(&placed[sl], 1, __ATOMIC_RELAXED) != 0) twice = 1;
        }
#pragma omp parallel for schedule(static) reduction(| : unplaced)
        for (size_t k = 0; k < ns; ++k) unplaced |= placed[k] == 0;
        if (twice) throw Error(TVEGPU_E_ARG, "internal: contribution gathered twice");
        if (unplaced) throw Error(TVEGPU_E_ARG, "internal: unplaced contribution");
    }
    lap("exactly-once check");
    build_chunks(r);
    return r;
}

// Shared-memory slot assignment of one chunk's nodes.  Element kernels read
// node a of the 8 elements of a quarter-warp with one 16-byte shared load; the
// 8 lanes are conflict-free iff their slots differ mod 8 (eight 16-byte bank
// groups).  So the nodes are 8-coloured greedily over those co-read groups and
// slot = 8 * (rank within colour) + colour; empty slots hold node -1.
// Per-thread scratch of the chunk build (capacity kept across chunks: no allocation per
// chunk), with an open-addressing map node id -> index in the chunk's sorted node list.
struct ColourScratch {
    std::vector<int> gdata, gsize, moff, mlist, fill, colour;
    std::vector<int32_t> hkey, hval;
    std::vector<unsigned> used;  // occupied slots (cleared after each chunk)
    unsigned hmask = 0;
    void map_reserve(size_t n) {
        size_t cap = 64;
        while (cap < 2 * n) cap *= 2;
        if (hkey.size() < cap) {  // (only between chunks: the map is empty)
            hkey.assign(cap, -1);
            hval.assign(cap, 0);
        }
        hmask = (unsigned)hkey.size() - 1;
    }
    unsigned slot(int32_t n) const {
        unsigned h = (unsigned)n * 2654435761u;
        while (hkey[h & hmask] != -1 && hkey[h & hmask] != n) ++h;
        return h & hmask;
    }
    bool insert(int32_t n) {  // true if new
        const unsigned h = slot(n);
        if (hkey[h] == n) return false;
        hkey[h] = n;
        used.push_back(h);
        return true;
    }
    int index(int32_t n) const { return hval[slot(n)]; }
    void set_index(int32_t n, int v) { hval[slot(n)] = v; }
    void clear() {
        for (unsigned h : used) hkey[h] = -1;
        used.clear();
    }
};

static void colour_slots(const std::vector<int32_t>& nodes, const int32_t* conn, int ne, int nn,
                         std::vector<int32_t>& slot_of, std::vector<int32_t>& slots, ColourScratch& w) {
    const int nu = (int)nodes.size();
    auto idx = [&](int32_t n) { return w.index(n); };
    // groups: (quarter-warp q, local a) -> distinct node indices, flat (<= 8 per group);
    // member: per node the groups it belongs to, ascending (CSR)
    const int ngmax = ((ne + 7) / 8) * nn;
    w.gdata.resize((size_t)ngmax * 8);
    w.gsize.resize(ngmax);
    w.moff.assign(nu + 1, 0);
    int* gdata = w.gdata.data();
    int* gsize = w.gsize.data();
    int* moff = w.moff.data();
    int ng = 0;
    for (int q = 0; q * 8 < ne; ++q)
        for (int a = 0; a < nn; ++a) {
            int g[8], k = 0;
            for (int l = q * 8; l < std::min(ne, q * 8 + 8); ++l) g[k++] = idx(conn[(size_t)l * nn + a]);
            for (int x = 1; x < k; ++x)  // insertion sort of <= 8 ids
                for (int y = x; y > 0 && g[y - 1] > g[y]; --y) std::swap(g[y - 1], g[y]);
            k = (int)(std::unique(g, g + k) - g);
            if (k < 2) continue;
            for (int j = 0; j < k; ++j) {
                gdata[(size_t)ng * 8 + j] = g[j];
                moff[g[j] + 1]++;
            }
            gsize[ng++] = k;
        }
    for (int v = 0; v < nu; ++v) moff[v + 1] += moff[v];
    w.mlist.resize(moff[nu]);
    int* mlist = w.mlist.data();
    w.fill.assign(moff, moff + nu);
    for (int gi = 0; gi < ng; ++gi)
        for (int j = 0; j < gsize[gi]; ++j) mlist[w.fill[gdata[(size_t)gi * 8 + j]]++] = gi;
    auto group = [&](int gi) { return std::make_pair(&gdata[(size_t)gi * 8], &gdata[(size_t)gi * 8] + gsize[gi]); };
    // Colour group by group in issue order: the uncoloured members of a group take
    // the colours still free in that group (this propagates the 2x2x2 parity
    // colouring through structured meshes); when a group has no free colour left,
    // fall back to the colour least used across all of the node's groups.
    w.colour.assign(nu, -1);
    int* colour = w.colour.data();
    for (int gi = 0; gi < ng; ++gi) {
        const auto [g0, g1] = group(gi);
        bool used[8] = {false, false, false, false, false, false, false, false};
        for (const int* x = g0; x < g1; ++x)
            if (colour[*x] >= 0) used[colour[*x]] = true;
        for (const int* pv = g0; pv < g1; ++pv) {
            const int v = *pv;
            if (colour[v] >= 0) continue;
            int c = 0;
            while (c < 8 && used[c]) ++c;
            if (c == 8) {
                int uses[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                for (int m = moff[v]; m < moff[v + 1]; ++m) {
                    const auto [h0, h1] = group(mlist[m]);
                    for (const int* x = h0; x < h1; ++x)
                        if (colour[*x] >= 0) uses[colour[*x]]++;
                }
                c = 0;
                for (int k = 1; k < 8; ++k)
                    if (uses[k] < uses[c]) c = k;
            }
            colour[v] = c;
            used[c] = true;
        }
    }
    // local refinement (helps unstructured / tetrahedral chunks): move each node to the
    // colour with the fewest same-colour partners across its groups
    for (int sweep = 0; sweep < 4; ++sweep) {
        bool moved = false;
        for (int v = 0; v < nu; ++v) {
            if (colour[v] < 0 || moff[v] == moff[v + 1]) continue;
            int cost[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int m = moff[v]; m < moff[v + 1]; ++m) {
                const auto [h0, h1] = group(mlist[m]);
                for (const int* x = h0; x < h1; ++x)
                    if (*x != v && colour[*x] >= 0) cost[colour[*x]]++;
            }
            int best = colour[v];
            for (int c = 0; c < 8; ++c)
                if (cost[c] < cost[best]) best = c;
            if (best != colour[v]) {
                colour[v] = best;
                moved = true;
            }
        }
        if (!moved) break;
    }
    {
        int count[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int v = 0; v < nu; ++v)
            if (colour[v] >= 0) count[colour[v]]++;
        for (int v = 0; v < nu; ++v)
            if (colour[v] < 0) {  // in no conflict group: balance the colour classes
                const int c = (int)(std::min_element(count, count + 8) - count);
                colour[v] = c;
                count[c]++;
            }
    }
    int count[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    slot_of.resize(nu);
    for (int v = 0; v < nu; ++v) slot_of[v] = 8 * count[colour[v]]++ + colour[v];
    int rows = 0;
    for (int c = 0; c < 8; ++c) rows = std::max(rows, count[c]);
    slots.assign((size_t)8 * rows, -1);
    for (int v = 0; v < nu; ++v) slots[slot_of[v]] = nodes[v];
}

void build_chunks(RankPlan& r) {
    StageTimer tm("build_chunks");
    LapTimer lap;
    const int nn = r.nn;
    r.chunk_start.clear();
    r.chunk_node_off.assign(1, 0);
    r.chunk_nodes.clear();
    r.chunk_node_slot.clear();
    r.lconn.resize((size_t)r.E * nn);  // every entry written below
    r.max_chunk_nodes = 0;
    // chunk ranges: boundary elements [0, Eb) then interior [Eb, E), kChunk at a time
    std::vector<int32_t> starts;
    for (int c0 = 0; c0 < r.Eb; c0 += kChunk) starts.push_back(c0);
    r.nchunks_boundary = (int)starts.size();
    for (int c0 = r.Eb; c0 < r.E; c0 += kChunk) starts.push_back(c0);
    const int nc = (int)starts.size();
    auto chunk_end = [&](int c) { return c + 1 < nc ? starts[c + 1] : r.E; };
    // chunks are independent: unique nodes, colouring and 16-bit connectivity in parallel
    std::vector<std::vector<int32_t>> cnodes(nc), cslot(nc);
    std::vector<int32_t> nslots(nc, 0);
#pragma omp parallel
    {
        ColourScratch w;
        std::vector<int32_t> slots;
#pragma omp for schedule(dynamic, 16)
        for (int c = 0; c < nc; ++c) {
            const int c0 = starts[c], c1 = chunk_end(c);
            const int32_t* cc = r.conn.data() + (size_t)c0 * nn;
            const int m = (c1 - c0) * nn;
            w.map_reserve(m);
            std::vector<int32_t> nodes;
            nodes.reserve(m);
            for (int k = 0; k < m; ++k)
                if (w.insert(cc[k])) nodes.push_back(cc[k]);
            std::sort(nodes.begin(), nodes.end());
            for (int v = 0; v < (int)nodes.size(); ++v) w.set_index(nodes[v], v);
            std::vector<int32_t> slot_of;
            colour_slots(nodes, cc, c1 - c0, nn, slot_of, slots, w);
            for (int k = 0; k < m; ++k) r.lconn[(size_t)c0 * nn + k] = (uint16_t)slot_of[w.index(cc[k])];
            w.clear();
            nslots[c] = (int)slots.size();
            cnodes[c] = std::move(nodes);
            cslot[c] = std::move(slot_of);
        }
    }
    lap("unique nodes + colouring");
    // staging walks each chunk's nodes in ascending id (coalesced loads), storing each to its slot
    r.chunk_start.assign(starts.begin(), starts.end());
    r.chunk_start.push_back(r.E);
    r.chunk_node_off.resize((size_t)nc + 1);
    r.chunk_node_off[0] = 0;
    for (int c = 0; c < nc; ++c) {
        r.chunk_node_off[c + 1] = r.chunk_node_off[c] + (int32_t)cnodes[c].size();
        r.max_chunk_nodes = std::max(r.max_chunk_nodes, nslots[c]);
    }
    r.chunk_nodes.resize(r.chunk_node_off[nc]);
    r.chunk_node_slot.resize(r.chunk_node_off[nc]);
#pragma omp parallel for schedule(static)
    for (int c = 0; c < nc; ++c) {
        std::copy(cnodes[c].begin(), cnodes[c].end(), r.chunk_nodes.begin() + r.chunk_node_off[c]);
        for (size_t k = 0; k < cslot[c].size(); ++k) r.chunk_node_slot[r.chunk_node_off[c] + k] = (uint16_t)cslot[c][k];
    }
}

void critical_timestep_from_edge(const tvegpu_problem& p, double L, double* thermal, double* mechanical) {
    const double cd = std::sqrt((p.kappa + 4.0 * p.mu / 3.0) / p.density);
    double cmin = std::numeric_limits<double>::infinity(), kmax = -std::numeric_limits<double>::infinity();
    for (int i = 0; i < p.c_table_len; ++i) cmin = std::min(cmin, p.c_table_value[i]);
    for (int i = 0; i < p.k_table_len; ++i) kmax = std::max(kmax, sym_max_eig(p.k_table_tensor + 9 * (size_t)i));
    *mechanical = 0.9 * L / cd;
    *thermal = 0.9 * (p.density * cmin * L * L) / (2.0 * kmax * 3.0);
}

void critical_timestep(const tvegpu_problem& p, double* thermal, double* mechanical) {
    static const int t4e[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    static const int h8e[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6},
                                   {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
    const bool t4 = p.kind == TVEGPU_T4;
    const int nn = t4 ? 4 : 8, ne = t4 ? 6 : 12;
    double L = std::numeric_limits<double>::infinity();
#pragma omp parallel for schedule(static) reduction(min : L)
    for (int e = 0; e < p.num_elements; ++e) {
        const int32_t* el = p.elements + (size_t)e * nn;
        for (int k = 0; k < ne; ++k) {
            const int a = t4 ? t4e[k][0] : h8e[k][0], b = t4 ? t4e[k][1] : h8e[k][1];
            double d2 = 0;
            for (int i = 0; i < 3; ++i) {
                const double d = p.nodes[3 * (size_t)el[a] + i] - p.nodes[3 * (size_t)el[b] + i];
                d2 += d * d;
            }
            L = std::min(L, std::sqrt(d2));
        }
    }
    critical_timestep_from_edge(p, L, thermal, mechanical);
}

}  // namespace tvegpu
