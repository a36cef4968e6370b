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

// inverse-transpose via the adjugate: (J^-1)^T = cof(J) / det J
void inv_transpose(const double J[3][3], double d, double out[3][3]) {
    out[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / d;
    out[0][1] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / d;
    out[0][2] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / d;
    out[1][0] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / d;
    out[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / d;
    out[1][2] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / d;
    out[2][0] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / d;
    out[2][1] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / d;
    out[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / d;
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
    for (int64_t k = 0; k < (int64_t)p.num_elements * nn; ++k) {
        const int v = p.elements[k];
        if (v < 0 || v >= p.num_nodes)
            invalid("element " + std::to_string(k / nn + 1) + " references out-of-range node " + std::to_string(v + 1));
    }
    if (!(p.mu > 0) || !(p.kappa > 0) || p.eta_a < 0) invalid("hyperelastic parameters need mu > 0, kappa > 0, eta_a >= 0");
    double sphi = 0;
    for (int i = 0; i < p.prony_count; ++i) {
        if (!(p.prony_phi[i] > 0) || !(p.prony_tau[i] > 0)) invalid("Prony terms need phi > 0 and tau > 0");
        sphi += p.prony_phi[i];
    }
    if (p.prony_count > 0 && !(sphi < 1.0)) invalid("Prony weights must sum to < 1");
    if (p.prony_count > 4) invalid("at most 4 Prony terms are supported on the device");
    if (!(p.density > 0)) invalid("density must be > 0");
    if (p.c_table_len < 1 || p.c_table_len > 16 || p.k_table_len < 1 || p.k_table_len > 16)
        invalid("property tables need 1..16 entries");
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
    g.A.resize((size_t)9 * E);
    g.vol.resize(E);
    g.centroid.resize((size_t)3 * E);
    for (int k = 0; k < 3; ++k) {
        g.lo[k] = std::numeric_limits<double>::infinity();
        g.hi[k] = -std::numeric_limits<double>::infinity();
    }
    int bad = -1;
#pragma omp parallel for schedule(static) reduction(max : bad)
    for (int e = 0; e < E; ++e) {
        const int32_t* el = p.elements + (size_t)e * nn;
        double J[3][3];
        if (nn == 4) {
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) J[i][j] = p.nodes[3 * (size_t)el[j + 1] + i] - p.nodes[3 * (size_t)el[0] + i];
        } else {
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    double s = 0;
                    for (int a = 0; a < 8; ++a) s += p.nodes[3 * (size_t)el[a] + i] * kH8Sign[a][j];
                    J[i][j] = s / 8.0;
                }
        }
        const double d = det3(J);
        const double V = nn == 4 ? d / 6.0 : 8.0 * d;
        if (!(V > 0)) {
            bad = std::max(bad, E - e);  // keep the LOWEST failing element
            continue;
        }
        double Ai[3][3];
        inv_transpose(J, d, Ai);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) g.A[(size_t)9 * e + i * 3 + j] = nn == 4 ? Ai[i][j] : Ai[i][j] / 8.0;
        g.vol[e] = V;
        for (int k = 0; k < 3; ++k) {
            double s = 0;
            for (int a = 0; a < nn; ++a) s += p.nodes[3 * (size_t)el[a] + k];
            g.centroid[(size_t)3 * e + k] = s / nn;
        }
    }
    if (bad >= 0) invalid("degenerate or inverted element " + std::to_string(E - bad + 1));
    {
        static const int t4e[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
        static const int h8e[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6},
                                       {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
        double L = std::numeric_limits<double>::infinity();
#pragma omp parallel for schedule(static) reduction(min : L)
        for (int e = 0; e < E; ++e) {
            const int32_t* el = p.elements + (size_t)e * nn;
            for (int k = 0; k < (nn == 4 ? 6 : 12); ++k) {
                const int a = nn == 4 ? t4e[k][0] : h8e[k][0], b = nn == 4 ? t4e[k][1] : h8e[k][1];
                double d2 = 0;
                for (int i = 0; i < 3; ++i) {
                    const double d = p.nodes[3 * (size_t)el[a] + i] - p.nodes[3 * (size_t)el[b] + i];
                    d2 += d * d;
                }
                L = std::min(L, std::sqrt(d2));
            }
        }
        g.min_edge = L;
    }
    for (int e = 0; e < E; ++e)
        for (int k = 0; k < 3; ++k) {
            g.lo[k] = std::min(g.lo[k], g.centroid[(size_t)3 * e + k]);
            g.hi[k] = std::max(g.hi[k], g.centroid[(size_t)3 * e + k]);
        }
    lap("element geometry + bounds");
    // canonical adjacency over original ids
    g.adj_off.assign(N + 1, 0);
    for (int64_t k = 0; k < (int64_t)E * nn; ++k) g.adj_off[p.elements[k] + 1]++;
    for (int i = 0; i < N; ++i) g.adj_off[i + 1] += g.adj_off[i];
    g.adj_elem.resize((size_t)E * nn);
    g.adj_local.resize((size_t)E * nn);
    {
        std::vector<int32_t> fill(g.adj_off.begin(), g.adj_off.end() - 1);
        for (int e = 0; e < E; ++e)
            for (int a = 0; a < nn; ++a) {
                const int i = p.elements[(size_t)e * nn + a];
                g.adj_elem[fill[i]] = e;
                g.adj_local[fill[i]] = a;
                fill[i]++;
            }
    }
    lap("adjacency");
    g.mass.assign(N, 0.0);
    g.vnode.assign(N, 0.0);
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
    // sharers of each node: bitmask of ranks touching it (nranks <= 64)
    if (nranks > 64) throw Error(TVEGPU_E_ARG, "at most 64 ranks");
    std::vector<uint64_t> touch(N, 0);
    for (int e = 0; e < E; ++e)
        for (int a = 0; a < nn; ++a) touch[p.elements[(size_t)e * nn + a]] |= 1ULL << r.owner[e];
    const uint64_t me = 1ULL << rank;
    // owned elements, split into boundary (touches a shared node) and interior
    std::vector<int32_t> bnd, inr;
    for (int e = 0; e < E; ++e) {
        if (r.owner[e] != rank) continue;
        bool b = false;
        for (int a = 0; a < nn && !b; ++a) b = (touch[p.elements[(size_t)e * nn + a]] & ~me) != 0;
        (b ? bnd : inr).push_back(e);
    }
    if (reorder) {
        std::vector<uint64_t> key(E);
        const double mscale = morton_scale(g);
        auto sort_group = [&](std::vector<int32_t>& v) {
#pragma omp parallel for schedule(static)
            for (size_t q = 0; q < v.size(); ++q) key[v[q]] = morton_key(&g.centroid[(size_t)3 * v[q]], g.lo, mscale);
            // a total order (ties broken by id): the parallel sort's result is unique
            __gnu_parallel::sort(v.begin(), v.end(),
                                 [&](int32_t x, int32_t y) { return key[x] < key[y] || (key[x] == key[y] && x < y); });
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
    r.elem_orig = bnd;
    r.elem_orig.insert(r.elem_orig.end(), inr.begin(), inr.end());
    r.E = (int)r.elem_orig.size();
    // first-touch node numbering (identity when reorder = 0, nranks = 1)
    std::vector<int32_t> local(N, -1);
    if (reorder) {
        for (int le = 0; le < r.E; ++le)
            for (int a = 0; a < nn; ++a) {
                const int i = p.elements[(size_t)r.elem_orig[le] * nn + a];
                if (local[i] < 0) {
                    local[i] = (int)r.node_orig.size();
                    r.node_orig.push_back(i);
                }
            }
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
    std::vector<int32_t> elem_local(E, -1);
#pragma omp parallel for schedule(static)
    for (int le = 0; le < r.E; ++le) {
        elem_local[r.elem_orig[le]] = le;
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
        std::vector<uint8_t> placed(ns, 0);
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
static std::vector<int32_t> colour_slots(const std::vector<int32_t>& nodes, const int32_t* conn, int ne, int nn,
                                         std::vector<int32_t>& slot_of) {
    const int nu = (int)nodes.size();
    auto idx = [&](int32_t n) { return (int)(std::lower_bound(nodes.begin(), nodes.end(), n) - nodes.begin()); };
    // groups: (quarter-warp q, local a) -> distinct node indices, flat (<= 8 per group);
    // member: per node the groups it belongs to, ascending (CSR)
    const int ngmax = ((ne + 7) / 8) * nn;
    std::vector<int> gdata((size_t)ngmax * 8), gsize(ngmax), moff(nu + 1, 0);
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
    std::vector<int> mlist(moff[nu]);
    {
        std::vector<int> fill(moff.begin(), moff.end() - 1);
        for (int gi = 0; gi < ng; ++gi)
            for (int j = 0; j < gsize[gi]; ++j) mlist[fill[gdata[(size_t)gi * 8 + j]]++] = gi;
    }
    auto group = [&](int gi) { return std::make_pair(&gdata[(size_t)gi * 8], &gdata[(size_t)gi * 8] + gsize[gi]); };
    // Colour group by group in issue order: the uncoloured members of a group take
    // the colours still free in that group (this propagates the 2x2x2 parity
    // colouring through structured meshes); when a group has no free colour left,
    // fall back to the colour least used across all of the node's groups.
    std::vector<int> colour(nu, -1);
    for (int gi = 0; gi < ng; ++gi) {
        const auto [g0, g1] = group(gi);
        bool used[8] = {false, false, false, false, false, false, false, false};
        for (const int* w = g0; w < g1; ++w)
            if (colour[*w] >= 0) used[colour[*w]] = true;
        for (const int* pv = g0; pv < g1; ++pv) {
            const int v = *pv;
            if (colour[v] >= 0) continue;
            int c = 0;
            while (c < 8 && used[c]) ++c;
            if (c == 8) {
                int uses[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                for (int m = moff[v]; m < moff[v + 1]; ++m) {
                    const auto [h0, h1] = group(mlist[m]);
                    for (const int* w = h0; w < h1; ++w)
                        if (colour[*w] >= 0) uses[colour[*w]]++;
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
                for (const int* w = h0; w < h1; ++w)
                    if (*w != v && colour[*w] >= 0) cost[colour[*w]]++;
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
    slot_of.assign(nu, 0);
    for (int v = 0; v < nu; ++v) slot_of[v] = 8 * count[colour[v]]++ + colour[v];
    int rows = 0;
    for (int c = 0; c < 8; ++c) rows = std::max(rows, count[c]);
    std::vector<int32_t> slots((size_t)8 * rows, -1);
    for (int v = 0; v < nu; ++v) slots[slot_of[v]] = nodes[v];
    return slots;
}

void build_chunks(RankPlan& r) {
    StageTimer tm("build_chunks");
    LapTimer lap;
    const int nn = r.nn;
    r.chunk_start.clear();
    r.chunk_node_off.assign(1, 0);
    r.chunk_nodes.clear();
    r.chunk_node_slot.clear();
    r.lconn.assign((size_t)r.E * nn, 0);
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
#pragma omp parallel for schedule(dynamic, 16)
    for (int c = 0; c < nc; ++c) {
        const int c0 = starts[c], c1 = chunk_end(c);
        std::vector<int32_t> nodes(r.conn.begin() + (size_t)c0 * nn, r.conn.begin() + (size_t)c1 * nn);
        std::sort(nodes.begin(), nodes.end());
        nodes.erase(std::unique(nodes.begin(), nodes.end()), nodes.end());
        std::vector<int32_t> slot_of;
        const std::vector<int32_t> slots = colour_slots(nodes, r.conn.data() + (size_t)c0 * nn, c1 - c0, nn, slot_of);
        for (int le = c0; le < c1; ++le)
            for (int a = 0; a < nn; ++a) {
                const int32_t n = r.conn[(size_t)le * nn + a];
                const int v = (int)(std::lower_bound(nodes.begin(), nodes.end(), n) - nodes.begin());
                r.lconn[(size_t)le * nn + a] = (uint16_t)slot_of[v];
            }
        nslots[c] = (int)slots.size();
        cnodes[c] = std::move(nodes);
        cslot[c] = std::move(slot_of);
    }
    lap("unique nodes + colouring");
    // staging walks each chunk's nodes in ascending id (coalesced loads), storing each to its slot
    for (int c = 0; c < nc; ++c) {
        r.chunk_start.push_back(starts[c]);
        r.chunk_nodes.insert(r.chunk_nodes.end(), cnodes[c].begin(), cnodes[c].end());
        for (int32_t s : cslot[c]) r.chunk_node_slot.push_back((uint16_t)s);
        r.chunk_node_off.push_back((int32_t)r.chunk_nodes.size());
        r.max_chunk_nodes = std::max(r.max_chunk_nodes, nslots[c]);
    }
    r.chunk_start.push_back(r.E);
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
