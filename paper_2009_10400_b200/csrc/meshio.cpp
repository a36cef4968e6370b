// meshio.cpp — load_mesh (mesh.hpp:73-79; file format SPEC.md:88) for the setup
// pipeline at scale: the text is split into lines once, section
// headers are found serially, and the node / element / direction lines — the bulk of
// a 16M-element file — are parsed in parallel (OpenMP) straight into the flat arrays
// tvegpu_problem takes.  Validation as the reference states it: ParseError with a
// line number; ValidationError for mixed element kinds, out-of-range node indices
// (naming the element), inverted elements (naming the element), non-unit directions.
//
// Format decisions where SPEC.md:88 is silent: section headers are
// case-insensitive; every node / element id 1..N appears exactly once (any order);
// a set body is N whitespace-separated 1-based ids over any number of lines;
// `$expansion_axes` lines carry `elem_id mx my mz nx ny nz`; `#` starts a comment.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "plan.hpp"

namespace tvegpu {
void set_create_error(const std::string& m);
}

using namespace tvegpu;

struct tvegpu_mesh {
    int32_t kind = TVEGPU_T4;
    std::vector<double> nodes, fibers, axes;
    std::vector<int32_t> elements;
    std::vector<std::string> nset_names, eset_names;
    std::vector<const char*> nset_cstr, eset_cstr;
    std::vector<int32_t> nset_off{0}, nset_items, eset_off{0}, eset_items;
};

namespace {

struct Line {
    const char* b;
    const char* e;
};

[[noreturn]] void parse_fail(size_t line, const std::string& m) {
    throw Error(TVEGPU_E_PARSE, "line " + std::to_string(line + 1) + ": " + m);
}
[[noreturn]] void invalid(const std::string& m) { throw Error(TVEGPU_E_VALIDATION, m); }

// strip comment and surrounding blanks
Line clean(Line l) {
    const char* h = static_cast<const char*>(std::memchr(l.b, '#', l.e - l.b));
    if (h) l.e = h;
    while (l.b < l.e && std::isspace((unsigned char)*l.b)) ++l.b;
    while (l.e > l.b && std::isspace((unsigned char)l.e[-1])) --l.e;
    return l;
}

// Tokenizer over one line: numbers are parsed with strtod / strtol on a NUL-terminated copy.
struct Tok {
    char buf[512];
    std::string big;  // lines longer than buf (long set lines)
    char* p;
    explicit Tok(Line l) {
        const size_t n = (size_t)(l.e - l.b);
        if (n < sizeof buf) {
            std::memcpy(buf, l.b, n);
            buf[n] = 0;
            p = buf;
        } else {
            big.assign(l.b, n);
            p = &big[0];
        }
    }
    bool more() {
        while (*p && std::isspace((unsigned char)*p)) ++p;
        return *p != 0;
    }
    bool num(double& v) {
        if (!more()) return false;
        char* q;
        v = std::strtod(p, &q);
        if (q == p || (*q && !std::isspace((unsigned char)*q))) return false;
        p = q;
        return true;
    }
    bool integer(long& v) {
        if (!more()) return false;
        char* q;
        v = std::strtol(p, &q, 10);
        if (q == p || (*q && !std::isspace((unsigned char)*q))) return false;
        p = q;
        return true;
    }
    std::string word() {
        more();
        const char* s = p;
        while (*p && !std::isspace((unsigned char)*p)) ++p;
        return std::string(s, (size_t)(p - s));
    }
};

std::string lower(std::string s) {
    for (char& c : s) c = (char)std::tolower((unsigned char)c);
    return s;
}

double det3(const double a[3], const double b[3], const double c[3]) {
    return a[0] * (b[1] * c[2] - b[2] * c[1]) - a[1] * (b[0] * c[2] - b[2] * c[0]) + a[2] * (b[0] * c[1] - b[1] * c[0]);
}

// Parses `count` data lines of a section starting after header line h, in parallel:
// fn(line index, cleaned line) for each; data lines are the next non-blank lines.
template <class Fn>
size_t parse_rows(const std::vector<Line>& lines, size_t h, long count, Fn&& fn) {
    std::vector<size_t> rows;
    rows.reserve((size_t)count);
    size_t i = h + 1;
    for (; i < lines.size() && (long)rows.size() < count; ++i) {
        const Line l = clean(lines[i]);
        if (l.b == l.e) continue;
        if (*l.b == '$') parse_fail(i, "section ends after " + std::to_string(rows.size()) + " of " +
                                           std::to_string(count) + " lines");
        rows.push_back(i);
    }
    if ((long)rows.size() < count) parse_fail(lines.size() - 1, "unexpected end of file in section");
    std::string err;
    size_t err_line = 0;
    tvegpu_status err_status = TVEGPU_E_PARSE;
    bool failed = false;
#pragma omp parallel for schedule(static)
    for (long r = 0; r < count; ++r) {
        if (failed) continue;
        try {
            fn(rows[r], clean(lines[rows[r]]));
        } catch (const Error& ex) {
#pragma omp critical
            if (!failed || rows[r] < err_line) {
                failed = true;
                err = ex.what();
                err_status = ex.status;
                err_line = rows[r];
            }
        }
    }
    if (failed) throw Error(err_status, err);
    return i;
}

}  // namespace

namespace tvegpu {

tvegpu_mesh* load_mesh_text(const char* text, size_t len) {
    auto m = std::make_unique<tvegpu_mesh>();
    std::vector<Line> lines;
    {
        const char* p = text;
        const char* end = text + len;
        while (p < end) {
            const char* nl = static_cast<const char*>(std::memchr(p, '\n', end - p));
            const char* e = nl ? nl : end;
            lines.push_back({p, e});
            p = nl ? nl + 1 : end;
        }
    }
    long N = -1, E = -1;
    int nn = 0;
    bool have_fibers = false, have_axes = false;
    size_t i = 0;
    while (i < lines.size()) {
        const Line l = clean(lines[i]);
        if (l.b == l.e) {
            ++i;
            continue;
        }
        if (*l.b != '$') parse_fail(i, "expected a section header ($nodes, $elements, ...)");
        Tok t(l);
        const std::string sec = lower(t.word());
        long count = 0;
        if (sec == "$nodes") {
            if (N >= 0) parse_fail(i, "second $nodes section");
            if (!t.integer(count) || count < 1) parse_fail(i, "$nodes needs a positive count");
            N = count;
            m->nodes.assign(3 * (size_t)N, 0.0);
            std::vector<char> seen(N, 0);
            i = parse_rows(lines, i, count, [&](size_t ln, Line row) {
                Tok r(row);
                long id;
                double x[3];
                if (!r.integer(id) || !r.num(x[0]) || !r.num(x[1]) || !r.num(x[2]) || r.more())
                    parse_fail(ln, "node line must be `id x y z`");
                if (id < 1 || id > N) parse_fail(ln, "node id " + std::to_string(id) + " outside 1.." + std::to_string(N));
                if (seen[id - 1]) parse_fail(ln, "duplicate node id " + std::to_string(id));
                seen[id - 1] = 1;
                for (int c = 0; c < 3; ++c) m->nodes[3 * (size_t)(id - 1) + c] = x[c];
            });
        } else if (sec == "$elements") {
            if (E >= 0) parse_fail(i, "second $elements section");
            if (!t.integer(count) || count < 1) parse_fail(i, "$elements needs a positive count");
            const std::string kind = lower(t.word());
            if (kind == "t4") m->kind = TVEGPU_T4, nn = 4;
            else if (kind == "h8") m->kind = TVEGPU_H8, nn = 8;
            else parse_fail(i, "element kind must be t4 or h8");
            E = count;
            m->elements.assign((size_t)nn * E, -1);
            std::vector<char> seen(E, 0);
            i = parse_rows(lines, i, count, [&](size_t ln, Line row) {
                Tok r(row);
                long id, v[9];
                int k = 0;
                if (!r.integer(id)) parse_fail(ln, "element line must be `id n1 n2 ...`");
                while (r.more()) {
                    if (k == 9 || !r.integer(v[k])) parse_fail(ln, "element line must be `id n1 n2 ...`");
                    ++k;
                }
                if (k != nn) {
                    if (k == 4 || k == 8)
                        invalid("mixed element kinds: element " + std::to_string(id) + " has " + std::to_string(k) +
                                " nodes in a " + (nn == 4 ? "t4" : "h8") + " mesh");
                    parse_fail(ln, "element needs " + std::to_string(nn) + " node ids");
                }
                if (id < 1 || id > E) parse_fail(ln, "element id " + std::to_string(id) + " outside 1.." + std::to_string(E));
                if (seen[id - 1]) parse_fail(ln, "duplicate element id " + std::to_string(id));
                seen[id - 1] = 1;
                for (int a = 0; a < nn; ++a) m->elements[(size_t)nn * (id - 1) + a] = (int32_t)(v[a] - 1);
            });
        } else if (sec == "$nodeset" || sec == "$elemset") {
            const std::string name = t.word();
            if (name.empty() || !t.integer(count) || count < 0) parse_fail(i, sec + " needs `name count`");
            std::vector<int32_t> ids;
            ids.reserve(count);
            size_t j = i + 1;
            for (; j < lines.size() && (long)ids.size() < count; ++j) {
                const Line row = clean(lines[j]);
                if (row.b == row.e) continue;
                if (*row.b == '$') break;
                Tok r(row);
                long v;
                while (r.more()) {
                    if (!r.integer(v)) parse_fail(j, "set entries must be integer ids");
                    ids.push_back((int32_t)(v - 1));
                }
            }
            if ((long)ids.size() != count) parse_fail(j - 1, sec + " " + name + ": expected " + std::to_string(count) + " ids");
            auto& names = sec == "$nodeset" ? m->nset_names : m->eset_names;
            auto& off = sec == "$nodeset" ? m->nset_off : m->eset_off;
            auto& items = sec == "$nodeset" ? m->nset_items : m->eset_items;
            names.push_back(name);
            items.insert(items.end(), ids.begin(), ids.end());
            off.push_back((int32_t)items.size());
            i = j;
        } else if (sec == "$fibers" || sec == "$expansion_axes") {
            const bool fib = sec == "$fibers";
            if (E < 0) parse_fail(i, sec + " must follow $elements");
            if (!t.integer(count) || count != E) parse_fail(i, sec + " count must equal the element count");
            const int w = fib ? 3 : 6;
            auto& dst = fib ? m->fibers : m->axes;
            dst.assign((size_t)w * E, 0.0);
            (fib ? have_fibers : have_axes) = true;
            std::vector<char> seen(E, 0);
            i = parse_rows(lines, i, count, [&](size_t ln, Line row) {
                Tok r(row);
                long id;
                double v[6];
                if (!r.integer(id)) parse_fail(ln, "direction line must start with the element id");
                for (int k = 0; k < w; ++k)
                    if (!r.num(v[k])) parse_fail(ln, fib ? "fiber line must be `elem ax ay az`" : "axes line must be `elem mx my mz nx ny nz`");
                if (r.more()) parse_fail(ln, "trailing tokens");
                if (id < 1 || id > E) parse_fail(ln, "element id " + std::to_string(id) + " outside 1.." + std::to_string(E));
                if (seen[id - 1]) parse_fail(ln, "duplicate element id " + std::to_string(id));
                seen[id - 1] = 1;
                for (int q = 0; q < w; q += 3)
                    if (std::fabs(std::sqrt(v[q] * v[q] + v[q + 1] * v[q + 1] + v[q + 2] * v[q + 2]) - 1.0) > 1e-6)
                        invalid("non-unit direction vector for element " + std::to_string(id));
                for (int k = 0; k < w; ++k) dst[(size_t)w * (id - 1) + k] = v[k];
            });
        } else {
            parse_fail(i, "unknown section " + sec);
        }
    }
    if (N < 0) invalid("mesh has no $nodes section");
    if (E < 0) invalid("mesh has no $elements section");
    // validation (mesh.hpp:73-75): out-of-range indices and inverted elements, lowest element id first
    long bad_range = -1, bad_vol = -1;
#pragma omp parallel for schedule(static) reduction(max : bad_range, bad_vol)
    for (long e = 0; e < E; ++e) {
        const int32_t* el = m->elements.data() + (size_t)nn * e;
        bool ok = true;
        for (int a = 0; a < nn; ++a) ok &= el[a] >= 0 && el[a] < N;
        if (!ok) {
            bad_range = std::max(bad_range, E - e);
            continue;
        }
        auto X = [&](int a, int c) { return m->nodes[3 * (size_t)el[a] + c]; };
        double v;
        if (nn == 4) {
            double a[3], b[3], c[3];
            for (int q = 0; q < 3; ++q) a[q] = X(1, q) - X(0, q), b[q] = X(2, q) - X(0, q), c[q] = X(3, q) - X(0, q);
            v = det3(a, b, c);  // columns: edges from node 0
        } else {  // centroid Jacobian of the trilinear brick map (sign of det J0)
            static const int s[8][3] = {{-1, -1, -1}, {1, -1, -1}, {1, 1, -1}, {-1, 1, -1},
                                        {-1, -1, 1},  {1, -1, 1},  {1, 1, 1},  {-1, 1, 1}};
            double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
            for (int a = 0; a < 8; ++a)
                for (int i2 = 0; i2 < 3; ++i2)
                    for (int j = 0; j < 3; ++j) J[j][i2] += s[a][j] * X(a, i2);
            v = det3(J[0], J[1], J[2]);
        }
        if (!(v > 0)) bad_vol = std::max(bad_vol, E - e);
    }
    if (bad_range >= 0) invalid("element " + std::to_string(E - bad_range + 1) + " references a node outside 1.." + std::to_string(N));
    if (bad_vol >= 0) invalid("inverted or degenerate element " + std::to_string(E - bad_vol + 1));
    for (const auto& items : {&m->nset_items})
        for (int32_t v : *items)
            if (v < 0 || v >= N) invalid("node set entry " + std::to_string(v + 1) + " outside 1.." + std::to_string(N));
    for (int32_t v : m->eset_items)
        if (v < 0 || v >= E) invalid("element set entry " + std::to_string(v + 1) + " outside 1.." + std::to_string(E));
    if (!have_fibers) m->fibers.clear();
    if (!have_axes) m->axes.clear();
    for (auto& s : m->nset_names) m->nset_cstr.push_back(s.c_str());
    for (auto& s : m->eset_names) m->eset_cstr.push_back(s.c_str());
    return m.release();
}

}  // namespace tvegpu

extern "C" {

tvegpu_status tvegpu_load_mesh(const char* text, uint64_t len, tvegpu_mesh** out, tvegpu_mesh_view* view) {
    if (!text || !out) return TVEGPU_E_ARG;
    *out = nullptr;
    try {
        tvegpu_mesh* m = load_mesh_text(text, (size_t)len);
        *out = m;
        if (view) tvegpu_mesh_get_view(m, view);
        return TVEGPU_OK;
    } catch (const Error& e) {
        set_create_error(e.what());
        return e.status;
    } catch (const std::exception& e) {
        set_create_error(e.what());
        return TVEGPU_E_PARSE;
    }
}

void tvegpu_mesh_get_view(const tvegpu_mesh* m, tvegpu_mesh_view* v) {
    if (!m || !v) return;
    const int nn = m->kind == TVEGPU_H8 ? 8 : 4;
    v->kind = m->kind;
    v->num_nodes = (int32_t)(m->nodes.size() / 3);
    v->num_elements = (int32_t)(m->elements.size() / nn);
    v->nodes = m->nodes.data();
    v->elements = m->elements.data();
    v->fiber_dirs = m->fibers.empty() ? nullptr : m->fibers.data();
    v->expansion_axes = m->axes.empty() ? nullptr : m->axes.data();
    v->num_node_sets = (int32_t)m->nset_names.size();
    v->node_set_names = m->nset_cstr.data();
    v->node_set_offsets = m->nset_off.data();
    v->node_set_items = m->nset_items.data();
    v->num_element_sets = (int32_t)m->eset_names.size();
    v->element_set_names = m->eset_cstr.data();
    v->element_set_offsets = m->eset_off.data();
    v->element_set_items = m->eset_items.data();
}

void tvegpu_mesh_destroy(tvegpu_mesh* m) { delete m; }

}  // extern "C"
