// tve_gpu_cli.cpp — the reference's command-line entry point (run |
// check | verify | bench, exit codes 0 success / 1 config or validation / 2 instability
// / 3 verification failure) over the B200 engine's C++ facade (include/tve_gpu.hpp).
// SURVEY §8 f-4.  Host plumbing: parsing, output files, timing; all physics runs in
// libtvegpu.
//
// Config: flat sectioned key = value text, SI units, °C, '#' comments;
// unknown sections / keys are errors; `--override section.key=value` applies after
// parsing (repeatable).  Keys are listed in kKeys below; tables are `T:v, T:v`.
//
//   g++ -std=c++17 -O2 -I include tools/tve_gpu_cli.cpp -L paper_2009_10400_b200/lib -ltvegpu
//       -Wl,-rpath,$PWD/paper_2009_10400_b200/lib -o build/tve_gpu
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "tve_gpu.hpp"

using namespace tve::gpu;
namespace fs = std::filesystem;

namespace {

struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };

// section -> allowed keys (repeatable keys may appear several times, in order)
const std::map<std::string, std::set<std::string>> kKeys = {
    {"mesh", {"file"}},
    {"material", {"mu", "kappa", "eta_a", "fiber"}},
    {"thermal", {"density", "specific_heat", "conductivity", "perfusion_rate", "blood_specific_heat",
                 "arterial_temperature", "metabolic_rate", "initial_temperature", "reference_specific_heat"}},
    {"expansion", {"kind", "alpha_i", "alpha_m", "alpha_n", "reference_temperature", "axis_m", "axis_n"}},
    {"viscoelastic", {"prony"}},
    {"sources", {"sphere", "element_set"}},
    {"bcs", {"fixed", "prescribed", "fixed_temperature", "body_force"}},
    {"sim", {"dt", "duration", "coupling", "expansion", "temperature_dependent", "damping_gamma",
             "hourglass_stiffness", "allow_unstable_dt", "workers"}},
    {"output", {"snapshot_interval", "probe_nodes", "ablation_threshold", "write_det_f", "write_stress"}}};
const std::set<std::string> kRepeatable = {"sources.sphere", "sources.element_set", "bcs.prescribed",
                                           "bcs.fixed_temperature", "bcs.fixed"};

using Config = std::vector<std::pair<std::string, std::string>>;  // "section.key" -> value, file order

std::string trim(const std::string& s) {
    const size_t a = s.find_first_not_of(" \t\r"), b = s.find_last_not_of(" \t\r");
    return a == std::string::npos ? "" : s.substr(a, b - a + 1);
}

void check_key(const std::string& dotted, const std::string& where) {
    const size_t d = dotted.find('.');
    const std::string sec = dotted.substr(0, d), key = d == std::string::npos ? "" : dotted.substr(d + 1);
    auto it = kKeys.find(sec);
    if (it == kKeys.end()) throw ConfigError(where + ": unknown section [" + sec + "]");
    if (!it->second.count(key)) throw ConfigError(where + ": unknown key '" + key + "' in [" + sec + "]");
}

Config parse_config(const std::string& text) {
    Config c;
    std::istringstream in(text);
    std::string line, sec;
    for (int ln = 1; std::getline(in, line); ++ln) {
        const size_t h = line.find('#');
        if (h != std::string::npos) line = line.substr(0, h);
        line = trim(line);
        if (line.empty()) continue;
        const std::string where = "config line " + std::to_string(ln);
        if (line.front() == '[') {
            if (line.back() != ']') throw ConfigError(where + ": malformed section header");
            sec = trim(line.substr(1, line.size() - 2));
            if (!kKeys.count(sec)) throw ConfigError(where + ": unknown section [" + sec + "]");
            continue;
        }
        const size_t eq = line.find('=');
        if (eq == std::string::npos || sec.empty()) throw ConfigError(where + ": expected key = value inside a section");
        const std::string key = sec + "." + trim(line.substr(0, eq));
        check_key(key, where);
        if (!kRepeatable.count(key))
            for (const auto& kv : c)
                if (kv.first == key) throw ConfigError(where + ": duplicate key " + key);
        c.push_back({key, trim(line.substr(eq + 1))});
    }
    return c;
}

void apply_override(Config& c, const std::string& kv) {
    const size_t eq = kv.find('=');
    if (eq == std::string::npos) throw ConfigError("override '" + kv + "' is not section.key=value");
    const std::string key = trim(kv.substr(0, eq)), val = trim(kv.substr(eq + 1));
    check_key(key, "override");
    c.erase(std::remove_if(c.begin(), c.end(), [&](const auto& p) { return p.first == key; }), c.end());
    c.push_back({key, val});
}

std::vector<std::string> all(const Config& c, const std::string& key) {
    std::vector<std::string> v;
    for (const auto& kv : c)
        if (kv.first == key) v.push_back(kv.second);
    return v;
}
bool has(const Config& c, const std::string& key) { return !all(c, key).empty(); }
std::string get(const Config& c, const std::string& key, const std::string& dflt = "") {
    const auto v = all(c, key);
    return v.empty() ? dflt : v.back();
}
double num(const std::string& s, const std::string& key) {
    char* e = nullptr;
    const double v = std::strtod(s.c_str(), &e);
    if (e == s.c_str() || trim(e) != "") throw ConfigError(key + ": '" + s + "' is not a number");
    return v;
}
double getd(const Config& c, const std::string& key, double dflt) { return has(c, key) ? num(get(c, key), key) : dflt; }
bool getb(const Config& c, const std::string& key, bool dflt) {
    if (!has(c, key)) return dflt;
    const std::string v = get(c, key);
    if (v == "on" || v == "true" || v == "1" || v == "yes") return true;
    if (v == "off" || v == "false" || v == "0" || v == "no") return false;
    throw ConfigError(key + ": expected on/off");
}
std::vector<double> nums(const std::string& s, const std::string& key) {
    std::vector<double> v;
    std::istringstream in(s);
    std::string t;
    while (in >> t) v.push_back(num(t, key));
    return v;
}
// "T:v, T:v"; with allow_scalar a bare value is a constant property (a one-point table)
std::vector<std::pair<double, double>> table(const std::string& s, const std::string& key, bool allow_scalar = false) {
    std::vector<std::pair<double, double>> t;
    if (allow_scalar && s.find(':') == std::string::npos && s.find(',') == std::string::npos)
        return {{37.0, num(trim(s), key)}};
    std::string item;
    std::istringstream in(s);
    while (std::getline(in, item, ',')) {
        const size_t c = item.find(':');
        if (c == std::string::npos) throw ConfigError(key + ": table entries are T:value");
        t.push_back({num(trim(item.substr(0, c)), key), num(trim(item.substr(c + 1)), key)});
    }
    if (t.empty()) throw ConfigError(key + ": empty table");
    return t;
}

struct Setup {
    Mesh mesh;
    MaterialModel mat;
    MechBCs mb;
    ThermalBCs tb;
    HeatSourceSet src;
    SimulationConfig cfg;
    double snapshot_interval = 0, ablation_threshold = 60.0;
    std::vector<int> probes;
    fs::path mesh_path;
};

const std::vector<int>& nodeset(const Mesh& m, const std::string& name) {
    auto it = m.node_sets.find(name);
    if (it == m.node_sets.end()) throw ConfigError("unknown node set '" + name + "'");
    return it->second;
}

Setup build_setup(const Config& c, const fs::path& base) {
    Setup s;
    if (!has(c, "mesh.file")) throw ConfigError("missing required key mesh.file");
    for (const char* k : {"sim.dt", "thermal.density", "material.mu", "material.kappa"})
        if (!has(c, k)) throw ConfigError(std::string("missing required key ") + k);
    s.mesh_path = fs::path(get(c, "mesh.file"));
    if (s.mesh_path.is_relative()) s.mesh_path = base / s.mesh_path;
    s.mesh = load_mesh_file(s.mesh_path.string());
    auto& m = s.mat;
    m.hyperelastic = {getd(c, "material.mu", 0), getd(c, "material.kappa", 0), getd(c, "material.eta_a", 0)};
    if (m.hyperelastic.mu <= 0 || m.hyperelastic.kappa <= 0) throw ConfigError("material.mu and material.kappa must be > 0");
    if (has(c, "material.fiber")) {
        const auto f = nums(get(c, "material.fiber"), "material.fiber");
        if (f.size() != 3) throw ConfigError("material.fiber needs 3 numbers");
        m.fiber = Vec3{f[0], f[1], f[2]};
    }
    m.thermal.density = getd(c, "thermal.density", 0);
    if (m.thermal.density <= 0) throw ConfigError("thermal.density must be > 0");
    for (auto [T, v] : table(get(c, "thermal.specific_heat", "37:3600"), "thermal.specific_heat", true))
        m.thermal.specific_heat.entries.push_back({T, v});
    m.thermal.conductivity.entries.clear();
    for (auto [T, k] : table(get(c, "thermal.conductivity", "37:0.53"), "thermal.conductivity", true))
        m.thermal.conductivity.entries.push_back({T, {k, 0, 0, 0, k, 0, 0, 0, k}});
    m.thermal.perfusion_rate = getd(c, "thermal.perfusion_rate", 0);
    m.thermal.blood_specific_heat = getd(c, "thermal.blood_specific_heat", 0);
    m.thermal.arterial_temperature = getd(c, "thermal.arterial_temperature", 37.0);
    m.thermal.metabolic_rate = getd(c, "thermal.metabolic_rate", 0);
    s.tb.initial_temperature = getd(c, "thermal.initial_temperature", 37.0);
    if (has(c, "expansion.kind") || has(c, "expansion.alpha_i")) {
        ExpansionSpec e;
        const std::string k = get(c, "expansion.kind", "isotropic");
        e.kind = k == "isotropic" ? ExpansionKind::Isotropic
                 : k == "transversely_isotropic" ? ExpansionKind::TransverselyIsotropic
                 : k == "orthotropic" ? ExpansionKind::Orthotropic
                                      : throw ConfigError("expansion.kind: isotropic | transversely_isotropic | orthotropic");
        e.alpha_i = getd(c, "expansion.alpha_i", 0);
        e.alpha_m = getd(c, "expansion.alpha_m", 0);
        e.alpha_n = getd(c, "expansion.alpha_n", 0);
        e.reference_temperature = getd(c, "expansion.reference_temperature", 37.0);
        m.expansion = e;
        for (const char* ax : {"expansion.axis_m", "expansion.axis_n"})
            if (has(c, ax)) {
                const auto v = nums(get(c, ax), ax);
                if (v.size() != 3) throw ConfigError(std::string(ax) + " needs 3 numbers");
                (std::string(ax) == "expansion.axis_m" ? m.axis_m : m.axis_n) = Vec3{v[0], v[1], v[2]};
            }
    }
    if (has(c, "viscoelastic.prony"))
        for (auto [phi, tau] : table(get(c, "viscoelastic.prony"), "viscoelastic.prony")) m.prony.terms.push_back({phi, tau});
    // sources: sphere = cx cy cz diameter q_r [t_start t_end];  element_set = name q_r [t_start t_end]
    for (const auto& v : all(c, "sources.sphere")) {
        const auto a = nums(v, "sources.sphere");
        if (a.size() != 5 && a.size() != 7) throw ConfigError("sources.sphere = cx cy cz diameter q_r [t_start t_end]");
        SourceRegion r;
        r.q_r = a[4];
        if (a.size() == 7) r.t_start = a[5], r.t_end = a[6];
        const int nn = s.mesh.kind == ElementKind::H8 ? 8 : 4;
        for (int e = 0; e < s.mesh.element_count(); ++e) {  // centroid inclusion
            double x[3] = {0, 0, 0};
            for (int q = 0; q < nn; ++q)
                for (int k = 0; k < 3; ++k) x[k] += s.mesh.nodes[s.mesh.elements[e][q]][k] / nn;
            const double d2 = (x[0] - a[0]) * (x[0] - a[0]) + (x[1] - a[1]) * (x[1] - a[1]) + (x[2] - a[2]) * (x[2] - a[2]);
            if (d2 <= 0.25 * a[3] * a[3]) r.elements.push_back(e);
        }
        s.src.regional.push_back(r);
    }
    for (const auto& v : all(c, "sources.element_set")) {
        std::istringstream in(v);
        std::string name;
        in >> name;
        std::string rest((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        const auto a = nums(rest, "sources.element_set");
        if (a.size() != 1 && a.size() != 3) throw ConfigError("sources.element_set = name q_r [t_start t_end]");
        auto it = s.mesh.element_sets.find(name);
        if (it == s.mesh.element_sets.end()) throw ConfigError("unknown element set '" + name + "'");
        SourceRegion r;
        r.elements = it->second;
        r.q_r = a[0];
        if (a.size() == 3) r.t_start = a[1], r.t_end = a[2];
        s.src.regional.push_back(r);
    }
    // bcs: fixed = nodeset ...;  prescribed = nodeset component target [ramp_time];
    //      fixed_temperature = nodeset value;  body_force = bx by bz
    for (const auto& v : all(c, "bcs.fixed")) {
        std::istringstream in(v);
        std::string name;
        while (in >> name) for (int n : nodeset(s.mesh, name)) s.mb.fixed_nodes.push_back(n);
    }
    for (const auto& v : all(c, "bcs.prescribed")) {
        std::istringstream in(v);
        std::string name;
        in >> name;
        std::string rest((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        const auto a = nums(rest, "bcs.prescribed");
        if (a.size() != 2 && a.size() != 3) throw ConfigError("bcs.prescribed = nodeset component target [ramp_time]");
        PrescribedDisplacement p;
        p.nodes = nodeset(s.mesh, name);
        p.component = (int)a[0];
        p.target = a[1];
        p.ramp_time = a.size() == 3 ? a[2] : 0.0;
        s.mb.prescribed.push_back(p);
    }
    for (const auto& v : all(c, "bcs.fixed_temperature")) {
        std::istringstream in(v);
        std::string name;
        double T;
        if (!(in >> name >> T)) throw ConfigError("bcs.fixed_temperature = nodeset value");
        for (int n : nodeset(s.mesh, name)) s.tb.fixed.push_back({n, T});
    }
    if (has(c, "bcs.body_force")) {
        const auto b = nums(get(c, "bcs.body_force"), "bcs.body_force");
        if (b.size() != 3) throw ConfigError("bcs.body_force needs 3 numbers");
        s.mb.body_force = Vec3{b[0], b[1], b[2]};
    }
    auto& g = s.cfg;
    g.dt = getd(c, "sim.dt", 0);
    g.duration = getd(c, "sim.duration", g.dt);
    if (g.dt <= 0) throw ConfigError("sim.dt must be > 0");
    const std::string mode = get(c, "sim.coupling", "coupled");
    g.mode = mode == "coupled" ? CouplingMode::Coupled
             : mode == "thermal_only" ? CouplingMode::ThermalOnly
             : mode == "mechanical_only" ? CouplingMode::MechanicalOnly
                                         : throw ConfigError("sim.coupling: coupled | thermal_only | mechanical_only");
    g.expansion_enabled = getb(c, "sim.expansion", m.expansion.has_value());
    g.temperature_dependent = getb(c, "sim.temperature_dependent", false);
    g.damping_gamma = getd(c, "sim.damping_gamma", 0);
    g.hourglass_stiffness = getd(c, "sim.hourglass_stiffness", 0.1);
    g.allow_unstable_dt = getb(c, "sim.allow_unstable_dt", false);
    s.snapshot_interval = getd(c, "output.snapshot_interval", 0);
    s.ablation_threshold = getd(c, "output.ablation_threshold", 60.0);
    for (double v : nums(get(c, "output.probe_nodes", ""), "output.probe_nodes")) s.probes.push_back((int)v - 1);
    return s;
}

// legacy-style unstructured-grid text snapshot, 9 significant digits
void write_snapshot(const fs::path& path, const Mesh& m, double time, long step, const std::vector<double>& T,
                    const std::vector<double>& u) {
    std::ofstream f(path);
    if (!f) throw IoError("cannot write " + path.string());
    char b[160];
    f << "# vtk DataFile Version 3.0\ntve_gpu snapshot step " << step << " time ";
    std::snprintf(b, sizeof b, "%.9g", time);
    f << b << "\nASCII\nDATASET UNSTRUCTURED_GRID\nPOINTS " << m.node_count() << " double\n";
    for (const auto& x : m.nodes) {
        std::snprintf(b, sizeof b, "%.9g %.9g %.9g\n", x[0], x[1], x[2]);
        f << b;
    }
    const int nn = m.kind == ElementKind::H8 ? 8 : 4;
    f << "CELLS " << m.element_count() << " " << (size_t)m.element_count() * (nn + 1) << "\n";
    for (const auto& e : m.elements) {
        f << nn;
        for (int a = 0; a < nn; ++a) f << " " << e[a];
        f << "\n";
    }
    f << "CELL_TYPES " << m.element_count() << "\n";
    for (int e = 0; e < m.element_count(); ++e) f << (nn == 8 ? 12 : 10) << "\n";
    f << "POINT_DATA " << m.node_count() << "\nSCALARS temperature double 1\nLOOKUP_TABLE default\n";
    for (double t : T) {
        std::snprintf(b, sizeof b, "%.9g\n", t);
        f << b;
    }
    f << "VECTORS displacement double\n";
    for (int i = 0; i < m.node_count(); ++i) {
        std::snprintf(b, sizeof b, "%.9g %.9g %.9g\n", u[3 * i], u[3 * i + 1], u[3 * i + 2]);
        f << b;
    }
}

tvegpu_problem geometry_problem(const Mesh& m, const MaterialModel& mat, std::vector<double>& xs,
                                std::vector<int32_t>& el, std::vector<double>& cT, std::vector<double>& cV,
                                std::vector<double>& kT, std::vector<double>& kK) {
    tvegpu_problem p{};
    const int nn = m.kind == ElementKind::H8 ? 8 : 4;
    for (const auto& x : m.nodes) xs.insert(xs.end(), x.begin(), x.end());
    for (const auto& e : m.elements) el.insert(el.end(), e.begin(), e.begin() + nn);
    for (auto [T, v] : mat.thermal.specific_heat.entries) cT.push_back(T), cV.push_back(v);
    for (const auto& e : mat.thermal.conductivity.entries) {
        kT.push_back(e.temperature);
        kK.insert(kK.end(), e.tensor.begin(), e.tensor.end());
    }
    p.kind = nn == 8 ? TVEGPU_H8 : TVEGPU_T4;
    p.num_nodes = m.node_count();
    p.num_elements = m.element_count();
    p.nodes = xs.data();
    p.elements = el.data();
    p.density = mat.thermal.density;
    p.mu = mat.hyperelastic.mu;
    p.kappa = mat.hyperelastic.kappa;
    p.eta_a = mat.hyperelastic.eta_a;
    p.c_table_len = (int32_t)cT.size();
    p.c_table_T = cT.data();
    p.c_table_value = cV.data();
    p.k_table_len = (int32_t)kT.size();
    p.k_table_T = kT.data();
    p.k_table_tensor = kK.data();
    static thread_local std::vector<double> fib;  // per-element fibres (lives as long as p is used)
    fib.clear();
    for (const auto& f : m.fiber_dirs) fib.insert(fib.end(), f.begin(), f.end());
    p.fiber_dirs = fib.empty() ? nullptr : fib.data();
    if (mat.fiber) {
        p.has_fiber = 1;
        for (int k = 0; k < 3; ++k) p.fiber[k] = (*mat.fiber)[k];
    }
    p.dt = 1.0;  // critical_timestep needs a valid problem; the configured dt is checked by the caller
    p.allow_unstable_dt = 1;
    return p;
}

double mesh_volume(const Mesh& m) {
    const int nn = m.kind == ElementKind::H8 ? 8 : 4;
    static const int t6[6][4] = {{0, 1, 2, 6}, {0, 2, 3, 6}, {0, 3, 7, 6}, {0, 7, 4, 6}, {0, 4, 5, 6}, {0, 5, 1, 6}};
    double V = 0;
    for (const auto& e : m.elements)
        for (int k = 0; k < (nn == 4 ? 1 : 6); ++k) {
            const int* id = nn == 4 ? nullptr : t6[k];
            auto X = [&](int q) { return m.nodes[e[id ? id[q] : q]]; };
            double a[3], b[3], c[3];
            for (int i = 0; i < 3; ++i) a[i] = X(1)[i] - X(0)[i], b[i] = X(2)[i] - X(0)[i], c[i] = X(3)[i] - X(0)[i];
            V += std::fabs(a[0] * (b[1] * c[2] - b[2] * c[1]) - a[1] * (b[0] * c[2] - b[2] * c[0]) + a[2] * (b[0] * c[1] - b[1] * c[0])) / 6;
        }
    return V;
}

int cmd_check(const Setup& s, bool json) {
    std::vector<double> xs, cT, cV, kT, kK;
    std::vector<int32_t> el;
    const tvegpu_problem p = geometry_problem(s.mesh, s.mat, xs, el, cT, cV, kT, kK);
    double th = 0, me = 0;
    if (tvegpu_critical_timestep(&p, &th, &me) != TVEGPU_OK) throw ValidationError(tvegpu_create_error());
    const double V = mesh_volume(s.mesh);
    const char* kind = s.mesh.kind == ElementKind::H8 ? "H8" : "T4";
    // the engine refuses dt above the critical step of the physics it runs
    const double crit = s.cfg.mode == CouplingMode::ThermalOnly ? th
                        : s.cfg.mode == CouplingMode::MechanicalOnly ? me : std::min(th, me);
    if (s.cfg.dt > crit && !s.cfg.allow_unstable_dt) {
        std::fprintf(stderr, "validation error: dt %.6g s exceeds the critical step (thermal %.6g s, mechanical %.6g s)\n",
                     s.cfg.dt, th, me);
        return 1;
    }
    if (json)
        std::printf("{\"kind\": \"%s\", \"elements\": %d, \"nodes\": %d, \"dofs\": %d, \"volume_m3\": %.9g, "
                    "\"dt_thermal\": %.9g, \"dt_mechanical\": %.9g, \"dt\": %.9g}\n",
                    kind, s.mesh.element_count(), s.mesh.node_count(), 4 * s.mesh.node_count(), V, th, me, s.cfg.dt);
    else
        std::printf("%s mesh: %d elements, %d nodes, %d degrees of freedom (x, y, z, T per node)\n"
                    "volume %.9g m^3; critical dt thermal %.6g s, mechanical %.6g s; configured dt %.6g s\n",
                    kind, s.mesh.element_count(), s.mesh.node_count(), 4 * s.mesh.node_count(), V, th, me, s.cfg.dt);
    return 0;
}

int cmd_run(const Setup& s, const fs::path& out, bool json) {
    fs::create_directories(out);
    Engine eng(s.mesh, s.mat, s.mb, s.tb, s.src, s.cfg);
    const long total = std::max(1L, (long)std::llround(s.cfg.duration / s.cfg.dt));
    const long every = s.snapshot_interval > 0 ? std::max(1L, (long)std::llround(s.snapshot_interval / s.cfg.dt)) : total;
    std::ofstream probes(out / "probes.csv"), abl(out / "ablation.csv");
    probes << "time,node_id,T,ux,uy,uz\n";
    abl << "time,threshold,volume_m3,elements_above\n";
    std::vector<double> T, u, per_step;
    char b[200];
    auto emit = [&](long step) {
        eng.make_snapshot(T, u);
        std::snprintf(b, sizeof b, "snapshot_%08ld.vtk", step);
        write_snapshot(out / b, s.mesh, eng.time(), step, T, u);
        for (int n : s.probes) {
            std::snprintf(b, sizeof b, "%.9g,%d,%.9g,%.9g,%.9g,%.9g\n", eng.time(), n + 1, T[n], u[3 * n], u[3 * n + 1],
                          u[3 * n + 2]);
            probes << b;
        }
        if (s.ablation_threshold > 0) {
            const auto [v, n] = eng.ablation_volume(s.ablation_threshold);
            std::snprintf(b, sizeof b, "%.9g,%.9g,%.9g,%ld\n", eng.time(), s.ablation_threshold, v, n);
            abl << b;
        }
    };
    emit(0);
    for (long done = 0; done < total;) {
        const long k = std::min(every, total - done);
        const auto t0 = std::chrono::steady_clock::now();
        eng.steps(k);  // throws InstabilityError (exit 2)
        per_step.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / k);
        done += k;
        emit(done);
    }
    const tvegpu_summary sm = eng.summary();
    std::sort(per_step.begin(), per_step.end());
    const double med = per_step[per_step.size() / 2];
    const double iqr = per_step[(3 * per_step.size()) / 4] - per_step[per_step.size() / 4];
    if (json)
        std::printf("{\"steps\": %ld, \"time\": %.9g, \"max_temperature\": %.9g, \"min_disp\": [%.9g, %.9g, %.9g], "
                    "\"max_disp\": [%.9g, %.9g, %.9g], \"median_step_seconds\": %.6g, \"iqr_step_seconds\": %.6g}\n",
                    (long)sm.steps, sm.time, sm.max_temperature, sm.min_disp[0], sm.min_disp[1], sm.min_disp[2],
                    sm.max_disp[0], sm.max_disp[1], sm.max_disp[2], med, iqr);
    else
        std::printf("%ld steps to t = %.6g s: T_max %.6f degC; u min (%.4g, %.4g, %.4g) max (%.4g, %.4g, %.4g) m; "
                    "median %.4g ms/step\n",
                    (long)sm.steps, sm.time, sm.max_temperature, sm.min_disp[0], sm.min_disp[1], sm.min_disp[2],
                    sm.max_disp[0], sm.max_disp[1], sm.max_disp[2], 1e3 * med);
    return 0;
}

// ---- structured meshes for verify / bench
Mesh box_h8(int nx, int ny, int nz, double h) {
    Mesh m;
    m.kind = ElementKind::H8;
    auto id = [&](int i, int j, int k) { return i + (nx + 1) * (j + (ny + 1) * k); };
    for (int k = 0; k <= nz; ++k)
        for (int j = 0; j <= ny; ++j)
            for (int i = 0; i <= nx; ++i) m.nodes.push_back({i * h, j * h, k * h});
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i)
                m.elements.push_back({id(i, j, k), id(i + 1, j, k), id(i + 1, j + 1, k), id(i, j + 1, k),
                                      id(i, j, k + 1), id(i + 1, j, k + 1), id(i + 1, j + 1, k + 1), id(i, j + 1, k + 1)});
    return m;
}
MaterialModel table5(bool td) {
    MaterialModel m;
    m.hyperelastic = {1190.476, 19444.444, 0};
    m.thermal.density = 1060;
    m.thermal.specific_heat.entries = {{37, 3600}};
    m.thermal.conductivity = ConductivityTable::isotropic(37, 0.53);
    if (td) {
        m.thermal.specific_heat.entries.push_back({90, 4300});
        m.thermal.conductivity.entries.push_back({90, {0.75, 0, 0, 0, 0.75, 0, 0, 0, 0.75}});
    }
    return m;
}

struct CaseResult { std::string name, metric; double value, tol; bool pass; };

std::vector<CaseResult> run_verify(const std::string& only) {
    std::vector<CaseResult> r;
    auto want = [&](const char* n) { return only.empty() || only == n; };
    if (want("perfusion_decay")) {
        Mesh m = box_h8(2, 2, 2, 0.005);
        MaterialModel mat = table5(false);
        mat.thermal.perfusion_rate = 26.6;
        mat.thermal.blood_specific_heat = 3617;
        SimulationConfig c;
        c.dt = 0.01;
        c.mode = CouplingMode::ThermalOnly;
        c.allow_unstable_dt = true;
        ThermalBCs tb;
        tb.initial_temperature = 47;
        Engine e(m, mat, MechBCs{}, tb, HeatSourceSet{}, c);
        const double tau = 1060.0 * 3600 / (26.6 * 3617);
        e.steps((long)std::llround(tau / c.dt));
        const auto& T = e.state().temperatures;
        double mean = 0;
        for (double t : T) mean += t / T.size();
        const double want_ = 10 * std::exp(-e.time() / tau);
        const double err = std::fabs((mean - 37) - want_) / want_;
        r.push_back({"perfusion_decay", "rel error in T - Ta at one time constant", err, 5e-3, err < 5e-3});
    }
    if (want("slab_conduction")) {
        const double rho = 1060, cp = 3700, k = 0.518, L = 0.05;
        const int nx = 20;
        Mesh m = box_h8(nx, 1, 1, L / nx);
        MaterialModel mat = table5(false);
        mat.thermal.specific_heat.entries = {{37, cp}};
        mat.thermal.conductivity = ConductivityTable::isotropic(37, k);
        ThermalBCs tb;
        for (int i = 0; i < m.node_count(); ++i) {
            if (m.nodes[i][0] < 1e-12) tb.fixed.push_back({i, 37.0});
            if (m.nodes[i][0] > L - 1e-12) tb.fixed.push_back({i, 90.0});
        }
        SimulationConfig c;
        c.mode = CouplingMode::ThermalOnly;
        c.allow_unstable_dt = true;
        const double tcheck = 0.1 * rho * cp * L * L / k;
        const long n = 200;
        c.dt = tcheck / n;
        Engine e(m, mat, MechBCs{}, tb, HeatSourceSet{}, c);
        e.steps(n);
        const auto& T = e.state().temperatures;
        const double a = k / (rho * cp), t = e.time();
        double num2 = 0, den2 = 0;
        for (int i = 0; i < m.node_count(); ++i) {
            const double x = m.nodes[i][0];
            if (x < 1e-12 || x > L - 1e-12) continue;
            double ex = 37 + 53 * x / L;
            for (int q = 1; q <= 50; ++q) {
                const double bq = 2.0 / (q * M_PI) * (53.0 * (q % 2 ? -1.0 : 1.0));
                ex += bq * std::sin(q * M_PI * x / L) * std::exp(-a * std::pow(q * M_PI / L, 2) * t);
            }
            num2 += (T[i] - ex) * (T[i] - ex);
            den2 += (ex - 37) * (ex - 37);
        }
        const double err = std::sqrt(num2 / den2);
        r.push_back({"slab_conduction", "relative L2 error vs 50-term Fourier series", err, 0.02, err < 0.02});
    }
    if (want("free_expansion")) {
        const int n = 2;
        const double L = 0.01;
        Mesh m = box_h8(n, n, n, L / n);
        MaterialModel mat = table5(false);
        mat.expansion = ExpansionSpec{ExpansionKind::Isotropic, 1e-4, 0, 0, 37.0};
        SimulationConfig c;
        c.dt = 0.4 * 0.9 * (L / n) / std::sqrt((19444.444 + 4 * 1190.476 / 3) / 1060);
        c.expansion_enabled = true;
        c.damping_gamma = 30;
        MechBCs mb;
        mb.fixed_nodes = {0};
        mb.prescribed = {{{n}, 1, 0.0, 0}, {{n}, 2, 0.0, 0}, {{n * (n + 1)}, 2, 0.0, 0}};
        ThermalBCs tb;
        tb.initial_temperature = 87;
        Engine e(m, mat, mb, tb, HeatSourceSet{}, c);
        e.steps(4000);
        const auto& u = e.state().disp;
        const double lam = (L + u[3 * n] - u[0]) / L;
        const double err = std::fabs(lam - 1.005) / 1.005;
        r.push_back({"free_expansion", "rel error of edge stretch vs 1 + alpha dT", err, 1e-3, err < 1e-3});
    }
    if (want("stress_relaxation")) {  // SPEC.md:565-573 (via the displacement-free uniaxial hold)
        Mesh m = box_h8(1, 1, 1, 0.01);
        MaterialModel mat = table5(false);
        mat.prony.terms = {{0.5, 0.58}};
        MechBCs mb;
        for (int i = 0; i < 8; ++i)
            for (int q = 0; q < 3; ++q) mb.prescribed.push_back({{i}, q, q == 0 ? 1e-3 * m.nodes[i][0] : 0.0, 0});
        SimulationConfig c;
        c.dt = 1e-3;
        c.mode = CouplingMode::MechanicalOnly;
        c.allow_unstable_dt = true;
        DeviceOptions o;
        o.diagnostics = true;
        Engine e(m, mat, mb, ThermalBCs{}, HeatSourceSet{}, c, o);
        auto& w = e.mutable_state();
        for (int i = 0; i < 8; ++i) w.disp[3 * i] = w.disp_prev[3 * i] = 1e-3 * m.nodes[i][0];
        e.step();
        std::vector<double> S(9);
        tvegpu_get_diagnostics(e.handle(), nullptr, nullptr, S.data());
        const double s0 = S[0] / (1.0 - c.dt * 0.5 / (c.dt + 0.58));  // undo step 1 of the recurrence (materials.hpp:122-127)
        double worst = 0;
        for (int k = 0; k < 10; ++k) {
            e.steps(290);
            tvegpu_get_diagnostics(e.handle(), nullptr, nullptr, S.data());
            const double want_ = 0.5 + 0.5 * std::exp(-e.time() / 0.58);
            worst = std::max(worst, std::fabs(S[0] / s0 - want_) / want_);
        }
        r.push_back({"stress_relaxation", "max rel error vs phi(t) on [0, 5 tau]", worst, 1e-2, worst < 1e-2});
    }
    return r;
}

int cmd_verify(const std::string& only, bool list) {
    const char* names[] = {"perfusion_decay", "slab_conduction", "free_expansion", "stress_relaxation"};
    if (list) {
        for (const char* n : names) std::printf("%s\n", n);
        return 0;
    }
    const auto res = run_verify(only);
    if (res.empty()) throw ConfigError("unknown verify case '" + only + "'");
    bool ok = true;
    std::printf("case,metric,value,tolerance,pass\n");
    for (const auto& c : res) {
        std::printf("%s,%s,%.6g,%.3g,%s\n", c.name.c_str(), c.metric.c_str(), c.value, c.tol, c.pass ? "yes" : "NO");
        ok &= c.pass;
    }
    return ok ? 0 : 3;
}

int cmd_bench(const std::string& kind, int steps) {  // engine.hpp:145-162 run_bench / bench_scaling_slope
    const bool h8 = kind == "h8";
    const std::vector<int> ladder = h8 ? std::vector<int>{40, 50, 63, 80, 100} : std::vector<int>{20, 25, 32, 40, 50};
    const auto res = run_bench(ladder, h8 ? ElementKind::H8 : ElementKind::T4, steps);
    std::printf("elements,nodes,TherMechTI_ms,TherMechExpanTI_ms,TherMechExpanTD_ms\n");
    for (const auto& r : res)
        std::printf("%d,%d,%.5f,%.5f,%.5f\n", r.elements, r.nodes, 1e3 * r.ther_mech_ti, 1e3 * r.ther_mech_expan_ti,
                    1e3 * r.ther_mech_expan_td);
    std::printf("# scaling slope (log step time vs log elements, TherMechExpanTD): %.3f\n", bench_scaling_slope(res));
    return 0;
}

int usage() {
    std::fprintf(stderr,
                 "usage: tve_gpu run|check --config PATH [--out DIR] [--override section.key=value]... [--json]\n"
                 "       tve_gpu verify [--case NAME] [--list]\n"
                 "       tve_gpu bench [--mesh-kind t4|h8] [--steps N]\n");
    return 1;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    std::string config, out = "out", only, kind = "t4";
    std::vector<std::string> overrides;
    bool json = false, list = false;
    int steps = 100;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto next = [&]() -> std::string {
            if (i + 1 >= argc) throw ConfigError(a + " needs a value");
            return argv[++i];
        };
        try {
            if (a == "--config") config = next();
            else if (a == "--out") out = next();
            else if (a == "--override") overrides.push_back(next());
            else if (a == "--json") json = true;
            else if (a == "--case") only = next();
            else if (a == "--list") list = true;
            else if (a == "--mesh-kind") kind = next();
            else if (a == "--steps") steps = std::atoi(next().c_str());
            else if (a == "--workers") next();  // parallelism lives in the engine
            else return usage();
        } catch (const ConfigError& e) {
            std::fprintf(stderr, "error: %s\n", e.what());
            return 1;
        }
    }
    try {
        if (cmd == "verify") return cmd_verify(only, list);
        if (cmd == "bench") return cmd_bench(kind, steps);
        if (cmd != "run" && cmd != "check") return usage();
        if (config.empty()) throw ConfigError("--config PATH is required");
        std::ifstream f(config);
        if (!f) throw ConfigError("cannot read config " + config);
        const std::string text((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
        Config c = parse_config(text);
        for (const auto& o : overrides) apply_override(c, o);
        const Setup s = build_setup(c, fs::path(config).parent_path());
        return cmd == "check" ? cmd_check(s, json) : cmd_run(s, out, json);
    } catch (const ConfigError& e) {
        std::fprintf(stderr, "config error: %s\n", e.what());
        return 1;
    } catch (const ParseError& e) {
        std::fprintf(stderr, "parse error: %s\n", e.what());
        return 1;
    } catch (const ValidationError& e) {
        std::fprintf(stderr, "validation error: %s\n", e.what());
        return 1;
    } catch (const InstabilityError& e) {
        std::fprintf(stderr, "instability at step %ld, node %d: %s\n", e.step, e.node, e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
