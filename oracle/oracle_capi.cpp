// oracle_capi.cpp — extern "C" shim over the oracle for the Python tests.
// TEST INFRASTRUCTURE ONLY (see tve_oracle.hpp).  Takes the same flat problem
// descriptor as the product ABI (include/tvegpu.h) and rebuilds the
// reference-shaped types (Mesh, MaterialModel, MechBCs, ...) from it, so both
// sides consume byte-identical inputs.
#include <cstring>
#include <memory>
#include <string>

#include "../include/tvegpu.h"
#include "tve_oracle.hpp"

using namespace tve_oracle;

namespace {
thread_local std::string g_err;

Mat3 m9(const double* p) {
    Mat3 m;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m.m[i][j] = p[i * 3 + j];
    return m;
}
void put9(const Mat3& m, double* p) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) p[i * 3 + j] = m.m[i][j];
}
Vec3 v3(const double* p) { return Vec3{{p[0], p[1], p[2]}}; }

struct Bundle {
    Mesh mesh;
    MaterialModel mat;
    MechBCs mbc;
    ThermalBCs tbc;
    HeatSourceSet src;
    SimulationConfig cfg;
    PrecomputedMesh pre;
    std::unique_ptr<Engine> eng;
    int last_status = 0;
    long err_step = -1;
    int err_node = -1;
};

void build(const tvegpu_problem& p, Bundle& b) {
    if (p.kind != TVEGPU_T4 && p.kind != TVEGPU_H8) throw ValidationError("bad element kind");
    const int nn = p.kind == TVEGPU_T4 ? 4 : 8;
    b.mesh.kind = p.kind == TVEGPU_T4 ? ElementKind::T4 : ElementKind::H8;
    b.mesh.nodes.resize(p.num_nodes);
    for (int i = 0; i < p.num_nodes; ++i) b.mesh.nodes[i] = v3(p.nodes + 3 * (size_t)i);
    b.mesh.elements.resize(p.num_elements);
    for (int e = 0; e < p.num_elements; ++e) {
        std::array<int, 8> el{};
        for (int a = 0; a < nn; ++a) el[a] = p.elements[(size_t)e * nn + a];
        b.mesh.elements[e] = el;
    }
    if (p.fiber_dirs) {
        b.mesh.fiber_dirs.resize(p.num_elements);
        for (int e = 0; e < p.num_elements; ++e) b.mesh.fiber_dirs[e] = v3(p.fiber_dirs + 3 * (size_t)e);
    }
    if (p.expansion_axes) {
        b.mesh.expansion_axes.resize(p.num_elements);
        for (int e = 0; e < p.num_elements; ++e)
            b.mesh.expansion_axes[e] = {v3(p.expansion_axes + 6 * (size_t)e), v3(p.expansion_axes + 6 * (size_t)e + 3)};
    }
    b.mat.hyperelastic = {p.mu, p.kappa, p.eta_a};
    std::vector<PronyTerm> terms;
    for (int i = 0; i < p.prony_count; ++i) terms.push_back({p.prony_phi[i], p.prony_tau[i]});
    b.mat.prony = terms.empty() ? PronySeries{} : PronySeries::from_terms(terms);
    b.mat.thermal.density = p.density;
    for (int i = 0; i < p.c_table_len; ++i) b.mat.thermal.specific_heat.entries.push_back({p.c_table_T[i], p.c_table_value[i]});
    for (int i = 0; i < p.k_table_len; ++i)
        b.mat.thermal.conductivity.entries.push_back({p.k_table_T[i], m9(p.k_table_tensor + 9 * (size_t)i)});
    b.mat.thermal.perfusion_rate = p.perfusion_rate;
    b.mat.thermal.blood_specific_heat = p.blood_specific_heat;
    b.mat.thermal.arterial_temperature = p.arterial_temperature;
    b.mat.thermal.metabolic_rate = p.metabolic_rate;
    if (p.has_expansion) {
        ExpansionSpec s;
        s.kind = (ExpansionKind)p.expansion_kind;
        s.alpha_i = p.alpha_i;
        s.alpha_m = p.alpha_m;
        s.alpha_n = p.alpha_n;
        s.reference_temperature = p.reference_temperature;
        b.mat.expansion = s;
    }
    if (p.has_fiber) b.mat.fiber = v3(p.fiber);
    b.mat.axis_m = v3(p.axis_m);
    b.mat.axis_n = v3(p.axis_n);
    for (int i = 0; i < p.num_fixed_nodes; ++i) b.mbc.fixed_nodes.push_back(p.fixed_nodes[i]);
    for (int i = 0; i < p.num_prescribed; ++i) {
        const auto& q = p.prescribed[i];
        PrescribedDisplacement d;
        d.nodes.assign(q.nodes, q.nodes + q.num_nodes);
        d.component = q.component;
        d.target = q.target;
        d.ramp_time = q.ramp_time;
        b.mbc.prescribed.push_back(d);
    }
    if (p.external_force) b.mbc.external_force.assign(p.external_force, p.external_force + 3 * (size_t)p.num_nodes);
    b.mbc.body_force = v3(p.body_force);
    for (int i = 0; i < p.num_fixed_temperatures; ++i)
        b.tbc.fixed.push_back({p.fixed_temperature_nodes[i], p.fixed_temperature_values[i]});
    b.tbc.initial_temperature = p.initial_temperature;
    for (int i = 0; i < p.num_sources; ++i) {
        const auto& s = p.sources[i];
        SourceRegion r;
        r.elements.assign(s.elements, s.elements + s.num_elements);
        r.q_r = s.q_r;
        r.t_start = s.t_start;
        r.t_end = s.t_end;
        b.src.regional.push_back(r);
    }
    b.cfg.dt = p.dt;
    b.cfg.duration = p.duration;
    b.cfg.mode = (CouplingMode)p.mode;
    b.cfg.expansion_enabled = p.expansion_enabled != 0;
    b.cfg.temperature_dependent = p.temperature_dependent != 0;
    b.cfg.damping_gamma = p.damping_gamma;
    b.cfg.hourglass_stiffness = p.hourglass_stiffness;
    b.cfg.allow_unstable_dt = p.allow_unstable_dt != 0;
    b.cfg.workers = p.workers;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const InstabilityError& e) {
        g_err = e.what();
        return 3;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return 2;
    } catch (const ParseError& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 7;
    }
}
}  // namespace

extern "C" {

const char* oracle_error() { return g_err.c_str(); }

void* oracle_create(const tvegpu_problem* p) {
    auto b = std::make_unique<Bundle>();
    int rc = guarded([&] {
        build(*p, *b);
        b->pre = precompute(b->mesh, p->density, p->ref_specific_heat);
        b->eng = std::make_unique<Engine>(b->mesh, b->pre, b->mat, b->mbc, b->tbc, b->src, b->cfg);
    });
    if (rc) return nullptr;
    return b.release();
}
// The same with MechBCs::motion_override (mechanics.hpp:43-46) bound to a C callback:
// fn(user, node, t, disp) returns nonzero and fills disp[3] to pin the node at time t.
typedef int (*oracle_motion_fn)(void* user, int node, double t, double* disp);
void* oracle_create_motion(const tvegpu_problem* p, oracle_motion_fn fn, void* user) {
    auto b = std::make_unique<Bundle>();
    int rc = guarded([&] {
        build(*p, *b);
        if (fn)
            b->mbc.motion_override = [fn, user](int n, double t) -> std::optional<Vec3> {
                double d[3];
                if (!fn(user, n, t, d)) return std::nullopt;
                return Vec3{d[0], d[1], d[2]};
            };
        b->pre = precompute(b->mesh, p->density, p->ref_specific_heat);
        b->eng = std::make_unique<Engine>(b->mesh, b->pre, b->mat, b->mbc, b->tbc, b->src, b->cfg);
    });
    if (rc) return nullptr;
    return b.release();
}
void oracle_destroy(void* h) { delete static_cast<Bundle*>(h); }

int oracle_step(void* h, long n, long* err_step, int* err_node) {
    auto* b = static_cast<Bundle*>(h);
    try {
        for (long k = 0; k < n; ++k) b->eng->step();
    } catch (const InstabilityError& e) {
        g_err = e.what();
        if (err_step) *err_step = e.step;
        if (err_node) *err_node = e.node;
        return 3;
    } catch (const ElementError& e) {
        g_err = e.what();
        if (err_step) *err_step = e.step;
        if (err_node) *err_node = e.element;
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 7;
    }
    return 0;
}

void oracle_get_state(void* h, double* T, double* u, double* uprev, double* viscous) {
    auto* b = static_cast<Bundle*>(h);
    const auto& s = b->eng->state();
    if (T) std::memcpy(T, s.thermal.temperatures.data(), s.thermal.temperatures.size() * 8);
    if (u) std::memcpy(u, s.mech.disp.data(), s.mech.disp.size() * 8);
    if (uprev) std::memcpy(uprev, s.mech.disp_prev.data(), s.mech.disp_prev.size() * 8);
    if (viscous)
        for (size_t k = 0; k < s.mech.viscous.size(); ++k) put9(s.mech.viscous[k], viscous + 9 * k);
}
void oracle_set_state(void* h, const double* T, const double* u, const double* uprev, const double* viscous,
                      double time, long step) {
    auto* b = static_cast<Bundle*>(h);
    auto& s = b->eng->state();
    if (T) std::memcpy(s.thermal.temperatures.data(), T, s.thermal.temperatures.size() * 8);
    if (u) std::memcpy(s.mech.disp.data(), u, s.mech.disp.size() * 8);
    if (uprev) std::memcpy(s.mech.disp_prev.data(), uprev, s.mech.disp_prev.size() * 8);
    if (viscous)
        for (size_t k = 0; k < s.mech.viscous.size(); ++k) s.mech.viscous[k] = m9(viscous + 9 * k);
    s.thermal.time = time;
    s.step = step;
}
double oracle_time(void* h) { return static_cast<Bundle*>(h)->eng->time(); }
long oracle_step_count(void* h) { return static_cast<Bundle*>(h)->eng->state().step; }
void oracle_set_nodal_sources(void* h, const double* power) {
    static_cast<Bundle*>(h)->eng->set_nodal_source_override(power);
}
void oracle_get_diagnostics(void* h, double* f_int, double* F, double* S, double* th_loads, double* forces,
                            double* nodal_sources) {
    auto* b = static_cast<Bundle*>(h);
    const auto& e = *b->eng;
    if (f_int) std::memcpy(f_int, e.last_internal_forces().data(), e.last_internal_forces().size() * 8);
    if (F)
        for (size_t k = 0; k < e.deformation_gradients().size(); ++k) put9(e.deformation_gradients()[k], F + 9 * k);
    if (S)
        for (size_t k = 0; k < e.element_stresses().size(); ++k) put9(e.element_stresses()[k], S + 9 * k);
    if (th_loads) std::memcpy(th_loads, e.element_thermal_loads().data(), e.element_thermal_loads().size() * 8);
    if (forces) std::memcpy(forces, e.element_forces().data(), e.element_forces().size() * 8);
    if (nodal_sources) std::memcpy(nodal_sources, e.nodal_sources().data(), e.nodal_sources().size() * 8);
}
double oracle_total_energy(void* h) { return static_cast<Bundle*>(h)->eng->total_energy(); }

// precompute() arrays in the reference layout (mesh.hpp:45-71).
int oracle_precompute(const tvegpu_problem* p, double* grads, double* vol, double* detj, double* mass,
                      double* cref, double* vnode, double* hg, int* adj_off, int* adj_elem, int* adj_local) {
    Bundle b;
    return guarded([&] {
        build(*p, b);
        PrecomputedMesh pre = precompute(b.mesh, p->density, p->ref_specific_heat);
        auto cp = [](double* dst, const std::vector<double>& v) {
            if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * 8);
        };
        cp(grads, pre.shape_gradients);
        cp(vol, pre.ref_volume);
        cp(detj, pre.det_jacobian);
        cp(mass, pre.lumped_mass);
        cp(cref, pre.lumped_heat_capacity_ref);
        cp(vnode, pre.node_volume);
        cp(hg, pre.hourglass_basis);
        if (adj_off) std::memcpy(adj_off, pre.adjacency_offsets.data(), pre.adjacency_offsets.size() * 4);
        for (size_t k = 0; k < pre.adjacency.size(); ++k) {
            if (adj_elem) adj_elem[k] = pre.adjacency[k].first;
            if (adj_local) adj_local[k] = pre.adjacency[k].second;
        }
    });
}

int oracle_critical_timestep(const tvegpu_problem* p, double* out2) {
    Bundle b;
    return guarded([&] {
        build(*p, b);
        auto ct = critical_timestep(b.mesh, b.mat);
        out2[0] = ct.thermal;
        out2[1] = ct.mechanical;
    });
}

// ---- unit-level functions (row-major 3x3, column a of 3xNN stored at [a*3+i]) ----
int oracle_strain_energy(const double* C, double mu, double kappa, double eta, const double* fiber, double* out) {
    return guarded([&] {
        Vec3 f = fiber ? v3(fiber) : Vec3{};
        *out = strain_energy(m9(C), {mu, kappa, eta}, fiber ? &f : nullptr);
    });
}
int oracle_pk2_stress(const double* C, double mu, double kappa, double eta, const double* fiber, double* out) {
    return guarded([&] {
        Vec3 f = fiber ? v3(fiber) : Vec3{};
        put9(pk2_stress(m9(C), {mu, kappa, eta}, fiber ? &f : nullptr), out);
    });
}
int oracle_total_pk2_stress(const double* F, const double* Fth, double mu, double kappa, double eta,
                            const double* fiber, double* out) {
    return guarded([&] {
        Vec3 f = fiber ? v3(fiber) : Vec3{};
        put9(total_pk2_stress(m9(F), m9(Fth), {mu, kappa, eta}, fiber ? &f : nullptr), out);
    });
}
int oracle_thermal_deformation_gradient(double T, int kind, double ai, double am, double an, double Tref,
                                        const double* m, const double* n, double* out) {
    return guarded([&] {
        ExpansionSpec s{(ExpansionKind)kind, ai, am, an, Tref};
        put9(thermal_deformation_gradient(T, s, v3(m), v3(n)), out);
    });
}
int oracle_prony_update(const double* S, double* hist, int P, const double* phi, const double* tau, double dt,
                        double* out) {
    return guarded([&] {
        std::vector<PronyTerm> t;
        for (int i = 0; i < P; ++i) t.push_back({phi[i], tau[i]});
        PronySeries pr = PronySeries::from_terms(t);
        std::vector<Mat3> h(P);
        for (int i = 0; i < P; ++i) h[i] = m9(hist + 9 * i);
        put9(prony_update(m9(S), h, dt, pr), out);
        for (int i = 0; i < P; ++i) put9(h[i], hist + 9 * i);
    });
}
int oracle_relaxation_function(double t, int P, const double* phi, const double* tau, double* out) {
    return guarded([&] {
        std::vector<PronyTerm> v;
        for (int i = 0; i < P; ++i) v.push_back({phi[i], tau[i]});
        *out = relaxation_function(t, PronySeries::from_terms(v));
    });
}
int oracle_interp_property(int n, const double* Ts, const double* vs, double T, double* out) {
    return guarded([&] {
        ScalarTable tab;
        for (int i = 0; i < n; ++i) tab.entries.push_back({Ts[i], vs[i]});
        *out = interp_property(tab, T);
    });
}
int oracle_deformation_gradient(int nn, const double* U, const double* G, double* out) {
    return guarded([&] { put9(nn == 4 ? deformation_gradient<4>(U, G) : deformation_gradient<8>(U, G), out); });
}
int oracle_element_thermal_load(int nn, const double* F, const double* G, const double* D, const double* Te,
                                double V, double* out) {
    return guarded([&] {
        if (nn == 4) {
            auto f = element_thermal_load<4>(m9(F), G, m9(D), Te, V);
            std::memcpy(out, f.data(), 32);
        } else {
            auto f = element_thermal_load<8>(m9(F), G, m9(D), Te, V);
            std::memcpy(out, f.data(), 64);
        }
    });
}
int oracle_element_internal_force(int nn, const double* F, const double* G, double mu, double kappa, double eta,
                                  const double* fiber, const double* Fth, double* hist, int P, const double* phi,
                                  const double* tau, double dt, double V, double* out) {
    return guarded([&] {
        std::vector<PronyTerm> t;
        for (int i = 0; i < P; ++i) t.push_back({phi[i], tau[i]});
        PronySeries pr = P ? PronySeries::from_terms(t) : PronySeries{};
        std::vector<Mat3> h(P);
        for (int i = 0; i < P; ++i) h[i] = m9(hist + 9 * i);
        Vec3 f = fiber ? v3(fiber) : Vec3{};
        if (nn == 4)
            element_internal_force<4>(m9(F), G, {mu, kappa, eta}, fiber ? &f : nullptr, m9(Fth), h, dt, pr, V, out);
        else
            element_internal_force<8>(m9(F), G, {mu, kappa, eta}, fiber ? &f : nullptr, m9(Fth), h, dt, pr, V, out);
        for (int i = 0; i < P; ++i) put9(h[i], hist + 9 * i);
    });
}
void oracle_hourglass_force(const double* U, const double* gamma, double k, double* out) {
    hourglass_force(U, gamma, k, out);
}
void oracle_hourglass_basis(const double* X, const double* G, double* out) {
    hourglass_basis_for_element(X, G, out);
}
int oracle_step_displacement(int N, double* u, double* uprev, const double* f, const double* M, const double* R,
                             double gamma, double dt) {
    return guarded([&] {
        MechState s;
        s.disp.assign(u, u + 3 * (size_t)N);
        s.disp_prev.assign(uprev, uprev + 3 * (size_t)N);
        MechBCs bc;
        if (R) bc.external_force.assign(R, R + 3 * (size_t)N);
        step_displacement(s, std::span<const double>(f, 3 * (size_t)N), bc, std::span<const double>(M, N), gamma,
                          dt, dt);
        std::memcpy(u, s.disp.data(), s.disp.size() * 8);
        std::memcpy(uprev, s.disp_prev.data(), s.disp_prev.size() * 8);
    });
}
int oracle_step_temperature(int N, double* T, const double* loads, const double* Qr, const double* Vn, double rho,
                            int ctab_n, const double* cT, const double* cv, double wb, double cb, double Ta,
                            double Qm, double dt, int td) {
    return guarded([&] {
        ThermalState s;
        s.temperatures.assign(T, T + N);
        ThermalProps p;
        p.density = rho;
        for (int i = 0; i < ctab_n; ++i) p.specific_heat.entries.push_back({cT[i], cv[i]});
        p.perfusion_rate = wb;
        p.blood_specific_heat = cb;
        p.arterial_temperature = Ta;
        p.metabolic_rate = Qm;
        ThermalBCs bc;
        step_temperature(s, std::span<const double>(loads, N), std::span<const double>(Qr, N), p,
                         std::span<const double>(Vn, N), bc, dt, td != 0, 37.0);
        std::memcpy(T, s.temperatures.data(), (size_t)N * 8);
    });
}


// ablation_volume over raw arrays: kind 0 = T4, 1 = H8.
int oracle_ablation_volume(int kind, int num_nodes, int num_elements, const double* nodes, const int* elements,
                           const double* T, const double* disp, double threshold, double* volume, long* count) {
    return guarded([&] {
        Mesh m;
        m.kind = kind == 1 ? ElementKind::H8 : ElementKind::T4;
        const int nn = kind == 1 ? 8 : 4;
        m.nodes.resize(num_nodes);
        for (int i = 0; i < num_nodes; ++i)
            for (int c = 0; c < 3; ++c) m.nodes[i][c] = nodes[3 * (size_t)i + c];
        m.elements.resize(num_elements);
        for (int e = 0; e < num_elements; ++e)
            for (int a = 0; a < nn; ++a) m.elements[e][a] = elements[(size_t)nn * e + a];
        std::vector<double> u;
        if (disp) u.assign(disp, disp + 3 * (size_t)num_nodes);
        const AblationReport r = ablation_volume(m, std::span<const double>(T, num_nodes), threshold, disp ? &u : nullptr);
        *volume = r.volume;
        *count = r.elements_above;
    });
}
}  // extern "C"
