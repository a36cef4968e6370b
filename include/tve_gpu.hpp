// tve_gpu.hpp — header-only C++ facade over the C ABI (tvegpu.h) with the class
// shape of the reference's tve::Engine (/root/reference/proj/include/tve/engine.hpp:83-143).
//
// The reference types (mesh.hpp, materials.hpp, mechanics.hpp, bioheat.hpp,
// engine.hpp) are mirrored field for field with std::array<double,3> in place of
// Eigen::Vector3d (the reference vendors Eigen, which is absent).
// Errors are the reference exception taxonomy (errors.hpp:8-33).  Porting a
// caller means: include this header, use tve::gpu:: instead of tve::, and link
// libtvegpu.so.  See INTEGRATION.md.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <istream>
#include <iterator>
#include <algorithm>
#include <chrono>
#include <fstream>
#include <functional>
#include <limits>
#include <map>
#include <ostream>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "tvegpu.h"

namespace tve::gpu {

using Vec3 = std::array<double, 3>;

// ---------------------------------------------------------------- errors.hpp:8-33
struct ParseError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ValidationError : std::runtime_error { using std::runtime_error::runtime_error; };
struct InstabilityError : std::runtime_error {
    InstabilityError(const std::string& m, long s, int n) : std::runtime_error(m), step(s), node(n) {}
    long step = -1;
    int node = -1;
};
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

// ---------------------------------------------------------------- mesh.hpp:15-37
enum class ElementKind { T4, H8 };
inline int nodes_per_element(ElementKind k) { return k == ElementKind::T4 ? 4 : 8; }
struct Mesh {
    std::vector<Vec3> nodes;
    ElementKind kind = ElementKind::T4;
    std::vector<std::array<int, 8>> elements;      // first nodes_per_element() entries used
    std::vector<Vec3> fiber_dirs;                   // empty or one per element
    std::vector<std::array<Vec3, 2>> expansion_axes;
    std::map<std::string, std::vector<int>> node_sets, element_sets;  // 0-based
    int node_count() const { return (int)nodes.size(); }
    int element_count() const { return (int)elements.size(); }
};

// ---------------------------------------------------------------- materials.hpp:13-97
struct HyperelasticParams { double mu = 0, kappa = 0, eta_a = 0; };
struct PronyTerm { double phi = 0, tau = 0; };
struct PronySeries { std::vector<PronyTerm> terms; };
struct ScalarTable { std::vector<std::pair<double, double>> entries; };
struct ConductivityTable {
    struct Entry { double temperature = 0; std::array<double, 9> tensor{}; };  // row-major
    std::vector<Entry> entries;
    static ConductivityTable isotropic(double T, double k) {
        ConductivityTable t;
        t.entries.push_back({T, {k, 0, 0, 0, k, 0, 0, 0, k}});
        return t;
    }
};
struct ThermalProps {
    double density = 0;
    ScalarTable specific_heat;
    ConductivityTable conductivity;
    double perfusion_rate = 0, blood_specific_heat = 0, arterial_temperature = 37.0, metabolic_rate = 0;
};
enum class ExpansionKind { Isotropic, TransverselyIsotropic, Orthotropic };
struct ExpansionSpec {
    ExpansionKind kind = ExpansionKind::Isotropic;
    double alpha_i = 0, alpha_m = 0, alpha_n = 0, reference_temperature = 37.0;
};
struct MaterialModel {
    HyperelasticParams hyperelastic;
    PronySeries prony;
    ThermalProps thermal;
    std::optional<ExpansionSpec> expansion;
    std::optional<Vec3> fiber;
    Vec3 axis_m{1, 0, 0};
    Vec3 axis_n{0, 1, 0};
};

// ---------------------------------------------------------------- bioheat.hpp / mechanics.hpp
struct SourceRegion {
    std::vector<int> elements;
    double q_r = 0, t_start = 0, t_end = std::numeric_limits<double>::infinity();
};
struct HeatSourceSet { std::vector<SourceRegion> regional; };
struct ThermalBCs { std::vector<std::pair<int, double>> fixed; double initial_temperature = 37.0; };
struct PrescribedDisplacement {
    std::vector<int> nodes;
    int component = 0;
    double target = 0, ramp_time = 0;
};
struct MechBCs {
    std::vector<int> fixed_nodes;
    std::vector<PrescribedDisplacement> prescribed;
    std::vector<double> external_force;  // 3 per node or empty
    Vec3 body_force{0, 0, 0};
    // mechanics.hpp:43-46: optional per-node trajectory; a returned value pins the node at
    // time t (applied last).  A host callback: the GPU engine evaluates it every step for
    // motion_nodes (empty = every node) and uploads the pins (tvegpu_set_motion_override).
    std::function<std::optional<Vec3>(int node, double t)> motion_override;
    std::vector<int> motion_nodes;  // candidate nodes of motion_override (a GPU-side restriction; empty = all)
};

// ---------------------------------------------------------------- engine.hpp:16-45
enum class CouplingMode { Coupled, ThermalOnly, MechanicalOnly };
struct OutputSpec {                  // engine.hpp:18-24
    double snapshot_interval = 0;    // [s]; <= 0 disables periodic snapshots
    std::vector<int> probe_nodes;    // 0-based (carried for callers; snapshots hold every node)
    bool write_det_f = false;        // needs DeviceOptions::diagnostics
    bool write_stress = false;       // needs DeviceOptions::diagnostics
    double ablation_threshold = 60.0;  // [degC]; <= 0 disables the report
};
struct SimulationConfig {
    double dt = 0, duration = 0;
    CouplingMode mode = CouplingMode::Coupled;
    bool expansion_enabled = false, temperature_dependent = false;
    double damping_gamma = 0, hourglass_stiffness = 0.1;
    bool allow_unstable_dt = false;
    int workers = 0;
    OutputSpec output;
};
// engine.hpp:47-55: field snapshot handed to sinks (copies, safe to retain)
struct Snapshot {
    double time = 0;
    long step = 0;
    std::vector<double> temperatures, displacements, det_f, max_principal_stress;
};
// engine.hpp:57-66
struct RunSummary {
    long steps = 0;
    double final_time = 0, max_temperature = 0;
    Vec3 min_displacement{0, 0, 0}, max_displacement{0, 0, 0};
    double ablation_volume = 0;  // [m^3] at the final step, deformed configuration (0 if disabled)
    double median_step_seconds = 0, iqr_step_seconds = 0;
};
using SnapshotSink = std::function<void(const Snapshot&)>;
struct SimulationState {
    std::vector<double> temperatures;  // ThermalState::temperatures
    double time = 0;                   // ThermalState::time
    std::vector<double> disp, disp_prev;
    std::vector<std::array<double, 9>> viscous;  // num_elements * prony_terms (row-major)
    long step = 0;
};

struct DeviceOptions {
    int device = -1;
    int steps_per_graph = 64;
    bool diagnostics = false;
    // one RCB partition per process and GPU (nranks > 1): NCCL id from tvegpu_nccl_unique_id
    // on one rank, shared by the caller; then peer_export / all-gather / peer_attach
    int nranks = 1, rank = 0;
    std::vector<unsigned char> nccl_unique_id;  // 128 bytes when nranks > 1
    int halo_transport = TVEGPU_HALO_PEER;
    bool slot_fp32 = false;  // mixed precision: fp32 contributions between element and node kernels
};

// tve::Engine (engine.hpp:83-143) on a B200.
class Engine {
public:
    Engine(const Mesh& mesh, const MaterialModel& material, const MechBCs& mech_bcs, const ThermalBCs& thermal_bcs,
           const HeatSourceSet& sources, const SimulationConfig& config, const DeviceOptions& opt = {})
        : N_(mesh.node_count()), E_(mesh.element_count()), P_((int)material.prony.terms.size()),
          dt_(config.dt), dur_(config.duration), out_(config.output) {
        build(mesh, material, mech_bcs, thermal_bcs, sources, config);
        tvegpu_options o;
        tvegpu_default_options(&o);
        o.device = opt.device;
        o.steps_per_graph = opt.steps_per_graph;
        o.diagnostics = opt.diagnostics ? 1 : 0;
        o.nranks = opt.nranks;
        o.rank = opt.rank;
        o.nccl_unique_id = opt.nccl_unique_id.empty() ? nullptr : opt.nccl_unique_id.data();
        o.halo_transport = opt.halo_transport;
        o.slot_fp32 = opt.slot_fp32 ? 1 : 0;
        const tvegpu_status st = tvegpu_create(&p_, &o, &h_);
        if (st != TVEGPU_OK) rethrow(st, tvegpu_create_error(), -1, -1);
        if (mech_bcs.motion_override) {
            motion_ = mech_bcs.motion_override;
            motion_nodes_ = mech_bcs.motion_nodes;
            check(tvegpu_set_motion_override(h_, &Engine::motion_trampoline, this, (int32_t)motion_nodes_.size(),
                                             motion_nodes_.empty() ? nullptr : motion_nodes_.data()));
        }
    }
    ~Engine() { tvegpu_destroy(h_); }

    // C callback -> MechBCs::motion_override
    static int32_t motion_trampoline(void* self, int32_t node, double t, double* disp) {
        const std::optional<Vec3> v = static_cast<Engine*>(self)->motion_(node, t);
        if (!v) return 0;
        disp[0] = (*v)[0], disp[1] = (*v)[1], disp[2] = (*v)[2];
        return 1;
    }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    // Peer-memory halo across processes (tvegpu.h tvegpu_peer_export / tvegpu_peer_attach):
    // every rank exports, the caller all-gathers the descriptors, every rank attaches.
    std::vector<unsigned char> peer_export() {
        size_t n = 0;
        check(tvegpu_peer_export(h_, nullptr, 0, &n));
        std::vector<unsigned char> b(n);
        check(tvegpu_peer_export(h_, b.data(), b.size(), &n));
        return b;
    }
    void peer_attach(const std::vector<std::vector<unsigned char>>& by_rank) {
        std::vector<const void*> p;
        std::vector<size_t> n;
        for (const auto& b : by_rank) {
            p.push_back(b.data());
            n.push_back(b.size());
        }
        check(tvegpu_peer_attach(h_, p.data(), n.data(), (int32_t)p.size()));
    }

    // engine.hpp:89-90
    void step() { steps(1); }
    void steps(int64_t n) {
        push_if_dirty();
        check(tvegpu_step(h_, n));
        mirror_valid_ = false;
    }
    // engine.hpp:95-97: state() returns a host mirror synced on access; writes made
    // through mutable_state() are pushed to the device before the next step.
    const SimulationState& state() {
        pull_if_stale();
        return mirror_;
    }
    SimulationState& mutable_state() {
        pull_if_stale();
        dirty_ = true;
        return mirror_;
    }
    double time() const { return tvegpu_time(h_); }
    long step_count() const { return (long)tvegpu_step_count(h_); }

    // engine.hpp:99 (fields only)
    void make_snapshot(std::vector<double>& T, std::vector<double>& u) {
        T.resize(N_);
        u.resize(3 * (size_t)N_);
        check(tvegpu_make_snapshot(h_, T.data(), u.data()));
    }
    // engine.hpp:101-105 (needs DeviceOptions::diagnostics): assembled internal force of the
    // last mechanics phase (3 per node), S~ and F per element (row-major 3x3, original ids)
    std::vector<double> last_internal_forces() {
        std::vector<double> f(3 * (size_t)N_);
        check(tvegpu_get_diagnostics(h_, f.data(), nullptr, nullptr));
        return f;
    }
    std::vector<std::array<double, 9>> element_stresses() {
        std::vector<std::array<double, 9>> S((size_t)E_);
        check(tvegpu_get_diagnostics(h_, nullptr, nullptr, S.empty() ? nullptr : S[0].data()));
        return S;
    }
    std::vector<std::array<double, 9>> deformation_gradients() {
        std::vector<std::array<double, 9>> F((size_t)E_);
        check(tvegpu_get_diagnostics(h_, nullptr, F.empty() ? nullptr : F[0].data(), nullptr));
        return F;
    }
    // bioheat.hpp:57 nodal source override (power per node [W]); empty restores regions
    void set_nodal_sources(const std::vector<double>& power) {
        check_power(power);
        check(tvegpu_set_nodal_sources(h_, power.empty() ? nullptr : power.data()));
    }
    // Closed-loop iteration: sources + n steps + T/u read-back, copies overlapped with
    // the step (tvegpu_step_io); empty power keeps the current sources.
    void step_io(const std::vector<double>& power, int64_t n, std::vector<double>& T, std::vector<double>& u) {
        check_power(power);
        push_if_dirty();
        T.resize(N_);
        u.resize(3 * (size_t)N_);
        check(tvegpu_step_io(h_, power.empty() ? nullptr : power.data(), n, T.data(), u.data()));
        mirror_valid_ = false;
    }

    // a power vector is one value per node (the C side reads num_nodes doubles)
    void check_power(const std::vector<double>& power) const {
        if (!power.empty() && power.size() != (size_t)N_)
            throw std::invalid_argument("nodal source power needs one value per node (" + std::to_string(N_) +
                                        "), got " + std::to_string(power.size()));
    }

    // engine.hpp:57-66 RunSummary extrema and SPEC.md:435-443 ablation volume, on the device
    tvegpu_summary summary() {
        push_if_dirty();
        tvegpu_summary s;
        check(tvegpu_get_summary(h_, &s));
        return s;
    }
    std::pair<double, long> ablation_volume(double threshold, bool deformed = true) {
        push_if_dirty();
        double v = 0;
        int64_t n = 0;
        check(tvegpu_ablation_volume(h_, threshold, deformed ? 1 : 0, &v, &n));
        return {v, (long)n};
    }

    // engine.hpp:108: kinetic plus hyperelastic strain energy of the current state [J]
    double total_energy() {
        push_if_dirty();
        double k = 0, e = 0;
        check(tvegpu_total_energy(h_, &k, &e));
        return k + e;
    }

    // engine.hpp:110-111
    void save_checkpoint(std::ostream& out) {
        push_if_dirty();
        uint64_t n = 0;
        check(tvegpu_checkpoint_size(h_, &n));
        std::vector<char> buf(n);
        check(tvegpu_save_checkpoint(h_, buf.data(), n));
        out.write(buf.data(), (std::streamsize)n);
        if (!out) throw IoError("save_checkpoint: write failed");
    }
    void load_checkpoint(std::istream& in) {
        std::vector<char> buf((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        check(tvegpu_load_checkpoint(h_, buf.data(), buf.size()));
        dirty_ = false;
        mirror_valid_ = false;
    }

    // engine.hpp:99: Snapshot with the optional element fields of OutputSpec
    Snapshot make_snapshot() {
        Snapshot s;
        s.time = time();
        s.step = step_count();
        make_snapshot(s.temperatures, s.displacements);
        if (out_.write_det_f || out_.write_stress) {
            std::vector<double> d(E_), m(E_);
            check(tvegpu_element_fields(h_, out_.write_det_f ? d.data() : nullptr,
                                        out_.write_stress ? m.data() : nullptr));
            if (out_.write_det_f) s.det_f = std::move(d);
            if (out_.write_stress) s.max_principal_stress = std::move(m);
        }
        return s;
    }

    // engine.hpp:92: run duration/dt steps, calling the sink on the output schedule
    // (every snapshot_interval, and at the end); per-step wall time from the chunks
    // between snapshots.  Throws InstabilityError like step().
    RunSummary run(const SnapshotSink& sink = nullptr) {
        push_if_dirty();
        const long total = std::max(1L, (long)std::llround(dur_ / dt_));
        const long every =
            out_.snapshot_interval > 0 ? std::max(1L, (long)std::llround(out_.snapshot_interval / dt_)) : total;
        std::vector<double> per;
        for (long done = 0; done < total;) {
            const long k = std::min(every, total - done);
            const auto t0 = std::chrono::steady_clock::now();
            steps(k);
            (void)time();
            per.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / k);
            done += k;
            if (sink && (out_.snapshot_interval > 0 || done == total)) sink(make_snapshot());
        }
        RunSummary r;
        const tvegpu_summary sm = summary();
        r.steps = (long)sm.steps;
        r.final_time = sm.time;
        r.max_temperature = sm.max_temperature;
        for (int c = 0; c < 3; ++c) r.min_displacement[c] = sm.min_disp[c], r.max_displacement[c] = sm.max_disp[c];
        if (out_.ablation_threshold > 0) r.ablation_volume = ablation_volume(out_.ablation_threshold).first;
        std::sort(per.begin(), per.end());
        r.median_step_seconds = per[per.size() / 2];
        r.iqr_step_seconds = per[(3 * per.size()) / 4] - per[per.size() / 4];
        return r;
    }

    tvegpu_engine* handle() { return h_; }

private:
    void build(const Mesh& m, const MaterialModel& mat, const MechBCs& mb, const ThermalBCs& tb,
               const HeatSourceSet& src, const SimulationConfig& c) {
        const int nn = nodes_per_element(m.kind);
        for (const auto& x : m.nodes) nodes_.insert(nodes_.end(), x.begin(), x.end());
        for (const auto& e : m.elements) elems_.insert(elems_.end(), e.begin(), e.begin() + nn);
        for (const auto& f : m.fiber_dirs) fibers_.insert(fibers_.end(), f.begin(), f.end());
        for (const auto& ax : m.expansion_axes)
            for (const auto& v : ax) axes_.insert(axes_.end(), v.begin(), v.end());
        for (const auto& t : mat.prony.terms) {
            phi_.push_back(t.phi);
            tau_.push_back(t.tau);
        }
        for (const auto& [T, v] : mat.thermal.specific_heat.entries) {
            cT_.push_back(T);
            cV_.push_back(v);
        }
        for (const auto& e : mat.thermal.conductivity.entries) {
            kT_.push_back(e.temperature);
            kK_.insert(kK_.end(), e.tensor.begin(), e.tensor.end());
        }
        fixed_ = mb.fixed_nodes;
        for (const auto& q : mb.prescribed)
            presc_.push_back({(int32_t)q.nodes.size(), q.nodes.data(), q.component, q.target, q.ramp_time});
        for (const auto& [n, v] : tb.fixed) {
            tfixN_.push_back(n);
            tfixV_.push_back(v);
        }
        for (const auto& r : src.regional)
            srcs_.push_back({(int32_t)r.elements.size(), r.elements.data(), r.q_r, r.t_start, r.t_end});
        ext_ = mb.external_force;
        tvegpu_problem& p = p_;
        p = tvegpu_problem{};
        p.kind = m.kind == ElementKind::T4 ? TVEGPU_T4 : TVEGPU_H8;
        p.num_nodes = m.node_count();
        p.num_elements = m.element_count();
        p.nodes = nodes_.data();
        p.elements = elems_.data();
        p.fiber_dirs = fibers_.empty() ? nullptr : fibers_.data();
        p.expansion_axes = axes_.empty() ? nullptr : axes_.data();
        p.ref_specific_heat = cV_.empty() ? 0.0 : interp(37.0);
        p.mu = mat.hyperelastic.mu;
        p.kappa = mat.hyperelastic.kappa;
        p.eta_a = mat.hyperelastic.eta_a;
        p.prony_count = (int32_t)phi_.size();
        p.prony_phi = phi_.data();
        p.prony_tau = tau_.data();
        p.density = mat.thermal.density;
        p.c_table_len = (int32_t)cT_.size();
        p.c_table_T = cT_.data();
        p.c_table_value = cV_.data();
        p.k_table_len = (int32_t)kT_.size();
        p.k_table_T = kT_.data();
        p.k_table_tensor = kK_.data();
        p.perfusion_rate = mat.thermal.perfusion_rate;
        p.blood_specific_heat = mat.thermal.blood_specific_heat;
        p.arterial_temperature = mat.thermal.arterial_temperature;
        p.metabolic_rate = mat.thermal.metabolic_rate;
        if (mat.expansion) {
            p.has_expansion = 1;
            p.expansion_kind = (int32_t)mat.expansion->kind;
            p.alpha_i = mat.expansion->alpha_i;
            p.alpha_m = mat.expansion->alpha_m;
            p.alpha_n = mat.expansion->alpha_n;
            p.reference_temperature = mat.expansion->reference_temperature;
        }
        if (mat.fiber) {
            p.has_fiber = 1;
            for (int k = 0; k < 3; ++k) p.fiber[k] = (*mat.fiber)[k];
        }
        for (int k = 0; k < 3; ++k) {
            p.axis_m[k] = mat.axis_m[k];
            p.axis_n[k] = mat.axis_n[k];
            p.body_force[k] = mb.body_force[k];
        }
        p.num_fixed_nodes = (int32_t)fixed_.size();
        p.fixed_nodes = fixed_.data();
        p.num_prescribed = (int32_t)presc_.size();
        p.prescribed = presc_.data();
        p.external_force = ext_.empty() ? nullptr : ext_.data();
        p.num_fixed_temperatures = (int32_t)tfixN_.size();
        p.fixed_temperature_nodes = tfixN_.data();
        p.fixed_temperature_values = tfixV_.data();
        p.initial_temperature = tb.initial_temperature;
        p.num_sources = (int32_t)srcs_.size();
        p.sources = srcs_.data();
        p.dt = c.dt;
        p.duration = c.duration;
        p.mode = (int32_t)c.mode;
        p.expansion_enabled = c.expansion_enabled;
        p.temperature_dependent = c.temperature_dependent;
        p.damping_gamma = c.damping_gamma;
        p.hourglass_stiffness = c.hourglass_stiffness;
        p.allow_unstable_dt = c.allow_unstable_dt;
        p.workers = c.workers;
    }
    double interp(double T) const {  // ScalarTable::at (materials.hpp:46)
        if (cT_.size() == 1 || T <= cT_.front()) return cV_.front();
        if (T >= cT_.back()) return cV_.back();
        size_t j = 0;
        while (j + 2 < cT_.size() && T >= cT_[j + 1]) ++j;
        return cV_[j] + (cV_[j + 1] - cV_[j]) * ((T - cT_[j]) / (cT_[j + 1] - cT_[j]));
    }
    void check(tvegpu_status st) {
        if (st == TVEGPU_OK) return;
        char msg[512];
        int64_t s = -1;
        int32_t n = -1;
        tvegpu_last_error(h_, msg, sizeof msg, &s, &n);
        rethrow(st, msg, s, n);
    }
    [[noreturn]] static void rethrow(tvegpu_status st, const std::string& msg, int64_t s, int32_t n) {
        switch (st) {
            case TVEGPU_E_PARSE: throw ParseError(msg);
            case TVEGPU_E_VALIDATION: throw ValidationError(msg);
            case TVEGPU_E_INSTABILITY: throw InstabilityError(msg, (long)s, (int)n);
            case TVEGPU_E_IO: throw IoError(msg);
            default: throw DeviceError(std::string(tvegpu_status_string(st)) + ": " + msg);
        }
    }
    void pull_if_stale() {
        if (mirror_valid_) return;
        mirror_.temperatures.resize(N_);
        mirror_.disp.resize(3 * (size_t)N_);
        mirror_.disp_prev.resize(3 * (size_t)N_);
        check(tvegpu_get_temperatures(h_, mirror_.temperatures.data()));
        check(tvegpu_get_displacements(h_, mirror_.disp.data(), mirror_.disp_prev.data()));
        mirror_.viscous.resize((size_t)E_ * P_);
        if (P_) check(tvegpu_get_viscous(h_, mirror_.viscous.data()->data()));
        mirror_.time = tvegpu_time(h_);
        mirror_.step = (long)tvegpu_step_count(h_);
        mirror_valid_ = true;
    }
    void push_if_dirty() {
        if (!dirty_) return;
        check(tvegpu_set_state(h_, mirror_.temperatures.data(), mirror_.disp.data(), mirror_.disp_prev.data(),
                               P_ ? mirror_.viscous.data()->data() : nullptr, mirror_.time, mirror_.step));
        dirty_ = false;
    }

    int N_, E_, P_;
    double dt_, dur_;
    OutputSpec out_;
    tvegpu_engine* h_ = nullptr;
    std::function<std::optional<Vec3>(int, double)> motion_;  // MechBCs::motion_override (copied, like the reference)
    std::vector<int32_t> motion_nodes_;
    tvegpu_problem p_{};
    std::vector<double> nodes_, fibers_, axes_, phi_, tau_, cT_, cV_, kT_, kK_, tfixV_, ext_;
    std::vector<int32_t> elems_, fixed_, tfixN_;
    std::vector<tvegpu_prescribed> presc_;
    std::vector<tvegpu_source> srcs_;
    SimulationState mirror_;
    bool mirror_valid_ = false, dirty_ = false;
};

// mesh.hpp:73-79 load_mesh / load_mesh_file: the library's parallel parser (SPEC.md:88 format).
inline Mesh load_mesh(std::string_view text) {
    tvegpu_mesh* h = nullptr;
    tvegpu_mesh_view v;
    const tvegpu_status st = tvegpu_load_mesh(text.data(), text.size(), &h, &v);
    if (st == TVEGPU_E_PARSE) throw ParseError(tvegpu_create_error());
    if (st == TVEGPU_E_VALIDATION) throw ValidationError(tvegpu_create_error());
    if (st != TVEGPU_OK) throw std::runtime_error(tvegpu_create_error());
    Mesh m;
    const int nn = v.kind == TVEGPU_H8 ? 8 : 4;
    m.kind = v.kind == TVEGPU_H8 ? ElementKind::H8 : ElementKind::T4;
    m.nodes.resize(v.num_nodes);
    for (int i = 0; i < v.num_nodes; ++i) m.nodes[i] = {v.nodes[3 * i], v.nodes[3 * i + 1], v.nodes[3 * i + 2]};
    m.elements.assign(v.num_elements, std::array<int, 8>{});
    for (int e = 0; e < v.num_elements; ++e)
        for (int a = 0; a < nn; ++a) m.elements[e][a] = v.elements[(size_t)nn * e + a];
    if (v.fiber_dirs)
        for (int e = 0; e < v.num_elements; ++e)
            m.fiber_dirs.push_back({v.fiber_dirs[3 * e], v.fiber_dirs[3 * e + 1], v.fiber_dirs[3 * e + 2]});
    if (v.expansion_axes)
        for (int e = 0; e < v.num_elements; ++e) {
            const double* q = v.expansion_axes + 6 * (size_t)e;
            m.expansion_axes.push_back({Vec3{q[0], q[1], q[2]}, Vec3{q[3], q[4], q[5]}});
        }
    for (int k = 0; k < v.num_node_sets; ++k)
        m.node_sets[v.node_set_names[k]].assign(v.node_set_items + v.node_set_offsets[k],
                                                v.node_set_items + v.node_set_offsets[k + 1]);
    for (int k = 0; k < v.num_element_sets; ++k)
        m.element_sets[v.element_set_names[k]].assign(v.element_set_items + v.element_set_offsets[k],
                                                      v.element_set_items + v.element_set_offsets[k + 1]);
    tvegpu_mesh_destroy(h);
    return m;
}
inline Mesh load_mesh_file(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoError("load_mesh_file: cannot open " + path);
    const std::string text((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    return load_mesh(text);
}

// ---------------------------------------------------------------- small reference free functions
inline std::string to_string(ElementKind k) { return k == ElementKind::T4 ? "T4" : "H8"; }  // mesh.hpp:18
inline std::string to_string(CouplingMode m) {                                              // engine.hpp:18
    return m == CouplingMode::Coupled ? "Coupled" : m == CouplingMode::ThermalOnly ? "ThermalOnly" : "MechanicalOnly";
}
// mesh.hpp:100: shortest edge of element e
inline double min_edge_length(const Mesh& m, int e) {
    static const int t4e[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    static const int h8e[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6},
                                   {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
    const bool t4 = m.kind == ElementKind::T4;
    double L = std::numeric_limits<double>::infinity();
    for (int k = 0; k < (t4 ? 6 : 12); ++k) {
        const auto& a = m.nodes[m.elements[e][t4 ? t4e[k][0] : h8e[k][0]]];
        const auto& b = m.nodes[m.elements[e][t4 ? t4e[k][1] : h8e[k][1]]];
        L = std::min(L, std::sqrt((a[0] - b[0]) * (a[0] - b[0]) + (a[1] - b[1]) * (a[1] - b[1]) + (a[2] - b[2]) * (a[2] - b[2])));
    }
    return L;
}
struct CriticalTimestep { double thermal = 0, mechanical = 0; };
// mesh.hpp:92-97 (host-only, through the C ABI)
inline CriticalTimestep critical_timestep(const Mesh& m, const MaterialModel& mat) {
    const int nn = nodes_per_element(m.kind);
    std::vector<double> xs, cT, cV, kT, kK;
    std::vector<int32_t> el;
    for (const auto& x : m.nodes) xs.insert(xs.end(), x.begin(), x.end());
    for (const auto& e : m.elements) el.insert(el.end(), e.begin(), e.begin() + nn);
    for (const auto& [T, v] : mat.thermal.specific_heat.entries) cT.push_back(T), cV.push_back(v);
    for (const auto& e : mat.thermal.conductivity.entries) {
        kT.push_back(e.temperature);
        kK.insert(kK.end(), e.tensor.begin(), e.tensor.end());
    }
    tvegpu_problem p{};
    p.kind = m.kind == ElementKind::T4 ? TVEGPU_T4 : TVEGPU_H8;
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
    std::vector<double> fib;
    for (const auto& f : m.fiber_dirs) fib.insert(fib.end(), f.begin(), f.end());
    p.fiber_dirs = fib.empty() ? nullptr : fib.data();
    if (mat.fiber) {
        p.has_fiber = 1;
        for (int k = 0; k < 3; ++k) p.fiber[k] = (*mat.fiber)[k];
    }
    p.dt = 1.0;
    p.allow_unstable_dt = 1;
    CriticalTimestep ct;
    if (tvegpu_critical_timestep(&p, &ct.thermal, &ct.mechanical) != TVEGPU_OK)
        throw ValidationError(tvegpu_create_error());
    return ct;
}

// ---------------------------------------------------------------- engine.hpp:145-162
// Structured cube meshes for run_bench: n^3 bricks of side h (H8), or 6 positively
// oriented tetrahedra per brick around its 0-6 diagonal (T4).
inline Mesh structured_cube(int n, double h, ElementKind kind) {
    Mesh m;
    m.kind = ElementKind::H8;
    auto id = [&](int i, int j, int k) { return i + (n + 1) * (j + (n + 1) * k); };
    for (int k = 0; k <= n; ++k)
        for (int j = 0; j <= n; ++j)
            for (int i = 0; i <= n; ++i) m.nodes.push_back({i * h, j * h, k * h});
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i)
                m.elements.push_back({id(i, j, k), id(i + 1, j, k), id(i + 1, j + 1, k), id(i, j + 1, k),
                                      id(i, j, k + 1), id(i + 1, j, k + 1), id(i + 1, j + 1, k + 1), id(i, j + 1, k + 1)});
    if (kind == ElementKind::H8) return m;
    static const int t6[6][4] = {{0, 1, 2, 6}, {0, 2, 3, 6}, {0, 3, 7, 6}, {0, 7, 4, 6}, {0, 4, 5, 6}, {0, 5, 1, 6}};
    Mesh t;
    t.kind = ElementKind::T4;
    t.nodes = m.nodes;
    for (const auto& e : m.elements)
        for (const auto& q : t6) {
            std::array<int, 8> v{e[q[0]], e[q[1]], e[q[2]], e[q[3]], 0, 0, 0, 0};
            const auto &a = t.nodes[v[0]], &b = t.nodes[v[1]], &c = t.nodes[v[2]], &d = t.nodes[v[3]];
            double x[3], y[3], z[3];
            for (int r = 0; r < 3; ++r) x[r] = b[r] - a[r], y[r] = c[r] - a[r], z[r] = d[r] - a[r];
            if (x[0] * (y[1] * z[2] - y[2] * z[1]) - x[1] * (y[0] * z[2] - y[2] * z[0]) + x[2] * (y[0] * z[1] - y[1] * z[0]) < 0)
                std::swap(v[1], v[2]);
            t.elements.push_back(v);
        }
    return t;
}

struct BenchResult {
    int elements = 0, nodes = 0;
    ElementKind kind = ElementKind::T4;
    // median / IQR of per-step wall time [s] per coupled mode
    double ther_mech_ti = 0, ther_mech_ti_iqr = 0;
    double ther_mech_expan_ti = 0, ther_mech_expan_ti_iqr = 0;
    double ther_mech_expan_td = 0, ther_mech_expan_td_iqr = 0;
};

// run_bench: per-step wall time of the three coupled modes (TI, +expansion, +temperature-
// dependent properties) on structured cubes with Table-5 tissue, bottom face fixed, dt at
// 0.4 of the dilatational transit of one cell.  Per-step samples are 10-step chunks (one
// device sync per chunk).  `workers` is accepted for signature parity (host threads only
// build the plan).
inline std::vector<BenchResult> run_bench(const std::vector<int>& cells_ladder, ElementKind kind,
                                          int steps_per_measurement, int workers = 0) {
    (void)workers;
    std::vector<BenchResult> out;
    for (int n : cells_ladder) {
        const double h = 0.001;
        const Mesh m = structured_cube(n, h, kind);
        BenchResult r;
        r.elements = m.element_count();
        r.nodes = m.node_count();
        r.kind = kind;
        double* med[3] = {&r.ther_mech_ti, &r.ther_mech_expan_ti, &r.ther_mech_expan_td};
        double* iqr[3] = {&r.ther_mech_ti_iqr, &r.ther_mech_expan_ti_iqr, &r.ther_mech_expan_td_iqr};
        for (int mode = 0; mode < 3; ++mode) {
            MaterialModel mat;
            mat.hyperelastic = {1190.476, 19444.444, 0};
            mat.prony.terms = {{0.5, 0.58}};
            mat.thermal.density = 1060;
            mat.thermal.specific_heat.entries = {{37, 3600}};
            mat.thermal.conductivity = ConductivityTable::isotropic(37, 0.53);
            if (mode == 2) {
                mat.thermal.specific_heat.entries.push_back({90, 4300});
                mat.thermal.conductivity.entries.push_back({90, {0.75, 0, 0, 0, 0.75, 0, 0, 0, 0.75}});
            }
            mat.expansion = ExpansionSpec{ExpansionKind::Isotropic, 1e-4, 0, 0, 37.0};
            SimulationConfig c;
            c.dt = 0.4 * 0.9 * h / std::sqrt((19444.444 + 4 * 1190.476 / 3) / 1060);
            c.expansion_enabled = mode >= 1;
            c.temperature_dependent = mode == 2;
            c.damping_gamma = 1;
            MechBCs mb;
            for (int i = 0; i < m.node_count(); ++i)
                if (m.nodes[i][2] < 1e-12) mb.fixed_nodes.push_back(i);
            Engine e(m, mat, mb, ThermalBCs{}, HeatSourceSet{}, c);
            e.steps(20);
            std::vector<double> t;
            for (int done = 0; done < steps_per_measurement; done += 10) {
                const int k = std::min(10, steps_per_measurement - done);
                const auto t0 = std::chrono::steady_clock::now();
                e.steps(k);
                t.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / k);
            }
            std::sort(t.begin(), t.end());
            *med[mode] = t[t.size() / 2];
            *iqr[mode] = t[(3 * t.size()) / 4] - t[t.size() / 4];
        }
        out.push_back(r);
    }
    return out;
}

// bench_scaling_slope: least-squares slope of log(median step time) vs log(elements),
// on the TherMechExpanTD column.
inline double bench_scaling_slope(const std::vector<BenchResult>& results) {
    double mx = 0, my = 0;
    const double n = (double)results.size();
    for (const auto& r : results) mx += std::log((double)r.elements) / n, my += std::log(r.ther_mech_expan_td) / n;
    double sxy = 0, sxx = 0;
    for (const auto& r : results) {
        const double dx = std::log((double)r.elements) - mx, dy = std::log(r.ther_mech_expan_td) - my;
        sxy += dx * dy;
        sxx += dx * dx;
    }
    return sxx > 0 ? sxy / sxx : 0.0;
}

}  // namespace tve::gpu
