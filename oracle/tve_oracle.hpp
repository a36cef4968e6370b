// tve_oracle.hpp — CPU fp64 restatement of the reference solver API.
//
// TEST INFRASTRUCTURE ONLY.  This is the parity oracle for the B200 path: only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
// legs may load it.  The product (paper_2009_10400_b200) never links it.
//
// The reference (/root/reference/proj/include/tve/*.hpp) ships declarations
// only: no bodies, no Eigen.  This file re-declares the
// same names, argument order, units and error types, written fresh and
// implemented from SPEC.md's formulas, in the reference's own data layout
// (explicit 3 x nn shape gradients, stored hourglass basis, (element, local)
// adjacency CSR, per-element F / F_ther / S_tilde caches).  Parity is pinned
// against SPEC.md's golden examples (tests/test_oracle_golden.py) — there is no
// runnable reference to compare with.  Eigen (unpinned, absent) is replaced by
// the small Mat3/Vec3 types below.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <map>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace tve_oracle {

// ---------------------------------------------------------------- errors.hpp:8-33
struct ParseError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ValidationError : std::runtime_error { using std::runtime_error::runtime_error; };
struct InstabilityError : std::runtime_error {
    InstabilityError(const std::string& m, long s, int n) : std::runtime_error(m), step(s), node(n) {}
    long step = -1;
    int node = -1;
};
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };
// A ValidationError raised by an element kernel inside Engine::step() (non-SPD C,
// materials.hpp:100; singular F): carries the step and lowest element.
struct ElementError : ValidationError {
    ElementError(const std::string& m, long s, int e) : ValidationError(m), step(s), element(e) {}
    long step = -1;
    int element = -1;
};

// ---------------------------------------------------------------- small linear algebra
struct Vec3 {
    double v[3] = {0, 0, 0};
    double& operator[](int i) { return v[i]; }
    double operator[](int i) const { return v[i]; }
};
struct Mat3 {  // row-major m[i][j]
    double m[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    static Mat3 identity() { Mat3 r; r.m[0][0] = r.m[1][1] = r.m[2][2] = 1; return r; }
    double* operator[](int i) { return m[i]; }
    const double* operator[](int i) const { return m[i]; }
};
Mat3 operator*(const Mat3& a, const Mat3& b);
Mat3 operator+(const Mat3& a, const Mat3& b);
Mat3 operator-(const Mat3& a, const Mat3& b);
Mat3 operator*(double s, const Mat3& a);
Vec3 operator*(const Mat3& a, const Vec3& x);
Mat3 transpose(const Mat3& a);
double det(const Mat3& a);
Mat3 inverse(const Mat3& a);  // general 3x3 inverse (Gaussian elimination, partial pivoting)
double trace(const Mat3& a);
Mat3 outer(const Vec3& a, const Vec3& b);

// ---------------------------------------------------------------- mesh.hpp:15-100
enum class ElementKind { T4, H8 };
inline int nodes_per_element(ElementKind k) { return k == ElementKind::T4 ? 4 : 8; }

struct Mesh {
    std::vector<Vec3> nodes;
    ElementKind kind = ElementKind::T4;
    std::vector<std::array<int, 8>> elements;
    std::map<std::string, std::vector<int>> node_sets, element_sets;
    std::vector<Vec3> fiber_dirs;                       // empty or one per element
    std::vector<std::array<Vec3, 2>> expansion_axes;    // empty or {m, n} per element
    int node_count() const { return (int)nodes.size(); }
    int element_count() const { return (int)elements.size(); }
    int nodes_per_elem() const { return nodes_per_element(kind); }
};

struct PrecomputedMesh {
    ElementKind kind = ElementKind::T4;
    int num_nodes = 0, num_elements = 0;
    std::vector<double> shape_gradients;   // 3*nn per element, column-major (col a = grad N_a)
    std::vector<double> ref_volume;
    std::vector<double> det_jacobian;      // H8 only
    std::vector<double> lumped_mass;
    std::vector<double> lumped_heat_capacity_ref;
    std::vector<double> node_volume;
    std::vector<double> hourglass_basis;   // H8 only: 4 x 8 per element, row-major (gamma_alpha rows)
    std::vector<int> adjacency_offsets;    // num_nodes + 1
    std::vector<std::pair<int, int>> adjacency;  // (element, local), ascending element then local
    int nodes_per_elem() const { return nodes_per_element(kind); }
    const double* gradients(int e) const { return shape_gradients.data() + (size_t)e * 3 * nodes_per_elem(); }
    double geometry_factor(int e) const { return ref_volume[e]; }
};

PrecomputedMesh precompute(const Mesh& mesh, double density, double ref_specific_heat);

// ---------------------------------------------------------------- materials.hpp:13-133
struct HyperelasticParams { double mu = 0, kappa = 0, eta_a = 0; };
struct PronyTerm { double phi = 0, tau = 0; };
struct PronySeries {
    std::vector<PronyTerm> terms;
    double phi_inf = 1.0;
    bool empty() const { return terms.empty(); }
    static PronySeries from_terms(std::vector<PronyTerm> terms);
};
struct ScalarTable {
    std::vector<std::pair<double, double>> entries;
    double at(double T) const;
    double min_value() const;
    double max_value() const;
};
struct ConductivityTable {
    struct Entry { double temperature = 0; Mat3 tensor; };
    std::vector<Entry> entries;
    Mat3 at(double T) const;
    double max_eigenvalue() const;
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
    Vec3 axis_m{{1, 0, 0}};
    Vec3 axis_n{{0, 1, 0}};
};

double strain_energy(const Mat3& C, const HyperelasticParams& p, const Vec3* fiber = nullptr);
Mat3 pk2_stress(const Mat3& C, const HyperelasticParams& p, const Vec3* fiber = nullptr);
Mat3 thermal_deformation_gradient(double T, const ExpansionSpec& spec, const Vec3& m, const Vec3& n);
Mat3 total_pk2_stress(const Mat3& F, const Mat3& F_ther, const HyperelasticParams& p,
                      const Vec3* fiber = nullptr);
Mat3 prony_update(const Mat3& S, std::span<Mat3> history, double dt, const PronySeries& prony);
double relaxation_function(double t, const PronySeries& prony);
double interp_property(const ScalarTable& table, double T);

struct CriticalTimestep { double thermal = 0, mechanical = 0; };
CriticalTimestep critical_timestep(const Mesh& mesh, const MaterialModel& material);
double min_edge_length(const Mesh& mesh, int e);

// ---------------------------------------------------------------- bioheat.hpp:13-76
struct ThermalState { std::vector<double> temperatures; double time = 0; };
struct SourceRegion {
    std::vector<int> elements;
    double q_r = 0, t_start = 0, t_end = std::numeric_limits<double>::infinity();
    bool active_at(double t) const { return t >= t_start && t < t_end; }
};
struct HeatSourceSet { std::vector<SourceRegion> regional; };
struct ThermalBCs { std::vector<std::pair<int, double>> fixed; double initial_temperature = 37.0; };

template <int NN>
std::array<double, NN> element_thermal_load(const Mat3& F, const double* grad /*3xNN col-major*/,
                                            const Mat3& conductivity, const double* Te,
                                            double geometry_factor);
void step_temperature(ThermalState& state, std::span<const double> assembled_loads,
                      std::span<const double> nodal_source_power, const ThermalProps& props,
                      std::span<const double> node_volume, const ThermalBCs& bcs, double dt,
                      bool temperature_dependent, double fixed_property_temperature);
void accumulate_nodal_sources(std::vector<double>& nodal_power, const HeatSourceSet& sources,
                              const Mesh& mesh, const PrecomputedMesh& pre, double time);

// ---------------------------------------------------------------- mechanics.hpp:15-110
struct MechState {
    std::vector<double> disp, disp_prev;
    std::vector<Mat3> viscous;  // num_elements * prony_terms
    static MechState zero(int num_nodes, int num_elements, int prony_terms);
};
struct PrescribedDisplacement {
    std::vector<int> nodes;
    int component = 0;
    double target = 0, ramp_time = 0;
    double value_at(double t) const {
        if (ramp_time <= 0) return target;
        return target * std::min(t / ramp_time, 1.0);
    }
};
struct MechBCs {
    std::vector<int> fixed_nodes;
    std::vector<PrescribedDisplacement> prescribed;
    std::vector<double> external_force;
    Vec3 body_force;
    std::function<std::optional<Vec3>(int, double)> motion_override;
};

template <int NN>
Mat3 deformation_gradient(const double* u_e /*3xNN col-major*/, const double* grad);
template <int NN>
void element_internal_force(const Mat3& F, const double* grad, const HyperelasticParams& params,
                            const Vec3* fiber, const Mat3& F_ther, std::span<Mat3> viscous_history,
                            double dt, const PronySeries& prony, double geometry_factor,
                            double* out /*3xNN col-major*/, Mat3* S_tilde_out = nullptr);
void hourglass_force(const double* u_e /*3x8*/, const double* gamma /*4x8 row-major*/,
                     double stiffness, double* out /*3x8*/);
void hourglass_basis_for_element(const double* coords /*3x8*/, const double* grad /*3x8*/,
                                 double* gamma /*4x8*/);
// R = bcs.external_force (the engine passes external + body force, engine.hpp:139).
void step_displacement(MechState& state, std::span<const double> assembled_forces,
                       const MechBCs& bcs, std::span<const double> lumped_mass,
                       double damping_gamma, double dt, double next_time);

// ---------------------------------------------------------------- engine.hpp:16-162
enum class CouplingMode { Coupled, ThermalOnly, MechanicalOnly };
struct SimulationConfig {
    double dt = 0, duration = 0;
    CouplingMode mode = CouplingMode::Coupled;
    bool expansion_enabled = false, temperature_dependent = false;
    double damping_gamma = 0, hourglass_stiffness = 0.1;
    bool allow_unstable_dt = false;
    int workers = 0;
};
struct SimulationState { ThermalState thermal; MechState mech; long step = 0; };

class Engine {
public:
    Engine(const Mesh& mesh, const PrecomputedMesh& pre, const MaterialModel& material,
           const MechBCs& mech_bcs, const ThermalBCs& thermal_bcs, const HeatSourceSet& sources,
           const SimulationConfig& config);
    void step();
    SimulationState& state() { return state_; }
    const SimulationState& state() const { return state_; }
    double time() const { return state_.thermal.time; }
    const std::vector<double>& last_internal_forces() const { return assembled_force_; }
    const std::vector<Mat3>& element_stresses() const { return stress_cache_; }
    const std::vector<Mat3>& deformation_gradients() const { return f_cache_; }
    const std::vector<double>& element_thermal_loads() const { return element_thermal_loads_; }
    const std::vector<double>& element_forces() const { return element_forces_; }
    const std::vector<double>& nodal_sources() const { return nodal_source_; }
    double total_energy() const;
    void set_nodal_source_override(const double* power);  // NULL = regional schedule

private:
    template <int NN> void step_impl();
    template <int NN> void thermal_element_phase(bool compute_f);
    void thermal_node_phase();
    template <int NN> void mechanics_element_phase(bool compute_f);
    void mechanics_node_phase();
    void refresh_nodal_sources();
    void check_finite(std::span<const double> values, const char* field, int stride) const;
    int element_error_ = -1;  // lowest element whose kernel hit a non-SPD C / singular F this step

    const Mesh& mesh_;
    const PrecomputedMesh& pre_;
    const MaterialModel& material_;
    MechBCs mech_bcs_;
    ThermalBCs thermal_bcs_;
    HeatSourceSet sources_;
    SimulationConfig config_;

    SimulationState state_;
    std::vector<Mat3> f_cache_, f_ther_cache_, stress_cache_;
    std::vector<Mat3> f_ther_delta_;  // F_ther - I (exact small-strain form, see pk2_from_strain)
    std::vector<double> element_thermal_loads_, element_forces_;
    std::vector<double> assembled_load_, assembled_force_;
    std::vector<double> nodal_source_, external_force_total_;
    std::vector<char> source_active_;
    bool sources_initialized_ = false;
    bool source_override_ = false;
    double fixed_property_temperature_ = 37.0;
    int workers_ = 1;
};

// ---- run-level outputs ----
// ablation_volume: exact volume of {x : T_h(x) >= threshold} for
// the piecewise-linear field, by analytic clipping of each tetrahedron; an H8 is
// split into 6 tetrahedra around its 0-6 diagonal first.  Measured at X + u when
// disp is given (deformed is the default when displacements exist).
// *elements_above counts the elements with a non-zero clipped volume.
struct AblationReport {
    double volume = 0;
    long elements_above = 0;
};
AblationReport ablation_volume(const Mesh& mesh, std::span<const double> T, double threshold,
                               const std::vector<double>* disp);
// Volume fraction of a tetrahedron above `threshold` given its nodal values.
double tet_fraction_above(const double T[4], double threshold);

}  // namespace tve_oracle
