// facade_demo.cpp — a reference-style C++ caller of the B200 engine through the
// tve::gpu facade (include/tve_gpu.hpp): the cfg1 problem (H8 10^3 unit cube,
// Table-5 liver tissue, central source, bottom fixed, top u_z ramp), N steps,
// then the Table-6 style summary (max T, displacement extrema).
//
//   g++ -std=c++17 -O2 -I include examples/facade_demo.cpp -L paper_2009_10400_b200/lib
//       -ltvegpu -Wl,-rpath,$PWD/paper_2009_10400_b200/lib -o facade_demo
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <sstream>

#include "tve_gpu.hpp"

using namespace tve::gpu;

int main(int argc, char** argv) {
    const int n = 10, steps = argc > 1 ? std::atoi(argv[1]) : 1000;
    const double L = 1.0, h = L / n;
    Mesh mesh;
    mesh.kind = ElementKind::H8;
    auto nid = [&](int i, int j, int k) { return i + (n + 1) * (j + (n + 1) * k); };
    for (int k = 0; k <= n; ++k)
        for (int j = 0; j <= n; ++j)
            for (int i = 0; i <= n; ++i) mesh.nodes.push_back({i * h, j * h, k * h});
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i)
                mesh.elements.push_back({nid(i, j, k), nid(i + 1, j, k), nid(i + 1, j + 1, k), nid(i, j + 1, k),
                                         nid(i, j, k + 1), nid(i + 1, j, k + 1), nid(i + 1, j + 1, k + 1),
                                         nid(i, j + 1, k + 1)});
    MaterialModel mat;  // Table 5
    mat.hyperelastic = {1190.476, 19444.444, 2 * 1190.476};
    mat.fiber = Vec3{1, 0, 0};
    mat.prony.terms = {{0.5, 0.58}};
    mat.thermal.density = 1060;
    mat.thermal.specific_heat.entries = {{37, 3600}, {90, 4300}};
    mat.thermal.conductivity = ConductivityTable::isotropic(37, 0.53);
    mat.thermal.conductivity.entries.push_back({90, {0.75, 0, 0, 0, 0.75, 0, 0, 0, 0.75}});
    mat.thermal.perfusion_rate = 26.6;
    mat.thermal.blood_specific_heat = 3617;
    mat.thermal.metabolic_rate = 33800;
    mat.expansion = ExpansionSpec{ExpansionKind::Isotropic, 1e-4, 0, 0, 37.0};
    MechBCs mb;
    PrescribedDisplacement top;
    top.component = 2;
    top.target = 0.1;
    // ramp over the run, never faster than ten dilatational wave transits (configs.ramp_time)
    const double cd = std::sqrt((mat.hyperelastic.kappa + 4.0 * mat.hyperelastic.mu / 3.0) / mat.thermal.density);
    top.ramp_time = std::max(0.01 * steps, 10.0 * L / cd);
    for (int i = 0; i < mesh.node_count(); ++i) {
        if (std::fabs(mesh.nodes[i][2]) < 1e-12) mb.fixed_nodes.push_back(i);
        if (std::fabs(mesh.nodes[i][2] - L) < 1e-12) top.nodes.push_back(i);
    }
    mb.prescribed.push_back(top);
    HeatSourceSet src;
    SourceRegion r;
    r.q_r = 9705360.0;
    for (int e = 0; e < mesh.element_count(); ++e) {
        double c[3] = {0, 0, 0};
        for (int a = 0; a < 8; ++a)
            for (int k = 0; k < 3; ++k) c[k] += mesh.nodes[mesh.elements[e][a]][k] / 8;
        const double d = std::sqrt((c[0] - .5) * (c[0] - .5) + (c[1] - .5) * (c[1] - .5) + (c[2] - .5) * (c[2] - .5));
        if (d <= 0.1) r.elements.push_back(e);
    }
    src.regional.push_back(r);
    SimulationConfig cfg;
    cfg.dt = 0.01;
    cfg.duration = 0.01 * steps;
    cfg.expansion_enabled = true;
    cfg.temperature_dependent = true;
    cfg.damping_gamma = 1.0;
    try {
        const CriticalTimestep ct = critical_timestep(mesh, mat);  // mesh.hpp:97
        std::printf("%s mesh, %s: critical dt thermal %.6g s, mechanical %.6g s, min edge %.6g m\n",
                    to_string(mesh.kind).c_str(), to_string(CouplingMode::Coupled).c_str(), ct.thermal, ct.mechanical,
                    min_edge_length(mesh, 0));
        Engine eng(mesh, mat, mb, ThermalBCs{}, src, cfg);
        eng.steps(steps);
        const SimulationState& s = eng.state();
        const double Tmax = *std::max_element(s.temperatures.begin(), s.temperatures.end());
        double umin[3] = {1e300, 1e300, 1e300}, umax[3] = {-1e300, -1e300, -1e300};
        for (int i = 0; i < mesh.node_count(); ++i)
            for (int k = 0; k < 3; ++k) {
                umin[k] = std::min(umin[k], s.disp[3 * i + k]);
                umax[k] = std::max(umax[k], s.disp[3 * i + k]);
            }
        std::printf("steps %ld time %.17g  T_max %.17g  u_z [%.17g, %.17g]\n", s.step, s.time, Tmax, umin[2],
                    umax[2]);
        // run-level outputs on the device: RunSummary extrema and the 40 degC isotherm volume
        const tvegpu_summary sm = eng.summary();
        const auto abl = eng.ablation_volume(40.0);
        std::printf("device summary: T_max %.17g  u_z max %.17g  ablation(40C) %.17g m^3 in %ld elements\n",
                    sm.max_temperature, sm.max_disp[2], abl.first, abl.second);
        // checkpoint / restart (engine.hpp:110-111): resume a copy and compare after 10 more steps
        std::stringstream ck;
        eng.save_checkpoint(ck);
        Engine twin(mesh, mat, mb, ThermalBCs{}, src, cfg);
        twin.load_checkpoint(ck);
        eng.steps(10);
        twin.steps(10);
        const bool same = eng.state().temperatures == twin.state().temperatures && eng.state().disp == twin.state().disp;
        std::printf("checkpoint resume bit-identical: %s\n", same ? "yes" : "NO");
        // engine.hpp:92 run(): a fresh engine over 50 steps, a snapshot sink every 10 steps
        {
            SimulationConfig c2 = cfg;
            c2.duration = 50 * cfg.dt;
            c2.output.snapshot_interval = 10 * cfg.dt;
            c2.output.ablation_threshold = 37.5;
            Engine e2(mesh, mat, mb, ThermalBCs{}, src, c2);
            int nsnap = 0;
            const RunSummary rs = e2.run([&](const Snapshot& s) { nsnap += s.step > 0 ? 1 : 0; });
            std::printf("run(): %ld steps, %d snapshots, T_max %.6f, ablation(37.5C) %.6g m^3\n", rs.steps, nsnap,
                        rs.max_temperature, rs.ablation_volume);
        }
        // reference-style state() write: cool the whole block back to 37 degC, keep stepping
        SimulationState& w = eng.mutable_state();
        std::fill(w.temperatures.begin(), w.temperatures.end(), 37.0);
        eng.step();
        std::printf("after reset + 1 step: T_max %.6f\n",
                    *std::max_element(eng.state().temperatures.begin(), eng.state().temperatures.end()));
    } catch (const InstabilityError& e) {
        std::printf("instability at step %ld node %d: %s\n", e.step, e.node, e.what());
        return 2;
    } catch (const std::exception& e) {
        std::printf("error: %s\n", e.what());
        return 1;
    }
    return 0;
}
