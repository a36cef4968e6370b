"""The reference's verify module and acceptance criteria 1-4, 6-8,
10 run on the GPU engine: closed-form physics, not just agreement with the oracle.
Expected values are computed here from the formulas SPEC states (the oracle module is
used only for precompute constants and the elastic PK2 of a given F)."""
import math

import numpy as np
import pytest

import paper_2009_10400_b200 as tg
from oracle import oracle as O
from paper_2009_10400_b200 import configs, meshgen
from paper_2009_10400_b200.problem import (COUPLED, EXP_ISOTROPIC, H8, MECHANICAL_ONLY, T4, THERMAL_ONLY,
                                           Prescribed, Problem, SourceRegion)

pytestmark = pytest.mark.gpu
MU, KAPPA = 1190.476, 19444.444


def box(kind, nx, ny, nz, h):
    """nx*ny*nz cubic cells of size h: H8, or 6 Kuhn tetrahedra per cell."""
    nodes, el = meshgen.structured_h8(1, h * nx, nx=nx, ny=ny, nz=nz)
    nodes = nodes * (h / (h * nx / 1))  # structured_h8 uses h = length / n with n = 1
    if kind == H8:
        return nodes, el
    loc = meshgen._kuhn_local()
    corner = np.array([0, 1, 3, 2, 4, 5, 7, 6])  # bit code x + 2y + 4z -> brick index
    return nodes, el[:, corner[loc]].reshape(-1, 4).astype(np.int32)


def test_zero_loads_state_invariant():
    p = configs.small_problem(kind=H8, n=3, perturb=False)
    p.sources, p.prescribed, p.expansion = [], [], None
    p.metabolic_rate = 0.0
    g = tg.Engine(p)
    g.step(200)
    s = g.state()
    assert not s["u"].any() and (s["T"] == p.initial_temperature).all()


@pytest.mark.parametrize("kind", [T4, H8])
def test_conservation_adiabatic(kind):  # acceptance 4: sum C_diag T constant to 1e-8 over 1e4 steps
    nodes, el = box(kind, 3, 3, 3, 0.01)
    p = Problem(kind=kind, nodes=nodes, elements=el, dt=0.05, mode=THERMAL_ONLY, c_table=[(37.0, 3600.0)],
                k_table=[(37.0, 0.53)], allow_unstable_dt=True)
    T0 = 37 + 20 * np.random.default_rng(0).uniform(size=p.num_nodes)
    g = tg.Engine(p)
    g.set_state(T=T0)
    Cd = O.precompute(p)["heat_capacity_ref"]
    e0 = (Cd * T0).sum()
    g.step(10000)
    assert abs((Cd * g.temperatures()).sum() - e0) / e0 < 1e-8


def test_perfusion_decay():  # SPEC.md:547-555, acceptance 2 (time constant within 1 %)
    nodes, el = meshgen.structured_h8(2, 0.01)
    rho, c, wb, cb = 1060.0, 3600.0, 26.6, 3617.0
    tau = rho * c / (wb * cb)
    dt = 0.01
    p = Problem(kind=H8, nodes=nodes, elements=el, dt=dt, mode=THERMAL_ONLY, c_table=[(37.0, c)],
                perfusion_rate=wb, blood_specific_heat=cb, initial_temperature=47.0, allow_unstable_dt=True)
    g = tg.Engine(p)
    ts, Ts = [], []
    for _ in range(8):
        g.step(int(round(tau / dt / 4)))
        ts.append(g.time())
        Ts.append(g.temperatures().mean())
    fit_tau = -1.0 / np.polyfit(ts, np.log(np.array(Ts) - 37.0), 1)[0]
    assert abs(fit_tau - tau) / tau < 1e-2
    t1 = ts[3]  # one time constant: error < 0.5 % in (T - Ta)
    assert abs((Ts[3] - 37) - 10 * math.exp(-t1 / tau)) / (10 * math.exp(-t1 / tau)) < 5e-3


@pytest.mark.parametrize("kind", [T4, H8])
def test_slab_conduction_fourier(kind):  # SPEC.md:537-546, acceptance 3 (< 2 % relative L2)
    rho, c, k = 1060.0, 3700.0, 0.518  # Table 1
    L, nx = 0.05, 20
    h = L / nx
    nodes, el = box(kind, nx, 1, 1, h)
    Ta, Tb, T0 = 37.0, 90.0, 37.0
    x = nodes[:, 0]
    ends = [(int(i), Ta) for i in np.nonzero(x < 1e-12)[0]] + [(int(i), Tb) for i in np.nonzero(x > L - 1e-12)[0]]
    p = Problem(kind=kind, nodes=nodes, elements=el, dt=1.0, mode=THERMAL_ONLY, density=rho, c_table=[(37.0, c)],
                k_table=[(37.0, k)], fixed_temperatures=ends, initial_temperature=T0, allow_unstable_dt=True)
    dt_th, _ = tg.engine.critical_timestep(p)
    t_check = 0.1 * rho * c * L * L / k  # = 1892.8 s
    nsteps = int(math.ceil(t_check / (0.5 * dt_th)))
    p.dt = t_check / nsteps
    g = tg.Engine(p)
    g.step(nsteps)
    a = k / (rho * c)
    t = g.time()
    n = np.arange(1, 51)
    bn = 2.0 / (n * np.pi) * ((T0 - Ta) * (1 - (-1.0) ** n) + (Tb - Ta) * (-1.0) ** n)
    exact = Ta + (Tb - Ta) * x / L + (bn[None, :] * np.sin(np.outer(x, n) * np.pi / L)
                                      * np.exp(-a * (n * np.pi / L) ** 2 * t)[None, :]).sum(axis=1)
    inner = (x > 1e-12) & (x < L - 1e-12)
    T = g.temperatures()
    err = np.linalg.norm(T[inner] - exact[inner]) / np.linalg.norm(exact[inner] - Ta)
    assert err < 0.02, err


def test_free_thermal_expansion():  # SPEC.md:556-564, acceptance 1
    n, L = 2, 0.01
    nodes, el = meshgen.structured_h8(n, L)
    cd = math.sqrt((KAPPA + 4 * MU / 3) / 1060)
    dt = 0.4 * 0.9 * (L / n) / cd
    origin, xnode, ynode = 0, n, n * (n + 1)
    p = Problem(kind=H8, nodes=nodes, elements=el, dt=dt, mu=MU, kappa=KAPPA, c_table=[(37.0, 3600.0)],
                initial_temperature=87.0, expansion_enabled=True, damping_gamma=30.0,
                expansion=dict(kind=EXP_ISOTROPIC, alpha_i=1e-4, reference_temperature=37.0),
                fixed_nodes=np.array([origin], np.int32),
                prescribed=[Prescribed(np.array([xnode]), 1, 0.0), Prescribed(np.array([xnode]), 2, 0.0),
                            Prescribed(np.array([ynode]), 2, 0.0)])
    g = tg.Engine(p, diagnostics=True)
    g.step(4000)
    x = nodes + g.state()["u"].reshape(-1, 3)
    expect = 1 + 1e-4 * 50
    lam_x = (x[xnode, 0] - x[origin, 0]) / L
    top = np.argmax(nodes.sum(axis=1))
    lam_diag = np.linalg.norm(x[top] - x[origin]) / np.linalg.norm(nodes[top] - nodes[origin])
    assert abs(lam_x - expect) / expect < 1e-3 and abs(lam_diag - expect) / expect < 1e-3
    assert np.abs(g.diagnostics()["S"]).max() < 1e-4 * MU  # residual stress


def test_stress_relaxation_matches_phi():  # SPEC.md:565-573, acceptance 6 (within 1 % on [0, 5 tau])
    nodes, el = meshgen.structured_h8(1, 0.01)
    phi, tau = [0.5], [0.58]
    eps = 1e-3
    u_target = np.zeros_like(nodes)
    u_target[:, 0] = eps * nodes[:, 0]  # uniaxial step strain, held: F = diag(1 + eps, 1, 1)
    pres = [Prescribed(np.array([i]), c, float(u_target[i, c])) for i in range(len(nodes)) for c in range(3)]
    dt = 1e-3
    p = Problem(kind=H8, nodes=nodes, elements=el, dt=dt, mu=MU, kappa=KAPPA, prony_phi=phi, prony_tau=tau,
                mode=MECHANICAL_ONLY, prescribed=pres, c_table=[(37.0, 3600.0)], allow_unstable_dt=True)
    g = tg.Engine(p, diagnostics=True)
    g.set_state(u=u_target.reshape(-1), u_prev=u_target.reshape(-1))
    F = np.diag([1 + eps, 1.0, 1.0])
    S0 = O.total_pk2_stress(F, np.eye(3), MU, KAPPA)[0, 0]
    worst = 0.0
    for k in range(1, 11):
        g.step(int(round(0.5 * tau[0] / dt)))  # every tau/2 up to 5 tau
        t = g.time()
        got = g.diagnostics()["S"].reshape(-1, 3, 3)[0, 0, 0] / S0
        want = 0.5 + 0.5 * math.exp(-t / tau[0])
        worst = max(worst, abs(got - want) / want)
    assert worst < 1e-2, worst


def test_rigid_rotation_indifference():  # SPEC.md:574-583, acceptance 7
    p = configs.small_problem(kind=H8, n=3, steps=60, perturb=False)
    p.expansion = None
    p.expansion_enabled = False
    L = np.ptp(p.nodes[:, 0])
    c = p.nodes.mean(axis=0)
    p.sources = [SourceRegion(meshgen.elements_in_sphere(p.nodes, p.elements, c, 0.5 * L), 5e6)]
    th = 0.5 * math.pi
    R = np.array([[math.cos(th), -math.sin(th), 0], [math.sin(th), math.cos(th), 0], [0, 0, 1]])
    urot = (p.nodes - c) @ R.T + c - p.nodes
    p.fixed_nodes = np.zeros(0, np.int32)
    p.prescribed = [Prescribed(np.array([i]), q, float(urot[i, q])) for i in range(p.num_nodes) for q in range(3)]
    b = tg.Engine(p, diagnostics=True)
    b.set_state(u=urot.reshape(-1), u_prev=urot.reshape(-1))
    p2 = configs.small_problem(kind=H8, n=3, steps=60, perturb=False)
    p2.expansion, p2.expansion_enabled, p2.sources = None, False, p.sources
    p2.prescribed = [Prescribed(np.array([i]), q, 0.0) for i in range(p.num_nodes) for q in range(3)]
    p2.fixed_nodes = np.zeros(0, np.int32)
    a = tg.Engine(p2)
    a.step(60)
    b.step(60)
    assert np.abs(b.temperatures() - a.temperatures()).max() <= 1e-10 * (a.temperatures().max() - 37.0)
    f = b.diagnostics()["f_int"]
    assert np.abs(f).max() < 1e-9 * MU * L * L


def test_paired_run_trends():  # acceptance 8 (directions of Table 6)
    def peak(**kw):
        p = configs.cfg1(steps=300)
        for k, v in kw.items():
            setattr(p, k, v)
        g = tg.Engine(p)
        g.step(300)
        return g.summary()["max_temperature"]
    with_exp = peak(expansion_enabled=True, temperature_dependent=False)
    no_exp = peak(expansion_enabled=False, temperature_dependent=False)
    td = peak(expansion_enabled=True, temperature_dependent=True)
    assert with_exp <= no_exp
    assert td < with_exp


def test_determinism_bit_identical():  # acceptance 10
    p = configs.small_problem(kind=T4, n=4, steps=50)
    a, b = tg.Engine(p), tg.Engine(p)
    a.step(50)
    b.step(50)
    np.testing.assert_array_equal(a.state()["u"], b.state()["u"])
    np.testing.assert_array_equal(a.state()["T"], b.state()["T"])
