"""Pin the CPU oracle against the reference's own golden examples.

The reference ships no runnable code; its tests exist only as the
per-operation examples and invariants of SPEC.md.  Every expected value below is
COMPUTED from the stated formula (never copied: SPEC.md:240 has a typo, see
SURVEY Appendix C17), and each test cites the SPEC line it pins.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2009_10400_b200 import meshgen
from paper_2009_10400_b200.problem import (COUPLED, EXP_ISOTROPIC, EXP_ORTHOTROPIC, EXP_TRANSVERSELY_ISOTROPIC,
                                           H8, MECHANICAL_ONLY, T4, THERMAL_ONLY, Prescribed, Problem,
                                           SourceRegion)

MU, KAPPA = 1190.476, 19444.444
UNIT_TET = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)


def tet_problem(**kw):
    return Problem(kind=T4, nodes=UNIT_TET.copy(), elements=np.array([[0, 1, 2, 3]]), dt=1e-6,
                   c_table=[(37.0, 3700.0)], k_table=[(37.0, 0.518)], allow_unstable_dt=True, **kw)


def cube_problem(**kw):
    nodes, el = meshgen.structured_h8(1, 1.0)
    return Problem(kind=H8, nodes=nodes, elements=el, dt=1e-6, allow_unstable_dt=True, **kw)


# ------------------------------------------------------------------ mesh / precompute
def test_precompute_unit_tet():
    pre = O.precompute(tet_problem(density=1060.0))
    assert pre["ref_volume"][0] == pytest.approx(1 / 6, rel=1e-15)
    G = pre["grads"].reshape(4, 3)
    np.testing.assert_allclose(G, [[-1, -1, -1], [1, 0, 0], [0, 1, 0], [0, 0, 1]], atol=1e-15)
    np.testing.assert_allclose(pre["lumped_mass"], 1060 / 24, rtol=1e-14)


def test_precompute_unit_cube_h8():
    pre = O.precompute(cube_problem(density=1060.0))
    assert pre["det_jacobian"][0] == pytest.approx(1 / 8, rel=1e-15)
    assert pre["ref_volume"][0] == pytest.approx(1.0, rel=1e-15)
    np.testing.assert_allclose(pre["lumped_mass"], 1060 / 8, rtol=1e-14)


@pytest.mark.parametrize("kind", [T4, H8])
def test_precompute_invariants(kind):
    from paper_2009_10400_b200 import configs
    p = configs.small_problem(kind=kind, n=3)
    p.nodes = p.nodes + np.random.default_rng(1).uniform(-0.1, 0.1, p.nodes.shape) * (p.nodes[1, 0] - p.nodes[0, 0])
    pre = O.precompute(p)
    V = pre["ref_volume"].sum()
    assert pre["lumped_mass"].sum() == pytest.approx(p.density * V, rel=1e-10)
    c_ref = 3600.0
    assert pre["heat_capacity_ref"].sum() == pytest.approx(p.density * c_ref * V, rel=1e-10)
    G = pre["grads"].reshape(p.num_elements, p.nn, 3)
    scale = np.abs(G).max()
    assert np.abs(G.sum(axis=1)).max() <= 1e-12 * scale  # partition of unity
    # adjacency: ascending element, then local (mesh.hpp:58-61)
    off, el, loc = pre["adj_offsets"], pre["adj_elem"], pre["adj_local"]
    for i in range(p.num_nodes):
        pairs = list(zip(el[off[i]:off[i + 1]], loc[off[i]:off[i + 1]]))
        assert pairs == sorted(pairs)
        for e, a in pairs:
            assert p.elements[e, a] == i
    assert (pre["lumped_mass"] > 0).all()


def test_inverted_element_rejected():
    p = tet_problem()
    p.elements = np.array([[0, 2, 1, 3]])
    with pytest.raises(O.OracleError) as ei:
        O.precompute(p)
    assert ei.value.status == 2 and "1" in str(ei.value)


def test_out_of_range_node_names_element():
    p = tet_problem()
    p.elements = np.array([[0, 1, 2, 9]])
    with pytest.raises(O.OracleError) as ei:
        O.precompute(p)
    assert "element 1" in str(ei.value)


def test_critical_timestep():
    L = 0.005
    p = tet_problem(mu=MU, kappa=KAPPA, density=1060.0)
    p.nodes = UNIT_TET * L
    th, mech = O.critical_timestep(p)
    cd = math.sqrt((KAPPA + 4 * MU / 3) / 1060)
    assert cd == pytest.approx(4.454354, rel=1e-6)
    assert mech == pytest.approx(0.9 * L / cd, rel=1e-14)
    assert mech == pytest.approx(1.010248e-3, rel=1e-6)
    assert th == pytest.approx(0.9 * 1060 * 3700 * L * L / (2 * 0.518 * 3), rel=1e-14)
    assert th == pytest.approx(28.3929, rel=1e-5)
    p.nodes = UNIT_TET * L / 2
    th2, mech2 = O.critical_timestep(p)
    assert mech2 == pytest.approx(mech / 2, rel=1e-14) and th2 == pytest.approx(th / 4, rel=1e-14)


# ------------------------------------------------------------------ materials
def test_strain_energy_goldens():
    assert O.strain_energy(np.eye(3), MU, KAPPA) == 0.0
    psi = O.strain_energy(1.21 * np.eye(3), MU, KAPPA)
    assert psi == pytest.approx(KAPPA / 2 * (1.331 - 1) ** 2, rel=1e-12)
    assert psi == pytest.approx(1065.1764, rel=1e-7)
    lam = 1.2
    Cf = np.diag([lam ** 2, 1 / lam, 1 / lam])
    a = np.array([1.0, 0, 0])
    aniso = O.strain_energy(Cf, MU, KAPPA, 2 * MU, a) - O.strain_energy(Cf, MU, KAPPA, 0.0, a)
    assert aniso == pytest.approx(MU * (1.44 - 1) ** 2, rel=1e-12)


def _rand_spd(rng):
    Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    return Q @ np.diag(rng.uniform(0.5, 2.0, 3)) @ Q.T


@pytest.mark.parametrize("eta", [0.0, 2 * MU])
def test_pk2_matches_fd_of_energy(eta):  # SPEC.md:138, 187, acceptance 5
    rng = np.random.default_rng(5)
    worst = 0.0
    for _ in range(100):
        Cm = _rand_spd(rng)
        a = rng.normal(size=3)
        a /= np.linalg.norm(a)
        S = O.pk2_stress(Cm, MU, KAPPA, eta, a)
        Sfd = np.zeros((3, 3))
        h = 1e-6
        for i in range(3):
            for j in range(3):
                E = np.zeros((3, 3))
                E[i, j] += 0.5 * h
                E[j, i] += 0.5 * h
                Sfd[i, j] = 2 * (O.strain_energy(Cm + E, MU, KAPPA, eta, a) -
                                 O.strain_energy(Cm - E, MU, KAPPA, eta, a)) / (2 * h)
        worst = max(worst, np.linalg.norm(S - Sfd) / max(np.linalg.norm(S), 1e-30))
    assert worst < 1e-4


def test_pk2_goldens():
    assert np.abs(O.pk2_stress(np.eye(3), MU, KAPPA, 2 * MU, np.array([1.0, 0, 0]))).max() < 1e-12
    lam = 1.1
    Cm = lam ** 2 * np.eye(3)
    J = lam ** 3
    np.testing.assert_allclose(O.pk2_stress(Cm, MU, KAPPA), KAPPA * J * (J - 1) * np.linalg.inv(Cm), rtol=1e-12,
                               atol=1e-9)


def test_energy_objectivity():
    rng = np.random.default_rng(7)
    for _ in range(20):
        Cm = _rand_spd(rng)
        a = rng.normal(size=3)
        a /= np.linalg.norm(a)
        Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        assert O.strain_energy(Q.T @ Cm @ Q, MU, KAPPA, 2 * MU, Q.T @ a) == pytest.approx(
            O.strain_energy(Cm, MU, KAPPA, 2 * MU, a), rel=1e-10)


def test_thermal_deformation_gradient_goldens():
    np.testing.assert_allclose(O.thermal_deformation_gradient(47.0, EXP_ISOTROPIC, 0.1), 2 * np.eye(3), rtol=1e-15)
    np.testing.assert_array_equal(O.thermal_deformation_gradient(37.0, EXP_ORTHOTROPIC, 0.1, 0.2, 0.3), np.eye(3))
    np.testing.assert_allclose(O.thermal_deformation_gradient(38.0, EXP_TRANSVERSELY_ISOTROPIC, 0.0, 0.2),
                               np.diag([1.2, 1.0, 1.0]), rtol=1e-15)
    with pytest.raises(O.OracleError):
        O.thermal_deformation_gradient(38.0, EXP_ORTHOTROPIC, 0.0, 0.2, 0.1, m=(1, 0, 0), n=(1, 1, 0))


def test_total_pk2_goldens():
    Fth = np.diag([1.01, 1.02, 0.99])
    assert np.abs(O.total_pk2_stress(Fth, Fth, MU, KAPPA)).max() < 1e-10
    rng = np.random.default_rng(3)
    F = np.eye(3) + 0.2 * rng.uniform(-1, 1, (3, 3))
    Sa, Sb = O.total_pk2_stress(F, np.eye(3), MU, KAPPA), O.pk2_stress(F.T @ F, MU, KAPPA)
    assert np.abs(Sa - Sb).max() <= 1e-14 * np.abs(Sb).max()  # same path or within 1e-14
    S = O.total_pk2_stress(np.eye(3), 1.01 * np.eye(3), MU, KAPPA)
    assert (np.diag(S) < 0).all()  # compressive
    # value: FD of W(F) = det(Fth) Psi((F Fth^-1)^T (F Fth^-1)) w.r.t. C = F^T F at F = I
    Fi = np.linalg.inv(1.01 * np.eye(3))
    W = lambda Cm: 1.01 ** 3 * O.strain_energy(Fi.T @ Cm @ Fi, MU, KAPPA)  # noqa: E731
    h = 1e-7
    Sfd = np.zeros((3, 3))
    for i in range(3):
        for j in range(3):
            E = np.zeros((3, 3))
            E[i, j] += 0.5 * h
            E[j, i] += 0.5 * h
            Sfd[i, j] = 2 * (W(np.eye(3) + E) - W(np.eye(3) - E)) / (2 * h)
    np.testing.assert_allclose(S, Sfd, rtol=1e-5, atol=1e-6 * np.abs(S).max())


def test_prony_goldens():
    S = np.array([[3.0, 1.0, 0.5], [1.0, 2.0, 0.0], [0.5, 0.0, 1.0]])
    St, h = O.prony_update(np.zeros((3, 3)), np.zeros(9), [0.5], [0.58], 0.01)
    assert not St.any() and not h.any()
    St, h = O.prony_update(S, np.zeros(9), [0.5], [0.58], 0.58)
    np.testing.assert_allclose(h[0], 0.25 * S, rtol=1e-15)
    np.testing.assert_allclose(St, 0.75 * S, rtol=1e-15)
    hist = np.zeros(9)
    for _ in range(2000):
        St, hist = O.prony_update(S, hist, [0.5], [0.58], 0.01)
    np.testing.assert_allclose(St, 0.5 * S, rtol=1e-12)


def test_relaxation_goldens():
    assert O.relaxation_function(0.0, [0.5], [0.58]) == pytest.approx(1.0, rel=1e-15)
    assert O.relaxation_function(1e6, [0.5], [0.58]) == pytest.approx(0.5, rel=1e-15)
    assert O.relaxation_function(0.58, [0.5], [0.58]) == pytest.approx(0.5 + 0.5 / math.e, rel=1e-14)
    assert O.relaxation_function(0.58, [0.5], [0.58]) == pytest.approx(0.6839397, rel=1e-7)
    ts = np.logspace(-3, 2, 50)
    vals = [O.relaxation_function(t, [0.3, 0.2], [0.58, 0.058]) for t in ts]
    assert all(a >= b for a, b in zip(vals, vals[1:]))


def test_interp_goldens():
    tab = [(37.0, 3600.0), (90.0, 4300.0)]
    assert O.interp_property(tab, 37.0) == 3600.0
    assert O.interp_property(tab, 63.5) == pytest.approx(3950.0, rel=1e-15)
    assert O.interp_property(tab, 120.0) == 4300.0
    assert O.interp_property(tab, 0.0) == 3600.0


# ------------------------------------------------------------------ bioheat
def _tet_grad():
    return np.array([[-1, -1, -1], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)


def test_element_thermal_load_goldens():
    G = _tet_grad()
    D = 0.53 * np.eye(3)
    rng = np.random.default_rng(2)
    F = np.eye(3) + 0.3 * rng.uniform(-1, 1, (3, 3))
    assert np.abs(O.element_thermal_load(F, G, D, np.full(4, 55.0), 1 / 6)).max() < 1e-12
    Te = np.array([37.0, 41.0, 50.0, 45.0])
    dense = (1 / 6) * (G @ D @ G.T) @ Te  # independent F = I assembly
    np.testing.assert_allclose(O.element_thermal_load(np.eye(3), G, D, Te, 1 / 6), dense, rtol=1e-13)
    Tlin = UNIT_TET[:, 0] * 10.0
    f0 = O.element_thermal_load(np.eye(3), G, D, Tlin, 1 / 6)
    f1 = O.element_thermal_load(np.diag([2.0, 1, 1]), G, D, Tlin, 1 / 6)
    np.testing.assert_allclose(f1, 0.5 * f0, rtol=1e-14)
    Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))  # rigid rotation indifference
    Q *= np.sign(np.linalg.det(Q))
    np.testing.assert_allclose(O.element_thermal_load(Q, G, D, Te, 1 / 6), dense, rtol=1e-12)


def test_step_temperature_goldens():
    N = 3
    Vn = np.array([0.1, 0.2, 0.3])
    T = np.array([37.0, 47.0, 60.0])
    out = O.step_temperature(T, np.zeros(N), np.zeros(N), Vn, 1060.0, [(37.0, 3600.0)], 0.0, 0.0, 37.0, 0.0, 0.01)
    np.testing.assert_array_equal(out, T)
    rate = -26.6 * 3617 * 10.0 / (1060 * 3600)
    assert rate == pytest.approx(-0.2521284, rel=1e-6)
    out = O.step_temperature(np.array([47.0]), np.zeros(1), np.zeros(1), np.array([1e-6]), 1060.0,
                             [(37.0, 3600.0)], 26.6, 3617.0, 37.0, 0.0, 2e-4)
    assert out[0] - 47.0 == pytest.approx(rate * 2e-4, rel=1e-9)
    assert out[0] - 47.0 == pytest.approx(-5.042568e-5, rel=1e-6)
    V = 1e-6
    out = O.step_temperature(np.array([37.0]), np.zeros(1), np.array([9705360.0 * V]), np.array([V]), 1060.0,
                             [(37.0, 3600.0)], 0.0, 0.0, 37.0, 0.0, 1.0)
    assert out[0] - 37.0 == pytest.approx(9705360.0 / (1060 * 3600), rel=1e-12)
    assert out[0] - 37.0 == pytest.approx(2.543333, rel=1e-6)


# ------------------------------------------------------------------ mechanics
def test_deformation_gradient_goldens():
    X = UNIT_TET
    G = _tet_grad()
    np.testing.assert_array_equal(O.deformation_gradient(np.zeros((4, 3)), G), np.eye(3))
    U = np.zeros((4, 3))
    U[:, 2] = 0.4 * X[:, 2]
    np.testing.assert_allclose(O.deformation_gradient(U, G), np.diag([1, 1, 1.4]), atol=1e-15)
    R = np.array([[0, -1, 0], [1, 0, 0], [0, 0, 1.0]])
    F = O.deformation_gradient(X @ R.T - X, G)
    np.testing.assert_allclose(F, R, atol=1e-15)
    assert np.linalg.det(F) == pytest.approx(1.0, abs=1e-15)


def test_element_internal_force_goldens():
    G = _tet_grad()
    f, _ = O.element_internal_force(np.eye(3), G, MU, KAPPA, 0.0, None, np.eye(3), np.zeros(0), [], [], 0.01, 1 / 6)
    assert np.abs(f).max() == 0.0
    Fth = 1.01 * np.eye(3)
    f, _ = O.element_internal_force(Fth, G, MU, KAPPA, 0.0, None, Fth, np.zeros(0), [], [], 0.01, 1 / 6)
    assert np.abs(f).max() < 1e-10
    F = np.diag([1.0, 1.0, 1.05])
    f, _ = O.element_internal_force(F, G, MU, KAPPA, 0.0, None, np.eye(3), np.zeros(0), [], [], 0.01, 1 / 6)
    # independent dense evaluation: V F S G with S from closed-form neo-Hookean
    Cm = F.T @ F
    J = math.sqrt(np.linalg.det(Cm))
    Ci = np.linalg.inv(Cm)
    S = MU * J ** (-2 / 3) * (np.eye(3) - np.trace(Cm) / 3 * Ci) + KAPPA * J * (J - 1) * Ci
    dense = ((1 / 6) * F @ S @ G.T).T
    np.testing.assert_allclose(f, dense, rtol=1e-10, atol=1e-12 * np.abs(dense).max())


def _distorted_hex(seed=4):
    X, el = meshgen.structured_h8(1, 1.0)
    X = X[el[0]]  # brick ordering
    return X + np.random.default_rng(seed).uniform(-0.15, 0.15, X.shape)


def _h8_grad(X):
    signs = np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                      [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], float)
    J0 = X.T @ signs / 8
    return (np.linalg.inv(J0).T @ signs.T / 8).T  # (8, 3)


def test_hourglass_goldens():
    X = _distorted_hex()
    G = _h8_grad(X)
    gamma = O.hourglass_basis(X, G)
    np.testing.assert_allclose(np.linalg.norm(gamma, axis=1), 1.0, rtol=1e-14)
    L = np.random.default_rng(1).uniform(-0.2, 0.2, (3, 3))
    U_lin = np.array([0.01, -0.02, 0.03]) + X @ L.T
    assert np.abs(O.hourglass_force(U_lin, gamma, 50.0)).max() <= 1e-12 * 50.0
    R = np.array([[0, -1, 0], [1, 0, 0], [0, 0, 1.0]])
    assert np.abs(O.hourglass_force(X @ R.T - X, gamma, 50.0)).max() <= 1e-12 * 50.0
    U = np.zeros((8, 3))
    U[:, 0] = 1e-3 * gamma[2]  # pure mode on x
    f = O.hourglass_force(U, gamma, 50.0)
    assert (f * U).sum() > 0  # f is added to f_int, so -f resists the mode
    Xc, elc = meshgen.structured_h8(1, 1.0)
    Xc = Xc[elc[0]]  # on a regular cube the gammas are orthonormal: eigen-relation
    gc = O.hourglass_basis(Xc, _h8_grad(Xc))
    np.testing.assert_allclose(gc @ gc.T, np.eye(4), atol=1e-14)
    U[:, 0] = 1e-3 * gc[2]
    np.testing.assert_allclose(O.hourglass_force(U, gc, 50.0)[:, 0], 50.0 * 1e-3 * gc[2], rtol=1e-12)


def test_step_displacement_goldens():
    z = np.zeros(3)
    u, up = O.step_displacement(z, z, z, np.array([1.0]), None, 0.0, 1.0)
    assert not u.any()
    u, up = O.step_displacement(z, z, z, np.array([1.0]), np.array([1.0, 0, 0]), 0.0, 1.0)
    assert u[0] == pytest.approx(1.0, rel=1e-15)
    # SPEC.md:315 says u+ -> u for huge gamma, but the header form it also fixes
    # (mechanics.hpp:88, the standard central difference) gives u+ -> u- : the centred
    # velocity (u+ - u-)/(2dt) -> 0.  We follow the header (DESIGN.md decision C24).
    u, up = O.step_displacement(np.array([1.0, 2, 3]), np.array([0.5, 0.5, 0.5]), z, np.array([1.0]), None, 1e12,
                                1.0)
    np.testing.assert_allclose(u, [0.5, 0.5, 0.5], rtol=1e-10)
    np.testing.assert_array_equal(up, [1, 2, 3])


# ------------------------------------------------------------------ engine
def test_engine_zero_loads_invariant():
    p = cube_problem(mu=MU, kappa=KAPPA)
    p.c_table = [(37.0, 3600.0)]
    eng = O.OracleEngine(p)
    eng.step(50)
    s = eng.state()
    assert not s["u"].any() and (s["T"] == 37.0).all()
    assert s["step"] == 50 and s["time"] == pytest.approx(50e-6)


def test_engine_conservation_adiabatic():  # SPEC.md:244, acceptance 4
    nodes, el = meshgen.kuhn_t4(3, 0.03)
    p = Problem(kind=T4, nodes=nodes, elements=el, dt=0.05, mode=THERMAL_ONLY, c_table=[(37.0, 3600.0)],
                k_table=[(37.0, 0.53)], allow_unstable_dt=True)  # thermal-only: mech limit irrelevant
    rng = np.random.default_rng(0)
    eng = O.OracleEngine(p)
    T0 = 37 + 20 * rng.uniform(size=p.num_nodes)
    eng.set_state(T=T0)
    Cd = O.precompute(p)["heat_capacity_ref"]
    e0 = (Cd * T0).sum()
    eng.step(10000)
    e1 = (Cd * eng.state()["T"]).sum()
    assert abs(e1 - e0) / e0 < 1e-8


def test_engine_perfusion_decay():  # SPEC.md:547-555, acceptance 2
    nodes, el = meshgen.structured_h8(1, 0.01)
    rho, c, wb, cb = 1060.0, 3600.0, 26.6, 3617.0
    tau = rho * c / (wb * cb)
    assert tau == pytest.approx(39.66233, rel=1e-6)
    dt = 0.01
    steps = int(round(tau / dt))
    p = Problem(kind=H8, nodes=nodes, elements=el, dt=dt, mode=THERMAL_ONLY, c_table=[(37.0, c)],
                perfusion_rate=wb, blood_specific_heat=cb, initial_temperature=47.0, allow_unstable_dt=True)
    eng = O.OracleEngine(p)
    eng.step(steps)
    t = eng.time()
    T = eng.state()["T"]
    expect = 37 + 10 * math.exp(-t / tau)
    assert abs((T.mean() - 37) - (expect - 37)) / (expect - 37) < 5e-3


def test_engine_free_expansion():  # SPEC.md:556-564, acceptance 1
    n = 2
    L = 0.01
    nodes, el = meshgen.structured_h8(n, L)
    h = L / n
    cd = math.sqrt((KAPPA + 4 * MU / 3) / 1060)
    dt = 0.4 * 0.9 * h / cd
    origin = 0
    xnode = n
    ynode = n * (n + 1)
    p = Problem(kind=H8, nodes=nodes, elements=el, dt=dt, mu=MU, kappa=KAPPA, c_table=[(37.0, 3600.0)],
                initial_temperature=87.0, expansion_enabled=True, damping_gamma=30.0,
                expansion=dict(kind=EXP_ISOTROPIC, alpha_i=1e-4, reference_temperature=37.0),
                fixed_nodes=np.array([origin], np.int32),
                prescribed=[Prescribed(np.array([xnode]), 1, 0.0), Prescribed(np.array([xnode]), 2, 0.0),
                            Prescribed(np.array([ynode]), 2, 0.0)])
    eng = O.OracleEngine(p)
    eng.step(4000)
    u = eng.state()["u"].reshape(-1, 3)
    x = nodes + u
    lam_x = (x[xnode, 0] - x[origin, 0]) / L
    top = np.argmax(nodes.sum(axis=1))
    lam_diag = np.linalg.norm(x[top] - x[origin]) / np.linalg.norm(nodes[top] - nodes[origin])
    expect = 1 + 1e-4 * 50
    assert abs(lam_x - expect) / expect < 1e-3
    assert abs((lam_x - 1) / (expect - 1) - 1) < 1e-2
    assert abs(lam_diag - expect) / expect < 1e-3


def test_engine_modes_consistency():
    from paper_2009_10400_b200 import configs
    p = configs.small_problem(kind=H8, n=3, perturb=False)
    p.sources = []
    p.expansion = None
    p.perfusion_rate = 0.0
    p.metabolic_rate = 0.0
    a = O.OracleEngine(p)
    a.step(20)
    p.mode = MECHANICAL_ONLY
    b = O.OracleEngine(p)
    b.step(20)
    np.testing.assert_allclose(a.state()["u"], b.state()["u"], rtol=0, atol=1e-14 * np.abs(b.state()["u"]).max())


def test_engine_determinism_and_restart():
    from paper_2009_10400_b200 import configs
    p = configs.small_problem(kind=H8, n=3)
    a = O.OracleEngine(p, workers=3)
    a.step(30)
    b = O.OracleEngine(p, workers=1)
    b.step(10)
    s = b.state()
    c = O.OracleEngine(p, workers=2)
    c.set_state(s["T"], s["u"], s["u_prev"], s["viscous"], s["time"], s["step"])
    c.step(20)
    for k in ("T", "u", "u_prev", "viscous"):
        np.testing.assert_array_equal(a.state()[k], c.state()[k])
    assert a.time() == c.time()


def test_engine_instability_reports_step_and_node():  # errors.hpp:21-27
    from paper_2009_10400_b200 import configs
    p = configs.small_problem(kind=T4, n=2, steps=10)
    p.mode = THERMAL_ONLY
    p.dt *= 3e5  # far above the thermal critical step: T oscillates and overflows
    p.allow_unstable_dt = True
    eng = O.OracleEngine(p)
    with pytest.raises(O.OracleError) as ei:
        eng.step(100000)
    assert ei.value.status == 3 and ei.value.step >= 0 and 0 <= ei.value.node < p.num_nodes
    assert eng.step_count() == ei.value.step  # the failing step is not counted
    T = eng.state()["T"]
    assert not np.isfinite(T[ei.value.node]) and np.isfinite(T[:ei.value.node]).all()


def test_engine_mechanical_blowup_reports_element():  # materials.hpp:100 (non-SPD C); C25
    from paper_2009_10400_b200 import configs
    p = configs.small_problem(kind=T4, n=2, steps=10)
    p.dt *= 40
    p.allow_unstable_dt = True
    eng = O.OracleEngine(p)
    with pytest.raises(O.OracleError) as ei:
        eng.step(100000)
    assert ei.value.status in (2, 3) and ei.value.step >= 0


def test_engine_unstable_dt_refused():
    from paper_2009_10400_b200 import configs
    p = configs.small_problem(kind=H8, n=2)
    p.dt *= 10
    with pytest.raises(O.OracleError) as ei:
        O.OracleEngine(p)
    assert ei.value.status == 2


def test_expansion_lowers_nothing_at_zero_alpha_thermal_only_equiv():
    from paper_2009_10400_b200 import configs
    p = configs.small_problem(kind=T4, n=3, perturb=False)
    p.prescribed = []
    p.expansion = dict(kind=EXP_ISOTROPIC, alpha_i=0.0)
    a = O.OracleEngine(p)
    a.step(15)
    p.mode = THERMAL_ONLY
    b = O.OracleEngine(p)
    b.step(15)
    np.testing.assert_array_equal(a.state()["T"], b.state()["T"])
