"""GPU parity: the sm_100a engine (through the C ABI) against the CPU oracle.

Tolerance (north_star): fp64 path, after N steps,
    ||x_gpu - x_cpu||_inf / max(||x_cpu - x0||_inf, 1e-300) <= 1e-10
for u (x0 = 0) and T (x0 = initial temperature); integer maps bit-exact
(tests/test_abi_and_maps.py).  Partition / reorder invariance and determinism
are bit-exact by construction and tested as such.
"""
import math

import numpy as np
import pytest

import paper_2009_10400_b200 as tg
from oracle import oracle as O
from paper_2009_10400_b200 import configs
from paper_2009_10400_b200.problem import (COUPLED, EXP_ISOTROPIC, EXP_ORTHOTROPIC, EXP_TRANSVERSELY_ISOTROPIC, H8,
                                           MECHANICAL_ONLY, T4, THERMAL_ONLY)

pytestmark = pytest.mark.gpu
TOL = 1e-10


def inc_err(x, ref, x0):
    return float(np.abs(x - ref).max() / max(np.abs(ref - x0).max(), 1e-300))


def compare(p, steps, tol=TOL, check_viscous=True, **kw):
    g = tg.Engine(p, **kw)
    o = O.OracleEngine(p)
    g.step(steps)
    o.step(steps)
    a, b = g.state(), o.state()
    eT = inc_err(a["T"], b["T"], p.initial_temperature)
    eu = inc_err(a["u"], b["u"], 0.0)
    eup = inc_err(a["u_prev"], b["u_prev"], 0.0)
    assert a["step"] == b["step"] == steps
    assert a["time"] == b["time"]  # same fp64 accumulation t += dt
    assert eT <= tol, f"T err {eT:.3e}"
    assert eu <= tol, f"u err {eu:.3e}"
    assert eup <= tol, f"u_prev err {eup:.3e}"
    if check_viscous and p.prony_count:
        ev = inc_err(a["viscous"], b["viscous"], 0.0)
        assert ev <= tol, f"viscous err {ev:.3e}"
    return g, o, dict(T=eT, u=eu)


@pytest.mark.parametrize("kind", [T4, H8])
@pytest.mark.parametrize("variant", ["base", "global_fiber", "no_prony", "prony2", "iso_noTD", "no_expansion"])
def test_small_coupled(kind, variant):
    p = configs.small_problem(kind=kind, n=4, steps=60)
    if variant == "global_fiber":
        p.fiber_dirs = None
        p.fiber = (0.6, 0.8, 0.0)
    elif variant == "no_prony":
        p.prony_phi, p.prony_tau = [], []
    elif variant == "prony2":
        p.prony_phi, p.prony_tau = [0.3, 0.2], [0.58, 0.0058]
    elif variant == "iso_noTD":
        p.temperature_dependent = False
        p.eta_a = 0.0
        p.fiber_dirs = None
    elif variant == "no_expansion":
        p.expansion_enabled = False
    compare(p, 60)


@pytest.mark.parametrize("kind", [T4, H8])
@pytest.mark.parametrize("exp_kind", [EXP_TRANSVERSELY_ISOTROPIC, EXP_ORTHOTROPIC])
@pytest.mark.parametrize("per_element_axes", [False, True])
def test_anisotropic_expansion(kind, exp_kind, per_element_axes):
    p = configs.small_problem(kind=kind, n=3, steps=40)
    p.expansion = dict(kind=exp_kind, alpha_i=1e-4, alpha_m=3e-4, alpha_n=-2e-4, reference_temperature=37.0)
    p.initial_temperature = 45.0
    if per_element_axes:
        rng = np.random.default_rng(11)
        Q = np.linalg.qr(rng.normal(size=(p.num_elements, 3, 3)))[0]
        p.expansion_axes = np.concatenate([Q[:, :, 0], Q[:, :, 1]], axis=1)
    else:
        s = 1 / math.sqrt(2)
        p.axis_m, p.axis_n = (s, s, 0.0), (-s, s, 0.0)
    compare(p, 40)


@pytest.mark.parametrize("kind", [T4, H8])
@pytest.mark.parametrize("exp_kind", [EXP_ISOTROPIC, EXP_ORTHOTROPIC])
def test_long_tables_and_prony_series(kind, exp_kind):
    """PronySeries / ScalarTable / ConductivityTable have no length limit (materials.hpp:27-65):
    six Prony terms (two beyond the staged history rows) and 20- / 24-entry c(T), k(T)
    tables (beyond the launch-parameter copies) whose entries the run's 37.0-37.12 degC
    range crosses several of."""
    p = configs.small_problem(kind=kind, n=4, steps=60)
    p.prony_phi = [0.2, 0.15, 0.1, 0.08, 0.06, 0.05]
    p.prony_tau = [0.58, 0.058, 0.0058, 5.8, 0.0012, 0.021]
    Tc = np.linspace(36.99, 37.13, 20)
    p.c_table = [(float(t), 3600.0 + 700.0 * math.sin(9.0 * i)) for i, t in enumerate(Tc)]
    Tk = np.linspace(36.995, 37.125, 24)
    p.k_table = [(float(t), np.array([[0.53 + 0.1 * math.cos(i), 0.01 * i, 0.0], [0.01 * i, 0.6, 0.02],
                                      [0.0, 0.02, 0.5 + 0.004 * i]])) for i, t in enumerate(Tk)]
    if exp_kind == EXP_ORTHOTROPIC:
        p.expansion = dict(kind=EXP_ORTHOTROPIC, alpha_i=1e-4, alpha_m=3e-4, alpha_n=-5e-5,
                           reference_temperature=37.0)
        p.axis_m, p.axis_n = (0.0, 0.6, 0.8), (1.0, 0.0, 0.0)
    compare(p, 60)


@pytest.mark.parametrize("kind", [T4, H8])
@pytest.mark.parametrize("mode", [THERMAL_ONLY, MECHANICAL_ONLY])
def test_modes(kind, mode):
    p = configs.small_problem(kind=kind, n=4, steps=50)
    p.mode = mode
    if mode == THERMAL_ONLY:
        p.initial_temperature = 40.0
    compare(p, 50)


def test_bcs_forces_and_fixed_temperatures():
    p = configs.small_problem(kind=H8, n=4, steps=40)
    rng = np.random.default_rng(5)
    p.external_force = rng.normal(scale=1e-6, size=(p.num_nodes, 3))
    p.body_force = (0.0, 0.0, -9.81 * p.density)
    p.fixed_temperatures = [(int(i), 37.0 + 10 * k) for k, i in enumerate(range(0, p.num_nodes, 7))]
    p.sources[0].t_start, p.sources[0].t_end = 5 * p.dt, 25.5 * p.dt  # window switches mid-run
    compare(p, 40)


def test_cfg1_reference_run():
    """configs[0]: H8 10^3, central source, 1000 steps — the reference CPU run."""
    p = configs.cfg1()
    _, _, err = compare(p, 1000)
    print("cfg1 increment-relative errors", err)


def test_cfg2_t4_anisotropic():
    p = configs.cfg2(steps=200)
    compare(p, 200)


def test_cfg3_liver():
    p = configs.cfg3(steps=100)
    compare(p, 100)


@pytest.mark.slow
def test_cfg4_1m_h8_parity():
    p = configs.cfg4(steps=20)
    compare(p, 20)


def test_reorder_and_determinism_bit_exact():
    p = configs.small_problem(kind=H8, n=6, steps=30)
    a = tg.Engine(p)
    b = tg.Engine(p, reorder=False)
    c = tg.Engine(p, steps_per_graph=7)
    for e in (a, b, c):
        e.step(30)
    sa, sb, sc = a.state(), b.state(), c.state()
    for k in ("T", "u", "u_prev", "viscous"):
        np.testing.assert_array_equal(sa[k], sb[k], err_msg=k)
        np.testing.assert_array_equal(sa[k], sc[k], err_msg=k)


def test_restart_bit_exact():
    p = configs.small_problem(kind=T4, n=4, steps=40)
    a = tg.Engine(p)
    a.step(40)
    b = tg.Engine(p)
    b.step(15)
    s = b.state()
    c = tg.Engine(p)
    c.set_state(s["T"], s["u"], s["u_prev"], s["viscous"], s["time"], s["step"])
    c.step(25)
    for k in ("T", "u", "u_prev", "viscous"):
        np.testing.assert_array_equal(a.state()[k], c.state()[k], err_msg=k)
    assert a.time() == c.time() and c.step_count() == 40


@pytest.mark.parametrize("kind", [T4, H8])  # T4: the two-threads-per-node K4 writes f_int
def test_diagnostics_match_oracle(kind):
    p = configs.small_problem(kind=kind, n=3, steps=10)
    g = tg.Engine(p, diagnostics=True)
    o = O.OracleEngine(p)
    g.step(10)
    o.step(10)
    dg, do = g.diagnostics(), o.diagnostics()
    for k in ("f_int", "F", "S"):
        scale = np.abs(do[k]).max()
        assert np.abs(dg[k] - do[k]).max() <= 1e-10 * scale, k


def test_nodal_source_override():
    p = configs.small_problem(kind=T4, n=3, steps=20)
    q = np.random.default_rng(1).uniform(0, 1e-3, p.num_nodes)
    g = tg.Engine(p)
    o = O.OracleEngine(p)
    g.set_nodal_sources(q)
    o.set_nodal_sources(q)
    g.step(20)
    o.step(20)
    assert inc_err(g.temperatures(), o.state()["T"], 37.0) <= TOL


@pytest.mark.parametrize("kind", [T4, H8])
def test_instability_matches_oracle(kind):
    """A non-finite temperature injected at one node: both engines raise InstabilityError
    at the same step naming the same (lowest) node, and leave the same state behind."""
    p = configs.small_problem(kind=kind, n=4, steps=30)
    p.expansion_enabled = False  # else the NaN reaches F_ther and both report a non-SPD C element error
    g = tg.Engine(p)
    o = O.OracleEngine(p)
    g.step(5)
    o.step(5)
    s = o.state()
    T = s["T"].copy()
    T[37] = np.nan
    for e in (g, o):
        e.set_state(T, s["u"], s["u_prev"], s["viscous"], s["time"], s["step"])
    with pytest.raises(O.OracleError) as eo:
        o.step(10)
    with pytest.raises(tg.InstabilityError) as eg:
        g.step(10)
    assert eo.value.status == 3
    assert (eg.value.step, eg.value.node) == (eo.value.step, eo.value.node) == (5, eo.value.node)
    assert g.step_count() == o.step_count() == 5 and g.time() == o.time()
    np.testing.assert_array_equal(np.isfinite(g.temperatures()), np.isfinite(o.state()["T"]))
    with pytest.raises(tg.InstabilityError):  # halted until the state is reset
        g.step(1)


def test_blowup_is_reported():
    """Explicit-scheme blow-up (dt far above critical): both engines stop with
    InstabilityError within a few steps of each other — the exact overflow step
    depends on intermediate magnitudes near 1e308, which legitimately differ."""
    p = configs.small_problem(kind=T4, n=2, steps=10)
    p.mode = THERMAL_ONLY
    p.dt *= 3e5
    p.allow_unstable_dt = True
    g = tg.Engine(p)
    o = O.OracleEngine(p)
    with pytest.raises(O.OracleError) as eo:
        o.step(5000)
    with pytest.raises(tg.InstabilityError) as eg:
        g.step(5000)
    assert eo.value.status == 3 and abs(eg.value.step - eo.value.step) <= 5


def test_mechanical_blowup_matches_oracle():
    p = configs.small_problem(kind=T4, n=2, steps=10)
    p.dt *= 40
    p.allow_unstable_dt = True
    g = tg.Engine(p)
    o = O.OracleEngine(p)
    with pytest.raises(O.OracleError) as eo:
        o.step(5000)
    with pytest.raises(tg.TveError) as eg:
        g.step(5000)
    assert eg.value.status in (2, 3) and abs(eg.value.step - eo.value.step) <= 5


def test_unstable_dt_refused():
    p = configs.small_problem(kind=H8, n=2)
    p.dt *= 10
    with pytest.raises(tg.ValidationError, match="critical"):
        tg.Engine(p)


@pytest.mark.parametrize("kind", [T4, H8])
@pytest.mark.parametrize("mode", [COUPLED, THERMAL_ONLY, MECHANICAL_ONLY])
@pytest.mark.parametrize("n", [1, 2, 70])
def test_step_io_matches_separate_calls(kind, mode, n):
    """tvegpu_step_io (copies overlapped on a side stream) == set_nodal_sources +
    step + make_snapshot, bit for bit, for every source vector of a changing schedule."""
    p = configs.small_problem(kind=kind, n=4, steps=6 * n)
    p.mode = mode
    a, b = tg.Engine(p), tg.Engine(p)
    rng = np.random.default_rng(n)
    Ta, ua = np.empty(p.num_nodes), np.empty(3 * p.num_nodes)
    for it in range(3):
        q = rng.uniform(0, 2e-3, p.num_nodes)
        a.set_nodal_sources(q)
        a.step(n)
        Tb_, ub_ = a.make_snapshot()
        b.step_io(q, n, Ta, ua)
        np.testing.assert_array_equal(Ta, Tb_)
        np.testing.assert_array_equal(ua, ub_)
    b.step_io(None, 1, Ta, None)  # keep the last sources, temperatures only
    a.step(1)
    np.testing.assert_array_equal(Ta, a.temperatures())
    assert a.step_count() == b.step_count() and a.time() == b.time()
    sa, sb = a.state(), b.state()
    for k in ("T", "u", "u_prev", "viscous"):
        np.testing.assert_array_equal(sa[k], sb[k], err_msg=k)


@pytest.mark.parametrize("kind", [T4, H8])
def test_single_element_mesh(kind):
    """Edge case: one element (one partially filled chunk, every node on the boundary)."""
    from paper_2009_10400_b200 import meshgen
    nodes, el = meshgen.structured_h8(1, 0.01) if kind == H8 else meshgen.kuhn_t4(1, 0.01)
    if kind == T4:
        el = el[:1]
        nodes = nodes[np.unique(el)]
        el = np.searchsorted(np.unique(meshgen.kuhn_t4(1, 0.01)[1][:1]), el).astype(np.int32)
    p = configs.small_problem(kind=kind, n=1, steps=40)
    p.nodes, p.elements = nodes, el
    p.fiber_dirs = None
    p.fixed_nodes = np.array([0], np.int32)
    p.prescribed = [tg.Prescribed(np.array([len(nodes) - 1]), 2, 1e-4, 0.002)]
    p.sources = [tg.SourceRegion(np.array([0], np.int32), 5e6)]
    compare(p, 40)


@pytest.mark.slow
def test_table1_length_run_is_stable_and_deterministic():
    """the Table-1 demo runs 62,500 steps (5 s at dt = 8e-5 s).  The liver-
    shaped T4 mesh for that many steps through the graph path: finite, physically bounded,
    the RunSummary equal to the host fields, and bit-identical on a second engine."""
    p = configs.cfg3(steps=62_500)
    p.dt = 8e-5
    a = tg.Engine(p)
    a.step(62_500)
    s, st = a.summary(), a.state()
    assert s["steps"] == 62_500 and abs(s["time"] - 5.0) < 1e-9
    assert np.isfinite(st["T"]).all() and np.isfinite(st["u"]).all()
    assert 37.0 < s["max_temperature"] < 100.0
    assert s["max_temperature"] == st["T"].max()
    b = tg.Engine(p)
    b.step(62_500)
    np.testing.assert_array_equal(b.state()["T"], st["T"])
    np.testing.assert_array_equal(b.state()["u"], st["u"])


@pytest.mark.parametrize("kind", [T4, H8])
@pytest.mark.parametrize("mode", [COUPLED, THERMAL_ONLY, MECHANICAL_ONLY])
def test_one_step_from_random_state(kind, mode):
    """Kernel-level parity (test plan item 2): one step from a random
    state — temperatures, displacements (≈1 % strain), previous displacements and a
    symmetric viscous history — on GPU and oracle; the step's increments agree to
    1e-12 (relative to the increment itself)."""
    p = configs.small_problem(kind=kind, n=4, steps=4)
    p.mode = mode
    rng = np.random.default_rng(5)
    N, E, P = p.num_nodes, p.num_elements, p.prony_count
    T = 37.0 + rng.uniform(-2.0, 10.0, N)
    u = 1e-4 * rng.normal(size=3 * N)
    up = u + 1e-6 * rng.normal(size=3 * N)
    th = rng.normal(size=(E, P, 3, 3)) * 50.0
    th = (th + np.swapaxes(th, -1, -2)).reshape(-1)
    g = tg.Engine(p)
    o = O.OracleEngine(p)
    for eng in (g, o):
        eng.set_state(T=T, u=u, u_prev=up, viscous=th, time=0.0, step=0)
        eng.step(1)
    a, b = g.state(), o.state()
    assert a["step"] == b["step"] == 1
    errs = {"T": inc_err(a["T"], b["T"], T), "u": inc_err(a["u"], b["u"], u),
            "u_prev": inc_err(a["u_prev"], b["u_prev"], up)}
    if P and mode != THERMAL_ONLY:
        errs["viscous"] = inc_err(a["viscous"], b["viscous"], th)
    for k, e in errs.items():
        if mode == THERMAL_ONLY and k != "T" or mode == MECHANICAL_ONLY and k == "T":
            continue  # untouched fields (compared bit-exactly below)
        assert e <= 1e-12, f"{k} increment err {e:.3e}"
    if mode == THERMAL_ONLY:
        assert np.array_equal(a["u"], u) and np.array_equal(b["u"], u)
    if mode == MECHANICAL_ONLY:
        assert np.array_equal(a["T"], T) and np.array_equal(b["T"], T)


def _jitter(p, frac, seed=9, where=None):
    """Move nodes by up to frac of the spacing (only those selected by `where`): distorted,
    non-affine H8 elements whose hourglass geometry c_al = X h_al is genuinely non-zero."""
    h = (p.nodes[:, 0].max() - p.nodes[:, 0].min()) / round(p.num_elements ** (1 / 3))
    d = np.random.default_rng(seed).uniform(-frac * h, frac * h, p.nodes.shape)
    if where is not None:
        d[~where(p.nodes)] = 0.0
    p.nodes = p.nodes + d
    return p


@pytest.mark.parametrize("kind", [H8, T4])
def test_distorted_mesh(kind):
    """Every node jittered by up to 15 % of the spacing: the general element path (H8: the
    hourglass geometry rows staged and used; no element is affine) against the oracle."""
    p = _jitter(configs.small_problem(kind=kind, n=5, steps=60), 0.15)
    compare(p, 60)


def test_mixed_affine_mesh_and_partitions():
    """Half the block distorted, half regular: affine chunks skip the hourglass rows, the
    others stage them, per chunk.  Parity with the oracle, and 2 / 3 / 4 partitions (whose
    chunks mix differently) bit-identical to one engine: an element's values do not depend on
    whether its chunk is all affine."""
    from paper_2009_10400_b200.engine import PartitionGroup
    p = configs.small_problem(kind=H8, n=6, steps=80)
    L = p.nodes[:, 0].max()
    p = _jitter(p, 0.12, where=lambda X: X[:, 0] < 0.5 * L - 1e-9)
    g, _, _ = compare(p, 80)
    a = g.state()
    for nparts in (2, 3, 4):
        grp = PartitionGroup(p, nparts, steps_per_graph=16)
        grp.step(80)
        b = grp.state()
        for k in ("T", "u", "u_prev", "viscous"):
            np.testing.assert_array_equal(a[k], b[k], err_msg=f"{nparts} parts {k}")


def test_affine_branch_value_identical_to_general_path(monkeypatch):
    """K3 takes its short hourglass branch per all-affine chunk; an affine element in a mixed
    chunk goes through the general branch.  Both give the same values for c_al = 0, so (1)
    an engine with affine detection off (TVEGPU_NO_AFFINE: every element general) matches
    the default engine, and (2) partitionings that put the interface elements in
    different chunks match one engine bit for bit.  (1) within 1e-12: without detection the
    hourglass rows keep the rounding-level c_al of a regular element, which detection snaps
    to zero.)"""
    from paper_2009_10400_b200.engine import PartitionGroup
    p = configs.small_problem(kind=H8, n=16, steps=60)
    L = p.nodes[:, 0].max()
    p = _jitter(p, 0.1, where=lambda X: X[:, 0] > 0.75 * L + 1e-9)
    g = tg.Engine(p)
    assert g.affine_chunks() > 0  # the short branch is exercised
    g.step(60)
    a = g.state()
    monkeypatch.setenv("TVEGPU_NO_AFFINE", "1")
    h = tg.Engine(p)
    assert h.affine_chunks() == 0
    h.step(60)
    b = h.state()
    monkeypatch.delenv("TVEGPU_NO_AFFINE")
    assert inc_err(b["u"], a["u"], 0.0) <= 1e-12
    assert inc_err(b["T"], a["T"], p.initial_temperature) <= 1e-12
    for nparts in (2, 3, 5):
        grp = PartitionGroup(p, nparts, steps_per_graph=16)
        grp.step(60)
        c = grp.state()
        for k in ("T", "u", "u_prev", "viscous"):
            np.testing.assert_array_equal(a[k], c[k], err_msg=f"{nparts} parts {k}")
    o = O.OracleEngine(p)
    o.step(60)
    r = o.state()
    assert inc_err(a["u"], r["u"], 0.0) <= 1e-10


# Mixed-precision mode (tvegpu_options.slot_fp32): element and node math in fp64, the
# per-element contributions between them stored as fp32 and summed in fp64.  Stated bound
# (measured ~2e-8 for u and ~5e-13 for T after 200 steps):
FP32_TOL_U, FP32_TOL_T = 1e-6, 1e-9


@pytest.mark.parametrize("kind", [T4, H8])
def test_fp32_slots_within_stated_bound(kind):
    p = configs.small_problem(kind=kind, n=5, steps=200)
    g = tg.Engine(p, slot_fp32=True)
    o = O.OracleEngine(p)
    g.step(200)
    o.step(200)
    a, b = g.state(), o.state()
    eu = inc_err(a["u"], b["u"], 0.0)
    eT = inc_err(a["T"], b["T"], p.initial_temperature)
    assert eu <= FP32_TOL_U and eT <= FP32_TOL_T, (eu, eT)
    assert eu > 0  # the mode is really in effect (fp32 rounding shows)


@pytest.mark.parametrize("halo", [tg.HALO_PEER, tg.HALO_NCCL])
def test_fp32_slots_partitions_bit_identical(halo):
    """The mixed mode keeps partition invariance: same kernels, same fp32 roundings, same
    canonical fp64 sums at any partition count (both halo paths carry fp32 slots)."""
    from paper_2009_10400_b200.engine import PartitionGroup
    p = configs.small_problem(kind=H8, n=6, steps=80)
    one = tg.Engine(p, slot_fp32=True)
    one.step(80)
    for nparts in (2, 4):
        grp = PartitionGroup(p, nparts, steps_per_graph=16, halo_transport=halo, slot_fp32=True)
        grp.step(80)
        a, b = one.state(), grp.state()
        for k in ("T", "u", "u_prev", "viscous"):
            np.testing.assert_array_equal(a[k], b[k], err_msg=f"{nparts} {k}")
