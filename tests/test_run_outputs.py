"""Run-level outputs on the device: RunSummary extrema,
ablation_volume by exact tet clipping, snapshot element fields — each against the
oracle (ablation: oracle/tve_oracle.cpp ablation_volume, pinned by
tests/test_ablation_oracle.py) on the same fields."""
import numpy as np
import pytest

import paper_2009_10400_b200 as tg
from oracle import oracle as O
from paper_2009_10400_b200 import configs
from paper_2009_10400_b200.problem import H8, T4

pytestmark = pytest.mark.gpu


def gaussian_T(nodes, peak=90.0, width=None):
    c = nodes.mean(axis=0)
    L = np.ptp(nodes[:, 0])
    w = width or 0.25 * L
    return 37.0 + (peak - 37.0) * np.exp(-np.sum((nodes - c) ** 2, axis=1) / (2 * w * w))


@pytest.mark.parametrize("kind", [T4, H8])
def test_summary_matches_state(kind):
    p = configs.small_problem(kind=kind, n=4, steps=30)
    g = tg.Engine(p)
    g.step(30)
    s, st = g.summary(), g.state()
    u = st["u"].reshape(-1, 3)
    assert s["steps"] == 30 and s["time"] == st["time"]
    assert s["max_temperature"] == st["T"].max()  # extrema are exact
    np.testing.assert_array_equal(s["min_disp"], u.min(axis=0))
    np.testing.assert_array_equal(s["max_disp"], u.max(axis=0))
    o = O.OracleEngine(p)
    o.step(30)
    ou = o.state()["u"].reshape(-1, 3)
    assert abs(s["max_temperature"] - o.state()["T"].max()) <= 1e-10 * 60
    assert np.abs(s["max_disp"] - ou.max(axis=0)).max() <= 1e-10 * np.abs(ou).max()


@pytest.mark.parametrize("kind", [T4, H8])
@pytest.mark.parametrize("deformed", [False, True])
def test_ablation_volume_matches_oracle(kind, deformed):
    p = configs.small_problem(kind=kind, n=6, steps=10)
    g = tg.Engine(p)
    T = gaussian_T(p.nodes)
    u = 0.02 * (p.nodes - p.nodes.mean(axis=0))  # 2 % dilation about the centre
    g.set_state(T=T, u=u, u_prev=u)
    for thr in (40.0, 60.0, 75.0, 89.0, 95.0):
        v, n = g.ablation_volume(thr, deformed=deformed)
        vo, no = O.ablation_volume("H8" if kind == H8 else "T4", p.nodes, p.elements, T, thr,
                                   disp=u if deformed else None)
        assert n == no
        assert abs(v - vo) <= 1e-12 * max(vo, 1e-300), (thr, v, vo)


def test_ablation_spec_uniform_cases():
    p = configs.small_problem(kind=H8, n=4, steps=10)
    g = tg.Engine(p)
    total = 0.04 ** 3
    g.set_state(T=np.full(p.num_nodes, 70.0))
    v, n = g.ablation_volume(60.0, deformed=False)
    assert abs(v - total) <= 1e-12 * total and n == p.num_elements
    g.set_state(T=np.full(p.num_nodes, 37.0))
    assert g.ablation_volume(60.0) == (0.0, 0)


def test_ablation_after_heating_run_is_deterministic():
    p = configs.cfg1(steps=200)
    g = tg.Engine(p)
    g.step(200)
    a = g.ablation_volume(40.0)
    b = g.ablation_volume(40.0)
    assert a == b  # fixed-order device reduction
    st = g.state()
    vo, no = O.ablation_volume("H8", p.nodes, p.elements, st["T"], 40.0, disp=st["u"])
    assert a[1] == no and abs(a[0] - vo) <= 1e-12 * max(vo, 1e-300)


@pytest.mark.parametrize("kind", [T4, H8])
def test_element_fields(kind):
    p = configs.small_problem(kind=kind, n=4, steps=20)
    g = tg.Engine(p, diagnostics=True)
    g.step(20)
    detf, smax = g.element_fields()
    d = g.diagnostics()
    F = d["F"].reshape(-1, 3, 3)
    S = d["S"].reshape(-1, 3, 3)
    np.testing.assert_allclose(detf, np.linalg.det(F), rtol=1e-13, atol=0)
    ev = np.linalg.eigvalsh(0.5 * (S + S.transpose(0, 2, 1)))[:, -1]
    scale = np.abs(ev).max()
    assert np.abs(smax - ev).max() <= 1e-10 * scale
    with pytest.raises(tg.engine.TveError):
        tg.Engine(p).element_fields()  # needs diagnostics


def test_run_with_sink_matches_stepping():  # engine.hpp:92 run(sink) -> RunSummary
    p = configs.cfg1(steps=120)
    a = tg.Engine(p)
    snaps = []
    r = a.run(sink=snaps.append, snapshot_interval=40 * p.dt, ablation_threshold=37.2)
    assert r["steps"] == 120 and [s["step"] for s in snaps] == [40, 80, 120]
    b = tg.Engine(p)
    b.step(120)
    st = b.state()
    np.testing.assert_array_equal(snaps[-1]["temperatures"], st["T"])
    np.testing.assert_array_equal(snaps[-1]["displacements"], st["u"])
    assert r["max_temperature"] == st["T"].max()
    assert r["ablation_volume"] == b.ablation_volume(37.2)[0]
    assert r["median_step_seconds"] > 0


@pytest.mark.parametrize("kind", [T4, H8])
@pytest.mark.parametrize("variant", ["coupled", "orthotropic"])
def test_total_energy_matches_oracle(kind, variant):  # engine.hpp:108
    from paper_2009_10400_b200.problem import EXP_ORTHOTROPIC
    p = configs.small_problem(kind=kind, n=4, steps=30)
    if variant == "orthotropic":
        p.expansion = dict(kind=EXP_ORTHOTROPIC, alpha_i=1e-4, alpha_m=3e-4, alpha_n=2e-4, reference_temperature=37.0)
        p.initial_temperature = 60.0
    g = tg.Engine(p)
    o = O.OracleEngine(p)
    g.step(30)
    o.step(30)
    ek, es = g.total_energy(split=True)
    eo = o.total_energy()
    assert ek > 0 and es > 0
    assert abs((ek + es) - eo) <= 1e-8 * eo, (ek + es, eo)
