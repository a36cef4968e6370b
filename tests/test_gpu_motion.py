"""MechBCs::motion_override (mechanics.hpp:43-46) on the GPU and SPEC.md's rigid-motion
oracle case (acceptance 7: interior forces < 1e-9 mu scale under a rigid
trajectory, cycle-return displacement error < 1e-10 scale).

The override is a host callback, so the engine runs it as a slow path: each step the
host evaluates it at t + dt for the candidate nodes, uploads the pins, and K4 applies
them after the fixed / prescribed components (C9).  Parity with the oracle (which
evaluates the same callback for every node) is checked at <= 1e-10 increment-relative.
"""
import math

import numpy as np
import pytest

import paper_2009_10400_b200 as tg
from oracle import oracle as O
from paper_2009_10400_b200 import configs, meshgen
from paper_2009_10400_b200.problem import H8, T4, SourceRegion

pytestmark = pytest.mark.gpu
MU = configs.T5["mu"]


def rigid_trajectory(nodes, center, total_time, theta_max=0.5 * math.pi, shift=1e-3):
    """u(X, t) of a rigid rotation about z through `center` by theta(t) plus a translation
    d(t), both following sin(pi t / total_time): out to the peak and back to rest."""
    def u_at(node, t):
        s = math.sin(math.pi * t / total_time)
        th = theta_max * s
        c, sn = math.cos(th), math.sin(th)
        x, y, z = nodes[node] - center
        return (c * x - sn * y - x + shift * s, sn * x + c * y - y + 0.5 * shift * s, 0.2 * shift * s)
    return u_at


def boundary_nodes(nodes):
    lo, hi = nodes.min(axis=0), nodes.max(axis=0)
    tol = 1e-9 * np.ptp(nodes)
    on = np.any(np.abs(nodes - lo) <= tol, axis=1) | np.any(np.abs(nodes - hi) <= tol, axis=1)
    return np.nonzero(on)[0].astype(np.int32)


def inc_err(x, ref, x0):
    return float(np.abs(x - ref).max() / max(np.abs(ref - x0).max(), 1e-300))


@pytest.mark.parametrize("kind", [H8, T4])
def test_motion_override_matches_oracle(kind):
    """Boundary nodes on a rigid translation + rotation trajectory, interior free: the
    GPU (callback on the boundary candidates) against the oracle (callback on every
    node, None for the interior) after a forward-and-back cycle."""
    steps = 80
    p = configs.small_problem(kind=kind, n=4, steps=steps)
    p.fixed_nodes = np.zeros(0, np.int32)
    p.prescribed = []
    c = p.nodes.mean(axis=0)
    bnd = boundary_nodes(p.nodes)
    on = np.zeros(p.num_nodes, bool)
    on[bnd] = True
    traj = rigid_trajectory(p.nodes, c, steps * p.dt, theta_max=0.05)
    g = tg.Engine(p)
    g.set_motion_override(traj, nodes=bnd)
    o = O.OracleEngine(p, motion_override=lambda n, t: traj(n, t) if on[n] else None)
    g.step(30)
    g.step(steps - 30)
    o.step(steps)
    a, b = g.state(), o.state()
    assert a["step"] == b["step"] == steps and a["time"] == b["time"]
    for k, x0 in (("T", p.initial_temperature), ("u", 0.0), ("u_prev", 0.0), ("viscous", 0.0)):
        e = inc_err(a[k], b[k], x0)
        assert e <= 1e-10, f"{k} {e:.3e}"
    # the pins are exact: boundary nodes sit on the trajectory
    want = np.array([traj(int(i), a["time"]) for i in bnd])
    np.testing.assert_array_equal(a["u"].reshape(-1, 3)[bnd], want)
    # removing the override returns to the plain (graph-replayed) path
    g.set_motion_override(None)
    g.step(5)


@pytest.mark.parametrize("kind", [H8, T4])
def test_rigid_motion_load_cycle(kind):
    """SPEC.md:574-583 / acceptance 7 with motion_override on every node: a rigid
    translation + 90-degree rotation out and back, with an interior heat source.
    Internal forces stay < 1e-9 mu scale at every sampled time, temperatures equal the
    undeformed run within 1e-10 of the rise (isotropic k), and after the cycle the
    displacements are back at zero within 1e-10 scale (no accumulation)."""
    steps = 60
    p = configs.small_problem(kind=kind, n=3, steps=steps, perturb=False)
    p.expansion, p.expansion_enabled = None, False
    p.fixed_nodes, p.prescribed = np.zeros(0, np.int32), []
    L = float(np.ptp(p.nodes[:, 0]))
    c = p.nodes.mean(axis=0)
    p.sources = [SourceRegion(meshgen.elements_in_sphere(p.nodes, p.elements, c, 0.5 * L), 5e6)]
    traj = rigid_trajectory(p.nodes, c, steps * p.dt, shift=0.1 * L)
    moving = tg.Engine(p, diagnostics=True)
    moving.set_motion_override(traj)
    static = tg.Engine(p)
    static.set_motion_override(lambda n, t: (0.0, 0.0, 0.0))
    worst_f = 0.0
    for k in range(6):
        moving.step(steps // 6)
        static.step(steps // 6)
        worst_f = max(worst_f, float(np.abs(moving.diagnostics()["f_int"]).max()))
        rise = static.temperatures().max() - p.initial_temperature
        assert np.abs(moving.temperatures() - static.temperatures()).max() <= 1e-10 * rise
    assert worst_f < 1e-9 * MU * L * L, worst_f
    s = moving.state()
    assert np.abs(s["u"]).max() <= 1e-10 * L
    assert np.abs(s["viscous"]).max() < 1e-9 * MU
