"""The oracle side of SPEC.md's rigid-motion case (acceptance 7) with
MechBCs::motion_override (mechanics.hpp:43-46) bound through oracle_create_motion:
every node on a rigid translation + 90-degree rotation trajectory out and back, with an
interior heat source — internal forces < 1e-9 mu scale, temperatures equal to the
undeformed run (isotropic k), displacements back at zero after the cycle."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2009_10400_b200 import configs, meshgen
from paper_2009_10400_b200.problem import H8, T4, SourceRegion

MU = configs.T5["mu"]


@pytest.mark.parametrize("kind", [H8, T4])
def test_oracle_rigid_motion_load_cycle(kind):
    steps = 40
    p = configs.small_problem(kind=kind, n=3, steps=steps, perturb=False)
    p.expansion, p.expansion_enabled = None, False
    p.fixed_nodes, p.prescribed = np.zeros(0, np.int32), []
    L = float(np.ptp(p.nodes[:, 0]))
    c = p.nodes.mean(axis=0)
    p.sources = [SourceRegion(meshgen.elements_in_sphere(p.nodes, p.elements, c, 0.5 * L), 5e6)]
    T_total = steps * p.dt

    def traj(n, t):
        s = math.sin(math.pi * t / T_total)
        th = 0.5 * math.pi * s
        x, y, z = p.nodes[n] - c
        return (math.cos(th) * x - math.sin(th) * y - x + 0.1 * L * s,
                math.sin(th) * x + math.cos(th) * y - y, 0.02 * L * s)

    moving = O.OracleEngine(p, motion_override=traj)
    static = O.OracleEngine(p, motion_override=lambda n, t: (0.0, 0.0, 0.0))
    for k in range(4):
        moving.step(steps // 4)
        static.step(steps // 4)
        f = moving.diagnostics()["f_int"]
        assert np.abs(f).max() < 1e-9 * MU * L * L
        Ts, Tm = static.state()["T"], moving.state()["T"]
        assert np.abs(Tm - Ts).max() <= 1e-10 * (Ts.max() - p.initial_temperature)
    s = moving.state()
    assert np.abs(s["u"]).max() <= 1e-10 * L
    # mid-cycle the nodes really moved (the check is not vacuous)
    assert moving.step_count() == steps
