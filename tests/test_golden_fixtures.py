"""Frozen oracle trajectories (tests/golden/trajectories.npz, made by
tests/golden/make_golden.py) for the seeded parity problems: T4 / H8 cubes (n = 3,
perturbed per-element fibres) in the three coupling modes, 40 steps.

CPU: the problem generator still produces the same inputs (sha256) and the oracle the
same states (it is deterministic: fixed-order gathers).  GPU: the sm_100a engine matches
the frozen states within the north_star tolerance, with no live oracle involved.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import make_golden as G  # noqa: E402

FIX = np.load(os.path.join(ROOT, "tests", "golden", "trajectories.npz"))
CASES = [c[0] for c in G.cases()]
KINDS = {c[0]: (c[1], c[2]) for c in G.cases()}


def inc_err(x, ref, x0):
    return float(np.abs(x - ref).max() / max(np.abs(ref - x0).max(), 1e-300))


def check_state(s, name, p, tol):
    assert int(s["step"]) == int(FIX[f"{name}/step"]) == G.STEPS
    assert float(s["time"]) == float(FIX[f"{name}/time"])
    assert inc_err(np.asarray(s["T"]), FIX[f"{name}/T"], p.initial_temperature) <= tol
    for k in ("u", "u_prev", "viscous"):
        ref = FIX[f"{name}/{k}"]
        if np.abs(ref).max() == 0.0:
            assert np.abs(np.asarray(s[k])).max() == 0.0, k
        else:
            assert inc_err(np.asarray(s[k]).ravel(), ref.ravel(), 0.0) <= tol, k


@pytest.mark.parametrize("name", CASES)
def test_inputs_unchanged(name):
    kind, mode = KINDS[name]
    assert G.input_digest(G.case_problem(kind, mode)) == str(FIX[f"{name}/digest"])


@pytest.mark.parametrize("name", CASES)
def test_oracle_reproduces_fixture(name):
    from oracle import oracle as O
    kind, mode = KINDS[name]
    p = G.case_problem(kind, mode)
    o = O.OracleEngine(p)
    o.step(G.STEPS)
    check_state(o.state(), name, p, 1e-13)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_matches_fixture(name):
    import paper_2009_10400_b200 as tg
    kind, mode = KINDS[name]
    p = G.case_problem(kind, mode)
    g = tg.Engine(p)
    g.step(G.STEPS)
    check_state(g.state(), name, p, 1e-10)
