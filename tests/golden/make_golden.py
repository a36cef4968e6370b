"""Regenerates tests/golden/trajectories.npz: oracle trajectories of small seeded problems.

The reference (/root/reference) has no runnable code, so its golden
vectors are SPEC.md's worked examples, checked inline in tests/test_oracle_golden.py.
This file freezes what the oracle — pinned to those examples — produces on the seeded
parity problems (configs.small_problem), so that

  * tests/test_golden_fixtures.py (CPU) catches any drift of the oracle or of the
    problem generator (input checksums are stored with the states), and
  * the GPU engine is also compared with a frozen fixture, not only with a live oracle.

    python tests/golden/make_golden.py      (writes tests/golden/trajectories.npz)
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2009_10400_b200 import configs  # noqa: E402
from paper_2009_10400_b200.problem import COUPLED, H8, MECHANICAL_ONLY, T4, THERMAL_ONLY  # noqa: E402

STEPS = 40
MODES = {"coupled": COUPLED, "thermal": THERMAL_ONLY, "mechanical": MECHANICAL_ONLY}


def case_problem(kind, mode):
    p = configs.small_problem(kind=kind, n=3, steps=STEPS)
    p.mode = MODES[mode]
    return p


def input_digest(p):
    h = hashlib.sha256()
    for a in (p.nodes, p.elements, p.fiber_dirs if p.fiber_dirs is not None else np.zeros(0)):
        h.update(np.ascontiguousarray(a).tobytes())
    h.update(repr((p.dt, p.initial_temperature, p.mode)).encode())
    return h.hexdigest()


def cases():
    for kind, kname in ((T4, "T4"), (H8, "H8")):
        for mode in MODES:
            yield f"{kname}_{mode}", kind, mode


def main():
    out = {}
    for name, kind, mode in cases():
        p = case_problem(kind, mode)
        o = O.OracleEngine(p)
        o.step(STEPS)
        s = o.state()
        out[f"{name}/digest"] = np.array(input_digest(p))
        for k in ("T", "u", "u_prev", "viscous"):
            out[f"{name}/{k}"] = np.asarray(s[k], dtype=np.float64)
        out[f"{name}/time"] = np.array(s["time"])
        out[f"{name}/step"] = np.array(s["step"])
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "trajectories.npz"), **out)
    print(f"{len(out)} arrays")


if __name__ == "__main__":
    main()
