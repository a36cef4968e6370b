"""Checkpoint / restart (engine.hpp:110-111; "serializing state at step n
and resuming yields bit-identical state at step n+k versus an uninterrupted run")."""
import numpy as np
import pytest

import paper_2009_10400_b200 as tg
from paper_2009_10400_b200 import configs
from paper_2009_10400_b200.problem import H8, T4

pytestmark = pytest.mark.gpu


def fields(e):
    s = e.state()
    return {k: s[k] for k in ("T", "u", "u_prev", "viscous")}, s["time"], s["step"]


@pytest.mark.parametrize("kind", [T4, H8])
@pytest.mark.parametrize("override", [False, True])
def test_restart_bit_identical(kind, override, tmp_path):
    p = configs.small_problem(kind=kind, n=4, steps=40)
    a = tg.Engine(p)
    if override:
        a.set_nodal_sources(np.random.default_rng(0).uniform(0, 1e-3, p.num_nodes))
    a.step(15)
    blob = a.save_checkpoint(tmp_path / "ck.bin")
    a.step(25)
    b = tg.Engine(p, reorder=False)  # a different local numbering: the image is in original ids
    b.load_checkpoint(tmp_path / "ck.bin")
    assert b.step_count() == 15
    b.step(25)
    fa, ta, sa = fields(a)
    fb, tb, sb = fields(b)
    assert ta == tb and sa == sb == 40
    for k in fa:
        np.testing.assert_array_equal(fa[k], fb[k], err_msg=k)
    c = tg.Engine(p)
    c.load_checkpoint(blob)  # from bytes
    c.step(25)
    np.testing.assert_array_equal(fields(c)[0]["u"], fa["u"])


def test_checkpoint_errors():
    p = configs.small_problem(kind=H8, n=3, steps=10)
    a = tg.Engine(p)
    a.step(3)
    blob = a.save_checkpoint()
    with pytest.raises(tg.engine.IoError):
        tg.Engine(p).load_checkpoint(blob[:100])
    with pytest.raises(tg.engine.IoError):
        tg.Engine(p).load_checkpoint(b"NOTACKPT" + blob[8:])
    q = configs.small_problem(kind=H8, n=4, steps=10)
    with pytest.raises(tg.engine.IoError):
        tg.Engine(q).load_checkpoint(blob)
