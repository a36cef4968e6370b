"""Mixed-precision (fp32 slot) mode: deviation from the oracle / the fp64 engine and speed.
    python scripts/fp32_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_10400_b200 as tg
from oracle import oracle as O
from paper_2009_10400_b200 import configs
from paper_2009_10400_b200.problem import H8, T4


def inc(x, ref, x0):
    return float(np.abs(x - ref).max() / max(np.abs(ref - x0).max(), 1e-300))


for kind in (H8, T4):
    p = configs.small_problem(kind=kind, n=5, steps=200)
    o = O.OracleEngine(p)
    g = tg.Engine(p, slot_fp32=True)
    for n in (60, 140):
        o.step(n)
        g.step(n)
        a, b = g.state(), o.state()
        print(kind, "steps", b["step"], "T", inc(a["T"], b["T"], p.initial_temperature), "u", inc(a["u"], b["u"], 0.0))
for name, make in (("cfg4", lambda: configs.cfg4(steps=1200)), ("cfg3", lambda: configs.cfg3(steps=3000))):
    p = make()
    e64, e32 = tg.Engine(p), tg.Engine(p, slot_fp32=True)
    for e in (e64, e32):
        e.step(200)
    a, b = e32.state(), e64.state()
    print(name, "200 steps fp32 vs fp64: T", inc(a["T"], b["T"], p.initial_temperature), "u", inc(a["u"], b["u"], 0.0))
    for tag, e in (("fp64", e64), ("fp32", e32)):
        st = torch.cuda.ExternalStream(e.stream)
        x, y = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x.record(st)
        e.enqueue(640)
        y.record(st)
        y.synchronize()
        e.sync()
        print(name, tag, f"{x.elapsed_time(y) / 640:.4f} ms/step", {k: round(v * 1e3, 1) for k, v in e.profile_kernels(30).items()})
