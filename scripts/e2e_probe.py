"""Breaks the e2e step (bench.py) into its calls and measures raw pinned PCIe copies."""
import time

import numpy as np
import torch

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2009_10400_b200 import Engine, configs

p = configs.cfg4()
N = p.num_nodes
for nbytes in (8 * N, 32 * N):
    h = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True)
    d = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
    for direction in ("h2d", "d2h"):
        for _ in range(3):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(20):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 20
        print(f"{direction} {nbytes/1e6:.1f} MB: {dt*1e3:.3f} ms  {nbytes/dt/1e9:.1f} GB/s")
eng = Engine(p)
power = torch.from_numpy(bench.lumped_source_power(p)).pin_memory().numpy()
Th = torch.empty(N, dtype=torch.float64, pin_memory=True).numpy()
uh = torch.empty(3 * N, dtype=torch.float64, pin_memory=True).numpy()
eng.step(5)
ts = np.zeros(3)
for k in range(23):
    t0 = time.perf_counter()
    eng.set_nodal_sources(power)
    t1 = time.perf_counter()
    eng.step(1)
    t2 = time.perf_counter()
    eng.make_snapshot(Th, uh)
    t3 = time.perf_counter()
    if k >= 3:
        ts += [t1 - t0, t2 - t1, t3 - t2]
ts /= 20
print("set_nodal_sources %.3f ms  step(1) %.3f ms  make_snapshot %.3f ms  total %.3f" % (*(ts * 1e3), ts.sum() * 1e3))

# set_nodal_sources alone, back to back (no step in between)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20):
    eng.set_nodal_sources(power)
print("set_nodal_sources alone %.3f ms" % ((time.perf_counter() - t) / 20 * 1e3))
t = time.perf_counter()
for _ in range(20):
    eng.make_snapshot(Th, uh)
print("make_snapshot alone %.3f ms" % ((time.perf_counter() - t) / 20 * 1e3))
t = time.perf_counter()
for _ in range(20):
    eng.step(1)
print("step(1) alone %.3f ms" % ((time.perf_counter() - t) / 20 * 1e3))
pw = torch.from_numpy(power)
dd = torch.empty_like(pw, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20):
    dd.copy_(pw, non_blocking=True)
    torch.cuda.synchronize()
print("torch H2D 8MB + sync %.3f ms  (pinned=%s)" % ((time.perf_counter() - t) / 20 * 1e3, pw.is_pinned()))
pg = np.array(power)  # pageable copy
t = time.perf_counter()
for _ in range(20):
    eng.set_nodal_sources(pg)
print("set_nodal_sources pageable %.3f ms" % ((time.perf_counter() - t) / 20 * 1e3))
import ctypes
from paper_2009_10400_b200 import engine as _e
L = _e.lib()
src = _e._f64(power)
ptr = src.ctypes.data_as(_e._dp)
t = time.perf_counter()
for _ in range(20):
    L.tvegpu_set_nodal_sources(eng._h, ptr)
print("raw C call (pinned) %.3f ms" % ((time.perf_counter() - t) / 20 * 1e3))
