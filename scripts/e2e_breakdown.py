"""tvegpu_step_io cost by component on cfg4: which copies and syncs the closed-loop call pays."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2009_10400_b200 import Engine, configs

p = configs.cfg4()
N = p.num_nodes
eng = Engine(p)
power = torch.from_numpy(bench.lumped_source_power(p)).pin_memory().numpy()
Th = torch.empty(N, dtype=torch.float64, pin_memory=True).numpy()
uh = torch.empty(3 * N, dtype=torch.float64, pin_memory=True).numpy()
eng.step(64)
cases = {"step only": (None, None, None), "power": (power, None, None), "T": (None, Th, None),
         "u": (None, None, uh), "power+T": (power, Th, None), "power+T+u": (power, Th, uh)}
for name, (pw, T, u) in list(cases.items()) + list(cases.items())[::-1]:
    for _ in range(3):
        eng.step_io(pw, 1, T, u)
    t = time.perf_counter()
    for _ in range(30):
        eng.step_io(pw, 1, T, u)
    print(f"{name:12s} {(time.perf_counter() - t) / 30 * 1e3:.3f} ms")
t = time.perf_counter()
for _ in range(30):
    eng.step(1)
print(f"{'step(1)':12s} {(time.perf_counter() - t) / 30 * 1e3:.3f} ms")
