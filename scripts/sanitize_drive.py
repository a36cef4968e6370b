"""Exercises every kernel of libtvegpu.so on small problems — run on the bounds-checking
build by scripts/gpu_bounds_check.sh (compute-sanitizer is not available on the GPU
pool; SURVEY.md §5 'Race detection / sanitizers').  Graph replays (steps_per_graph = 4), PDL chains,
step_io, run-level reductions, diagnostics, checkpoint and the lockstep partition
group (halo pack/unpack) all run; no oracle, no torch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2009_10400_b200 as tg
from paper_2009_10400_b200.engine import PartitionGroup
from paper_2009_10400_b200 import configs
from paper_2009_10400_b200.problem import COUPLED, H8, MECHANICAL_ONLY, T4, THERMAL_ONLY

for kind in (T4, H8):
    for mode in (COUPLED, THERMAL_ONLY, MECHANICAL_ONLY):
        p = configs.small_problem(kind=kind, n=3, steps=64)
        p.mode = mode
        e = tg.Engine(p, steps_per_graph=4, diagnostics=(mode == COUPLED))
        e.step(3)   # plain launches
        e.step(8)   # graph replays
        if mode == COUPLED:
            power = np.full(p.num_nodes, 1e-3)
            T = np.empty(p.num_nodes)
            u = np.empty(3 * p.num_nodes)
            e.step_io(power, 1, T, u)
            e.step_io(power, 2)
            e.summary()
            e.ablation_volume(37.001)
            e.element_fields()
            e.total_energy(split=True)
            ck = e.save_checkpoint()
            e.step(2)
            e.load_checkpoint(ck)
            e.step(1)
            e.profile_kernels(2)
        e.state()
        e.close()
    g = PartitionGroup(configs.small_problem(kind=kind, n=4, steps=16), 3)
    g.step(4)
    g.fields()
print("sanitize drive ok")
