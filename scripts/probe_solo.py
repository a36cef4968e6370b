"""Per-kernel times (direct launches) of one solo partition vs a standalone cube of the
same size: where a partition's step spends its extra time.
    python scripts/probe_solo.py [cfg4|cfg5_16m] P"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_10400_b200 as tg
from paper_2009_10400_b200 import configs
from paper_2009_10400_b200.problem import H8

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 2
p = configs.cfg4(steps=400) if wl == "cfg4" else configs.cfg5_h8(252, steps=400)
n = 100 if wl == "cfg4" else 252
e = tg.Engine(p, nranks=P, rank=0)
e.peer_attach_solo()
e.step(20)
try:
    e.sync()
except tg.TveError:
    pass
print(f"rank 0 of {P}", {k: round(v * 1e3, 1) for k, v in e.profile_kernels(30).items()}, flush=True)
e.close()
# standalone block of the partition's size: n x n x n/P (z split first by RCB for a cube? use the same count)
q = configs.cube_problem(H8, n, 0.1 * n / 100, p.dt, 400, 1e-2, 0.01) if P == 1 else None
nz = n // P if P in (2,) else n
q = configs.cfg4(steps=400) if wl == "cfg4" and P == 1 else None
from paper_2009_10400_b200 import meshgen
import numpy as np
nodes, el = meshgen.structured_h8(n, 0.1 * n / 100)
keep = el[(nodes[el].mean(axis=1)[:, 0] < 0.05 * n / 100)]  # half the block along x
used, inv = np.unique(keep, return_inverse=True)
sub = configs._base(H8, nodes[used], inv.reshape(keep.shape).astype(np.int32), p.dt, 400)
sub.fixed_nodes = np.nonzero(sub.nodes[:, 2] <= 1e-12)[0].astype(np.int32)
s1 = tg.Engine(sub)
s1.step(20)
print("standalone half block", sub.num_elements, {k: round(v * 1e3, 1) for k, v in s1.profile_kernels(30).items()})
