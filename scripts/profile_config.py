"""Per-kernel device times (CUDA events, direct launches) of one configuration:
    python scripts/profile_config.py cfg5_t4 100     (or cfg3, cfg4, cfg5_h8 N)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_10400_b200 as tg
from paper_2009_10400_b200 import configs

name = sys.argv[1]
args = [int(a) for a in sys.argv[2:]]
p = getattr(configs, name)(*args) if args else getattr(configs, name)()
eng = tg.Engine(p)
eng.step(50)
prof = eng.profile_kernels(50)
tot = sum(prof.values())
print(f"{name}{args}: {p.num_elements:,} elements, {p.num_nodes:,} nodes; "
      + "  ".join(f"{k}={v * 1e3:.1f}us" for k, v in prof.items()) + f"  sum={tot * 1e3:.1f}us")
