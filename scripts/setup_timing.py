"""Setup-time breakdown: tvegpu_create stage timings (TVEGPU_TIMING=1)
on the 16M-element H8 mesh (and cfg4), as the engine is created by bench.py.

    python scripts/setup_timing.py [n ...]      (H8 n^3; default 100 252)"""
import os
import sys
import time

os.environ["TVEGPU_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_10400_b200 as tg  # noqa: E402
from paper_2009_10400_b200 import configs  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [100, 252]:
    t = time.perf_counter()
    p = configs.cfg5_h8(n, steps=50) if n != 100 else configs.cfg4(steps=50)
    print(f"H8 n={n}: {p.num_elements:,} elements; problem generation {time.perf_counter() - t:.2f} s",
          file=sys.stderr, flush=True)
    for rep in range(2):
        t = time.perf_counter()
        e = tg.Engine(p)
        dt = time.perf_counter() - t
        e.step(2)
        print(f"H8 n={n} rep {rep}: tvegpu_create {dt:.3f} s (threads {os.cpu_count()})", file=sys.stderr, flush=True)
        e.close()
