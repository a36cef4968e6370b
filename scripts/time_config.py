"""Graph-replayed ms/step of one configuration (CUDA events on the engine stream), as bench.py
times it:  python scripts/time_config.py cfg5_h8 252 [steps]   (cfg3 - 2000: no size argument)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_10400_b200 as tg
from paper_2009_10400_b200 import configs

name = sys.argv[1]
args = [int(a) for a in sys.argv[2:3] if a != "-"]  # the config's size argument ("-": none)
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 256
p = getattr(configs, name)(*args, steps=steps + 200) if args else getattr(configs, name)(steps=steps + 200)
e = tg.Engine(p)
st = torch.cuda.ExternalStream(e.stream)
e.step(64)
e.sync()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
e.enqueue(steps)
b.record(st)
b.synchronize()
e.sync()
print(f"{name}{args}: {p.num_elements:,} elements, {a.elapsed_time(b) / steps:.4f} ms/step (graph replay)")
