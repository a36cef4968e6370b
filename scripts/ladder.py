"""Size ladder on one B200 — the reference's run_bench / bench_scaling_slope
(engine.hpp:145-162; SPEC.md:371-378 and criterion 9): per-step time of the three
coupled modes TherMechTI < TherMechExpanTI < TherMechExpanTD on structured cubes
(H8 n^3 for n = 100..252, i.e. 1M..16M elements; Kuhn T4 n^3), the log-log slope of
step time vs element count, and the host setup time.  Device-timed (CUDA events on
the engine's stream, graph-replayed steps after warm-up).

    python scripts/ladder.py [--kinds H8,T4] [--steps 200] [--out profiles/ladder_r1.json]
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_10400_b200 as tg
from bench import ClockSampler, canonical_bytes, load_peaks
from paper_2009_10400_b200 import configs
from paper_2009_10400_b200.problem import H8, T4

MODES = {"TherMechTI": dict(expansion_enabled=False, temperature_dependent=False),
         "TherMechExpanTI": dict(expansion_enabled=True, temperature_dependent=False),
         "TherMechExpanTD": dict(expansion_enabled=True, temperature_dependent=True)}
LADDER = {H8: [100, 126, 159, 200, 252], T4: [55, 69, 87, 110, 126, 139]}  # up to 16.0M / 16.1M elements


def time_steps(eng, steps, warmup, sampler, soak=0.3):
    """ms per step (CUDA events on the engine stream, graph replays) and the clocks
    sampled by nvidia-smi during the timed window (the bench's clock record)."""
    stream = torch.cuda.ExternalStream(eng.stream)
    eng.step(warmup)
    eng.sync()
    t0 = time.perf_counter()  # keep the GPU busy until clocks settle (the first rung ran cold)
    while time.perf_counter() - t0 < soak:
        eng.step(64)
        eng.sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.time()
    a.record(stream)
    eng.enqueue(steps)
    b.record(stream)
    b.synchronize()
    w1 = time.time()
    eng.sync()
    return a.elapsed_time(b) / steps, sampler.summary(w0, w1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kinds", default="H8,T4")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--out", default="gpurun_out/ladder.json")
    args = ap.parse_args()
    rows = []
    sampler = ClockSampler(0)
    peak, _ = load_peaks()
    for kname in args.kinds.split(","):
        kind = H8 if kname == "H8" else T4
        for n in LADDER[kind]:
            t0 = time.perf_counter()
            p = configs.cfg5_h8(n, steps=args.steps + args.warmup + 64) if kind == H8 else \
                configs.cfg5_t4(n, steps=args.steps + args.warmup + 64)
            t_mesh = time.perf_counter() - t0
            row = dict(kind=kname, n=n, elements=p.num_elements, nodes=p.num_nodes, mesh_gen_s=t_mesh)
            for mname, flags in MODES.items():
                for k, v in flags.items():
                    setattr(p, k, v)
                t0 = time.perf_counter()
                eng = tg.Engine(p)
                eng.sync()
                setup = time.perf_counter() - t0
                ms, clk = time_steps(eng, args.steps, args.warmup, sampler)
                row[mname] = ms
                row[mname + "_setup_s"] = setup
                row[mname + "_clocks"] = clk
                if mname == "TherMechExpanTD":  # the bench mode: element-steps/s and canonical HBM fraction
                    cb = sum(canonical_bytes(p).values())
                    row["element_steps_per_s"] = p.num_elements / (ms / 1e3)
                    row["canonical_bytes_per_step"] = cb
                    row["hbm_frac"] = cb / (ms / 1e3) / 1e9 / peak
                del eng
                torch.cuda.empty_cache()
            rows.append(row)
            print(json.dumps(row), flush=True)
    out = {"rows": rows, "slopes": {}, "steps": args.steps, "warmup": args.warmup}
    for kname in args.kinds.split(","):
        r = [x for x in rows if x["kind"] == kname]
        for mname in MODES:
            x = np.log([q["elements"] for q in r])
            y = np.log([q[mname] for q in r])
            out["slopes"][f"{kname}/{mname}"] = float(np.polyfit(x, y, 1)[0])
        out[f"{kname}_mode_order_holds"] = all(q["TherMechTI"] < q["TherMechExpanTI"] < q["TherMechExpanTD"] for q in r)
    sampler.stop()
    print(json.dumps(out["slopes"]), flush=True)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
