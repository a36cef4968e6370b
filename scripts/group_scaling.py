"""Partitioning overhead of the multi-GPU step, measured on one B200.

A tvegpu_group of P RCB partitions runs the multi-GPU step code (boundary SEND launches
with peer-memory halo stores + flags, interior launches, node kernels that wait for
the flags, P streams, CUDA graphs) on ONE device, so its per-step time holds the whole
mesh's work plus everything partitioning adds: P-fold launches, the boundary/interior
split, replicated interface nodes, the halo stores.  T(1) / T(P) is therefore the
efficiency one B200 sees for the same total work split P ways; the real P-GPU run adds
the NVLink transfer of the halo (per rank ~ halo bytes / 900 GB/s, overlapped with the
interior chunks) and divides the work by P.

    python scripts/group_scaling.py [--workload cfg5_16m|cfg4] [--parts 1,2,4,8] [--steps 100]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_10400_b200 as tg
from bench import WORKLOADS, ClockSampler
from paper_2009_10400_b200.engine import PartitionGroup


def per_step_ms(run, steps, warmup):
    run(warmup)
    t0 = time.perf_counter()
    run(steps)  # synchronous: returns after the device finite check
    return 1e3 * (time.perf_counter() - t0) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg5_16m", choices=sorted(WORKLOADS))
    ap.add_argument("--parts", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=64)
    ap.add_argument("--halo", default="peer", choices=["peer", "nccl"])
    ap.add_argument("--out", default="gpurun_out/group_scaling.json")
    args = ap.parse_args()
    label, make = WORKLOADS[args.workload]
    p = make(args.steps + args.warmup + 64)
    halo = tg.HALO_PEER if args.halo == "peer" else tg.HALO_NCCL
    sampler = ClockSampler(0)
    rows = []
    for P in [int(x) for x in args.parts.split(",")]:
        if P == 1:
            e = tg.Engine(p)
            w0 = time.time()
            ms = per_step_ms(e.step, args.steps, args.warmup)
            w1 = time.time()
            kps = e.kernels_per_step()
            e.close()
        else:
            g = PartitionGroup(p, P, halo_transport=halo)
            w0 = time.time()
            ms = per_step_ms(g.step, args.steps, args.warmup)
            w1 = time.time()
            kps = None
            g.close()
        row = {"parts": P, "ms_per_step": ms, "element_steps_per_s": p.num_elements / (ms / 1e3),
               "clocks": sampler.summary(w0, w1)}
        if kps:
            row["kernels_per_step"] = kps
        rows.append(row)
        print(json.dumps(row), flush=True)
    t1 = rows[0]["ms_per_step"] if rows[0]["parts"] == 1 else None
    for r in rows:
        r["efficiency_vs_1"] = (t1 / r["ms_per_step"]) if t1 else None
    out = {"workload": label, "elements": p.num_elements, "nodes": p.num_nodes, "halo": args.halo,
           "steps": args.steps, "warmup": args.warmup, "rows": rows,
           "timing": "wall clock around synchronous step(n) calls (one host sync per call), after warm-up"}
    sampler.stop()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({r["parts"]: round(r["efficiency_vs_1"] or 0, 3) for r in rows}))


if __name__ == "__main__":
    main()
