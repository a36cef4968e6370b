"""One rank's step of a P-GPU run, timed on one B200 (projected strong scaling).

For P in {1, 2, 4, 8}: every RCB partition of the mesh is created as rank r of P with no
NCCL id and stepped ALONE (tvegpu_peer_attach_solo: the peer-memory halo's stores go to
a local scratch buffer and the waits pass), with the bench's protocol: graph-replayed
steps, CUDA events on the engine stream, clocks sampled.  The slowest rank bounds the
P-GPU step; the halo transfer over NVLink is added as an estimate (bytes per step per
rank / 900 GB/s, NOT overlapped — a conservative bound: the step code overlaps it with
the interior chunks).  The results are a projection from one GPU, not a P-GPU
measurement.

    python scripts/partition_solo.py [--workload cfg5_16m|cfg4] [--parts 2,4,8]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2009_10400_b200 as tg
from bench import WORKLOADS, ClockSampler

NVLINK_GBS = 900.0  # B200 NVLink 5, per direction


def time_engine(eng, steps, warmup, sampler, soak=0.5):
    st = torch.cuda.ExternalStream(eng.stream)
    eng.step(warmup)
    t0 = time.time()  # keep the GPU busy until clocks settle (the bench's soak)
    while time.time() - t0 < soak:
        try:
            eng.step(32)
        except tg.TveError:
            break
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.time()
    a.record(st)
    eng.enqueue(steps)
    b.record(st)
    b.synchronize()
    w1 = time.time()
    try:
        eng.sync()
    except tg.TveError:
        pass  # solo partitions gather scratch halo values: their physics is not the point
    return a.elapsed_time(b) / steps, sampler.summary(w0, w1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg5_16m", choices=sorted(WORKLOADS))
    ap.add_argument("--parts", default="2,4,8")
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=32)
    ap.add_argument("--out", default="gpurun_out/partition_solo.json")
    args = ap.parse_args()
    label, make = WORKLOADS[args.workload]
    p = make(args.steps + args.warmup + 64)
    sampler = ClockSampler(0)
    e1 = tg.Engine(p)
    t1, c1 = time_engine(e1, args.steps, args.warmup, sampler)
    e1.close()
    del e1
    out = {"workload": label, "elements": p.num_elements, "one_gpu_ms": t1, "one_gpu_clocks": c1, "parts": []}
    print(json.dumps({"P": 1, "ms": t1}), flush=True)
    for P in [int(x) for x in args.parts.split(",")]:
        ranks = []
        for r in range(P):
            eng = tg.Engine(p, nranks=P, rank=r)
            eng.peer_attach_solo()
            ms, clk = time_engine(eng, args.steps, args.warmup, sampler)
            nb, sb, rb = eng.halo_info()
            ranks.append({"rank": r, "ms": ms, "kernels_per_step": eng.kernels_per_step(), "neighbors": nb,
                          "send_bytes": sb, "recv_bytes": rb, "clocks": clk})
            eng.close()
            del eng
            torch.cuda.empty_cache()
        worst = max(ranks, key=lambda x: x["ms"])
        xfer_ms = max(max(x["send_bytes"], x["recv_bytes"]) for x in ranks) / (NVLINK_GBS * 1e9) * 1e3
        proj = worst["ms"] + xfer_ms
        row = {"P": P, "ranks": ranks, "max_rank_ms": worst["ms"], "halo_transfer_ms_bound": xfer_ms,
               "projected_step_ms": proj, "projected_element_steps_per_s": p.num_elements / (proj / 1e3),
               "projected_efficiency": t1 / (P * proj)}
        out["parts"].append(row)
        print(json.dumps({k: v for k, v in row.items() if k != "ranks"}), flush=True)
    sampler.stop()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
