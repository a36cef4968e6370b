#!/usr/bin/env python
"""Benchmark of the coupled TLED time step (BASELINE.json metric: element-steps/s,
achieved HBM GB/s, ms per explicit step).

Workload at N=1: cfg4 (BASELINE configs[3]) — H8 block 100^3 = 1,000,000 elements,
1,030,301 nodes, coupled TherMechExpanTD (temperature-dependent c/k, isotropic
thermal expansion), hourglass control, one Prony term, central RFA source.  It is
the configuration the north_star's >= 60 % HBM-roofline target is stated on.
At N>1 (torchrun, one rank per GPU): strong scaling of the fixed 16M-element H8 mesh
(BASELINE configs[4], cfg5 H8 252^3) split by RCB into N partitions with the NCCL halo
exchange overlapped with the interior elements; --workload cfg4 runs
configs[3] at N GPUs instead.  Each rank reports its halo volume and exchange time.

--impl reference: the reference's algorithm on the host CPU (the fp64 oracle,
OpenMP over all host threads) on the same workload — the reference ships no
runnable code, so the oracle restatement is its CPU implementation.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2009_10400_b200 import configs  # noqa: E402
from paper_2009_10400_b200.problem import H8  # noqa: E402

METRIC = "element-steps/s"


WORKLOADS = {
    # BASELINE configs[3]: the N = 1 headline and the 2-GPU cfg4 point
    "cfg4": ("cfg4: H8 100^3 (1,000,000 el) TherMechExpanTD, hourglass, Prony P=1",
             lambda steps: configs.cfg4(steps=steps)),
    # BASELINE configs[4] top rung: the fixed 16M-element mesh strong-scaled over 1/2/4/8 GPUs
    "cfg5_16m": ("cfg5: H8 252^3 (16,003,008 el) TherMechExpanTD, hourglass, Prony P=1, dt = 1/2 critical",
                 lambda steps: configs.cfg5_h8(252, steps=steps)),
}


def workload_for(args, world):
    """N = 1: cfg4 (the metric's configuration).  N > 1: the fixed 16M-element mesh split
    by RCB over the N GPUs (strong scaling), or --workload cfg4."""
    name = args.workload or ("cfg4" if world == 1 else "cfg5_16m")
    label, make = WORKLOADS[name]
    return name, label, make


def bench_config(name, label, p, world, graph_steps):
    """The config dict both arms print (identical for the same workload and N)."""
    return {"workload": label, "elements": p.num_elements, "nodes": p.num_nodes,
            "parallelism": f"rcb{world}" if world > 1 else "single",
            "l2": "working set > 1 GB per GPU vs 126 MB L2: no flush needed",
            "graph_steps": graph_steps, "name": name}


def canonical_bytes(p):
    """SURVEY.md §8(d) algorithmic bytes per launch of each kernel (fp64 values, int32 indices)."""
    E, N, nn, P = p.num_elements, p.num_nodes, p.nn, p.prony_count
    fib = 24 if p.fiber_dirs is not None else 0
    axes = 48 if p.expansion_axes is not None else 0
    hasR = p.external_force is not None or any(b != 0 for b in p.body_force)
    return {
        "thermal_element": E * (12 * nn + 80) + N * 32,
        "thermal_node": E * 12 * nn + N * 37,
        "mech_element": E * (28 * nn + 80 + 96 * P + fib + axes) + N * (32 + (24 if p.kind == H8 else 0)),
        "mech_node": E * 28 * nn + N * (85 + (24 if hasR else 0)),
    }


def lumped_source_power(p):
    """accumulate_nodal_sources (bioheat.hpp:65-69) in numpy: q_r V_e / nn to each node."""
    X = p.nodes[p.elements]
    if p.kind == H8:
        s = np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                      [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], float)
        V = 8.0 * np.linalg.det(np.einsum("eai,aj->eij", X, s) / 8.0)
    else:
        V = np.linalg.det(np.stack([X[:, 1] - X[:, 0], X[:, 2] - X[:, 0], X[:, 3] - X[:, 0]], axis=2)) / 6.0
    q = np.zeros(p.num_nodes)
    for r in p.sources:
        for a in range(p.nn):
            np.add.at(q, p.elements[r.elements, a], r.q_r * V[r.elements] / p.nn)
    return q


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


KERNEL_REGEX = {"thermal_element": "k_thermal_element", "thermal_node": "k_thermal_node",
                "mech_element": "k_mech_element", "mech_node": "k_mech_node"}
_UNITS = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "kib": 1024, "mib": 1024 ** 2, "gib": 1024 ** 3}


def ncu_traffic_live(args, kernel, timeout_s=300):
    """DRAM bytes of ONE launch of `kernel`, measured in this bench run: ncu (dram__bytes_read.sum
    + dram__bytes_write.sum, cache flushed before the launch as in a --set full capture) on a
    short probe of the same workload (`bench.py --traffic-probe`), after the probe's own warm-up
    steps.  A byte count, not a time: the bench's timings never run under the profiler.
    Returns (bytes, note) or (None, why)."""
    import shutil
    ncu = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu" if os.path.exists("/usr/local/cuda/bin/ncu") else None)
    if ncu is None:
        return None, "ncu not found"
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control", "none",
           "-k", f"regex:{KERNEL_REGEX[kernel]}", "-s", "6", "-c", "1", "--csv",
           sys.executable, os.path.join(ROOT, "bench.py"), "--traffic-probe"]
    if args.workload:
        cmd += ["--workload", args.workload]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s, cwd=ROOT)
    except Exception as ex:  # noqa: BLE001
        return None, f"ncu probe failed: {type(ex).__name__}"
    import csv
    import io
    tot, seen = 0.0, set()
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith('"')]
    try:
        rows = list(csv.reader(io.StringIO("\n".join(lines))))
        h = rows[0]
        im, iu, iv = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
        for row in rows[1:]:
            if row[im] in ("dram__bytes_read.sum", "dram__bytes_write.sum") and row[im] not in seen:
                seen.add(row[im])
                tot += float(row[iv].replace(",", "")) * _UNITS.get(row[iu].strip().lower(), float("nan"))
    except Exception:  # noqa: BLE001
        return None, "ncu probe output not parsed (rc %d): %s" % (r.returncode, (r.stderr or r.stdout)[-200:])
    if len(seen) != 2 or not math.isfinite(tot):
        return None, "ncu probe: metrics missing (rc %d)" % r.returncode
    return tot, "measured in this run: ncu dram__bytes_read.sum + dram__bytes_write.sum of one launch"


def traffic_probe(args):
    """--traffic-probe: the bench workload, a few direct steps (the ncu pass in ncu_traffic_live)."""
    import paper_2009_10400_b200 as tg
    _, _, make = workload_for(args, 1)
    eng = tg.Engine(make(64), steps_per_graph=1)
    eng.step(8)
    eng.close()
    return 0


def ncu_traffic(workload_key, kernel):
    """dram bytes per launch from a committed `ncu --set full` capture (profiles/ncu_dram_bytes.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_dram_bytes.json")) as f:
            return json.load(f).get(workload_key, {}).get(kernel)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 100 ms while the bench runs."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id):
        self.rows = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(gpu_id)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), line.strip()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0, t1):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sel = [r for t, r in self.rows if t0 - 0.15 <= t <= t1 + 0.15] or [r for _, r in self.rows[-5:]]
        sm, smax, reasons = [], [], set()
        for r in sel:
            parts = [x.strip() for x in r.split(",")]
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
                for n, v in zip(names, parts[4:8]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
            except Exception:
                continue
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_oracle_rate(problem, budget_s, max_steps, warmup=1, threads=None):
    """Element-steps/s of the fp64 oracle (OpenMP, all host threads unless `threads`) on the same problem."""
    from oracle import oracle as O
    threads = threads or os.cpu_count() or 1
    o = O.OracleEngine(problem, workers=threads)
    o.step(warmup)
    t0 = time.perf_counter()
    n = 0
    while n < max_steps:
        o.step(1)
        n += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return problem.num_elements * n / dt, n, dt, threads


def single_thread_rate(problem, budget_s):
    """BASELINE.md §3 asks for the CPU baseline at all host threads and also at 1: the
    same oracle on one thread, a bounded sample (informational beside the main figure)."""
    if budget_s <= 0:
        return None
    rate, n, dt, _ = cpu_oracle_rate(problem, budget_s=budget_s, max_steps=1000, warmup=1, threads=1)
    return {"value": rate, "unit": METRIC, "cores": 1, "steps": n, "seconds": dt}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    name, label, make = workload_for(args, world)
    p = make(args.steps)
    warm = max(1, min(args.warmup, 10))  # ~0.1 s per CPU step on cfg4: bounded, >= 3 when asked for >= 3
    rate, n, dt, threads = cpu_oracle_rate(p, budget_s=args.ref_budget, max_steps=args.steps, warmup=warm)
    sample = (f"{n} of {args.steps} requested steps of the full {p.num_elements:,}-element workload "
              f"({dt:.1f} s, fp64 oracle, OpenMP {threads} threads on {cpu_model()})")
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": METRIC, "n_gpus": world,
            "steps": n, "warmup": warm, "ms_per_step": 1e3 * dt / n, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(name, label, p, world, args.graph_steps),
            "cpu_baseline": {"value": rate, "unit": METRIC, "cores": threads, "kind": "port", "sample": sample,
                             "single_thread": single_thread_rate(p, args.single_budget)},
            "e2e": {"value": rate, "unit": METRIC, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import paper_2009_10400_b200 as tg

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"bench.py --gpus {args.gpus} needs {args.gpus} ranks (torchrun --nproc-per-node "
                         f"{args.gpus}); this process group has {world}")
    if world > torch.cuda.device_count():
        raise SystemExit(f"--gpus {world}: only {torch.cuda.device_count()} CUDA device(s) visible")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        # a halo wait that cannot complete fails the run in seconds instead of stalling it
        os.environ.setdefault("TVEGPU_HALO_TIMEOUT_MS", "5000")
        # communicator-init lines (rank count) of the halo communicator and torch's
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wname, workload, make = workload_for(args, world)
    p = make(args.steps + args.warmup + 64)
    nccl_id = None
    if world > 1:
        obj = [tg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    eng = tg.Engine(p, device=local, nranks=world, rank=rank, nccl_id=nccl_id, steps_per_graph=args.graph_steps)
    halo_transport = None
    if world > 1:
        # peer-memory halo: all-gather the partitions' descriptors (CUDA IPC handles of the
        # receive areas + flag inboxes), attach; the boundary element kernels then store the
        # interface contributions straight into the neighbours' memory over NVLink.
        # TVEGPU_HALO=nccl keeps the pack + ncclSend/ncclRecv path.
        halo_transport = "nccl"
        if os.environ.get("TVEGPU_HALO", "peer") != "nccl":
            blobs = [None] * world
            dist.all_gather_object(blobs, eng.peer_export())
            ok = 1
            try:
                eng.peer_attach(blobs)
            except Exception as ex:  # noqa: BLE001 — e.g. no peer access between these GPUs
                print(f"rank {rank}: peer-memory halo unavailable ({ex}); NCCL halo", file=sys.stderr)
                ok = 0
            t = torch.tensor([ok], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            if int(t.item()) == 1:
                halo_transport = "peer"
            elif eng.halo_peer:  # every rank must step with the same transport
                eng.peer_detach()
    stream = torch.cuda.ExternalStream(eng.stream, device=local)
    props = torch.cuda.get_device_properties(local)
    sampler = ClockSampler(getattr(props, "uuid", None) and f"GPU-{props.uuid}" or local)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up: W steps, then keep the GPU busy ~0.5 s so clocks settle (untimed)
    eng.step(args.warmup)
    t_soak = time.time()
    while time.time() - t_soak < args.soak:
        eng.step(args.graph_steps)
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    wall0 = time.time()
    ev0.record(stream)
    eng.enqueue(args.steps)
    ev1.record(stream)
    ev1.synchronize()
    wall1 = time.time()
    eng.sync()  # finite check of the timed steps (raises on instability)
    barrier()
    ms = ev0.elapsed_time(ev1)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clocks = sampler.summary(wall0, wall1)
    sampler.stop()
    E_total = p.num_elements  # the whole mesh (split over the ranks)
    value = E_total * args.steps / (ms / 1e3)
    ms_step = ms / args.steps

    # per-kernel durations (CUDA events on the engine stream, direct launches)
    prof = eng.profile_kernels(min(args.steps, 50))
    local_bytes = canonical_bytes(p)
    kname = {"thermal_element": "k_thermal_element", "thermal_node": "k_thermal_node",
             "mech_element": "k_mech_element", "mech_node": "k_mech_node"}
    per_kernel = {}
    for k, b in local_bytes.items():
        for n, t in prof.items():
            if n.startswith(kname[k]):
                per_kernel[k] = (b / world, t)
    dom = max(per_kernel, key=lambda k: per_kernel[k][1])
    b_dom, t_dom = per_kernel[dom]
    peak, peak_src = load_peaks()
    ach = b_dom / (t_dom / 1e3) / 1e9
    step_bytes = sum(local_bytes.values())
    step_gbs = step_bytes * args.steps / (ms / 1e3) / 1e9
    wkey = wname if world == 1 else f"{wname}_n{world}"
    traffic, tsrc = (None, "skipped (--no-ncu-traffic)")
    if rank == 0 and world == 1 and not args.no_ncu_traffic:
        traffic, tsrc = ncu_traffic_live(args, dom)
    if traffic is None:  # fall back to the committed capture, saying so
        traffic = ncu_traffic(wkey, dom)
        tsrc = (f"{tsrc}; profiles/ncu_dram_bytes.json (dram__bytes_read.sum + dram__bytes_write.sum of the "
                f"committed ncu --set full capture of this workload)")
    roofline = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": traffic, "kernel": dom, "kernel_ms": t_dom,
                "algorithmic_bytes_per_launch": b_dom, "peak_source": peak_src, "traffic_source": tsrc}
    halo = None
    if world > 1:  # per rank: halo volume and the transfer time on the comm stream
        nb, sb, rb = eng.halo_info()
        mine = [float(nb), float(sb), float(rb), 1e3 * prof.get("halo_exchange_thermal", 0.0),
                1e3 * prof.get("halo_exchange_mech", 0.0), float(eng.problem.num_elements)]
        t = torch.tensor(mine, device="cuda", dtype=torch.float64)
        allr = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(allr, t)
        halo = [{"rank": r, "neighbors": int(v[0]), "send_bytes_per_step": int(v[1]), "recv_bytes_per_step": int(v[2]),
                 "exchange_us_thermal": v[3], "exchange_us_mech": v[4]} for r, v in
                enumerate(x.tolist() for x in allr)]

    # end to end through the public API with host buffers: per step upload this step's
    # nodal source powers (pinned H2D, bioheat.hpp:57), step (finite check D2H), read T and u (D2H)
    e2e_steps = max(3, min(args.steps, args.e2e_steps))
    # pinned host buffers (the contract's "from pinned host memory"); the power vector is
    # the lumped regional source, re-sent every step as a generator control loop would
    power = torch.from_numpy(lumped_source_power(p)).pin_memory().numpy()
    Th = torch.empty(p.num_nodes, dtype=torch.float64, pin_memory=True).numpy()
    uh = torch.empty(3 * p.num_nodes, dtype=torch.float64, pin_memory=True).numpy()
    # untimed: first-call allocations (device I/O buffers); the first few dozen DMA
    # reads of a freshly pinned buffer run ~2x slower (measured, scripts/e2e_breakdown.py)
    for k in range(200):  # ~0.2 s; a fresh box's first pinned transfers run slower for longer
        eng.step_io(power, 1, Th, uh)
    barrier()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        eng.step_io(power, 1, Th, uh)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": E_total * e2e_steps / e2e_s, "unit": METRIC, "ms_per_step": 1e3 * e2e_s / e2e_steps,
           "h2d_bytes_per_step": 8 * p.num_nodes, "d2h_bytes_per_step": 32 * p.num_nodes + 40,
           "steps": e2e_steps,
           "calls": "tvegpu_step_io(power, 1, T, u): source upload + 1 step + T/u read-back (C ABI, pinned host "
                    "buffers, copies overlapped with the step on a side stream)"}

    # informational: the closed control loop a thermal-ablation controller runs — upload the
    # source powers, step, read back the RunSummary (T_max, displacement extrema; 56 B)
    for k in range(20):
        eng.step_io(power, 1)
        eng.summary()
    barrier()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        eng.step_io(power, 1)
        eng.summary()
    torch.cuda.synchronize()
    ctl_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([ctl_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ctl_s = float(t.item())
    e2e_control = {"value": E_total * e2e_steps / ctl_s, "unit": METRIC, "ms_per_step": 1e3 * ctl_s / e2e_steps,
                   "h2d_bytes_per_step": 8 * p.num_nodes, "d2h_bytes_per_step": 56 + 40, "steps": e2e_steps,
                   "calls": "tvegpu_step_io(power, 1, NULL, NULL) + tvegpu_get_summary (device reductions)"}

    line = {"metric": METRIC, "value": value, "unit": METRIC, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(wname, workload, p, world, args.graph_steps),
            "achieved_hbm_gbs_step": step_gbs, "canonical_bytes_per_element_step": step_bytes / p.num_elements,
            "step_roofline_frac": step_gbs / peak,
            "kernel_ms": prof, "roofline": roofline, "e2e": e2e, "e2e_control": e2e_control,
            "gpu_launches": eng.kernels_per_step() * args.steps, "clocks": clocks}
    if halo is not None:
        line["halo"] = halo
        line["halo_transport"] = halo_transport

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, n, dt, threads = cpu_oracle_rate(p, budget_s=args.cpu_budget, max_steps=1000)
        line["cpu_baseline"] = {"value": rate, "unit": METRIC, "cores": threads, "kind": "port",
                                "sample": f"{n} steps of the full cfg4 mesh in {dt:.1f} s (fp64 oracle, OpenMP "
                                          f"{threads} threads, {cpu_model()})",
                                "single_thread": single_thread_rate(p, args.single_budget)}
    if rank == 0 and world == 1 and not args.no_extras:
        # the other BASELINE configurations on one GPU (not the headline; ms per step, per-kernel split)
        def side(p, n_steps, regime, slot_fp32=False):
            e = tg.Engine(p, device=local, steps_per_graph=args.graph_steps, slot_fp32=slot_fp32)
            e.step(200)
            dev = None
            if slot_fp32:  # deviation from the fp64 engine after the same 200 steps
                ref = tg.Engine(p, device=local, steps_per_graph=args.graph_steps)
                ref.step(200)
                a, b = e.state(), ref.state()
                ref.close()
                dev = {"u": float(np.abs(a["u"] - b["u"]).max() / max(np.abs(b["u"]).max(), 1e-300)),
                       "T": float(np.abs(a["T"] - b["T"]).max() /
                                  max(np.abs(b["T"] - p.initial_temperature).max(), 1e-300)),
                       "steps": 200, "measure": "increment-relative vs the fp64 engine"}
            st = torch.cuda.ExternalStream(e.stream, device=local)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            e.enqueue(n_steps)
            b.record(st)
            b.synchronize()
            e.sync()
            t = a.elapsed_time(b) / n_steps
            by = sum(canonical_bytes(p).values())
            pk = e.profile_kernels(100)
            e.close()
            return {"elements": p.num_elements, "nodes": p.num_nodes, "ms_per_step": t,
                    "element_steps_per_s": p.num_elements / (t / 1e3), "steps": n_steps,
                    "canonical_bytes_per_step": by, "achieved_gbs": by / (t / 1e3) / 1e9,
                    "hbm_frac": by / (t / 1e3) / 1e9 / peak, "regime": regime,
                    "kernel_us_direct_launches": {k: 1e3 * v for k, v in pk.items()},
                    "launch_overhead_us": 1e3 * (sum(pk.values()) - t),
                    **({"deviation_from_fp64": dev} if dev else {})}
        l2 = ("L2-resident: the step's canonical traffic fits the 126 MB L2, so the fraction can exceed 1; "
              "four launches of a few us each")
        # configs[2], the real-time target: liver-shaped T4 (~100k el), 3 RFA sources, perfusion
        p3 = configs.cfg3(steps=100000)
        line["cfg3_liver"] = side(p3, 2000, l2)
        line["cfg3_liver"]["realtime_dt_ms"] = 1e3 * p3.dt
        line["cfg3_liver"]["hbm_frac_l2_regime"] = line["cfg3_liver"]["hbm_frac"]
        # configs[1]: T4 Kuhn n=20 (48k el), per-element helical fibres, temperature-dependent
        line["cfg2_t4_fibres"] = side(configs.cfg2(steps=100000), 2000, l2)
        # configs[3] with the anisotropic expansion class (orthotropic, per-element axes): the
        # K3 variant with the most register pressure (EXP = 2)
        p4o = configs.cfg4(steps=args.steps + 400)
        p4o.expansion = dict(kind=2, alpha_i=1e-4, alpha_m=3e-4, alpha_n=-5e-5, reference_temperature=37.0)
        rng = np.random.default_rng(5)
        Q = np.linalg.qr(rng.normal(size=(p4o.num_elements, 3, 3)))[0]
        p4o.expansion_axes = np.concatenate([Q[:, :, 0], Q[:, :, 1]], axis=1)
        line["cfg4_orthotropic_axes"] = side(p4o, 400, "working set > L2 (HBM-bound)")
        # configs[3] with every node jittered by up to 5 % of the spacing: no element is affine,
        # so K3 stages and reads the hourglass geometry (the general H8 path; the structured
        # headline cube takes the affine fast path, as voxel-derived hex meshes do)
        p4j = configs.cfg4(steps=args.steps + 400)
        h = 0.1 / 100
        p4j.nodes = p4j.nodes + np.random.default_rng(6).uniform(-0.05 * h, 0.05 * h, p4j.nodes.shape)
        line["cfg4_jittered_general_h8"] = side(p4j, 400, "working set > L2 (HBM-bound)")
        # the optional mixed-precision mode (tvegpu_options.slot_fp32: fp32 contributions
        # between the fp64 element and node kernels) on the headline workload, with its
        # deviation from the fp64 engine after 200 steps (not the headline: dtype stays f64)
        line["cfg4_fp32_slots"] = side(p, 400, "working set > L2 (HBM-bound)", slot_fp32=True)
    if rank == 0:
        print(json.dumps(line), flush=True)
    eng.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: cfg4 at N = 1, the 16M-element cfg5 mesh at N > 1")
    ap.add_argument("--graph-steps", type=int, default=64)
    ap.add_argument("--soak", type=float, default=0.5)
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-budget", type=float, default=90.0)
    ap.add_argument("--single-budget", type=float, default=8.0, help="seconds of the 1-thread CPU sample (0: skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-ncu-traffic", action="store_true", help="roofline.traffic from the committed capture")
    ap.add_argument("--traffic-probe", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.traffic_probe:
        return traffic_probe(args)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    return run_reference(args) if args.impl == "reference" else run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
