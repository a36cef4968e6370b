#!/usr/bin/env python
"""Summarise an `ncu --set full` report and a `--metrics gpu__time_duration.sum`
launch list into profiles/: a markdown table per kernel and the per-launch DRAM
traffic JSON bench.py reports as roofline.traffic.

    python scripts/ncu_summary.py .ncu_reports/prof_r1a.ncu-rep gpurun_out/launches_r1a.csv r1 cfg4
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration [us]", 1e-3),
    ("dram__bytes_read.sum", "DRAM read [MB]", 1e-6),
    ("dram__bytes_write.sum", "DRAM write [MB]", 1e-6),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak", 1),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 %", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("smsp__inst_executed.sum", "warp-instr [M]", 1e-6),
]
KEY = {"k_thermal_element": "thermal_element", "k_thermal_node": "thermal_node", "k_mech_element": "mech_element",
       "k_mech_node": "mech_node"}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def num(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return float("nan")


def main(rep, launches, tag, workload):
    h, units, rows = raw_rows(rep)
    ki = h.index("Kernel Name")
    table, traffic = [], {}
    for r in rows:
        name = r[ki].split("(")[0].replace("void ", "").replace("tvegpu::", "")
        vals = {}
        for m, label, scale in METRICS:
            if m in h:
                v = num(r[h.index(m)])
                if m.startswith("dram__bytes"):  # ncu reports bytes in the unit row (MB/GB) -> normalise
                    u = units[h.index(m)]
                    v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
                elif m == "gpu__time_duration.sum":
                    u = units[h.index(m)]
                    v *= {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(u, 1)
                vals[label] = v * scale
        stalls = {c.split("issue_stalled_")[1].split("_per")[0]: num(r[i]) for i, c in enumerate(h)
                  if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
        vals["top stalls"] = ", ".join(f"{k} {v:.1f}" for k, v in top)
        table.append((name, vals))
        for pre, key in KEY.items():
            if name.startswith(pre):
                traffic[key] = vals["DRAM read [MB]"] * 1e6 + vals["DRAM write [MB]"] * 1e6
    # launch list: per-kernel share of the step
    shares = collections.defaultdict(list)
    if launches and os.path.exists(launches):
        lrows = [r for r in csv.reader(open(launches)) if len(r) > 10]
        i0 = next(i for i, r in enumerate(lrows) if "Kernel Name" in r)
        lh = lrows[i0]
        for r in lrows[i0 + 1:]:
            shares[r[lh.index("Kernel Name")].split("(")[0].replace("void ", "").replace("tvegpu::", "")].append(
                num(r[lh.index("Metric Value")]))
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    md = [f"# ncu summary {tag} — workload {workload}", "",
          f"Source: `{os.path.basename(rep)}` (`ncu --set full --clock-control none`, one launch per kernel after "
          "warm-up; times are cold-cache and serialised — compare shares, not absolutes).", ""]
    cols = [m[1] for m in METRICS] + ["top stalls"]
    md.append("| kernel | " + " | ".join(cols) + " |")
    md.append("|---" * (len(cols) + 1) + "|")
    for name, vals in table:
        md.append(f"| {name} | " + " | ".join(
            (f"{vals[c]:.1f}" if isinstance(vals.get(c), float) else str(vals.get(c, ""))) for c in cols) + " |")
    if shares:
        tot = sum(sum(v) for v in shares.values())
        md += ["", "Launch list (`--metrics gpu__time_duration.sum`): share of the measured step time", "",
               "| kernel | launches | mean [us] | share |", "|---|---|---|---|"]
        for k, v in sorted(shares.items(), key=lambda kv: -sum(kv[1])):
            md.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.3f} |")
    path = os.path.join(ROOT, "profiles", f"ncu_{tag}_{workload}.md")
    open(path, "w").write("\n".join(md) + "\n")
    jpath = os.path.join(ROOT, "profiles", "ncu_dram_bytes.json")
    data = json.load(open(jpath)) if os.path.exists(jpath) else {}
    data[workload] = {k: v for k, v in traffic.items()}
    data[workload]["_source"] = f"profiles/ncu_{tag}_{workload}.md (dram__bytes_read.sum + dram__bytes_write.sum)"
    json.dump(data, open(jpath, "w"), indent=1)
    print(open(path).read())


if __name__ == "__main__":
    main(*sys.argv[1:5])
