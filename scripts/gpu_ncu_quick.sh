#!/bin/bash
# Quick ncu metric capture (a few launches of each step kernel) of a short bench run.
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 64 --warmup 3 --soak 0 --no-cpu-baseline --no-extras --e2e-steps 3"
METRICS=${METRICS:-gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__sass_inst_executed_op_shared_ld.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum}
$CMD > gpurun_out/plain_quick.log 2>&1 && \
timeout 900 ncu --metrics $METRICS --clock-control none -k regex:"k_(mech|thermal)_(element|node)" -s 40 -c 4 --csv $CMD > gpurun_out/ncu_quick.csv 2> gpurun_out/ncu_quick.err
echo "ncu quick rc=$?"
python3 - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/ncu_quick.csv")) if len(r) > 10]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
for r in rows[1:]:
    print(f"{r[ki][:28]:28s} {r[mi][:60]:60s} {r[vi]}")
PY
