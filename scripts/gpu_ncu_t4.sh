#!/bin/bash
# ncu evidence for the T4 path: cfg5 Kuhn n=100 (6M elements), one launch of each step kernel
set -u
mkdir -p gpurun_out
TAG=${TAG:-r2}
CMD="python scripts/time_config.py cfg5_t4 100 128"
$CMD > gpurun_out/t4_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(mech|thermal)_(element|node)" -s 200 -c 40 --csv \
    --log-file gpurun_out/launches_${TAG}_cfg5_t4.csv $CMD > /dev/null 2>&1
echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_(mech|thermal)_(element|node)" -s 200 -c 4 \
    -o gpurun_out/prof_${TAG}_cfg5_t4 $CMD > gpurun_out/ncu_t4.log 2>&1
echo "ncu full rc=$?"
cat gpurun_out/t4_plain.log
