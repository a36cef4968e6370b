#!/bin/bash
# Full ncu capture of the step kernels on cfg4 (one launch each after warm-up).
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 64 --warmup 3 --soak 0 --no-cpu-baseline --no-extras --e2e-steps 3"
$CMD > gpurun_out/plain_full.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_(mech|thermal)_(element|node)" \
    -s 40 -c 4 -o gpurun_out/prof_${TAG:-r1} $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
tail -5 gpurun_out/ncu_full.log
