#!/bin/bash
# round 2: K3 register parking in shared memory (5 CTAs/SM) — parity subset, then A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py -x -q -p no:cacheprovider -m "gpu and not slow" 2>&1 | tail -5 > gpurun_out/gputest_r2e.log
echo "tests rc=${PIPESTATUS[0]}" >> gpurun_out/gputest_r2e.log
ARMS="nopark:nopark: park5:: park4:park4:" bash scripts/gpu_ab_env.sh > gpurun_out/ab_r2e.txt 2>&1
cat gpurun_out/gputest_r2e.log gpurun_out/ab_r2e.txt
