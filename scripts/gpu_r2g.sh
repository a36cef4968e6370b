#!/bin/bash
# round 2: K3 Hd/slot parking x element rows by TMA or L1 — parity subset (default build), A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py -x -q -p no:cacheprovider -m "gpu and not slow" 2>&1 | tail -3 > gpurun_out/gputest_r2g.log
echo "tests rc=${PIPESTATUS[0]}" >> gpurun_out/gputest_r2g.log
ARMS="nopark:nopark: park4tma:: notmap5:notmap5: notmanp:notmanp:" bash scripts/gpu_ab_env.sh > gpurun_out/ab_r2g.txt 2>&1
cat gpurun_out/gputest_r2g.log gpurun_out/ab_r2g.txt
