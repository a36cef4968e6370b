#!/bin/bash
# round 2: node-major chunk slot blocks — parity subset, then A/B against the previous kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py -x -q -p no:cacheprovider -m "gpu and not slow" 2>&1 | tail -5 > gpurun_out/gputest_r2d.log
echo "tests rc=${PIPESTATUS[0]}" >> gpurun_out/gputest_r2d.log
ARMS="base:base: nmaj:: emaj::TVEGPU_NODE_MAJOR=0 k1mb6:k1mb6:" bash scripts/gpu_ab_env.sh > gpurun_out/ab_r2d.txt 2>&1
for c in "cfg5_t4 100" cfg3; do for l in base ""; do TVEGPU_LIB=${l:+paper_2009_10400_b200/lib/libtvegpu_$l.so} python scripts/profile_config.py $c 2>&1 | tail -1; done; done >> gpurun_out/ab_r2d.txt
cat gpurun_out/gputest_r2d.log gpurun_out/ab_r2d.txt
