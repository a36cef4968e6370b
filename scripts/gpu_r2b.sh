#!/bin/bash
# round 2: GPU suite on the TMA-rows kernels, then A/B bench against the L1-prefetch variant
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_gpu_parity_large.py 2>&1 | tail -15 > gpurun_out/gputest_r2b.log
echo "tests rc=${PIPESTATUS[0]}" >> gpurun_out/gputest_r2b.log
LIBS="notma" bash scripts/ab_lib.sh > gpurun_out/ab_r2b.txt 2>&1
cat gpurun_out/gputest_r2b.log gpurun_out/ab_r2b.txt
