#!/bin/bash
# round 2: peer-memory halo (SEND element kernels + device flags) — partitioned suite, parity subset, bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_partitioned.py -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/gputest_r2i.log
echo "partitioned rc=${PIPESTATUS[0]}" >> gpurun_out/gputest_r2i.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -m "gpu and not slow" 2>&1 | tail -3 >> gpurun_out/gputest_r2i.log
python bench.py --steps 1000 --no-cpu-baseline --no-extras --no-ncu-traffic --single-budget 0 --e2e-steps 20 2>&1 | tail -1 | cut -c1-400 >> gpurun_out/gputest_r2i.log
cat gpurun_out/gputest_r2i.log
