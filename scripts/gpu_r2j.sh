#!/bin/bash
# round 2: bench with the side configurations, then the size ladder (H8 1M..16M, T4 1M..16.1M)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r2j.log 2>&1; echo "bench rc=$?" > gpurun_out/r2j.txt
timeout 2400 python scripts/ladder.py --steps 100 --out gpurun_out/ladder_r2.json > gpurun_out/ladder_r2.log 2>&1; echo "ladder rc=$?" >> gpurun_out/r2j.txt
cat gpurun_out/r2j.txt; tail -3 gpurun_out/ladder_r2.log
