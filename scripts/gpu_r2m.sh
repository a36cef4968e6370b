#!/bin/bash
# round 2: PDL on the peer path; partitioned suite; per-rank timing of P-GPU partitions (projection)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_partitioned.py -x -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/r2m.txt
echo "partitioned rc=${PIPESTATUS[0]}" >> gpurun_out/r2m.txt
timeout 1500 python scripts/partition_solo.py --workload cfg5_16m --out gpurun_out/partition_solo_16m.json > gpurun_out/ps16.log 2>&1
timeout 900 python scripts/partition_solo.py --workload cfg4 --parts 2,4,8 --out gpurun_out/partition_solo_cfg4.json > gpurun_out/ps4.log 2>&1
cat gpurun_out/r2m.txt; tail -n 5 gpurun_out/ps16.log; tail -n 5 gpurun_out/ps4.log
