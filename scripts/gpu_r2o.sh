#!/bin/bash
# round 2: early vs late PDL trigger (A/B, cfg4 + cfg3), parity subset on the early build
mkdir -p gpurun_out
ARMS="late:: early:early:" bash scripts/gpu_ab_env.sh > gpurun_out/ab_r2o.txt 2>&1
for l in "" early; do for c in cfg3 "cfg5_h8 252"; do TVEGPU_LIB=${l:+paper_2009_10400_b200/lib/libtvegpu_$l.so} python scripts/time_config.py $c; done; done >> gpurun_out/ab_r2o.txt 2>&1
TVEGPU_LIB=paper_2009_10400_b200/lib/libtvegpu_early.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py -x -q -p no:cacheprovider -m "gpu and not slow" 2>&1 | tail -1 >> gpurun_out/ab_r2o.txt
cat gpurun_out/ab_r2o.txt
