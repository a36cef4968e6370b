#!/bin/bash
# round 2: shared-memory carve-out A/B (one carve-out for all step kernels) x K3 parking
mkdir -p gpurun_out
ARMS="nopark:nopark: noparkC100:nopark:TVEGPU_CARVEOUT=100 noparkC44:nopark:TVEGPU_CARVEOUT=44 park4C100:park4:TVEGPU_CARVEOUT=100 park5C100::TVEGPU_CARVEOUT=100" bash scripts/gpu_ab_env.sh > gpurun_out/ab_r2f.txt 2>&1
cat gpurun_out/ab_r2f.txt
