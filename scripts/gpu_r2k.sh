#!/bin/bash
# round 2: element kernels rebuilding the H8 geometry from the chunk coordinate block (K1 / K3 xstage) A/B
mkdir -p gpurun_out
ARMS="base:: k1x3:k1x3: k1x3m6:k1x3m6: k3x3:k3x3:" bash scripts/gpu_ab_env.sh > gpurun_out/ab_r2k.txt 2>&1
cat gpurun_out/ab_r2k.txt
