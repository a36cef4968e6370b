#!/bin/bash
# round 2: partitioning overhead of the multi-GPU step on one device (peer and NCCL-copy halo paths)
mkdir -p gpurun_out
timeout 1200 python scripts/group_scaling.py --workload cfg5_16m --out gpurun_out/group_scaling_16m_peer.json > gpurun_out/gs1.log 2>&1
timeout 900 python scripts/group_scaling.py --workload cfg5_16m --halo nccl --parts 1,8 --out gpurun_out/group_scaling_16m_nccl.json > gpurun_out/gs2.log 2>&1
timeout 600 python scripts/group_scaling.py --workload cfg4 --out gpurun_out/group_scaling_cfg4_peer.json > gpurun_out/gs3.log 2>&1
tail -2 gpurun_out/gs1.log gpurun_out/gs2.log gpurun_out/gs3.log
