# round 2 (final code): size ladder with clock records, and the 16M partition projection
mkdir -p gpurun_out
timeout 2400 python scripts/ladder.py --steps 100 --out gpurun_out/ladder_r2v.json > gpurun_out/ladder_r2v.log 2>&1; echo "ladder rc=$?"
timeout 1500 python scripts/partition_solo.py --workload cfg5_16m --out gpurun_out/partition_solo_r2v_16m.json > gpurun_out/ps16_r2v.log 2>&1; echo "ps16 rc=$?"
tail -3 gpurun_out/ladder_r2v.log; tail -3 gpurun_out/ps16_r2v.log
