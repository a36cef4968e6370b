#!/bin/bash
# One gpurun session producing the round's evidence: full GPU test suite (incl. slow),
# the default bench line, the reference arm, an ncu launch list and one --set full capture.
set -u
mkdir -p gpurun_out
TAG=${TAG:-r1}
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -s -rs --durations=25 > gpurun_out/pytest_gpu_all.log 2>&1; echo "pytest all rc=$?" >> gpurun_out/summary.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/summary.txt
timeout 900 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?" >> gpurun_out/summary.txt
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref_${TAG}.log 2>&1; echo "bench ref rc=$?" >> gpurun_out/summary.txt
CMD="python bench.py --steps 64 --warmup 3 --soak 0 --no-cpu-baseline --no-extras --e2e-steps 3 --no-ncu-traffic --single-budget 0"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 80 --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/summary.txt
$CMD > gpurun_out/plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_(mech|thermal)_(element|node)" -s 40 -c 4 \
    -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/pytest_gpu_all.log >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
timeout 900 python scripts/partition_solo.py --workload cfg4 --out gpurun_out/partition_solo_${TAG}_cfg4.json > gpurun_out/ps_cfg4.log 2>&1; echo "partition solo cfg4 rc=$?" >> gpurun_out/summary.txt
