#!/bin/bash
# One gpurun session: GPU parity tests, smoke, bench, then the ncu launch list of a
# short bench command that has just exited 0 without ncu.
set -u
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/summary.txt
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/summary.txt
if [ "${NCU:-1}" = "1" ]; then
  CMD="python bench.py --steps 64 --warmup 3 --soak 0 --no-cpu-baseline --no-extras --e2e-steps 3"
  $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 60 --csv \
      --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
  echo "ncu launches rc=$?" >> gpurun_out/summary.txt
fi
tail -3 gpurun_out/pytest_gpu.log >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
