#!/bin/bash
# A/B of library variants and environment settings on cfg4 (graph-replayed step + per-kernel
# event times).  ARMS="name:lib:ENV=VAL,ENV2=VAL ..." (lib empty = default library).
mkdir -p gpurun_out
for rep in ${REPS:-1 2}; do
  for arm in ${ARMS}; do
    IFS=: read -r name lib envs <<< "$arm"
    [ -n "$lib" ] && lib=paper_2009_10400_b200/lib/libtvegpu_$lib.so
    env TVEGPU_LIB=$lib ${envs//,/ } python bench.py --steps 1000 --no-cpu-baseline --no-extras --e2e-steps 20 \
        ${BENCH_ARGS:-} > gpurun_out/abe_$name.log 2>&1
    python - "$name" <<'PY'
import json, sys
name = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/abe_{name}.log").read().strip().splitlines()[-1])
    print(f"{name:12s} ms/step {d['ms_per_step']:.4f}  e2e {d['e2e']['ms_per_step']:.3f}  kernels " +
          " ".join(f"{k.split('<')[0][2:]}={v*1e3:.1f}us" for k, v in d["kernel_ms"].items()) +
          f"  sm {d['clocks']['sm_mhz']}")
except Exception as ex:
    print(name, "FAILED", open(f"gpurun_out/abe_{name}.log").read()[-800:])
PY
  done
done
