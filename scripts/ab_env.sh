#!/bin/bash
# A/B of the default library under environment toggles: ENVS="A=1 B=1" runs one bench
# per toggle (plus the plain default), kernel times only.
mkdir -p gpurun_out
for e in "" ${ENVS:-}; do
  name=${e:-default}
  env $e python bench.py --steps 1000 --no-cpu-baseline --no-extras --e2e-steps 3 ${BENCH_ARGS:-} > gpurun_out/ab_$name.log 2>&1
  python - "$name" <<'PY'
import json, sys
name = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{name}.log").read().strip().splitlines()[-1])
    print(f"{name:22s} ms/step {d['ms_per_step']:.4f}  e2e {d['e2e']['ms_per_step']:.3f}  kernels " +
          " ".join(f"{k.split('<')[0][2:]}={v*1e3:.1f}us" for k, v in d["kernel_ms"].items()))
except Exception as ex:
    print(name, "FAILED", open(f"gpurun_out/ab_{name}.log").read()[-800:])
PY
done
