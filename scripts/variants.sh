#!/bin/bash
# Bench each built variant of libtvegpu (short runs, kernel times only).
mkdir -p gpurun_out
for v in "" ${VARIANTS:-}; do
  if [ -z "$v" ]; then lib=""; name=default; else lib=$PWD/paper_2009_10400_b200/lib/libtvegpu_$v.so; name=$v; fi
  TVEGPU_LIB=$lib python bench.py --steps 1000 --no-cpu-baseline --no-extras --e2e-steps 3 ${BENCH_ARGS:-} > gpurun_out/var_$name.log 2>&1
  python - "$name" <<'PY'
import json, sys
name = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/var_{name}.log").read().strip().splitlines()[-1])
    print(f"{name:10s} ms/step {d['ms_per_step']:.4f}  value {d['value']:.3e}  kernels " +
          " ".join(f"{k.split('<')[0][2:]}={v*1e3:.1f}us" for k, v in d["kernel_ms"].items()))
except Exception as e:
    print(name, "FAILED", open(f"gpurun_out/var_{name}.log").read()[-800:])
PY
done
