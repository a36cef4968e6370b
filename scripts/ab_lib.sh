#!/bin/bash
# A/B of build variants: LIBS="mw3 k3b2" benches lib/libtvegpu_<name>.so against the default
# library (kernel times only; csrc/Makefile `variant` target builds them).
mkdir -p gpurun_out
for n in default ${LIBS:-}; do
  if [ "$n" = default ]; then lib=""; else lib=paper_2009_10400_b200/lib/libtvegpu_$n.so; fi
  TVEGPU_LIB=$lib python bench.py --steps 1000 --no-cpu-baseline --no-extras --e2e-steps 3 ${BENCH_ARGS:-} > gpurun_out/abl_$n.log 2>&1
  python - "$n" <<'PY'
import json, sys
name = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/abl_{name}.log").read().strip().splitlines()[-1])
    print(f"{name:10s} ms/step {d['ms_per_step']:.4f}  e2e {d['e2e']['ms_per_step']:.3f}  kernels " +
          " ".join(f"{k.split('<')[0][2:]}={v*1e3:.1f}us" for k, v in d["kernel_ms"].items()))
except Exception as ex:
    print(name, "FAILED", open(f"gpurun_out/abl_{name}.log").read()[-800:])
PY
  for c in "cfg5_t4 100" cfg3; do TVEGPU_LIB=$lib python scripts/profile_config.py $c 2>&1 | tail -1; done
done
