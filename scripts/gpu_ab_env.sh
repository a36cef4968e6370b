#!/bin/bash
# A/B of environment settings on cfg4: ENVS="A=1 B=2" (each run alone), LIB=<variant or empty>
mkdir -p gpurun_out
for rep in 1 2; do
for e in default ${ENVS}; do
  if [ "$e" = default ]; then envs=""; else envs="$e"; fi
  if [ "${e%%=*}" = LIB ]; then lib=paper_2009_10400_b200/lib/libtvegpu_${e#LIB=}.so; envs=""; else lib=""; fi
  env $envs TVEGPU_LIB=$lib python bench.py --steps 1000 --no-cpu-baseline --no-extras --e2e-steps 3 > gpurun_out/abe.log 2>&1
  python - "$e" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/abe.log").read().strip().splitlines()[-1])
    print(f"{sys.argv[1]:24s} ms/step {d['ms_per_step']:.4f}  kernels " +
          " ".join(f"{k.split('<')[0][2:]}={v*1e3:.1f}us" for k, v in d["kernel_ms"].items()) + f"  clk {d['clocks']['sm_mhz']}")
except Exception as ex:
    print(sys.argv[1], "FAILED", open("gpurun_out/abe.log").read()[-600:])
PY
done
done
