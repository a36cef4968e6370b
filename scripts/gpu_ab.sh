#!/bin/bash
# A/B of build variants on cfg4 (graph-replayed step + per-kernel event times): LIBS="a b"
mkdir -p gpurun_out
for rep in 1 2; do
LIBS="${LIBS}" bash scripts/ab_lib.sh 2>&1 | grep -v "^cfg5\|^cfg3" 
done
