#!/bin/bash
# The GPU parity suite (non-slow) under every runtime switch and the main build variants
# (INTEGRATION.md §8): results may change only within the documented tolerance.
L=paper_2009_10400_b200/lib
declare -A FLAGS=([geo0]=-DTVEGPU_GEO=0 [mw4]=-DTVEGPU_MW=4 [ch64]=-DTVEGPU_CHUNK=64 [ch256]=-DTVEGPU_CHUNK=256)
for v in geo0 mw4 ch64 ch256; do
  [ -f $L/libtvegpu_$v.so ] || make -C paper_2009_10400_b200/csrc variant NAME=$v VFLAGS=${FLAGS[$v]} > /dev/null 2>&1 \
    || { echo "$v: build failed"; continue; }
  echo "$v: $(TVEGPU_LIB=$L/libtvegpu_$v.so timeout 900 python -m pytest tests -m gpu -q -x -k 'not slow' 2>&1 | tail -1)"
done
for e in TVEGPU_NO_PDL=1 TVEGPU_NO_ELL=1 TVEGPU_NO_PAIR=1; do
  echo "$e: $(env $e timeout 900 python -m pytest tests -m gpu -q -x -k 'not slow' 2>&1 | tail -1)"
done
