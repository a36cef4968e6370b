#!/bin/bash
# The bounds-checking build (TVEGPU_BOUNDS_CHECK=1: device asserts on every index the step
# kernels dereference) under the GPU test suite and the all-kernels driver.  Stands in for
# compute-sanitizer memcheck, which the GPU pool does not allow.
set -u
make -C paper_2009_10400_b200/csrc variant NAME=chk VFLAGS=-DTVEGPU_BOUNDS_CHECK=1 > /dev/null 2>&1 || \
  { [ -f paper_2009_10400_b200/lib/libtvegpu_chk.so ] || { echo "chk build failed"; exit 1; }; }
export TVEGPU_LIB=paper_2009_10400_b200/lib/libtvegpu_chk.so
timeout 1500 python -m pytest tests -m gpu -x -q -k "not slow" 2>&1 | tail -2
timeout 600 python scripts/sanitize_drive.py 2>&1 | tail -1
