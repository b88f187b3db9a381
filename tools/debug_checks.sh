#!/bin/bash
# Device-assert build (SDNN_DEBUG_CHECKS=1) + the GPU parity tests that reach
# every pass kernel variant, in place of compute-sanitizer (closed on the pool).
#   gpurun --timeout 1800 -- 'bash tools/debug_checks.sh'
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
L=$PWD/paper_2004_10908_b200/libsdnn_dbg.so
[ -f "$L" ] || SDNN_LIB=$L SDNN_NVCC_FLAGS="-DSDNN_DEBUG_CHECKS=1" python -m paper_2004_10908_b200.build
SDNN_LIB=$L timeout 1500 python -m pytest tests/test_gpu_parity.py -q -k "c1_full or fused or large_caps or knob or full_size_c2 or full_size_c4 or ragged or edge" \
  > gpurun_out/debug_checks.log 2>&1
tail -1 gpurun_out/debug_checks.log
