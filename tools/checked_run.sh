#!/bin/bash
# Checked build run (compute-sanitizer is closed on this GPU pool): the
# library built with -DSPX_DEBUG_CHECKS (device bounds / invariant checks
# that trap) runs the sanitizer cases and the GPU suite's kernel and pipeline
# tests, then the cases again under every lanes-per-cell template and with
# CUDA graphs off (a data race shows up as a result that depends on the
# launch shape; every run is compared with the oracle).
#   python tools/build_variants.py checked:-DSPX_DEBUG_CHECKS   (here)
#   bash tools/checked_run.sh > gpurun_out/checked.log 2>&1     (GPU box)
set -u
export SPX_LIB_VARIANT=variants/libspx_checked.so
rc=0
echo "== sanitizer cases (checked build)"; python tools/sanitize_cases.py || rc=1
for lpc in 4 8 16 32; do
  echo "== SPX_LPC=$lpc"; SPX_LPC=$lpc python tools/sanitize_cases.py | tail -1 || rc=1
done
echo "== SPX_NO_GRAPHS=1"; SPX_NO_GRAPHS=1 python tools/sanitize_cases.py | tail -1 || rc=1
echo "== GPU tests (checked build)"
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py tests/test_gpu_errors.py \
  tests/test_gpu_large.py -q -x -p no:cacheprovider 2>&1 | tail -3
[ "${PIPESTATUS[0]}" = 0 ] || rc=1
echo "checked run rc=$rc"
exit $rc
