#!/bin/bash
# compute-sanitizer passes over smoke() (C1 through the C ABI): memcheck, synccheck, racecheck
O=gpurun_out/san; mkdir -p $O
if [ -z "${1:-}" ]; then for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/$tool.log 2>&1; echo "rc=$?" >> $O/$tool.log
done; fi
# one C3 plan creation + solve (scripts/profile_step.py C3) under memcheck / synccheck when asked
if [ "${1:-}" = "c3" ]; then
  for tool in memcheck synccheck; do
    timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/profile_step.py C3 > $O/c3_$tool.log 2>&1; echo "rc=$?" >> $O/c3_$tool.log
  done
fi
# C4' (N = 128, 256 orders: the 128-register QR build, d = 512) under memcheck when asked
if [ "${1:-}" = "c4p" ]; then
  timeout 1800 compute-sanitizer --tool memcheck --print-limit 20 python scripts/profile_step.py C4p > $O/c4p_memcheck.log 2>&1; echo "rc=$?" >> $O/c4p_memcheck.log
fi
# the batch API (concurrent plans on their own threads/streams, lean QR build) and the kernel tests under memcheck
if [ "${1:-}" = "batch" ]; then
  timeout 1800 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -q -p no:cacheprovider \
    tests/test_gpu_capi.py tests/test_gpu_kernels.py tests/test_gpu_multidevice.py > $O/batch_memcheck.log 2>&1; echo "rc=$?" >> $O/batch_memcheck.log
fi
