#!/bin/bash
# compute-sanitizer passes over smoke() (C1 through the C ABI): memcheck, synccheck, racecheck
O=gpurun_out/san; mkdir -p $O
if [ "${1:-}" != "c3" ]; then for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/$tool.log 2>&1; echo "rc=$?" >> $O/$tool.log
done; fi
# one C3 plan creation + solve (scripts/profile_step.py C3) under memcheck / synccheck when asked
if [ "${1:-}" = "c3" ]; then
  for tool in memcheck synccheck; do
    timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/profile_step.py C3 > $O/c3_$tool.log 2>&1; echo "rc=$?" >> $O/c3_$tool.log
  done
fi
