#!/bin/bash
# compute-sanitizer passes over smoke() (C1 through the C ABI): memcheck, synccheck, racecheck
O=gpurun_out/san; mkdir -p $O
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/$tool.log 2>&1; echo "rc=$?" >> $O/$tool.log
done
