#!/bin/bash
# Re-run of the per-configuration bench records at the current code (one B200).
set -u
O=gpurun_out/rr; mkdir -p $O
for c in C1 C2 C3F; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.log 2>&1; done
timeout 900 python bench.py --config C4p --steps 3 --warmup 1 --no-cpu-baseline > $O/bench_C4p.log 2>&1
timeout 900 python bench.py --config R3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_R3.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_c3.log 2>&1
timeout 600 python scripts/shard_probe.py C3 2,4,8 4 > $O/shard_c3.jsonl 2>&1
timeout 900 python scripts/shard_probe.py C4p 2,4,8 > $O/shard_c4p.jsonl 2>&1
