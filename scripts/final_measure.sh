#!/bin/bash
# Round-end measurement pass on one B200 (run under gpurun from the repo root);
# results in gpurun_out/final/.  See profiles/README.md for what each file is.
set -u
O=gpurun_out/final
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c3.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_c3.log 2>&1
for c in C1 C2 C3F; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.log 2>&1; done
timeout 900 python bench.py --config C4p --steps 3 --warmup 1 --no-cpu-baseline > $O/bench_C4p.log 2>&1
timeout 900 python bench.py --config C5 --steps 3 --warmup 1 --no-cpu-baseline > $O/bench_C5.log 2>&1
timeout 900 python bench.py --config R3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_R3.log 2>&1
timeout 900 python bench.py --config MC7 --steps 1 --warmup 1 > $O/bench_MC7.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python scripts/profile_step.py C3 > $O/prof.log 2>&1
timeout 600 python scripts/shard_probe.py C3 2,4,8 4 > $O/shard_c3.jsonl 2>&1
timeout 900 python scripts/shard_probe.py C4p 2,4,8 > $O/shard_c4p.jsonl 2>&1
timeout 600 python scripts/qr_profile.py C3 > $O/qr_profile_c3.json 2>/dev/null
# ncu --set full of the top kernels, summarised on the box (the reports are large)
bash scripts/ncu_capture.sh
python scripts/ncu_summary.py $O/ncu_summary.json gpurun_out/ncu_*.ncu-rep > $O/ncu_summary.log 2>&1
rm -f gpurun_out/ncu_*.ncu-rep
