set -u
O=gpurun_out/q1; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c3.log 2>&1
timeout 900 python bench.py --config C5 --steps 3 --warmup 1 --no-cpu-baseline > $O/bench_C5.log 2>&1
