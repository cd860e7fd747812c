O=gpurun_out/sw; mkdir -p $O
for k in 2 3 4 5 6 8; do timeout 600 python bench.py --config C5 --steps 3 --warmup 1 --no-cpu-baseline --concurrency $k > $O/c5_k$k.log 2>&1; done
