"""Order-shard timing on ONE GPU (emulates the multi-GPU modes of bench.py):
  single : one full-order plan, solves/s
  shardW : the W order shards of one solve (m = r mod W), each alone -> the
           per-rank time of a solve sharded over W GPUs (latency mode)
  concW  : the W shards run concurrently (W host threads / streams) -> the
           per-GPU work of W in-flight solves each sharded over W GPUs
           (throughput mode)
Usage: python scripts/shard_probe.py [C3|C4p] [W,...] [concurrency,...]"""
import json, os, sys, tempfile, threading, time
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # (as bench.py: many streams in flight)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench, paper_1707_05882_b200 as V
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
Ws = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]
Ks = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0]  # 0: all W at once
w = bench.workload(cfg)
nodes = bench.quad_nodes(w.N)
L = w.material.order_count
mat = V.Material.load(w.material.write(tempfile.mkdtemp(), "m"))
opts = V.options(w.N)
steps = 4 if cfg == "C3" else 1
out = {"config": cfg}
p = V.Plan(mat, opts, nodes, w.n_dphi, device=0)
p.run(1)
out["single_ms"] = p.run(steps) * 1e3
p.close()
for W in Ws:
    # pooled plans, as the distributed layer uses them (the lean kernel builds)
    plans = [V.Plan(mat, opts, nodes, w.n_dphi, device=0, m_begin=r, m_stride=W, n_orders=len(range(r, L, W)),
                    pooled=True) for r in range(W)]
    alone = []
    for q in plans:
        q.run(1)
        alone.append(q.run(steps) * 1e3)
    rec = {"shard_alone_ms_max": max(alone), "shard_alone_ms": alone}
    for K in Ks:
        K = K or W
        groups = [plans[i::K] for i in range(K)]
        ths = [threading.Thread(target=lambda g=g: [q.run(steps) for q in g]) for g in groups]
        t = time.perf_counter()
        for th in ths: th.start()
        for th in ths: th.join()
        rec[f"concurrent{K}_ms_per_solve"] = (time.perf_counter() - t) / steps * 1e3
    out[f"W{W}"] = rec
    for q in plans: q.close()
    print(json.dumps(out), flush=True)
