"""Throughput of K concurrent device-resident C3 plans (K host threads, one
CUDA stream per plan)."""
import os, sys, tempfile, threading, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench, paper_1707_05882_b200 as V
w = bench.workload("C3"); nodes = bench.quad_nodes(w.N)
for K in (1, 2, 3, 4):
    plans = []
    for k in range(K):
        mat = V.Material.load(w.material.write(tempfile.mkdtemp(), "m"))
        plans.append(V.Plan(mat, V.options(w.N), nodes, w.n_dphi, device=0))
    steps = 6
    for p in plans: p.run(1)
    ths = [threading.Thread(target=p.run, args=(steps,)) for p in plans]
    t = time.perf_counter()
    for th in ths: th.start()
    for th in ths: th.join()
    dt = time.perf_counter() - t
    print("K=%d  %.1f solves/s  (%.2f ms per solve)" % (K, K * steps / dt, 1e3 * dt / (K * steps)), os.environ.get("VRTE_QR_CLUSTER", ""))
    for p in plans: p.close()
