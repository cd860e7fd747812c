import os, sys, time, tempfile, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1707_05882_b200 as V, bench
path = os.path.join(ROOT, "build", "debug", "fe_c3.bin")
if not os.path.exists(path):
    os.environ["VRTE_DUMP_FE"] = path
    w = bench.workload("C3"); nodes = bench.quad_nodes(w.N)
    mat = V.Material.load(w.material.write(tempfile.mkdtemp(), "m"))
    V.Plan(mat, V.options(w.N), nodes[:2], 3, device=0)
    del os.environ["VRTE_DUMP_FE"]
d = 256
A = np.fromfile(path).reshape(-1, d, d).transpose(0, 2, 1).copy()
V.schur(A[:2])
ts = []
for _ in range(3):
    t = time.perf_counter(); V.schur(A); ts.append(time.perf_counter() - t)
print("schur batch", A.shape[0], "wall ms", ["%.1f" % (1e3 * x) for x in ts], "NOZ" if os.environ.get("VRTE_QR_NOZ_DEBUG") else "")
