import sys, os, numpy as np, tempfile
which = sys.argv[1]
root = os.getcwd()
if which == "old":
    sys.path.insert(0, os.path.join(root, "_old"))
sys.path.insert(1, root)
import paper_1707_05882_b200 as V
print(which, V.LIB_PATH)
import bench
for cfg in ["C3", "C1", "C2"]:
    w = bench.workload(cfg); nodes = bench.quad_nodes(w.N)
    mat = V.Material.load(w.material.write(tempfile.mkdtemp(), "m"))
    b = V.compute_brdf(mat, V.options(w.N), nodes, w.n_dphi)
    np.save(f"/tmp/{which}_{cfg}.npy", b.table())
if which == "new":
    for cfg in ["C3", "C1", "C2"]:
        a, c = np.load(f"/tmp/old_{cfg}.npy"), np.load(f"/tmp/new_{cfg}.npy")
        print(cfg, "bitwise equal:", np.array_equal(a, c), "max diff", np.abs(a - c).max())
