"""One warm-up + one timed C3 solve through a device-resident plan (for ncu)."""
import os, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import paper_1707_05882_b200 as V
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
w = bench.workload(cfg)
nodes = bench.quad_nodes(w.N)
mat = V.Material.load(w.material.write(tempfile.mkdtemp(), "m"))
plan = V.Plan(mat, V.options(w.N), nodes, w.n_dphi, device=0)   # first solve (warm-up)
print("solve s", plan.run(1), plan.last.as_dict()["kernel_launches"])
