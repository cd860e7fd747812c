"""C4 eigen stage check (all 256 orders, 4 incidents): which QR settings converge."""
import os, sys, tempfile, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench, paper_1707_05882_b200 as V
w = bench.workload("C4"); nodes = bench.quad_nodes(w.N)
mat = V.Material.load(w.material.write(tempfile.mkdtemp(), "m"))
t = time.time()
try:
    p = V.Plan(mat, V.options(w.N), nodes[:4], 5, device=0)
    r = p.last
    print("ok", "t_hqr %.1f ms" % (r.t_hqr * 1e3), "hess %.1f" % (r.t_hessenberg * 1e3), "sweeps", r.qr_sweeps,
          "refl", r.qr_steps, "maxres %.1e" % r.max_eigen_residual, "wall %.1f s" % (time.time() - t))
except V.VrteError as e:
    print("FAIL", e, "wall %.1f s" % (time.time() - t))
