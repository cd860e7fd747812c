import time, tempfile, numpy as np, sys
sys.path.insert(0, '.')
import paper_1707_05882_b200 as V
from paper_1707_05882_b200 import materials as M
w = M.config("C3")
d = tempfile.mkdtemp()
mat = V.Material.load(w.material.write(d, "m"))
import bench
nodes = bench.quad_nodes(w.N)
for i in range(6):
    t0 = time.perf_counter()
    b = V.compute_brdf(mat, V.options(w.N), nodes, w.n_dphi)
    t1 = time.perf_counter()
    tm = b.timings() if hasattr(b, "timings") else None
    st = V.DeviceStats(); 
    V.lib().vrte_brdf_device_stats_get(b._h, V.C.byref(st)) if hasattr(V, "DeviceStats") else None
    dev = st.t_homogeneous + st.t_particular + st.t_boundary + st.t_synthesis
    print("py %.2f ms  device stages %.2f ms" % ((t1 - t0) * 1e3, dev * 1e3))
    b.close() if hasattr(b, "close") else None
