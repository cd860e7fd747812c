"""Compare the GPU reduced operators E, F of C4 orders with the oracle (the
plan handle is kept even when the solve fails)."""
import ctypes as C, os, sys, tempfile, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)
import paper_1707_05882_b200 as V, bench
import pyoracle as O
from paper_1707_05882_b200 import materials as M
from helpers import oracle_material
w = M.config("C4"); nodes = bench.quad_nodes(w.N)
mat = V.Material.load(w.material.write(tempfile.mkdtemp(), "m"))
om = oracle_material(w.material)
m0 = int(sys.argv[1]) if len(sys.argv) > 1 else 151
mu = np.ascontiguousarray(nodes[:4])
h = C.c_void_p()
rc = V.lib().vrte_brdf_plan_create(mat._h, C.byref(V.options(w.N)), V._dp(mu), len(mu), 5, None, 0, m0, 1, 1, C.byref(h))
print("plan rc", rc, V.lib().vrte_last_error().decode() if rc else "")
d = 4 * w.N
E = np.zeros(d * d); F = np.zeros(d * d)
V.lib().vrte_cuda_plan_fetch_ef(h, V._dp(E), V._dp(F))
E = E.reshape(d, d).T; F = F.reshape(d, d).T
e, f = O.reduced_ops(om, 0, w.N, m0)[:2]
print("m", m0, "finite", np.isfinite(E).all(), np.isfinite(F).all(),
      "E err %.2e F err %.2e" % (np.abs(E - e).max() / np.abs(e).max(), np.abs(F - f).max() / np.abs(f).max()))
bad = np.argwhere(~np.isfinite(E))
print("nonfinite E entries", len(bad), bad[:5])
