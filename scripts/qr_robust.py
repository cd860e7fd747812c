"""QR robustness: the C4 order-m F E with tiny random perturbations (1 ulp
level), batch of copies through the kernel-level Schur API."""
import os, sys, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)
import paper_1707_05882_b200 as V
import pyoracle as O
from paper_1707_05882_b200 import materials as M
from helpers import oracle_material
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 151
n = int(sys.argv[3]) if len(sys.argv) > 3 else 16
w = M.config(cfg)
E, F = O.reduced_ops(oracle_material(w.material), 0, w.N, m)[:2]
A0 = F @ E
rng = np.random.default_rng(1)
A = np.array([A0 * (1 + 2e-16 * rng.standard_normal(A0.shape)) for _ in range(n)])
fails = 0
for i in range(n):
    try:
        V.schur(A[i:i + 1])
    except V.VrteError:
        fails += 1
print(cfg, "m", m, "QR failures %d / %d" % (fails, n))
