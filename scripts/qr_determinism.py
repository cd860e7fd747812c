import os, sys, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1707_05882_b200 as V
A = np.load(os.path.join(ROOT, "build", "debug", "c4_fe151.npy"))
res = []
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    try:
        T, Z, lam = V.schur(A[None])
        res.append(("ok", float(np.abs(T).sum())))
    except V.VrteError:
        res.append(("FAIL", 0.0))
print(os.environ.get("VRTE_HQR", "multi"), [r[0] for r in res], "distinct T sums", len(set(r[1] for r in res)))
