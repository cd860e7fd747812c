import os, sys, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1707_05882_b200 as V
d = 512
A = np.fromfile(sys.argv[1]).reshape(-1, d, d).transpose(0, 2, 1)  # column-major dump
print("dumped", A.shape, "finite", np.isfinite(A).all())
for env in ("multi",):
    try:
        T, Z, lam = V.schur(A)
        print("schur ok on the dumped matrix")
    except V.VrteError as e:
        print("schur FAIL on the dumped matrix:", e)
lam = np.linalg.eigvals(A[0])
print("numpy eig ok; min |lam| %.3e, n complex %d" % (np.abs(lam).min(), (np.abs(lam.imag) > 0).sum()))
np.save(os.path.join(ROOT, "gpurun_out", "c4_fe151.npy"), A[0])
