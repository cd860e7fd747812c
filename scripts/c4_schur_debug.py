"""Run the C4 order-151 F E (and neighbours) through the kernel-level Schur API."""
import os, sys, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)
import paper_1707_05882_b200 as V
import pyoracle as O
from paper_1707_05882_b200 import materials as M
from helpers import oracle_material
w = M.config("C4")
mat = oracle_material(w.material)
ms = [int(x) for x in sys.argv[1:]] or [151]
A = []
for m in ms:
    E, F = O.reduced_ops(mat, 0, w.N, m)[:2]
    A.append(F @ E)
A = np.array(A)
for blocked in (True, False):
    H, Q = V.hessenberg(A, blocked)
    print("hessenberg blocked=%d finite %s recon %.2e" % (blocked, np.isfinite(H).all(),
          max(np.abs(Q[i] @ H[i] @ Q[i].T - A[i]).max() / np.abs(A[i]).max() for i in range(len(ms)))))
try:
    T, Z, lam = V.schur(A)
    for i, m in enumerate(ms):
        ref = np.sort_complex(np.linalg.eigvals(A[i]))
        got = np.sort_complex(lam[i])
        print(m, "schur ok, recon %.2e, eig rel err %.2e" % (np.abs(Z[i] @ T[i] @ Z[i].T - A[i]).max() / np.abs(A[i]).max(),
              (np.abs(got - ref) / np.abs(ref)).max()))
except V.VrteError as e:
    print("schur FAIL", e)
