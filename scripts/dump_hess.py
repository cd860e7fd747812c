import os, sys, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1707_05882_b200 as V
A = np.load(os.path.join(ROOT, "build", "debug", "c4_fe151.npy"))
for blocked in (1, 0):
    H, Q = V.hessenberg(A[None], bool(blocked))
    np.save(os.path.join(ROOT, "gpurun_out", "c4_h151_%s.npy" % ("blocked" if blocked else "unblocked")), H[0])
    try:
        V.schur(A[None]) if blocked else None
    except V.VrteError as e:
        print("schur fails", e)
print("saved")
