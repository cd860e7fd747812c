import os, sys, ctypes as C, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1707_05882_b200 as V
A = np.load(os.path.join(ROOT, "build", "debug", "c4_fe151.npy"))[None]
batch, d, _ = A.shape
Ac = np.ascontiguousarray(A.transpose(0, 2, 1))
T, Z = np.zeros_like(Ac), np.zeros_like(Ac)
wr, wi = np.zeros((batch, d)), np.zeros((batch, d))
code = V.lib().vrte_cuda_schur(V._dp(Ac), d, batch, V._dp(T), V._dp(Z), V._dp(wr), V._dp(wi), 0)
T = T[0].T
print("code", code)
np.save(os.path.join(ROOT, "gpurun_out", "c4_fail_T.npy"), T)
np.set_printoptions(linewidth=200, precision=6)
print(T[504:512, 504:512])
