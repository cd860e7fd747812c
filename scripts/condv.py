"""Conditioning study of the eigenvector matrices of F E per (medium, order):
cond(V) (numpy eig, unit columns) -> can V^-1 replace the Schur form as the
approximate inverse?  Writes gpurun_out/condv_<cfg>.txt"""
import os, sys, tempfile, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench, paper_1707_05882_b200 as V
for cfg in sys.argv[1:] or ["C3"]:
    w = bench.workload(cfg); nodes = bench.quad_nodes(w.N)
    mat = V.Material.load(w.material.write(tempfile.mkdtemp(), "m"))
    p = V.Plan(mat, V.options(w.N), nodes[:2], 3, device=0)
    S = 2 if cfg in ("C3",) else 1
    E, F = p.ef(S)
    lines = []
    for s in range(S):
        for m in range(E.shape[1]):
            A = F[s, m] @ E[s, m]
            lam, X = np.linalg.eig(A)
            X = X / np.linalg.norm(X, axis=0)
            c = np.linalg.cond(X)
            rel = np.sort(np.abs(lam))
            gap = np.min(np.abs(lam[:, None] - lam[None, :]) + np.eye(len(lam)) * 1e300, axis=1) / np.abs(lam)
            lines.append("s=%d m=%2d cond(V)=%9.2e  |lam| %.2e..%.2e  min rel gap %.1e  n_complex %d" % (
                s, m, c, rel[0], rel[-1], gap.min(), int((np.abs(lam.imag) > 0).sum())))
    open(f"{ROOT}/gpurun_out/condv_{cfg}.txt", "w").write("\n".join(lines) + "\n")
    print(cfg, "max cond", max(float(l.split("cond(V)=")[1].split()[0]) for l in lines))
