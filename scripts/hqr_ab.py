"""A/B: windowed vs simple Francis QR must give bitwise identical Schur forms."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, tempfile, numpy as np
sys.path.insert(0, "%s"); sys.path.insert(0, "%s/oracle")
import paper_1707_05882_b200 as V, pyoracle as O, bench
out = {}
for cfg in ("C1", "C2", "C3"):
    w = bench.workload(cfg); nodes = bench.quad_nodes(w.N)
    mat = V.Material.load(w.material.write(tempfile.mkdtemp(), "m"))
    p = V.Plan(mat, V.options(w.N), nodes[:4], 5, device=0)
    S = 2 if cfg == "C3" else 1
    wr, wi, res, nu = p.modes(S)
    t = p.run(2)
    out[cfg] = (wr, wi, p.table(), t, p.last.t_hqr)
np.savez(sys.argv[1], **{k + "_" + n: v for k, tup in out.items() for n, v in zip(("wr","wi","tab","t","thqr"), tup)})
''' % (ROOT, ROOT)
for mode in ("simple", "windowed"):
    env = dict(os.environ)
    env["VRTE_HQR"] = "band" if mode == "simple" else "window"
    subprocess.run([sys.executable, "-c", code, f"{ROOT}/gpurun_out/hqr_{mode}.npz"], env=env, check=True)
import numpy as np
a = np.load(f"{ROOT}/gpurun_out/hqr_simple.npz"); b = np.load(f"{ROOT}/gpurun_out/hqr_windowed.npz")
for cfg in ("C1", "C2", "C3"):
    la = np.sort_complex((a[cfg+"_wr"] + 1j*a[cfg+"_wi"]).ravel()); lb = np.sort_complex((b[cfg+"_wr"] + 1j*b[cfg+"_wi"]).ravel())
    ta, tb = a[cfg+"_tab"], b[cfg+"_tab"]
    print(cfg, "eig max rel diff %.2e" % (np.abs(la-lb)/np.abs(la)).max(), "table max rel diff %.2e" % (np.abs(ta-tb).max()/np.abs(ta).max()),
          "hqr ms band %.2f window %.2f" % (1e3*a[cfg+"_thqr"], 1e3*b[cfg+"_thqr"]))
