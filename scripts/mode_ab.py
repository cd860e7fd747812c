"""A/B two settings of one env switch (e.g. VRTE_HESS=unblocked vs blocked):
eigenvalues, BRDF tables and stage times must agree.
usage: python scripts/mode_ab.py VAR valueA valueB [configs...]"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
var, va, vb = sys.argv[1:4]
cfgs = sys.argv[4:] or ["C1", "C2", "C3"]
code = r'''
import os, sys, tempfile, numpy as np
sys.path.insert(0, "%s")
import paper_1707_05882_b200 as V, bench
out = {}
for cfg in sys.argv[2].split(","):
    w = bench.workload(cfg); nodes = bench.quad_nodes(w.N)
    mat = V.Material.load(w.material.write(tempfile.mkdtemp(), "m"))
    p = V.Plan(mat, V.options(w.N), nodes, w.n_dphi, device=0)
    S = 2 if cfg in ("C3", "C5") else 1
    wr, wi, res, nu = p.modes(S)
    t = p.run(3)
    r = p.last
    out[cfg] = (wr, wi, res, p.table(), t, r.t_hessenberg, r.t_hqr, r.t_refine, r.t_particular, r.t_boundary)
np.savez(sys.argv[1], **{k + "_" + n: v for k, tup in out.items()
         for n, v in zip(("wr","wi","res","tab","t","th","tq","tr","tp","tb"), tup)})
''' % ROOT
files = []
for val in (va, vb):
    env = dict(os.environ); env[var] = val
    f = f"{ROOT}/gpurun_out/ab_{var}_{val}.npz"
    subprocess.run([sys.executable, "-c", code, f, ",".join(cfgs)], env=env, check=True)
    files.append(f)
import numpy as np
a, b = np.load(files[0]), np.load(files[1])
for cfg in cfgs:
    la = np.sort_complex((a[cfg+"_wr"] + 1j*a[cfg+"_wi"]).ravel()); lb = np.sort_complex((b[cfg+"_wr"] + 1j*b[cfg+"_wi"]).ravel())
    ta, tb = a[cfg+"_tab"], b[cfg+"_tab"]
    print(cfg, "eig max rel diff %.2e" % (np.abs(la-lb)/np.maximum(np.abs(la),1e-300)).max(),
          "table max rel diff %.2e" % (np.abs(ta-tb).max()/np.abs(ta).max()),
          "max residual %.1e / %.1e" % (a[cfg+"_res"].max(), b[cfg+"_res"].max()))
    for key, name in (("t","solve"),("th","hess"),("tq","hqr"),("tr","refine"),("tp","partic"),("tb","bound")):
        print("   %-7s ms  %s=%-10s %8.3f   %s=%-10s %8.3f" % (name, var, va, 1e3*a[cfg+"_"+key], var, vb, 1e3*b[cfg+"_"+key]))
