import os, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench, paper_1707_05882_b200 as V
for cfg in sys.argv[1:] or ["C3"]:
    w = bench.workload(cfg); nodes = bench.quad_nodes(w.N)
    mat = V.Material.load(w.material.write(tempfile.mkdtemp(), "m"))
    p = V.Plan(mat, V.options(w.N), nodes, w.n_dphi, device=0)
    p.run(1)
    r = p.last
    nmat = 2 * w.material.order_count if cfg in ("C3", "C5") else w.material.order_count
    cyc = list(r.qr_cycles)
    print(cfg, "sweeps", r.qr_sweeps, "reflectors", r.qr_steps, "t_hqr ms %.2f" % (r.t_hqr * 1e3),
          "cycles/reflector/matrix %.0f" % (r.t_hqr * 1.9e9 / (r.qr_steps / nmat)))
    st = max(r.qr_steps, 1)
    print("   per reflector (thread-0 clock): defl+shift=%.0f winload=%.0f chase=%.0f update=%.0f" %
          tuple(c / st for c in cyc[:4]), " AED deflations %d, %.0f%% of reflectors in multi-bulge sweeps" % (cyc[4], 100.0 * cyc[5] / st))
    print("   AED calls %d, %.0f cycles per call (warp-0 Schur of the window)" % (cyc[7], cyc[6] / max(cyc[7], 1)))
