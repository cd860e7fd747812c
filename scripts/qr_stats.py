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
    print(cfg, "sweeps", r.qr_sweeps, "steps", r.qr_steps, "t_hqr ms %.2f" % (r.t_hqr * 1e3),
          "cycles/step/matrix-par %.0f" % (r.t_hqr * 1.9e9 / (r.qr_steps / (2 * w.material.order_count if cfg == "C3" else w.material.order_count))))
    cyc = list(r.qr_cycles); tot = sum(cyc) or 1
    print("   phase cycles per step: " + " ".join("%s=%.0f" % (n, c / r.qr_steps) for n, c in zip(("shift+Msearch", "winload", "chase", "writeback+update", "?", "deflation"), cyc)))
