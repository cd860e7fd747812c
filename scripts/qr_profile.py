"""Per-matrix profile of the multishift QR kernel on the C3 (or given config)
F E matrices: E, F fetched from a plan, F E formed on the host, then the
kernel-level Schur call with the kernel's trace.  Prints the distribution of
rank-0 cycles, sweeps, AED calls and the AED / chase / update-wait shares."""
import json, os, sys, tempfile
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench, paper_1707_05882_b200 as V
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
w = bench.workload(cfg)
nodes = bench.quad_nodes(w.N)
mat = V.Material.load(w.material.write(tempfile.mkdtemp(), "m"))
S = len({(l.omega, l.coeffs.tobytes()) for l in w.material.layers})
p = V.Plan(mat, V.options(w.N), nodes[:1], 5, device=0)
E, F = p.ef(S)
L = E.shape[1]
FE = np.einsum("smij,smjk->smik", F, E).reshape(S * L, 4 * w.N, 4 * w.N)
Be = int(p.last.eigen_slots) if p.last.eigen_slots else S * L
FE = FE[:Be] if Be else FE
tr, ms = V.schur_trace(FE)
tr2, ms2 = V.schur_trace(FE)
cyc = tr[:, 0]
order = np.argsort(-cyc)
out = {"config": cfg, "matrices": len(FE), "qr_ms": ms2, "clock_ghz_est": float(cyc.max() / (ms2 * 1e6)),
       "cycles_max": float(cyc.max()), "cycles_median": float(np.median(cyc)), "cycles_p90": float(np.percentile(cyc, 90)),
       "slowest": [{"slot": int(b), "cycles": float(tr[b, 0]), "sweeps": float(tr[b, 2]), "aed_calls": float(tr[b, 3]),
                    "aed_cycles": float(tr[b, 4]), "chase_cycles": float(tr[b, 5]), "wait_cycles": float(tr[b, 6]),
                    "aed_deflations": float(tr[b, 7])} for b in order[:8]],
       "mean_share": {"aed": float((tr[:, 4] / cyc).mean()), "chase": float((tr[:, 5] / cyc).mean()),
                      "wait": float((tr[:, 6] / cyc).mean())}}
print(json.dumps(out, indent=1))
