"""Measured parity of the GPU path (numbers behind the tolerances in
tests/test_gpu_parity.py): golden fixtures vs the exact (mpmath) answer and vs
the fp64 reference restatement, C2 full table and C3 incidents vs the oracle
(as written and in accurate mode).  Prints one JSON object."""
import glob, json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)
import paper_1707_05882_b200 as V
import pyoracle as O
from paper_1707_05882_b200 import materials as M
from helpers import (GOLDEN, desc_from_golden, load_golden, matrix_metric, oracle_material,
                     product_material, survey_metric)

out = {"env": {k: v for k, v in os.environ.items() if k.startswith("VRTE_")}, "golden": {}}
for path in sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))):
    case = os.path.basename(path)[:-4]
    z, meta = load_golden(case)
    desc = desc_from_golden(z, meta)
    b = V.compute_brdf(product_material(desc), V.options(meta["N"]), z["mu_in"], meta["n_dphi"])
    g = b.table()
    ex, orc = z["exact"], z["oracle"]
    if np.abs(ex).max() == 0:
        out["golden"][case] = {"max_abs": float(np.abs(g).max())}
        continue
    out["golden"][case] = {"gpu_vs_exact_matrix": matrix_metric(g, ex), "gpu_vs_exact_survey": survey_metric(g, ex),
                           "ref_vs_exact_matrix": matrix_metric(orc, ex), "ref_vs_exact_survey": survey_metric(orc, ex),
                           "gpu_vs_ref_survey": survey_metric(g, orc)}
for cfg, pick in (("C2", None), ("C3", [0, 40, 63])):
    w = M.config(cfg)
    nodes, _ = O.quadrature(w.N)
    b = V.compute_brdf(product_material(w.material), V.options(w.N), nodes, 19)
    g = b.table()
    st = b.device_stats()
    mu = nodes if pick is None else nodes[pick]
    gs = g if pick is None else g[pick]
    t = time.time()
    r, _ = O.brdf(oracle_material(w.material), w.N, mu, 19)
    acc_pick = list(range(len(mu))) if cfg == "C2" else [1]
    with O.accurate():
        ra, _ = O.brdf(oracle_material(w.material), w.N, mu[acc_pick], 19)
    out[cfg] = {"incidents": "all" if pick is None else pick, "gpu_vs_ref_matrix": matrix_metric(gs, r),
                "gpu_vs_accurate_ref_matrix": matrix_metric(gs[acc_pick], ra),
                "ref_vs_accurate_ref_matrix": matrix_metric(r[acc_pick], ra),
                "max_eigen_residual": st["max_eigen_residual"], "oracle_s": round(time.time() - t, 1)}
print(json.dumps(out, indent=1))
