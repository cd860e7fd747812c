"""Dump GPU BRDF tables for the golden cases and C2/C3 (dev analysis)."""
import glob, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)
import paper_1707_05882_b200 as V
import pyoracle as O
from paper_1707_05882_b200 import materials as M
from helpers import load_golden, desc_from_golden, product_material
out = {}
for f in sorted(glob.glob(os.path.join(ROOT, "tests/golden/*.npz"))):
    name = os.path.basename(f)[:-4]
    z, meta = load_golden(name)
    desc = desc_from_golden(z, meta)
    b = V.compute_brdf(product_material(desc), V.options(meta["N"]), z["mu_in"], meta["n_dphi"])
    out[name] = b.table()
for cfg, pick in (("C2", None), ("C3", [0, 40, 63])):
    w = M.config(cfg)
    nodes, _ = O.quadrature(w.N)
    mat = product_material(w.material)
    b = V.compute_brdf(mat, V.options(w.N), nodes, 19)
    t = b.table()
    out[cfg] = t if pick is None else t[pick]
    for it in (1, 5):
        os.environ["VRTE_REFINE_ITERS"] = str(it); os.environ["VRTE_NO_RESIDUAL_GATE"] = "1"
        b = V.compute_brdf(mat, V.options(w.N), nodes, 19)
        out[f"{cfg}_ref{it}"] = b.table() if pick is None else b.table()[pick]
    os.environ.pop("VRTE_REFINE_ITERS"); os.environ.pop("VRTE_NO_RESIDUAL_GATE")
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez_compressed(os.path.join(ROOT, "gpurun_out", "gpu_tables.npz"), **out)
print("saved", list(out))
# particular-refinement ablation on the golden cases
for pit in (0, 1, 3):
    os.environ["VRTE_PART_REFINE_ITERS"] = str(pit)
    res = {}
    for f in sorted(glob.glob(os.path.join(ROOT, "tests/golden/*.npz"))):
        name = os.path.basename(f)[:-4]
        z, meta = load_golden(name)
        desc = desc_from_golden(z, meta)
        b = V.compute_brdf(product_material(desc), V.options(meta["N"]), z["mu_in"], meta["n_dphi"])
        res[name] = b.table()
    np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"gpu_tables_pit{pit}.npz"), **res)
