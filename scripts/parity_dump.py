"""Diagnostics: save the GPU table and the accurate-mode oracle's for one
config to gpurun_out/dump_<cfg>_<tag>.npz (VRTE_ORACLE_BND_STEPS /
VRTE_ORACLE_POLISH select the oracle variant) for offline analysis."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)
import paper_1707_05882_b200 as V
import pyoracle as O
from paper_1707_05882_b200 import materials as M
from helpers import oracle_material, product_material

cfg, tag = sys.argv[1], sys.argv[2]
band = int(sys.argv[3]) if len(sys.argv) > 3 else 0
w = M.config(cfg, band)
nodes, _ = O.quadrature(w.N)
b = V.compute_brdf(product_material(w.material), V.options(w.N), nodes, 19)
g = b.table()
print("stats", b.device_stats(), flush=True)
om = oracle_material(w.material)
with O.cached_boundary(), O.accurate():
    ra, _ = O.brdf(om, w.N, nodes, 19)
np.savez_compressed(f"gpurun_out/dump_{w.name}_{tag}.npz", gpu=g, acc=ra)
