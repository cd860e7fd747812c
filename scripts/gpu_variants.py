"""Diagnostics: GPU C3 tables at a few incidents under refinement variants
(env knobs of the experiment), saved to gpurun_out/variants.npz."""
import os, sys, subprocess, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
VARIANTS = {"base": {}, "bnd": {"VRTE_BND_FORCE_REFINE": "1"}, "part2": {"VRTE_PART_REFINE_ITERS": "2"},
            "eig2": {"VRTE_REFINE_ITERS": "2"},
            "all": {"VRTE_BND_FORCE_REFINE": "1", "VRTE_PART_REFINE_ITERS": "2", "VRTE_REFINE_ITERS": "2"}}
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import paper_1707_05882_b200 as V
    import pyoracle as O
    from paper_1707_05882_b200 import materials as M
    from helpers import product_material
    w = M.config(sys.argv[2])
    nodes, _ = O.quadrature(w.N)
    pick = [int(x) for x in sys.argv[3].split(",")]
    b = V.compute_brdf(product_material(w.material), V.options(w.N), nodes[pick], 19)
    np.save(sys.argv[4], b.table())
    print(json.dumps(b.device_stats()))
    sys.exit(0)
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
pick = sys.argv[2] if len(sys.argv) > 2 else "0,1,2,40"
out = {}
for name, env in VARIANTS.items():
    e = dict(os.environ, **env)
    f = f"/tmp/var_{name}.npy"
    r = subprocess.run([sys.executable, __file__, "child", cfg, pick, f], env=e, capture_output=True, text=True)
    print(name, r.stdout.strip()[-300:], r.stderr[-500:])
    out[name] = np.load(f)
np.savez_compressed(f"gpurun_out/variants_{cfg}.npz", **out)
