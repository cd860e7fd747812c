"""Experiment: C3 tables with and without the eigenpair Newton step (env
variants), each against the accurate oracle at a few incidents, with the
device stage times.  Usage: python scripts/refine_experiment.py [out.json]"""
import os, sys, subprocess, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
VARIANTS = {"base": {}, "no_newton": {"VRTE_REFINE_ITERS": "0", "VRTE_REFINE_EXTRA": "0"},
            "adaptive": {"VRTE_REFINE_ITERS": "0", "VRTE_REFINE_EXTRA": "2"}}
PICK = [0, 1, 2, 8, 20, 40, 63]
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import paper_1707_05882_b200 as V
    import pyoracle as O
    from paper_1707_05882_b200 import materials as M
    from helpers import product_material
    w = M.config("C3")
    nodes, _ = O.quadrature(w.N)
    mat = product_material(w.material)
    full = V.compute_brdf(mat, V.options(w.N), nodes, 19)
    np.save(sys.argv[2], full.table()[PICK])
    st = full.device_stats()
    plan = V.Plan(mat, V.options(w.N), nodes, 19)
    plan.run(3)
    sec = plan.run(10)
    res = plan.last.as_dict()
    print(json.dumps({"ms_per_solve": sec * 1e3, "t_refine_ms": res["t_refine"] * 1e3,
                      "max_eigen_residual": res["max_eigen_residual"], "stats": st}))
    sys.exit(0)
import pyoracle as O
from paper_1707_05882_b200 import materials as M
from helpers import matrix_metric, oracle_material, survey_metric, survey_per_matrix
w = M.config("C3")
nodes, _ = O.quadrature(w.N)
with O.cached_boundary(), O.accurate():
    acc, _ = O.brdf(oracle_material(w.material), w.N, nodes[PICK], 19)
rep = {"incidents": PICK}
for name, env in VARIANTS.items():
    e = dict(os.environ, **env)
    f = f"/tmp/refx_{name}.npy"
    r = subprocess.run([sys.executable, __file__, "child", f], env=e, capture_output=True, text=True)
    if r.returncode != 0:
        rep[name] = {"error": r.stderr[-800:]}
        continue
    g = np.load(f)
    info = json.loads(r.stdout.strip().splitlines()[-1])
    pm = survey_per_matrix(g, acc)
    info.update({"survey_vs_accurate": survey_metric(g, acc), "matrix_vs_accurate": matrix_metric(g, acc),
                 "survey_excl_grazing": float(pm[3:, 4:].max()),
                 "survey_per_incident": [float(pm[i].max()) for i in range(len(PICK))]})
    rep[name] = info
    print(name, json.dumps(info)[:600], flush=True)
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/refine_experiment.json"
json.dump(rep, open(out, "w"), indent=1)
