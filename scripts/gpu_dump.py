"""Dump GPU tables / modes / tau=0 stacks for offline comparison with the oracle."""
import os, sys, json, tempfile
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1707_05882_b200 as V
from paper_1707_05882_b200 import materials as M
import pyoracle as O

CASES = {
    "rayleigh_N6": (lambda: M.single_layer(M.RAYLEIGH, 0.9, 1.0, "lambertian", 0.3), 6, [0.7], 6),
    "C1": (lambda: M.config("C1").material, 8, None, 19),
    "conservative_N8": (lambda: M.single_layer(M.ISOTROPIC, 1.0, 10.0, "lambertian", 1.0), 8, None, 19),
    "paint_N8": (lambda: M.MaterialDesc([M.LayerDesc(0.95, 2.0, M.generator_G(0.5, 12)), M.LayerDesc(0.6, 5.0, M.RAYLEIGH)], "lambertian", 0.2), 8, None, 19),
    "C2": (lambda: M.config("C2").material, 32, None, 19),
    "C3": (lambda: M.config("C3").material, 64, None, 19),
}
out = os.path.join(ROOT, "gpurun_out"); os.makedirs(out, exist_ok=True)
for name in sys.argv[1:]:
    mk, N, mu_in, nd = CASES[name]
    desc = mk()
    tmp = tempfile.mkdtemp()
    mat = V.Material.load(desc.write(tmp, "m"))
    nodes, _ = O.quadrature(N)
    mu = nodes if mu_in is None else np.asarray(mu_in, float)
    ident = np.eye(4).ravel()
    res = {}
    try:
        pl = V.Plan(mat, V.options(N), mu, nd, ident)
        res["table"] = pl.table(); res["up"] = pl.up()
        S = len({(l.omega, l.coeffs.tobytes()) for l in desc.layers})
        wr, wi, rr, nu = pl.modes(S)
        res.update(wr=wr, wi=wi, res=rr, nu=nu)
        t = pl.run(3); res["t"] = t
        res["last"] = pl.last.message.decode()
    except V.VrteError as e:
        res["error"] = str(e)
    try:
        b = V.compute_brdf(mat, V.options(N), mu, nd)
        res["table_default"] = b.table(); res["stats"] = json.dumps(b.device_stats())
    except V.VrteError as e:
        res["error2"] = str(e)
    big = N >= 64
    if big: res.pop("up", None); res.pop("table_default", None)
    np.savez_compressed(os.path.join(out, f"dump_{name}.npz"), mu=mu, **res)
    print(name, "t=%s" % res.get("t"), res.get("error"), res.get("error2"), res.get("stats"), flush=True)
