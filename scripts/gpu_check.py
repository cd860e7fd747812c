"""Quick GPU-vs-oracle check used during development (run under gpurun)."""
import os, sys, time, json, tempfile
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1707_05882_b200 as V
from paper_1707_05882_b200 import materials as M
import pyoracle as O

def parity(g, r):
    r00 = np.abs(r[..., 0, 0])[..., None, None]
    den = np.maximum(np.abs(r), 1e-3 * r00)
    den = np.where(den == 0, 1e-300, den)
    return float(np.max(np.abs(g - r) / den))

def omat(desc):
    bt = {"black": 0, "lambertian": 1, "mueller_table": 2}[desc.base]
    return O.Material(np.array([l.omega for l in desc.layers]), np.array([l.tau for l in desc.layers]),
                      desc.padded_coeffs(), bt, desc.albedo, desc.table)

def run(name, desc, N, mu_in=None, n_dphi=19, oracle=True):
    tmp = tempfile.mkdtemp()
    path = desc.write(tmp, "m")
    mat = V.Material.load(path)
    nodes, _ = O.quadrature(N)
    mu = nodes if mu_in is None else np.asarray(mu_in)
    t = time.time()
    try:
        b = V.compute_brdf(mat, V.options(N), mu, n_dphi)
    except V.VrteError as e:
        print(name, "GPU ERROR", e); return
    tg = time.time() - t
    g = b.table()
    st = b.device_stats()
    line = {"case": name, "N": N, "gpu_s": round(tg, 4), "stats": {k: (float(v) if isinstance(v, float) else int(v)) for k, v in st.items()}}
    if oracle:
        t = time.time()
        r, tm = O.brdf(omat(desc), N, mu, n_dphi)
        line["oracle_s"] = round(time.time() - t, 3)
        line["parity"] = parity(g, r)
        line["maxabs"] = float(np.abs(g - r).max())
        line["oracle_maxres"] = tm["max_eigen_residual"]
    print(json.dumps(line), flush=True)

if __name__ == "__main__":
    which = sys.argv[1:] or ["small"]
    D = "/root/repo/tests/golden/data"
    if "small" in which:
        run("iso_half_N4", M.single_layer(M.ISOTROPIC, 0.5, 1.0), 4, [0.6, 1.0], 5)
        run("rayleigh_N6", M.single_layer(M.RAYLEIGH, 0.9, 1.0, "lambertian", 0.3), 6, [0.7], 6)
        run("full_N5", M.single_layer(M.FULL, 0.85, 1.0, "lambertian", 0.2), 5, None, 7)
        w = M.config("C1"); run("C1", w.material, w.N)
        run("paint_N8", M.MaterialDesc([M.LayerDesc(0.95, 2.0, M.generator_G(0.5, 12)), M.LayerDesc(0.6, 5.0, M.RAYLEIGH)], "lambertian", 0.2), 8)
        run("conservative_N8", M.single_layer(M.ISOTROPIC, 1.0, 10.0, "lambertian", 1.0), 8)
    if "c2" in which:
        w = M.config("C2"); run("C2", w.material, w.N)
    if "c3p" in which:
        w = M.config("C3")
        nodes, _ = O.quadrature(64)
        run("C3_partial", w.material, 64, nodes[[0, 31, 63]])
    if "c3" in which:
        w = M.config("C3"); run("C3_gpu_only", w.material, 64, oracle=False)
