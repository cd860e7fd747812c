"""Generate the committed golden fixtures for the parity tests (TEST INFRASTRUCTURE).

For each small case this writes tests/golden/<case>.npz with
  exact   : the mpmath restatement at 32 digits (oracle/mp_oracle.py) -- the
            discrete-ordinate solution with no fp64 rounding
  oracle  : the fp64 CPU restatement (oracle/vrte_oracle.cpp, LAPACK)
  mu_in, N, n_dphi and the material description.
Run here (CPU, no GPU needed):  python tests/golden/gen_golden.py [case ...]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import mp_oracle as MP  # noqa: E402
import pyoracle as O  # noqa: E402
from paper_1707_05882_b200 import materials as M  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def cases():
    nodes = lambda n: O.quadrature(n)[0]
    return {
        # test_capi.cpp:85-119 BRDF case
        "iso_half_N4": (M.single_layer(M.ISOTROPIC, 0.5, 1.0), 4, [0.6, 1.0], 5),
        "rayleigh_lam_N6": (M.single_layer(M.RAYLEIGH, 0.9, 1.0, "lambertian", 0.3), 6, [0.7], 6),
        "full_lam_N5": (M.single_layer(M.FULL, 0.85, 1.0, "lambertian", 0.2), 5, nodes(5), 7),
        "vacuum_N4": (M.single_layer(M.ISOTROPIC, 0.0, 1.0), 4, [0.6], 8),
        "paint_N6": (M.MaterialDesc([M.LayerDesc(0.95, 2.0, M.generator_G(0.5, 12)),
                                     M.LayerDesc(0.6, 5.0, M.RAYLEIGH)], "lambertian", 0.2),
                     6, nodes(6)[[0, 2, 5]], 9),
        "C1": (M.config("C1").material, 8, nodes(8), 19),
    }


def omat(desc):
    bt = {"black": 0, "lambertian": 1, "mueller_table": 2}[desc.base]
    return O.Material(np.array([l.omega for l in desc.layers]), np.array([l.tau for l in desc.layers]),
                      desc.padded_coeffs(), bt, desc.albedo, desc.table)


def main(names):
    allc = cases()
    for name in names or list(allc):
        desc, N, mu, nd = allc[name]
        mu = np.asarray(mu, float)
        t = time.time()
        oracle, tm = O.brdf(omat(desc), N, mu, nd)
        exact = MP.brdf([l.omega for l in desc.layers], [l.tau for l in desc.layers],
                        desc.padded_coeffs(), {"black": 0, "lambertian": 1}[desc.base],
                        desc.albedo, N, mu, nd)
        meta = {"N": N, "n_dphi": nd, "base": desc.base, "albedo": desc.albedo,
                "layers": [{"omega": l.omega, "tau": l.tau} for l in desc.layers]}
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), exact=exact, oracle=oracle, mu_in=mu,
                            coeffs=desc.padded_coeffs(), meta=json.dumps(meta))
        sc = np.abs(exact).reshape(exact.shape[:3] + (16,)).max(-1)[..., None, None]
        sc = np.where(sc == 0, 1.0, sc)
        print(name, "%.1fs" % (time.time() - t), "oracle-vs-exact (rel. to matrix max) %.2e"
              % (np.abs(oracle - exact) / sc).max(), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
