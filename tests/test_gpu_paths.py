"""Round-2 paths of the device pipeline, each against the oracle or against
the path it replaces:

* the boundary residual probes (boundary.cuh): the default BRDF path solves the
  R right-hand sides through layer 0 only and checks K = 4 random combinations
  through every row; the forced full-solution fallback (the reference's exact
  per-right-hand-side gate, boundary.cpp:233-257) gives the same table;
* media ordered by expansion length: the free-streaming orders of a short
  expansion are skipped whatever the layer order (C3 with the layers swapped).
"""
import numpy as np
import pytest

import paper_1707_05882_b200 as V
import pyoracle as O
from paper_1707_05882_b200 import materials as M

from helpers import matrix_metric, oracle_material, product_material, survey_metric

pytestmark = pytest.mark.gpu


def test_forced_fallback_matches_the_probe_path():
    w = M.config("C3")
    N = 16
    nodes, _ = O.quadrature(N)
    mat = product_material(w.material)
    b = V.compute_brdf(mat, V.options(N), nodes, 7)
    g = b.table()
    s = b.device_stats()
    assert s["boundary_fallback"] == 0 and 0.0 < s["max_boundary_residual"] < 1e-12
    with V.forced_boundary_fallback():
        bf = V.compute_brdf(mat, V.options(N), nodes, 7)
    gf = bf.table()
    sf = bf.device_stats()
    assert sf["boundary_fallback"] == 1 and sf["boundary_refined"] == 0
    assert 0.0 < sf["max_boundary_residual"] < 1e-12
    assert matrix_metric(gf, g) < 1e-12
    # the radiance path always runs the full gate; the probe path is back afterwards
    b2 = V.compute_brdf(mat, V.options(N), nodes, 7)
    assert b2.device_stats()["boundary_fallback"] == 0 and np.array_equal(b2.table(), g)


@pytest.mark.parametrize("swap", [False, True])
def test_free_streaming_orders_skipped_in_either_layer_order(swap):
    w = M.config("C3")
    layers = list(reversed(w.material.layers)) if swap else w.material.layers
    desc = M.MaterialDesc(layers, base="lambertian", albedo=0.2)
    N = 16
    nodes, _ = O.quadrature(N)
    b = V.compute_brdf(product_material(desc), V.options(N), nodes[::3], 7)
    s = b.device_stats()
    # G(0.6, 64): 64 orders through the eigen pipeline; Rayleigh (L = 3): 3
    assert s["eigen_slots"] == 67
    with O.accurate():
        r, _ = O.brdf(oracle_material(desc), N, nodes[::3], 7)
    assert matrix_metric(b.table(), r) < 2e-10
