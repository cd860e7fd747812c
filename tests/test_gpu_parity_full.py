"""Headline parity on FULL tables: C3 (all 64 x 64 x 19 Mueller matrices) and
the C5 bands 0/15/30, GPU through the C ABI against the oracle (tests only:
boundary LU memoized across incidents, bit-identical to the per-incident
factorization), in accurate mode (every mode polished, every solve refined:
the reference's algorithm at its fp64 limit) and as written.

Measured on the B200 (profiles/parity_r02.json, scripts/parity_full.py):

                         GPU vs accurate          reference-as-written vs accurate
  per matrix max|d|/max|M|   3.7e-11 .. 8.7e-11     1.4e-9 .. 3.4e-9
  SURVEY §8(d) metric        5.4e-9  .. 3.2e-8      1.6e-6 .. 4.7e-6
  matrices with SURVEY <= 1e-9   99.79% .. 99.98%

The SURVEY metric floors the denominator at 1e-3 |M00|; at grazing incidence /
exit (mu < 0.01) some entries of the exact answer itself move by up to 3.8e-8
in that metric under a 1e-15 relative change of omega
(accurate_rounding_sensitivity_survey), i.e. 1e-9 per element is below the
fp64 conditioning of the problem there; the reference implementation is 2e-6
off.  Asserted (tolerances with margin over the measurement):
  * per matrix vs accurate                         <= 2e-10
  * SURVEY metric <= 1e-9 on >= 99.5% of the matrices
  * SURVEY metric vs accurate <= 2% of the reference's own error (and <= 5e-8)
  * vs the oracle AS WRITTEN: the difference is the reference's own error
    (SURVEY <= 1.05 x |ref - accurate| + 1e-9, per matrix <= 1.05 x + 1e-10)
"""
import numpy as np
import pytest

import paper_1707_05882_b200 as V
import pyoracle as O
from paper_1707_05882_b200 import materials as M

from helpers import matrix_metric, oracle_material, product_material, survey_metric, survey_per_matrix

pytestmark = pytest.mark.gpu

CASES = [("C3", 0), ("C5", 0), ("C5", 15), ("C5", 30)]


@pytest.fixture(scope="module", params=CASES, ids=lambda c: f"{c[0]}b{c[1]}" if c[0] == "C5" else c[0])
def tables(request):
    cfg, band = request.param
    w = M.config(cfg, band)
    nodes, _ = O.quadrature(w.N)
    b = V.compute_brdf(product_material(w.material), V.options(w.N), nodes, 19)
    g = b.table()
    om = oracle_material(w.material)
    with O.cached_boundary():
        r, _ = O.brdf(om, w.N, nodes, 19)
        with O.accurate():
            a, _ = O.brdf(om, w.N, nodes, 19)
    return w.name, g, r, a, b.device_stats()


def test_full_table_vs_accurate_oracle(tables):
    name, g, r, a, st = tables
    assert g.shape == (64, 64, 19, 4, 4)
    assert matrix_metric(g, a) <= 2e-10, name
    frac = float((survey_per_matrix(g, a) <= 1e-9).mean())
    assert frac >= 0.995, (name, frac)
    own = survey_metric(r, a)
    err = survey_metric(g, a)
    assert err <= min(0.02 * own, 5e-8), (name, err, own)


def test_full_table_vs_oracle_as_written(tables):
    name, g, r, a, st = tables
    assert survey_metric(g, r) <= 1.05 * survey_metric(r, a) + 1e-9, name
    assert matrix_metric(g, r) <= 1.05 * matrix_metric(r, a) + 1e-10, name


def test_gates_on_full_tables(tables):
    name, g, r, a, st = tables
    assert st["max_eigen_residual"] < 1e-10
    assert st["max_boundary_residual"] < 1e-10 and st["boundary_refined"] == 0
    assert st["max_balance_residual"] < 1e-6
