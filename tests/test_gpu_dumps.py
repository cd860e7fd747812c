"""The debug dumps of vrte_options (pipeline.cpp:333-357, kernel.cpp:188-214)
in the reference's file formats, checked against the oracle:
  dump_kernel_path  : the Fourier kernel blocks A^m(+-mu_i, +-mu_j) of layer 0
                      (a4, assemble_azimuth_kernel) for every order;
  dump_eigen_path   : lambda, nu and the 8N residual of every mode, sorted as
                      the reference sorts them (homogeneous.cpp:272-276);
  dump_boundary_path: per order the condition lower bound and the residual
                      (one line per order: the matrix is factored once)."""
import csv

import numpy as np
import pytest

import paper_1707_05882_b200 as V
import pyoracle as O
from paper_1707_05882_b200 import materials as M

from helpers import oracle_material, product_material

pytestmark = pytest.mark.gpu


def test_dumps_match_the_oracle(tmp_path):
    w = M.config("C1")
    N = w.N
    kp, ep, bp = (str(tmp_path / f) for f in ("kernel.csv", "eigen.csv", "boundary.csv"))
    o = V.options(N, dump_kernel_path=kp.encode(), dump_eigen_path=ep.encode(), dump_boundary_path=bp.encode())
    nodes, _ = O.quadrature(N)
    V.compute_brdf(product_material(w.material), o, nodes[:2], 5)
    om = oracle_material(w.material)
    L = w.material.order_count
    # kernel blocks
    rows = list(csv.reader(open(kp)))
    assert rows[0] == ["m", "i", "j", "sign_i", "sign_j"] + [f"a{r}{c}" for r in range(4) for c in range(4)]
    assert len(rows) == 1 + L * 4 * N * N
    got = np.array([[float(x) for x in r[5:]] for r in rows[1:]]).reshape(L, 2, 2, N, N, 4, 4)
    for m in range(L):
        pp, pm, mp, mm = O.kernel_blocks(om, 0, N, m)
        ref = np.array([[pp, pm], [mp, mm]])
        assert np.abs(got[m] - ref).max() <= 1e-12 * max(np.abs(ref).max(), 1e-300), m
    # modes
    rows = list(csv.reader(open(ep)))
    assert rows[0] == ["m", "lambda_re", "lambda_im", "nu_re", "nu_im", "residual"]
    body = np.array([[float(x) for x in r] for r in rows[1:]])
    assert body.shape == (L * 4 * N, 6)
    for m in (0, 5, L - 1):
        onu, _ = O.homogeneous(om, 0, N, m)
        g = body[body[:, 0] == m]
        gnu = g[:, 3] + 1j * g[:, 4]
        assert np.all(np.diff(g[:, 3]) <= 0)  # the reference's order: nu_re descending
        for v in onu:
            assert np.min(np.abs(gnu - v)) <= 1e-9 * abs(v)
        assert g[:, 5].max() < 1e-9
    # boundary
    rows = list(csv.reader(open(bp)))
    assert rows[0] == ["m", "condition_estimate", "residual"] and len(rows) == 1 + L
    b = np.array([[float(x) for x in r] for r in rows[1:]])
    assert np.array_equal(b[:, 0], np.arange(L)) and np.all(b[:, 1] >= 1) and np.all(b[:, 2] < 1e-10)


def test_kernel_dump_unwritable_path_is_a_validation_error():
    w = M.config("C1")
    o = V.options(w.N, dump_kernel_path=b"/nonexistent-dir/kernel.csv")
    with pytest.raises(V.VrteError) as e:
        V.compute_brdf(product_material(w.material), o, [0.5], 5)
    assert e.value.code == 2 and "cannot open kernel dump file" in e.value.message
