"""Kernel-level checks of the dense building blocks against numpy/LAPACK
(the reference's PartialPivLU call sites boundary.cpp:230 and the eigen
basis inverse), on sizes and pivoting patterns the BRDF path produces."""
import numpy as np
import pytest

import paper_1707_05882_b200 as V

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G,batch,ncol", [(1, 2, 3), (7, 3, 5), (64, 2, 16), (100, 3, 37),
                                          (256, 4, 256), (1024, 2, 96), (1536, 1, 8)])
def test_row_major_lu_solve_matches_lapack(G, batch, ncol):
    rng = np.random.default_rng(G * 7 + batch)
    A = rng.standard_normal((batch, G, G))
    # graded rows/columns like the boundary system (attenuation factors)
    A *= np.exp(-rng.uniform(0, 6, (batch, G, 1))) * np.exp(-rng.uniform(0, 3, (batch, 1, G)))
    B = rng.standard_normal((batch, G, ncol))
    X = V.lu_solve(A, B)
    for b in range(batch):
        ref = np.linalg.solve(A[b], B[b])
        res = np.abs(A[b] @ X[b] - B[b]).max() / (np.abs(A[b]).max() * np.abs(X[b]).max() * G)
        assert res < 1e-15, res
        assert np.abs(X[b] - ref).max() <= 1e-8 * np.abs(ref).max()


def test_row_major_lu_pivots_like_lapack():
    # exact ties and a zero leading pivot: first-index argmax, row interchanges
    A = np.array([[[0.0, 2.0, 1.0], [3.0, 1.0, 0.0], [3.0, 0.0, 5.0]]])
    B = np.eye(3)[None]
    X = V.lu_solve(A, B)
    assert np.allclose(X[0] @ A[0], np.eye(3), atol=1e-15)


def test_row_major_lu_reports_singular():
    A = np.zeros((1, 8, 8))
    with pytest.raises(V.VrteError):
        V.lu_solve(A, np.ones((1, 8, 1)))
