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


@pytest.mark.parametrize("d,batch", [(4, 2), (32, 3), (100, 2), (256, 3), (512, 2), (520, 1)])
@pytest.mark.parametrize("blocked", [True, False])
def test_hessenberg_reduction(d, batch, blocked):
    rng = np.random.default_rng(d + batch)
    # graded like F E (row/column scales 1 .. 1e6)
    sc = np.exp(rng.uniform(0, 14, d))
    A = rng.standard_normal((batch, d, d)) * sc[None, :, None] * 1e-3 + np.diag(sc)[None]
    H, Q = V.hessenberg(A, blocked)
    for b in range(batch):
        nrm = np.abs(A[b]).max()
        assert np.abs(np.tril(H[b], -2)).max() == 0.0
        assert np.abs(Q[b].T @ Q[b] - np.eye(d)).max() < 1e-13 * d
        assert np.abs(Q[b] @ H[b] @ Q[b].T - A[b]).max() < 1e-14 * d * nrm


@pytest.mark.parametrize("d,batch", [(16, 4), (64, 3), (256, 2)])
def test_schur_form_of_graded_matrices(d, batch):
    rng = np.random.default_rng(7 * d + batch)
    sc = np.exp(rng.uniform(0, 14, d))  # graded like F E (1 .. 1e6)
    A = rng.standard_normal((batch, d, d)) * 1e-2 * np.sqrt(sc[None, :, None] * sc[None, None, :]) + np.diag(sc)[None]
    T, Z, lam = V.schur(A)
    for b in range(batch):
        nrm = np.abs(A[b]).max()
        assert np.abs(np.tril(T[b], -2)).max() == 0.0
        assert np.abs(Z[b].T @ Z[b] - np.eye(d)).max() < 1e-13 * d
        assert np.abs(Z[b] @ T[b] @ Z[b].T - A[b]).max() < 1e-14 * d * nrm
        ref = np.sort_complex(np.linalg.eigvals(A[b]))
        got = np.sort_complex(lam[b])
        assert np.abs(got - ref).max() < 1e-12 * nrm


def test_qr_converges_through_underflowing_bulge():
    # Trailing 3x3 block with a repeated diagonal entry and a subdiagonal of
    # 1e-182: the Ahues-Kressner test cannot deflate it (bb = 0), so the QR
    # sweep must keep chasing a bulge whose squared entries underflow
    # (LAPACK dlarfg: tau = 2 sign flip, not the identity).  This stalled the
    # round-1 kernels on a C4 order (m = 151, d = 512).
    d = 12
    H = np.triu(np.random.default_rng(3).standard_normal((d, d))) * 1e-3 + np.diag(np.linspace(2.0, 8.0, d))
    for k in range(1, d):
        H[k, k - 1] = 1e-3
    a = 1.000175
    H[d - 2, d - 2] = H[d - 1, d - 1] = a
    H[d - 2, d - 1] = 2.8e-33
    H[d - 1, d - 2] = -3.0e-182
    T, Z, lam = V.schur(H[None])
    assert np.isfinite(T).all()
    assert np.abs(Z[0] @ T[0] @ Z[0].T - H).max() < 1e-13
    ref = np.sort_complex(np.linalg.eigvals(H))
    assert np.abs(np.sort_complex(lam[0]) - ref).max() < 1e-12


@pytest.mark.parametrize("G,ncols,batch", [(384, 384, 3), (1024, 1280, 4), (1000, 1100, 2), (2048, 2056, 1)])
def test_lu_lookahead_schedule_is_bitwise_identical(G, ncols, batch):
    """The boundary stage's look-ahead schedule (panels of block K+1 under the
    rest of block K's trailing update, lu.cu) performs the same operations on
    every row as the serial schedule: identical factors and row maps; and the
    factors reproduce P A = L U on the augmented columns too."""
    rng = np.random.default_rng(G + ncols)
    A = rng.standard_normal((batch, G, ncols))
    A *= np.exp(-rng.uniform(0, 6, (batch, G, 1)))
    F1, p1 = V.lu_factor(A, G, lookahead=True)
    F0, p0 = V.lu_factor(A, G, lookahead=False)
    assert np.array_equal(p0, p1)
    assert np.array_equal(F0, F1)
    for b in range(batch):
        P = F1[b][p1[b]]  # position order
        Lm = np.tril(P[:, :G], -1) + np.eye(G)
        U = np.triu(P[:, :G])
        PA = A[b][p1[b]]
        assert np.abs(Lm @ U - PA[:, :G]).max() <= 1e-13 * np.abs(A[b]).max() * np.sqrt(G)
        if ncols > G:  # the carried columns hold L^-1 P B
            assert np.abs(Lm @ P[:, G:] - PA[:, G:]).max() <= 1e-13 * np.abs(A[b]).max() * np.sqrt(G)


@pytest.mark.parametrize("G,ncols,batch", [(1024, 1280, 3), (1000, 1100, 2), (384, 640, 2)])
def test_deferred_right_hand_sides_are_bitwise_the_augmented_elimination(G, ncols, batch):
    """The BRDF pipeline factors the boundary system before its right-hand sides
    exist and eliminates them afterwards through the row map saved after each
    outer block's panels (lu.cu LuRhsDefer): identical to carrying them along,
    in both schedules."""
    rng = np.random.default_rng(3 * G + ncols)
    A = rng.standard_normal((batch, G, ncols))
    A *= np.exp(-rng.uniform(0, 6, (batch, G, 1)))
    F0, p0 = V.lu_factor(A, G, lookahead=True)
    F1, p1 = V.lu_factor(A, G, lookahead=True, deferred=True)
    F2, p2 = V.lu_factor(A, G, lookahead=False, deferred=True)
    assert np.array_equal(p0, p1) and np.array_equal(p0, p2)
    assert np.array_equal(F0, F1)
    assert np.array_equal(F0, F2)
