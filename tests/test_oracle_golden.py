"""Pin the CPU oracle to the reference's own golden values and oracle identities.

Ports of the reference known-answer tests:
quadrature (test_core.cpp:30-68), Wigner explicit sums (oracles.hpp:24-41,
test_phase.cpp:14-43), kernel parity / isotropic structure (test_phase.cpp:
78-161), E/F kernel-vs-stacked routes (test_homogeneous.cpp:77-89), vacuum
spectrum (:91-113), residual bound (:115-129), conjugate pairs (:131-150),
diffusion nu golden (:191-207), particular golden Z and reduced-vs-unreduced
(test_particular.cpp:67-110), dither (:139-160).
"""
import math

import numpy as np
import pytest

import pyoracle as O
from paper_1707_05882_b200 import materials as M


def mat(coeffs, omega=0.5, tau=1.0, base=0, rho=0.0):
    c = np.asarray(coeffs, float)
    return O.Material(np.array([omega]), np.array([tau]), c[None], base, rho)


# ------------------------------------------------------------ quadrature
def test_quadrature_one_point_is_midpoint():
    n, w = O.quadrature(1)
    assert n[0] == pytest.approx(0.5, rel=1e-15) and w[0] == pytest.approx(1.0, rel=1e-15)


def test_quadrature_two_point_roots():
    n, w = O.quadrature(2)
    assert n[0] == pytest.approx(0.5 - 1 / (2 * math.sqrt(3)), rel=1e-13)
    assert n[1] == pytest.approx(0.5 + 1 / (2 * math.sqrt(3)), rel=1e-13)
    assert np.allclose(w, 0.5, rtol=1e-14)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 13, 16, 64])
def test_quadrature_exactness(n):
    x, w = O.quadrature(n)
    assert abs(w.sum() - 1) < 1e-12
    for k in range(2 * n):
        assert abs((w * x ** k).sum() - 1.0 / (k + 1)) < 1e-12
    assert np.all(np.diff(x) > 0) and x[0] > 0 and x[-1] < 1


# ------------------------------------------------------------ Wigner / GSF
def wigner_explicit(l, m, n, theta):
    """oracles.hpp:24-41 explicit finite sum."""
    if l < max(abs(m), abs(n)):
        return 0.0
    f = math.factorial
    c, s = math.cos(theta / 2), math.sin(theta / 2)
    pref = math.sqrt(f(l + m) * f(l - m) * f(l + n) * f(l - n))
    tot = 0.0
    for k in range(max(0, n - m), min(l + n, l - m) + 1):
        den = f(l + n - k) * f(k) * f(m - n + k) * f(l - m - k)
        sg = 1.0 if (m - n + k) % 2 == 0 else -1.0
        tot += sg * c ** (2 * l + n - m - 2 * k) * s ** (m - n + 2 * k) / den
    return pref * tot


def test_wigner_recurrence_matches_explicit_sum():
    rng = np.random.default_rng(7)
    for m in (0, 1, 2, 3, 7, 12):
        for n in (0, 2, -2):
            for x in rng.uniform(-1, 1, 6):
                seq = O.wigner_d_sequence(m, n, 20, x)
                for l in range(21):
                    ex = wigner_explicit(l, m, n, math.acos(x))
                    assert abs(seq[l] - ex) <= 1e-11 * max(1.0, abs(ex))


def test_wigner_spot_values():
    th = 0.7
    c, s = math.cos(th), math.sin(th)
    assert wigner_explicit(1, 0, 0, th) == pytest.approx(c, rel=1e-14)
    assert wigner_explicit(1, 1, 0, th) == pytest.approx(-s / math.sqrt(2), rel=1e-14)
    assert wigner_explicit(2, 0, 2, th) == pytest.approx(math.sqrt(6) / 4 * s * s, rel=1e-14)
    assert wigner_explicit(2, 2, 2, th) == pytest.approx(0.25 * (1 + c) ** 2, rel=1e-14)
    assert wigner_explicit(2, 2, -2, th) == pytest.approx(0.25 * (1 - c) ** 2, rel=1e-14)


def test_gsf_parity_identity():
    # Pi(-mu) = (-1)^(l-m) D Pi(mu) D : P, R even/odd with l-m, T flips sign extra
    for m in (0, 1, 2, 4):
        for mu in (0.15, 0.5, 0.93):
            p1, r1, t1 = O.gsf_sequence(m, 7, mu)
            p2, r2, t2 = O.gsf_sequence(m, 7, -mu)
            for l in range(m, 8):
                s = (-1) ** (l - m)
                assert abs(p2[l] - s * p1[l]) < 1e-12
                assert abs(r2[l] - s * r1[l]) < 1e-12
                assert abs(t2[l] + s * t1[l]) < 1e-12


# ------------------------------------------------------------ kernels
def test_isotropic_kernel_structure():
    k = O.kernel_blocks(mat(M.ISOTROPIC, 0.9), 0, 4, 0)
    e = np.zeros((4, 4))
    e[0, 0] = 1.0
    for blocks in (k[0], k[1], k[2]):
        assert np.abs(blocks - e).max() < 1e-14
    wide = np.zeros((3, 4, 4))
    wide[0] = M.ISOTROPIC[0]
    k1 = O.kernel_blocks(mat(wide, 0.9), 0, 4, 1)
    assert np.abs(k1[0]).max() == 0.0


def test_kernel_parity_identity():
    D = np.diag([1, 1, -1, -1.0])
    for m in range(4):
        pp, pm, mp_, mm = O.kernel_blocks(mat(M.FULL, 0.8), 0, 5, m)
        assert np.abs(mm - D @ pp @ D).max() < 1e-12
        assert np.abs(mp_ - D @ pm @ D).max() < 1e-12


def stacked_ef(coeffs, omega, N, m):
    """homogeneous.cpp:75-107 stacked GSF route, restated in numpy."""
    x, w = O.quadrature(N)
    d, L = 4 * N, len(coeffs)
    D4 = np.diag([1, 1, -1, -1.0])
    se, sf = np.zeros((d, d)), np.zeros((d, d))
    tabs = [O.gsf_sequence(m, L - 1, xi) for xi in x]
    for l in range(m, L):
        Pi = np.zeros((d, 4))
        for i, (p, r, t) in enumerate(tabs):
            Pi[4 * i:4 * i + 4] = [[p[l], 0, 0, 0], [0, r[l], -t[l], 0], [0, -t[l], r[l], 0], [0, 0, 0, p[l]]]
        s = -1 if (l - m) % 2 else 1
        se += Pi @ (coeffs[l] @ (np.eye(4) + s * D4)) @ Pi.T
        sf += Pi @ (coeffs[l] @ (np.eye(4) - s * D4)) @ Pi.T
    W = np.diag(np.repeat(w, 4))
    Minv = np.diag(1 / np.repeat(x, 4))
    return (np.eye(d) - omega / 2 * se @ W) @ Minv, (np.eye(d) - omega / 2 * sf @ W) @ Minv


@pytest.mark.parametrize("coeffs,omega", [(M.RAYLEIGH, 0.7), (M.FULL, 0.95)])
def test_reduced_operators_two_routes(coeffs, omega):
    for m in range(len(coeffs)):
        e, f = O.reduced_ops(mat(coeffs, omega), 0, 5, m)
        e2, f2 = stacked_ef(coeffs, omega, 5, m)
        sc = np.abs(e).max()
        assert np.abs(e - e2).max() < 1e-12 * sc and np.abs(f - f2).max() < 1e-12 * sc


def test_reduced_operators_vacuum():
    e, f = O.reduced_ops(mat(M.ISOTROPIC, 0.0), 0, 3, 0)
    x, _ = O.quadrature(3)
    assert np.allclose(np.diag(e), 1 / np.repeat(x, 4))
    assert np.abs(e - f).max() == 0.0


# ------------------------------------------------------------ homogeneous
def test_vacuum_spectrum_is_node_cosines_times_four():
    nu, _ = O.homogeneous(mat(M.ISOTROPIC, 0.0), 0, 4, 0)
    x, _ = O.quadrature(4)
    assert np.all(np.abs(nu.imag) < 1e-12)
    counts = [int(np.sum(np.abs(nu.real - xi) < 1e-10)) for xi in x]
    assert counts == [4, 4, 4, 4]


@pytest.mark.parametrize("coeffs,omega", [(M.ISOTROPIC, 0.99), (M.RAYLEIGH, 0.9), (M.FULL, 0.85)])
def test_mode_residual_bound(coeffs, omega):
    for m in range(len(coeffs)):
        nu, res = O.homogeneous(mat(coeffs, omega), 0, 8, m)
        assert res.max() < 1e-9 and np.all(nu.real > 0)


def test_conjugate_pairs():
    for m in range(4):
        nu, _ = O.homogeneous(mat(M.FULL, 0.9), 0, 6, m)
        for v in nu:
            if abs(v.imag) < 1e-12 * abs(v):
                continue
            assert np.min(np.abs(nu - np.conj(v))) < 1e-9 * abs(v)


def diffusion_nu(N, omega):
    """test_homogeneous.cpp:27-49 characteristic equation by bisection."""
    x, w = O.quadrature(N)
    f = lambda nu: 1 - omega * np.sum(w / (1 - x * x / (nu * nu)))
    lo = x[-1] * (1 + 1e-12)
    while f(lo) > 0:
        lo = x[-1] + 0.5 * (lo - x[-1])
    hi = 1e6
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        lo, hi = (mid, hi) if f(mid) <= 0 else (lo, mid)
    return 0.5 * (lo + hi)


def test_diffusion_mode_golden():
    nu, _ = O.homogeneous(mat(M.ISOTROPIC, 0.99), 0, 8, 0)
    largest = nu.real.max()
    assert largest == pytest.approx(diffusion_nu(8, 0.99), rel=1e-10)
    assert largest == pytest.approx(5.79672945130218, rel=1e-10)  # test_homogeneous.cpp:206


# ------------------------------------------------------------ particular
def unreduced_particular(coeffs, omega, N, m, k, mu0, stokes):
    """unreduced.hpp:14-38: dense 8N solve ((1/mu0) M + I - (omega/2) A w) z = x."""
    x, w = O.quadrature(N)
    d = 4 * N
    pp, pm, mp_, mm = O.kernel_blocks(mat(coeffs, omega), 0, N, m)
    sys_ = np.zeros((2 * d, 2 * d))
    c = omega / 2
    for i in range(N):
        for j in range(N):
            for blk, (r0, c0) in ((pp, (0, 0)), (pm, (0, d)), (mp_, (d, 0)), (mm, (d, d))):
                sys_[r0 + 4 * i:r0 + 4 * i + 4, c0 + 4 * j:c0 + 4 * j + 4] -= c * w[j] * blk[i, j]
    for i in range(N):
        for cc in range(4):
            sys_[4 * i + cc, 4 * i + cc] += 1 + x[i] / mu0
            sys_[d + 4 * i + cc, d + 4 * i + cc] += 1 - x[i] / mu0
    up, dn = O.beam_column(mat(coeffs, omega), 0, N, m, -mu0)
    sel = np.array([stokes[cc] if ((k == 1) == (cc < 2)) else 0.0 for cc in range(4)])
    sc = omega / (2 * math.pi)
    rhs = np.concatenate([sc * (up @ sel).ravel(), sc * (dn @ sel).ravel()])
    z = np.linalg.solve(sys_, rhs)
    return z[:d], z[d:]


def test_particular_golden_values():
    zp, zm, _, _ = O.particular(mat(M.ISOTROPIC, 0.5), 0, 4, 0, 1, 0.6, [1, 0, 0, 0])
    # test_particular.cpp:107-109
    assert zp[0] == pytest.approx(0.0509350198293183, rel=1e-9)
    assert zm[0] == pytest.approx(0.0642660587264871, rel=1e-9)
    assert zp[12] == pytest.approx(0.0222776908886489, rel=1e-9)


@pytest.mark.parametrize("coeffs,omega", [(M.ISOTROPIC, 0.5), (M.RAYLEIGH, 0.9), (M.FULL, 0.7)])
def test_particular_reduced_matches_unreduced(coeffs, omega):
    st = [1.0, 0.3, -0.2, 0.1]
    for m in range(len(coeffs)):
        for k in (1, 2):
            zp, zm, _, res = O.particular(mat(coeffs, omega), 0, 4, m, k, 0.6, st)
            up, dn = unreduced_particular(coeffs, omega, 4, m, k, 0.6, st)
            sc = max(np.abs(up).max(), np.abs(dn).max(), 1e-30)
            assert np.abs(zp - up).max() < 1e-10 * sc and np.abs(zm - dn).max() < 1e-10 * sc
            assert res < 1e-9


def test_particular_dither_at_resonance():
    nu, _ = O.homogeneous(mat(M.ISOTROPIC, 0.5), 0, 2, 0)
    resonant = [v.real for v in nu if v.real < 1 and abs(v.imag) < 1e-14][-1]
    _, _, mu_eff, res = O.particular(mat(M.ISOTROPIC, 0.5), 0, 2, 0, 1, resonant, [1, 0, 0, 0])
    assert mu_eff != resonant and mu_eff == pytest.approx(resonant * (1 - 1e-7), rel=1e-15)
    assert res < 1e-9


# ------------------------------------------------------------ BRDF properties on the oracle
def test_oracle_vacuum_brdf_is_zero():
    fr, _ = O.brdf(mat(M.ISOTROPIC, 0.0), 4, np.array([0.6]), 8)
    assert np.abs(fr).max() < 1e-12


def test_oracle_basis_invariance_and_ill_conditioned_rejection():
    m = mat(M.RAYLEIGH, 0.9)
    a, _ = O.brdf(m, 6, np.array([0.7]), 6)
    alt = np.array([[1, 0, 0, 0], [1, -0.8, 0, 0], [1, 0.2, 0.7, 0], [1, 0.1, -0.2, 0.6]], float)
    b, _ = O.brdf(m, 6, np.array([0.7]), 6, basis=alt)
    assert np.abs(a - b).max() < 1e-8 * np.abs(a).max()
    bad = np.array([[1, 0, 0, 0], [1, 1e-9, 0, 0], [1, 0, 1, 0], [1, 0, 0, 1]], float)
    with pytest.raises(O.OracleError) as e:
        O.brdf(m, 4, np.array([0.6]), 4, basis=bad)
    assert e.value.code == 2
