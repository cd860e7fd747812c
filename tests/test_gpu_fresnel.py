"""Fresnel top interface (extension; absent from the
reference, so there is no oracle): validated against closed forms and physical
properties, with an independent numpy restatement of the Fresnel matrices and
the split quadrature here.

* pure absorber over a Lambertian base: the DOM answer in closed form (beam
  refracted and attenuated along mu0', base reflection, the internal
  reflections between interface and base as a geometric series over the
  quadrature, exit through T_out / n^2) -- checks T_in, T_out, R and the
  radiance / irradiance factors to 1e-12;
* reciprocity of the scattering table on a square grid (mu_in = the table's
  own exit directions), as satisfied by the table without an interface;
* energy: a lossless slab over a white base returns everything but the outer
  specular reflection, 1 - R_ext(mu0);
* the interface's input validation and the paths that do not model it.
"""
import numpy as np
import pytest

import paper_1707_05882_b200 as V
import pyoracle as O
from paper_1707_05882_b200 import materials as M

from helpers import product_material

pytestmark = pytest.mark.gpu


def amp(n1, n2, c1):
    s2 = (n1 / n2) ** 2 * (1 - c1 * c1)
    c2 = np.sqrt(1 - s2 + 0j) if s2 <= 1 else 1j * np.sqrt(s2 - 1)
    rs = (n1 * c1 - n2 * c2) / (n1 * c1 + n2 * c2)
    rp = (n2 * c1 - n1 * c2) / (n2 * c1 + n1 * c2)
    ts = 2 * n1 * c1 / (n1 * c1 + n2 * c2)
    tp = 2 * n1 * c1 / (n2 * c1 + n1 * c2)
    return rs, rp, ts, tp, c2


def mueller(p, s, k):
    pp, ss, x = abs(p) ** 2, abs(s) ** 2, p * np.conj(s)
    return k * np.array([[0.5 * (pp + ss), 0.5 * (pp - ss), 0, 0], [0.5 * (pp - ss), 0.5 * (pp + ss), 0, 0],
                         [0, 0, x.real, x.imag], [0, 0, -x.imag, x.real]])


def R_in(n, mu):
    rs, rp, *_ = amp(n, 1.0, mu)
    return mueller(rp, rs, 1.0)


def T_in(n, mu_out):
    rs, rp, ts, tp, c2 = amp(1.0, n, mu_out)
    return mueller(tp, ts, n * c2.real / mu_out)


def T_out(n, mu):
    rs, rp, ts, tp, c2 = amp(n, 1.0, mu)
    return mueller(tp, ts, c2.real / (n * mu)) if c2.real > 0 else np.zeros((4, 4))


def split_quadrature(N, n):
    mu_c = np.sqrt(1 - 1 / n ** 2)
    hi = (N + 1) // 2
    x, w = np.polynomial.legendre.leggauss(N - hi)
    xl, wl = mu_c * 0.5 * (x + 1), mu_c * 0.5 * w
    x, w = np.polynomial.legendre.leggauss(hi)
    xh, wh = mu_c + (1 - mu_c) * 0.5 * (x + 1), (1 - mu_c) * 0.5 * w
    return np.concatenate([xl, xh]), np.concatenate([wl, wh]), N - hi


def slab(coeffs, omega, tau, base, albedo, n):
    d = M.MaterialDesc([M.LayerDesc(omega, tau, np.asarray(coeffs, float))], base=base, albedo=albedo)
    d.interface_n = n
    return d


def test_pure_absorber_matches_the_closed_form():
    n, tau, rho, N = 1.5, 0.8, 0.3, 8
    mu0 = np.array([0.35, 0.9])
    b = V.compute_brdf(product_material(slab(M.RAYLEIGH, 0.0, tau, "lambertian", rho, n)), V.options(N), mu0, 3)
    g = b.table()
    nodes, w, lo = split_quadrature(N, n)
    mu_air = np.sqrt(1 - n * n * (1 - nodes[lo:] ** 2))
    assert np.allclose(b.mu_out(), mu_air, rtol=0, atol=1e-14)
    denom = 1 - 2 * rho * sum(w[j] * nodes[j] * R_in(n, nodes[j])[0, 0] * np.exp(-2 * tau / nodes[j]) for j in range(N))
    for ii, m0 in enumerate(mu0):
        m0p = np.sqrt(1 - (1 - m0 * m0) / n ** 2)
        Ti = T_in(n, m0)
        for k, i in enumerate(range(lo, N)):
            u = rho / np.pi * np.exp(-tau / nodes[i]) / denom
            ex = np.outer(T_out(n, nodes[i])[:, 0] / n ** 2 * u, m0 * Ti[0, :] * np.exp(-tau / m0p)) / m0
            for ip in range(3):
                assert np.abs(g[ii, k, ip] - ex).max() < 1e-12 * np.abs(ex).max(), (ii, k, ip)


def test_reciprocity_on_a_square_grid():
    """F(a -> b, dphi) = D F(b -> a, -dphi)^T D, D = diag(1, 1, -1, 1), on
    mu_in = the exit directions; holds for the table without an interface to
    roundoff (the oracle: 2e-11), and with it to the same level -- a check of
    the interface matrices' U/V conventions as well."""
    w = M.config("C1")

    def recip_err(n):
        desc = slab(w.material.layers[0].coeffs, 0.95, 1.0, "lambertian", 0.1, n)
        mat = product_material(desc)
        mu = V.compute_brdf(mat, V.options(8), [0.5], 5).mu_out()
        F = V.compute_brdf(mat, V.options(8), mu, 5).table()
        D = np.diag([1.0, 1.0, -1.0, 1.0])
        err = 0.0
        for a in range(len(mu)):
            for c in range(len(mu)):
                for ip in range(5):
                    lhs = F[a, c, ip]
                    rhs = D @ F[c, a, (-ip) % 5].T @ D
                    err = max(err, np.abs(lhs - rhs).max() / np.abs(F[a, c, ip]).max())
        return err

    e0, e1 = recip_err(1.0), recip_err(1.5)
    assert e0 < 1e-9
    assert e1 < max(10 * e0, 1e-9), (e0, e1)


def test_lossless_slab_returns_all_but_the_outer_specular_reflection():
    n, N = 1.5, 16
    mu0 = np.array([0.3, 0.7, 1.0])
    b = V.compute_brdf(product_material(slab(M.ISOTROPIC, 1.0, 10.0, "lambertian", 1.0, n)), V.options(N), mu0, 7,
                       basis=np.eye(4).ravel())
    for ii, m0 in enumerate(mu0):
        rs, rp, *_ = amp(1.0, n, m0)
        R_ext = 0.5 * (abs(rs) ** 2 + abs(rp) ** 2)
        assert b.reflectance(ii)[0] == pytest.approx(1.0 - R_ext, abs=1e-3), m0


def test_interface_validation_and_unsupported_paths(tmp_path):
    bad = slab(M.ISOTROPIC, 0.5, 1.0, "black", 0.0, 0.8)
    with pytest.raises(V.VrteError) as e:
        product_material(bad)
    assert e.value.code == 2 and "interface: refractive index" in e.value.message
    mat = product_material(slab(M.ISOTROPIC, 0.5, 1.0, "black", 0.0, 1.33))
    with pytest.raises(V.VrteError) as e:
        V.solve_radiance(mat, V.options(8), [0.0])
    assert e.value.code == 2 and "BRDF-only" in e.value.message
    # n = 1 is the reference's model exactly (no interface)
    one = product_material(slab(M.ISOTROPIC, 0.5, 1.0, "black", 0.0, 1.0))
    ref = product_material(slab(M.ISOTROPIC, 0.5, 1.0, "black", 0.0, 1.0 + 0.0))
    assert np.array_equal(V.compute_brdf(one, V.options(8), [0.5], 5).table(),
                          V.compute_brdf(ref, V.options(8), [0.5], 5).table())


def test_c3_with_a_fresnel_interface():
    w = M.config("C3F")
    nodes, _ = O.quadrature(w.N)
    b = V.compute_brdf(product_material(w.material), V.options(w.N), nodes[::8], 19)
    g = b.table()
    st = b.device_stats()
    mu_out = b.mu_out()
    assert g.shape == (8, 32, 19, 4, 4) and np.all(np.isfinite(g))
    assert np.all(np.diff(mu_out) > 0) and 0 < mu_out[0] and mu_out[-1] < 1
    assert st["max_eigen_residual"] < 1e-9 and st["boundary_fallback"] == 0
    assert np.all(g[..., 0, 0] >= 0)
