"""Pin the oracle's radiance-field restatement (SURVEY §8(f) rank 1:
reconstruction.cpp:28-227, pipeline.cpp:253-309, capi.cpp:138-174) to the
reference's own reconstruction tests (test_reconstruction.cpp) and to the
BRDF path it shares state with (brdf.cpp:127-160).  Test infrastructure only.
"""
import math

import numpy as np
import pytest

import pyoracle as O
from paper_1707_05882_b200 import materials as M

from helpers import oracle_material

ISO = np.array([M.greek(1, 0, 0, 0, 0, 0)])


def layer(coeffs, omega, tau):
    return M.LayerDesc(omega, tau, np.asarray(coeffs, float))


def mat(layers, base="black", albedo=0.0, mu0=0.6):
    return M.MaterialDesc(layers, base=base, albedo=albedo, mu0=mu0)


CASES = {
    # test_reconstruction.cpp:23-33
    "iso_half": mat([layer(ISO, 0.5, 1.0)]),
    "rayleigh_lam": mat([layer(M.RAYLEIGH, 0.9, 2.0)], "lambertian", 0.3),
    "two_layer": mat([layer(M.RAYLEIGH, 0.8, 1.0), layer(ISO, 0.4, 0.5)]),
}


@pytest.mark.parametrize("name", list(CASES))
def test_reconstruction_reproduces_nodal_values_at_the_nodes(name):
    # test_reconstruction.cpp:22-63: the source-function integration along +-mu_i
    # equals the discrete-ordinate solution at the nodes, at the top, inside, bottom
    d = CASES[name]
    m = oracle_material(d)
    N = 8
    nodes, _ = O.quadrature(N)
    tot = sum(l.tau for l in d.layers)
    taus = [0.0, 0.37 * tot, tot]
    phis = [0.3 + 2 * math.pi * j / 7 for j in range(7)]
    stokes = [1.0, 0.2, -0.1, 0.05]
    nod, *_ = O.radiance(m, N, 0.6, 0.3, stokes, taus, mus=None, phis=phis, nodal=True)
    mus = np.concatenate([nodes, -nodes])
    rec, *_ = O.radiance(m, N, 0.6, 0.3, stokes, taus, mus=mus, phis=phis)
    for it in range(len(taus)):
        scale = max(np.abs(nod[it]).max(), 1e-12)
        assert np.abs(rec[it] - nod[it]).max() < 1e-8 * scale, (it, np.abs(rec[it] - nod[it]).max(), scale)


def test_top_field_at_nodes_matches_the_brdf_path():
    # tau = 0, mu = node: I = F_r(mu0, mu_i, dphi) mu0 I0 (brdf.cpp:100-117)
    d = CASES["rayleigh_lam"]
    m = oracle_material(d)
    N = 6
    nodes, _ = O.quadrature(N)
    mu0, I0 = 0.6, np.array([1.0, 0.3, -0.2, 0.1])
    table, _ = O.brdf(m, N, [mu0], n_dphi=19)
    phis = [2 * math.pi * j / 19 for j in range(19)]
    f, *_ = O.radiance(m, N, mu0, 0.0, I0, [0.0], mus=nodes, phis=phis)
    want = np.einsum("ojrc,c->ojr", table[0], mu0 * I0)
    assert np.abs(f[0] - want).max() < 1e-10 * np.abs(want).max()


def test_isotropic_medium_gives_azimuth_independent_field():
    # test_reconstruction.cpp:167-188
    m = oracle_material(mat([layer(ISO, 0.7, 1.0)]))
    phis = [2 * math.pi * j / 8 for j in range(8)]
    f, *_ = O.radiance(m, 8, 0.6, 0.0, [1, 0, 0, 0], [0.0], mus=[0.9, -0.35], phis=phis)
    for imu in range(2):
        first = f[0, imu, 0]
        assert np.allclose(f[0, imu, :, 0], first[0], rtol=1e-12, atol=0)
        assert np.abs(f[0, imu, :, 1] - first[1]).max() < 1e-12
        assert np.abs(f[0, imu, :, 2:]).max() < 1e-12


def test_unpolarized_beam_leaves_no_u_or_v_in_the_beam_meridian_plane():
    # test_reconstruction.cpp:190-...
    m = oracle_material(mat([layer(M.RAYLEIGH, 0.9, 1.0)]))
    f, *_ = O.radiance(m, 8, 0.6, 0.0, [1, 0, 0, 0], [0.0], mus=[0.8], phis=[0.0, math.pi])
    assert np.abs(f[0, 0, :, 2:]).max() < 1e-12 * abs(f[0, 0, 0, 0])


def test_standard_grid_and_reflectance():
    # capi.cpp:138-174: 2*zenith signed directions x azimuth grid from phi0; the
    # field reflectance equals the BRDF-table reflectance at the same incident
    d = CASES["rayleigh_lam"]
    m = oracle_material(d)
    N, mu0, phi0 = 8, 0.6, 0.4
    f, mus, phis, refl = O.radiance(m, N, mu0, phi0, [1, 0, 0, 0], [0.0, 1.0], zenith=11, azimuth=19)
    assert f.shape == (2, 22, 19, 4) and np.all(np.isfinite(f))
    assert mus[0] == 1e-6 and mus[10] == 1.0 and mus[11] == -1e-6 and mus[21] == -1.0
    assert phis[0] == pytest.approx(phi0) and phis[-1] == pytest.approx(phi0 + math.pi)
    table, _ = O.brdf(m, N, [mu0], n_dphi=19)
    nodes, w = O.quadrature(N)
    # brdf.cpp:142-160: exiting flux per Stokes channel over mu0 I0 -- for I0 = e0
    # the first COLUMN of F_r integrated over the upper hemisphere
    r = np.einsum("o,ojc->c", w * nodes * 2 * math.pi / 19, table[0][:, :, :, 0])
    assert np.allclose(refl, r, rtol=1e-10, atol=1e-14)
