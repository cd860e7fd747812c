"""Radiance path (vrte_solve_radiance, capi.cpp:138-232):
the sm_100a reconstruction (radiance.cu) against the oracle restatement
(tests/test_oracle_radiance.py pins it to the reference's reconstruction tests)."""
import math
import os
import tempfile

import numpy as np
import pytest

import paper_1707_05882_b200 as V
import pyoracle as O
from paper_1707_05882_b200 import materials as M

from helpers import oracle_material, product_material

pytestmark = pytest.mark.gpu

ISO = np.array([M.greek(1, 0, 0, 0, 0, 0)])


def desc(layers, base="black", albedo=0.0, mu0=0.6, phi0=0.0, stokes=(1.0, 0.0, 0.0, 0.0)):
    d = M.MaterialDesc([M.LayerDesc(o, t, np.asarray(c, float)) for c, o, t in layers], base=base, albedo=albedo)
    d.mu0, d.phi0, d.stokes = mu0, phi0, tuple(stokes)
    return d


CASES = {
    "iso_half": (desc([(ISO, 0.5, 1.0)]), 8),
    "rayleigh_lam": (desc([(M.RAYLEIGH, 0.9, 2.0)], "lambertian", 0.3, stokes=(1.0, 0.3, -0.2, 0.1)), 8),
    "two_layer": (desc([(M.RAYLEIGH, 0.8, 1.0), (ISO, 0.4, 0.5)], mu0=0.45, phi0=0.7), 8),
    "paint": (desc([(M.generator_G(0.6, 16), 0.95, 2.0), (M.RAYLEIGH, 0.6, 5.0)], "lambertian", 0.2,
                   mu0=0.8, phi0=1.3, stokes=(1.0, 0.0, 0.4, 0.0)), 12),
}


def run_pair(d, N, taus, zen=6, azi=7):
    f = V.solve_radiance(product_material(d), V.options(N, out_zenith=zen, out_azimuth=azi), taus)
    t, mus, phis, g = f.values()
    r, omu, ophi, orefl = O.radiance(oracle_material(d), N, d.mu0, d.phi0, d.stokes, taus, zenith=zen, azimuth=azi)
    return f, (t, mus, phis, g), (omu, ophi, r, orefl)


@pytest.mark.parametrize("name", list(CASES))
def test_radiance_field_matches_oracle(name):
    d, N = CASES[name]
    tot = sum(l.tau for l in d.layers)
    taus = [0.0, 0.3 * tot, d.layers[0].tau, tot]
    f, (t, mus, phis, g), (omu, ophi, r, orefl) = run_pair(d, N, taus)
    assert np.array_equal(t, taus) and np.array_equal(mus, omu) and np.allclose(phis, ophi, rtol=0, atol=1e-15)
    scale = np.abs(r).max()
    err = np.abs(g - r).max() / scale
    assert err < 1e-9, (name, err)
    assert np.allclose(f.reflectance(), orefl, rtol=1e-10, atol=1e-13)


def test_radiance_defaults_and_csv():
    # n_tau = 0 -> {0}; the standard 11 x 19 grid; CSV in csv.cpp:28-40 format
    d, N = CASES["rayleigh_lam"]
    f = V.solve_radiance(product_material(d), V.options(N), [])
    assert f.shape == (1, 22, 19)
    p = os.path.join(tempfile.mkdtemp(), "field.csv")
    f.write_csv(p)
    lines = open(p).read().splitlines()
    assert lines[0] == "tau,mu,phi,I,Q,U,V" and len(lines) == 1 + 22 * 19
    row = [float(x) for x in lines[1].split(",")]
    assert np.array_equal(np.array(row), f.row(0, 0, 0))
    tm = f.timings()
    assert tm.boundary_solves > 0 and tm.reconstruction_items == 22


def test_incident_override_and_isotropy():
    # options.incident_override replaces the material's beam (capi.cpp:151-155);
    # an isotropic medium gives an azimuth-independent field (test_reconstruction.cpp:167-188)
    d, N = CASES["iso_half"]
    o = V.options(N, out_zenith=4, out_azimuth=8, incident_override=1, incident_mu0=0.33, incident_phi0=2.0)
    f = V.solve_radiance(product_material(d), o, [0.0, 0.5])
    _, mus, phis, g = f.values()
    assert phis[0] == pytest.approx(2.0)
    r, *_ = O.radiance(oracle_material(d), N, 0.33, 2.0, d.stokes, [0.0, 0.5], zenith=4, azimuth=8)
    assert np.abs(g - r).max() < 1e-9 * np.abs(r).max()
    assert np.abs(g[..., 0] - g[..., :1, 0]).max() < 1e-12 * np.abs(g[..., 0]).max()


def table_base(N, rho=0.2):
    # smooth, partially polarizing Mueller table on the quadrature nodes (boundary.cpp:37-71)
    nodes, _ = O.quadrature(N)
    t = np.zeros((N, N, 4, 4))
    for i, a in enumerate(nodes):
        for j, b in enumerate(nodes):
            f = 2 * rho * (1.0 + 0.3 * (a - b))
            t[i, j] = f * np.array([[1, 0.1 * (a - b), 0, 0], [0.1 * (a - b), 0.5, 0, 0],
                                    [0, 0, 0.3, 0.05], [0, 0, -0.05, 0.3]])
    return t


def test_mueller_table_base_brdf_and_radiance_match_oracle():
    # the bilinear Mueller-table base (base_type 2) through both product paths
    N = 8
    d = desc([(M.RAYLEIGH, 0.9, 1.5)], "mueller_table", mu0=0.55, phi0=0.4, stokes=(1.0, 0.2, 0.1, -0.1))
    d.table = table_base(N)
    nodes, _ = O.quadrature(N)
    g = V.compute_brdf(product_material(d), V.options(N), nodes, 7).table()
    r, _ = O.brdf(oracle_material(d), N, nodes, 7)
    assert np.abs(g - r).max() < 1e-9 * np.abs(r).max()
    f, (t, mus, phis, gf), (omu, ophi, rf, orefl) = run_pair(d, N, [0.0, 0.7, 1.5], zen=5, azi=6)
    assert np.abs(gf - rf).max() < 1e-9 * np.abs(rf).max()
    assert np.allclose(f.reflectance(), orefl, rtol=1e-10, atol=1e-13)


def test_degenerate_grids_and_many_depths():
    # out_zenith = 1 -> mu = {1, -1}; out_azimuth = 1 -> phi = {phi0} (pipeline.cpp:358-390);
    # depths outside [0, tau_total] clamp into the stack (reconstruction.cpp:12-19)
    d, N = CASES["two_layer"]
    taus = [-0.5, 0.0, 0.2, 1.0, 1.0000001, 1.3, 1.5, 9.0]
    f, (t, mus, phis, g), (omu, ophi, r, orefl) = run_pair(d, N, taus, zen=1, azi=1)
    assert list(mus) == [1.0, -1.0] and len(phis) == 1
    assert np.abs(g - r).max() < 1e-9 * np.abs(r).max()


def stokes_metric(g, r):
    """Per output Stokes vector: max_c |G_c - R_c| / max(|R_c|, 1e-3 |R_I|, 1e-6 max|R|) -- the
    SURVEY §8(d) per-Mueller-matrix metric applied to the field's Stokes vectors (the absolute
    floor keeps the exactly-zero downward field at tau = 0 out of the ratio)."""
    scale = np.abs(r).max()
    den = np.maximum(np.maximum(np.abs(r), 1e-3 * np.abs(r[..., :1])), 1e-6 * scale)
    return float((np.abs(g - r) / den).max())


@pytest.mark.parametrize("name", list(CASES))
def test_radiance_per_element_parity(name):
    d, N = CASES[name]
    tot = sum(l.tau for l in d.layers)
    f, (t, mus, phis, g), (omu, ophi, r, orefl) = run_pair(d, N, [0.0, 0.5 * tot, tot])
    assert stokes_metric(g, r) <= 1e-9, name


def test_radiance_grid_edge_cases_follow_the_reference():
    d, N = CASES["rayleigh_lam"]
    mat = product_material(d)
    full = V.solve_radiance(mat, V.options(N, out_zenith=3, out_azimuth=4), [0.0])
    # an empty zenith or azimuth grid: an empty field, VRTE_OK, the reflectance still solved
    for zen, azi, shape in ((0, 4, (1, 0, 4)), (3, 0, (1, 6, 0)), (0, 0, (1, 0, 0))):
        f = V.solve_radiance(mat, V.options(N, out_zenith=zen, out_azimuth=azi), [0.0])
        assert f.shape == shape
        assert np.array_equal(f.reflectance(), full.reflectance())
    # a negative count is std::vector's length_error in the reference: status 3
    for zen, azi in ((-1, 4), (3, -2)):
        with pytest.raises(V.VrteError) as e:
            V.solve_radiance(mat, V.options(N, out_zenith=zen, out_azimuth=azi), [0.0])
        assert e.value.code == 3
    # validation order: the solver's quadrature check precedes the incident check
    bad = V.options(0, incident_override=1, incident_mu0=2.0)
    with pytest.raises(V.VrteError) as e:
        V.solve_radiance(mat, bad, [0.0])
    assert e.value.code == 2 and "quadrature size" in str(e.value)
    with pytest.raises(V.VrteError) as e:
        V.solve_radiance(mat, V.options(N, incident_override=1, incident_mu0=2.0), [0.0])
    assert e.value.code == 2 and "incident mu0" in str(e.value)
