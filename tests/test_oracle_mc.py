"""Pin the oracle's Monte Carlo restatement (mc.cpp) with the
reference's own tracer tests (test_mc.cpp) and against the oracle's DOM radiance
field (test_mc.cpp:96-130).  Test infrastructure only."""
import math

import numpy as np
import pytest

import pyoracle as O
from paper_1707_05882_b200 import materials as M

from helpers import oracle_material

ISO = np.array([M.greek(1, 0, 0, 0, 0, 0)])


def mat(coeffs, omega, tau, base="black", albedo=0.0):
    return oracle_material(M.MaterialDesc([M.LayerDesc(omega, tau, np.asarray(coeffs, float))], base=base,
                                          albedo=albedo))


def test_vacuum_tallies_nothing():
    t = O.mc_trace(mat(ISO, 0.0, 1.0), 0.6, 0.0, [1, 0, 0, 0], 20000, 7, 6, 6, threads=2)
    assert np.abs(t.sum).max() == 0.0


def test_reproducible_across_thread_counts():
    m = mat(M.RAYLEIGH, 0.8, 1.0)
    a = O.mc_trace(m, 0.6, 0.0, [1, 0, 0, 0], 50000, 123, 5, 6, threads=1)
    b = O.mc_trace(m, 0.6, 0.0, [1, 0, 0, 0], 50000, 123, 5, 6, threads=4)
    c = O.mc_trace(m, 0.6, 0.0, [1, 0, 0, 0], 50000, 124, 5, 6, threads=4)
    assert np.array_equal(a.sum, b.sum) and np.array_equal(a.sum_sq, b.sum_sq) and np.array_equal(a.hits, b.hits)
    assert not np.array_equal(a.sum, c.sum)


def test_lossless_slab_over_perfect_diffuse_base_returns_all_flux():
    t = O.mc_trace(mat(ISO, 1.0, 10.0, "lambertian", 1.0), 0.6, 0.0, [1, 0, 0, 0], 200000, 42, 8, 8)
    n = t.photons
    flux = t.sum[0, ..., 0].sum()
    var = t.sum_sq[0, ..., 0].sum()
    mean = flux / n
    se = math.sqrt(max(0.0, var / n - mean * mean) / n)
    assert abs(t.mu0 * mean - t.mu0) < 3.0 * t.mu0 * se + 1e-9


def test_isotropic_unpolarized_beam_stays_unpolarized():
    t = O.mc_trace(mat(ISO, 0.5, 1.0), 0.6, 0.0, [1, 0, 0, 0], 200000, 99, 5, 5)
    for h in range(2):
        for iz in range(5):
            for ia in range(5):
                if t.hits[h, iz, ia] < 10:
                    continue
                s, se = t.radiance(h, iz, ia), t.std_error(h, iz, ia)
                assert np.all(np.abs(s[1:]) < 3.0 * se[1:] + 1e-12)


def test_tracer_agrees_with_the_dom_field_for_a_polarizing_slab():
    # test_mc.cpp:96-130: flux-weighted bin averages of the solved field (2x2 Gauss
    # points per bin) against the tracer's bins
    m = mat(M.RAYLEIGH, 0.9, 1.0)
    zb, ab = 6, 8
    t = O.mc_trace(m, 0.6, 0.0, [1, 0, 0, 0], 400000, 31415, zb, ab)
    ga, gb = 0.5 - 0.5 / math.sqrt(3), 0.5 + 0.5 / math.sqrt(3)
    checked = passed = 0
    for h in range(2):
        tau = 0.0 if h == 0 else 1.0
        for iz in range(zb):
            mus = [(iz + f) / zb for f in (ga, gb)]
            for ia in range(ab):
                if t.hits[h, iz, ia] < 50:
                    continue
                phis = [2 * math.pi * (ia + f) / ab for f in (ga, gb)]
                sm = [mu if h == 0 else -mu for mu in mus]
                f, *_ = O.radiance(m, 16, 0.6, 0.0, [1, 0, 0, 0], [tau], mus=sm, phis=phis)
                w = np.array(mus)[:, None, None]
                dom = (w * f[0]).sum(axis=(0, 1)) / (2 * sum(mus))
                s, se = t.radiance(h, iz, ia), t.std_error(h, iz, ia)
                checked += 1
                if abs(s[0] - dom[0]) < 4.0 * se[0] + 0.02 * abs(dom[0]):
                    passed += 1
    assert checked > 20 and passed >= 0.9 * checked, (checked, passed)
