"""The drop-in C ABI end to end on the GPU (reference test_capi.cpp:85-119,
test_pipeline.cpp:25-42 counters, csv.cpp:111-168 output formats)."""
import math
import os

import numpy as np
import pytest

import paper_1707_05882_b200 as V
import pyoracle as O
from paper_1707_05882_b200 import materials as M

from helpers import product_material

pytestmark = pytest.mark.gpu


def test_brdf_through_the_shared_library_interface(tmp_path):
    mat = product_material(M.single_layer(M.ISOTROPIC, 0.5, 1.0))  # isotropic_half.json
    b = V.compute_brdf(mat, V.options(4), [0.6, 1.0], 5)
    assert b.shape == (2, 4, 5)
    assert b.entry(0, 0, 0)[0, 0] >= 0.0
    r = b.reflectance(0)
    assert 0.0 < r[0] <= 1.0 + 1e-6
    csv, binp = str(tmp_path / "t.csv"), str(tmp_path / "t.bin")
    b.write_csv(csv)
    b.write_binary(binp)
    lines = open(csv).read().splitlines()
    assert lines[0] == "mu_in,mu_out,dphi," + ",".join(f"m{r}{c}" for r in range(4) for c in range(4))
    assert len(lines) == 1 + 2 * 4 * 5
    tab = b.table()
    vals = [float(x) for x in lines[1].split(",")]
    assert vals[0] == 0.6 and vals[2] == 0.0 and np.array_equal(np.array(vals[3:]), tab[0, 0, 0].ravel())
    mi, mo, dp, t2 = V.read_brdf_binary(binp)
    assert np.array_equal(t2, tab) and list(mi) == [0.6, 1.0]
    assert np.array_equal(mo, O.quadrature(4)[0])
    assert np.allclose(dp, 2 * math.pi * np.arange(5) / 5, rtol=0, atol=0)
    os.remove(csv)


def test_default_dphi_and_index_errors():
    mat = product_material(M.single_layer(M.RAYLEIGH, 0.9, 1.0))
    b = V.compute_brdf(mat, V.options(4), [0.6], 0)
    assert b.shape == (1, 4, 19)
    with pytest.raises(V.VrteError) as e:
        b.entry(1, 0, 0)
    assert e.value.code == V.VRTE_E_ARGUMENT and "out of range" in e.value.message
    with pytest.raises(V.VrteError):
        b.reflectance(3)


def test_timings_and_counters():
    w = M.config("C1")
    mat = product_material(w.material)
    nodes, _ = O.quadrature(8)
    b = V.compute_brdf(mat, V.options(8), nodes, 19)
    t = b.timings()
    L, S, n_in = 12, 1, 8
    assert t["homogeneous_solves"] == S * L
    assert t["particular_solves"] == n_in * 4 * 2 * L * S
    assert t["boundary_solves"] == n_in * 4 * L
    assert t["reconstruction"] == 0.0 and t["total_wall"] > 0.0
    assert t["homogeneous"] > 0 and t["boundary"] > 0
    s = b.device_stats()
    assert s["kernel_launches"] > 0 and s["max_eigen_residual"] < 1e-10


def test_order_cap_truncates_orders():
    w = M.config("C1")
    mat = product_material(w.material)
    b = V.compute_brdf(mat, V.options(8, order_cap=3), [0.5], 7)
    r, _ = O.brdf(__import__("helpers").oracle_material(w.material), 8, np.array([0.5]), 7, order_cap=3)
    assert np.abs(b.table() - r).max() < 1e-10 * np.abs(r).max()


def test_f00_roundoff_clamp_counts_like_the_reference():
    """brdf.cpp:106-117: F00 in [-1e-9, 0) is clamped to 0 and counted; the
    count matches the oracle's on a case that has such entries: a forward-peaked
    G(0.9, 24) phase matrix under-resolved at N = 6 has negative F00 lobes, and
    omega = 1e-10 scales them into the clamp window (90 entries)."""
    from helpers import oracle_material
    desc = M.single_layer(M.generator_G(0.9, 24), 1e-10, 1.0)
    nodes, _ = O.quadrature(6)
    b = V.compute_brdf(product_material(desc), V.options(6), nodes, 6)
    assert np.all(b.table()[..., 0, 0] >= 0)
    _, tm = O.brdf(oracle_material(desc), 6, nodes, 6)
    assert tm["clamped_entries"] == 90
    assert b.device_stats()["clamped"] == tm["clamped_entries"]
    # ten times larger lobes leave the window: the reference's error, same text
    with pytest.raises(V.VrteError) as ei:
        V.compute_brdf(product_material(M.single_layer(M.generator_G(0.9, 24), 1e-6, 1.0)), V.options(6), nodes, 6)
    assert ei.value.code == 3 and ei.value.message.startswith("brdf: negative intensity entry -0.000000")


def test_spectral_batch_matches_individual_solves():
    """vrte_compute_brdf_batch (spectral bands, BASELINE config 5 shape at small
    N): every band's table equals the single-request table bit for bit, for any
    concurrency."""
    nodes, _ = O.quadrature(8)
    mats = [product_material(M.config("C5", band=b).material) for b in (0, 15, 30)]
    single = [V.compute_brdf(m, V.options(8), nodes[:3], 5).table() for m in mats]
    for conc in (1, 3):
        out = V.compute_brdf_batch(mats, V.options(8), nodes[:3], 5, concurrency=conc)
        for b, s in zip(out, single):
            assert np.array_equal(b.table(), s)


def test_batch_reports_first_failure():
    nodes, _ = O.quadrature(16)
    ok = product_material(M.config("C1").material)
    bad = product_material(M.config("C4").material)  # at N=16 the reference rejects m = 0
    with pytest.raises(V.VrteError) as ei:
        V.compute_brdf_batch([ok, bad], V.options(16, 24), nodes[:2], 5)
    assert ei.value.code == 3 and "negative real axis" in ei.value.message


def test_pinned_host_buffers_are_recycled_per_size():
    import ctypes as C
    L = V.lib()
    L.vrte_cuda_host_alloc.restype = C.c_void_p
    L.vrte_cuda_host_alloc.argtypes = [C.c_size_t]
    L.vrte_cuda_host_free.argtypes = [C.c_void_p, C.c_size_t]
    n = 1 << 20
    p = L.vrte_cuda_host_alloc(n)
    assert p
    buf = (C.c_ubyte * n).from_address(p)
    buf[0], buf[n - 1] = 7, 9
    assert buf[0] == 7 and buf[n - 1] == 9
    L.vrte_cuda_host_free(p, n)
    q = L.vrte_cuda_host_alloc(n)  # the freed buffer of the same size comes back
    assert q == p
    L.vrte_cuda_host_free(q, n)
    L.vrte_cuda_host_free(None, 0)  # null is a no-op
