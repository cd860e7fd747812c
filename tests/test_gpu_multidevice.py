"""Order sharding inside the product: VRTE_DEVICES lists the
devices one vrte_compute_brdf call shards its Fourier orders over (cyclic,
m = k, k + D, ...); the tau = 0 stacks are gathered to the first device by peer
copies and synthesized there in order 0..L-1, so the table is bitwise equal to
the single-device one.  This box has one B200: repeated ordinals run several
shards (each with its own plan, stream and host thread) on it, which exercises
the same sharding, gather and synthesis code as distinct devices.  Band
sharding of vrte_compute_brdf_batch follows the same list."""
import os

import numpy as np
import pytest

import paper_1707_05882_b200 as V
import pyoracle as O
from paper_1707_05882_b200 import materials as M

from helpers import product_material

pytestmark = pytest.mark.gpu


class devices:
    def __init__(self, spec):
        self.spec = spec

    def __enter__(self):
        os.environ["VRTE_DEVICES"] = self.spec

    def __exit__(self, *exc):
        os.environ.pop("VRTE_DEVICES", None)


@pytest.mark.parametrize("cfg,spec", [("C1", "0,0"), ("C1", "0,0,0,0,0"), ("C3", "0,0,0"), ("C3", "0,0,0,0,0,0,0,0")])
def test_order_sharded_call_is_bitwise_single_device(cfg, spec):
    w = M.config(cfg)
    nodes, _ = O.quadrature(w.N)
    mu = nodes[:: max(1, w.N // 8)]
    mat = product_material(w.material)
    one = V.compute_brdf(mat, V.options(w.N), mu, 19)
    with devices(spec):
        many = V.compute_brdf(mat, V.options(w.N), mu, 19)
    assert np.array_equal(one.table(), many.table())
    s1, s2 = one.device_stats(), many.device_stats()
    assert s2["max_eigen_residual"] == s1["max_eigen_residual"]
    assert s2["kernel_launches"] > s1["kernel_launches"]


def test_more_devices_than_orders():
    # a Rayleigh layer has L = 3 orders: shards beyond the third stay idle
    mat = product_material(M.single_layer(M.RAYLEIGH, 0.9, 1.0, "lambertian", 0.3))
    one = V.compute_brdf(mat, V.options(6), [0.4, 0.9], 7)
    with devices("0,0,0,0,0"):
        many = V.compute_brdf(mat, V.options(6), [0.4, 0.9], 7)
    assert np.array_equal(one.table(), many.table())


def test_sharded_failure_reports_the_reference_message():
    w = M.config("C4")
    nodes, _ = O.quadrature(16)
    mat = product_material(w.material)
    with devices("0,0"):
        with pytest.raises(V.VrteError) as ei:
            V.compute_brdf(mat, V.options(16), nodes[:2], 5)
    assert ei.value.code == 3 and "negative real axis" in ei.value.message


def test_band_sharded_batch():
    nodes, _ = O.quadrature(8)
    mats = [product_material(M.config("C5", band=b).material) for b in (0, 7, 15, 30)]
    single = [V.compute_brdf(m, V.options(8), nodes[:3], 5).table() for m in mats]
    with devices("0,0"):
        out = V.compute_brdf_batch(mats, V.options(8), nodes[:3], 5, concurrency=2)
    for b, s in zip(out, single):
        assert np.array_equal(b.table(), s)


def test_bad_device_list_is_a_validation_error():
    mat = product_material(M.config("C1").material)
    with devices("0,x"):
        with pytest.raises(V.VrteError) as ei:
            V.compute_brdf(mat, V.options(8), [0.5], 5)
    assert ei.value.code == 2
