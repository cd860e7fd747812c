"""C-ABI checks that need no GPU: the library loads, exports every symbol of
include/vrte/*.h, and reproduces the reference's host-side behaviour
(test_capi.cpp:19-37 material loading/errors, capi.cpp:21-32 error mapping,
brdf.cpp:45-62 validation order, vrte_options_init defaults)."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

import paper_1707_05882_b200 as V
from paper_1707_05882_b200 import materials as M

from helpers import product_material

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    syms = set()
    for h in ("vrte.h", "vrte_ext.h", "vrte_cuda.h"):
        text = open(os.path.join(ROOT, "include", "vrte", h)).read()
        syms |= set(re.findall(r"VRTE_API[^;(]*?\b(vrte_\w+)\s*\(", text, flags=re.S))
    return syms


def test_library_exports_every_declared_symbol():
    lib = V.lib()
    declared = header_symbols()
    assert len(declared) >= 35
    assert declared == set(V.EXPORTED)
    for s in declared:
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", V.LIB_PATH], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert declared <= exported
    # nothing else leaks (hidden visibility)
    assert {s for s in exported if not s.startswith("vrte_")} == set()


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", V.LIB_PATH],
                         capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_\d+a?", out))
    assert arches == {"sm_100a"}, arches


def test_version_and_options_init():
    assert V.version() == "1.0.0"
    o = V.Options()
    V.lib().vrte_options_init(C.byref(o))
    assert (o.quadrature_n, o.out_zenith, o.out_azimuth, o.order_cap, o.threads) == (40, 11, 19, 0, 0)
    assert o.dump_eigen_path is None and o.incident_override == 0


def write_rayleigh_slab(d):
    m = M.single_layer(M.RAYLEIGH, 0.9, 1.0, "lambertian", 0.3)
    return m.write(d, "rayleigh_slab")


def test_material_loading_and_errors():
    d = tempfile.mkdtemp()
    mat = V.Material.load(write_rayleigh_slab(d))
    assert mat.info() == (3, 1)
    with pytest.raises(V.VrteError) as e:
        V.Material.load(os.path.join(d, "does_not_exist.json"))
    assert e.value.code == V.VRTE_E_VALIDATION and "cannot open material file" in e.value.message
    bad = '{"layers":[{"omega": 1.5, "tau": 1.0, "coeff_file": "x.coef"}]}'
    with pytest.raises(V.VrteError) as e:
        V.Material.parse(bad, ".")
    assert e.value.code == V.VRTE_E_VALIDATION
    h = C.c_void_p()
    assert V.lib().vrte_material_load(None, C.byref(h)) == V.VRTE_E_ARGUMENT
    assert V.lib().vrte_material_info(None, None, None) == V.VRTE_E_ARGUMENT


def test_validation_messages_match_reference_wording():
    d = tempfile.mkdtemp()
    M.write_coef(os.path.join(d, "iso.coef"), M.ISOTROPIC)
    doc = ('{"layers":[{"omega": 1.5, "tau": -1.0, "coeff_file": "iso.coef"}],'
           '"base":{"type":"lambertian","albedo":2.0},"source":{"mu0":0.6}}')
    with pytest.raises(V.VrteError) as e:
        V.Material.parse(doc, d)
    msg = e.value.message
    assert "layer 0: albedo out of range (omega = 1.5, expected [0,1])" in msg
    assert "layer 0: optical thickness must be positive (tau = -1)" in msg
    assert "base: lambertian albedo out of range (rho = 2.000000)" in msg
    assert msg.count("; ") == 2
    # coefficient file errors
    with open(os.path.join(d, "bad.coef"), "w") as f:
        f.write("0 1 0 0 0 0 0\n2 0.5 0 0 0 0 0\n")
    with pytest.raises(V.VrteError) as e:
        V.Material.parse('{"layers":[{"omega":0.5,"tau":1,"coeff_file":"bad.coef"}]}', d)
    assert "missing coefficient row for l = 1" in e.value.message
    with pytest.raises(V.VrteError) as e:
        V.Material.parse('{"layers":[{"omega":0.5,"tau":1,"coeff_file":"iso.coef"}],"base":{"type":"mirror"}}', d)
    assert 'base: unknown type "mirror"' in e.value.message
    with pytest.raises(V.VrteError) as e:
        V.Material.parse("{not json", d)
    assert e.value.message.startswith("material JSON parse error")


def test_block_structure_and_normalization_checks():
    d = tempfile.mkdtemp()
    c = M.generator_G(0.5, 4)
    c[2, 0, 2] = 0.1  # breaks the 2+2 block structure
    M.write_coef(os.path.join(d, "c.coef"), M.ISOTROPIC)
    with open(os.path.join(d, "c.coef"), "a"):
        pass
    m = M.single_layer(M.ISOTROPIC * 0.5, 0.5, 1.0)  # beta_0 = 0.5 violates normalization
    with pytest.raises(V.VrteError) as e:
        V.Material.parse(m.json_text(d, "norm"), d)
    assert "violates the phase normalization B_0(0,0) = 1" in e.value.message


def test_brdf_argument_and_validation_errors_precede_device_work():
    d = tempfile.mkdtemp()
    mat = V.Material.load(write_rayleigh_slab(d))
    lib = V.lib()
    h = C.c_void_p()
    o = V.options(4)
    mu = np.array([0.6])
    dp = mu.ctypes.data_as(C.POINTER(C.c_double))
    assert lib.vrte_compute_brdf(mat._h, C.byref(o), None, 1, 5, None, C.byref(h)) == V.VRTE_E_ARGUMENT
    assert lib.vrte_compute_brdf(mat._h, C.byref(o), dp, 0, 5, None, C.byref(h)) == V.VRTE_E_ARGUMENT
    assert lib.vrte_compute_brdf(None, C.byref(o), dp, 1, 5, None, C.byref(h)) == V.VRTE_E_ARGUMENT
    # ill-conditioned basis rejected before any solve (test_brdf.cpp:87-96)
    bad = np.array([[1, 0, 0, 0], [1, 1e-9, 0, 0], [1, 0, 1, 0], [1, 0, 0, 1]], float)
    with pytest.raises(V.VrteError) as e:
        V.compute_brdf(mat, o, mu, 4, bad)
    assert e.value.code == V.VRTE_E_VALIDATION and "ill-conditioned" in e.value.message
    with pytest.raises(V.VrteError) as e:
        V.compute_brdf(mat, o, [1.5], 4)
    assert e.value.code == V.VRTE_E_VALIDATION and "incident cosines must lie in (0,1]" in e.value.message
    with pytest.raises(V.VrteError) as e:
        V.compute_brdf(mat, V.options(0), mu, 4)
    assert e.value.code == V.VRTE_E_VALIDATION and "quadrature size must be at least 1" in e.value.message


def test_mc_argument_checks_before_any_device_work():
    # mc.cpp:258-261 validation (2), capi.cpp:331-332 null checks (5); free accepts NULL
    d = tempfile.mkdtemp()
    mat = V.Material.load(write_rayleigh_slab(d))
    lib = V.lib()
    h = C.c_void_p()
    assert lib.vrte_mc_trace(None, C.byref(V.options(4)), 100, 7, 4, 4, C.byref(h)) == V.VRTE_E_ARGUMENT
    assert lib.vrte_mc_trace(mat._h, C.byref(V.options(4)), 0, 7, 4, 4, C.byref(h)) == V.VRTE_E_VALIDATION
    assert "mc: photon count must be positive" in lib.vrte_last_error().decode()
    assert lib.vrte_mc_trace(mat._h, C.byref(V.options(4)), 10, 7, 0, 4, C.byref(h)) == V.VRTE_E_VALIDATION
    assert "mc: bin counts must be positive" in lib.vrte_last_error().decode()
    row = np.zeros(10)
    assert lib.vrte_mc_tally_row(None, 0, 0, 0, row.ctypes.data_as(C.POINTER(C.c_double))) == V.VRTE_E_ARGUMENT
    lib.vrte_field_free(None)
    lib.vrte_mc_tally_free(None)
    lib.vrte_brdf_free(None)
    lib.vrte_material_free(None)


def test_radiance_argument_checks_before_any_device_work():
    # capi.cpp:138-140 null checks (5), pipeline.cpp:97-98 incident validation (2)
    d = tempfile.mkdtemp()
    mat = V.Material.load(write_rayleigh_slab(d))
    lib = V.lib()
    h = C.c_void_p()
    assert lib.vrte_solve_radiance(None, C.byref(V.options(4)), None, 0, C.byref(h)) == V.VRTE_E_ARGUMENT
    assert lib.vrte_solve_radiance(mat._h, C.byref(V.options(4)), None, 1, C.byref(h)) == V.VRTE_E_ARGUMENT
    o = V.options(4, incident_override=1, incident_mu0=1.5)
    with pytest.raises(V.VrteError) as e:
        V.solve_radiance(mat, o, [0.0])
    assert e.value.code == V.VRTE_E_VALIDATION and "incident mu0 must lie in (0,1]" in e.value.message
    row = np.zeros(7)
    assert lib.vrte_field_row(None, 0, 0, 0, row.ctypes.data_as(C.POINTER(C.c_double))) == V.VRTE_E_ARGUMENT
    assert lib.vrte_field_size(None, None, None, None) == V.VRTE_E_ARGUMENT


def test_last_error_is_thread_local():
    import threading
    lib = V.lib()
    h = C.c_void_p()
    assert lib.vrte_material_load(b"/nonexistent.json", C.byref(h)) == V.VRTE_E_VALIDATION
    seen = []

    def other():
        seen.append(lib.vrte_last_error().decode())

    t = threading.Thread(target=other)
    t.start()
    t.join()
    assert seen == [""]
    assert "cannot open material file" in lib.vrte_last_error().decode()


def test_binary_reader_roundtrip_format(tmp_path):
    # VRTEBRDF v1 layout (csv.cpp:147-168) written by hand, read by the python reader
    ni, no, npd = 2, 3, 2
    rng = np.random.default_rng(3)
    tab = rng.uniform(-1, 1, (ni, no, npd, 4, 4))
    p = tmp_path / "t.bin"
    with open(p, "wb") as f:
        f.write(b"VRTEBRDF")
        f.write(np.array([1, ni, no, npd], "<u4").tobytes())
        for a in ([0.5, 1.0], [0.3, 0.7, 0.9], [0.0, 3.14]):
            f.write(np.array(a, "<f8").tobytes())
        f.write(tab.astype("<f8").tobytes())
    mi, mo, dp, t2 = V.read_brdf_binary(str(p))
    assert list(mo) == [0.3, 0.7, 0.9] and np.array_equal(t2, tab)
