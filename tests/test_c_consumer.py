"""A compiled C program linked against libvrte.so.1 (the reference's SONAME,
src/CMakeLists.txt:37-42) through the reference header alone: the drop-in as
an existing application would see it.  Loads the reference's own data/*.json
(tests/golden/proj_data, verbatim copies); the GPU test also solves them."""
import os
import subprocess

import numpy as np
import pytest

import paper_1707_05882_b200 as V

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
DATA = os.path.join(HERE, "golden", "proj_data")
MATERIALS = ["rayleigh_slab.json", "isotropic_half.json", "conservative_diffuse.json", "paint_film.json"]


@pytest.fixture(scope="module")
def consumer(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("c") / "consumer")
    libdir = os.path.dirname(V.LIB_PATH)
    # link by SONAME the way a reference build links -lvrte: the executable's
    # NEEDED entry must be libvrte.so.1
    subprocess.run(["cc", "-std=c11", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(HERE, "c", "consumer.c"),
                    "-L", libdir, "-l:libvrte.so.1", "-Wl,-rpath," + libdir, "-o", exe], check=True)
    need = subprocess.run(["readelf", "-d", exe], capture_output=True, text=True).stdout
    assert "[libvrte.so.1]" in need
    return exe


def run(exe, *args):
    return subprocess.run([exe, *args], capture_output=True, text=True, timeout=300)


def test_library_soname():
    out = subprocess.run(["readelf", "-d", V.LIB_PATH], capture_output=True, text=True).stdout
    assert "Library soname: [libvrte.so.1]" in out


@pytest.mark.parametrize("name", MATERIALS)
def test_c_consumer_loads_reference_data(consumer, name):
    r = run(consumer, os.path.join(DATA, name))
    assert r.returncode == 0, r.stderr
    L = {"rayleigh_slab.json": 3, "isotropic_half.json": 1, "conservative_diffuse.json": 1, "paint_film.json": 12}[name]
    layers = 2 if name == "paint_film.json" else 1
    assert r.stdout.strip() == f"version 1.0.0 L {L} layers {layers}"


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/data"), reason="reference tree not present")
def test_c_consumer_loads_the_reference_tree_in_place(consumer):
    for name in MATERIALS:
        r = run(consumer, os.path.join("/root/reference/proj/data", name))
        assert r.returncode == 0, r.stderr


def test_c_consumer_validation_error(consumer, tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text('{"layers": [{"omega": 1.5, "tau": 1.0, "coeff_file": "%s"}], "base": {"type": "black"}}'
                   % os.path.join(DATA, "isotropic.coef"))
    r = run(consumer, str(bad))
    assert r.returncode == 2 and r.stderr.startswith("vrte status 2:")


@pytest.mark.gpu
@pytest.mark.parametrize("name", MATERIALS)
def test_c_consumer_solves_reference_data(consumer, name):
    import pyoracle as O
    r = run(consumer, os.path.join(DATA, name), "8", "--solve")
    assert r.returncode == 0, r.stderr
    line = r.stdout.splitlines()[1].split()
    assert line[:4] == ["size", "2", "8", "5"]
    f00 = float(line[5])
    mat = V.Material.load(os.path.join(DATA, name))
    b = V.compute_brdf(mat, V.options(8), [0.6, 1.0], 5)
    assert f00 == b.table()[0, 0, 0, 0, 0]  # the same library, bit for bit
    L = mat.info()[0]
    S = 2 if name == "paint_film.json" else 1  # distinct media (pipeline.cpp:37-54)
    assert line[8] == "solves"
    assert line[9:] == [str(S * L), str(2 * 4 * 2 * L * S), str(2 * 4 * L)]
