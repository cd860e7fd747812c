"""In-tree build of libvrte.so (host C++ + sm_100a CUDA, one shared object).

nvcc compiles the device pipeline for `-gencode arch=compute_100a,code=sm_100a`
(no other architectures: sm_100a only), g++ compiles the host C ABI, and nvcc
links both with the static CUDA runtime so the library does not depend on the
runtime PyTorch happens to load.  Objects go to build/, the library to
paper_1707_05882_b200/lib/libvrte.so (git-ignored; it travels to the GPU box).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "vrte")
LIB = os.path.join(PKG, "lib", "libvrte.so")
SONAME = "libvrte.so.1"
INCLUDE = os.path.join(ROOT, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _json_include() -> str:
    site = sysconfig.get_paths()["purelib"]
    cand = os.path.join(site, "include", "cudnn_frontend", "thirdparty")
    if os.path.exists(os.path.join(cand, "nlohmann", "json.hpp")):
        return cand
    for d in ("/usr/include", "/usr/local/include"):
        if os.path.exists(os.path.join(d, "nlohmann", "json.hpp")):
            return d
    raise RuntimeError("nlohmann/json.hpp not found")


def sources():
    cu = sorted(os.path.join(CSRC, "cuda", f) for f in os.listdir(os.path.join(CSRC, "cuda"))
                if f.endswith(".cu"))
    cpp = sorted(os.path.join(CSRC, "host", f) for f in os.listdir(os.path.join(CSRC, "host"))
                 if f.endswith(".cpp"))
    return cu, cpp


def _headers():
    hs = []
    for d in (os.path.join(CSRC, "cuda"), os.path.join(CSRC, "host"), os.path.join(INCLUDE, "vrte")):
        hs += [os.path.join(d, f) for f in os.listdir(d) if f.endswith((".h", ".hpp", ".cuh"))]
    return hs


def _stale(obj, src, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src] + deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    nvcc = _nvcc()
    cu, cpp = sources()
    deps = _headers()
    jobs = []
    objs = []
    for s in cu:
        o = os.path.join(BUILD, os.path.basename(s) + ".o")
        objs.append(o)
        if force or _stale(o, s, deps):
            jobs.append([nvcc, "-std=c++17", "-O3", *ARCH, "-lineinfo", "-Xptxas", "-v",
                         "-Xcompiler", "-fPIC,-fvisibility=hidden", "--expt-relaxed-constexpr",
                         "-I", INCLUDE, "-c", s, "-o", o])
    for s in cpp:
        o = os.path.join(BUILD, os.path.basename(s) + ".o")
        objs.append(o)
        if force or _stale(o, s, deps):
            jobs.append(["g++", "-std=c++20", "-O2", "-fPIC", "-fvisibility=hidden", "-Wall",
                         "-I", INCLUDE, "-I", _json_include(), "-I", "/usr/local/cuda/include",
                         "-c", s, "-o", o])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        for out in ex.map(_run, jobs):
            if verbose:
                sys.stdout.write(out)
    if jobs or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        # SONAME libvrte.so.1: the reference's SOVERSION 1 (src/CMakeLists.txt:37-42), so
        # binaries linked against the reference's libvrte resolve to this library
        _run([nvcc, "-shared", *ARCH, "-cudart", "static", "-Xlinker", "-soname=" + SONAME, "-o", LIB, *objs,
              "-lpthread", "-ldl", "-lrt"])
    link = os.path.join(os.path.dirname(LIB), SONAME)
    if os.path.lexists(link) and os.readlink(link) != os.path.basename(LIB):
        os.remove(link)
    if not os.path.lexists(link):
        os.symlink(os.path.basename(LIB), link)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
