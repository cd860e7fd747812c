"""ctypes binding of the CPU restatement oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference leg
import this module.  The product path (libvrte.so, paper_1707_05882_b200)
never imports or calls it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libvrte_oracle.so")


def build() -> str:
    """Compile the oracle (make) if needed; returns the .so path."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


class OracleMaterial(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int32),
        ("order_count", C.c_int32),
        ("omega", C.POINTER(C.c_double)),
        ("tau", C.POINTER(C.c_double)),
        ("coeffs", C.POINTER(C.c_double)),
        ("base_type", C.c_int32),
        ("rho", C.c_double),
        ("table_n", C.c_int32),
        ("table", C.POINTER(C.c_double)),
    ]


class OracleTimings(C.Structure):
    _fields_ = [
        ("homogeneous", C.c_double),
        ("particular", C.c_double),
        ("boundary", C.c_double),
        ("reconstruction", C.c_double),
        ("total_wall", C.c_double),
        ("homogeneous_solves", C.c_uint64),
        ("particular_solves", C.c_uint64),
        ("boundary_solves", C.c_uint64),
        ("reconstruction_items", C.c_uint64),
        ("clamped_entries", C.c_uint64),
        ("dithered", C.c_uint64),
        ("max_eigen_residual", C.c_double),
        ("max_boundary_condition", C.c_double),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        dp = C.POINTER(C.c_double)
        mp = C.POINTER(OracleMaterial)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_quadrature.argtypes = [C.c_int32, dp, dp]
        L.oracle_wigner_d_sequence.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_double, dp]
        L.oracle_gsf_sequence.argtypes = [C.c_int32, C.c_int32, C.c_double, dp, dp, dp]
        L.oracle_kernel_blocks.argtypes = [mp, C.c_int32, C.c_int32, C.c_int32, dp, dp, dp, dp]
        L.oracle_beam_column.argtypes = [mp, C.c_int32, C.c_int32, C.c_int32, C.c_double, dp, dp]
        L.oracle_reduced_ops.argtypes = [mp, C.c_int32, C.c_int32, C.c_int32, dp, dp]
        L.oracle_homogeneous.argtypes = [mp, C.c_int32, C.c_int32, C.c_int32, dp, dp, dp, dp]
        L.oracle_particular.argtypes = [mp, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_double, dp, dp, dp, dp, dp]
        L.oracle_set_accurate.argtypes = [C.c_int32]
        L.oracle_set_cache_boundary.argtypes = [C.c_int32]
        L.oracle_brdf.argtypes = [mp, C.c_int32, C.c_int32, C.c_int32, dp, C.c_size_t,
                                  C.c_int32, dp, dp, C.POINTER(OracleTimings), dp]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def _check(code):
    if code != 0:
        raise OracleError(code, lib().oracle_last_error().decode())


@dataclass
class Material:
    """Plain-array material (layers top first), see oracle_material."""
    omega: np.ndarray           # [P]
    tau: np.ndarray             # [P]
    coeffs: np.ndarray          # [P, L, 4, 4]
    base_type: int = 0          # 0 black, 1 lambertian, 2 table
    rho: float = 0.0
    table: np.ndarray | None = None  # [n, n, 4, 4]

    def c(self):
        self._keep = [np.ascontiguousarray(self.omega, np.float64),
                      np.ascontiguousarray(self.tau, np.float64),
                      np.ascontiguousarray(self.coeffs, np.float64)]
        tab = None
        n = 0
        if self.table is not None:
            tab = np.ascontiguousarray(self.table, np.float64)
            n = tab.shape[0]
            self._keep.append(tab)
        return OracleMaterial(len(self.omega), self.coeffs.shape[1], _dp(self._keep[0]),
                              _dp(self._keep[1]), _dp(self._keep[2]), self.base_type,
                              float(self.rho), n, _dp(tab))


class accurate:
    """Context manager: run the oracle in accurate mode (see vrte_oracle.h)."""

    def __enter__(self):
        lib().oracle_set_accurate(1)

    def __exit__(self, *exc):
        lib().oracle_set_accurate(0)


class cached_boundary:
    """Context manager: reuse each order's boundary LU across incidents (bit-identical
    results, see oracle_set_cache_boundary); for full-table parity tests only."""

    def __enter__(self):
        lib().oracle_set_cache_boundary(1)

    def __exit__(self, *exc):
        lib().oracle_set_cache_boundary(0)


def quadrature(n):
    nodes = np.zeros(n)
    w = np.zeros(n)
    _check(lib().oracle_quadrature(n, _dp(nodes), _dp(w)))
    return nodes, w


def wigner_d_sequence(m, n, lmax, x):
    out = np.zeros(lmax + 1)
    lib().oracle_wigner_d_sequence(m, n, lmax, x, _dp(out))
    return out


def gsf_sequence(m, lmax, x):
    p, r, t = np.zeros(lmax + 1), np.zeros(lmax + 1), np.zeros(lmax + 1)
    lib().oracle_gsf_sequence(m, lmax, x, _dp(p), _dp(r), _dp(t))
    return p, r, t


def kernel_blocks(mat: Material, layer, N, m):
    arrs = [np.zeros((N * N, 4, 4)) for _ in range(4)]
    cm = mat.c()
    _check(lib().oracle_kernel_blocks(C.byref(cm), layer, N, m, *[_dp(a) for a in arrs]))
    return [a.reshape(N, N, 4, 4) for a in arrs]


def beam_column(mat: Material, layer, N, m, mu_beam):
    up, dn = np.zeros((N, 4, 4)), np.zeros((N, 4, 4))
    cm = mat.c()
    _check(lib().oracle_beam_column(C.byref(cm), layer, N, m, mu_beam, _dp(up), _dp(dn)))
    return up, dn


def reduced_ops(mat: Material, layer, N, m):
    d = 4 * N
    e, f = np.zeros(d * d), np.zeros(d * d)
    cm = mat.c()
    _check(lib().oracle_reduced_ops(C.byref(cm), layer, N, m, _dp(e), _dp(f)))
    return e.reshape(d, d).T.copy(), f.reshape(d, d).T.copy()  # col-major -> [i, j]


def homogeneous(mat: Material, layer, N, m, vectors=False):
    d = 4 * N
    nu = np.zeros(2 * d)
    res = np.zeros(d)
    pp = np.zeros(2 * d * d) if vectors else None
    pm = np.zeros(2 * d * d) if vectors else None
    cm = mat.c()
    _check(lib().oracle_homogeneous(C.byref(cm), layer, N, m, _dp(nu), _dp(res), _dp(pp),
                                    _dp(pm)))
    nu_c = nu[0::2] + 1j * nu[1::2]
    if not vectors:
        return nu_c, res
    pp_c = (pp[0::2] + 1j * pp[1::2]).reshape(d, d)
    pm_c = (pm[0::2] + 1j * pm[1::2]).reshape(d, d)
    return nu_c, res, pp_c, pm_c


def particular(mat: Material, layer, N, m, k, mu0, stokes):
    d = 4 * N
    zp, zm = np.zeros(d), np.zeros(d)
    mu_eff = C.c_double(0)
    res = C.c_double(0)
    st = np.ascontiguousarray(stokes, np.float64)
    cm = mat.c()
    _check(lib().oracle_particular(C.byref(cm), layer, N, m, k, mu0, _dp(st), _dp(zp), _dp(zm),
                                   C.byref(mu_eff), C.byref(res)))
    return zp, zm, mu_eff.value, res.value


def brdf(mat: Material, N, mu_in, n_dphi=19, basis=None, order_cap=0, threads=0,
         components=False):
    """Full F_r table [n_in, N, n_dphi, 4, 4] (+ timings dict)."""
    mu = np.ascontiguousarray(mu_in, np.float64)
    out = np.zeros((len(mu), N, n_dphi, 4, 4))
    b = None if basis is None else np.ascontiguousarray(basis, np.float64).reshape(16)
    tm = OracleTimings()
    L = mat.coeffs.shape[1] if order_cap <= 0 else min(order_cap, mat.coeffs.shape[1])
    comps = np.zeros(len(mu) * 4 * L * 2 * 4 * N * 2) if components else None
    cm = mat.c()
    _check(lib().oracle_brdf(C.byref(cm), N, order_cap, threads, _dp(mu), len(mu), n_dphi,
                             _dp(b), _dp(out), C.byref(tm), _dp(comps)))
    t = {f: getattr(tm, f) for f, _ in OracleTimings._fields_}
    if components:
        cc = comps[0::2] + 1j * comps[1::2]
        return out, t, cc.reshape(len(mu), 4, L, 2, 4 * N)
    return out, t


def radiance(mat: Material, N, mu0, phi0, stokes, taus=(0.0,), zenith=11, azimuth=19, mus=None,
             phis=None, nodal=False, order_cap=0, threads=0):
    """capi.cpp:138-174 restated: (values [n_tau, n_mu, n_phi, 4], mus, phis,
    reflectance[4]).  nodal=True: discrete-ordinate stacks at +nodes, -nodes."""
    tv = np.ascontiguousarray(taus, np.float64)
    st = np.ascontiguousarray(stokes, np.float64)
    mu_in = None if mus is None else np.ascontiguousarray(mus, np.float64)
    ph_in = None if phis is None else np.ascontiguousarray(phis, np.float64)
    n_mu = 2 * N if nodal else (len(mu_in) if mu_in is not None else 2 * zenith)
    n_ph = len(ph_in) if ph_in is not None else azimuth
    vals = np.zeros((max(1, len(tv)), n_mu, n_ph, 4))
    mo = np.zeros(n_mu)
    po = np.zeros(n_ph)
    refl = np.zeros(4)
    tm = OracleTimings()
    cm = mat.c()
    lib().oracle_radiance_at.argtypes = None
    _check(lib().oracle_radiance_at(C.byref(cm), N, order_cap, threads, C.c_double(mu0), C.c_double(phi0),
                                    _dp(st), _dp(tv), C.c_size_t(len(tv)), zenith, azimuth, _dp(mu_in),
                                    C.c_size_t(0 if mu_in is None else len(mu_in)), _dp(ph_in),
                                    C.c_size_t(0 if ph_in is None else len(ph_in)), 1 if nodal else 0,
                                    _dp(mo), _dp(po), _dp(vals), _dp(refl), C.byref(tm)))
    return vals, mo, po, refl


class McTally:
    """mc.hpp TallyGrid: raw sums [2, zb, ab, 4], hits [2, zb, ab] and the flux-weighted
    bin-average radiance / standard error of mc.cpp:233-253."""

    def __init__(self, s, sq, hits, photons, mu0, zb, ab):
        self.sum, self.sum_sq, self.hits = s, sq, hits
        self.photons, self.mu0, self.zb, self.ab = photons, mu0, zb, ab

    def bin_flux_measure(self, iz):
        lo, hi = iz / self.zb, (iz + 1) / self.zb
        return 0.5 * (hi * hi - lo * lo) * (2 * np.pi / self.ab)

    def radiance(self, hemi, iz, ia):
        return self.sum[hemi, iz, ia] * self.mu0 / (self.photons * self.bin_flux_measure(iz))

    def std_error(self, hemi, iz, ia):
        n = float(self.photons)
        mean = self.sum[hemi, iz, ia] / n
        var = np.maximum(0.0, self.sum_sq[hemi, iz, ia] / n - mean * mean)
        return self.mu0 / self.bin_flux_measure(iz) * np.sqrt(var / max(1.0, n - 1.0))


def mc_trace(mat: Material, mu0, phi0, stokes, photons, seed, zb, ab, threads=0) -> McTally:
    s = np.zeros((2, zb, ab, 4))
    sq = np.zeros((2, zb, ab, 4))
    h = np.zeros((2, zb, ab), dtype=np.uint64)
    st = np.ascontiguousarray(stokes, np.float64)
    cm = mat.c()
    _check(lib().oracle_mc_trace(C.byref(cm), C.c_double(mu0), C.c_double(phi0), _dp(st), C.c_uint64(photons),
                                 C.c_uint64(seed), zb, ab, threads, _dp(s), _dp(sq),
                                 h.ctypes.data_as(C.POINTER(C.c_uint64))))
    return McTally(s, sq, h, photons, mu0, zb, ab)
