"""B200-native drop-in for the reference `vrte` BRDF path (arXiv 1707.05882).

Python mirror of the reference C ABI (/root/reference/proj/include/vrte/vrte.h)
over the in-tree libvrte.so (host C++ + sm_100a kernels).  Same names,
argument meaning, status codes and error text as the reference; there is no
CPU fallback: importing without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libvrte.so")

VRTE_OK = 0
VRTE_E_VALIDATION = 2
VRTE_E_NUMERICAL = 3
VRTE_E_ARGUMENT = 5


class VrteError(RuntimeError):
    """A non-zero vrte_status with vrte_last_error() text."""

    def __init__(self, code: int, message: str):
        super().__init__(f"vrte status {code}: {message}")
        self.code = code
        self.message = message


class Options(C.Structure):
    """vrte_options (vrte.h:54-66); layout is ABI."""
    _fields_ = [
        ("quadrature_n", C.c_int32),
        ("order_cap", C.c_int32),
        ("threads", C.c_int32),
        ("out_zenith", C.c_int32),
        ("out_azimuth", C.c_int32),
        ("incident_mu0", C.c_double),
        ("incident_phi0", C.c_double),
        ("incident_override", C.c_int32),
        ("dump_eigen_path", C.c_char_p),
        ("dump_boundary_path", C.c_char_p),
        ("dump_kernel_path", C.c_char_p),
    ]


class Timings(C.Structure):
    """vrte_timings (vrte.h:75-85)."""
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
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class DeviceStats(C.Structure):
    """vrte_brdf_device_stats (vrte_ext.h)."""
    _fields_ = [
        ("t_homogeneous", C.c_double),
        ("t_particular", C.c_double),
        ("t_boundary", C.c_double),
        ("t_synthesis", C.c_double),
        ("dithered", C.c_uint64),
        ("clamped", C.c_uint64),
        ("polished", C.c_uint64),
        ("kernel_launches", C.c_uint64),
        ("max_eigen_residual", C.c_double),
        ("max_particular_residual", C.c_double),
        ("material_hash", C.c_uint64),
        ("max_balance_residual", C.c_double),
        ("max_boundary_residual", C.c_double),
        ("max_boundary_condition", C.c_double),
        ("boundary_refined", C.c_uint64),
        ("boundary_cond_warnings", C.c_uint64),
        ("boundary_fallback", C.c_uint64),
        ("eigen_slots", C.c_uint64),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class CudaResult(C.Structure):
    """vrte_cuda_result (vrte_cuda.h)."""

    def as_dict(self):
        return {f: (getattr(self, f) if f != "message" else self.message.decode(errors="replace"))
                for f, _ in self._fields_}

    _fields_ = [
        ("t_homogeneous", C.c_double),
        ("t_particular", C.c_double),
        ("t_boundary", C.c_double),
        ("t_synthesis", C.c_double),
        ("t_device", C.c_double),
        ("t_hessenberg", C.c_double),
        ("t_hqr", C.c_double),
        ("t_trevc", C.c_double),
        ("t_refine", C.c_double),
        ("t_lu_factor", C.c_double),
        ("t_lu_solve", C.c_double),
        ("dithered", C.c_uint64),
        ("clamped", C.c_uint64),
        ("polished", C.c_uint64),
        ("kernel_launches", C.c_uint64),
        ("qr_sweeps", C.c_uint64),
        ("qr_steps", C.c_uint64),
        ("qr_cycles", C.c_uint64 * 8),
        ("max_eigen_residual", C.c_double),
        ("max_particular_residual", C.c_double),
        ("max_balance_residual", C.c_double),
        ("max_boundary_residual", C.c_double),
        ("max_boundary_condition", C.c_double),
        ("boundary_refined", C.c_uint64),
        ("boundary_cond_warnings", C.c_uint64),
        ("eigen_slots", C.c_uint64),
        ("slots", C.c_uint64),
        ("boundary_fallback", C.c_uint64),
        ("particular_extra_steps", C.c_uint64),
        ("status", C.c_int32),
        ("message", C.c_char * 512),
    ]


_lib = None

# every symbol include/vrte/*.h exports (tests check the .so against this)
EXPORTED = [
    "vrte_last_error", "vrte_version", "vrte_material_load", "vrte_material_parse",
    "vrte_material_free", "vrte_material_info", "vrte_options_init", "vrte_solve_radiance",
    "vrte_field_size", "vrte_field_row", "vrte_field_write_csv", "vrte_field_timings",
    "vrte_field_reflectance", "vrte_field_free", "vrte_compute_brdf", "vrte_brdf_size",
    "vrte_brdf_entry", "vrte_brdf_write_csv", "vrte_brdf_write_binary", "vrte_brdf_reflectance",
    "vrte_brdf_timings", "vrte_brdf_free", "vrte_mc_trace", "vrte_mc_tally_row",
    "vrte_mc_tally_write_csv", "vrte_mc_tally_free",
    # vrte_ext.h
    "vrte_brdf_device_stats_get", "vrte_brdf_plan_create", "vrte_brdf_from_stacks", "vrte_brdf_grid",
    "vrte_compute_brdf_batch", "vrte_mc_tally_hits",
    # vrte_cuda.h
    "vrte_cuda_brdf", "vrte_cuda_plan_create", "vrte_cuda_plan_run", "vrte_cuda_plan_fetch",
    "vrte_cuda_plan_fetch_up", "vrte_cuda_plan_fetch_modes", "vrte_cuda_plan_fetch_ef",
    "vrte_cuda_plan_destroy",
    "vrte_cuda_synthesize", "vrte_cuda_device_count", "vrte_cuda_current_device", "vrte_cuda_lu_solve", "vrte_cuda_lu_factor", "vrte_cuda_hessenberg", "vrte_cuda_schur",
    "vrte_cuda_radiance_field", "vrte_cuda_mc_trace", "vrte_cuda_host_alloc", "vrte_cuda_host_free",
    "vrte_cuda_debug_force_boundary_fallback", "vrte_cuda_plan_up_device", "vrte_cuda_plan_synthesize_device",
    "vrte_cuda_plan_acquire", "vrte_cuda_plan_release", "vrte_brdf_plan_acquire", "vrte_cuda_schur_trace",
]


def lib():
    """Load libvrte.so (fails loudly if it was not built: no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libvrte.so not built at {LIB_PATH}; run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    vp, dp = C.c_void_p, C.POINTER(C.c_double)
    L.vrte_last_error.restype = C.c_char_p
    L.vrte_version.restype = C.c_char_p
    L.vrte_material_load.argtypes = [C.c_char_p, C.POINTER(vp)]
    L.vrte_material_parse.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(vp)]
    L.vrte_material_free.argtypes = [vp]
    L.vrte_material_info.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.vrte_options_init.argtypes = [C.POINTER(Options)]
    L.vrte_compute_brdf_batch.argtypes = [C.POINTER(vp), C.c_size_t, C.POINTER(Options), dp, C.c_size_t,
                                          C.c_int32, dp, C.c_int32, C.POINTER(vp)]
    L.vrte_compute_brdf.argtypes = [vp, C.POINTER(Options), dp, C.c_size_t, C.c_int32, dp,
                                    C.POINTER(vp)]
    L.vrte_brdf_size.argtypes = [vp, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t),
                                 C.POINTER(C.c_size_t)]
    L.vrte_brdf_entry.argtypes = [vp, C.c_size_t, C.c_size_t, C.c_size_t, dp]
    L.vrte_brdf_write_csv.argtypes = [vp, C.c_char_p]
    L.vrte_brdf_write_binary.argtypes = [vp, C.c_char_p]
    L.vrte_brdf_reflectance.argtypes = [vp, C.c_size_t, dp]
    L.vrte_brdf_timings.argtypes = [vp, C.POINTER(Timings)]
    L.vrte_brdf_free.argtypes = [vp]
    L.vrte_brdf_device_stats_get.argtypes = [vp, C.POINTER(DeviceStats)]
    L.vrte_brdf_grid.argtypes = [vp, dp, dp, dp]
    L.vrte_brdf_plan_create.argtypes = [vp, C.POINTER(Options), dp, C.c_size_t, C.c_int32, dp,
                                        C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(vp)]
    L.vrte_brdf_plan_acquire.argtypes = [vp, C.POINTER(Options), dp, C.c_size_t, C.c_int32, dp,
                                        C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(vp)]
    L.vrte_brdf_from_stacks.argtypes = [vp, C.POINTER(Options), dp, C.c_size_t, C.c_int32, dp, dp,
                                        C.POINTER(vp)]
    L.vrte_cuda_plan_run.argtypes = [vp, C.c_int32, dp, C.POINTER(CudaResult)]
    L.vrte_cuda_plan_fetch.argtypes = [vp, dp]
    L.vrte_cuda_plan_fetch_up.argtypes = [vp, dp]
    L.vrte_cuda_plan_fetch_modes.argtypes = [vp, dp, dp, dp, dp]
    L.vrte_cuda_plan_destroy.argtypes = [vp]
    L.vrte_cuda_plan_fetch_ef.argtypes = [vp, dp, dp]
    L.vrte_cuda_lu_solve.argtypes = [dp, C.c_int32, C.c_int32, dp, C.c_int32, dp, C.c_int32]
    L.vrte_cuda_lu_factor.argtypes = [dp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int32]
    L.vrte_cuda_hessenberg.argtypes = [dp, C.c_int32, C.c_int32, dp, dp, C.c_int32, C.c_int32]
    L.vrte_cuda_debug_force_boundary_fallback.argtypes = [C.c_int32]
    L.vrte_cuda_debug_force_boundary_fallback.restype = None
    L.vrte_cuda_plan_up_device.argtypes = [vp, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]
    L.vrte_cuda_plan_release.argtypes = [vp]
    L.vrte_cuda_plan_release.restype = None
    L.vrte_cuda_plan_synthesize_device.argtypes = [vp, C.c_void_p, dp, C.POINTER(CudaResult)]
    L.vrte_cuda_schur.argtypes = [dp, C.c_int32, C.c_int32, dp, dp, dp, dp, C.c_int32]
    L.vrte_cuda_schur_trace.argtypes = [dp, C.c_int32, C.c_int32, dp, dp, dp, dp, C.c_int32, dp, dp]
    L.vrte_solve_radiance.argtypes = [vp, C.POINTER(Options), dp, C.c_size_t, C.POINTER(vp)]
    L.vrte_field_size.argtypes = [vp, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]
    L.vrte_field_row.argtypes = [vp, C.c_size_t, C.c_size_t, C.c_size_t, dp]
    L.vrte_field_write_csv.argtypes = [vp, C.c_char_p]
    L.vrte_field_timings.argtypes = [vp, C.POINTER(Timings)]
    L.vrte_field_reflectance.argtypes = [vp, dp]
    L.vrte_field_free.argtypes = [vp]
    L.vrte_mc_trace.argtypes = [vp, C.POINTER(Options), C.c_uint64, C.c_uint64, C.c_int32,
                                C.c_int32, C.POINTER(vp)]
    L.vrte_mc_tally_row.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, dp]
    L.vrte_mc_tally_write_csv.argtypes = [vp, C.c_char_p]
    L.vrte_mc_tally_free.argtypes = [vp]
    L.vrte_mc_tally_hits.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_uint64)]
    _lib = L
    return L


def _check(code: int):
    if code != VRTE_OK:
        raise VrteError(code, lib().vrte_last_error().decode(errors="replace"))


def _dp(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def lu_solve(A, B, device: int = 0) -> np.ndarray:
    """Batched dense solve through the boundary stage's row-major LU kernels
    (kernel-level check): A [batch, G, G], B [batch, G, ncol] -> A^-1 B."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    batch, G, _ = A.shape
    ncol = B.shape[2]
    X = np.zeros_like(B)
    code = lib().vrte_cuda_lu_solve(_dp(A), G, batch, _dp(B), ncol, _dp(X), device)
    if code != 0:
        raise VrteError(code, "vrte_cuda_lu_solve failed (singular or bad arguments)")
    return X


def lu_factor(A, G: int, lookahead: bool = True, device: int = 0, deferred: bool = False):
    """Batched in-place row-major LU (kernel-level check): A [batch, G, ncols]
    (columns past G carried along, or with deferred=True eliminated after the
    matrix's factorization through per-block row-map snapshots) -> (factors at
    the physical rows, perm [batch, G]: physical row of each position)."""
    A = np.array(A, dtype=np.float64, order="C", copy=True)
    batch, g, ncols = A.shape
    if g != G:
        raise ValueError("lu_factor: A must be [batch, G, ncols]")
    perm = np.zeros((batch, G), dtype=np.int32)
    code = lib().vrte_cuda_lu_factor(_dp(A), G, ncols, batch, int(bool(lookahead)) | (2 if deferred else 0),
                                     perm.ctypes.data_as(C.POINTER(C.c_int32)), device)
    if code != 0:
        raise VrteError(code, "vrte_cuda_lu_factor failed (singular or bad arguments)")
    return A, perm


class forced_boundary_fallback:
    """Context manager (tests): every BRDF call takes the boundary stage's
    full-solution fallback (vrte_cuda_debug_force_boundary_fallback)."""

    def __enter__(self):
        lib().vrte_cuda_debug_force_boundary_fallback(1)

    def __exit__(self, *exc):
        lib().vrte_cuda_debug_force_boundary_fallback(0)


def hessenberg(A, blocked: bool = True, device: int = 0):
    """Kernel-level check of the Hessenberg stage: A [batch, d, d] (row index
    first) -> (H, Q) with A = Q H Q^T."""
    A = np.asarray(A, dtype=np.float64)
    batch, d, _ = A.shape
    Ac = np.ascontiguousarray(A.transpose(0, 2, 1))  # column-major per matrix
    H, Q = np.zeros_like(Ac), np.zeros_like(Ac)
    code = lib().vrte_cuda_hessenberg(_dp(Ac), d, batch, _dp(H), _dp(Q), int(blocked), device)
    if code != 0:
        raise VrteError(code, "vrte_cuda_hessenberg failed")
    return H.transpose(0, 2, 1).copy(), Q.transpose(0, 2, 1).copy()


def schur(A, device: int = 0):
    """Kernel-level check of the eigen stage: A [batch, d, d] -> (T, Z, w) with
    A = Z T Z^T, T quasi-triangular, w the eigenvalues [batch, d] (complex)."""
    A = np.asarray(A, dtype=np.float64)
    batch, d, _ = A.shape
    Ac = np.ascontiguousarray(A.transpose(0, 2, 1))
    T, Z = np.zeros_like(Ac), np.zeros_like(Ac)
    wr, wi = np.zeros((batch, d)), np.zeros((batch, d))
    code = lib().vrte_cuda_schur(_dp(Ac), d, batch, _dp(T), _dp(Z), _dp(wr), _dp(wi), device)
    if code != 0:
        raise VrteError(code, "vrte_cuda_schur: QR did not converge")
    return T.transpose(0, 2, 1).copy(), Z.transpose(0, 2, 1).copy(), wr + 1j * wi


def schur_trace(A, device: int = 0):
    """Debug: schur() plus the QR kernel's per-matrix profile [batch, 8] (cycles,
    reflectors, sweeps, AED calls, AED cycles, chase cycles, update-wait cycles,
    AED deflations) and its device time in ms."""
    A = np.asarray(A, dtype=np.float64)
    batch, d, _ = A.shape
    Ac = np.ascontiguousarray(A.transpose(0, 2, 1))
    T, Z = np.zeros_like(Ac), np.zeros_like(Ac)
    wr, wi = np.zeros((batch, d)), np.zeros((batch, d))
    tr, ms = np.zeros((batch, 8)), np.zeros(1)
    code = lib().vrte_cuda_schur_trace(_dp(Ac), d, batch, _dp(T), _dp(Z), _dp(wr), _dp(wi), device, _dp(tr), _dp(ms))
    if code != 0:
        raise VrteError(code, "vrte_cuda_schur: QR did not converge")
    return tr, float(ms[0])


def version() -> str:
    return lib().vrte_version().decode()


def options(quadrature_n: int = 40, order_cap: int = 0, **kw) -> Options:
    """vrte_options_init + overrides."""
    o = Options()
    lib().vrte_options_init(C.byref(o))
    o.quadrature_n = quadrature_n
    o.order_cap = order_cap
    for k, v in kw.items():
        setattr(o, k, v)
    return o


class Material:
    """Opaque vrte_material handle (vrte_material_load / vrte_material_parse)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def load(cls, path: str) -> "Material":
        h = C.c_void_p()
        _check(lib().vrte_material_load(path.encode(), C.byref(h)))
        return cls(h)

    @classmethod
    def parse(cls, json_text: str, base_dir: str = "") -> "Material":
        h = C.c_void_p()
        _check(lib().vrte_material_parse(json_text.encode(), base_dir.encode(), C.byref(h)))
        return cls(h)

    def info(self):
        L, P = C.c_int32(), C.c_int32()
        _check(lib().vrte_material_info(self._h, C.byref(L), C.byref(P)))
        return L.value, P.value

    def close(self):
        if self._h:
            lib().vrte_material_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Brdf:
    """Opaque vrte_brdf handle with the table mirrored as a numpy array."""

    def __init__(self, handle):
        self._h = handle
        ni, no, npd = C.c_size_t(), C.c_size_t(), C.c_size_t()
        _check(lib().vrte_brdf_size(handle, C.byref(ni), C.byref(no), C.byref(npd)))
        self.shape = (ni.value, no.value, npd.value)

    def entry(self, i, o, p) -> np.ndarray:
        e = np.zeros(16)
        _check(lib().vrte_brdf_entry(self._h, i, o, p, _dp(e)))
        return e.reshape(4, 4)

    def table(self) -> np.ndarray:
        """[n_in, n_out, n_dphi, 4, 4] (row-major Mueller entries)."""
        ni, no, npd = self.shape
        out = np.zeros((ni, no, npd, 4, 4))
        e = np.zeros(16)
        for i in range(ni):
            for o in range(no):
                for p in range(npd):
                    _check(lib().vrte_brdf_entry(self._h, i, o, p, _dp(e)))
                    out[i, o, p] = e.reshape(4, 4)
        return out

    def mu_out(self) -> np.ndarray:
        """Exit cosines of the table (vrte_brdf_grid, vrte_ext.h)."""
        out = np.zeros(self.shape[1])
        _check(lib().vrte_brdf_grid(self._h, None, _dp(out), None))
        return out

    def reflectance(self, i) -> np.ndarray:
        r = np.zeros(4)
        _check(lib().vrte_brdf_reflectance(self._h, i, _dp(r)))
        return r

    def timings(self) -> dict:
        t = Timings()
        _check(lib().vrte_brdf_timings(self._h, C.byref(t)))
        return t.as_dict()

    def device_stats(self) -> dict:
        s = DeviceStats()
        _check(lib().vrte_brdf_device_stats_get(self._h, C.byref(s)))
        return s.as_dict()

    def write_csv(self, path: str):
        _check(lib().vrte_brdf_write_csv(self._h, path.encode()))

    def write_binary(self, path: str):
        _check(lib().vrte_brdf_write_binary(self._h, path.encode()))

    def close(self):
        if self._h:
            lib().vrte_brdf_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def compute_brdf(material: Material, opts: Options, mu_in, n_dphi: int = 19, basis=None) -> Brdf:
    """vrte_compute_brdf (vrte.h:110-112) on the sm_100a pipeline."""
    mu = np.ascontiguousarray(mu_in, dtype=np.float64)
    b = None if basis is None else np.ascontiguousarray(basis, dtype=np.float64).reshape(16)
    h = C.c_void_p()
    _check(lib().vrte_compute_brdf(material._h, C.byref(opts), _dp(mu), len(mu), n_dphi, _dp(b),
                                   C.byref(h)))
    return Brdf(h)


class Field:
    """Opaque vrte_field handle (vrte.h:87-98): radiance on the (tau, signed mu, phi) grid."""

    def __init__(self, handle):
        self._h = handle
        nt, nm, npd = C.c_size_t(), C.c_size_t(), C.c_size_t()
        _check(lib().vrte_field_size(handle, C.byref(nt), C.byref(nm), C.byref(npd)))
        self.shape = (nt.value, nm.value, npd.value)

    def row(self, it, imu, ip) -> np.ndarray:
        r = np.zeros(7)
        _check(lib().vrte_field_row(self._h, it, imu, ip, _dp(r)))
        return r

    def values(self):
        """(taus, mus, phis, stokes [n_tau, n_mu, n_phi, 4]) via vrte_field_row."""
        nt, nm, npd = self.shape
        out = np.zeros((nt, nm, npd, 4))
        taus, mus, phis = np.zeros(nt), np.zeros(nm), np.zeros(npd)
        r = np.zeros(7)
        for it in range(nt):
            for im in range(nm):
                for ip in range(npd):
                    _check(lib().vrte_field_row(self._h, it, im, ip, _dp(r)))
                    out[it, im, ip] = r[3:]
                    taus[it], mus[im], phis[ip] = r[0], r[1], r[2]
        return taus, mus, phis, out

    def reflectance(self) -> np.ndarray:
        r = np.zeros(4)
        _check(lib().vrte_field_reflectance(self._h, _dp(r)))
        return r

    def timings(self) -> Timings:
        t = Timings()
        _check(lib().vrte_field_timings(self._h, C.byref(t)))
        return t

    def write_csv(self, path: str):
        _check(lib().vrte_field_write_csv(self._h, path.encode()))

    def close(self):
        if self._h:
            lib().vrte_field_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_radiance(material: Material, opts: Options, taus=()) -> Field:
    """vrte_solve_radiance (vrte.h:87-89) on the sm_100a pipeline + radiance.cu."""
    t = np.ascontiguousarray(taus, dtype=np.float64)
    h = C.c_void_p()
    _check(lib().vrte_solve_radiance(material._h, C.byref(opts), _dp(t) if len(t) else None, len(t),
                                     C.byref(h)))
    return Field(h)


class McTally:
    """Opaque vrte_mc_tally handle (vrte.h:119-129): binned exiting radiance of the tracer."""

    def __init__(self, handle, zb, ab):
        self._h, self.zb, self.ab = handle, zb, ab

    def row(self, hemisphere, iz, ia) -> np.ndarray:
        """(mu center, phi center, I, Q, U, V, se_I, se_Q, se_U, se_V)"""
        r = np.zeros(10)
        _check(lib().vrte_mc_tally_row(self._h, hemisphere, iz, ia, _dp(r)))
        return r

    def rows(self) -> np.ndarray:
        return np.array([[[self.row(h, iz, ia) for ia in range(self.ab)] for iz in range(self.zb)] for h in (0, 1)])

    def hits(self) -> np.ndarray:
        """[2, zb, ab] photon counts (vrte_mc_tally_hits, vrte_ext.h)"""
        out = np.zeros((2, self.zb, self.ab), dtype=np.int64)
        v = C.c_uint64()
        for h in (0, 1):
            for iz in range(self.zb):
                for ia in range(self.ab):
                    _check(lib().vrte_mc_tally_hits(self._h, h, iz, ia, C.byref(v)))
                    out[h, iz, ia] = v.value
        return out

    def write_csv(self, path: str):
        _check(lib().vrte_mc_tally_write_csv(self._h, path.encode()))

    def close(self):
        if self._h:
            lib().vrte_mc_tally_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def mc_trace(material: Material, opts: Options, photons: int, seed: int, zenith_bins: int,
             azimuth_bins: int) -> McTally:
    """vrte_mc_trace (vrte.h:123-125) on the GPU tracer (mc.cu)."""
    h = C.c_void_p()
    _check(lib().vrte_mc_trace(material._h, C.byref(opts), photons, seed, zenith_bins, azimuth_bins, C.byref(h)))
    return McTally(h, zenith_bins, azimuth_bins)


def compute_brdf_batch(materials, opts: Options, mu_in, n_dphi: int = 19, basis=None,
                       concurrency: int = 2):
    """vrte_compute_brdf_batch (vrte_ext.h): independent requests (e.g. spectral
    bands) solved concurrently, one plan / CUDA stream each.  Returns a list of
    Brdf handles; raises VrteError with the first failure."""
    mu = np.ascontiguousarray(mu_in, dtype=np.float64)
    b = None if basis is None else np.ascontiguousarray(basis, dtype=np.float64).reshape(16)
    n = len(materials)
    mats = (C.c_void_p * n)(*[m._h for m in materials])
    outs = (C.c_void_p * n)()
    code = lib().vrte_compute_brdf_batch(mats, n, C.byref(opts), _dp(mu), len(mu), n_dphi, _dp(b),
                                         concurrency, outs)
    handles = [Brdf(C.c_void_p(outs[i])) if outs[i] else None for i in range(n)]
    if code != VRTE_OK:
        msg = lib().vrte_last_error().decode(errors="replace")
        for h in handles:
            if h is not None:
                h.close()
        raise VrteError(code, msg)
    return handles


def brdf_from_stacks(material: Material, opts: Options, mu_in, n_dphi, basis, up_all) -> Brdf:
    """vrte_brdf_from_stacks: BRDF handle from gathered per-order tau=0 stacks
    [L, n_in, 4, N, 4] (the multi-GPU root step; synthesis runs on the GPU)."""
    mu = np.ascontiguousarray(mu_in, dtype=np.float64)
    b = None if basis is None else np.ascontiguousarray(basis, dtype=np.float64).reshape(16)
    up = np.ascontiguousarray(up_all, dtype=np.float64)
    h = C.c_void_p()
    _check(lib().vrte_brdf_from_stacks(material._h, C.byref(opts), _dp(mu), len(mu), n_dphi, _dp(b),
                                       _dp(up), C.byref(h)))
    return Brdf(h)


def read_brdf_binary(path: str):
    """VRTEBRDF v1 reader (csv.cpp:170-203): (mu_in, mu_out, dphi, table)."""
    with open(path, "rb") as f:
        raw = f.read()
    if raw[:8] != b"VRTEBRDF":
        raise ValueError(path + ": not a brdf table")
    ver, ni, no, npd = np.frombuffer(raw[8:24], dtype="<u4")
    if ver != 1:
        raise ValueError(path + ": unsupported brdf table version")
    off = 24
    mu_in = np.frombuffer(raw, "<f8", ni, off); off += 8 * ni
    mu_out = np.frombuffer(raw, "<f8", no, off); off += 8 * no
    dphi = np.frombuffer(raw, "<f8", npd, off); off += 8 * npd
    tab = np.frombuffer(raw, "<f8", ni * no * npd * 16, off).reshape(ni, no, npd, 4, 4)
    return mu_in.copy(), mu_out.copy(), dphi.copy(), tab.copy()


class Plan:
    """Device-resident solve plan (vrte_brdf_plan_create / vrte_cuda_plan_*)."""

    def __init__(self, material: Material, opts: Options, mu_in, n_dphi=19, basis=None,
                 device=-1, m_begin=0, m_stride=1, n_orders=0, pooled=False):
        """Creating the plan solves once.  pooled: lease the device buffers from
        the process pool (vrte_brdf_plan_acquire; close() returns them)."""
        mu = np.ascontiguousarray(mu_in, dtype=np.float64)
        b = None if basis is None else np.ascontiguousarray(basis, dtype=np.float64).reshape(16)
        h = C.c_void_p()
        fn = lib().vrte_brdf_plan_acquire if pooled else lib().vrte_brdf_plan_create
        _check(fn(material._h, C.byref(opts), _dp(mu), len(mu), n_dphi, _dp(b), device, m_begin, m_stride, n_orders,
                  C.byref(h)))
        self._h = h
        self.pooled = pooled
        self.device = device if device >= 0 else lib().vrte_cuda_current_device()
        self.n_in, self.n_dphi = len(mu), n_dphi
        self.N = opts.quadrature_n
        self.L = min(material.info()[0], opts.order_cap) if opts.order_cap > 0 else material.info()[0]
        self.n_orders = n_orders if n_orders > 0 else self.L
        self.last = CudaResult()

    def run(self, iters: int = 1) -> float:
        """Average device seconds per solve over `iters` back-to-back solves."""
        s = C.c_double()
        code = lib().vrte_cuda_plan_run(self._h, iters, C.byref(s), C.byref(self.last))
        if code != 0:
            raise VrteError(code, self.last.message.decode(errors="replace"))
        return s.value

    def table(self) -> np.ndarray:
        out = np.zeros((self.n_in, self.N, self.n_dphi, 4, 4))
        _check(lib().vrte_cuda_plan_fetch(self._h, _dp(out)))
        return out

    def up(self) -> np.ndarray:
        """tau=0 upward stacks [n_orders, n_in, 4 channels, N, 4 Stokes]."""
        out = np.zeros((self.n_orders, self.n_in, 4, self.N, 4))
        _check(lib().vrte_cuda_plan_fetch_up(self._h, _dp(out)))
        return out

    def up_device(self):
        """The tau = 0 stacks on the device, zero-copy, as a torch tensor
        [n_orders, 4 n_in, 4N] (valid until the plan's next run or close)."""
        import torch
        ptr, n = C.c_void_p(), C.c_size_t()
        _check(lib().vrte_cuda_plan_up_device(self._h, C.byref(ptr), C.byref(n)))
        shape = (self.n_orders, 4 * self.n_in, 4 * self.N)

        class _View:  # __cuda_array_interface__ v3 over the plan's buffer
            __cuda_array_interface__ = {"shape": shape, "typestr": "<f8", "data": (ptr.value, False),
                                        "version": 3, "strides": None}

        return torch.as_tensor(_View(), device=torch.device("cuda", self.device))

    def synthesize_device(self, up_all, fetch: bool = True):
        """Synthesis of all L orders from device stacks up_all (torch tensor
        [L, 4 n_in, 4N] on this plan's device, order m at index m); returns the
        host table [n_in, N, n_dphi, 4, 4] (fetch) or None."""
        import torch
        assert up_all.is_cuda and up_all.dtype == torch.float64 and up_all.is_contiguous()
        torch.cuda.current_stream(up_all.device).synchronize()  # its writes precede the plan's stream
        out = np.zeros((self.n_in, self.N, self.n_dphi, 4, 4)) if fetch else None
        r = CudaResult()
        code = lib().vrte_cuda_plan_synthesize_device(self._h, C.c_void_p(up_all.data_ptr()),
                                                      _dp(out) if fetch else None, C.byref(r))
        if code != 0:
            raise VrteError(code, r.message.decode(errors="replace"))
        return out

    def modes(self, n_media: int):
        d = 4 * self.N
        n = n_media * self.n_orders * d
        wr, wi, res, nu = np.zeros(n), np.zeros(n), np.zeros(n), np.zeros(2 * n)
        _check(lib().vrte_cuda_plan_fetch_modes(self._h, _dp(wr), _dp(wi), _dp(res), _dp(nu)))
        sh = (n_media, self.n_orders, d)
        return (wr.reshape(sh), wi.reshape(sh), res.reshape(sh),
                (nu[0::2] + 1j * nu[1::2]).reshape(sh))

    def ef(self, n_media: int):
        """Reduced operators E, F as [n_media, n_orders, d, d] (row index i, column j)."""
        d = 4 * self.N
        n = n_media * self.n_orders * d * d
        E, F = np.zeros(n), np.zeros(n)
        _check(lib().vrte_cuda_plan_fetch_ef(self._h, _dp(E), _dp(F)))
        sh = (n_media, self.n_orders, d, d)
        return E.reshape(sh).transpose(0, 1, 3, 2).copy(), F.reshape(sh).transpose(0, 1, 3, 2).copy()

    def close(self):
        if getattr(self, "_h", None):
            if getattr(self, "pooled", False):
                lib().vrte_cuda_plan_release(self._h)
            else:
                lib().vrte_cuda_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
