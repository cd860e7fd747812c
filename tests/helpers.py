"""Shared helpers for the parity tests (test infrastructure)."""
import json
import os
import tempfile

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def survey_metric(got, ref):
    """per Mueller matrix, max_rc |G-R| / max(|R_rc|, 1e-3 |R_00|)."""
    r00 = np.abs(ref[..., 0, 0])[..., None, None]
    den = np.maximum(np.abs(ref), 1e-3 * r00)
    den = np.where(den == 0, 1e-300, den)
    return float(np.max(np.abs(got - ref) / den))


def element_metric(got, ref):
    """Plain per-element relative error over the entries with |R_rc| >= 1e-3 |R_00|."""
    r00 = np.abs(ref[..., 0, 0])[..., None, None]
    keep = (np.abs(ref) >= 1e-3 * r00) & (np.abs(ref) > 0)
    if not keep.any():
        return 0.0
    return float(np.max(np.abs(got - ref)[keep] / np.abs(ref)[keep]))


def matrix_metric(got, ref):
    """Per Mueller matrix, max_rc |G-R| / max_rc |R_rc| (relative to the matrix scale)."""
    sc = np.abs(ref).reshape(ref.shape[:-2] + (16,)).max(-1)[..., None, None]
    sc = np.where(sc == 0, 1.0, sc)
    return float(np.max(np.abs(got - ref) / sc))


def oracle_material(desc):
    import pyoracle as O
    bt = {"black": 0, "lambertian": 1, "mueller_table": 2}[desc.base]
    return O.Material(np.array([l.omega for l in desc.layers]), np.array([l.tau for l in desc.layers]),
                      desc.padded_coeffs(), bt, desc.albedo, desc.table)


def product_material(desc):
    """Write the material as JSON + coefficient files and load it through the C ABI."""
    import paper_1707_05882_b200 as V
    d = tempfile.mkdtemp(prefix="vrte_mat_")
    return V.Material.load(desc.write(d, "m"))


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)
    meta = json.loads(str(z["meta"]))
    return z, meta


def desc_from_golden(z, meta):
    from paper_1707_05882_b200 import materials as M
    layers = [M.LayerDesc(l["omega"], l["tau"], z["coeffs"][p]) for p, l in enumerate(meta["layers"])]
    return M.MaterialDesc(layers, base=meta["base"], albedo=meta["albedo"])


def survey_den(ref):
    r00 = np.abs(ref[..., 0, 0])[..., None, None]
    den = np.maximum(np.abs(ref), 1e-3 * r00)
    return np.where(den == 0, 1e-300, den)


def sensitivity_metric(got, ref, ref_perturbed, k=2.0):
    """SURVEY §8(d) metric with the reference's own rounding sensitivity allowed
    for: max over elements of (|G-R| - k |R'-R|) / den, where R' is the same
    reference run on inputs perturbed by ~1e-15 relative (its fp64 noise floor
    at that element).  <= 1e-9 means: within 1e-9 wherever the reference's
    answer is itself stable to 1e-9, and within k times its own rounding
    movement where it is not."""
    den = survey_den(ref)
    return float(np.max((np.abs(got - ref) - k * np.abs(ref_perturbed - ref)) / den))


def survey_per_matrix(got, ref):
    return (np.abs(got - ref) / survey_den(ref)).max(axis=(-1, -2))


def perturbed(om, rel=1e-15):
    """The oracle material with every single-scattering albedo scaled by (1 + rel)."""
    import copy
    q = copy.copy(om)
    q.omega = np.asarray(om.omega, float) * (1.0 + rel)
    return q
