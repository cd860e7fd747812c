"""Material inputs for the BRDF path (host-side plumbing, no compute).

Mirrors the reference's material ingest (/root/reference/proj/src/core/
material.cpp:111-161 coefficient rows "l beta alpha gamma delta epsilon zeta",
material.cpp:195-250 JSON schema) and the synthetic workloads of SURVEY.md
§8(d): the Greek generator G(g, L) and configs C1..C5.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field

import numpy as np


def greek(beta, alpha, gamma, delta, eps, zeta):
    """4x4 B_l in the 2+2 block layout (material.cpp:147-154)."""
    b = np.zeros((4, 4))
    b[0, 0] = beta
    b[1, 1] = alpha
    b[0, 1] = b[1, 0] = gamma
    b[3, 3] = delta
    b[2, 2] = zeta
    b[2, 3] = -eps
    b[3, 2] = eps
    return b


def greek_rows(coeffs):
    """Inverse of greek(): rows (beta, alpha, gamma, delta, eps, zeta)."""
    return [(b[0, 0], b[1, 1], b[0, 1], b[3, 3], b[3, 2], b[2, 2]) for b in coeffs]


def generator_G(g: float, L: int, pol: float = 1.0) -> np.ndarray:
    """SURVEY.md §8(d) Greek generator; G(0.5, 12) == data/forward12.coef.

    `pol` scales every polarization coefficient (alpha, gamma, delta, epsilon,
    zeta; beta untouched): pol = 0.5 is the C4' set (see config("C4p"))."""
    out = np.zeros((L, 4, 4))
    for l in range(L):
        beta = (2 * l + 1) * g ** l
        if l >= 2:
            a, gm, e, z = 0.9 * pol * beta, -0.35 * pol * beta, 0.12 * pol * beta, 0.8 * pol * beta
        else:
            a = gm = e = z = 0.0
        dl = 0.3 * pol if l == 0 else 0.7 * pol * beta
        out[l] = greek(beta, a, gm, dl, e, z)
    return out


ISOTROPIC = np.array([greek(1, 0, 0, 0, 0, 0)])
RAYLEIGH = np.array([greek(1, 0, 0, 0, 0, 0), greek(0, 0, 0, 1.5, 0, 0),
                     greek(0.5, 3.0, -math.sqrt(6.0) / 2.0, 0, 0, 0)])
# tests/support/materials.hpp:44-51 (all Greek channels, not physical)
FULL = np.array([greek(1, 0, 0, 0.3, 0, 0), greek(0.5, 0, 0, 0.6, 0, 0),
                 greek(0.7, 2.5, -0.9, 0.4, 0.3, 1.1), greek(0.3, 1.2, 0.4, 0.2, -0.2, 0.5)])


def format_double(v: float) -> str:
    """%.17g, the reference's lossless text format (csv.cpp:11-15)."""
    return "%.17g" % v


def write_coef(path: str, coeffs: np.ndarray) -> None:
    with open(path, "w") as f:
        f.write("# l beta alpha gamma delta epsilon zeta\n")
        for l, row in enumerate(greek_rows(coeffs)):
            f.write(str(l) + " " + " ".join(format_double(float(x)) for x in row) + "\n")


def read_coef(path: str) -> np.ndarray:
    rows = {}
    with open(path) as f:
        for line in f:
            s = line.strip()
            if not s or s.startswith("#"):
                continue
            t = s.split()
            rows[int(t[0])] = [float(x) for x in t[1:7]]
    return np.array([greek(*rows[l]) for l in range(max(rows) + 1)])


@dataclass
class LayerDesc:
    omega: float
    tau: float
    coeffs: np.ndarray


@dataclass
class MaterialDesc:
    """Layer stack (top first) over a base; mirrors MaterialSpec (material.hpp:59-71)."""
    layers: list
    base: str = "black"          # black | lambertian | mueller_table
    albedo: float = 0.0
    table: np.ndarray | None = None   # [n, n, 4, 4] for mueller_table
    mu0: float = 0.6
    phi0: float = 0.0
    stokes: tuple = (1.0, 0.0, 0.0, 0.0)
    interface_n: float = 1.0      # Fresnel top interface (extension; 1 = none, the reference's model)

    @property
    def order_count(self) -> int:
        return max(l.coeffs.shape[0] for l in self.layers)

    def padded_coeffs(self) -> np.ndarray:
        """[P, L, 4, 4] zero-padded to the common order count (material.cpp:106-108)."""
        L = self.order_count
        out = np.zeros((len(self.layers), L, 4, 4))
        for p, l in enumerate(self.layers):
            out[p, :l.coeffs.shape[0]] = l.coeffs
        return out

    def write(self, directory: str, name: str = "material") -> str:
        """Write the JSON + coefficient (+ table) files; returns the JSON path."""
        os.makedirs(directory, exist_ok=True)
        doc = {"layers": []}
        for p, l in enumerate(self.layers):
            cf = f"{name}_layer{p}.coef"
            write_coef(os.path.join(directory, cf), l.coeffs)
            doc["layers"].append({"omega": l.omega, "tau": l.tau, "coeff_file": cf})
        if self.base == "lambertian":
            doc["base"] = {"type": "lambertian", "albedo": self.albedo}
        elif self.base == "mueller_table":
            tf = f"{name}_base.txt"
            n = self.table.shape[0]
            with open(os.path.join(directory, tf), "w") as f:
                f.write(f"{n}\n")
                for i in range(n):
                    for j in range(n):
                        f.write(" ".join(format_double(float(x)) for x in self.table[i, j].ravel()) + "\n")
            doc["base"] = {"type": "mueller_table", "table_file": tf}
        else:
            doc["base"] = {"type": "black"}
        doc["source"] = {"mu0": self.mu0, "phi0": self.phi0, "stokes": list(self.stokes)}
        if self.interface_n != 1.0:
            doc["interface"] = {"type": "fresnel", "n": self.interface_n}
        path = os.path.join(directory, f"{name}.json")
        with open(path, "w") as f:
            json.dump(doc, f, indent=2)
        return path

    def json_text(self, directory: str, name: str = "material") -> str:
        with open(self.write(directory, name)) as f:
            return f.read()


def single_layer(coeffs, omega, tau, base="black", albedo=0.0, mu0=0.6) -> MaterialDesc:
    return MaterialDesc([LayerDesc(omega, tau, np.asarray(coeffs, float))], base=base,
                        albedo=albedo, mu0=mu0)


# ---------------------------------------------------------------- SURVEY §8(d) configs
@dataclass
class Workload:
    name: str
    material: MaterialDesc
    N: int
    n_dphi: int
    note: str = ""
    mu_in: np.ndarray | None = field(default=None)   # None -> the N quadrature nodes


def config(name: str, band: int = 0) -> Workload:
    if name == "C1":
        m = single_layer(generator_G(0.5, 12), 0.95, 1.0, "lambertian", 0.1)
        return Workload("C1", m, 8, 19, "forward12, omega=0.95, tau=1, Lambertian 0.1")
    if name == "C2":
        m = single_layer(generator_G(0.7, 64), 0.9, 1000.0, "black")
        return Workload("C2", m, 32, 19, "G(0.7,64), omega=0.9, tau=1000 (semi-infinite stand-in)")
    if name == "C3":
        m = MaterialDesc([LayerDesc(0.95, 2.0, generator_G(0.6, 64)),
                          LayerDesc(0.6, 5.0, RAYLEIGH)], base="lambertian", albedo=0.2)
        return Workload("C3", m, 64, 19, "paint: G(0.6,64) over rayleigh, Lambertian 0.2")
    if name == "C4":
        m = single_layer(generator_G(0.9, 256), 0.99, 10.0, "black")
        return Workload("C4", m, 128, 72, "G(0.9,256), omega=0.99, tau=10")
    if name == "C3F":
        # C3 with the Fresnel top interface of the paint's binder (n = 1.5; BASELINE
        # config 3 "with a Fresnel interface" -- an extension, absent from the reference)
        w = config("C3")
        w.material.interface_n = 1.5
        return Workload("C3F", w.material, 64, 19, "paint C3 under a Fresnel interface, n = 1.5")
    if name == "C4p":
        # C4': the survey's C4 shape with the polarization ratios halved.  G(0.9, 256)
        # itself is rejected by the reference (F E has negative real eigenvalues at
        # m = 0, 1, 2: homogeneous.cpp:177-181); with pol = 0.5 every order m = 0..255
        # passes the reference's checks (the oracle accepts all 256, 8N residual <= 5e-10).
        m = single_layer(generator_G(0.9, 256, 0.5), 0.99, 10.0, "black")
        return Workload("C4p", m, 128, 72, "C4': G(0.9,256) with polarization x0.5, omega=0.99, tau=10")
    if name == "C5":
        b = band
        om = 0.80 + 0.19 * b / 30.0
        g = 0.75 - 0.25 * b / 30.0
        m = MaterialDesc([LayerDesc(om, 2.0, generator_G(g, 64)), LayerDesc(0.6, 5.0, RAYLEIGH)],
                         base="lambertian", albedo=0.2)
        return Workload(f"C5b{b}", m, 64, 19, f"band {b}: omega={om:.4f}, g={g:.4f}")
    raise KeyError(name)
