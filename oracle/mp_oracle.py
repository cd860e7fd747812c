"""High-precision (mpmath) restatement of the BRDF path -- TEST INFRASTRUCTURE.

Same algorithm as the reference (/root/reference/proj/src): GSF recurrences
(wigner.cpp:11-81), kernel blocks (kernel.cpp:29-65, 89-109), reduced
operators (homogeneous.cpp:43-73), eigen-modes with the lambda floor / nu
clamp rules (homogeneous.cpp:131-210), particular solution with the resonance
dither (particular.cpp:27-84), the global boundary system (boundary.cpp:142-265)
and the tau = 0 Fourier/Mueller synthesis (reconstruction.cpp:201-227,
brdf.cpp:100-117) -- evaluated at `dps` decimal digits so that its answer is
the exact discrete-ordinate solution to well below fp64 precision.  It exists
to measure the fp64 error floor of both the fp64 oracle and the GPU path
("use mpmath at N <= 8 to show the fp64 floor").

Linearity in the incident Stokes vector (pinned by test_brdf.cpp:63-85) is
used to solve the four unit Stokes channels instead of four basis vectors;
F_r = E_unit B (mu0 B)^+ is then exact algebra.  Slow (pure Python): N <= 8.
"""
from __future__ import annotations

import math

import mpmath as mp
import numpy as np


def _quadrature(n):
    """types.cpp:27-68 at working precision (Newton on P_n)."""
    nodes, weights = [mp.mpf(0)] * n, [mp.mpf(0)] * n
    half = (n + 1) // 2
    for k in range(half):
        x = mp.cos(mp.pi * (k + mp.mpf(3) / 4) / (n + mp.mpf(1) / 2))
        for _ in range(200):
            p0, p1 = mp.mpf(1), x
            for l in range(2, n + 1):
                p0, p1 = p1, ((2 * l - 1) * x * p1 - (l - 1) * p0) / l
            dp = n * (x * p1 - p0) / (x * x - 1)
            dx = p1 / dp
            x -= dx
            if abs(dx) < mp.mpf(10) ** (-mp.mp.dps + 3):
                break
        w = 2 / ((1 - x * x) * dp * dp)
        nodes[n - 1 - k], weights[n - 1 - k] = (1 + x) / 2, w / 2
        nodes[k], weights[k] = (1 - x) / 2, w / 2
    if n == 1:
        nodes, weights = [mp.mpf(1) / 2], [mp.mpf(1)]
    return nodes, weights


def _wigner(m, n, lmax, x):
    d = [mp.mpf(0)] * (lmax + 1)
    lmin = max(abs(m), abs(n))
    if lmin > lmax:
        return d
    a, b = abs(m - n), abs(m + n)
    v = mp.sqrt(mp.factorial(2 * lmin) / (mp.factorial(a) * mp.factorial(b))) / mp.mpf(2) ** lmin
    v *= mp.power(max(mp.mpf(0), 1 - x), mp.mpf(a) / 2) * mp.power(max(mp.mpf(0), 1 + x), mp.mpf(b) / 2)
    if n < m and (m - n) % 2:
        v = -v
    d[lmin] = v
    prev, cur = mp.mpf(0), v
    for l in range(lmin, lmax):
        if l == 0:
            nxt = x
        else:
            lp = l + 1
            c0 = l * mp.sqrt((lp * lp - m * m) * (lp * lp - n * n))
            c1 = (2 * l + 1) * (l * lp * x - m * n)
            c2 = lp * mp.sqrt((l * l - m * m) * (l * l - n * n))
            nxt = (c1 * cur - c2 * prev) / c0
        prev, cur = cur, nxt
        d[l + 1] = nxt
    return d


def _gsf(m, lmax, x):
    sgn = -1 if m % 2 else 1
    d0, d2p, d2m = _wigner(m, 0, lmax, x), _wigner(m, 2, lmax, x), _wigner(m, -2, lmax, x)
    return ([sgn * d0[l] for l in range(lmax + 1)],
            [sgn * (d2p[l] + d2m[l]) / 2 for l in range(lmax + 1)],
            [-sgn * (d2p[l] - d2m[l]) / 2 for l in range(lmax + 1)])


def _pi(g, l, flip):
    P, R, T = g[0][l], g[1][l], g[2][l]
    t = T if flip else -T
    M = mp.zeros(4, 4)
    M[0, 0] = P
    M[1, 1] = R
    M[2, 2] = R
    M[3, 3] = P
    M[1, 2] = t
    M[2, 1] = t
    return M


def _mat4(b):
    M = mp.zeros(4, 4)
    for r in range(4):
        for c in range(4):
            M[r, c] = mp.mpf(float(b[r, c]))
    return M


D4 = [1, 1, -1, -1]


class _Order:
    """Kernel, reduced operators and modes of one (medium, order)."""

    def __init__(self, m, omega, coeffs, nodes, weights):
        n, L = len(nodes), len(coeffs)
        d = 4 * n
        self.m, self.n, self.d = m, n, d
        self.omega = mp.mpf(float(omega))
        B = [_mat4(c) for c in coeffs]
        self.B = B
        self.nodes, self.weights = nodes, weights
        tab = [_gsf(m, L - 1, x) for x in nodes] if m < L else None
        self.app = [[mp.zeros(4, 4) for _ in range(n)] for _ in range(n)]
        self.apm = [[mp.zeros(4, 4) for _ in range(n)] for _ in range(n)]
        if m < L:
            for i in range(n):
                for j in range(n):
                    for l in range(m, L):
                        left = _pi(tab[i], l, False) * B[l]
                        s = -1 if (l - m) % 2 else 1
                        self.app[i][j] += left * _pi(tab[j], l, False)
                        self.apm[i][j] += s * (left * _pi(tab[j], l, True))
        ho = self.omega / 2
        K1, K2 = mp.zeros(d, d), mp.zeros(d, d)
        for i in range(n):
            for j in range(n):
                sc = ho * weights[j]
                for r in range(4):
                    for c in range(4):
                        K1[4 * i + r, 4 * j + c] = sc * self.app[i][j][r, c]
                        K2[4 * i + r, 4 * j + c] = sc * self.apm[i][j][r, c] * D4[c]
        self.E, self.F = mp.zeros(d, d), mp.zeros(d, d)
        for i in range(d):
            for j in range(d):
                idm = 1 if i == j else 0
                self.E[i, j] = (idm - K1[i, j] - K2[i, j]) / nodes[j // 4]
                self.F[i, j] = (idm - K1[i, j] + K2[i, j]) / nodes[j // 4]
        self.FE = self.F * self.E
        self._modes()

    def _modes(self):
        d = self.d
        lam, V = mp.eig(self.FE)
        femax = max(abs(self.FE[i, j]) for i in range(d) for j in range(d))
        floor = mp.mpf("1e-12") * max(1, femax)
        self.nu, self.pp, self.pm = [], [], []
        for j in range(d):
            l = lam[j]
            x = [V[i, j] for i in range(d)]
            xm = max(abs(v) for v in x)
            x = [v / xm for v in x]
            cons = abs(l) < floor
            if cons:
                nu = mp.mpf("4e9")
                pp = [x[i] / self.nodes[i // 4] / 2 for i in range(d)]
                pm = list(pp)
            else:
                if mp.re(l) < 0 and abs(mp.im(l)) < 1e-10 * abs(mp.re(l)) and abs(l) < 1e-10:
                    l = abs(l)
                nu = 1 / mp.sqrt(l)
                if mp.re(nu) < 0:
                    nu = -nu
                if abs(nu) > 4e9:
                    nu = 4e9 * nu / abs(nu)
                ex = self.E * mp.matrix(x)
                pp = [(x[i] - nu * ex[i]) / self.nodes[i // 4] / 2 for i in range(d)]
                pm = [(x[i] + nu * ex[i]) / self.nodes[i // 4] / 2 for i in range(d)]
            self.nu.append(nu)
            self.pp.append(pp)
            self.pm.append(pm)

    def particular(self, mu0_in, c, L):
        """Z+, Z- for the unit Stokes channel c (k = 1 for c < 2), particular.cpp:7-107."""
        n, d = self.n, self.d
        mu0 = mp.mpf(float(mu0_in))
        if self.omega == 0 or self.m >= L:
            return [mp.mpf(0)] * d, [mp.mpf(0)] * d
        gb = _gsf(self.m, L - 1, -mu0)
        tab = [_gsf(self.m, L - 1, x) for x in self.nodes]
        xp, xm = [mp.mpf(0)] * d, [mp.mpf(0)] * d
        sc = self.omega / (2 * mp.pi)
        for i in range(n):
            up, dn = mp.zeros(4, 4), mp.zeros(4, 4)
            for l in range(self.m, L):
                right = self.B[l] * _pi(gb, l, False)
                s = -1 if (l - self.m) % 2 else 1
                up += _pi(tab[i], l, False) * right
                dn += s * (_pi(tab[i], l, True) * right)
            for r in range(4):
                xp[4 * i + r] = sc * up[r, c]
                xm[4 * i + r] = sc * dn[r, c]
        if max(abs(v) for v in xp + xm) == 0:
            return [mp.mpf(0)] * d, [mp.mpf(0)] * d
        mu = mu0
        for nu in self.nu:
            lam = 1 / (nu * nu)
            if abs(lam - 1 / (mu * mu)) < 1e-8 * abs(lam):
                mu = mu * (1 - mp.mpf("1e-7"))
                break
        sp = [xp[i] + D4[i % 4] * xm[i] for i in range(d)]
        sm = [xp[i] - D4[i % 4] * xm[i] for i in range(d)]
        lhs = self.FE - mp.eye(d) / (mu * mu)
        rhs = self.F * mp.matrix(sp) - mp.matrix(sm) / mu
        g = mp.lu_solve(lhs, rhs)
        eg = self.E * g
        zp, zm = [], []
        for i in range(d):
            h = mu * (sp[i] - eg[i])
            zp.append((g[i] + h) / self.nodes[i // 4] / 2)
            zm.append(D4[i % 4] * (g[i] - h) / self.nodes[i // 4] / 2)
        return zp, zm


def brdf(omegas, taus, coeffs, base_type, rho, N, mu_in, n_dphi, basis=None, dps=32):
    """Exact (high-precision) F_r table [n_in, N, n_dphi, 4, 4] as float64.

    omegas/taus: per layer; coeffs: [P, L, 4, 4]; base_type 0 black / 1 lambertian.
    """
    if base_type not in (0, 1):
        raise NotImplementedError("mp oracle: black or lambertian base only")
    with mp.workdps(dps):
        P, L = len(omegas), coeffs.shape[1]
        nodes, weights = _quadrature(N)
        d = 4 * N
        # medium dedup (pipeline.cpp:37-54)
        sig, reps = [], []
        for p in range(P):
            s = next((sig[q] for q in range(p) if omegas[q] == omegas[p]
                      and np.array_equal(coeffs[q], coeffs[p])), -1)
            if s < 0:
                s = len(reps)
                reps.append(p)
            sig.append(s)
        states = [[_Order(m, omegas[r], coeffs[r], nodes, weights) for m in range(L)] for r in reps]
        tau = [mp.mpf(float(t)) for t in taus]
        tau_top = [mp.mpf(0)]
        for p in range(1, P):
            tau_top.append(tau_top[-1] + tau[p - 1])
        tau_tot = tau_top[-1] + tau[-1]
        G = 2 * d * P
        basis = np.array([[1, 0, 0, 0], [1, 1, 0, 0], [1, 0, 1, 0], [1, 0, 0, 1]], float) \
            if basis is None else np.asarray(basis, float).reshape(4, 4)
        n_in = len(mu_in)
        up = {}
        for m in range(L):
            ms = [states[sig[p]][m] for p in range(P)]
            att = [[mp.exp(-tau[p] / ms[p].nu[j]) for j in range(d)] for p in range(P)]
            A = mp.matrix(G, G)
            for j in range(d):
                col_a, col_b = lambda p: 2 * d * p + j, lambda p: 2 * d * p + d + j
                m0 = ms[0]
                for i in range(d):
                    A[i, col_a(0)] = D4[i % 4] * m0.pm[j][i]
                    A[i, col_b(0)] = att[0][j] * D4[i % 4] * m0.pp[j][i]
                for p in range(P - 1):
                    ru, rd = d + 2 * d * p, 2 * d + 2 * d * p
                    mp_, mq = ms[p], ms[p + 1]
                    for i in range(d):
                        A[ru + i, col_a(p)] = att[p][j] * mp_.pp[j][i]
                        A[ru + i, col_b(p)] = mp_.pm[j][i]
                        A[rd + i, col_a(p)] = att[p][j] * D4[i % 4] * mp_.pm[j][i]
                        A[rd + i, col_b(p)] = D4[i % 4] * mp_.pp[j][i]
                        A[ru + i, col_a(p + 1)] = -mq.pp[j][i]
                        A[ru + i, col_b(p + 1)] = -att[p + 1][j] * mq.pm[j][i]
                        A[rd + i, col_a(p + 1)] = -D4[i % 4] * mq.pm[j][i]
                        A[rd + i, col_b(p + 1)] = -att[p + 1][j] * D4[i % 4] * mq.pp[j][i]
                rb, mqq = d + 2 * d * (P - 1), ms[P - 1]
                for i in range(d):
                    A[rb + i, col_a(P - 1)] = att[P - 1][j] * mqq.pp[j][i]
                    A[rb + i, col_b(P - 1)] = mqq.pm[j][i]
                if m == 0 and base_type == 1 and rho != 0:
                    fa = sum(weights[k] * nodes[k] * att[P - 1][j] * D4[0] * mqq.pm[j][4 * k]
                             for k in range(N))
                    fb = sum(weights[k] * nodes[k] * D4[0] * mqq.pp[j][4 * k] for k in range(N))
                    for i in range(N):
                        A[rb + 4 * i, col_a(P - 1)] -= 2 * mp.mpf(rho) * fa
                        A[rb + 4 * i, col_b(P - 1)] -= 2 * mp.mpf(rho) * fb
            Ainv = mp.inverse(A)
            for ii, mu0f in enumerate(mu_in):
                mu0 = mp.mpf(float(mu0f))
                for c in range(4):
                    parts = [st.particular(mu0f, c, L) for st in [states[s][m] for s in range(len(reps))]]
                    zp = [parts[sig[p]][0] for p in range(P)]
                    zm = [parts[sig[p]][1] for p in range(P)]
                    rhs = mp.matrix(G, 1)
                    for i in range(d):
                        rhs[i] = -zm[0][i]
                    for p in range(P - 1):
                        bn = mp.exp(-tau_top[p + 1] / mu0)
                        ru = d + 2 * d * p
                        for i in range(d):
                            rhs[ru + i] = bn * (zp[p + 1][i] - zp[p][i])
                            rhs[ru + d + i] = bn * (zm[p + 1][i] - zm[p][i])
                    bb = mp.exp(-tau_tot / mu0)
                    rb = d + 2 * d * (P - 1)
                    for i in range(d):
                        rhs[rb + i] = -(bb * zp[P - 1][i])
                    if m == 0 and base_type == 1 and rho != 0:
                        flux = sum(weights[k] * nodes[k] * bb * zm[P - 1][4 * k] for k in range(N))
                        beam = (mu0 / mp.pi) * 2 * mp.mpf(rho) * bb if c == 0 else 0
                        for i in range(N):
                            rhs[rb + 4 * i] += 2 * mp.mpf(rho) * flux + beam
                    coef = Ainv * rhs
                    m0 = ms[0]
                    u = [zp[0][i] for i in range(d)]
                    for j in range(d):
                        a, b = coef[j], coef[d + j]
                        for i in range(d):
                            u[i] += a * m0.pp[j][i] + b * att[0][j] * m0.pm[j][i]
                    up[(m, ii, c)] = u
        # synthesis + Mueller recovery
        out = np.zeros((n_in, N, n_dphi, 4, 4))
        for ii, mu0f in enumerate(mu_in):
            mu0 = mp.mpf(float(mu0f))
            Bm = mp.matrix([[mp.mpf(float(basis[b][c])) for b in range(4)] for c in range(4)])
            I = mu0 * Bm
            pinv = I.T * mp.inverse(I * I.T)
            post = Bm * pinv
            for io in range(N):
                for ip in range(n_dphi):
                    x = -2 * mp.pi * ip / n_dphi
                    Eu = mp.zeros(4, 4)
                    for m in range(L):
                        sc = 1 if m == 0 else 2
                        cs, sn = mp.cos(m * x), mp.sin(m * x)
                        p1 = [sc * cs, sc * cs, sc * sn, sc * sn]
                        p2 = [-sc * sn, -sc * sn, sc * cs, sc * cs]
                        for c in range(4):
                            v = up[(m, ii, c)]
                            for r in range(4):
                                Eu[r, c] += (p1[r] if c < 2 else p2[r]) * mp.re(v[4 * io + r]) / 2
                    F = Eu * post
                    for r in range(4):
                        for c in range(4):
                            out[ii, io, ip, r, c] = float(F[r, c])
        return out
