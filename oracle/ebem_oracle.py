"""CPU restatement of the reference's FDS hot path -- TEST INFRASTRUCTURE ONLY.

A from-scratch numpy/scipy restatement of the algorithm the reference C++
library implements (the checker for the CUDA path; never imported by the
product).  Only tests/, bench.py's CPU legs and __graft_entry__.smoke() may
use it.  Independent of both the reference code and the CUDA code:

* H0/H1 come from scipy.special.hankel1 (AMOS) instead of Chebyshev tables;
* Gauss-Legendre rules from numpy.polynomial.legendre.leggauss;
* everything is vectorised over element pairs x quadrature points;
* the column-pivoted QR is a numpy restatement of LAPACK zlaqp2;
* LU solves use scipy.linalg (LAPACK zgetrf/zgetrs, as the reference).

Each function cites the reference file:line it follows.  Pinned by
tests/test_oracle.py against the reference's golden vectors
(tests/golden/reference_values.json) and against the reference library
compiled in place (oracle/_ref).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.special as sps

PI = math.pi
EULER = 0.57721566490153286060651209008240
SERIES_TERMS = 16      # proj/src/kernel_scalars.cpp:19
PIVOT_FLOOR = 1e-14    # proj/src/compression.cpp:15


# ------------------------------------------------------------------ medium
@dataclass
class Medium:
    """proj/include/ebem/medium.hpp:14-60 (from_lame keeps lambda, mu exact)."""
    lam: float
    mu: float
    rho: float
    omega: float

    @property
    def cL(self):
        return math.sqrt((self.lam + 2 * self.mu) / self.rho)

    @property
    def cT(self):
        return math.sqrt(self.mu / self.rho)

    @property
    def kL(self):
        return self.omega / self.cL

    @property
    def kT(self):
        return self.omega / self.cT

    def default_coupling(self):
        return 1j / self.kT


def gauss01(n):
    """Gauss-Legendre rule on [0, 1] (proj/src/quadrature.cpp:16-56)."""
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


def hankel01(x):
    """H0^(1), H1^(1) at real x > 0 (proj/src/hankel.cpp:34-71)."""
    x = np.asarray(x, dtype=np.float64)
    return sps.hankel1(0, x), sps.hankel1(1, x)


# ---------------------------------------------------- remainder series
class _Series:
    """sum_q (a_q + b_q ln r) r^q as dense arrays over q in [lo, lo+len)
    (LogSeries, proj/src/kernel_scalars.cpp:28-121)."""

    def __init__(self, lo=0, a=None, b=None):
        self.lo = lo
        self.a = np.zeros(0, complex) if a is None else np.asarray(a, complex)
        self.b = np.zeros(0, complex) if b is None else np.asarray(b, complex)

    def _span(self, lo, hi):
        out_a = np.zeros(hi - lo, complex)
        out_b = np.zeros(hi - lo, complex)
        i = self.lo - lo
        out_a[i:i + len(self.a)] = self.a
        out_b[i:i + len(self.b)] = self.b
        return out_a, out_b

    def plus(self, o, f=1.0):
        lo = min(self.lo, o.lo)
        hi = max(self.lo + len(self.a), o.lo + len(o.a))
        a1, b1 = self._span(lo, hi)
        a2, b2 = o._span(lo, hi)
        return _Series(lo, a1 + f * a2, b1 + f * b2)

    def times(self, f):
        return _Series(self.lo, f * self.a, f * self.b)

    def over_r(self, p=1):
        return _Series(self.lo - p, self.a.copy(), self.b.copy())

    def d(self):
        q = self.lo + np.arange(len(self.a))
        return _Series(self.lo - 1, q * self.a + self.b, q * self.b)

    def prune(self, rel=1e-25):
        mag = lambda z: np.abs(z.real) + np.abs(z.imag)  # noqa: E731
        peak = max(mag(self.a).max(initial=0.0), mag(self.b).max(initial=0.0))
        cut = rel * peak
        self.a = np.where(mag(self.a) > cut, self.a, 0)
        self.b = np.where(mag(self.b) > cut, self.b, 0)
        return self

    def drop_log(self, q):
        i = q - self.lo
        if 0 <= i < len(self.b):
            self.b[i] = 0
        return self

    def trimmed(self):
        nz = np.nonzero((self.a != 0) | (self.b != 0))[0]
        if len(nz) == 0:
            return _Series(0, np.zeros(1, complex), np.zeros(1, complex))
        return _Series(self.lo + nz[0], self.a[nz[0]:nz[-1] + 1], self.b[nz[0]:nz[-1] + 1])

    def eval(self, r):
        r = np.asarray(r, dtype=np.float64)
        lr = np.log(r)
        out = np.zeros(r.shape, complex)
        for i, (a, b) in enumerate(zip(self.a, self.b)):
            if a != 0 or b != 0:
                out += (a + b * lr) * r ** (self.lo + i)
        return out

    def integrate(self, c, j):
        """int_0^1 u^j [series](c u) du (closed form, :108-121)."""
        lc = math.log(c)
        s = 0j
        for i, (a, b) in enumerate(zip(self.a, self.b)):
            q = self.lo + i
            inv = 1.0 / (q + j + 1)
            s += c ** q * ((a + b * lc) * inv - b * inv * inv)
        return s


def _chi_series(k):
    """chi_a + ln(r)/(2 pi), chi_a = (i/4) H0(k r) (kernel_scalars.cpp:133-151)."""
    c0 = 0.25j - (math.log(0.5 * k) + EULER) / (2 * PI)
    a = np.zeros(2 * SERIES_TERMS + 1, complex)
    b = np.zeros(2 * SERIES_TERMS + 1, complex)
    ap, harm = 1.0, 0.0
    for p in range(SERIES_TERMS + 1):
        if p > 0:
            ap *= -0.25 * k * k / (p * p)
            harm += 1.0 / p
        a[2 * p] = ap * (c0 + harm / (2 * PI))
        b[2 * p] = 0 if p == 0 else -ap / (2 * PI)
    return _Series(0, a, b)


class Scalars:
    """The ten radial scalars (KernelScalars, proj/src/kernel_scalars.cpp:123-379).
    Order: gpsi, gchi, d1, d2, d3, n1, n2, n4, n5, n7."""

    def __init__(self, med: Medium):
        self.med = med
        kL, kT, lam, mu = med.kL, med.kT, med.lam, med.mu
        self.kL, self.kT, self.lam, self.mu = kL, kT, lam, mu
        self.ar = lam / (lam + 2 * mu)
        self.cc = (lam + mu) / (8 * PI * (lam + 2 * mu))
        self.qfac = 8 * mu * self.cc
        self.radius = 0.25 / kT   # the reference's pointwise switch (:131)
        # The restatement switches to the series later (k_T r < 1, where the
        # series still converges to ~1e-20): scipy's H0/H1 lose more digits in
        # the static/full cancellation than the reference's own evaluator.
        self.switch = 1.0 / kT
        self.kappa = mu / (2 * PI * (lam + 2 * mu))
        cT, cL = _chi_series(kT), _chi_series(kL)
        psi = cT.plus(cL, -1.0).times(1.0 / (kT * kT))
        psi = psi.plus(_Series(2, [0], [-self.cc]))
        psi.drop_log(2)
        psi.prune()
        p1 = psi.d()
        p2 = p1.d()
        p3 = p2.d()
        p4 = p3.d()
        t1 = cT.d()
        t2 = t1.d()
        l1 = cL.d()
        l2 = l1.d()
        gpsi = cT.plus(p1.over_r())
        gchi = p2.plus(p1.over_r(), -1.0).prune()
        w = gchi.over_r()
        gam = gchi.over_r(2)
        bet = p3.plus(w, -3.0).over_r().prune()
        alf = p4.plus(p3.over_r(), -6.0).plus(gam, 15.0).prune()
        d1 = l1.times(self.ar).plus(w, 2.0)
        d2 = t1.plus(w, 2.0)
        d3 = p3.plus(w, -3.0).times(2.0)
        n1 = t1.over_r().times(-2 * mu).plus(gam, -4 * mu)
        n2 = t2.plus(t1.over_r(), -1.0).times(-mu).plus(bet, -4 * mu)
        n4 = alf.times(-4 * mu)
        n5 = (cL.times(lam * self.ar * kL * kL).plus(l1.over_r(), -4 * mu * self.ar)
              .plus(gam, -4 * mu))
        n5 = n5.plus(_Series(0, [0], [-lam * self.ar * kL * kL / (2 * PI)]))
        n7 = l2.plus(l1.over_r(), -1.0).times(-2 * mu * self.ar).plus(bet, -4 * mu)
        self.series = [s.prune().trimmed() for s in
                       (gpsi, gchi, d1, d2, d3, n1, n2, n4, n5, n7)]
        for s in self.series:
            assert s.lo >= 0, "remainder series kept a negative power"
        # dense (10, L) tables over powers 0..L-1 for vectorised evaluation
        L = max(s.lo + len(s.a) for s in self.series)
        self._A = np.zeros((10, L), complex)
        self._B = np.zeros((10, L), complex)
        for k, s in enumerate(self.series):
            self._A[k, s.lo:s.lo + len(s.a)] = s.a
            self._B[k, s.lo:s.lo + len(s.b)] = s.b
        self._q = np.arange(L)

    # -- static part (:283-299)
    def static(self, r):
        r = np.asarray(r, dtype=np.float64)
        lr = np.log(r)
        lam, mu, cc = self.lam, self.mu, self.cc
        l2m = lam + 2 * mu
        r2 = r * r
        d1 = mu / (2 * PI * l2m * r)
        return np.stack([-lr / (2 * PI) + cc * (2 * lr + 1), np.full_like(r, 2 * cc), d1, -d1,
                         -8 * cc / r, mu * mu / (PI * l2m * r2), mu * lam / (PI * l2m * r2),
                         -8 * self.qfac / r2, mu * (lam - mu) / (PI * l2m * r2),
                         2 * mu * mu / (PI * l2m * r2)], axis=-1).astype(complex)

    def _series(self, r):
        r = np.asarray(r, dtype=np.float64)
        lr = np.log(r)[..., None]
        rp = r[..., None] ** self._q                       # (..., L)
        return (rp @ self._A.T) + (lr * rp) @ self._B.T

    def _hankel_branch(self, r):
        kT, kL, mu, lam, ar = self.kT, self.kL, self.mu, self.lam, self.ar
        zT, zL = kT * r, kL * r
        h0T, h1T = hankel01(zT)
        h0L, h1L = hankel01(zL)
        i4 = 0.25j
        chiT, chiL = i4 * h0T, i4 * h0L
        chiT1, chiL1 = -i4 * kT * h1T, -i4 * kL * h1L
        chiT2 = -i4 * kT ** 2 * (h0T - h1T / zT)
        chiL2 = -i4 * kL ** 2 * (h0L - h1L / zL)
        chiT3 = -i4 * kT ** 3 * (-h1T - h0T / zT + 2 * h1T / zT ** 2)
        chiL3 = -i4 * kL ** 3 * (-h1L - h0L / zL + 2 * h1L / zL ** 2)
        chiT4 = -i4 * kT ** 4 * (-h0T + 2 * h1T / zT + 3 * h0T / zT ** 2 - 6 * h1T / zT ** 3)
        chiL4 = -i4 * kL ** 4 * (-h0L + 2 * h1L / zL + 3 * h0L / zL ** 2 - 6 * h1L / zL ** 3)
        ik = 1.0 / (kT * kT)
        p1, p2 = (chiT1 - chiL1) * ik, (chiT2 - chiL2) * ik
        p3, p4 = (chiT3 - chiL3) * ik, (chiT4 - chiL4) * ik
        gpsi = chiT + p1 / r
        gchi = p2 - p1 / r
        w = gchi / r
        gam = gchi / r ** 2
        bet = (p3 - 3 * w) / r
        alf = p4 - 6 * p3 / r + 15 * gam
        return np.stack([gpsi, gchi, ar * chiL1 + 2 * w, chiT1 + 2 * w, 2 * (p3 - 3 * w),
                         -2 * mu * chiT1 / r - 4 * mu * gam,
                         -mu * (chiT2 - chiT1 / r) - 4 * mu * bet, -4 * mu * alf,
                         lam * ar * kL * kL * chiL - 4 * mu * ar * chiL1 / r - 4 * mu * gam,
                         -2 * mu * ar * (chiL2 - chiL1 / r) - 4 * mu * bet], axis=-1)

    def split(self, r):
        """(full, remainder), proj/src/kernel_scalars.cpp:214-331."""
        r = np.asarray(r, dtype=np.float64)
        full = np.empty(r.shape + (10,), complex)
        rem = np.empty(r.shape + (10,), complex)
        s0 = self.static(r)
        small = r < self.switch
        if small.any():
            rs = self._series(r[small])
            rem[small] = rs
            full[small] = rs + s0[small]
        big = ~small
        if big.any():
            fb = self._hankel_branch(r[big])
            full[big] = fb
            rem[big] = fb - s0[big]
        return full, rem

    def full(self, r):
        return self.split(r)[0]

    def remainder(self, r):
        return self.split(r)[1]

    def integrated_remainder(self, scale, upow):
        if not self.kT * scale < 2.5:
            raise ValueError("KernelScalars: element too long for this frequency")
        lc = math.log(scale)
        inv = 1.0 / (self._q + upow + 1.0)
        cp = scale ** self._q
        return ((self._A + self._B * lc) * (cp * inv) - self._B * (cp * inv * inv)).sum(1)


# ----------------------------------------------------------- combiners
def combine_D(s, zh, ny):
    """proj/src/kernels.cpp:22-37; s (...,10), zh/ny (...,2) -> (...,2,2)."""
    nz = np.sum(ny * zh, -1)
    d1, d2, d3 = s[..., 2], s[..., 3], s[..., 4]
    out = np.empty(s.shape[:-1] + (2, 2), complex)
    for i in range(2):
        for j in range(2):
            dij = 1.0 if i == j else 0.0
            out[..., i, j] = -(d1 * (ny[..., j] * zh[..., i]) +
                               d2 * (nz * dij + ny[..., i] * zh[..., j]) +
                               d3 * (nz * zh[..., i] * zh[..., j]))
    return out


def combine_N(s, zh, m, n):
    """proj/src/kernels.cpp:39-68 (m observation normal, n source normal)."""
    mn = np.sum(m * n, -1)
    mz = np.sum(m * zh, -1)
    nz = np.sum(n * zh, -1)
    out = np.empty(s.shape[:-1] + (2, 2), complex)
    for i in range(2):
        for j in range(2):
            dij = 1.0 if i == j else 0.0
            zi, zj = zh[..., i], zh[..., j]
            out[..., i, j] = (s[..., 5] * (mn * dij + n[..., i] * m[..., j]) +
                              s[..., 6] * (mn * zi * zj + mz * nz * dij + mz * n[..., i] * zj
                                           + nz * zi * m[..., j]) +
                              s[..., 7] * (mz * nz * zi * zj) + s[..., 8] * (m[..., i] * n[..., j]) +
                              s[..., 9] * (mz * zi * n[..., j] + nz * m[..., i] * zj))
    return out


def q0_kernel(qfac, r, zh):
    """proj/src/kernels.cpp:70-78."""
    lr = qfac * np.log(r)
    out = np.empty(r.shape + (2, 2))
    out[..., 0, 0] = lr - qfac * zh[..., 0] ** 2
    out[..., 0, 1] = out[..., 1, 0] = -qfac * zh[..., 0] * zh[..., 1]
    out[..., 1, 1] = lr - qfac * zh[..., 1] ** 2
    return out


# --------------------------------------------------------------- geometry
class Curve:
    """Closed polyline: element e from node e to (e+1) mod N, normal = +90 deg
    rotation of the tangent (proj/src/geometry.cpp:15-37)."""

    def __init__(self, xy):
        self.xy = np.asarray(xy, dtype=np.float64).reshape(-1, 2)
        self.n = len(self.xy)
        self.d = np.roll(self.xy, -1, axis=0) - self.xy
        self.h = np.hypot(self.d[:, 0], self.d[:, 1])
        self.t = self.d / self.h[:, None]
        self.nrm = np.stack([-self.t[:, 1], self.t[:, 0]], axis=1)


def _seg_dist(p, a, b):
    ab = b - a
    l2 = np.sum(ab * ab, -1)
    t = np.where(l2 > 0, np.sum((p - a) * ab, -1) / np.where(l2 > 0, l2, 1), 0.0)
    t = np.clip(t, 0.0, 1.0)
    q = p - (a + t[..., None] * ab)
    return np.hypot(q[..., 0], q[..., 1])


def element_distance(c: Curve, ea, eb):
    """proj/src/geometry.cpp:83-96 (vectorised)."""
    a0, a1 = c.xy[ea], c.xy[ea] + c.d[ea]
    b0, b1 = c.xy[eb], c.xy[eb] + c.d[eb]
    d = np.minimum(_seg_dist(a0, b0, b1), _seg_dist(a1, b0, b1))
    d = np.minimum(d, _seg_dist(b0, a0, a1))
    return np.minimum(d, _seg_dist(b1, a0, a1))


# ---------------------------------------------------------- pair integrals
SHAPE_SLOPE = np.array([-1.0, 1.0])


class Integrator:
    """Galerkin pair integrals (PairIntegrator, proj/src/assembly.cpp:27-286),
    returned as V[la, lb, i, j] = D + alpha N (+ M/2 on coincident diagonals)."""

    def __init__(self, curve: Curve, med: Medium, alpha, corner=10, far=4, refine=1.0):
        self.c, self.med, self.alpha = curve, med, complex(alpha)
        self.S = Scalars(med)
        self.corner, self.far, self.refine = corner, far, refine
        self.kappa = self.S.kappa
        self.ccon = self.S.cc

    def scaled(self, n):
        return int(n * self.refine + 0.5)

    def tier(self, q):
        """tier_nodes, proj/src/assembly.cpp:27-38 (vectorised)."""
        add = np.where(q >= 8.0, 0, np.where(q >= 4.0, 2, np.where(q >= 2.0, 5, 9)))
        return ((self.far + add) * self.refine + 0.5).astype(int)

    def separated(self, ea, eb):
        """proj/src/assembly.cpp:248-286, vectorised over pairs of one tier."""
        c, S, al = self.c, self.S, self.alpha
        out = np.zeros((len(ea), 2, 2, 2, 2), complex)
        if len(ea) == 0:
            return out
        dist = element_distance(c, ea, eb)
        n_of = self.tier(dist / np.maximum(c.h[ea], c.h[eb]))
        for n in np.unique(n_of):
            sel = np.nonzero(n_of == n)[0]
            a, b = ea[sel], eb[sel]
            s, w = gauss01(int(n))
            x = c.xy[a][:, None, :] + s[None, :, None] * c.d[a][:, None, :]   # (P, n, 2)
            y = c.xy[b][:, None, :] + s[None, :, None] * c.d[b][:, None, :]
            z = x[:, :, None, :] - y[:, None, :, :]                           # (P, n, n, 2)
            r = np.hypot(z[..., 0], z[..., 1])
            zh = z / r[..., None]
            fs, rs = S.split(r)
            nx = np.broadcast_to(c.nrm[a][:, None, None, :], zh.shape)
            ny = np.broadcast_to(c.nrm[b][:, None, None, :], zh.shape)
            dm = combine_D(fs, zh, ny)
            nm = combine_N(rs, zh, nx, ny)
            qm = q0_kernel(S.qfac, r, zh)
            ww = w[:, None] * w[None, :]
            wgt = ww[None] * (c.h[a] * c.h[b])[:, None, None]
            P = np.stack([1 - s, s])  # (2, n)
            km = dm + al * nm
            acc = np.einsum("pij,ai,bj,pijkl->pabkl", wgt, P, P, km)
            slope = np.outer(SHAPE_SLOPE, SHAPE_SLOPE)
            acc += al * np.einsum("ij,ab,pijkl->pabkl", ww, slope, qm)
            out[sel] = acc
        return out

    def coincident(self, e):
        """proj/src/assembly.cpp:70-146."""
        c, S = self.c, self.S
        h, tau, nrm = c.h[e], c.t[e], c.nrm[e]
        D = np.zeros((2, 2, 2, 2), complex)
        N = np.zeros((2, 2, 2, 2), complex)
        M = np.array([[h / 3, h / 6], [h / 6, h / 3]])
        dc = 0.5 * self.kappa * h
        D[0, 1, 0, 1] += dc
        D[0, 1, 1, 0] -= dc
        D[1, 0, 0, 1] -= dc
        D[1, 0, 1, 0] += dc
        f0, f1, f2, f3 = (S.integrated_remainder(h, j) for j in range(4))
        i1, i2 = f2[2] - f1[2], f2[3] - f1[3]
        val = -h * h * (i1 * np.outer(tau, nrm) + i2 * np.outer(nrm, tau))
        D[0, 1] += val
        D[1, 0] -= val
        for a in range(2):
            for b in range(2):
                sg = SHAPE_SLOPE[a] * SHAPE_SLOPE[b]
                N[a, b] += sg * S.qfac * ((math.log(h) - 1.5) * np.eye(2) - np.outer(tau, tau))
        sdiag = f3 / 3 - f1 + 2 * f0 / 3
        soff = (f0 - f3) / 3
        nd = combine_N(sdiag, tau, nrm, nrm)
        no = combine_N(soff, tau, nrm, nrm)
        N[0, 0] += h * h * nd
        N[1, 1] += h * h * nd
        N[0, 1] += h * h * no
        N[1, 0] += h * h * no
        V = D + self.alpha * N
        for a in range(2):
            for b in range(2):
                V[a, b] += 0.5 * M[a, b] * np.eye(2)
        return V

    def adjacent(self, ea, eb):
        """proj/src/assembly.cpp:148-246 (Duffy, two triangles)."""
        c, S = self.c, self.S
        end_start = (ea + 1) % c.n == eb
        hx, hy = c.h[ea], c.h[eb]
        if end_start:
            tx, bx0, bx1 = -c.t[ea], [0.0, 1.0], [1.0, -1.0]
            ty, by0, by1 = c.t[eb], [1.0, 0.0], [-1.0, 1.0]
        else:
            tx, bx0, bx1 = c.t[ea], [1.0, 0.0], [-1.0, 1.0]
            ty, by0, by1 = -c.t[eb], [0.0, 1.0], [1.0, -1.0]
        nx, ny = c.nrm[ea], c.nrm[eb]
        dhat = np.zeros(10, complex)
        dhat[2], dhat[3], dhat[4] = self.kappa, -self.kappa, -8 * self.ccon
        D = np.zeros((2, 2, 2, 2), complex)
        N = np.zeros((2, 2, 2, 2), complex)
        gx, gw = gauss01(self.scaled(self.corner))
        for tri in range(2):
            for w, wt in zip(gx, gw):
                zv = hx * tx - (w * hy) * ty if tri == 0 else (w * hx) * tx - hy * ty
                g = math.hypot(zv[0], zv[1])
                zh = zv / g
                dm = [combine_D(S.integrated_remainder(g, j + 1), zh, ny) for j in range(3)]
                nm = [combine_N(S.integrated_remainder(g, j + 1), zh, nx, ny) for j in range(3)]
                ds = combine_D(dhat, zh, ny)
                for a in range(2):
                    for b in range(2):
                        t0, u0 = bx0[a], by0[b]
                        t1 = bx1[a] if tri == 0 else bx1[a] * w
                        u1 = by1[b] * w if tri == 0 else by1[b]
                        cf = [t0 * u0, t0 * u1 + t1 * u0, t1 * u1]
                        cint = cf[0] + cf[1] / 2 + cf[2] / 3
                        D[a, b] += ds * (wt * hx * hy * cint / g)
                        for j in range(3):
                            D[a, b] += dm[j] * (wt * hx * hy * cf[j])
                            N[a, b] += nm[j] * (wt * hx * hy * cf[j])
                        sg = SHAPE_SLOPE[a] * SHAPE_SLOPE[b]
                        ql = S.qfac * (math.log(g) * 0.5 - 0.25)
                        qz = S.qfac * 0.5
                        N[a, b] += wt * sg * (ql * np.eye(2) - qz * np.outer(zh, zh))
        return D + self.alpha * N

    def bundles(self, ea, eb):
        """Bundle of every (ea[p], eb[p]) pair (PairIntegrator::bundle, :53-68)."""
        n = self.c.n
        out = np.zeros((len(ea), 2, 2, 2, 2), complex)
        coin = ea == eb
        adj = ((ea + 1) % n == eb) | ((eb + 1) % n == ea)
        sep = ~(coin | adj)
        out[sep] = self.separated(ea[sep], eb[sep])
        for p in np.nonzero(coin)[0]:
            out[p] = self.coincident(ea[p])
        for p in np.nonzero(adj & ~coin)[0]:
            out[p] = self.adjacent(ea[p], eb[p])
        return out


def _support(nodes, n):
    """Elements carrying the hat functions of the listed nodes (node g owns
    elements g-1 and g), ascending (proj/src/assembly.cpp:342-368)."""
    s = set()
    for g in nodes:
        s.add(int(g))
        s.add(int(g - 1) % n)
    return np.array(sorted(s), dtype=np.int64)


def _scatter(rows, cols, nr_curve, nc_curve, res, ces, B):
    """Ordered scatter of bundles B[ra, cb] into the (rows x cols) block
    (proj/src/assembly.cpp:383-407, :493-506)."""
    nr = len(rows[0]) + len(rows[1])
    nc = len(cols[0]) + len(cols[1])
    A = np.zeros((nr, nc), complex)
    rpos = [dict((int(g), k + (0 if p == 0 else len(rows[0]))) for k, g in enumerate(rows[p]))
            for p in range(2)]
    cpos = [dict((int(g), k + (0 if q == 0 else len(cols[0]))) for k, g in enumerate(cols[q]))
            for q in range(2)]
    # vectorised per (la, lb, i, j): contributions ordered by (ea, eb) ascending
    for la in range(2):
        ga = (res + la) % nr_curve
        for lb in range(2):
            gb = (ces + lb) % nc_curve
            for i in range(2):
                ri = np.array([rpos[i].get(int(g), -1) for g in ga])
                for j in range(2):
                    cj = np.array([cpos[j].get(int(g), -1) for g in gb])
                    okr = np.nonzero(ri >= 0)[0]
                    okc = np.nonzero(cj >= 0)[0]
                    if len(okr) == 0 or len(okc) == 0:
                        continue
                    sub = B[np.ix_(okr, okc)][:, :, la, lb, i, j]
                    np.add.at(A, (ri[okr][:, None], cj[okc][None, :]), sub)
    return A


def true_block(itg: Integrator, rows, cols):
    """BlockAssembler::true_block (proj/src/assembly.cpp:332-409)."""
    n = itg.c.n
    rows = [np.asarray(r, dtype=np.int64) for r in rows]
    cols = [np.asarray(q, dtype=np.int64) for q in cols]
    res = _support(np.concatenate(rows), n)
    ces = _support(np.concatenate(cols), n)
    ea = np.repeat(res, len(ces))
    eb = np.tile(ces, len(res))
    B = itg.bundles(ea, eb).reshape(len(res), len(ces), 2, 2, 2, 2)
    return _scatter(rows, cols, n, n, res, ces, B)


def cross_block(test: Curve, rows, src: Curve, cols, S: Scalars, alpha, n_gauss):
    """kernel_cross_block (proj/src/assembly.cpp:424-509): plain full kernel,
    n_gauss x n_gauss tensor Gauss per element pair."""
    rows = [np.asarray(r, dtype=np.int64) for r in rows]
    cols = [np.asarray(q, dtype=np.int64) for q in cols]
    res = _support(np.concatenate(rows), test.n)
    ces = _support(np.concatenate(cols), src.n)
    s, w = gauss01(n_gauss)
    x = test.xy[res][:, None, :] + s[None, :, None] * test.d[res][:, None, :]   # (A, n, 2)
    y = src.xy[ces][:, None, :] + s[None, :, None] * src.d[ces][:, None, :]     # (B, n, 2)
    z = x[:, None, :, None, :] - y[None, :, None, :, :]                           # (A,B,n,n,2)
    r = np.hypot(z[..., 0], z[..., 1])
    zh = z / r[..., None]
    fs = S.full(r)
    nx = np.broadcast_to(test.nrm[res][:, None, None, None, :], zh.shape)
    ny = np.broadcast_to(src.nrm[ces][None, :, None, None, :], zh.shape)
    km = combine_D(fs, zh, ny) + complex(alpha) * combine_N(fs, zh, nx, ny)
    P = np.stack([1 - s, s])
    wgt = np.outer(w, w)[None, None] * (test.h[res][:, None] * src.h[ces][None, :])[:, :, None, None]
    B = np.einsum("abij,li,mj,abijkq->ablmkq", wgt, P, P, km)
    return _scatter(rows, cols, test.n, src.n, res, ces, B)


# ------------------------------------------------------------------- proxy
@dataclass
class Proxy:
    center: tuple
    radius: float
    polygon: Curve
    enclosed: np.ndarray


def build_proxy(curve: Curve, begin, end, radius_factor=1.5, m_prime=64):
    """proj/src/compression.cpp:25-69."""
    if radius_factor <= 1.0:
        raise ValueError("build_proxy: radius_factor must exceed 1")
    n = curve.n
    idx = np.array([(g % n + n) % n for g in range(begin - 1, end + 1)])
    p = curve.xy[idx]
    lo, hi = p.min(0), p.max(0)
    cx, cy = 0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1])
    rad = radius_factor * max(0.5 * math.hypot(hi[0] - lo[0], hi[1] - lo[1]), 1e-300)
    t = np.array([2.0 * PI * j / m_prime for j in range(m_prime)])
    poly = Curve(np.stack([cx + rad * np.cos(t), cy + rad * np.sin(t)], axis=1))
    d = np.hypot(curve.xy[:, 0] - cx, curve.xy[:, 1] - cy)
    g = np.arange(n)
    enc = np.nonzero((d < rad) & ((g < begin) | (g >= end)))[0]
    return Proxy((cx, cy), rad, poly, enc)


# ------------------------------------------------------------------- CPQR
def cpqr(a, gaps=None):
    """Column-pivoted Householder QR with LAPACK zlaqp2 pivoting (zgeqp3 as
    called by Cpqr, proj/src/lapack.cpp:101-119).  Returns (R, jpvt).
    With a list `gaps`, appends per step the gap between the largest and
    second-largest partial column norm among the candidates, divided by the
    largest initial column norm |R_00| (1.0 when a single candidate is left):
    the matrix entries carry rounding of order eps |R_00|, so a gap near that
    level means the pivot is a tie that rounding decides."""
    A = np.array(a, dtype=complex, order="F")
    m, n = A.shape
    jp = np.arange(n)
    vn1 = np.linalg.norm(A, axis=0)
    vn2 = vn1.copy()
    tol3z = math.sqrt(2.0 ** -53)
    r00 = float(vn1.max()) if n else 0.0
    for i in range(min(m, n)):
        if gaps is not None:
            c = np.sort(vn1[i:])[::-1]
            gaps.append(1.0 if c.size < 2 or r00 == 0 else float((c[0] - c[1]) / r00))
        pvt = i + int(np.argmax(vn1[i:]))
        if pvt != i:
            A[:, [i, pvt]] = A[:, [pvt, i]]
            jp[[i, pvt]] = jp[[pvt, i]]
            vn1[pvt], vn2[pvt] = vn1[i], vn2[i]
        alpha = A[i, i]
        xn = np.linalg.norm(A[i + 1:, i])
        if xn == 0 and alpha.imag == 0:
            tau = 0
            beta = alpha.real
        else:
            beta = -math.copysign(math.sqrt(abs(alpha) ** 2 + xn ** 2), alpha.real)
            tau = complex((beta - alpha.real) / beta, -alpha.imag / beta)
            A[i + 1:, i] *= 1.0 / (alpha - beta)
        A[i, i] = beta
        if i + 1 < n and tau != 0:
            v = np.concatenate([[1.0], A[i + 1:, i]])
            wv = v.conj() @ A[i:, i + 1:]
            A[i:, i + 1:] -= np.conj(tau) * np.outer(v, wv)
        for j in range(i + 1, n):
            if vn1[j] == 0:
                continue
            temp = max(1.0 - (abs(A[i, j]) / vn1[j]) ** 2, 0.0)
            temp2 = temp * (vn1[j] / vn2[j]) ** 2
            if temp2 <= tol3z:
                vn1[j] = np.linalg.norm(A[i + 1:, j]) if i + 1 < m else 0.0
                vn2[j] = vn1[j]
            else:
                vn1[j] *= math.sqrt(temp)
    return np.triu(A[: min(m, n)]), jp


def eps_rank(R, eps):
    """Cpqr::eps_rank (proj/src/lapack.cpp:127-138)."""
    d = np.abs(np.diag(R))
    if d[0] == 0:
        return 0
    hit = np.nonzero(d <= eps * d[0])[0]
    return int(hit[0]) if len(hit) else len(d)


def interpolation(R, jp, k):
    """Cpqr::interpolation (proj/src/lapack.cpp:140-158)."""
    n = R.shape[1]
    coeff = np.zeros((k, n), complex)
    if k == 0:
        return jp[:0].copy(), coeff
    T = sla.solve_triangular(R[:k, :k], R[:k, k:], lower=False)
    coeff[np.arange(k), jp[:k]] = 1.0
    coeff[:, jp[k:]] = T
    return jp[:k].copy(), coeff


@dataclass
class CellBasis:
    k: int
    saturated: bool
    row_skeleton: list
    col_skeleton: list
    u: list
    v: list


def basis_from_interactions(mv, mu, rows, cols, eps):
    """proj/src/compression.cpp:71-118."""
    nr0, nc0 = len(rows[0]), len(cols[0])
    qs = [cpqr(mv[:, :nc0]), cpqr(mv[:, nc0:]), cpqr(mu[:nr0].conj().T),
          cpqr(mu[nr0:].conj().T)]
    k = max(eps_rank(R, eps) for R, _ in qs)
    k = min(k, min(eps_rank(R, PIVOT_FLOOR) for R, _ in qs))
    ip = [interpolation(R, jp, k) for R, jp in qs]
    sat = k >= min(len(cols[0]), len(cols[1]), len(rows[0]), len(rows[1]))
    return CellBasis(
        k=k, saturated=bool(sat),
        col_skeleton=[np.asarray(cols[0])[ip[0][0]], np.asarray(cols[1])[ip[1][0]]],
        row_skeleton=[np.asarray(rows[0])[ip[2][0]], np.asarray(rows[1])[ip[3][0]]],
        v=[ip[0][1], ip[1][1]], u=[ip[2][1].conj().T, ip[3][1].conj().T])


# ----------------------------------------------------------------- problem
class Problem:
    """Mesh + medium + assembler + AssemblerSource in one object."""

    def __init__(self, xy, med: Medium, alpha=None, corner=10, far=4, rhs_nodes=8,
                 refine=1.0, radius_factor=1.5, m_prime=64, n_gauss=6):
        self.c = Curve(xy)
        self.med = med
        self.alpha = med.default_coupling() if alpha is None else complex(alpha)
        self.itg = Integrator(self.c, med, self.alpha, corner, far, refine)
        self.rf, self.mp, self.ng = radius_factor, m_prime, n_gauss
        self.rhs_nodes = int(rhs_nodes * refine + 0.5)

    @property
    def n(self):
        return self.c.n

    def block(self, rows, cols):
        return true_block(self.itg, rows, cols)

    def cell_mats(self, rows, cols, begin, end):
        """AssemblerSource::cell_basis interaction matrices (compression.cpp:139-166)."""
        px = build_proxy(self.c, begin, end, self.rf, self.mp)
        poly = [np.arange(self.mp)] * 2
        mv = cross_block(px.polygon, poly, self.c, cols, self.itg.S, self.alpha, self.ng)
        mu = cross_block(self.c, rows, px.polygon, poly, self.itg.S, self.alpha, self.ng)
        if len(px.enclosed):
            enc = [px.enclosed, px.enclosed]
            mv = np.vstack([mv, self.block(enc, cols)])
            mu = np.hstack([mu, self.block(rows, enc)])
        return mv, mu

    def cell_basis(self, rows, cols, begin, end, eps):
        mv, mu = self.cell_mats(rows, cols, begin, end)
        return basis_from_interactions(mv, mu, rows, cols, eps)

    def rhs(self, angles, amplitude=1.0, kind=0):
        """BlockAssembler::rhs for plane waves (proj/include/ebem/assembly.hpp:94-119);
        kind 0: PlanePWave (proj/src/kernels.cpp:99-118), kind 1: SV."""
        c, med = self.c, self.med
        s, w = gauss01(self.rhs_nodes)
        angles = np.atleast_1d(angles)
        out = np.zeros((2 * c.n, len(angles)), complex)
        x = c.xy[:, None, :] + s[None, :, None] * c.d[:, None, :]          # (E, q, 2)
        for col, ang in enumerate(angles):
            d = np.array([math.cos(ang), math.sin(ang)])
            k = med.kL if kind == 0 else med.kT
            ph = amplitude * np.exp(-1j * k * (x @ d))
            f = -1j * k * ph
            nd = c.nrm @ d
            if kind == 0:
                u = ph[..., None] * d
                t = f[..., None] * (med.lam * c.nrm[:, None, :] + 2 * med.mu * nd[:, None, None] * d)
            else:
                p = np.array([-d[1], d[0]])
                npp = c.nrm @ p
                u = ph[..., None] * p
                t = f[..., None] * (med.mu * (nd[:, None, None] * p + npp[:, None, None] * d))
            v = u + self.alpha * t                                         # (E, q, 2)
            wh = w[None, :] * c.h[:, None]
            for a, shp in enumerate((1 - s, s)):
                contrib = np.einsum("eq,eqi->ei", shp[None, :] * wh, v)
                ga = (np.arange(c.n) + a) % c.n
                np.add.at(out[:, col], ga, contrib[:, 0])
                np.add.at(out[:, col], c.n + ga, contrib[:, 1])
        return out

    def dense(self):
        g = np.arange(self.n)
        return self.block([g, g], [g, g])


# --------------------------------------------------------------------- FDS
@dataclass
class _Cell:
    jrow: list = None
    jcol: list = None
    nloc: int = 0
    k: int = 0
    srow: list = None
    scol: list = None
    v: list = None
    lu: tuple = None
    ainv_u: np.ndarray = None
    atilde: np.ndarray = None


class Fds:
    """FdsSolver (proj/src/fds.cpp:18-263) over a Problem."""

    def __init__(self, prob: Problem, depth: int, eps: float, ell0: int = 1):
        n = prob.n
        if ell0 < 0 or ell0 >= depth:
            raise ValueError("FdsSolver: dense level must lie strictly above the leaves")
        if n % (1 << depth):
            raise ValueError("ClusterTree: node count must be divisible by 2^depth")
        self.p, self.depth, self.eps, self.ell0 = prob, depth, eps, ell0
        self.cells = [_Cell() for _ in range((2 << depth) - 1)]
        self.max_rank = [0] * (depth + 1)
        self.saturated = False
        leaf = n >> depth
        for c in range((1 << depth) - 1, (2 << depth) - 1):
            a = (c - ((1 << depth) - 1)) * leaf
            r = list(range(a, a + leaf))
            self.cells[c].jrow = [r, r]
            self.cells[c].jcol = [r, r]
            self.cells[c].nloc = leaf
        for level in range(depth, ell0, -1):
            first, last = (1 << level) - 1, (2 << level) - 2
            size = n >> level
            for c in range(first, last + 1):
                C = self.cells[c]
                b0 = (c - first) * size
                B = prob.cell_basis(C.jrow, C.jcol, b0, b0 + size, eps)
                C.k, C.srow, C.scol, C.v = B.k, B.row_skeleton, B.col_skeleton, B.v
                diag = prob.block(C.jrow, C.jcol) if level == depth else self._reduced(c)
                C.lu = sla.lu_factor(diag)
                U = np.zeros((2 * C.nloc, 2 * C.k), complex)
                U[:C.nloc, :C.k] = B.u[0]
                U[C.nloc:, C.k:] = B.u[1]
                C.ainv_u = sla.lu_solve(C.lu, U)
                W = np.vstack([C.v[0] @ C.ainv_u[:C.nloc], C.v[1] @ C.ainv_u[C.nloc:]])
                C.atilde = np.linalg.inv(W) if C.k else np.zeros((0, 0), complex)
                self.max_rank[level] = max(self.max_rank[level], C.k)
                self.saturated |= B.saturated
            for c in range((1 << (level - 1)) - 1, (2 << (level - 1)) - 1):
                c1, c2 = self.cells[2 * c + 1], self.cells[2 * c + 2]
                P = self.cells[c]
                P.jrow = [list(c1.srow[q]) + list(c2.srow[q]) for q in range(2)]
                P.jcol = [list(c1.scol[q]) + list(c2.scol[q]) for q in range(2)]
                P.nloc = c1.k + c2.k
        self.top = list(range((1 << ell0) - 1, (2 << ell0) - 1))
        offs = np.cumsum([0] + [2 * self.cells[c].nloc for c in self.top])
        self.top_off = offs
        T = np.zeros((offs[-1], offs[-1]), complex)
        for i, ci in enumerate(self.top):
            for j, cj in enumerate(self.top):
                blk = self._reduced(ci) if i == j else prob.block(self.cells[ci].jrow,
                                                                  self.cells[cj].jcol)
                T[offs[i]:offs[i + 1], offs[j]:offs[j + 1]] = blk
        self.top_lu = sla.lu_factor(T)

    def _reduced(self, cell):
        """FdsSolver::reduced_diagonal (proj/src/fds.cpp:33-54)."""
        c1, c2 = self.cells[2 * cell + 1], self.cells[2 * cell + 2]
        k1, k2 = c1.k, c2.k
        npp = k1 + k2
        x12 = self.p.block(c1.srow, c2.scol)
        x21 = self.p.block(c2.srow, c1.scol)
        a = np.zeros((2 * npp, 2 * npp), complex)
        for p in range(2):
            for q in range(2):
                a[p * npp:p * npp + k1, q * npp:q * npp + k1] = c1.atilde[p * k1:(p + 1) * k1, q * k1:(q + 1) * k1]
                a[p * npp + k1:(p + 1) * npp, q * npp + k1:(q + 1) * npp] = c2.atilde[p * k2:(p + 1) * k2, q * k2:(q + 1) * k2]
                a[p * npp:p * npp + k1, q * npp + k1:(q + 1) * npp] = x12[p * k1:(p + 1) * k1, q * k2:(q + 1) * k2]
                a[p * npp + k1:(p + 1) * npp, q * npp:q * npp + k1] = x21[p * k2:(p + 1) * k2, q * k1:(q + 1) * k1]
        return a

    def rank_of(self, cell):
        return self.cells[cell].k

    def solve(self, rhs):
        """FdsSolver::solve (proj/src/fds.cpp:156-263)."""
        n, depth = self.p.n, self.depth
        rhs = np.asarray(rhs, complex).reshape(2 * n, -1)
        leaf = n >> depth
        f, ft, af, x = {}, {}, {}, {}
        for c in range((1 << depth) - 1, (2 << depth) - 1):
            a = (c - ((1 << depth) - 1)) * leaf
            f[c] = np.vstack([rhs[a:a + leaf], rhs[n + a:n + a + leaf]])
        for level in range(depth, self.ell0, -1):
            for c in range((1 << level) - 1, (2 << level) - 1):
                C = self.cells[c]
                af[c] = sla.lu_solve(C.lu, f[c])
                vf = np.vstack([C.v[0] @ af[c][:C.nloc], C.v[1] @ af[c][C.nloc:]])
                ft[c] = C.atilde @ vf
            for c in range((1 << (level - 1)) - 1, (2 << (level - 1)) - 1):
                k1, k2 = self.cells[2 * c + 1].k, self.cells[2 * c + 2].k
                a1, a2 = ft[2 * c + 1], ft[2 * c + 2]
                f[c] = np.vstack([a1[:k1], a2[:k2], a1[k1:], a2[k2:]])
        ftop = np.vstack([f[c] for c in self.top])
        xt = sla.lu_solve(self.top_lu, ftop)
        for i, c in enumerate(self.top):
            x[c] = xt[self.top_off[i]:self.top_off[i + 1]]
        for level in range(self.ell0, depth):
            for c in range((1 << level) - 1, (2 << level) - 1):
                k1, k2 = self.cells[2 * c + 1].k, self.cells[2 * c + 2].k
                for side in range(2):
                    cc = 2 * c + 1 + side
                    C = self.cells[cc]
                    r0 = 0 if side == 0 else k1
                    y = np.vstack([x[c][r0:r0 + C.k], x[c][k1 + k2 + r0:k1 + k2 + r0 + C.k]])
                    x[cc] = af[cc] + C.ainv_u @ (C.atilde @ y - ft[cc])
        out = np.zeros((2 * n, rhs.shape[1]), complex)
        for c in range((1 << depth) - 1, (2 << depth) - 1):
            a = (c - ((1 << depth) - 1)) * leaf
            out[a:a + leaf] = x[c][:leaf]
            out[n + a:n + a + leaf] = x[c][leaf:]
        return out


def circle_nodes(n, radius=1.0):
    """Mesh::star(n, StarShape{r, 0, b}) nodes (proj/src/geometry.cpp:10-13,39-46)."""
    th = np.array([2.0 * PI * t / n for t in range(n)])
    return np.stack([radius * np.cos(th), radius * np.sin(th)], axis=1)
