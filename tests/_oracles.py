"""ctypes wrappers for the oracles -- TEST INFRASTRUCTURE ONLY.

* ``RefLib``   : oracle/_ref/libebem_ref.so, the reference library compiled in
                 place from /root/reference/proj/src (see oracle/Makefile and
                 oracle/ref_capi.cpp for the file:line of every entry point).
(The from-scratch CPU restatement is the numpy module oracle/ebem_oracle.py,
imported directly.)

Only tests/, bench.py's CPU legs and __graft_entry__.smoke() import this.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF_SO = ROOT / "oracle" / "_ref" / "libebem_ref.so"

_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


def _ci(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def cplx_from(buf, rows, cols):
    """Column-major interleaved complex buffer -> (rows, cols) complex array."""
    return buf.view(np.complex128).reshape(cols, rows).T.copy()


def to_buf(m):
    """(rows, cols) complex array -> column-major interleaved float64 buffer."""
    m = np.asarray(m, dtype=np.complex128)
    return np.asfortranarray(m).ravel(order="F").view(np.float64).copy()


class OracleError(RuntimeError):
    pass


class _Base:
    prefix = ""

    def _chk(self, rc):
        if rc != 0:
            msg = getattr(self.lib, self.prefix + "last_error")()
            raise OracleError(f"rc={rc}: {msg.decode()}")


class RefLib(_Base):
    """The reference library, compiled in place."""

    prefix = "ref_"

    def __init__(self, path=REF_SO):
        if not Path(path).exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref`")
        self.lib = ctypes.CDLL(str(path))
        self.lib.ref_last_error.restype = ctypes.c_char_p

    def set_threads(self, n):
        self.lib.ref_set_threads(int(n))

    def max_threads(self):
        return self.lib.ref_max_threads()

    def hankel(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros(4 * x.size)
        self._chk(self.lib.ref_hankel1_01(_ptr(x), x.size, _ptr(out)))
        o = out.reshape(-1, 4)
        return o[:, 0] + 1j * o[:, 1], o[:, 2] + 1j * o[:, 3]

    def scalars(self, lam, mu, rho, omega, r, which=0):
        r = np.ascontiguousarray(r, dtype=np.float64)
        out = np.zeros(20 * r.size)
        self._chk(self.lib.ref_scalars(_D(lam), _D(mu), _D(rho), _D(omega),
                                       _ptr(r), r.size, which, _ptr(out)))
        return out.view(np.complex128).reshape(-1, 10)

    def integrated_remainder(self, lam, mu, rho, omega, scale, upow):
        out = np.zeros(20)
        self._chk(self.lib.ref_integrated_remainder(
            _D(lam), _D(mu), _D(rho), _D(omega), _D(scale), upow, _ptr(out)))
        return out.view(np.complex128)

    def gauss_rule(self, n):
        x = np.zeros(n)
        w = np.zeros(n)
        self._chk(self.lib.ref_gauss_rule(n, _ptr(x), _ptr(w)))
        return x, w

    def cpqr(self, a, eps=(1e-10, 1e-14), k_interp=0):
        a = np.asarray(a, dtype=np.complex128)
        m, n = a.shape
        buf = to_buf(a)
        kmax = min(m, n)
        jpvt = np.zeros(kmax, dtype=np.int32)
        rdiag = np.zeros(kmax)
        e = np.ascontiguousarray(eps, dtype=np.float64)
        ranks = np.zeros(len(e), dtype=np.int32)
        coeff = np.zeros(2 * max(k_interp, 1) * n)
        self._chk(self.lib.ref_cpqr(_ptr(buf), m, n, _ptr(jpvt), _ptr(rdiag),
                                    _ptr(e), len(e), _ptr(ranks), k_interp,
                                    _ptr(coeff)))
        c = cplx_from(coeff, k_interp, n) if k_interp > 0 else None
        return jpvt, rdiag, ranks, c

    def problem(self, nodes, lam, mu, rho, omega, alpha, corner=10, far=4,
                rhs_nodes=8, refine=1.0, radius_factor=1.5, m_prime=64,
                n_gauss=6):
        return RefProblem(self, nodes, lam, mu, rho, omega, alpha, corner, far,
                          rhs_nodes, refine, radius_factor, m_prime, n_gauss)


class RefProblem:
    def __init__(self, ref, nodes, lam, mu, rho, omega, alpha, corner, far,
                 rhs_nodes, refine, radius_factor, m_prime, n_gauss):
        self.ref = ref
        lib = ref.lib
        xy = np.ascontiguousarray(nodes, dtype=np.float64).reshape(-1)
        self.n = xy.size // 2
        icfg = _ci([corner, far, rhs_nodes, m_prime])
        dcfg = np.array([refine, radius_factor])
        h = _P()
        ref._chk(lib.ref_problem_new(_ptr(xy), self.n, _D(lam), _D(mu), _D(rho),
                                     _D(omega), _D(alpha.real), _D(alpha.imag),
                                     _ptr(icfg), _ptr(dcfg), n_gauss,
                                     ctypes.byref(h)))
        self.h = h
        self.m_prime = m_prime

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_problem_free(self.h)
            self.h = None

    def true_block(self, rows, cols):
        r0, r1 = _ci(rows[0]), _ci(rows[1])
        c0, c1 = _ci(cols[0]), _ci(cols[1])
        nr, nc = r0.size + r1.size, c0.size + c1.size
        out = np.zeros(2 * max(nr * nc, 1))
        self.ref._chk(self.ref.lib.ref_true_block(
            self.h, _ptr(r0), r0.size, _ptr(r1), r1.size, _ptr(c0), c0.size,
            _ptr(c1), c1.size, _ptr(out)))
        return cplx_from(out[: 2 * nr * nc], nr, nc)

    def dense(self):
        out = np.zeros(2 * (2 * self.n) ** 2)
        self.ref._chk(self.ref.lib.ref_dense(self.h, _ptr(out)))
        return cplx_from(out, 2 * self.n, 2 * self.n)

    def build_proxy(self, begin, end):
        o3 = np.zeros(3)
        ne = _I()
        self.ref._chk(self.ref.lib.ref_build_proxy(self.h, begin, end, _ptr(o3),
                                                   ctypes.byref(ne), None, 0))
        enc = np.zeros(max(ne.value, 1), dtype=np.int32)
        self.ref._chk(self.ref.lib.ref_build_proxy(self.h, begin, end, _ptr(o3),
                                                   ctypes.byref(ne), _ptr(enc),
                                                   enc.size))
        return o3, enc[: ne.value]

    def cell_mats(self, rows, cols, begin, end):
        r0, r1 = _ci(rows[0]), _ci(rows[1])
        c0, c1 = _ci(cols[0]), _ci(cols[1])
        nout = _I()
        args = (self.h, _ptr(r0), r0.size, _ptr(r1), r1.size, _ptr(c0),
                c0.size, _ptr(c1), c1.size, begin, end, ctypes.byref(nout))
        self.ref._chk(self.ref.lib.ref_cell_mats(*args, None, None))
        no = nout.value
        nr, nc = r0.size + r1.size, c0.size + c1.size
        mv = np.zeros(2 * no * nc)
        mu = np.zeros(2 * nr * no)
        self.ref._chk(self.ref.lib.ref_cell_mats(*args, _ptr(mv), _ptr(mu)))
        return cplx_from(mv, no, nc), cplx_from(mu, nr, no)

    def cell_basis(self, rows, cols, begin, end, eps):
        r0, r1 = _ci(rows[0]), _ci(rows[1])
        c0, c1 = _ci(cols[0]), _ci(cols[1])
        k = _I()
        sat = _I()
        args = (self.h, _ptr(r0), r0.size, _ptr(r1), r1.size, _ptr(c0),
                c0.size, _ptr(c1), c1.size, begin, end, _D(eps),
                ctypes.byref(k), ctypes.byref(sat))
        self.ref._chk(self.ref.lib.ref_cell_basis(*args, None, None, None,
                                                  None, None))
        kk = k.value
        skel = np.zeros(max(4 * kk, 1), dtype=np.int32)
        u0 = np.zeros(2 * max(r0.size * kk, 1))
        u1 = np.zeros(2 * max(r1.size * kk, 1))
        v0 = np.zeros(2 * max(kk * c0.size, 1))
        v1 = np.zeros(2 * max(kk * c1.size, 1))
        self.ref._chk(self.ref.lib.ref_cell_basis(*args, _ptr(skel), _ptr(u0),
                                                  _ptr(u1), _ptr(v0), _ptr(v1)))
        s = skel[: 4 * kk].reshape(4, kk)
        return dict(k=kk, saturated=bool(sat.value),
                    row_skeleton=(s[0].copy(), s[1].copy()),
                    col_skeleton=(s[2].copy(), s[3].copy()),
                    u=(cplx_from(u0[: 2 * r0.size * kk], r0.size, kk),
                       cplx_from(u1[: 2 * r1.size * kk], r1.size, kk)),
                    v=(cplx_from(v0[: 2 * kk * c0.size], kk, c0.size),
                       cplx_from(v1[: 2 * kk * c1.size], kk, c1.size)))

    def rhs_plane_p(self, angles, amplitude=1.0):
        a = np.ascontiguousarray(np.atleast_1d(angles), dtype=np.float64)
        out = np.zeros(4 * self.n * a.size)
        self.ref._chk(self.ref.lib.ref_rhs_plane_p(self.h, _ptr(a), a.size,
                                                   _D(amplitude), _ptr(out)))
        return cplx_from(out, 2 * self.n, a.size)

    def evaluate_field(self, u, pts, ng=8, angle=None, amplitude=1.0):
        """evaluate_scattered (angle None) / evaluate_field with a P wave:
        (m, 2) complex displacements."""
        ub = to_buf(np.asarray(u, dtype=np.complex128).reshape(-1, 1))
        p = np.ascontiguousarray(pts, dtype=np.float64).ravel()
        m = p.size // 2
        out = np.zeros(4 * m)
        self.ref._chk(self.ref.lib.ref_evaluate_field(
            self.h, _ptr(ub), _ptr(p), m, ng, _D(-100.0 if angle is None else angle),
            _D(amplitude), _ptr(out)))
        return out.view(np.complex128).reshape(m, 2)

    def conv_solve(self, rhs):
        rhs = np.asarray(rhs, dtype=np.complex128).reshape(2 * self.n, -1)
        m = rhs.shape[1]
        b = to_buf(rhs)
        x = np.zeros_like(b)
        rc = _D()
        self.ref._chk(self.ref.lib.ref_conv_solve(self.h, _ptr(b), m, _ptr(x),
                                                  ctypes.byref(rc)))
        return cplx_from(x, 2 * self.n, m), rc.value

    def fds(self, depth, eps, ell0=1, record=True):
        return RefFds(self, depth, eps, ell0, record)


class RefFds:
    def __init__(self, prob, depth, eps, ell0, record):
        self.prob = prob
        self.depth = depth
        lib = prob.ref.lib
        h = _P()
        stats = np.zeros(5)
        mr = np.zeros(depth + 1, dtype=np.int32)
        prob.ref._chk(lib.ref_fds_new(prob.h, depth, _D(eps), ell0,
                                      1 if record else 0, ctypes.byref(h),
                                      _ptr(stats), _ptr(mr)))
        self.h = h
        self.stats = dict(upward_seconds=stats[0], top_factor_seconds=stats[1],
                          basis_cpu_seconds=stats[2], top_dim=int(stats[3]),
                          saturated=bool(stats[4]), max_rank=mr.tolist())

    def __del__(self):
        if getattr(self, "h", None):
            self.prob.ref.lib.ref_fds_free(self.h)
            self.h = None

    def solve(self, rhs):
        n = self.prob.n
        rhs = np.asarray(rhs, dtype=np.complex128).reshape(2 * n, -1)
        m = rhs.shape[1]
        b = to_buf(rhs)
        x = np.zeros_like(b)
        t = np.zeros(3)
        self.prob.ref._chk(self.prob.ref.lib.ref_fds_solve(self.h, _ptr(b), m,
                                                           _ptr(x), _ptr(t)))
        return cplx_from(x, 2 * n, m), t

    def rank_of(self, cell):
        return self.prob.ref.lib.ref_fds_rank_of(self.h, cell)

    def cell(self, begin, end):
        sizes = np.zeros(5, dtype=np.int32)
        lib = self.prob.ref.lib
        self.prob.ref._chk(lib.ref_fds_cell(self.h, begin, end, _ptr(sizes),
                                            None, None, None))
        nr0, nr1, nc0, nc1, k = sizes.tolist()
        rows = np.zeros(max(nr0 + nr1, 1), dtype=np.int32)
        cols = np.zeros(max(nc0 + nc1, 1), dtype=np.int32)
        skel = np.zeros(max(4 * k, 1), dtype=np.int32)
        self.prob.ref._chk(lib.ref_fds_cell(self.h, begin, end, _ptr(sizes),
                                            _ptr(rows), _ptr(cols), _ptr(skel)))
        s = skel[: 4 * k].reshape(4, k)
        return dict(k=k, rows=(rows[:nr0], rows[nr0:nr0 + nr1]),
                    cols=(cols[:nc0], cols[nc0:nc0 + nc1]),
                    row_skeleton=(s[0], s[1]), col_skeleton=(s[2], s[3]))


def star_nodes(n, r=1.0, a=0.3, b=3):
    """Mesh::star node positions (proj/src/geometry.cpp:10-13, :39-46)."""
    t = 2.0 * np.pi * np.arange(n) / n
    # same operation order as StarShape::point
    theta = np.array([2.0 * 3.14159265358979323846 * i / n for i in range(n)])
    rad = (r + a * np.cos(b * theta)) / (1.0 + a)
    del t
    return np.stack([rad * np.cos(theta), rad * np.sin(theta)], axis=1)
