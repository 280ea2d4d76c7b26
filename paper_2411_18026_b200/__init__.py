"""B200-native (sm_100a) fast direct solver path of the `ebem` library.

Python mirror of the reference C++ API for the hot path (SURVEY.md section
8b), backed by ``libebem_gpu.so`` (CUDA kernels + native runtime) through the
C ABI declared in ``include/ebem_gpu.h``:

    Mesh, StarShape                  proj/include/ebem/geometry.hpp:16-75
    Medium                           proj/include/ebem/medium.hpp:14-60
    ClusterTree                      proj/include/ebem/geometry.hpp:82-114
    AssemblyConfig, BlockAssembler   proj/include/ebem/assembly.hpp:21-130
    PlanePWave (+ PlaneSVWave)       proj/include/ebem/kernels.hpp:74-89
    ProxyConfig, CellBasis,
    BlockSource, AssemblerSource     proj/include/ebem/compression.hpp:14-123
    FdsConfig, FdsStats,
    FdsSolveTiming, FdsSolver        proj/include/ebem/fds.hpp:13-94

Matrices are numpy complex128 arrays; global vectors are component-major
``[u1(0..N-1); u2(0..N-1)]``.  There is no CPU fallback: without a CUDA
device every compute call raises :class:`CudaError`.
"""
from __future__ import annotations

import ctypes
import os
import math
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "StarShape", "Mesh", "Medium", "ClusterTree", "AssemblyConfig",
    "ProxyConfig", "FdsConfig", "FdsStats", "FdsSolveTiming", "CellBasis",
    "BlockAssembler", "BlockSource", "AssemblerSource", "FdsSolver",
    "PlanePWave", "PlaneSVWave", "EbemError", "InvalidArgument",
    "SingularMatrix", "DomainError", "LengthError", "CudaError", "lib",
    "eval_hankel", "device_info", "launch_count",
]

K_PI = 3.14159265358979323846

# --------------------------------------------------------------------- errors


class EbemError(RuntimeError):
    """Base of the errors raised by the native library."""


class InvalidArgument(EbemError, ValueError):
    """std::invalid_argument in the reference."""


class SingularMatrix(EbemError):
    """std::runtime_error from LuFactor (zero pivot)."""


class DomainError(EbemError, ValueError):
    """std::domain_error (element too long for the frequency)."""


class LengthError(EbemError, MemoryError):
    """std::length_error (memory budget)."""


class CudaError(EbemError):
    """No CUDA device or a CUDA failure (there is no CPU fallback)."""


class LogicError(EbemError):
    """std::logic_error."""


_ERRORS = {1: InvalidArgument, 2: SingularMatrix, 3: DomainError,
           4: LengthError, 5: CudaError, 6: LogicError}

# ----------------------------------------------------------------- native lib

# EBEM_GPU_LIB: an alternative in-tree build of the library (A/B measurements)
_LIB_PATH = Path(os.environ.get("EBEM_GPU_LIB") or Path(__file__).resolve().parent / "libebem_gpu.so")
_lib = None


class _AsmCfg(ctypes.Structure):
    _fields_ = [("corner_nodes", ctypes.c_int), ("far_nodes", ctypes.c_int),
                ("rhs_nodes", ctypes.c_int), ("refine", ctypes.c_double),
                ("max_dense_bytes", ctypes.c_size_t)]


class _ProxyCfg(ctypes.Structure):
    _fields_ = [("radius_factor", ctypes.c_double), ("m_prime", ctypes.c_int),
                ("n_gauss", ctypes.c_int)]


class _FdsCfg(ctypes.Structure):
    _fields_ = [("epsilon", ctypes.c_double), ("ell0", ctypes.c_int)]


_MAX_LEVELS = 32


class _FdsStats(ctypes.Structure):
    _fields_ = [("depth", ctypes.c_int), ("max_rank", ctypes.c_int * _MAX_LEVELS),
                ("top_dim", ctypes.c_int), ("saturated", ctypes.c_int),
                ("upward_seconds", ctypes.c_double),
                ("top_factor_seconds", ctypes.c_double),
                ("basis_cpu_seconds", ctypes.c_double),
                ("factorize_device_seconds", ctypes.c_double)]


class _SolveTiming(ctypes.Structure):
    _fields_ = [("upward_seconds", ctypes.c_double),
                ("top_seconds", ctypes.c_double),
                ("downward_seconds", ctypes.c_double),
                ("device_seconds", ctypes.c_double)]


class _ConvStats(ctypes.Structure):
    _fields_ = [("assemble_seconds", ctypes.c_double), ("factor_seconds", ctypes.c_double),
                ("rcond", ctypes.c_double), ("min_pivot", ctypes.c_double),
                ("condition_warning", ctypes.c_int)]


def lib():
    """The loaded native library (raises ImportError when it is not built)."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise ImportError(
                f"{_LIB_PATH} is missing: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(str(_LIB_PATH))
        L.ebem_gpu_last_error.restype = ctypes.c_char_p
        L.ebem_gpu_launch_count.restype = ctypes.c_longlong
        L.ebem_gpu_problem_size.restype = ctypes.c_int
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        msg = lib().ebem_gpu_last_error().decode()
        raise _ERRORS.get(rc, EbemError)(msg)


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _ints(v):
    return np.ascontiguousarray(np.asarray(v, dtype=np.int64).astype(np.int32))


def _to_cbuf(m, rows, cols):
    """complex (rows, cols) -> column-major interleaved float64 buffer."""
    a = np.asarray(m, dtype=np.complex128).reshape(rows, cols)
    return np.asfortranarray(a).ravel(order="F").view(np.float64).copy()


def _from_cbuf(buf, rows, cols):
    return buf.view(np.complex128).reshape(cols, rows).T.copy()


def device_info() -> str:
    buf = ctypes.create_string_buffer(256)
    _check(lib().ebem_gpu_device_info(buf, 256))
    return buf.value.decode()


def launch_count() -> int:
    """Kernel launches issued by the library since it was loaded."""
    return int(lib().ebem_gpu_launch_count())


def eval_hankel(x):
    """(H0(x), H1(x)) from the device evaluator (parity hook)."""
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    out = np.zeros(4 * x.size)
    _check(lib().ebem_gpu_eval_hankel(_p(x), x.size, _p(out)))
    o = out.reshape(-1, 4)
    return o[:, 0] + 1j * o[:, 1], o[:, 2] + 1j * o[:, 3]


# ------------------------------------------------------------------ geometry


@dataclass
class StarShape:
    """x(t) = (r + a cos(b t)) (cos t, sin t) / (1 + a), geometry.cpp:10-13."""
    r: float = 1.0
    a: float = 0.3
    b: int = 3

    def point(self, theta: float):
        rad = (self.r + self.a * math.cos(float(self.b) * theta)) / (1.0 + self.a)
        return rad * math.cos(theta), rad * math.sin(theta)


class Mesh:
    """Closed piecewise-linear boundary; element e runs from node e to e+1."""

    def __init__(self, nodes):
        xy = np.ascontiguousarray(np.asarray(nodes, dtype=np.float64).reshape(-1, 2))
        if xy.shape[0] < 4:
            raise InvalidArgument("Mesh: needs at least 4 nodes")
        d = np.roll(xy, -1, axis=0) - xy
        h = np.hypot(d[:, 0], d[:, 1])
        if not np.all(h > 0.0):
            raise InvalidArgument("Mesh: zero-length element")
        self._xy = xy

    @staticmethod
    def star(n_elements: int, shape: StarShape = StarShape()) -> "Mesh":
        if n_elements < 4:
            raise InvalidArgument("Mesh::star: n too small")
        pts = [shape.point(2.0 * K_PI * t / n_elements) for t in range(n_elements)]
        return Mesh(pts)

    def size(self) -> int:
        return self._xy.shape[0]

    def node(self, i: int):
        return tuple(self._xy[i])

    @property
    def nodes(self) -> np.ndarray:
        return self._xy

    def next(self, e: int) -> int:
        return 0 if e + 1 == self.size() else e + 1

    def prev(self, e: int) -> int:
        return self.size() - 1 if e == 0 else e - 1


class Medium:
    """Isotropic elastic medium and angular frequency, medium.hpp:14-60."""

    def __init__(self, cL: float, cT: float, density: float, ang_freq: float):
        if not (cL > 0 and cT > 0 and density > 0 and ang_freq > 0):
            raise InvalidArgument("Medium: all parameters must be positive")
        if not cL > cT:
            raise InvalidArgument("Medium: requires c_L > c_T")
        self._cL, self._cT, self._rho, self._omega = cL, cT, density, ang_freq
        self._mu = density * cT * cT
        self._lambda = density * (cL * cL - 2.0 * cT * cT)

    @staticmethod
    def from_lame(lam: float, mu: float, density: float, ang_freq: float) -> "Medium":
        if not (mu > 0 and lam + mu > 0):
            raise InvalidArgument("Medium: Lame constants out of range")
        m = Medium(math.sqrt((lam + 2.0 * mu) / density), math.sqrt(mu / density),
                   density, ang_freq)
        m._lambda, m._mu = lam, mu
        return m

    def c_L(self): return self._cL
    def c_T(self): return self._cT
    def rho(self): return self._rho
    def omega(self): return self._omega
    def mu(self): return self._mu
    def lambda_(self): return self._lambda
    def k_L(self): return self._omega / self._cL
    def k_T(self): return self._omega / self._cT

    def default_coupling(self) -> complex:
        return 1j / self.k_T()


class ClusterTree:
    """Uniform binary tree over node indices, geometry.hpp:82-114."""

    def __init__(self, n_nodes: int, depth: int):
        if depth < 0:
            raise InvalidArgument("ClusterTree: negative depth")
        if n_nodes <= 0 or n_nodes % (1 << depth) != 0:
            raise InvalidArgument(
                f"ClusterTree: node count must be divisible by 2^depth (got "
                f"{n_nodes} nodes, depth {depth})")
        self._n, self._depth = n_nodes, depth

    def depth(self): return self._depth
    def n_nodes(self): return self._n
    def n_cells(self): return (2 << self._depth) - 1

    @staticmethod
    def first_cell(level): return (1 << level) - 1

    @staticmethod
    def last_cell(level): return (2 << level) - 2

    @staticmethod
    def child1(cell): return 2 * cell + 1

    @staticmethod
    def child2(cell): return 2 * cell + 2

    @staticmethod
    def parent(cell): return (cell - 1) // 2

    @staticmethod
    def depth_for(n_nodes: int, max_leaf: int) -> int:
        if n_nodes <= 0 or max_leaf <= 0:
            raise InvalidArgument("ClusterTree: sizes must be positive")
        d = 0
        while (n_nodes >> d) > max_leaf and n_nodes % (2 << d) == 0:
            d += 1
        return d

    def level_of(self, cell):
        level = 0
        while cell > self.last_cell(level):
            level += 1
        return level

    def is_leaf(self, cell): return cell >= self.first_cell(self._depth)
    def leaf_size(self): return self._n >> self._depth
    def leaf_begin(self, cell): return (cell - self.first_cell(self._depth)) * self.leaf_size()
    def leaf_end(self, cell): return self.leaf_begin(cell) + self.leaf_size()

    def cell_begin(self, cell):
        lv = self.level_of(cell)
        return (cell - self.first_cell(lv)) * (self._n >> lv)

    def cell_end(self, cell):
        return self.cell_begin(cell) + (self._n >> self.level_of(cell))


# -------------------------------------------------------------------- configs


@dataclass
class AssemblyConfig:
    corner_nodes: int = 10
    far_nodes: int = 4
    rhs_nodes: int = 8
    refine: float = 1.0
    max_dense_bytes: int = 4 << 30

    def _c(self):
        return _AsmCfg(self.corner_nodes, self.far_nodes, self.rhs_nodes,
                       self.refine, self.max_dense_bytes)


@dataclass
class ProxyConfig:
    radius_factor: float = 1.5
    m_prime: int = 64
    n_gauss: int = 6

    def _c(self):
        return _ProxyCfg(self.radius_factor, self.m_prime, self.n_gauss)


@dataclass
class FdsConfig:
    epsilon: float = 1e-8
    ell0: int = 1


@dataclass
class FdsStats:
    max_rank: list = field(default_factory=list)
    top_dim: int = 0
    saturated: bool = False
    upward_seconds: float = 0.0
    top_factor_seconds: float = 0.0
    basis_cpu_seconds: float = 0.0
    factorize_device_seconds: float = 0.0


@dataclass
class ConvStats:
    """ConvStats, dense_solver.hpp:10-19."""
    assemble_seconds: float = 0.0
    factor_seconds: float = 0.0
    rcond: float = 1.0
    min_pivot: float = 0.0
    condition_warning: bool = False


@dataclass
class FdsSolveTiming:
    upward_seconds: float = 0.0
    top_seconds: float = 0.0
    downward_seconds: float = 0.0
    device_seconds: float = 0.0


@dataclass
class CellBasis:
    k: int = 0
    saturated: bool = False
    row_skeleton: tuple = ((), ())
    col_skeleton: tuple = ((), ())
    u: tuple = (None, None)  # each |rows[p]| x k
    v: tuple = (None, None)  # each k x |cols[q]|


# -------------------------------------------------------------- incident waves


class PlanePWave:
    """u = A d exp(-i kL d.x), kernels.hpp:74-89 (kind 0 on device)."""
    kind = 0

    def __init__(self, medium: Medium, amplitude: float, angle_rad: float):
        self.medium, self.amplitude, self.angle = medium, amplitude, angle_rad

    def direction(self):
        return (math.cos(self.angle), math.sin(self.angle))


class PlaneSVWave(PlanePWave):
    """u = A p exp(-i kT d.x), p = (-d_y, d_x).  Not in the reference (config
    4 of BASELINE.json); traction from the same constitutive law."""
    kind = 1


# ------------------------------------------------------------------- problem


class _Handle:
    def __init__(self, mesh: Mesh, medium: Medium, alpha: complex,
                 acfg: AssemblyConfig, pcfg: ProxyConfig):
        L = lib()
        h = ctypes.c_void_p()
        xy = np.ascontiguousarray(mesh.nodes).ravel()
        a, p = acfg._c(), pcfg._c()
        _check(L.ebem_gpu_problem_create(
            _p(xy), mesh.size(), ctypes.c_double(medium.lambda_()),
            ctypes.c_double(medium.mu()), ctypes.c_double(medium.rho()),
            ctypes.c_double(medium.omega()), ctypes.c_double(complex(alpha).real),
            ctypes.c_double(complex(alpha).imag), ctypes.byref(a), ctypes.byref(p),
            ctypes.byref(h)))
        self.h = h
        self.n = mesh.size()

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ebem_gpu_problem_destroy(self.h)
            self.h = None

    def true_block(self, rows, cols):
        r0, r1 = _ints(rows[0]), _ints(rows[1])
        c0, c1 = _ints(cols[0]), _ints(cols[1])
        nr, nc = r0.size + r1.size, c0.size + c1.size
        out = np.zeros(2 * max(nr * nc, 1))
        _check(lib().ebem_gpu_true_block(self.h, _p(r0), r0.size, _p(r1), r1.size,
                                         _p(c0), c0.size, _p(c1), c1.size, _p(out)))
        return _from_cbuf(out[: 2 * nr * nc], nr, nc)

    def dense(self):
        d = 2 * self.n
        out = np.zeros(2 * d * d)
        _check(lib().ebem_gpu_dense(self.h, _p(out)))
        return _from_cbuf(out, d, d)

    def rhs(self, kind, angles, amplitude):
        a = np.ascontiguousarray(np.atleast_1d(angles), dtype=np.float64)
        out = np.zeros(4 * self.n * a.size)
        _check(lib().ebem_gpu_rhs_plane(self.h, int(kind), _p(a), a.size,
                                        ctypes.c_double(amplitude), _p(out)))
        return _from_cbuf(out, 2 * self.n, a.size)


class BlockAssembler:
    """Galerkin matrix of D + I/2 + alpha N, assembly.hpp:68-130."""

    def __init__(self, mesh: Mesh, medium: Medium, alpha: complex,
                 config: AssemblyConfig = None):
        self._mesh, self._medium = mesh, medium
        self._alpha = complex(alpha)
        self._config = config or AssemblyConfig()
        self._h = _Handle(mesh, medium, self._alpha, self._config, ProxyConfig())

    def n_nodes(self): return self._mesh.size()
    def alpha(self): return self._alpha
    def mesh(self): return self._mesh
    def medium(self): return self._medium
    def config(self): return self._config

    def true_block(self, rows, cols) -> np.ndarray:
        return self._h.true_block(rows, cols)

    def dense(self) -> np.ndarray:
        """The full 2N x 2N Galerkin matrix (assembly.cpp:311-330)."""
        return self._h.dense()

    def rhs(self, wave) -> np.ndarray:
        return self._h.rhs(wave.kind, [wave.angle], wave.amplitude)[:, 0]

    def rhs_batch(self, medium: Medium, angles_rad: Sequence[float],
                  amplitude: float, kind: int = 0) -> np.ndarray:
        return self._h.rhs(kind, angles_rad, amplitude)


class BlockSource:
    """Entry provider interface, compression.hpp:66-87."""

    def n_nodes(self) -> int:
        raise NotImplementedError

    def block(self, rows, cols) -> np.ndarray:
        raise NotImplementedError

    def cell_basis(self, rows, cols, node_begin, node_end, epsilon) -> CellBasis:
        raise NotImplementedError


class AssemblerSource(BlockSource):
    """Production source: proxy-surface bases, compression.hpp:106-123."""

    def __init__(self, assembler: BlockAssembler, proxy: ProxyConfig = None):
        self._asm = assembler
        self._proxy = proxy or ProxyConfig()
        # the assembler's native problem (geometry, series tables on the device)
        # already carries the default proxy settings: share it when they match
        if self._proxy == ProxyConfig():
            self._h = assembler._h
        else:
            self._h = _Handle(assembler.mesh(), assembler.medium(), assembler.alpha(),
                              assembler.config(), self._proxy)

    def n_nodes(self): return self._asm.n_nodes()
    def assembler(self): return self._asm
    def proxy(self): return self._proxy

    def block(self, rows, cols):
        return self._h.true_block(rows, cols)

    def cell_basis(self, rows, cols, node_begin, node_end, epsilon) -> CellBasis:
        L = lib()
        r0, r1 = _ints(rows[0]), _ints(rows[1])
        c0, c1 = _ints(cols[0]), _ints(cols[1])
        k, sat = ctypes.c_int(), ctypes.c_int()
        args = (self._h.h, _p(r0), r0.size, _p(r1), r1.size, _p(c0), c0.size,
                _p(c1), c1.size, int(node_begin), int(node_end),
                ctypes.c_double(epsilon), ctypes.byref(k), ctypes.byref(sat))
        _check(L.ebem_gpu_cell_basis(*args, None, None, None, None, None))
        kk = k.value
        skel = np.zeros(max(4 * kk, 1), dtype=np.int32)
        bufs = [np.zeros(2 * max(s * kk, 1)) for s in (r0.size, r1.size, c0.size, c1.size)]
        _check(L.ebem_gpu_cell_basis(*args, _p(skel), *[_p(b) for b in bufs]))
        s = skel[: 4 * kk].reshape(4, kk)
        return CellBasis(
            k=kk, saturated=bool(sat.value),
            row_skeleton=(s[0].copy(), s[1].copy()),
            col_skeleton=(s[2].copy(), s[3].copy()),
            u=(_from_cbuf(bufs[0][: 2 * r0.size * kk], r0.size, kk),
               _from_cbuf(bufs[1][: 2 * r1.size * kk], r1.size, kk)),
            v=(_from_cbuf(bufs[2][: 2 * kk * c0.size], kk, c0.size),
               _from_cbuf(bufs[3][: 2 * kk * c1.size], kk, c1.size)))

    def cell_bases(self, begins, ends, epsilon, skeletons=False):
        """Batched cell_basis over contiguous cells (one device pass);
        returns (ranks, device seconds) or, with skeletons=True,
        (ranks, device seconds, [(row0, row1, col0, col1) per cell])."""
        b = _ints(begins)
        e = _ints(ends)
        k = np.zeros(b.size, dtype=np.int32)
        t = ctypes.c_double()
        sk = np.zeros(max(4 * int((e - b).sum()), 1), np.int32) if skeletons else None
        _check(lib().ebem_gpu_cell_bases(self._h.h, b.size, _p(b), _p(e),
                                         ctypes.c_double(epsilon), _p(k), _p(sk),
                                         ctypes.byref(t)))
        if not skeletons:
            return k, float(t.value)
        out, o = [], 0
        for kk in k.tolist():
            out.append(tuple(sk[o + q * kk: o + (q + 1) * kk].copy() for q in range(4)))
            o += 4 * kk
        return k, float(t.value), out

    def interaction_matrices(self, rows, cols, node_begin, node_end):
        """(M_V, M_U) of cell_basis (compression.cpp:139-166), for tests."""
        L = lib()
        r0, r1 = _ints(rows[0]), _ints(rows[1])
        c0, c1 = _ints(cols[0]), _ints(cols[1])
        no = ctypes.c_int()
        args = (self._h.h, _p(r0), r0.size, _p(r1), r1.size, _p(c0), c0.size,
                _p(c1), c1.size, int(node_begin), int(node_end), ctypes.byref(no))
        _check(L.ebem_gpu_cell_mats(*args, None, None))
        n_out = no.value
        nr, nc = r0.size + r1.size, c0.size + c1.size
        mv = np.zeros(2 * n_out * nc)
        mu = np.zeros(2 * nr * n_out)
        _check(L.ebem_gpu_cell_mats(*args, _p(mv), _p(mu)))
        return _from_cbuf(mv, n_out, nc), _from_cbuf(mu, nr, n_out)

    def build_proxy(self, node_begin, node_end):
        o3 = np.zeros(3)
        ne = ctypes.c_int()
        L = lib()
        _check(L.ebem_gpu_build_proxy(self._h.h, int(node_begin), int(node_end),
                                      _p(o3), ctypes.byref(ne), None, 0))
        enc = np.zeros(max(ne.value, 1), dtype=np.int32)
        _check(L.ebem_gpu_build_proxy(self._h.h, int(node_begin), int(node_end),
                                      _p(o3), ctypes.byref(ne), _p(enc), enc.size))
        return (o3[0], o3[1]), o3[2], enc[: ne.value]

    def eval_scalars(self, r, which=0):
        r = np.ascontiguousarray(r, dtype=np.float64).ravel()
        out = np.zeros(20 * r.size)
        _check(lib().ebem_gpu_eval_scalars(self._h.h, _p(r), r.size, int(which), _p(out)))
        return out.view(np.complex128).reshape(-1, 10)


_IP = ctypes.POINTER(ctypes.c_int)
_DP = ctypes.POINTER(ctypes.c_double)
_BLOCK_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, _IP, ctypes.c_int, _IP,
                             ctypes.c_int, _IP, ctypes.c_int, _IP, ctypes.c_int, _DP)
_BASIS_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, _IP, ctypes.c_int, _IP,
                             ctypes.c_int, _IP, ctypes.c_int, _IP, ctypes.c_int,
                             ctypes.c_int, ctypes.c_int, ctypes.c_double, _IP, _IP, _IP,
                             _DP, _DP, _DP, _DP)


def _ilist(p, n):
    return np.ctypeslib.as_array(p, (n,)).copy() if n > 0 else np.zeros(0, np.int32)


def _host_callbacks(source: BlockSource, errors: list):
    """ctypes trampolines exposing a Python BlockSource to the device solver."""

    def block(_, r0, nr0, r1, nr1, c0, nc0, c1, nc1, out):
        try:
            rows = (_ilist(r0, nr0), _ilist(r1, nr1))
            cols = (_ilist(c0, nc0), _ilist(c1, nc1))
            a = np.asarray(source.block(rows, cols), dtype=np.complex128)
            nr, nc = nr0 + nr1, nc0 + nc1
            if a.shape != (nr, nc):
                raise InvalidArgument(f"BlockSource::block returned {a.shape}, need {(nr, nc)}")
            if nr and nc:
                np.ctypeslib.as_array(out, (2 * nr * nc,))[:] = _to_cbuf(a, nr, nc)
            return 0
        except Exception as e:  # noqa: BLE001
            errors.append(e)
            return 1 if isinstance(e, ValueError) else 2

    def basis(_, r0, nr0, r1, nr1, c0, nc0, c1, nc1, b, e, eps, k, sat, skel, u0, u1,
              v0, v1):
        try:
            rows = (_ilist(r0, nr0), _ilist(r1, nr1))
            cols = (_ilist(c0, nc0), _ilist(c1, nc1))
            cb = source.cell_basis(rows, cols, b, e, eps)
            kk = int(cb.k)
            k[0] = kk
            sat[0] = 1 if cb.saturated else 0
            if kk:
                sk = np.concatenate([np.asarray(cb.row_skeleton[0]), np.asarray(cb.row_skeleton[1]),
                                     np.asarray(cb.col_skeleton[0]), np.asarray(cb.col_skeleton[1])])
                np.ctypeslib.as_array(skel, (4 * kk,))[:] = sk.astype(np.int32)
                for ptr, m, (r_, c_) in ((u0, cb.u[0], (nr0, kk)), (u1, cb.u[1], (nr1, kk)),
                                         (v0, cb.v[0], (kk, nc0)), (v1, cb.v[1], (kk, nc1))):
                    np.ctypeslib.as_array(ptr, (2 * r_ * c_,))[:] = _to_cbuf(m, r_, c_)
            return 0
        except Exception as ex:  # noqa: BLE001
            errors.append(ex)
            return 1 if isinstance(ex, ValueError) else 2

    return _BLOCK_FN(block), _BASIS_FN(basis)


@dataclass
class FieldSample:
    """FieldSample, postprocess.hpp:13-18."""
    location: tuple
    displacement: tuple  # (u1, u2) complex
    intensity: float


def circle_probes(radius: float, count: int, center=(0.0, 0.0)) -> np.ndarray:
    """Evenly spaced points on a circle (postprocess.cpp:46-54)."""
    if radius <= 0.0 or count <= 0:
        raise InvalidArgument("circle_probes: radius and count must be positive")
    phi = 2.0 * math.pi * np.arange(count) / count
    return np.stack([center[0] + radius * np.cos(phi), center[1] + radius * np.sin(phi)], 1)


def _field(mesh, medium, u, points, n_gauss, kind, angle, amplitude, assembler):
    u = np.asarray(u, dtype=np.complex128).ravel()
    if u.size != 2 * mesh.size():
        raise InvalidArgument("evaluate_scattered: boundary data size")
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 2))
    m = pts.shape[0]
    asm = assembler or BlockAssembler(mesh, medium, medium.default_coupling())
    ub = np.ascontiguousarray(u).view(np.float64)
    out = np.zeros(4 * max(m, 1))
    inten = np.zeros(max(m, 1))
    _check(lib().ebem_gpu_field(asm._h.h, _p(ub), _p(pts.ravel()), m, int(n_gauss), int(kind),
                                ctypes.c_double(angle), ctypes.c_double(amplitude), _p(out),
                                _p(inten)))
    return pts, out[: 4 * m].view(np.complex128).reshape(m, 2), inten[:m]


def evaluate_scattered(mesh: Mesh, medium: Medium, boundary_u, points, n_gauss: int = 8,
                       assembler: "BlockAssembler" = None) -> np.ndarray:
    """Scattered displacement at points off the boundary (postprocess.cpp:56-97):
    (m, 2) complex.  Pass an existing assembler to reuse its device geometry."""
    return _field(mesh, medium, boundary_u, points, n_gauss, -1, 0.0, 0.0, assembler)[1]


def evaluate_field(mesh: Mesh, medium: Medium, wave, boundary_u, points, n_gauss: int = 8,
                   assembler: "BlockAssembler" = None):
    """Total field (incident plane wave + scattered) with intensities
    (postprocess.cpp:99-119); PlaneSVWave also accepted."""
    pts, u, inten = _field(mesh, medium, boundary_u, points, n_gauss, wave.kind,
                           wave.angle, wave.amplitude, assembler)
    return [FieldSample((float(p[0]), float(p[1])), (complex(v[0]), complex(v[1])), float(i))
            for p, v, i in zip(pts, u, inten)]


class ConvSolver:
    """Dense reference solver, dense_solver.hpp:21-45: full Galerkin matrix
    and one partial-pivoted LU on the device."""

    def __init__(self, mesh: Mesh, medium: Medium, alpha: complex,
                 config: AssemblyConfig = None):
        self._asm = BlockAssembler(mesh, medium, alpha, config)
        st = _ConvStats()
        h = ctypes.c_void_p()
        _check(lib().ebem_gpu_conv_create(self._asm._h.h, ctypes.byref(h), ctypes.byref(st)))
        self._c = h
        self._stats = ConvStats(st.assemble_seconds, st.factor_seconds, st.rcond,
                                st.min_pivot, bool(st.condition_warning))

    def __del__(self):
        if getattr(self, "_c", None) and _lib is not None:
            _lib.ebem_gpu_conv_destroy(self._c)
            self._c = None

    def assembler(self) -> BlockAssembler:
        return self._asm

    def stats(self) -> ConvStats:
        return self._stats

    def size(self) -> int:
        return 2 * self._asm.n_nodes()

    def solve(self, rhs) -> np.ndarray:
        b = np.asarray(rhs, dtype=np.complex128)
        vec = b.ndim == 1
        b2 = b.reshape(-1, 1) if vec else b
        if b2.shape[0] != self.size():
            raise InvalidArgument(f"LuFactor: right-hand side has {b2.shape[0]} rows, "
                                  f"need {self.size()}")
        m = b2.shape[1]
        buf = np.asfortranarray(b2).ravel(order="F").view(np.float64).copy()
        out = np.zeros_like(buf)
        _check(lib().ebem_gpu_conv_solve(self._c, _p(buf), m, _p(out)))
        x = out.view(np.complex128).reshape(m, self.size()).T
        return x[:, 0].copy() if vec else np.ascontiguousarray(x)


class FdsSolver:
    """Hierarchical direct solver, fds.hpp:44-94.  Construction factorizes.

    AssemblerSource runs entirely on the device.  Any other BlockSource (the
    reference tests' MatrixSource / DirectSource fakes) supplies entries and
    bases through host callbacks; the merges and solves still run on the
    device."""

    def __init__(self, source: BlockSource, tree: ClusterTree,
                 config: FdsConfig = None):
        self._source, self._tree = source, tree
        self._config = config or FdsConfig()
        if tree.n_nodes() != source.n_nodes():
            raise InvalidArgument("FdsSolver: tree and source node counts differ")
        cfg = _FdsCfg(self._config.epsilon, self._config.ell0)
        st = _FdsStats()
        h = ctypes.c_void_p()
        if isinstance(source, AssemblerSource):
            _check(lib().ebem_gpu_fds_create(source._h.h, tree.depth(), ctypes.byref(cfg),
                                             ctypes.byref(h), ctypes.byref(st)))
        else:
            self._errors = []
            self._cbs = _host_callbacks(source, self._errors)
            rc = lib().ebem_gpu_fds_create_source(tree.n_nodes(), tree.depth(),
                                                  ctypes.byref(cfg), self._cbs[0],
                                                  self._cbs[1], None, ctypes.byref(h),
                                                  ctypes.byref(st))
            if rc != 0 and self._errors:
                raise self._errors[0]
            _check(rc)
        self._h = h
        self._stats = FdsStats(
            max_rank=list(st.max_rank)[: tree.depth() + 1], top_dim=st.top_dim,
            saturated=bool(st.saturated), upward_seconds=st.upward_seconds,
            top_factor_seconds=st.top_factor_seconds,
            basis_cpu_seconds=st.basis_cpu_seconds,
            factorize_device_seconds=st.factorize_device_seconds)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ebem_gpu_fds_destroy(self._h)
            self._h = None

    def solve(self, rhs, timing: Optional[FdsSolveTiming] = None) -> np.ndarray:
        n = self._tree.n_nodes()
        rhs = np.asarray(rhs, dtype=np.complex128)
        vec = rhs.ndim == 1
        if rhs.shape[0] != 2 * n:
            raise InvalidArgument(
                f"FdsSolver: right-hand side has {rhs.shape[0]} rows, need {2 * n}")
        b = rhs.reshape(2 * n, -1)
        m = b.shape[1]
        buf = _to_cbuf(b, 2 * n, m)
        t = _SolveTiming()
        _check(lib().ebem_gpu_fds_solve(self._h, _p(buf), m, _p(buf), ctypes.byref(t)))
        if timing is not None:
            timing.upward_seconds = t.upward_seconds
            timing.top_seconds = t.top_seconds
            timing.downward_seconds = t.downward_seconds
            timing.device_seconds = t.device_seconds
        x = _from_cbuf(buf, 2 * n, m)
        return x[:, 0] if vec else x

    def stats(self) -> FdsStats:
        return self._stats

    def tree(self) -> ClusterTree:
        return self._tree

    def rank_of(self, cell: int) -> int:
        return int(lib().ebem_gpu_fds_rank_of(self._h, int(cell)))

    def cell(self, cell: int):
        """Sequences' sizes and skeletons of one cell (introspection)."""
        sizes = np.zeros(5, dtype=np.int32)
        _check(lib().ebem_gpu_fds_cell(self._h, int(cell), _p(sizes), None))
        k = int(sizes[4])
        skel = np.zeros(max(4 * k, 1), dtype=np.int32)
        _check(lib().ebem_gpu_fds_cell(self._h, int(cell), _p(sizes), _p(skel)))
        s = skel[: 4 * k].reshape(4, k)
        return dict(sizes=sizes.tolist(), k=k, row_skeleton=(s[0], s[1]),
                    col_skeleton=(s[2], s[3]))

    @property
    def handle(self):
        return self._h


# ------------------------------------------------------------- measurement


def prof_enable(on: bool = True) -> None:
    """Per-kernel CUDA-event timing on the launching stream (bench hooks)."""
    _check(lib().ebem_gpu_prof_enable(1 if on else 0))


def prof_read(reset: bool = False) -> dict:
    """{kernel: (milliseconds, launches, work units, algorithmic HBM bytes)}
    since the last reset."""
    L = lib()
    L.ebem_gpu_prof_name.restype = ctypes.c_char_p
    n = L.ebem_gpu_prof_kernels()
    ms = np.zeros(n)
    cnt = np.zeros(n, dtype=np.int64)
    units = np.zeros(n)
    byts = np.zeros(n)
    _check(L.ebem_gpu_prof_bytes(_p(byts), n))
    _check(L.ebem_gpu_prof_read(1 if reset else 0, _p(ms), _p(cnt), _p(units), n))
    return {L.ebem_gpu_prof_name(i).decode(): (float(ms[i]), int(cnt[i]), float(units[i]),
                                                float(byts[i]))
            for i in range(n)}


def fp64_peak_tflops() -> float:
    """Measured FP64 FMA throughput (DFMA chains on every SM)."""
    v = ctypes.c_double()
    _check(lib().ebem_gpu_fp64_peak(ctypes.byref(v)))
    return float(v.value)
