"""Compare one leaf cell's device merge factors with numpy on reference data
(development aid)."""
import ctypes
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
os.environ["EBEM_DEBUG_NOTHROW"] = "1"
import paper_2411_18026_b200 as eb  # noqa: E402
from _oracles import RefLib  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def get(fds, cell, which, shape, dtype=np.complex128):
    L = eb.lib()
    if dtype == np.int32:
        out = np.zeros(shape[0], dtype=np.int32)
    else:
        out = np.zeros(2 * shape[0] * shape[1])
    rc = L.ebem_gpu_fds_debug_cell(fds.handle, cell, which, out.ctypes.data_as(ctypes.c_void_p))
    assert rc == 0, L.ebem_gpu_last_error()
    if dtype == np.int32:
        return out
    return out.view(np.complex128).reshape(shape[1], shape[0]).T


N = 1024
mesh = eb.Mesh.star(N, eb.StarShape(1.0, 0.0, 3))
med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
alpha = med.default_coupling()
asm = eb.BlockAssembler(mesh, med, alpha)
src = eb.AssemblerSource(asm, eb.ProxyConfig())
tree = eb.ClusterTree(N, 5)
fds = eb.FdsSolver(src, tree, eb.FdsConfig(1e-10, 1))
cell = 31
k = fds.rank_of(cell)
n = 32
leaf = list(range(32))
A = asm.true_block((leaf, leaf), (leaf, leaf))
b = src.cell_basis((leaf, leaf), (leaf, leaf), 0, 32, 1e-10)
U = np.zeros((64, 2 * k), complex)
U[:32, :k] = b.u[0]
U[32:, k:] = b.u[1]
AU = np.linalg.solve(A, U)
W = np.vstack([b.v[0] @ AU[:32], b.v[1] @ AU[32:]])
print("k", k, "cond W", np.linalg.cond(W))
lu = get(fds, cell, 0, (64, 64))
piv = get(fds, cell, 1, (64,), np.int32)
# reconstruct A from LU
L = np.tril(lu, -1) + np.eye(64)
Um = np.triu(lu)
PA = L @ Um
Ar = A.copy()
for i, p in enumerate(piv):
    Ar[[i, p]] = Ar[[p, i]]
print("LU reconstruct rel", rel(PA, Ar))
au = get(fds, cell, 2, (64, 2 * k))
print("ainv_u rel", rel(au, AU))
v = get(fds, cell, 3, (k, 2 * n))
print("v0 rel", rel(v[:, :32], b.v[0]), "v1 rel", rel(v[:, 32:], b.v[1]))
at = get(fds, cell, 4, (2 * k, 2 * k))
print("atilde rel", rel(at, np.linalg.inv(W)))
