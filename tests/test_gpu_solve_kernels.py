"""LU-solve kernel variants through the dense solver (ConvSolver::solve =
LuFactor::solve, proj/src/lapack.cpp:73-89): the batched solve dispatches on
the order n = 2N and the right-hand-side count m to the one-warp-per-column
kernel (n <= 128, m <= 8), the CTA-per-column kernel (larger n, few m), the
blocked panel kernel (n >= 96, m >= 16) and the staged register kernel, each
checked against a numpy solve of the same dense matrix.  GPU."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("n_nodes,m", [
    (24, 1), (24, 3),      # n = 48: one warp per column
    (24, 20),              # n = 48, many columns: staged register kernel
    (100, 1), (100, 5),    # n = 200: one CTA per column
    (100, 16), (100, 37),  # n = 200: blocked panels (full and ragged column tiles)
    (60, 33),              # n = 120: blocked panels, order not a multiple of 32
    (65, 1), (128, 2),     # n = 130, 256: column blocks of 16 (ragged / exact last block)
    (129, 1), (250, 3),    # n = 258, 500: two rows per thread, column blocks of 8
    (200, 2),              # n = 400: CTA per column, two rows per thread
    (200, 20),             # n = 400: blocked panels, eight rows per lane group
    (700, 1),              # n = 1400: CTA per column, eight rows per thread
])
def test_lu_solve_variants_match_numpy(eb, n_nodes, m):
    mesh = eb.Mesh.star(n_nodes, eb.StarShape(1.0, 0.0, 3))
    med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
    conv = eb.ConvSolver(mesh, med, med.default_coupling())
    a = conv.assembler().dense()
    rng = np.random.default_rng(n_nodes * 100 + m)
    f = rng.standard_normal((2 * n_nodes, m)) + 1j * rng.standard_normal((2 * n_nodes, m))
    x = conv.solve(f)
    xr = np.linalg.solve(a, f)
    assert rel(x, xr) < 1e-10
    assert rel(a @ x, f) < 1e-12
