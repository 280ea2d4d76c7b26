"""The ID's TSQR stage (reduction of the tall interaction matrices before the
column-pivoted QR, proj/src/lapack.cpp:101-119) through the C ABI: the
reduced block has the input's Gram matrix (hence its column norms and zlaqp2
pivot sequence), is upper triangular, and matches LAPACK's |R_ii|.  GPU."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def tall_reduce(eb, a):
    a = np.asfortranarray(a, dtype=np.complex128)
    rows, n = a.shape
    out = np.zeros(2 * rows * n)
    rr = ctypes.c_int()
    buf = a.ravel(order="F").view(np.float64)
    rc = eb.lib().ebem_gpu_tall_reduce(buf.ctypes.data_as(ctypes.c_void_p), rows, n, rows,
                                       out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(rr))
    assert rc == 0, eb.lib().ebem_gpu_last_error()
    m = rr.value
    c = out[: 2 * m * n].reshape(n, m, 2)
    return (c[..., 0] + 1j * c[..., 1]).T


def check(eb, a, tol=1e-12, diag=True):
    r = tall_reduce(eb, a)
    n = a.shape[1]
    assert np.all(np.isfinite(r))
    g = a.conj().T @ a
    scale = np.linalg.norm(g)
    assert np.linalg.norm(r.conj().T @ r - g) <= tol * scale
    if r.shape[0] == n < a.shape[0]:
        assert np.all(r[np.tril_indices(n, -1)] == 0)
    if r.shape[0] == n < a.shape[0] and diag:  # |R_ii| is unique while R stays nonsingular
        ref = np.linalg.qr(a, mode="r")
        d, dr = np.abs(np.diag(r)), np.abs(np.diag(ref))
        big = dr > 1e-8 * dr.max()
        assert np.allclose(d[big], dr[big], rtol=1e-9)
    return r


@pytest.mark.parametrize("rows,n", [(3000, 94), (20000, 94), (5000, 40), (700, 128),
                                    (129, 128), (1000, 1), (64, 64), (4100, 65),
                                    (100000, 122), (333, 17)])
def test_random_blocks(eb, rows, n):
    rng = np.random.default_rng(rows * 1000 + n)
    a = rng.standard_normal((rows, n)) + 1j * rng.standard_normal((rows, n))
    r = check(eb, a)
    if rows > n:
        assert r.shape == (n, n)
    else:  # nothing to reduce: the block comes back unchanged
        assert np.array_equal(r, a)


def test_rank_deficient_and_zero_columns(eb):
    rng = np.random.default_rng(7)
    rows, n, k = 6000, 94, 10
    a = (rng.standard_normal((rows, k)) + 1j * rng.standard_normal((rows, k))) @ \
        (rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n)))
    a[:, 5] = 0.0
    a[:, 40] = 0.0
    r = check(eb, a, diag=False)
    assert np.abs(r[k + 1:, :]).max() <= 1e-12 * np.abs(r).max()
    assert np.all(r[:, 5] == 0) and np.all(r[:, 40] == 0)


def test_stacked_triangles_with_geometric_residues(eb):
    # stacked R factors cut mid-triangle: the eliminated rows' residues shrink
    # geometrically (down to |x|^2 underflow) -- the case Smith's division covers
    rng = np.random.default_rng(1)
    n = 94
    tri = [np.linalg.qr(rng.standard_normal((200, n)) + 1j * rng.standard_normal((200, n)),
                        mode="r") for _ in range(30)]
    s = np.vstack(tri)
    for r0, rows in ((417, 417), (41, 2459), (0, 2820)):
        check(eb, s[r0:r0 + rows], diag=False)


def test_graded_columns_like_interaction_matrices(eb):
    # singular values decaying to 1e-16 relative, as the proxy interactions
    rng = np.random.default_rng(11)
    rows, n = 12000, 110
    q1, _ = np.linalg.qr(rng.standard_normal((rows, n)) + 1j * rng.standard_normal((rows, n)))
    q2, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    s = np.logspace(0, -16, n)
    a = (q1 * s) @ q2
    check(eb, a, tol=1e-12)


def test_real_and_pure_imaginary_leading_entries(eb):
    # zlarfg's H = I branch (x = 0, alpha real) and alpha = i * t
    rows, n = 4096, 70
    a = np.zeros((rows, n), complex)
    a[0, :] = 1.0 + 0j
    a[1, 3:] = 1j
    a[rows - 1, 10:] = -2.0
    check(eb, a, diag=False)
