"""Host tables of libebem_gpu.so (medium_setup.cpp) against the reference
compiled in place -- no device needed.

* The remainder expansion of the ten kernel scalars, derived in
  medium_setup.cpp from the ascending Hankel expansion and closed-form
  derivative coefficients, evaluated below the series radius vs
  KernelScalars::remainder (proj/src/kernel_scalars.cpp:381-409) and its
  integrated form vs KernelScalars::integrated_remainder (:353-379).
* Gauss-Legendre rules (Jacobi-matrix eigenvalues + Christoffel weights) vs
  gauss_rule (proj/src/quadrature.cpp:16-56).
"""
import ctypes

import numpy as np
import pytest

MAXP = 48
MEDIA = [(1.0, 1.0, 1.0, 1.0), (1.0, 1.0, 1.0, 2.0), (1.0, 1.0, 1.0, 4.0),
         (1.0, 1.0, 1.0, 8.0), (1.5, 1.0, 1.0, 16.0 / 1.3), (2.0, 0.5, 1.3, 3.0)]


def series(eb, med):
    out = np.zeros(10 * MAXP * 4)
    mq = ctypes.c_int()
    rc = eb.lib().ebem_gpu_series_table(*[ctypes.c_double(v) for v in med],
                                        out.ctypes.data_as(ctypes.c_void_p), MAXP,
                                        ctypes.byref(mq))
    assert rc == 0
    t = out.reshape(10, MAXP, 4)
    return t[..., 0] + 1j * t[..., 1], t[..., 2] + 1j * t[..., 3], mq.value


def eval_series(a, b, r):
    q = np.arange(MAXP)
    rp = r[:, None] ** q[None, :]
    lr = np.log(r)[:, None]
    return np.stack([((a[k][None, :] + b[k][None, :] * lr) * rp).sum(1) for k in range(10)], 1)


@pytest.mark.parametrize("med", MEDIA)
def test_remainder_expansion_vs_reference(eb, ref, med):
    a, b, mq = series(eb, med)
    assert 0 < mq < MAXP
    kT = med[3] / np.sqrt(med[1] / med[2])
    r = np.geomspace(1e-6, 0.999 * 0.25 / kT, 40)
    got = eval_series(a, b, r)
    want = ref.scalars(*med, r, which=1)
    scale = np.abs(want).max(axis=0) + 1e-300
    assert np.max(np.abs(got - want) / scale) < 1e-13


@pytest.mark.parametrize("med", MEDIA)
def test_integrated_remainder_vs_reference(eb, ref, med):
    a, b, _ = series(eb, med)
    kT = med[3] / np.sqrt(med[1] / med[2])
    q = np.arange(MAXP)
    for c in (1e-4, 0.03 / kT, 0.8 / kT, 2.4 / kT):
        for j in (0, 1, 2):
            inv = 1.0 / (q + j + 1)
            got = ((c ** q) * ((a + b * np.log(c)) * inv - b * inv ** 2)).sum(1)
            want = ref.integrated_remainder(*med, c, j)
            assert np.max(np.abs(got - want)) <= 1e-13 * np.abs(want).max()


def test_expansion_has_single_parity_and_no_singular_power(eb):
    for med in MEDIA:
        a, b, _ = series(eb, med)
        for k in range(10):
            nz = np.nonzero((a[k] != 0) | (b[k] != 0))[0]
            assert nz.size and np.all(nz % 2 == nz[0] % 2)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 6, 8, 9, 10, 13, 20, 40, 64])
def test_gauss_rule_vs_reference(eb, ref, n):
    x = np.zeros(n)
    w = np.zeros(n)
    assert eb.lib().ebem_gpu_gauss_rule(n, x.ctypes.data_as(ctypes.c_void_p),
                                        w.ctypes.data_as(ctypes.c_void_p)) == 0
    xr, wr = ref.gauss_rule(n)
    assert np.max(np.abs(x - xr)) < 4e-16
    # the reference's Newton weights carry up to ~9e-14 relative error at the
    # ends (vs 40-digit mpmath); the Christoffel weights here ~1e-15
    assert np.max(np.abs(w - wr) / wr) < 2e-13
    # exact for polynomials of degree 2n - 1
    for d in range(2 * n):
        assert abs(np.dot(w, x ** d) - 1.0 / (d + 1)) < 1e-14
