"""The oracles themselves, pinned before they are trusted (CPU only).

* the reference compiled in place (oracle/_ref) against the reference's own
  golden vectors (proj/tests/reference_values.hpp via tests/golden/);
* the numpy restatement (oracle/ebem_oracle.py) against the same golden
  vectors and against the compiled reference on small cases.
Tolerances are the reference's own (proj/tests/test_hankel.cpp:22-29,
proj/tests/test_kernels.cpp:75-157)."""
import math

import numpy as np
import pytest

import ebem_oracle as eo

GOLD_MED = eo.Medium(1.0, 1.0, 1.0, 2.0)


def cplx(v, k):
    return complex(v[2 * k], v[2 * k + 1])


def test_ref_hankel_golden(ref, golden):
    for h in golden["hankel"]:
        h0, h1 = ref.hankel([h["x"]])
        assert abs(h0[0] - complex(h["h0r"], h["h0i"])) <= 5e-15 * abs(h0[0])
        assert abs(h1[0] - complex(h["h1r"], h["h1i"])) <= 5e-15 * abs(h1[0])


def test_oracle_hankel_golden(golden):
    for h in golden["hankel"]:
        h0, h1 = eo.hankel01(h["x"])
        assert abs(h0 - complex(h["h0r"], h["h0i"])) <= 5e-15 * abs(h0)
        assert abs(h1 - complex(h["h1r"], h["h1i"])) <= 5e-15 * abs(h1)


@pytest.mark.parametrize("which", ["full", "rem", "stat"])
def test_scalars_golden_ref_and_oracle(ref, golden, which):
    S = eo.Scalars(GOLD_MED)
    kT = GOLD_MED.kT
    for sv in golden["scalars"]:
        r = sv["r"]
        o = {"full": S.full, "rem": S.remainder, "stat": S.static}[which](np.array([r]))[0]
        g = ref.scalars(1.0, 1.0, 1.0, 2.0, [r], {"full": 0, "rem": 1, "stat": 2}[which])[0]
        for k in range(10):
            if which == "stat":
                want = sv["stat"][k]
                scale = max(abs(v) for v in sv["stat"])
                tol = 1e-13 * max(scale * 1e-10, abs(want))
            elif which == "full":
                want = cplx(sv["full"], k)
                tol = max(5e-12, 1e-14 / (kT * r) ** 2) * abs(want)
            else:
                want = cplx(sv["rem"], k)
                tol = 1e-12 * (abs(want) + 5e-2 * abs(cplx(sv["full"], k))) + 1e-25
            # the restatement's remainder above the switch is full - static from
            # scipy's H0/H1; it concedes ~4x the reference's cancellation margin
            otol = 4 * tol if which == "rem" else tol
            assert abs(o[k] - want) <= otol, (which, r, k, "oracle")
            assert abs(g[k] - want) <= tol, (which, r, k, "reference")


def test_oracle_kernel_matrices_golden(golden):
    S = eo.Scalars(GOLD_MED)
    for kv in golden["kernels"]:
        z, m, n = np.array(kv["z"]), np.array(kv["m"]), np.array(kv["n"])
        r = math.hypot(*z)
        zh = z / r
        s = S.full(np.array([r]))[0]
        D = eo.combine_D(s, zh, n)
        N = eo.combine_N(s, zh, m, n)
        wD = np.array(kv["D"]).view(complex).reshape(2, 2)
        wN = np.array(kv["N"]).view(complex).reshape(2, 2)
        tol = max(1e-12, 1e-14 / (GOLD_MED.kT * r) ** 2)
        assert np.max(np.abs(D - wD)) <= tol * np.max(np.abs(wD))
        assert np.max(np.abs(N - wN)) <= tol * np.max(np.abs(wN))


def test_oracle_incident_golden(golden):
    med = GOLD_MED
    for iv in golden["incident"]:
        d, x, n = np.array(iv["d"]), np.array(iv["x"]), np.array(iv["n"])
        ph = np.exp(-1j * med.kL * (d @ x))
        u = ph * d
        t = -1j * med.kL * ph * (med.lam * n + 2 * med.mu * (n @ d) * d)
        wu = np.array(iv["u"]).view(complex)
        wt = np.array(iv["t"]).view(complex)
        assert np.max(np.abs(u - wu)) < 1e-14
        assert np.max(np.abs(t - wt)) < 1e-14 * np.max(np.abs(wt))


def test_oracle_log_galerkin_golden(golden):
    # sum of the log-Galerkin table is -3/2 (coincident static N, assembly.cpp:118-123)
    assert abs(np.sum(golden["log_galerkin"]) + 1.5) < 1e-15


def _small_problem(ref, n=128, omega=1.0):
    xy = eo.circle_nodes(n)
    med = eo.Medium(1.0, 1.0, 1.0, omega)
    return eo.Problem(xy, med), ref.problem(xy, 1.0, 1.0, 1.0, omega, med.default_coupling())


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_oracle_true_block_vs_reference(ref):
    p, rp = _small_problem(ref, 96)
    leaf = list(range(24))
    assert rel(p.block([leaf, leaf], [leaf, leaf]), rp.true_block((leaf, leaf), (leaf, leaf))) < 1e-12
    rows = ([95, 0, 1, 40, 41], [2, 3, 60])
    cols = ([94, 95, 0, 10], [1, 50, 51, 52])
    assert rel(p.block(rows, cols), rp.true_block(rows, cols)) < 1e-11


def test_oracle_cell_mats_and_basis_vs_reference(ref):
    p, rp = _small_problem(ref, 128)
    leaf = list(range(32, 64))
    mv, mu = p.cell_mats([leaf, leaf], [leaf, leaf], 32, 64)
    rmv, rmu = rp.cell_mats((leaf, leaf), (leaf, leaf), 32, 64)
    assert mv.shape == rmv.shape and mu.shape == rmu.shape
    assert rel(mv, rmv) < 1e-12 and rel(mu, rmu) < 1e-12
    b = eo.basis_from_interactions(rmv, rmu, [leaf, leaf], [leaf, leaf], 1e-10)
    rb = rp.cell_basis((leaf, leaf), (leaf, leaf), 32, 64, 1e-10)
    assert b.k == rb["k"]
    for q in range(2):
        assert np.array_equal(b.col_skeleton[q], rb["col_skeleton"][q])
        assert np.array_equal(b.row_skeleton[q], rb["row_skeleton"][q])


def test_oracle_cpqr_pivots_match_lapack(ref):
    rng = np.random.default_rng(7)
    for m, n in [(40, 12), (164, 32), (30, 30)]:
        a = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
        R, jp = eo.cpqr(a)
        rjp, rd, _, _ = ref.cpqr(a)
        assert np.array_equal(jp[: len(rjp)], rjp)
        assert np.allclose(np.abs(np.diag(R)), rd, rtol=1e-12)
    # rank one -> k = 1; zero -> k = 0 (proj/tests/test_dense_solver.cpp:99-120)
    u = rng.standard_normal((20, 1)) + 0j
    R, _ = eo.cpqr(u @ u.T[:, :8].conj())
    assert eo.eps_rank(R, 1e-10) == 1
    R, _ = eo.cpqr(np.zeros((6, 4), complex))
    assert eo.eps_rank(R, 1e-10) == 0


def test_oracle_rhs_vs_reference(ref):
    p, rp = _small_problem(ref, 64, omega=2.0)
    for ang in (0.0, 1.1):
        assert rel(p.rhs([ang])[:, 0], rp.rhs_plane_p([ang])[:, 0]) < 1e-13


def test_oracle_fds_vs_reference(ref):
    p, rp = _small_problem(ref, 128)
    f = rp.rhs_plane_p([0.0])
    F = eo.Fds(p, 2, 1e-10, 1)
    rF = rp.fds(2, 1e-10, 1)
    x = F.solve(f)
    xr, _ = rF.solve(f)
    assert rel(x, xr) < 1e-10
    assert F.max_rank == rF.stats["max_rank"]
