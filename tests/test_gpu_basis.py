"""Cell bases (proxy ID) on the device vs the reference: ranks, skeleton
index sets, coefficients and the low-rank consistency property.  GPU."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(eb, ref, n, omega=1.0, shape=None, m_prime=64):
    mesh = eb.Mesh.star(n, shape or eb.StarShape(1.0, 0.0, 3))
    med = eb.Medium.from_lame(1.0, 1.0, 1.0, omega)
    asm = eb.BlockAssembler(mesh, med, med.default_coupling())
    src = eb.AssemblerSource(asm, eb.ProxyConfig(1.5, m_prime, 6))
    rp = ref.problem(mesh.nodes, 1.0, 1.0, 1.0, omega, med.default_coupling(), m_prime=m_prime)
    return src, rp


@pytest.mark.parametrize("eps", [1e-8, 1e-10])
def test_leaf_basis_matches_reference(eb, ref, eps):
    src, rp = _setup(eb, ref, 1024)
    for b in (0, 480, 992):
        r = list(range(b, b + 32))
        got = src.cell_basis((r, r), (r, r), b, b + 32, eps)
        want = rp.cell_basis((r, r), (r, r), b, b + 32, eps)
        assert got.k == want["k"] and got.saturated == want["saturated"]
        for q in range(2):
            assert np.array_equal(got.col_skeleton[q], want["col_skeleton"][q])
            assert np.array_equal(got.row_skeleton[q], want["row_skeleton"][q])
            # coefficients carry cond(R11) ~ 1/eps of the fill's 1e-14 noise
            assert np.linalg.norm(got.v[q] - want["v"][q]) <= 1e-3 * np.linalg.norm(want["v"][q])
            assert np.linalg.norm(got.u[q] - want["u"][q]) <= 1e-3 * np.linalg.norm(want["u"][q])


def test_basis_identity_on_skeleton_and_low_rank(eb, ref):
    n = 1024
    src, rp = _setup(eb, ref, n)
    r = list(range(64, 96))
    B = src.cell_basis((r, r), (r, r), 64, 96, 1e-10)
    for q in range(2):
        cols = np.searchsorted(r, B.col_skeleton[q])
        assert np.allclose(B.v[q][:, cols], np.eye(B.k), atol=0)
    # far interactions reconstruct to ~ eps (DirectSource-style consistency)
    far = list(range(400, 700))
    a = src.block((far, far), (r, r))
    sk = src.block((far, far), (list(B.col_skeleton[0]), list(B.col_skeleton[1])))
    v = np.zeros((2 * B.k, 64), complex)
    v[:B.k, :32] = B.v[0]
    v[B.k:, 32:] = B.v[1]
    assert np.linalg.norm(a - sk @ v) <= 1e-8 * np.linalg.norm(a)


def test_upper_level_basis_with_skeleton_sequences(eb, ref):
    # A level-3 style call: non-contiguous per-component sequences.
    n = 2048
    src, rp = _setup(eb, ref, n)
    rng = np.random.default_rng(5)
    base = np.arange(256, 512)
    rows = (sorted(rng.choice(base, 48, replace=False)), sorted(rng.choice(base, 48, replace=False)))
    cols = (sorted(rng.choice(base, 48, replace=False)), sorted(rng.choice(base, 48, replace=False)))
    got = src.cell_basis(rows, cols, 256, 512, 1e-10)
    want = rp.cell_basis(rows, cols, 256, 512, 1e-10)
    assert got.k == want["k"]
    for q in range(2):
        assert set(got.col_skeleton[q]) == set(want["col_skeleton"][q])
        assert set(got.row_skeleton[q]) == set(want["row_skeleton"][q])


def test_empty_lists_raise(eb, ref):
    src, _ = _setup(eb, ref, 256)
    with pytest.raises(eb.InvalidArgument):
        src.cell_basis(([], [1, 2]), ([3], [4]), 0, 32, 1e-10)
    with pytest.raises(eb.InvalidArgument):
        src.cell_basis(([1], [2]), ([1], [2]), 0, 32, 0.0)
