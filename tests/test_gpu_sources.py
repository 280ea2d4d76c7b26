"""Any BlockSource through the device solver: the reference's synthetic
FDS tests (proj/tests/test_fds.cpp:36-187) with the MatrixSource and
DirectSource fakes restated in numpy (bases by the restatement oracle's
basis_from_interactions).  The merges and solves run on the device.  GPU."""
import numpy as np
import pytest

import ebem_oracle as eo

pytestmark = pytest.mark.gpu


class MatrixSource:
    """Entries from an explicit component-major matrix (test_fds.cpp:36-67)."""

    def __init__(self, a, n):
        self.a, self.n = a, n

    def n_nodes(self):
        return self.n

    def block(self, rows, cols):
        r = np.concatenate([np.asarray(rows[0]), self.n + np.asarray(rows[1])]).astype(int)
        c = np.concatenate([np.asarray(cols[0]), self.n + np.asarray(cols[1])]).astype(int)
        return self.a[np.ix_(r, c)]


def direct_source(eb, entries):
    """DirectSource (compression.hpp:129-146): bases from the full far field."""

    class Direct(eb.BlockSource):
        def n_nodes(self):
            return entries.n

        def block(self, rows, cols):
            return entries.block(rows, cols)

        def cell_basis(self, rows, cols, b, e, eps):
            others = np.array([g for g in range(entries.n) if g < b or g >= e])
            far = (others, others)
            mv = entries.block(far, cols)
            mu = entries.block(rows, far)
            cb = eo.basis_from_interactions(mv, mu, rows, cols, eps)
            return eb.CellBasis(k=cb.k, saturated=cb.saturated,
                                row_skeleton=tuple(cb.row_skeleton),
                                col_skeleton=tuple(cb.col_skeleton),
                                u=tuple(cb.u), v=tuple(cb.v))

    return Direct()


def rmat(rng, r, c):
    return rng.standard_normal((r, c)) + 1j * rng.standard_normal((r, c))


def synthetic_system(n, n_leaves, ranks, seed):
    """Off-diagonal leaf blocks exactly low rank (test_fds.cpp:80-119)."""
    m = n // n_leaves
    rng = np.random.default_rng(seed)
    a = np.zeros((2 * n, 2 * n), complex)
    uf = [[rmat(rng, m, ranks[i]) for _ in range(2)] for i in range(n_leaves)]
    vf = [[rmat(rng, ranks[i], m) for _ in range(2)] for i in range(n_leaves)]
    for i in range(n_leaves):
        for j in range(n_leaves):
            if i == j or ranks[i] == 0 or ranks[j] == 0:
                continue
            scale = 1.0 / np.sqrt(m * ranks[i] * ranks[j])
            for p in range(2):
                for q in range(2):
                    c = scale * rmat(rng, ranks[i], ranks[j])
                    a[p * n + i * m:p * n + (i + 1) * m, q * n + j * m:q * n + (j + 1) * m] = \
                        uf[i][p] @ c @ vf[j][q]
    for i in range(n_leaves):
        d = rmat(rng, 2 * m, 2 * m) / np.sqrt(2.0 * m) + 8.0 * np.eye(2 * m)
        for p in range(2):
            for q in range(2):
                a[p * n + i * m:p * n + (i + 1) * m, q * n + i * m:q * n + (i + 1) * m] = \
                    d[p * m:(p + 1) * m, q * m:(q + 1) * m]
    return a


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_synthetic_low_rank_exact(eb):
    n, depth, n_leaves = 128, 3, 8
    ranks = [2, 3, 4, 2, 4, 3, 2, 3]
    entries = MatrixSource(synthetic_system(n, n_leaves, ranks, 91), n)
    src = direct_source(eb, entries)
    tree = eb.ClusterTree(n, depth)
    f = rmat(np.random.default_rng(17), 2 * n, 2)
    want = np.linalg.solve(entries.a, f)
    for ell0 in (0, 1, 2):
        fds = eb.FdsSolver(src, tree, eb.FdsConfig(1e-10, ell0))
        assert rel(fds.solve(f), want) <= 1e-11
        for c in range(eb.ClusterTree.first_cell(depth), eb.ClusterTree.last_cell(depth) + 1):
            assert fds.rank_of(c) == ranks[c - eb.ClusterTree.first_cell(depth)]


def test_block_diagonal_zero_ranks(eb):
    n, depth, n_leaves = 64, 2, 4
    entries = MatrixSource(synthetic_system(n, n_leaves, [0] * 4, 7), n)
    src = direct_source(eb, entries)
    tree = eb.ClusterTree(n, depth)
    fds = eb.FdsSolver(src, tree, eb.FdsConfig(1e-10, 1))
    assert fds.stats().top_dim == 0
    for c in range(3, 7):
        assert fds.rank_of(c) == 0
    f = rmat(np.random.default_rng(3), 2 * n, 1)[:, 0]
    assert rel(fds.solve(f), np.linalg.solve(entries.a, f)) <= 1e-12


def test_inconsistent_inputs(eb):
    n = 64
    entries = MatrixSource(synthetic_system(n, 4, [1, 1, 1, 1], 5), n)
    src = direct_source(eb, entries)
    tree = eb.ClusterTree(n, 2)
    with pytest.raises(eb.InvalidArgument):
        eb.FdsSolver(src, tree, eb.FdsConfig(1e-8, 2))
    with pytest.raises(eb.InvalidArgument):
        eb.FdsSolver(src, tree, eb.FdsConfig(1e-8, -1))
    with pytest.raises(eb.InvalidArgument):
        eb.FdsSolver(src, eb.ClusterTree(32, 1), eb.FdsConfig())
    fds = eb.FdsSolver(src, tree, eb.FdsConfig())
    with pytest.raises(eb.InvalidArgument):
        fds.solve(np.zeros(2 * n + 2, complex))


def test_callback_errors_propagate(eb):
    class Broken(eb.BlockSource):
        def n_nodes(self):
            return 64

        def block(self, rows, cols):
            raise RuntimeError("boom")

        def cell_basis(self, rows, cols, b, e, eps):
            raise RuntimeError("basis boom")

    with pytest.raises(RuntimeError, match="basis boom"):
        eb.FdsSolver(Broken(), eb.ClusterTree(64, 2), eb.FdsConfig(1e-8, 1))


def test_device_source_through_host_path_matches(eb, ref):
    # The scattering system through the callback path (AssemblerSource
    # entries and bases wrapped as a plain BlockSource) == the device path.
    n = 512
    mesh = eb.Mesh.star(n, eb.StarShape(1.0, 0.0, 3))
    med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
    asm = eb.BlockAssembler(mesh, med, med.default_coupling())
    dev = eb.AssemblerSource(asm)

    class Wrapped(eb.BlockSource):
        def n_nodes(self):
            return n

        def block(self, rows, cols):
            return dev.block(rows, cols)

        def cell_basis(self, rows, cols, b, e, eps):
            return dev.cell_basis(rows, cols, b, e, eps)

    tree = eb.ClusterTree(n, 4)
    f = asm.rhs(eb.PlanePWave(med, 1.0, 0.2))
    x_dev = eb.FdsSolver(dev, tree, eb.FdsConfig(1e-10, 1)).solve(f)
    x_host = eb.FdsSolver(Wrapped(), tree, eb.FdsConfig(1e-10, 1)).solve(f)
    assert rel(x_host, x_dev) < 1e-12
