"""End-to-end factorize + solve on the device vs the reference FdsSolver
(same inputs): solution to 1e-8 relative, identical ranks and skeleton sets,
dense-LU agreement within the ID tolerance, determinism, error behaviour.
GPU."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def build(eb, n, omega=1.0, shape=None, leaf=32, m_prime=64, eps=1e-10, ell0=1, lam=1.0):
    mesh = eb.Mesh.star(n, shape or eb.StarShape(1.0, 0.0, 3))
    med = eb.Medium.from_lame(lam, 1.0, 1.0, omega)
    asm = eb.BlockAssembler(mesh, med, med.default_coupling())
    src = eb.AssemblerSource(asm, eb.ProxyConfig(1.5, m_prime, 6))
    tree = eb.ClusterTree(n, eb.ClusterTree.depth_for(n, leaf))
    fds = eb.FdsSolver(src, tree, eb.FdsConfig(eps, ell0))
    return mesh, med, asm, src, tree, fds


def ref_side(ref, mesh, med, tree, eps, ell0=1, m_prime=64, lam=1.0):
    rp = ref.problem(mesh.nodes, lam, 1.0, 1.0, med.omega(), med.default_coupling(),
                     m_prime=m_prime)
    return rp, rp.fds(tree.depth(), eps, ell0)


def test_config1_plumbing_vs_reference_and_dense(eb, ref):
    # BASELINE.json configs[0]: N=1024 circle, k_T a = 1, eps 1e-10, leaf 32.
    mesh, med, asm, src, tree, fds = build(eb, 1024)
    rp, rf = ref_side(ref, mesh, med, tree, 1e-10)
    f = asm.rhs(eb.PlanePWave(med, 1.0, 0.0))
    x = fds.solve(f)
    xr, _ = rf.solve(rp.rhs_plane_p([0.0]))
    assert rel(x, xr[:, 0]) < 1e-8
    assert fds.stats().max_rank == rf.stats["max_rank"]
    assert fds.stats().top_dim == rf.stats["top_dim"]
    # within the ID tolerance of the dense LU (proj/tests/test_fds.cpp:241: 100 eps)
    xc, _ = rp.conv_solve(f)
    assert rel(x, xc[:, 0]) < 100 * 1e-10
    # identical skeleton sets, every compressed cell
    for cell in range(3, tree.n_cells()):
        got = fds.cell(cell)
        want = rf.cell(tree.cell_begin(cell), tree.cell_end(cell))
        assert got["k"] == want["k"] == fds.rank_of(cell)
        for q in range(2):
            assert set(got["col_skeleton"][q]) == set(want["col_skeleton"][q])
            assert set(got["row_skeleton"][q]) == set(want["row_skeleton"][q])


@pytest.mark.parametrize("ell0", [0, 2])
def test_other_dense_levels(eb, ref, ell0):
    mesh, med, asm, src, tree, fds = build(eb, 512, ell0=ell0)
    rp, rf = ref_side(ref, mesh, med, tree, 1e-10, ell0=ell0)
    f = rp.rhs_plane_p([0.3])
    assert rel(fds.solve(f[:, 0]), rf.solve(f)[0][:, 0]) < 1e-8


def test_star_cavity_vs_reference(eb, ref):
    # non-convex star (default StarShape), omega 2 (the reference tests' medium)
    mesh, med, asm, src, tree, fds = build(eb, 1024, omega=2.0, shape=eb.StarShape(), eps=1e-8)
    rp, rf = ref_side(ref, mesh, med, tree, 1e-8)
    f = rp.rhs_plane_p([0.7])
    assert rel(fds.solve(f[:, 0]), rf.solve(f)[0][:, 0]) < 1e-8
    assert fds.stats().max_rank == rf.stats["max_rank"]


def test_config4_shape_small(eb, ref):
    # r(theta) = 1 + 0.3 cos 5 theta through Mesh(nodes), nu = 0.3, leaf 64,
    # m' = 128, eps 1e-8 (BASELINE configs[3] at reduced N and frequency).
    n = 4096
    th = np.array([2.0 * 3.14159265358979323846 * t / n for t in range(n)])
    rr = 1.0 + 0.3 * np.cos(5 * th)
    nodes = np.stack([rr * np.cos(th), rr * np.sin(th)], 1)
    mesh = eb.Mesh(nodes)
    med = eb.Medium.from_lame(1.5, 1.0, 1.0, 4.0)
    asm = eb.BlockAssembler(mesh, med, med.default_coupling())
    src = eb.AssemblerSource(asm, eb.ProxyConfig(1.5, 128, 6))
    tree = eb.ClusterTree(n, eb.ClusterTree.depth_for(n, 64))
    fds = eb.FdsSolver(src, tree, eb.FdsConfig(1e-8, 1))
    rp = ref.problem(nodes, 1.5, 1.0, 1.0, 4.0, med.default_coupling(), m_prime=128)
    rf = rp.fds(tree.depth(), 1e-8, 1)
    f = rp.rhs_plane_p([np.radians(30.0)])
    assert rel(fds.solve(f[:, 0]), rf.solve(f)[0][:, 0]) < 1e-8
    assert fds.stats().max_rank == rf.stats["max_rank"]


def test_multi_rhs_batch_equals_single_and_reuse(eb, ref):
    mesh, med, asm, src, tree, fds = build(eb, 1024, omega=4.0)
    angles = [2 * np.pi * j / 12 for j in range(12)]
    F = asm.rhs_batch(med, angles, 1.0)
    X = fds.solve(F)
    for j in (0, 5, 11):
        assert rel(X[:, j], fds.solve(F[:, j])) < 1e-12
    rp, rf = ref_side(ref, mesh, med, tree, 1e-10)
    assert rel(X, rf.solve(F)[0]) < 1e-8


def test_bitwise_determinism(eb):
    mesh, med, asm, src, tree, fds = build(eb, 1024)
    f = asm.rhs(eb.PlanePWave(med, 1.0, 0.0))
    x1 = fds.solve(f)
    fds2 = eb.FdsSolver(src, tree, eb.FdsConfig(1e-10, 1))
    assert np.array_equal(x1, fds2.solve(f))
    assert np.array_equal(x1, fds.solve(f))


def test_argument_errors_match_reference_messages(eb):
    mesh = eb.Mesh.star(256, eb.StarShape(1.0, 0.0, 3))
    med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
    src = eb.AssemblerSource(eb.BlockAssembler(mesh, med, med.default_coupling()))
    with pytest.raises(eb.InvalidArgument, match="dense level must lie strictly above"):
        eb.FdsSolver(src, eb.ClusterTree(256, 3), eb.FdsConfig(1e-8, 3))
    with pytest.raises(eb.InvalidArgument, match="node counts differ"):
        eb.FdsSolver(src, eb.ClusterTree(128, 2))
    fds = eb.FdsSolver(src, eb.ClusterTree(256, 3), eb.FdsConfig(1e-8, 1))
    with pytest.raises(eb.InvalidArgument, match="right-hand side has 10 rows, need 512"):
        fds.solve(np.zeros(10, complex))


def test_domain_error_for_coarse_mesh_at_high_frequency(eb):
    # element length * k_T >= 2.5 -> the reference's std::domain_error
    mesh = eb.Mesh.star(64, eb.StarShape(1.0, 0.0, 3))
    med = eb.Medium.from_lame(1.0, 1.0, 1.0, 40.0)
    asm = eb.BlockAssembler(mesh, med, med.default_coupling())
    with pytest.raises(eb.DomainError):
        asm.true_block(([0, 1], [0, 1]), ([0, 1], [0, 1]))


@pytest.mark.slow
def test_config2_n16384_vs_reference(eb, ref):
    # a config-2 sweep point at full parity (reference ~20 s on the host)
    mesh, med, asm, src, tree, fds = build(eb, 16384)
    rp, rf = ref_side(ref, mesh, med, tree, 1e-10)
    f = rp.rhs_plane_p([0.0])
    assert rel(fds.solve(f[:, 0]), rf.solve(f)[0][:, 0]) < 1e-8
    assert fds.stats().max_rank == rf.stats["max_rank"]


def test_large_n_properties(eb):
    # 2N = 2^19: size-independent checks (linearity in the RHS, finite, ranks)
    mesh, med, asm, src, tree, fds = build(eb, 262144)
    f1 = asm.rhs(eb.PlanePWave(med, 1.0, 0.0))
    f2 = asm.rhs(eb.PlanePWave(med, 1.0, 1.3))
    X = fds.solve(np.stack([f1, f2, 2 * f1 - 3j * f2], 1))
    assert np.all(np.isfinite(X))
    assert rel(X[:, 2], 2 * X[:, 0] - 3j * X[:, 1]) < 1e-10  # ~ cond * eps
    st = fds.stats()
    assert st.max_rank[tree.depth()] == 25 and not st.saturated
