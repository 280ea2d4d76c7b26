"""Dense reference path on the device: BlockAssembler::dense
and ConvSolver (proj/src/assembly.cpp:311-330, proj/src/dense_solver.cpp:9-29)
against the compiled reference.  GPU."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def setup(eb, ref, n, omega=1.0, shape=None):
    mesh = eb.Mesh.star(n, shape or eb.StarShape(1.0, 0.0, 3))
    med = eb.Medium.from_lame(1.0, 1.0, 1.0, omega)
    rp = ref.problem(mesh.nodes, 1.0, 1.0, 1.0, omega, med.default_coupling())
    return mesh, med, rp


@pytest.mark.parametrize("n,omega", [(256, 1.0), (512, 4.0)])
def test_dense_matches_reference(eb, ref, n, omega):
    mesh, med, rp = setup(eb, ref, n, omega)
    asm = eb.BlockAssembler(mesh, med, med.default_coupling())
    a = asm.dense()
    assert rel(a, rp.dense()) < 1e-12
    # sub-blocks equal true_block (the reference's guarantee, assembly.cpp:318-321)
    rows = (list(range(10, 60)), list(range(200, 230)))
    cols = (list(range(0, 40)) + [n - 1], list(range(100, 170)))
    ri = np.array(rows[0] + [n + g for g in rows[1]])
    ci = np.array(cols[0] + [n + g for g in cols[1]])
    assert rel(a[np.ix_(ri, ci)], asm.true_block(rows, cols)) < 1e-13


def test_conv_solve_matches_reference_and_fds(eb, ref):
    n = 512
    mesh, med, rp = setup(eb, ref, n)
    conv = eb.ConvSolver(mesh, med, med.default_coupling())
    assert conv.size() == 2 * n
    asm = conv.assembler()
    f = asm.rhs_batch(med, [0.0, 1.0, 2.5], 1.0)
    x = conv.solve(f)
    xr, rc = rp.conv_solve(f)
    assert rel(x, xr) < 1e-11
    st = conv.stats()
    # zgecon's estimate and ours agree to the estimator's own slack
    assert 0.2 < st.rcond / rc < 5.0
    assert not st.condition_warning and st.min_pivot > 0.0
    # vector overload; residual
    x0 = conv.solve(f[:, 0])
    assert rel(x0, x[:, 0]) < 1e-14
    a = asm.dense()
    assert rel(a @ x, f) < 1e-12
    # the FDS solution is within the ID tolerance of the dense one
    src = eb.AssemblerSource(asm, eb.ProxyConfig())
    fds = eb.FdsSolver(src, eb.ClusterTree(n, eb.ClusterTree.depth_for(n, 32)),
                       eb.FdsConfig(1e-10, 1))
    assert rel(fds.solve(f), x) < 1e-8


def test_conv_errors(eb):
    mesh = eb.Mesh.star(64, eb.StarShape(1.0, 0.0, 3))
    med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
    small = eb.AssemblyConfig(max_dense_bytes=1000)
    with pytest.raises(eb.LengthError, match="exceeds the configured memory budget"):
        eb.ConvSolver(mesh, med, med.default_coupling(), small)
    with pytest.raises(eb.LengthError):
        eb.BlockAssembler(mesh, med, med.default_coupling(), small).dense()
    conv = eb.ConvSolver(mesh, med, med.default_coupling())
    with pytest.raises(eb.InvalidArgument, match="right-hand side has 10 rows, need 128"):
        conv.solve(np.zeros(10, complex))
