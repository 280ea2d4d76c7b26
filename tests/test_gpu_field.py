"""Field evaluation on the device: evaluate_scattered /
evaluate_field (proj/src/postprocess.cpp:56-119) against the compiled
reference, and the representation's physics: the total field of the solved
scattering problem satisfies the boundary data it was built from.  GPU."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def solved(eb, n=512, omega=2.0):
    mesh = eb.Mesh.star(n, eb.StarShape(1.0, 0.0, 3))
    med = eb.Medium.from_lame(1.0, 1.0, 1.0, omega)
    asm = eb.BlockAssembler(mesh, med, med.default_coupling())
    src = eb.AssemblerSource(asm, eb.ProxyConfig())
    fds = eb.FdsSolver(src, eb.ClusterTree(n, eb.ClusterTree.depth_for(n, 32)),
                       eb.FdsConfig(1e-10, 1))
    wave = eb.PlanePWave(med, 1.0, 0.3)
    u = fds.solve(asm.rhs(wave))
    return mesh, med, asm, wave, u


def test_scattered_and_total_field_match_reference(eb, ref):
    mesh, med, asm, wave, u = solved(eb)
    pts = np.vstack([eb.circle_probes(1.5, 36), eb.circle_probes(3.0, 12, (0.5, -0.2))])
    us = eb.evaluate_scattered(mesh, med, u, pts, assembler=asm)
    rp = ref.problem(mesh.nodes, 1.0, 1.0, 1.0, 2.0, med.default_coupling())
    assert rel(us, rp.evaluate_field(u, pts)) < 1e-12
    samples = eb.evaluate_field(mesh, med, wave, u, pts, n_gauss=10, assembler=asm)
    tot = np.array([s.displacement for s in samples])
    assert rel(tot, rp.evaluate_field(u, pts, ng=10, angle=0.3)) < 1e-12
    inten = np.array([s.intensity for s in samples])
    assert np.allclose(inten, np.sum(np.abs(tot) ** 2, axis=1), rtol=1e-14)


def test_interior_points_see_no_total_field(eb):
    # Exterior problem: at points inside the cavity the representation of the
    # scattered field cancels the incident one (extinction), up to the
    # discretisation error.
    mesh, med, asm, wave, u = solved(eb, n=2048, omega=1.0)
    pts = eb.circle_probes(0.4, 16)
    samples = eb.evaluate_field(mesh, med, wave, u, pts, assembler=asm)
    tot = np.array([s.displacement for s in samples])
    inc = np.array([[np.cos(0.3), np.sin(0.3)]]) * np.exp(
        -1j * med.k_L() * (pts[:, :1] * np.cos(0.3) + pts[:, 1:] * np.sin(0.3)))
    assert np.linalg.norm(tot) < 1e-3 * np.linalg.norm(inc)


def test_field_errors(eb):
    mesh, med, asm, wave, u = solved(eb, n=256)
    with pytest.raises(eb.InvalidArgument, match="from the boundary; offset it beyond"):
        eb.evaluate_scattered(mesh, med, u, [[1.0 + 1e-4, 0.0]], assembler=asm)
    with pytest.raises(eb.InvalidArgument, match="boundary data size"):
        eb.evaluate_scattered(mesh, med, u[:10], [[3.0, 0.0]], assembler=asm)
    with pytest.raises(eb.InvalidArgument, match="radius and count must be positive"):
        eb.circle_probes(-1.0, 4)
