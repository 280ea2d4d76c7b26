"""Device special functions, Galerkin fill and proxy geometry vs the oracles
(the reference compiled in place and its golden vectors).  GPU."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def cplx(v, k):
    return complex(v[2 * k], v[2 * k + 1])


def test_hankel_golden(eb, golden):
    x = np.array([h["x"] for h in golden["hankel"]])
    h0, h1 = eb.eval_hankel(x)
    for i, h in enumerate(golden["hankel"]):
        assert abs(h0[i] - complex(h["h0r"], h["h0i"])) <= 5e-15 * abs(h0[i])
        assert abs(h1[i] - complex(h["h1r"], h["h1i"])) <= 5e-15 * abs(h1[i])


def test_hankel_vs_reference_and_wronskian(eb, ref):
    x = np.exp(np.linspace(math.log(1e-8), math.log(1e3), 3001))
    x = np.concatenate([x, [8.0 * (1 - 1e-12), 8.0, 8.0 * (1 + 1e-12)]])
    h0, h1 = eb.eval_hankel(x)
    r0, r1 = ref.hankel(x)
    assert np.max(np.abs(h0 - r0) / np.abs(r0)) < 1e-13
    assert np.max(np.abs(h1 - r1) / np.abs(r1)) < 1e-13
    lhs = np.imag(np.conj(h0) * h1)
    assert np.all(np.abs(lhs + 2 / (np.pi * x)) < 1e-13 * np.abs(h0) * np.abs(h1))


def _source(eb, n=1024, omega=1.0, shape=None, m_prime=64, leaf=32):
    mesh = eb.Mesh.star(n, shape or eb.StarShape(1.0, 0.0, 3))
    med = eb.Medium.from_lame(1.0, 1.0, 1.0, omega)
    asm = eb.BlockAssembler(mesh, med, med.default_coupling())
    src = eb.AssemblerSource(asm, eb.ProxyConfig(1.5, m_prime, 6))
    return mesh, med, asm, src


def test_scalars_golden(eb, golden):
    _, med, _, src = _source(eb, 64, omega=2.0)
    r = np.array([s["r"] for s in golden["scalars"]])
    full, rem, stat = (src.eval_scalars(r, w) for w in (0, 1, 2))
    kT = med.k_T()
    for i, sv in enumerate(golden["scalars"]):
        for k in range(10):
            want = cplx(sv["full"], k)
            assert abs(full[i, k] - want) <= max(5e-12, 1e-14 / (kT * sv["r"]) ** 2) * abs(want)
            wr = cplx(sv["rem"], k)
            # direct subtraction above the series switch: the device concedes up
            # to 3x the reference's cancellation margin (reciprocal products
            # instead of divisions in the derivative chain)
            assert abs(rem[i, k] - wr) <= 3e-12 * (abs(wr) + 5e-2 * abs(want)) + 1e-25
            ws = sv["stat"][k]
            scale = max(abs(v) for v in sv["stat"])
            assert abs(stat[i, k].real - ws) <= 1e-13 * max(scale * 1e-10, abs(ws))


@pytest.mark.parametrize("case", ["leaf", "wrap", "mixed", "skeletal"])
def test_true_block_vs_reference(eb, ref, case):
    n = 1024
    mesh, med, asm, _ = _source(eb, n, omega=1.0)
    rp = ref.problem(mesh.nodes, 1.0, 1.0, 1.0, 1.0, med.default_coupling())
    rng = np.random.default_rng(3)
    if case == "leaf":
        r = list(range(32, 64))
        rows = cols = (r, r)
    elif case == "wrap":  # node 0 and N-1 (element wrap-around)
        r = list(range(n - 16, n)) + list(range(0, 16))
        rows = cols = (r, r)
    elif case == "mixed":
        rows = (list(range(100, 140)), list(range(120, 150)))
        cols = (list(range(0, 20)) + [n - 1], list(range(90, 110)))
    else:  # scattered skeleton-like lists, different per component
        rows = (sorted(rng.choice(n, 40, replace=False)), sorted(rng.choice(n, 40, replace=False)))
        cols = (list(rng.choice(n, 30, replace=False)), list(rng.choice(n, 30, replace=False)))
    a = asm.true_block(rows, cols)
    b = rp.true_block(rows, cols)
    assert a.shape == b.shape
    assert rel(a, b) < 1e-12
    assert np.max(np.abs(a - b)) <= 1e-11 * np.max(np.abs(b))


def test_true_block_is_deterministic(eb):
    _, _, asm, _ = _source(eb, 512)
    r = list(range(0, 64))
    a = asm.true_block((r, r), (r, r))
    b = asm.true_block((r, r), (r, r))
    assert np.array_equal(a, b)


def test_proxy_geometry_and_enclosed_sets(eb, ref):
    for shape, n in [(None, 1024), (eb.StarShape(1.0, 0.3, 3), 2048)]:
        mesh, med, _, src = _source(eb, n, shape=shape)
        rp = ref.problem(mesh.nodes, 1.0, 1.0, 1.0, 1.0, med.default_coupling())
        for size in (32, 64, 256, n // 4):
            for b in range(0, n, max(size, n // 16)):
                c, rad, enc = src.build_proxy(b, b + size)
                o3, renc = rp.build_proxy(b, b + size)
                assert (c[0], c[1], rad) == (o3[0], o3[1], o3[2])
                assert np.array_equal(enc, renc)


@pytest.mark.parametrize("m_prime,leaf,omega", [(64, 32, 1.0), (128, 64, 8.0)])
def test_interaction_matrices_vs_reference(eb, ref, m_prime, leaf, omega):
    n = 2048
    mesh, med, _, src = _source(eb, n, omega=omega, m_prime=m_prime)
    rp = ref.problem(mesh.nodes, 1.0, 1.0, 1.0, omega, med.default_coupling(), m_prime=m_prime)
    for b in (0, n - leaf, 5 * leaf):
        r = list(range(b, b + leaf))
        mv, mu = src.interaction_matrices((r, r), (r, r), b, b + leaf)
        rmv, rmu = rp.cell_mats((r, r), (r, r), b, b + leaf)
        assert mv.shape == rmv.shape and mu.shape == rmu.shape
        assert rel(mv, rmv) < 1e-12 and rel(mu, rmu) < 1e-12
        assert np.max(np.abs(mv - rmv)) <= 1e-12 * np.max(np.abs(rmv))


def test_rhs_plane_p_vs_reference(eb, ref):
    mesh, med, asm, _ = _source(eb, 1024, omega=4.0)
    rp = ref.problem(mesh.nodes, 1.0, 1.0, 1.0, 4.0, med.default_coupling())
    angles = [2 * np.pi * j / 7 for j in range(7)]
    a = asm.rhs_batch(med, angles, 1.0)
    b = rp.rhs_plane_p(angles)
    assert rel(a, b) < 1e-13
    f1 = asm.rhs(eb.PlanePWave(med, 2.5, angles[3]))
    assert rel(f1, 2.5 * b[:, 3]) < 1e-13


def test_rhs_plane_sv_vs_restatement(eb):
    # SV incidence is not in the reference (SURVEY.md orientation item 4):
    # pinned against the numpy restatement only.
    import ebem_oracle as eo
    mesh, med, asm, _ = _source(eb, 512, omega=3.0)
    p = eo.Problem(mesh.nodes, eo.Medium(1.0, 1.0, 1.0, 3.0))
    ang = math.radians(30.0)
    a = asm.rhs(eb.PlaneSVWave(med, 1.0, ang))
    b = p.rhs([ang], 1.0, kind=1)[:, 0]
    assert rel(a, b) < 1e-13
