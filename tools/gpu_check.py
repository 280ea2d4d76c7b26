"""Quick GPU-vs-reference parity probe (development aid; the real gates are
the pytest suites).  Usage: python tools/gpu_check.py [N]"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2411_18026_b200 as eb  # noqa: E402
from _oracles import RefLib  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    print(eb.device_info())
    ref = RefLib()
    x = np.array([1e-8, 1e-3, 0.5, 1.0, 7.99, 8.01, 10.0, 100.0, 1000.0])
    g0, g1 = eb.eval_hankel(x)
    r0, r1 = ref.hankel(x)
    print("hankel rel", np.max(np.abs(g0 - r0) / np.abs(r0)), np.max(np.abs(g1 - r1) / np.abs(r1)))

    mesh = eb.Mesh.star(N, eb.StarShape(1.0, 0.0, 3))
    med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
    alpha = med.default_coupling()
    asm = eb.BlockAssembler(mesh, med, alpha)
    src = eb.AssemblerSource(asm, eb.ProxyConfig())
    rp = ref.problem(mesh.nodes, 1.0, 1.0, 1.0, 1.0, alpha)

    rr = np.array([1e-5, 0.01, 0.2, 0.26, 1.0, 3.0])
    for which in (0, 1, 2):
        a = src.eval_scalars(rr, which)
        b = ref.scalars(1.0, 1.0, 1.0, 1.0, rr, which)
        print("scalars", which, np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))

    leaf = list(range(0, 32))
    t = time.time()
    A = asm.true_block((leaf, leaf), (leaf, leaf))
    print("true_block leaf", time.time() - t, rel(A, rp.true_block((leaf, leaf), (leaf, leaf))))
    rows = (list(range(100, 140)), list(range(120, 150)))
    cols = (list(range(0, 20)) + [N - 1], list(range(90, 110)))
    print("true_block mixed", rel(asm.true_block(rows, cols), rp.true_block(rows, cols)))

    mv, mu = src.interaction_matrices((leaf, leaf), (leaf, leaf), 0, 32)
    rmv, rmu = rp.cell_mats((leaf, leaf), (leaf, leaf), 0, 32)
    print("cell_mats", mv.shape, rmv.shape, rel(mv, rmv), rel(mu, rmu))
    print("  entry max rel", np.max(np.abs(mv - rmv)) / np.max(np.abs(rmv)))
    print("  poly part", rel(mv[:128], rmv[:128]), "near part", rel(mv[128:], rmv[128:]))
    print("  U poly part", rel(mu[:, :128], rmu[:, :128]), "near part", rel(mu[:, 128:], rmu[:, 128:]))
    np.set_printoptions(linewidth=200, precision=4)

    b = src.cell_basis((leaf, leaf), (leaf, leaf), 0, 32, 1e-10)
    rb = rp.cell_basis((leaf, leaf), (leaf, leaf), 0, 32, 1e-10)
    print("cell_basis k", b.k, rb["k"])
    for p in range(2):
        print("  col skel", p, np.array_equal(b.col_skeleton[p], rb["col_skeleton"][p]),
              "row skel", np.array_equal(b.row_skeleton[p], rb["row_skeleton"][p]))
        print("  v rel", rel(b.v[p], rb["v"][p]), "u rel", rel(b.u[p], rb["u"][p]))

    f = asm.rhs(eb.PlanePWave(med, 1.0, 0.0))
    rf = rp.rhs_plane_p([0.0])[:, 0]
    print("rhs rel", rel(f, rf))

    depth = eb.ClusterTree.depth_for(N, 32)
    tree = eb.ClusterTree(N, depth)
    t = time.time()
    fds = eb.FdsSolver(src, tree, eb.FdsConfig(1e-10, 1))
    tf = time.time() - t
    print("gpu factorize", tf, fds.stats())
    t = time.time()
    xg = fds.solve(f)
    print("gpu solve", time.time() - t)
    t = time.time()
    rfds = rp.fds(depth, 1e-10, 1)
    print("ref factorize", time.time() - t, rfds.stats["max_rank"])
    xr, _ = rfds.solve(rf)
    print("solution rel vs ref", rel(xg, xr[:, 0]))
    # skeleton parity on every cell
    same = tot = 0
    for cell in range(tree.n_cells()):
        lv = tree.level_of(cell)
        if lv <= 1:
            continue
        c = fds.cell(cell)
        rc = rfds.cell(tree.cell_begin(cell), tree.cell_end(cell))
        tot += 1
        ok = c["k"] == rc["k"] and all(np.array_equal(np.sort(c["col_skeleton"][p]), np.sort(rc["col_skeleton"][p])) for p in range(2))
        same += ok
    print("cells with identical skeleton sets", same, "/", tot)


if __name__ == "__main__":
    main()
