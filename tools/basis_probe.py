"""cell_basis of one FDS cell recomputed through the API vs the reference
(development aid).  Usage: python tools/basis_probe.py N cell"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2411_18026_b200 as eb  # noqa: E402
from _oracles import RefLib  # noqa: E402

N, cell = int(sys.argv[1]), int(sys.argv[2])
mesh = eb.Mesh.star(N, eb.StarShape(1.0, 0.0, 3))
med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
asm = eb.BlockAssembler(mesh, med, med.default_coupling())
src = eb.AssemblerSource(asm, eb.ProxyConfig())
depth = eb.ClusterTree.depth_for(N, 32)
fds = eb.FdsSolver(src, eb.ClusterTree(N, depth), eb.FdsConfig(1e-10, 1))
lvl = (cell + 1).bit_length() - 1
size = N >> lvl
b, e = (cell - ((1 << lvl) - 1)) * size, (cell - ((1 << lvl) - 1) + 1) * size
c1, c2 = fds.cell(2 * cell + 1), fds.cell(2 * cell + 2)
rows = tuple(np.concatenate([c1["row_skeleton"][q], c2["row_skeleton"][q]]) for q in range(2))
cols = tuple(np.concatenate([c1["col_skeleton"][q], c2["col_skeleton"][q]]) for q in range(2))
print("cell", cell, "range", b, e, "n", [len(x) for x in rows + cols])
gb = src.cell_basis(rows, cols, b, e, 1e-10)
print("k", gb.k, "u finite", [bool(np.all(np.isfinite(u))) for u in gb.u],
      "v finite", [bool(np.all(np.isfinite(v))) for v in gb.v])
ref = RefLib()
rp = ref.problem(mesh.nodes, 1.0, 1.0, 1.0, 1.0, med.default_coupling())
rb = rp.cell_basis(rows, cols, b, e, 1e-10)
print("ref k", rb["k"], "same skel", [bool(np.array_equal(rb["col_skeleton"][q], gb.col_skeleton[q])) for q in range(2)],
      [bool(np.array_equal(rb["row_skeleton"][q], gb.row_skeleton[q])) for q in range(2)])
for q in range(2):
    print("u", q, np.linalg.norm(gb.u[q] - rb["u"][q]) / np.linalg.norm(rb["u"][q]),
          "v", q, np.linalg.norm(gb.v[q] - rb["v"][q]) / np.linalg.norm(rb["v"][q]))
sys.path.insert(0, str(ROOT / "tests"))
from test_gpu_tsqr import tall_reduce  # noqa: E402
mv, mu = src.interaction_matrices(rows, cols, b, e)
tu = mu.conj().T
nr0 = len(rows[0])
for name, blk in (("V0", mv[:, :len(cols[0])]), ("V1", mv[:, len(cols[0]):]),
                  ("U0", tu[:, :nr0]), ("U1", tu[:, nr0:])):
    r = tall_reduce(eb, blk)
    g = blk.conj().T @ blk
    print(name, blk.shape, "finite", bool(np.all(np.isfinite(blk))), "R finite",
          bool(np.all(np.isfinite(r))), "gram err", np.linalg.norm(r.conj().T @ r - g) / np.linalg.norm(g))
