"""Where the GPU-vs-reference solution difference comes from -- TEST
INFRASTRUCTURE.  At config 2, size N:
  d_full    GPU FdsSolver (device fill + ID + merges) vs the reference
  d_hybrid  GPU merges + solves fed with the REFERENCE's blocks and bases
            (a host BlockSource over oracle/_ref) vs the reference
  d_blocks  device blocks (true_block), reference bases
  d_bases   reference blocks, device bases (interaction-matrix fill + ID)
so d_hybrid isolates the merge / solve arithmetic, d_blocks the exact-block
fill and d_bases the basis construction.  Prints one JSON line."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import paper_2411_18026_b200 as eb  # noqa: E402
from _oracles import RefLib, star_nodes  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ref = RefLib()
rp = ref.problem(star_nodes(n, 1.0, 0.0, 3), 1.0, 1.0, 1.0, 1.0, 1j)
depth = eb.ClusterTree.depth_for(n, 32)
rf = rp.fds(depth, 1e-10, 1, record=False)
f = rp.rhs_plane_p([0.0])
xr = rf.solve(f)[0][:, 0]


class RefSource(eb.BlockSource):
    def n_nodes(self):
        return n

    def block(self, rows, cols):
        return rp.true_block(rows, cols)

    def cell_basis(self, rows, cols, b, e, eps):
        c = rp.cell_basis(rows, cols, b, e, eps)
        return eb.CellBasis(c["k"], c["saturated"], c["row_skeleton"], c["col_skeleton"],
                            c["u"], c["v"])


mesh = eb.Mesh.star(n, eb.StarShape(1.0, 0.0, 3))
med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
asm = eb.BlockAssembler(mesh, med, med.default_coupling())
tree = eb.ClusterTree(n, depth)
dev = eb.AssemblerSource(asm)


class DevBlocks(RefSource):
    def block(self, rows, cols):
        return dev.block(rows, cols)


class DevBases(RefSource):
    def cell_basis(self, rows, cols, b, e, eps):
        return dev.cell_basis(rows, cols, b, e, eps)


cfg = eb.FdsConfig(1e-10, 1)
xg = eb.FdsSolver(dev, tree, cfg).solve(f[:, 0])
xh = eb.FdsSolver(RefSource(), tree, cfg).solve(f[:, 0])
xb = eb.FdsSolver(DevBlocks(), tree, cfg).solve(f[:, 0])
xs = eb.FdsSolver(DevBases(), tree, cfg).solve(f[:, 0])
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
print(json.dumps({"n": n, "d_full": rel(xg, xr), "d_hybrid": rel(xh, xr),
                  "d_blocks": rel(xb, xr), "d_bases": rel(xs, xr)}))
