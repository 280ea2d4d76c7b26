"""Entry-level deviation of the device true_block from the reference's
(BlockAssembler::true_block, assembly.cpp:332-409) by pair type -- TEST
INFRASTRUCTURE.  Config 2 circle at N, k_T = 1."""
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
mesh = eb.Mesh.star(n, eb.StarShape(1.0, 0.0, 3))
med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
asm = eb.BlockAssembler(mesh, med, med.default_coupling())
out = {}
for name, rows, cols in [
        ("leaf_diag", np.arange(0, 32), np.arange(0, 32)),
        ("near_gap", np.arange(0, 32), np.arange(40, 72)),
        ("mid_r", np.arange(0, 32), np.arange(n // 16, n // 16 + 32)),      # r ~ 0.39
        ("far_r", np.arange(0, 32), np.arange(n // 4, n // 4 + 32))]:         # r ~ 1.4
    A = asm.true_block((rows, rows), (cols, cols))
    B = rp.true_block((rows, rows), (cols, cols))
    d = np.abs(A - B)
    rel = d / np.abs(B).max()
    entry_rel = d / np.maximum(np.abs(B), 1e-300)
    m = len(rows)
    # per (row, col) node offset along the curve for the diagonal block
    off = {}
    if name == "leaf_diag":
        for k in range(0, 6):
            mask = np.zeros((2 * m, 2 * m), bool)
            for i in range(m):
                for j in range(m):
                    if abs(i - j) == k:
                        for p in range(2):
                            for q in range(2):
                                mask[p * m + i, q * m + j] = True
            off[k] = float(entry_rel[mask].max())
    out[name] = {"max_rel_to_blockmax": float(rel.max()),
                 "median_entry_rel": float(np.median(entry_rel)),
                 "max_entry_rel": float(entry_rel.max()), "by_offset": off}
print(json.dumps(out, indent=1))
