"""Per-cell NaN / rank check of a factorization against the reference
(development aid).  Usage: python tools/nan_probe.py [N]"""
import ctypes
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2411_18026_b200 as eb  # noqa: E402
from _oracles import RefLib  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
mesh = eb.Mesh.star(N, eb.StarShape(1.0, 0.0, 3))
med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
asm = eb.BlockAssembler(mesh, med, med.default_coupling())
src = eb.AssemblerSource(asm, eb.ProxyConfig())
depth = eb.ClusterTree.depth_for(N, 32)
tree = eb.ClusterTree(N, depth)
fds = eb.FdsSolver(src, tree, eb.FdsConfig(1e-10, 1))
L = eb.lib()
ref = RefLib()
rp = ref.problem(mesh.nodes, 1.0, 1.0, 1.0, 1.0, med.default_coupling())
rf = rp.fds(depth, 1e-10, 1)
buf = np.zeros(2 * 4096 * 4096)
for lvl in range(depth, 1, -1):
    first = (1 << lvl) - 1
    nan_cells, rank_diff = [], 0
    for c in range(first, first + (1 << lvl)):
        info = fds.cell(c)
        k = info["k"]
        if k != rf.rank_of(c):
            rank_diff += 1
        nl = info["sizes"][2] + info["sizes"][3]
        for which, nr in ((0, 2 * nl * nl), (2, 2 * nl * 2 * k), (3, 2 * k * nl), (4, 8 * k * k)):
            buf[:nr] = 0
            rc = L.ebem_gpu_fds_debug_cell(fds.handle, c, which, buf.ctypes.data_as(ctypes.c_void_p))
            if rc == 0 and not np.all(np.isfinite(buf[:nr])):
                nan_cells.append((c, which))
    print(f"level {lvl}: cells {1 << lvl} rank_diff {rank_diff} nan_V {nan_cells[:8]} ({len(nan_cells)})",
          flush=True)
f = asm.rhs(eb.PlanePWave(med, 1.0, 0.0))
x = fds.solve(f)
print("solve finite", np.all(np.isfinite(x)), "stats", fds.stats().top_dim)
