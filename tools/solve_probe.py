"""Solve-phase timing at config 2 (development aid): factorize once, solve
one right-hand side several times; per-phase device times.  With --ncu the
solves are bracketed by cudaProfilerStart/Stop for
`ncu --profile-from-start off`."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2411_18026_b200 as eb  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1
med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
mesh = eb.Mesh.star(N, eb.StarShape(1.0, 0.0, 3))
asm = eb.BlockAssembler(mesh, med, med.default_coupling())
src = eb.AssemblerSource(asm)
tree = eb.ClusterTree(N, eb.ClusterTree.depth_for(N, 32))
fds = eb.FdsSolver(src, tree, eb.FdsConfig(1e-10, 1))
f = asm.rhs_batch(med, list(np.linspace(0.0, 6.0, m)), 1.0) if m > 1 \
    else asm.rhs(eb.PlanePWave(med, 1.0, 0.0))
ncu = "--ncu" in sys.argv
if ncu:
    import torch
    fds.solve(f)
    torch.cuda.cudart().cudaProfilerStart()
for i in range(3):
    tm = eb.FdsSolveTiming()
    fds.solve(f, tm)
    print(f"solve {i}: device {tm.device_seconds*1e3:.3f} ms (up {tm.upward_seconds*1e3:.3f}, "
          f"top {tm.top_seconds*1e3:.3f}, down {tm.downward_seconds*1e3:.3f})", flush=True)
if ncu:
    torch.cuda.cudart().cudaProfilerStop()
