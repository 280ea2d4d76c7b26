"""One single-RHS solve at config 2 (N), bracketed by cudaProfilerStart/Stop
for `ncu --profile-from-start off` (kernel list of the solve graphs)."""
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2411_18026_b200 as eb  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1
med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
mesh = eb.Mesh.star(N, eb.StarShape(1.0, 0.0, 3))
asm = eb.BlockAssembler(mesh, med, med.default_coupling())
fds = eb.FdsSolver(eb.AssemblerSource(asm), eb.ClusterTree(N, eb.ClusterTree.depth_for(N, 32)),
                   eb.FdsConfig(1e-10, 1))
import numpy as np  # noqa: E402
F = asm.rhs_batch(med, [0.1 * j for j in range(m)], 1.0)
fds.solve(F)  # records the graphs
cudart = ctypes.CDLL("libcudart.so.12") if False else None
import torch  # noqa: E402
tm = eb.FdsSolveTiming()
torch.cuda.profiler.start()
fds.solve(F, tm)
torch.cuda.profiler.stop()
print(f"solve({m}) device {tm.device_seconds * 1e3:.3f} ms")
