"""The config-3 block solve (N=65536, k_T a=4, 180 P waves) bracketed by
cudaProfilerStart/Stop for `ncu --profile-from-start off` (development aid)."""
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2411_18026_b200 as eb  # noqa: E402
import torch  # noqa: E402

n = 65536
med = eb.Medium.from_lame(1.0, 1.0, 1.0, 4.0)
mesh = eb.Mesh.star(n, eb.StarShape(1.0, 0.0, 3))
asm = eb.BlockAssembler(mesh, med, med.default_coupling())
fds = eb.FdsSolver(eb.AssemblerSource(asm), eb.ClusterTree(n, eb.ClusterTree.depth_for(n, 32)),
                   eb.FdsConfig(1e-10, 1))
F = asm.rhs_batch(med, [2 * math.pi * j / 180 for j in range(180)], 1.0)
fds.solve(F)
tm = eb.FdsSolveTiming()
torch.cuda.profiler.start()
fds.solve(F, tm)
torch.cuda.profiler.stop()
print(f"solve(180) device {tm.device_seconds * 1e3:.3f} ms")
