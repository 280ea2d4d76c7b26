"""Per-point FP64 flop count of the fill kernels on the bench workload family.

Run once plainly (prints the point evaluations per kernel from the library's
profiler) and once under
  ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,
      smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,
      smsp__sass_thread_inst_executed_op_dadd_pred_on.sum -k regex:<kernel>
then flops/point = (2 DFMA + DMUL + DADD) / points (tools/flops_from_ncu.py)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2411_18026_b200 as eb  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
eb.prof_enable(True)
med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
mesh = eb.Mesh.star(N, eb.StarShape(1.0, 0.0, 3))
src = eb.AssemblerSource(eb.BlockAssembler(mesh, med, med.default_coupling()))
fds = eb.FdsSolver(src, eb.ClusterTree(N, eb.ClusterTree.depth_for(N, 32)), eb.FdsConfig(1e-10, 1))
for k, (ms, c, u, _b) in eb.prof_read().items():
    if c:
        print(f"POINTS {k} {u:.0f} launches {c}")
