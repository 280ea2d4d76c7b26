"""Per-kernel device time of one factorization at config 2 (development aid)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2411_18026_b200 as eb  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
mesh = eb.Mesh.star(N, eb.StarShape(1.0, 0.0, 3))
src = eb.AssemblerSource(eb.BlockAssembler(mesh, med, med.default_coupling()))
tree = eb.ClusterTree(N, eb.ClusterTree.depth_for(N, 32))
eb.prof_enable(True)
for i in range(2):
    f = eb.FdsSolver(src, tree, eb.FdsConfig(1e-10, 1))
    p = eb.prof_read(reset=True)
tot = sum(v[0] for v in p.values())
print(f"factorize {f.stats().factorize_device_seconds:.4f} s, kernels {tot:.1f} ms: " +
      ", ".join(f"{k} {v[0]:.1f}" for k, v in sorted(p.items(), key=lambda kv: -kv[1][0]) if v[0] > 0.05))
