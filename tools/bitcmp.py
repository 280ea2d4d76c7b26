"""Solution of one factorize + solve at config 2, saved for bitwise A/B of
two builds or env switches (development aid).
  python tools/bitcmp.py N out.npy          (save)
  python tools/bitcmp.py --cmp a.npy b.npy  (compare)"""
import sys
from pathlib import Path

import numpy as np

if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    d = np.linalg.norm(a - b) / np.linalg.norm(a)
    print(f"{sys.argv[2]} vs {sys.argv[3]}: bitwise {'EQUAL' if np.array_equal(a, b) else 'DIFFER'}, rel {d:.3e}")
    sys.exit(0)
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2411_18026_b200 as eb  # noqa: E402

N = int(sys.argv[1])
med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
mesh = eb.Mesh.star(N, eb.StarShape(1.0, 0.0, 3))
asm = eb.BlockAssembler(mesh, med, med.default_coupling())
src = eb.AssemblerSource(asm)
tree = eb.ClusterTree(N, eb.ClusterTree.depth_for(N, 32))
fds = eb.FdsSolver(src, tree, eb.FdsConfig(1e-10, 1))
x = fds.solve(asm.rhs(eb.PlanePWave(med, 1.0, 0.0)))
np.save(sys.argv[2], x)
print(f"N={N} factorize {fds.stats().factorize_device_seconds:.4f} s")
