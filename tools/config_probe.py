"""Runs BASELINE.json configs 3 and 4 at full size (development aid)."""
import math
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2411_18026_b200 as eb  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "3"
eb.prof_enable(True)
if which == "3":
    # config 3: circle N=65536, kT a = 4, nu 0.25, 180 P waves
    n = 65536
    med = eb.Medium.from_lame(1.0, 1.0, 1.0, 4.0)
    mesh = eb.Mesh.star(n, eb.StarShape(1.0, 0.0, 3))
    leaf, mp, eps = 32, 64, 1e-10
    angles = [2 * math.pi * j / 180 for j in range(180)]
    kind = 0
else:
    # config 4: r = 1 + 0.3 cos 5 theta, N = 131072, kT a_max = 16, nu 0.3, leaf 64, m' 128
    n = 131072
    th = np.array([2.0 * 3.14159265358979323846 * t / n for t in range(n)])
    rr = 1.0 + 0.3 * np.cos(5 * th)
    mesh = eb.Mesh(np.stack([rr * np.cos(th), rr * np.sin(th)], 1))
    med = eb.Medium.from_lame(1.5, 1.0, 1.0, 16.0 / 1.3)
    leaf, mp, eps = 64, 128, 1e-8
    angles = [math.radians(30.0)]
    kind = 1
asm = eb.BlockAssembler(mesh, med, med.default_coupling())
src = eb.AssemblerSource(asm, eb.ProxyConfig(1.5, mp, 6))
tree = eb.ClusterTree(n, eb.ClusterTree.depth_for(n, leaf))
t = time.time()
fds = eb.FdsSolver(src, tree, eb.FdsConfig(eps, 1))
tf = time.time() - t
st = fds.stats()
F = asm.rhs_batch(med, angles, 1.0, kind=kind)
tm = eb.FdsSolveTiming()
x1 = fds.solve(F[:, 0], tm)
t1 = tm.device_seconds
tm2 = eb.FdsSolveTiming()
X = fds.solve(F, tm2)
print(f"config {which}: N={n} factorize {tf:.3f}s (device {st.factorize_device_seconds:.3f}s) "
      f"ranks {st.max_rank} top {st.top_dim} solve1 {t1*1e3:.2f} ms, "
      f"solve{len(angles)} {tm2.device_seconds*1e3:.2f} ms "
      f"per-RHS {(tm2.device_seconds - t1) / max(len(angles) - 1, 1) * 1e3:.3f} ms, "
      f"first-RHS {st.factorize_device_seconds + t1:.3f}s", flush=True)
print("batch vs single", np.linalg.norm(X[:, 0] - x1) / np.linalg.norm(x1))
for k, (ms, c, u, _b) in sorted(eb.prof_read(reset=True).items(), key=lambda kv: -kv[1][0]):
    if c:
        print(f"   {k:18s} {ms:9.2f} ms  {c:5d} launches")
