"""Wall-time breakdown of the e2e path of bench.py (development aid)."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2411_18026_b200 as eb  # noqa: E402

N = 262144
med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
mesh0 = eb.Mesh.star(N, eb.StarShape(1.0, 0.0, 3))
xy = np.array(mesh0.nodes)
tree = eb.ClusterTree(N, eb.ClusterTree.depth_for(N, 32))
for rep in range(4):
    t = [time.perf_counter()]
    m2 = eb.Mesh(xy); t.append(time.perf_counter())
    a2 = eb.BlockAssembler(m2, med, med.default_coupling()); t.append(time.perf_counter())
    s2 = eb.AssemblerSource(a2, eb.ProxyConfig()); t.append(time.perf_counter())
    fds = eb.FdsSolver(s2, tree, eb.FdsConfig(1e-10, 1)); t.append(time.perf_counter())
    b = a2.rhs(eb.PlanePWave(med, 1.0, 0.0)); t.append(time.perf_counter())
    x = fds.solve(b); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"rep {rep}: mesh {d[0]:.1f} asm {d[1]:.1f} src {d[2]:.1f} fds {d[3]:.1f} "
          f"(device {fds.stats().factorize_device_seconds*1e3:.1f}) rhs {d[4]:.1f} solve {d[5]:.1f} total {sum(d):.1f} ms")
    del fds
# recording vs replay of the solve graphs
fds = eb.FdsSolver(s2, tree, eb.FdsConfig(1e-10, 1))
for k in range(3):
    t0 = time.perf_counter()
    tm = eb.FdsSolveTiming()
    x = fds.solve(b, tm)
    print(f"solve {k}: wall {1e3 * (time.perf_counter() - t0):.2f} ms device {tm.device_seconds * 1e3:.2f} ms")
