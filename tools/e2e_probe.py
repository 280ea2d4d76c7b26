"""Wall-clock split of the bench's end-to-end sequence (development aid)."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2411_18026_b200 as eb  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
xy = np.array(eb.Mesh.star(N, eb.StarShape(1.0, 0.0, 3)).nodes)
tree = eb.ClusterTree(N, eb.ClusterTree.depth_for(N, 32))
for rep in range(3):
    t = [time.perf_counter()]
    m2 = eb.Mesh(xy); t.append(time.perf_counter())
    a2 = eb.BlockAssembler(m2, med, med.default_coupling()); t.append(time.perf_counter())
    s2 = eb.AssemblerSource(a2, eb.ProxyConfig()); t.append(time.perf_counter())
    fds = eb.FdsSolver(s2, tree, eb.FdsConfig(1e-10, 1)); t.append(time.perf_counter())
    b = a2.rhs(eb.PlanePWave(med, 1.0, 0.0)); t.append(time.perf_counter())
    x = fds.solve(b); t.append(time.perf_counter())
    x = fds.solve(b); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"rep {rep}: mesh {d[0]:.1f} asm {d[1]:.1f} src {d[2]:.1f} fds {d[3]:.1f} "
          f"(device {fds.stats().factorize_device_seconds*1e3:.1f}) rhs {d[4]:.1f} "
          f"solve1 {d[5]:.1f} solve2 {d[6]:.1f} ms", flush=True)
    del fds, s2, a2
