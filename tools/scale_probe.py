"""Factorize/solve timings over the config-2 sweep (development aid)."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2411_18026_b200 as eb  # noqa: E402

ns = [int(a) for a in sys.argv[1:]] or [4096, 16384, 65536, 262144]
med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
eb.prof_enable(True)
for N in ns:
    mesh = eb.Mesh.star(N, eb.StarShape(1.0, 0.0, 3))
    asm = eb.BlockAssembler(mesh, med, med.default_coupling())
    src = eb.AssemblerSource(asm, eb.ProxyConfig())
    tree = eb.ClusterTree(N, eb.ClusterTree.depth_for(N, 32))
    t = time.time()
    fds = eb.FdsSolver(src, tree, eb.FdsConfig(1e-10, 1))
    tf = time.time() - t
    f = asm.rhs(eb.PlanePWave(med, 1.0, 0.0))
    t = time.time()
    x = fds.solve(f)
    ts = time.time() - t
    st = fds.stats()
    print(f"N={N} factorize {tf:.3f}s ({2*N/tf:.3e} unknowns/s) basis {st.basis_cpu_seconds:.3f}s "
          f"top {st.top_factor_seconds:.3f}s solve {ts*1e3:.2f} ms ranks {st.max_rank} top_dim {st.top_dim}",
          flush=True)
    for k, (ms, c, u, _b) in sorted(eb.prof_read(reset=True).items(), key=lambda kv: -kv[1][0]):
        if c:
            print(f"   {k:18s} {ms:9.2f} ms  {c:5d} launches  units {u:.3e}  rate {u/ms*1e3 if ms else 0:.3e}/s")
