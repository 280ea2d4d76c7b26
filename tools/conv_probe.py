"""Dense reference path timings (ConvSolver on the device) (development aid)."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2411_18026_b200 as eb  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [1024, 2048, 4096]:
    mesh = eb.Mesh.star(n, eb.StarShape(1.0, 0.0, 3))
    med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
    t = time.perf_counter()
    conv = eb.ConvSolver(mesh, med, med.default_coupling())
    tc = time.perf_counter() - t
    f = conv.assembler().rhs(eb.PlanePWave(med, 1.0, 0.0))
    t = time.perf_counter()
    x = conv.solve(f)
    ts = time.perf_counter() - t
    st = conv.stats()
    print(f"N={n}: create {tc:.3f}s (assemble {st.assemble_seconds:.3f}s, factor "
          f"{st.factor_seconds:.3f}s), solve {ts * 1e3:.1f} ms, rcond {st.rcond:.3e}, "
          f"min pivot {st.min_pivot:.3e}", flush=True)
    if n <= 2048:
        from _oracles import RefLib
        ref = RefLib()
        rp = ref.problem(mesh.nodes, 1.0, 1.0, 1.0, 1.0, med.default_coupling())
        t = time.perf_counter()
        xr, rc = rp.conv_solve(f)
        tr = time.perf_counter() - t
        print(f"   reference ConvSolver ({ref.max_threads()} threads) {tr:.2f}s; "
              f"rel diff {np.linalg.norm(x - xr[:, 0]) / np.linalg.norm(xr):.2e}; rcond {rc:.3e}",
              flush=True)
