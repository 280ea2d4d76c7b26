"""Per-kernel device time of one factorization (+ one solve) on a BASELINE
config-2 point: ms, launches, work units, achieved rate.  Usage:
  python tools/kernel_table.py [N] [reps] [nrhs]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import paper_2411_18026_b200 as eb  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
nrhs = int(sys.argv[3]) if len(sys.argv) > 3 else 1
med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
mesh = eb.Mesh.star(N, eb.StarShape(1.0, 0.0, 3))
asm = eb.BlockAssembler(mesh, med, med.default_coupling())
src = eb.AssemblerSource(asm)
tree = eb.ClusterTree(N, eb.ClusterTree.depth_for(N, 32))
F = asm.rhs_batch(med, [2 * np.pi * j / nrhs for j in range(nrhs)], 1.0)
eb.prof_enable(True)
for rep in range(reps):
    eb.prof_read(reset=True)
    fds = eb.FdsSolver(src, tree, eb.FdsConfig(1e-10, 1))
    fp = eb.prof_read(reset=True)
    fds.solve(F)  # records the solve graphs
    eb.prof_read(reset=True)
    tm = eb.FdsSolveTiming()
    fds.solve(F, tm)
    sp = eb.prof_read(reset=True)
    if rep < reps - 1:
        del fds
        continue
    print(f"N={N} factorize {fds.stats().factorize_device_seconds * 1e3:.1f} ms, "
          f"solve({nrhs}) {tm.device_seconds * 1e3:.2f} ms")
    for title, pr in (("factorize", fp), ("solve", sp)):
        tot = sum(v[0] for v in pr.values())
        print(f"-- {title}: kernels {tot:.1f} ms")
        for k, (ms, c, u, b) in sorted(pr.items(), key=lambda kv: -kv[1][0]):
            if not c:
                continue
            rate = ""
            if ms > 0 and b > 0:
                rate += f" {b / ms / 1e6:8.1f} GB/s"
            if ms > 0 and k not in ("k_proxy_pairs", "k_near_sym", "k_near_onesided",
                                    "k_near_singular", "k_gather"):
                rate += f" {u / ms / 1e9:7.2f} TFLOP/s"
            print(f"   {k:16s} {ms:9.2f} ms {c:6d} launches units {u:.3e}{rate}")
