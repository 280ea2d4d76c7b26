"""Repeated factorizations on one handle: per-step device time (variance)."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2411_18026_b200 as eb  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
mesh = eb.Mesh.star(N, eb.StarShape(1.0, 0.0, 3))
src = eb.AssemblerSource(eb.BlockAssembler(mesh, med, med.default_coupling()))
tree = eb.ClusterTree(N, eb.ClusterTree.depth_for(N, 32))
eb.prof_enable("--prof" in sys.argv)
for i in range(reps):
    t = time.perf_counter()
    fds = eb.FdsSolver(src, tree, eb.FdsConfig(1e-10, 1))
    w = time.perf_counter() - t
    print(f"rep {i}: wall {w:.3f}s device {fds.stats().factorize_device_seconds:.3f}s", flush=True)
    if "--prof" in sys.argv:
        pr = eb.prof_read(reset=True)
        tot = sum(v[0] for v in pr.values())
        top = sorted(pr.items(), key=lambda kv: -kv[1][0])[:4]
        print(f"   kernels {tot:.1f} ms: " + ", ".join(f"{k} {v[0]:.0f}" for k, v in top), flush=True)
    del fds
