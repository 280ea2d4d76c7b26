"""N>1 plumbing of bench.py on CPU with gloo, world_size 2.  The solver path
does not shard (replicas only), so ranks run independent replicas
and only the timing reductions (max over ranks, summed units) cross ranks."""
import os
import socket
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

WORKER = r"""
import os, sys
sys.path.insert(0, sys.argv[1])
import bench
dist, rank, world = bench.dist_init()
assert world == 2 and dist is not None
t = bench.dist_max(dist, 1.0 + rank)
u = bench.dist_sum(dist, 10.0)
bench.barrier(dist)
assert t == 2.0, t
assert u == 20.0, u
print("ok", rank)
"""


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_two_rank_reductions(tmp_path):
    script = tmp_path / "w.py"
    script.write_text(WORKER)
    port = str(_free_port())
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE="2",
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
        procs.append(subprocess.Popen([sys.executable, str(script), str(ROOT)], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=120) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e
        assert o.startswith("ok")
