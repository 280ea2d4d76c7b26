"""Time of the streaming TSQR on single matrices (development aid):
EBEM_TSQR_PIECES=1 python tools/tsqr_bench.py -> one CTA per matrix, i.e.
the per-block time of one reflector pipeline."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2411_18026_b200 as eb  # noqa: E402
from test_gpu_tsqr import tall_reduce  # noqa: E402

eb.prof_enable(True)
shapes = [(32768, 100), (32768, 128), (32768, 72), (32768, 64), (32768, 32)]
if len(sys.argv) > 2:  # n rows1 rows2 ...
    shapes = [(int(r), int(sys.argv[1])) for r in sys.argv[2:]]
for rows, n in shapes:
    rng = np.random.default_rng(0)
    a = rng.standard_normal((rows, n)) + 1j * rng.standard_normal((rows, n))
    tall_reduce(eb, a)
    eb.prof_read(reset=True)
    tall_reduce(eb, a)
    ms = eb.prof_read(reset=True)["k_qr_reduce"][0]
    blocks = rows // 32
    print(f"rows {rows} n {n}: {ms:.3f} ms, {ms * 1e-3 * 1.965e9 / blocks:.0f} cycles per 32-row block", flush=True)
