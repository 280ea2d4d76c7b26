"""Cycles per reflector step of the streaming TSQR on one CTA (development aid).
EBEM_TSQR_PIECES=1 python tools/tsqr_bench.py"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2411_18026_b200 as eb  # noqa: E402
from test_gpu_tsqr import tall_reduce  # noqa: E402

eb.prof_enable(True)
for rows, n in [(6400, 94), (6400, 122), (12800, 60), (6400, 32)]:
    rng = np.random.default_rng(0)
    a = rng.standard_normal((rows, n)) + 1j * rng.standard_normal((rows, n))
    tall_reduce(eb, a)
    eb.prof_read(reset=True)
    tall_reduce(eb, a)
    ms = eb.prof_read(reset=True)["k_qr_reduce"][0]
    b = 128 if n <= 64 else 64
    steps = (rows // b) * n
    print(f"rows {rows} n {n}: {ms:.3f} ms, {ms * 1e-3 * 1.965e9 / steps:.0f} cycles/step", flush=True)
