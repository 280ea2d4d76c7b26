import sys, os, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2411_18026_b200 as eb
from test_gpu_tsqr import tall_reduce
cases = [(80, 40), (120, 40), (200, 40), (5000, 40), (5000, 33), (5000, 48), (5000, 64), (5000, 20), (96, 48)]
for rows, n in cases:
    rng = np.random.default_rng(1)
    a = rng.standard_normal((rows, n)) + 1j * rng.standard_normal((rows, n))
    r = tall_reduce(eb, a)
    g = a.conj().T @ a
    bad = np.argwhere(~np.isfinite(r))
    err = np.linalg.norm(r.conj().T @ r - g) / np.linalg.norm(g) if not len(bad) else -1
    print(os.environ.get('EBEM_TSQR_PIECES'), rows, n, r.shape, 'nan', len(bad), sorted(set(bad[:, 1].tolist()))[:6], sorted(set(bad[:, 0].tolist()))[:6], 'err', err, flush=True)
