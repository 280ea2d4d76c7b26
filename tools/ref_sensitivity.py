"""Rounding sensitivity of the reference solver itself -- TEST INFRASTRUCTURE.

Builds on oracle/_ref_fma/libebem_ref.so: the reference compiled in place
with the same sources and flags as oracle/_ref plus -mfma -ffp-contract=fast
(fused multiply-adds change only the rounding).  Solves config 2 at N and
compares with the committed -O2 reference fixture (tests/golden/configs/
cfg2_n<N>.*): the relative difference between two builds of the SAME
reference is the floor below which no other implementation can be expected
to agree with it.  Writes tests/golden/configs/ref_sensitivity.json.

  make -C oracle ref OUT=_ref_fma REFFLAGS="-std=c++20 -O2 -g -fPIC -fopenmp \
      -mfma -mavx2 -ffp-contract=fast -I/root/reference/proj/include -Ieigen_shim"
  python tools/ref_sensitivity.py 65536 262144
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT / "tests"), str(ROOT / "tools")]
from _oracles import RefLib, star_nodes  # noqa: E402
from gen_ref_fixtures import depth_for, probes  # noqa: E402

GOLD = ROOT / "tests" / "golden" / "configs"
OUT = GOLD / "ref_sensitivity.json"


def main(ns):
    ref = RefLib(ROOT / "oracle" / "_ref_fma" / "libebem_ref.so")
    ref.set_threads(int(os.environ.get("REF_THREADS", os.cpu_count())))
    res = json.loads(OUT.read_text()) if OUT.exists() else {}
    for n in ns:
        meta = json.loads((GOLD / f"cfg2_n{n}.json").read_text())
        fx = dict(np.load(GOLD / f"cfg2_n{n}.npz"))
        rp = ref.problem(star_nodes(n, 1.0, 0.0, 3), 1.0, 1.0, 1.0, 1.0, 1j)
        t0 = time.perf_counter()
        rf = rp.fds(depth_for(n, 32), 1e-10, 1, record=False)
        tf = time.perf_counter() - t0
        x, _ = rf.solve(rp.rhs_plane_p([0.0]))
        s = meta["stride"]
        xs = x[::s]
        rel = float(np.linalg.norm(xs - fx["x_sample"]) / np.linalg.norm(fx["x_sample"]))
        P = probes(2 * n, meta["n_probes"], meta["probe_seed"])
        est = np.abs(P.conj().T @ x - fx["x_probe"]) / (np.sqrt(2.0) * fx["x_norm"][None, :])
        res[f"cfg2_n{n}"] = {"rel_sample_fma_vs_O2": rel,
                             "rel_probe_median_fma_vs_O2": float(np.median(est)),
                             "max_rank_fma": rf.stats["max_rank"],
                             "max_rank_O2": meta["max_rank"],
                             "factorize_seconds": tf, "threads": ref.max_threads()}
        print(n, res[f"cfg2_n{n}"], flush=True)
        OUT.write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]])
