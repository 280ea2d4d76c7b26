"""BASELINE config 5: batched level microbenchmark (fill + ID) on 4096 boxes.

Boxes of 64 consecutive nodes of the unit-circle 262144-gon at seeded random
positions (the per-box random rotation quantised to the mesh grid, SURVEY.md
8d), 128-point proxy circles, k_T = 8, nu = 0.25, eps = 1e-10.  One batched
cell_basis pass (proxy fill in both orientations, enclosed near rows, TSQR,
CPQR, interpolation).  Also checks ranks/skeletons of sample boxes against
the reference (when oracle/_ref is present) and times the reference on them.
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2411_18026_b200 as eb  # noqa: E402

N, BOXES, BOX = 262144, 4096, 64
rng = np.random.default_rng(2411)
begins = np.sort(rng.choice(N - BOX, BOXES, replace=False))
ends = begins + BOX
mesh = eb.Mesh.star(N, eb.StarShape(1.0, 0.0, 3))
med = eb.Medium.from_lame(1.0, 1.0, 1.0, 8.0)
src = eb.AssemblerSource(eb.BlockAssembler(mesh, med, med.default_coupling()),
                         eb.ProxyConfig(1.5, 128, 6))
eb.prof_enable(True)
src.cell_bases(begins[:64], ends[:64], 1e-10)  # warm-up
eb.prof_read(reset=True)
times = []
for _ in range(3):
    k, t = src.cell_bases(begins, ends, 1e-10)
    times.append(t)
prof = eb.prof_read(reset=True)
med_t = float(np.median(times))
out = {"config": "5", "boxes": BOXES, "box": BOX, "m_prime": 128, "kT": 8.0,
       "device_seconds": med_t, "boxes_per_second": BOXES / med_t,
       "rank_min": int(k.min()), "rank_max": int(k.max()),
       "kernels_ms": {kk: v[0] / 3 for kk, v in prof.items() if v[1]}}
try:
    from _oracles import REF_SO, RefLib
    if REF_SO.exists():
        ref = RefLib()
        ref.set_threads(1)
        rp = ref.problem(mesh.nodes, 1.0, 1.0, 1.0, 8.0, med.default_coupling(), m_prime=128)
        same, sample, tref = 0, 8, 0.0
        for i in range(sample):
            b, e = int(begins[i * 500]), int(ends[i * 500])
            r = list(range(b, e))
            t0 = time.perf_counter()
            rb = rp.cell_basis((r, r), (r, r), b, e, 1e-10)
            tref += time.perf_counter() - t0
            gb = src.cell_basis((r, r), (r, r), b, e, 1e-10)
            same += int(rb["k"] == gb.k and all(
                np.array_equal(rb["col_skeleton"][q], gb.col_skeleton[q]) for q in range(2)))
        out["reference_seconds_per_box_1_core"] = tref / sample
        out["reference_boxes_per_second_all_cores_est"] = sample / tref * ref.max_threads()
        out["identical_rank_and_skeletons_vs_reference"] = f"{same}/{sample}"
except Exception as ex:  # noqa: BLE001
    out["reference"] = f"unavailable: {ex}"
print(json.dumps(out))
