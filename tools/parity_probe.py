"""Diagnostics of the config-2 parity at one N against the committed
reference fixture: skeleton agreement per level (identical / tie / cascade)
and the solution's relative difference (test infrastructure)."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests"), str(ROOT / "oracle")]
import paper_2411_18026_b200 as eb  # noqa: E402
import test_gpu_configs as T  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2_n262144"
meta, fx = T.fixture(name)
med, asm, src, tree, fds = T.circle_solver(eb, meta)
x = fds.solve(asm.rhs(eb.PlanePWave(med, 1.0, 0.0)))
s = meta["stride"]
out = {"rel_sample": T.rel(x[::s], fx["x_sample"][:, 0])}
P = T.probes(2 * meta["n"], meta["n_probes"], meta["probe_seed"])
got = P.conj().T @ x
out["probe_rel"] = (np.abs(got - fx["x_probe"][:, 0]) / (np.sqrt(2.0) * fx["x_norm"][0])).tolist()
try:
    T.check_fds(eb, src, fds, tree, meta, fx, name)
except AssertionError as e:
    out["check_fds"] = str(e)[:3000]
rep = json.loads((ROOT / "gpurun_out" / f"parity_{name}.json").read_text())
cells = fx["cell_id"].tolist()
lev = {c: tree.level_of(c) for c in cells}
notes = rep.pop("notes", [])
out["report"] = rep
out["tie_levels"] = sorted({lev[n["cell"]] for n in notes})
print(json.dumps(out, indent=1))
