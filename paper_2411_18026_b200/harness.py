"""Experiment harness on the device solver: the reference's scaling,
multi-RHS and FDS-vs-Conv experiments with its CSV / JSON report schema.

Mirrors (same experiment protocol, same CSV columns, same JSON keys):
  scaling      cmd_scaling   proj/tools/ebem_cli.cpp:326-381 (+ fit_exponent,
               proj/src/report.cpp:102-121; median-of-3 below 1600 elements,
               single runs above, proj/include/ebem/report.hpp:76)
  multi_rhs    cmd_multi_rhs proj/tools/ebem_cli.cpp:383-459 (first RHS,
               per-column solves j >= 1, block solve and its deviation)
  error_table  cmd_error_table proj/tools/ebem_cli.cpp:218-275 (FDS vs the
               dense Conv solver over an (N, epsilon) ladder)
  CSV          csv_render / CsvTable, proj/src/report.cpp:14-56 (integers
               plain, doubles %.16e, no quoting)
  JSON         RunReport::to_json, proj/src/report.cpp:66-84, plus "summary"
               (save_outputs, ebem_cli.cpp:206-214)

Times are device seconds (CUDA events on the library stream: factorization
and solve) unless stated; the reference records steady-clock wall time, so
wall seconds of the same calls are reported beside them.

Usage:
  python -m paper_2411_18026_b200.harness scaling --n-max 262144 --omega 1 \
      --epsilon 1e-10 --leaf 32 --out scaling.csv
  python -m paper_2411_18026_b200.harness multi_rhs --n 65536 --omega 4 \
      --rhs-count 180 --epsilon 1e-10 --out multi_rhs.csv
  python -m paper_2411_18026_b200.harness error_table --out error_table.csv
"""
from __future__ import annotations

import argparse
import json
import math
import os
import time
from pathlib import Path
from typing import Callable, Dict, List, Sequence

import numpy as np

from . import (AssemblerSource, BlockAssembler, ClusterTree, ConvSolver, FdsConfig,
               FdsSolveTiming, FdsSolver, Medium, Mesh, PlanePWave, ProxyConfig, StarShape,
               device_info)


# ------------------------------------------------------------------ report

def csv_render(cell) -> str:
    """csv_render (report.cpp:14-25): ints plain, doubles %.16e."""
    if isinstance(cell, bool):
        raise TypeError("csv_render: bool cell")
    if isinstance(cell, (int, np.integer)):
        return str(int(cell))
    if isinstance(cell, (float, np.floating)):
        return "%.16e" % float(cell)
    s = str(cell)
    if any(c in s for c in ',"\n'):
        raise ValueError("csv_render: cell would need quoting: " + s)
    return s


class CsvTable:
    """CsvTable (report.cpp:27-56)."""

    def __init__(self, header: Sequence[str]):
        if not header:
            raise ValueError("CsvTable: header must not be empty")
        self.n_cols = len(header)
        self.text = ",".join(csv_render(h) for h in header) + "\n"
        self.n_rows = 0

    def row(self, cells: Sequence) -> None:
        if len(cells) != self.n_cols:
            raise ValueError(f"CsvTable: row width {len(cells)} != header {self.n_cols}")
        self.text += ",".join(csv_render(c) for c in cells) + "\n"
        self.n_rows += 1

    def save(self, path: str) -> None:
        Path(path).write_text(self.text)


def fit_exponent(n: Sequence[float], t: Sequence[float]) -> float:
    """Least-squares slope of log t against log n (report.cpp:102-121)."""
    if len(n) != len(t) or len(n) < 2:
        raise ValueError("fit_exponent: need matching samples, >= 2")
    x = np.log(np.asarray(n, dtype=float))
    y = np.log(np.asarray(t, dtype=float))
    if np.any(~np.isfinite(x)) or np.any(~np.isfinite(y)):
        raise ValueError("fit_exponent: samples must be positive")
    m = float(len(n))
    denom = m * float(x @ x) - float(x.sum()) ** 2
    if denom <= 0.0:
        raise ValueError("fit_exponent: degenerate abscissae")
    return (m * float(x @ y) - float(x.sum()) * float(y.sum())) / denom


def timing_repeats(n_elements: int) -> int:
    """report.hpp:76: median of 3 up to 1600 elements, single runs above."""
    return 3 if n_elements <= 1600 else 1


def median_seconds(fn: Callable[[], float], repeats: int, warm_up: bool) -> float:
    """median_seconds (report.cpp:86-100) over the seconds fn returns."""
    if repeats <= 0:
        raise ValueError("median_seconds: repeats must be positive")
    if warm_up:
        fn()
    return float(np.median([fn() for _ in range(repeats)]))


def peak_memory_mib() -> float:
    """VmHWM of this process (report.cpp:123-135)."""
    try:
        for line in open("/proc/self/status"):
            if line.startswith("VmHWM:"):
                return float(line.split()[1]) / 1024.0
    except OSError:
        pass
    return 0.0


def run_report(config: dict, phases: dict, max_rank: List[int], errors: Dict[str, float],
               summary: dict) -> dict:
    """RunReport::to_json (report.cpp:66-79) + "summary"."""
    keys = ("assembly_seconds", "compression_seconds", "factorization_seconds",
            "top_solve_seconds", "downward_seconds", "per_rhs_seconds", "total_seconds")
    return {"config": config, "phases": {k: float(phases.get(k, 0.0)) for k in keys},
            "max_rank_per_level": list(max_rank), "relative_errors": errors,
            "peak_memory_mib": peak_memory_mib(), "summary": summary}


def save_outputs(table: CsvTable, report: dict, csv_path: str) -> None:
    table.save(csv_path)
    jp = str(Path(csv_path).with_suffix(".json"))
    Path(jp).write_text(json.dumps(report, indent=2) + "\n")
    print(f"wrote {csv_path} and {jp}")


# ------------------------------------------------------------- experiments

def _problem(n: int, omega: float, m_prime: int = 64, lam: float = 1.0):
    mesh = Mesh.star(n, StarShape(1.0, 0.0, 3))
    med = Medium.from_lame(lam, 1.0, 1.0, omega)
    asm = BlockAssembler(mesh, med, med.default_coupling())
    src = AssemblerSource(asm, ProxyConfig(1.5, m_prime, 6))
    return mesh, med, asm, src


def run_fds(n: int, omega: float, eps: float, leaf: int, ell0: int = 1, angle: float = 0.0):
    """run_fds (ebem_cli.cpp:164-185) on the device: build, RHS, one solve.
    Returns a dict of device and wall seconds, the solution and stats."""
    mesh, med, asm, src = _problem(n, omega)
    tree = ClusterTree(n, ClusterTree.depth_for(n, leaf))
    t0 = time.perf_counter()
    fds = FdsSolver(src, tree, FdsConfig(eps, ell0))
    build_wall = time.perf_counter() - t0
    t0 = time.perf_counter()
    f = asm.rhs(PlanePWave(med, 1.0, angle))
    rhs_wall = time.perf_counter() - t0
    tm = FdsSolveTiming()
    t0 = time.perf_counter()
    x = fds.solve(f, tm)
    solve_wall = time.perf_counter() - t0
    st = fds.stats()
    return {"x": x, "stats": st, "levels": tree.depth(), "ell0": ell0,
            "build_seconds": st.factorize_device_seconds, "build_wall_seconds": build_wall,
            "solve_seconds": tm.device_seconds, "solve_wall_seconds": solve_wall,
            "assemble_rhs_seconds": rhs_wall}


def scaling(n_min: int = 4096, n_max: int = 262144, omega: float = 1.0, eps: float = 1e-10,
            leaf: int = 32, conv_max: int = 4096, out: str = "scaling.csv",
            reference: Dict[int, float] = None) -> dict:
    """cmd_scaling on the device: FDS factorization time over N = n_min ..
    n_max (doubling), the dense Conv solver up to conv_max, both exponents.
    `reference` ({N: seconds}) adds the reference's CPU times as "ref_fds"
    rows (measured by bench.py --sweep, which may run the oracle)."""
    table = CsvTable(["solver", "n_elements", "levels", "ell0", "epsilon", "seconds"])
    fn, ft, cn, ct = [], [], [], []
    rows = []
    n = n_min
    while n <= n_max:
        res = {}

        def once():
            r = run_fds(n, omega, eps, leaf)
            res.update(r)
            return r["build_seconds"]

        sec = median_seconds(once, timing_repeats(n), True)  # first call warms the context
        table.row(["fds", n, res["levels"], res["ell0"], eps, sec])
        rows.append({"n_elements": n, "levels": res["levels"], "factorize_seconds": sec,
                     "factorize_wall_seconds": res["build_wall_seconds"],
                     "solve_seconds": res["solve_seconds"],
                     "max_rank": res["stats"].max_rank})
        fn.append(n)
        ft.append(sec)
        print(f"fds  n={n:7d}: {sec:10.4f} s (device)", flush=True)
        n *= 2
    n = 400
    while n <= min(conv_max, n_max):
        mesh, med, asm, src = _problem(n, omega)

        def conv_once():
            c = ConvSolver(mesh, med, med.default_coupling())
            s = c.stats()
            return s.assemble_seconds + s.factor_seconds

        sec = median_seconds(conv_once, timing_repeats(n), timing_repeats(n) > 1)
        table.row(["conv", n, 0, 0, 0.0, sec])
        cn.append(n)
        ct.append(sec)
        print(f"conv n={n:7d}: {sec:10.4f} s", flush=True)
        n *= 2
    for nn, sec in sorted((reference or {}).items()):
        table.row(["ref_fds", int(nn), ClusterTree.depth_for(int(nn), leaf), 1, eps, float(sec)])
    summary = {"fds_exponent": fit_exponent(fn, ft) if len(fn) > 1 else None,
               "conv_exponent": fit_exponent(cn, ct) if len(cn) > 1 else None,
               "fds_max_n": n_max, "conv_max_n": conv_max, "device": device_info(),
               "rows": rows}
    if reference and len(reference) > 1:
        ks = sorted(reference)
        summary["ref_fds_exponent"] = fit_exponent(ks, [reference[k] for k in ks])
    cfg = {"experiment": "scaling", "n_elements": n_max, "leaf_size": leaf, "epsilon": eps,
           "omega": omega, "solver": "fds-gpu", "out": out}
    rep = run_report(cfg, {"compression_seconds": sum(ft), "total_seconds": sum(ft) + sum(ct)},
                     rows[-1]["max_rank"] if rows else [], {}, summary)
    if out:
        save_outputs(table, rep, out)
    return rep


def multi_rhs(n: int = 65536, omega: float = 4.0, count: int = 180, eps: float = 1e-10,
              leaf: int = 32, angle0: float = 0.0, out: str = "multi_rhs.csv") -> dict:
    """cmd_multi_rhs (ebem_cli.cpp:383-459) on the device: one build, the
    first solve, then every column alone (j >= 1 averaged) and the block
    solve with its deviation from the columns."""
    if count < 2:
        raise ValueError("--rhs-count must be >= 2")
    mesh, med, asm, src = _problem(n, omega)
    tree = ClusterTree(n, ClusterTree.depth_for(n, leaf))
    t0 = time.perf_counter()
    fds = FdsSolver(src, tree, FdsConfig(eps, 1))
    build_wall = time.perf_counter() - t0
    build = fds.stats().factorize_device_seconds
    angles = [angle0 + 2.0 * math.pi * j / count for j in range(count)]
    t0 = time.perf_counter()
    batch = asm.rhs_batch(med, angles, 1.0)
    rhs_seconds = time.perf_counter() - t0
    tm = FdsSolveTiming()
    fds.solve(batch[:, 0], tm)  # first solve of the process also records the graphs
    first = tm.device_seconds
    tb = FdsSolveTiming()
    allx = fds.solve(batch, tb)
    table = CsvTable(["rhs_index", "angle_deg", "solve_seconds", "deviation_vs_batch"])
    max_dev, per, worst = 0.0, [], 0.0
    for j in range(count):
        tj = FdsSolveTiming()
        xj = fds.solve(batch[:, j], tj)
        dev = float(np.linalg.norm(allx[:, j] - xj) / np.linalg.norm(xj))
        table.row([j, angles[j] * 180.0 / math.pi, tj.device_seconds, dev])
        max_dev = max(max_dev, dev)
        if j > 0:
            per.append(tj.device_seconds)
            worst = max(worst, tj.device_seconds)
    per_mean = float(np.mean(per))
    first_total = build + first
    summary = {"build_seconds": build, "build_wall_seconds": build_wall,
               "first_solve_seconds": first, "first_total_seconds": first_total,
               "per_rhs_mean_seconds": per_mean, "per_rhs_worst_seconds": worst,
               "speedup_vs_rebuild": first_total / per_mean,
               "block_solve_seconds": tb.device_seconds,
               "block_per_rhs_seconds": tb.device_seconds / count,
               "max_deviation_vs_batch": max_dev, "device": device_info()}
    cfg = {"experiment": "multi_rhs", "n_elements": n, "leaf_size": leaf, "epsilon": eps,
           "omega": omega, "rhs_count": count, "solver": "fds-gpu", "out": out}
    rep = run_report(cfg, {"compression_seconds": build, "assembly_seconds": rhs_seconds,
                           "per_rhs_seconds": per_mean, "total_seconds": first_total},
                     fds.stats().max_rank, {"max_deviation_vs_batch": max_dev}, summary)
    if out:
        save_outputs(table, rep, out)
    return rep


def error_table(ns: Sequence[int] = (400, 1600, 6400), epss: Sequence[float] = (1e-8, 1e-10),
                omega: float = 2.0, out: str = "error_table.csv") -> dict:
    """cmd_error_table (ebem_cli.cpp:218-275): FDS against the dense Conv
    solver for every (N, epsilon), tree depth from the CLI's default leaf
    size 100 and ell0 = min(1, levels - 1) (resolve_levels / resolve_ell0,
    ebem_cli.cpp:77-88)."""
    table = CsvTable(["n_elements", "levels", "ell0", "epsilon", "error_vs_conv",
                      "fds_build_seconds", "fds_solve_seconds", "conv_build_seconds",
                      "conv_solve_seconds"])
    errors, worst, max_rank = {}, 0.0, []
    for n in ns:
        mesh = Mesh.star(n, StarShape())
        med = Medium.from_lame(1.0, 1.0, 1.0, omega)
        asm = BlockAssembler(mesh, med, med.default_coupling())
        src = AssemblerSource(asm)
        levels = ClusterTree.depth_for(n, 100)
        ell0 = min(1, levels - 1)
        tree = ClusterTree(n, levels)
        f = asm.rhs(PlanePWave(med, 1.0, 0.0))
        conv = ConvSolver(mesh, med, med.default_coupling())
        t0 = time.perf_counter()
        xc = conv.solve(f)
        conv_solve = time.perf_counter() - t0
        cs = conv.stats()
        for eps in epss:
            fds = FdsSolver(src, tree, FdsConfig(eps, ell0))
            tm = FdsSolveTiming()
            x = fds.solve(f, tm)
            err = float(np.linalg.norm(x - xc) / np.linalg.norm(xc))
            table.row([n, levels, ell0, eps, err, fds.stats().factorize_device_seconds,
                       tm.device_seconds, cs.assemble_seconds + cs.factor_seconds, conv_solve])
            errors[f"n{n}_eps{csv_render(float(eps))}"] = err
            worst = max(worst, err / eps)
            max_rank = fds.stats().max_rank
    summary = {"worst_error_over_epsilon": worst, "device": device_info()}
    cfg = {"experiment": "error_table", "omega": omega, "solver": "fds-gpu", "out": out}
    rep = run_report(cfg, {}, max_rank, errors, summary)
    if out:
        save_outputs(table, rep, out)
    return rep


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2411_18026_b200.harness")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("scaling")
    s.add_argument("--n-min", type=int, default=4096)
    s.add_argument("--n-max", type=int, default=262144)
    s.add_argument("--conv-max", type=int, default=4096)
    m = sub.add_parser("multi_rhs")
    m.add_argument("--n", type=int, default=65536)
    m.add_argument("--rhs-count", type=int, default=180)
    e = sub.add_parser("error_table")
    e.add_argument("--n", type=int, action="append")
    for p in (s, m, e):
        p.add_argument("--omega", type=float, default=None)
        p.add_argument("--epsilon", type=float, default=None)
        p.add_argument("--leaf", type=int, default=32)
        p.add_argument("--out", default="")
    a = ap.parse_args(argv)
    if a.cmd == "scaling":
        scaling(a.n_min, a.n_max, a.omega or 1.0, a.epsilon or 1e-10, a.leaf, a.conv_max,
                a.out or "scaling.csv")
    elif a.cmd == "multi_rhs":
        multi_rhs(a.n, a.omega or 4.0, a.rhs_count, a.epsilon or 1e-10, a.leaf,
                  out=a.out or "multi_rhs.csv")
    else:
        error_table(a.n or (400, 1600, 6400), (a.epsilon,) if a.epsilon else (1e-8, 1e-10),
                    a.omega or 2.0, a.out or "error_table.csv")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
