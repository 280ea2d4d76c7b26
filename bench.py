"""Benchmark of the B200 fast-direct-solver path (BASELINE.json config 2).

Workload (BASELINE.json configs[1], the config the metric is quoted on):
circular cavity, N = 262144 straight elements (2N = 2^19 = 524288 complex
unknowns), mu = rho = 1, Poisson 0.25 (lambda = mu), omega = k_T = 1, leaf 32
(depth 13), proxy circle m' = 64 at 1.5 x half-diagonal, 6-point proxy
Gauss, ID tolerance 1e-10, ell0 = 1, one unit plane P wave along (1, 0).

A "step" = one factorization (FdsSolver construction) + one single-RHS
solve.  `value` = factorize unknowns/s = 2N / (mean device time of the
factorization, CUDA events on the library's stream).  `e2e` = the same metric
through the public Python API from host buffers (mesh upload, factorize,
rhs assembly, solve with host copies), steady-clock.  The working set of a
factorization is several GB (far above the 126 MB L2) and L2 is flushed
between steps anyway.

--impl reference times the reference C++ library compiled in place
(oracle/_ref/libebem_ref.so) on the host cores with all threads, on a
bounded sample of the same workload family (config 2 at N = 16384).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "factorize unknowns/s (2N / t_factorize) at 2N=2^19"
UNIT = "unknowns/s"
N_BENCH = 262144
N_CPU_SAMPLE = 16384
EPS = 1e-10
LEAF = 32
# Algorithmic FP64 flops per quadrature-point evaluation (DESIGN.md,
# "Roofline"): FP64 instructions per point counted by ncu on the kernels
# (DADD + DMUL + 2 DFMA), divided by the point evaluations of the launch.
FLOPS_PER_POINT = {"k_near_onesided": 723.1, "k_proxy_pairs": 837.8, "k_near_sym": 1006.5}


def config_dict():
    return {"workload": "config2: circle N=262144 (2N=2^19), k_T*a=1, nu=0.25, "
                        "leaf 32, m'=64, eps=1e-10, 1 plane P wave",
            "n_elements": N_BENCH, "unknowns": 2 * N_BENCH, "leaf": LEAF,
            "epsilon": EPS, "m_prime": 64, "kT": 1.0, "ell0": 1,
            "parallelism": "replicas", "l2": "flushed between steps (512 MiB write); "
                                              "working set >> L2"}


# ------------------------------------------------------------------ helpers

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self):
        self.rows = []
        self._p = None

    def start(self):
        try:
            self._p = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-i", os.environ.get("LOCAL_RANK", "0"),
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self._p = None

    def _read(self):
        for line in self._p.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self._p is not None:
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, nm in enumerate(names):
                if len(r) > 3 + i and r[3 + i].lower() == "active":
                    reasons.add(nm)
        loaded = sorted(sm)[len(sm) // 4:] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def flush_l2():
    try:
        import torch
        if torch.cuda.is_available():
            buf = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
            buf.fill_(1)
            torch.cuda.synchronize()
            del buf
    except Exception:
        pass


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws <= 1:
        return None, 0, 1
    import torch.distributed as dist
    dist.init_process_group(backend="gloo")
    return dist, dist.get_rank(), ws


def dist_max(dist, v):
    if dist is None:
        return v
    import torch
    t = torch.tensor([float(v)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_sum(dist, v):
    if dist is None:
        return v
    import torch
    t = torch.tensor([float(v)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# --------------------------------------------------------- reference (CPU)

def run_reference(n, threads, steps=1, warmup=0):
    """Times the reference FdsSolver (compiled in place) on the host cores."""
    sys.path.insert(0, str(ROOT / "tests"))
    from _oracles import RefLib, star_nodes
    ref = RefLib()
    ref.set_threads(threads)
    nodes = star_nodes(n, 1.0, 0.0, 3)
    p = ref.problem(nodes, 1.0, 1.0, 1.0, 1.0, 1j)
    depth = 0
    while (n >> depth) > LEAF and n % (2 << depth) == 0:
        depth += 1
    rhs = p.rhs_plane_p([0.0])
    tf, ts = [], []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        f = p.fds(depth, EPS, 1, record=False)
        t1 = time.perf_counter()
        f.solve(rhs)
        t2 = time.perf_counter()
        del f
        if i >= warmup:
            tf.append(t1 - t0)
            ts.append(t2 - t1)
    return float(np.mean(tf)), float(np.mean(ts))


def cpu_info():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ------------------------------------------------------------------- main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_BENCH)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    dist, rank, world = dist_init()
    threads = os.cpu_count() or 1

    if args.impl == "reference":
        if rank != 0:
            return 0
        tf, ts = run_reference(N_CPU_SAMPLE, threads, steps=args.steps, warmup=min(args.warmup, 1))
        v = 2 * N_CPU_SAMPLE / tf
        sample = (f"reference FdsSolver (oracle/_ref, -O2 -g, OpenMP) on config 2 at "
                  f"N={N_CPU_SAMPLE} (2N={2 * N_CPU_SAMPLE}); bounded sample of the "
                  f"N={N_BENCH} workload, mean of {args.steps} factorizations")
        line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": (tf + ts) * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "c128 (f64)", "data": "synthetic (seeded geometry, analytic plane wave)",
                "config": config_dict(), "impl": "reference",
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                                 "sample": sample, "cpu": cpu_info()},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0},
                "solve_seconds_per_rhs": ts}
        print(json.dumps(line))
        return 0

    import paper_2411_18026_b200 as eb
    n = args.n
    med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
    shape = eb.StarShape(1.0, 0.0, 3)
    mesh = eb.Mesh.star(n, shape)
    depth = eb.ClusterTree.depth_for(n, LEAF)
    tree = eb.ClusterTree(n, depth)
    asm = eb.BlockAssembler(mesh, med, med.default_coupling())
    src = eb.AssemblerSource(asm, eb.ProxyConfig())
    f_host = asm.rhs(eb.PlanePWave(med, 1.0, 0.0))

    def step():
        fds = eb.FdsSolver(src, tree, eb.FdsConfig(EPS, 1))
        tm = eb.FdsSolveTiming()
        x = fds.solve(f_host, tm)
        return fds.stats().factorize_device_seconds, tm.device_seconds, x

    for _ in range(args.warmup):
        step()
        flush_l2()
    fp64_peak = eb.fp64_peak_tflops()
    barrier(dist)
    # timed region: the library's per-kernel event profiler is off
    clocks = ClockSampler()
    clocks.start()
    l0 = eb.launch_count()
    tfs, tss = [], []
    for _ in range(args.steps):
        tf, ts, x = step()
        tfs.append(tf)
        tss.append(ts)
        flush_l2()
    launches = eb.launch_count() - l0
    clk = clocks.stop()
    # one extra, untimed step with the event profiler on: kernel breakdown and
    # the dominant kernel's roofline
    eb.prof_enable(True)
    eb.prof_read(reset=True)
    step()
    prof = eb.prof_read(reset=True)
    eb.prof_enable(False)
    flush_l2()
    t_fact = dist_max(dist, float(np.mean(tfs)))
    t_solve = dist_max(dist, float(np.mean(tss)))
    units_total = dist_sum(dist, 2 * n)
    value = units_total / t_fact

    # end to end through the public API from host buffers
    xy_host = np.array(mesh.nodes)
    e2e_t = []
    for _ in range(max(1, min(args.steps, 3))):
        flush_l2()
        t0 = time.perf_counter()
        m2 = eb.Mesh(xy_host)
        a2 = eb.BlockAssembler(m2, med, med.default_coupling())
        s2 = eb.AssemblerSource(a2, eb.ProxyConfig())
        fds = eb.FdsSolver(s2, tree, eb.FdsConfig(EPS, 1))
        b = a2.rhs(eb.PlanePWave(med, 1.0, 0.0))
        xe = fds.solve(b)
        e2e_t.append(time.perf_counter() - t0)
        del fds, s2, a2
    t_e2e = dist_max(dist, float(np.mean(e2e_t)))
    h2d = 2 * 16 * n + 8 + 32 * n
    d2h = 32 * n + 32 * n

    # roofline of the dominant kernel
    top = max(prof.items(), key=lambda kv: kv[1][0])
    kname, (kms, kcount, kunits) = top
    # DRAM traffic per launch of the dominant kernel from an ncu capture of
    # every launch of one factorization at this workload (committed summary)
    traffic = None
    tf_path = ROOT / "profiles" / "r1_ncu_traffic_k_near_sym.json"
    if kname == "k_near_sym" and tf_path.exists():
        traffic = json.load(open(tf_path))["dram_bytes_per_launch"]
    roof = None
    if kname in FLOPS_PER_POINT and kms > 0:
        ach = FLOPS_PER_POINT[kname] * kunits / (kms * 1e-3) / 1e12
        roof = {"bound": "fp64", "kernel": kname, "achieved": ach, "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": ach / fp64_peak if fp64_peak else None,
                "traffic": traffic,
                "traffic_unit": "DRAM bytes per launch (ncu dram__bytes_read.sum + "
                                "dram__bytes_write.sum over all launches of one factorization, "
                                "profiles/r1_ncu_traffic_k_near_sym.json); the kernel is FP64-bound",
                "peak_source": "measured on this box by ebem_gpu_fp64_peak (DFMA chains); "
                               "MEASURED_PEAKS.json has no FP64 entry",
                "units": "quadrature points", "units_per_launch": kunits / max(kcount, 1),
                "flops_per_unit": FLOPS_PER_POINT[kname],
                "avg_launch_ms": kms / max(kcount, 1), "share_of_step":
                    kms * 1e-3 / (float(np.mean(tfs)) + float(np.mean(tss)))}
    else:
        roof = {"bound": "fp64", "kernel": kname, "achieved": None, "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": None, "traffic": None}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            tf_c, ts_c = run_reference(N_CPU_SAMPLE, threads)
            cpu = {"value": 2 * N_CPU_SAMPLE / tf_c, "unit": UNIT, "cores": threads,
                   "kind": "reference",
                   "sample": f"reference FdsSolver (oracle/_ref) factorize on config 2 at "
                             f"N={N_CPU_SAMPLE}, all {threads} host threads; a bounded sample "
                             f"(the reference is O(N log N), so its rate at N={N_BENCH} is lower)",
                   "cpu": cpu_info(), "solve_seconds_per_rhs": ts_c}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        kernels = {k: {"ms": v[0], "launches": v[1], "units": v[2]}
                   for k, v in prof.items() if v[1]}  # the one profiled step
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": (t_fact + t_solve) * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
                "data": "synthetic (analytic circle mesh, plane P wave)",
                "config": config_dict(),
                "factorize_seconds": t_fact, "solve_seconds_per_rhs": t_solve,
                "e2e": {"value": units_total / t_e2e, "unit": UNIT,
                        "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                        "seconds": t_e2e},
                "gpu_launches": launches // max(args.steps, 1),
                "clocks": clk, "roofline": roof, "cpu_baseline": cpu,
                "kernels_per_step": kernels, "ranks": tree.depth()}
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
    return 0


if __name__ == "__main__":
    sys.exit(main())
