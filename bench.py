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
(oracle/_ref/libebem_ref.so) on the host cores with all threads, on the SAME
workload: one factorization + one solve at N = 262144 (about 8-10 min on 16
cores; the reference's own protocol for large N is a single run,
proj/include/ebem/report.hpp:76), so the line reports steps = 1 whatever
--steps asks for.  A bounded N = 16384 sample rides along under
"sample_n16384".

Roofline sections (each reproducible from profiles/):
  roofline        the dominant kernel (k_near_sym), FP64: executed FP64 flops
                  per quadrature point from the ncu calibration in
                  profiles/calibration.json (tagged with its commit)
  roofline_merge  the merge GEMMs (k_gemm on DMMA) and LU / solves, FP64
  roofline_id     the ID (TSQR + pivoted QR): HBM GB/s of the algorithmic
                  bytes and FP64 rate
  roofline_solve  one right-hand side: factor bytes read once / time, HBM
Extra configs (BASELINE configs[2..4], CUDA events, once after the timed
region): config 3 multi-RHS, config 4 star + SV wave, config 5 level bases.
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
CALIBRATION = ROOT / "profiles" / "calibration.json"


def calibration():
    """FP64 flops per quadrature point (ncu DADD + DMUL + 2 DFMA over all
    launches of one factorization / the points the library counted), DRAM
    traffic per launch of the dominant kernel and the DMMA pipe activity of
    the merge GEMMs, with the commit they were measured at
    (tools/calibrate.sh)."""
    try:
        return json.loads(CALIBRATION.read_text())
    except (OSError, ValueError):
        return {}


def config_dict(n=N_BENCH):
    return {"workload": f"config2: circle N={n} (2N={2 * n}), k_T*a=1, nu=0.25, "
                        "leaf 32, m'=64, eps=1e-10, 1 plane P wave",
            "n_elements": n, "unknowns": 2 * n, "leaf": LEAF,
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
                 "-lms", os.environ.get("EBEM_BENCH_SMI_MS", "200")], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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
    ap.add_argument("--no-extra-configs", action="store_true")
    args = ap.parse_args()
    dist, rank, world = dist_init()
    threads = os.cpu_count() or 1

    if args.impl == "reference":
        if rank != 0:
            return 0
        # the same workload as our arm: one factorization + one solve at
        # N = 262144 (single run, the reference's protocol for large N)
        n_ref = args.n
        tf, ts = run_reference(n_ref, threads, steps=1, warmup=0)
        v = 2 * n_ref / tf
        tf_s, ts_s = run_reference(N_CPU_SAMPLE, threads, steps=1, warmup=0)
        sample = (f"reference FdsSolver (oracle/_ref: the reference compiled in place, "
                  f"-O2 -g, OpenMP, its merge products through the Eigen-subset shim's "
                  f"plain loops) on config 2 at N={n_ref} (2N={2 * n_ref}), one "
                  f"factorization + one solve on all {threads} host threads")
        line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
                "steps": 1, "warmup": 0, "ms_per_step": (tf + ts) * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "c128 (f64)", "data": "synthetic (seeded geometry, analytic plane wave)",
                "config": config_dict(n_ref), "impl": "reference",
                "steps_note": (f"one timed factorization (the reference's single-run protocol "
                               f"for large N); --steps {args.steps} --warmup {args.warmup} "
                               f"would take {args.steps + args.warmup} x {tf:.0f} s"),
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                                 "sample": sample, "cpu": cpu_info()},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0},
                "factorize_seconds": tf, "solve_seconds_per_rhs": ts,
                "sample_n16384": {"value": 2 * N_CPU_SAMPLE / tf_s, "unit": UNIT,
                                  "factorize_seconds": tf_s, "solve_seconds_per_rhs": ts_s}}
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
        return fds.stats().factorize_device_seconds, tm.device_seconds, x, fds

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
        tf, ts, x, f_ = step()
        del f_  # device arenas are released before the next factorization
        tfs.append(tf)
        tss.append(ts)
        flush_l2()
    launches = eb.launch_count() - l0
    clk = clocks.stop()
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
    # one extra, untimed step with the event profiler on: kernel breakdown and
    # the rooflines
    eb.prof_enable(True)
    eb.prof_read(reset=True)
    _, _, _, fds_p = step()
    prof = eb.prof_read(reset=True)
    eb.prof_enable(False)
    flush_l2()

    h2d = 2 * 16 * n + 8 + 32 * n
    d2h = 32 * n + 32 * n

    cal = calibration()
    hbm = hbm_peak()
    roof = fill_roofline(prof, cal, fp64_peak, float(np.mean(tfs)) + float(np.mean(tss)))
    roof_merge = rate_roofline(prof, ("k_gemm",), fp64_peak, hbm, "merge GEMMs W = V A^-1U "
                               "(fds.cpp:99-100) on DMMA")
    roof_merge["lu_and_solves"] = rate_roofline(prof, ("k_getrf", "k_getrs"), fp64_peak, hbm,
                                                "LU + A^-1U / W^-1 solves (fds.cpp:89-101)")
    if cal.get("k_gemm_mma"):
        roof_merge["ncu"] = cal["k_gemm_mma"]
    roof_id = rate_roofline(prof, ("k_qr_reduce", "k_cpqr"), fp64_peak, hbm,
                            "ID: TSQR + pivoted QR (Cpqr, lapack.cpp:101-119)", bound="hbm")
    fb = factor_bytes(fds_p, tree, n)
    roof_solve = {"bound": "hbm", "what": "one right-hand side: every factor (LU, A^-1U, "
                  "V, W^-1 of every cell, top LU) read once + RHS / solution",
                  "bytes": fb, "seconds": t_solve, "achieved": fb / t_solve / 1e9,
                  "peak": hbm, "unit": "GB/s", "frac": fb / t_solve / 1e9 / hbm}

    extra = {}
    if not args.no_extra_configs:
        try:
            extra = extra_configs(eb, fp64_peak, hbm)
        except Exception as e:  # noqa: BLE001
            extra = {"error": repr(e)}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            tf_c, ts_c = run_reference(N_CPU_SAMPLE, threads)
            cpu = {"value": 2 * N_CPU_SAMPLE / tf_c, "unit": UNIT, "cores": threads,
                   "kind": "reference",
                   "sample": f"reference FdsSolver (oracle/_ref) factorize on config 2 at "
                             f"N={N_CPU_SAMPLE} (not {N_BENCH}: a bounded ~20 s sample), all "
                             f"{threads} host threads; the reference is O(N log N), so its rate "
                             f"at N={N_BENCH} is lower (bench.py --impl reference times that)",
                   "n_elements": N_CPU_SAMPLE, "cpu": cpu_info(),
                   "solve_seconds_per_rhs": ts_c}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        kernels = {k: {"ms": v[0], "launches": v[1], "units": v[2], "bytes": v[3]}
                   for k, v in prof.items() if v[1]}  # the one profiled step
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": (t_fact + t_solve) * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
                "data": "synthetic (analytic circle mesh, plane P wave)",
                "config": config_dict(n),
                "factorize_seconds": t_fact, "solve_seconds_per_rhs": t_solve,
                "e2e": {"value": units_total / t_e2e, "unit": UNIT,
                        "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                        "seconds": t_e2e},
                "gpu_launches": launches // max(args.steps, 1),
                "clocks": clk, "roofline": roof, "roofline_merge": roof_merge,
                "roofline_id": roof_id, "roofline_solve": roof_solve,
                "cpu_baseline": cpu, "extra_configs": extra,
                "kernels_per_step": kernels, "max_rank": fds_p.stats().max_rank,
                "calibration_commit": cal.get("commit")}
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
    return 0


# ---------------------------------------------------------------- rooflines

def hbm_peak():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6545.6  # the pool's last MEASURED_PEAKS.json value


def fill_roofline(prof, cal, fp64_peak, step_s):
    """The dominant kernel: executed FP64 flops per point (calibration) x the
    points the library counted / its CUDA-event time."""
    kname, (kms, kcount, kunits, _b) = max(prof.items(), key=lambda kv: kv[1][0])
    fpp = cal.get("flops_per_point", {}).get(kname)
    roof = {"bound": "fp64", "kernel": kname, "peak": fp64_peak, "unit": "TFLOP/s",
            "peak_source": "measured on this box by ebem_gpu_fp64_peak (DFMA chains on "
                           "every SM); MEASURED_PEAKS.json has no FP64 entry",
            "units": "quadrature points", "units_per_launch": kunits / max(kcount, 1),
            "avg_launch_ms": kms / max(kcount, 1),
            "share_of_step": kms * 1e-3 / step_s}
    if fpp and kms > 0:
        ach = fpp * kunits / (kms * 1e-3) / 1e12
        roof.update(achieved=ach, frac=ach / fp64_peak if fp64_peak else None,
                    flops_per_unit=fpp)
    else:
        roof.update(achieved=None, frac=None)
    tr = cal.get("dram_bytes_per_launch", {}).get(kname)
    roof["traffic"] = tr
    roof["traffic_unit"] = ("DRAM bytes per launch (ncu dram__bytes_read.sum + "
                            "dram__bytes_write.sum over every launch of one factorization, "
                            "profiles/calibration.json)")
    roof["points_per_second"] = kunits / (kms * 1e-3) if kms > 0 else None
    return roof


def rate_roofline(prof, names, fp64_peak, hbm, what, bound="fp64"):
    ms = sum(prof.get(k, (0, 0, 0, 0))[0] for k in names)
    fl = sum(prof.get(k, (0, 0, 0, 0))[2] for k in names)
    by = sum(prof.get(k, (0, 0, 0, 0))[3] for k in names)
    if ms <= 0:
        return {"what": what, "kernels": list(names), "ms": 0.0}
    tf = fl / (ms * 1e-3) / 1e12
    gb = by / (ms * 1e-3) / 1e9
    out = {"what": what, "kernels": list(names), "bound": bound, "ms": ms,
           "flops": fl, "bytes": by, "tflops": tf, "fp64_frac": tf / fp64_peak,
           "gbs": gb, "hbm_frac": gb / hbm}
    out.update(achieved=gb if bound == "hbm" else tf, peak=hbm if bound == "hbm" else fp64_peak,
               unit="GB/s" if bound == "hbm" else "TFLOP/s",
               frac=gb / hbm if bound == "hbm" else tf / fp64_peak)
    return out


def factor_bytes(fds, tree, n):
    """Bytes one single-RHS solve must read: per compressed cell LU (2n)^2,
    A^-1U 2n x 2k, V 2 x k x n, W^-1 (2k)^2 (n = sequence length per
    component, k = rank), the top LU, plus the RHS in and solution out."""
    depth = tree.depth()
    ell0 = 1
    ks = {}
    total = 0.0
    for lev in range(depth, ell0, -1):
        first = (1 << lev) - 1
        for c in range(first, first + (1 << lev)):
            k = fds.rank_of(c)
            ks[c] = k
            nl = (n >> depth) if lev == depth else ks[2 * c + 1] + ks[2 * c + 2]
            total += 16.0 * ((2 * nl) ** 2 + 2 * nl * 2 * k + 2 * k * nl + (2 * k) ** 2)
    top = fds.stats().top_dim
    total += 16.0 * top * top + 2 * 16.0 * 2 * n
    return total


# ------------------------------------------------------------ extra configs

def extra_configs(eb, fp64_peak, hbm):
    """BASELINE configs[2..4] once each, device time by CUDA events on the
    library stream (factorization device seconds, solve timing, batched
    cell_basis seconds)."""
    out = {}
    # config 3: N=65536, k_T a = 4, 180 P waves as one block
    n3 = 65536
    med3 = eb.Medium.from_lame(1.0, 1.0, 1.0, 4.0)
    m3 = eb.Mesh.star(n3, eb.StarShape(1.0, 0.0, 3))
    a3 = eb.BlockAssembler(m3, med3, med3.default_coupling())
    s3 = eb.AssemblerSource(a3)
    t3 = eb.ClusterTree(n3, eb.ClusterTree.depth_for(n3, LEAF))
    F = a3.rhs_batch(med3, [2 * np.pi * j / 180 for j in range(180)], 1.0)
    f3 = eb.FdsSolver(s3, t3, eb.FdsConfig(EPS, 1))  # warm-up (as the headline's warm-up steps)
    del f3
    f3 = eb.FdsSolver(s3, t3, eb.FdsConfig(EPS, 1))  # a second factorization, warm
    tm1, tm = eb.FdsSolveTiming(), eb.FdsSolveTiming()
    f3.solve(F[:, 0], tm1)  # records the one-column graphs
    f3.solve(F[:, 0], tm1)
    f3.solve(F, tm)  # records the 180-column graphs
    f3.solve(F, tm)
    # the solve replays CUDA graphs (no per-kernel events): its flops from the
    # factor sizes, one complex multiply-add per factor entry and column
    ent = (factor_bytes(f3, t3, n3) - 2 * 16.0 * 2 * n3) / 16.0
    fl = 8.0 * 180 * ent
    out["config3"] = {
        "workload": "circle N=65536, k_T a=4, 180 plane P waves theta_j=2 pi j/180, one block",
        "factorize_seconds": f3.stats().factorize_device_seconds,
        "first_rhs_seconds": f3.stats().factorize_device_seconds + tm1.device_seconds,
        "solve1_seconds": tm1.device_seconds, "solve180_seconds": tm.device_seconds,
        "per_rhs_seconds": (tm.device_seconds - tm1.device_seconds) / 179,
        "solve180_flops": fl, "solve180_tflops": fl / tm.device_seconds / 1e12 if fl else None,
        "solve180_fp64_frac": fl / tm.device_seconds / 1e12 / fp64_peak if fl else None,
        "max_rank": f3.stats().max_rank}
    del f3
    # config 4: star r = 1 + 0.3 cos 5 theta, N = 131072, nu 0.3, k_T = 16/1.3
    n4 = 131072
    th = np.array([2.0 * 3.14159265358979323846 * t / n4 for t in range(n4)])
    rr = 1.0 + 0.3 * np.cos(5 * th)
    m4 = eb.Mesh(np.stack([rr * np.cos(th), rr * np.sin(th)], 1))
    med4 = eb.Medium.from_lame(1.5, 1.0, 1.0, 16.0 / 1.3)
    a4 = eb.BlockAssembler(m4, med4, med4.default_coupling())
    s4 = eb.AssemblerSource(a4, eb.ProxyConfig(1.5, 128, 6))
    t4 = eb.ClusterTree(n4, eb.ClusterTree.depth_for(n4, 64))
    f4 = eb.FdsSolver(s4, t4, eb.FdsConfig(1e-8, 1))
    sv = a4.rhs(eb.PlaneSVWave(med4, 1.0, np.radians(30.0)))
    tm4 = eb.FdsSolveTiming()
    f4.solve(sv, tm4)
    f4.solve(sv, tm4)
    f4b = eb.FdsSolver(s4, t4, eb.FdsConfig(1e-8, 1))  # a second factorization, warm
    out["config4"] = {
        "workload": "star 1+0.3cos5t, N=131072, nu=0.3, k_T=16/1.3, leaf 64, m'=128, "
                    "eps=1e-8, plane SV wave at 30 deg",
        "factorize_seconds": f4b.stats().factorize_device_seconds,
        "unknowns_per_second": 2 * n4 / f4b.stats().factorize_device_seconds,
        "solve_seconds": tm4.device_seconds, "max_rank": f4b.stats().max_rank}
    del f4, f4b
    # config 5: 4096 boxes x 64 nodes, m' 128, k_T 8: the batched level bases
    n5, box = 262144, 64
    rng = np.random.default_rng(2411)
    begins = np.sort(rng.choice(n5 - box, 4096, replace=False))
    med5 = eb.Medium.from_lame(1.0, 1.0, 1.0, 8.0)
    m5 = eb.Mesh.star(n5, eb.StarShape(1.0, 0.0, 3))
    s5 = eb.AssemblerSource(eb.BlockAssembler(m5, med5, med5.default_coupling()),
                            eb.ProxyConfig(1.5, 128, 6))
    s5.cell_bases(begins[:64], begins[:64] + box, 1e-10)
    ts5 = [s5.cell_bases(begins, begins + box, 1e-10)[1] for _ in range(3)]
    out["config5"] = {"workload": "4096 boxes x 64 nodes of the 262144-gon, seeded, m'=128, "
                                  "k_T=8, eps=1e-10: fill + ID of the level (one batched pass)",
                      "seconds": float(np.median(ts5)),
                      "boxes_per_second": 4096 / float(np.median(ts5))}
    return out


if __name__ == "__main__":
    sys.exit(main())
