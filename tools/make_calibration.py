"""Builds profiles/calibration.json from the ncu CSVs of tools/calibrate.sh.
Usage: make_calibration.py <commit> <points.log> <fill.csv> <gemm.csv>"""
import collections
import csv
import json
import re
import sys

commit, points_log, fill_csv, gemm_csv = sys.argv[1:5]


def rows_of(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    return rows[h], rows[h + 1:]


def kname(full):
    name = re.sub(r"^void ", "", full).split("(")[0].split("<")[0].replace("ebem_gpu::", "")
    if name == "k_proxy_pp":
        name = "k_proxy_pairs"  # the thread-per-pair body of the proxy blocks (profiler name)
    if name == "k_near_sym" and re.search(r"k_near_sym<(\(bool\))?(0|false)>", full):
        name = "k_near_onesided"  # the one-sided instantiation (profiler name)
    return name


def agg(path):
    hdr, rows = rows_of(path)
    ik, im, iv, iid = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                       hdr.index("Metric Value"), hdr.index("ID"))
    acc = collections.defaultdict(collections.Counter)
    launches = collections.defaultdict(set)
    for r in rows:
        k = kname(r[ik])
        acc[k][r[im]] += float(r[iv].replace(",", ""))
        launches[k].add(r[iid])
    return acc, {k: len(v) for k, v in launches.items()}


pts = {}
for line in open(points_log):
    if line.startswith("POINTS"):
        _, k, u, *_ = line.split()
        pts[k] = float(u)
fill, nl = agg(fill_csv)
out = {"commit": commit, "workload": "config 2, N=262144, one factorization",
       "flops_per_point": {}, "dram_bytes_per_launch": {}, "launches": nl}
for k, c in fill.items():
    fl = (2 * c["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
          + c["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]
          + c["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"])
    if pts.get(k):
        out["flops_per_point"][k] = fl / pts[k]
    out["dram_bytes_per_launch"][k] = (c["dram__bytes_read.sum"] + c["dram__bytes_write.sum"]) / nl[k]
gm, gl = agg(gemm_csv)
for k, c in gm.items():
    n = gl[k]
    out[k] = {"launches": n,
              "ncu_seconds": c["gpu__time_duration.sum"] * 1e-9,
              "dmma_warp_instructions": c["sm__inst_executed_pipe_tensor_subpipe_dmma.sum"],
              "dmma_flops": 512.0 * c["sm__inst_executed_pipe_tensor_subpipe_dmma.sum"],
              "dmma_pipe_active_pct_mean":
                  c["smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"] / n,
              "fp64_pipe_active_pct_mean":
                  c["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"] / n}
print(json.dumps(out, indent=1))
