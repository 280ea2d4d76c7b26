"""Sum FP64 thread instructions per kernel from an ncu --csv metrics log and
divide by the point counts printed by tools/calibrate_flops.py."""
import collections
import csv
import re
import sys

ncu_csv, plain_log = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(ncu_csv)))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
acc = collections.defaultdict(lambda: collections.Counter())
for r in rows[h + 1:]:
    if len(r) <= iv:
        continue
    full = r[ik]
    name = re.sub(r"^void ", "", full).split("(")[0].split("<")[0].replace("ebem_gpu::", "")
    if name == "k_near_sym" and re.search(r"k_near_sym<(\(bool\))?(0|false)>", full):
        name = "k_near_onesided"  # the one-sided instantiation (profiler name)
    acc[name][r[im]] += float(r[iv].replace(",", ""))
pts = {}
for line in open(plain_log):
    if line.startswith("POINTS"):
        _, k, u, *_ = line.split()
        pts[k] = float(u)
for k, c in acc.items():
    fl = (2 * c["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
          + c["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]
          + c["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"])
    p = pts.get(k)
    print(f"{k}: fp64 flops {fl:.4e} points {p} flops/point {fl / p if p else float('nan'):.1f}")
