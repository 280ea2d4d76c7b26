"""Summaries of ncu output for profiles/ (development aid).

  python tools/ncu_summary.py launches <launches.csv> [title]
      per-kernel launch count / total / share from a
      `--metrics gpu__time_duration.sum --csv` launch list
  python tools/ncu_summary.py full <report.ncu-rep>
      key sections of one `--set full` capture
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def launches(path, title=""):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = csv.DictReader(io.StringIO("".join(lines)))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("ebem_gpu::", "")
        name = name.replace("void ", "").replace("<unnamed>::", "")
        name = name.replace("(anonymous namespace)::", "")
        name = re.sub(r"<[^<>]*>$", "", name).strip()
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(r["Metric Unit"], 1e-6)
        tot[name] += v * scale
        cnt[name] += 1
    s = sum(tot.values())
    if title:
        print(title)
    print("cold-cache serialised launches: compare shares, not absolutes")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k:28s} launches {cnt[k]:5d}  total {tot[k]:10.3f} ms  share {100 * tot[k] / s:5.1f}%")
    print(f"{'all':28s} launches {sum(cnt.values()):5d}  total {s:10.3f} ms")


KEYS = ["Duration", "Registers Per Thread", "Block Size", "Grid Size",
        "Dynamic Shared Memory Per Block", "Theoretical Occupancy",
        "Achieved Occupancy", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "No Eligible", "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Local Memory Spilling Requests"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ki = hdr.index("Kernel Name")
    si, mi, ui, vi = (hdr.index(x) for x in ("Section Name", "Metric Name",
                                              "Metric Unit", "Metric Value"))
    seen = set()
    print(re.sub(r"\(.*", "", rows[1][ki]))
    for r in rows[1:]:
        if r[mi] in KEYS and (r[si], r[mi]) not in seen:
            seen.add((r[si], r[mi]))
            print(f"  {r[si][:34]:34s} {r[mi]:38s} {r[vi]:>12s} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    want = ["dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
            "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
            "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
    for w in want:
        if w in rr[0]:
            i = rr[0].index(w)
            print(f"  {w:60s} {rr[2][i]:>16s} {rr[1][i]}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
    else:
        full(sys.argv[2])
