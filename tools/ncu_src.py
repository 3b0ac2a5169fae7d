"""Summarise an ncu --set full report of k_sector_eval_real: stall samples per
SASS line (top lines) and the headline pipe metrics."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.005
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:]]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data)
acc = 0.0
for d in data:
    s = f(d["Warp Stall Sampling (All Samples)"])
    acc += s
    if s / tot > thr or "BAR" in d["Source"]:
        print(d["Address"][-5:], f"{s / tot * 100:5.1f}% cum {acc / tot * 100:5.1f}%",
              f"{f(d['Instructions Executed']) / 1e6:6.2f}M", d["Source"][:64],
              d["L1 Wavefronts Shared"], d["L1 Wavefronts Shared Ideal"])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
d = dict(zip(r[0], r[2]))
for k in ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
          "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_shared.avg",
          "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "smsp__inst_executed.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"]:
    print(k, d.get(k))
for k in r[0]:
    if "pcsamp_warps_issue_stalled" in k and "not_issued" not in k and d[k] not in ("", "0"):
        print(k.replace("smsp__pcsamp_warps_issue_stalled_", "stall "), d[k])
