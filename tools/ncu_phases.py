"""Split an ncu --set full source page of k_sector_eval_real into its phases
(init | generator steps | expectation) by the barrier-heavy generator loop:
stall reasons, warp instructions and shared wavefronts per phase.
Usage: python tools/ncu_phases.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


stalls = [c for c in h if c.startswith("stall_")]
heavy = [i for i, d in enumerate(data) if "BAR.SYNC" in d["Source"] and f(d["Instructions Executed"]) > 1e5]
g0, g1 = min(heavy), max(heavy)
tot_s = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data)
for name, lo, hi in (("init", 0, g0), ("generators", g0, g1 + 1), ("expectation", g1 + 1, len(data))):
    part = data[lo:hi]
    s = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in part)
    inst = sum(f(d["Instructions Executed"]) for d in part)
    wf = sum(f(d["L1 Wavefronts Shared"]) for d in part)
    st = sorted(((c, sum(f(d[c]) for d in part)) for c in stalls), key=lambda x: -x[1])
    print(f"{name:12s} samples {s / tot_s * 100:5.1f}%  warp-instructions {inst / 1e6:7.2f}M  "
          f"shared wavefronts {wf / 1e6:6.2f}M")
    print("    " + ", ".join(f"{c[6:]} {v / max(s, 1) * 100:.0f}%" for c, v in st[:8]))
