"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel: launches, total ns, share of the process's GPU time."""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
tot = defaultdict(lambda: [0, 0])
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"]
    name = re.sub(r"\(.*", "", name).replace("void ", "").replace("ffq::", "")
    if name.startswith("at::"):
        name = "torch elementwise (L2 flush, buffers)"
    tot[name][0] += 1
    tot[name][1] += int(float(d["Metric Value"]))
all_ns = sum(v[1] for v in tot.values())
print(f"{'kernel':48s} {'launches':>8s} {'total_ns':>12s} {'share':>7s}")
for k, (n, ns) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"{k:48s} {n:8d} {ns:12d} {100 * ns / all_ns:6.1f}%")
