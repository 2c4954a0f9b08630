"""Summarise an ncu launch-list CSV (gpu__time_duration + DRAM/L2 bytes per launch):
per kernel name, launches, total ms, share, DRAM and L2 bytes."""
import csv
import signal
import sys

signal.signal(signal.SIGPIPE, signal.SIG_DFL)
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
i0 = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[i0]
k_name, k_met, k_val = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
k_id = h.index("ID")
per = defaultdict(dict)
names = {}
for r in rows[i0 + 1:]:
    if len(r) <= k_val:
        continue
    lid = r[k_id]
    names[lid] = r[k_name]
    try:
        per[lid][r[k_met]] = float(r[k_val].replace(",", ""))
    except ValueError:
        pass
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for lid, m in per.items():
    nm = names[lid]
    short = nm.split("(")[0]
    if len(short) > 90:
        short = short[:90]
    a = agg[short]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0) / 1e6  # ns -> ms
    a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    a[3] += m.get("lts__t_bytes.sum", 0)
tot = sum(a[1] for a in agg.values())
skip = tuple(sys.argv[2:]) if len(sys.argv) > 2 else ()
print(f"{'kernel':92s} {'n':>4s} {'ms':>10s} {'share':>6s} {'DRAM GB':>9s} {'DRAM GB/s':>9s} {'L2 GB':>8s}")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    if any(s in k for s in skip):
        continue
    bw = a[2] / (a[1] / 1e3) / 1e9 if a[1] else 0
    print(f"{k:92s} {a[0]:4d} {a[1]:10.3f} {100 * a[1] / tot:5.1f}% {a[2] / 1e9:9.3f} {bw:9.1f} {a[3] / 1e9:8.2f}")
print(f"total {tot:.3f} ms over {sum(a[0] for a in agg.values())} launches")
