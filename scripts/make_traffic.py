"""profiles/r2/traffic.json from ncu launch lists: DRAM and L2 bytes of the enumeration
kernels (filter_kernel, enum_kernel, sub_kernel) of one count, keyed by the bench workload
string and stamped with the source hash of the build that was captured (bench.py uses an
entry only for that build).  Run it on the launch list of the current tree.

    python scripts/make_traffic.py '<workload>' <launches.csv> [<workload> <csv> ...]
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_07858_b200 import build  # noqa: E402

out_path = os.path.join(ROOT, "profiles", "r2", "traffic.json")
try:
    out = json.load(open(out_path))
except (OSError, ValueError):
    out = {}
args = sys.argv[1:]
for work, path in zip(args[::2], args[1::2]):
    rows = list(csv.reader(open(path)))
    i0 = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[i0]
    kn, mn, mv, ki = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = {}
    for r in rows[i0 + 1:]:
        if len(r) <= mv or not any(k in r[kn] for k in ("enum_kernel", "sub_kernel", "filter_kernel")):
            continue
        per.setdefault(r[ki], {})[r[mn]] = float(r[mv].replace(",", ""))
    dram = sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in per.values())
    l2 = sum(m.get("lts__t_bytes.sum", 0) for m in per.values())
    ms = sum(m.get("gpu__time_duration.sum", 0) for m in per.values()) / 1e6
    out[work] = {"dram_bytes": int(dram), "l2_bytes": int(l2), "ncu_ms": round(ms, 3),
                 "launches": len(per), "source": os.path.relpath(path, ROOT),
                 "src_sha": build.source_hash()}
    print(work, out[work])
json.dump(out, open(out_path, "w"), indent=1)
