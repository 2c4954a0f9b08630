"""Emulated multi-GPU scaling on one B200: every shard of an N-way split is counted in
turn on the same device (each shard is exactly what rank k of N runs: its own
preprocessing, level 1 and enumeration); the job time of N GPUs is the slowest shard,
the count the sum.  Usage: python scripts/shard_scaling.py [config] [shard_mode] > out.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07858_b200 import DeviceGraph, EngineConfig, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
mode = sys.argv[2] if len(sys.argv) > 2 else "root"
p, q = synth.CONFIGS[name][1][0]
if name == "C5":
    dg = DeviceGraph.from_device_csr(*synth.fr_shaped_csr(device="cuda"))
    cap = 1 << 17
else:
    dg = DeviceGraph(synth.build_config(name))
    cap = 4096
cfg = EngineConfig(batch_buffer_capacity=cap, shard_mode=mode)
out = {"config": name, "p": p, "q": q, "shard_mode": mode, "runs": []}
for n in (1, 2, 4, 8):
    shards, total = [], 0
    for k in range(n):
        for _ in range(2):  # warm, then timed
            r, _ = dg.count_raw(p, q, cfg, shard=(k, n))
        total += int(r.count_lo) | (int(r.count_hi) << 64)
        shards.append({"shard": k, "tasks": r.tasks_consumed, "prep_ms": 1e3 * r.time_prep,
                       "level1_ms": 1e3 * r.time_level1, "enum_ms": 1e3 * r.time_enum,
                       "total_ms": 1e3 * r.time_total})
    out["runs"].append({"n": n, "count": str(total), "job_ms": max(s["total_ms"] for s in shards),
                        "search_ms": max(s["level1_ms"] + s["enum_ms"] for s in shards),
                        "shards": shards})
base = out["runs"][0]
for run in out["runs"]:
    run["speedup"] = base["job_ms"] / run["job_ms"]
    run["search_speedup"] = base["search_ms"] / run["search_ms"]
print(json.dumps(out, indent=1))
