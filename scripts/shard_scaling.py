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
if name in synth.DEVICE_CONFIGS:  # C5, C5H: generated on the device
    dg = DeviceGraph.from_device_csr(*synth.build_device_config(name))
    cap = 1 << 17
else:
    dg = DeviceGraph(synth.build_config(name))
    cap = 4096
cfg = EngineConfig(batch_buffer_capacity=cap, shard_mode=mode)
out = {"config": name, "p": p, "q": q, "shard_mode": mode, "runs": []}
sharded_prep = os.environ.get("SHARD_PREP", "1") == "1"
out["sharded_prep"] = sharded_prep
if sharded_prep:
    import time

    import torch

    from paper_2403_07858_b200.engine import assemble_upper_device

    out["note"] = ("job = max slice time + assemble + max count time; the all-gather of the "
                   "slices (NVLink, a few MB) is not emulated and is estimated at "
                   "50 us + bytes / 300 GB/s")
for n in (1, 2, 4, 8):
    shards, total = [], 0
    upper, slice_ms, asm_ms, gather_ms = None, 0.0, 0.0, 0.0
    if sharded_prep and n > 1:
        sl = []
        for k in range(n):
            for _ in range(2):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                x = dg.twohop_slice(p, q, cfg, shard=(k, n))
                torch.cuda.synchronize()
                dt = 1e3 * (time.perf_counter() - t0)
            sl.append(x)
            slice_ms = max(slice_ms, dt)
        nbytes = sum(4 * (x[0].numel() + x[1].numel()) for x in sl)
        gather_ms = 0.05 + nbytes / 300e9 * 1e3
        stride = max(max(x[1].numel() for x in sl), 1)
        ids_all = torch.zeros(n * stride, dtype=torch.int32, device="cuda")
        for k, x in enumerate(sl):
            ids_all[k * stride:k * stride + x[1].numel()] = x[1]
        lens_all = torch.cat([x[0] for x in sl])
        total_pairs = sum(x[1].numel() for x in sl)
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            upper = assemble_upper_device(lens_all, ids_all, stride, total_pairs, world=n)
            torch.cuda.synchronize()
            asm_ms = 1e3 * (time.perf_counter() - t0)
    for k in range(n):
        for _ in range(2):  # warm, then timed
            r, _ = dg.count_raw(p, q, cfg, shard=(k, n), upper=upper)
        total += int(r.count_lo) | (int(r.count_hi) << 64)
        shards.append({"shard": k, "tasks": r.tasks_consumed, "prep_ms": 1e3 * r.time_prep,
                       "level1_ms": 1e3 * r.time_level1, "enum_ms": 1e3 * r.time_enum,
                       "total_ms": 1e3 * r.time_total})
    out["runs"].append({"n": n, "count": str(total),
                        "job_ms": slice_ms + gather_ms + asm_ms + max(s["total_ms"] for s in shards),
                        "slice_ms": slice_ms, "gather_ms_est": gather_ms, "assemble_ms": asm_ms,
                        "search_ms": max(s["level1_ms"] + s["enum_ms"] for s in shards),
                        "shards": shards})
base = out["runs"][0]
for run in out["runs"]:
    run["speedup"] = base["job_ms"] / run["job_ms"]
    run["search_speedup"] = base["search_ms"] / run["search_ms"]
print(json.dumps(out, indent=1))
