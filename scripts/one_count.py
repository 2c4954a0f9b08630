"""Run W+K counts of one config through the resident-graph API (for ncu / nsys-less profiling).

    python scripts/one_count.py <config> [reps] [p q]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07858_b200 import DeviceGraph, EngineConfig, synth  # noqa: E402

CAPACITY = {"C5": 1 << 17, "C5H": 1 << 17}  # bench.py: the hub slices of C5 need 122,855 words
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p, q = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else synth.CONFIGS[name][1][0]
if name in synth.DEVICE_CONFIGS:
    dg = DeviceGraph.from_device_csr(*synth.build_device_config(name))
else:
    dg = DeviceGraph(synth.build_config(name))
cfg = EngineConfig(batch_buffer_capacity=CAPACITY.get(name, 4096))
for i in range(reps):
    t = time.time()
    rep, _ = dg.count_raw(p, q, cfg)
    dt = time.time() - t
    print(name, p, q, int(rep.count_lo) | (int(rep.count_hi) << 64), f"{dt*1e3:.1f} ms",
          f"prep {rep.time_prep*1e3:.2f} l1 {rep.time_level1*1e3:.2f} enum {rep.time_enum*1e3:.2f}",
          flush=True)
