"""Run W+K counts of one config through the resident-graph API (for ncu / nsys-less profiling)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07858_b200 import synth, DeviceGraph, EngineConfig
name = sys.argv[1]; reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p, q = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else synth.CONFIGS[name][1][0]
g = synth.build_config(name)
dg = DeviceGraph(g)
for i in range(reps):
    t = time.time(); rep, _ = dg.count_raw(p, q); dt = time.time() - t
    print(name, p, q, int(rep.count_lo) | (int(rep.count_hi) << 64), f"{dt*1e3:.1f} ms",
          f"prep {rep.time_prep*1e3:.2f} l1 {rep.time_level1*1e3:.2f} enum {rep.time_enum*1e3:.2f}", flush=True)
