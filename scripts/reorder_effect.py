"""Measurement: count time of a config with no reorder / degree presort / Border
(apply_reorder, cli.py:124-145), reorder time itself on the device.
usage: python scripts/reorder_effect.py [CONFIG ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07858_b200 import DeviceGraph, EngineConfig, reorder, synth  # noqa: E402

for name in sys.argv[1:] or ["C2", "C3", "C4"]:
    g0 = synth.build_config(name)
    for p, q in synth.CONFIGS[name][1]:
        for kind in ("none", "degree", "border"):
            t = time.perf_counter()
            g = reorder.apply_reorder(g0, kind, 1000, p, q)
            tr = time.perf_counter() - t
            dg = DeviceGraph(g)
            best = None
            for _ in range(4):
                r, _ = dg.count_raw(p, q, EngineConfig())
                tt = r.time_prep + r.time_enum
                best = tt if best is None else min(best, tt)
            print(f"{name} ({p},{q}) {kind:7s} reorder {tr*1e3:8.1f} ms  count {best*1e3:7.3f} ms  "
                  f"{int(r.count_lo) | (int(r.count_hi) << 64)}", flush=True)
            dg.close()
