"""Development: C2 (4,4) enumeration/prep times (BC_DEBUG=1 for phases, INSTR=1 for
reference-equivalent tallies)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07858_b200 import DeviceGraph, EngineConfig, synth  # noqa: E402

name = os.environ.get("CFG", "C2")
g = synth.build_config(name)
p, q = synth.CONFIGS[name][1][0]
dg = DeviceGraph(g)
for i in range(int(os.environ.get("REPS", "3"))):
    r, _ = dg.count_raw(p, q, EngineConfig(instrument=bool(int(os.environ.get("INSTR", "0")))))
    print(f"enum {r.time_enum*1e3:.3f} prep {r.time_prep*1e3:.3f} level1 {r.time_level1*1e3:.3f} "
          f"alive {r.tasks_alive} emitted {r.tasks_emitted} batches {r.batches_executed} "
          f"inter {r.intersections} opw {r.operand_words} split {r.tasks_split}", file=sys.stderr)
