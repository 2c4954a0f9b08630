"""Quick GPU-vs-oracle check on the named configs (dev tool; oracle as checker)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O
from paper_2403_07858_b200 import synth, DeviceGraph, EngineConfig

names = sys.argv[1:] or ["C1", "C3", "C4", "C2"]
for name in names:
    g = synth.build_config(name)
    for p, q in synth.CONFIGS[name][1]:
        t = time.time(); ref = O.count(g, p, q, workers=os.cpu_count()); tref = time.time() - t
        dg = DeviceGraph(g)
        dg.count_raw(p, q)
        t = time.time(); rep, _ = dg.count_raw(p, q); tg = time.time() - t
        ins, _ = dg.count_raw(p, q, EngineConfig(instrument=True))
        cnt = int(rep.count_lo) | (int(rep.count_hi) << 64)
        ok = (cnt == ref.count and rep.batches_executed == ref.batches_executed
              and ins.operand_words == ref.operand_words and ins.intersections == ref.intersections)
        print(f"{name} ({p},{q}) {'OK ' if ok else 'BAD'} gpu={cnt} ref={ref.count} "
              f"batches {rep.batches_executed}/{ref.batches_executed} opw {ins.operand_words}/{ref.operand_words} "
              f"inter {ins.intersections}/{ref.intersections} | gpu wall {tg*1e3:.1f} ms "
              f"(prep {rep.time_prep*1e3:.2f} l1 {rep.time_level1*1e3:.2f} enum {rep.time_enum*1e3:.2f}) "
              f"alive {rep.tasks_alive} launches {rep.kernel_launches} | cpu {tref:.2f}s", flush=True)
        dg.close()
