"""Development probe of the FR-shaped config (C5) on one GPU: generation time,
preprocessing stage times (BC_DEBUG), level-1 workload shape (BC_LEVEL1_STATS).

    BC_DEBUG=1 BC_LEVEL1_STATS=1 [BC_LEVEL1_ONLY=1] python scripts/c5_probe.py [p q] [n_cores]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2403_07858_b200 import synth  # noqa: E402
from paper_2403_07858_b200.engine import DeviceGraph, EngineConfig  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 8
q = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cores = int(sys.argv[3]) if len(sys.argv) > 3 else 64
torch.cuda.synchronize()
t = time.time()
uo, ui, vo, vi = synth.fr_shaped_csr(device="cuda", n_cores=cores)
torch.cuda.synchronize()
print(f"gen {time.time() - t:.2f} s  E={int(uo[-1])}", flush=True)
dg = DeviceGraph.from_device_csr(uo, ui, vo, vi, 0)
del uo, ui, vo, vi
torch.cuda.empty_cache()
for it in range(int(os.environ.get("REPS", "1"))):
    t = time.time()
    rep, _ = dg.count_raw(p, q, EngineConfig(instrument=bool(os.environ.get("INSTR")), batch_buffer_capacity=1 << 17, order_mode=os.environ.get("ORDER", "reference")))
    d = rep.as_dict()
    print(f"({p},{q}) wall {time.time() - t:.3f} s count {d['count']} prep {rep.time_prep:.3f} "
          f"l1 {rep.time_level1:.3f} enum {rep.time_enum:.3f} tasks {rep.tasks_emitted} "
          f"alive {rep.tasks_alive} und {rep.und_pairs} dir2 {rep.dir2_pairs} "
          f"adjw {rep.adj_words} dirw {rep.dir2_words} maxslice {rep.max_slice_words} "
          f"opw {rep.operand_words} inter {rep.intersections}", flush=True)
print("peak mem GB", torch.cuda.max_memory_allocated() / 1e9)
