"""Development/measurement: device Border pass vs the C oracle (one host thread) on a
config graph, both layers: wall time per call, rounds, final 1-block totals, parity.
usage: python scripts/border_bench.py [CONFIG] [ITERS]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402  (the checker / CPU leg only)
from paper_2403_07858_b200 import DeviceGraph, _abi, reorder, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
g = synth.build_config(name)
dg = DeviceGraph(g)
for layer in ("U", "V"):
    reorder.border_reorder(dg, layer, min(iters, 8))  # warm-up
    t = time.perf_counter()
    res = reorder.border_reorder(dg, layer, iters)
    tg = time.perf_counter() - t
    launches = _abi.load().bc_last_launch_count()
    line = (f"{name} layer {layer}: {len(res.one_block_history) - 1} swaps, 1-blocks "
            f"{res.one_block_history[0]} -> {res.one_block_history[-1]}; GPU {tg*1e3:.1f} ms "
            f"({launches} launches)")
    if os.environ.get("NO_CPU") != "1":
        t = time.perf_counter()
        perm, hist = O.border_reorder(g, layer, iters)
        tc = time.perf_counter() - t
        same = perm.tolist() == res.permutation.tolist() and hist == res.one_block_history
        line += f"; CPU oracle {tc*1e3:.1f} ms; identical {same}"
    print(line, flush=True)
dg.close()
