"""Randomised parity sweep on the GPU against the CPU oracle (development / confidence):
random bipartite graphs (sizes, densities, planted dense blocks), p, q in 1..9, every anchor,
hybrid / dfs, forced level-1 and row paths, order modes, task shards.  Compares count,
batches_executed, tasks_emitted, roots_filtered (reference order) and counts (fast orders).
usage: python scripts/stress_parity.py [SECONDS] [SEED]"""
import os
import sys
import time
from math import comb

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402  (the checker)
from paper_2403_07858_b200 import DeviceGraph, EngineConfig, synth  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
t_end = time.time() + secs
n_checks = n_graphs = 0
bad = []
while time.time() < t_end:
    hi = int(os.environ.get("STRESS_MAXN", "320"))
    nu, nv = int(rng.integers(1, hi)), int(rng.integers(1, hi))
    t_graph = time.time()
    g = synth.random_bipartite(nu, nv, float(rng.uniform(0.003, 0.35)), int(rng.integers(1 << 30)))
    if rng.random() < 0.4 and nu > 8 and nv > 8:  # plant a dense block
        a, b = int(rng.integers(4, min(nu, 24) + 1)), int(rng.integers(4, min(nv, 24) + 1))
        us, vs = rng.choice(nu, a, replace=False), rng.choice(nv, b, replace=False)
        m = rng.random((a, b)) < rng.uniform(0.7, 1.0)
        i, j = np.nonzero(m)
        uo, ui = g.u_csr.off, g.u_csr.idx
        eu = np.concatenate([np.repeat(np.arange(nu), np.diff(uo)), us[i]])
        ev = np.concatenate([ui.astype(np.int64), vs[j]])
        g = synth.from_edges(nu, nv, eu, ev)
    n_graphs += 1
    dg = DeviceGraph(g)
    for _ in range(4):
        p, q = int(rng.integers(1, 10)), int(rng.integers(1, 10))
        anchor = ["auto", "U", "V"][int(rng.integers(3))]
        mode = ["hybrid", "dfs"][int(rng.integers(2))]
        # skip searches the single-threaded oracle cannot finish in seconds: the leaves of
        # a (p, q) search number about sum_v C(deg v, p) (anchor U) / sum_u C(deg u, q)
        du, dv = np.diff(g.u_csr.off), np.diff(g.v_csr.off)
        size = sum(comb(int(d), p) for d in dv) + sum(comb(int(d), q) for d in du)
        if size > 2e7:
            continue
        t_o = time.time()
        want = O.count(g, p, q, anchor=anchor, mode=mode)
        t_o = time.time() - t_o
        l1 = ["auto", "scatter", "probe"][int(rng.integers(3))]
        rows = ["auto", "scatter", "probe"][int(rng.integers(3))]
        cfg = EngineConfig(anchor=anchor, mode=mode, level1=l1, rows=rows)
        t_g = time.time()
        r, _ = dg.count_raw(p, q, cfg)
        t_g = time.time() - t_g
        if os.environ.get("STRESS_VERBOSE") or t_o + t_g > 2:
            print(f"  ({nu}x{nv}, p={p}, q={q}, {anchor}, {mode}, {l1}, {rows}) oracle {t_o:.2f}s "
                  f"gpu {t_g:.2f}s", flush=True)
        got = int(r.count_lo) | (int(r.count_hi) << 64)
        n_checks += 1
        key = (nu, nv, p, q, anchor, mode, l1, rows)
        if (got != want.count or r.batches_executed != want.batches_executed
                or r.tasks_emitted != want.tasks_emitted or r.roots_filtered != want.roots_filtered):
            bad.append(("ref", key, got, want.count, r.batches_executed, want.batches_executed))
        k = int(rng.integers(2, 6))
        tot = 0
        if os.environ.get("STRESS_VERBOSE"):
            print(f"    shards {k}", flush=True)
        for s in range(k):
            rr, _ = dg.count_raw(p, q, cfg, shard=(s, k))
            tot += int(rr.count_lo) | (int(rr.count_hi) << 64)
        n_checks += 1
        if tot != want.count:
            bad.append(("shards", key, k, tot, want.count))
        om = ["fast", "fast-reorder"][int(rng.integers(2))]
        if os.environ.get("STRESS_VERBOSE"):
            print(f"    order {om}", flush=True)
        rf, _ = dg.count_raw(p, q, EngineConfig(anchor=anchor, mode=mode, order_mode=om))
        n_checks += 1
        if (int(rf.count_lo) | (int(rf.count_hi) << 64)) != want.count:
            bad.append((om, key))
    dg.close()
    if n_graphs % 20 == 0:
        print(f"... graphs {n_graphs} checks {n_checks} mismatches {len(bad)}", flush=True)
print(f"graphs {n_graphs} checks {n_checks} mismatches {len(bad)}")
for b in bad[:20]:
    print("MISMATCH", b)
sys.exit(1 if bad else 0)
