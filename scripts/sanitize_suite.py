"""Counts for compute-sanitizer runs (memcheck / racecheck / synccheck): every kernel
path the library can take, forced by EngineConfig flags, on small graphs and the C4 /
C3 configs, each checked against the CPU oracle (test infrastructure).

    compute-sanitizer --tool memcheck python scripts/sanitize_suite.py [quick]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2403_07858_b200 import DeviceGraph, EngineConfig, count_bicliques, synth  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
PATHS = [dict(), dict(level1="scatter", rows="scatter"), dict(level1="probe", rows="probe"),
         dict(level1="scatter", rows="probe"), dict(level1="probe", rows="scatter"),
         dict(force_triage=True), dict(force_triage=True, restricted_rows=False),
         dict(mode="dfs"), dict(order_mode="fast-reorder")]
n_checked = 0


def check(g, p, q, kw, tag):
    global n_checked
    want = O.count(g, p, q, anchor=kw.get("anchor", "auto"), mode=kw.get("mode", "hybrid"))
    rep = count_bicliques(g, p, q, EngineConfig(**kw))
    assert rep.count == want.count, (tag, p, q, kw, rep.count, want.count)
    if kw.get("order_mode", "reference") == "reference":
        assert rep.batches_executed == want.batches_executed, (tag, p, q, kw)
    n_checked += 1


rng = np.random.default_rng(7)
for i in range(3 if quick else 8):
    nu, nv = int(rng.integers(40, 120)), int(rng.integers(40, 120))
    g = synth.random_bipartite(nu, nv, float(rng.uniform(0.2, 0.5)), int(rng.integers(1 << 30)))
    p, q = int(rng.integers(5, 9)), int(rng.integers(2, 6))
    for kw in PATHS:
        check(g, p, q, dict(kw, anchor=["auto", "U", "V"][i % 3]), f"random{i}")
for name, (p, q) in (("C4", (8, 8)), ("C3", (6, 3))):
    g = synth.build_config(name)
    for kw in (PATHS[:1] + PATHS[5:7]) if quick else PATHS:
        check(g, p, q, kw, name)
# per-task counts, claim log and nesting check, enumeration, shards
g = synth.build_config("C4")
dg = DeviceGraph(g)
rep, per_task = dg.count_raw(8, 8, EngineConfig(force_triage=True), task_counts=True)
assert per_task == O.count(g, 8, 8, per_task=True, workers=8).task_counts
for k in range(3):
    dg.count_raw(8, 8, EngineConfig(), shard=(k, 3))
dg.close()
r = count_bicliques(g, 8, 8, EngineConfig(track_tasks=True, check_nesting=True))
assert r.task_tally is not None
g = synth.random_bipartite(30, 30, 0.4, 5)
r = count_bicliques(g, 3, 3, EngineConfig(enumerate_results=True))
assert r.count == O.count(g, 3, 3).count
print(f"sanitize suite ok: {n_checked} oracle-checked counts", flush=True)
