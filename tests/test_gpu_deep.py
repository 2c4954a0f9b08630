"""Deep searches on the device: p, q in 9..12 (the paper runs p + q up to 24,
PAPER.md:847; the reference engine has no depth limit, engine.py:306-374).

Graphs are random bipartite noise around a planted near-complete core, so the
(p,q) counts are large and the search goes 9-12 levels deep; the oracle
(reference order, bisect intersections) finishes each in well under a second.
Every kernel path (level 1 scatter/probe x rows scatter/probe, split and
whole-task enumeration) must give the exact count and the reference's
counters, batch accounting and intersection tallies."""

import itertools

import numpy as np
import pytest

from oracle import oracle as O
from paper_2403_07858_b200 import DeviceGraph, EngineConfig, count_bicliques
from paper_2403_07858_b200.graph import from_edges

pytestmark = pytest.mark.gpu

DEEP_PQ = [(9, 9), (10, 9), (9, 12), (12, 10), (11, 11), (12, 12), (10, 12), (12, 9)]


def deep_graph(seed, nu=80, nv=70, core=(22, 22), dens=0.93, noise=0.1, n_cores=1):
    rng = np.random.default_rng(seed)
    m = rng.random((nu, nv)) < noise
    for _ in range(n_cores):
        cu = rng.choice(nu, core[0], replace=False)
        cv = rng.choice(nv, core[1], replace=False)
        m[np.ix_(cu, cv)] |= rng.random(core) < dens
    i, j = np.nonzero(m)
    return from_edges(nu, nv, i.astype(np.int64), j.astype(np.int64))


def _check(rep, want, tag):
    assert rep.count == want.count, tag
    assert rep.tasks_emitted == want.tasks_emitted, tag
    assert rep.roots_filtered == want.roots_filtered, tag
    assert rep.batches_executed == want.batches_executed, tag
    assert rep.device["operand_words"] == want.operand_words, tag
    assert rep.device["intersections"] == want.intersections, tag


@pytest.mark.parametrize("i,pq", list(enumerate(DEEP_PQ)))
def test_deep_pq_all_paths(i, pq):
    p, q = pq
    g = deep_graph(i)
    for anchor, mode in (("auto", "hybrid"), ("V", "dfs"), ("U", "hybrid")):
        want = O.count(g, p, q, anchor=anchor, mode=mode)
        assert want.count > 0 or anchor != "auto"
        for l1, rows in itertools.product(("scatter", "probe"), ("scatter", "probe")):
            cfg = EngineConfig(anchor=anchor, mode=mode, level1=l1, rows=rows, instrument=True)
            _check(count_bicliques(g, p, q, cfg), want, (p, q, anchor, mode, l1, rows))


@pytest.mark.parametrize("seed", [101, 202, 303])
def test_deep_multi_core_split_and_shards(seed):
    """Several planted cores and a larger noise graph: heavy tasks are split into
    sub-tasks; per-task u128 counts equal the oracle's and shards sum exactly."""
    rng = np.random.default_rng(seed)
    p, q = int(rng.integers(9, 13)), int(rng.integers(9, 13))
    g = deep_graph(seed, nu=160, nv=150, core=(20, 21), dens=0.95, noise=0.05, n_cores=3)
    want = O.count(g, p, q, per_task=True, workers=4)
    dg = DeviceGraph(g)
    try:
        for flags in ({}, {"level1": "probe"}, {"rows": "probe"}):
            rep, per_task = dg.count_raw(p, q, EngineConfig(**flags), task_counts=True)
            got = int(rep.count_lo) | (int(rep.count_hi) << 64)
            assert got == want.count, (seed, p, q, flags)
            assert per_task == want.task_counts
            assert rep.batches_executed == want.batches_executed
        total = 0
        for k in range(4):
            r, _ = dg.count_raw(p, q, EngineConfig(), shard=(k, 4))
            total += int(r.count_lo) | (int(r.count_hi) << 64)
        assert total == want.count
    finally:
        dg.close()


def test_deep_fast_order_matches():
    """(q,p)-core pruning and degree relabelling keep deep counts exact."""
    for i, (p, q) in enumerate(DEEP_PQ[:4]):
        g = deep_graph(50 + i)
        want = O.count(g, p, q).count
        for order in ("fast", "fast-reorder"):
            assert count_bicliques(g, p, q, EngineConfig(order_mode=order)).count == want
