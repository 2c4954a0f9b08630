"""GPU parity of the alternative kernel paths the library picks by cost estimate:
level 1 by root-grouped wedge scatter vs per-task HTB intersections, and
candidate rows by wedge scatter vs per-candidate probes.  Every combination
must give the oracle's exact count, CountReport counters, batch accounting and
reference-equivalent intersection tallies (B_enum), and shard sums must add up.
"""

import itertools

import numpy as np
import pytest

from oracle import oracle as O
from paper_2403_07858_b200 import DeviceGraph, EngineConfig, count_bicliques, synth

pytestmark = pytest.mark.gpu

COMBOS = list(itertools.product(("scatter", "probe"), ("scatter", "probe")))


def _cfg(l1, rows, **kw):
    return EngineConfig(level1=l1, rows=rows, **kw)


@pytest.mark.parametrize("l1,rows", COMBOS)
def test_random_graphs_all_paths(l1, rows):
    rng = np.random.default_rng(11)
    for i in range(30):
        nu, nv = int(rng.integers(20, 140)), int(rng.integers(20, 140))
        g = synth.random_bipartite(nu, nv, float(rng.uniform(0.08, 0.45)), int(rng.integers(1 << 30)))
        p, q = int(rng.integers(2, 9)), int(rng.integers(2, 8))
        anchor = ["auto", "U", "V"][i % 3]
        mode = ["hybrid", "dfs"][i % 2]
        want = O.count(g, p, q, anchor=anchor, mode=mode)
        rep = count_bicliques(g, p, q, _cfg(l1, rows, anchor=anchor, mode=mode, instrument=True))
        assert rep.count == want.count, (i, p, q, l1, rows)
        assert rep.batches_executed == want.batches_executed, (i, p, q)
        assert rep.tasks_emitted == want.tasks_emitted
        assert rep.roots_filtered == want.roots_filtered
        assert rep.device["operand_words"] == want.operand_words
        assert rep.device["intersections"] == want.intersections


@pytest.mark.parametrize("name,p,q", [("C3", 3, 6), ("C3", 6, 3), ("C4", 8, 8), ("C1", 2, 2)])
@pytest.mark.parametrize("l1,rows", [("scatter", "scatter"), ("probe", "scatter"),
                                     ("scatter", "probe")])
def test_configs_alt_paths(golden, name, p, q, l1, rows):
    g = synth.build_config(name)
    want = golden["configs"][name][f"({p},{q})"]["hybrid"]
    rep = count_bicliques(g, p, q, _cfg(l1, rows))
    assert str(rep.count) == want["count"]
    assert rep.batches_executed == want["batches"]
    assert rep.tasks_emitted == want["emitted"]


def test_scatter_shards_and_task_counts():
    g = synth.build_config("C4")
    want = O.count(g, 8, 8, per_task=True, workers=8)
    dg = DeviceGraph(g)
    cfg = _cfg("scatter", "scatter")
    rep, per_task = dg.count_raw(8, 8, cfg, task_counts=True)
    assert per_task == want.task_counts
    total = 0
    for k in range(3):
        r, _ = dg.count_raw(8, 8, cfg, shard=(k, 3))
        total += int(r.count_lo) | (int(r.count_hi) << 64)
    assert total == want.count
    dg.close()


@pytest.mark.parametrize("order", ["fast", "fast-reorder"])
def test_fast_order_counts(golden, order):
    """(q,p)-core pruning (+ degree relabel): same exact counts as the reference order
    on random graphs (all anchors, both modes), corpus300 and the C1-C4 configs."""
    rng = np.random.default_rng(5)
    for i in range(40):
        nu, nv = int(rng.integers(10, 140)), int(rng.integers(10, 140))
        g = synth.random_bipartite(nu, nv, float(rng.uniform(0.05, 0.45)), int(rng.integers(1 << 30)))
        p, q = int(rng.integers(1, 9)), int(rng.integers(1, 8))
        anchor = ["auto", "U", "V"][i % 3]
        want = O.count(g, p, q, anchor=anchor).count
        for rows in ("probe", "scatter"):
            rep = count_bicliques(g, p, q, EngineConfig(anchor=anchor, order_mode=order, rows=rows,
                                                        mode=["hybrid", "dfs"][i % 2]))
            assert rep.count == want, (i, p, q, anchor, order, rows)
    corpus = synth.corpus300()[:60]
    pq = golden["corpus300"]["pq"]
    for g, row in zip(corpus, golden["corpus300"]["counts"]):
        dg = DeviceGraph(g)
        for (p, q), want in zip(pq, row):
            r, _ = dg.count_raw(p, q, EngineConfig(order_mode=order))
            assert str(int(r.count_lo) | (int(r.count_hi) << 64)) == want, (p, q)
        dg.close()
    for name, (p, q) in [("C1", (2, 2)), ("C3", (3, 6)), ("C3", (6, 3)), ("C4", (8, 8))]:
        g = synth.build_config(name)
        want = golden["configs"][name][f"({p},{q})"]["hybrid"]["count"]
        dg = DeviceGraph(g)
        r, _ = dg.count_raw(p, q, EngineConfig(order_mode=order))
        assert str(int(r.count_lo) | (int(r.count_hi) << 64)) == want, (name, order)
        total = 0
        for k in range(3):
            rr, _ = dg.count_raw(p, q, EngineConfig(order_mode=order), shard=(k, 3))
            total += int(rr.count_lo) | (int(rr.count_hi) << 64)
        assert str(total) == want
        dg.close()


def test_fast_order_rejects_reference_only_inputs():
    g = synth.random_bipartite(40, 40, 0.3, 3)
    with pytest.raises(ValueError):
        count_bicliques(g, 3, 3, EngineConfig(order_mode="fast"), roots=[0, 1])


@pytest.mark.parametrize("shard_mode", ["root", "task"])
def test_shard_modes_sum_to_total(shard_mode):
    """Both multi-GPU shard rules (whole roots dealt degree-balanced; task interleave)
    partition the tasks: per-shard counts and consumed tasks add up, on every path."""
    for name, (p, q) in [("C4", (8, 8)), ("C3", (6, 3)), ("C1", (2, 2))]:
        g = synth.build_config(name)
        dg = DeviceGraph(g)
        full, _ = dg.count_raw(p, q)
        total = int(full.count_lo) | (int(full.count_hi) << 64)
        for n in (2, 3, 8):
            parts = consumed = 0
            for k in range(n):
                r, _ = dg.count_raw(p, q, EngineConfig(shard_mode=shard_mode), shard=(k, n))
                parts += int(r.count_lo) | (int(r.count_hi) << 64)
                consumed += r.tasks_consumed
            assert parts == total, (name, n, shard_mode)
            assert consumed == full.tasks_consumed
        dg.close()


def test_u128_counts_and_overflow():
    """Complete bipartite graphs: counts above 2^64 are exact (u128 accumulation, limb
    reduction), a count of 2^128 or more is an error, never a wrapped value."""
    from math import comb

    nu = nv = 200
    k = np.arange(nu * nv)
    g = synth.from_edges(nu, nv, k // nv, k % nv)
    want = comb(nu, 2) * comb(nv, 20)
    assert want > 2**64
    assert count_bicliques(g, 2, 20).count == want
    with pytest.raises(RuntimeError):
        count_bicliques(g, 2, 40)  # C(200,2) * C(200,40) > 2^128


@pytest.mark.parametrize("p", [1, 2])
def test_u128_sum_overflow_of_small_terms(p):
    """Every term C(131, 65) < 2^128, but three of them pass 2^128: the per-warp and
    global 128-bit sums must report the overflow, not wrap (K_{3,131})."""
    from math import comb

    nu, nv = 3, 131
    k = np.arange(nu * nv)
    g = synth.from_edges(nu, nv, k // nv, k % nv)
    assert comb(131, 65) < 2**128 <= 3 * comb(131, 65)
    with pytest.raises(RuntimeError, match="128 bits"):
        count_bicliques(g, p, 65, EngineConfig(anchor="U"))
    g1 = synth.from_edges(1, nv, np.zeros(nv, np.int64), np.arange(nv))
    assert count_bicliques(g1, 1, 65, EngineConfig(anchor="U")).count == comb(131, 65)


def test_enumeration_matches_brute_force():
    """enumerate_results (reference engine.py:301-304, 480-483): the device search emits
    every biclique; sorted (L, R) pairs equal an independent brute-force enumeration,
    for both anchors and p_eff 1..4."""
    from itertools import combinations

    def brute(g, p, q):
        uo, ui = g.u_csr.off, g.u_csr.idx
        rows = [frozenset(ui[uo[i]:uo[i + 1]].tolist()) for i in range(g.u_count)]
        out = []
        for L in combinations(range(g.u_count), p):
            common = frozenset.intersection(*(rows[u] for u in L))
            for R in combinations(sorted(common), q):
                out.append((L, R))
        return sorted(out)

    g = synth.recon_graph()
    rep = count_bicliques(g, 3, 2, EngineConfig(enumerate_results=True, anchor="U"))
    assert rep.bicliques == [((0, 1, 2), (1, 2)), ((0, 1, 3), (0, 2))]  # test_engine.py:42-46
    for seed, (nu, nv) in enumerate([(9, 9), (8, 10), (12, 7)]):
        g = synth.random_bipartite(nu, nv, 0.4, seed + 5)
        for p, q in ((1, 2), (2, 2), (3, 2), (2, 3), (4, 2), (2, 4)):
            want = brute(g, p, q)
            for anchor in ("U", "V", "auto"):
                rep = count_bicliques(g, p, q, EngineConfig(enumerate_results=True, anchor=anchor))
                assert rep.bicliques == want, (seed, p, q, anchor)
                assert rep.count == len(want)


def test_wide_counters_and_light_boundaries():
    """2-hop multiplicities past the 16-bit counters (k > 60000: 32-bit tile counters, no
    light path) and anchors whose wedge pools straddle the light-kernel bound (1024)."""
    from math import comb

    nu, nv = 3, 60005
    k = np.arange(nu * nv)
    g = synth.from_edges(nu, nv, k // nv, k % nv)
    rep = count_bicliques(g, 2, 60001, EngineConfig(anchor="U"))
    assert rep.count == comb(3, 2) * comb(nv, 60001)
    # stars of growing size around shared centres: pools 1000..1100 per anchor
    rng = np.random.default_rng(2)
    for deg in (31, 32, 33, 64):
        eu, ev = [], []
        for u in range(40):
            vs = rng.choice(200, size=deg, replace=False)
            eu += [u] * deg
            ev += vs.tolist()
        g = synth.from_edges(40, 200, eu, ev)
        for p, q in ((2, 3), (3, 2), (3, 3)):
            want = O.count(g, p, q, anchor="U")
            got = count_bicliques(g, p, q, EngineConfig(anchor="U"))
            assert got.count == want.count and got.batches_executed == want.batches_executed


def test_degenerate_inputs():
    """Empty layers, isolated vertices, p or q above every degree: the reference's counts
    and counters (all zero or filtered) without a device error."""
    cases = [synth.from_edges(0, 0, [], []), synth.from_edges(5, 0, [], []),
             synth.from_edges(0, 7, [], []), synth.from_edges(4, 4, [0], [0]),
             synth.from_edges(6, 5, [0, 1, 2], [0, 0, 0])]
    for g in cases:
        for p, q in ((1, 1), (2, 2), (3, 1), (1, 4), (5, 5)):
            for anchor in ("auto", "U", "V"):
                want = O.count(g, p, q, anchor=anchor)
                got = count_bicliques(g, p, q, EngineConfig(anchor=anchor))
                assert got.count == want.count, (p, q, anchor)
                assert got.tasks_emitted == want.tasks_emitted
                assert got.roots_filtered == want.roots_filtered
                assert got.batches_executed == want.batches_executed


@pytest.mark.parametrize("name,p,q", [("C2", 4, 4), ("C4", 8, 8), ("C3", 6, 3), ("C1", 2, 2)])
def test_sharded_preprocessing(golden, name, p, q):
    """Sharded 2-hop construction: the shards' upper-list slices partition the anchors,
    their assembly equals the one-shard slice, and counting with the injected lists gives
    the reference's count, batches and tasks, whole and per task shard."""
    import torch

    from paper_2403_07858_b200.engine import assemble_upper

    g = synth.build_config(name)
    want = golden["configs"][name][f"({p},{q})"]["hybrid"]
    dg = DeviceGraph(g)
    whole = assemble_upper([dg.twohop_slice(p, q)])
    for n in (2, 3, 8):
        sl = [dg.twohop_slice(p, q, shard=(k, n)) for k in range(n)]
        owned = torch.stack([(x[0] > 0).to(torch.int32) for x in sl]).sum(0)
        assert int(owned.max().item()) <= 1
        off, ids = assemble_upper(sl)
        assert torch.equal(off, whole[0]) and torch.equal(ids, whole[1])
        total = 0
        for k in range(n):
            r, _ = dg.count_raw(p, q, shard=(k, n), upper=(off, ids))
            total += int(r.count_lo) | (int(r.count_hi) << 64)
        assert str(total) == want["count"]
    r, _ = dg.count_raw(p, q, upper=whole)
    assert str(int(r.count_lo) | (int(r.count_hi) << 64)) == want["count"]
    assert r.batches_executed == want["batches"] and r.tasks_emitted == want["emitted"]
    dg.close()


def test_assemble_upper_device_matches_host():
    import torch

    from paper_2403_07858_b200.engine import assemble_upper, assemble_upper_device

    g = synth.build_config("C3")
    dg = DeviceGraph(g)
    for n in (1, 3, 8):
        sl = [dg.twohop_slice(6, 3, shard=(k, n)) for k in range(n)]
        stride = max(max(x[1].numel() for x in sl), 1)
        ids_all = torch.zeros(n * stride, dtype=torch.int32, device="cuda")
        for k, x in enumerate(sl):
            ids_all[k * stride:k * stride + x[1].numel()] = x[1]
        off, ids = assemble_upper_device(torch.cat([x[0] for x in sl]), ids_all, stride,
                                         sum(x[1].numel() for x in sl), world=n)
        off2, ids2 = assemble_upper(sl)
        assert torch.equal(off, off2) and torch.equal(ids, ids2)
    dg.close()


# The survivor filter + triage path (chosen by size for C5-scale task counts) forced on
# small graphs, with the root-restricted rows (rank-position filter) and with whole
# opposite-layer rows: exact counts, per-task counts, batches and shard sums.
TRIAGE_PATHS = [dict(force_triage=True),
                dict(force_triage=True, restricted_rows=False),
                dict(force_triage=True, level1="scatter", rows="scatter"),
                dict(force_triage=True, level1="probe", rows="scatter"),
                dict(force_triage=True, level1="scatter", rows="probe"),
                dict(restricted_rows=False)]


@pytest.mark.parametrize("kw", TRIAGE_PATHS)
def test_forced_triage_paths_random_deep(kw):
    rng = np.random.default_rng(29)
    for i in range(9):
        nu, nv = int(rng.integers(40, 100)), int(rng.integers(40, 100))
        g = synth.random_bipartite(nu, nv, float(rng.uniform(0.15, 0.4)), int(rng.integers(1 << 30)))
        p, q = int(rng.integers(5, 9)), int(rng.integers(2, 6))
        anchor = ["auto", "U", "V"][i % 3]
        want = O.count(g, p, q, anchor=anchor, per_task=True)
        dg = DeviceGraph(g)
        try:
            cfg = EngineConfig(anchor=anchor, **kw)
            rep, per_task = dg.count_raw(p, q, cfg, task_counts=True)
            got = int(rep.count_lo) | (int(rep.count_hi) << 64)
            assert got == want.count, (i, p, q, kw)
            assert per_task == want.task_counts, (i, p, q, kw)
            assert rep.batches_executed == want.batches_executed, (i, p, q, kw)
            assert rep.tasks_emitted == want.tasks_emitted
            total = 0
            for k in range(3):
                r, _ = dg.count_raw(p, q, cfg, shard=(k, 3))
                total += int(r.count_lo) | (int(r.count_hi) << 64)
            assert total == want.count, (i, p, q, kw)
        finally:
            dg.close()


@pytest.mark.parametrize("name,p,q", [("C3", 6, 3), ("C4", 8, 8)])
@pytest.mark.parametrize("kw", TRIAGE_PATHS[:2])
def test_forced_triage_configs(golden, name, p, q, kw):
    g = synth.build_config(name)
    want = golden["configs"][name][f"({p},{q})"]["hybrid"]
    rep = count_bicliques(g, p, q, EngineConfig(**kw))
    assert str(rep.count) == want["count"]
    assert rep.batches_executed == want["batches"]
    assert rep.tasks_emitted == want["emitted"]


@pytest.mark.parametrize("kw", TRIAGE_PATHS[:3])
def test_rank_override_any_values_on_restricted_rows(kw):
    """A rank override (a partitioned count passes the full graph's ranks, partition.py:
    246-249) may hold any distinct int64s: the restricted rows' rank positions must follow
    their order, not their magnitude.  Order-preserving rescalings of the reference rank
    (large, negative) give the reference's counts, batches and per-task counts."""
    rng = np.random.default_rng(41)
    for i in range(4):
        g = synth.random_bipartite(int(rng.integers(60, 110)), int(rng.integers(60, 110)),
                                   float(rng.uniform(0.2, 0.4)), int(rng.integers(1 << 30)))
        p, q = int(rng.integers(5, 8)), int(rng.integers(2, 5))
        prep = O.Prepared(g, p, q, anchor="U")
        rank = prep.export(O.X_RANK).astype(np.int64)
        want = O.count(g, p, q, anchor="U", per_task=True)
        dg = DeviceGraph(g)
        try:
            for rk in (rank * 1_000_003 + 7, rank - 10**15):
                rep, per_task = dg.count_raw(p, q, EngineConfig(anchor="U", **kw), rank=rk,
                                             task_counts=True)
                got = int(rep.count_lo) | (int(rep.count_hi) << 64)
                assert got == want.count, (i, p, q, kw)
                assert per_task == want.task_counts, (i, p, q, kw)
                assert rep.batches_executed == want.batches_executed, (i, p, q, kw)
        finally:
            dg.close()
