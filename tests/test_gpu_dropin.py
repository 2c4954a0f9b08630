"""Drop-in contract of ``count_bicliques`` beyond the count: the reference's own
assertions on ``track_tasks`` / ``task_tally`` / ``task_counts``, ``check_nesting``,
``wall_time`` and enumeration together with ``roots=`` / ``structures=``, restated
against this package (reference ``pkg/tests/test_engine.py:234-284``,
``test_acceptance.py:140-155``, ``engine.py:419-500``)."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2403_07858_b200 import EngineConfig, count_bicliques, prepare_structures, synth

pytestmark = pytest.mark.gpu


def brute_pairs(g, p, q):
    """Every (L, R) biclique of g, sorted: the reference's oracle.enumerate_bicliques."""
    from itertools import combinations

    adj = [set(g.u_csr.row(u).tolist()) for u in range(g.u_count)]
    out = []
    for L in combinations(range(g.u_count), p):
        common = set.intersection(*(adj[u] for u in L)) if L else set()
        for R in combinations(sorted(common), q):
            out.append((L, R))
    return sorted(out)


def test_nesting_assert_mode_runs_clean():
    # test_engine.py:234-237, plus the device's tally of checked ids
    g = synth.random_bipartite(15, 15, 0.4, 31)
    rep = count_bicliques(g, 4, 2, EngineConfig(check_nesting=True))
    assert rep.count == O.brute_force_count(g, 4, 2)
    for seed in (3, 4, 5):
        g = synth.random_bipartite(40, 36, 0.5, seed)
        for anchor in ("U", "V"):  # p_eff 5 / 4: both descend below level 2
            rep = count_bicliques(g, 5, 4, EngineConfig(check_nesting=True, anchor=anchor))
            assert rep.count == O.count(g, 5, 4, anchor=anchor).count > 0
            assert rep.device["nesting_checked"] > 0


def test_workers_agree_and_tally_exactly_once():
    # test_engine.py:240-252: exactly-once claims through the device claim log
    g = synth.random_bipartite(40, 40, 0.25, 77)
    base = count_bicliques(g, 3, 2, EngineConfig(worker_count=1, track_tasks=True))
    assert base.task_tally == [(0, i) for i in range(base.tasks_emitted)]
    assert base.task_counts == [base.tasks_emitted]
    for w in (2, 4):
        rep = count_bicliques(g, 3, 2, EngineConfig(worker_count=w, track_tasks=True))
        assert rep.count == base.count
        assert rep.tasks_consumed == rep.tasks_emitted == base.tasks_emitted
        assert len(rep.task_tally) == rep.tasks_emitted
        assert set(rep.task_tally) == {
            (e, i) for e, n in enumerate(rep.task_counts) for i in range(n)}


@pytest.mark.parametrize("name,p,q", [("C4", 8, 8), ("C3", 6, 3), ("C1", 2, 2)])
def test_tally_exactly_once_on_configs(golden, name, p, q):
    """Criterion 5 (test_acceptance.py:140-155) on every kernel path the configs take:
    each emitted task is claimed exactly once (split, triage and whole-task paths)."""
    g = synth.build_config(name)
    for w in (1, 8):
        r = count_bicliques(g, p, q, EngineConfig(worker_count=w, track_tasks=True))
        assert str(r.count) == golden["configs"][name][f"({p},{q})"]["hybrid"]["count"]
        want = [(e, i) for e in range(len(r.task_counts)) for i in range(r.task_counts[e])]
        assert sorted(r.task_tally) == want
        assert r.tasks_consumed == r.tasks_emitted


def test_p1_tally():
    g = synth.random_bipartite(30, 20, 0.3, 2)
    r = count_bicliques(g, 1, 3, EngineConfig(track_tasks=True, anchor="U"))
    assert r.task_tally == [(0, i) for i in range(r.tasks_emitted)] and r.tasks_emitted == 30
    assert r.count == O.brute_force_count(g, 1, 3)


def test_wall_time_is_counting_phase():
    g = synth.build_config("C3")
    r = count_bicliques(g, 6, 3)
    assert r.wall_time == pytest.approx(r.time_1hop + r.time_2hop)
    assert 0 < r.wall_time < r.device["time_total"]
    assert r.device["time_prep"] > 0


def test_root_restriction_splits_count():
    # test_engine.py:261-269 through the drop-in's structures= / roots=
    g = synth.random_bipartite(16, 16, 0.35, 41)
    s = prepare_structures(g, 3, 2, anchor="U")
    total = count_bicliques(g, 3, 2, EngineConfig(anchor="U"), structures=s).count
    a = count_bicliques(g, 3, 2, EngineConfig(anchor="U"), structures=s, roots=range(0, 8)).count
    b = count_bicliques(g, 3, 2, EngineConfig(anchor="U"), structures=s, roots=range(8, 16)).count
    assert a + b == total == O.brute_force_count(g, 3, 2)


def test_rank_override_changes_order_not_count():
    # test_engine.py:272-278
    g = synth.random_bipartite(12, 12, 0.4, 53)
    want = O.brute_force_count(g, 2, 2)
    rank = np.random.default_rng(1).permutation(12) + 1
    s = prepare_structures(g, 2, 2, anchor="U", rank=rank)
    assert count_bicliques(g, 2, 2, EngineConfig(anchor="U"), structures=s).count == want


@pytest.mark.parametrize("anchor", ["U", "V"])
def test_enumeration_with_roots_and_structures(anchor):
    """Enumeration together with roots= / structures= (engine.py:480-483): the root-
    restricted enumerations partition the whole set, and a V-anchored structures= run
    is normalised back to (L, R) of the caller's graph."""
    g = synth.random_bipartite(12, 13, 0.45, 9)
    p, q = 3, 2
    want = brute_pairs(g, p, q)
    s = prepare_structures(g, p, q, anchor=anchor)
    cfg = EngineConfig(enumerate_results=True, anchor=anchor)
    whole = count_bicliques(g, p, q, cfg, structures=s)
    assert whole.bicliques == want and whole.count == len(want)
    n = s.work.u_count
    parts = []
    for lo, hi in ((0, n // 2), (n // 2, n)):
        r = count_bicliques(g, p, q, cfg, structures=s, roots=range(lo, hi))
        assert r.count == len(r.bicliques)
        parts += r.bicliques
    assert sorted(parts) == want
    r = count_bicliques(g, p, q, EngineConfig(enumerate_results=True, anchor=anchor),
                        roots=range(0, 5))
    assert r.count == len(r.bicliques) and set(r.bicliques) <= set(want)


@pytest.mark.parametrize("devs", [(0, 0), (0, 0, 0)])
def test_one_call_over_several_devices(golden, devs):
    """The reference's in-call parallelism (engine.py:449-478: one count_bicliques call,
    several workers) as EngineConfig(devices=...): a host thread per listed GPU counts its
    shard and the call sums the exact partials.  Only one GPU is reachable here, so the
    shards share device 0 (the library serialises calls per device); the merge, the
    counters and the claim log are what is checked."""
    for name, (p, q) in (("C4", (8, 8)), ("C3", (6, 3)), ("C1", (2, 2))):
        g = synth.build_config(name)
        want = golden["configs"][name][f"({p},{q})"]["hybrid"]
        rep = count_bicliques(g, p, q, EngineConfig(devices=devs, track_tasks=True))
        assert str(rep.count) == want["count"], name
        assert rep.batches_executed == want["batches"], name
        assert rep.tasks_emitted == want["emitted"]
        assert rep.tasks_consumed == want["emitted"]  # every task by exactly one shard
        assert sorted(rep.task_tally) == [(0, i) for i in range(want["emitted"])]
    with pytest.raises(ValueError):
        EngineConfig(devices=()).validate()


def test_shutdown_releases_cache_and_counts_again(golden):
    """bc_shutdown hands the library pools' cached scratch back to the device; a live graph
    keeps working and later calls re-reserve (same counts)."""
    from paper_2403_07858_b200 import DeviceGraph, _abi

    g = synth.build_config("C4")
    want = golden["configs"]["C4"]["(8,8)"]["hybrid"]["count"]
    dg = DeviceGraph(g)
    try:
        r1, _ = dg.count_raw(8, 8)
        _abi.load().bc_shutdown()
        r2, _ = dg.count_raw(8, 8)
    finally:
        dg.close()
    assert str(int(r1.count_lo) | (int(r1.count_hi) << 64)) == want
    assert str(int(r2.count_lo) | (int(r2.count_hi) << 64)) == want
    assert str(count_bicliques(g, 8, 8).count) == want
