"""GPU parity: the sm_100a path through the C-ABI vs the pinned oracle and
the reference goldens (tests/golden/golden.json).  Bit-exact throughout:
structures, counts, CountReport counters, per-task partial counts and the
reference-equivalent intersection tallies (B_enum / B_min)."""

import hashlib

import numpy as np
import pytest

from oracle import oracle as O
from paper_2403_07858_b200 import (DeviceGraph, EngineConfig, count_bicliques, prepare_structures,
                                   synth)
from paper_2403_07858_b200 import _abi

pytestmark = pytest.mark.gpu

FIELDS = {
    "und_size": lambda s: s.und_sizes, "rank": lambda s: s.order.rank,
    "order": lambda s: s.order.order, "dir_off": lambda s: s.dir2.csr.off,
    "dir_idx": lambda s: s.dir2.csr.idx, "hadj_off": lambda s: s.adj_htb.off,
    "hadj_idx": lambda s: s.adj_htb.idx, "hadj_val": lambda s: s.adj_htb.val,
    "hdir_off": lambda s: s.dir2_htb.off, "hdir_idx": lambda s: s.dir2_htb.idx,
    "hdir_val": lambda s: s.dir2_htb.val, "tasks": lambda s: s.tasks.ravel(),
}


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).astype("<i8").tobytes()).hexdigest()


def check_structures(g, p, q, anchor, rec):
    s = prepare_structures(g, p, q, anchor)
    assert (s.choice.layer, s.choice.p_eff, s.choice.q_eff) == (rec["anchor"], rec["p_eff"], rec["q_eff"])
    for k, h in rec["sha256"].items():
        got = FIELDS[k](s)
        if "arrays" in rec:
            assert np.asarray(got, dtype=np.int64).tolist() == rec["arrays"][k], k
        assert digest(got) == h, k


def check_reports(g, p, q, anchor, recs):
    for mode, r in recs.items():
        rep = count_bicliques(g, p, q, EngineConfig(mode=mode, anchor=anchor))
        assert str(rep.count) == r["count"], (p, q, anchor, mode)
        assert rep.tasks_emitted == r["emitted"]
        assert rep.roots_filtered == r["filtered"]
        assert rep.tasks_consumed == r["consumed"]
        assert rep.batches_executed == r["batches"], (p, q, anchor, mode)
        assert rep.anchor_layer == r["anchor"]


def test_recon(golden):
    g = synth.recon_graph()
    check_structures(g, 3, 2, "U", golden["recon"]["structures_3_2_U"])
    for key, recs in golden["recon"]["reports"].items():
        p, q, anchor = key.split(",")
        check_reports(g, int(p), int(q), anchor, recs)


def test_random_structures_and_reports(golden):
    for c in golden["random"]:
        g = synth.random_bipartite(c["nu"], c["nv"], c["density"], c["seed"])
        check_structures(g, c["p"], c["q"], c["anchor"], c["structures"])
        check_reports(g, c["p"], c["q"], c["anchor"], c["reports"])


def test_medium_and_instrumented_operand_words(golden):
    for c in golden["medium"]:
        g = synth.random_bipartite(c["nu"], c["nv"], c["density"], c["seed"])
        check_structures(g, c["p"], c["q"], "auto", c["structures"])
        check_reports(g, c["p"], c["q"], "auto", c["reports"])
        rep = count_bicliques(g, c["p"], c["q"], EngineConfig(instrument=True))
        ins = c["instrumented"]
        d = rep.device
        assert (d["intersections"], d["operand_words"], d["min_words"]) == (
            ins["intersections"], ins["operand_words"], ins["min_words"])


def test_corpus300(golden):
    corpus = synth.corpus300()
    pq = golden["corpus300"]["pq"]
    for g, row in zip(corpus, golden["corpus300"]["counts"]):
        dg = DeviceGraph(g)
        for (p, q), want in zip(pq, row):
            rep, _ = dg.count_raw(p, q)
            got = int(rep.count_lo) | (int(rep.count_hi) << 64)
            assert str(got) == want, (p, q)
        dg.close()


def test_random_vs_oracle_dense():
    """Wider/deeper searches than the corpus: p, q up to 7, both anchors, both modes."""
    rng = np.random.default_rng(7)
    for i in range(40):
        nu, nv = int(rng.integers(20, 120)), int(rng.integers(20, 120))
        g = synth.random_bipartite(nu, nv, float(rng.uniform(0.1, 0.45)), int(rng.integers(1 << 30)))
        p, q = int(rng.integers(2, 8)), int(rng.integers(2, 8))
        anchor = ["auto", "U", "V"][i % 3]
        mode = ["hybrid", "dfs"][i % 2]
        cap = [4096, 64, 7][i % 3]
        want = O.count(g, p, q, anchor=anchor, mode=mode, capacity=max(cap, 64))
        rep = count_bicliques(g, p, q, EngineConfig(anchor=anchor, mode=mode,
                                                    batch_buffer_capacity=max(cap, 64),
                                                    instrument=True))
        assert rep.count == want.count, (i, p, q)
        assert rep.batches_executed == want.batches_executed, (i, p, q)
        assert rep.tasks_emitted == want.tasks_emitted
        assert rep.device["operand_words"] == want.operand_words
        assert rep.device["intersections"] == want.intersections


def test_per_task_counts_and_shards():
    g = synth.build_config("C4")
    want = O.count(g, 8, 8, per_task=True, workers=8)
    dg = DeviceGraph(g)
    rep, per_task = dg.count_raw(8, 8, task_counts=True)
    assert per_task == want.task_counts
    total = 0
    for k in range(3):
        r, _ = dg.count_raw(8, 8, shard=(k, 3))
        total += int(r.count_lo) | (int(r.count_hi) << 64)
    assert total == want.count
    dg.close()


def test_roots_and_rank_override():
    g = synth.random_bipartite(60, 50, 0.3, 41)
    total = count_bicliques(g, 3, 3, EngineConfig(anchor="U")).count
    a = count_bicliques(g, 3, 3, EngineConfig(anchor="U"), roots=range(0, 30)).count
    b = count_bicliques(g, 3, 3, EngineConfig(anchor="U"), roots=range(30, 60)).count
    assert a + b == total == O.count(g, 3, 3, anchor="U").count
    rank = np.random.default_rng(1).permutation(60) + 1
    s = prepare_structures(g, 3, 3, "U", rank=rank)
    assert np.array_equal(s.order.rank, rank)
    assert count_bicliques(g, 3, 3, EngineConfig(anchor="U"), structures=s).count == total
    with pytest.raises(ValueError):
        prepare_structures(g, 3, 3, "U", rank=np.ones(60, dtype=np.int64))


def test_errors_match_reference():
    g = synth.random_bipartite(200, 200, 0.2, 9)
    with pytest.raises(ValueError, match="batch-words"):
        count_bicliques(g, 2, 2, EngineConfig(batch_buffer_capacity=2))
    assert count_bicliques(synth.recon_graph(), 5, 2, EngineConfig(anchor="U")).count == 0
    empty = synth.from_edges(5, 3, [], [])
    assert count_bicliques(empty, 2, 2).count == 0


@pytest.mark.parametrize("name,p,q", [("C1", 2, 2), ("C3", 3, 6), ("C3", 6, 3), ("C4", 8, 8),
                                      ("C2", 4, 4)])
def test_configs(golden, name, p, q):
    g = synth.build_config(name)
    cf = golden["configs"][name]
    check_structures(g, p, q, "auto", cf[f"structures_({p},{q})"])
    key = f"({p},{q})"
    want = cf[key]["hybrid"] if key in cf else None
    ref = O.count(g, p, q, workers=8)
    rep = count_bicliques(g, p, q, EngineConfig(instrument=True))
    assert rep.count == ref.count
    if want:
        assert str(rep.count) == want["count"]
        assert rep.batches_executed == want["batches"]
        assert rep.tasks_emitted == want["emitted"] and rep.roots_filtered == want["filtered"]
    assert rep.batches_executed == ref.batches_executed
    assert rep.device["intersections"] == ref.intersections
    assert rep.device["operand_words"] == ref.operand_words
    assert rep.device["min_words"] == ref.min_words


def test_library_is_the_path():
    """The count came from the .so: the ABI reports kernel launches."""
    rep = count_bicliques(synth.build_config("C1"), 2, 2)
    assert rep.count == 2482
    assert rep.device["kernel_launches"] > 0
    assert _abi.load().bc_device_count() >= 1
