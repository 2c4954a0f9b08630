"""Pin the CPU oracle (oracle/) to the reference's own outputs (CPU only).

Every fixture in tests/golden/golden.json was produced by running the
reference package (tests/golden/make_golden.py); the oracle must reproduce
structures bit for bit and every CountReport field the reference makes
deterministic.  The GPU parity tests then compare the device against this
pinned oracle.
"""

import hashlib

import numpy as np
import pytest

from oracle import oracle as O
from paper_2403_07858_b200 import synth

EXPORTS = {
    "und_size": O.X_UND_SIZE, "rank": O.X_RANK, "order": O.X_ORDER, "dir_off": O.X_DIR_OFF,
    "dir_idx": O.X_DIR_IDX, "hadj_off": O.X_HADJ_OFF, "hadj_idx": O.X_HADJ_IDX,
    "hadj_val": O.X_HADJ_VAL, "hdir_off": O.X_HDIR_OFF, "hdir_idx": O.X_HDIR_IDX,
    "hdir_val": O.X_HDIR_VAL,
}


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).astype("<i8").tobytes()).hexdigest()


def oracle_arrays(g, p, q, anchor="auto"):
    s = O.Prepared(g, p, q, anchor)
    arr = {k: s.export(w) for k, w in EXPORTS.items()}
    arr["tasks"] = O.tasks(s).ravel()
    return s, arr


def check_structures(g, p, q, anchor, rec):
    s, arr = oracle_arrays(g, p, q, anchor)
    assert s.anchor == rec["anchor"] and s.p_eff == rec["p_eff"] and s.q_eff == rec["q_eff"]
    for k, h in rec["sha256"].items():
        assert digest(arr[k]) == h, k
    if "arrays" in rec:
        for k, v in rec["arrays"].items():
            assert np.asarray(arr[k], dtype=np.int64).tolist() == v, k


def check_reports(g, p, q, anchor, recs, workers=1):
    for mode, r in recs.items():
        got = O.count(g, p, q, mode=mode, anchor=anchor, workers=workers)
        assert str(got.count) == r["count"]
        assert got.tasks_emitted == r["emitted"]
        assert got.roots_filtered == r["filtered"]
        assert got.tasks_consumed == r["consumed"]
        assert got.batches_executed == r["batches"]
        assert got.anchor_layer == r["anchor"]


def test_htb_goldens(golden):
    h = golden["htb"]
    # set A as row 0 and set B as row 1 of the anchor layer
    g = synth.from_edges(2, 128, [0] * len(h["set_a"]) + [1] * len(h["set_b"]),
                         h["set_a"] + h["set_b"])
    s = O.Prepared(g, 1, 1, "U")
    off, idx, val = s.export(O.X_HADJ_OFF), s.export(O.X_HADJ_IDX), s.export(O.X_HADJ_VAL)
    assert idx[off[0]:off[1]].tolist() == h["a_idx"] == [0, 2]
    assert val[off[0]:off[1]].tolist() == h["a_val"] == [132360, 295424]
    assert idx[off[1]:off[2]].tolist() == h["b_idx"]
    assert val[off[1]:off[2]].tolist() == h["b_val"] == [8389640, 64]
    # intersection {3,10}: both rows share exactly these two V neighbours -> (2,2) count 1
    assert O.count(g, 2, 2, anchor="U").count == 1
    assert h["isect_ids"] == [3, 10] and h["isect_val"] == [1032]


def test_recon_structures_and_trace(golden):
    g = synth.recon_graph()
    rec = golden["recon"]["structures_3_2_U"]
    check_structures(g, 3, 2, "U", rec)
    a = rec["arrays"]
    # SURVEY Appendix C trace
    assert a["rank"] == [4, 3, 2, 1]
    assert a["hadj_val"] == [7, 23, 14, 29]
    assert a["hdir_val"] == [14, 12, 8]
    assert a["tasks"] == [0, 1, 0, 2, 0, 3, 1, 2, 1, 3, 2, 3]


def test_recon_reports(golden):
    g = synth.recon_graph()
    for key, recs in golden["recon"]["reports"].items():
        p, q, anchor = key.split(",")
        check_reports(g, int(p), int(q), anchor, recs)
    assert O.count(g, 3, 2).count == 2
    assert O.count(g, 2, 2).count == 10
    assert O.count(g, 1, 2).count == 18
    assert O.count(g, 1, 1).count == 14


def test_random_structures_and_reports(golden):
    for c in golden["random"]:
        g = synth.random_bipartite(c["nu"], c["nv"], c["density"], c["seed"])
        check_structures(g, c["p"], c["q"], c["anchor"], c["structures"])
        check_reports(g, c["p"], c["q"], c["anchor"], c["reports"])


def test_medium_structures_reports_and_operand_bytes(golden):
    for c in golden["medium"]:
        g = synth.random_bipartite(c["nu"], c["nv"], c["density"], c["seed"])
        check_structures(g, c["p"], c["q"], "auto", c["structures"])
        check_reports(g, c["p"], c["q"], "auto", c["reports"])
        r = O.count(g, c["p"], c["q"])
        ins = c["instrumented"]
        assert (r.intersections, r.operand_words, r.min_words) == (
            ins["intersections"], ins["operand_words"], ins["min_words"])


def test_corpus300_counts(golden):
    corpus = synth.corpus300()
    pq = golden["corpus300"]["pq"]
    for g, row in zip(corpus, golden["corpus300"]["counts"]):
        for (p, q), want in zip(pq, row):
            assert str(O.count(g, p, q).count) == want


def test_brute_restatement(golden):
    corpus = synth.corpus300()[:20]
    pq = golden["corpus300"]["pq"]
    for g, row, eng in zip(corpus, golden["corpus300"]["brute_first20"], golden["corpus300"]["counts"]):
        for (p, q), want, e in zip(pq, row, eng):
            assert str(O.brute_force_count(g, p, q)) == want == e
            cf = O.closed_form_count(g, p, q)
            if cf is not None:
                assert str(cf) == want


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_config_fingerprints(golden, name):
    g = synth.build_config(name)
    assert g.fingerprint() == synth.FINGERPRINTS[name] == golden["configs"][name]["fingerprint"]


def test_config_structures(golden):
    for name, keys in [("C1", [("structures_(2,2)", 2, 2)]),
                       ("C3", [("structures_(3,6)", 3, 6), ("structures_(6,3)", 6, 3)]),
                       ("C2", [("structures_(4,4)", 4, 4)]),
                       ("C4", [("structures_(8,8)", 8, 8)])]:
        g = synth.build_config(name)
        for key, p, q in keys:
            check_structures(g, p, q, "auto", golden["configs"][name][key])


def test_config_counts(golden):
    cf = golden["configs"]
    g1 = synth.build_config("C1")
    check_reports(g1, 2, 2, "auto", cf["C1"]["(2,2)"])
    r = O.count(g1, 2, 2)
    ins = cf["C1"]["instrumented_(2,2)"]
    assert (r.intersections, r.operand_words, r.min_words) == (
        ins["intersections"], ins["operand_words"], ins["min_words"])
    g3 = synth.build_config("C3")
    r = O.count(g3, 3, 6, workers=4)
    ins = cf["C3"]["instrumented_(3,6)"]
    assert str(r.count) == cf["C3"]["(3,6)"]["hybrid"]["count"] == ins["count"]
    assert r.batches_executed == cf["C3"]["(3,6)"]["hybrid"]["batches"]
    assert (r.intersections, r.operand_words, r.min_words) == (
        ins["intersections"], ins["operand_words"], ins["min_words"])
    for name, key, p, q in [("C2", "(4,4)", 4, 4), ("C3", "(6,3)", 6, 3), ("C4", "(8,8)", 8, 8)]:
        if key not in cf[name]:
            pytest.skip("heavy reference goldens not generated")
        g = synth.build_config(name)
        r = O.count(g, p, q, workers=8)
        want = cf[name][key]["hybrid"]
        assert str(r.count) == want["count"]
        assert (r.tasks_emitted, r.roots_filtered, r.batches_executed, r.tasks_consumed) == (
            want["emitted"], want["filtered"], want["batches"], want["consumed"])


def test_survey_operand_bytes():
    """B_enum / B_min of SURVEY 8(d) (reference instrumented by the survey)."""
    g = synth.build_config("C4")
    r = O.count(g, 8, 8, workers=8)
    assert (r.intersections, r.operand_words, r.min_words) == (29754436, 4034850823, 416685192)
    assert r.count == 90068795717


def test_root_restriction_and_rank_override():
    g = synth.random_bipartite(16, 16, 0.35, 41)
    total = O.count(g, 3, 2, anchor="U").count
    a = O.count(g, 3, 2, anchor="U", roots=range(0, 8)).count
    b = O.count(g, 3, 2, anchor="U", roots=range(8, 16)).count
    assert a + b == total
    g = synth.random_bipartite(12, 12, 0.4, 53)
    rank = np.random.default_rng(1).permutation(12) + 1
    assert O.count(g, 2, 2, anchor="U", rank=rank).count == O.brute_force_count(g, 2, 2)
    with pytest.raises(ValueError):
        O.Prepared(synth.random_bipartite(5, 5, 0.4, 1), 2, 2, "U", rank=[1, 1, 2, 3, 4])


def test_per_task_counts_sum():
    g = synth.random_bipartite(40, 40, 0.25, 77)
    r = O.count(g, 3, 2, per_task=True)
    assert sum(r.task_counts) == r.count
    assert len(r.task_counts) == r.tasks_emitted


def test_capacity_check():
    g = synth.random_bipartite(200, 200, 0.2, 9)
    with pytest.raises(ValueError, match="batch-words"):
        O.count(g, 2, 2, capacity=2)
