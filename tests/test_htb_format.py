"""HTB encoding and the HTBDUMP1 format (reference htb.py,
test_htb.py).  CPU: the host encoder and dump against the reference's bytes
(tests/golden/htb_dumps.json, make_htb_golden.py) and its known answers.  GPU:
the device-built adjacency / directed-2-hop arenas dump to the reference's files.
"""

import hashlib
import json
import os
import sys

import numpy as np
import pytest

from paper_2403_07858_b200 import htb, synth

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "htb_dumps.json")))
sys.path.insert(0, os.path.join(HERE, "golden"))

FIG_SET_A = [3, 8, 10, 17, 73, 79, 82]
FIG_SET_B = [3, 10, 23, 102]


def _families():
    src = open(os.path.join(HERE, "golden", "make_htb_golden.py")).read()
    start, end = src.index("def families():"), src.index("def digest(")
    ns = {"np": np}
    exec(src[start:end], ns)
    return ns["families"]()


def _dump_digest(h, tmp_path, name="h.bin"):
    p = tmp_path / name
    htb.dump_htb(h, p)
    b = p.read_bytes()
    return {"sha256": hashlib.sha256(b).hexdigest(), "bytes": len(b)}


def test_known_answers():
    h = htb.htb_build([FIG_SET_A])  # test_htb.py:25-37
    assert h.idx.tolist() == [0, 2] and h.val.tolist() == [132360, 295424] and h.off.tolist() == [0, 2]
    h = htb.htb_build([FIG_SET_B])
    assert h.idx.tolist() == [0, 3] and h.val.tolist() == [8389640, 64]
    h = htb.htb_build([[]])
    assert h.off.tolist() == [0, 0] and h.n_words == 0 and htb.htb_decode(h, 0) == []
    assert htb.htb_build([[0, 33, 66]]).n_words == 3 and htb.htb_build([[0, 1, 2]]).n_words == 1
    with pytest.raises(ValueError):
        htb.htb_build([[3, 2]])
    with pytest.raises(ValueError):
        htb.htb_build([[1, 1]])
    with pytest.raises(ValueError):
        htb.htb_build([[-1, 4]])


@pytest.mark.parametrize("name", sorted(_families()))
def test_dump_bytes_match_reference(name, tmp_path):
    sets = _families()[name]
    h = htb.htb_build(sets)
    assert _dump_digest(h, tmp_path) == GOLD["families"][name]
    g = htb.load_htb(tmp_path / "h.bin")
    assert g.off.tolist() == h.off.tolist() and g.idx.tolist() == h.idx.tolist()
    for s in range(len(sets)):
        assert htb.htb_decode(g, s) == sorted(sets[s])


def test_load_rejects_bad_and_truncated(tmp_path):
    p = tmp_path / "junk.htb"
    p.write_bytes(b"NOTADUMP" + b"\x00" * 16)
    with pytest.raises(ValueError, match="magic"):
        htb.load_htb(p)
    h = htb.htb_build([FIG_SET_A, [], FIG_SET_B])
    q = tmp_path / "t.htb"
    htb.dump_htb(h, q)
    raw = q.read_bytes()
    assert len(raw) == 8 + 4 * (2 + len(h.off) + 2 * h.n_words)  # test_htb.py:194-203
    q.write_bytes(raw[:-4])
    with pytest.raises(ValueError, match="truncated"):
        htb.load_htb(q)


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(GOLD["structures"]))
def test_device_arenas_dump_like_reference(key, tmp_path):
    from paper_2403_07858_b200 import prepare_structures

    name, pq = key.split("|")
    p, q = map(int, pq.split(","))
    s = prepare_structures(synth.build_config(name), p, q)
    assert _dump_digest(s.adj_htb, tmp_path, "a.bin") == GOLD["structures"][key]["adj"]
    assert _dump_digest(s.dir2_htb, tmp_path, "d.bin") == GOLD["structures"][key]["dir2"]


def test_slices_and_intersections():
    """test_htb.py:39-52, 121-127 and random sets against Python sets."""
    a, b = htb.HtbSlice.from_ids(FIG_SET_B), htb.HtbSlice.from_ids(FIG_SET_A)
    out = htb.htb_intersect(a, b, htb.HtbSlice([0] * 8, [0] * 8, 0, 0))
    assert len(out) == 1 and out.idx[out.lo] == 0 and out.val[out.lo] == 1032
    assert out.decode() == [3, 10] and htb.htb_intersect_count(a, b) == 2
    got = htb.htb_intersect(htb.HtbSlice.from_ids([3, 40]), htb.HtbSlice.from_ids([3, 40, 70]),
                            htb.HtbSlice([0] * 6, [0] * 6, 3, 3))
    assert got.lo == 3 and got.hi == 5 and got.decode() == [3, 40]
    with pytest.raises(ValueError):
        htb.htb_intersect(a, b, htb.HtbSlice([0], [0], 0, 0))
    rng = np.random.default_rng(9)
    for _ in range(50):
        xs = sorted(rng.choice(400, size=int(rng.integers(0, 60)), replace=False).tolist())
        ys = sorted(rng.choice(400, size=int(rng.integers(0, 60)), replace=False).tolist())
        sa, sb = htb.HtbSlice.from_ids(xs), htb.HtbSlice.from_ids(ys)
        cap = min(len(sa), len(sb))
        r = htb.htb_intersect(sa, sb, htb.HtbSlice([0] * cap, [0] * cap, 0, 0))
        assert r.decode() == sorted(set(xs) & set(ys))
        assert htb.htb_intersect_count(sa, sb) == len(set(xs) & set(ys)) == r.cardinality()
        assert sa.cardinality() == len(xs)


def test_stats_json_payload_matches_reference_schema(tmp_path):
    """cli.py:252-257: {"schema": 1, **asdict(report)} over the reference's CountReport
    fields (engine.py:64-79), json with default=int and a trailing newline."""
    import json

    from paper_2403_07858_b200 import CountReport, stats_payload, write_stats_json

    r = CountReport(count=1 << 70, time_1hop=0.5, time_2hop=1.5, batches_executed=7,
                    tasks_stolen=0, roots_filtered=2, wall_time=2.0, tasks_emitted=9,
                    tasks_consumed=9, workers=1, anchor_layer="U", device={"kernel_launches": 3})
    d = stats_payload(r)
    assert list(d) == ["schema", "count", "time_1hop", "time_2hop", "batches_executed",
                       "tasks_stolen", "roots_filtered", "wall_time", "tasks_emitted",
                       "tasks_consumed", "workers", "anchor_layer", "bicliques", "task_tally",
                       "task_counts"]
    p = tmp_path / "s.json"
    write_stats_json(r, p)
    raw = p.read_text()
    assert raw.endswith("}\n") and json.loads(raw)["count"] == 1 << 70
    assert "device" in stats_payload(r, include_device=True)


@pytest.mark.gpu
def test_dump_loads_straight_into_device_arenas(tmp_path):
    """A HTBDUMP1 dump of the device-built arenas, loaded back straight into device memory
    (htb.load_htb_device), equals the arenas word for word."""
    import torch

    from paper_2403_07858_b200 import DeviceGraph, prepare_structures

    g = synth.build_config("C4")
    s = prepare_structures(g, 8, 8)
    dg = DeviceGraph(g)
    try:
        arenas = dg.htb_arenas(8, 8)
    finally:
        dg.close()
    for name, h in (("adj", s.adj_htb), ("dir2", s.dir2_htb)):
        htb.dump_htb(h, tmp_path / f"{name}.bin")
        got = htb.load_htb_device(tmp_path / f"{name}.bin", 0)
        for a, b in zip(got, arenas[name]):
            assert a.dtype == b.dtype and torch.equal(a, b), name
