"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container only (needs /root/reference, read-only):

    python tests/golden/make_golden.py [--heavy]

Imports the reference package from /root/reference/pkg/src and records, for
seeded inputs, its structures (2-hop lists, priority, HTB arrays, tasks) and
CountReport fields.  The fixtures pin the oracle (oracle/) and, through it,
the GPU path.  Nothing on the GPU box reads /root/reference.

--heavy additionally runs the reference on the large configs C2, C3(6,3)
and C4 with 8 fork workers (minutes each).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from bicount import htb as rhtb  # noqa: E402
from bicount.engine import (  # noqa: E402
    EngineConfig, _build_shared, count_bicliques, pre_runtime_tasks, prepare_structures)
from bicount.graph import BipartiteGraph as RGraph  # noqa: E402
from bicount.oracle import brute_force_count  # noqa: E402

from paper_2403_07858_b200 import synth  # noqa: E402


def to_ref(g) -> RGraph:
    return RGraph([np.asarray(a, np.int32) for a in g.u_adj], [np.asarray(a, np.int32) for a in g.v_adj])


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).astype("<i8").tobytes()).hexdigest()


def csr_of(lists):
    off = np.zeros(len(lists) + 1, dtype=np.int64)
    np.cumsum([len(x) for x in lists], out=off[1:])
    idx = np.concatenate([np.asarray(x, np.int64) for x in lists]) if off[-1] else np.zeros(0, np.int64)
    return off, idx


def structures_record(rg, p, q, anchor="auto", full=False):
    s = prepare_structures(rg, p, q, anchor=anchor)
    lists, emitted, filtered = pre_runtime_tasks(s.dir2, s.order, s.choice.p_eff, 1, s.und_sizes)
    tasks = np.asarray(lists[0], dtype=np.int64).reshape(-1, 2)
    doff, didx = csr_of(s.dir2.lists)
    arrays = {
        "und_size": np.asarray(s.und_sizes), "rank": np.asarray(s.order.rank),
        "order": np.asarray(s.order.order), "dir_off": doff, "dir_idx": didx,
        "hadj_off": s.adj_htb.off, "hadj_idx": s.adj_htb.idx, "hadj_val": s.adj_htb.val,
        "hdir_off": s.dir2_htb.off, "hdir_idx": s.dir2_htb.idx, "hdir_val": s.dir2_htb.val,
        "tasks": tasks.ravel(),
    }
    rec = {"anchor": s.choice.layer, "p_eff": s.choice.p_eff, "q_eff": s.choice.q_eff,
           "emitted": emitted, "filtered": filtered,
           "sha256": {k: digest(v) for k, v in arrays.items()}}
    if full:
        rec["arrays"] = {k: np.asarray(v, dtype=np.int64).tolist() for k, v in arrays.items()}
    return rec


def report_record(rg, p, q, anchor="auto", workers=1, modes=("hybrid", "dfs")):
    out = {}
    for mode in modes:
        t = time.time()
        r = count_bicliques(rg, p, q, EngineConfig(mode=mode, anchor=anchor, worker_count=workers))
        out[mode] = {"count": str(r.count), "batches": r.batches_executed,
                     "emitted": r.tasks_emitted, "filtered": r.roots_filtered,
                     "consumed": r.tasks_consumed, "anchor": r.anchor_layer,
                     "seconds": round(time.time() - t, 3)}
    return out


def instrumented(rg, p, q):
    """Reference search with htb_intersect wrapped: calls, sum(|a|+|b|), sum(min)."""
    import bicount.engine as E
    tally = [0, 0, 0]
    orig = E.htb_intersect

    def wrapped(a, b, out):
        la, lb = a.hi - a.lo, b.hi - b.lo
        tally[0] += 1
        tally[1] += la + lb
        tally[2] += min(la, lb)
        return orig(a, b, out)

    E.htb_intersect = wrapped
    try:
        r = count_bicliques(rg, p, q, EngineConfig(worker_count=1))
    finally:
        E.htb_intersect = orig
    return {"count": str(r.count), "intersections": tally[0], "operand_words": tally[1],
            "min_words": tally[2]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heavy", action="store_true")
    args = ap.parse_args()
    gold = {}

    # HTB goldens (test_htb.py:17-52)
    a, b = [3, 8, 10, 17, 73, 79, 82], [3, 10, 23, 102]
    ha, hb = rhtb.htb_build([a]), rhtb.htb_build([b])
    out = rhtb.htb_intersect(hb.slice(0), ha.slice(0), rhtb.HtbSlice([0] * 8, [0] * 8, 0, 0))
    gold["htb"] = {"set_a": a, "set_b": b, "a_idx": ha.idx, "a_val": ha.val, "b_idx": hb.idx,
                   "b_val": hb.val, "isect_idx": out.idx[out.lo:out.hi],
                   "isect_val": out.val[out.lo:out.hi], "isect_ids": out.decode()}

    # recon graph (helpers.py:10-24; test_engine.py:35-63)
    rg = to_ref(synth.recon_graph())
    gold["recon"] = {"structures_3_2_U": structures_record(rg, 3, 2, "U", full=True), "reports": {}}
    for p, q, anc in [(3, 2, "auto"), (3, 2, "U"), (2, 2, "auto"), (1, 2, "auto"), (1, 1, "auto"),
                      (5, 2, "U"), (2, 6, "U"), (4, 2, "V"), (2, 3, "V")]:
        gold["recon"]["reports"][f"{p},{q},{anc}"] = report_record(rg, p, q, anc)

    # seeded random graphs: full structures + reports
    cases = []
    rng = np.random.default_rng(2026)
    for i in range(24):
        nu, nv = int(rng.integers(5, 60)), int(rng.integers(5, 60))
        dens = float(rng.uniform(0.05, 0.5))
        seed = int(rng.integers(0, 2**31))
        p, q = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        anchor = ["auto", "U", "V"][i % 3]
        g = synth.random_bipartite(nu, nv, dens, seed)
        rg = to_ref(g)
        cases.append({"nu": nu, "nv": nv, "density": dens, "seed": seed, "p": p, "q": q,
                      "anchor": anchor, "structures": structures_record(rg, p, q, anchor, full=True),
                      "reports": report_record(rg, p, q, anchor)})
    gold["random"] = cases

    # medium random graphs: digests + reports (bigger than brute force can do)
    med = []
    for (nu, nv, dens, seed, p, q) in [(300, 200, 0.06, 1, 3, 3), (400, 400, 0.03, 2, 4, 2),
                                       (250, 300, 0.08, 3, 2, 4), (150, 150, 0.15, 4, 5, 3),
                                       (500, 120, 0.05, 5, 3, 5), (200, 200, 0.1, 6, 6, 2)]:
        g = synth.random_bipartite(nu, nv, dens, seed)
        rg = to_ref(g)
        med.append({"nu": nu, "nv": nv, "density": dens, "seed": seed, "p": p, "q": q,
                    "structures": structures_record(rg, p, q),
                    "reports": report_record(rg, p, q),
                    "instrumented": instrumented(rg, p, q)})
    gold["medium"] = med

    # corpus300 x (p,q) in {1..4}^2 (test_acceptance.py:115-120): reference engine counts
    t = time.time()
    corpus = synth.corpus300()
    counts = []
    for g in corpus:
        rg = to_ref(g)
        row = []
        for p in range(1, 5):
            for q in range(1, 5):
                row.append(str(count_bicliques(rg, p, q).count))
        counts.append(row)
    gold["corpus300"] = {"pq": [[p, q] for p in range(1, 5) for q in range(1, 5)], "counts": counts,
                         "seconds": round(time.time() - t, 2)}
    # brute-force cross-check of a slice, as the reference's criterion 3 does
    gold["corpus300"]["brute_first20"] = [
        [str(brute_force_count(to_ref(g), p, q)) for p in range(1, 5) for q in range(1, 5)]
        for g in corpus[:20]]

    # S2 (reference test graph) and the small configs
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        s2 = synth.synth_generate(12720, 11100, 2.6, 7)
    cfgs = {"S2": {"fingerprint": s2.fingerprint(),
                   "(2,2)": report_record(to_ref(s2), 2, 2, workers=8, modes=("hybrid",)),
                   "(4,4)": report_record(to_ref(s2), 4, 4, workers=8, modes=("hybrid",)),
                   "structures_(4,4)": structures_record(to_ref(s2), 4, 4)}}
    g1 = synth.build_config("C1")
    cfgs["C1"] = {"fingerprint": g1.fingerprint(),
                  "(2,2)": report_record(to_ref(g1), 2, 2, modes=("hybrid", "dfs")),
                  "structures_(2,2)": structures_record(to_ref(g1), 2, 2),
                  "instrumented_(2,2)": instrumented(to_ref(g1), 2, 2)}
    g3 = synth.build_config("C3")
    cfgs["C3"] = {"fingerprint": g3.fingerprint(),
                  "(3,6)": report_record(to_ref(g3), 3, 6, workers=8, modes=("hybrid",)),
                  "structures_(3,6)": structures_record(to_ref(g3), 3, 6),
                  "structures_(6,3)": structures_record(to_ref(g3), 6, 3),
                  "instrumented_(3,6)": instrumented(to_ref(g3), 3, 6)}
    g2 = synth.build_config("C2")
    cfgs["C2"] = {"fingerprint": g2.fingerprint(), "structures_(4,4)": structures_record(to_ref(g2), 4, 4)}
    g4 = synth.build_config("C4")
    cfgs["C4"] = {"fingerprint": g4.fingerprint(), "structures_(8,8)": structures_record(to_ref(g4), 8, 8)}
    if args.heavy:
        cfgs["C2"]["(4,4)"] = report_record(to_ref(g2), 4, 4, workers=8, modes=("hybrid",))
        cfgs["C3"]["(6,3)"] = report_record(to_ref(g3), 6, 3, workers=8, modes=("hybrid",))
        cfgs["C4"]["(8,8)"] = report_record(to_ref(g4), 8, 8, workers=8, modes=("hybrid",))
    gold["configs"] = cfgs

    path = os.path.join(HERE, "golden.json")
    prev = {}
    if os.path.exists(path) and not args.heavy:
        prev = json.load(open(path)).get("configs", {})
    for name, rec in prev.items():  # keep previously computed heavy results
        for k, v in rec.items():
            gold["configs"].setdefault(name, {}).setdefault(k, v)
    with open(path, "w") as fh:
        json.dump(gold, fh, indent=1, sort_keys=True)
        fh.write("\n")
    print(f"wrote {path}")


if __name__ == "__main__":
    main()
