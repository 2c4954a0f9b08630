"""Generate tests/golden/partition.json by running the REFERENCE BCPar partitioner.

Run in the build container only (needs /root/reference, read-only):

    python tests/golden/make_partition_golden.py

Records, for seeded inputs, the reference's undirected 2-hop index digest
(``graph.py:192-215``), ``budgeted_partition`` output (``partition.py:74-171``:
groups in admission order, closures, costs, oversize flags) and
``count_partitioned`` report fields (``partition.py:203-272``).  These pin
``paper_2403_07858_b200.partition`` (host greedy + device counts per closure).
Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from bicount.engine import EngineConfig  # noqa: E402
from bicount.graph import BipartiteGraph as RGraph  # noqa: E402
from bicount.graph import build_two_hop_index, select_anchor_layer  # noqa: E402
from bicount.partition import budgeted_partition, count_partitioned, entry_weight  # noqa: E402

from paper_2403_07858_b200 import synth  # noqa: E402
from paper_2403_07858_b200.graph import from_edges  # noqa: E402


def to_ref(g) -> RGraph:
    return RGraph([np.asarray(a, np.int32) for a in g.u_adj], [np.asarray(a, np.int32) for a in g.v_adj])


def two_components():
    return from_edges(4, 4, [0, 0, 1, 1, 2, 2, 3, 3], [0, 1, 0, 1, 2, 3, 2, 3])


def chain():
    return from_edges(3, 4, [0, 0, 1, 1, 1, 1, 2, 2], [0, 1, 0, 1, 2, 3, 2, 3])


# (name, builder, layer, k, budget (int) or fraction of the total entry weight (float))
CASES = [
    ("recon_1000", synth.recon_graph, "U", 2, 1000),
    ("recon_26", synth.recon_graph, "U", 2, 26),
    ("recon_25", synth.recon_graph, "U", 2, 25),
    ("two_comp_6", two_components, "U", 2, 6),
    ("chain_11", chain, "U", 2, 11),
    ("chain_12", chain, "U", 2, 12),
    ("isolated_k1", lambda: from_edges(2, 2, [0, 0], [0, 1]), "U", 1, 10),
    ("empty", lambda: from_edges(0, 0, [], []), "U", 2, 5),
] + [(f"rb18x14_s{s}_f{f}", (lambda s=s: synth.random_bipartite(18, 14, 0.25, s)), "U", 2, f)
     for s in range(4) for f in (0.05, 0.3, 0.8)] + [
    ("rb9x13_V", lambda: synth.random_bipartite(9, 13, 0.35, 11), "V", 2, 0.5),
    ("rb200x150_k2", lambda: synth.random_bipartite(200, 150, 0.04, 3), "U", 2, 0.1),
    ("rb120x300_V_k3", lambda: synth.random_bipartite(120, 300, 0.06, 8), "V", 3, 0.2),
    ("C1_k2", lambda: synth.build_config("C1"), "U", 2, 0.05),
]

# (case name, p, q) -> count_partitioned report fields
COUNTS = [
    ("recon_1000", 3, 2), ("recon_25", 3, 2), ("recon_25", 2, 2), ("two_comp_6", 2, 2),
    ("chain_11", 2, 2), ("isolated_k1", 1, 1), ("empty", 2, 2),
    ("rb18x14_s0_f0.3", 2, 2), ("rb18x14_s1_f0.05", 3, 2), ("rb18x14_s2_f0.8", 2, 2),
    ("rb18x14_s3_f0.05", 2, 2), ("rb9x13_V", 2, 3), ("rb200x150_k2", 3, 2),
    ("rb120x300_V_k3", 3, 2), ("C1_k2", 2, 2), ("C1_k2", 3, 2),
]


def main() -> None:
    out = {"partition": {}, "count": {}}
    parts_of = {}
    for name, build, layer, k, budget in CASES:
        rg = to_ref(build())
        idx = build_two_hop_index(rg, layer, k)
        w = entry_weight(rg, idx)
        b = budget if isinstance(budget, int) else max(1, int(budget * int(w.sum())))
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            parts = budgeted_partition(rg, idx, b)
        parts_of[name] = (rg, parts)
        out["partition"][name] = {
            "layer": layer, "k": k, "budget": b,
            "und_sizes": [int(len(x)) for x in idx.lists],
            "groups": [[int(u) for u in gr] for gr in parts.groups],
            "closures": [[int(u) for u in cl] for cl in parts.closures],
            "costs": [int(c) for c in parts.costs], "oversize": [bool(o) for o in parts.oversize]}
        print(name, "groups", parts.group_count, flush=True)
    for name, p, q in COUNTS:
        rg, parts = parts_of[name]
        if select_anchor_layer(rg, p, q, force=parts.layer).q_eff != parts.k:
            raise SystemExit(f"{name} ({p},{q}): k mismatch")
        rep = count_partitioned(rg, parts, p, q, EngineConfig())
        out["count"][f"{name}|{p},{q}"] = {
            "count": str(rep.count), "roots_filtered": rep.roots_filtered,
            "tasks_emitted": rep.tasks_emitted, "tasks_consumed": rep.tasks_consumed,
            "batches_executed": rep.batches_executed, "anchor_layer": rep.anchor_layer}
        print(name, p, q, rep.count, flush=True)
    with open(os.path.join(HERE, "partition.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))


if __name__ == "__main__":
    main()
