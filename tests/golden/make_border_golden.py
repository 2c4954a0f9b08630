"""Generate tests/golden/border.json by running the REFERENCE Border pass.

Run in the build container only (needs /root/reference, read-only):

    python tests/golden/make_border_golden.py

Records, for seeded inputs, the reference's ``border_reorder`` permutation and
1-block history (``reorder.py:146-179``), ``degree_order`` (``reorder.py:137-143``)
and the full ``apply_reorder`` pipeline of the CLI (``cli.py:124-145``: degree
presort, then Border on the anchor layer and then the other layer) as a digest of
the relabelled graph.  These pin ``oracle.border_reorder`` and, through it, the
device pass.  Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from bicount.cli import apply_reorder  # noqa: E402
from bicount.graph import BipartiteGraph as RGraph  # noqa: E402
from bicount.reorder import border_reorder, degree_order  # noqa: E402

from paper_2403_07858_b200 import synth  # noqa: E402
from paper_2403_07858_b200.graph import from_edges  # noqa: E402


def to_ref(g) -> RGraph:
    return RGraph([np.asarray(a, np.int32) for a in g.u_adj], [np.asarray(a, np.int32) for a in g.v_adj])


def graph_digest(rg) -> str:
    h = hashlib.sha256()
    for lists in (rg.u_adj, rg.v_adj):
        off = np.zeros(len(lists) + 1, np.int64)
        np.cumsum([len(a) for a in lists], out=off[1:])
        h.update(off.astype("<i8").tobytes())
        for a in lists:
            h.update(np.asarray(a, np.int64).astype("<i8").tobytes())
    return h.hexdigest()


# (name, graph builder, layer, iterations)
CASES = [
    ("recon_U", synth.recon_graph, "U", 10),
    ("recon_V", synth.recon_graph, "V", 10),
    ("lone_bits", lambda: from_edges(64, 1, [0, 32], [0, 0]), "U", 10),
    ("tiny_cols", lambda: from_edges(1, 3, [0, 0], [0, 2]), "U", 5),
    ("empty", lambda: from_edges(0, 0, [], []), "U", 5),
] + [(f"rb50x90_s{s}", (lambda s=s: synth.random_bipartite(50, 90, 0.08, s)), "V", 10)
     for s in range(4)] + [
    (f"rb70x30_s{s}", (lambda s=s: synth.random_bipartite(70, 30, 0.15, s)), "U", 25)
    for s in range(3)] + [
    ("rb12_s5", lambda: synth.random_bipartite(12, 12, 0.35, 5), "U", 8),
    ("rb300x400_U", lambda: synth.random_bipartite(300, 400, 0.02, 3), "U", 120),
    ("rb300x400_V", lambda: synth.random_bipartite(300, 400, 0.02, 3), "V", 120),
    ("rb200x150_dense_U", lambda: synth.random_bipartite(200, 150, 0.3, 9), "U", 60),
    ("rb100x80_mid_U", lambda: synth.random_bipartite(100, 80, 0.12, 13), "U", 50),
    ("rb60x200_V", lambda: synth.random_bipartite(60, 200, 0.1, 17), "V", 80),
    ("C1_U", lambda: synth.build_config("C1"), "U", 300),
    ("C1_V", lambda: synth.build_config("C1"), "V", 150),
]

PIPELINES = [  # (name, builder, iters, p, q, anchor)
    ("pipe_rb_auto", lambda: synth.random_bipartite(160, 220, 0.05, 21), 30, 3, 3, "auto"),
    ("pipe_rb_V", lambda: synth.random_bipartite(120, 90, 0.08, 4), 20, 2, 3, "V"),
    ("pipe_recon", synth.recon_graph, 10, 2, 2, "auto"),
]


def main() -> None:
    out = {"border": {}, "degree_order": {}, "pipeline": {}}
    for name, build, layer, iters in CASES:
        g = build()
        t = time.time()
        res = border_reorder(to_ref(g), layer, iters)
        out["border"][name] = {"layer": layer, "iterations": iters,
                               "permutation": np.asarray(res.permutation).tolist(),
                               "history": [int(x) for x in res.one_block_history]}
        print(f"{name}: {len(res.one_block_history) - 1} swaps, {time.time() - t:.1f} s", flush=True)
    for name, build in [("recon", synth.recon_graph),
                        ("rb70x30", lambda: synth.random_bipartite(70, 30, 0.15, 1))]:
        rg = to_ref(build())
        out["degree_order"][name] = {"U": degree_order(rg, "U").tolist(),
                                     "V": degree_order(rg, "V").tolist()}
    for name, build, iters, p, q, anchor in PIPELINES:
        rg = apply_reorder(to_ref(build()), "border", iters, p, q, anchor)
        out["pipeline"][name] = {"iterations": iters, "p": p, "q": q, "anchor": anchor,
                                 "digest": graph_digest(rg)}
    with open(os.path.join(HERE, "border.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))


if __name__ == "__main__":
    main()
