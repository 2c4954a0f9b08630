"""Generate tests/golden/htb_dumps.json by running the REFERENCE HTB encoder and dump
(``htb.py:89-115``, ``186-206``).  Build container only (needs /root/reference):

    python tests/golden/make_htb_golden.py

Records the sha256 and size of the reference's HTBDUMP1 file for seeded id-set families
and for the reference's own adjacency / directed 2-hop HTBs of small configs
(``prepare_structures``), so the repo's ``htb.dump_htb`` (host encoder and the device
arenas exported by ``prepare_structures``) can be checked byte for byte.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from bicount.engine import prepare_structures  # noqa: E402
from bicount.graph import BipartiteGraph as RGraph  # noqa: E402
from bicount.htb import dump_htb, htb_build  # noqa: E402

from paper_2403_07858_b200 import synth  # noqa: E402


def families():
    out = {"fig_a": [[3, 8, 10, 17, 73, 79, 82]], "fig_ab": [[3, 8, 10, 17, 73, 79, 82], [3, 10, 23, 102]],
           "empty_sets": [[], [5], [], [31, 32, 33]]}
    rng = np.random.default_rng(3)
    for i in range(4):
        n = int(rng.integers(1, 60))
        out[f"rand{i}"] = [sorted(rng.choice(5000, size=int(rng.integers(0, 80)), replace=False).tolist())
                           for _ in range(n)]
    return out


def digest(h) -> dict:
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "h.bin")
        dump_htb(h, p)
        b = open(p, "rb").read()
    return {"sha256": hashlib.sha256(b).hexdigest(), "bytes": len(b)}


def main() -> None:
    out = {"families": {}, "structures": {}}
    for name, sets in families().items():
        out["families"][name] = digest(htb_build(sets))
    for name, p, q in (("C1", 2, 2), ("C4", 3, 3)):
        g = synth.build_config(name)
        rg = RGraph([np.asarray(a, np.int32) for a in g.u_adj], [np.asarray(a, np.int32) for a in g.v_adj])
        s = prepare_structures(rg, p, q)
        out["structures"][f"{name}|{p},{q}"] = {"adj": digest(s.adj_htb), "dir2": digest(s.dir2_htb)}
    with open(os.path.join(HERE, "htb_dumps.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
