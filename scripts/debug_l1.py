"""Development: compare level-1 Info / C_R1 lists of the scatter path with the
probe path and with numpy on one random graph (BC_DUMP_L1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2403_07858_b200 import EngineConfig, count_bicliques, prepare_structures, synth  # noqa: E402


def load(path):
    with open(path, "rb") as fh:
        n = int(np.frombuffer(fh.read(8), np.int64)[0])
        info = np.frombuffer(fh.read(16 * n), np.int32).reshape(n, 4)
        nl = int(np.frombuffer(fh.read(8), np.int64)[0])
        ro = li = None
        if nl:
            ro = np.frombuffer(fh.read(8 * (n + 1)), np.int64)
            li = np.frombuffer(fh.read(4 * nl), np.int32)
    return info, ro, li


rng = np.random.default_rng(11)
for i in range(30):
    nu, nv = int(rng.integers(20, 140)), int(rng.integers(20, 140))
    g = synth.random_bipartite(nu, nv, float(rng.uniform(0.08, 0.45)), int(rng.integers(1 << 30)))
    p, q = int(rng.integers(2, 9)), int(rng.integers(2, 8))
    anchor = ["auto", "U", "V"][i % 3]
    mode = ["hybrid", "dfs"][i % 2]
    want = O.count(g, p, q, anchor=anchor, mode=mode)
    res = {}
    for l1 in ("probe", "scatter"):
        for rows in ("probe", "scatter"):
            os.environ["BC_DUMP_L1"] = f"/tmp/l1_{l1}.bin"
            r = count_bicliques(g, p, q, EngineConfig(anchor=anchor, mode=mode, level1=l1, rows=rows))
            res[(l1, rows)] = r.count
    print(i, p, q, anchor, "want", want.count, res, flush=True)
    if any(v != want.count for v in res.values()):
        a, _, _ = load("/tmp/l1_probe.bin")
        b, ro, li = load("/tmp/l1_scatter.bin")
        s = prepare_structures(g, p, q, anchor)
        tasks = s.tasks
        work = s.work
        bad = np.nonzero((a[:, 0] != b[:, 0]) | (a[:, 1] != b[:, 1]))[0]
        print("info mismatches", len(bad), "of", len(a))
        for t in bad[:5]:
            r_, s_ = tasks[t]
            want_l = np.intersect1d(work.u_csr.row(r_), work.u_csr.row(s_))
            print(" task", t, (r_, s_), "probe", a[t], "scatter", b[t], "list", li[ro[t]:ro[t + 1]],
                  "numpy", want_l)
        # list correctness everywhere
        nbad = 0
        for t in range(len(tasks)):
            r_, s_ = tasks[t]
            want_l = np.intersect1d(work.u_csr.row(r_), work.u_csr.row(s_))
            if not np.array_equal(li[ro[t]:ro[t + 1]], want_l):
                nbad += 1
        print("list mismatches", nbad)
        break
