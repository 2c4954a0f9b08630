"""Pin the full C5 (8,8) total with the CPU oracle (TEST INFRASTRUCTURE ONLY).

A whole C5 count is hours of CPU, so the anchor roots are counted in contiguous
chunks through the reference's own root decomposition: a root-restricted count
emits exactly the tasks whose root is in the set (``engine.py:155-162``), and
root-restricted counts over a partition of the roots sum to the whole count
(``partition.py:244-250``, ``test_engine.py:261-269``).

Each chunk's result is appended to ``--out`` (JSON lines) as soon as it ends, so
the run resumes where it stopped.  ``--finish`` sums the chunks, checks that they
cover every root exactly once, and writes the total plus the per-chunk counts
into ``tests/golden/c5_full.json``.

    python scripts/c5_full_oracle.py --threads 6            # hours, resumable
    python scripts/c5_full_oracle.py --finish
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2403_07858_b200 import synth  # noqa: E402

CAP = 1 << 17
DEFAULT_OUT = os.path.join(ROOT, "profiles", "r2", "c5_oracle_chunks.jsonl")
GOLDEN = os.path.join(ROOT, "tests", "golden", "c5_full.json")


def load_done(path):
    done = {}
    if os.path.exists(path):
        with open(path) as f:
            for line in f:
                line = line.strip()
                if line:
                    r = json.loads(line)
                    done[(r["lo"], r["hi"])] = r
    return done


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=len(os.sched_getaffinity(0)))
    ap.add_argument("--chunk", type=int, default=1000)
    ap.add_argument("--out", default=DEFAULT_OUT)
    ap.add_argument("--finish", action="store_true")
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)

    if a.finish:
        done = load_done(a.out)
        spans = sorted(done)
        n = done[spans[0]]["n_roots_total"]
        pos = 0
        for lo, hi in spans:
            assert lo == pos, f"gap or overlap at {lo} (expected {pos})"
            pos = hi
        assert pos == n, f"chunks cover {pos} of {n} roots"
        chunks = [done[s] for s in spans]
        total = sum(int(c["count"]) for c in chunks)
        out = {
            "config": "C5", "p": 8, "q": 8, "capacity": CAP,
            "generator": "synth.fr_shaped_csr() defaults (44,000 x 8,956,000, m=1e8, 64 planted core triples)",
            "count": str(total),
            "tasks_emitted": sum(c["tasks_emitted"] for c in chunks),
            "roots_filtered": sum(c["roots_filtered"] for c in chunks),
            "batches_executed": sum(c["batches_executed"] for c in chunks),
            "intersections": sum(c["intersections"] for c in chunks),
            "operand_words": sum(c["operand_words"] for c in chunks),
            "cpu_seconds_wall": sum(c["seconds"] for c in chunks),
            "threads": chunks[0]["threads"],
            "chunks": [{"lo": c["lo"], "hi": c["hi"], "count": c["count"]} for c in chunks],
            "made_by": "scripts/c5_full_oracle.py (oracle/bicount_oracle.c, reference rank and task order)",
        }
        with open(GOLDEN, "w") as f:
            json.dump(out, f, indent=1)
        print(json.dumps({k: v for k, v in out.items() if k != "chunks"}, indent=1))
        return

    t0 = time.perf_counter()
    csr = synth.fr_shaped_csr(device="cpu")
    g = synth.graph_from_torch_csr(*csr)
    del csr
    print(f"graph: {g.u_count} x {g.v_count}, {time.perf_counter() - t0:.1f} s", flush=True)
    t0 = time.perf_counter()
    prep = O.Prepared(g, 8, 8, threads=a.threads)
    print(f"prepare: anchor {prep.anchor}, n={prep.n}, {time.perf_counter() - t0:.1f} s", flush=True)
    done = load_done(a.out)
    n = prep.n
    for lo in range(0, n, a.chunk):
        hi = min(n, lo + a.chunk)
        if (lo, hi) in done:
            continue
        t1 = time.perf_counter()
        r = O.count(g, 8, 8, workers=a.threads, capacity=CAP, roots=np.arange(lo, hi),
                    prepared=prep)
        dt = time.perf_counter() - t1
        assert not r.overflow
        rec = {"lo": lo, "hi": hi, "n_roots_total": n, "count": str(r.count),
               "tasks_emitted": r.tasks_emitted, "roots_filtered": r.roots_filtered,
               "batches_executed": r.batches_executed, "intersections": r.intersections,
               "operand_words": r.operand_words, "seconds": dt, "threads": a.threads}
        with open(a.out, "a") as f:
            f.write(json.dumps(rec) + "\n")
        print(f"[{lo},{hi}) count={r.count} tasks={r.tasks_emitted} {dt:.1f} s", flush=True)


if __name__ == "__main__":
    main()
