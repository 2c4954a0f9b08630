"""Development: one forced-path count under compute-sanitizer (first random case of
tests/test_gpu_variants.py that uses p_eff >= 5)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2403_07858_b200 import EngineConfig, count_bicliques, synth  # noqa: E402

rng = np.random.default_rng(11)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    nu, nv = int(rng.integers(20, 140)), int(rng.integers(20, 140))
    g = synth.random_bipartite(nu, nv, float(rng.uniform(0.08, 0.45)), int(rng.integers(1 << 30)))
    p, q = int(rng.integers(2, 9)), int(rng.integers(2, 8))
    anchor = ["auto", "U", "V"][i % 3]
    mode = ["hybrid", "dfs"][i % 2]
    r = count_bicliques(g, p, q, EngineConfig(anchor=anchor, mode=mode, level1="scatter", rows="scatter", instrument=bool(os.environ.get("INSTR"))))
    print(i, p, q, r.count, flush=True)
