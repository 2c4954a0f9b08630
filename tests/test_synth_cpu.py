"""Host-side generators (CPU): the FR-shaped C5 recipe is integer-exact and counter
based, so it is bit-identical for any chunking of the draw counter (and on CPU vs GPU),
and its CSR views are consistent; the config recipes reproduce the SURVEY fingerprints."""

import numpy as np
import torch

from paper_2403_07858_b200 import synth


def _small(chunk):
    return synth.fr_shaped_csr(nu=300, nv=5000, m=20000, cap_u=2000, cap_v=40, n_cores=2,
                               device="cpu", chunk=chunk)


def test_fr_shaped_is_chunk_invariant_and_consistent():
    a = _small(1 << 25)
    b = _small(777)
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    uo, ui, vo, vi = (t.numpy() for t in a)
    assert uo[-1] == vo[-1] == len(ui) == len(vi)
    for r in range(len(uo) - 1):  # rows strictly increasing
        row = ui[uo[r]:uo[r + 1]]
        assert np.all(np.diff(row) > 0)
    g = synth.graph_from_torch_csr(*a)
    # the V view is the transpose of the U view
    eu = np.repeat(np.arange(g.u_count), np.diff(g.u_csr.off))
    key_u = np.sort(eu * g.v_count + g.u_csr.idx)
    ev = np.repeat(np.arange(g.v_count), np.diff(g.v_csr.off))
    key_v = np.sort(g.v_csr.idx.astype(np.int64) * g.v_count + ev)
    assert np.array_equal(key_u, key_v)


def test_planted_cores_are_in_the_graph():
    uo, ui, vo, vi = (t.numpy() for t in _small(1 << 25))
    for pu, pv, i, j in synth.planted_cores(300, 5000, 2, 9):
        for a, b in zip(pu[i], pv[j]):
            row = ui[uo[a]:uo[a + 1]]
            k = np.searchsorted(row, b)
            assert k < len(row) and row[k] == b


def test_config_fingerprints():
    for name in ("C1", "C4"):
        assert synth.build_config(name).fingerprint() == synth.FINGERPRINTS[name]


def test_bench_cpu_calibration_chunk():
    """bench.py's C5 CPU estimate scales a fixed chunk of roots by that chunk's measured
    share of the offline full oracle run (profiles/r2/c5_oracle_chunks.jsonl): the chunks
    must cover every root once and the calibration chunk must be among them."""
    import importlib.util
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    lo, hi, t_chunk, t_full, n_chunks, threads = bench.calibration_chunk("C5")
    assert (lo, hi) == bench.CAL_CHUNK["C5"] and 0 < t_chunk < t_full
    assert n_chunks == 44 and threads >= 1
    assert bench.calibration_chunk("C2") is None
