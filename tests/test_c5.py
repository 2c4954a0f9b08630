"""FR-shaped config C5 (SURVEY 8(c) config-5 parity).  A full CPU count is hours, so
(i) the whole total and the reference's counters are pinned by one offline chunked
oracle run (tests/golden/c5_full.json, scripts/c5_full_oracle.py: 3.1 h on 6 threads),
(ii) sampled roots -- planted-core roots, where the (8,8) bicliques live, plus seeded
random roots -- are re-counted by the CPU oracle on the same full graph in the test
(reference rank, reference task order), and (iii) task shards (the multi-GPU
decomposition) sum to the total.  The graph is generated on the GPU by the integer
counter-based recipe (synth.fr_shaped_csr), bit-identical to the CPU recipe the
offline run used."""

import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2403_07858_b200 import DeviceGraph, EngineConfig, synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CAP = 1 << 17


@pytest.fixture(scope="module")
def c5():
    import torch

    csr = synth.fr_shaped_csr(device="cuda")
    g = synth.graph_from_torch_csr(*csr)
    dg = DeviceGraph.from_device_csr(*csr, 0)
    del csr
    torch.cuda.empty_cache()
    yield g, dg
    dg.close()


def test_c5_sampled_roots_match_oracle(c5):
    g, dg = c5
    nu, nv = g.u_count, g.v_count
    cores = synth.planted_cores(nu, nv)
    core_roots = sorted({int(c[0][0]) for c in cores[:12]} | {int(c[0][1]) for c in cores[:6]})
    rnd = np.random.default_rng(3).choice(nu, 120, replace=False).tolist()
    roots = sorted(set(core_roots) | set(rnd))
    rep, _ = dg.count_raw(8, 8, EngineConfig(batch_buffer_capacity=CAP), roots=roots)
    gpu = int(rep.count_lo) | (int(rep.count_hi) << 64)
    prep = O.Prepared(g, 8, 8, threads=len(os.sched_getaffinity(0)))
    want = O.count(g, 8, 8, workers=8, capacity=CAP, roots=roots, prepared=prep)
    assert gpu == want.count
    assert gpu > 0  # the planted cores are in the sample
    assert rep.tasks_emitted == want.tasks_emitted
    assert rep.roots_filtered == want.roots_filtered
    assert rep.batches_executed == want.batches_executed


def test_c5_shards_sum_to_total(c5):
    _, dg = c5
    cfg = EngineConfig(batch_buffer_capacity=CAP)
    rep, _ = dg.count_raw(8, 8, cfg)
    total = int(rep.count_lo) | (int(rep.count_hi) << 64)
    parts = 0
    for k in range(3):
        r, _ = dg.count_raw(8, 8, cfg, shard=(k, 3))
        parts += int(r.count_lo) | (int(r.count_hi) << 64)
    assert parts == total
    assert rep.tasks_emitted == 18900520


def test_c5_full_total_matches_chunked_oracle(c5):
    """The whole C5 (8,8) count and the reference's counters against the full offline
    CPU oracle run (tests/golden/c5_full.json, 44 root chunks summed by
    scripts/c5_full_oracle.py, the decomposition of engine.py:155-162)."""
    import json

    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c5_full.json")))
    _, dg = c5
    rep, _ = dg.count_raw(8, 8, EngineConfig(batch_buffer_capacity=CAP))
    assert (int(rep.count_lo) | (int(rep.count_hi) << 64)) == int(gold["count"])
    assert rep.tasks_emitted == gold["tasks_emitted"]
    assert rep.roots_filtered == gold["roots_filtered"]
    assert rep.batches_executed == gold["batches_executed"]
    ins, _ = dg.count_raw(8, 8, EngineConfig(batch_buffer_capacity=CAP, instrument=True))
    assert ins.intersections == gold["intersections"]
    assert ins.operand_words == gold["operand_words"]
