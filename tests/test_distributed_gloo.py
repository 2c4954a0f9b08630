"""Multi-rank host logic on CPU (gloo, world size 2).

Each rank takes the tasks t with t % world == rank -- the device's shard rule
(bc_config.shard_index/shard_count) -- and sums their exact per-task counts,
here produced by the CPU oracle standing in for the GPU partials; the
product's allreduce_count (4 x 32-bit limbs, one all_reduce) must return the
exact total on every rank, including totals far above 2^64.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, partials, total, q):
    import torch.distributed as dist

    from paper_2403_07858_b200.engine import allreduce_count

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        got = allreduce_count(partials[rank])
        big = allreduce_count((2**100 + 12345) * (rank + 1))
        q.put((rank, got == total, big == (2**100 + 12345) * 3))
    finally:
        dist.destroy_process_group()


def _run(partials, total, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, partials, total, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in procs)
    assert all(ok and big for _, ok, big in res), res


def test_shard_partials_allreduce_to_exact_total():
    from oracle import oracle as O
    from paper_2403_07858_b200 import synth

    g = synth.random_bipartite(45, 40, 0.3, 5)
    r = O.count(g, 4, 3, per_task=True)
    world = 2
    partials = [sum(r.task_counts[k::world]) for k in range(world)]
    assert sum(partials) == r.count
    _run(partials, r.count, world)


def test_c4_shard_partials():
    from oracle import oracle as O
    from paper_2403_07858_b200 import synth

    g = synth.build_config("C4")
    r = O.count(g, 8, 8, per_task=True, workers=8)
    partials = [sum(r.task_counts[k::2]) for k in range(2)]
    assert r.count == 90068795717
    _run(partials, r.count)


def test_assemble_upper_cpu():
    """Slices of an upper CSR dealt to 3 shards reassemble into the original (CPU tensors)."""
    import torch

    from paper_2403_07858_b200.engine import assemble_upper

    rng = np.random.default_rng(1)
    n = 50
    lists = [np.sort(rng.choice(np.arange(u + 1, n + 40), size=int(rng.integers(0, 6)),
                                replace=False)) if u < n else [] for u in range(n)]
    lens = torch.tensor([len(x) for x in lists], dtype=torch.int32)
    owner = torch.tensor([u % 3 for u in range(n)])
    slices = []
    for k in range(3):
        lk = torch.where(owner == k, lens, torch.zeros_like(lens))
        ids = [int(v) for u in range(n) if u % 3 == k for v in lists[u]]
        slices.append((lk, torch.tensor(ids, dtype=torch.int32)))
    off, ids = assemble_upper(slices)
    assert off.tolist() == np.concatenate([[0], np.cumsum([len(x) for x in lists])]).tolist()
    assert ids.tolist() == [int(v) for x in lists for v in x]
