"""The multi-rank product path, executed: world = 2 and 3 processes, all on cuda:0,
joined by a gloo group (NCCL needs one GPU per rank; only one is reachable here).

Each rank runs exactly what it runs on an 8-GPU box -- ``count_bicliques_distributed``
with sharded preprocessing (its anchors' 2-hop slice, ``gather_upper`` all-gather,
device assembly, its task shard, the limb all-reduce), the replicated-preprocessing
path under both shard rules, and ``count_partitioned_distributed`` over BCPar
closures -- and the totals must equal the reference's goldens (reference
``engine.py:449-478``: one call splits its tasks across workers; ``partition.py:244-258``).
bench.py's N > 1 branch runs the same way through torchrun (``--dist-backend gloo``).
"""

import json
import os
import socket
import subprocess
import sys
import warnings

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, scenario, outq):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_2403_07858_b200 import partition as P
    from paper_2403_07858_b200 import synth
    from paper_2403_07858_b200.engine import (DeviceGraph, EngineConfig,
                                              count_bicliques_distributed, gather_upper)

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        out = {}
        if scenario == "counts":
            for name, (p, q) in (("C4", (8, 8)), ("C3", (6, 3)), ("C1", (2, 2))):
                g = synth.build_config(name)
                dg = DeviceGraph(g)
                for tag, kw in (("shardprep", dict(shard_prep=True)),
                                ("root", dict()),
                                ("task", dict(cfg=EngineConfig(shard_mode="task")))):
                    total, local = count_bicliques_distributed(g, p, q, rank=rank, world=world,
                                                               dgraph=dg, **kw)
                    out[f"{name}|{tag}"] = (str(total), local.tasks_consumed, local.tasks_emitted)
                # the gathered upper CSR equals the single-GPU one (same structures)
                off, ids = gather_upper(dg, p, q, EngineConfig(), rank, world)
                r1, _ = dg.count_raw(p, q, upper=(off, ids))
                r0, _ = dg.count_raw(p, q)
                out[f"{name}|upper"] = (r1.und_pairs == r0.und_pairs and
                                        r1.dir2_pairs == r0.dir2_pairs and
                                        r1.count_lo == r0.count_lo and
                                        r1.batches_executed == r0.batches_executed)
                dg.close()
        elif scenario == "partitioned":
            g = synth.build_config("C3")
            idx = P.build_two_hop_index(g, "U", 6)
            w = P.entry_weight(g, idx)
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                parts = P.budgeted_partition(g, idx, int(w.sum() // 4))
            total, local = P.count_partitioned_distributed(g, parts, 3, 6, rank=rank, world=world)
            out["C3|partitioned"] = (str(total), local.tasks_consumed, parts.group_count)
        outq.put((rank, out))
    finally:
        dist.destroy_process_group()


def _run(world, scenario):
    ctx = mp.get_context("spawn")
    outq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scenario, outq))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, out = outq.get(timeout=600)  # a rank that died raises queue.Empty, not a hang
        res[r] = out
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_counts_match_goldens(golden, world):
    res = _run(world, "counts")
    for name, (p, q) in (("C4", (8, 8)), ("C3", (6, 3)), ("C1", (2, 2))):
        want = golden["configs"][name][f"({p},{q})"]["hybrid"]
        for tag in ("shardprep", "root", "task"):
            key = f"{name}|{tag}"
            totals = {res[r][key][0] for r in range(world)}
            assert totals == {want["count"]}, (key, totals)
            # every task of the job is consumed by exactly one rank
            assert sum(res[r][key][1] for r in range(world)) == want["emitted"], key
        assert all(res[r][f"{name}|upper"] for r in range(world)), name


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_distributed_c3(world):
    res = _run(world, "partitioned")
    totals = {res[r]["C3|partitioned"][0] for r in range(world)}
    assert totals == {"141893943"}
    assert res[0]["C3|partitioned"][2] > 1


def test_bench_multirank_branch_gloo():
    """bench.py's N > 1 branch (sharded 2-hop + all-gather + limb all-reduce + max-over-ranks
    timing) under torchrun, two ranks on one GPU over gloo."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", "bench.py", "--gpus", "2",
           "--config", "C4", "--steps", "2", "--warmup", "3", "--dist-backend", "gloo",
           "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["n_gpus"] == 2 and line["count"] == 90068795717
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
