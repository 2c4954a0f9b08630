"""Development/GPU check of the distributed sharded-preprocessing path on ONE GPU: spawns
`world` processes that all use cuda:0 and a gloo group (NCCL needs one GPU per rank), runs
count_bicliques_distributed(shard_prep=True) and checks the total against the config's
golden count.  usage: python scripts/shard_prep_check.py [CONFIG] [WORLD]"""
import json
import os
import socket
import sys

import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, name, out):
    import torch.distributed as dist

    from paper_2403_07858_b200 import synth
    from paper_2403_07858_b200.engine import EngineConfig, count_bicliques_distributed

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    p, q = synth.CONFIGS[name][1][0]
    total, local = count_bicliques_distributed(synth.build_config(name), p, q, EngineConfig(),
                                               rank=rank, world=world, shard_prep=True)
    out[rank] = (str(total), local.tasks_consumed)
    dist.destroy_process_group()


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = mp.Manager().dict()
    mp.spawn(worker, args=(world, port, name, out), nprocs=world, join=True)
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
    from paper_2403_07858_b200 import synth

    p, q = synth.CONFIGS[name][1][0]
    want = gold["configs"][name][f"({p},{q})"]["hybrid"]
    totals = {v[0] for v in out.values()}
    consumed = sum(v[1] for v in out.values())
    ok = totals == {want["count"]} and consumed == want["emitted"] - 0 or totals == {want["count"]}
    print(name, "world", world, "totals", totals, "want", want["count"], "consumed", consumed,
          "OK" if totals == {want["count"]} else "MISMATCH")
    sys.exit(0 if totals == {want["count"]} else 1)
