"""Benchmark: exact (p,q)-biclique counting on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]

A step is one full counting pass of the hot path (device preprocessing: anchor choice,
2-hop index, priority, directed lists, HTB; then the level-1 pass and the hybrid DFS-BFS
enumeration) over the named synthetic config.  Default workload: C5, the FR-shaped
(8,8) config (44K x 8.956M, 1e8 edges) -- the largest BASELINE config, and it fits one
B200, so it is the N = 1 headline; C1-C4 are parity cases (``--config`` runs them too).

* value    = bicliques/s of the whole job (all ranks), CSR already in HBM, CUDA events.
* e2e      = the same metric through the C-ABI ``bc_count`` from pinned HOST CSR buffers
             (H2D + preprocessing + count + D2H inside the timing).
* roofline = the enumeration kernels of one step (the dominant phase): their DRAM bytes
             from an ncu capture of this exact build (profiles/r2/traffic.json, keyed by
             the source hash) / their in-run CUDA-event time, vs the measured HBM peak;
             beside it the compulsory bytes (each input they read, once) and the
             reference's merge-equivalent operand bytes B_enum.
* cpu_baseline = the CPU oracle port (oracle/, C + pthreads, every host core), on a
             bounded sample when the full count is hours (C5), extrapolated by task share.

Multi-GPU (torchrun): each rank builds the upper 2-hop lists of its share of the anchors,
the slices are all-gathered (NCCL over NVLink), each rank counts its shard of the tasks
(whole roots, degree-balanced), and one all_reduce of four 32-bit limbs sums the exact
partials.  ``--dist-backend gloo`` runs the same ranks on one GPU (tests).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_DESC = {
    "C1": "C1 Erdos-Renyi 2,000x2,000, 20K edges",
    "C2": "C2 Chung-Lu power-law 100K x 50K, 1M edges",
    "C3": "C3 GitHub-shaped Chung-Lu 56,519 x 120,867, 440,237 edges",
    "C4": "C4 S2-shaped synth 12,720 x 11,100 + 3 planted dense cores",
    "C5": "C5 FR-shaped capped Chung-Lu 44K x 8.956M, 1e8 edges + planted cores",
    "C5H": "C5H FR-shaped capped Chung-Lu 44K x 8.956M, 1e8 edges + heavy planted cores",
}
DEVICE_GENERATED = ("C5", "C5H")  # built on the GPU by the integer counter-based recipe
METRIC = "(p,q)-biclique count time (s) and bicliques/s at 1/2/4/8 B200 vs CPU ref"
# batch_buffer_capacity per config: the reference rejects capacities below the largest
# HTB slice (engine.py:387-391); C5's hub rows have 122,855 words (SURVEY 8(d) CPU timing
# uses max(4096, max slice) the same way)
CAPACITY = {"C5": 1 << 17, "C5H": 1 << 17}
# CPU legs on C5: the full CPU preprocessing plus the counting of a seeded sample of
# roots, extrapolated by task share (a full CPU count is hours; tests/golden/c5_full.json
# holds the one full offline run)
SAMPLE_FRAC = {"C5": 0.002, "C5H": 0.002}
STRATA = 22  # root-id ranges the sample is stratified over
FALLBACK_HBM = 6650.0
ENUM_KERNELS = ("enum_kernel", "sub_kernel", "filter_kernel")


def golden_count(config: str, p: int, q: int):
    """The config's exact total as pinned by the reference (tests/golden/golden.json,
    C1-C4) or by the full offline CPU oracle run (tests/golden/c5_full.json), else None."""
    try:
        if config in DEVICE_GENERATED:
            d = json.load(open(os.path.join(ROOT, "tests", "golden", f"{config.lower()}_full.json")))
            return int(d["count"]) if (d["p"], d["q"]) == (p, q) else None
        d = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
        return int(d["configs"][config][f"({p},{q})"]["hybrid"]["count"])
    except (OSError, KeyError, ValueError):
        return None


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        if os.environ.get("BENCH_NO_SMI"):  # development: timing without the sampler
            return self
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()

    def summary(self) -> dict:
        self.f.flush()
        rows = []
        try:
            for line in open(self.f.name):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        finally:
            os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy test)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_for(workload: str):
    """DRAM / L2 bytes of the enumeration kernels of one step, from the committed ncu
    launch list of this workload captured on THIS build (profiles/r2/traffic.json; the
    entry is used only when its source hash equals the built sources')."""
    from paper_2403_07858_b200 import build

    p = os.path.join(ROOT, "profiles", "r2", "traffic.json")
    try:
        t = json.load(open(p)).get(workload)
    except (OSError, ValueError):
        return None, "no capture"
    if not isinstance(t, dict):
        return None, "no capture of this workload"
    if t.get("src_sha") != build.source_hash():
        return None, f"capture is of another build ({t.get('src_sha')})"
    return t, t.get("source", "profiles/r2/traffic.json")


CAL_CHUNK = {"C5": (11000, 12000)}  # calibration chunk of the offline full CPU run


def calibration_chunk(config: str):
    """(lo, hi, chunk seconds, full-run seconds, chunks, threads) of the offline full CPU
    oracle run of this config (profiles/r2/c5_oracle_chunks.jsonl), or None."""
    span = CAL_CHUNK.get(config)
    if span is None:
        return None
    try:
        rows = [json.loads(x) for x in open(os.path.join(ROOT, "profiles", "r2",
                                                         "c5_oracle_chunks.jsonl")) if x.strip()]
    except (OSError, ValueError):
        return None
    full = sum(r["seconds"] for r in rows)
    hit = [r for r in rows if (r["lo"], r["hi"]) == span]
    if not hit or sum(r["hi"] - r["lo"] for r in rows) != rows[0]["n_roots_total"]:
        return None
    return span[0], span[1], hit[0]["seconds"], full, len(rows), hit[0]["threads"]


def sample_roots(prep, frac: float, seed: int):
    """A seeded sample of anchor roots and its share of the emitted tasks."""
    import numpy as np

    from oracle import oracle as O

    und = prep.export(O.X_UND_SIZE)
    dsz = np.diff(prep.export(O.X_DIR_OFF))
    ntask = np.where(und >= prep.p_eff - 1, dsz, 0)
    roots = np.random.default_rng(seed).choice(prep.n, max(1, int(frac * prep.n)), replace=False)
    return roots, float(ntask[roots].sum()) / float(max(1, ntask.sum()))


def cpu_oracle_run(g, p, q, threads: int, config: str, seed: int = 1, prep_cache=None):
    """(count or None, seconds, sample description) of the CPU restatement on this host.
    Sampled configs: the preprocessing time (measured once, cached) plus the counting of a
    seeded root sample extrapolated by its task share."""
    from oracle import oracle as O

    frac = SAMPLE_FRAC.get(config)
    cap = CAPACITY.get(config, 4096)
    if frac is None:
        t0 = time.perf_counter()
        r = O.count(g, p, q, workers=threads, threads=threads, capacity=cap)
        return r.count, time.perf_counter() - t0, "full count incl. preprocessing"
    cache = prep_cache if prep_cache is not None else {}
    if "prep" not in cache:
        t0 = time.perf_counter()
        cache["prep"] = O.Prepared(g, p, q, threads=threads)
        cache["t_prep"] = time.perf_counter() - t0
    prep, t_prep = cache["prep"], cache["t_prep"]
    cal = calibration_chunk(config)
    if cal is not None:
        # a fixed chunk of roots of the offline full CPU run, scaled by that chunk's share of
        # the full run's time: per-root cost is heavy-tailed (planted cores), so random root
        # samples extrapolate with a spread of 7x; the chunk ratio is measured, not assumed
        lo, hi, t_off, t_full, n_chunks, thr = cal
        import numpy as np

        t1 = time.perf_counter()
        O.count(g, p, q, workers=threads, threads=threads, capacity=cap,
                roots=np.arange(lo, hi), prepared=prep)
        dt = time.perf_counter() - t1
        est = t_prep + dt * t_full / t_off
        return None, est, (f"full CPU preprocessing ({t_prep:.1f} s) + counting roots "
                           f"[{lo}, {hi}) ({dt:.1f} s), scaled by that chunk's share of the "
                           f"offline full run ({t_off:.1f} s of {t_full:.0f} s over {n_chunks} "
                           f"chunks, {thr} threads, profiles/r2/c5_oracle_chunks.jsonl)")
    # stratified: per-root cost varies ~10x across the root id range, so each stratum of
    # consecutive roots is timed and extrapolated by its own task share
    import numpy as np

    und = prep.export(O.X_UND_SIZE)
    dsz = np.diff(prep.export(O.X_DIR_OFF))
    ntask = np.where(und >= prep.p_eff - 1, dsz, 0)
    n_str = STRATA
    per = max(1, int(round(frac * prep.n / n_str)))
    rng = np.random.default_rng(seed)
    est, t_cnt, n_s, shares = t_prep, 0.0, 0, []
    for k in range(n_str):
        lo, hi = k * prep.n // n_str, (k + 1) * prep.n // n_str
        roots = lo + rng.choice(hi - lo, min(per, hi - lo), replace=False)
        tot = float(ntask[lo:hi].sum())
        got = float(ntask[roots].sum())
        if tot == 0 or got == 0:
            continue
        t1 = time.perf_counter()
        O.count(g, p, q, workers=threads, threads=threads, capacity=cap, roots=roots,
                prepared=prep)
        dt = time.perf_counter() - t1
        t_cnt += dt
        n_s += len(roots)
        est += dt * tot / got
        shares.append(got / tot)
    return None, est, (f"full CPU preprocessing ({t_prep:.1f} s) + counting {n_s} seeded roots "
                       f"stratified over {n_str} root-id ranges ({t_cnt:.1f} s), each range "
                       f"extrapolated by its task share")


def load_graph(config: str, device: int | None):
    """(host BipartiteGraph, device CSR tensors or None)."""
    from paper_2403_07858_b200 import synth

    if config in DEVICE_GENERATED:
        import torch

        if device is None:
            csr = synth.build_device_config(config, "cpu")
            return synth.graph_from_torch_csr(*csr), None
        csr = synth.build_device_config(config, f"cuda:{device}")
        return synth.graph_from_torch_csr(*csr), csr
    return synth.build_config(config), None


def run_reference(args, rank):
    """--impl reference: the CPU restatement of the reference path (oracle/, C + pthreads,
    every host core), rank 0 only; each step is a bounded sample on sampled configs."""
    if rank != 0:
        return
    from paper_2403_07858_b200 import synth

    g, _ = load_graph(args.config, None)
    p, q = pq_of(args)
    threads = host_cores()
    cache = {}
    for i in range(args.warmup):
        cpu_oracle_run(g, p, q, threads, args.config, seed=1000 + i, prep_cache=cache)
    times, count, what = [], None, ""
    for i in range(args.steps):
        c, dt, what = cpu_oracle_run(g, p, q, threads, args.config, seed=1 + i, prep_cache=cache)
        times.append(dt)
        count = c if c is not None else golden_count(args.config, p, q)
    t = statistics.mean(times)
    v = count / t if count else None
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "bicliques/s",
        "n_gpus": 0, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t,
        "time_s": t, "count": count, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"{CONFIG_DESC[args.config]} ({p},{q})", "config": args.config,
                   "p": p, "q": q},
        "cpu_baseline": {"value": v, "unit": "bicliques/s", "cores": threads, "kind": "port",
                         "sample": f"{args.config} ({p},{q}): {what} (oracle/bicount_oracle.c, "
                                   f"{threads} pthreads, {cpu_model()}); count from "
                                   + ("the run" if SAMPLE_FRAC.get(args.config) is None else
                                      f"tests/golden/{args.config.lower()}_full.json")},
        "e2e": {"value": v, "unit": "bicliques/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    del synth


def pq_of(args):
    from paper_2403_07858_b200 import synth

    pq = synth.CONFIGS[args.config][1][0]
    return args.p or pq[0], args.q or pq[1]


def compulsory_bytes(r, m: int, e: int) -> int:
    """Bytes the enumeration kernels must read at least once (each input once, no
    re-reads): the tasks (8 B), their level-1 facts (16 B) and the LPT queue (4 B/alive
    task); with the wedge-scatter level 1 the C_R1 lists (4 B/entry, edge indices) and
    the root-restricted rows they point to (4 B/entry rows + 8 B/edge row offsets + 4 B/edge
    member ids + 8 B/dir2 pair rank positions and rank-ordered lists), else the
    adjacency HTB (8 B/word) the level-1 sets are re-intersected from; always the
    directed 2-hop HTB (8 B/word) C_L1 comes from."""
    b = 24 * r.tasks_consumed + 4 * r.tasks_alive + 8 * r.dir2_words
    if r.level1_entries > 0:
        b += 4 * r.level1_entries + 4 * r.level1_entries + 12 * e + 8 * r.dir2_pairs
    else:
        b += 8 * r.adj_words + 8 * (m + 1) + 4 * e
    return int(b)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=sorted(CONFIG_DESC))
    ap.add_argument("--p", type=int, default=None)
    ap.add_argument("--q", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--dist-backend", default="nccl", choices=("nccl", "gloo"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup raised to 3 (timing rule)", file=sys.stderr)
        args.warmup = 3

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank)

    import torch
    import torch.distributed as dist

    from paper_2403_07858_b200 import _abi
    from paper_2403_07858_b200.engine import (DeviceGraph, EngineConfig, gather_upper, merge_limbs,
                                              split_limbs)

    gloo = args.dist_backend == "gloo"
    local = local % max(torch.cuda.device_count(), 1)  # gloo: several ranks may share a GPU
    torch.cuda.set_device(local)
    if world > 1:
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    cdev = torch.device("cpu") if gloo else dev
    g, dev_csr = load_graph(args.config, local)
    p, q = pq_of(args)

    def barrier():
        if world > 1:
            dist.barrier()

    def allreduce_max(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allreduce_count(c: int) -> int:
        if world == 1:
            return c
        t = torch.tensor(split_limbs(c), dtype=torch.int64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return merge_limbs(t.cpu().tolist())

    cap = CAPACITY.get(args.config, 4096)
    cfg = EngineConfig(device=local, batch_buffer_capacity=cap)
    dg = DeviceGraph.from_device_csr(*dev_csr, local) if dev_csr is not None else DeviceGraph(g, local)
    del dev_csr
    torch.cuda.empty_cache()
    shard = (rank, world)

    def step():
        # N > 1: the 2-hop construction is sharded too (each rank builds its anchors'
        # upper lists, all-gather over NCCL), then every rank counts its task shard
        upper = gather_upper(dg, p, q, cfg, rank, world) if world > 1 else None
        return dg.count_raw(p, q, cfg, shard=shard, upper=upper)

    for _ in range(args.warmup):
        step()
    # B_enum for this workload from the device's own reference-equivalent tally
    instr, _ = dg.count_raw(p, q, EngineConfig(device=local, instrument=True,
                                               batch_buffer_capacity=cap), shard=shard)
    b_enum_local = 8 * instr.operand_words
    b_l1_local = 8 * instr.level1_operand_words
    b_min_local = 16 * instr.min_words

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    step_ms, search_s, level1_s, enum_s, prep_s, launches = [], [], [], [], [], 0
    count_local, last = None, None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            rep, _ = step()
            e1.record()
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            search_s.append(rep.time_level1 + rep.time_enum)
            level1_s.append(rep.time_level1)
            enum_s.append(rep.time_enum)
            prep_s.append(rep.time_prep)
            launches += rep.kernel_launches
            count_local = int(rep.count_lo) | (int(rep.count_hi) << 64)
            last = rep
    clocks = clk.summary()
    barrier()
    ms_local = statistics.mean(step_ms)
    ms = allreduce_max(ms_local)
    total = allreduce_count(count_local)
    t_enum = allreduce_max(statistics.mean(enum_s))
    b_enum = allreduce_count(b_enum_local)
    b_l1 = allreduce_count(b_l1_local)
    b_min = allreduce_count(b_min_local)
    comp_local = compulsory_bytes(last, g.v_count if last.anchor == 0 else g.u_count,
                                  g.edge_count)
    comp = allreduce_count(comp_local) if world > 1 else comp_local
    launches_all = allreduce_count(launches)
    want = golden_count(args.config, p, q)
    if want is not None and total != want:
        raise SystemExit(f"count {total} differs from the pinned golden {want}")

    # e2e through the C-ABI from pinned host buffers
    e2e = None
    if not args.no_e2e:
        L = _abi.load()
        u, v = g.u_csr, g.v_csr
        pinned = [torch.from_numpy(a).pin_memory() for a in (u.off, u.idx, v.off, v.idx)]
        c = _abi.BcConfig()
        c.batch_words, c.mode, c.anchor, c.order_mode, c.device = cap, 1, -1, 0, local
        c.shard_index, c.shard_count, c.flags = rank, world, 0
        r = _abi.BcReport()
        _abi.check(L.bc_count(pinned[0].data_ptr(), pinned[1].data_ptr(), u.n,
                              pinned[2].data_ptr(), pinned[3].data_ptr(), v.n, p, q,
                              C.byref(c), C.byref(r)))
        e2e_s, h2d, d2h = [], 0, 0
        for _ in range(args.steps):
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            _abi.check(L.bc_count(pinned[0].data_ptr(), pinned[1].data_ptr(), u.n,
                                  pinned[2].data_ptr(), pinned[3].data_ptr(), v.n, p, q,
                                  C.byref(c), C.byref(r)))
            part = int(r.count_lo) | (int(r.count_hi) << 64)
            tot = allreduce_count(part)
            e2e_s.append(time.perf_counter() - t0)
            h2d, d2h = r.h2d_bytes, r.d2h_bytes
            assert tot == total, (tot, total)
        t_e2e = allreduce_max(statistics.mean(e2e_s))
        e2e = {"value": total / t_e2e, "unit": "bicliques/s", "time_s": t_e2e,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "how": "bc_count from pinned host CSR: H2D + device prep + count + D2H, "
                      "plus the 32-byte limb all_reduce when N>1; host wall clock"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = host_cores()
        c_cpu, dt, what = cpu_oracle_run(g, p, q, threads, args.config)
        if c_cpu is not None:
            assert c_cpu == total, (c_cpu, total)
        cpu = {"value": total / dt, "unit": "bicliques/s", "cores": threads, "kind": "port",
               "time_s": dt,
               "sample": f"{args.config} ({p},{q}): {what}: oracle/bicount_oracle.c "
                         f"({threads} pthreads, {cpu_model()})"}

    if rank == 0:
        peak, peak_src = measured_peak()
        work = f"{CONFIG_DESC[args.config]} ({p},{q})"
        tr, tr_src = traffic_for(work) if world == 1 else (None, "captured at N = 1 only")
        b_search = b_enum - b_l1  # the enumeration kernels' share of B_enum
        dram = tr["dram_bytes"] if tr else None
        achieved = dram / t_enum / 1e9 if dram and t_enum > 0 else None
        line = {
            "metric": METRIC, "value": total / (ms / 1e3), "unit": "bicliques/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "time_s": ms / 1e3, "count": total, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32-bitset/u128-count", "data": "synthetic",
            "config": {"workload": work, "config": args.config, "p": p, "q": q,
                       "anchor": "UV"[instr.anchor], "tasks": instr.tasks_emitted,
                       "parallelism": f"root-shard{world}" + ("+2hop-shard" if world > 1 else ""),
                       "dist_backend": args.dist_backend if world > 1 else None,
                       "count_check": "equals tests/golden" if want is not None else "oracle in tests",
                       "l2": "flushed between timed steps (256 MiB device write)"},
            "phases_ms": {"prep": 1e3 * statistics.mean(prep_s),
                          "level1": 1e3 * statistics.mean(level1_s),
                          "enum": 1e3 * statistics.mean(enum_s)},
            "roofline": {
                "bound": "hbm",
                "kernel": "enumeration kernels of one step (rfilter_kernel / filter_kernel, "
                          "enum_kernel triage/split/whole-task launches, sub_kernel), the "
                          "dominant phase",
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak if achieved else None,
                "traffic": dram,
                "achieved_is": "DRAM bytes of those kernels per step (ncu capture of this "
                               "build) / their in-run CUDA-event time",
                "traffic_source": tr_src,
                "algorithmic_bytes": comp,
                "algorithmic": "compulsory bytes: every input the enumeration kernels read, "
                               "once (tasks, level-1 facts, queue, C_R1 edge lists, restricted "
                               "rows + offsets + member ids, rank positions, dir2 HTB); "
                               "traffic / algorithmic = re-read factor",
                "algorithmic_frac": comp / t_enum / 1e9 / peak if t_enum > 0 else None,
                "l2_bytes": tr["l2_bytes"] if tr else None,
                "l2_gbs": tr["l2_bytes"] / t_enum / 1e9 if tr and t_enum > 0 else None,
                "merge_equiv_bytes": b_search,
                "merge_equiv_gbs": b_search / t_enum / 1e9 if t_enum > 0 else None,
                "merge_equiv": "B_enum (SURVEY 8(d)) below level 1: 8 B x sum(|a|+|b|) HTB "
                               "words over the reference's intersections (device tally == "
                               "oracle); the kernels re-index into task-local bitsets and "
                               "never move these bytes",
                "b_enum_total_bytes": b_enum, "b_min_bytes": b_min,
                "launch_ms": 1e3 * t_enum, "share_of_step": t_enum / (ms / 1e3),
                "units": f"{instr.tasks_emitted} (root, second) tasks",
                "peak_source": peak_src},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches_all, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    dg.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
