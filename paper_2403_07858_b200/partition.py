"""BCPar: memory-budgeted partitioning of the anchor layer, and counting by closures.

Mirrors the reference's ``bicount.partition`` interface (``pkg/src/bicount/
partition.py``) on top of the device path:

* ``build_two_hop_index(g, layer, k)`` — the undirected 2-hop index
  (``graph.py:192-215``), built on the GPU (``bc_prepare``: upper-triangle wedge
  counts, rank split) and symmetrised on the host from the directed lists.
* ``budgeted_partition(g, index, budget)`` — the greedy closure growth of
  ``partition.py:74-171`` (seed by descending average 2-hop weight; admit the
  root whose closure overlaps most; close at the budget; oversize singletons
  warn).  Sequential, host-side, same tie rules (heap on (-benefit, id)).
* ``closure_subgraph(work, closure, group)`` (``partition.py:174-200``).
* ``count_partitioned(g, parts, p, q, cfg, structures=)`` (``partition.py:203-
  272``): every group is counted ON THE GPU on its closure subgraph with the
  global priority order carried in (``rank_override``) and its roots
  (``bc_config.roots``), so each biclique lands in exactly one group.  With
  ``shard=(rank, world)`` a process counts only its share of the groups (dealt
  LPT by closure cost) — closures are the multi-GPU shards for graphs past one
  GPU's memory; ``count_partitioned_distributed`` adds the exact limb allreduce.
* ``write_manifest`` (``partition.py:275-283``).
"""

from __future__ import annotations

import heapq
import warnings
from dataclasses import dataclass
from time import perf_counter

import numpy as np

from .engine import (CountReport, DeviceGraph, EngineConfig, TwoHopIndex, allreduce_count,
                     prepare_structures)
from .graph import BipartiteGraph, CsrView, LAYERS, as_csr, from_edges, transpose


class PartitionError(RuntimeError):
    """Partition does not fit the graph it is being applied to."""


@dataclass
class PartitionSet:
    layer: str
    k: int
    budget: int
    groups: list[list[int]]
    closures: list[list[int]]
    costs: list[int]
    oversize: list[bool]

    @property
    def group_count(self) -> int:
        return len(self.groups)


def _work(g, layer: str) -> BipartiteGraph:
    if layer not in LAYERS:
        raise ValueError(f"layer must be one of {LAYERS}, got {layer!r}")
    u, v = as_csr(g)
    return BipartiteGraph(u_csr=u, v_csr=v) if layer == "U" else BipartiteGraph(u_csr=v, v_csr=u)


def build_two_hop_index(g, layer: str, k: int, *, device: int = 0) -> TwoHopIndex:
    """Undirected 2-hop lists of ``layer`` with multiplicity >= k (graph.py:192-215), from
    the device: the directed lists hold each pair once, so the union of both directions
    is the undirected index."""
    if k < 1:
        raise ValueError("k must be >= 1")
    work = _work(g, layer)
    n = work.u_count
    if n == 0 or work.edge_count == 0:
        return TwoHopIndex(k, layer, CsrView(np.zeros(n + 1, np.int64), np.empty(0, np.int32)),
                           directed=False)
    s = prepare_structures(work, 2, k, anchor="U", device=device)
    d = s.dir2.csr
    src = np.repeat(np.arange(n, dtype=np.int64), d.degrees())
    dst = d.idx.astype(np.int64)
    key = np.sort(np.concatenate([src * n + dst, dst * n + src]))
    a = key // n
    off = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(a, minlength=n), out=off[1:])
    return TwoHopIndex(k, layer, CsrView(off, (key - a * n).astype(np.int32)), directed=False)


def entry_weight(g, index: TwoHopIndex) -> np.ndarray:
    """Per-vertex entry cost: 1-hop plus 2-hop list lengths (partition.py:61-65)."""
    work = _work(g, index.layer)
    return work.u_csr.degrees().astype(np.int64) + index.csr.degrees().astype(np.int64)


def closure_cost(g, index: TwoHopIndex, closure) -> int:
    return int(entry_weight(g, index)[np.asarray(list(closure), dtype=np.int64)].sum())


def budgeted_partition(g, index: TwoHopIndex, budget: int) -> PartitionSet:
    """Greedy groups whose closures fit ``budget`` entries (partition.py:74-171)."""
    if index.directed:
        raise ValueError("partitioning needs the undirected 2-hop index")
    if budget < 1:
        raise ValueError("budget must be >= 1")
    work = _work(g, index.layer)
    n = work.u_count
    two = index.csr
    if two.n != n:
        raise ValueError("index does not match the graph layer")
    w = entry_weight(g, index)
    toff, tidx = two.off, two.idx.astype(np.int64)
    tdeg = np.diff(toff)
    # average weight of each vertex's 2-hop neighbours (float64 sum / count, as the reference)
    seg = np.add.reduceat(w[tidx], toff[:-1][tdeg > 0]) if len(tidx) else np.empty(0, np.int64)
    avg = np.zeros(n, np.float64)
    avg[tdeg > 0] = seg.astype(np.float64) / tdeg[tdeg > 0]
    # reverse reach: roots v whose 2-hop list holds x, ascending v
    order = np.argsort(tidx, kind="stable")
    rin_idx = np.repeat(np.arange(n, dtype=np.int64), tdeg)[order]
    rin_off = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(tidx, minlength=n), out=rin_off[1:])
    seeds = np.lexsort((np.arange(n), -avg))

    wl = w.tolist()
    tl = [tidx[toff[i]:toff[i + 1]].tolist() for i in range(n)]
    rl = [rin_idx[rin_off[i]:rin_off[i + 1]].tolist() for i in range(n)]
    assigned = bytearray(n)
    in_closure = bytearray(n)
    groups, closures, costs, oversize = [], [], [], []
    for seed in seeds.tolist():
        if assigned[seed]:
            continue
        assigned[seed] = 1
        group = [seed]
        members = sorted({seed, *tl[seed]})
        for x in members:
            in_closure[x] = 1
        cost = sum(wl[x] for x in members)
        benefit: dict[int, int] = {}
        heap: list[tuple[int, int]] = []

        def admit(xs):
            for x in xs:  # x just joined: every unassigned root reaching x saves w(x)
                wx = wl[x]
                for v in rl[x]:
                    if not assigned[v]:
                        b = benefit.get(v, 0) + wx
                        benefit[v] = b
                        heapq.heappush(heap, (-b, v))

        admit(members)
        while True:
            cand = None
            while heap:
                nb, v = heapq.heappop(heap)
                if not assigned[v] and benefit.get(v) == -nb:
                    cand = v
                    break
            if cand is None:
                break
            fresh = [x for x in [cand] + tl[cand] if not in_closure[x]]
            added = sum(wl[x] for x in fresh)
            if cost + added > budget:
                break
            assigned[cand] = 1
            del benefit[cand]
            group.append(cand)
            cost += added
            for x in fresh:
                in_closure[x] = 1
            members.extend(fresh)
            admit(fresh)
        over = cost > budget
        if over:
            warnings.warn(f"vertex {seed} needs {cost} entries alone, over budget {budget}; "
                          "kept as its own oversize group", RuntimeWarning)
        members.sort()
        for x in members:
            in_closure[x] = 0
        groups.append(group)
        closures.append(members)
        costs.append(cost)
        oversize.append(over)
    return PartitionSet(layer=index.layer, k=index.k, budget=budget, groups=groups,
                        closures=closures, costs=costs, oversize=oversize)


def closure_subgraph(work, closure, group):
    """Closure rows plus their whole 1-hop fringe (partition.py:174-200): returns
    (subgraph, anchor ids, local root ids).  ``work`` has the partitioned layer as U."""
    u, _ = as_csr(work)
    anchor = np.asarray(closure, dtype=np.int64)
    m = len(anchor)
    deg = (u.off[anchor + 1] - u.off[anchor]) if m else np.empty(0, np.int64)
    if m and deg.sum():
        starts = np.repeat(u.off[anchor] - np.concatenate([[0], np.cumsum(deg)[:-1]]), deg)
        flat = u.idx[starts + np.arange(int(deg.sum()))].astype(np.int64)
        vids, ev = np.unique(flat, return_inverse=True)
        eu = np.repeat(np.arange(m, dtype=np.int64), deg)
    else:
        vids = np.empty(0, np.int64)
        eu = ev = np.empty(0, np.int64)
    amap = np.full(u.n, -1, dtype=np.int64)
    amap[anchor] = np.arange(m)
    roots_local = amap[np.asarray(group, dtype=np.int64)]
    if np.any(roots_local < 0):
        raise PartitionError("integrity: group member missing from its closure")
    return from_edges(m, len(vids), eu, ev), anchor, roots_local


def shard_groups(parts: PartitionSet, world: int) -> list[list[int]]:
    """Group indices per rank: LPT by closure cost, snake order (heaviest first)."""
    order = sorted(range(parts.group_count), key=lambda i: (-parts.costs[i], i))
    out: list[list[int]] = [[] for _ in range(world)]
    for j, i in enumerate(order):
        r = j % (2 * world)
        out[r if r < world else 2 * world - 1 - r].append(i)
    return [sorted(x) for x in out]


def count_partitioned(g, parts: PartitionSet, p: int, q: int, cfg: EngineConfig | None = None,
                      *, structures=None, shard: tuple[int, int] = (0, 1)) -> CountReport:
    """Count group by group on the GPU and sum (partition.py:203-272); with ``shard``,
    only this process's share of the groups."""
    cfg = cfg if cfg is not None else EngineConfig()
    cfg.validate()
    if p < 1 or q < 1:
        raise ValueError("p and q must be >= 1")
    p_eff, q_eff = (p, q) if parts.layer == "U" else (q, p)
    if parts.k != q_eff:
        raise PartitionError(f"partition was built on k={parts.k} 2-hop lists but counting "
                             f"({p},{q}) anchored on {parts.layer} needs k={q_eff}")
    work = g if parts.layer == "U" else transpose(g)
    work = _work(work, "U")
    n = work.u_count
    flat = (np.concatenate([np.asarray(x, dtype=np.int64) for x in parts.groups])
            if parts.groups else np.empty(0, np.int64))
    if not np.array_equal(np.sort(flat), np.arange(n)):
        raise PartitionError("groups must cover the anchor layer exactly once")
    if structures is not None:
        if structures.choice.layer != parts.layer or structures.choice.q_eff != q_eff:
            raise PartitionError("supplied structures disagree with the partition")
        grank = np.asarray(structures.order.rank, np.int64)
        und = np.asarray(structures.und_sizes, np.int64)
    elif n and work.edge_count:
        s = prepare_structures(work, p_eff, q_eff, anchor="U", device=cfg.device)
        grank, und = s.order.rank, np.asarray(s.und_sizes, np.int64)
    else:
        grank = np.arange(n, 0, -1, dtype=np.int64)
        und = np.zeros(n, np.int64)
    sub_cfg = EngineConfig(worker_count=cfg.worker_count,
                           batch_buffer_capacity=cfg.batch_buffer_capacity, mode=cfg.mode,
                           anchor="U", check_nesting=cfg.check_nesting, device=cfg.device)
    mine = shard_groups(parts, shard[1])[shard[0]] if shard[1] > 1 else range(parts.group_count)
    total = 0
    t1 = t2 = wall = 0.0
    batches = stolen = emitted = consumed = filtered = 0
    for i in mine:
        if p_eff >= 2 and (not parts.groups[i] or und[parts.groups[i]].max() < p_eff - 1):
            # every root fails the task filter (engine.py:155-162; a root's 2-hop list
            # lies inside its closure, so its size is the global one): no device call
            filtered += len(parts.groups[i])
            continue
        sub, anchor, roots_local = closure_subgraph(work, parts.closures[i], parts.groups[i])
        dg = DeviceGraph(sub, cfg.device)
        try:
            t0 = perf_counter()
            rep, _ = dg.count_raw(p_eff, q_eff, sub_cfg, anchor="U", rank=grank[anchor],
                                  roots=roots_local)
            wall += perf_counter() - t0
        finally:
            dg.close()
        total += int(rep.count_lo) | (int(rep.count_hi) << 64)
        t1 += rep.time_level1
        t2 += rep.time_enum
        batches += rep.batches_executed
        stolen += rep.tasks_stolen
        emitted += rep.tasks_emitted
        consumed += rep.tasks_consumed
        filtered += rep.roots_filtered
    return CountReport(count=total, time_1hop=t1, time_2hop=t2, batches_executed=batches,
                       tasks_stolen=stolen, roots_filtered=filtered, wall_time=wall,
                       tasks_emitted=emitted, tasks_consumed=consumed, workers=cfg.worker_count,
                       anchor_layer=parts.layer)


def count_partitioned_distributed(g, parts: PartitionSet, p: int, q: int,
                                  cfg: EngineConfig | None = None, *, rank: int, world: int,
                                  group=None, structures=None) -> tuple[int, CountReport]:
    """One process per GPU: this rank counts its closures; the exact total is the
    allreduce of the partial counts' 32-bit limbs.  Returns (total, local report)."""
    local = count_partitioned(g, parts, p, q, cfg, structures=structures, shard=(rank, world))
    import torch

    dev = torch.device("cuda", (cfg or EngineConfig()).device) if torch.cuda.is_available() else None
    return allreduce_count(local.count, group, dev), local


def write_manifest(parts: PartitionSet, path) -> None:
    """Audit dump, one line per group: id, cost, oversize flag, roots (partition.py:275-283)."""
    with open(path, "w") as fh:
        fh.write(f"# layer {parts.layer} k {parts.k} budget {parts.budget} "
                 f"groups {parts.group_count}\n")
        fh.write("# group cost oversize roots...\n")
        for i, grp in enumerate(parts.groups):
            fh.write(f"{i} {parts.costs[i]} {int(parts.oversize[i])} {' '.join(map(str, grp))}\n")
