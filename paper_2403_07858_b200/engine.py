"""Drop-in counting entry point backed by the sm_100a library.

Mirrors the reference engine surface (``pkg/src/bicount/engine.py``):

* ``EngineConfig`` (engine.py:43-61) — same fields, defaults and
  ``validate()`` errors, plus device knobs (``device``, ``order_mode``).
* ``CountReport`` (engine.py:64-79) — same fields; ``device`` carries the
  library's own measurements (phase times, structure sizes, counters).
* ``count_bicliques(g, p, q, cfg, *, structures=None, roots=None)``
  (engine.py:419-500) — exact Python-int count computed on the GPU.
* ``prepare_structures(g, p, q, anchor="auto", rank=None)``
  (engine.py:115-144) — built on the GPU, exported back to host arrays.

``worker_count`` is validated exactly as in the reference but does not
change the device schedule (warps pull tasks from one atomic queue).  The
reference's in-call parallelism (engine.py:449-478: one call, several workers)
maps to ``EngineConfig(devices=(0, 1, ...))``: one host thread per listed GPU,
each counting its shard of the tasks, exact partials summed in the call.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from time import perf_counter

import numpy as np

from . import _abi
from .graph import BipartiteGraph, CsrView, as_csr

MODES = ("dfs", "hybrid")
ANCHOR_FLAGS = ("auto", "U", "V")
ORDER_MODES = ("reference", "fast", "fast-reorder")
KERNEL_CHOICES = ("auto", "scatter", "probe")


@dataclass
class EngineConfig:
    worker_count: int = 1
    batch_buffer_capacity: int = 4096  # scratch words per level (reference semantics)
    mode: str = "hybrid"
    anchor: str = "auto"
    enumerate_results: bool = False
    track_tasks: bool = False
    check_nesting: bool = False
    # device knobs (not in the reference)
    device: int = 0
    order_mode: str = "reference"
    instrument: bool = False  # tally reference-equivalent intersections (B_enum)
    level1: str = "auto"      # "scatter" (root-grouped wedge walk) | "probe" (per-task HTB)
    rows: str = "auto"        # candidate rows: "scatter" | "probe"
    restricted_rows: bool = True  # scatter walks read N(v) & dir2(root), not all of N(v)
    force_triage: bool = False    # p_eff >= 5: filter + triage path whatever the task count
    shard_mode: str = "root"  # multi-GPU: whole roots, degree-balanced | "task" interleave
    devices: tuple | None = None  # one call over several GPUs (thread per device); None: device

    def validate(self) -> None:
        if self.worker_count < 1:
            raise ValueError("worker_count must be >= 1")
        if self.batch_buffer_capacity < 1:
            raise ValueError("batch_buffer_capacity must be >= 1")
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")
        if self.anchor not in ANCHOR_FLAGS:
            raise ValueError(f"anchor must be one of {ANCHOR_FLAGS}")
        if self.order_mode not in ORDER_MODES:
            raise ValueError(f"order_mode must be one of {ORDER_MODES}")
        if self.level1 not in KERNEL_CHOICES or self.rows not in KERNEL_CHOICES:
            raise ValueError(f"level1 / rows must be one of {KERNEL_CHOICES}")
        if self.shard_mode not in ("root", "task"):
            raise ValueError("shard_mode must be one of ('root', 'task')")
        if self.devices is not None and (len(self.devices) < 1 or
                                         any(int(d) < 0 for d in self.devices)):
            raise ValueError("devices must list at least one device index >= 0")


@dataclass
class CountReport:
    count: int
    time_1hop: float
    time_2hop: float
    batches_executed: int
    tasks_stolen: int
    roots_filtered: int
    wall_time: float
    tasks_emitted: int
    tasks_consumed: int
    workers: int
    anchor_layer: str
    bicliques: list | None = None
    task_tally: list | None = None
    task_counts: list | None = None
    device: dict = field(default_factory=dict)


@dataclass
class AnchorChoice:  # graph.py:76-80
    layer: str
    p_eff: int
    q_eff: int


@dataclass
class PriorityOrder:  # graph.py:67-73
    rank: np.ndarray
    order: np.ndarray


@dataclass
class TwoHopIndex:  # graph.py:52-64 (directed lists as CSR)
    k: int
    layer: str
    csr: CsrView
    directed: bool

    @property
    def lists(self) -> list[np.ndarray]:
        return [self.csr.row(i) for i in range(self.csr.n)]

    @property
    def sizes(self) -> np.ndarray:
        return self.csr.degrees()


@dataclass
class Htb:  # htb.py:64-86
    off: np.ndarray
    idx: np.ndarray
    val: np.ndarray

    @property
    def n_sets(self) -> int:
        return len(self.off) - 1

    @property
    def n_words(self) -> int:
        return len(self.idx)


@dataclass
class SearchStructures:  # engine.py:82-92, exported from device
    choice: AnchorChoice
    work: BipartiteGraph
    und_sizes: np.ndarray
    order: PriorityOrder
    dir2: TwoHopIndex
    adj_htb: Htb
    dir2_htb: Htb
    tasks: np.ndarray  # int32[(emitted, 2)] in emission order (engine.py:147-173)


def _csr_arrays(g):
    u, v = as_csr(g)
    arrs = [np.ascontiguousarray(u.off, np.int64), np.ascontiguousarray(u.idx, np.int32),
            np.ascontiguousarray(v.off, np.int64), np.ascontiguousarray(v.idx, np.int32)]
    return arrs, u.n, v.n


def _make_config(cfg: EngineConfig, anchor: str, rank, roots, shard=(0, 1), flags=0):
    c = _abi.BcConfig()
    c.batch_words = int(cfg.batch_buffer_capacity)
    c.mode = 0 if cfg.mode == "dfs" else 1
    c.anchor = {"auto": -1, "U": 0, "V": 1}[anchor]
    c.order_mode = ORDER_MODES.index(cfg.order_mode)
    c.device = int(cfg.device)
    c.shard_index, c.shard_count = int(shard[0]), int(shard[1])
    c.flags = flags | (_abi.BC_FLAG_INSTRUMENT if cfg.instrument else 0)
    c.flags |= {"auto": 0, "scatter": _abi.BC_FLAG_L1_SCATTER, "probe": _abi.BC_FLAG_L1_PROBE}[cfg.level1]
    c.flags |= {"auto": 0, "scatter": _abi.BC_FLAG_ROWR_SCATTER,
                "probe": _abi.BC_FLAG_ROWR_PROBE}[cfg.rows]
    if not cfg.restricted_rows:
        c.flags |= _abi.BC_FLAG_FULL_ROWS
    if cfg.force_triage:
        c.flags |= _abi.BC_FLAG_FORCE_TRIAGE
    if cfg.shard_mode == "task":
        c.flags |= _abi.BC_FLAG_TASK_SHARD
    keep = []
    if rank is not None:
        r = np.ascontiguousarray(rank, dtype=np.int64)
        keep.append(r)
        c.rank_override = r.ctypes.data
        c.n_rank = len(r)
    if roots is not None:
        rr = np.fromiter((int(x) for x in roots), dtype=np.int64)
        rr = rr[(rr >= -(2**31)) & (rr < 2**31)].astype(np.int32)
        keep.append(rr)
        c.roots = rr.ctypes.data if len(rr) else keep_empty(keep)
        c.n_roots = len(rr)
    return c, keep


def keep_empty(keep):
    z = np.zeros(1, dtype=np.int32)
    keep.append(z)
    return z.ctypes.data


class DeviceGraph:
    """A graph resident in HBM (``bc_graph``): upload once, count many times."""

    def __init__(self, g, device: int = 0):
        L = _abi.load()
        (uo, ui, vo, vi), nu, nv = _csr_arrays(g)
        h = C.c_void_p()
        _abi.check(L.bc_graph_create(uo.ctypes.data, ui.ctypes.data, nu, vo.ctypes.data,
                                     vi.ctypes.data, nv, device, C.byref(h)))
        self._h = h
        self.device = device
        self.u_count, self.v_count = nu, nv

    @classmethod
    def from_device_csr(cls, u_off, u_idx, v_off, v_idx, device: int = 0) -> "DeviceGraph":
        """Adopt a CSR already in HBM (torch CUDA tensors: int64 offsets, int32
        ids), e.g. ``synth.fr_shaped_csr(device="cuda")``; copied device to device."""
        L = _abi.load()
        ts = [u_off, u_idx, v_off, v_idx]
        for t, dt in zip(ts, ("int64", "int32", "int64", "int32")):
            if not t.is_cuda or str(t.dtype) != f"torch.{dt}" or not t.is_contiguous():
                raise ValueError("device CSR must be contiguous CUDA tensors (int64 off, int32 idx)")
        self = cls.__new__(cls)
        h = C.c_void_p()
        nu, nv = u_off.numel() - 1, v_off.numel() - 1
        _abi.check(L.bc_graph_create_device(u_off.data_ptr(), u_idx.data_ptr(), nu,
                                            v_off.data_ptr(), v_idx.data_ptr(), nv, device,
                                            C.byref(h)))
        self._h = h
        self.device = device
        self.u_count, self.v_count = nu, nv
        return self

    def twohop_slice(self, p: int, q: int, cfg: EngineConfig | None = None, *, anchor=None,
                     shard=(0, 1)):
        """This shard's upper 2-hop lists (sharded preprocessing): (lens int32[n] with 0 for
        anchors of other shards, ids int32[]) as CUDA tensors (bc_graph_twohop_slice)."""
        import torch

        cfg = cfg if cfg is not None else EngineConfig()
        cfg.validate()
        L = _abi.load()
        c, keep = _make_config(cfg, anchor or cfg.anchor, None, None)
        h = C.c_void_p()
        _abi.check(L.bc_graph_twohop_slice(self._h, int(p), int(q), C.byref(c), int(shard[0]),
                                           int(shard[1]), C.byref(h)))
        try:
            dev = torch.device("cuda", cfg.device)
            out = []
            for what in (_abi.BC_X_SLICE_LENS, _abi.BC_X_SLICE_IDS):
                t = torch.empty(max(int(L.bc_export_len(h, what)), 0), dtype=torch.int32, device=dev)
                _abi.check(L.bc_export_device(h, what, t.data_ptr() if t.numel() else None))
                out.append(t)
        finally:
            L.bc_structs_destroy(h)
        del keep
        return out[0], out[1]

    def htb_arenas(self, p: int, q: int, cfg: EngineConfig | None = None, *, anchor=None,
                   rank=None):
        """The device-built HTB arenas of (p, q) as CUDA tensors, without a host round trip:
        {"adj": (off int64, idx int32, val int32), "dir2": (...)} -- the u32 words of
        htb.py:64-86 viewed as int32 (compare with ``htb.load_htb_device``)."""
        import torch

        cfg = cfg if cfg is not None else EngineConfig()
        cfg.validate()
        L = _abi.load()
        c, keep = _make_config(cfg, anchor or cfg.anchor, rank, None)
        h = C.c_void_p()
        _abi.check(L.bc_prepare(self._h, int(p), int(q), C.byref(c), C.byref(h)))
        try:
            dev = torch.device("cuda", cfg.device)
            out = {}
            for name, ids in (("adj", (_abi.BC_X_HADJ_OFF, _abi.BC_X_HADJ_IDX, _abi.BC_X_HADJ_VAL)),
                              ("dir2", (_abi.BC_X_HDIR_OFF, _abi.BC_X_HDIR_IDX, _abi.BC_X_HDIR_VAL))):
                ts = []
                for what, dt in zip(ids, (torch.int64, torch.int32, torch.int32)):
                    t = torch.empty(max(int(L.bc_export_len(h, what)), 0), dtype=dt, device=dev)
                    _abi.check(L.bc_export_device(h, what, t.data_ptr() if t.numel() else None))
                    ts.append(t)
                out[name] = tuple(ts)
        finally:
            L.bc_structs_destroy(h)
        del keep
        return out

    def count_raw(self, p: int, q: int, cfg: EngineConfig | None = None, *, anchor=None,
                  rank=None, roots=None, shard=(0, 1), task_counts: bool = False, upper=None):
        """One counting pass; returns (BcReport, per-task counts or None).  ``upper`` =
        (off int64[n+1], ids int32[]) CUDA tensors: the whole upper 2-hop CSR from the
        shards' slices (``assemble_upper``), so the 2-hop construction is skipped."""
        cfg = cfg if cfg is not None else EngineConfig()
        cfg.validate()
        if p < 1 or q < 1:
            raise ValueError("p and q must be >= 1")
        L = _abi.load()
        flags = _abi.BC_FLAG_TASK_COUNTS if task_counts else 0
        c, keep = _make_config(cfg, anchor or cfg.anchor, rank, roots, shard, flags)
        tc = None
        if task_counts:
            # the emitted count is only known on device: size by directed pairs bound
            cap = max(1, _task_bound(self, p, q, cfg, anchor, rank))
            tc = np.zeros(2 * cap, dtype=np.uint64)
            c.task_counts = tc.ctypes.data
            c.task_counts_cap = cap
        rep = _abi.BcReport()
        if upper is None:
            _abi.check(L.bc_graph_count(self._h, int(p), int(q), C.byref(c), C.byref(rep)))
        else:
            off, ids = upper
            _abi.check(L.bc_graph_count_upper(self._h, int(p), int(q), C.byref(c),
                                              off.data_ptr(), ids.data_ptr() if ids.numel() else None,
                                              int(ids.numel()), C.byref(rep)))
        del keep
        per_task = None
        if task_counts:
            e = rep.tasks_emitted
            lo = tc[0:2 * e:2].astype(object)
            hi = tc[1:2 * e:2].astype(object)
            per_task = [int(a) | (int(b) << 64) for a, b in zip(lo, hi)]
        return rep, per_task

    def close(self):
        if getattr(self, "_h", None):
            _abi.load().bc_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _task_bound(dg: DeviceGraph, p, q, cfg, anchor, rank) -> int:
    s = _prepare_device(dg, p, q, cfg, anchor or cfg.anchor, rank)
    try:
        return int(_export(s, _abi.BC_X_TASKS).size // 2)
    finally:
        _abi.load().bc_structs_destroy(s)


def _prepare_device(dg: DeviceGraph, p, q, cfg, anchor, rank, roots=None):
    L = _abi.load()
    c, keep = _make_config(cfg, anchor, rank, roots)
    h = C.c_void_p()
    _abi.check(L.bc_prepare(dg._h, int(p), int(q), C.byref(c), C.byref(h)))
    del keep
    return h


_EXPORT_DT = {
    _abi.BC_X_UND_SIZE: np.int64, _abi.BC_X_RANK: np.int64, _abi.BC_X_ORDER: np.int64,
    _abi.BC_X_DIR_OFF: np.int64, _abi.BC_X_DIR_IDX: np.int32, _abi.BC_X_HADJ_OFF: np.int64,
    _abi.BC_X_HADJ_IDX: np.uint32, _abi.BC_X_HADJ_VAL: np.uint32, _abi.BC_X_HDIR_OFF: np.int64,
    _abi.BC_X_HDIR_IDX: np.uint32, _abi.BC_X_HDIR_VAL: np.uint32, _abi.BC_X_TASKS: np.int32,
    _abi.BC_X_META: np.int64,
}


def _export(h, what: int) -> np.ndarray:
    L = _abi.load()
    n = L.bc_export_len(h, what)
    out = np.empty(max(n, 0), dtype=_EXPORT_DT[what])
    if n > 0:
        _abi.check(L.bc_export(h, what, out.ctypes.data))
    return out


def prepare_structures(g, p: int, q: int, anchor: str = "auto", rank=None,
                       device: int = 0, roots=None) -> SearchStructures:
    """Device-built structures, exported (engine.py:115-144)."""
    if p < 1 or q < 1:
        raise ValueError("p and q must be >= 1")
    if anchor not in ANCHOR_FLAGS:
        raise ValueError(f"anchor must be one of {ANCHOR_FLAGS}")
    dg = DeviceGraph(g, device)
    cfg = EngineConfig(device=device)
    h = _prepare_device(dg, p, q, cfg, anchor, rank, roots)
    L = _abi.load()
    try:
        meta = _export(h, _abi.BC_X_META)
        layer = "UV"[int(meta[0])]
        choice = AnchorChoice(layer, int(meta[1]), int(meta[2]))
        u, v = as_csr(g)
        work = BipartiteGraph(u_csr=u, v_csr=v) if layer == "U" else BipartiteGraph(u_csr=v, v_csr=u)
        dir2 = TwoHopIndex(choice.q_eff, "U",
                           CsrView(_export(h, _abi.BC_X_DIR_OFF), _export(h, _abi.BC_X_DIR_IDX)),
                           directed=True)
        return SearchStructures(
            choice=choice, work=work, und_sizes=_export(h, _abi.BC_X_UND_SIZE),
            order=PriorityOrder(_export(h, _abi.BC_X_RANK), _export(h, _abi.BC_X_ORDER)),
            dir2=dir2,
            adj_htb=Htb(_export(h, _abi.BC_X_HADJ_OFF), _export(h, _abi.BC_X_HADJ_IDX),
                        _export(h, _abi.BC_X_HADJ_VAL)),
            dir2_htb=Htb(_export(h, _abi.BC_X_HDIR_OFF), _export(h, _abi.BC_X_HDIR_IDX),
                         _export(h, _abi.BC_X_HDIR_VAL)),
            tasks=_export(h, _abi.BC_X_TASKS).reshape(-1, 2))
    finally:
        L.bc_structs_destroy(h)
        dg.close()


def _report(rep: _abi.BcReport, cfg: EngineConfig, wall: float, anchor_layer: str,
            per_task=None) -> CountReport:
    d = rep.as_dict()
    return CountReport(
        count=d["count"], time_1hop=rep.time_level1, time_2hop=rep.time_enum,
        batches_executed=rep.batches_executed, tasks_stolen=rep.tasks_stolen,
        roots_filtered=rep.roots_filtered, wall_time=wall, tasks_emitted=rep.tasks_emitted,
        tasks_consumed=rep.tasks_consumed, workers=cfg.worker_count, anchor_layer=anchor_layer,
        task_counts=per_task, device=d)


def task_bound(u_off, u_idx, v_off, v_idx, p: int) -> int:
    """Upper bound on tasks_emitted for either anchor layer, from host CSR: one task per
    anchor when p_eff = 1, else one per directed 2-hop pair, and an anchor's undirected
    2-hop list holds at most min(n - 1, sum over its neighbours v of deg(v) - 1) ids
    (graph.py:192-224), each pair counted from both ends."""
    best = 0
    for aoff, aidx, boff in ((u_off, u_idx, v_off), (v_off, v_idx, u_off)):
        n = len(aoff) - 1
        if p <= 1 or n == 0:
            best = max(best, n)
            continue
        dm1 = np.diff(boff) - 1
        per = np.zeros(n, dtype=np.int64)
        if len(aidx):
            w = np.concatenate([[0], np.cumsum(dm1[aidx], dtype=np.int64)])
            per = w[aoff[1:]] - w[aoff[:-1]]
        best = max(best, int((np.minimum(per, n - 1).sum() + 1) // 2), n)
    return best


def task_tally(claims: np.ndarray, emitted: int, workers: int):
    """(task_tally, task_counts) in the reference's terms (engine.py:446,462,473,498-499):
    task t of the round-robin emission is entry (t % workers, t // workers); the device
    logs how many times each task was claimed, so a task run twice appears twice and a
    task never run does not appear."""
    c = claims[:emitted].astype(np.int64)
    t = np.repeat(np.arange(emitted, dtype=np.int64), c)
    tally = list(zip((t % workers).tolist(), (t // workers).tolist()))
    counts = [(emitted - w + workers - 1) // workers for w in range(workers)]
    return tally, counts


def count_bicliques(g, p: int, q: int, cfg: EngineConfig | None = None, *,
                    structures=None, roots=None) -> CountReport:
    """Exact (p,q)-biclique count on the GPU (engine.py:419-500).

    ``structures`` (ours or the reference's ``SearchStructures``) fixes the
    anchor layer and the priority rank, as in the reference's partitioned
    counting (partition.py:246-249); the device rebuilds the rest itself.
    ``roots`` restricts which anchor vertices root tasks (engine.py:155-162).
    ``wall_time`` covers the counting phase (level 1 + enumeration, device
    events), not structure preparation, as in the reference (engine.py:432,492);
    ``device["time_total"]`` is the whole call.  ``track_tasks`` fills
    ``task_tally`` / ``task_counts`` from the device's per-task claim log;
    ``check_nesting`` runs the device nesting check (AssertionError on a
    violation, as the reference's assert, engine.py:365-366).
    """
    cfg = cfg if cfg is not None else EngineConfig()
    cfg.validate()
    if p < 1 or q < 1:
        raise ValueError("p and q must be >= 1")
    anchor, rank, graph, pp, qq = cfg.anchor, None, g, p, q
    if structures is not None:
        # the reference reads s.work / s.choice / s.order only (engine.py:430-434)
        graph = structures.work
        anchor = "U"
        pp, qq = structures.choice.p_eff, structures.choice.q_eff
        rank = np.asarray(structures.order.rank, dtype=np.int64)
    L = _abi.load()
    (uo, ui, vo, vi), nu, nv = _csr_arrays(graph)
    flags = (_abi.BC_FLAG_TRACK_TASKS if cfg.track_tasks else 0) | (
        _abi.BC_FLAG_CHECK_NESTING if cfg.check_nesting else 0)
    c, keep = _make_config(cfg, anchor, rank, roots, flags=flags)
    claims = None
    if cfg.track_tasks:
        cap = max(1, task_bound(uo, ui, vo, vi, int(pp)))
        claims = np.zeros(cap, dtype=np.uint32)
        c.task_claims = claims.ctypes.data
        c.task_claims_cap = cap
    devs = tuple(int(d) for d in cfg.devices) if cfg.devices else (int(cfg.device),)
    if len(devs) == 1:
        c.device = devs[0]
        rep = _abi.BcReport()
        _abi.check(L.bc_count(uo.ctypes.data, ui.ctypes.data, nu, vo.ctypes.data, vi.ctypes.data,
                              nv, int(pp), int(qq), C.byref(c), C.byref(rep)))
        wall = rep.time_level1 + rep.time_enum
    else:
        rep, wall = _count_devices(L, (uo, ui, vo, vi), nu, nv, pp, qq, c, devs, claims)
    del keep
    layer = structures.choice.layer if structures is not None else "UV"[rep.anchor]
    out = _report(rep, cfg, wall, layer)
    if claims is not None:
        out.task_tally, out.task_counts = task_tally(claims, rep.tasks_emitted, cfg.worker_count)
    if cfg.enumerate_results:
        out.bicliques = enumerate_bicliques(graph, pp, qq, cfg, out.count, layer, anchor=anchor,
                                            rank=rank, roots=roots)
    return out


# CountReport fields of the reference (engine.py:64-79); cli.py:252-257 writes them as
# {"schema": 1, **asdict(report)} for --stats-json
REFERENCE_REPORT_FIELDS = ("count", "time_1hop", "time_2hop", "batches_executed", "tasks_stolen",
                           "roots_filtered", "wall_time", "tasks_emitted", "tasks_consumed",
                           "workers", "anchor_layer", "bicliques", "task_tally", "task_counts")


def stats_payload(report: CountReport, include_device: bool = False) -> dict:
    """The reference CLI's --stats-json payload for this report (cli.py:252-257): schema 1
    plus the reference's CountReport fields, in its order; ``device`` (this library's own
    measurements) only when asked for."""
    d = {"schema": 1}
    for k in REFERENCE_REPORT_FIELDS:
        d[k] = getattr(report, k)
    if include_device:
        d["device"] = dict(report.device)
    return d


def write_stats_json(report: CountReport, path, include_device: bool = False) -> None:
    """cli.py:252-257: json.dump(payload, indent=2, default=int) and a newline."""
    import json

    with open(path, "w") as fh:
        json.dump(stats_payload(report, include_device), fh, indent=2, default=int)
        fh.write("\n")


# report fields summed over the shards of one multi-device call (the rest are global:
# equal on every shard) and the phase times taken as the slowest shard's
_SUMMED = ("tasks_consumed", "tasks_stolen", "batches_executed", "tasks_alive", "tasks_split",
           "intersections", "operand_words", "min_words", "kernel_launches", "h2d_bytes",
           "d2h_bytes", "level1_operand_words", "nesting_checked", "level1_entries")
_MAXED = ("time_h2d", "time_prep", "time_level1", "time_enum", "time_total")


def _count_devices(L, csr, nu, nv, p, q, c, devs, claims):
    """One call over several GPUs (the reference's in-call workers, engine.py:449-478):
    shard k of len(devs) on devs[k], one host thread each (ctypes drops the GIL; the
    library locks per device), exact u128 partials summed.  Returns (merged report,
    wall time of the counting phase = the slowest shard's level 1 + enumeration)."""
    import threading

    uo, ui, vo, vi = csr
    n = len(devs)
    reps = [_abi.BcReport() for _ in range(n)]
    cfgs, logs, errs = [], [], [None] * n
    for k, d in enumerate(devs):
        ck = _abi.BcConfig()
        C.pointer(ck)[0] = c  # copy every field, then this shard's device and index
        ck.device, ck.shard_index, ck.shard_count = d, k, n
        if claims is not None:
            lg = np.zeros_like(claims)
            ck.task_claims, ck.task_claims_cap = lg.ctypes.data, len(lg)
            logs.append(lg)
        cfgs.append(ck)

    def run(k):
        try:
            _abi.check(L.bc_count(uo.ctypes.data, ui.ctypes.data, nu, vo.ctypes.data,
                                  vi.ctypes.data, nv, int(p), int(q), C.byref(cfgs[k]),
                                  C.byref(reps[k])))
        except Exception as e:  # re-raised on the calling thread
            errs[k] = e

    th = [threading.Thread(target=run, args=(k,)) for k in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    out = _abi.BcReport()
    C.pointer(out)[0] = reps[0]
    total = sum(int(r.count_lo) | (int(r.count_hi) << 64) for r in reps)
    if total >> 128:
        raise RuntimeError("bicount_b200 error: the count reached 2^128")
    out.count_lo, out.count_hi = total & ((1 << 64) - 1), total >> 64
    out.overflow = max(r.overflow for r in reps)
    for f in _SUMMED:
        setattr(out, f, sum(getattr(r, f) for r in reps))
    for f in _MAXED:
        setattr(out, f, max(getattr(r, f) for r in reps))
    if claims is not None:
        claims[:] = np.sum(logs, axis=0)
    return out, max(r.time_level1 + r.time_enum for r in reps)


ENUM_GUARD = 10**7


def enumerate_bicliques(g, p: int, q: int, cfg: EngineConfig, count: int, layer: str, *,
                        anchor=None, rank=None, roots=None):
    """Every (p,q)-biclique as (L, R) tuples, sorted (engine.py:301-304, 480-483).

    The search runs on the GPU (``bc_graph_enumerate``: one record per leaf, [L, |C_R|,
    C_R]); the host only expands each record into combinations(C_R, q_eff), swaps the
    pair for a V anchor and sorts.  ``anchor`` / ``rank`` / ``roots`` as in
    ``count_bicliques`` (a caller's ``structures`` fixes the first two)."""
    from itertools import combinations

    if count > ENUM_GUARD:
        raise ValueError(f"refusing enumeration: {count} results exceeds guard {ENUM_GUARD}")
    L = _abi.load()
    dg = DeviceGraph(g, cfg.device)
    try:
        c, keep = _make_config(cfg, anchor or cfg.anchor, rank, roots)
        need = C.c_int64(0)
        cap = 1 << 16
        while True:
            buf = np.zeros(cap, dtype=np.int32)
            rep = _abi.BcReport()
            _abi.check(L.bc_graph_enumerate(dg._h, int(p), int(q), C.byref(c), buf.ctypes.data,
                                            cap, C.byref(need), C.byref(rep)))
            if need.value <= cap:
                break
            cap = int(need.value)
        del keep
    finally:
        dg.close()
    p_eff, q_eff = rep.p_eff, rep.q_eff
    found = []
    rec = buf[:need.value].tolist()
    i = 0
    while i < len(rec):
        left = tuple(sorted(rec[i:i + p_eff]))
        cnt = rec[i + p_eff]
        right = rec[i + p_eff + 1:i + p_eff + 1 + cnt]
        i += p_eff + 1 + cnt
        for r in combinations(right, q_eff):
            found.append((left, r))
    if layer == "V":
        found = [(r, l) for (l, r) in found]
    found.sort()
    return found


# ---------------------------------------------------------------------------
# multi-GPU: shard tasks across ranks, one allreduce of the 128-bit partials
# ---------------------------------------------------------------------------
def split_limbs(x: int) -> list[int]:
    """128-bit count -> four 32-bit limbs (each summed in a u64 lane)."""
    if x < 0 or x >= 1 << 128:
        raise ValueError("partial count outside [0, 2^128)")
    return [(x >> (32 * i)) & 0xFFFFFFFF for i in range(4)]


def merge_limbs(limbs) -> int:
    """Carry-normalise summed limbs (exact for up to 2^32 ranks)."""
    return sum(int(v) << (32 * i) for i, v in enumerate(limbs))


def allreduce_count(partial: int, group=None, device=None) -> int:
    """Sum exact partial counts over a torch.distributed group.

    One ``all_reduce(SUM)`` of 4 x int64 limbs (NCCL over NVLink on GPUs,
    gloo on CPU); each limb holds < 2^32, so the sum is exact for < 2^31
    ranks in a signed 64-bit lane.
    """
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "gloo":
        device = None  # gloo reduces host tensors (CPU tests, one-GPU multi-rank runs)
    t = torch.tensor(split_limbs(partial), dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return merge_limbs(t.cpu().tolist())


def assemble_upper(slices):
    """Whole upper 2-hop CSR from every shard's (lens, ids) slice (each anchor's list comes
    from exactly one shard, in anchor order within a slice): (off int64[n+1], ids int32[])."""
    import torch

    lens = torch.stack([sl[0] for sl in slices]).sum(0).to(torch.int64)
    n = lens.numel()
    off = torch.zeros(n + 1, dtype=torch.int64, device=lens.device)
    torch.cumsum(lens, 0, out=off[1:])
    ids = torch.empty(int(off[-1].item()), dtype=torch.int32, device=lens.device)
    for sl_lens, sl_ids in slices:
        if sl_ids.numel() == 0:
            continue
        l64 = sl_lens.to(torch.int64)
        starts = off[:-1][l64 > 0]
        cnt = l64[l64 > 0]
        first = torch.repeat_interleave(starts - (torch.cumsum(cnt, 0) - cnt), cnt)
        ids[first + torch.arange(sl_ids.numel(), device=lens.device)] = sl_ids
    return off, ids


def assemble_upper_device(lens_all, ids_all, stride: int, n_pairs: int, device: int = 0, *,
                          world: int):
    """``assemble_upper`` on the device (bc_assemble_upper): lens_all int32[world * n],
    ids_all int32[world * stride] (rank r's slice ids at r * stride)."""
    import torch

    L = _abi.load()
    if world < 1 or stride < 1 or lens_all.numel() % world or ids_all.numel() < world * stride:
        raise ValueError("assemble_upper_device: need world >= 1, stride >= 1, "
                         "lens_all of world * n entries and ids_all of world * stride")
    n = lens_all.numel() // world
    off = torch.empty(n + 1, dtype=torch.int64, device=lens_all.device)
    ids = torch.empty(max(n_pairs, 1), dtype=torch.int32, device=lens_all.device)
    got = C.c_int64(0)
    _abi.check(L.bc_assemble_upper(int(device), int(world), int(n), lens_all.data_ptr(),
                                   ids_all.data_ptr(), int(stride), off.data_ptr(), ids.data_ptr(),
                                   int(ids.numel()), C.byref(got)))
    return off, ids[:got.value]


def gather_upper(dg: DeviceGraph, p: int, q: int, cfg: EngineConfig, rank: int, world: int,
                 group=None, anchor=None):
    """Sharded preprocessing: build this rank's 2-hop slice, all-gather every slice
    (NCCL over NVLink; variable sizes padded to the largest), assemble the whole upper CSR."""
    import torch
    import torch.distributed as dist

    lens, ids = dg.twohop_slice(p, q, cfg, anchor=anchor, shard=(rank, world))
    dev = lens.device
    # NCCL gathers device memory directly; gloo (CPU tests) goes through host copies
    cdev = torch.device("cpu") if dist.get_backend(group) == "gloo" else dev
    sizes = [torch.zeros(1, dtype=torch.int64, device=cdev) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([ids.numel()], dtype=torch.int64, device=cdev), group=group)
    mx = max(int(x.item()) for x in sizes)
    pad = torch.zeros(max(mx, 1), dtype=torch.int32, device=cdev)
    pad[:ids.numel()] = ids.to(cdev)
    all_ids = [torch.empty_like(pad) for _ in range(world)]
    all_lens = [torch.empty(lens.numel(), dtype=torch.int32, device=cdev) for _ in range(world)]
    dist.all_gather(all_ids, pad, group=group)
    dist.all_gather(all_lens, lens.to(cdev), group=group)
    total = sum(int(x.item()) for x in sizes)
    return assemble_upper_device(torch.cat(all_lens).to(dev), torch.cat(all_ids).to(dev),
                                 pad.numel(), total, dev.index or 0, world=world)


def count_bicliques_distributed(g, p: int, q: int, cfg: EngineConfig | None = None, *,
                                rank: int, world: int, group=None, dgraph: DeviceGraph | None = None,
                                roots=None, shard_prep: bool = False) -> tuple[int, CountReport]:
    """This rank counts its shard of the tasks (cfg.shard_mode); returns (total, local
    report).  With ``shard_prep`` the 2-hop construction is split across the ranks too
    (``gather_upper``) instead of being replicated."""
    cfg = cfg if cfg is not None else EngineConfig()
    dg = dgraph if dgraph is not None else DeviceGraph(g, cfg.device)
    t0 = perf_counter()
    upper = None
    if shard_prep and world > 1 and cfg.order_mode == "reference":
        upper = gather_upper(dg, p, q, cfg, rank, world, group)
    rep, _ = dg.count_raw(p, q, cfg, roots=roots, shard=(rank, world), upper=upper)
    wall = perf_counter() - t0
    local = _report(rep, cfg, wall, "UV"[rep.anchor])
    import torch

    dev = torch.device("cuda", cfg.device) if torch.cuda.is_available() else None
    total = allreduce_count(local.count, group, dev)
    return total, local
