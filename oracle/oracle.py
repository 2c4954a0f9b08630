"""ctypes front-end of the C oracle (``oracle/bicount_oracle.c``) plus pure
Python restatements for tiny inputs — TEST INFRASTRUCTURE ONLY.

``count(g, p, q, ...)`` restates the reference ``count_bicliques``
(``pkg/src/bicount/engine.py:419-500``) and returns the same report fields
plus the intersection tallies that define B_enum / B_min.
``prepare(g, p, q, ...)`` restates ``prepare_structures``
(``engine.py:115-144``) and exports every intermediate array so the GPU
structures can be compared bit for bit.

``brute_force_count`` restates the reference's independent ground truth
(``pkg/src/bicount/oracle.py:31-56``): subset recursion over U with a
binomial R-count; pure Python, tiny graphs only.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from itertools import combinations
from math import comb

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liborc.so")

X_UND_SIZE, X_RANK, X_ORDER, X_UND_OFF, X_UND_IDX, X_DIR_OFF, X_DIR_IDX, \
    X_HADJ_OFF, X_HADJ_IDX, X_HADJ_VAL, X_HDIR_OFF, X_HDIR_IDX, X_HDIR_VAL, X_META = range(14)

_I64, _I32, _U32 = np.int64, np.int32, np.uint32
_EXPORT_DT = {X_UND_SIZE: _I64, X_RANK: _I64, X_ORDER: _I64, X_UND_OFF: _I64,
              X_UND_IDX: _I32, X_DIR_OFF: _I64, X_DIR_IDX: _I32, X_HADJ_OFF: _I64,
              X_HADJ_IDX: _U32, X_HADJ_VAL: _U32, X_HDIR_OFF: _I64, X_HDIR_IDX: _U32,
              X_HDIR_VAL: _U32, X_META: _I64}


class OrcConfig(C.Structure):
    _fields_ = [("p", C.c_int32), ("q", C.c_int32), ("workers", C.c_int32),
                ("capacity", C.c_int32), ("mode", C.c_int32), ("anchor", C.c_int32),
                ("rank_override", C.c_void_p), ("root_mask", C.c_void_p),
                ("task_words", C.c_void_p), ("task_count", C.c_void_p),
                ("task_l1", C.c_void_p)]


class OrcReport(C.Structure):
    _fields_ = [("count_lo", C.c_uint64), ("count_hi", C.c_uint64),
                ("overflow", C.c_int32), ("anchor", C.c_int32),
                ("p_eff", C.c_int32), ("q_eff", C.c_int32),
                ("batches", C.c_int64), ("stolen", C.c_int64),
                ("roots_filtered", C.c_int64), ("emitted", C.c_int64),
                ("consumed", C.c_int64), ("intersections", C.c_int64),
                ("operand_words", C.c_int64), ("min_words", C.c_int64),
                ("prep_time", C.c_double), ("wall_time", C.c_double),
                ("time_1hop", C.c_double), ("time_2hop", C.c_double)]


def build(force: bool = False) -> str:
    srcs = [os.path.join(HERE, f) for f in ("bicount_oracle.c", "border_oracle.c", "Makefile")]
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            os.path.getmtime(s) for s in srcs):
        subprocess.run(["make", "-s", "-C", HERE, "liborc.so"], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        L.orc_prepare.restype = C.c_void_p
        L.orc_prepare.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                  C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                  C.c_int32]
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_export_len.restype = C.c_int64
        L.orc_export_len.argtypes = [C.c_void_p, C.c_int]
        L.orc_export.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.orc_count.restype = C.c_int
        L.orc_count.argtypes = [C.c_void_p, C.POINTER(OrcConfig), C.POINTER(OrcReport)]
        L.orc_last_error.restype = C.c_char_p
        L.orc_border.restype = C.c_int64
        L.orc_border.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                 C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


def _csr(g):
    """(u_off, u_idx, v_off, v_idx) for this repo's graph or a reference graph."""
    if hasattr(g, "u_csr"):
        return g.u_csr.off, g.u_csr.idx, g.v_csr.off, g.v_csr.idx

    def flat(lists):
        off = np.zeros(len(lists) + 1, dtype=np.int64)
        if lists:
            np.cumsum([len(a) for a in lists], out=off[1:])
        idx = (np.concatenate([np.asarray(a, np.int32) for a in lists])
               if off[-1] else np.empty(0, np.int32))
        return off, np.ascontiguousarray(idx, np.int32)

    uo, ui = flat(list(g.u_adj))
    vo, vi = flat(list(g.v_adj))
    return uo, ui, vo, vi


_ANCHOR = {"auto": -1, "U": 0, "V": 1}


class Prepared:
    """Handle on the oracle's prepared structures (engine.py:82-92)."""

    def __init__(self, g, p: int, q: int, anchor: str = "auto", rank=None, threads: int = 0):
        self._keep = [np.ascontiguousarray(a) for a in _csr(g)]
        uo, ui, vo, vi = self._keep
        rk = None
        if rank is not None:
            rk = np.ascontiguousarray(rank, dtype=np.int64)
            self._keep.append(rk)
        n_u, n_v = len(uo) - 1, len(vo) - 1
        L = lib()
        if anchor not in _ANCHOR:
            raise ValueError(f"anchor must be one of ('auto', 'U', 'V')")
        if rk is not None:
            n_anchor = _anchor_size(uo, vo, anchor)
            if len(rk) != n_anchor:
                raise ValueError("rank override must give one distinct value per anchor vertex")
        h = L.orc_prepare(uo.ctypes.data, ui.ctypes.data, n_u, vo.ctypes.data, vi.ctypes.data,
                          n_v, p, q, _ANCHOR[anchor],
                          rk.ctypes.data if rk is not None else None, threads)
        if not h:
            raise ValueError(L.orc_last_error().decode())
        self.h = h
        meta = self.export(X_META)
        self.anchor = "UV"[int(meta[0])]
        self.p_eff, self.q_eff, self.n = int(meta[1]), int(meta[2]), int(meta[3])

    def export(self, what: int) -> np.ndarray:
        L = lib()
        n = L.orc_export_len(self.h, what)
        out = np.empty(n, dtype=_EXPORT_DT[what])
        if n:
            L.orc_export(self.h, what, out.ctypes.data)
        return out

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            lib().orc_free(h)
            self.h = None


def _anchor_size(uo, vo, anchor):
    if anchor == "U":
        return len(uo) - 1
    if anchor == "V":
        return len(vo) - 1
    du, dv = np.diff(uo), np.diff(vo)
    wu, wv = int((du * (du - 1) // 2).sum()), int((dv * (dv - 1) // 2).sum())
    return len(uo) - 1 if wv <= wu else len(vo) - 1


@dataclass
class OracleReport:
    count: int
    overflow: bool
    anchor_layer: str
    p_eff: int
    q_eff: int
    batches_executed: int
    tasks_stolen: int
    roots_filtered: int
    tasks_emitted: int
    tasks_consumed: int
    intersections: int
    operand_words: int
    min_words: int
    prep_time: float
    wall_time: float
    time_1hop: float
    time_2hop: float
    workers: int
    task_words: np.ndarray | None = None
    task_counts: list | None = None
    task_l1: np.ndarray | None = None

    @property
    def b_enum(self) -> int:
        return 8 * self.operand_words

    @property
    def b_min(self) -> int:
        return 16 * self.min_words


def count(g, p: int, q: int, *, workers: int = 1, capacity: int = 4096, mode: str = "hybrid",
          anchor: str = "auto", rank=None, roots=None, prepared: Prepared | None = None,
          per_task: bool = False, threads: int = 0) -> OracleReport:
    """Restatement of count_bicliques (engine.py:419-500)."""
    if workers < 1:
        raise ValueError("worker_count must be >= 1")
    if capacity < 1:
        raise ValueError("batch_buffer_capacity must be >= 1")
    if mode not in ("dfs", "hybrid"):
        raise ValueError("mode must be one of ('dfs', 'hybrid')")
    if p < 1 or q < 1:
        raise ValueError("p and q must be >= 1")
    s = prepared if prepared is not None else Prepared(g, p, q, anchor, rank, threads)
    mask = None
    if roots is not None:
        mask = np.zeros(s.n, dtype=np.uint8)
        r = np.asarray(list(roots), dtype=np.int64)
        r = r[(r >= 0) & (r < s.n)]
        mask[r] = 1
    cfg = OrcConfig(p, q, workers, capacity, 0 if mode == "dfs" else 1, -1,
                    None, mask.ctypes.data if mask is not None else None, None, None, None)
    tw = tc = None
    if per_task:
        # emitted is unknown until counted; upper bound = directed pairs (or n for p_eff=1)
        ub = max(int(s.export(X_DIR_OFF)[-1]), s.n, 1)
        tw = np.zeros(ub, dtype=np.int64)
        tc = np.zeros(2 * ub, dtype=np.uint64)
        l1 = np.zeros(4 * ub, dtype=np.int64)
        cfg.task_words = tw.ctypes.data
        cfg.task_count = tc.ctypes.data
        cfg.task_l1 = l1.ctypes.data
    rep = OrcReport()
    if lib().orc_count(s.h, C.byref(cfg), C.byref(rep)) != 0:
        raise ValueError(lib().orc_last_error().decode())
    out = OracleReport(
        count=int(rep.count_lo) | (int(rep.count_hi) << 64), overflow=bool(rep.overflow),
        anchor_layer="UV"[rep.anchor], p_eff=rep.p_eff, q_eff=rep.q_eff,
        batches_executed=rep.batches, tasks_stolen=rep.stolen,
        roots_filtered=rep.roots_filtered, tasks_emitted=rep.emitted,
        tasks_consumed=rep.consumed, intersections=rep.intersections,
        operand_words=rep.operand_words, min_words=rep.min_words,
        prep_time=rep.prep_time, wall_time=rep.wall_time, time_1hop=rep.time_1hop,
        time_2hop=rep.time_2hop, workers=workers)
    if per_task:
        e = rep.emitted
        out.task_words = tw[:e]
        out.task_counts = [int(tc[2 * i]) | (int(tc[2 * i + 1]) << 64) for i in range(e)]
        out.task_l1 = l1[:4 * e].reshape(e, 4)
    return out


def tasks(prepared: Prepared, roots=None) -> np.ndarray:
    """pre_runtime_tasks (engine.py:147-173) for one worker: int64[(emitted, 2)]."""
    order = prepared.export(X_ORDER)
    und = prepared.export(X_UND_SIZE)
    doff = prepared.export(X_DIR_OFF)
    didx = prepared.export(X_DIR_IDX)
    allowed = None if roots is None else set(int(r) for r in roots)
    out = []
    for r in order.tolist():
        if allowed is not None and r not in allowed:
            continue
        if und[r] < prepared.p_eff - 1:
            continue
        if prepared.p_eff == 1:
            out.append((r, -1))
        else:
            out.extend((r, int(w)) for w in didx[doff[r]:doff[r + 1]])
    return np.asarray(out, dtype=np.int64).reshape(-1, 2)


# ---------------------------------------------------------------------------
# pure-Python restatements (tiny graphs)
# ---------------------------------------------------------------------------
PAIR_GUARD = 10**8


def brute_force_count(g, p: int, q: int) -> int:
    """Subset recursion over U, prune on |common| < q (reference oracle.py:31-56)."""
    if p < 1 or q < 1:
        raise ValueError("p and q must be >= 1")
    uo, ui, vo, vi = _csr(g)
    nu, nv = len(uo) - 1, len(vo) - 1
    if comb(nu, p) * comb(nv, q) > PAIR_GUARD:
        raise ValueError("refusing brute force: candidate pairs exceed guard")
    if p > nu or q > nv:
        return 0
    rows = [frozenset(ui[uo[i]:uo[i + 1]].tolist()) for i in range(nu)]
    total = 0

    def walk(start, depth, common):
        nonlocal total
        if depth == p:
            total += comb(len(common), q)
            return
        for u in range(start, nu - (p - depth) + 1):
            c = rows[u] if common is None else common & rows[u]
            if len(c) >= q:
                walk(u + 1, depth + 1, c)

    walk(0, 0, None)
    return total


def closed_form_count(g, p: int, q: int):
    """(1,q), (p,1), (2,2) closed forms (reference oracle.py:59-79)."""
    uo, ui, vo, vi = _csr(g)
    du, dv = np.diff(uo), np.diff(vo)
    if p == 1:
        return sum(comb(int(d), q) for d in du)
    if q == 1:
        return sum(comb(int(d), p) for d in dv)
    if p == 2 and q == 2:
        shared: dict = {}
        for v in range(len(dv)):
            lst = vi[vo[v]:vo[v + 1]].tolist()
            for a, b in combinations(lst, 2):
                shared[a, b] = shared.get((a, b), 0) + 1
        return sum(comb(c, 2) for c in shared.values())
    return None


def border_reorder(g, layer: str, iterations: int):
    """Restates reference ``border_reorder`` (``reorder.py:146-179``) in C
    (``border_oracle.c``): returns (permutation int64[n], one_block_history list)."""
    if iterations < 0:
        raise ValueError("iterations must be >= 0")
    uo, ui, vo, vi = (np.ascontiguousarray(a) for a in _csr(g))
    if layer == "U":
        coff, cidx, roff, ridx = uo, ui, vo, vi
    elif layer == "V":
        coff, cidx, roff, ridx = vo, vi, uo, ui
    else:
        raise ValueError(f"layer must be 'U' or 'V', got {layer!r}")
    coff = np.ascontiguousarray(coff, np.int64)
    roff = np.ascontiguousarray(roff, np.int64)
    cidx = np.ascontiguousarray(cidx, np.int32)
    ridx = np.ascontiguousarray(ridx, np.int32)
    n, m = len(coff) - 1, len(roff) - 1
    perm = np.empty(max(n, 1), np.int64)
    hist = np.empty(iterations + 1, np.int64)
    nh = lib().orc_border(coff.ctypes.data, cidx.ctypes.data, n, roff.ctypes.data,
                          ridx.ctypes.data, m, iterations, perm.ctypes.data, hist.ctypes.data)
    if nh < 0:
        raise MemoryError("orc_border: allocation failed")
    return perm[:n].copy(), hist[:nh].tolist()
