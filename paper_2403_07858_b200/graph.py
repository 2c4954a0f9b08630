"""Bipartite graph container for the B200 path, CSR-native.

Mirrors the reference's ``BipartiteGraph`` (``pkg/src/bicount/graph.py:15-49``):
both adjacency views, each list sorted and duplicate-free, ``u_adj`` /
``v_adj`` exposed as lists of int32 arrays so reference callers keep working.
Internally each view is one CSR pair (``int64 off[n+1]``, ``int32 idx[E]``),
which is exactly what the C-ABI (``include/bicount_b200.h``) consumes — no
per-vertex Python objects on the hot path, which matters at the FR-shaped
config (9 M vertices).

``as_csr`` accepts either this class or any object with ``u_adj``/``v_adj``
lists (e.g. the reference's own ``BipartiteGraph``) and flattens it.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

LAYERS = ("U", "V")


@dataclass
class CsrView:
    off: np.ndarray  # int64[n+1]
    idx: np.ndarray  # int32[E]

    @property
    def n(self) -> int:
        return len(self.off) - 1

    def row(self, i: int) -> np.ndarray:
        return self.idx[self.off[i]:self.off[i + 1]]

    def degrees(self) -> np.ndarray:
        return np.diff(self.off)


class BipartiteGraph:
    """Both adjacency views of a bipartite graph as CSR.

    Construct with ``BipartiteGraph.from_csr`` / ``from_edges`` or from
    reference-style lists ``BipartiteGraph(u_adj, v_adj)``.
    """

    def __init__(self, u_adj=None, v_adj=None, u_orig=None, v_orig=None, *,
                 u_csr: CsrView | None = None, v_csr: CsrView | None = None):
        if u_csr is None:
            u_csr = _lists_to_csr(u_adj)
            v_csr = _lists_to_csr(v_adj)
        self.u_csr = u_csr
        self.v_csr = v_csr
        self.u_orig = u_orig
        self.v_orig = v_orig
        self._u_lists = None
        self._v_lists = None

    @classmethod
    def from_csr(cls, u_off, u_idx, v_off, v_idx) -> "BipartiteGraph":
        return cls(u_csr=CsrView(np.ascontiguousarray(u_off, np.int64),
                                 np.ascontiguousarray(u_idx, np.int32)),
                   v_csr=CsrView(np.ascontiguousarray(v_off, np.int64),
                                 np.ascontiguousarray(v_idx, np.int32)))

    # --- reference-compatible surface (graph.py:23-49) ---
    @property
    def u_adj(self) -> list[np.ndarray]:
        if self._u_lists is None:
            self._u_lists = _csr_to_lists(self.u_csr)
        return self._u_lists

    @property
    def v_adj(self) -> list[np.ndarray]:
        if self._v_lists is None:
            self._v_lists = _csr_to_lists(self.v_csr)
        return self._v_lists

    @property
    def u_count(self) -> int:
        return self.u_csr.n

    @property
    def v_count(self) -> int:
        return self.v_csr.n

    @property
    def edge_count(self) -> int:
        return int(self.u_csr.off[-1])

    def adj(self, layer: str) -> list[np.ndarray]:
        _check_layer(layer)
        return self.u_adj if layer == "U" else self.v_adj

    def degrees(self, layer: str) -> np.ndarray:
        _check_layer(layer)
        return (self.u_csr if layer == "U" else self.v_csr).degrees()

    def fingerprint(self) -> str:
        """sha256 of sorted keys u*|V|+v as LE int64."""
        u = np.repeat(np.arange(self.u_count, dtype=np.int64), self.u_csr.degrees())
        key = u * np.int64(self.v_count) + self.u_csr.idx.astype(np.int64)
        return hashlib.sha256(key.astype("<i8").tobytes()).hexdigest()


def _check_layer(layer: str) -> None:
    if layer not in LAYERS:
        raise ValueError(f"layer must be one of {LAYERS}, got {layer!r}")


def _lists_to_csr(lists) -> CsrView:
    lists = list(lists)
    n = len(lists)
    off = np.zeros(n + 1, dtype=np.int64)
    if n:
        np.cumsum([len(a) for a in lists], out=off[1:])
    idx = (np.concatenate([np.asarray(a, dtype=np.int32) for a in lists])
           if n and off[-1] else np.empty(0, dtype=np.int32))
    return CsrView(off, idx.astype(np.int32, copy=False))


def _csr_to_lists(c: CsrView) -> list[np.ndarray]:
    off = c.off
    return [c.idx[off[i]:off[i + 1]] for i in range(c.n)]


def as_csr(g) -> tuple[CsrView, CsrView]:
    """(U view, V view) CSR for this class or any reference-style graph."""
    if isinstance(g, BipartiteGraph):
        return g.u_csr, g.v_csr
    return _lists_to_csr(g.u_adj), _lists_to_csr(g.v_adj)


def from_edges(u_count: int, v_count: int, eu, ev) -> BipartiteGraph:
    """Both views from parallel edge arrays; duplicates collapse, rows sorted.

    Same contract and errors as the reference ``from_edges``
    (``pkg/src/bicount/graph.py:88-108``), built as CSR with one sort.
    """
    eu = np.asarray(eu, dtype=np.int64)
    ev = np.asarray(ev, dtype=np.int64)
    if eu.shape != ev.shape:
        raise ValueError("edge arrays must have equal length")
    if eu.size:
        if eu.min() < 0 or eu.max() >= u_count:
            raise ValueError("u id out of range")
        if ev.min() < 0 or ev.max() >= v_count:
            raise ValueError("v id out of range")
    key = np.unique(eu * np.int64(v_count) + ev)
    return csr_from_sorted_keys(u_count, v_count, key)


def csr_from_sorted_keys(u_count: int, v_count: int, key: np.ndarray) -> BipartiteGraph:
    """Graph from strictly increasing keys u*|V|+v."""
    su = key // v_count
    sv = key - su * v_count
    u_off = np.zeros(u_count + 1, dtype=np.int64)
    np.cumsum(np.bincount(su, minlength=u_count), out=u_off[1:])
    # V view: stable order by v keeps u ascending inside each row
    rev = np.argsort(sv, kind="stable")
    v_off = np.zeros(v_count + 1, dtype=np.int64)
    np.cumsum(np.bincount(sv, minlength=v_count), out=v_off[1:])
    return BipartiteGraph.from_csr(u_off, sv.astype(np.int32), v_off,
                                   su[rev].astype(np.int32))


def transpose(g) -> BipartiteGraph:
    """Swap the two views (reference ``graph.py:160-161``)."""
    u, v = as_csr(g)
    return BipartiteGraph(u_csr=v, v_csr=u)
