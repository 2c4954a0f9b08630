"""Vertex reordering before the count: degree presort and Border on the device.

Mirrors the reference's reordering interface (``pkg/src/bicount/reorder.py``,
``graph.py:164-189``, ``cli.py:124-145``) for the caller side of the hot path
(SURVEY 8(f) rank 2):

* ``border_reorder(g, layer, iterations)`` -> ``ReorderResult`` — the greedy
  1-block reduction (``reorder.py:146-179``) run by ``csrc/border.cu`` through
  ``bc_graph_border``; permutation and history are bit-identical to the
  reference's (same argmax / partner tie rules).  There is no CPU fallback.
* ``degree_order(g, layer)`` (``reorder.py:137-143``) and ``relabel(g, pu, pv)``
  (``graph.py:169-183``): small host permutations (CSR rebuilt with one sort).
* ``apply_reorder(g, kind, iters, p, q, anchor)`` — the CLI pipeline
  (``cli.py:124-145``): degree presort, then Border on the anchor layer, then on
  the other layer.  Counts are invariant under it (``test_reorder.py:147-154``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from .graph import BipartiteGraph, LAYERS, as_csr, csr_from_sorted_keys


@dataclass
class ReorderResult:
    permutation: np.ndarray      # int64[n]: new position of each old id
    one_block_history: list[int]  # 1-block total before and after every accepted swap


def _check_layer(layer: str) -> None:
    if layer not in LAYERS:
        raise ValueError(f"layer must be one of {LAYERS}, got {layer!r}")


def degree_order(g, layer: str) -> np.ndarray:
    """Permutation placing high-degree vertices first, ties by id (reorder.py:137-143)."""
    _check_layer(layer)
    u, v = as_csr(g)
    deg = (u if layer == "U" else v).degrees()
    order = np.lexsort((np.arange(len(deg)), -deg))
    perm = np.empty(len(deg), dtype=np.int64)
    perm[order] = np.arange(len(deg))
    return perm


def _check_permutation(perm: np.ndarray, n: int, name: str) -> None:
    if len(perm) != n or not np.array_equal(np.sort(perm), np.arange(n)):
        raise ValueError(f"{name} is not a bijection on [0, {n})")


def relabel(g, perm_u, perm_v) -> BipartiteGraph:
    """Rename vertices (new id of u is perm_u[u]); rows re-sorted (graph.py:169-183)."""
    u, v = as_csr(g)
    pu = np.asarray(perm_u, dtype=np.int64)
    pv = np.asarray(perm_v, dtype=np.int64)
    _check_permutation(pu, u.n, "perm_u")
    _check_permutation(pv, v.n, "perm_v")
    src = np.repeat(np.arange(u.n, dtype=np.int64), u.degrees())
    key = np.sort(pu[src] * np.int64(max(v.n, 1)) + pv[u.idx.astype(np.int64)])
    out = csr_from_sorted_keys(u.n, v.n, key)
    for name, perm in (("u_orig", pu), ("v_orig", pv)):
        orig = getattr(g, name, None)
        if orig is not None:
            o = np.empty_like(orig)
            o[perm] = orig
            setattr(out, name, o)
    return out


def border_reorder(g, layer: str, iterations: int, *, device: int = 0) -> ReorderResult:
    """Greedy 1-block reduction by column swaps of ``layer`` (reorder.py:146-179), on
    the GPU.  ``g`` is a graph or a ``DeviceGraph`` already in HBM."""
    from .engine import DeviceGraph

    if iterations < 0:
        raise ValueError("iterations must be >= 0")
    _check_layer(layer)
    own = not isinstance(g, DeviceGraph)
    dg = DeviceGraph(g, device) if own else g
    try:
        n = dg.u_count if layer == "U" else dg.v_count
        perm = np.empty(max(n, 1), dtype=np.int64)
        hist = np.empty(iterations + 1, dtype=np.int64)
        nh = C.c_int64(0)
        L = _abi.load()
        _abi.check(L.bc_graph_border(dg._h, 0 if layer == "U" else 1, int(iterations),
                                     perm.ctypes.data, hist.ctypes.data, C.byref(nh)))
    finally:
        if own:
            dg.close()
    return ReorderResult(permutation=perm[:n].copy(),
                         one_block_history=[int(x) for x in hist[:nh.value]])


def wedge_mass(g, layer: str) -> int:
    """Sum of C(d, 2) over a layer (graph.py:246-249)."""
    u, v = as_csr(g)
    d = (u if layer == "U" else v).degrees().astype(np.int64)
    return int((d * (d - 1) // 2).sum())


def anchor_layer(g, p: int, q: int, force: str | None = None) -> str:
    """select_anchor_layer(...).layer (graph.py:252-269)."""
    if p < 1 or q < 1:
        raise ValueError("p and q must be >= 1")
    if force is not None:
        _check_layer(force)
        return force
    return "U" if wedge_mass(g, "V") <= wedge_mass(g, "U") else "V"


REORDER_KINDS = ("none", "degree", "border")


def apply_reorder(g, kind: str, iters: int, p: int, q: int, anchor: str = "auto",
                  *, device: int = 0):
    """Degree presort, then for ``border`` a device pass per layer, anchor layer first
    (cli.py:124-145).  Returns the relabelled graph (``g`` itself for ``none``)."""
    if kind not in REORDER_KINDS:
        raise ValueError(f"reorder must be one of {REORDER_KINDS}")
    if iters < 0:
        raise ValueError("--border-iters must be >= 0")
    if kind == "none":
        return g
    g = relabel(g, degree_order(g, "U"), degree_order(g, "V"))
    if kind == "degree":
        return g
    first = anchor_layer(g, p, q, None if anchor == "auto" else anchor)
    for layer in (first, "V" if first == "U" else "U"):
        res = border_reorder(g, layer, iters, device=device)
        if layer == "U":
            g = relabel(g, res.permutation, np.arange(g.v_count))
        else:
            g = relabel(g, np.arange(g.u_count), res.permutation)
    return g
