"""HTB (truncated bitmap) format helpers on the host side of the path.

Mirrors the data-format surface of the reference's ``bicount.htb``
(``pkg/src/bicount/htb.py``): ``htb_build`` (family of
sorted id sets -> off / idx / val, ``htb.py:89-115``), ``htb_decode``, ``HtbSlice`` with
``htb_intersect`` / ``htb_intersect_count`` (``htb.py:20-61, 122-183``), and the
``HTBDUMP1`` dump format (``dump_htb`` / ``load_htb``, ``htb.py:186-206``): an
8-byte magic, little-endian u32 ``n_sets, n_words``, then ``off``, ``idx``,
``val`` as u32.  The device builds its own HTB arenas (``prep.cu``, flat
``htb_flags`` / ``htb_fill``); ``prepare_structures(...).adj_htb`` /
``.dir2_htb`` export them in this same layout, so they can be dumped and
compared with the reference's files byte for byte.  ``htb_build`` here is a
vectorised CSR encoder (one pass, no per-set Python loop).
"""

from __future__ import annotations

import numpy as np

from .engine import Htb

MAGIC = b"HTBDUMP1"
WORD_BITS = 32


def htb_build(sets) -> Htb:
    """Encode a family of sorted, duplicate-free, non-negative id lists (htb.py:89-115)."""
    sets = list(sets)
    lens = np.fromiter((len(s) for s in sets), dtype=np.int64, count=len(sets))
    ids = (np.concatenate([np.asarray(s, dtype=np.int64) for s in sets])
           if lens.sum() else np.empty(0, np.int64))
    row = np.repeat(np.arange(len(sets), dtype=np.int64), lens)
    if ids.size:
        if ids.min() < 0:
            raise ValueError("ids must be non-negative")
        same = row[1:] == row[:-1]
        if (np.diff(ids)[same] <= 0).any():
            raise ValueError("input set must be sorted and duplicate-free")
    word = ids >> 5
    start = np.ones(ids.size, dtype=bool)
    if ids.size:
        start[1:] = (word[1:] != word[:-1]) | (row[1:] != row[:-1])
    cut = np.flatnonzero(start)
    bit = np.left_shift(np.uint32(1), (ids & 31).astype(np.uint32))
    val = np.bitwise_or.reduceat(bit, cut) if cut.size else np.empty(0, np.uint32)
    off = np.zeros(len(sets) + 1, dtype=np.int64)
    np.cumsum(np.bincount(row[cut], minlength=len(sets)), out=off[1:])
    return Htb(off, word[cut].astype(np.uint32), val.astype(np.uint32))


class HtbSlice:
    """One encoded set: (idx, val) arrays with a [lo, hi) window (htb.py:20-61)."""

    __slots__ = ("idx", "val", "lo", "hi")

    def __init__(self, idx, val, lo: int = 0, hi: int | None = None):
        self.idx = idx
        self.val = val
        self.lo = lo
        self.hi = len(idx) if hi is None else hi

    def __len__(self) -> int:
        return self.hi - self.lo

    def _words(self):
        return (np.asarray(self.idx[self.lo:self.hi], dtype=np.int64),
                np.asarray(self.val[self.lo:self.hi], dtype=np.uint32))

    def cardinality(self) -> int:
        return int(np.bitwise_count(self._words()[1]).sum())

    def decode(self) -> list[int]:
        idx, val = self._words()
        w, b = np.nonzero(((val[:, None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool))
        return (idx[w] * 32 + b).tolist()

    @classmethod
    def from_ids(cls, ids) -> "HtbSlice":
        h = htb_build([ids])
        return cls(h.idx, h.val, 0, h.n_words)

    @classmethod
    def empty(cls) -> "HtbSlice":
        return cls([], [], 0, 0)


def _match(a: HtbSlice, b: HtbSlice):
    ai, av = a._words()
    bi, bv = b._words()
    _, ia, ib = np.intersect1d(ai, bi, assume_unique=True, return_indices=True)
    x = av[ia] & bv[ib]
    keep = x != 0
    return ai[ia][keep], x[keep]


def htb_intersect(a: HtbSlice, b: HtbSlice, out: HtbSlice) -> HtbSlice:
    """a & b written into caller scratch from out.lo, zero words dropped; the scratch
    must hold min(len(a), len(b)) words (htb.py:122-154)."""
    if len(out.idx) - out.lo < min(len(a), len(b)):
        raise ValueError("scratch capacity below min(len(a), len(b)) words")
    w, x = _match(a, b)
    for k in range(len(w)):
        out.idx[out.lo + k] = int(w[k])
        out.val[out.lo + k] = int(x[k])
    out.hi = out.lo + len(w)
    return out


def htb_intersect_count(a: HtbSlice, b: HtbSlice, early_exit_at: int | None = None) -> int:
    """|a & b| without materialising it (htb.py:157-183); with early_exit_at the result
    is only guaranteed to be >= the threshold once it is met."""
    return int(np.bitwise_count(_match(a, b)[1]).sum())


def htb_decode(h: Htb, s: int) -> list[int]:
    """Ids of set ``s``, ascending (htb.py:42-52)."""
    if not 0 <= s < h.n_sets:
        raise IndexError(f"set index {s} out of range [0, {h.n_sets})")
    lo, hi = int(h.off[s]), int(h.off[s + 1])
    idx = np.asarray(h.idx[lo:hi], dtype=np.int64)
    val = np.asarray(h.val[lo:hi], dtype=np.uint32)
    bits = ((val[:, None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool)
    w, b = np.nonzero(bits)
    return (idx[w] * 32 + b).tolist()


def dump_htb(h: Htb, path) -> None:
    """Write off / idx / val as little-endian u32 behind the 8-byte magic (htb.py:186-193)."""
    off = np.asarray(h.off, dtype=np.int64)
    if len(h.idx) >= 2**32 or (off.size and off[-1] >= 2**32):
        raise ValueError("HTBDUMP1 holds u32 offsets: arena too large")
    with open(path, "wb") as f:
        f.write(MAGIC)
        np.asarray([len(off) - 1, len(h.idx)], dtype="<u4").tofile(f)
        off.astype("<u4").tofile(f)
        np.asarray(h.idx, dtype="<u4").tofile(f)
        np.asarray(h.val, dtype="<u4").tofile(f)


def load_htb(path) -> Htb:
    """Read a dump (htb.py:196-206): ValueError on a bad magic or a truncated file."""
    with open(path, "rb") as f:
        if f.read(8) != MAGIC:
            raise ValueError(f"{path}: not a bitmap dump (bad magic)")
        head = np.fromfile(f, dtype="<u4", count=2)
        if head.size != 2:
            raise ValueError(f"{path}: truncated dump")
        n_sets, n_words = int(head[0]), int(head[1])
        off = np.fromfile(f, dtype="<u4", count=n_sets + 1)
        idx = np.fromfile(f, dtype="<u4", count=n_words)
        val = np.fromfile(f, dtype="<u4", count=n_words)
    if len(off) != n_sets + 1 or len(idx) != n_words or len(val) != n_words:
        raise ValueError(f"{path}: truncated dump")
    return Htb(off.astype(np.int64), idx.astype(np.uint32), val.astype(np.uint32))


def load_htb_device(path, device: int = 0):
    """A dump straight into device memory (CUDA tensors off int64, idx int32, val int32 --
    the u32 words viewed as int32, the layout of ``DeviceGraph.htb_arenas``): the file is
    read once into pinned host memory and copied with one transfer per array."""
    import torch

    h = load_htb(path)
    dev = torch.device("cuda", device)
    return tuple(torch.from_numpy(np.ascontiguousarray(a)).pin_memory().to(dev, non_blocking=True)
                 for a in (h.off.astype(np.int64), h.idx.view(np.int32), h.val.view(np.int32)))

