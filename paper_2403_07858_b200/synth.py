"""Seeded synthetic inputs: the five BASELINE.json configs and the test corpora.

Recipes follow SURVEY.md Appendix B (RNG call sequences reproduced exactly
so the sha256 fingerprints there match). Two generators restate reference
code because the parity graphs are defined by it:

* ``synth_generate`` — power-law 2-hop generator, reference
  ``pkg/src/bicount/cli.py:58-110`` (C4's background graph).
* ``random_bipartite`` / ``corpus300`` / ``recon_graph`` — reference test
  fixtures ``pkg/tests/helpers.py:7-55``.

All are deterministic per seed (numpy PCG64 ``default_rng``).
"""

from __future__ import annotations

import warnings
from math import comb

import numpy as np

from .graph import BipartiteGraph, csr_from_sorted_keys, from_edges

# cli.py:34-36 synthesis knobs
TARGET_FLOOR = 40
SHARE_BIAS = 0.55
STALL_LIMIT = 24

FINGERPRINTS = {
    "C1": "3ab2e3e23871d9015d46a92a21676aac8a23c3fd7aca34e13902f531c1df9117",
    "C2": "5971ce6f3745cc286c68e95cf0fd0e5ef7244f449019e1dbd5114a696e0b2c14",
    "C3": "7b3cfe96d091cbad4bdce0ceeeb9ef21e0cfb7db002fcc71a016c1e607ae8b2d",
    "C4": "cf71d0fac1cc00b4a5a5749833c6de35811bd50268f90c4637ebdec3903962ed",
}

RECON_U_NEIGHBORS = [[0, 1, 2], [0, 1, 2, 4], [1, 2, 3], [0, 2, 3, 4]]
CORPUS_SEED = 20260822


def recon_graph() -> BipartiteGraph:
    """The 4x5 example graph of the paper's Examples 1-3 (helpers.py:10-24)."""
    eu = [u for u, nb in enumerate(RECON_U_NEIGHBORS) for _ in nb]
    ev = [v for nb in RECON_U_NEIGHBORS for v in nb]
    return from_edges(4, 5, eu, ev)


def random_bipartite(nu: int, nv: int, density: float, seed) -> BipartiteGraph:
    """Dense Bernoulli mask graph (helpers.py:27-31)."""
    rng = np.random.default_rng(seed)
    mask = rng.random((nu, nv)) < density
    eu, ev = np.nonzero(mask)
    return from_edges(nu, nv, eu, ev)


def corpus300() -> list[BipartiteGraph]:
    """300 seeded graphs <= 30+30 vertices, density 0.1-0.5 (helpers.py:37-55)."""
    rng = np.random.default_rng(CORPUS_SEED)
    out = []
    while len(out) < 300:
        nu = int(rng.integers(2, 31))
        nv = int(rng.integers(2, 31))
        if comb(nu, 4) * comb(nv, 4) > 10**8:
            continue
        density = float(rng.uniform(0.1, 0.5))
        out.append(random_bipartite(nu, nv, density, rng.integers(0, 2**31)))
    return out


def synth_generate(u_count: int, v_count: int, alpha: float, seed: int) -> BipartiteGraph:
    """Power-law 2-hop generator (reference cli.py:58-110).

    Each U vertex draws a 2-hop target from a truncated power law and adds
    V neighbours (biased towards popular ones) until the target is met or
    the pick loop stalls. The draw order of ``rng`` is part of the contract.
    """
    if u_count < 1 or v_count < 1:
        raise ValueError("layer sizes must be >= 1")
    if alpha <= 1:
        raise ValueError("power-law exponent must be > 1")
    rng = np.random.default_rng(seed)
    cap = max(1, u_count - 1)
    raw = np.floor(TARGET_FLOOR * (1.0 - rng.random(u_count))
                   ** (-1.0 / (alpha - 1.0))).astype(np.int64)
    if int((raw > cap).sum()):
        warnings.warn(f"{int((raw > cap).sum())} of {u_count} two-hop targets "
                      f"exceed {cap} and were clipped", RuntimeWarning)
    targets = np.minimum(raw, cap).tolist()
    holders: list[list[int]] = [[] for _ in range(v_count)]
    picks: list[int] = []
    eu: list[int] = []
    ev: list[int] = []
    for u in range(u_count):
        goal = targets[u]
        seen: set[int] = set()
        mine: set[int] = set()
        misses = 0
        while len(seen) < goal and misses < STALL_LIMIT and len(mine) < v_count:
            if picks and rng.random() < SHARE_BIAS:
                v = picks[int(rng.integers(len(picks)))]
            else:
                v = int(rng.integers(v_count))
            if v in mine:
                misses += 1
                continue
            had = len(seen)
            mine.add(v)
            seen.update(holders[v])
            holders[v].append(u)
            picks.append(v)
            misses = 0 if len(seen) > had else misses + 1
        for v in sorted(mine):
            eu.append(u)
            ev.append(v)
    return from_edges(u_count, v_count, eu, ev)


def erdos_renyi(nu: int, nv: int, m: int, seed: int) -> BipartiteGraph:
    rng = np.random.default_rng(seed)
    keys = rng.choice(nu * nv, size=m, replace=False)
    return from_edges(nu, nv, keys // nv, keys % nv)


def chung_lu(nu: int, nv: int, m: int, gamma: float, seed: int, over: float) -> BipartiteGraph:
    """Chung-Lu power-law bipartite graph (SURVEY App. B recipe)."""
    rng = np.random.default_rng(seed)

    def w(n):
        x = (np.arange(n) + 1.0) ** (-1.0 / (gamma - 1.0))
        return x / x.sum()

    k = int(m * over)
    eu = rng.choice(nu, k, p=w(nu))
    ev = rng.choice(nv, k, p=w(nv))
    key = np.unique(eu.astype(np.int64) * nv + ev)
    key = rng.permutation(key)[:m]
    return from_edges(nu, nv, key // nv, key % nv)


PLANTED_CORES = [(32, 48, 0.85), (24, 32, 0.9), (20, 24, 0.95)]


def planted_dense(seed_base: int = 7, seed_cores: int = 3) -> BipartiteGraph:
    """C4: S2-shaped synth + 3 planted dense cores."""
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        base = synth_generate(12720, 11100, 2.6, seed_base)
    rng = np.random.default_rng(seed_cores)
    eu = [np.repeat(np.arange(base.u_count, dtype=np.int64), base.u_csr.degrees())]
    ev = [base.u_csr.idx.astype(np.int64)]
    for a, b, dens in PLANTED_CORES:
        cu = rng.choice(12720, a, replace=False)
        cv = rng.choice(11100, b, replace=False)
        mask = rng.random((a, b)) < dens
        i, j = np.nonzero(mask)
        eu.append(cu[i].astype(np.int64))
        ev.append(cv[j].astype(np.int64))
    return from_edges(12720, 11100, np.concatenate(eu), np.concatenate(ev))


def _s64(x: int) -> int:
    """Unsigned 64-bit constant as a signed int64 value (two's complement)."""
    return x - (1 << 64) if x >= 1 << 63 else x


_SM_GAMMA, _SM_M1, _SM_M2 = _s64(0x9E3779B97F4A7C15), _s64(0xBF58476D1CE4E5B9), _s64(0x94D049BB133111EB)


def _lsr(x, s: int):
    """Logical right shift of an int64 torch tensor."""
    return (x >> s) & ((1 << (64 - s)) - 1)


def splitmix64(x):
    """SplitMix64 finaliser on int64 torch tensors (wrapping arithmetic): a
    counter-based hash, so the stream is identical on CPU and GPU and for any
    chunking of the counter range."""
    z = x + _SM_GAMMA
    z = (z ^ _lsr(z, 30)) * _SM_M1
    z = (z ^ _lsr(z, 27)) * _SM_M2
    return z ^ _lsr(z, 31)


def _capped_cdf(n: int, gamma: float, cap: float, m: int, scale_bits: int = 40) -> np.ndarray:
    """Integer cumulative Chung-Lu weights (i+1)^(-1/(gamma-1)), clipped at
    cap/m and renormalised 30 times, in fixed point so the
    inverse-CDF sampling below is exact integer arithmetic on any device."""
    w = (np.arange(n) + 1.0) ** (-1.0 / (gamma - 1.0))
    w /= w.sum()
    lim = cap / m
    for _ in range(30):
        w = np.minimum(w, lim)
        w /= w.sum()
    wi = np.maximum(np.floor(w * float(1 << scale_bits)), 1).astype(np.int64)
    return np.cumsum(wi)


def fr_shaped_csr(nu: int = 44_000, nv: int = 8_956_000, m: int = 100_000_000,
                  gamma_u: float = 2.5, gamma_v: float = 2.5, cap_u: float = 200_000,
                  cap_v: float = 64, seed: int = 5, n_cores: int = 64, core_seed: int = 9,
                  device=None, chunk: int = 1 << 25):
    """C5 built directly as device CSR (both views), FR-shaped:
    a small dense U (44K) against a huge sparse V (8.956M), capped Chung-Lu
    degrees, plus ``n_cores`` copies of C4's three planted core shapes.

    Endpoint draws are SplitMix64(seed-keyed counter) mod the integer weight
    total, inverted by ``searchsorted`` on the integer CDF; edges are the
    distinct keys u*|V|+v of ``m`` draws (so |E| is slightly below m).  All
    arithmetic is integer, so the graph is bit-identical on CPU and GPU; on a
    B200 it takes about a second instead of the numpy recipe's minutes.
    Returns torch tensors (u_off, u_idx, v_off, v_idx) on ``device``.
    """
    import torch

    dev = torch.device(device) if device is not None else torch.device("cpu")
    cdf_u = torch.from_numpy(_capped_cdf(nu, gamma_u, cap_u, m)).to(dev)
    cdf_v = torch.from_numpy(_capped_cdf(nv, gamma_v, cap_v, m)).to(dev)
    tot_u, tot_v = int(cdf_u[-1]), int(cdf_v[-1])
    ku, kv = _s64((seed * 0x632BE59BD9B4E019 + 1) % (1 << 64)), _s64((seed * 0x8CB92BA72F3D8DD7 + 2) % (1 << 64))
    keys = torch.empty(m, dtype=torch.int64, device=dev)
    mask63 = (1 << 63) - 1
    for c0 in range(0, m, chunk):
        c1 = min(m, c0 + chunk)
        ctr = torch.arange(c0, c1, dtype=torch.int64, device=dev)
        ru = (splitmix64(ctr ^ ku) & mask63) % tot_u
        rv = (splitmix64(ctr ^ kv) & mask63) % tot_v
        eu = torch.searchsorted(cdf_u, ru, right=True)
        ev = torch.searchsorted(cdf_v, rv, right=True)
        keys[c0:c1] = eu * nv + ev
        del ctr, ru, rv, eu, ev
    extra = [pu[i] * nv + pv[j] for pu, pv, i, j in planted_cores(nu, nv, n_cores, core_seed)]
    if extra:
        keys = torch.cat([keys, torch.from_numpy(np.concatenate(extra)).to(dev)])
    keys = torch.unique(keys, sorted=True)
    return csr_from_sorted_keys_torch(nu, nv, keys)


def planted_cores(nu: int, nv: int, n_cores: int = 64, core_seed: int = 9):
    """The C5 planted cores: (U ids, V ids, edge rows, edge cols) per core, in
    generation order (``n_cores`` copies of C4's three core shapes)."""
    crng = np.random.default_rng(core_seed)
    out = []
    for _ in range(n_cores):
        for a, b, dens in PLANTED_CORES:
            pu = crng.choice(nu, a, replace=False).astype(np.int64)
            pv = crng.choice(nv, b, replace=False).astype(np.int64)
            i, j = np.nonzero(crng.random((a, b)) < dens)
            out.append((pu, pv, i, j))
    return out


def csr_from_sorted_keys_torch(nu: int, nv: int, key):
    """(u_off, u_idx, v_off, v_idx) torch tensors from strictly increasing keys."""
    import torch

    dev = key.device
    su = key // nv
    sv = key - su * nv
    u_off = torch.zeros(nu + 1, dtype=torch.int64, device=dev)
    u_off[1:] = torch.cumsum(torch.bincount(su, minlength=nu), 0)
    u_idx = sv.to(torch.int32)
    k2 = torch.sort(sv * nu + su).values  # V-major, u ascending inside each row
    del sv
    v_of = k2 // nu
    v_off = torch.zeros(nv + 1, dtype=torch.int64, device=dev)
    v_off[1:] = torch.cumsum(torch.bincount(v_of, minlength=nv), 0)
    v_idx = (k2 - v_of * nu).to(torch.int32)
    return u_off, u_idx, v_off, v_idx


def _gen_device() -> str:
    import torch

    return "cuda" if torch.cuda.is_available() else "cpu"


def graph_from_torch_csr(u_off, u_idx, v_off, v_idx) -> BipartiteGraph:
    return BipartiteGraph.from_csr(u_off.cpu().numpy(), u_idx.cpu().numpy(),
                                   v_off.cpu().numpy(), v_idx.cpu().numpy())


# C5H: C5's base graph with many more planted core triples, so the (8,8) search -- not
# the level-1 pass -- dominates and one GPU runs for seconds: the multi-GPU scaling
# workload; calibrated on a B200
C5H_CORES, C5H_CORE_SEED = 8192, 11

DEVICE_CONFIGS = {
    "C5": {},
    "C5H": {"n_cores": C5H_CORES, "core_seed": C5H_CORE_SEED},
}


def build_device_config(name: str, device: str = "cuda"):
    """(u_off, u_idx, v_off, v_idx) torch tensors of a device-generated config."""
    return fr_shaped_csr(device=device, **DEVICE_CONFIGS[name])


CONFIGS = {
    # name: (builder, [(p, q), ...])
    "C1": (lambda: erdos_renyi(2000, 2000, 20000, 1), [(2, 2)]),
    "C2": (lambda: chung_lu(100000, 50000, 1000000, 2.5, 7, 1.15), [(4, 4)]),
    "C3": (lambda: chung_lu(56519, 120867, 440237, 2.5, 11, 1.3), [(3, 6), (6, 3)]),
    "C4": (planted_dense, [(8, 8)]),
    "C5": (lambda: graph_from_torch_csr(*build_device_config("C5", _gen_device())), [(8, 8)]),
    "C5H": (lambda: graph_from_torch_csr(*build_device_config("C5H", _gen_device())), [(8, 8)]),
}


def build_config(name: str) -> BipartiteGraph:
    return CONFIGS[name][0]()
