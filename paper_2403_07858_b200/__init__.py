"""B200-native (sm_100a) exact (p,q)-biclique counting — the GBC hot path.

Drop-in for the reference ``bicount`` counting entry point
(``pkg/src/bicount/engine.py:419``): ``count_bicliques(g, p, q, cfg)`` returns
a ``CountReport`` whose ``count`` is an exact Python int, computed by the
hand-written CUDA kernels in ``csrc/`` behind the C-ABI in
``include/bicount_b200.h``.  There is no CPU fallback.
"""

from .engine import (
    AnchorChoice,
    CountReport,
    DeviceGraph,
    EngineConfig,
    Htb,
    PriorityOrder,
    SearchStructures,
    TwoHopIndex,
    allreduce_count,
    count_bicliques,
    count_bicliques_distributed,
    merge_limbs,
    prepare_structures,
    split_limbs,
    stats_payload,
    write_stats_json,
)
from .graph import BipartiteGraph, CsrView, as_csr, from_edges, transpose

__version__ = "0.1.0"

__all__ = [
    "AnchorChoice", "BipartiteGraph", "CountReport", "CsrView", "DeviceGraph", "EngineConfig",
    "Htb", "PriorityOrder", "SearchStructures", "TwoHopIndex", "allreduce_count", "as_csr",
    "count_bicliques", "count_bicliques_distributed", "from_edges", "merge_limbs",
    "prepare_structures", "split_limbs", "stats_payload", "transpose", "write_stats_json",
    "__version__",
]
