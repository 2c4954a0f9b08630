"""ctypes binding of ``libbicount_b200.so`` (declared in ``include/bicount_b200.h``).

No CPU fallback: if the library or a CUDA device is missing, ``load()``
raises ``RuntimeError`` — the product path fails loudly.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# BC_LIB selects a development build (e.g. the phase-profiling one); default in-tree .so
LIB_PATH = os.environ.get("BC_LIB") or os.path.join(HERE, "libbicount_b200.so")

BC_OK, BC_EINVAL, BC_ECUDA, BC_ENCCL, BC_EOOM, BC_EOVERFLOW, BC_EASSERT = 0, -1, -2, -3, -4, -5, -6
ABI_VERSION = 3
BC_FLAG_TASK_COUNTS, BC_FLAG_INSTRUMENT, BC_FLAG_NO_SPLIT = 1, 2, 4
BC_FLAG_L1_SCATTER, BC_FLAG_L1_PROBE, BC_FLAG_ROWR_SCATTER, BC_FLAG_ROWR_PROBE = 8, 16, 32, 64
BC_FLAG_TASK_SHARD, BC_FLAG_TRACK_TASKS, BC_FLAG_CHECK_NESTING = 128, 256, 512
BC_FLAG_FULL_ROWS, BC_FLAG_FORCE_TRIAGE = 1024, 2048

(BC_X_UND_SIZE, BC_X_RANK, BC_X_ORDER, BC_X_DIR_OFF, BC_X_DIR_IDX, BC_X_HADJ_OFF,
 BC_X_HADJ_IDX, BC_X_HADJ_VAL, BC_X_HDIR_OFF, BC_X_HDIR_IDX, BC_X_HDIR_VAL, BC_X_TASKS,
 BC_X_META, BC_X_SLICE_LENS, BC_X_SLICE_IDS) = range(15)

# every symbol include/bicount_b200.h declares (checked by tests/test_abi.py)
EXPORTED = ("bc_abi_version", "bc_last_error", "bc_device_count", "bc_count", "bc_graph_create",
            "bc_graph_create_device", "bc_graph_count", "bc_graph_enumerate", "bc_graph_destroy", "bc_prepare", "bc_export_len", "bc_export",
            "bc_structs_destroy", "bc_shutdown", "bc_debug_phase_cycles", "bc_graph_border",
            "bc_last_launch_count", "bc_graph_twohop_slice", "bc_graph_count_upper",
            "bc_export_device", "bc_assemble_upper")


class BcConfig(C.Structure):
    _fields_ = [("batch_words", C.c_int32), ("mode", C.c_int32), ("anchor", C.c_int32),
                ("order_mode", C.c_int32), ("device", C.c_int32), ("shard_index", C.c_int32),
                ("shard_count", C.c_int32), ("flags", C.c_int32),
                ("rank_override", C.c_void_p), ("n_rank", C.c_int64),
                ("roots", C.c_void_p), ("n_roots", C.c_int64),
                ("task_counts", C.c_void_p), ("task_counts_cap", C.c_int64),
                ("task_claims", C.c_void_p), ("task_claims_cap", C.c_int64)]


class BcReport(C.Structure):
    _fields_ = [("count_lo", C.c_uint64), ("count_hi", C.c_uint64), ("overflow", C.c_int32),
                ("anchor", C.c_int32), ("p_eff", C.c_int32), ("q_eff", C.c_int32),
                ("tasks_emitted", C.c_int64), ("tasks_consumed", C.c_int64),
                ("tasks_stolen", C.c_int64), ("roots_filtered", C.c_int64),
                ("batches_executed", C.c_int64), ("tasks_alive", C.c_int64),
                ("tasks_split", C.c_int64), ("und_pairs", C.c_int64), ("dir2_pairs", C.c_int64),
                ("adj_words", C.c_int64), ("dir2_words", C.c_int64),
                ("max_slice_words", C.c_int64), ("intersections", C.c_int64),
                ("operand_words", C.c_int64), ("min_words", C.c_int64),
                ("kernel_launches", C.c_int64), ("h2d_bytes", C.c_int64),
                ("d2h_bytes", C.c_int64), ("time_h2d", C.c_double),
                ("time_prep", C.c_double), ("time_level1", C.c_double),
                ("time_enum", C.c_double), ("time_total", C.c_double),
                ("level1_operand_words", C.c_int64), ("nesting_checked", C.c_int64),
                ("level1_entries", C.c_int64)]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["count"] = int(self.count_lo) | (int(self.count_hi) << 64)
        return d


_lib = None


def _declare(L):
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    L.bc_abi_version.restype = C.c_int
    L.bc_abi_version.argtypes = []
    L.bc_last_error.restype = C.c_char_p
    L.bc_last_error.argtypes = []
    L.bc_device_count.restype = C.c_int
    L.bc_device_count.argtypes = []
    L.bc_count.restype = C.c_int
    L.bc_count.argtypes = [vp, vp, i64, vp, vp, i64, i32, i32, C.POINTER(BcConfig),
                           C.POINTER(BcReport)]
    L.bc_graph_create.restype = C.c_int
    L.bc_graph_create.argtypes = [vp, vp, i64, vp, vp, i64, i32, C.POINTER(C.c_void_p)]
    if hasattr(L, "bc_graph_create_device"):  # (absent from development A/B builds of older trees)
        L.bc_graph_create_device.restype = C.c_int
        L.bc_graph_create_device.argtypes = [vp, vp, i64, vp, vp, i64, i32, C.POINTER(C.c_void_p)]
    L.bc_graph_count.restype = C.c_int
    L.bc_graph_count.argtypes = [vp, i32, i32, C.POINTER(BcConfig), C.POINTER(BcReport)]
    if hasattr(L, "bc_graph_enumerate"):
        L.bc_graph_enumerate.restype = C.c_int
        L.bc_graph_enumerate.argtypes = [vp, i32, i32, C.POINTER(BcConfig), vp, i64,
                                         C.POINTER(C.c_int64), C.POINTER(BcReport)]
    if hasattr(L, "bc_graph_twohop_slice"):
        L.bc_graph_twohop_slice.restype = C.c_int
        L.bc_graph_twohop_slice.argtypes = [vp, i32, i32, C.POINTER(BcConfig), i32, i32,
                                            C.POINTER(C.c_void_p)]
        L.bc_graph_count_upper.restype = C.c_int
        L.bc_graph_count_upper.argtypes = [vp, i32, i32, C.POINTER(BcConfig), vp, vp, i64,
                                           C.POINTER(BcReport)]
        L.bc_export_device.restype = C.c_int
        L.bc_export_device.argtypes = [vp, i32, vp]
        L.bc_assemble_upper.restype = C.c_int
        L.bc_assemble_upper.argtypes = [i32, i32, i64, vp, vp, i64, vp, vp, i64,
                                        C.POINTER(C.c_int64)]
    if hasattr(L, "bc_graph_border"):
        L.bc_graph_border.restype = C.c_int
        L.bc_graph_border.argtypes = [vp, i32, i64, vp, vp, C.POINTER(C.c_int64)]
        L.bc_last_launch_count.restype = C.c_int64
        L.bc_last_launch_count.argtypes = []
    L.bc_graph_destroy.restype = None
    L.bc_graph_destroy.argtypes = [vp]
    L.bc_prepare.restype = C.c_int
    L.bc_prepare.argtypes = [vp, i32, i32, C.POINTER(BcConfig), C.POINTER(C.c_void_p)]
    L.bc_export_len.restype = C.c_int64
    L.bc_export_len.argtypes = [vp, i32]
    L.bc_export.restype = C.c_int
    L.bc_export.argtypes = [vp, i32, vp]
    L.bc_structs_destroy.restype = None
    L.bc_structs_destroy.argtypes = [vp]
    L.bc_shutdown.restype = None
    L.bc_shutdown.argtypes = []
    L.bc_debug_phase_cycles.restype = C.c_int
    L.bc_debug_phase_cycles.argtypes = [vp, i32]


def open_library():
    """dlopen the library without touching a GPU (symbol checks on CPU hosts)."""
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python __graft_entry__.py build` "
                           "(or paper_2403_07858_b200/build.py); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    _declare(L)
    return L


def load():
    """The library, checked to have a CUDA device behind it."""
    global _lib
    if _lib is None:
        L = open_library()
        if L.bc_abi_version() != ABI_VERSION:
            raise RuntimeError("libbicount_b200.so ABI version mismatch")
        if L.bc_device_count() < 1:
            raise RuntimeError("no CUDA device visible: the B200 path has no CPU fallback")
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == BC_OK:
        return
    msg = (_lib or open_library()).bc_last_error().decode(errors="replace")
    if rc == BC_EINVAL:
        raise ValueError(msg)
    if rc == BC_EASSERT:  # check_nesting (the reference's assert, engine.py:365-366)
        raise AssertionError(msg)
    raise RuntimeError(f"bicount_b200 error {rc}: {msg}")
