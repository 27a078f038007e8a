"""ctypes binding of libcapt_b200.so (include/capt_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every entry point raises.  Error codes map to the reference's
exceptions: CAPT_EINVAL / CAPT_ERANGE -> ValueError, CAPT_ENOMEM ->
MemoryError, CAPT_ECUDA -> RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcapt_b200.so")
# experiments only: load a variant built with build_ext --out (never rebuilt)
VARIANT = os.environ.get("CAPT_LIB_VARIANT")

CAPT_OK, CAPT_EINVAL, CAPT_ERANGE, CAPT_ECUDA, CAPT_ENOMEM = range(5)
PREFILTER = 0x1
CHECK_RADII = 0x2
STATS = 0x4
INPUT_F64 = 0x8
HOST_IO = 0x10
MODE_DIRECT = 0x100
MODE_BINNED = 0x200
MODE_THREAD = 0x400
K5_FFMA = 0x800
MODE_WARP = 0x1000
MODE_FIELD = 0x2000
SLAB_BORROW = 0x1  # capt_tree_from_slab flag


class CaptTreeInfo(C.Structure):
    _fields_ = [("k", C.c_int32), ("depth", C.c_int32), ("n_leaves", C.c_int64),
                ("n_points", C.c_int64), ("total_stored", C.c_int64),
                ("max_affordance", C.c_int64), ("r_min", C.c_double),
                ("r_max", C.c_double), ("device_bytes", C.c_int64),
                ("device", C.c_int32), ("reserved", C.c_int32), ("n_ties", C.c_int64)]


class CaptFieldInfo(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("n_cand", C.c_int32), ("n_cells", C.c_int64), ("lo", C.c_float * 3),
                ("h", C.c_float), ("box_lo", C.c_float * 3), ("box_hi", C.c_float * 3),
                ("rcap", C.c_float), ("q_step", C.c_float), ("c0", C.c_float * 3),
                ("q_err", C.c_float)]


_lib = None


def lib():
    """Load the extension (building it in-tree first if sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH) or os.environ.get("CAPT_AUTOBUILD", "1") == "1":
        try:
            from . import build_ext
            if not build_ext.up_to_date():
                build_ext.build()
        except Exception as exc:  # noqa: BLE001 - surface the real cause below
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"libcapt_b200.so is not built and building failed: {exc}")
    L = C.CDLL(os.path.join(HERE, VARIANT) if VARIANT else LIB_PATH)
    if VARIANT:  # an experiment build may predate an entry point: bind what it has
        class _Tolerant:
            def __init__(self, lib):
                object.__setattr__(self, "_l", lib)

            def __getattr__(self, name):
                try:
                    return getattr(self._l, name)
                except AttributeError:
                    return C.CFUNCTYPE(C.c_int)(lambda *a: CAPT_EINVAL)

            def __setattr__(self, name, value):
                setattr(self._l, name, value)
        L = _Tolerant(L)
    vp, i64, i32, u32, dbl = C.c_void_p, C.c_int64, C.c_int, C.c_uint32, C.c_double
    L.capt_last_error.restype = C.c_char_p
    L.capt_version.restype = C.c_int
    L.capt_tree_create.argtypes = [i32, i32, i64, i64, dbl, dbl, vp, vp, vp, vp, vp,
                                   C.POINTER(vp)]
    L.capt_tree_build.argtypes = [i32, i32, vp, i64, dbl, dbl, i32, u32, vp, C.POINTER(vp)]
    L.capt_tree_info_get.argtypes = [vp, C.POINTER(CaptTreeInfo)]
    L.capt_tree_export.argtypes = [vp, vp, vp, vp, vp, vp]
    L.capt_tree_destroy.argtypes = [vp]
    L.capt_tree_destroy.restype = None
    L.capt_tree_slab.argtypes = [vp, C.POINTER(vp), C.POINTER(i64)]
    L.capt_tree_from_slab.argtypes = [i32, vp, i64, u32, vp, C.POINTER(vp)]
    L.capt_query.argtypes = [vp, vp, vp, i64, i32, vp, u32, vp, vp, vp, vp]
    L.capt_leaf_indices.argtypes = [vp, vp, i64, u32, vp, vp]
    L.capt_filter_cloud.argtypes = [i32, i32, vp, i64, dbl, i32, vp, dbl, u32, vp, vp, vp]
    L.capt_measure_fp32_peak.argtypes = [i32, C.POINTER(dbl)]
    L.capt_tc_selftest.argtypes = [i32, C.POINTER(dbl)]
    L.capt_nn_distances.argtypes = [i32, i32, vp, i64, u32, vp, vp]
    L.capt_tree_field.argtypes = [vp, C.POINTER(CaptFieldInfo), vp, vp]
    L.capt_stage_timing.argtypes = [i32]
    L.capt_stage_times.argtypes = [C.POINTER(dbl), C.POINTER(i64)]
    L.capt_field_list_counts.argtypes = [vp, C.POINTER(u32)]
    L.capt_tree_field_blocks.argtypes = [vp, vp, vp, vp]
    L.capt_kernel_launches.restype = C.c_int64
    L.capt_kernel_launches.argtypes = []
    for name in ("capt_tree_create", "capt_tree_build", "capt_tree_info_get",
                 "capt_tree_export", "capt_tree_slab", "capt_tree_from_slab", "capt_query",
                 "capt_leaf_indices", "capt_filter_cloud", "capt_measure_fp32_peak",
                 "capt_tc_selftest", "capt_nn_distances", "capt_tree_field",
                 "capt_stage_timing", "capt_stage_times", "capt_field_list_counts",
                 "capt_tree_field_blocks"):
        getattr(L, name).restype = C.c_int
    _lib = L
    return L


def last_error() -> str:
    msg = lib().capt_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == CAPT_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc in (CAPT_EINVAL, CAPT_ERANGE):
        raise ValueError(msg)
    if rc == CAPT_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def ptr(a) -> int | None:
    """Raw address of a numpy array or torch tensor (None for None)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def default_device() -> int:
    env = os.environ.get("CAPT_DEVICE")
    if env is not None:
        return int(env)
    import sys
    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_available():
        return torch.cuda.current_device()
    local = os.environ.get("LOCAL_RANK")
    return int(local) if local is not None else 0


EXPORTED_SYMBOLS = (
    "capt_last_error", "capt_version", "capt_tree_create", "capt_tree_build",
    "capt_tree_info_get", "capt_tree_export", "capt_tree_destroy", "capt_tree_slab",
    "capt_tree_from_slab", "capt_query", "capt_leaf_indices", "capt_filter_cloud",
    "capt_measure_fp32_peak", "capt_kernel_launches", "capt_tc_selftest", "capt_nn_distances",
    "capt_tree_field", "capt_stage_timing", "capt_stage_times", "capt_field_list_counts",
    "capt_tree_field_blocks",
)
