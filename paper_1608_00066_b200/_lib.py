"""ctypes prototypes of libpbvd.so (include/pbvd.h).  Argument marshalling
only: every step of the decode runs in the library's CUDA kernels.  There is
no CPU fallback -- if the library is missing this module raises."""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libpbvd.so"

PBVD_OK = 0
PBVD_TERMINATED = 1
PBVD_ALLOW_CATASTROPHIC = 2
PBVD_START_ZERO = 4

EXPORTS = (
    "pbvd_create", "pbvd_destroy", "pbvd_llr_count", "pbvd_stage_count", "pbvd_block_count",
    "pbvd_decode", "pbvd_decode_blocks", "pbvd_decode_host", "pbvd_set_lanes", "pbvd_get_lanes",
    "pbvd_set_fused", "pbvd_get_fused",
    "pbvd_set_workspace_limit", "pbvd_set_profiling", "pbvd_kernel_times", "pbvd_get_info",
    "pbvd_supported", "pbvd_strerror", "pbvd_last_error", "pbvd_probe_acs_peak",
    "pbvd_probe_acs_balanced", "pbvd_jit_prebuild",
    "pbvd_stream_open", "pbvd_stream_push", "pbvd_stream_finish", "pbvd_stream_close",
    "pbvd_decode_blocks_mirrored", "pbvd_ipc_export", "pbvd_ipc_open", "pbvd_ipc_close",
)
PBVD_IPC_HANDLE_BYTES = 64


class PbvdInfo(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int), ("R", ctypes.c_int), ("N", ctypes.c_int),
                ("lanes", ctypes.c_int), ("D", ctypes.c_int), ("L", ctypes.c_int),
                ("P", ctypes.c_int), ("dec_bytes_per_block", ctypes.c_int64),
                ("span", ctypes.c_int64), ("workspace_bytes", ctypes.c_size_t),
                ("jit", ctypes.c_int), ("host_lanes", ctypes.c_int)]


_lib = None


def load(path: os.PathLike | None = None):
    """Load libpbvd.so (build it first with paper_1608_00066_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    # PBVD_LIB: an alternative build of the same library (A/B experiments,
    # tools/ only); the default is the in-tree libpbvd.so
    p = Path(path) if path else Path(os.environ.get("PBVD_LIB", str(LIB_PATH)))
    if not p.exists():
        raise ImportError(f"{p} not found: build the CUDA library first "
                          "(python -m paper_1608_00066_b200.build); there is no CPU fallback")
    L = ctypes.CDLL(str(p))
    i32, i64, u32 = ctypes.c_int, ctypes.c_int64, ctypes.c_uint
    vp, cp = ctypes.c_void_p, ctypes.c_char_p
    h = ctypes.c_void_p
    L.pbvd_create.argtypes = [ctypes.POINTER(h), i32, i32, ctypes.POINTER(ctypes.c_uint32), i32,
                              ctypes.POINTER(ctypes.c_uint8), i32, i32, i32, u32, i32]
    L.pbvd_create.restype = i32
    L.pbvd_destroy.argtypes = [h]
    L.pbvd_destroy.restype = None
    for fn in ("pbvd_llr_count", "pbvd_stage_count", "pbvd_block_count"):
        getattr(L, fn).argtypes = [h, i64]
        getattr(L, fn).restype = i64
    L.pbvd_decode.argtypes = [h, vp, i64, vp, i64, vp]
    L.pbvd_decode.restype = i32
    L.pbvd_decode_blocks.argtypes = [h, vp, i64, i64, i64, i64, i64, vp, vp]
    L.pbvd_decode_blocks.restype = i32
    L.pbvd_decode_blocks_mirrored.argtypes = [h, vp, i64, i64, i64, i64, i64, vp,
                                              ctypes.POINTER(ctypes.c_void_p), i32, vp]
    L.pbvd_decode_blocks_mirrored.restype = i32
    L.pbvd_decode_host.argtypes = [h, vp, i64, i64, i64, i64, i64, vp, i32]
    L.pbvd_decode_host.restype = i32
    L.pbvd_set_lanes.argtypes = [h, i32]
    L.pbvd_set_lanes.restype = i32
    L.pbvd_get_lanes.argtypes = [h]
    L.pbvd_get_lanes.restype = i32
    L.pbvd_set_fused.argtypes = [h, i32]
    L.pbvd_set_fused.restype = i32
    L.pbvd_get_fused.argtypes = [h]
    L.pbvd_get_fused.restype = i32
    L.pbvd_set_workspace_limit.argtypes = [h, ctypes.c_size_t]
    L.pbvd_set_workspace_limit.restype = i32
    L.pbvd_set_profiling.argtypes = [h, i32]
    L.pbvd_set_profiling.restype = i32
    L.pbvd_kernel_times.argtypes = [h, ctypes.POINTER(ctypes.c_float),
                                    ctypes.POINTER(ctypes.c_float), ctypes.POINTER(i32)]
    L.pbvd_kernel_times.restype = i32
    L.pbvd_get_info.argtypes = [h, ctypes.POINTER(PbvdInfo)]
    L.pbvd_get_info.restype = i32
    L.pbvd_probe_acs_peak.argtypes = [i32, ctypes.POINTER(ctypes.c_double),
                                      ctypes.POINTER(ctypes.c_double)]
    L.pbvd_probe_acs_peak.restype = i32
    L.pbvd_probe_acs_balanced.argtypes = [i32, ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_double)]
    L.pbvd_probe_acs_balanced.restype = i32
    L.pbvd_jit_prebuild.argtypes = [i32, i32, ctypes.POINTER(ctypes.c_uint32), i32, cp,
                                     ctypes.c_size_t]
    L.pbvd_jit_prebuild.restype = i32
    L.pbvd_stream_open.argtypes = [h, ctypes.POINTER(h)]
    L.pbvd_stream_open.restype = i32
    L.pbvd_stream_push.argtypes = [h, vp, i64, vp, i64, ctypes.POINTER(i64), vp]
    L.pbvd_stream_push.restype = i32
    L.pbvd_stream_finish.argtypes = [h, vp, i64, ctypes.POINTER(i64), vp]
    L.pbvd_stream_finish.restype = i32
    L.pbvd_stream_close.argtypes = [h]
    L.pbvd_stream_close.restype = None
    L.pbvd_supported.argtypes = []
    L.pbvd_supported.restype = cp
    L.pbvd_strerror.argtypes = [i32]
    L.pbvd_strerror.restype = cp
    L.pbvd_last_error.argtypes = [h]
    L.pbvd_last_error.restype = cp
    L.pbvd_ipc_export.argtypes = [vp, vp, ctypes.POINTER(i64)]
    L.pbvd_ipc_export.restype = i32
    L.pbvd_ipc_open.argtypes = [vp, i64, i32, ctypes.POINTER(vp)]
    L.pbvd_ipc_open.restype = i32
    L.pbvd_ipc_close.argtypes = [vp, i64, i32]
    L.pbvd_ipc_close.restype = i32
    _lib = L
    return L
