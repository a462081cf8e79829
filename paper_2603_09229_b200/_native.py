"""ctypes binding of the C ABI (include/flashkmeans.h).

The library is AOT-built into ``paper_2603_09229_b200/_lib/libflashkmeans.so``
(``python -m paper_2603_09229_b200._build``).  There is deliberately no
fallback: if the library is missing or the device is not an sm_100 part, the
operators raise instead of silently computing on the CPU.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FK_LIB_PATH") or os.path.join(_HERE, "_lib", "libflashkmeans.so")

FK_OK, FK_EINVAL, FK_EUNSUPPORTED, FK_ECUDA, FK_EWORKSPACE = range(5)
FK_F32, FK_BF16, FK_F16, FK_F64 = range(4)

_lock = threading.Lock()
_lib = None


class NativeLibraryError(RuntimeError):
    """The sm_100a library is missing, failed to load, or reported a CUDA error."""


def _declare(L):
    P, I64, I32, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
    L.fk_version.restype = ctypes.c_char_p
    L.fk_status_string.restype = ctypes.c_char_p
    L.fk_status_string.argtypes = [ctypes.c_int]
    L.fk_last_cuda_error.restype = ctypes.c_char_p
    L.fk_device_supported.restype = ctypes.c_int
    L.fk_device_supported.argtypes = [ctypes.c_int]
    L.fk_preload.restype = ctypes.c_int
    L.fk_preload.argtypes = []
    L.fk_assign_workspace.restype = SZ
    L.fk_assign_workspace.argtypes = [ctypes.c_int, I64, I64, I64, I64]
    L.fk_assign_bias_rows.restype = I64
    L.fk_assign_bias_rows.argtypes = [I64]
    L.fk_assign_bias.restype = ctypes.c_int
    L.fk_assign_bias.argtypes = [ctypes.c_int, P, I64, I64, I64, P, P]
    L.fk_assign.restype = ctypes.c_int
    L.fk_assign.argtypes = [ctypes.c_int, P, P, P, I64, I64, I64, I64, P, P, P, P, P, SZ, P]
    L.fk_assign_xsplit_bytes.restype = SZ
    L.fk_assign_xsplit_bytes.argtypes = [ctypes.c_int, I64, I64, I64]
    L.fk_assign_xsplit.restype = ctypes.c_int
    L.fk_assign_xsplit.argtypes = [ctypes.c_int, P, I64, I64, I64, P, P]
    L.fk_assign_split_workspace.restype = SZ
    L.fk_assign_split_workspace.argtypes = [ctypes.c_int, I64, I64, I64, I64]
    L.fk_assign_split_fallback_rows.restype = ctypes.c_int
    L.fk_assign_split_fallback_rows.argtypes = [ctypes.c_int, I64, I64, I64, I64, P, P, P]
    L.fk_assign_split.restype = ctypes.c_int
    L.fk_assign_split.argtypes = [ctypes.c_int, P, P, P, I64, I64, I64, I64, I32, P, P, P, P, P, SZ, P]
    L.fk_update_workspace.restype = SZ
    L.fk_update_workspace.argtypes = [ctypes.c_int, I64, I64, I64, I64]
    L.fk_update.restype = ctypes.c_int
    L.fk_update.argtypes = [ctypes.c_int, P, P, I64, I64, I64, I64, I64, I32, P, P, P, P, SZ, P]
    L.fk_update_prehist.restype = ctypes.c_int
    L.fk_update_prehist.argtypes = [ctypes.c_int, P, P, I64, I64, I64, I64, I64, I32, P, P, P, P, SZ, P]
    L.fk_update_hist_slots.restype = ctypes.c_int
    L.fk_update_hist_slots.argtypes = [ctypes.c_int, I64, I64, I64, I64, P, ctypes.POINTER(P),
                                       ctypes.POINTER(P), ctypes.POINTER(I64), ctypes.POINTER(I64),
                                       ctypes.POINTER(I64)]
    L.fk_assign_hist.restype = ctypes.c_int
    L.fk_assign_hist.argtypes = [ctypes.c_int, P, P, P, I64, I64, I64, I64, P, P, P, P, P, SZ, P, P, I64,
                                 I64, P, P]
    L.fk_assign_row_norms.restype = ctypes.c_int
    L.fk_assign_row_norms.argtypes = [ctypes.c_int, P, I64, I64, I64, I64, P, P]
    L.fk_argsort.restype = ctypes.c_int
    L.fk_argsort.argtypes = [P, I64, I64, I64, P, P, P, SZ, P]
    L.fk_normalize.restype = ctypes.c_int
    L.fk_normalize.argtypes = [ctypes.c_int, P, P, P, P, ctypes.c_int, P, P, P, I64, I64, I64, P, P]
    L.fk_objective_partials.restype = ctypes.c_int
    L.fk_objective_partials.argtypes = [ctypes.c_int, P, I64, I64, P, P]
    L.fk_normalize_loop_tail.restype = ctypes.c_int
    L.fk_normalize_loop_tail.argtypes = [ctypes.c_int, P, P, P, P, ctypes.c_int, P, P, P, I64, I64, I64, P,
                                         ctypes.c_int, P, I64, P, P, P, P, P, P, P, P, P]
    L.fk_loop_tail.restype = ctypes.c_int
    L.fk_loop_tail.argtypes = [P, I64, I64, P, P, P, P, P, P, P, P]
    L.fk_row_norms.restype = ctypes.c_int
    L.fk_row_norms.argtypes = [ctypes.c_int, P, I64, I64, P, P]
    L.fk_objective_workspace.restype = SZ
    L.fk_objective_workspace.argtypes = [I64, I64]
    L.fk_objective.restype = ctypes.c_int
    L.fk_objective.argtypes = [ctypes.c_int, P, I64, I64, P, P, SZ, P]
    L.fk_scatter.restype = ctypes.c_int
    L.fk_scatter.argtypes = [ctypes.c_int, P, P, I64, I64, I64, I64, P, P, P]
    L.fk_stats_pack.restype = ctypes.c_int
    L.fk_stats_pack.argtypes = [I32, P, P, P, P, I64, I64, P]
    L.fk_merges_from_counts.restype = ctypes.c_int
    L.fk_merges_from_counts.argtypes = [P, I64, I64, I64, P, I32, P]
    L.fk_farthest_workspace.restype = SZ
    L.fk_farthest_workspace.argtypes = [I64, I64]
    L.fk_farthest.restype = ctypes.c_int
    L.fk_farthest.argtypes = [ctypes.c_int, P, I64, I64, I64, P, P, SZ, P]
    L.fk_kmeanspp_workspace.restype = SZ
    L.fk_kmeanspp_workspace.argtypes = [I64, I64, I64, I64]
    L.fk_kmeanspp.restype = ctypes.c_int
    L.fk_kmeanspp.argtypes = [ctypes.c_int, P, I64, I64, I64, I64, P, P, P, P, P, SZ, P]
    L.fk_kmeanspp_init.restype = ctypes.c_int
    L.fk_kmeanspp_init.argtypes = [P, I64, I64, I64, P, SZ, P]
    L.fk_kmeanspp_sweep.restype = ctypes.c_int
    L.fk_kmeanspp_sweep.argtypes = [ctypes.c_int, P, I64, I64, I64, I64, P, I64, P, I64, I32, P,
                                    I64, P]
    L.fk_kmeanspp_select.restype = ctypes.c_int
    L.fk_kmeanspp_select.argtypes = [P, I64, I64, P, I64, I64, P, P, P, SZ, P]


EXPORTED = (
    "fk_version", "fk_status_string", "fk_last_cuda_error", "fk_device_supported", "fk_preload",
    "fk_assign_workspace", "fk_assign_bias_rows", "fk_assign_bias", "fk_assign", "fk_assign_xsplit_bytes",
    "fk_assign_xsplit", "fk_assign_split_workspace", "fk_assign_split", "fk_assign_split_fallback_rows",
    "fk_update_workspace",
    "fk_update", "fk_update_prehist", "fk_update_hist_slots", "fk_assign_hist", "fk_assign_row_norms", "fk_argsort", "fk_normalize", "fk_row_norms", "fk_objective_workspace", "fk_objective",
    "fk_objective_partials", "fk_loop_tail", "fk_normalize_loop_tail", "fk_scatter",
    "fk_stats_pack", "fk_merges_from_counts", "fk_farthest_workspace", "fk_farthest",
    "fk_kmeanspp_workspace", "fk_kmeanspp",
    "fk_kmeanspp_init", "fk_kmeanspp_sweep", "fk_kmeanspp_select",
)


def lib():
    """Load (once) and return the ctypes handle; raises NativeLibraryError if absent."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise NativeLibraryError(
                        f"{LIB_PATH} is missing: build it with "
                        "`python -m paper_2603_09229_b200._build` (there is no CPU fallback)")
                L = ctypes.CDLL(LIB_PATH)
                _declare(L)
                _lib = L
    return _lib


def check(status: int, what: str) -> None:
    if status == FK_OK:
        return
    L = lib()
    msg = f"{what}: {L.fk_status_string(status).decode()}"
    if status == FK_EINVAL:
        raise ValueError(msg)
    if status == FK_EUNSUPPORTED:
        raise NotImplementedError(msg + " (an sm_100 / B200 device is required)")
    if status == FK_ECUDA:
        raise NativeLibraryError(msg + ": " + L.fk_last_cuda_error().decode())
    raise NativeLibraryError(msg)
