"""ctypes binding of the in-tree C ABI (include/fireiron_b200.h).

The product path is the native library ``_lib/libfireiron_b200.so`` built by
``__graft_entry__.build()``; importing this module fails loudly when it is
missing -- there is no CPU or PyTorch fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FI_LIB_PATH") or os.path.join(_HERE, "_lib", "libfireiron_b200.so")  # override: A/B builds

FI_OK = 0
FI_F32, FI_F16, FI_BF16 = 0, 1, 2
FI_KIND_GENERIC, FI_KIND_TCGEN05 = 0, 1

ERROR_KINDS = [
    "ZeroDim", "ShapeMismatch", "NonDivisible", "NotMatMul", "CNotInGL", "HierarchyViolation",
    "UnitCountMismatch", "UpwardLoad", "InvalidMoveDecomp", "PatternMismatch", "NoExecutableMatch",
    "AmbiguousMatch", "DuplicatePattern", "SwizzleNotBijective", "InvalidRefinement", "UnboundVar",
    "DivisionByZero", "CapacityExceeded", "ReuseBufferUnavailable", "OwnershipViolation",
    "UnsimulatableResidual", "ParseError", "InvalidTree", "IoError",
]
BACKEND_ERRORS = {100: "CudaError", 101: "NvrtcError", 102: "NcclError", 103: "Unsupported",
                  104: "ArgumentError"}


def status_name(code: int) -> str:
    if 1 <= code <= len(ERROR_KINDS):
        return ERROR_KINDS[code - 1]
    return BACKEND_ERRORS.get(code, f"status{code}")


class FiError(RuntimeError):
    """Mirror of anvil::Error (proj/include/anvil/error.hpp:67-76): carries the kind."""

    def __init__(self, code: int, message: str):
        self.code = code
        self.kind = status_name(code)
        super().__init__(f"{self.kind}: {message}")


class TcConfig(C.Structure):
    _fields_ = [("cta_group", C.c_int32), ("tile_n", C.c_int32), ("split_k", C.c_int32),
                ("ab_elem", C.c_int32), ("a_row_major", C.c_int32), ("b_row_major", C.c_int32),
                ("c_row_major", C.c_int32), ("c_elem", C.c_int32), ("group_m", C.c_int32),
                ("max_ctas", C.c_int32)]


class PlanInfo(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64), ("kind", C.c_int32),
                ("is_move", C.c_int32), ("elem_a", C.c_int32), ("elem_b", C.c_int32),
                ("elem_c", C.c_int32), ("a_row_major", C.c_int32), ("b_row_major", C.c_int32),
                ("c_row_major", C.c_int32), ("grid_x", C.c_int64), ("grid_y", C.c_int64),
                ("block_threads", C.c_int64), ("launch_ctas", C.c_int64), ("cluster", C.c_int32),
                ("stages", C.c_int32), ("tmem_cols", C.c_int32), ("cta_group", C.c_int32),
                ("tile_m", C.c_int32), ("tile_n", C.c_int32), ("split_k", C.c_int32),
                ("shared_bytes", C.c_int64), ("flops", C.c_double), ("streamk", C.c_int32),
                ("remainder", C.c_int32), ("entry_name", C.c_char * 128)]


class AsyncCheckOptions(C.Structure):
    _fields_ = [("num_sms", C.c_int32), ("max_active_clusters", C.c_int32), ("streamk", C.c_int32),
                ("remainder", C.c_int32), ("c_tma", C.c_int32), ("ring_drain", C.c_int32),
                ("mutation", C.c_int32), ("pull_d", C.c_int32), ("head", C.c_int32),
                ("gated_chunks", C.c_int32), ("gated_first", C.c_int32)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"native library missing: {LIB_PATH}; run __graft_entry__.build() "
            "(the backend has no CPU fallback)")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
    sigs = {
        "fi_version": ([], C.c_char_p),
        "fi_last_error": ([], C.c_char_p),
        "fi_tc_gemm": ([C.POINTER(TcConfig), vp, vp, vp, i64, i64, i64, i64, i64, i64, vp, vp], C.c_int),
        "fi_convert_f32": ([vp, vp, i64, C.c_int, vp], C.c_int),
        "fi_host_snap_f32": ([vp, vp, i64, C.c_int], C.c_int),
        "fi_ipc_export": ([vp, vp, C.POINTER(i64)], C.c_int),
        "fi_ipc_open": ([vp, i64, C.POINTER(vp)], C.c_int),
        "fi_ipc_close": ([vp, i64], C.c_int),
        "fi_copy_async": ([vp, vp, i64, vp], C.c_int),
    }
    optional = {
        "fi_plan_create": ([C.c_char_p, i64, i64, i64, C.c_int, C.c_uint32, C.POINTER(vp)], C.c_int),
        "fi_plan_launch": ([vp, vp, vp, vp, vp], C.c_int),
        "fi_plan_host_bytes": ([vp, C.POINTER(i64), C.POINTER(i64)], C.c_int),
        "fi_plan_launch_gated": ([vp, vp, vp, vp, vp, vp, C.c_uint32, i64, i32], C.c_int),
        "fi_stream_write_u32": ([vp, C.c_uint32, vp], C.c_int),
        "fi_plan_run_host": ([vp, vp, vp, vp], C.c_int),
        "fi_plan_query": ([vp, C.POINTER(PlanInfo)], C.c_int),
        "fi_plan_source": ([vp, C.c_char_p, i64], i64),
        "fi_plan_destroy": ([vp], None),
        "fi_script_validate": ([C.c_char_p, i64, i64, i64, C.c_char_p, i64], i64),
        "fi_script_elaborate": ([C.c_char_p, C.c_int, C.c_char_p, i64], i64),
        "fi_script_print": ([C.c_char_p, C.c_char_p, i64], i64),
        "fi_script_codegen": ([C.c_char_p, i64, i64, i64, C.c_char_p, i64], i64),
        "fi_script_check_async": ([C.c_char_p, i64, i64, i64, C.POINTER(AsyncCheckOptions), C.c_char_p, i64], i64),
    }
    for name, (args, res) in list(sigs.items()) + list(optional.items()):
        if not hasattr(lib, name):
            if name in sigs:
                raise ImportError(f"{LIB_PATH} does not export {name}")
            continue
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


lib = _load()


def last_error() -> str:
    return (lib.fi_last_error() or b"").decode()


def check(code: int) -> None:
    if code != FI_OK:
        raise FiError(code, last_error())
