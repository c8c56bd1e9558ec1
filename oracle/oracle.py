"""ctypes binding of the oracle (TEST INFRASTRUCTURE ONLY).

* liboracle.so  -- C restatement of the reference numerics (oracle/fi_oracle.c)
* _ref/libanvil_ref.so -- the unmodified reference compiled in place
  (oracle/Makefile); optional, present where it was built.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module. The product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libanvil_ref.so")


def build():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(os.path.join(HERE, "fi_oracle.c")):
        subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)


def _load():
    build()
    lib = C.CDLL(LIB)
    i64, f32p, vp = C.c_int64, C.POINTER(C.c_float), C.c_void_p
    lib.fio_fill_parallel.argtypes = [vp, i64, i64, C.c_int, i64, C.c_uint64, C.c_int, C.c_int]
    lib.fio_fill_integers.argtypes = [vp, i64, i64, C.c_int, i64, C.c_uint64, i64, i64]
    lib.fio_fill_uniform.argtypes = [vp, i64, i64, C.c_int, i64, C.c_uint64]
    lib.fio_round_to_f16.argtypes = [C.c_float]
    lib.fio_round_to_f16.restype = C.c_float
    lib.fio_round_to_bf16.argtypes = [C.c_float]
    lib.fio_round_to_bf16.restype = C.c_float
    lib.fio_round_array.argtypes = [vp, i64, C.c_int]
    lib.fio_digest.argtypes = [vp, i64, i64, C.c_int, i64]
    lib.fio_digest.restype = C.c_uint64
    gemm = [vp, vp, vp, i64, i64, i64, C.c_int, i64, C.c_int, i64, C.c_int, i64, C.c_int]
    lib.fio_seqk_f32.argtypes = gemm
    lib.fio_gemm_f64.argtypes = gemm
    lib.fio_sample_f64.argtypes = [vp, vp, i64, C.c_int, i64, C.c_int, i64, vp, vp, i64, vp]
    lib.fio_max_abs_error.argtypes = [vp, vp, i64]
    lib.fio_max_abs_error.restype = C.c_double
    return lib


lib = _load()
THREADS = os.cpu_count() or 1


def fill(rows: int, cols: int, seed: int, integers: bool) -> np.ndarray:
    """Logical row-major rows x cols matrix, bit-identical to anvil's
    fill_integers / fill_uniform (matrix.hpp:48-63)."""
    out = np.empty((rows, cols), dtype=np.float32)
    lib.fio_fill_parallel(out.ctypes.data, rows, cols, 1, cols, seed, int(integers), THREADS)
    return out


def fill_sequential(rows: int, cols: int, seed: int, integers: bool) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.float32)
    if integers:
        lib.fio_fill_integers(out.ctypes.data, rows, cols, 1, cols, seed, -3, 3)
    else:
        lib.fio_fill_uniform(out.ctypes.data, rows, cols, 1, cols, seed)
    return out


def round_elem(x: np.ndarray, elem: str) -> np.ndarray:
    """Grid snapping on ingestion: f16 = anvil round_to_f16, bf16 = RNE."""
    y = np.ascontiguousarray(x, dtype=np.float32).copy()
    code = {"f32": 0, "f16": 1, "bf16": 2}[elem]
    lib.fio_round_array(y.ctypes.data, y.size, code)
    return y


def digest(c_logical: np.ndarray) -> str:
    """anvil::digest (matrix.hpp:86-103) of a logical row-major matrix."""
    c = np.ascontiguousarray(c_logical, dtype=np.float32)
    return f"0x{lib.fio_digest(c.ctypes.data, c.shape[0], c.shape[1], 1, c.shape[1]):016x}"


def _gemm(fn, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    m, k = a.shape
    k2, n = b.shape
    assert k == k2
    c = np.empty((m, n), dtype=np.float32)
    fn(a.ctypes.data, b.ctypes.data, c.ctypes.data, m, n, k, 1, k, 1, n, 1, n, THREADS)
    return c


def seqk_f32(a, b) -> np.ndarray:
    """The reference simulator's FMA-leaf result: ascending k, unfused fp32."""
    return _gemm(lib.fio_seqk_f32, a, b)


def gemm_f64(a, b) -> np.ndarray:
    """tests/support/oracle.hpp naive_matmul: fp64 accumulate, rounded to fp32."""
    return _gemm(lib.fio_gemm_f64, a, b)


def sample_f64(a, b, rows, cols) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    r = np.ascontiguousarray(rows, dtype=np.int64)
    c = np.ascontiguousarray(cols, dtype=np.int64)
    out = np.empty(len(r), dtype=np.float64)
    lib.fio_sample_f64(a.ctypes.data, b.ctypes.data, a.shape[1], 1, a.shape[1], 1, b.shape[1],
                       r.ctypes.data, c.ctypes.data, len(r), out.ctypes.data)
    return out


def max_abs_error(got, want) -> float:
    g = np.ascontiguousarray(got, dtype=np.float32)
    w = np.ascontiguousarray(want, dtype=np.float32)
    return float(lib.fio_max_abs_error(g.ctypes.data, w.ctypes.data, g.size))


# ------------------------------------------------------------ reference (_ref)
def have_reference() -> bool:
    return os.path.exists(REF_LIB)


_ref = None


def ref():
    global _ref
    if _ref is None:
        r = C.CDLL(REF_LIB)
        i64 = C.c_int64
        r.ref_run.argtypes = [C.c_char_p, i64, i64, i64, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.POINTER(i64), C.POINTER(i64)]
        r.ref_time_blocks.argtypes = [C.c_char_p, i64, i64, i64, i64, C.c_int, C.POINTER(C.c_double),
                                      C.POINTER(i64)]
        r.ref_last_error.restype = C.c_char_p
        _ref = r
    return _ref


def ref_run(script: str, a: np.ndarray, b=None, m=0, n=0, k=0):
    """The reference simulator (anvil::run) on logical row-major inputs."""
    r = ref()
    a = np.ascontiguousarray(a, dtype=np.float32)
    bb = np.ascontiguousarray(b, dtype=np.float32) if b is not None else None
    rows = a.shape[0]
    cols = bb.shape[1] if bb is not None else a.shape[1]
    out = np.empty((rows, cols), dtype=np.float32)
    races = C.c_int64(0)
    rc = r.ref_run(script.encode(), m, n, k, a.ctypes.data, bb.ctypes.data if bb is not None else None,
                   out.ctypes.data, C.byref(races), None)
    if rc:
        raise RuntimeError(r.ref_last_error().decode())
    return out, races.value


def ref_time_blocks(script: str, m: int, n: int, k: int, blocks: int, threads: int):
    """Times `blocks` CTA blocks of the reference Machine; returns (secs, grid_blocks)."""
    r = ref()
    secs = C.c_double(0)
    grid = C.c_int64(0)
    rc = r.ref_time_blocks(script.encode(), m, n, k, blocks, threads, C.byref(secs), C.byref(grid))
    if rc:
        raise RuntimeError(r.ref_last_error().decode())
    return secs.value, grid.value
