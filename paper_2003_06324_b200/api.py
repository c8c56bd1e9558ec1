"""Python host API over the C ABI (include/fireiron_b200.h).

Mirrors the reference's execution-path interface (proj/include/anvil):
  validate / elaborate / print_script / generate  -> IR services (no GPU)
  Plan(script).run_host(A, B)                      -> anvil::run (sim.hpp:495)
  Plan(script).launch(dA, dB, dC, stream)          -> device-resident execution
Errors raise FiError whose .kind is the anvil::ErrorKind name
(proj/include/anvil/error.hpp:8-33) or a backend error name.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _native as N
from ._native import FiError

ELEM_NAMES = {N.FI_F32: "f32", N.FI_F16: "f16", N.FI_BF16: "bf16"}


def _text(fn, *args) -> str:
    cap = 1 << 16
    while True:
        buf = C.create_string_buffer(cap)
        n = fn(*args, buf, cap)
        if n < 0:
            raise FiError(int(-n), N.last_error())
        if n < cap:
            return buf.value.decode()
        cap = int(n) + 1


def _enc(script: str) -> bytes:
    return script.encode() if isinstance(script, str) else script


def validate(script: str, m: int = 0, n: int = 0, k: int = 0) -> str:
    """ValidationReport::to_string of validate_with_plan (decomp.hpp:397-411)."""
    return _text(N.lib.fi_script_validate, _enc(script), m, n, k)


def elaborate(script: str, with_subs: bool = False) -> str:
    """render_trace(elaborate(...)) (decomp.hpp:739-770)."""
    return _text(N.lib.fi_script_elaborate, _enc(script), int(with_subs))


def print_script(script: str) -> str:
    """Canonical script text (script.hpp:739-793)."""
    return _text(N.lib.fi_script_print, _enc(script))


def generate(script: str, m: int = 0, n: int = 0, k: int = 0) -> str:
    """sm_100a CUDA translation unit for the strategy (the anvil::generate seam)."""
    return _text(N.lib.fi_script_codegen, _enc(script), m, n, k)


def plan_summary(script: str, m: int = 0, n: int = 0, k: int = 0) -> str:
    """Launch + buffer plan of lower() (program.hpp:628), one line per buffer."""
    return _text(N.lib.fi_script_plan, _enc(script), m, n, k)


MUTATIONS = {"none": 0, "skip_empty_wait": 1, "ring_drain_every_unit": 2, "flag_before_bulk_wait": 3,
             "skip_tmem_empty_wait": 4, "remainder_slot_collision": 5, "unpacked_peer_staging": 6,
             "tx_undercount": 7, "mcast_single_release": 8, "gate_skip_acquire": 9}


class AsyncReport:
    """Result of check_async: counts plus the report text."""

    def __init__(self, text: str):
        import re
        self.text = text
        self.ok = text.startswith("async protocol check: ok")
        nums = dict(re.findall(r"(events|races|capacity|coverage|deadlocks) (\d+)", text))
        self.events = int(nums.get("events", 0))
        self.races = int(nums.get("races", 0))
        self.capacity_errors = int(nums.get("capacity", 0))
        self.coverage_errors = int(nums.get("coverage", 0))
        self.deadlocks = int(nums.get("deadlocks", 0))
        m = re.search(r"schedule: (\d+) clusters x (\d+) CTAs, (\d+) tiles, (\d+) units, mode (\d+), "
                      r"slices (\d+)( \+ remainder)?( \(pull fixup(, first)?\))?, split-k (\d+), stages (\d+)", text)
        if m:
            self.clusters, self.cluster_size, self.tiles, self.units, self.mode, self.slices = \
                (int(x) for x in m.groups()[:6])
            self.remainder = m.group(7) is not None
            self.pull = m.group(8) is not None
            self.head = m.group(9) is not None
            self.split_k, self.stages = int(m.group(10)), int(m.group(11))

    def __repr__(self):
        return self.text


def check_async(script: str, m: int = 0, n: int = 0, k: int = 0, *, num_sms: int = 148,
                max_active_clusters: int = 0, streamk: int = -1, remainder: int = 1, c_tma: int = -1,
                ring_drain: int = 1, pull_d: int = -2, head: int = 1, mutation: str = "none",
                gated_chunks: int = 0, gated_first: int = 0) -> AsyncReport:
    """CPU check of the asynchronous protocol (mbarrier phases, TMA, tcgen05
    commits, TMEM hand-off, bulk copies, epoch flags) of the launch a tcgen05
    strategy lowers to: races, capacity, coverage, deadlock
    (include/fireiron/async_check.hpp). No GPU needed. gated_chunks > 0 models
    a gated launch (fi_plan_launch_gated): B in that many column chunks, each
    landed by a copy engine and released by its ready flag."""
    o = N.AsyncCheckOptions(num_sms, max_active_clusters, streamk, remainder, c_tma, ring_drain,
                            MUTATIONS[mutation], pull_d, head, gated_chunks, gated_first)
    return AsyncReport(_text(N.lib.fi_script_check_async, _enc(script), m, n, k, C.byref(o)))


def host_snap(x: np.ndarray, elem: str = "f16") -> np.ndarray:
    """fp32 -> f16/bf16 bit patterns (uint16) on the host, as fi_plan_run_host
    snaps input panels before they cross PCIe (fi_host_snap_f32)."""
    src = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(src.shape, dtype=np.uint16)
    code = {"f16": 1, "bf16": 2}[elem]
    N.check(N.lib.fi_host_snap_f32(src.ctypes.data, out.ctypes.data, src.size, code))
    return out


def _np_elem(code: int):
    return {N.FI_F32: np.float32, N.FI_F16: np.float16}.get(code)


class Plan:
    """A compiled strategy: parse -> validate -> lower -> emit -> compile -> load."""

    def __init__(self, script: str, m: int = 0, n: int = 0, k: int = 0, device: int = 0):
        h = C.c_void_p()
        N.check(N.lib.fi_plan_create(_enc(script), m, n, k, device, 0, C.byref(h)))
        self._h = h
        info = N.PlanInfo()
        N.check(N.lib.fi_plan_query(self._h, C.byref(info)))
        self.info = info

    def close(self):
        h = getattr(self, "_h", None)
        self._h = None
        if h and N is not None and getattr(N, "lib", None) is not None:
            N.lib.fi_plan_destroy(h)

    __del__ = close

    # ---- shapes / layouts of the root operands -------------------------
    @property
    def m(self): return int(self.info.m)

    @property
    def n(self): return int(self.info.n)

    @property
    def k(self): return int(self.info.k)

    @property
    def kind(self) -> str:
        return "tcgen05" if self.info.kind == N.FI_KIND_TCGEN05 else "generic"

    @property
    def flops(self) -> float:
        return float(self.info.flops)

    def source(self) -> str:
        return _text(N.lib.fi_plan_source, self._h)

    def shapes(self):
        """(rows, cols, row_major) of the physical A, B, C roots."""
        i = self.info
        if i.is_move:
            return (i.m, i.n, bool(i.a_row_major)), None, (i.m, i.n, bool(i.c_row_major))
        return ((i.m, i.k, bool(i.a_row_major)), (i.k, i.n, bool(i.b_row_major)),
                (i.m, i.n, bool(i.c_row_major)))

    # ---- execution -------------------------------------------------------
    def launch(self, dA: int, dB: Optional[int], dC: int, stream: int = 0) -> None:
        """Stream-ordered launch on device pointers (root element types/layouts)."""
        N.check(N.lib.fi_plan_launch(self._h, C.c_void_p(dA), C.c_void_p(dB or 0) if dB else None,
                                     C.c_void_p(dC), C.c_void_p(stream) if stream else None))

    def launch_gated(self, dA: int, dB: int, dC: int, stream: int, ready: int, epoch: int, chunk_cols: int,
                     first_chunk: int) -> None:
        """Launch with B's column chunks (chunk_cols wide) gated by the device
        flags ready[j] >= epoch, scheduling chunk first_chunk first (the fused
        all-gather -> GEMM of the multi-GPU driver)."""
        N.check(N.lib.fi_plan_launch_gated(self._h, C.c_void_p(dA), C.c_void_p(dB), C.c_void_p(dC),
                                           C.c_void_p(stream) if stream else None, C.c_void_p(ready),
                                           C.c_uint32(epoch), C.c_int64(chunk_cols), C.c_int32(first_chunk)))

    def run_host(self, A: np.ndarray, B: Optional[np.ndarray] = None) -> np.ndarray:
        """anvil::run semantics: logical fp32 matrices in, logical fp32 C out.

        A is M x K (B is K x N); they are laid out into the root layouts here,
        snapped to the root element grid on the device, executed, and C is
        returned as a logical M x N float32 array."""
        sa, sb, sc = self.shapes()

        def phys(x, shape):
            rows, cols, row_major = shape
            x = np.asarray(x, dtype=np.float32)
            if x.shape != (rows, cols):
                raise FiError(2, f"input must be {rows}x{cols}, got {x.shape}")
            return np.ascontiguousarray(x if row_major else x.T)

        pa = phys(A, sa)
        pb = phys(B, sb) if sb is not None else None
        rows, cols, c_row = sc
        out = np.empty((rows, cols) if c_row else (cols, rows), dtype=np.float32)
        N.check(N.lib.fi_plan_run_host(self._h, pa.ctypes.data, pb.ctypes.data if pb is not None else None,
                                       out.ctypes.data))
        return out if c_row else out.T.copy()

    def host_bytes(self):
        """(H2D, D2H) bytes the last run_host moved across PCIe."""
        up, down = C.c_int64(), C.c_int64()
        N.check(N.lib.fi_plan_host_bytes(self._h, C.byref(up), C.byref(down)))
        return int(up.value), int(down.value)

    def run_host_ptr(self, pA: int, pB: Optional[int], pC: int) -> None:
        """fi_plan_run_host on raw host pointers (physical root layouts, fp32)."""
        N.check(N.lib.fi_plan_run_host(self._h, C.c_void_p(pA), C.c_void_p(pB) if pB else None,
                                       C.c_void_p(pC)))
