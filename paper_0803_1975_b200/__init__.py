"""paper_0803_1975_b200 — B200-native compressed modular GEMM (Dumas et al.,
arXiv 0803.1975), host-side mirror of the reference's ``qgemm`` header API.

The reference API (``/root/reference/proj/include/qgemm/*.hpp``) is
restated here with the same names, argument meaning and error behaviour;
every computation goes through the C ABI of ``_lib/libqgemm_b200.so``
(``include/qgemm_b200.h``), i.e. through hand-written sm_100a kernels.
There is no CPU fallback: if the library is missing this module raises
on import, and device calls without a CUDA device raise ``CudaError``.

PyTorch is used only as plumbing: device buffers, the current CUDA stream
and pinned host memory.

Reference mapping (file:line):
  plan_compression / uncompressed_plan / plan_packed_axis / choose_panel
      plan.hpp:125-224
  compress_rows_reversed / compress_cols_forward / compress_outer_cols /
  compress_outer_rows                      gemm.hpp:104-178
  uncompress                               gemm.hpp:182-204
  packed_common_product                    gemm.hpp:210-244
  reduce_common_entry                      gemm.hpp:247-250
  mul_common_compressed                    gemm.hpp:254-271
  mul_common_repacked                      gemm.hpp:275-280
  packed_right_product / redq_in_place / mul_right_compressed
                                           gemm.hpp:285-335
  blocked_accumulate                       gemm.hpp:450-489
  random_residue_matrix                    prng.hpp:31-38
  residue_checksum                         bench.hpp:43-47
"""
from __future__ import annotations

import ctypes
import dataclasses
import enum
import os
from typing import Optional, Union

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QG_LIB_PATH") or os.path.join(_HERE, "_lib", "libqgemm_b200.so")  # QG_LIB_PATH: experiment builds
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "qgemm_b200.h")


# ----------------------------------------------------------------- errors
class Error(RuntimeError):
    """qgemm::Error, errors.hpp:8-10."""


class InvalidModulus(Error):
    pass


class NoCompression(Error):
    pass


class SlotOverflow(Error):
    pass


class DigitOverflow(Error):
    pass


class DimensionMismatch(Error):
    pass


class PlanMismatch(Error):
    pass


class UnsupportedAlgorithm(Error):
    pass


class ParseError(Error):
    pass


class InvalidArgument(ValueError):
    """std::invalid_argument (plan.hpp:128-129, gemm.hpp:455)."""


class CudaError(Error):
    pass


class NotExact(Error):
    pass


_STATUS = {
    1: InvalidModulus,
    2: NoCompression,
    3: SlotOverflow,
    4: DigitOverflow,
    5: DimensionMismatch,
    6: PlanMismatch,
    7: UnsupportedAlgorithm,
    8: ParseError,
    9: InvalidArgument,
    10: CudaError,
    11: Error,
    12: NotExact,
}


# ----------------------------------------------------------------- C types
class _Plan(ctypes.Structure):
    _fields_ = [
        ("p", ctypes.c_uint32),
        ("t", ctypes.c_int32),
        ("d", ctypes.c_int32),
        ("e", ctypes.c_int32),
        ("beta", ctypes.c_int32),
        ("kmax", ctypes.c_uint64),
        ("inv_qd", ctypes.c_double),
        ("extraction", ctypes.c_int32),
    ]


class _GpuPlan(ctypes.Structure):
    _fields_ = [("plan", _Plan), ("kblock_words", ctypes.c_uint64), ("max_exact_words", ctypes.c_uint64),
                ("balanced", ctypes.c_int32), ("anchored", ctypes.c_int32)]


class _FullPlan(ctypes.Structure):
    _fields_ = [("base", _Plan), ("dq", ctypes.c_int32), ("dtheta", ctypes.c_int32),
                ("theta_exponent", ctypes.c_int32)]


class _Orientation(ctypes.Structure):
    _fields_ = [("direction", ctypes.c_int32), ("axis", ctypes.c_int32), ("slots", ctypes.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_0803_1975_b200). There is no CPU fallback."
        )
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    sz, u32, u64, i32, vp = ctypes.c_size_t, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
    sig = {
        "qg_abi_version": ([], i32),
        "qg_status_string": ([i32], ctypes.c_char_p),
        "qg_plan_compression": ([u32, u64, i32, i32, P(_Plan)], i32),
        "qg_uncompressed_plan": ([u32, u64, i32, P(_Plan)], i32),
        "qg_plan_packed_axis": ([u32, u64, u64, i32, P(_Plan)], i32),
        "qg_choose_panel": ([u32, u64, i32, P(u64)], i32),
        "qg_max_exact_block": ([P(_Plan), P(u64)], i32),
        "qg_gpu_plan_from": ([P(_Plan), u64, P(_GpuPlan)], i32),
        "qg_plan_gpu": ([u32, u64, P(_GpuPlan)], i32),
        "qg_plan_gpu_ex": ([u32, u64, i32, P(_GpuPlan)], i32),
        "qg_max_exact_block_balanced": ([P(_Plan), P(u64)], i32),
        "qg_gpu_plan_kmax": ([P(_GpuPlan), P(u64)], i32),
        "qg_max_exact_block_anchored": ([P(_Plan), P(u64), P(i32)], i32),
        "qg_gen_residues": ([u64, u32, sz, sz, sz, vp, i32, vp], i32),
        "qg_compress_rows_reversed": ([P(_Plan), vp, i32, sz, sz, sz, vp, sz, vp], i32),
        "qg_compress_cols_forward": ([P(_Plan), vp, i32, sz, sz, sz, vp, sz, vp], i32),
        "qg_compress_outer_cols": ([P(_Plan), vp, i32, sz, sz, sz, vp, sz, vp], i32),
        "qg_compress_outer_rows": ([P(_Plan), vp, i32, sz, sz, sz, vp, sz, vp], i32),
        "qg_packed_common_product": ([P(_Plan), vp, vp, sz, sz, sz, vp, vp], i32),
        "qg_reduce_common": ([P(_Plan), vp, sz, vp, vp], i32),
        "qg_mul_common": ([P(_GpuPlan), vp, vp, sz, sz, sz, vp, sz, vp], i32),
        "qg_mul_common_repacked": ([P(_GpuPlan), vp, vp, sz, sz, sz, vp, vp, vp], i32),
        "qg_mul_right": ([P(_Plan), vp, sz, vp, sz, sz, sz, vp, vp], i32),
        "qg_packed_right_product": ([P(_Plan), vp, sz, vp, sz, sz, sz, vp, vp], i32),
        "qg_redq": ([P(_Plan), vp, sz, vp], i32),
        "qg_uncompress": ([P(_Plan), _Orientation, vp, sz, sz, sz, sz, vp, vp], i32),
        "qg_host_mul_common": ([P(_Plan), vp, vp, sz, sz, sz, vp], i32),
        "qg_host_mul_common_gpu": ([P(_GpuPlan), vp, vp, sz, sz, sz, vp], i32),
        "qg_host_mul_common_multi": ([P(_GpuPlan), P(i32), i32, vp, vp, sz, sz, sz, vp], i32),
        "qg_host_blocked_accumulate": ([P(_Plan), vp, vp, sz, sz, sz, sz, vp], i32),
        "qg_host_mul_right": ([P(_Plan), vp, vp, sz, sz, sz, vp], i32),
        "qg_tiled_stage_words": ([P(_GpuPlan), u64, P(u32)], i32),
        "qg_tiled_words": ([sz, sz, i32, u32], sz),
        "qg_pack_a_tiled": ([P(_GpuPlan), u32, vp, i32, sz, sz, sz, vp, vp], i32),
        "qg_pack_b_tiled": ([P(_GpuPlan), u32, vp, i32, sz, sz, sz, vp, vp], i32),
        "qg_mul_common_tiled": ([P(_GpuPlan), vp, vp, sz, sz, sz, vp, sz, vp], i32),
        "qg_mul_common_compressed": ([P(_GpuPlan), vp, sz, vp, sz, i32, sz, sz, sz, vp, sz, vp], i32),
        "qg_plan_right_gpu": ([u32, u64, u64, P(_GpuPlan)], i32),
        "qg_right_tiled_stage": ([P(_GpuPlan), u64, P(u32)], i32),
        "qg_pack_residues_tiled": ([u32, vp, i32, sz, sz, sz, vp, vp], i32),
        "qg_pack_outer_cols_tiled": ([P(_Plan), u32, vp, i32, sz, sz, sz, vp, vp], i32),
        "qg_mul_right_tiled": ([P(_GpuPlan), vp, vp, sz, sz, sz, vp, sz, vp], i32),
        "qg_pack_outer_rows_tiled": ([P(_Plan), u32, vp, i32, sz, sz, sz, vp, vp], i32),
        "qg_pack_residues_b_tiled": ([u32, vp, i32, sz, sz, sz, vp, vp], i32),
        "qg_mul_left_tiled": ([P(_GpuPlan), vp, vp, sz, sz, sz, vp, sz, vp], i32),
        "qg_pack_residues_tiled_bal": ([u32, u32, vp, i32, sz, sz, sz, vp, vp], i32),
        "qg_pack_residues_b_tiled_bal": ([u32, u32, vp, i32, sz, sz, sz, vp, vp], i32),
        "qg_pack_outer_cols_tiled_bal": ([P(_Plan), u32, vp, i32, sz, sz, sz, vp, vp], i32),
        "qg_pack_outer_rows_tiled_bal": ([P(_Plan), u32, vp, i32, sz, sz, sz, vp, vp], i32),
        "qg_plan_full": ([u32, u64, i32, P(_FullPlan)], i32),
        "qg_plan_full_gpu": ([u32, u64, P(_FullPlan), P(u64)], i32),
        "qg_full_tiled_stage": ([P(_FullPlan), u64, u64, P(u32)], i32),
        "qg_mul_full_tiled": ([P(_FullPlan), u64, vp, vp, sz, sz, sz, vp, sz, vp], i32),
        "qg_uncompress_full": ([P(_FullPlan), vp, sz, sz, sz, vp, sz, vp], i32),
        "qg_host_mul_left": ([P(_Plan), vp, vp, sz, sz, sz, vp], i32),
        "qg_host_mul_left_gpu": ([P(_GpuPlan), vp, vp, sz, sz, sz, vp], i32),
        "qg_host_mul_right_gpu": ([P(_GpuPlan), vp, vp, sz, sz, sz, vp], i32),
        "qg_host_mul_full": ([P(_FullPlan), u64, vp, vp, sz, sz, sz, vp], i32),
        "qg_naive_gemm": ([u32, vp, vp, sz, sz, sz, vp, sz, vp], i32),
        "qg_extract_coefficients": ([P(_Plan), vp, sz, vp, vp], i32),
        "qg_reduce_and_compress": ([P(_Plan), vp, sz, sz, sz, vp, sz, vp], i32),
        "qg_host_naive_gemm": ([u32, vp, vp, sz, sz, sz, vp], i32),
        "qg_host_uncompress": ([P(_Plan), _Orientation, vp, sz, sz, sz, sz, vp], i32),
        "qg_host_random_residue_matrix": ([sz, sz, u32, u64, vp], i32),
        "qg_last_phase_seconds": ([P(ctypes.c_double), P(ctypes.c_double)], None),
        "qg_set_phase_timing": ([i32], None),
        "qg_parse_matrix": ([ctypes.c_char_p, sz, P(u32), P(sz), P(sz), P(P(u32))], i32),
        "qg_read_matrix_file": ([ctypes.c_char_p, P(u32), P(sz), P(sz), P(P(u32))], i32),
        "qg_write_matrix_file": ([ctypes.c_char_p, u32, vp, sz, sz], i32),
        "qg_free": ([vp], None),
        "qg_compress_rows_reversed_u64": ([P(_Plan), vp, i32, sz, sz, sz, vp, sz, vp], i32),
        "qg_compress_cols_forward_u64": ([P(_Plan), vp, i32, sz, sz, sz, vp, sz, vp], i32),
        "qg_compress_outer_cols_u64": ([P(_Plan), vp, i32, sz, sz, sz, vp, sz, vp], i32),
        "qg_compress_outer_rows_u64": ([P(_Plan), vp, i32, sz, sz, sz, vp, sz, vp], i32),
        "qg_packed_common_product_u64": ([P(_Plan), vp, vp, sz, sz, sz, vp, vp], i32),
        "qg_reduce_common_u64": ([P(_Plan), vp, sz, vp, vp], i32),
        "qg_extract_coefficients_u64": ([P(_Plan), vp, sz, vp, vp], i32),
        "qg_reduce_and_compress_u64": ([P(_Plan), vp, sz, sz, sz, vp, sz, vp], i32),
        "qg_redq_u64": ([P(_Plan), vp, sz, vp], i32),
        "qg_uncompress_u64": ([P(_Plan), _Orientation, vp, sz, sz, sz, sz, vp, vp], i32),
        "qg_packed_right_product_u64": ([P(_Plan), vp, i32, sz, vp, sz, sz, sz, vp, vp], i32),
        "qg_mul_right_u64": ([P(_Plan), vp, i32, sz, vp, sz, sz, sz, vp, vp], i32),
        "qg_packed_left_product_u64": ([P(_Plan), vp, vp, i32, sz, sz, sz, sz, vp, vp], i32),
        "qg_mul_left_u64": ([P(_Plan), vp, vp, i32, sz, sz, sz, sz, vp, vp], i32),
        "qg_mul_full_u64": ([P(_FullPlan), vp, i32, vp, i32, sz, sz, sz, vp, sz, vp], i32),
        "qg_host_mul_common_i64": ([P(_Plan), vp, vp, sz, sz, sz, vp], i32),
        "qg_host_blocked_accumulate_i64": ([P(_Plan), vp, vp, sz, sz, sz, sz, vp], i32),
        "qg_host_mul_right_i64": ([P(_Plan), vp, vp, sz, sz, sz, vp], i32),
        "qg_host_mul_left_i64": ([P(_Plan), vp, vp, sz, sz, sz, vp], i32),
        "qg_host_mul_full_i64": ([P(_FullPlan), vp, vp, sz, sz, sz, vp], i32),
        "qg_mul_common_repacked_tiled": ([P(_GpuPlan), vp, vp, sz, sz, sz, vp, sz, vp], i32),
        "qg_mul_common_repacked_compressed": ([P(_GpuPlan), vp, sz, vp, sz, i32, sz, sz, sz, vp, sz, vp], i32),
        "qg_host_mul_common_repacked": ([P(_Plan), vp, vp, sz, sz, sz, vp], i32),
        "qg_host_mul_common_repacked_gpu": ([P(_GpuPlan), vp, vp, sz, sz, sz, vp], i32),
        "qg_packed_left_product": ([P(_Plan), vp, sz, vp, i32, sz, sz, sz, sz, vp, vp], i32),
        "qg_mul_left": ([P(_Plan), vp, sz, vp, i32, sz, sz, sz, sz, vp, vp], i32),
        "qg_extract_digits": ([P(_Plan), vp, sz, vp, vp], i32),
        "qg_extract_digits_u64": ([P(_Plan), vp, sz, vp, vp], i32),
        "qg_device_alloc": ([sz, P(vp)], i32),
        "qg_device_free": ([vp], i32),
        "qg_copy_to_device": ([vp, vp, sz], i32),
        "qg_copy_to_host": ([vp, vp, sz], i32),
        "qg_host_pack_b_slot_tiled": ([P(_GpuPlan), u32, vp, sz, sz, sz, sz, vp, vp], i32),
        "qg_host_mul_common_packed_b": ([P(_GpuPlan), vp, sz, sz, vp, sz, vp, vp], i32),
        "qg_set_dynamic_tiles": ([i32], None),
        "qg_kernel_launches": ([], u64),
        "qg_last_kernel": ([], ctypes.c_char_p),
        "qg_last_error": ([], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


lib = _load()
EXPORTED_SYMBOLS = tuple(
    n for n in dir(lib) if n.startswith("qg_")
)  # populated lazily by ctypes; use header_symbols() for the declared list


def header_symbols(path: str = HEADER_PATH) -> list:
    """Function names declared in include/qgemm_b200.h."""
    import re

    text = open(path).read()
    return sorted(set(re.findall(r"\b(qg_[a-z0-9_]+)\s*\(", text)))


def _check(status: int) -> None:
    if status != 0:
        cls = _STATUS.get(status, Error)
        msg = lib.qg_status_string(status).decode()
        if status == 10:
            msg += ": " + lib.qg_last_error().decode()
        raise cls(msg)


# ----------------------------------------------------------------- plans
class ExtractionMode(enum.IntEnum):
    """plan.hpp:14-17."""

    ReciprocalMul = 0
    AddHighBits = 1


@dataclasses.dataclass(frozen=True)
class CompressionPlan:
    """CompressionPlan, plan.hpp:29-42."""

    p: int
    t: int
    d: int
    e: int
    beta: int
    kmax: int
    inv_qd: float
    extraction: int = 0

    def q(self) -> int:
        return 1 << self.t

    def q_mask(self) -> int:
        return (1 << self.t) - 1

    def _c(self) -> _Plan:
        return _Plan(self.p, self.t, self.d, self.e, self.beta, self.kmax, self.inv_qd, self.extraction)

    @staticmethod
    def _from(c: _Plan) -> "CompressionPlan":
        return CompressionPlan(c.p, c.t, c.d, c.e, c.beta, c.kmax, c.inv_qd, c.extraction)


@dataclasses.dataclass(frozen=True)
class GpuPlan:
    """A CompressionPlan k-blocked for the FP64 tensor-core contraction."""

    plan: CompressionPlan
    kblock_words: int
    max_exact_words: int
    balanced: int = 0
    anchored: int = 0

    def _c(self) -> _GpuPlan:
        return _GpuPlan(self.plan._c(), self.kblock_words, self.max_exact_words, self.balanced, self.anchored)

    @staticmethod
    def _from(c: "_GpuPlan") -> "GpuPlan":
        return GpuPlan(CompressionPlan._from(c.plan), c.kblock_words, c.max_exact_words, c.balanced, c.anchored)

    def eq3_kmax(self) -> int:
        """Residues a k-block may hold (Eq. 3) for this plan's digits
        (qg_gpu_plan_kmax): plan.kmax's bound for unsigned digits, the
        balanced-digit bound for balanced ones."""
        out = ctypes.c_uint64()
        g = self._c()
        _check(lib.qg_gpu_plan_kmax(ctypes.byref(g), ctypes.byref(out)))
        return out.value


def make_plan(p: int, t: int, e: int, beta: int = 53) -> CompressionPlan:
    """The hand-built plan of the reference tests (test_pack.cpp:15-24)."""
    import math

    if p < 2 or any(p % f == 0 for f in range(2, int(math.isqrt(p)) + 1)):
        raise InvalidModulus(f"modulus {p} is not prime")
    return CompressionPlan(p, t, e - 1, e, beta, ((1 << t) - 1) // ((p - 1) ** 2), math.ldexp(1.0, -t * (e - 1)), 0)


def plan_compression(p: int, k: int, beta: int = 53, mode: int = ExtractionMode.ReciprocalMul) -> CompressionPlan:
    out = _Plan()
    _check(lib.qg_plan_compression(p, k, beta, int(mode), ctypes.byref(out)))
    return CompressionPlan._from(out)


def uncompressed_plan(p: int, k: int, beta: int = 53) -> CompressionPlan:
    out = _Plan()
    _check(lib.qg_uncompressed_plan(p, k, beta, ctypes.byref(out)))
    return CompressionPlan._from(out)


def plan_packed_axis(p: int, k: int, axis_len: int, beta: int = 53) -> CompressionPlan:
    out = _Plan()
    _check(lib.qg_plan_packed_axis(p, k, axis_len, beta, ctypes.byref(out)))
    return CompressionPlan._from(out)


def choose_panel(p: int, k: int, beta: int = 53) -> int:
    out = ctypes.c_uint64()
    _check(lib.qg_choose_panel(p, k, beta, ctypes.byref(out)))
    return out.value


def max_exact_block(plan: CompressionPlan) -> int:
    out = ctypes.c_uint64()
    pl = plan._c()
    _check(lib.qg_max_exact_block(ctypes.byref(pl), ctypes.byref(out)))
    return out.value


def gpu_plan_from(plan: CompressionPlan, k: int) -> GpuPlan:
    out = _GpuPlan()
    pl = plan._c()
    _check(lib.qg_gpu_plan_from(ctypes.byref(pl), k, ctypes.byref(out)))
    return GpuPlan._from(out)


def plan_gpu(p: int, k: int, balanced: bool = True, anchored: bool = True) -> GpuPlan:
    """(t, e, k-block[, balanced digits][, anchored accumulation]) for the
    tensor-core path; balanced=False restricts to the reference's unsigned
    packing, anchored=False to the FP64-add block flush (K4)."""
    out = _GpuPlan()
    _check(lib.qg_plan_gpu_ex(p, k, (0 if balanced else 1) | (0 if anchored else 2), ctypes.byref(out)))
    return GpuPlan._from(out)


def max_exact_block_anchored(plan: CompressionPlan):
    """(words, E): the largest k-block of the anchored accumulation (DESIGN.md
    §3g) and the binade exponent its anchor uses; (0, 0) if none is exact."""
    out = ctypes.c_uint64()
    ex = ctypes.c_int()
    pl = plan._c()
    _check(lib.qg_max_exact_block_anchored(ctypes.byref(pl), ctypes.byref(out), ctypes.byref(ex)))
    return out.value, ex.value


def max_exact_block_balanced(plan: CompressionPlan) -> int:
    out = ctypes.c_uint64()
    pl = plan._c()
    _check(lib.qg_max_exact_block_balanced(ctypes.byref(pl), ctypes.byref(out)))
    return out.value


def kernel_launches() -> int:
    return int(lib.qg_kernel_launches())


def last_kernel() -> str:
    return lib.qg_last_kernel().decode()


# ----------------------------------------------------------------- device data
def _torch():
    import torch

    return torch


def _stream() -> ctypes.c_void_p:
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _dtype_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.float64:
        return 0
    if t.dtype == torch.int32:
        return 2
    if getattr(torch, "uint32", None) is not None and t.dtype == torch.uint32:
        return 1
    raise InvalidArgument(f"residues must be float64, int32 or uint32 tensors, got {t.dtype}")


def _require_cuda(*ts):
    for t in ts:
        if not t.is_cuda:
            raise InvalidArgument("device entry points take CUDA tensors (use the *_host functions for host data)")
        if not t.is_contiguous():
            raise InvalidArgument("tensors must be contiguous row-major")


class PackDirection(enum.IntEnum):
    Forward = 0
    Reversed = 1


class PackAxis(enum.IntEnum):
    Row = 0
    Column = 1


@dataclasses.dataclass
class PackOrientation:
    """PackOrientation, matrix.hpp:33-39."""

    direction: int = PackDirection.Forward
    axis: int = PackAxis.Column
    slots: int = 1


@dataclasses.dataclass
class CompressedMatrix:
    """CompressedMatrix<DoubleWord>, matrix.hpp:44-63: row-major packed words
    (a float64 CUDA tensor of shape stored_rows x stored_cols) plus the
    metadata needed to undo the packing."""

    logical_rows: int
    logical_cols: int
    stored_rows: int
    stored_cols: int
    orientation: PackOrientation
    plan: CompressionPlan
    data: object  # torch.Tensor, float64, cuda


def random_residue_matrix(rows: int, cols: int, p: int, seed: int, *, dtype=None, device="cuda",
                          row0: int = 0):
    """random_residue_matrix(rows, cols, PrimeModulus(p), seed), prng.hpp:31-38,
    generated on the device (K0); rows [row0, row0+rows) of the seeded matrix."""
    torch = _torch()
    dtype = torch.float64 if dtype is None else dtype
    out = torch.empty((rows, cols), dtype=dtype, device=device)
    code = 0 if dtype == torch.float64 else 1
    if code == 1 and dtype not in (torch.int32, getattr(torch, "uint32", torch.int32)):
        raise InvalidArgument("dtype must be float64, int32 or uint32")
    _check(lib.qg_gen_residues(seed, p, row0, rows, cols, _ptr(out), code, _stream()))
    return out


def compress_rows_reversed(a, plan: CompressionPlan) -> CompressedMatrix:
    """gemm.hpp:104-118: m x ceil(k/e) words, {Reversed, Column, e}."""
    torch = _torch()
    _require_cuda(a)
    m, k = a.shape
    groups = (k + plan.e - 1) // plan.e
    out = torch.empty((m, groups), dtype=torch.float64, device=a.device)
    pl = plan._c()
    _check(lib.qg_compress_rows_reversed(ctypes.byref(pl), _ptr(a), _dtype_code(a), m, k, k, _ptr(out), groups, _stream()))
    return CompressedMatrix(m, k, m, groups, PackOrientation(PackDirection.Reversed, PackAxis.Column, plan.e), plan, out)


def compress_cols_forward(b, plan: CompressionPlan) -> CompressedMatrix:
    """gemm.hpp:122-140: ceil(k/e) x n words, {Forward, Row, e}."""
    torch = _torch()
    _require_cuda(b)
    k, n = b.shape
    groups = (k + plan.e - 1) // plan.e
    out = torch.empty((groups, n), dtype=torch.float64, device=b.device)
    pl = plan._c()
    _check(lib.qg_compress_cols_forward(ctypes.byref(pl), _ptr(b), _dtype_code(b), k, n, n, _ptr(out), n, _stream()))
    return CompressedMatrix(k, n, groups, n, PackOrientation(PackDirection.Forward, PackAxis.Row, plan.e), plan, out)


def compress_outer_cols(b, plan: CompressionPlan) -> CompressedMatrix:
    """gemm.hpp:145-158: rows x ceil(cols/e) words, {Forward, Column, e}."""
    torch = _torch()
    _require_cuda(b)
    rows, cols = b.shape
    groups = (cols + plan.e - 1) // plan.e
    out = torch.empty((rows, groups), dtype=torch.float64, device=b.device)
    pl = plan._c()
    _check(lib.qg_compress_outer_cols(ctypes.byref(pl), _ptr(b), _dtype_code(b), rows, cols, cols, _ptr(out), groups, _stream()))
    return CompressedMatrix(rows, cols, rows, groups, PackOrientation(PackDirection.Forward, PackAxis.Column, plan.e), plan, out)


def compress_outer_rows(a, plan: CompressionPlan) -> CompressedMatrix:
    """gemm.hpp:161-178: ceil(rows/e) x cols words, {Forward, Row, e}."""
    torch = _torch()
    _require_cuda(a)
    rows, cols = a.shape
    groups = (rows + plan.e - 1) // plan.e
    out = torch.empty((groups, cols), dtype=torch.float64, device=a.device)
    pl = plan._c()
    _check(lib.qg_compress_outer_rows(ctypes.byref(pl), _ptr(a), _dtype_code(a), rows, cols, cols, _ptr(out), cols, _stream()))
    return CompressedMatrix(rows, cols, groups, cols, PackOrientation(PackDirection.Forward, PackAxis.Row, plan.e), plan, out)


def uncompress(cm: CompressedMatrix):
    """gemm.hpp:182-204 -> int32 logical_rows x logical_cols residues."""
    torch = _torch()
    out = torch.empty((cm.logical_rows, cm.logical_cols), dtype=torch.int32, device=cm.data.device)
    pl = cm.plan._c()
    o = _Orientation(int(cm.orientation.direction), int(cm.orientation.axis), int(cm.orientation.slots))
    _check(lib.qg_uncompress(ctypes.byref(pl), o, _ptr(cm.data), cm.stored_rows, cm.stored_cols,
                             cm.logical_rows, cm.logical_cols, _ptr(out), _stream()))
    return out


def _plans_compatible(a: CompressionPlan, b: CompressionPlan) -> bool:  # gemm.hpp:37-39
    return a.p == b.p and a.t == b.t and a.e == b.e and a.beta == b.beta


def _check_common_operands(ca: CompressedMatrix, cb: CompressedMatrix) -> None:
    """The checks of packed_common_product, gemm.hpp:213-225."""
    if not _plans_compatible(ca.plan, cb.plan):
        raise PlanMismatch("operands were packed under different plans")
    if (ca.orientation.direction != PackDirection.Reversed or ca.orientation.axis != PackAxis.Column
            or cb.orientation.direction != PackDirection.Forward or cb.orientation.axis != PackAxis.Row):
        raise PlanMismatch("common product needs a row-reversed left operand and a column-forward right operand")
    if ca.logical_cols != cb.logical_rows or ca.stored_cols != cb.stored_rows:
        raise DimensionMismatch(
            f"inner dimensions disagree: {ca.logical_rows}x{ca.logical_cols} times {cb.logical_rows}x{cb.logical_cols}")


def packed_common_product(ca: CompressedMatrix, cb: CompressedMatrix):
    """gemm.hpp:210-244 with the reference's per-product high part
    (word.hpp:28-30): the m x n float64 accumulators, bit-identical."""
    torch = _torch()
    _check_common_operands(ca, cb)
    if ca.logical_cols > ca.plan.kmax:
        raise PlanMismatch(f"common dimension {ca.logical_cols} exceeds kmax={ca.plan.kmax}")
    out = torch.empty((ca.logical_rows, cb.logical_cols), dtype=torch.float64, device=ca.data.device)
    pl = ca.plan._c()
    _check(lib.qg_packed_common_product(ctypes.byref(pl), _ptr(ca.data), _ptr(cb.data), ca.logical_rows,
                                        cb.logical_cols, ca.logical_cols, _ptr(out), _stream()))
    return out


def reduce_common_entry(acc, plan: CompressionPlan):
    """gemm.hpp:247-250 over a tensor of accumulators -> int32 residues."""
    torch = _torch()
    out = torch.empty(acc.shape, dtype=torch.int32, device=acc.device)
    pl = plan._c()
    _check(lib.qg_reduce_common(ctypes.byref(pl), _ptr(acc), acc.numel(), _ptr(out), _stream()))
    return out


def _as_gpu_plan(plan: Union[CompressionPlan, GpuPlan], k: int) -> GpuPlan:
    return plan if isinstance(plan, GpuPlan) else gpu_plan_from(plan, k)


def mul_common_compressed(a_or_ca, b_or_cb, plan: Optional[Union[CompressionPlan, GpuPlan]] = None):
    """mul_common_compressed, gemm.hpp:254-271, on the FP64 tensor cores.

    (a, b, plan): residue tensors, packed on the device under ``plan``;
    (ca, cb): operands compressed already (their plan is used).
    A GpuPlan (plan_gpu) may cover k > kmax through in-kernel k-blocks.
    Returns int32 C (m x n)."""
    torch = _torch()
    if isinstance(a_or_ca, CompressedMatrix):
        ca, cb = a_or_ca, b_or_cb
        _check_common_operands(ca, cb)
        gp = _as_gpu_plan(plan if plan is not None else ca.plan, ca.logical_cols)
        if gp.balanced:
            raise PlanMismatch("operands packed in the reference layout hold unsigned words; "
                               "use plan_gpu(p, k, balanced=False)")
    else:
        a, b = a_or_ca, b_or_cb
        if a.shape[1] != b.shape[0]:  # check_inner_dims, gemm.hpp:22-27
            raise DimensionMismatch(
                f"inner dimensions disagree: {a.shape[0]}x{a.shape[1]} times {b.shape[0]}x{b.shape[1]}")
        gp = _as_gpu_plan(plan, a.shape[1])
        base = gp.plan
        k = a.shape[1]
        if not isinstance(plan, GpuPlan) and k > base.kmax:  # compress_rows_reversed's check
            raise PlanMismatch(f"common dimension {k} exceeds kmax={base.kmax}")
        if not os.environ.get("QG_FORCE_ROW_LAYOUT"):
            return mul_common_residues(a, b, gp)
        if gp.balanced:  # the row layout holds the reference's unsigned words
            gp = plan_gpu(base.p, k, balanced=False)
            base = gp.plan
            plan = gp
        if isinstance(plan, GpuPlan) and k > base.kmax:
            # blocked plan: pack with a kmax-free plan view (blocks enforce Eq. 3)
            big = dataclasses.replace(base, kmax=max(base.kmax, k))
            ca, cb = compress_rows_reversed(a, big), compress_cols_forward(b, big)
            ca.plan = cb.plan = base
        else:
            ca, cb = compress_rows_reversed(a, base), compress_cols_forward(b, base)
    m, n, k = ca.logical_rows, cb.logical_cols, ca.logical_cols
    out = torch.empty((m, n), dtype=torch.int32, device=ca.data.device)
    g = gp._c()
    _check(lib.qg_mul_common(ctypes.byref(g), _ptr(ca.data), _ptr(cb.data), m, n, k, _ptr(out), n, _stream()))
    return out


def tiled_stage_words(gp: GpuPlan, k: int) -> int:
    out = ctypes.c_uint32()
    g = gp._c()
    _check(lib.qg_tiled_stage_words(ctypes.byref(g), k, ctypes.byref(out)))
    return out.value


def pack_tiled(a, plan: Union[CompressionPlan, GpuPlan], bk: int, operand: str):
    """Tiled packed layout of A ('a': compress_rows_reversed words) or B
    ('b': compress_cols_forward words, transposed) as dense zero-padded
    128 x bk blocks (include/qgemm_b200.h); balanced digits if the GpuPlan says
    so. Returns a flat float64 tensor."""
    torch = _torch()
    _require_cuda(a)
    rows, cols = a.shape
    gp = plan if isinstance(plan, GpuPlan) else GpuPlan(plan, 1, 0, 0)
    plan = gp.plan
    pl = gp._c()
    if operand == "a":
        out = torch.empty(lib.qg_tiled_words(rows, cols, plan.e, bk), dtype=torch.float64, device=a.device)
        _check(lib.qg_pack_a_tiled(ctypes.byref(pl), bk, _ptr(a), _dtype_code(a), rows, cols, cols, _ptr(out), _stream()))
    else:
        out = torch.empty(lib.qg_tiled_words(cols, rows, plan.e, bk), dtype=torch.float64, device=a.device)
        _check(lib.qg_pack_b_tiled(ctypes.byref(pl), bk, _ptr(a), _dtype_code(a), rows, cols, cols, _ptr(out), _stream()))
    return out


def mul_common_residues(a, b, plan: Union[CompressionPlan, GpuPlan]):
    """mul_common_compressed(A, B, plan) on device residues through one ABI
    call (qg_mul_common_compressed): tiled packs into stream-ordered
    workspaces, then the tiled contraction (64x64 tiles with k split over a
    thread-block cluster for small products). Returns int32 C (m x n)."""
    torch = _torch()
    _require_cuda(a, b)
    if a.dtype != b.dtype:
        b = b.to(a.dtype)
    m, k = a.shape
    n = b.shape[1]
    gp = _as_gpu_plan(plan, k)
    out = torch.empty((m, n), dtype=torch.int32, device=a.device)
    g = gp._c()
    _check(lib.qg_mul_common_compressed(ctypes.byref(g), _ptr(a), k, _ptr(b), n, _dtype_code(a), m, k, n,
                                        _ptr(out), n, _stream()))
    return out


def mul_common_tiled(a, b, plan: Union[CompressionPlan, GpuPlan]):
    """mul_common_compressed on residue tensors through the tiled packed
    layout and the tiled DMMA contraction (n must be even)."""
    torch = _torch()
    m, k = a.shape
    n = b.shape[1]
    gp = _as_gpu_plan(plan, k)
    bk = tiled_stage_words(gp, k)
    ca = pack_tiled(a, gp, bk, "a")
    cb = pack_tiled(b, gp, bk, "b")
    out = torch.empty((m, n), dtype=torch.int32, device=a.device)
    g = gp._c()
    _check(lib.qg_mul_common_tiled(ctypes.byref(g), _ptr(ca), _ptr(cb), m, n, k, _ptr(out), n, _stream()))
    return out


def mul_common_repacked(a, b, plan: Union[CompressionPlan, GpuPlan]) -> CompressedMatrix:
    """mul_common_repacked, gemm.hpp:275-280: C reduced and its rows re-packed
    forward in groups of e (ReduceAndCompress, pack.hpp:141-155) under the
    plan's (t, e), fused into the contraction's epilogue
    (qg_mul_common_repacked_compressed: no int32 C in HBM). Under a
    CompressionPlan the words are the reference's bit for bit."""
    torch = _torch()
    _require_cuda(a, b)
    if a.shape[1] != b.shape[0]:  # check_inner_dims, gemm.hpp:22-27
        raise DimensionMismatch(f"inner dimensions disagree: {a.shape[0]}x{a.shape[1]} times {b.shape[0]}x{b.shape[1]}")
    m, k = a.shape
    n = b.shape[1]
    if not isinstance(plan, GpuPlan) and k > plan.kmax:  # compress_rows_reversed's check
        raise PlanMismatch(f"common dimension {k} exceeds kmax={plan.kmax}")
    gp = _as_gpu_plan(plan, k)
    base = gp.plan
    if b.dtype != a.dtype:
        b = b.to(a.dtype)
    a, b = a.contiguous(), b.contiguous()
    H = (n + base.e - 1) // base.e
    out = torch.empty((m, H), dtype=torch.float64, device=a.device)
    g = gp._c()
    _check(lib.qg_mul_common_repacked_compressed(ctypes.byref(g), _ptr(a), k, _ptr(b), n, _dtype_code(a), m, k, n,
                                                 _ptr(out), H, _stream()))
    return CompressedMatrix(m, n, m, H, PackOrientation(PackDirection.Forward, PackAxis.Column, base.e), base, out)


def mul_common_repacked_host(a, b, plan: Union[CompressionPlan, GpuPlan], out=None) -> np.ndarray:
    """mul_common_repacked on host ResidueMatrix data (uint32): m x ceil(n/e)
    float64 words (qg_host_mul_common_repacked[_gpu], pipelined)."""
    a, b = _host_u32(a), _host_u32(b)
    if a.shape[1] != b.shape[0]:
        raise DimensionMismatch(f"inner dimensions disagree: {a.shape} times {b.shape}")
    m, k = a.shape
    n = b.shape[1]
    base = plan.plan if isinstance(plan, GpuPlan) else plan
    cc = np.empty((m, (n + base.e - 1) // base.e), dtype=np.float64) if out is None else out
    vp = ctypes.c_void_p
    if isinstance(plan, GpuPlan):
        g = plan._c()
        _check(lib.qg_host_mul_common_repacked_gpu(ctypes.byref(g), a.ctypes.data_as(vp), b.ctypes.data_as(vp), m, k,
                                                   n, cc.ctypes.data_as(vp)))
    else:
        pl = plan._c()
        _check(lib.qg_host_mul_common_repacked(ctypes.byref(pl), a.ctypes.data_as(vp), b.ctypes.data_as(vp), m, k, n,
                                               cc.ctypes.data_as(vp)))
    return cc


def packed_right_product(a, cb: CompressedMatrix) -> CompressedMatrix:
    """gemm.hpp:285-310: exact A x CB (pre-REDQ words)."""
    return _right(a, cb, redq=False)


def mul_right_compressed(a, cb: CompressedMatrix) -> CompressedMatrix:
    """gemm.hpp:320-335: packed_right_product + redq_in_place, fused. ``a``
    may also be a Forward CompressedMatrix (it is uncompressed first)."""
    if isinstance(a, CompressedMatrix):
        if a.orientation.direction != PackDirection.Forward:
            raise PlanMismatch("left operand must be packed forward to be unpacked")
        a = uncompress(a)
    return _right(a, cb, redq=True)


def _right(a, cb: CompressedMatrix, redq: bool) -> CompressedMatrix:
    torch = _torch()
    if cb.orientation.direction != PackDirection.Forward or cb.orientation.axis != PackAxis.Column:
        raise PlanMismatch("right product needs the right operand packed forward on its columns")
    m, k = a.shape
    if k != cb.logical_rows:
        raise DimensionMismatch(
            f"inner dimensions disagree: {m}x{k} times {cb.logical_rows}x{cb.logical_cols}")
    if k > cb.plan.kmax:
        raise PlanMismatch(f"common dimension {k} exceeds kmax={cb.plan.kmax}")
    ad = a if a.dtype == torch.float64 else a.to(torch.float64)
    ad = ad.contiguous()
    out = torch.empty((m, cb.stored_cols), dtype=torch.float64, device=cb.data.device)
    pl = cb.plan._c()
    fn = lib.qg_mul_right if redq else lib.qg_packed_right_product
    _check(fn(ctypes.byref(pl), _ptr(ad), k, _ptr(cb.data), m, k, cb.logical_cols, _ptr(out), _stream()))
    return CompressedMatrix(m, cb.logical_cols, m, cb.stored_cols, dataclasses.replace(cb.orientation), cb.plan, out)


def redq_in_place(cm: CompressedMatrix) -> None:
    """gemm.hpp:313-316."""
    pl = cm.plan._c()
    _check(lib.qg_redq(ctypes.byref(pl), _ptr(cm.data), cm.data.numel(), _stream()))


def plan_right_gpu(p: int, k: int, n: int) -> GpuPlan:
    """(t, e, k-block in residues) for the mixed variant on the tensor-core path."""
    out = _GpuPlan()
    _check(lib.qg_plan_right_gpu(p, k, n, ctypes.byref(out)))
    return GpuPlan._from(out)


def mul_right_tiled(a, b, plan: Union[CompressionPlan, GpuPlan]) -> CompressedMatrix:
    """mul_right_compressed(A, compress_outer_cols(B, plan)) on residue
    tensors through the tiled layout and the blocked mixed contraction. With a
    CompressionPlan the words equal the reference's bit for bit; a GpuPlan from
    plan_right_gpu may block k past plan.kmax (in-place REDQ between blocks)."""
    torch = _torch()
    _require_cuda(a, b)
    m, k = a.shape
    n = b.shape[1]
    if b.shape[0] != k:
        raise DimensionMismatch(f"inner dimensions disagree: {m}x{k} times {b.shape[0]}x{n}")
    gp = plan if isinstance(plan, GpuPlan) else GpuPlan(plan, k, k, 0)
    pl = gp.plan
    g = gp._c()
    bk = ctypes.c_uint32()
    _check(lib.qg_right_tiled_stage(ctypes.byref(g), k, ctypes.byref(bk)))
    bk = bk.value
    H = (n + pl.e - 1) // pl.e
    kt = -(-k // bk)
    a_t = torch.empty(-(-m // 128) * 128 * kt * bk, dtype=torch.float64, device=a.device)
    bo_t = torch.empty(-(-H // 128) * 128 * kt * bk, dtype=torch.float64, device=a.device)
    c_pl = pl._c()
    if gp.balanced:  # balanced digits: twice the k-block between in-place REDQs
        _check(lib.qg_pack_residues_tiled_bal(pl.p, bk, _ptr(a), _dtype_code(a), m, k, k, _ptr(a_t), _stream()))
        _check(lib.qg_pack_outer_cols_tiled_bal(ctypes.byref(c_pl), bk, _ptr(b), _dtype_code(b), k, n, n, _ptr(bo_t),
                                                _stream()))
    else:
        _check(lib.qg_pack_residues_tiled(bk, _ptr(a), _dtype_code(a), m, k, k, _ptr(a_t), _stream()))
        _check(lib.qg_pack_outer_cols_tiled(ctypes.byref(c_pl), bk, _ptr(b), _dtype_code(b), k, n, n, _ptr(bo_t),
                                            _stream()))
    cc = torch.empty((m, H), dtype=torch.float64, device=a.device)
    _check(lib.qg_mul_right_tiled(ctypes.byref(g), _ptr(a_t), _ptr(bo_t), m, k, n, _ptr(cc), H, _stream()))
    return CompressedMatrix(m, n, m, H, PackOrientation(PackDirection.Forward, PackAxis.Column, pl.e), pl, cc)


# ------------------------------------------- left and full compression
def mul_left_tiled(a, b, plan: Union[CompressionPlan, GpuPlan]) -> CompressedMatrix:
    """mul_left_compressed(compress_outer_rows(A, plan), B), gemm.hpp:340-371,
    on residue tensors: A's outer-row words and B's residues as tiled blocks,
    the REDQ contraction of the mixed variant. ceil(m/e) x n words,
    {Forward, Row, e}; bit-identical to the reference's under a
    CompressionPlan, k-blocked past kmax under a GpuPlan (plan_right_gpu(p, k, m))."""
    torch = _torch()
    _require_cuda(a, b)
    m, k = a.shape
    n = b.shape[1]
    if b.shape[0] != k:
        raise DimensionMismatch(f"inner dimensions disagree: {m}x{k} times {b.shape[0]}x{n}")
    gp = plan if isinstance(plan, GpuPlan) else GpuPlan(plan, k, k, 0)
    pl = gp.plan
    g = gp._c()
    bk = ctypes.c_uint32()
    _check(lib.qg_right_tiled_stage(ctypes.byref(g), k, ctypes.byref(bk)))
    bk = bk.value
    G = (m + pl.e - 1) // pl.e
    kt = -(-k // bk)
    ao_t = torch.empty(-(-G // 128) * 128 * kt * bk, dtype=torch.float64, device=a.device)
    b_t = torch.empty(-(-n // 128) * 128 * kt * bk, dtype=torch.float64, device=a.device)
    c_pl = pl._c()
    if gp.balanced:
        _check(lib.qg_pack_outer_rows_tiled_bal(ctypes.byref(c_pl), bk, _ptr(a), _dtype_code(a), m, k, k, _ptr(ao_t),
                                                _stream()))
        _check(lib.qg_pack_residues_b_tiled_bal(pl.p, bk, _ptr(b), _dtype_code(b), k, n, n, _ptr(b_t), _stream()))
    else:
        _check(lib.qg_pack_outer_rows_tiled(ctypes.byref(c_pl), bk, _ptr(a), _dtype_code(a), m, k, k, _ptr(ao_t),
                                            _stream()))
        _check(lib.qg_pack_residues_b_tiled(bk, _ptr(b), _dtype_code(b), k, n, n, _ptr(b_t), _stream()))
    cc = torch.empty((G, n), dtype=torch.float64, device=a.device)
    _check(lib.qg_mul_left_tiled(ctypes.byref(g), _ptr(ao_t), _ptr(b_t), m, k, n, _ptr(cc), n, _stream()))
    return CompressedMatrix(m, n, G, n, PackOrientation(PackDirection.Forward, PackAxis.Row, pl.e), pl, cc)


def mul_left_compressed(ca, b, plan: Optional[Union[CompressionPlan, GpuPlan]] = None) -> CompressedMatrix:
    """mul_left_compressed(ca, b), gemm.hpp:340-371. ``ca`` is the
    compress_outer_rows matrix (its words are unpacked on the device and
    re-packed into the tiled layout) or a residue tensor with ``plan``."""
    if isinstance(ca, CompressedMatrix):
        if ca.orientation.direction != PackDirection.Forward or ca.orientation.axis != PackAxis.Row:
            raise PlanMismatch("left product needs the left operand packed forward on its rows")
        if ca.logical_cols != b.shape[0]:
            raise DimensionMismatch(f"inner dimensions disagree: {ca.logical_rows}x{ca.logical_cols} "
                                    f"times {b.shape[0]}x{b.shape[1]}")
        if ca.logical_cols > ca.plan.kmax:
            raise PlanMismatch("common dimension exceeds the plan's kmax")
        return mul_left_tiled(uncompress(ca), b, ca.plan)
    if plan is None:
        raise InvalidArgument("a residue operand needs a plan")
    return mul_left_tiled(ca, b, plan)


@dataclasses.dataclass
class FullPlan:
    """FullPlan, plan.hpp:44-57: base.e = (dq+1)(dtheta+1) base-Q digits per
    word, rows of A in dq+1 slots of radix Q, columns of B in dtheta+1 slots of
    radix Theta = 2^theta_exponent = Q^(dq+1)."""

    base: CompressionPlan
    dq: int
    dtheta: int
    theta_exponent: int

    def q_slots(self) -> int:
        return self.dq + 1

    def theta_slots(self) -> int:
        return self.dtheta + 1

    def _c(self) -> _FullPlan:
        return _FullPlan(self.base._c(), self.dq, self.dtheta, self.theta_exponent)

    @staticmethod
    def _from(c: _FullPlan) -> "FullPlan":
        return FullPlan(CompressionPlan._from(c.base), c.dq, c.dtheta, c.theta_exponent)


def plan_full(p: int, k: int, beta: int = 53) -> FullPlan:
    """plan_full(PrimeModulus(p), k, beta), plan.hpp:229-252."""
    out = _FullPlan()
    _check(lib.qg_plan_full(p, k, beta, ctypes.byref(out)))
    return FullPlan._from(out)


def plan_full_gpu(p: int, k: int):
    """(FullPlan, kblock residues) for the full variant on the tensor-core path."""
    out = _FullPlan()
    kb = ctypes.c_uint64()
    _check(lib.qg_plan_full_gpu(p, k, ctypes.byref(out), ctypes.byref(kb)))
    return FullPlan._from(out), kb.value


def mul_full_compressed(a, b, fp: FullPlan, kblock_words: int = 0):
    """mul_full_compressed(A, B, fp), gemm.hpp:377-445, on residue tensors:
    int32 m x n residues of A B mod p. kblock_words = 0 keeps the reference's
    single block (k <= kmax); plan_full_gpu's value blocks k past it."""
    torch = _torch()
    _require_cuda(a, b)
    m, k = a.shape
    n = b.shape[1]
    if b.shape[0] != k:
        raise DimensionMismatch(f"inner dimensions disagree: {m}x{k} times {b.shape[0]}x{n}")
    if fp.base.beta > 53:
        raise PlanMismatch("plan word width exceeds the DoubleWord backend")
    if not kblock_words and k > fp.base.kmax:
        raise PlanMismatch("common dimension exceeds the plan's kmax")
    f = fp._c()
    bk = ctypes.c_uint32()
    _check(lib.qg_full_tiled_stage(ctypes.byref(f), kblock_words, k, ctypes.byref(bk)))
    bk = bk.value
    qs, ts = fp.q_slots(), fp.theta_slots()
    G, H = -(-m // qs), -(-n // ts)
    kt = -(-k // bk)
    ao_t = torch.empty(-(-G // 128) * 128 * kt * bk, dtype=torch.float64, device=a.device)
    bo_t = torch.empty(-(-H // 128) * 128 * kt * bk, dtype=torch.float64, device=a.device)
    pa = _Plan(fp.base.p, fp.base.t, qs - 1, qs, fp.base.beta, fp.base.kmax, 1.0, 0)
    pb = _Plan(fp.base.p, fp.theta_exponent, ts - 1, ts, fp.base.beta, fp.base.kmax, 1.0, 0)
    _check(lib.qg_pack_outer_rows_tiled(ctypes.byref(pa), bk, _ptr(a), _dtype_code(a), m, k, k, _ptr(ao_t), _stream()))
    _check(lib.qg_pack_outer_cols_tiled(ctypes.byref(pb), bk, _ptr(b), _dtype_code(b), k, n, n, _ptr(bo_t), _stream()))
    cc = torch.empty((G, H), dtype=torch.float64, device=a.device)
    _check(lib.qg_mul_full_tiled(ctypes.byref(f), kblock_words, _ptr(ao_t), _ptr(bo_t), m, k, n, _ptr(cc), H,
                                 _stream()))
    c = torch.empty((m, n), dtype=torch.int32, device=a.device)
    _check(lib.qg_uncompress_full(ctypes.byref(f), _ptr(cc), H, m, n, _ptr(c), n, _stream()))
    return c


def extract_coefficients(words, plan: CompressionPlan):
    """extract_coefficient, pack.hpp:78-100, elementwise (float64 CUDA tensor
    -> int32 residues) in the plan's extraction mode."""
    torch = _torch()
    _require_cuda(words)
    w = words if words.dtype == torch.float64 else words.to(torch.float64)
    out = torch.empty(w.shape, dtype=torch.int32, device=w.device)
    pl = plan._c()
    _check(lib.qg_extract_coefficients(ctypes.byref(pl), _ptr(w), w.numel(), _ptr(out), _stream()))
    return out


def reduce_and_compress(words, plan: CompressionPlan) -> CompressedMatrix:
    """reduce_and_compress, pack.hpp:141-155, on every row of a 2-D tensor of
    accumulated words: rows x ceil(cols/e) words, {Forward, Column, e}."""
    torch = _torch()
    _require_cuda(words)
    w = words if words.dtype == torch.float64 else words.to(torch.float64)
    rows, cols = w.shape
    groups = (cols + plan.e - 1) // plan.e
    out = torch.empty((rows, groups), dtype=torch.float64, device=w.device)
    pl = plan._c()
    _check(lib.qg_reduce_and_compress(ctypes.byref(pl), _ptr(w), rows, cols, cols, _ptr(out), groups, _stream()))
    return CompressedMatrix(rows, cols, rows, groups, PackOrientation(PackDirection.Forward, PackAxis.Column, plan.e),
                            plan, out)


def residue_checksum(c) -> int:
    """bench.hpp:43-47: sum of residues mod 2^32."""
    torch = _torch()
    if hasattr(c, "is_cuda"):
        return int(c.to(torch.int64).sum().item()) & 0xFFFFFFFF
    return int(np.asarray(c, dtype=np.uint64).sum()) & 0xFFFFFFFF


# ----------------------------------------------------------------- host data
def _host_u32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint32))


def mul_common_compressed_host(a, b, plan: Union[CompressionPlan, GpuPlan], out=None) -> np.ndarray:
    """mul_common_compressed(A, B, plan) on host ResidueMatrix data
    (uint32 row-major): copies in, runs the kernels, copies C out. A GpuPlan
    (plan_gpu) k-blocks the common dimension past plan.kmax. ``out`` may be a
    preallocated (pinned) uint32 array."""
    a, b = _host_u32(a), _host_u32(b)
    if a.shape[1] != b.shape[0]:
        raise DimensionMismatch(f"inner dimensions disagree: {a.shape} times {b.shape}")
    m, k = a.shape
    n = b.shape[1]
    c = np.empty((m, n), dtype=np.uint32) if out is None else out
    vp = ctypes.c_void_p
    if isinstance(plan, GpuPlan):
        g = plan._c()
        _check(lib.qg_host_mul_common_gpu(ctypes.byref(g), a.ctypes.data_as(vp), b.ctypes.data_as(vp), m, k, n,
                                          c.ctypes.data_as(vp)))
    else:
        pl = plan._c()
        _check(lib.qg_host_mul_common(ctypes.byref(pl), a.ctypes.data_as(vp), b.ctypes.data_as(vp), m, k, n,
                                      c.ctypes.data_as(vp)))
    return c


def mul_common_multi_host(a, b, plan: Union[CompressionPlan, GpuPlan], devices=(0,), out=None) -> np.ndarray:
    """mul_common_compressed on host data over several GPUs of this process
    (qg_host_mul_common_multi): rows of A and C sharded over `devices`, B
    packed once and broadcast as packed words over NCCL."""
    a, b = _host_u32(a), _host_u32(b)
    if a.shape[1] != b.shape[0]:
        raise DimensionMismatch(f"inner dimensions disagree: {a.shape} times {b.shape}")
    m, k = a.shape
    n = b.shape[1]
    gp = _as_gpu_plan(plan, k)
    c = np.empty((m, n), dtype=np.uint32) if out is None else out
    devs = (ctypes.c_int * len(devices))(*devices)
    g = gp._c()
    _check(lib.qg_host_mul_common_multi(ctypes.byref(g), devs, len(devices), a.ctypes.data_as(ctypes.c_void_p),
                                        b.ctypes.data_as(ctypes.c_void_p), m, k, n, c.ctypes.data_as(ctypes.c_void_p)))
    return c


def blocked_accumulate_host(a, b, plan: CompressionPlan, kpanel: int) -> np.ndarray:
    """blocked_accumulate(A, B, plan, kpanel), gemm.hpp:450-489, host data."""
    a, b = _host_u32(a), _host_u32(b)
    if a.shape[1] != b.shape[0]:
        raise DimensionMismatch(f"inner dimensions disagree: {a.shape} times {b.shape}")
    m, k = a.shape
    n = b.shape[1]
    c = np.empty((m, n), dtype=np.uint32)
    pl = plan._c()
    _check(lib.qg_host_blocked_accumulate(ctypes.byref(pl), a.ctypes.data_as(ctypes.c_void_p),
                                          b.ctypes.data_as(ctypes.c_void_p), m, k, n, kpanel,
                                          c.ctypes.data_as(ctypes.c_void_p)))
    return c


def mul_right_compressed_host(a, b, plan: Union[CompressionPlan, GpuPlan], out=None) -> np.ndarray:
    """mul_right_compressed(A, compress_outer_cols(B, plan)) on host data:
    the post-REDQ words, m x ceil(n/e) float64. A GpuPlan (plan_right_gpu)
    blocks k past kmax."""
    a, b = _host_u32(a), _host_u32(b)
    if a.shape[1] != b.shape[0]:
        raise DimensionMismatch(f"inner dimensions disagree: {a.shape} times {b.shape}")
    m, k = a.shape
    n = b.shape[1]
    e = plan.plan.e if isinstance(plan, GpuPlan) else plan.e
    cc = np.empty((m, (n + e - 1) // e), dtype=np.float64) if out is None else out
    fn = lib.qg_host_mul_right_gpu if isinstance(plan, GpuPlan) else lib.qg_host_mul_right
    pl = plan._c()
    _check(fn(ctypes.byref(pl), a.ctypes.data_as(ctypes.c_void_p), b.ctypes.data_as(ctypes.c_void_p),
              m, k, n, cc.ctypes.data_as(ctypes.c_void_p)))
    return cc


def mul_left_compressed_host(a, b, plan: Union[CompressionPlan, GpuPlan], out=None) -> np.ndarray:
    """mul_left_compressed(compress_outer_rows(A, plan), B) on host data: the
    post-REDQ words, ceil(m/e) x n float64. A GpuPlan (plan_right_gpu(p, k,
    m)) blocks k past kmax."""
    a, b = _host_u32(a), _host_u32(b)
    if a.shape[1] != b.shape[0]:
        raise DimensionMismatch(f"inner dimensions disagree: {a.shape} times {b.shape}")
    m, k = a.shape
    n = b.shape[1]
    e = plan.plan.e if isinstance(plan, GpuPlan) else plan.e
    cc = np.empty(((m + e - 1) // e, n), dtype=np.float64) if out is None else out
    fn = lib.qg_host_mul_left_gpu if isinstance(plan, GpuPlan) else lib.qg_host_mul_left
    pl = plan._c()
    _check(fn(ctypes.byref(pl), a.ctypes.data_as(ctypes.c_void_p), b.ctypes.data_as(ctypes.c_void_p),
              m, k, n, cc.ctypes.data_as(ctypes.c_void_p)))
    return cc


def mul_full_compressed_host(a, b, fp: FullPlan, kblock_words: int = 0, out=None) -> np.ndarray:
    """mul_full_compressed(A, B, fp), gemm.hpp:377-445, on host data."""
    a, b = _host_u32(a), _host_u32(b)
    if a.shape[1] != b.shape[0]:
        raise DimensionMismatch(f"inner dimensions disagree: {a.shape} times {b.shape}")
    m, k = a.shape
    n = b.shape[1]
    c = np.empty((m, n), dtype=np.uint32) if out is None else out
    f = fp._c()
    _check(lib.qg_host_mul_full(ctypes.byref(f), kblock_words, a.ctypes.data_as(ctypes.c_void_p),
                                b.ctypes.data_as(ctypes.c_void_p), m, k, n, c.ctypes.data_as(ctypes.c_void_p)))
    return c


# ----------------------------------------------------------------- matrix files
def _check_parse(status: int) -> None:
    if status == 8:  # ParseError carries the reference's message (matrix_io.hpp:27-62)
        raise ParseError(lib.qg_last_error().decode())
    _check(status)


def _adopt(p, rows, cols, data):
    n = rows.value * cols.value
    out = np.ctypeslib.as_array(data, shape=(max(n, 1),))[:n].copy().reshape(rows.value, cols.value)
    lib.qg_free(ctypes.cast(data, ctypes.c_void_p))
    return p.value, out


def parse_matrix(text: str):
    """read_matrix, matrix_io.hpp:27-52: (p, uint32 rows x cols array)."""
    raw = text.encode()
    p, rows, cols, data = ctypes.c_uint32(), ctypes.c_size_t(), ctypes.c_size_t(), ctypes.POINTER(ctypes.c_uint32)()
    _check_parse(lib.qg_parse_matrix(raw, len(raw), ctypes.byref(p), ctypes.byref(rows), ctypes.byref(cols),
                                     ctypes.byref(data)))
    return _adopt(p, rows, cols, data)


def read_matrix_file(path: str):
    """read_matrix_file, matrix_io.hpp:54-62: (p, uint32 array)."""
    p, rows, cols, data = ctypes.c_uint32(), ctypes.c_size_t(), ctypes.c_size_t(), ctypes.POINTER(ctypes.c_uint32)()
    _check_parse(lib.qg_read_matrix_file(os.fsencode(path), ctypes.byref(p), ctypes.byref(rows), ctypes.byref(cols),
                                         ctypes.byref(data)))
    return _adopt(p, rows, cols, data)


def write_matrix_file(path: str, m, p: int) -> None:
    """write_matrix_file, matrix_io.hpp:64-75."""
    m = _host_u32(m)
    rows, cols = m.shape
    _check_parse(lib.qg_write_matrix_file(os.fsencode(path), p, m.ctypes.data_as(ctypes.c_void_p), rows, cols))


CLI_PATH = os.path.join(_HERE, "_lib", "qgemm_b200")


# ----------------------------------------------------------------- Int64Word
class Int64Word:
    """The Int64Word backend (word.hpp:36-54) on the device: packed words are
    uint64 (held bit for bit in int64 tensors), word products wrap modulo
    2^64, plans may use beta up to 63. Same routines as the DoubleWord API."""

    KINDS = {"rows_reversed": 0, "cols_forward": 1, "outer_cols": 2, "outer_rows": 3}

    @staticmethod
    def compress(x, plan: CompressionPlan, kind: str):
        """compress_rows_reversed / cols_forward / outer_cols / outer_rows
        (gemm.hpp:104-178) into uint64 words."""
        torch = _torch()
        _require_cuda(x)
        rows, cols = x.shape
        e = plan.e
        shape = {"rows_reversed": (rows, -(-cols // e)), "cols_forward": (-(-rows // e), cols),
                 "outer_cols": (rows, -(-cols // e)), "outer_rows": (-(-rows // e), cols)}[kind]
        out = torch.empty(shape, dtype=torch.int64, device=x.device)
        fn = {"rows_reversed": lib.qg_compress_rows_reversed_u64, "cols_forward": lib.qg_compress_cols_forward_u64,
              "outer_cols": lib.qg_compress_outer_cols_u64, "outer_rows": lib.qg_compress_outer_rows_u64}[kind]
        pl = plan._c()
        _check(fn(ctypes.byref(pl), _ptr(x), _dtype_code(x), rows, cols, cols, _ptr(out), shape[1], _stream()))
        return out

    @staticmethod
    def packed_common_product(ca, cb, plan: CompressionPlan):
        torch = _torch()
        m, groups = ca.shape
        n = cb.shape[1]
        acc = torch.empty((m, n), dtype=torch.int64, device=ca.device)
        pl = plan._c()
        _check(lib.qg_packed_common_product_u64(ctypes.byref(pl), _ptr(ca), _ptr(cb), m, n, groups, _ptr(acc),
                                                _stream()))
        return acc

    @staticmethod
    def reduce_common(acc, plan: CompressionPlan):
        torch = _torch()
        out = torch.empty(acc.shape, dtype=torch.int32, device=acc.device)
        pl = plan._c()
        _check(lib.qg_reduce_common_u64(ctypes.byref(pl), _ptr(acc), acc.numel(), _ptr(out), _stream()))
        return out

    @staticmethod
    def extract_coefficients(words, plan: CompressionPlan):
        torch = _torch()
        out = torch.empty(words.shape, dtype=torch.int32, device=words.device)
        pl = plan._c()
        _check(lib.qg_extract_coefficients_u64(ctypes.byref(pl), _ptr(words), words.numel(), _ptr(out), _stream()))
        return out

    @staticmethod
    def reduce_and_compress(words, plan: CompressionPlan):
        torch = _torch()
        rows, cols = words.shape
        g = -(-cols // plan.e)
        out = torch.empty((rows, g), dtype=torch.int64, device=words.device)
        pl = plan._c()
        _check(lib.qg_reduce_and_compress_u64(ctypes.byref(pl), _ptr(words), rows, cols, cols, _ptr(out), g, _stream()))
        return out

    @staticmethod
    def redq_in_place(words, plan: CompressionPlan) -> None:
        pl = plan._c()
        _check(lib.qg_redq_u64(ctypes.byref(pl), _ptr(words), words.numel(), _stream()))

    @staticmethod
    def uncompress(words, plan: CompressionPlan, orientation: PackOrientation, logical_rows: int, logical_cols: int):
        torch = _torch()
        out = torch.empty((logical_rows, logical_cols), dtype=torch.int32, device=words.device)
        pl = plan._c()
        o = _Orientation(int(orientation.direction), int(orientation.axis), int(orientation.slots))
        _check(lib.qg_uncompress_u64(ctypes.byref(pl), o, _ptr(words), words.shape[0], words.shape[1], logical_rows,
                                     logical_cols, _ptr(out), _stream()))
        return out

    @staticmethod
    def right_product(a, cbo, plan: CompressionPlan, n: int, redq: bool = True):
        """packed_right_product / mul_right_compressed (gemm.hpp:285-325)."""
        torch = _torch()
        m, k = a.shape
        H = cbo.shape[1]
        cc = torch.empty((m, H), dtype=torch.int64, device=a.device)
        fn = lib.qg_mul_right_u64 if redq else lib.qg_packed_right_product_u64
        pl = plan._c()
        _check(fn(ctypes.byref(pl), _ptr(a), _dtype_code(a), k, _ptr(cbo), m, k, n, _ptr(cc), _stream()))
        return cc

    @staticmethod
    def left_product(ca, b, plan: CompressionPlan, m: int, redq: bool = True):
        """packed_left_product / mul_left_compressed (gemm.hpp:340-371)."""
        torch = _torch()
        G, k = ca.shape
        n = b.shape[1]
        cc = torch.empty((G, n), dtype=torch.int64, device=b.device)
        fn = lib.qg_mul_left_u64 if redq else lib.qg_packed_left_product_u64
        pl = plan._c()
        _check(fn(ctypes.byref(pl), _ptr(ca), _ptr(b), _dtype_code(b), n, m, k, n, _ptr(cc), _stream()))
        return cc

    @staticmethod
    def mul_full_compressed(a, b, fp: FullPlan):
        torch = _torch()
        m, k = a.shape
        n = b.shape[1]
        c = torch.empty((m, n), dtype=torch.int32, device=a.device)
        f = fp._c()
        _check(lib.qg_mul_full_u64(ctypes.byref(f), _ptr(a), _dtype_code(a), _ptr(b), _dtype_code(b), m, k, n, _ptr(c),
                                   n, _stream()))
        return c

    # host data (value semantics)
    @staticmethod
    def mul_common_compressed_host(a, b, plan: CompressionPlan) -> np.ndarray:
        a, b = _host_u32(a), _host_u32(b)
        m, k = a.shape
        n = b.shape[1]
        c = np.empty((m, n), dtype=np.uint32)
        pl = plan._c()
        _check(lib.qg_host_mul_common_i64(ctypes.byref(pl), a.ctypes.data_as(ctypes.c_void_p),
                                          b.ctypes.data_as(ctypes.c_void_p), m, k, n, c.ctypes.data_as(ctypes.c_void_p)))
        return c

    @staticmethod
    def blocked_accumulate_host(a, b, plan: CompressionPlan, kpanel: int) -> np.ndarray:
        a, b = _host_u32(a), _host_u32(b)
        m, k = a.shape
        n = b.shape[1]
        c = np.empty((m, n), dtype=np.uint32)
        pl = plan._c()
        _check(lib.qg_host_blocked_accumulate_i64(ctypes.byref(pl), a.ctypes.data_as(ctypes.c_void_p),
                                                  b.ctypes.data_as(ctypes.c_void_p), m, k, n, kpanel,
                                                  c.ctypes.data_as(ctypes.c_void_p)))
        return c

    @staticmethod
    def mul_right_compressed_host(a, b, plan: CompressionPlan) -> np.ndarray:
        a, b = _host_u32(a), _host_u32(b)
        m, k = a.shape
        n = b.shape[1]
        cc = np.empty((m, -(-n // plan.e)), dtype=np.uint64)
        pl = plan._c()
        _check(lib.qg_host_mul_right_i64(ctypes.byref(pl), a.ctypes.data_as(ctypes.c_void_p),
                                         b.ctypes.data_as(ctypes.c_void_p), m, k, n, cc.ctypes.data_as(ctypes.c_void_p)))
        return cc

    @staticmethod
    def mul_left_compressed_host(a, b, plan: CompressionPlan) -> np.ndarray:
        a, b = _host_u32(a), _host_u32(b)
        m, k = a.shape
        n = b.shape[1]
        cc = np.empty((-(-m // plan.e), n), dtype=np.uint64)
        pl = plan._c()
        _check(lib.qg_host_mul_left_i64(ctypes.byref(pl), a.ctypes.data_as(ctypes.c_void_p),
                                        b.ctypes.data_as(ctypes.c_void_p), m, k, n, cc.ctypes.data_as(ctypes.c_void_p)))
        return cc

    @staticmethod
    def mul_full_compressed_host(a, b, fp: FullPlan) -> np.ndarray:
        a, b = _host_u32(a), _host_u32(b)
        m, k = a.shape
        n = b.shape[1]
        c = np.empty((m, n), dtype=np.uint32)
        f = fp._c()
        _check(lib.qg_host_mul_full_i64(ctypes.byref(f), a.ctypes.data_as(ctypes.c_void_p),
                                        b.ctypes.data_as(ctypes.c_void_p), m, k, n, c.ctypes.data_as(ctypes.c_void_p)))
        return c
