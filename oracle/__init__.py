"""oracle — CPU checkers for the compressed modular GEMM. TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package. The product
(paper_0803_1975_b200) never imports it and has no CPU fallback.

* ``C``   — oracle/_build/libqg_oracle.so: the plain-C restatement of the
            reference algorithm (qg_oracle.c, every routine cites the
            reference file:line it follows).
* ``REF`` — oracle/_ref/libqgref.so: the unmodified reference headers
            (/root/reference/proj/include) compiled behind a C ABI
            (ref_harness.cpp). Present wherever it was built (it travels to
            the GPU box with the snapshot); None otherwise.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libqg_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libqgref.so")


class Plan(ctypes.Structure):
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

    def astuple(self):
        return (self.p, self.t, self.d, self.e, self.beta, self.kmax, self.inv_qd, self.extraction)


class FullPlan(ctypes.Structure):
    _fields_ = [("base", Plan), ("dq", ctypes.c_int32), ("dtheta", ctypes.c_int32), ("theta_exponent", ctypes.c_int32)]


class Orientation(ctypes.Structure):
    _fields_ = [("direction", ctypes.c_int32), ("axis", ctypes.c_int32), ("slots", ctypes.c_int32)]


def build(quiet: bool = True) -> None:
    """make -C oracle (the C restatement; the reference harness only where
    /root/reference exists)."""
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/include"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _load_c():
    if not os.path.exists(ORACLE_SO):
        build()
    lib = ctypes.CDLL(ORACLE_SO)
    P, vp, sz, u32, u64, i32 = ctypes.POINTER, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
    sig = {
        "qgo_plan_compression": ([u32, u64, i32, i32, P(Plan)], i32),
        "qgo_uncompressed_plan": ([u32, u64, i32, P(Plan)], i32),
        "qgo_plan_packed_axis": ([u32, u64, u64, i32, P(Plan)], i32),
        "qgo_make_plan": ([u32, i32, i32, i32, P(Plan)], i32),
        "qgo_choose_panel": ([u32, u64, i32], u64),
        "qgo_splitmix64_at": ([u64, u64], u64),
        "qgo_random_residue_matrix": ([sz, sz, u32, u64, vp], None),
        "qgo_random_residue_rows": ([sz, sz, sz, u32, u64, vp], None),
        "qgo_compress_forward": ([vp, sz, P(Plan), P(ctypes.c_double)], i32),
        "qgo_compress_reverse": ([vp, sz, P(Plan), P(ctypes.c_double)], i32),
        "qgo_extract_coefficient": ([ctypes.c_double, P(Plan)], u32),
        "qgo_extract_all": ([ctypes.c_double, P(Plan), vp], i32),
        "qgo_redq": ([ctypes.c_double, P(Plan), P(ctypes.c_double)], i32),
        "qgo_reduce_and_compress": ([vp, sz, P(Plan), vp], i32),
        "qgo_compress_rows_reversed": ([P(Plan), vp, sz, sz, vp], i32),
        "qgo_compress_cols_forward": ([P(Plan), vp, sz, sz, vp], i32),
        "qgo_compress_outer_cols": ([P(Plan), vp, sz, sz, vp], i32),
        "qgo_compress_outer_rows": ([P(Plan), vp, sz, sz, vp], i32),
        "qgo_uncompress": ([P(Plan), Orientation, vp, sz, sz, sz, sz, vp], i32),
        "qgo_packed_common_product": ([P(Plan), vp, vp, sz, sz, sz, sz, vp, i32], i32),
        "qgo_reduce_common_entry": ([ctypes.c_double, P(Plan)], u32),
        "qgo_mul_common_compressed": ([P(Plan), vp, vp, sz, sz, sz, vp, i32], i32),
        "qgo_mul_common_repacked": ([P(Plan), vp, vp, sz, sz, sz, vp, i32], i32),
        "qgo_packed_right_product": ([P(Plan), vp, vp, sz, sz, sz, vp, i32], i32),
        "qgo_redq_in_place": ([P(Plan), vp, sz], i32),
        "qgo_mul_right_compressed": ([P(Plan), vp, vp, sz, sz, sz, vp, i32], i32),
        "qgo_blocked_accumulate": ([P(Plan), vp, vp, sz, sz, sz, sz, vp, i32], i32),
        "qgo_plan_full": ([u32, u64, i32, P(FullPlan)], i32),
        "qgo_packed_left_product": ([P(Plan), vp, vp, sz, sz, sz, vp, i32], i32),
        "qgo_mul_left_compressed": ([P(Plan), vp, vp, sz, sz, sz, vp, i32], i32),
        "qgo_mul_full_compressed": ([P(FullPlan), vp, vp, sz, sz, sz, vp], i32),
        "qgo_compress_rows_reversed_i64": ([P(Plan), vp, sz, sz, vp], i32),
        "qgo_compress_cols_forward_i64": ([P(Plan), vp, sz, sz, vp], i32),
        "qgo_compress_outer_cols_i64": ([P(Plan), vp, sz, sz, vp], i32),
        "qgo_compress_outer_rows_i64": ([P(Plan), vp, sz, sz, vp], i32),
        "qgo_packed_common_product_i64": ([P(Plan), vp, vp, sz, sz, sz, vp], i32),
        "qgo_reduce_common_entry_i64": ([u64, P(Plan)], u32),
        "qgo_extract_coefficient_i64": ([u64, P(Plan)], u32),
        "qgo_redq_i64": ([u64, P(Plan), P(u64)], i32),
        "qgo_redq_in_place_i64": ([P(Plan), vp, sz], i32),
        "qgo_uncompress_i64": ([P(Plan), Orientation, vp, sz, sz, sz, sz, vp], i32),
        "qgo_packed_right_product_i64": ([P(Plan), vp, vp, sz, sz, sz, vp], i32),
        "qgo_packed_left_product_i64": ([P(Plan), vp, vp, sz, sz, sz, vp], i32),
        "qgo_mul_full_compressed_i64": ([P(FullPlan), vp, vp, sz, sz, sz, vp], i32),
        "qgo_blocked_accumulate_i64": ([P(Plan), vp, vp, sz, sz, sz, sz, vp], i32),
        "qgo_reduce_and_compress_i64": ([vp, sz, P(Plan), vp], i32),
        "qgo_naive_gemm": ([u32, vp, vp, sz, sz, sz, vp, i32], i32),
        "qgo_residue_checksum": ([vp, sz], u32),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


def _load_ref():
    if not os.path.exists(REF_SO):
        if os.path.isdir("/root/reference/proj/include"):
            build()
        if not os.path.exists(REF_SO):
            return None
    lib = ctypes.CDLL(REF_SO)
    P, vp, sz, u32, u64, i32 = ctypes.POINTER, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
    dp = P(ctypes.c_double)
    sig = {
        "qgref_plan_compression": ([u32, u64, i32, i32, P(Plan)], i32),
        "qgref_uncompressed_plan": ([u32, u64, i32, P(Plan)], i32),
        "qgref_plan_packed_axis": ([u32, u64, u64, i32, P(Plan)], i32),
        "qgref_choose_panel": ([u32, u64, i32, P(u64)], i32),
        "qgref_random_residue_matrix": ([sz, sz, u32, u64, vp], None),
        "qgref_compress_forward": ([P(Plan), vp, sz, dp], i32),
        "qgref_compress_reverse": ([P(Plan), vp, sz, dp], i32),
        "qgref_extract_coefficient": ([P(Plan), ctypes.c_double, P(u32)], i32),
        "qgref_extract_all": ([P(Plan), ctypes.c_double, vp], i32),
        "qgref_redq": ([P(Plan), ctypes.c_double, dp], i32),
        "qgref_compress_rows_reversed": ([P(Plan), vp, sz, sz, vp], i32),
        "qgref_compress_cols_forward": ([P(Plan), vp, sz, sz, vp], i32),
        "qgref_compress_outer_cols": ([P(Plan), vp, sz, sz, vp], i32),
        "qgref_compress_outer_rows": ([P(Plan), vp, sz, sz, vp], i32),
        "qgref_packed_common_product": ([P(Plan), vp, vp, sz, sz, sz, vp], i32),
        "qgref_mul_common": ([P(Plan), vp, vp, sz, sz, sz, vp, i32, dp, dp], i32),
        "qgref_cb_create": ([P(Plan), vp, sz, sz, dp], vp),
        "qgref_cb_free": ([vp], None),
        "qgref_mul_common_cb": ([P(Plan), vp, vp, sz, sz, vp, i32, dp], i32),
        "qgref_mul_right": ([P(Plan), vp, vp, sz, sz, sz, vp, vp, i32, dp, dp], i32),
        "qgref_blocked_accumulate": ([P(Plan), vp, vp, sz, sz, sz, sz, vp], i32),
        "qgref_plan_full": ([u32, u64, i32, P(FullPlan)], i32),
        "qgref_parse_matrix": ([ctypes.c_char_p, sz, P(u32), P(sz), P(sz), vp, sz, ctypes.c_char_p, sz], i32),
        "qgref_write_matrix": ([vp, sz, sz, u32, ctypes.c_char_p, sz], sz),
        "qgref_mul_left": ([P(Plan), vp, vp, sz, sz, sz, vp], i32),
        "qgref_mul_full": ([P(FullPlan), vp, vp, sz, sz, sz, vp], i32),
        "qgref_pack_i64": ([i32, P(Plan), vp, sz, sz, vp], i32),
        "qgref_common_i64": ([P(Plan), vp, vp, sz, sz, sz, vp, vp], i32),
        "qgref_right_i64": ([P(Plan), vp, vp, sz, sz, sz, vp, vp], i32),
        "qgref_left_i64": ([P(Plan), vp, vp, sz, sz, sz, vp, vp], i32),
        "qgref_full_i64": ([P(FullPlan), vp, vp, sz, sz, sz, vp], i32),
        "qgref_blocked_i64": ([P(Plan), vp, vp, sz, sz, sz, sz, vp], i32),
        "qgref_extract_i64": ([P(Plan), u64, P(u32)], i32),
        "qgref_redq_i64": ([P(Plan), u64, P(u64)], i32),
        "qgref_naive_gemm": ([u32, vp, vp, sz, sz, sz, vp], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


C = _load_c()
REF = _load_ref()


class OracleError(RuntimeError):
    def __init__(self, status):
        super().__init__(f"oracle status {status}")
        self.status = status


def _ok(st):
    if st:
        raise OracleError(st)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _u32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


def threads() -> int:
    return max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1)


# ---------------------------------------------------------------- C restatement
def plan_compression(p, k, beta=53, mode=0) -> Plan:
    pl = Plan()
    _ok(C.qgo_plan_compression(p, k, beta, mode, ctypes.byref(pl)))
    return pl


def uncompressed_plan(p, k, beta=53) -> Plan:
    pl = Plan()
    _ok(C.qgo_uncompressed_plan(p, k, beta, ctypes.byref(pl)))
    return pl


def plan_packed_axis(p, k, axis, beta=53) -> Plan:
    pl = Plan()
    _ok(C.qgo_plan_packed_axis(p, k, axis, beta, ctypes.byref(pl)))
    return pl


def make_plan(p, t, e, beta=53) -> Plan:
    pl = Plan()
    _ok(C.qgo_make_plan(p, t, e, beta, ctypes.byref(pl)))
    return pl


def plan_of(x) -> Plan:
    """Oracle Plan from any object with the CompressionPlan fields."""
    if isinstance(x, Plan):
        return x
    return Plan(x.p, x.t, x.d, x.e, x.beta, x.kmax, x.inv_qd, getattr(x, "extraction", 0))


def random_residue_matrix(rows, cols, p, seed, row0=0) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.uint32)
    C.qgo_random_residue_rows(row0, rows, cols, p, seed, _p(out))
    return out


def compress_rows_reversed(plan, a) -> np.ndarray:
    a = _u32(a)
    m, k = a.shape
    out = np.empty((m, -(-k // plan.e)), dtype=np.float64)
    _ok(C.qgo_compress_rows_reversed(ctypes.byref(plan_of(plan)), _p(a), m, k, _p(out)))
    return out


def compress_cols_forward(plan, b) -> np.ndarray:
    b = _u32(b)
    k, n = b.shape
    out = np.empty((-(-k // plan.e), n), dtype=np.float64)
    _ok(C.qgo_compress_cols_forward(ctypes.byref(plan_of(plan)), _p(b), k, n, _p(out)))
    return out


def compress_outer_cols(plan, b) -> np.ndarray:
    b = _u32(b)
    k, n = b.shape
    out = np.empty((k, -(-n // plan.e)), dtype=np.float64)
    _ok(C.qgo_compress_outer_cols(ctypes.byref(plan_of(plan)), _p(b), k, n, _p(out)))
    return out


def compress_outer_rows(plan, a) -> np.ndarray:
    a = _u32(a)
    m, k = a.shape
    out = np.empty((-(-m // plan.e), k), dtype=np.float64)
    _ok(C.qgo_compress_outer_rows(ctypes.byref(plan_of(plan)), _p(a), m, k, _p(out)))
    return out


def packed_common_product(plan, ca, cb, k) -> np.ndarray:
    ca, cb = np.ascontiguousarray(ca, np.float64), np.ascontiguousarray(cb, np.float64)
    m, groups = ca.shape
    n = cb.shape[1]
    out = np.empty((m, n), dtype=np.float64)
    _ok(C.qgo_packed_common_product(ctypes.byref(plan_of(plan)), _p(ca), _p(cb), m, n, groups, k, _p(out), threads()))
    return out


def mul_common_compressed(plan, a, b) -> np.ndarray:
    a, b = _u32(a), _u32(b)
    m, k = a.shape
    n = b.shape[1]
    c = np.empty((m, n), dtype=np.uint32)
    _ok(C.qgo_mul_common_compressed(ctypes.byref(plan_of(plan)), _p(a), _p(b), m, k, n, _p(c), threads()))
    return c


def mul_common_repacked(plan, a, b) -> np.ndarray:
    a, b = _u32(a), _u32(b)
    m, k = a.shape
    n = b.shape[1]
    cc = np.empty((m, -(-n // plan.e)), dtype=np.float64)
    _ok(C.qgo_mul_common_repacked(ctypes.byref(plan_of(plan)), _p(a), _p(b), m, k, n, _p(cc), threads()))
    return cc


def packed_right_product(plan, a, cbo, n) -> np.ndarray:
    a = _u32(a)
    cbo = np.ascontiguousarray(cbo, np.float64)
    m, k = a.shape
    cc = np.empty((m, -(-n // plan.e)), dtype=np.float64)
    _ok(C.qgo_packed_right_product(ctypes.byref(plan_of(plan)), _p(a), _p(cbo), m, k, n, _p(cc), threads()))
    return cc


def mul_right_compressed(plan, a, cbo, n) -> np.ndarray:
    a = _u32(a)
    cbo = np.ascontiguousarray(cbo, np.float64)
    m, k = a.shape
    cc = np.empty((m, -(-n // plan.e)), dtype=np.float64)
    _ok(C.qgo_mul_right_compressed(ctypes.byref(plan_of(plan)), _p(a), _p(cbo), m, k, n, _p(cc), threads()))
    return cc


def redq_words(plan, words) -> np.ndarray:
    w = np.array(words, dtype=np.float64, copy=True)
    _ok(C.qgo_redq_in_place(ctypes.byref(plan_of(plan)), _p(w), w.size))
    return w


def uncompress(plan, words, orientation, logical_rows, logical_cols) -> np.ndarray:
    w = np.ascontiguousarray(words, np.float64)
    out = np.empty((logical_rows, logical_cols), dtype=np.uint32)
    o = Orientation(*orientation)
    _ok(C.qgo_uncompress(ctypes.byref(plan_of(plan)), o, _p(w), w.shape[0], w.shape[1], logical_rows, logical_cols, _p(out)))
    return out


def blocked_accumulate(plan, a, b, kpanel) -> np.ndarray:
    a, b = _u32(a), _u32(b)
    m, k = a.shape
    n = b.shape[1]
    c = np.empty((m, n), dtype=np.uint32)
    _ok(C.qgo_blocked_accumulate(ctypes.byref(plan_of(plan)), _p(a), _p(b), m, k, n, kpanel, _p(c), threads()))
    return c


def plan_full(p, k, beta=53) -> FullPlan:
    fp = FullPlan()
    _ok(C.qgo_plan_full(p, k, beta, ctypes.byref(fp)))
    return fp


def mul_left_compressed(plan, a, b) -> np.ndarray:
    """mul_left_compressed(compress_outer_rows(A), B): ceil(m/e) x n post-REDQ words."""
    a, b = _u32(a), _u32(b)
    m, k = a.shape
    n = b.shape[1]
    ca = compress_outer_rows(plan, a)
    cc = np.empty((-(-m // plan.e), n), dtype=np.float64)
    _ok(C.qgo_mul_left_compressed(ctypes.byref(plan_of(plan)), _p(ca), _p(b), m, k, n, _p(cc), threads()))
    return cc


def mul_full_compressed(fp, a, b) -> np.ndarray:
    a, b = _u32(a), _u32(b)
    m, k = a.shape
    n = b.shape[1]
    c = np.empty((m, n), dtype=np.uint32)
    _ok(C.qgo_mul_full_compressed(ctypes.byref(fp), _p(a), _p(b), m, k, n, _p(c)))
    return c


def naive_gemm(p, a, b, nthreads=None) -> np.ndarray:
    a, b = _u32(a), _u32(b)
    m, k = a.shape
    n = b.shape[1]
    c = np.empty((m, n), dtype=np.uint32)
    _ok(C.qgo_naive_gemm(p, _p(a), _p(b), m, k, n, _p(c), nthreads or threads()))
    return c


def residue_checksum(c) -> int:
    c = _u32(c)
    return int(C.qgo_residue_checksum(_p(c), c.size))
