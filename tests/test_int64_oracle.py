"""The Int64Word backend (word.hpp:36-54) in the oracle, pinned to the
reference's own Int64Word instantiations (oracle/_ref) on random shapes and
plans up to beta = 63 (where word products wrap modulo 2^64), plus the
reference's Int64Word known answers (test_pack.cpp / test_gemm.cpp run every
case for both backends) and golden vectors (tests/golden/golden_i64.json)."""
import ctypes
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O

needs_ref = pytest.mark.skipif(O.REF is None, reason="oracle/_ref not built here")
vp = ctypes.c_void_p
GOLDEN_PATH = os.path.join(os.path.dirname(__file__), "golden", "golden_i64.json")
GOLDEN = json.load(open(GOLDEN_PATH)) if os.path.exists(GOLDEN_PATH) else None


def P(a):
    return a.ctypes.data_as(vp)


def o_pack(kind, plan, src):
    rows, cols = src.shape
    fn = [O.C.qgo_compress_rows_reversed_i64, O.C.qgo_compress_cols_forward_i64, O.C.qgo_compress_outer_cols_i64,
          O.C.qgo_compress_outer_rows_i64][kind]
    shape = [(rows, -(-cols // plan.e)), (-(-rows // plan.e), cols), (rows, -(-cols // plan.e)),
             (-(-rows // plan.e), cols)][kind]
    out = np.zeros(shape, np.uint64)
    st = fn(ctypes.byref(plan), P(np.ascontiguousarray(src, np.uint32)), rows, cols, P(out))
    return st, out


def plans(p, k):
    out = []
    for beta in (53, 63):
        pl = O.Plan()
        if O.C.qgo_plan_compression(p, k, beta, 0, ctypes.byref(pl)) == 0:
            out.append(pl)
    return out


@needs_ref
@pytest.mark.parametrize("seed", range(12))
def test_int64_oracle_matches_reference(seed):
    rng = np.random.default_rng(900 + seed)
    p = int(rng.choice([2, 3, 5, 7, 11, 13, 31]))
    m, k, n = (int(x) for x in rng.integers(1, 30, size=3))
    a, b = O.random_residue_matrix(m, k, p, 10 * seed + 1), O.random_residue_matrix(k, n, p, 10 * seed + 2)
    for pl in plans(p, k):
        for kind, src in ((0, a), (1, b), (2, b), (3, a)):
            st, mine = o_pack(kind, pl, src)
            ref = np.zeros_like(mine)
            assert O.REF.qgref_pack_i64(kind, ctypes.byref(pl), P(np.ascontiguousarray(src)), src.shape[0], src.shape[1],
                                        P(ref)) == st
            if st == 0:
                assert np.array_equal(mine, ref), (kind, pl.beta)
        # common product words + C
        K = -(-k // pl.e)
        _, ca = o_pack(0, pl, a)
        _, cb = o_pack(1, pl, b)
        acc = np.zeros((m, n), np.uint64)
        assert O.C.qgo_packed_common_product_i64(ctypes.byref(pl), P(ca), P(cb), m, n, K, P(acc)) == 0
        racc, rc = np.zeros((m, n), np.uint64), np.zeros((m, n), np.uint32)
        assert O.REF.qgref_common_i64(ctypes.byref(pl), P(a), P(b), m, k, n, P(racc), P(rc)) == 0
        assert np.array_equal(acc, racc)
        assert np.array_equal(np.vectorize(lambda w: O.C.qgo_reduce_common_entry_i64(int(w), ctypes.byref(pl)))(acc)
                              .astype(np.uint32), rc)
        assert np.array_equal(rc, O.naive_gemm(p, a, b))
        # right / left: pre-REDQ and post-REDQ words
        rp, lp = O.Plan(), O.Plan()
        for axis_len, which in ((n, "right"), (m, "left")):
            pl2 = O.Plan()
            if O.C.qgo_plan_packed_axis(p, k, axis_len, pl.beta, ctypes.byref(pl2)):
                continue
            if which == "right":
                _, cbo = o_pack(2, pl2, b)
                pre = np.zeros((m, -(-n // pl2.e)), np.uint64)
                assert O.C.qgo_packed_right_product_i64(ctypes.byref(pl2), P(a), P(cbo), m, k, n, P(pre)) == 0
                rpre, rcc = np.zeros_like(pre), np.zeros_like(pre)
                assert O.REF.qgref_right_i64(ctypes.byref(pl2), P(a), P(b), m, k, n, P(rpre), P(rcc)) == 0
            else:
                _, cao = o_pack(3, pl2, a)
                pre = np.zeros((-(-m // pl2.e), n), np.uint64)
                assert O.C.qgo_packed_left_product_i64(ctypes.byref(pl2), P(cao), P(b), m, k, n, P(pre)) == 0
                rpre, rcc = np.zeros_like(pre), np.zeros_like(pre)
                assert O.REF.qgref_left_i64(ctypes.byref(pl2), P(a), P(b), m, k, n, P(rpre), P(rcc)) == 0
            assert np.array_equal(pre, rpre), which
            post = pre.copy()
            assert O.C.qgo_redq_in_place_i64(ctypes.byref(pl2), P(post), post.size) == 0
            assert np.array_equal(post, rcc), which
        # blocked: two panels
        kp = max(1, (k + 1) // 2)
        bp = O.Plan()
        if kp >= 2:
            stb = O.C.qgo_plan_compression(p, kp, 63, 0, ctypes.byref(bp))
        else:
            stb = O.C.qgo_uncompressed_plan(p, 1, 63, ctypes.byref(bp))
        if stb == 0:
            c1, c2 = np.zeros((m, n), np.uint32), np.zeros((m, n), np.uint32)
            assert O.C.qgo_blocked_accumulate_i64(ctypes.byref(bp), P(a), P(b), m, k, n, kp, P(c1)) == 0
            assert O.REF.qgref_blocked_i64(ctypes.byref(bp), P(a), P(b), m, k, n, kp, P(c2)) == 0
            assert np.array_equal(c1, c2) and np.array_equal(c1, O.naive_gemm(p, a, b))
    # full compression at beta 63
    fp = O.FullPlan()
    if O.C.qgo_plan_full(p, k, 63, ctypes.byref(fp)) == 0:
        c1, c2 = np.zeros((m, n), np.uint32), np.zeros((m, n), np.uint32)
        assert O.C.qgo_mul_full_compressed_i64(ctypes.byref(fp), P(a), P(b), m, k, n, P(c1)) == 0
        assert O.REF.qgref_full_i64(ctypes.byref(fp), P(a), P(b), m, k, n, P(c2)) == 0
        assert np.array_equal(c1, c2) and np.array_equal(c1, O.naive_gemm(p, a, b))


@needs_ref
def test_int64_word_routines_match_reference():
    rng = np.random.default_rng(5)
    for p, t, e, beta in [(3, 5, 2, 53), (3, 13, 4, 63), (7, 18, 3, 63), (2, 4, 15, 63), (5, 31, 2, 63), (3, 62, 1, 63)]:
        pl = O.make_plan(p, t, e, beta)
        words = [int(x) for x in rng.integers(0, 2 ** 63, size=300, dtype=np.uint64)]
        words += [int(x) >> int(s) for x, s in zip(rng.integers(0, 2 ** 63, size=300, dtype=np.uint64),
                                                   rng.integers(0, 63, size=300))]
        for w in words:
            out = ctypes.c_uint32()
            assert O.REF.qgref_extract_i64(ctypes.byref(pl), w, ctypes.byref(out)) == 0
            assert O.C.qgo_extract_coefficient_i64(w, ctypes.byref(pl)) == out.value
            r1, r2 = ctypes.c_uint64(), ctypes.c_uint64()
            s1 = O.REF.qgref_redq_i64(ctypes.byref(pl), w, ctypes.byref(r1))
            s2 = O.C.qgo_redq_i64(w, ctypes.byref(pl), ctypes.byref(r2))
            assert s1 == s2 and (s1 or r1.value == r2.value), (w, s1, s2)


def test_int64_known_answers():  # test_pack.cpp / test_gemm.cpp run these for Int64Word too
    kA = np.array([[1, 2], [0, 1]], np.uint32)
    kB = np.array([[2, 0], [1, 1]], np.uint32)
    kC = np.array([[1, 2], [1, 1]], np.uint32)
    plan = O.make_plan(3, 5, 2)
    _, ca = o_pack(0, plan, kA)
    _, cb = o_pack(1, plan, kB)
    acc = np.zeros((2, 2), np.uint64)
    assert O.C.qgo_packed_common_product_i64(ctypes.byref(plan), P(ca), P(cb), 2, 2, 1, P(acc)) == 0
    assert np.array_equal((acc & 31) % 3, kC)
    _, cbo = o_pack(2, plan, kB)
    assert cbo.tolist() == [[2], [33]]  # test_gemm.cpp:150-154
    _, cao = o_pack(3, plan, kA)
    assert cao.tolist() == [[1, 34]]  # test_gemm.cpp:177-181
    pre = np.zeros((1, 2), np.uint64)
    assert O.C.qgo_packed_left_product_i64(ctypes.byref(plan), P(cao), P(kB), 2, 2, 2, P(pre)) == 0
    assert O.C.qgo_redq_in_place_i64(ctypes.byref(plan), P(pre), 2) == 0
    assert pre.tolist() == [[33, 34]]  # test_gemm.cpp:183-185
    w = np.array([1156, 1156, 1156], np.uint64)  # test_pack.cpp:247-255
    out = np.zeros(2, np.uint64)
    assert O.C.qgo_reduce_and_compress_i64(P(w), 3, ctypes.byref(plan), P(out)) == 0
    assert out.tolist() == [33, 1]
    wide = O.make_plan(3, 17, 3, 63)  # test_pack.cpp:263-268: wider than DoubleWord, fine for Int64Word
    _, cw = o_pack(2, wide, np.array([[1, 2]], np.uint32))
    assert cw.tolist() == [[1 + (2 << 17)]]


@pytest.mark.skipif(GOLDEN is None, reason="golden_i64.json not generated")
@pytest.mark.parametrize("idx", range(len(GOLDEN["cases"])) if GOLDEN else [])
def test_int64_golden(idx):
    c = GOLDEN["cases"][idx]
    p, m, k, n = c["p"], c["m"], c["k"], c["n"]
    a, b = O.random_residue_matrix(m, k, p, c["seed_a"]), O.random_residue_matrix(k, n, p, c["seed_b"])
    pl = O.Plan(*[c["plan"][f] for f in ("p", "t", "d", "e", "beta", "kmax")], float.fromhex(c["plan"]["inv_qd_hex"]),
                c["plan"]["extraction"])
    K = -(-k // pl.e)
    _, ca = o_pack(0, pl, a)
    _, cb = o_pack(1, pl, b)
    acc = np.zeros((m, n), np.uint64)
    assert O.C.qgo_packed_common_product_i64(ctypes.byref(pl), P(ca), P(cb), m, n, K, P(acc)) == 0
    assert hashlib.sha256(acc.tobytes()).hexdigest() == c["acc_sha"]
    if "right_cc_sha" in c:
        rp = O.Plan(*[c["right_plan"][f] for f in ("p", "t", "d", "e", "beta", "kmax")],
                    float.fromhex(c["right_plan"]["inv_qd_hex"]), 0)
        _, cbo = o_pack(2, rp, b)
        pre = np.zeros((m, -(-n // rp.e)), np.uint64)
        assert O.C.qgo_packed_right_product_i64(ctypes.byref(rp), P(a), P(cbo), m, k, n, P(pre)) == 0
        assert O.C.qgo_redq_in_place_i64(ctypes.byref(rp), P(pre), pre.size) == 0
        assert hashlib.sha256(pre.tobytes()).hexdigest() == c["right_cc_sha"]
