"""Pin the oracle (oracle/qg_oracle.c, the C restatement) before trusting it:
(1) the known answers of the reference's own tests (proj/tests/*.cpp, README),
(2) golden vectors produced by the reference itself (tests/golden/golden.json),
(3) where oracle/_ref is built, direct comparison with the reference."""
import ctypes
import hashlib
import json
import math
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)


def fwd(v, plan):
    v = np.asarray(v, dtype=np.uint32)
    out = ctypes.c_double()
    st = O.C.qgo_compress_forward(v.ctypes.data_as(ctypes.c_void_p), v.size, ctypes.byref(plan), ctypes.byref(out))
    return st, out.value


def rev(v, plan):
    v = np.asarray(v, dtype=np.uint32)
    out = ctypes.c_double()
    st = O.C.qgo_compress_reverse(v.ctypes.data_as(ctypes.c_void_p), v.size, ctypes.byref(plan), ctypes.byref(out))
    return st, out.value


def extract(w, plan):
    return O.C.qgo_extract_coefficient(float(w), ctypes.byref(plan))


def digits(w, plan):
    d = np.zeros(64, dtype=np.uint64)
    st = O.C.qgo_extract_all(float(w), ctypes.byref(plan), d.ctypes.data_as(ctypes.c_void_p))
    return st, d[: plan.e].tolist()


def redq(w, plan):
    out = ctypes.c_double()
    st = O.C.qgo_redq(float(w), ctypes.byref(plan), ctypes.byref(out))
    return st, out.value


# ------------------------------------------------------------------ test_pack.cpp
def test_forward_packing():  # test_pack.cpp:41-50
    plan = O.make_plan(3, 5, 3)
    assert fwd([1, 2], plan) == (0, 65.0)
    assert fwd([], plan) == (0, 0.0)
    assert fwd([2, 1, 0], plan) == (0, 34.0)
    assert fwd([1, 1, 1, 1], plan)[0] == 3  # SlotOverflow


def test_reversed_packing():  # test_pack.cpp:52-62
    plan2 = O.make_plan(3, 5, 2)
    assert rev([1, 2], plan2) == (0, 34.0)
    assert rev([1], plan2) == (0, 32.0)
    assert rev([1, 2, 1], O.make_plan(3, 5, 3)) == (0, 1089.0)


def test_extraction():  # test_pack.cpp:64-73
    plan = O.make_plan(3, 5, 2)
    assert extract(1156, plan) == 1
    assert extract(0, plan) == 0
    assert extract(2 * (1 << 40), O.make_plan(3, 10, 5)) == 2


def test_digit_splitting():  # test_pack.cpp:75-91
    assert digits(1057, O.make_plan(3, 5, 3)) == (0, [1, 1, 1])
    assert digits(65, O.make_plan(3, 5, 2)) == (0, [1, 2])
    assert digits((1 << 50) - 1, O.make_plan(3, 10, 5)) == (0, [1023] * 5)
    assert digits(1 << 15, O.make_plan(3, 5, 3))[0] == 4  # DigitOverflow


def test_redq_known_answers():  # test_pack.cpp:93-117
    plan = O.make_plan(3, 5, 3)
    assert redq(4423, plan) == (0, 1057.0)
    assert redq(0, plan) == (0, 0.0)
    assert redq(1057, plan) == (0, 1057.0)
    rng = np.random.default_rng(5150)
    for t, e in [(5, 7), (6, 8), (7, 7), (8, 6), (10, 5), (13, 4), (17, 3)]:
        pl = O.make_plan(3, t, e)
        for _ in range(100):
            w = 0
            for s in range(e):
                w |= int(rng.integers(0, 1 << t)) << (t * s)
            st, r = redq(w, pl)
            assert st == 0
            d0, d1 = digits(w, pl)[1], digits(r, pl)[1]
            assert d1 == [x % 3 for x in d0]
            assert redq(r, pl) == (0, r)


def test_reversed_times_forward_dot_product():  # test_pack.cpp:160-185
    plan = O.make_plan(3, 5, 2)
    for a0 in range(3):
        for a1 in range(3):
            for b0 in range(3):
                for b1 in range(3):
                    w = rev([a0, a1], plan)[1] * fwd([b0, b1], plan)[1]
                    assert extract(w, plan) == (a0 * b0 + a1 * b1) % 3


def test_reduce_and_compress():  # test_pack.cpp:247-261
    plan = O.make_plan(3, 5, 2)
    row = np.full(3, 1156.0)
    out = np.zeros(2)
    assert O.C.qgo_reduce_and_compress(row.ctypes.data_as(ctypes.c_void_p), 3, ctypes.byref(plan),
                                       out.ctypes.data_as(ctypes.c_void_p)) == 0
    assert out.tolist() == [33.0, 1.0]


def test_plans_needing_more_bits_are_rejected():  # test_pack.cpp:263-268
    assert fwd([1, 2], O.make_plan(3, 17, 3, 63))[0] == 6  # PlanMismatch for the double backend


def test_accumulated_high_parts_are_exact():  # test_pack.cpp:187-223 with exact integers
    rng = np.random.default_rng(31337)
    for t, e in [(5, 7), (6, 8), (7, 7), (8, 6), (10, 5), (13, 4), (17, 3)]:
        pl = O.make_plan(3, t, e)
        k = 1 + int(rng.integers(0, pl.kmax))
        a = rng.integers(0, 3, size=(1, k)).astype(np.uint32)
        b = rng.integers(0, 3, size=(k, 1)).astype(np.uint32)
        ca, cb = O.compress_rows_reversed(pl, a), O.compress_cols_forward(pl, b)
        acc = O.packed_common_product(pl, ca, cb, k)[0, 0]
        shadow = sum((int(x) * int(y)) >> (t * (e - 1)) for x, y in zip(ca[0], cb[:, 0]))
        assert shadow < (1 << 53) and int(acc) == shadow
        assert (int(acc) & ((1 << t) - 1)) == int((a.astype(np.int64) @ b.astype(np.int64))[0, 0])


# ------------------------------------------------------------------ test_gemm.cpp / acceptance
kA = np.array([[1, 2], [0, 1]], dtype=np.uint32)
kB = np.array([[2, 0], [1, 1]], dtype=np.uint32)
kC = np.array([[1, 2], [1, 1]], dtype=np.uint32)


def test_naive_oracle():  # test_gemm.cpp:36-50, 310-328
    assert np.array_equal(O.naive_gemm(3, kA, kB), kC)
    r = O.random_residue_matrix(5, 4, 3, 11)
    assert np.array_equal(O.naive_gemm(3, np.eye(5, dtype=np.uint32), r), r)
    k = 5000
    c = O.naive_gemm(5, np.full((1, k), 4, np.uint32), np.full((k, 1), 4, np.uint32))
    assert c[0, 0] == (16 * k) % 5


def test_layouts():  # test_gemm.cpp:330-359
    plan = O.make_plan(3, 5, 2)
    assert O.compress_rows_reversed(plan, [[1, 2]]).tolist() == [[34.0]]
    assert O.compress_rows_reversed(plan, [[1]]).tolist() == [[32.0]]
    assert O.compress_cols_forward(plan, [[2], [1]]).tolist() == [[34.0]]
    assert O.compress_cols_forward(plan, np.eye(2, dtype=np.uint32)).tolist() == [[1.0, 32.0]]
    assert O.compress_cols_forward(plan, [[2, 1]]).tolist() == [[2.0, 1.0]]
    with pytest.raises(O.OracleError) as ex:
        O.compress_rows_reversed(plan, np.zeros((1, 8), np.uint32))
    assert ex.value.status == 6


def test_common_product_known_answers():  # test_gemm.cpp:375-397
    plan = O.make_plan(3, 5, 2)
    assert np.array_equal(O.mul_common_compressed(plan, kA, kB), kC)
    p7 = O.plan_compression(7, 4)
    eye = np.eye(4, dtype=np.uint32)
    assert np.array_equal(O.mul_common_compressed(p7, eye, eye), eye)
    for t, e in [(5, 2), (10, 5), (17, 3)]:
        pl = O.make_plan(3, t, e)
        k = pl.kmax
        c = O.mul_common_compressed(pl, np.full((1, k), 2, np.uint32), np.full((k, 1), 2, np.uint32))
        assert c[0, 0] == (k * 4) % 3


def test_right_compression_known_answers():  # test_gemm.cpp:417-443
    plan = O.make_plan(3, 5, 2)
    cbo = O.compress_outer_cols(plan, kB)
    assert cbo.tolist() == [[2.0], [33.0]]
    cc = O.mul_right_compressed(plan, kA, cbo, 2)
    assert np.array_equal(O.uncompress(plan, cc, (0, 1, 2), 2, 2), kC)
    same = O.mul_right_compressed(plan, np.eye(2, dtype=np.uint32), cbo, 2)
    assert np.array_equal(bits(same), bits(cbo))


def test_panel_blocking():  # test_gemm.cpp:503-523
    plan = O.make_plan(3, 5, 2)
    a, b = O.random_residue_matrix(3, 14, 3, 31), O.random_residue_matrix(14, 5, 3, 32)
    assert np.array_equal(O.blocked_accumulate(plan, a, b, 7), O.naive_gemm(3, a, b))
    a2, b2 = O.random_residue_matrix(4, 6, 3, 33), O.random_residue_matrix(6, 4, 3, 34)
    assert np.array_equal(O.blocked_accumulate(plan, a2, b2, 6), O.mul_common_compressed(plan, a2, b2))
    assert np.array_equal(O.blocked_accumulate(O.uncompressed_plan(3, 1), a2, b2, 1), O.naive_gemm(3, a2, b2))
    with pytest.raises(O.OracleError):
        O.blocked_accumulate(plan, a, b, 8)


def test_partial_compression():  # test_gemm.cpp:547-560
    p, m, k, n = 7, 7, 13, 9
    plan = O.plan_compression(p, k)
    assert plan.e == 5
    a, b = O.random_residue_matrix(m, k, p, 41), O.random_residue_matrix(k, n, p, 42)
    want = O.naive_gemm(p, a, b)
    assert np.array_equal(O.mul_common_compressed(plan, a, b), want)
    cc = O.mul_right_compressed(plan, a, O.compress_outer_cols(plan, b), n)
    assert np.array_equal(O.uncompress(plan, cc, (0, 1, plan.e), m, n), want)
    assert np.array_equal(O.blocked_accumulate(O.plan_compression(p, 5), a, b, 5), want)


def test_table1_and_planner():  # acceptance.cpp:91-111, test_plan.cpp:10-46, 186-193
    for k, t, e in [(7, 5, 7), (15, 6, 8), (31, 7, 7), (63, 8, 6), (255, 10, 5), (2047, 13, 4), (32767, 17, 3)]:
        pl = O.plan_compression(3, k)
        assert (pl.t, pl.e) == (t, e)
    pl = O.plan_compression(3, 200)
    assert (pl.t, pl.e, pl.kmax) == (10, 5, 255)
    assert O.plan_compression(3, 200, 53, 1).kmax == 222


def test_bound_edge():  # acceptance.cpp:163-221: p=3, t=17, e=3, k=32767, all-2
    pl = O.make_plan(3, 17, 3)
    k = 32767
    a, b = np.full((1, k), 2, np.uint32), np.full((k, 1), 2, np.uint32)
    acc = O.packed_common_product(pl, O.compress_rows_reversed(pl, a), O.compress_cols_forward(pl, b), k)[0, 0]
    assert acc < 2.0 ** 53
    assert O.C.qgo_reduce_common_entry(acc, ctypes.byref(pl)) == 1


def test_readme_checksum():  # README.md:97-99
    a, b = O.random_residue_matrix(512, 512, 3, 42), O.random_residue_matrix(512, 512, 3, 43)
    c = O.mul_common_compressed(O.plan_compression(3, 512), a, b)
    assert O.residue_checksum(c) == 262622


def test_splitmix_stream():  # prng.hpp:12-29: index i is the (i+1)-th next()
    state, gamma, mask = 99, 0x9E3779B97F4A7C15, (1 << 64) - 1
    for i in range(50):
        state = (state + gamma) & mask
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
        z ^= z >> 31
        assert O.C.qgo_splitmix64_at(99, i) == z


# ------------------------------------------------------------------ golden vectors
def _plan_tuple(d):
    return (d["p"], d["t"], d["d"], d["e"], d["beta"], d["kmax"], float.fromhex(d["inv_qd_hex"]), d["extraction"])


def _opl(d):
    return O.Plan(*_plan_tuple(d))


def test_golden_planners():
    for rec in GOLDEN["plan_compression"]:
        p, k, beta, mode = rec["args"]
        pl = O.Plan()
        st = O.C.qgo_plan_compression(p, k, beta, mode, ctypes.byref(pl))
        assert st == rec["status"], rec["args"]
        if st == 0:
            assert pl.astuple() == _plan_tuple(rec["plan"]), rec["args"]
    for rec in GOLDEN["plan_packed_axis"]:
        pl = O.Plan()
        st = O.C.qgo_plan_packed_axis(*rec["args"], ctypes.byref(pl))
        assert st == rec["status"]
        if st == 0:
            assert pl.astuple() == _plan_tuple(rec["plan"])
    for rec in GOLDEN["uncompressed_plan"]:
        pl = O.Plan()
        assert O.C.qgo_uncompressed_plan(*rec["args"], ctypes.byref(pl)) == rec["status"]
        if rec["status"] == 0:
            assert pl.astuple() == _plan_tuple(rec["plan"])
    for rec in GOLDEN["choose_panel"]:
        assert O.C.qgo_choose_panel(*rec["args"]) == rec["panel"]


def _hex_words(h, shape):
    return np.array([int(x, 16) for x in h], dtype=np.uint64).reshape(shape)


@pytest.mark.parametrize("idx", range(len(GOLDEN["cases"])))
def test_golden_cases(idx):
    c = GOLDEN["cases"][idx]
    p, m, k, n = c["p"], c["m"], c["k"], c["n"]
    a, b = O.random_residue_matrix(m, k, p, c["seed_a"]), O.random_residue_matrix(k, n, p, c["seed_b"])
    assert hashlib.sha256(a.tobytes()).hexdigest() == c["a_sha"]
    assert hashlib.sha256(b.tobytes()).hexdigest() == c["b_sha"]
    want = np.array(c["c"], dtype=np.uint32).reshape(m, n)
    assert np.array_equal(O.naive_gemm(p, a, b), want)
    if "plan" in c:
        pl = _opl(c["plan"])
        K = -(-k // pl.e)
        ca, cb = O.compress_rows_reversed(pl, a), O.compress_cols_forward(pl, b)
        assert np.array_equal(bits(ca), _hex_words(c["ca"], (m, K)))
        assert np.array_equal(bits(cb), _hex_words(c["cb"], (K, n)))
        assert np.array_equal(bits(O.packed_common_product(pl, ca, cb, k)), _hex_words(c["acc"], (m, n)))
        assert np.array_equal(O.mul_common_compressed(pl, a, b), want)
    if "right_plan" in c:
        rp = _opl(c["right_plan"])
        H = -(-n // rp.e)
        cbo = O.compress_outer_cols(rp, b)
        assert np.array_equal(bits(cbo), _hex_words(c["cbo"], (k, H)))
        assert np.array_equal(bits(O.mul_right_compressed(rp, a, cbo, n)), _hex_words(c["cc"], (m, H)))
        assert np.array_equal(bits(O.compress_outer_rows(rp, a)), _hex_words(c["cao"], (-(-m // rp.e), k)))
    if "blocked" in c:
        bl = c["blocked"]
        assert np.array_equal(O.blocked_accumulate(_opl(bl["plan"]), a, b, bl["kpanel"]), want)


@pytest.mark.parametrize("name", ["config1", "config3", "config2"])
def test_golden_configs_oracle(name):
    g = GOLDEN["configs"][name]
    p, m, k, n = g["p"], g["m"], g["k"], g["n"]
    a, b = O.random_residue_matrix(m, k, p, 42), O.random_residue_matrix(k, n, p, 43)
    c = O.mul_common_compressed(_opl(g["plan"]), a, b)
    assert O.residue_checksum(c) == g["checksum"]
    assert hashlib.sha256(c.astype(np.uint8).tobytes()).hexdigest() == g["sha256_u8"]


# ------------------------------------------------------------------ direct vs the reference
needs_ref = pytest.mark.skipif(O.REF is None, reason="oracle/_ref not built here")


@needs_ref
def test_oracle_matches_reference_random_sweep():
    rng = np.random.default_rng(77)
    vp = ctypes.c_void_p
    for trial in range(60):
        p = int(rng.choice([2, 3, 5, 7, 11, 13]))
        m, k, n = (int(x) for x in rng.integers(1, 40, size=3))
        a, b = O.random_residue_matrix(m, k, p, 7 * trial), O.random_residue_matrix(k, n, p, 7 * trial + 1)
        pl = O.Plan()
        if O.REF.qgref_plan_compression(p, k, 53, 0, ctypes.byref(pl)) == 0:
            acc = np.empty((m, n))
            assert O.REF.qgref_packed_common_product(ctypes.byref(pl), a.ctypes.data_as(vp), b.ctypes.data_as(vp),
                                                     m, k, n, acc.ctypes.data_as(vp)) == 0
            mine = O.packed_common_product(pl, O.compress_rows_reversed(pl, a), O.compress_cols_forward(pl, b), k)
            assert np.array_equal(bits(mine), bits(acc))
        c = np.empty((m, n), np.uint32)
        O.REF.qgref_naive_gemm(p, a.ctypes.data_as(vp), b.ctypes.data_as(vp), m, k, n, c.ctypes.data_as(vp))
        assert np.array_equal(O.naive_gemm(p, a, b), c)
        # scalar routines on random words
        for _ in range(20):
            w = float(int(rng.integers(0, 1 << 52)))
            if O.REF.qgref_plan_compression(p, max(k, 2), 53, 0, ctypes.byref(pl)) == 0:
                r1 = ctypes.c_double()
                s1 = O.REF.qgref_redq(ctypes.byref(pl), w, ctypes.byref(r1))
                s2, r2 = redq(w, pl)
                assert s1 == s2 and (s1 or r1.value == r2)
                u = ctypes.c_uint32()
                O.REF.qgref_extract_coefficient(ctypes.byref(pl), w, ctypes.byref(u))
                assert u.value == extract(w, pl)
