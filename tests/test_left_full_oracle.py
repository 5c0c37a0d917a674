"""Left and full compression (gemm.hpp:340-445) and plan_full (plan.hpp:229-252)
on CPU: the oracle restatement against the reference's own known answers
(test_gemm.cpp:177-229, test_plan.cpp:96-131, acceptance.cpp:258-332) and the
golden vectors the reference produced (tests/golden/golden_left_full.json);
the product's planners (qg_plan_full, qg_plan_full_gpu) against the same."""
import ctypes
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O
import paper_0803_1975_b200 as qg

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden_left_full.json")))
kA = np.array([[1, 2], [0, 1]], np.uint32)
kB = np.array([[2, 0], [1, 1]], np.uint32)
kC = np.array([[1, 2], [1, 1]], np.uint32)


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)


def _plan_tuple(d):
    return (d["p"], d["t"], d["d"], d["e"], d["beta"], d["kmax"], float.fromhex(d["inv_qd_hex"]), d["extraction"])


def _full(d):
    return O.FullPlan(O.Plan(*_plan_tuple(d["base"])), d["dq"], d["dtheta"], d["theta_exponent"])


def _hex_words(h, shape):
    return np.array([int(x, 16) for x in h], dtype=np.uint64).reshape(shape)


def test_left_compression_known_answers():  # test_gemm.cpp:177-199
    plan = O.make_plan(3, 5, 2)
    ca = O.compress_outer_rows(plan, kA)
    assert ca.tolist() == [[1.0, 34.0]]
    cc = O.mul_left_compressed(plan, kA, kB)
    assert cc.tolist() == [[33.0, 34.0]]
    assert np.array_equal(O.uncompress(plan, cc, (0, 0, 2), 2, 2), kC)
    assert np.array_equal(O.uncompress(plan, O.mul_left_compressed(plan, kA, np.eye(2, dtype=np.uint32)),
                                       (0, 0, 2), 2, 2), kA)
    a1, b1 = O.random_residue_matrix(1, 6, 5, 8), O.random_residue_matrix(6, 5, 5, 9)
    p5 = O.plan_packed_axis(5, 6, 1)
    cc1 = O.mul_left_compressed(p5, a1, b1)
    assert np.array_equal(O.uncompress(p5, cc1, (0, 0, p5.e), 1, 5), O.naive_gemm(5, a1, b1))


def test_full_compression_known_answers():  # test_gemm.cpp:201-229
    fp = O.FullPlan(O.make_plan(3, 5, 4), 1, 1, 10)
    assert np.array_equal(O.mul_full_compressed(fp, kA, kB), kC)
    assert not O.mul_full_compressed(fp, np.zeros((2, 2), np.uint32), kB).any()
    a1, b1 = O.random_residue_matrix(1, 7, 3, 5), O.random_residue_matrix(7, 1, 3, 6)
    assert np.array_equal(O.mul_full_compressed(O.plan_full(3, 7), a1, b1), O.naive_gemm(3, a1, b1))
    m, k, n = 9, 10, 8
    fp5 = O.plan_full(5, k)
    a, b = O.random_residue_matrix(m, k, 5, 21), O.random_residue_matrix(k, n, 5, 22)
    before = O.mul_full_compressed(fp5, a, b)
    a[4, 7] = (a[4, 7] + 1) % 5
    after = O.mul_full_compressed(fp5, a, b)
    keep = np.arange(m) != 4
    assert np.array_equal(before[keep], after[keep])
    assert np.array_equal(after, O.naive_gemm(5, a, b))


def test_plan_full_known_answers():  # test_plan.cpp:96-112
    fp = O.plan_full(3, 250)
    assert (fp.base.t, fp.dq + 1, fp.dtheta + 1, fp.theta_exponent, fp.base.e) == (10, 2, 2, 20, 4)
    fp = O.plan_full(3, 7)
    assert (fp.base.t, fp.dq + 1, fp.dtheta + 1) == (5, 3, 3)
    with pytest.raises(O.OracleError):
        O.plan_full(7, 10000)
    for lib_plan in (qg.plan_full(3, 250), qg.plan_full(3, 7)):
        assert lib_plan.theta_exponent == lib_plan.base.t * lib_plan.q_slots()
    with pytest.raises(qg.NoCompression):
        qg.plan_full(7, 10000)


def test_plan_full_consistency_sweep():  # test_plan.cpp:114-131, acceptance.cpp:307-329
    rng = np.random.default_rng(99)
    for _ in range(300):
        p = int(rng.choice([2, 3, 5, 7, 11, 13, 251]))
        k = 1 + int(rng.integers(1 << 16))
        beta = 24 + int(rng.integers(40))
        try:
            fp = qg.plan_full(p, k, beta)
        except qg.NoCompression:
            continue
        qs, ts = fp.q_slots(), fp.theta_slots()
        assert fp.base.t * qs * ts < beta
        assert qs >= 2 and ts >= qs
        assert fp.theta_exponent == fp.base.t * qs
        assert not fp.base.t * qs * (ts + 1) < beta


def test_golden_plan_full():
    for rec in GOLDEN["plan_full"]:
        p, k, beta = rec["args"]
        mine = O.FullPlan()
        st = O.C.qgo_plan_full(p, k, beta, ctypes.byref(mine))
        lib = qg._FullPlan()
        st_lib = qg.lib.qg_plan_full(p, k, beta, ctypes.byref(lib))
        assert st == st_lib == rec["status"], rec["args"]
        if st == 0:
            want = _full(rec["plan"])
            for got in (mine, lib):
                assert tuple(getattr(got.base, f) for f, _ in O.Plan._fields_) == _plan_tuple(rec["plan"]["base"])
                assert (got.dq, got.dtheta, got.theta_exponent) == (want.dq, want.dtheta, want.theta_exponent)


@pytest.mark.parametrize("idx", range(len(GOLDEN["cases"])))
def test_golden_left_full_cases(idx):
    c = GOLDEN["cases"][idx]
    p, m, k, n = c["p"], c["m"], c["k"], c["n"]
    a, b = O.random_residue_matrix(m, k, p, c["seed_a"]), O.random_residue_matrix(k, n, p, c["seed_b"])
    assert hashlib.sha256(a.tobytes()).hexdigest() == c["a_sha"]
    want = O.naive_gemm(p, a, b)
    assert hashlib.sha256(want.tobytes()).hexdigest() == c["c_sha"]
    if "left_plan" in c:
        lp = O.Plan(*_plan_tuple(c["left_plan"]))
        cc = O.mul_left_compressed(lp, a, b)
        assert np.array_equal(bits(cc), _hex_words(c["left_cc"], (-(-m // lp.e), n)))
        assert np.array_equal(O.uncompress(lp, cc, (0, 0, lp.e), m, n), want)
    if "full_plan" in c:
        assert np.array_equal(O.mul_full_compressed(_full(c["full_plan"]), a, b), want)


@pytest.mark.parametrize("p", [2, 3, 5, 7, 11])
def test_full_never_overflows(p):  # acceptance.cpp:258-304 (criterion 6), exact integers
    for seed in range(50):
        r = np.random.default_rng(seed * 31 + p)
        m, k, n = (1 + int(x) for x in r.integers(40, size=3))
        fp = O.plan_full(p, k)
        a, b = O.random_residue_matrix(m, k, p, seed + 1000), O.random_residue_matrix(k, n, p, seed + 2000)
        qs, ts, t = fp.dq + 1, fp.dtheta + 1, fp.base.t
        G, H = -(-m // qs), -(-n // ts)
        wa = [[sum(int(a[g * qs + s, l]) << (t * s) for s in range(min(qs, m - g * qs))) for l in range(k)]
              for g in range(G)]
        wb = [[sum(int(b[l, h * ts + s]) << (fp.theta_exponent * s) for s in range(min(ts, n - h * ts)))
               for h in range(H)] for l in range(k)]
        for g in range(G):
            for h in range(H):
                assert sum(wa[g][l] * wb[l][h] for l in range(k)) < (1 << 53)
        assert np.array_equal(O.mul_full_compressed(fp, a, b), O.naive_gemm(p, a, b))


@pytest.mark.parametrize("p", [2, 3, 5, 7, 11, 13, 251])
@pytest.mark.parametrize("k", [1, 7, 100, 256, 4096, 32768, 100000])
def test_full_gpu_planner_invariants(p, k):
    fp, kb = qg.plan_full_gpu(p, k)
    pl = fp.base
    qs, ts = fp.q_slots(), fp.theta_slots()
    assert pl.e == qs * ts and pl.t * pl.e <= 52
    assert fp.theta_exponent == pl.t * qs
    cap = 52 // pl.t  # word_capacity(t, 53): largest e with t e < 53
    assert qs * qs <= cap < (qs + 1) * (qs + 1) and ts == cap // qs  # plan.hpp:241-242 split
    if kb >= k:
        assert k <= pl.kmax
    else:
        assert (p - 1) + kb * (p - 1) ** 2 < (1 << pl.t)
        assert kb % 4 == 0
