"""GPU parity of the Int64Word backend (word.hpp:36-54): uint64 words,
wrapping products, beta = 63 plans. Device results against the oracle's
Int64Word restatement (pinned to the reference in tests/test_int64_oracle.py)
and the reference's golden vectors (tests/golden/golden_i64.json), bit for
bit (words compared as raw uint64)."""
import ctypes
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden_i64.json")))
vp = ctypes.c_void_p


def P(a):
    return a.ctypes.data_as(vp)


def u64(t):
    return t.cpu().numpy().view(np.uint64)


def dev(torch, x, cuda, dtype=np.float64):
    return torch.from_numpy(np.ascontiguousarray(x).astype(dtype)).to(cuda)


def qplan(qg, d):
    return qg.CompressionPlan(d["p"], d["t"], d["d"], d["e"], d["beta"], d["kmax"], float.fromhex(d["inv_qd_hex"]),
                              d["extraction"])


def oplan(orc, d):
    return orc.Plan(d["p"], d["t"], d["d"], d["e"], d["beta"], d["kmax"], float.fromhex(d["inv_qd_hex"]), d["extraction"])


def o_pack(orc, kind, pl, src):
    rows, cols = src.shape
    fn = [orc.C.qgo_compress_rows_reversed_i64, orc.C.qgo_compress_cols_forward_i64, orc.C.qgo_compress_outer_cols_i64,
          orc.C.qgo_compress_outer_rows_i64][kind]
    shape = [(rows, -(-cols // pl.e)), (-(-rows // pl.e), cols), (rows, -(-cols // pl.e)), (-(-rows // pl.e), cols)][kind]
    out = np.zeros(shape, np.uint64)
    assert fn(ctypes.byref(pl), P(np.ascontiguousarray(src, np.uint32)), rows, cols, P(out)) == 0
    return out


@pytest.mark.parametrize("idx", range(len(GOLDEN["cases"])))
def test_int64_golden_gpu(qg, orc, cuda, idx):
    import torch

    c = GOLDEN["cases"][idx]
    p, m, k, n = c["p"], c["m"], c["k"], c["n"]
    a, b = orc.random_residue_matrix(m, k, p, c["seed_a"]), orc.random_residue_matrix(k, n, p, c["seed_b"])
    ad, bd = dev(torch, a, cuda), dev(torch, b, cuda, np.int32)
    W = qg.Int64Word
    pl, opl = qplan(qg, c["plan"]), oplan(orc, c["plan"])
    ca = W.compress(ad, pl, "rows_reversed")
    cb = W.compress(bd, pl, "cols_forward")
    assert hashlib.sha256(u64(ca).tobytes()).hexdigest() == c["ca_sha"]
    assert np.array_equal(u64(cb), o_pack(orc, 1, opl, b))
    acc = W.packed_common_product(ca, cb, pl)
    assert hashlib.sha256(u64(acc).tobytes()).hexdigest() == c["acc_sha"]
    cc = W.reduce_common(acc, pl).cpu().numpy().astype(np.uint32)
    assert hashlib.sha256(cc.tobytes()).hexdigest() == c["c_sha"]
    assert np.array_equal(W.mul_common_compressed_host(a, b, pl), cc)
    if "right_plan" in c:
        rp = qplan(qg, c["right_plan"])
        cbo = W.compress(bd, rp, "outer_cols")
        pre = W.right_product(ad, cbo, rp, n, redq=False)
        assert hashlib.sha256(u64(pre).tobytes()).hexdigest() == c["right_pre_sha"]
        post = W.right_product(ad, cbo, rp, n)
        assert hashlib.sha256(u64(post).tobytes()).hexdigest() == c["right_cc_sha"]
        assert hashlib.sha256(W.mul_right_compressed_host(a, b, rp).tobytes()).hexdigest() == c["right_cc_sha"]
        un = W.uncompress(post, rp, qg.PackOrientation(0, 1, rp.e), m, n).cpu().numpy().astype(np.uint32)
        assert np.array_equal(un, cc)
    if "left_plan" in c:
        lp = qplan(qg, c["left_plan"])
        cao = W.compress(ad, lp, "outer_rows")
        pre = W.left_product(cao, bd, lp, m, redq=False)
        assert hashlib.sha256(u64(pre).tobytes()).hexdigest() == c["left_pre_sha"]
        post = W.left_product(cao, bd, lp, m)
        assert hashlib.sha256(u64(post).tobytes()).hexdigest() == c["left_cc_sha"]
        assert hashlib.sha256(W.mul_left_compressed_host(a, b, lp).tobytes()).hexdigest() == c["left_cc_sha"]
    if "full_plan" in c:
        d = c["full_plan"]
        fp = qg.FullPlan(qplan(qg, d["base"]), d["dq"], d["dtheta"], d["theta_exponent"])
        assert np.array_equal(W.mul_full_compressed(ad, bd, fp).cpu().numpy().astype(np.uint32), cc)
        assert np.array_equal(W.mul_full_compressed_host(a, b, fp), cc)
    if "blocked" in c:
        bl = c["blocked"]
        assert np.array_equal(W.blocked_accumulate_host(a, b, qplan(qg, bl["plan"]), bl["kpanel"]), cc)


@pytest.mark.parametrize("p,t,e", [(3, 5, 2), (3, 13, 4), (7, 18, 3), (2, 4, 15), (5, 31, 2), (3, 62, 1), (3, 9, 6)])
def test_int64_word_routines(qg, orc, cuda, p, t, e):
    """extract_coefficient / redq / reduce_and_compress on arbitrary uint64 words."""
    import torch

    W = qg.Int64Word
    pl, opl = qg.make_plan(p, t, e, 63), orc.make_plan(p, t, e, 63)
    rng = np.random.default_rng(t * 7 + e)
    words = rng.integers(0, 2 ** 63, size=4096, dtype=np.uint64) >> rng.integers(0, 63, size=4096).astype(np.uint64)
    wd = torch.from_numpy(words.view(np.int64).copy()).to(cuda)
    got = W.extract_coefficients(wd, pl).cpu().numpy().astype(np.uint32)
    want = np.array([orc.C.qgo_extract_coefficient_i64(int(w), ctypes.byref(opl)) for w in words], np.uint32)
    assert np.array_equal(got, want)
    fit = words[words < (np.uint64(1) << np.uint64(t * e))] if t * e < 64 else words
    fd = torch.from_numpy(fit.view(np.int64).copy()).to(cuda)
    W.redq_in_place(fd, pl)
    want = np.empty_like(fit)
    for i, w in enumerate(fit):
        r = ctypes.c_uint64()
        assert orc.C.qgo_redq_i64(int(w), ctypes.byref(opl), ctypes.byref(r)) == 0
        want[i] = r.value
    assert np.array_equal(u64(fd), want)
    if t * e < 64 and (words >= (np.uint64(1) << np.uint64(t * e))).any():
        with pytest.raises(qg.DigitOverflow):
            W.redq_in_place(wd.clone(), pl)
    rows = words[: 7 * 300].reshape(7, 300)
    rc = W.reduce_and_compress(torch.from_numpy(rows.view(np.int64).copy()).to(cuda), pl)
    for r in range(7):
        out = np.zeros(-(-300 // e), np.uint64)
        assert orc.C.qgo_reduce_and_compress_i64(P(np.ascontiguousarray(rows[r])), 300, ctypes.byref(opl), P(out)) == 0
        assert np.array_equal(u64(rc)[r], out)


@pytest.mark.parametrize("p,m,k,n", [(3, 37, 200, 45), (7, 70, 33, 130), (2, 5, 400, 3), (13, 64, 64, 64)])
def test_int64_products_vs_oracle(qg, orc, cuda, p, m, k, n):
    import torch

    W = qg.Int64Word
    a, b = orc.random_residue_matrix(m, k, p, 71), orc.random_residue_matrix(k, n, p, 72)
    want = orc.naive_gemm(p, a, b)
    ad, bd = dev(torch, a, cuda, np.uint32), dev(torch, b, cuda)
    pl = qg.plan_compression(p, k, 63)
    opl = orc.Plan(*[getattr(pl, f) for f in ("p", "t", "d", "e", "beta", "kmax", "inv_qd", "extraction")])
    ca, cb = W.compress(ad, pl, "rows_reversed"), W.compress(bd, pl, "cols_forward")
    acc = W.packed_common_product(ca, cb, pl)
    oca, ocb = o_pack(orc, 0, opl, a), o_pack(orc, 1, opl, b)
    oacc = np.zeros((m, n), np.uint64)
    assert orc.C.qgo_packed_common_product_i64(ctypes.byref(opl), P(oca), P(ocb), m, n, oca.shape[1], P(oacc)) == 0
    assert np.array_equal(u64(acc), oacc)
    assert np.array_equal(W.reduce_common(acc, pl).cpu().numpy().astype(np.uint32), want)
    rp = qg.plan_packed_axis(p, k, n, 63)
    cbo = W.compress(bd, rp, "outer_cols")
    post = W.right_product(ad, cbo, rp, n)
    assert np.array_equal(W.uncompress(post, rp, qg.PackOrientation(0, 1, rp.e), m, n).cpu().numpy().astype(np.uint32),
                          want)
    bp = qg.plan_compression(p, max(2, k // 3), 63)
    assert np.array_equal(W.blocked_accumulate_host(a, b, bp, max(2, k // 3)), want)
    with pytest.raises(qg.PlanMismatch):  # beta 53 DoubleWord entry points reject a 63-bit plan
        qg.mul_common_compressed_host(a, b, pl)
