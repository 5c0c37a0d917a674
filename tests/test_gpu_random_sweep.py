"""Randomized GPU parity sweep: many primes (2 .. 2^31-1), ragged shapes,
every variant (common under the GPU and the reference plans, blocked, right,
left, full, the Int64Word backend) against the oracle's naive product, and
the words of the reference-plan variants against the oracle restatement."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
PRIMES = [2, 3, 5, 7, 11, 13, 17, 31, 61, 101, 257, 1009, 8191, 65521, 131071, 1000003, 16777213, 2147483647]


def cases(n, seed):
    rng = np.random.default_rng(seed)
    for i in range(n):
        p = int(PRIMES[i % len(PRIMES)])
        m, k, n_ = (int(x) for x in rng.integers(1, 200, size=3))
        if rng.random() < 0.3:
            k = int(rng.integers(200, 3000))
        yield p, m, k, n_, 1000 * seed + i


@pytest.mark.parametrize("p,m,k,n,seed", list(cases(36, 11)))
def test_random_common_and_blocked(qg, orc, cuda, p, m, k, n, seed):
    import torch

    a, b = orc.random_residue_matrix(m, k, p, seed), orc.random_residue_matrix(k, n, p, seed + 1)
    want = orc.naive_gemm(p, a, b)
    ad = torch.from_numpy(a.astype(np.float64)).to(cuda)
    bd = torch.from_numpy(b.astype(np.float64)).to(cuda)
    try:
        gp = qg.plan_gpu(p, k)
    except qg.NoCompression:
        gp = None
    if gp is not None:
        c = qg.mul_common_compressed(ad, bd, gp)
        assert np.array_equal(c.cpu().numpy().astype(np.uint32), want)
        assert np.array_equal(qg.mul_common_compressed_host(a, b, gp), want)
    try:
        pl = qg.plan_compression(p, k)
    except qg.NoCompression:
        pl = None
    if pl is not None:
        assert np.array_equal(qg.mul_common_compressed_host(a, b, pl), want)
    kp = qg.choose_panel(p, k)
    if kp >= 2:
        bp = qg.plan_compression(p, kp)
        assert np.array_equal(qg.blocked_accumulate_host(a, b, bp, kp), want)


@pytest.mark.parametrize("p,m,k,n,seed", list(cases(36, 12)))
def test_random_right_left_full(qg, orc, cuda, p, m, k, n, seed):
    import torch

    a, b = orc.random_residue_matrix(m, k, p, seed), orc.random_residue_matrix(k, n, p, seed + 1)
    want = orc.naive_gemm(p, a, b)
    ad = torch.from_numpy(a.astype(np.float64)).to(cuda)
    bd = torch.from_numpy(b.astype(np.float64)).to(cuda)
    for axis, fn in ((n, qg.mul_right_tiled), (m, qg.mul_left_tiled)):
        try:
            gp = qg.plan_right_gpu(p, k, axis)
        except qg.NoCompression:
            continue
        cc = fn(ad, bd, gp)
        assert np.array_equal(qg.uncompress(cc).cpu().numpy().astype(np.uint32), want), fn.__name__
        try:
            rp = qg.plan_packed_axis(p, k, axis)
        except qg.NoCompression:
            continue
        if k <= rp.kmax:  # the reference plan: words equal the oracle restatement's
            cc = fn(ad, bd, rp)
            op = orc.plan_of(rp)
            if fn is qg.mul_right_tiled:
                ref = orc.mul_right_compressed(op, a, orc.compress_outer_cols(op, b), n)
            else:
                ref = orc.mul_left_compressed(op, a, b)
            assert np.array_equal(cc.data.cpu().numpy().view(np.uint64), ref.view(np.uint64)), fn.__name__
    try:
        fp, kb = qg.plan_full_gpu(p, k)
    except qg.NoCompression:
        fp = None
    if fp is not None:
        assert np.array_equal(qg.mul_full_compressed(ad, bd, fp, kb).cpu().numpy().astype(np.uint32), want)


@pytest.mark.parametrize("p,m,k,n,seed", list(cases(18, 13)))
def test_random_int64word(qg, orc, cuda, p, m, k, n, seed):
    a, b = orc.random_residue_matrix(m, k, p, seed), orc.random_residue_matrix(k, n, p, seed + 1)
    want = orc.naive_gemm(p, a, b)
    W = qg.Int64Word
    try:
        pl = qg.plan_compression(p, k, 63)
    except qg.NoCompression:
        return
    c = W.mul_common_compressed_host(a, b, pl)
    assert np.array_equal(c, want)
    opl = orc.Plan(*[getattr(pl, f) for f in ("p", "t", "d", "e", "beta", "kmax", "inv_qd", "extraction")])
    K = -(-k // pl.e)
    ca, cb = np.zeros((m, K), np.uint64), np.zeros((K, n), np.uint64)
    assert orc.C.qgo_compress_rows_reversed_i64(ctypes.byref(opl), a.ctypes.data_as(ctypes.c_void_p), m, k,
                                                ca.ctypes.data_as(ctypes.c_void_p)) == 0
    try:
        rp = qg.plan_packed_axis(p, k, n, 63)
    except qg.NoCompression:
        return
    cc = W.mul_right_compressed_host(a, b, rp)
    orp = orc.Plan(*[getattr(rp, f) for f in ("p", "t", "d", "e", "beta", "kmax", "inv_qd", "extraction")])
    H = -(-n // rp.e)
    cbo, pre = np.zeros((k, H), np.uint64), np.zeros((m, H), np.uint64)
    assert orc.C.qgo_compress_outer_cols_i64(ctypes.byref(orp), b.ctypes.data_as(ctypes.c_void_p), k, n,
                                             cbo.ctypes.data_as(ctypes.c_void_p)) == 0
    assert orc.C.qgo_packed_right_product_i64(ctypes.byref(orp), a.ctypes.data_as(ctypes.c_void_p),
                                              cbo.ctypes.data_as(ctypes.c_void_p), m, k, n,
                                              pre.ctypes.data_as(ctypes.c_void_p)) == 0
    assert orc.C.qgo_redq_in_place_i64(ctypes.byref(orp), pre.ctypes.data_as(ctypes.c_void_p), pre.size) == 0
    assert np.array_equal(cc, pre)


@pytest.mark.parametrize("p", [65521, 131071, 1000003])
def test_wide_digit_right_product_reference_layout(qg, orc, cuda, p):
    """One-digit words of large p (t > 31) through the reference-layout right
    product (qg_mul_right) and the device REDQ / uncompress."""
    import torch

    m, k, n = 37, 150, 29
    a, b = orc.random_residue_matrix(m, k, p, 91), orc.random_residue_matrix(k, n, p, 92)
    pl = qg.plan_packed_axis(p, k, n)
    ad = torch.from_numpy(a.astype(np.float64)).to(cuda)
    cbo = qg.compress_outer_cols(torch.from_numpy(b.astype(np.float64)).to(cuda), pl)
    cc = qg.mul_right_compressed(ad, cbo)
    op = orc.plan_of(pl)
    want = orc.mul_right_compressed(op, a, orc.compress_outer_cols(op, b), n)
    assert np.array_equal(cc.data.cpu().numpy().view(np.uint64), want.view(np.uint64))
    assert np.array_equal(qg.uncompress(cc).cpu().numpy().astype(np.uint32), orc.naive_gemm(p, a, b))


@pytest.mark.parametrize("p,m,k,n,seed", list(cases(36, 14)))
def test_random_reference_layouts_and_panels(qg, orc, cuda, p, m, k, n, seed):
    """Reference-layout operands (CompressedMatrix in), blocked products with a
    random panel width, and pack -> uncompress round trips."""
    import torch

    a, b = orc.random_residue_matrix(m, k, p, seed), orc.random_residue_matrix(k, n, p, seed + 1)
    want = orc.naive_gemm(p, a, b)
    ad = torch.from_numpy(a.astype(np.float64)).to(cuda)
    bd = torch.from_numpy(b.astype(np.int32)).to(cuda)
    rng = np.random.default_rng(seed)
    kp = int(rng.integers(1, k + 1))
    try:
        bp = qg.plan_compression(p, kp) if kp >= 2 else qg.uncompressed_plan(p, 1)
    except qg.NoCompression:
        bp = None
    if bp is not None:
        assert np.array_equal(qg.blocked_accumulate_host(a, b, bp, kp), want), kp
    try:
        pl = qg.plan_compression(p, k)
    except qg.NoCompression:
        return
    ca, cb = qg.compress_rows_reversed(ad, pl), qg.compress_cols_forward(bd, pl)
    op = orc.plan_of(pl)
    assert np.array_equal(ca.data.cpu().numpy().view(np.uint64), orc.compress_rows_reversed(op, a).view(np.uint64))
    assert np.array_equal(cb.data.cpu().numpy().view(np.uint64), orc.compress_cols_forward(op, b).view(np.uint64))
    c = qg.mul_common_compressed(ca, cb)
    assert np.array_equal(c.cpu().numpy().astype(np.uint32), want)
    for cm, src in ((ca, a), (cb, b), (qg.compress_outer_cols(bd, pl), b), (qg.compress_outer_rows(ad, pl), a)):
        assert np.array_equal(qg.uncompress(cm).cpu().numpy().astype(np.uint32), src)
