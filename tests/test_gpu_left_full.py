"""GPU parity of left and full compression (gemm.hpp:340-445) on the tiled
layout, through the C ABI, against the oracle (pinned to the reference in
tests/test_left_full_oracle.py) and the reference's golden vectors
(tests/golden/golden_left_full.json). Words compare as raw float64 bits,
C residue by residue."""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden_left_full.json")))


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)


def host(t):
    return t.cpu().numpy()


def _plan_tuple(d):
    return (d["p"], d["t"], d["d"], d["e"], d["beta"], d["kmax"], float.fromhex(d["inv_qd_hex"]), d["extraction"])


def _hex_words(h, shape):
    return np.array([int(x, 16) for x in h], dtype=np.uint64).reshape(shape)


def _dev(torch, x, cuda, dtype=None):
    return torch.from_numpy(x.astype(np.float64 if dtype is None else dtype)).to(cuda)


@pytest.mark.parametrize("p,t,e", [(3, 5, 7), (3, 8, 6), (3, 13, 4), (7, 12, 4), (2, 4, 13), (7, 18, 2)])
@pytest.mark.parametrize("m,k", [(1, 1), (5, 7), (33, 31), (300, 257)])
@pytest.mark.parametrize("bk", [4, 12, 36])
def test_outer_rows_tiled_layout(qg, orc, cuda, p, t, e, m, k, bk):
    """Block [g-tile][k-tile] holds compress_outer_rows words (g, l) row-major,
    zero past the logical shape."""
    import torch

    a = orc.random_residue_matrix(m, k, p, 500 + m + k)
    pl = qg.make_plan(p, t, e)
    big = orc.Plan(*orc.plan_of(pl).astuple())
    want = orc.compress_outer_rows(big, a)
    G = -(-m // e)
    kt = -(-k // bk)
    for dtype in (np.float64, np.int32):
        out = torch.full((-(-G // 128) * 128 * kt * bk,), -1.0, dtype=torch.float64, device=cuda)
        import ctypes

        c_pl = pl._c()
        ad = _dev(torch, a, cuda, dtype)
        qg._check(qg.lib.qg_pack_outer_rows_tiled(ctypes.byref(c_pl), bk, qg._ptr(ad), qg._dtype_code(ad), m, k, k,
                                                  qg._ptr(out), qg._stream()))
        tiles = host(out).reshape(-(-G // 128), kt, 128, bk).transpose(0, 2, 1, 3).reshape(-(-G // 128) * 128, kt * bk)
        assert np.array_equal(bits(tiles[:G, :k]), bits(want))
        assert not tiles[G:, :].any() and not tiles[:, k:].any()


@pytest.mark.parametrize("idx", range(len(GOLDEN["cases"])))
def test_golden_left_full_gpu(qg, orc, cuda, idx):
    import torch

    c = GOLDEN["cases"][idx]
    p, m, k, n = c["p"], c["m"], c["k"], c["n"]
    a, b = orc.random_residue_matrix(m, k, p, c["seed_a"]), orc.random_residue_matrix(k, n, p, c["seed_b"])
    assert hashlib.sha256(a.tobytes()).hexdigest() == c["a_sha"]
    ad, bd = _dev(torch, a, cuda), _dev(torch, b, cuda)
    want = orc.naive_gemm(p, a, b)
    if "left_plan" in c:
        lp = qg.CompressionPlan._from(qg._Plan(*_plan_tuple(c["left_plan"])))
        cc = qg.mul_left_tiled(ad, bd, lp)
        assert np.array_equal(bits(host(cc.data)), _hex_words(c["left_cc"], (-(-m // lp.e), n)))
        assert np.array_equal(host(qg.uncompress(cc)).astype(np.uint32), want)
        # the reference's API shape: mul_left_compressed(compress_outer_rows(A), B)
        cc2 = qg.mul_left_compressed(qg.compress_outer_rows(ad, lp), bd)
        assert np.array_equal(bits(host(cc2.data)), bits(host(cc.data)))
        assert np.array_equal(bits(qg.mul_left_compressed_host(a, b, lp)), bits(host(cc.data)))
    if "full_plan" in c:
        d = c["full_plan"]
        fp = qg.FullPlan(qg.CompressionPlan._from(qg._Plan(*_plan_tuple(d["base"]))), d["dq"], d["dtheta"],
                         d["theta_exponent"])
        assert np.array_equal(host(qg.mul_full_compressed(ad, bd, fp)).astype(np.uint32), want)
        assert np.array_equal(qg.mul_full_compressed_host(a, b, fp), want)
    assert hashlib.sha256(want.tobytes()).hexdigest() == c["c_sha"]


@pytest.mark.parametrize("p,k", [(3, 7), (3, 255), (5, 31), (7, 13), (3, 512), (2, 100), (11, 40), (7, 2000)])
@pytest.mark.parametrize("m,n", [(1, 1), (17, 33), (130, 70), (257, 300)])
def test_mul_left_tiled(qg, orc, cuda, p, k, m, n):
    """Reference plan: CC words equal mul_left_compressed's bit for bit;
    blocked GPU plan (in-place REDQ between k-blocks): CC equals
    compress_outer_rows(naive C)."""
    import torch

    a, b = orc.random_residue_matrix(m, k, p, 277), orc.random_residue_matrix(k, n, p, 278)
    ad, bd = _dev(torch, a, cuda), _dev(torch, b, cuda)
    want_c = orc.naive_gemm(p, a, b)
    try:
        lp = qg.plan_packed_axis(p, k, m)
    except qg.NoCompression:
        lp = None
    if lp is not None and k <= lp.kmax:
        cc = qg.mul_left_tiled(ad, bd, lp)
        want = orc.mul_left_compressed(orc.plan_of(lp), a, b)
        assert np.array_equal(bits(host(cc.data)), bits(want))
    gp = qg.plan_right_gpu(p, k, m)
    cc = qg.mul_left_tiled(ad, bd, gp)
    assert np.array_equal(host(qg.uncompress(cc)).astype(np.uint32), want_c)
    big = orc.Plan(*orc.plan_of(gp.plan).astuple())
    big.kmax = max(big.kmax, k)
    assert np.array_equal(bits(host(cc.data)), bits(orc.compress_outer_rows(big, want_c)))


@pytest.mark.parametrize("p,k", [(3, 7), (3, 250), (5, 10), (7, 13), (2, 100), (3, 4096), (7, 3000), (251, 600)])
@pytest.mark.parametrize("m,n", [(1, 1), (9, 8), (130, 70), (257, 383)])
def test_mul_full(qg, orc, cuda, p, k, m, n):
    """Reference plan_full (single block) and the blocked GPU plan both give
    naive C; int32 operands too."""
    import torch

    a, b = orc.random_residue_matrix(m, k, p, 377), orc.random_residue_matrix(k, n, p, 378)
    want = orc.naive_gemm(p, a, b)
    try:
        fp = qg.plan_full(p, k)
    except qg.NoCompression:
        fp = None
    if fp is not None:
        got = qg.mul_full_compressed(_dev(torch, a, cuda), _dev(torch, b, cuda), fp)
        assert np.array_equal(host(got).astype(np.uint32), want)
        assert np.array_equal(want, orc.mul_full_compressed(orc.FullPlan(orc.plan_of(fp.base), fp.dq, fp.dtheta,
                                                                         fp.theta_exponent), a, b))
    gfp, kb = qg.plan_full_gpu(p, k)
    got = qg.mul_full_compressed(_dev(torch, a, cuda, np.int32), _dev(torch, b, cuda, np.int32), gfp, kb)
    assert np.array_equal(host(got).astype(np.uint32), want)
    assert np.array_equal(qg.mul_full_compressed_host(a, b, gfp, kb), want)


def test_full_adversarial_all_max(qg, orc, cuda):
    """All residues p-1 at the largest single-block k of the plan (acceptance.cpp
    criterion 6's worst case) and past it under the blocked plan."""
    import torch

    for p in (3, 7):
        fp = qg.plan_full(p, 200)
        k = fp.base.kmax
        a = np.full((67, k), p - 1, np.uint32)
        b = np.full((k, 45), p - 1, np.uint32)
        want = np.full((67, 45), (k * (p - 1) ** 2) % p, np.uint32)
        assert np.array_equal(host(qg.mul_full_compressed(_dev(torch, a, cuda), _dev(torch, b, cuda), fp)), want)
        gfp, kb = qg.plan_full_gpu(p, 5 * k)
        a5, b5 = np.full((67, 5 * k), p - 1, np.uint32), np.full((5 * k, 45), p - 1, np.uint32)
        want5 = np.full((67, 45), (5 * k * (p - 1) ** 2) % p, np.uint32)
        got = qg.mul_full_compressed(_dev(torch, a5, cuda), _dev(torch, b5, cuda), gfp, kb)
        assert np.array_equal(host(got), want5)


def test_left_full_errors(qg, cuda):
    import torch

    a = torch.zeros((4, 300), dtype=torch.float64, device=cuda)
    b = torch.zeros((300, 5), dtype=torch.float64, device=cuda)
    pl = qg.plan_packed_axis(3, 8, 4)  # kmax far below 300
    with pytest.raises(qg.PlanMismatch):
        qg.mul_left_tiled(a, b, pl)
    with pytest.raises(qg.PlanMismatch):
        qg.mul_left_compressed(qg.compress_outer_cols(a, pl), b)
    with pytest.raises(qg.DimensionMismatch):
        qg.mul_left_tiled(a, b[:7].contiguous(), pl)
    fp = qg.plan_full(3, 8)
    with pytest.raises(qg.PlanMismatch):
        qg.mul_full_compressed(a, b, fp)  # k > kmax, single block
    bad = qg.FullPlan(fp.base, fp.dq, fp.dtheta, fp.theta_exponent + 1)
    with pytest.raises(qg.PlanMismatch):
        qg.mul_full_compressed(a[:, :8].contiguous(), b[:8].contiguous(), bad)
    with pytest.raises(qg.DimensionMismatch):
        qg.mul_full_compressed(a, b[:7].contiguous(), fp)


@pytest.mark.parametrize("p,k,m,n", [(5, 3000, 130, 70), (3, 20000, 67, 129), (7, 13, 9, 8)])
def test_host_entries_with_gpu_plans(qg, orc, p, k, m, n):
    """qg_host_mul_right_gpu / qg_host_mul_left_gpu: blocked plans on host data."""
    a, b = orc.random_residue_matrix(m, k, p, 477), orc.random_residue_matrix(k, n, p, 478)
    want = orc.naive_gemm(p, a, b)
    gr = qg.plan_right_gpu(p, k, n)
    big = orc.Plan(*orc.plan_of(gr.plan).astuple())
    big.kmax = max(big.kmax, k)
    assert np.array_equal(bits(qg.mul_right_compressed_host(a, b, gr)), bits(orc.compress_outer_cols(big, want)))
    gl = qg.plan_right_gpu(p, k, m)
    big = orc.Plan(*orc.plan_of(gl.plan).astuple())
    big.kmax = max(big.kmax, k)
    assert np.array_equal(bits(qg.mul_left_compressed_host(a, b, gl)), bits(orc.compress_outer_rows(big, want)))


@pytest.mark.parametrize("p,t,e,kb", [(5, 13, 4, 1008), (7, 13, 4, 448), (3, 10, 5, 252), (11, 12, 4, 72),
                                      (13, 13, 4, 36), (5, 13, 4, 28)])
@pytest.mark.parametrize("m,k,n", [(130, 3000, 70), (67, 1001, 129), (5, 37, 9)])
def test_balanced_redq_plans(qg, orc, cuda, p, t, e, kb, m, k, n):
    """Balanced-digit right/left products (signed operands, balanced in-place
    REDQ between k-blocks): the CC words are the canonical REDQ words of C."""
    import torch

    a, b = orc.random_residue_matrix(m, k, p, 577), orc.random_residue_matrix(k, n, p, 578)
    want = orc.naive_gemm(p, a, b)
    gp = qg.GpuPlan(qg.make_plan(p, t, e), kb, kb, 1)
    big = orc.Plan(*orc.plan_of(gp.plan).astuple())
    big.kmax = max(big.kmax, k)
    for dtype in (np.float64, np.int32):
        ad, bd = _dev(torch, a, cuda, dtype), _dev(torch, b, cuda, dtype)
        cc = qg.mul_right_tiled(ad, bd, gp)
        assert np.array_equal(bits(host(cc.data)), bits(orc.compress_outer_cols(big, want)))
        cl = qg.mul_left_tiled(ad, bd, gp)
        assert np.array_equal(bits(host(cl.data)), bits(orc.compress_outer_rows(big, want)))
    assert np.array_equal(bits(qg.mul_right_compressed_host(a, b, gp)), bits(orc.compress_outer_cols(big, want)))
    assert np.array_equal(bits(qg.mul_left_compressed_host(a, b, gp)), bits(orc.compress_outer_rows(big, want)))


def test_balanced_redq_bound_is_enforced(qg, cuda):
    import torch

    a = torch.zeros((8, 3000), dtype=torch.float64, device=cuda)
    b = torch.zeros((3000, 8), dtype=torch.float64, device=cuda)
    # p = 5, t = 13: h + kb h^2 < Q/2 allows 1023 residues per block, not 2016
    with pytest.raises(qg.PlanMismatch):
        qg.mul_right_tiled(a, b, qg.GpuPlan(qg.make_plan(5, 13, 4), 2016, 2016, 1))
