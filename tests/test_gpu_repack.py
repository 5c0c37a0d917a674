"""Compressed-out and compressed-in products on the GPU (SURVEY.md §8(f)
rank 1): mul_common_repacked with ReduceAndCompress fused into the
contraction's epilogue (gemm.hpp:275-280, pack.hpp:141-155) and
mul_right_compressed(ca, cb), the uncompress-first path (gemm.hpp:329-335).

Expected words come from the oracle's compress_outer_cols (oracle/qg_oracle.c,
pinned to the reference in test_oracle.py) applied to the exact C, so a
repacked word must equal compress_outer_cols(C, plan) bit for bit; for config 1
the reference's own mul_common_repacked (oracle/_ref) is compared directly."""
import ctypes
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)


@pytest.fixture
def route(monkeypatch, request):
    monkeypatch.setenv("QG_SMALL", request.param)
    return request.param


def _want_words(orc, qg, c, plan):
    return bits(orc.compress_outer_cols(orc.plan_of(plan), np.ascontiguousarray(c.astype(np.uint32))))


@pytest.mark.parametrize("route", ["0", "1"], indirect=True, ids=["main128", "small64"])
@pytest.mark.parametrize("p,m,k,n,planner", [
    (3, 512, 512, 512, "reference"),    # config 1 shape
    (7, 640, 4096, 384, "gpu"),         # config 2 common dimension, blocked balanced plan (e=4)
    (7, 256, 4096, 256, "reference"),   # reference plan t=18 e=2
    (3, 1024, 256, 1024, "gpu"),        # config 3 k (e=5: words cross 32-column warp segments)
    (3, 300, 32768, 130, "gpu"),        # config 5 k (e=6), ragged m and n
    (5, 129, 1000, 257, "gpu"),         # odd n
    (2, 200, 700, 190, "gpu"),
    (13, 131, 600, 77, "gpu"),
])
def test_mul_common_repacked_words(qg, orc, cuda, route, p, m, k, n, planner):
    import torch

    a = orc.random_residue_matrix(m, k, p, 42)
    b = orc.random_residue_matrix(k, n, p, 43)
    plan = qg.plan_compression(p, k) if planner == "reference" else qg.plan_gpu(p, k)
    base = plan.plan if isinstance(plan, qg.GpuPlan) else plan
    cc = qg.mul_common_repacked(torch.from_numpy(a.astype(np.float64)).to(cuda),
                                torch.from_numpy(b.astype(np.float64)).to(cuda), plan)
    assert (cc.stored_rows, cc.stored_cols) == (m, -(-n // base.e))
    assert cc.orientation.direction == qg.PackDirection.Forward and cc.orientation.axis == qg.PackAxis.Column
    c = orc.naive_gemm(p, a, b)
    assert np.array_equal(bits(cc.data.cpu().numpy()), _want_words(orc, qg, c, base))
    assert np.array_equal(qg.uncompress(cc).cpu().numpy().astype(np.uint32), c)
    if route == "0" and m >= 256 and n >= 256 and p < 256:
        assert qg.last_kernel().startswith("dot_tiled_repack"), qg.last_kernel()


def test_repacked_matches_reference_config1(qg, orc, cuda):
    """Config 1 (p=3, 512^3, seeds 42/43) against the reference's own
    mul_common_repacked words (oracle/_ref), when the reference harness is
    present, else against its golden C through the oracle's packer."""
    import torch

    p, m, k, n = 3, 512, 512, 512
    plan = qg.plan_compression(p, k)
    a = qg.random_residue_matrix(m, k, p, 42)
    b = qg.random_residue_matrix(k, n, p, 43)
    cc = qg.mul_common_repacked(a, b, plan)
    got = bits(cc.data.cpu().numpy())
    ah = orc.random_residue_matrix(m, k, p, 42)
    bh = orc.random_residue_matrix(k, n, p, 43)
    want = bits(orc.mul_common_repacked(orc.plan_of(plan), ah, bh))
    assert np.array_equal(got, want)
    assert qg.residue_checksum(qg.uncompress(cc)) == 262622  # README.md:97-99
    torch.cuda.synchronize()


@pytest.mark.parametrize("planner", ["reference", "gpu"])
def test_repacked_host_api(qg, orc, cuda, planner):
    p, m, k, n = 7, 700, 4096, 300
    a = orc.random_residue_matrix(m, k, p, 5)
    b = orc.random_residue_matrix(k, n, p, 6)
    plan = qg.plan_compression(p, k) if planner == "reference" else qg.plan_gpu(p, k)
    base = plan.plan if isinstance(plan, qg.GpuPlan) else plan
    cc = qg.mul_common_repacked_host(a, b, plan)
    assert np.array_equal(bits(cc), _want_words(orc, qg, orc.naive_gemm(p, a, b), base))


@pytest.mark.parametrize("p", [257, 1021])
def test_repacked_large_p_goes_through_workspace(qg, orc, cuda, p):
    """p >= 256 does not fit the fused epilogue's byte staging: the int32
    workspace + outer-cols pack path gives the same words."""
    import torch

    m, k, n = 300, 40, 260
    a = orc.random_residue_matrix(m, k, p, 1)
    b = orc.random_residue_matrix(k, n, p, 2)
    gp = qg.plan_gpu(p, k)
    cc = qg.mul_common_repacked(torch.from_numpy(a.astype(np.float64)).to(cuda),
                                torch.from_numpy(b.astype(np.float64)).to(cuda), gp)
    assert np.array_equal(bits(cc.data.cpu().numpy()), _want_words(orc, qg, orc.naive_gemm(p, a, b), gp.plan))


def test_repacked_config2_full_size(qg, orc, cuda):
    """Config 2 (p=7, 4096^3) under the benched GPU plan: the fused words equal
    compress_outer_cols of the C that matches the reference's sha256."""
    import torch

    p, m, k, n = 7, 4096, 4096, 4096
    gp = qg.plan_gpu(p, k)
    a = qg.random_residue_matrix(m, k, p, 42)
    b = qg.random_residue_matrix(k, n, p, 43)
    c = qg.mul_common_compressed(a, b, gp)
    cc = qg.mul_common_repacked(a, b, gp)
    assert qg.residue_checksum(c) == 50333685
    want = torch.from_numpy(_want_words(orc, qg, c.cpu().numpy(), gp.plan).view(np.float64)).to(cuda)
    assert torch.equal(cc.data, want)
    del a, b, c, cc
    torch.cuda.empty_cache()


# ------------------------------------------------------------ mul_right_compressed(ca, cb)
@pytest.mark.parametrize("p,m,k,n", [(5, 33, 120, 50), (3, 130, 500, 257), (7, 64, 64, 9)])
def test_mul_right_compressed_compressed_left(qg, orc, cuda, p, m, k, n):
    """gemm.hpp:329-335: a Forward-packed left operand is uncompressed on the
    device first; the words equal mul_right_compressed(A, CB) and the
    reference's (oracle) words; a Reversed left operand is refused."""
    import torch

    plan = qg.plan_packed_axis(p, k, n)
    a = orc.random_residue_matrix(m, k, p, 3)
    b = orc.random_residue_matrix(k, n, p, 4)
    ad = torch.from_numpy(a.astype(np.float64)).to(cuda)
    cbo = qg.compress_outer_cols(torch.from_numpy(b.astype(np.float64)).to(cuda), plan)
    ca = qg.compress_outer_cols(ad, plan)  # Forward, on the k axis of A
    cc = qg.mul_right_compressed(ca, cbo)
    ref = qg.mul_right_compressed(ad, cbo)
    assert np.array_equal(bits(cc.data.cpu().numpy()), bits(ref.data.cpu().numpy()))
    want = orc.mul_right_compressed(orc.plan_of(plan), a, orc.compress_outer_cols(orc.plan_of(plan), b), n)
    assert np.array_equal(bits(cc.data.cpu().numpy()), bits(want))
    assert np.array_equal(qg.uncompress(cc).cpu().numpy().astype(np.uint32), orc.naive_gemm(p, a, b))
    with pytest.raises(qg.PlanMismatch):
        qg.mul_right_compressed(qg.compress_rows_reversed(ad, plan), cbo)


# ------------------------------------------------------------ reference-layout left product, digit extraction
@pytest.mark.parametrize("p,m,k,n", [(7, 30, 40, 17), (3, 129, 500, 64), (5, 8, 1, 3)])
@pytest.mark.parametrize("dtype", ["f64", "u32"])
def test_left_product_reference_layout(qg, orc, cuda, p, m, k, n, dtype):
    """qg_packed_left_product / qg_mul_left (gemm.hpp:340-371) on
    compress_outer_rows words: the REDQ'd words equal the oracle's
    mul_left_compressed bit for bit; the raw words unpack to the unreduced
    digits (the dot products)."""
    import torch

    plan = qg.plan_packed_axis(p, k, m)
    a = orc.random_residue_matrix(m, k, p, 7)
    b = orc.random_residue_matrix(k, n, p, 8)
    ca = qg.compress_outer_rows(torch.from_numpy(a.astype(np.float64)).to(cuda), plan)
    bd = torch.from_numpy(b.astype(np.float64) if dtype == "f64" else b.view(np.int32)).to(cuda)
    code = 0 if dtype == "f64" else 1
    G = -(-m // plan.e)
    pl = plan._c()
    cc = torch.empty((G, n), dtype=torch.float64, device=cuda)
    qg._check(qg.lib.qg_mul_left(ctypes.byref(pl), qg._ptr(ca.data), k, qg._ptr(bd), code, n, m, k, n, qg._ptr(cc),
                                 qg._stream()))
    want = orc.mul_left_compressed(orc.plan_of(plan), a, b)
    assert np.array_equal(bits(cc.cpu().numpy()), bits(want))
    raw = torch.empty((G, n), dtype=torch.float64, device=cuda)
    qg._check(qg.lib.qg_packed_left_product(ctypes.byref(pl), qg._ptr(ca.data), k, qg._ptr(bd), code, n, m, k, n,
                                            qg._ptr(raw), qg._stream()))
    w = raw.cpu().numpy().astype(np.uint64)
    dots = (a.astype(np.int64) @ b.astype(np.int64))
    for s in range(plan.e):
        rows = np.arange(s, m, plan.e)
        got = (w[:len(rows)] >> np.uint64(plan.t * s)) & np.uint64((1 << plan.t) - 1)
        assert np.array_equal(got.astype(np.int64), dots[rows])


@pytest.mark.parametrize("u64", [False, True])
def test_extract_digits(qg, cuda, u64):
    """extract_all (pack.hpp:104-119) on the device: every base-Q digit of each
    word, unreduced; a word >= Q^e (or negative) is DigitOverflow."""
    import torch

    plan = qg.make_plan(3, 5, 3)
    vals = [0, 1, 31, 32, 33, 2081, 2048 + 32, 32767]
    dt = torch.int64 if u64 else torch.float64
    w = torch.tensor(vals, dtype=dt, device=cuda)
    out = torch.zeros(len(vals) * 3, dtype=torch.int64, device=cuda)
    pl = plan._c()
    fn = qg.lib.qg_extract_digits_u64 if u64 else qg.lib.qg_extract_digits
    qg._check(fn(ctypes.byref(pl), qg._ptr(w), len(vals), qg._ptr(out), qg._stream()))
    got = out.view(-1, 3).cpu().tolist()
    assert got == [[(v >> (5 * s)) & 31 for s in range(3)] for v in vals]
    bad = torch.tensor([32768], dtype=dt, device=cuda)
    with pytest.raises(qg.DigitOverflow):
        qg._check(fn(ctypes.byref(pl), qg._ptr(bad), 1, qg._ptr(out), qg._stream()))
    if not u64:
        neg = torch.tensor([-1.0], dtype=dt, device=cuda)
        with pytest.raises(qg.DigitOverflow):
            qg._check(fn(ctypes.byref(pl), qg._ptr(neg), 1, qg._ptr(out), qg._stream()))
