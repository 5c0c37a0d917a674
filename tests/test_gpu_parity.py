"""GPU parity: the sm_100a kernels, called through the C ABI, against the
oracle (oracle/qg_oracle.c, pinned to the reference in test_oracle.py) on the
same seeded inputs. Integer/byte work must be bit-exact: packed words are
compared as raw float64 bit patterns, C residue by residue."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)


def host(t):
    return t.cpu().numpy()


LADDER = [(3, 5, 7), (3, 6, 8), (3, 7, 7), (3, 8, 6), (3, 10, 5), (3, 13, 4), (3, 17, 3)]


@pytest.mark.parametrize("p,seed,rows,cols,row0", [(3, 42, 37, 53, 0), (7, 43, 64, 129, 5), (5, 1, 1, 1000, 17), (11, 9, 3, 3, 0)])
def test_gen_residues_bitexact(qg, orc, cuda, p, seed, rows, cols, row0):
    import torch

    want = orc.random_residue_matrix(rows, cols, p, seed, row0=row0)
    got = qg.random_residue_matrix(rows, cols, p, seed, row0=row0)
    assert np.array_equal(host(got).astype(np.uint32), want)
    got32 = qg.random_residue_matrix(rows, cols, p, seed, row0=row0, dtype=torch.int32)
    assert np.array_equal(host(got32).astype(np.uint32), want)


@pytest.mark.parametrize("p,t,e", LADDER + [(5, 9, 3), (7, 12, 4), (2, 4, 13), (7, 18, 2)])
@pytest.mark.parametrize("m,k", [(1, 1), (5, 7), (33, 31), (130, 257)])
def test_pack_kernels_bitexact(qg, orc, cuda, p, t, e, m, k):
    import torch

    plan = qg.make_plan(p, t, e)
    a = orc.random_residue_matrix(m, k, p, 1000 + m + k)
    oplan = orc.plan_of(plan)
    big = orc.Plan(*oplan.astuple())
    big.kmax = max(big.kmax, k, m)  # packing does not depend on kmax
    pbig = qg.CompressionPlan._from(qg._Plan(*big.astuple()))
    ad = torch.from_numpy(a.astype(np.float64)).to(cuda)
    for dev_in in (ad, torch.from_numpy(a.astype(np.int32)).to(cuda)):
        ca = qg.compress_rows_reversed(dev_in, pbig)
        assert np.array_equal(bits(host(ca.data)), bits(orc.compress_rows_reversed(big, a)))
        cb = qg.compress_cols_forward(dev_in, pbig)
        assert np.array_equal(bits(host(cb.data)), bits(orc.compress_cols_forward(big, a)))
        co = qg.compress_outer_cols(dev_in, pbig)
        assert np.array_equal(bits(host(co.data)), bits(orc.compress_outer_cols(big, a)))
        cr = qg.compress_outer_rows(dev_in, pbig)
        assert np.array_equal(bits(host(cr.data)), bits(orc.compress_outer_rows(big, a)))
        # uncompress inverts every packing (test_gemm.cpp:361-373)
        for cm in (ca, cb, co, cr):
            assert np.array_equal(host(qg.uncompress(cm)).astype(np.uint32), a)


@pytest.mark.parametrize("p,k", [(3, 7), (3, 255), (5, 31), (7, 13), (3, 512), (2, 100), (11, 40)])
@pytest.mark.parametrize("m,n", [(1, 1), (17, 33), (130, 70)])
def test_packed_common_product_bitexact(qg, orc, cuda, p, k, m, n):
    """gemm.hpp:210-244: the pre-mask accumulators equal the reference's doubles."""
    import torch

    plan = qg.plan_compression(p, k)
    a = orc.random_residue_matrix(m, k, p, 7 * m + k)
    b = orc.random_residue_matrix(k, n, p, 11 * n + k)
    ca = qg.compress_rows_reversed(torch.from_numpy(a.astype(np.float64)).to(cuda), plan)
    cb = qg.compress_cols_forward(torch.from_numpy(b.astype(np.float64)).to(cuda), plan)
    acc = host(qg.packed_common_product(ca, cb))
    oplan = orc.plan_of(plan)
    want = orc.packed_common_product(oplan, orc.compress_rows_reversed(oplan, a), orc.compress_cols_forward(oplan, b), k)
    assert np.array_equal(bits(acc), bits(want))
    red = host(qg.reduce_common_entry(qg.packed_common_product(ca, cb), plan)).astype(np.uint32)
    assert np.array_equal(red, orc.naive_gemm(p, a, b))


@pytest.mark.parametrize("p,m,k,n", [
    (3, 512, 512, 512),      # config 1 shape
    (3, 200, 256, 300),      # short k (config 3 flavour), ragged tiles
    (7, 129, 1000, 131),     # ragged everything
    (5, 1, 17, 1),
    (2, 64, 3000, 64),
    (11, 70, 40, 90),
    (7, 256, 113, 256),      # k = kmax(t=12) for p=7
])
def test_mul_common_reference_plan(qg, orc, cuda, p, m, k, n):
    import torch

    plan = qg.plan_compression(p, k)
    a = orc.random_residue_matrix(m, k, p, 42)
    b = orc.random_residue_matrix(k, n, p, 43)
    want = orc.naive_gemm(p, a, b)
    got = host(qg.mul_common_compressed(torch.from_numpy(a.astype(np.float64)).to(cuda),
                                        torch.from_numpy(b.astype(np.float64)).to(cuda), plan))
    assert np.array_equal(got.astype(np.uint32), want)
    if (p, m, k, n) == (3, 512, 512, 512):
        assert qg.residue_checksum(got) == 262622  # README.md:97-99


@pytest.mark.parametrize("p,m,k,n", [
    (7, 256, 4096, 256),     # config 2 common dimension, k >> kmax of the blocked plan
    (3, 192, 5000, 200),
    (5, 130, 2047, 129),
    (3, 64, 32768, 64),      # config 5 common dimension
])
def test_mul_common_gpu_plan_blocked(qg, orc, cuda, p, m, k, n):
    """plan_gpu picks (t, e, kblock) freely; C mod p is unique, so it must
    equal naive_gemm (gemm.hpp:80-100) exactly."""
    import torch

    gp = qg.plan_gpu(p, k)
    assert gp.kblock_words * gp.plan.e <= gp.eq3_kmax() or gp.kblock_words * gp.plan.e >= k
    assert gp.kblock_words <= gp.max_exact_words
    a = orc.random_residue_matrix(m, k, p, 4242)
    b = orc.random_residue_matrix(k, n, p, 4243)
    got = host(qg.mul_common_compressed(torch.from_numpy(a.astype(np.float64)).to(cuda),
                                        torch.from_numpy(b.astype(np.float64)).to(cuda), gp))
    assert np.array_equal(got.astype(np.uint32), orc.naive_gemm(p, a, b))


@pytest.mark.parametrize("p,k", [(3, 1023), (7, 113), (5, 255), (3, 32767), (7, 4096), (3, 4096), (5, 8192)])
def test_adversarial_all_max_residues(qg, orc, cuda, p, k):
    """All residues p-1 maximise every digit and the FP64 magnitude: the
    worst case of the exactness bound (test_gemm.cpp:383-393, acceptance.cpp:163-221)."""
    import torch

    for plan in (qg.plan_gpu(p, k),) + ((qg.plan_compression(p, k),) if k <= 65535 else ()):
        a = np.full((16, k), p - 1, dtype=np.uint32)
        b = np.full((k, 24), p - 1, dtype=np.uint32)
        got = host(qg.mul_common_compressed(torch.from_numpy(a.astype(np.float64)).to(cuda),
                                            torch.from_numpy(b.astype(np.float64)).to(cuda), plan))
        assert (got == (k * (p - 1) ** 2) % p).all()


def test_adversarial_sparse_low_digits(qg, orc, cuda):
    """Residues that make the low digits large and the wanted digit small."""
    import torch

    rng = np.random.default_rng(5)
    for p, k in ((3, 4096), (7, 4096), (5, 2000)):
        gp = qg.plan_gpu(p, k)
        e = gp.plan.e
        a = np.zeros((32, k), dtype=np.uint32)
        b = np.zeros((k, 40), dtype=np.uint32)
        # slot patterns: A's first residue of each word, B's last -> products land below digit d
        a[:, 0::e] = p - 1
        b[e - 1::e, :] = p - 1
        noise = rng.random(a.shape) < 0.05
        a[noise] = rng.integers(0, p, size=int(noise.sum()))
        got = host(qg.mul_common_compressed(torch.from_numpy(a.astype(np.float64)).to(cuda),
                                            torch.from_numpy(b.astype(np.float64)).to(cuda), gp))
        assert np.array_equal(got.astype(np.uint32), orc.naive_gemm(p, a, b))


@pytest.mark.parametrize("p,m,k,n", [(5, 96, 300, 250), (3, 130, 64, 77), (7, 33, 500, 9), (5, 1, 6, 1)])
def test_mul_right_bitexact(qg, orc, cuda, p, m, k, n):
    """Mixed variant: CC words equal the reference's post-REDQ words."""
    import torch

    plan = qg.plan_packed_axis(p, k, n)
    a = orc.random_residue_matrix(m, k, p, 77)
    b = orc.random_residue_matrix(k, n, p, 78)
    cbo = qg.compress_outer_cols(torch.from_numpy(b.astype(np.float64)).to(cuda), plan)
    oplan = orc.plan_of(plan)
    assert np.array_equal(bits(host(cbo.data)), bits(orc.compress_outer_cols(oplan, b)))
    ad = torch.from_numpy(a.astype(np.float64)).to(cuda)
    raw = qg.packed_right_product(ad, cbo)
    assert np.array_equal(bits(host(raw.data)), bits(orc.packed_right_product(oplan, a, orc.compress_outer_cols(oplan, b), n)))
    cc = qg.mul_right_compressed(ad, cbo)
    want = orc.mul_right_compressed(oplan, a, orc.compress_outer_cols(oplan, b), n)
    assert np.array_equal(bits(host(cc.data)), bits(want))
    assert np.array_equal(host(qg.uncompress(cc)).astype(np.uint32), orc.naive_gemm(p, a, b))
    qg.redq_in_place(raw)
    assert np.array_equal(bits(host(raw.data)), bits(want))


def test_redq_digit_overflow(qg, cuda):
    import torch

    plan = qg.make_plan(3, 5, 3)
    w = torch.tensor([4423.0, 0.0, 1057.0], dtype=torch.float64, device=cuda)
    cm = qg.CompressedMatrix(1, 9, 1, 3, qg.PackOrientation(0, 1, 3), plan, w.view(1, 3))
    qg.redq_in_place(cm)
    assert w.cpu().tolist() == [1057.0, 0.0, 1057.0]  # test_pack.cpp:93-99
    bad = torch.tensor([float(1 << 15)], dtype=torch.float64, device=cuda)
    with pytest.raises(qg.DigitOverflow):
        qg.redq_in_place(qg.CompressedMatrix(1, 3, 1, 1, qg.PackOrientation(0, 1, 3), plan, bad.view(1, 1)))


def test_host_entry_points(qg, orc, cuda):
    p, m, k, n = 3, 70, 300, 50
    a = orc.random_residue_matrix(m, k, p, 1)
    b = orc.random_residue_matrix(k, n, p, 2)
    want = orc.naive_gemm(p, a, b)
    plan = qg.plan_compression(p, k)
    assert np.array_equal(qg.mul_common_compressed_host(a, b, plan), want)
    for kp in (1, 2, 3, 7, 64, 150, 255):
        pl = qg.plan_compression(p, kp) if kp >= 2 else qg.uncompressed_plan(p, 1)
        assert np.array_equal(qg.blocked_accumulate_host(a, b, pl, kp), orc.blocked_accumulate(orc.plan_of(pl), a, b, kp)), kp
    rp = qg.plan_packed_axis(p, k, n)
    got = qg.mul_right_compressed_host(a, b, rp)
    oplan = orc.plan_of(rp)
    assert np.array_equal(bits(got), bits(orc.mul_right_compressed(oplan, a, orc.compress_outer_cols(oplan, b), n)))


def test_error_behaviour(qg, cuda):
    import torch

    a = torch.zeros((2, 3), dtype=torch.float64, device=cuda)
    with pytest.raises(qg.DimensionMismatch):
        qg.mul_common_compressed(a, a, qg.make_plan(3, 5, 2))
    with pytest.raises(qg.PlanMismatch):  # 8 columns exceed kmax = 7 at Q = 32 (test_gemm.cpp:357-358)
        qg.compress_rows_reversed(torch.zeros((1, 8), dtype=torch.float64, device=cuda), qg.make_plan(3, 5, 2))
    ca = qg.compress_rows_reversed(torch.zeros((2, 2), dtype=torch.float64, device=cuda), qg.make_plan(3, 5, 2))
    other = qg.compress_cols_forward(torch.zeros((2, 2), dtype=torch.float64, device=cuda), qg.make_plan(3, 7, 2))
    with pytest.raises(qg.PlanMismatch):
        qg.mul_common_compressed(ca, other)
    cb = qg.compress_cols_forward(torch.zeros((2, 2), dtype=torch.float64, device=cuda), qg.make_plan(3, 5, 2))
    with pytest.raises(qg.PlanMismatch):
        qg.packed_common_product(cb, cb)


def test_determinism(qg, orc, cuda):
    import torch

    p, m, k, n = 11, 170, 230, 190
    a = torch.from_numpy(orc.random_residue_matrix(m, k, p, 51).astype(np.float64)).to(cuda)
    b = torch.from_numpy(orc.random_residue_matrix(k, n, p, 52).astype(np.float64)).to(cuda)
    for plan in (qg.plan_compression(p, k), qg.plan_gpu(p, k)):
        once = host(qg.mul_common_compressed(a, b, plan))
        twice = host(qg.mul_common_compressed(a, b, plan))
        assert np.array_equal(once, twice)


def test_empty_shapes(qg, cuda):
    import torch

    plan = qg.plan_compression(3, 5)
    z = lambda r, c: torch.zeros((r, c), dtype=torch.float64, device=cuda)
    assert qg.mul_common_compressed(z(0, 5), z(5, 4), plan).shape == (0, 4)
    assert qg.mul_common_compressed(z(3, 5), z(5, 0), plan).shape == (3, 0)


@pytest.mark.parametrize("p,m,k,n", [(7, 300, 4096, 258), (3, 129, 512, 130), (5, 77, 8192, 64), (3, 512, 32768, 256),
                                     (2, 64, 3000, 66), (11, 70, 40, 90), (7, 1, 113, 2)])
@pytest.mark.parametrize("planner", ["gpu", "reference"])
def test_tiled_path(qg, orc, cuda, p, m, k, n, planner):
    """The tiled packed layout + tiled DMMA kernel (the fast path) equals naive_gemm."""
    import torch

    if planner == "reference" and k > 65535:
        pytest.skip()
    plan = qg.plan_gpu(p, k) if planner == "gpu" else qg.plan_compression(p, k)
    a = orc.random_residue_matrix(m, k, p, 900 + m)
    b = orc.random_residue_matrix(k, n, p, 901 + n)
    got = host(qg.mul_common_tiled(torch.from_numpy(a.astype(np.float64)).to(cuda),
                                   torch.from_numpy(b.astype(np.float64)).to(cuda), plan))
    assert "tiled" in qg.last_kernel()
    assert np.array_equal(got.astype(np.uint32), orc.naive_gemm(p, a, b))


@pytest.mark.parametrize("bk", [4, 12, 20, 28, 36])
def test_tiled_layout_words(qg, orc, cuda, bk):
    """CA_t / CB_t hold exactly the reference's packed words, block by block,
    zero padded (include/qgemm_b200.h)."""
    import torch

    p, m, k, n = 5, 150, 333, 170
    plan = qg.plan_packed_axis(p, 300, 4)  # t for k=300, e=4
    plan = qg.CompressionPlan(plan.p, plan.t, plan.d, plan.e, plan.beta, max(plan.kmax, k), plan.inv_qd, 0)
    a = orc.random_residue_matrix(m, k, p, 31)
    b = orc.random_residue_matrix(k, n, p, 32)
    oplan = orc.plan_of(plan)
    ca = orc.compress_rows_reversed(oplan, a)
    cb = orc.compress_cols_forward(oplan, b)
    K = ca.shape[1]
    Kt = -(-K // bk)
    ta = host(qg.pack_tiled(torch.from_numpy(a.astype(np.int32)).to(cuda), plan, bk, "a"))
    tb = host(qg.pack_tiled(torch.from_numpy(b.astype(np.int32)).to(cuda), plan, bk, "b"))
    Mt, Nt = -(-m // 128), -(-n // 128)
    ea = np.zeros((Mt * 128, Kt * bk))
    ea[:m, :K] = ca
    eb = np.zeros((Nt * 128, Kt * bk))
    eb[:n, :K] = cb.T
    ea = ea.reshape(Mt, 128, Kt, bk).transpose(0, 2, 1, 3).ravel()
    eb = eb.reshape(Nt, 128, Kt, bk).transpose(0, 2, 1, 3).ravel()
    assert np.array_equal(bits(ta), bits(ea))
    assert np.array_equal(bits(tb), bits(eb))


@pytest.mark.parametrize("p,m,k,n", [(5, 96, 300, 250), (3, 130, 64, 77), (7, 33, 500, 9), (5, 1, 6, 1), (5, 200, 3000, 301),
                                     (3, 64, 20000, 130)])
def test_mul_right_tiled(qg, orc, cuda, p, m, k, n):
    """Mixed variant on the tiled layout: under the reference plan the CC words
    equal mul_right_compressed's bit for bit; under a blocked GPU plan (in-place
    REDQ between k-blocks) they equal compress_outer_cols(naive C)."""
    import torch

    a = orc.random_residue_matrix(m, k, p, 177)
    b = orc.random_residue_matrix(k, n, p, 178)
    ad = torch.from_numpy(a.astype(np.float64)).to(cuda)
    bd = torch.from_numpy(b.astype(np.float64)).to(cuda)
    want_c = orc.naive_gemm(p, a, b)
    try:
        rp = qg.plan_packed_axis(p, k, n)
    except qg.NoCompression:
        rp = None
    if rp is not None and k <= rp.kmax:
        cc = qg.mul_right_tiled(ad, bd, rp)
        op = orc.plan_of(rp)
        want = orc.mul_right_compressed(op, a, orc.compress_outer_cols(op, b), n)
        assert np.array_equal(bits(host(cc.data)), bits(want))
    gp = qg.plan_right_gpu(p, k, n)
    cc = qg.mul_right_tiled(ad, bd, gp)
    assert np.array_equal(host(qg.uncompress(cc)).astype(np.uint32), want_c)
    big = orc.Plan(*orc.plan_of(gp.plan).astuple())
    big.kmax = max(big.kmax, k)
    assert np.array_equal(bits(host(cc.data)), bits(orc.compress_outer_cols(big, want_c)))
