"""GPU parity of the two-dimensional host pipeline (qg_abi.cu host_pipeline2d:
A in row chunks and B in column panels interleaved over PCIe, one contraction
per (chunk, panel) tile, 2-D copies of each tile's output), forced on with
QG_HOST_2D=1 on ragged shapes, against the oracle: C = naive_gemm
(gemm.hpp:80-100) for the dot-product variant, CC words bit-identical to
mul_right_compressed (gemm.hpp:320-335) for the mixed variant."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("p,m,k,n", [(3, 700, 300, 1000), (7, 1300, 4096, 515), (5, 129, 2000, 4099), (3, 2048, 256, 640)])
@pytest.mark.parametrize("panels,tiles", [("4", "96"), ("2", "8"), ("3", "1")])
def test_host_common_2d(qg, orc, cuda, monkeypatch, p, m, k, n, panels, tiles):
    monkeypatch.setenv("QG_HOST_2D", "1")
    monkeypatch.setenv("QG_HOST_PANELS", panels)
    monkeypatch.setenv("QG_HOST_TILES", tiles)
    a = orc.random_residue_matrix(m, k, p, 11)
    b = orc.random_residue_matrix(k, n, p, 12)
    want = orc.naive_gemm(p, a, b)
    for plan in (qg.plan_gpu(p, k), qg.plan_gpu(p, k, balanced=False)):
        assert np.array_equal(qg.mul_common_compressed_host(a, b, plan), want)


@pytest.mark.parametrize("p,m,k,n", [(5, 700, 1000, 3000), (3, 300, 257, 2049), (7, 1100, 600, 700)])
@pytest.mark.parametrize("panels", ["4", "2"])
def test_host_right_2d(qg, orc, cuda, monkeypatch, p, m, k, n, panels):
    monkeypatch.setenv("QG_HOST_2D", "1")
    monkeypatch.setenv("QG_HOST_PANELS", panels)
    monkeypatch.setenv("QG_HOST_TILES", "8")
    a = orc.random_residue_matrix(m, k, p, 21)
    b = orc.random_residue_matrix(k, n, p, 22)
    rp = qg.plan_packed_axis(p, k, n)
    oplan = orc.plan_of(rp)
    want = orc.mul_right_compressed(oplan, a, orc.compress_outer_cols(oplan, b), n)
    assert np.array_equal(bits(qg.mul_right_compressed_host(a, b, rp)), bits(want))
    gp = qg.plan_right_gpu(p, k, n)
    got = qg.mul_right_compressed_host(a, b, gp)
    # a blocked plan has its own (t, e): compare through the residues
    e = gp.plan.e
    digits = np.zeros((m, ((n + e - 1) // e) * e), dtype=np.uint64)
    w = got.astype(np.uint64)
    for s in range(e):
        digits[:, s::e] = (w >> np.uint64(gp.plan.t * s)) & np.uint64((1 << gp.plan.t) - 1)
    assert np.array_equal(digits[:, :n].astype(np.uint32), orc.naive_gemm(p, a, b))


@pytest.mark.parametrize("p,m,k,n,parts", [(5, 700, 5000, 3000, "8"), (3, 300, 4000, 2049, "3"), (7, 1100, 3000, 700, "2")])
def test_host_right_ksplit(qg, orc, cuda, monkeypatch, p, m, k, n, parts):
    """The k-split host path of the mixed variant (host_right_ksplit: parts of
    k contracted in turn, the accumulators continuing from the previous
    parts' REDQ'd words): the CC words of a blocked GPU plan decode to
    naive_gemm's C."""
    monkeypatch.setenv("QG_HOST_KSPLIT", "1")
    monkeypatch.setenv("QG_HOST_KPARTS", parts)
    a = orc.random_residue_matrix(m, k, p, 41)
    b = orc.random_residue_matrix(k, n, p, 42)
    gp = qg.plan_right_gpu(p, k, n)
    if gp.balanced:
        gp = qg.GpuPlan(gp.plan, gp.kblock_words, gp.max_exact_words, 0)
    got = qg.mul_right_compressed_host(a, b, gp)
    e = gp.plan.e
    digits = np.zeros((m, ((n + e - 1) // e) * e), dtype=np.uint64)
    w = got.astype(np.uint64)
    for s in range(e):
        digits[:, s::e] = (w >> np.uint64(gp.plan.t * s)) & np.uint64((1 << gp.plan.t) - 1)
    assert np.array_equal(digits[:, :n].astype(np.uint32), orc.naive_gemm(p, a, b))


@pytest.mark.parametrize("p,m,k,n,parts", [(5, 700, 5000, 3000, "8"), (7, 1100, 3000, 700, "2"), (3, 2100, 3100, 300, "3")])
def test_host_left_ksplit(qg, orc, cuda, monkeypatch, p, m, k, n, parts):
    """The k-split host path of the left variant: CC words (digit s of
    CC[g][j] = C[g e + s][j]) decode to naive_gemm's C."""
    monkeypatch.setenv("QG_HOST_KSPLIT", "1")
    monkeypatch.setenv("QG_HOST_KPARTS", parts)
    a = orc.random_residue_matrix(m, k, p, 51)
    b = orc.random_residue_matrix(k, n, p, 52)
    gp = qg.plan_right_gpu(p, k, m)
    if gp.balanced:
        gp = qg.GpuPlan(gp.plan, gp.kblock_words, gp.max_exact_words, 0)
    got = qg.mul_left_compressed_host(a, b, gp)
    e = gp.plan.e
    w = got.astype(np.uint64)
    c = np.zeros((((m + e - 1) // e) * e, n), dtype=np.uint64)
    for s in range(e):
        c[s::e, :] = (w >> np.uint64(gp.plan.t * s)) & np.uint64((1 << gp.plan.t) - 1)
    assert np.array_equal(c[:m].astype(np.uint32), orc.naive_gemm(p, a, b))

