"""K4A — the contraction with anchored accumulators (qg_anchor.cu, DESIGN.md
§3g; packed_common_product + reduce_common_entry + blocked_accumulate,
gemm.hpp:210-271, 450-489): every block length the kernel is built for, at and
below the anchored bound, on the operands that spend the exactness budget
(+-h residues, slot-skewed, random), ragged shapes whose K is not a whole
number of blocks or pipeline slots, against an exact integer product; the same
C as the FP64-flush kernel K4; plans past the anchored bound are refused."""
import numpy as np
import pytest

from test_gpu_edge import exact_c, operands

pytestmark = pytest.mark.gpu

# (p, t, e, block words): hand-built plans that reach every kernel instantiation (12 ... 52 words)
# and the planner's own plans for configs 5 and 2
CASES = [(3, 8, 6, 12), (7, 12, 4, 28), (7, 11, 4, 28), (5, 9, 5, 12), (3, 10, 5, 20), (3, 7, 2, 12), (3, 7, 2, 20),
         (3, 8, 2, 28), (3, 8, 2, 36), (3, 9, 2, 44), (3, 9, 2, 52), (11, 12, 4, 12)]


def anchored_plan(qg, p, t, e, kb):
    pl = qg.make_plan(p, t, e)
    amax, _ = qg.max_exact_block_anchored(pl)
    assert kb <= amax, (p, t, e, kb, amax)
    return qg.GpuPlan(pl, kb, amax, 1, 1)


@pytest.mark.parametrize("p,t,e,kb", CASES, ids=[f"p{c[0]}t{c[1]}e{c[2]}kb{c[3]}" for c in CASES])
@pytest.mark.parametrize("m,n,blocks", [(256, 256, 7), (384, 300, 40), (130, 258, 3)])
def test_anchored_worst_case(qg, cuda, monkeypatch, p, t, e, kb, m, n, blocks):
    import torch

    monkeypatch.setenv("QG_SMALL", "0")
    gp = anchored_plan(qg, p, t, e, kb)
    assert kb * e <= gp.eq3_kmax()
    k = blocks * kb * e - (e // 2 + 1)  # K not a whole number of blocks (nor of 2- / 3-block slots)
    a, b = operands(p, e, m, k, n, seed=kb)
    want = exact_c(a, b, p)
    got = qg.mul_common_compressed(torch.from_numpy(a.astype(np.float64)).to(cuda),
                                   torch.from_numpy(b.astype(np.float64)).to(cuda), gp)
    assert qg.last_kernel() == f"dot_tiled_anchor_kb{kb}_balanced", qg.last_kernel()
    got = got.cpu().numpy().astype(np.uint32)
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{len(bad)} mismatches, first at {bad[:4].tolist()}"


@pytest.mark.parametrize("p,k", [(3, 32768), (7, 4096), (5, 20000), (11, 8192)])
def test_anchored_equals_fp64_flush(qg, orc, cuda, monkeypatch, p, k):
    """The planner's anchored plan and its FP64-flush plan give the same C (= naive_gemm) on
    seeded residues, uint32 and float64 inputs, through the device and the host entry."""
    import torch

    monkeypatch.setenv("QG_SMALL", "0")
    m, n = 300, 520
    a = orc.random_residue_matrix(m, k, p, 11)
    b = orc.random_residue_matrix(k, n, p, 12)
    want = orc.naive_gemm(p, a, b)
    ga, gf = qg.plan_gpu(p, k), qg.plan_gpu(p, k, anchored=False)
    assert ga.anchored and not gf.anchored
    ad = torch.from_numpy(a.astype(np.float64)).to(cuda)
    bd = torch.from_numpy(b.astype(np.float64)).to(cuda)
    ca = qg.mul_common_compressed(ad, bd, ga).cpu().numpy().astype(np.uint32)
    assert "anchor" in qg.last_kernel()
    cf = qg.mul_common_compressed(ad, bd, gf).cpu().numpy().astype(np.uint32)
    assert "anchor" not in qg.last_kernel()
    assert np.array_equal(ca, want) and np.array_equal(cf, want)
    ch = qg.mul_common_compressed_host(a, b, ga)
    assert np.array_equal(np.asarray(ch).astype(np.uint32), want)


def test_anchored_plan_past_bound_refused(qg, cuda):
    """A block longer than the anchored bound is refused (NotExact) even though Eq. G would allow it
    with the FP64 flush; a block length without a kernel is an invalid argument."""
    import torch

    a = torch.ones((8, 4096), dtype=torch.float64, device=cuda)
    b = torch.ones((4096, 8), dtype=torch.float64, device=cuda)
    pl = qg.make_plan(3, 8, 6)
    amax, _ = qg.max_exact_block_anchored(pl)
    assert amax == 15
    with pytest.raises(qg.NotExact):
        qg.mul_common_compressed(a, b, qg.GpuPlan(pl, 20, 22, 1, 1))  # fine for K4 (Eq. G: 22), not anchored
    with pytest.raises(qg.NotExact):
        qg.mul_common_compressed(a, b, qg.GpuPlan(pl, 16, 22, 1, 1))
    ok = qg.mul_common_compressed(a, b, qg.GpuPlan(pl, 20, 22, 1, 0))
    assert int(ok[0, 0]) == 4096 % 3
    pl7 = qg.make_plan(7, 12, 4)
    with pytest.raises(qg.InvalidArgument):
        qg.mul_common_compressed(a, b, qg.GpuPlan(pl7, 24, 53, 1, 1))  # within the bound (28), no kernel
    torch.cuda.synchronize()


@pytest.mark.parametrize("p,k,m,n", [(3, 9000, 200, 260), (7, 4096, 1000, 1030), (5, 20000, 384, 514), (3, 32768, 256, 96)])
def test_anchored_repack(qg, orc, cuda, monkeypatch, p, k, m, n):
    """mul_common_repacked (gemm.hpp:275-280) under an anchored plan: K4A with the fused
    ReduceAndCompress epilogue; CC's words decode to naive_gemm's C and equal the FP64-flush
    kernel's words bit for bit (ragged shapes, e that does not divide 32)."""
    import torch

    monkeypatch.setenv("QG_SMALL", "0")
    a = orc.random_residue_matrix(m, k, p, 31)
    b = orc.random_residue_matrix(k, n, p, 32)
    want = orc.naive_gemm(p, a, b)
    ga = qg.plan_gpu(p, k)
    assert ga.anchored
    gf = qg.GpuPlan(ga.plan, ga.kblock_words, ga.max_exact_words, 1, 0)  # the same blocks, FP64 flush (K4R)
    ad = torch.from_numpy(a.astype(np.float64)).to(cuda)
    bd = torch.from_numpy(b.astype(np.float64)).to(cuda)
    cr = qg.mul_common_repacked(ad, bd, ga)
    assert "repack_anchor" in qg.last_kernel(), qg.last_kernel()
    assert np.array_equal(qg.uncompress(cr).cpu().numpy().astype(np.uint32), want)
    cf = qg.mul_common_repacked(ad, bd, gf)
    assert "anchor" not in qg.last_kernel()
    assert torch.equal(cr.data, cf.data)


def test_anchored_small_entry_accepts_the_plan(qg, orc, cuda, monkeypatch):
    """The small-product kernel (no anchored variant) runs an anchored plan's blocks with the FP64
    flush: same C."""
    import torch

    p, m, k, n = 3, 200, 9000, 260
    a = orc.random_residue_matrix(m, k, p, 21)
    b = orc.random_residue_matrix(k, n, p, 22)
    want = orc.naive_gemm(p, a, b)
    gp = qg.plan_gpu(p, k)
    assert gp.anchored
    ad = torch.from_numpy(a.astype(np.float64)).to(cuda)
    bd = torch.from_numpy(b.astype(np.float64)).to(cuda)
    monkeypatch.setenv("QG_SMALL", "1")
    cs = qg.mul_common_compressed(ad, bd, gp).cpu().numpy().astype(np.uint32)
    assert "anchor" not in qg.last_kernel()
    assert np.array_equal(cs, want)
