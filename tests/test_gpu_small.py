"""GPU parity of the small-product contraction (qg_small.cu, reached through
qg_mul_common_compressed / qg_mul_common_tiled): 64x64 tiles on the tiled
packed layout, k stages split over a thread-block cluster reduced through
distributed shared memory. C must equal the oracle's naive_gemm (gemm.hpp:80-100)
residue for residue on every shape, plan, dtype and split count."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def host(t):
    return t.cpu().numpy()


def dev(x, cuda, dtype="f64"):
    import torch

    if dtype == "f64":
        return torch.from_numpy(x.astype(np.float64)).to(cuda)
    return torch.from_numpy(x.astype(np.int32)).to(cuda)


def run(qg, a, b, plan, cuda, dtype="f64"):
    import ctypes

    import torch

    m, k = a.shape
    n = b.shape[1]
    ad, bd = dev(a, cuda, dtype), dev(b, cuda, dtype)
    gp = plan if isinstance(plan, qg.GpuPlan) else qg.gpu_plan_from(plan, k)
    out = torch.full((m, n), -1, dtype=torch.int32, device=cuda)
    g = gp._c()
    qg._check(qg.lib.qg_mul_common_compressed(ctypes.byref(g), qg._ptr(ad), k, qg._ptr(bd), n, qg._dtype_code(ad),
                                              m, k, n, qg._ptr(out), n, qg._stream()))
    torch.cuda.synchronize()
    return host(out).astype(np.uint32), qg.last_kernel()


SHAPES = [
    (3, 512, 512, 512),   # config 1
    (3, 65, 100, 67),     # ragged 64-tiles, odd n
    (5, 1, 1, 1),
    (7, 33, 257, 31),
    (3, 10, 2, 10),       # k < e: one short word
    (2, 130, 700, 64),
    (11, 64, 40, 128),
    (7, 200, 4096, 150),  # k >> the exact block: k-blocks inside every split
    (3, 96, 32768, 96),   # config 5 common dimension
    (5, 17, 8191, 300),
]


@pytest.mark.parametrize("p,m,k,n", SHAPES)
@pytest.mark.parametrize("planner", ["gpu", "gpu_unsigned", "reference"])
def test_small_path_matches_oracle(qg, orc, cuda, monkeypatch, p, m, k, n, planner):
    monkeypatch.setenv("QG_SMALL", "1")
    if planner == "reference":
        try:
            plan = qg.plan_compression(p, k)
        except qg.Error:
            pytest.skip("the reference planner refuses this k")
    else:
        plan = qg.plan_gpu(p, k, balanced=(planner == "gpu"))
    a = orc.random_residue_matrix(m, k, p, 42)
    b = orc.random_residue_matrix(k, n, p, 43)
    got, kern = run(qg, a, b, plan, cuda)
    assert np.array_equal(got, orc.naive_gemm(p, a, b)), kern
    t = plan.plan.t if isinstance(plan, qg.GpuPlan) else plan.t
    if t <= 31:
        assert kern.startswith("small_tiled"), kern
    if (p, m, k, n) == (3, 512, 512, 512):
        from paper_0803_1975_b200 import residue_checksum

        assert residue_checksum(got) == 262622  # README.md:97-99


@pytest.mark.parametrize("splits", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("p,m,k,n", [(3, 130, 2000, 70), (7, 64, 4096, 64), (3, 40, 300, 40)])
def test_small_path_any_split(qg, orc, cuda, monkeypatch, splits, p, m, k, n):
    """Any partition of k into pieces of <= the exact block is exact: every
    cluster size gives the same C (split counts are capped by the stages)."""
    monkeypatch.setenv("QG_SMALL", "1")
    monkeypatch.setenv("QG_SMALL_SPLITS", str(splits))
    a = orc.random_residue_matrix(m, k, p, 7)
    b = orc.random_residue_matrix(k, n, p, 8)
    want = orc.naive_gemm(p, a, b)
    for plan in (qg.plan_gpu(p, k), qg.plan_gpu(p, k, balanced=False)):
        got, kern = run(qg, a, b, plan, cuda)
        assert np.array_equal(got, want), kern


@pytest.mark.parametrize("dtype", ["f64", "i32"])
def test_small_path_dtypes(qg, orc, cuda, monkeypatch, dtype):
    monkeypatch.setenv("QG_SMALL", "1")
    p, m, k, n = 7, 100, 999, 77
    a = orc.random_residue_matrix(m, k, p, 1)
    b = orc.random_residue_matrix(k, n, p, 2)
    got, _ = run(qg, a, b, qg.plan_gpu(p, k), cuda, dtype)
    assert np.array_equal(got, orc.naive_gemm(p, a, b))


@pytest.mark.parametrize("p,k", [(3, 1023), (7, 113), (5, 8192), (3, 32767), (7, 4096)])
def test_small_path_all_max(qg, orc, cuda, monkeypatch, p, k):
    """All residues p-1: every digit and the FP64 magnitude at their maximum."""
    monkeypatch.setenv("QG_SMALL", "1")
    a = np.full((16, k), p - 1, dtype=np.uint32)
    b = np.full((k, 24), p - 1, dtype=np.uint32)
    for plan in (qg.plan_gpu(p, k), qg.plan_gpu(p, k, balanced=False)):
        got, _ = run(qg, a, b, plan, cuda)
        assert (got == (k * (p - 1) ** 2) % p).all()


def test_small_vs_tiled_paths_agree(qg, orc, cuda, monkeypatch):
    """The same product through the small kernel and through the tiled packs
    + contraction (QG_SMALL=0): identical C."""
    import torch

    p, m, k, n = 7, 384, 4096, 384
    a = qg.random_residue_matrix(m, k, p, 42)
    b = qg.random_residue_matrix(k, n, p, 43)
    gp = qg.plan_gpu(p, k)
    monkeypatch.setenv("QG_SMALL", "1")
    c1 = qg.mul_common_compressed(a, b, gp)
    k1 = qg.last_kernel()
    monkeypatch.setenv("QG_SMALL", "0")
    c2 = qg.mul_common_compressed(a, b, gp)
    k2 = qg.last_kernel()
    torch.cuda.synchronize()
    assert k1.startswith("small_tiled") and not k2.startswith("small_tiled"), (k1, k2)
    assert torch.equal(c1, c2)


def test_large_p_one_digit_words(qg, orc, cuda):
    """t > 31 (one residue per word, p = 65521): the entry routes through the
    reference layout; still C = naive_gemm."""
    p, m, k, n = 65521, 40, 300, 50
    a = orc.random_residue_matrix(m, k, p, 3)
    b = orc.random_residue_matrix(k, n, p, 4)
    plan = qg.uncompressed_plan(p, k)
    assert plan.t > 31
    got, _ = run(qg, a, b, plan, cuda)
    assert np.array_equal(got, orc.naive_gemm(p, a, b))
