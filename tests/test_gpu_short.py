"""Short common dimensions (the packed K fits one pipeline stage — BASELINE
config 3's case; packed_common_product + reduce_common_entry,
gemm.hpp:210-250) through the single-block tiled contraction: interior and
ragged tiles, many tiles per CTA and fewer tiles than CTAs, balanced and
unsigned plans, the static and the dynamic tile schedule, against
naive_gemm."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(qg, cuda, a, b, gp):
    import torch

    c = qg.mul_common_tiled(torch.from_numpy(a.astype(np.float64)).to(cuda),
                            torch.from_numpy(b.astype(np.float64)).to(cuda), gp)
    return c.cpu().numpy().astype(np.uint32), qg.last_kernel()


@pytest.mark.parametrize("p,k", [(3, 256), (3, 100), (7, 200), (5, 8), (3, 30), (13, 150), (2, 300)])
@pytest.mark.parametrize("m,n", [(1024, 2304), (2500, 2100), (130, 4000), (3000, 128), (128, 128)])
@pytest.mark.parametrize("balanced", [True, False], ids=["balanced", "unsigned"])
def test_short_k_parity(qg, orc, cuda, monkeypatch, p, k, m, n, balanced):
    monkeypatch.setenv("QG_SMALL", "0")
    gp = qg.plan_gpu(p, k, balanced=balanced)
    K = -(-k // gp.plan.e)
    if gp.kblock_words < K:
        pytest.skip("multi-block plan")
    a = orc.random_residue_matrix(m, k, p, 5 + m)
    b = orc.random_residue_matrix(k, n, p, 6 + n)
    got, kern = _run(qg, cuda, a, b, gp)
    assert "singleblock" in kern, kern
    assert np.array_equal(got, orc.naive_gemm(p, a, b))


def test_short_static_and_dynamic(qg, orc, cuda, monkeypatch):
    """Config 3's plan on a ragged shape under the static and the dynamic tile schedule; all-(p-1)
    and all-ones rows (the balanced extraction's extremes)."""
    monkeypatch.setenv("QG_SMALL", "0")
    p, k, m, n = 3, 256, 2100, 1700
    gp = qg.plan_gpu(p, k)
    a = orc.random_residue_matrix(m, k, p, 1)
    b = orc.random_residue_matrix(k, n, p, 2)
    a[:300] = p - 1
    b[:, :200] = p - 1
    a[300:600] = 1
    want = orc.naive_gemm(p, a, b)
    c1, k1 = _run(qg, cuda, a, b, gp)
    qg.lib.qg_set_dynamic_tiles(1)
    try:
        c2, k2 = _run(qg, cuda, a, b, gp)
    finally:
        qg.lib.qg_set_dynamic_tiles(0)
    assert np.array_equal(c1, want) and np.array_equal(c2, want)


def test_short_reference_plan(qg, orc, cuda, monkeypatch):
    """The reference's own plan (unsigned digits, one block)."""
    monkeypatch.setenv("QG_SMALL", "0")
    p, k, m, n = 3, 120, 900, 1300
    gp = qg.gpu_plan_from(qg.plan_compression(p, k), k)
    a = orc.random_residue_matrix(m, k, p, 3)
    b = orc.random_residue_matrix(k, n, p, 4)
    got, kern = _run(qg, cuda, a, b, gp)
    assert np.array_equal(got, orc.naive_gemm(p, a, b))
