"""The tiled contraction kernels with the dynamic tile schedule
(qg_set_dynamic_tiles / QG_DYN): tiles claimed from a per-launch atomic
counter instead of every gridDim.x-th tile. The results must be the same
words / residues as under the static schedule, including launches that run
concurrently on several streams (separate counters) and launches captured
into a CUDA graph and replayed (the counter's memset is a graph node)."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture
def dynamic(qg):
    qg.lib.qg_set_dynamic_tiles(1)
    yield
    qg.lib.qg_set_dynamic_tiles(0)


@pytest.mark.parametrize("p,m,k,n", [(7, 1000, 4096, 1030), (3, 1280, 256, 2048), (3, 384, 32768, 512)])
def test_dynamic_common(qg, orc, cuda, dynamic, p, m, k, n, monkeypatch):
    import torch

    monkeypatch.setenv("QG_SMALL", "0")
    a = orc.random_residue_matrix(m, k, p, 1)
    b = orc.random_residue_matrix(k, n, p, 2)
    gp = qg.plan_gpu(p, k)
    got = qg.mul_common_compressed(torch.from_numpy(a.astype(np.float64)).to(cuda),
                                   torch.from_numpy(b.astype(np.float64)).to(cuda), gp)
    assert np.array_equal(got.cpu().numpy().astype(np.uint32), orc.naive_gemm(p, a, b))


def test_dynamic_right_and_repack(qg, orc, cuda, dynamic):
    import torch

    p, m, k, n = 5, 700, 3000, 900
    a = orc.random_residue_matrix(m, k, p, 3)
    b = orc.random_residue_matrix(k, n, p, 4)
    want = orc.naive_gemm(p, a, b)
    ad = torch.from_numpy(a.astype(np.float64)).to(cuda)
    bd = torch.from_numpy(b.astype(np.float64)).to(cuda)
    cc = qg.mul_right_tiled(ad, bd, qg.plan_right_gpu(p, k, n))
    assert np.array_equal(qg.uncompress(cc).cpu().numpy().astype(np.uint32), want)
    cr = qg.mul_common_repacked(ad, bd, qg.plan_gpu(p, k))
    assert np.array_equal(qg.uncompress(cr).cpu().numpy().astype(np.uint32), want)


def test_dynamic_concurrent_streams_and_graph(qg, orc, cuda, dynamic, monkeypatch):
    """Four products at once on four streams, then a captured graph replayed
    three times: every launch owns its counter."""
    import torch

    monkeypatch.setenv("QG_SMALL", "0")
    p, k = 7, 4096
    gp = qg.plan_gpu(p, k)
    bk = qg.tiled_stage_words(gp, k)
    g = gp._c()
    jobs = []
    for i in range(4):
        m, n = 512 + 128 * i, 640
        a = orc.random_residue_matrix(m, k, p, 10 + i)
        b = orc.random_residue_matrix(k, n, p, 20 + i)
        ca = qg.pack_tiled(torch.from_numpy(a.astype(np.float64)).to(cuda), gp, bk, "a")
        cb = qg.pack_tiled(torch.from_numpy(b.astype(np.float64)).to(cuda), gp, bk, "b")
        c = torch.empty((m, n), dtype=torch.int32, device=cuda)
        jobs.append((a, b, ca, cb, c, torch.cuda.Stream()))
    torch.cuda.synchronize()
    for a, b, ca, cb, c, s in jobs:
        qg._check(qg.lib.qg_mul_common_tiled(ctypes.byref(g), qg._ptr(ca), qg._ptr(cb), a.shape[0], b.shape[1], k,
                                             qg._ptr(c), b.shape[1], ctypes.c_void_p(s.cuda_stream)))
    torch.cuda.synchronize()
    for a, b, ca, cb, c, s in jobs:
        assert np.array_equal(c.cpu().numpy().astype(np.uint32), orc.naive_gemm(p, a, b))
    a, b, ca, cb, c, s = jobs[0]
    c.zero_()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        qg._check(qg.lib.qg_mul_common_tiled(ctypes.byref(g), qg._ptr(ca), qg._ptr(cb), a.shape[0], b.shape[1], k,
                                             qg._ptr(c), b.shape[1], qg._stream()))
    want = orc.naive_gemm(p, a, b)
    for _ in range(3):
        c.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert np.array_equal(c.cpu().numpy().astype(np.uint32), want)
