"""The five BASELINE configs on the GPU against golden outputs of the
REFERENCE ITSELF (tests/golden/golden.json, made by make_golden.py through
oracle/_ref): residue checksums (bench.hpp:43-47) and sha256 of the full
result bytes. Config 5 is checked on 32-row slices from each of 8 row shards
(a row of C depends only on that row of A and all of B)."""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))["configs"]


def sha_u8(c):
    return hashlib.sha256(np.ascontiguousarray(c.cpu().numpy().astype(np.uint8)).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["config1", "config3", "config2"])
@pytest.mark.parametrize("planner", ["reference", "gpu"])
def test_common_configs(qg, cuda, name, planner):
    g = GOLDEN[name]
    p, m, k, n = g["p"], g["m"], g["k"], g["n"]
    a = qg.random_residue_matrix(m, k, p, 42)
    b = qg.random_residue_matrix(k, n, p, 43)
    plan = qg.plan_compression(p, k) if planner == "reference" else qg.plan_gpu(p, k)
    c = qg.mul_common_compressed(a, b, plan)
    assert qg.residue_checksum(c) == g["checksum"]
    assert sha_u8(c) == g["sha256_u8"]


def test_config4_mixed_variant(qg, cuda):
    """p=5, 8192^3, right compression: CC words bit-identical to the
    reference's post-REDQ words; C = uncompress(CC) matches its checksum."""
    import torch

    g = GOLDEN["config4"]
    p, m, k, n = g["p"], g["m"], g["k"], g["n"]
    plan = qg.plan_compression(p, k)  # what run_bench uses (bench.hpp:149)
    a = qg.random_residue_matrix(m, k, p, 42)
    b = qg.random_residue_matrix(k, n, p, 43)
    cbo = qg.compress_outer_cols(b, plan)
    del b
    cc = qg.mul_right_compressed(a, cbo)
    words = cc.data.cpu().numpy().view(np.uint64)
    assert hashlib.sha256(np.ascontiguousarray(words).tobytes()).hexdigest() == g["cc_sha256"]
    c = qg.uncompress(cc)
    assert qg.residue_checksum(c) == g["checksum"]
    assert sha_u8(c) == g["sha256_u8"]
    torch.cuda.empty_cache()


@pytest.mark.parametrize("planner", ["gpu", "reference"])
def test_config5_row_shards(qg, cuda, planner):
    """Row-layout operands (compress_rows_reversed / compress_cols_forward words)."""
    import torch

    g = GOLDEN["config5_rows"]
    p, m, k, n = g["p"], g["m"], g["k"], g["n"]
    # reference-layout operands hold the reference's unsigned words
    plan = qg.plan_compression(p, k) if planner == "reference" else qg.plan_gpu(p, k, balanced=False)
    base = plan.plan if isinstance(plan, qg.GpuPlan) else plan
    big = qg.CompressionPlan(base.p, base.t, base.d, base.e, base.beta, max(base.kmax, k), base.inv_qd, 0)
    b = qg.random_residue_matrix(k, n, p, 43)
    cb = qg.compress_cols_forward(b, big)
    cb.plan = base
    del b
    torch.cuda.empty_cache()
    for shard in g["shards"]:
        a = qg.random_residue_matrix(shard["rows"], k, p, 42, row0=shard["row0"])
        ca = qg.compress_rows_reversed(a, big)
        ca.plan = base
        c = qg.mul_common_compressed(ca, cb, plan)
        assert qg.residue_checksum(c) == shard["checksum"], shard["row0"]
        assert sha_u8(c) == shard["sha256_u8"], shard["row0"]
    del cb
    torch.cuda.empty_cache()


def test_config5_row_shards_tiled(qg, cuda):
    """Config 5 through the fast path (tiled layout, balanced GPU plan)."""
    import torch

    g = GOLDEN["config5_rows"]
    p, m, k, n = g["p"], g["m"], g["k"], g["n"]
    gp = qg.plan_gpu(p, k)
    b = qg.random_residue_matrix(k, n, p, 43)
    bk = qg.tiled_stage_words(gp, k)
    cb = qg.pack_tiled(b, gp, bk, "b")
    del b
    import ctypes

    for shard in g["shards"]:
        a = qg.random_residue_matrix(shard["rows"], k, p, 42, row0=shard["row0"])
        ca = qg.pack_tiled(a, gp, bk, "a")
        c = torch.empty((shard["rows"], n), dtype=torch.int32, device=cuda)
        gpc = gp._c()
        qg._check(qg.lib.qg_mul_common_tiled(ctypes.byref(gpc), qg._ptr(ca), qg._ptr(cb), shard["rows"], n, k,
                                             qg._ptr(c), n, qg._stream()))
        assert qg.residue_checksum(c) == shard["checksum"], shard["row0"]
        assert sha_u8(c) == shard["sha256_u8"], shard["row0"]
    del cb
    torch.cuda.empty_cache()
