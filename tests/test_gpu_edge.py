"""Worst-case parity of the benched plans at their exactness edge
(VERDICT r1 "What's weak" 1-2; the bound-edge test of the
reference is acceptance.cpp:163-221).

The benched plans pack residues in balanced form (v > p/2 enters as v - p,
DESIGN.md §3b), so every product term of a digit lies in [-h^2, h^2], h =
floor(p/2). Eq. G's budget is spent when all terms of all digits share one
sign at full magnitude: residues h and p-h (= +-h) in all-positive and
all-negative products; slot-skewed operands push the largest sums into the
digits below d (or above it) while digit d itself stays 0. Seeded random
inputs, or all-(p-1) (which enters as -1), sit far inside the budget.

Every plan is run at the k-block it is benched with (the largest block its
stage depths allow below Eq. G's maximum) on the main 128x128-tile kernel and
on the small cluster kernel, and C is compared with an exact integer product:
float64 sums of these small integers stay below 2^53, so A @ B in float64 is
exact in any order. Plans asking for one word past Eq. G are refused."""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))["configs"]

# (name, p, k) of the dot-product configs (BASELINE.json configs 1, 2, 3, 5)
COMMON = [("config1", 3, 512), ("config2", 7, 4096), ("config3", 3, 256), ("config5", 3, 32768)]
NPAT = 8


def pattern(idx, p, e, k, rng_seed):
    """Residue vector of length k for pattern `idx` (slot = position mod e)."""
    h = p // 2
    l = np.arange(k)
    slot = l % e
    rng = np.random.default_rng(rng_seed)
    if idx == 0:  # +h everywhere
        v = np.full(k, h)
    elif idx == 1:  # -h everywhere (residue p - h)
        v = np.full(k, p - h)
    elif idx == 2:  # +h on the upper half of the slots only
        v = np.where(slot >= (e + 1) // 2, h, 0)
    elif idx == 3:  # +h on the lower half of the slots only
        v = np.where(slot < (e + 1) // 2, h, 0)
    elif idx == 4:  # random signs at full magnitude
        v = np.where(rng.random(k) < 0.5, h, p - h)
    elif idx == 5:  # sign alternating with the slot
        v = np.where(slot % 2 == 0, h, p - h)
    elif idx == 6:  # all p-1 (the previous "adversarial" input: -1 in balanced form)
        v = np.full(k, p - 1)
    else:  # uniform residues
        v = rng.integers(0, p, k)
    return v.astype(np.int64)


def operands(p, e, m, k, n, seed=0):
    a = np.stack([pattern(r % NPAT, p, e, k, seed + r) for r in range(m)])
    b = np.stack([pattern(c % NPAT, p, e, k, seed + 10007 + c) for c in range(n)], axis=1)
    return a, b


def exact_c(a, b, p):
    import torch

    c = torch.from_numpy(a.astype(np.float64)) @ torch.from_numpy(b.astype(np.float64))
    return (c.numpy().astype(np.int64) % p).astype(np.uint32)


@pytest.fixture
def route(monkeypatch, request):
    monkeypatch.setenv("QG_SMALL", request.param)
    return request.param


@pytest.mark.parametrize("route", ["0", "1"], indirect=True, ids=["main128", "small64"])
@pytest.mark.parametrize("anchored", [True, False], ids=["anchored", "fp64flush"])
@pytest.mark.parametrize("name,p,k", COMMON, ids=[c[0] for c in COMMON])
def test_worst_case_common(qg, cuda, route, name, p, k, anchored):
    """The benched plan (plan_gpu, balanced digits; anchored accumulation K4A
    where the planner picks it, and the FP64-add flush K4) on +-h operands: all
    sign combinations, slot-skewed operands, at the plan's own block."""
    import torch

    gp = qg.plan_gpu(p, k, anchored=anchored)
    pl = gp.plan
    K = -(-k // pl.e)
    if gp.kblock_words < K and gp.anchored:
        # anchored blocks: the largest odd multiple of 4 words the anchored bound
        # (and Eq. 3) allow
        amax, _ = qg.max_exact_block_anchored(pl)
        lim = min(amax, gp.eq3_kmax() // pl.e, 52)
        assert gp.kblock_words <= lim and gp.kblock_words % 8 == 4
        assert gp.kblock_words + 8 > lim, (gp.kblock_words, lim)
    elif gp.kblock_words < K:  # blocked: the block uses >= 90 % of Eq. G's maximum
        assert gp.kblock_words <= gp.max_exact_words
        assert gp.kblock_words >= 0.9 * gp.max_exact_words, (gp.kblock_words, gp.max_exact_words)
    m = n = 256
    a, b = operands(p, pl.e, m, k, n)
    want = exact_c(a, b, p)
    got = qg.mul_common_compressed(torch.from_numpy(a.astype(np.float64)).to(cuda),
                                   torch.from_numpy(b.astype(np.float64)).to(cuda), gp)
    got = got.cpu().numpy().astype(np.uint32)
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{len(bad)} mismatches, first at {bad[:4].tolist()} (row/col pattern " \
                          f"{[(int(r) % NPAT, int(c) % NPAT) for r, c in bad[:4]]})"


@pytest.mark.parametrize("p,k", [(7, 4096), (3, 32768), (5, 8192), (3, 4096)])
@pytest.mark.parametrize("balanced", [True, False])
def test_block_past_eq_g_refused(qg, cuda, p, k, balanced):
    """A plan one word past Eq. G's maximum is refused (NotExact), never
    clamped or rounded into range; one residue past Eq. 3 likewise
    (PlanMismatch). The maximum itself is accepted by the checks."""
    import torch

    gp = qg.plan_gpu(p, k, balanced=balanced, anchored=False)
    pl = gp.plan
    K = -(-k // pl.e)
    if gp.max_exact_words >= K:
        pytest.skip("single-block plan: no block edge at this k")
    a = torch.ones((8, k), dtype=torch.float64, device=cuda)
    b = torch.ones((k, 8), dtype=torch.float64, device=cuda)
    over = qg.GpuPlan(pl, gp.max_exact_words + 1, gp.max_exact_words, gp.balanced)
    kmax_words = gp.eq3_kmax() // pl.e
    # one word past Eq. G; where that block also breaks Eq. 3 (config 5:
    # 23 words x 6 > 127 residues), the Eq. 3 check (PlanMismatch) fires first
    err = qg.PlanMismatch if gp.max_exact_words + 1 > kmax_words else qg.NotExact
    with pytest.raises(err):
        qg.mul_common_compressed(a, b, over)
    with pytest.raises(err):
        qg.mul_common_tiled(a, b, over)
    if kmax_words + 1 <= gp.max_exact_words:
        with pytest.raises(qg.PlanMismatch):
            qg.mul_common_compressed(a, b, qg.GpuPlan(pl, kmax_words + 1, gp.max_exact_words, gp.balanced))
    torch.cuda.synchronize()


def test_balanced_plan_kmax_not_inflated(qg):
    """plan_gpu's plan.kmax is the reference's unsigned Eq. 3 bound
    (plan.hpp:113-115) even for a balanced plan, so reusing gp.plan as a
    CompressionPlan (qg_host_mul_common / gpu_plan_from) checks the right
    bound."""
    for p, k in [(7, 4096), (3, 32768), (3, 256), (5, 8192)]:
        gp = qg.plan_gpu(p, k)
        assert gp.balanced
        assert gp.plan.kmax == ((1 << gp.plan.t) - 1) // (p - 1) ** 2
        assert gp.eq3_kmax() >= gp.plan.kmax
        gf = qg.gpu_plan_from(gp.plan, k)
        assert not gf.balanced and gf.kblock_words * gf.plan.e <= gf.plan.kmax or gf.kblock_words * gf.plan.e >= k


# ------------------------------------------------------------- mixed variant
def right_words(c, t, e):
    """The post-REDQ words of a right product (digits already in [0, p))."""
    m, n = c.shape
    h = -(-n // e)
    cp = np.zeros((m, h * e), dtype=np.uint64)
    cp[:, :n] = c
    w = np.zeros((m, h), dtype=np.uint64)
    for s in range(e):
        w |= cp[:, s::e] << np.uint64(t * s)
    return w


@pytest.mark.parametrize("balanced", [True, False])
def test_worst_case_right(qg, cuda, balanced):
    """Config 4's mixed variant under plan_right_gpu (in-place REDQ every
    kblock residues): +-h operands fill every digit to h + kb h^2 just below
    Q/2 (balanced) or (p-1) + kb (p-1)^2 below Q (unsigned)."""
    import torch

    p, k, n = 5, 8192, 8192
    gp = qg.plan_right_gpu(p, k, n)  # the benched plan: t=13, e=4, unsigned, 504-residue blocks
    pl = gp.plan
    if balanced != bool(gp.balanced):  # the same (t, e) in the other digit form, at its largest block
        h = p // 2 if balanced else p - 1
        lim = (1 << (pl.t - 1)) if balanced else (1 << pl.t)
        kb = (lim - 1 - h) // (h * h)
        bk = ctypes_stage(qg, qg.GpuPlan(pl, kb, kb, int(balanced)), k)
        gp = qg.GpuPlan(pl, kb // bk * bk, kb // bk * bk, int(balanced))
    assert bool(gp.balanced) == balanced
    h = p // 2 if gp.balanced else p - 1
    lim = (1 << (pl.t - 1)) if gp.balanced else (1 << pl.t)
    assert h + gp.kblock_words * h * h < lim
    m, nn = 256, 1024
    a, b = operands(p, 1, m, k, nn, seed=5)
    # the right variant packs B along n: make column patterns depend on the slot too
    b = np.ascontiguousarray(b[:, np.argsort(np.arange(nn) % pl.e, kind="stable")])
    want = exact_c(a, b, p)
    cc = qg.mul_right_tiled(torch.from_numpy(a.astype(np.float64)).to(cuda),
                            torch.from_numpy(b.astype(np.float64)).to(cuda), gp)
    words = cc.data.cpu().numpy().astype(np.uint64)  # exact integer words < 2^53
    assert np.array_equal(words, right_words(want, pl.t, pl.e))
    assert np.array_equal(qg.uncompress(cc).cpu().numpy().astype(np.uint32), want)


def ctypes_stage(qg, gp, k):
    import ctypes

    bk = ctypes.c_uint32()
    g = gp._c()
    qg._check(qg.lib.qg_right_tiled_stage(ctypes.byref(g), k, ctypes.byref(bk)))
    return bk.value


def test_right_block_past_bound_refused(qg, cuda):
    """One residue past the digit bound between in-place REDQs is refused,
    even where rounding the block down to whole stages would hide it."""
    import torch

    p, k = 5, 8192
    gp = qg.plan_right_gpu(p, k, k)
    pl = gp.plan
    h = p // 2 if gp.balanced else p - 1
    lim = (1 << (pl.t - 1)) if gp.balanced else (1 << pl.t)
    kb_max = (lim - 1 - h) // (h * h)
    a = torch.ones((8, k), dtype=torch.float64, device=cuda)
    b = torch.ones((k, 8), dtype=torch.float64, device=cuda)
    with pytest.raises(qg.PlanMismatch):
        qg.mul_right_tiled(a, b, qg.GpuPlan(pl, kb_max + 1, kb_max + 1, gp.balanced))
    qg.mul_right_tiled(a, b, qg.GpuPlan(pl, kb_max, kb_max, gp.balanced))  # the maximum itself runs
    torch.cuda.synchronize()


def test_config4_gpu_plan_full_size(qg, cuda):
    """The benched config-4 plan (plan_right_gpu: t=13, e=4, balanced, blocks
    of 504 residues) at full size: C = uncompress(CC) equals the reference's
    (golden sha256 of C, made by oracle/_ref)."""
    import torch

    g = GOLDEN["config4"]
    p, m, k, n = g["p"], g["m"], g["k"], g["n"]
    gp = qg.plan_right_gpu(p, k, n)
    a = qg.random_residue_matrix(m, k, p, 42)
    b = qg.random_residue_matrix(k, n, p, 43)
    cc = qg.mul_right_tiled(a, b, gp)
    del a, b
    c = qg.uncompress(cc)
    assert qg.residue_checksum(c) == g["checksum"]
    assert hashlib.sha256(np.ascontiguousarray(c.cpu().numpy().astype(np.uint8)).tobytes()).hexdigest() == \
        g["sha256_u8"]
    del cc, c
    torch.cuda.empty_cache()


# ------------------------------------------------------------- config 5, full size
def freivalds(c, a, b, p, vectors=32, seed=7):
    """C == A B (mod p) with probability >= 1 - p^-vectors: C x vs A (B x),
    every product an exact float64 integer sum (< 2^53). Checker only."""
    import torch

    g = torch.Generator(device=c.device).manual_seed(seed)
    x = torch.randint(0, p, (c.shape[1], vectors), generator=g, device=c.device).to(torch.float64)
    cx = torch.remainder(c.to(torch.float64) @ x, p)
    bx = torch.remainder(b.to(torch.float64) @ x, p)
    abx = torch.remainder(a.to(torch.float64) @ bx, p)
    return bool(torch.equal(cx, abx))


@pytest.mark.parametrize("inputs", ["seeded", "worst"])
def test_config5_full_size(qg, cuda, inputs):
    """Config 5 (p=3, 32768^3) under the benched plan over the WHOLE C:
    Freivalds over GF(3) with 32 vectors; the seeded product also matches the
    reference's golden row shards, the worst-case product (+-h row/column
    patterns at the plan's block) exact rows from every 4096-row shard."""
    import torch

    p, m, k, n = 3, 32768, 32768, 32768
    gp = qg.plan_gpu(p, k)
    if inputs == "seeded":
        a = qg.random_residue_matrix(m, k, p, 42)
        b = qg.random_residue_matrix(k, n, p, 43)
    else:
        pa, pb = operands(p, gp.plan.e, NPAT * 4, k, NPAT * 4, seed=11)
        a = torch.from_numpy(pa.astype(np.float64)).to(cuda).repeat(m // (NPAT * 4), 1)
        b = torch.from_numpy(pb.astype(np.float64)).to(cuda).repeat(1, n // (NPAT * 4))
    c = qg.mul_common_compressed(a, b, gp)
    assert freivalds(c, a, b, p)
    if inputs == "seeded":
        for sh in GOLDEN["config5_rows"]["shards"]:
            r0 = sh["row0"]
            blk = c[r0:r0 + sh["rows"]]
            assert qg.residue_checksum(blk) == sh["checksum"], r0
            assert hashlib.sha256(np.ascontiguousarray(blk.cpu().numpy().astype(np.uint8)).tobytes()).hexdigest() \
                == sh["sha256_u8"], r0
    else:
        rows = torch.arange(0, m, 4096 + 7, device=cuda)
        want = torch.remainder(a[rows] @ b, p).to(torch.int32)
        assert torch.equal(c[rows], want)
    del a, b, c
    torch.cuda.empty_cache()
