"""Anchored accumulation (K4A) on CPU: the library's bound
equals an independent big-integer evaluation; the scheme itself — start
every k-block from A0 = 1.5 2^E + Q^d/2 + Q^(d+1)/2, read digit d from fixed
bits of the result — is exact under ANY faithful rounding of every product
and every add (emulated with integers: always down, always up, nearest) on the
operands that spend the budget, at the largest block the bound allows; the
planner's anchored plans respect the bound, Eq. 3 and the kernel's block
lengths."""
import numpy as np
import pytest

import paper_0803_1975_b200 as qg


def _bitlen(v):
    return int(v).bit_length()


def _ulp(v):
    b = _bitlen(abs(v))
    return 1 << (b - 53) if b > 53 else 1


def anchored_exponent(p, t, e, kb):
    """Independent restatement of the bound."""
    d = e - 1
    h = p // 2
    if t < 2 or d < 1 or h == 0 or t * e > 53:
        return 0
    Q, Qd = 1 << t, 1 << (t * d)
    amax = sum(h << (t * i) for i in range(e))
    xmax = amax * amax
    err_x = _ulp(xmax) if _bitlen(xmax) > 53 else 0
    off = Qd // 2 + (Qd << t) // 2 + (Qd << t)
    L = sum(min(kb * min(s + 1, 2 * d + 1 - s) * h * h, Q // 2 - 1) << (t * s) for s in range(d))
    for E in range(max(_bitlen(kb * xmax) + 1, 53), t * d + 52):
        u = 1 << (E - 52)
        err = kb * (u + err_x)
        if off + kb * xmax + err >= 1 << (E - 1):
            continue
        s = t * d - (E - 52)
        if s + t > 32:
            continue
        return E if (s >= 1 and 2 * (L + err) < Qd) else 0
    return 0


PLANS = [(3, 8, 6), (7, 12, 4), (7, 11, 4), (3, 10, 5), (5, 12, 4), (5, 9, 5), (3, 9, 5), (11, 12, 4), (13, 12, 4),
         (31, 15, 3), (3, 7, 2), (3, 8, 2), (3, 9, 2), (2, 8, 6), (251, 23, 2), (17, 16, 3), (7, 13, 4)]


@pytest.mark.parametrize("p,t,e", PLANS)
def test_anchored_bound_equals_independent_evaluation(p, t, e):
    pl = qg.make_plan(p, t, e)
    words, E = qg.max_exact_block_anchored(pl)
    ok = [kb for kb in range(1, 400) if anchored_exponent(p, t, e, kb)]
    assert words == (max(ok) if ok else 0)
    assert E == (anchored_exponent(p, t, e, words) if words else 0)


def test_anchored_bound_known_values():
    """Hand-checked: config 5's plan 15 words in binade 85, config 2's 28 in 81."""
    assert qg.max_exact_block_anchored(qg.make_plan(3, 8, 6)) == (15, 85)
    assert qg.max_exact_block_anchored(qg.make_plan(7, 12, 4)) == (28, 81)


def _round(v, g, mode):
    """v rounded onto the grid g Z: toward -inf, +inf or to nearest (ties away)."""
    if g == 1:
        return v
    if mode == "down":
        return (v // g) * g
    if mode == "up":
        return -((-v) // g) * g
    return ((2 * v + g) // (2 * g)) * g


def _words(p, t, e, digits):
    """Balanced packed words of digit rows (n x e): A reversed, B forward share the form sum v Q^i."""
    h = p // 2
    v = np.where(digits > h, digits - p, digits).astype(object)
    return [sum(int(v[r, i]) << (t * i) for i in range(e)) for r in range(v.shape[0])]


@pytest.mark.parametrize("p,t,e", [(3, 8, 6), (7, 12, 4), (5, 9, 5), (3, 10, 5), (7, 11, 4), (11, 12, 4)])
@pytest.mark.parametrize("mode", ["down", "up", "nearest"])
def test_anchored_scheme_exact_under_any_faithful_rounding(p, t, e, mode):
    """One block of the largest exact length, products rounded (unfused) and
    added to the anchored accumulator with directed rounding: the digit field
    of the result is D_d + Q/2 for all-(+h), all-(-h), slot-skewed, alternating
    and random operands."""
    pl = qg.make_plan(p, t, e)
    kb, E = qg.max_exact_block_anchored(pl)
    assert kb >= 4
    d, Q, h = e - 1, 1 << t, p // 2
    u = 1 << (E - 52)
    s = t * d - (E - 52)
    A0 = 3 * (1 << (E - 1)) + (1 << (t * d - 1)) + (1 << (t * d + t - 1))
    rng = np.random.default_rng(p * 1000 + t)
    slot = np.arange(e)
    pats = [np.full((kb, e), h), np.full((kb, e), p - h), np.tile(np.where(slot >= (e + 1) // 2, h, 0), (kb, 1)),
            np.tile(np.where(slot < (e + 1) // 2, h, 0), (kb, 1)), np.tile(np.where(slot % 2 == 0, h, p - h), (kb, 1)),
            np.where(rng.random((kb, e)) < 0.5, h, p - h), rng.integers(0, p, (kb, e))]
    for pa in pats:
        for pb in pats:
            # A's word holds a row segment reversed, B's a column segment forward: digit d of a
            # word product is the dot product of the two segments
            wa = _words(p, t, e, pa[:, ::-1])
            wb = _words(p, t, e, pb)
            for anchor in (A0, A0 + (1 << (t * d + t))):
                acc = anchor
                for x, y in zip(wa, wb):
                    prod = _round(x * y, _ulp(x * y), mode)
                    acc = _round(acc + prod, u, mode)
                    assert (1 << E) <= acc < (1 << (E + 1))
                field = ((acc // u) >> s) & (Q - 1)
                va = np.where(pa > h, pa - p, pa)
                vb = np.where(pb > h, pb - p, pb)
                D = int((va * vb).sum())
                assert field == (D + Q // 2) % Q, (mode, D, field)
                assert (D % p) == (int((pa * pb).sum()) % p)


@pytest.mark.parametrize("p,k", [(3, 32768), (7, 4096), (5, 100000), (11, 8192), (3, 1200), (3, 100000)])
def test_planner_anchored_plans(p, k):
    gp = qg.plan_gpu(p, k)
    pl = gp.plan
    K = -(-k // pl.e)
    assert gp.anchored and gp.balanced
    amax, E = qg.max_exact_block_anchored(pl)
    assert gp.kblock_words % 8 == 4 and 12 <= gp.kblock_words <= min(amax, 52)
    assert gp.kblock_words * pl.e <= gp.eq3_kmax() or k <= gp.eq3_kmax()
    assert 16 * gp.kblock_words <= K
    assert anchored_exponent(p, pl.t, pl.e, gp.kblock_words)
    assert gp.kblock_words <= gp.max_exact_words  # an anchored block is always within Eq. G
    plain = qg.plan_gpu(p, k, anchored=False)
    assert not plain.anchored


def test_planner_config_plans():
    """The benched plans: config 5 (p=3, 32768) t=8 e=6 in 12-word anchored blocks, config 2
    (p=7, 4096) e=4 in 28-word anchored blocks; the short products (configs 1, 3) keep their
    single-block plans."""
    g5 = qg.plan_gpu(3, 32768)
    assert (g5.plan.t, g5.plan.e, g5.kblock_words, g5.anchored) == (8, 6, 12, 1)
    g2 = qg.plan_gpu(7, 4096)
    assert (g2.plan.e, g2.kblock_words, g2.anchored) == (4, 28, 1)
    for p, k in [(3, 512), (3, 256)]:
        assert not qg.plan_gpu(p, k).anchored
