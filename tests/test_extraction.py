"""extract_coefficient (pack.hpp:78-100) in both extraction modes and
reduce_and_compress (pack.hpp:141-155): the oracle pinned to the reference on
fuzzed words (in-range, boundary, out-of-range, negative), the device kernels
pinned to the oracle bit for bit, and the reference's own cases
(test_pack.cpp:64-73, 224-261) restated."""
import ctypes

import numpy as np
import pytest

import oracle as O

needs_ref = pytest.mark.skipif(O.REF is None, reason="oracle/_ref not built here")
PLANS = [(3, 5, 2), (3, 10, 5), (3, 13, 4), (7, 12, 4), (2, 4, 13), (5, 17, 3), (3, 26, 2), (7, 18, 2)]


def fuzz_words(plan, n, seed):
    rng = np.random.default_rng(seed)
    t, e, d = plan.t, plan.e, plan.d
    exact = [float(int(x)) for x in rng.integers(0, 2 ** min(52, t * e), size=n // 4, dtype=np.uint64)]
    mags = [float(m) * 2.0 ** float(s) for m, s in zip(rng.random(n // 4), rng.integers(-4, 80, size=n // 4))]
    # words just around digit boundaries: k Q^d - 1, k Q^d, k Q^d + 1/2 ulp ...
    edges = []
    for _ in range(n // 4):
        k = int(rng.integers(1, 2 ** t))
        base = float(k) * 2.0 ** (t * d)
        edges += [base, np.nextafter(base, 0.0), np.nextafter(base, np.inf), base - 0.5, base + 2.0 ** (t * d - 1)]
    special = [0.0, -0.0, -1.0, -2.0 ** 40, 2.0 ** 63, 2.0 ** 64, 2.0 ** 70, float("inf"), 2.0 ** (t * (2 * d + 1)),
               2.0 ** (t * (2 * d + 1)) - 1.0]
    return np.array(exact + mags + edges + special, dtype=np.float64)


def with_mode(plan, mode):
    q = O.Plan(*plan.astuple())
    q.extraction = mode
    return q


@needs_ref
@pytest.mark.parametrize("p,t,e", PLANS)
@pytest.mark.parametrize("mode", [0, 1])
def test_oracle_extraction_matches_reference(p, t, e, mode):
    plan = with_mode(O.make_plan(p, t, e), mode)
    out = ctypes.c_uint32()
    for w in fuzz_words(plan, 400, 11 * t + e):
        assert O.REF.qgref_extract_coefficient(ctypes.byref(plan), float(w), ctypes.byref(out)) == 0
        assert O.C.qgo_extract_coefficient(float(w), ctypes.byref(plan)) == out.value, (w, mode)


def test_additive_extraction_agrees_with_reciprocal():  # test_pack.cpp:224-244
    for p, t, e in [(3, 5, 2), (3, 10, 5), (3, 13, 4)]:
        base = O.make_plan(p, t, e)
        add = with_mode(base, 1)
        rng = np.random.default_rng(8080 + t)
        for _ in range(500):
            a = rng.integers(0, p, size=e).astype(np.uint32)
            b = rng.integers(0, p, size=e).astype(np.uint32)
            ra = sum(int(x) << (t * (e - 1 - i)) for i, x in enumerate(a))
            fb = sum(int(x) << (t * i) for i, x in enumerate(b))
            w = float(ra) * float(fb)
            want = ((ra * fb) >> (t * base.d)) & ((1 << t) - 1)
            assert O.C.qgo_extract_coefficient(w, ctypes.byref(add)) == want % p
            assert O.C.qgo_extract_coefficient(w, ctypes.byref(base)) == want % p


@pytest.mark.gpu
@pytest.mark.parametrize("p,t,e", PLANS)
@pytest.mark.parametrize("mode", [0, 1])
def test_device_extraction_bitexact(qg, cuda, p, t, e, mode):
    import torch

    oplan = with_mode(O.make_plan(p, t, e), mode)
    plan = qg.CompressionPlan._from(qg._Plan(*oplan.astuple()))
    words = fuzz_words(oplan, 4000, 7 * t + e + mode)
    got = qg.extract_coefficients(torch.from_numpy(words).to(cuda), plan).cpu().numpy().astype(np.uint32)
    want = np.array([O.C.qgo_extract_coefficient(float(w), ctypes.byref(oplan)) for w in words], np.uint32)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, [(words[i], got[i], want[i]) for i in bad[:5]]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1])
def test_device_reduce_and_compress(qg, cuda, mode):
    import torch

    # test_pack.cpp:247-261: three words of 1156 under make_plan(3, 5, 2) -> [33, 1]
    plan = qg.make_plan(3, 5, 2)
    if mode:
        plan = qg.CompressionPlan._from(qg._Plan(*with_mode(O.plan_of(plan), 1).astuple()))
    cm = qg.reduce_and_compress(torch.full((1, 3), 1156.0, dtype=torch.float64, device=cuda), plan)
    assert cm.data.cpu().tolist() == [[33.0, 1.0]]
    assert qg.reduce_and_compress(torch.zeros((1, 2), dtype=torch.float64, device=cuda), plan).data.cpu().tolist() == [[0.0]]
    # rows of accumulated dot-product words vs the oracle's restatement
    for p, t, e in PLANS:
        oplan = with_mode(O.make_plan(p, t, e), mode)
        words = fuzz_words(oplan, 400, 3 * t).reshape(-1)
        rows, cols = 7, len(words) // 7
        w2 = np.ascontiguousarray(words[: rows * cols].reshape(rows, cols))
        pl = qg.CompressionPlan._from(qg._Plan(*oplan.astuple()))
        got = qg.reduce_and_compress(torch.from_numpy(w2).to(cuda), pl).data.cpu().numpy()
        for r in range(rows):
            groups = -(-cols // e)
            want = np.empty(groups)
            assert O.C.qgo_reduce_and_compress(w2[r].ctypes.data_as(ctypes.c_void_p), cols, ctypes.byref(oplan),
                                               want.ctypes.data_as(ctypes.c_void_p)) == 0
            assert np.array_equal(got[r].view(np.uint64), want.view(np.uint64)), (p, t, e, r)
