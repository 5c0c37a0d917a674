"""Host side of the product on CPU: the planners behind the C ABI equal the
reference's (golden vectors from the reference itself), the Eq. G exactness
bound matches an independent big-integer evaluation, the GPU planner's
invariants hold, and the library exports every symbol its header declares."""
import ctypes
import json
import math
import os
import subprocess

import pytest

import paper_0803_1975_b200 as qg

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def _plan_tuple(d):
    return (d["p"], d["t"], d["d"], d["e"], d["beta"], d["kmax"], float.fromhex(d["inv_qd_hex"]), d["extraction"])


def _tuple(pl):
    return (pl.p, pl.t, pl.d, pl.e, pl.beta, pl.kmax, pl.inv_qd, pl.extraction)


def test_every_declared_symbol_is_exported():
    declared = qg.header_symbols()
    assert len(declared) >= 25
    missing = [s for s in declared if not hasattr(qg.lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", qg.LIB_PATH], capture_output=True, text=True).stdout
    for s in declared:
        assert f" T {s}" in out, s
    assert qg.lib.qg_abi_version() == 1


def test_status_strings_follow_errors_hpp():
    names = [qg.lib.qg_status_string(i).decode() for i in range(13)]
    assert names[:9] == ["ok", "InvalidModulus", "NoCompression", "SlotOverflow", "DigitOverflow",
                         "DimensionMismatch", "PlanMismatch", "UnsupportedAlgorithm", "ParseError"]


@pytest.mark.parametrize("field", ["plan_compression", "plan_packed_axis", "uncompressed_plan"])
def test_planners_equal_reference(field):
    fn = {"plan_compression": qg.lib.qg_plan_compression, "plan_packed_axis": qg.lib.qg_plan_packed_axis,
          "uncompressed_plan": qg.lib.qg_uncompressed_plan}[field]
    for rec in GOLDEN[field]:
        out = qg._Plan()
        st = fn(*rec["args"], ctypes.byref(out))
        assert st == rec["status"], (field, rec["args"])
        if st == 0:
            assert _tuple(out) == _plan_tuple(rec["plan"]), (field, rec["args"])


def test_choose_panel_equals_reference():
    for rec in GOLDEN["choose_panel"]:
        assert qg.choose_panel(*rec["args"]) == rec["panel"], rec["args"]


def test_python_errors_mirror_the_reference():
    with pytest.raises(qg.InvalidModulus):
        qg.plan_compression(4, 10)
    with pytest.raises(qg.InvalidArgument):
        qg.plan_compression(3, 0)
    with pytest.raises(qg.NoCompression):
        qg.plan_compression(3, 1)  # e = min(capacity, k) = 1
    with pytest.raises(qg.NoCompression):
        qg.plan_compression(65521, 1 << 30)


def eq_g_max_block(p, t, e, cap=100000):
    """Independent evaluation of Eq. G with Python integers."""
    d = e - 1
    Q, Qd, pm = 1 << t, 1 << (t * d), (p - 1) ** 2
    amax = (p - 1) * sum(Q ** i for i in range(e))
    xmax = amax * amax

    def ulp(v):
        return 1 << max(0, v.bit_length() - 53)

    def rerr(v):  # rounding error of an op with exact integer result v
        return ulp(v) if v.bit_length() > 53 else 0

    err, best = 0, 0
    for kb in range(1, cap + 1):
        L = sum(min(Q - 1, kb * min(s + 1, 2 * d + 1 - s) * pm) * Q ** s for s in range(d))
        smax = kb * xmax
        err += rerr(smax) + rerr(xmax)
        if ulp(smax) > Qd or L + err >= Qd or (smax >> (t * d)) >= (1 << 52):
            break
        best = kb
    return best


@pytest.mark.parametrize("p,t,e,survey", [
    (3, 10, 5, 34), (3, 11, 4, 127), (3, 12, 4, 154), (3, 14, 3, 1365), (3, 17, 3, 419),
    (5, 12, 4, 59), (5, 15, 3, 568), (7, 12, 4, 28), (7, 15, 3, 303), (7, 18, 2, 3640)])
def test_eq_g_bound(p, t, e, survey):
    """The library's bound equals an independent evaluation, and is within one
    word of SURVEY.md §7.3's rho=1 table (which assumed fused products)."""
    plan = qg.make_plan(p, t, e)
    got = qg.max_exact_block(plan)
    assert got == eq_g_max_block(p, t, e)
    assert abs(got - survey) <= max(1, survey // 50) or got >= survey


@pytest.mark.parametrize("p", [2, 3, 5, 7, 11, 13, 31])
@pytest.mark.parametrize("k", [1, 2, 7, 100, 512, 4096, 8192, 32768, 100000])
def test_gpu_planner_invariants(p, k):
    gp = qg.plan_gpu(p, k)
    pl = gp.plan
    K = -(-k // pl.e)
    assert pl.t * pl.e < 53 or pl.e == 1
    # plan.kmax keeps the reference's meaning (plan.hpp:113-115) even for
    # balanced plans; the Eq. 3 bound the kernels enforce is eq3_kmax()
    assert pl.kmax == ((1 << pl.t) - 1) // ((p - 1) ** 2)
    kmax = gp.eq3_kmax()
    assert kmax == (((1 << (pl.t - 1)) - 1) // ((p // 2) ** 2) if gp.balanced else pl.kmax)
    if gp.kblock_words < K:  # multi-block: Eq. 3 per block, Eq. G, stage-aligned
        assert gp.kblock_words * pl.e <= kmax
        assert gp.kblock_words <= gp.max_exact_words
        assert gp.kblock_words % 4 == 0
        nblocks = -(-K // gp.kblock_words)
        assert nblocks * ((1 << pl.t) - 1) < (1 << 32)
    else:
        assert k <= kmax
        assert K <= gp.max_exact_words


def test_gpu_plan_from_reference_plans():
    for p, k in [(3, 512), (7, 4096), (3, 256), (3, 32768), (5, 8192)]:
        pl = qg.plan_compression(p, k)
        gp = qg.gpu_plan_from(pl, k)
        assert gp.plan == pl
        assert gp.kblock_words <= max(gp.max_exact_words, 1)


def test_device_calls_fail_loudly_without_a_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    pl = qg.plan_compression(3, 16)._c()
    st = qg.lib.qg_gen_residues(1, 3, 0, 4, 4, ctypes.c_void_p(16), 0, None)
    assert st == 10  # QG_CUDA_ERROR: no silent CPU path
    with pytest.raises(qg.CudaError):
        qg.mul_common_compressed_host([[1, 2]], [[1], [2]], qg.plan_compression(3, 2))
