#!/usr/bin/env python3
"""Generate tests/golden/golden_i64.json from the REFERENCE ITSELF: the
Int64Word backend (word.hpp:36-54) at beta = 63 plans, whose words exceed
2^53 and whose word products wrap modulo 2^64. Computed by the unmodified
reference headers instantiated with Int64Word (oracle/_ref/libqgref.so).

    python tests/golden/make_golden_i64.py
"""
import ctypes
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402
from make_golden import P, plan_dict, ref_mat, sha  # noqa: E402

R = oracle.REF
assert R is not None, "needs oracle/_ref/libqgref.so (make -C oracle ref)"


def main():
    cases = []
    shapes = [(3, 9, 100, 7), (2, 33, 250, 17), (5, 20, 37, 41), (7, 130, 64, 70), (3, 64, 1000, 65), (11, 15, 23, 14),
              (3, 1, 5, 1), (13, 40, 12, 40)]
    for idx, (p, m, k, n) in enumerate(shapes):
        sa, sb = 5000 + idx, 6000 + idx
        a, b = ref_mat(m, k, p, sa), ref_mat(k, n, p, sb)
        pl = oracle.Plan()
        if R.qgref_plan_compression(p, k, 63, 0, ctypes.byref(pl)):
            continue
        case = {"p": p, "m": m, "k": k, "n": n, "seed_a": sa, "seed_b": sb, "plan": plan_dict(pl)}
        acc, c = np.zeros((m, n), np.uint64), np.zeros((m, n), np.uint32)
        assert R.qgref_common_i64(ctypes.byref(pl), P(a), P(b), m, k, n, P(acc), P(c)) == 0
        case["acc_sha"], case["c_sha"] = sha(acc), sha(c)
        K = -(-k // pl.e)
        ca = np.zeros((m, K), np.uint64)
        assert R.qgref_pack_i64(0, ctypes.byref(pl), P(a), m, k, P(ca)) == 0
        case["ca_sha"] = sha(ca)
        case["max_word_bits"] = int(max(int(x) for x in ca.ravel()).bit_length()) if ca.size else 0
        rp = oracle.Plan()
        if R.qgref_plan_packed_axis(p, k, n, 63, ctypes.byref(rp)) == 0:
            H = -(-n // rp.e)
            pre, cc = np.zeros((m, H), np.uint64), np.zeros((m, H), np.uint64)
            assert R.qgref_right_i64(ctypes.byref(rp), P(a), P(b), m, k, n, P(pre), P(cc)) == 0
            case["right_plan"], case["right_pre_sha"], case["right_cc_sha"] = plan_dict(rp), sha(pre), sha(cc)
        lp = oracle.Plan()
        if R.qgref_plan_packed_axis(p, k, m, 63, ctypes.byref(lp)) == 0:
            G = -(-m // lp.e)
            pre, cc = np.zeros((G, n), np.uint64), np.zeros((G, n), np.uint64)
            assert R.qgref_left_i64(ctypes.byref(lp), P(a), P(b), m, k, n, P(pre), P(cc)) == 0
            case["left_plan"], case["left_pre_sha"], case["left_cc_sha"] = plan_dict(lp), sha(pre), sha(cc)
        fp = oracle.FullPlan()
        if R.qgref_plan_full(p, k, 63, ctypes.byref(fp)) == 0:
            cf = np.zeros((m, n), np.uint32)
            assert R.qgref_full_i64(ctypes.byref(fp), P(a), P(b), m, k, n, P(cf)) == 0
            assert np.array_equal(cf, c)
            case["full_plan"] = {"base": plan_dict(fp.base), "dq": fp.dq, "dtheta": fp.dtheta,
                                 "theta_exponent": fp.theta_exponent}
        kp = max(1, (k + 1) // 2)
        bp = oracle.Plan()
        st = R.qgref_plan_compression(p, kp, 63, 0, ctypes.byref(bp)) if kp >= 2 else \
            R.qgref_uncompressed_plan(p, 1, 63, ctypes.byref(bp))
        if st == 0:
            cb = np.zeros((m, n), np.uint32)
            assert R.qgref_blocked_i64(ctypes.byref(bp), P(a), P(b), m, k, n, kp, P(cb)) == 0
            assert np.array_equal(cb, c)
            case["blocked"] = {"kpanel": kp, "plan": plan_dict(bp)}
        cases.append(case)
    json.dump({"source": "reference headers, Int64Word, via oracle/_ref/libqgref.so (tests/golden/make_golden_i64.py)",
               "cases": cases}, open(os.path.join(HERE, "golden_i64.json"), "w"), indent=0)
    print("wrote", len(cases), "cases; max word bits", [c["max_word_bits"] for c in cases])


if __name__ == "__main__":
    main()
