#!/usr/bin/env python3
"""Generate tests/golden/golden_left_full.json from the REFERENCE ITSELF.

Left and full compression (gemm.hpp:340-445) and plan_full (plan.hpp:229-252)
evaluated by the unmodified reference headers through oracle/_ref/libqgref.so
(oracle/Makefile). Pins the C restatement (tests/test_oracle.py) and the CUDA
path (tests/test_gpu_left_full.py). Run here, where /root/reference exists:

    python tests/golden/make_golden_left_full.py
"""
import ctypes
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402
from make_golden import P, plan_dict, ref_mat, sha, words_hex  # noqa: E402

R = oracle.REF
assert R is not None, "needs oracle/_ref/libqgref.so (make -C oracle ref)"


def full_dict(fp):
    return {"base": plan_dict(fp.base), "dq": fp.dq, "dtheta": fp.dtheta, "theta_exponent": fp.theta_exponent}


def main():
    g = {"source": "reference headers via oracle/_ref/libqgref.so (tests/golden/make_golden_left_full.py)"}
    plans = []
    for p in (2, 3, 5, 7, 11, 13, 251, 8191, 4, 1):
        for k in (1, 2, 3, 7, 10, 40, 100, 250, 256, 1000, 4096, 10000, 16384, 1 << 20):
            for beta in (24, 40, 53, 63):
                fp = oracle.FullPlan()
                st = R.qgref_plan_full(p, k, beta, ctypes.byref(fp))
                plans.append({"args": [p, k, beta], "status": st, "plan": full_dict(fp) if st == 0 else None})
    g["plan_full"] = plans

    cases = []
    shapes = [(3, 2, 2, 2), (3, 7, 13, 9), (5, 9, 10, 8), (7, 17, 31, 19), (2, 40, 40, 40), (11, 12, 23, 14),
              (3, 33, 250, 21), (5, 1, 6, 5), (3, 1, 7, 1), (13, 5, 6, 7), (3, 130, 64, 257), (2, 300, 100, 129)]
    for idx, (p, m, k, n) in enumerate(shapes):
        sa, sb = 3000 + idx, 4000 + idx
        a, b = ref_mat(m, k, p, sa), ref_mat(k, n, p, sb)
        case = {"p": p, "m": m, "k": k, "n": n, "seed_a": sa, "seed_b": sb, "a_sha": sha(a), "b_sha": sha(b)}
        c = np.empty((m, n), np.uint32)
        R.qgref_naive_gemm(p, P(a), P(b), m, k, n, P(c))
        case["c_sha"] = sha(c)
        lp = oracle.Plan()
        if R.qgref_plan_packed_axis(p, k, m, 53, ctypes.byref(lp)) == 0:
            cc = np.empty((-(-m // lp.e), n))
            assert R.qgref_mul_left(ctypes.byref(lp), P(a), P(b), m, k, n, P(cc)) == 0
            case["left_plan"] = plan_dict(lp)
            case["left_cc"] = words_hex(cc)
        fp = oracle.FullPlan()
        st = R.qgref_plan_full(p, k, 53, ctypes.byref(fp))
        case["full_status"] = st
        if st == 0:
            cf = np.empty((m, n), np.uint32)
            assert R.qgref_mul_full(ctypes.byref(fp), P(a), P(b), m, k, n, P(cf)) == 0
            assert np.array_equal(cf, c)
            case["full_plan"] = full_dict(fp)
        cases.append(case)
    g["cases"] = cases
    with open(os.path.join(HERE, "golden_left_full.json"), "w") as f:
        json.dump(g, f, indent=0)
    print("wrote", len(plans), "plans,", len(cases), "cases")


if __name__ == "__main__":
    main()
