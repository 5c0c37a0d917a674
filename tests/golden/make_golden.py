#!/usr/bin/env python3
"""Generate tests/golden/golden.json from the REFERENCE ITSELF.

Every value below is computed by the unmodified reference headers
(/root/reference/proj/include/qgemm, compiled into oracle/_ref/libqgref.so by
oracle/Makefile) — nothing comes from this repo's oracle or kernels. The
file pins both the C restatement (tests/test_oracle.py) and the CUDA path
(tests/test_gpu_golden.py). Run here (where /root/reference exists):

    python tests/golden/make_golden.py

Large outputs are stored as a checksum (residue_checksum, bench.hpp:43-47)
plus a sha256 of the raw bytes, small ones in full.
"""
import ctypes
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

R = oracle.REF
assert R is not None, "needs oracle/_ref/libqgref.so (make -C oracle ref)"
vp = ctypes.c_void_p
THREADS = oracle.threads()


def P(a):
    return a.ctypes.data_as(vp)


def ref_plan(p, k, beta=53, mode=0):
    pl = oracle.Plan()
    st = R.qgref_plan_compression(p, k, beta, mode, ctypes.byref(pl))
    return st, pl


def ref_mat(rows, cols, p, seed):
    out = np.empty((rows, cols), dtype=np.uint32)
    R.qgref_random_residue_matrix(rows, cols, p, seed, P(out))
    return out


def words_hex(w):
    return [format(int(x), "016x") for x in np.ascontiguousarray(w, np.float64).view(np.uint64).ravel()]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def checksum(c):
    return int(np.asarray(c, np.uint64).sum() & 0xFFFFFFFF)


def plan_dict(pl):
    return {"p": pl.p, "t": pl.t, "d": pl.d, "e": pl.e, "beta": pl.beta, "kmax": pl.kmax,
            "inv_qd_hex": float(pl.inv_qd).hex(), "extraction": pl.extraction}


def main():
    t0 = time.time()
    g = {"source": "reference headers via oracle/_ref/libqgref.so (tests/golden/make_golden.py)"}

    # ---- planners (plan.hpp:125-224)
    plans = []
    for p in (2, 3, 5, 7, 11, 13, 31, 65521, 4, 1):
        for k in (1, 2, 3, 7, 8, 15, 31, 63, 100, 200, 255, 256, 512, 1000, 2047, 4096, 8192, 32767, 32768, 1 << 20, 1 << 30):
            for beta in (53, 63, 24):
                for mode in (0, 1):
                    st, pl = ref_plan(p, k, beta, mode)
                    plans.append({"args": [p, k, beta, mode], "status": st, "plan": plan_dict(pl) if st == 0 else None})
    g["plan_compression"] = plans
    axis = []
    for p in (2, 3, 5, 7, 11):
        for k in (1, 6, 100, 8192, 1 << 20):
            for ax in (1, 2, 3, 5, 8192):
                pl = oracle.Plan()
                st = R.qgref_plan_packed_axis(p, k, ax, 53, ctypes.byref(pl))
                axis.append({"args": [p, k, ax, 53], "status": st, "plan": plan_dict(pl) if st == 0 else None})
    g["plan_packed_axis"] = axis
    un = []
    for p in (2, 3, 7):
        for k in (1, 5, 1000):
            pl = oracle.Plan()
            st = R.qgref_uncompressed_plan(p, k, 53, ctypes.byref(pl))
            un.append({"args": [p, k, 53], "status": st, "plan": plan_dict(pl) if st == 0 else None})
    g["uncompressed_plan"] = un
    panels = []
    for p in (2, 3, 5, 7, 11):
        for k in (1, 2, 7, 100, 512, 4096, 8192, 32768):
            out = ctypes.c_uint64()
            st = R.qgref_choose_panel(p, k, 53, ctypes.byref(out))
            panels.append({"args": [p, k, 53], "status": st, "panel": out.value})
    g["choose_panel"] = panels

    # ---- small seeded cases: every packing, the accumulators, C, mixed CC, blocked C
    cases = []
    rng = np.random.default_rng(2024)
    shapes = [(3, 2, 2, 2), (3, 7, 13, 9), (7, 7, 13, 9), (5, 17, 31, 19), (2, 9, 40, 11), (11, 12, 23, 14),
              (3, 33, 255, 21), (7, 16, 113, 16), (13, 5, 6, 7), (3, 1, 1, 1)]
    for idx, (p, m, k, n) in enumerate(shapes):
        sa, sb = 1000 + idx, 2000 + idx
        a, b = ref_mat(m, k, p, sa), ref_mat(k, n, p, sb)
        st, pl = ref_plan(p, k)
        case = {"p": p, "m": m, "k": k, "n": n, "seed_a": sa, "seed_b": sb,
                "a_sha": sha(a), "b_sha": sha(b)}
        c = np.empty((m, n), np.uint32)
        R.qgref_naive_gemm(p, P(a), P(b), m, k, n, P(c))
        case["c"] = c.ravel().tolist()
        if st == 0:
            case["plan"] = plan_dict(pl)
            K = -(-k // pl.e)
            ca, cb = np.empty((m, K)), np.empty((K, n))
            assert R.qgref_compress_rows_reversed(ctypes.byref(pl), P(a), m, k, P(ca)) == 0
            assert R.qgref_compress_cols_forward(ctypes.byref(pl), P(b), k, n, P(cb)) == 0
            acc = np.empty((m, n))
            assert R.qgref_packed_common_product(ctypes.byref(pl), P(a), P(b), m, k, n, P(acc)) == 0
            case["ca"], case["cb"], case["acc"] = words_hex(ca), words_hex(cb), words_hex(acc)
            cc_c = np.empty((m, n), np.uint32)
            mm, cv = ctypes.c_double(), ctypes.c_double()
            assert R.qgref_mul_common(ctypes.byref(pl), P(a), P(b), m, k, n, P(cc_c), 1, ctypes.byref(mm), ctypes.byref(cv)) == 0
            assert np.array_equal(cc_c, c)
        rp = oracle.Plan()
        if R.qgref_plan_packed_axis(p, k, n, 53, ctypes.byref(rp)) == 0:
            H = -(-n // rp.e)
            cbo = np.empty((k, H))
            assert R.qgref_compress_outer_cols(ctypes.byref(rp), P(b), k, n, P(cbo)) == 0
            cc = np.empty((m, H))
            cu = np.empty((m, n), np.uint32)
            mm, cv = ctypes.c_double(), ctypes.c_double()
            assert R.qgref_mul_right(ctypes.byref(rp), P(a), P(b), m, k, n, P(cc), P(cu), 1, ctypes.byref(mm), ctypes.byref(cv)) == 0
            case["right_plan"] = plan_dict(rp)
            case["cbo"], case["cc"] = words_hex(cbo), words_hex(cc)
            assert np.array_equal(cu, c)
            cao = np.empty((-(-m // rp.e), k))
            assert R.qgref_compress_outer_rows(ctypes.byref(rp), P(a), m, k, P(cao)) == 0
            case["cao"] = words_hex(cao)
        kp = max(1, k // 2)
        bp = oracle.Plan()
        if kp >= 2:
            stb = R.qgref_plan_compression(p, kp, 53, 0, ctypes.byref(bp))
        else:
            stb = R.qgref_uncompressed_plan(p, 1, 53, ctypes.byref(bp))
        if stb == 0:
            cbk = np.empty((m, n), np.uint32)
            assert R.qgref_blocked_accumulate(ctypes.byref(bp), P(a), P(b), m, k, n, kp, P(cbk)) == 0
            assert np.array_equal(cbk, c)
            case["blocked"] = {"kpanel": kp, "plan": plan_dict(bp)}
        cases.append(case)
    g["cases"] = cases

    # ---- BASELINE configs at seed 42 (A = seed, B = seed+1, bench.hpp:70-71)
    cfg = {}

    def common(name, p, m, k, n, rows=None):
        st, pl = ref_plan(p, k)
        r0 = 0
        mm = m if rows is None else rows
        a = ref_mat(m, k, p, 42)[:mm] if m * k <= (1 << 28) else oracle.random_residue_matrix(mm, k, p, 42)
        b = ref_mat(k, n, p, 43)
        c = np.empty((mm, n), np.uint32)
        s_mul, s_conv = ctypes.c_double(), ctypes.c_double()
        t = time.time()
        assert R.qgref_mul_common(ctypes.byref(pl), P(a), P(b), mm, k, n, P(c), THREADS, ctypes.byref(s_mul), ctypes.byref(s_conv)) == 0
        cfg[name] = {"p": p, "m": m, "k": k, "n": n, "rows": [r0, mm], "plan": plan_dict(pl),
                     "checksum": checksum(c), "sha256_u8": sha(c.astype(np.uint8)),
                     "row0_head": c[0, :64].tolist(), "ref_seconds": time.time() - t, "threads": THREADS}
        print(name, cfg[name]["checksum"], f"{time.time() - t:.1f}s", flush=True)

    common("config1", 3, 512, 512, 512)
    common("config3", 3, 8192, 256, 8192)
    common("config2", 7, 4096, 4096, 4096)
    # config 5: rows sampled from every one of 8 row shards (32 rows each)
    p, m, k, n = 3, 32768, 32768, 32768
    st, pl = ref_plan(p, k)
    b = oracle.random_residue_matrix(k, n, p, 43)
    shards = []
    t = time.time()
    for r in range(8):
        r0 = r * (m // 8)
        a = oracle.random_residue_matrix(32, k, p, 42, row0=r0)
        c = np.empty((32, n), np.uint32)
        s_mul, s_conv = ctypes.c_double(), ctypes.c_double()
        assert R.qgref_mul_common(ctypes.byref(pl), P(a), P(b), 32, k, n, P(c), THREADS, ctypes.byref(s_mul), ctypes.byref(s_conv)) == 0
        shards.append({"row0": r0, "rows": 32, "checksum": checksum(c), "sha256_u8": sha(c.astype(np.uint8))})
    cfg["config5_rows"] = {"p": p, "m": m, "k": k, "n": n, "plan": plan_dict(pl), "shards": shards,
                           "ref_seconds": time.time() - t}
    print("config5 rows", time.time() - t, flush=True)
    # config 4: mixed variant (bench.hpp:148-165: plan_compression, compress_outer_cols,
    # packed_right_product, redq_in_place, uncompress) on all rows
    p, m, k, n = 5, 8192, 8192, 8192
    st, pl = ref_plan(p, k)
    a = oracle.random_residue_matrix(m, k, p, 42)
    b = oracle.random_residue_matrix(k, n, p, 43)
    H = -(-n // pl.e)
    cc = np.empty((m, H))
    cu = np.empty((m, n), np.uint32)
    s_mul, s_conv = ctypes.c_double(), ctypes.c_double()
    t = time.time()
    assert R.qgref_mul_right(ctypes.byref(pl), P(a), P(b), m, k, n, P(cc), P(cu), THREADS, ctypes.byref(s_mul), ctypes.byref(s_conv)) == 0
    cfg["config4"] = {"p": p, "m": m, "k": k, "n": n, "plan": plan_dict(pl), "checksum": checksum(cu),
                      "sha256_u8": sha(cu.astype(np.uint8)), "cc_sha256": sha(cc.view(np.uint64)),
                      "cc_row0_head": words_hex(cc[0, :16]), "ref_seconds": time.time() - t}
    print("config4", cfg["config4"]["checksum"], time.time() - t, flush=True)
    g["configs"] = cfg
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json"), "w") as f:
        json.dump(g, f, indent=0, sort_keys=True)
    print("done", time.time() - t0)


if __name__ == "__main__":
    main()
