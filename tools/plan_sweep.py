#!/usr/bin/env python3
"""Calibrate the GPU planner: time the fused DMMA contraction (qg_mul_common)
for every candidate (t, e, k-block) of a (p, m, k, n) workload on one B200.

    python tools/plan_sweep.py --p 7 --m 4096 --k 4096 --n 4096

Prints one JSON line per candidate: packed words K, block words, stage
depth chosen by the dispatcher, kernel ms, packed TFLOP/s, effective
2mnk/s. Each candidate is checked against the first one (C mod p is unique).
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_0803_1975_b200 as qg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, default=7)
    ap.add_argument("--m", type=int, default=4096)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--tiled", action="store_true", help="tiled layout + balanced plans (the fast path)")
    args = ap.parse_args()
    p, m, k, n = args.p, args.m, args.k, args.n
    a = qg.random_residue_matrix(m, k, p, 42)
    b = qg.random_residue_matrix(k, n, p, 43)
    ref_c = None
    for bal in ((0, 1) if args.tiled else (0,)):
     for t in range(2, 27):
        km = ((1 << t) - 1) // ((p - 1) ** 2) if not bal else ((1 << (t - 1)) - 1) // ((p // 2) ** 2)
        if km < 1:
            continue
        cap = 53 // t - (1 if 53 % t == 0 else 0)
        for e in sorted({cap, cap - 1}):
            if e < 2:
                continue
            pl = qg.make_plan(p, t, e)
            pl = qg.CompressionPlan(pl.p, pl.t, pl.d, pl.e, pl.beta, km, pl.inv_qd, 0)
            exact = qg.max_exact_block_balanced(pl) if bal else qg.max_exact_block(pl)
            K = -(-k // e)
            kbw = exact if k <= km else min(exact, km // e)
            if kbw < 4 and K > kbw:
                continue
            cands = sorted({c for c in ((4, 12, 20, 28, 36, 44, 52, 56, 72, 104, 144, kbw) if args.tiled else
                                        (4, 8, 16, 24, 28, 32, 48, 64, 96, 128, 192, 256, kbw)) if c <= kbw})
            if K <= kbw and k <= km:
                cands = [K]
            big = qg.CompressionPlan(pl.p, pl.t, pl.d, pl.e, pl.beta, max(pl.kmax, k), pl.inv_qd, 0)
            c = torch.empty((m, n), dtype=torch.int32, device="cuda")
            if not args.tiled:
                ca = qg.compress_rows_reversed(a, big).data
                cb = qg.compress_cols_forward(b, big).data
            for kb in cands:
                gpp = qg.GpuPlan(pl, kb, exact, bal)
                gp = gpp._c()
                if args.tiled:
                    try:
                        bk = qg.tiled_stage_words(gpp, k)
                    except qg.Error:
                        continue
                    ca = qg.pack_tiled(a, gpp, bk, "a")
                    cb = qg.pack_tiled(b, gpp, bk, "b")
                    fn = qg.lib.qg_mul_common_tiled
                else:
                    fn = qg.lib.qg_mul_common
                run = lambda: qg._check(fn(ctypes.byref(gp), qg._ptr(ca), qg._ptr(cb), m, n, k, qg._ptr(c), n, qg._stream()))
                try:
                    run()
                except qg.Error as ex:  # plans the library refuses (e.g. digit sums would overflow)
                    print(json.dumps({"t": t, "e": e, "balanced": bal, "kblock": kb, "refused": str(ex)}), flush=True)
                    continue
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(args.reps):
                    run()
                e1.record()
                e1.synchronize()
                ms = e0.elapsed_time(e1) / args.reps
                if ref_c is None:
                    ref_c = c.clone()
                ok = bool(torch.equal(c, ref_c))
                print(json.dumps({"p": p, "m": m, "k": k, "n": n, "t": t, "e": e, "balanced": bal, "K": K, "kblock": kb, "exact": exact,
                                  "kernel": qg.last_kernel(), "ms": round(ms, 4),
                                  "packed_tflops": round(2 * m * n * K / ms / 1e9, 2),
                                  "eff_T": round(2 * m * n * k / ms / 1e9, 2), "agrees": ok}), flush=True)
            del c


if __name__ == "__main__":
    main()
