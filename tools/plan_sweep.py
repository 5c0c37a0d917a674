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
    args = ap.parse_args()
    p, m, k, n = args.p, args.m, args.k, args.n
    a = qg.random_residue_matrix(m, k, p, 42)
    b = qg.random_residue_matrix(k, n, p, 43)
    ref_c = None
    for t in range(2, 27):
        km = ((1 << t) - 1) // ((p - 1) ** 2)
        if km < 1:
            continue
        cap = 53 // t - (1 if 53 % t == 0 else 0)
        for e in sorted({cap, cap - 1}):
            if e < 2:
                continue
            pl = qg.make_plan(p, t, e)
            exact = qg.max_exact_block(pl)
            K = -(-k // e)
            kbw = exact if k <= km else min(exact, km // e)
            if kbw < 4 and K > kbw:
                continue
            cands = sorted({c for c in (4, 8, 16, 24, 28, 32, 48, 64, 96, 128, 192, 256, kbw) if c <= kbw})
            if K <= kbw and k <= km:
                cands = [K]
            big = qg.CompressionPlan(pl.p, pl.t, pl.d, pl.e, pl.beta, max(pl.kmax, k), pl.inv_qd, 0)
            ca = qg.compress_rows_reversed(a, big)
            cb = qg.compress_cols_forward(b, big)
            c = torch.empty((m, n), dtype=torch.int32, device="cuda")
            for kb in cands:
                gp = qg.GpuPlan(pl, kb, exact)._c()
                run = lambda: qg._check(qg.lib.qg_mul_common(ctypes.byref(gp), qg._ptr(ca.data), qg._ptr(cb.data), m, n, k,
                                                             qg._ptr(c), n, qg._stream()))
                run()
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
                print(json.dumps({"p": p, "m": m, "k": k, "n": n, "t": t, "e": e, "K": K, "kblock": kb, "exact": exact,
                                  "kernel": qg.last_kernel(), "ms": round(ms, 4),
                                  "packed_tflops": round(2 * m * n * K / ms / 1e9, 2),
                                  "eff_T": round(2 * m * n * k / ms / 1e9, 2), "agrees": ok}), flush=True)
            del ca, cb, c


if __name__ == "__main__":
    main()
