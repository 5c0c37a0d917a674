#!/usr/bin/env python3
"""One full BASELINE config 5 product on one B200: p=3, m=n=k=32768, seeds
42/43, through the fast path (tiled layout, plan_gpu). Prints one JSON line
with the device time and effective 2mnk/s, then verifies C:

* the 8 golden row shards (32 rows from each eighth of C) made by the
  reference itself (tests/golden/golden.json);
* Freivalds over GF(3): C x = A (B x) mod 3 for 8 random 0/1/2 vectors x
  (exact: float64 matrix-vector products of residues stay < 2^53; this is
  the checker, not the product path);
* the same 256 rows recomputed under the reference plan (t=18, e=2) are
  bit-identical.

Usage: python tools/run_config5.py [--m 32768]   (about 7 minutes)
"""
import argparse
import ctypes
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_0803_1975_b200 as qg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=32768)
    args = ap.parse_args()
    p, m, k, n = 3, args.m, 32768, 32768
    dev = torch.device("cuda", 0)
    gp = qg.plan_gpu(p, k)
    bk = qg.tiled_stage_words(gp, k)
    a = qg.random_residue_matrix(m, k, p, 42)
    b = qg.random_residue_matrix(k, n, p, 43)
    c = torch.empty((m, n), dtype=torch.int32, device=dev)
    g = gp._c()
    # warm-up on a 256-row slice (kernel load, clocks)
    ca_s = qg.pack_tiled(a[:256], gp, bk, "a")
    cb = qg.pack_tiled(b, gp, bk, "b")
    qg._check(qg.lib.qg_mul_common_tiled(ctypes.byref(g), qg._ptr(ca_s), qg._ptr(cb), 256, n, k, qg._ptr(c), n, qg._stream()))
    torch.cuda.synchronize()
    del ca_s
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    w0 = time.perf_counter()
    e0.record()
    ca = qg.pack_tiled(a, gp, bk, "a")
    cb = qg.pack_tiled(b, gp, bk, "b")
    e1.record()
    qg._check(qg.lib.qg_mul_common_tiled(ctypes.byref(g), qg._ptr(ca), qg._ptr(cb), m, n, k, qg._ptr(c), n, qg._stream()))
    e2.record()
    e2.synchronize()
    wall = time.perf_counter() - w0
    pack_ms, kern_ms = e0.elapsed_time(e1), e1.elapsed_time(e2)
    K = -(-k // gp.plan.e)
    line = {"workload": "config5: p=3 m=%d n=k=32768, one GPU" % m, "plan": {"t": gp.plan.t, "e": gp.plan.e,
            "kblock_words": gp.kblock_words, "balanced": gp.balanced, "stage_words": bk},
            "ms_total": pack_ms + kern_ms, "ms_pack": pack_ms, "ms_contraction": kern_ms, "wall_s": wall,
            "eff_mult_adds_per_s": 2.0 * m * n * k / ((pack_ms + kern_ms) * 1e-3),
            "packed_tflops": 2.0 * m * n * K / (kern_ms * 1e-3) / 1e12, "kernel": qg.last_kernel()}
    print(json.dumps(line), flush=True)
    del ca, cb
    torch.cuda.empty_cache()

    # ---- verification
    golden = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "golden.json")))
    shards = golden["configs"]["config5_rows"]["shards"]
    ok_shards = 0
    for sh in shards:
        if sh["row0"] + sh["rows"] > m:
            continue
        rows = c[sh["row0"]:sh["row0"] + sh["rows"]]
        cs = int(rows.to(torch.int64).sum().item()) & 0xFFFFFFFF
        sha = hashlib.sha256(rows.cpu().numpy().astype("uint8").tobytes()).hexdigest()
        ok_shards += int(cs == sh["checksum"] and sha == sh["sha256_u8"])
    frei = []
    gen = torch.Generator(device=dev).manual_seed(7)
    ad, bd = a.double(), b.double()
    cd = c.double()
    for _ in range(8):
        x = torch.randint(0, 3, (n,), generator=gen, device=dev, dtype=torch.int64).double()
        bx = torch.remainder(bd @ x, 3)
        lhs = torch.remainder(cd @ x, 3)
        rhs = torch.remainder(ad @ bx, 3)
        frei.append(bool(torch.equal(lhs, rhs)))
    del ad, bd, cd
    # same rows under the reference plan, row layout kernels
    rp = qg.plan_compression(p, k)
    a2 = qg.random_residue_matrix(256, k, p, 42)
    c2 = qg.mul_common_compressed(a2, b, rp)
    same = bool(torch.equal(c2, c[:256]))
    print(json.dumps({"golden_shards_ok": ok_shards, "golden_shards": len([s for s in shards if s["row0"] + s["rows"] <= m]),
                      "freivalds_ok": sum(frei), "freivalds_trials": len(frei),
                      "rows0_255_equal_reference_plan": same,
                      "checksum_c": int(c.to(torch.int64).sum().item()) & 0xFFFFFFFF}), flush=True)


if __name__ == "__main__":
    main()
