#!/usr/bin/env python3
"""Achieved HBM bandwidth of the memory-bound kernels (pack, unpack, REDQ,
extraction) at BASELINE config sizes.

Each kernel is timed with CUDA events on the launching stream (median of 10
after 3 warm-ups, L2 flushed before each timed launch); `achieved` =
algorithmic bytes (inputs read once + outputs written once, counted from the
shapes) / time, against the measured copy peak in MEASURED_PEAKS.json. Run it
plain for the numbers; run it under `ncu --metrics
gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum` for the
kernel-only durations and DRAM traffic (tools/summarize_memory_ncu.py).

    python tools/profile_memory_kernels.py > gpurun_out/memory_kernels.jsonl
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_0803_1975_b200 as qg  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
dev = torch.device("cuda", 0)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
sp = qg._stream
P = qg._ptr


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        fn()
        s1.record()
        s1.synchronize()
        ts.append(s0.elapsed_time(s1))
    ts.sort()
    return ts[len(ts) // 2]


def report(name, ref, nbytes, ms, note=""):
    gbs = nbytes / (ms * 1e-3) / 1e9
    print(json.dumps({"kernel": name, "replaces": ref, "algorithmic_bytes": int(nbytes), "ms": round(ms, 4),
                      "achieved_gbs": round(gbs, 1), "peak_gbs": PEAK, "frac_of_measured_copy": round(gbs / PEAK, 3),
                      "note": note}), flush=True)


def main():
    # config 2 operands: p=7, 4096^3, GPU plan (balanced t=12 e=4, 52-word stages)
    p, m, k, n = 7, 4096, 4096, 4096
    gp = qg.plan_gpu(p, k)
    g = gp._c()
    bk = ctypes.c_uint32()
    qg._check(qg.lib.qg_tiled_stage_words(ctypes.byref(g), k, ctypes.byref(bk)))
    bk = bk.value
    a = torch.empty((m, k), dtype=torch.float64, device=dev)
    report("k_gen_residues", "random_residue_matrix prng.hpp:31-38", m * k * 8,
           timed(lambda: qg._check(qg.lib.qg_gen_residues(42, p, 0, m, k, P(a), 0, sp()))), "4096 x 4096 f64 written")
    b = qg.random_residue_matrix(k, n, p, 43)
    wa, wb = qg.lib.qg_tiled_words(m, k, gp.plan.e, bk), qg.lib.qg_tiled_words(n, k, gp.plan.e, bk)
    ca = torch.empty(wa, dtype=torch.float64, device=dev)
    cb = torch.empty(wb, dtype=torch.float64, device=dev)
    report("k_pack_a_tiled", "compress_rows_reversed gemm.hpp:104-118", m * k * 8 + wa * 8,
           timed(lambda: qg._check(qg.lib.qg_pack_a_tiled(ctypes.byref(g), bk, P(a), 0, m, k, k, P(ca), sp()))),
           "config 2 A: f64 residues in, tiled balanced words out")
    report("k_pack_b_tiled", "compress_cols_forward gemm.hpp:122-140", k * n * 8 + wb * 8,
           timed(lambda: qg._check(qg.lib.qg_pack_b_tiled(ctypes.byref(g), bk, P(b), 0, k, n, n, P(cb), sp()))),
           "config 2 B: f64 residues in, transposed tiled words out")
    del a, b, ca, cb

    # config 4 shape: p=5, 8192^3, right/left/full packs and the unpack/REDQ kernels
    p, m, k, n = 5, 8192, 8192, 8192
    gr = qg.plan_right_gpu(p, k, n)
    pl = gr.plan
    gg = gr._c()
    bkr = ctypes.c_uint32()
    qg._check(qg.lib.qg_right_tiled_stage(ctypes.byref(gg), k, ctypes.byref(bkr)))
    bkr = bkr.value
    kt = -(-k // bkr)
    H = -(-n // pl.e)
    bmat = qg.random_residue_matrix(k, n, p, 43)
    bo = torch.empty(-(-H // 128) * 128 * kt * bkr, dtype=torch.float64, device=dev)
    plc = pl._c()
    report("k_pack_outer_tiled", "compress_outer_cols gemm.hpp:145-158", k * n * 8 + bo.numel() * 8,
           timed(lambda: qg._check(qg.lib.qg_pack_outer_cols_tiled(ctypes.byref(plc), bkr, P(bmat), 0, k, n, n, P(bo),
                                                                   sp()))), "config 4 B (t=13, e=4)")
    ao = torch.empty(-(-(m // pl.e) // 128) * 128 * kt * bkr, dtype=torch.float64, device=dev)
    report("k_pack_outer_rows_tiled", "compress_outer_rows gemm.hpp:160-176", m * k * 8 + ao.numel() * 8,
           timed(lambda: qg._check(qg.lib.qg_pack_outer_rows_tiled(ctypes.byref(plc), bkr, P(bmat), 0, m, k, k, P(ao),
                                                                    sp()))), "config-4-shape A of the left variant")
    del bo, ao
    # CC words of the right product (m x H), then unpack / REDQ / extraction over them
    a4 = qg.random_residue_matrix(m, k, p, 42)
    cc = qg.mul_right_tiled(a4, bmat, gr)
    del a4
    out = torch.empty((m, n), dtype=torch.int32, device=dev)
    o = qg._Orientation(0, 1, pl.e)
    report("k_uncompress", "uncompress gemm.hpp:182-204", cc.data.numel() * 8 + m * n * 4,
           timed(lambda: qg._check(qg.lib.qg_uncompress(ctypes.byref(plc), o, P(cc.data), m, H, m, n, P(out), sp()))),
           "config 4 CC -> int32 C (includes the DigitOverflow flag read-back)")
    w = cc.data.clone()
    report("k_redq", "redq_in_place gemm.hpp:313-316", w.numel() * 16,
           timed(lambda: qg._check(qg.lib.qg_redq(ctypes.byref(plc), P(w), w.numel(), sp()))),
           "in place over config 4 CC (includes the DigitOverflow flag read-back)")
    fp, kb = qg.plan_full_gpu(p, k)
    f = fp._c()
    G, Hf = -(-m // fp.q_slots()), -(-n // fp.theta_slots())
    words = (torch.rand((G, Hf), device=dev) * 2.0 ** 52).floor().to(torch.float64)
    report("k_uncompress_full", "mul_full_compressed unpack gemm.hpp:427-443", words.numel() * 8 + m * n * 4,
           timed(lambda: qg._check(qg.lib.qg_uncompress_full(ctypes.byref(f), P(words), words.shape[1], m, n, P(out), n,
                                                            sp()))), "config-4-shape full words -> int32 C")
    del words, w, cc
    # extraction / ReduceAndCompress over accumulated words (m x n doubles)
    acc = bmat * 1.0
    ext = torch.empty((m, n), dtype=torch.int32, device=dev)
    report("k_extract_coefficients", "extract_coefficient pack.hpp:78-100", m * n * 12,
           timed(lambda: qg._check(qg.lib.qg_extract_coefficients(ctypes.byref(plc), P(acc), m * n, P(ext), sp()))),
           "8192 x 8192 words -> int32")
    rc = torch.empty((m, H), dtype=torch.float64, device=dev)
    report("k_reduce_and_compress", "reduce_and_compress pack.hpp:141-155", m * n * 8 + m * H * 8,
           timed(lambda: qg._check(qg.lib.qg_reduce_and_compress(ctypes.byref(plc), P(acc), m, n, n, P(rc), H, sp()))),
           "8192 x 8192 words -> 8192 x 2048 words")


if __name__ == "__main__":
    main()
