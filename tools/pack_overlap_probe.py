"""Do the two tiled packs of a bench step overlap? Times pack A + pack B of
config 2 (and 3) serially on one stream and concurrently on two streams
(CUDA events, L2 flushed before each timed pair)."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_0803_1975_b200 as qg  # noqa: E402

flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
for (p, m, k, n) in [(7, 4096, 4096, 4096), (3, 8192, 256, 8192)]:
    gp = qg.plan_gpu(p, k)
    g = gp._c()
    bk = qg.tiled_stage_words(gp, k)
    a = qg.random_residue_matrix(m, k, p, 42)
    b = qg.random_residue_matrix(k, n, p, 43)
    ca = torch.empty(qg.lib.qg_tiled_words(m, k, gp.plan.e, bk), dtype=torch.float64, device="cuda")
    cb = torch.empty(qg.lib.qg_tiled_words(n, k, gp.plan.e, bk), dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def pa(s):
        qg._check(qg.lib.qg_pack_a_tiled(ctypes.byref(g), bk, qg._ptr(a), 0, m, k, k, qg._ptr(ca), ctypes.c_void_p(s.cuda_stream)))

    def pb(s):
        qg._check(qg.lib.qg_pack_b_tiled(ctypes.byref(g), bk, qg._ptr(b), 0, k, n, n, qg._ptr(cb), ctypes.c_void_p(s.cuda_stream)))

    res = {}
    for mode in ("serial", "concurrent", "a_only", "b_only"):
        ts = []
        for it in range(13):
            flush.fill_(1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            cur = torch.cuda.current_stream()
            e0.record(cur)
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            if mode == "serial":
                pa(s1)
                pb(s1)
            elif mode == "concurrent":
                pa(s1)
                pb(s2)
            elif mode == "a_only":
                pa(s1)
            else:
                pb(s1)
            cur.wait_stream(s1)
            cur.wait_stream(s2)
            e1.record(cur)
            e1.synchronize()
            if it >= 3:
                ts.append(e0.elapsed_time(e1))
        ts.sort()
        res[mode] = round(ts[len(ts) // 2] * 1e3, 1)
    print(json.dumps({"p": p, "m": m, "k": k, "n": n, "us": res}), flush=True)
