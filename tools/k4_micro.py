#!/usr/bin/env python3
"""K4 / K4A micro-benchmark: the tiled contraction alone on a product of
exactly `waves` full waves of 128x128 tiles (no tail), CUDA events, L2 flushed
between launches. Prints time, % of the DMMA peak and a checksum that must not
depend on the plan.

  python tools/k4_micro.py --p 3 --k 32768 [--kblock 12 --anchored 1] [--waves 8]
"""
import argparse, ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0803_1975_b200 as qg

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=3)
ap.add_argument("--k", type=int, default=32768)
ap.add_argument("--kblock", type=int, default=0)
ap.add_argument("--anchored", type=int, default=-1)
ap.add_argument("--waves", type=int, default=8)
ap.add_argument("--t", type=int, default=0, help="force the plan's (t, e) (with --e)")
ap.add_argument("--e", type=int, default=0)
ap.add_argument("--plain", type=int, default=0, help="1: plan_gpu(p, k, anchored=False), the best FP64-flush plan")
ap.add_argument("--m", type=int, default=0, help="explicit shape instead of whole waves")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--peak", type=float, default=37.09)
args = ap.parse_args()
dev = torch.device("cuda", 0)
sms = torch.cuda.get_device_properties(0).multi_processor_count
p, k = args.p, args.k
tiles_n = 32
tiles_m = sms * args.waves // tiles_n
m, n = tiles_m * 128, tiles_n * 128
if args.m:
    m, n = args.m, args.n or args.m
gp = qg.plan_gpu(p, k, anchored=not args.plain)
if args.t:
    gp = qg.GpuPlan(qg.make_plan(p, args.t, args.e), gp.kblock_words, 0, 1, 0)
if (args.kblock or args.anchored >= 0) and not args.plain:
    gp = qg.GpuPlan(gp.plan, args.kblock or gp.kblock_words, gp.max_exact_words, gp.balanced,
                    gp.anchored if args.anchored < 0 else args.anchored)
bk = qg.tiled_stage_words(gp, k)
a = qg.random_residue_matrix(m, k, p, 42)
b = qg.random_residue_matrix(k, n, p, 43)
ca = qg.pack_tiled(a, gp, bk, "a")
cb = qg.pack_tiled(b, gp, bk, "b")
c = torch.empty((m, n), dtype=torch.int32, device=dev)
g = gp._c()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
def run():
    qg._check(qg.lib.qg_mul_common_tiled(ctypes.byref(g), qg._ptr(ca), qg._ptr(cb), m, n, k, qg._ptr(c), n, qg._stream()))
for _ in range(2):
    run()
torch.cuda.synchronize()
ts = []
for _ in range(args.reps):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts) // 2]
K = -(-k // gp.plan.e)
tf = 2.0 * m * n * K / (ms * 1e-3) / 1e12
print(json.dumps({"kernel": qg.last_kernel(), "m": m, "n": n, "k": k, "t": gp.plan.t, "e": gp.plan.e, "kblock": gp.kblock_words,
                  "bk": bk, "anchored": gp.anchored, "ms": round(ms, 4), "tflops": round(tf, 3), "frac": round(tf / args.peak, 4),
                  "eff_T": round(2.0 * m * n * k / (ms * 1e-3) / 1e12, 2), "checksum": int(c.sum().item())}))
