#!/usr/bin/env python3
"""bench.py — effective mod-p multiply-adds per second (2mnk/s) of the
compressed modular GEMM on B200, the BASELINE.json metric.

Workload (N=1): BASELINE config 2 — p=7, m=n=k=4096, dot-product variant
(Q-adic rows reversed / columns forward, FP64 tensor-core contraction,
per-k-block digit extraction, mod-p accumulation between blocks).
A "step" = pack A (K1) + pack B (K2) + the fused DMMA contraction/extract/mod-p
kernel (K4) on device-resident residues (seeded SplitMix64, K0, generated
once). For N>1 (torchrun) every rank owns m=4096 rows of A and C (weak
scaling); rank 0 packs B and broadcasts the packed CB over NCCL each step.

Keys beyond the base contract:
  roofline      the contraction kernel's achieved packed FP64 TFLOP/s vs the
                measured DMMA peak (profiles/r01_fp64_peak.json)
  cpu_baseline  the reference's own CPU path (oracle/_ref, the unmodified
                reference headers) timed on this host's cores on a row sample
  e2e           the same metric through the public host-buffer API
                (mul_common_compressed_host: H2D of A,B + kernels + D2H of C)
``--impl reference`` runs only the reference CPU arm.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (p, m, k, n, description)
    "config1": (3, 512, 512, 512, "config1: p=3 m=n=k=512 dot-product variant"),
    "config2": (7, 4096, 4096, 4096, "config2: p=7 m=n=k=4096 dot-product variant, k-blocked"),
    "config3": (3, 8192, 256, 8192, "config3: p=3 m=n=8192 k=256 dot-product variant"),
    "config5": (3, 32768, 32768, 32768, "config5: p=3 m=n=k=32768 dot-product variant, k-blocked"),
    "config4": (5, 8192, 8192, 8192, "config4: p=5 m=n=k=8192 mixed (right) variant, REDQ epilogue -> CC"),
    # the left and full variants (gemm.hpp:340-445) on config 4's shape
    "config4_left": (5, 8192, 8192, 8192, "config4 shape: p=5 m=n=k=8192 left (outer-rows) variant, REDQ -> CC"),
    "config4_full": (5, 8192, 8192, 8192, "config4 shape: p=5 m=n=k=8192 full (two-axis) variant -> C"),
}
REDQ_VARIANTS = {"config4": "right", "config4_left": "left", "config4_full": "full"}
SEED = 42


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock and clock-event reasons while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h) if hasattr(
                    nv, "nvmlDeviceGetCurrentClocksEventReasons") else nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self._nv is not None:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread:
            self._thread.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


# ------------------------------------------------------------------ CPU reference
def reference_cpu_sample(p, m, k, n, target_s=4.0, threads=None, rows=None):
    """Time the reference's own dot-product path (oracle/_ref: unmodified
    compress_rows_reversed -> compress_cols_forward -> packed_common_product
    -> reduce_common_entry, bench.hpp:127-146) at its own plan on a row
    sample of the seeded workload, rows sharded over host threads.
    Returns (rate 2*rows*n*k/s, rows, threads, seconds, C rows, plan)."""
    import ctypes

    import numpy as np

    import oracle

    ref = oracle.REF
    kind = "reference"
    threads = threads or host_threads()
    pl = oracle.Plan()
    if ref is None:
        raise RuntimeError("oracle/_ref/libqgref.so is missing (built by __graft_entry__.build())")
    st = ref.qgref_plan_compression(p, k, 53, 0, ctypes.byref(pl))
    if st:
        raise RuntimeError(f"reference plan failed: {st}")
    b = oracle.random_residue_matrix(k, n, p, SEED + 1)

    def run(r):
        a = oracle.random_residue_matrix(r, k, p, SEED)
        c = np.empty((r, n), dtype=np.uint32)
        mul, conv = ctypes.c_double(), ctypes.c_double()
        t0 = time.perf_counter()
        st = ref.qgref_mul_common(ctypes.byref(pl), a.ctypes.data_as(ctypes.c_void_p), b.ctypes.data_as(ctypes.c_void_p),
                                  r, k, n, c.ctypes.data_as(ctypes.c_void_p), threads, ctypes.byref(mul), ctypes.byref(conv))
        dt = time.perf_counter() - t0
        if st:
            raise RuntimeError(f"reference mul_common failed: {st}")
        return dt, c

    if rows is None:
        pilot = max(threads, 8)
        dt, _ = run(pilot)
        rows = int(min(m, max(threads, pilot * target_s / max(dt, 1e-3))))
        rows = max(threads, rows // threads * threads) if rows >= threads else rows
    dt, c = run(rows)
    return 2.0 * rows * n * k / dt, rows, threads, dt, c, pl, kind


def reference_variant_sample(variant, p, m, k, n, target_s=4.0, threads=None, rows=None):
    """Time the reference's own right / left / full path (oracle/_ref: the
    unmodified mul_right_compressed / mul_left_compressed(compress_outer_rows)
    / mul_full_compressed, bench.hpp:108-152) at the reference's plan on a row
    sample of the seeded workload, row shards over host threads (B packed per
    shard for left/full, as the reference's single-threaded call would).
    Raises NoCompression when the reference planner refuses the shape."""
    import ctypes
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    import oracle

    ref = oracle.REF
    if ref is None:
        raise RuntimeError("oracle/_ref/libqgref.so is missing (built by __graft_entry__.build())")
    threads = threads or host_threads()
    vp = ctypes.c_void_p
    if variant == "full":
        plan = oracle.FullPlan()
        st = ref.qgref_plan_full(p, k, 53, ctypes.byref(plan))
        group = plan.dq + 1 if st == 0 else 1
    else:
        plan = oracle.Plan()
        st = ref.qgref_plan_compression(p, k, 53, 0, ctypes.byref(plan))
        group = plan.e if (st == 0 and variant == "left") else 1
    if st:
        raise RuntimeError(f"reference planner refused p={p} k={k} for the {variant} variant (status {st}: "
                           f"{'NoCompression' if st == 2 else 'error'})")
    b = oracle.random_residue_matrix(k, n, p, SEED + 1)

    pack_b_cache = []

    def pack_b_seconds():  # the reference's compress_outer_cols(B) alone (gemm.hpp:145-158)
        if not pack_b_cache:
            cbo = np.zeros((k, -(-n // plan.e)))
            runs = []
            for _ in range(2):
                t0 = time.perf_counter()
                ref.qgref_compress_outer_cols(ctypes.byref(plan), b.ctypes.data_as(vp), k, n, cbo.ctypes.data_as(vp))
                runs.append(time.perf_counter() - t0)
            pack_b_cache.append(min(runs))
        return pack_b_cache[0]

    def shard(a, r):
        if variant == "left":
            cc = np.empty((-(-r // plan.e), n))
            st = ref.qgref_mul_left(ctypes.byref(plan), a.ctypes.data_as(vp), b.ctypes.data_as(vp), r, k, n,
                                    cc.ctypes.data_as(vp))
        else:
            cc = np.empty((r, n), np.uint32)
            st = ref.qgref_mul_full(ctypes.byref(plan), a.ctypes.data_as(vp), b.ctypes.data_as(vp), r, k, n,
                                    cc.ctypes.data_as(vp))
        if st:
            raise RuntimeError(f"reference {variant} failed: {st}")

    def run(r):
        a = oracle.random_residue_matrix(r, k, p, SEED)
        t0 = time.perf_counter()
        if variant == "right":
            cc = np.empty((r, -(-n // plan.e)))
            mul, conv = ctypes.c_double(), ctypes.c_double()
            st = ref.qgref_mul_right(ctypes.byref(plan), a.ctypes.data_as(vp), b.ctypes.data_as(vp), r, k, n,
                                     cc.ctypes.data_as(vp), None, threads, ctypes.byref(mul), ctypes.byref(conv))
            if st:
                raise RuntimeError(f"reference right failed: {st}")
            # compress_outer_cols(B) runs once per call: charge it pro rata
            # (r/m), as a full-size run amortises it over all m rows
            dt = time.perf_counter() - t0
            pack_b = min(pack_b_seconds(), dt)
            return max(dt - pack_b + pack_b * r / m, mul.value)  # never below the multiply phase itself
        else:
            per = max(group, -(-r // threads) // group * group)
            parts = [(i, min(r, i + per)) for i in range(0, r, per)]
            with ThreadPoolExecutor(len(parts)) as ex:
                list(ex.map(lambda se: shard(np.ascontiguousarray(a[se[0]:se[1]]), se[1] - se[0]), parts))
        return time.perf_counter() - t0

    if rows is None:
        pilot = max(threads, 8) // group * group or group
        dt = run(pilot)
        rows = int(min(m, max(threads * group, pilot * target_s / max(dt, 1e-3))))
        rows = max(group, rows // (threads * group) * (threads * group)) if rows >= threads * group else \
            max(group, rows // group * group)
    dt = run(rows)
    kind = "reference"
    return 2.0 * rows * n * k / dt, rows, threads, dt, None, plan, kind


# ------------------------------------------------------------------ reference arm
def reference_arm(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    p, m, k, n, desc = CONFIGS[args.config]
    variant = REDQ_VARIANTS.get(args.config, "common")
    rates, rows_used, thr = [], None, host_threads()
    rows_used = None
    for i in range(args.warmup + args.steps):
        if variant == "common":
            rate, rows, thr, dt, _, pl, kind = reference_cpu_sample(p, m, k, n, target_s=args.ref_step_s, rows=rows_used)
        else:
            try:
                rate, rows, thr, dt, _, pl, kind = reference_variant_sample(variant, p, m, k, n,
                                                                            target_s=args.ref_step_s, rows=rows_used)
            except RuntimeError as ex:
                print(json.dumps({"impl": "reference", "unavailable": str(ex)}), flush=True)
                return 0
        rows_used = rows
        if i >= args.warmup:
            rates.append(rate)
    value = sum(rates) / len(rates)
    pdesc = (f"t={pl.base.t} dq={pl.dq} dtheta={pl.dtheta}" if variant == "full" else f"t={pl.t} e={pl.e}")
    sample = (f"rows 0..{rows_used - 1} of A ({rows_used}x{k}) x B ({k}x{n}), {variant} variant, reference plan "
              f"{pdesc}, {thr} threads")
    line = {
        "impl": "reference", "metric": "effective mod-p mult-adds/sec (2mnk/s)", "value": value, "unit": "mult-adds/s (2mnk/s)",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 2.0 * rows_used * n * k / value * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (SplitMix64 seed 42/43)",
        "config": {"workload": desc, "p": p, "m": m, "k": k, "n": n},
        "cpu_baseline": {"value": value, "unit": "mult-adds/s (2mnk/s)", "cores": thr, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "mult-adds/s (2mnk/s)", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def redq_arm(args):
    """Config 4 and its §8(f) siblings: the right (mixed, gemm.hpp:285-335),
    left (gemm.hpp:340-371) and full (gemm.hpp:377-445) variants on the tiled
    layout. Step = the operand packs into tiled blocks + the DMMA contraction
    with in-place REDQ between k-blocks and a REDQ epilogue (K5) [+ the full
    variant's digit scatter to C] on device-resident residues.
    --plan gpu: plan_right_gpu / plan_full_gpu; --plan reference: the plan the
    reference bench uses (plan_compression / plan_full, bench.hpp:108-152),
    output words bit-identical to the reference's."""
    import ctypes
    import hashlib

    import numpy as np
    import torch

    import paper_0803_1975_b200 as qg

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    p, m, k, n, desc = CONFIGS[args.config]
    variant = REDQ_VARIANTS[args.config]
    sp = qg._stream
    kblock = 0
    if variant == "full":
        if args.plan == "reference":
            try:
                fp = qg.plan_full(p, k)
            except qg.NoCompression:
                print(json.dumps({"metric": "effective mod-p mult-adds/sec (2mnk/s)", "value": None,
                                  "unavailable": f"plan_full({p}, {k}) raises NoCompression (plan.hpp:235-237)"}))
                return 0
            kblock = 0
        else:
            fp, kblock = qg.plan_full_gpu(p, k)
        plan = fp.base
        f = fp._c()
        bk_c = ctypes.c_uint32()
        qg._check(qg.lib.qg_full_tiled_stage(ctypes.byref(f), kblock, k, ctypes.byref(bk_c)))
        rows_a, rows_b = -(-m // fp.q_slots()), -(-n // fp.theta_slots())
        out_shape = (rows_a, rows_b)
        plan_desc = {"t": plan.t, "dq": fp.dq, "dtheta": fp.dtheta, "theta_exponent": fp.theta_exponent,
                     "kblock_residues": kblock or k}
    else:
        if args.plan == "reference":
            base = qg.plan_compression(p, k)
            gp = qg.GpuPlan(base, k, k, 0)
        else:
            gp = qg.plan_right_gpu(p, k, n if variant == "right" else m)
        if args.redq_plan:  # experiments: "t:e:kblock:balanced"
            t_, e_, kb_, bal_ = (int(x) for x in args.redq_plan.split(":"))
            gp = qg.GpuPlan(qg.make_plan(p, t_, e_), kb_, kb_, bal_)
        plan = gp.plan
        g = gp._c()
        bk_c = ctypes.c_uint32()
        qg._check(qg.lib.qg_right_tiled_stage(ctypes.byref(g), k, ctypes.byref(bk_c)))
        if variant == "right":
            rows_a, rows_b = m, -(-n // plan.e)
        else:
            rows_a, rows_b = -(-m // plan.e), n
        out_shape = (rows_a, rows_b)
        plan_desc = {"t": plan.t, "e": plan.e, "kblock_residues": gp.kblock_words, "balanced": bool(gp.balanced)}
    bk = bk_c.value
    kt = -(-k // bk)
    a = qg.random_residue_matrix(m, k, p, SEED)
    b = qg.random_residue_matrix(k, n, p, SEED + 1)
    a_t = torch.empty(-(-rows_a // 128) * 128 * kt * bk, dtype=torch.float64, device=dev)
    b_t = torch.empty(-(-rows_b // 128) * 128 * kt * bk, dtype=torch.float64, device=dev)
    cc = torch.empty(out_shape, dtype=torch.float64, device=dev)
    c_full = torch.empty((m, n), dtype=torch.int32, device=dev) if variant == "full" else None
    pl = plan._c()
    if variant == "full":
        qs, ts = fp.q_slots(), fp.theta_slots()
        pa = qg._Plan(p, plan.t, qs - 1, qs, 53, plan.kmax, 1.0, 0)
        pb = qg._Plan(p, fp.theta_exponent, ts - 1, ts, 53, plan.kmax, 1.0, 0)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)

    bal = variant != "full" and bool(gp.balanced)

    def step(ev=None):
        if variant == "right" and bal:
            qg._check(qg.lib.qg_pack_residues_tiled_bal(p, bk, qg._ptr(a), 0, m, k, k, qg._ptr(a_t), sp()))
            qg._check(qg.lib.qg_pack_outer_cols_tiled_bal(ctypes.byref(pl), bk, qg._ptr(b), 0, k, n, n, qg._ptr(b_t),
                                                          sp()))
        elif variant == "right":
            qg._check(qg.lib.qg_pack_residues_tiled(bk, qg._ptr(a), 0, m, k, k, qg._ptr(a_t), sp()))
            qg._check(qg.lib.qg_pack_outer_cols_tiled(ctypes.byref(pl), bk, qg._ptr(b), 0, k, n, n, qg._ptr(b_t), sp()))
        elif variant == "left" and bal:
            qg._check(qg.lib.qg_pack_outer_rows_tiled_bal(ctypes.byref(pl), bk, qg._ptr(a), 0, m, k, k, qg._ptr(a_t),
                                                          sp()))
            qg._check(qg.lib.qg_pack_residues_b_tiled_bal(p, bk, qg._ptr(b), 0, k, n, n, qg._ptr(b_t), sp()))
        elif variant == "left":
            qg._check(qg.lib.qg_pack_outer_rows_tiled(ctypes.byref(pl), bk, qg._ptr(a), 0, m, k, k, qg._ptr(a_t), sp()))
            qg._check(qg.lib.qg_pack_residues_b_tiled(bk, qg._ptr(b), 0, k, n, n, qg._ptr(b_t), sp()))
        else:
            qg._check(qg.lib.qg_pack_outer_rows_tiled(ctypes.byref(pa), bk, qg._ptr(a), 0, m, k, k, qg._ptr(a_t), sp()))
            qg._check(qg.lib.qg_pack_outer_cols_tiled(ctypes.byref(pb), bk, qg._ptr(b), 0, k, n, n, qg._ptr(b_t), sp()))
        if ev:
            ev[0].record(stream)
        if variant == "right":
            qg._check(qg.lib.qg_mul_right_tiled(ctypes.byref(g), qg._ptr(a_t), qg._ptr(b_t), m, k, n, qg._ptr(cc),
                                                rows_b, sp()))
        elif variant == "left":
            qg._check(qg.lib.qg_mul_left_tiled(ctypes.byref(g), qg._ptr(a_t), qg._ptr(b_t), m, k, n, qg._ptr(cc),
                                               rows_b, sp()))
        else:
            qg._check(qg.lib.qg_mul_full_tiled(ctypes.byref(f), kblock, qg._ptr(a_t), qg._ptr(b_t), m, k, n,
                                               qg._ptr(cc), rows_b, sp()))
        if ev:
            ev[1].record(stream)
        if variant == "full":
            qg._check(qg.lib.qg_uncompress_full(ctypes.byref(f), qg._ptr(cc), rows_b, m, n, qg._ptr(c_full), n, sp()))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    step_ms, kern_ms = [], []
    launches0 = qg.kernel_launches()
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            s0.record(stream)
            step(ev)
            s1.record(stream)
            s1.synchronize()
            step_ms.append(s0.elapsed_time(s1))
            kern_ms.append(ev[0].elapsed_time(ev[1]))
    launches = qg.kernel_launches() - launches0
    kernel = qg.last_kernel()
    ms = sum(step_ms) / len(step_ms)
    kms = sum(kern_ms) / len(kern_ms)
    flop = 2.0 * rows_a * rows_b * k  # DMMA flops of the contraction (words x words x k)
    peak = float((load_json(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) or {}).get("dmma_m8n8k4_tflops", 37.09))
    if variant == "full":
        c = c_full
    else:
        orient = qg.PackOrientation(0, 1, plan.e) if variant == "right" else qg.PackOrientation(0, 0, plan.e)
        c = qg.uncompress(qg.CompressedMatrix(m, n, rows_a, rows_b, orient, plan, cc))
    line = {"metric": "effective mod-p mult-adds/sec (2mnk/s)", "value": 2.0 * m * n * k / (ms * 1e-3),
            "unit": "mult-adds/s (2mnk/s)", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SplitMix64 seed 42/43, generated on device)",
            "config": {"workload": desc, "variant": variant, "p": p, "m": m, "k": k, "n": n,
                       "plan": dict(plan_desc, stage_words=bk, source=args.plan),
                       "l2": "256 MiB buffer written between timed steps"},
            "roofline": {"bound": "tensor", "achieved": round(flop / (kms * 1e-3) / 1e12, 3), "peak": peak,
                         "unit": "TFLOP/s", "frac": round(flop / (kms * 1e-3) / 1e12 / peak, 4),
                         "traffic": ((load_json(os.path.join(ROOT, "profiles", "ncu_summary.json")) or {})
                                     .get("contraction", {}).get(args.config, {}).get("dram_bytes")),
                         "kernel": kernel, "kernel_ms": round(kms, 4),
                         "per_unit": "2 flops per packed-word product; rows_a x rows_b x k products per launch"},
            "gpu_launches": launches, "checksum_c": qg.residue_checksum(c),
            "cc_sha256": hashlib.sha256(cc.cpu().numpy().view("uint64").tobytes()).hexdigest(),
            "clocks": clk.summary()}
    del flush
    if not args.no_e2e:
        an = torch.empty((m, k), dtype=torch.int32, pin_memory=True)
        bn = torch.empty((k, n), dtype=torch.int32, pin_memory=True)
        an.copy_(a.to(torch.int32))
        bn.copy_(b.to(torch.int32))
        an_u, bn_u = an.numpy().view(np.uint32), bn.numpy().view(np.uint32)
        if variant == "full":
            out = torch.empty((m, n), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
            call = lambda: qg.mul_full_compressed_host(an_u, bn_u, fp, kblock, out=out)  # noqa: E731
            api = "mul_full_compressed_host (qg_host_mul_full)"
        else:
            out = torch.empty(out_shape, dtype=torch.float64, pin_memory=True).numpy()
            fn = qg.mul_right_compressed_host if variant == "right" else qg.mul_left_compressed_host
            arg = gp if args.plan == "gpu" else plan
            call = lambda: fn(an_u, bn_u, arg, out=out)  # noqa: E731
            api = f"mul_{variant}_compressed_host (qg_host_mul_{variant}{'_gpu' if args.plan == 'gpu' else ''})"
        for _ in range(3):
            call()
        times = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            call()
            times.append(time.perf_counter() - t0)
        t = sum(times) / len(times)
        # the host path's result against the device product's, bit for bit
        dev_out = c.cpu().numpy().astype(np.uint32) if variant == "full" else cc.cpu().numpy()
        same = bool(np.array_equal(np.ascontiguousarray(out).view(np.uint32 if variant == "full" else np.uint64),
                                   np.ascontiguousarray(dev_out).view(np.uint32 if variant == "full" else np.uint64)))
        line["e2e"] = {"value": 2.0 * m * n * k / t, "unit": "mult-adds/s (2mnk/s)",
                       "h2d_bytes_per_step": int((m * k + k * n) * 4), "d2h_bytes_per_step": int(out.nbytes),
                       "ms_per_step": t * 1e3, "api": api, "matches_device": same}
    if not args.no_cpu:
        try:
            rate, rows, thr, dt, _, rpl, kind = reference_variant_sample(variant, p, m, k, n, target_s=args.cpu_s)
            pdesc = (f"t={rpl.base.t} dq={rpl.dq} dtheta={rpl.dtheta}" if variant == "full" else f"t={rpl.t} e={rpl.e}")
            line["cpu_baseline"] = {"value": rate, "unit": "mult-adds/s (2mnk/s)", "cores": thr, "kind": kind,
                                    "sample": f"rows 0..{rows - 1} of A x B ({k}x{n}), reference {variant} path, "
                                              f"plan {pdesc}, {dt:.1f} s"}
        except RuntimeError as ex:
            line["cpu_baseline"] = {"value": None, "unavailable": str(ex)}
    print(json.dumps(line), flush=True)
    return 0


def our_arm(args):
    import numpy as np
    import torch
    import ctypes

    import torch.distributed as dist

    import paper_0803_1975_b200 as qg
    from paper_0803_1975_b200.dist import (PanelOps, ShardOps, mul_common_sharded, mul_common_sharded_pipelined,
                                           panel_bounds)

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    # one process per GPU; with fewer GPUs than ranks (the gloo functional
    # check of the multi-rank path on one GPU) ranks share devices
    local_dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)

    p, m_rank, k, n, desc = CONFIGS[args.config]
    gp = qg.plan_gpu(p, k) if args.plan == "gpu" else qg.gpu_plan_from(qg.plan_compression(p, k), k)
    if args.kblock:  # experiments: override the k-block of the chosen plan
        gp = qg.GpuPlan(gp.plan, args.kblock, gp.max_exact_words, gp.balanced)
    pl = gp.plan
    K = -(-k // pl.e)
    m_total = m_rank * world
    row0 = rank * m_rank

    # device-resident seeded inputs (K0): this rank's rows of A, all of B on rank 0
    a = qg.random_residue_matrix(m_rank, k, p, SEED, row0=row0)
    b = qg.random_residue_matrix(k, n, p, SEED + 1) if rank == 0 else None
    bk_c = ctypes.c_uint32()
    gpc = gp._c()
    qg._check(qg.lib.qg_tiled_stage_words(ctypes.byref(gpc), k, ctypes.byref(bk_c)))
    bk = bk_c.value
    # tiled packed layouts (dense zero-padded 128 x bk blocks, CB transposed)
    ca = torch.empty(qg.lib.qg_tiled_words(m_rank, k, pl.e, bk), dtype=torch.float64, device=dev)
    cb = torch.empty(qg.lib.qg_tiled_words(n, k, pl.e, bk), dtype=torch.float64, device=dev)
    c = torch.empty((m_rank, n), dtype=torch.int32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()
    sp = qg._stream
    plc = pl._c()

    def pack_rows(a_):
        qg._check(qg.lib.qg_pack_a_tiled(ctypes.byref(gpc), bk, qg._ptr(a_), 0, m_rank, k, k, qg._ptr(ca), sp()))
        return ca

    def pack_cols(b_):
        qg._check(qg.lib.qg_pack_b_tiled(ctypes.byref(gpc), bk, qg._ptr(b_), 0, k, n, n, qg._ptr(cb), sp()))
        return cb

    ev = {}

    def contract(ca_, cb_):
        ev["c0"].record(stream)
        qg._check(qg.lib.qg_mul_common_tiled(ctypes.byref(gpc), qg._ptr(ca_), qg._ptr(cb_), m_rank, n, k, qg._ptr(c), n, sp()))
        ev["c1"].record(stream)
        return c

    ops = ShardOps(pack_rows=pack_rows, pack_cols=pack_cols, empty_cb=lambda shape: cb, contract=contract)
    # multi-rank: the packed B goes out in column panels, each broadcast queued
    # behind the pack that produced it, so rank 0's packing overlaps the wire
    Kt = (K + bk - 1) // bk
    Nt = (n + 127) // 128
    W = Kt * 128 * bk  # words per 128-column tile column of CB_t

    def panel_views(cb_, panels):
        return [cb_[t0 * W:t1 * W] for t0, t1 in (panel_bounds(Nt, panels, j) for j in range(panels))]

    def pack_cols_panel(b_, j, panels, cb_):
        t0, t1 = panel_bounds(Nt, panels, j)
        c0, c1 = t0 * 128, min(n, t1 * 128)
        if c1 > c0:
            qg._check(qg.lib.qg_pack_b_tiled(ctypes.byref(gpc), bk, ctypes.c_void_p(b_.data_ptr() + c0 * 8), 0, k,
                                             c1 - c0, n, ctypes.c_void_p(cb_.data_ptr() + t0 * W * 8), sp()))

    pops = PanelOps(pack_rows=pack_rows, panel_views=panel_views, pack_cols_panel=pack_cols_panel, contract=contract)
    panels = max(1, min(args.bcast_panels, Nt))

    def step():
        if world > 1 and panels > 1:
            return mul_common_sharded_pipelined(a, b, cb, pops, rank, world, panels)
        return mul_common_sharded(a, b, tuple(cb.shape), ops, rank, world)

    for _ in range(args.warmup):
        ev["c0"], ev["c1"] = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        step()
    torch.cuda.synchronize()

    # One GPU: the step's launches are captured once into one CUDA graph
    # (packs, then the contraction) and replayed, so host launch gaps stay out
    # of the step (they dominate small shapes such as config 1); the
    # contraction's timing events are record nodes inside the graph.
    use_graph = world == 1 and not args.no_graph
    launches_per_step = None
    kernel_name = None
    if use_graph:
        # the whole step (both packs, concurrent, + the contraction) is ONE graph; the
        # contraction's timing events are record nodes inside it (external
        # events), so no host launch gap sits between packs and contraction
        g_step = torch.cuda.CUDAGraph()
        gc0 = torch.cuda.Event(enable_timing=True, external=True)
        gc1 = torch.cuda.Event(enable_timing=True, external=True)
        n0 = qg.kernel_launches()
        side = torch.cuda.Stream()
        with torch.cuda.graph(g_step):
            # the two packs are independent: B's runs on a forked branch of the graph
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                pack_cols(b)
            pack_rows(a)
            torch.cuda.current_stream().wait_stream(side)
            gc0.record()
            qg._check(qg.lib.qg_mul_common_tiled(ctypes.byref(gpc), qg._ptr(ca), qg._ptr(cb), m_rank, n, k,
                                                 qg._ptr(c), n, sp()))
            gc1.record()
        launches_per_step = qg.kernel_launches() - n0
        kernel_name = qg.last_kernel()

        def step():  # noqa: F811
            g_step.replay()
            ev["c0"], ev["c1"] = gc0, gc1
            return c

        for _ in range(3):
            step()
        torch.cuda.synchronize()

    step_ms, contract_ms = [], []
    launches0 = qg.kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    with ClockSampler(local_dev) as clk:
        for _ in range(args.steps):
            flush.fill_(1)  # evict L2 between timed steps (outside the events)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev["c0"], ev["c1"] = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            step()
            s1.record(stream)
            s1.synchronize()
            step_ms.append(s0.elapsed_time(s1))
            contract_ms.append(ev["c0"].elapsed_time(ev["c1"]))
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - wall0
    launches = qg.kernel_launches() - launches0
    if use_graph:  # replays do not pass through the library's launch counter
        launches = launches_per_step * args.steps
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = 2.0 * m_total * n * k / (ms_per_step * 1e-3)

    # parity spot-check inside the bench: checksum of this rank's C
    checksum = qg.residue_checksum(c)

    contract_avg = sum(contract_ms) / len(contract_ms)
    packed_flop = 2.0 * m_rank * n * K  # per launch: packed words, not padding
    peak_doc = load_json(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) or {}
    peak = float(peak_doc.get("dmma_m8n8k4_tflops", 37.09))
    achieved = packed_flop / (contract_avg * 1e-3) / 1e12
    ncu = load_json(os.path.join(ROOT, "profiles", "ncu_summary.json")) or {}
    traffic = ncu.get("contraction", {}).get(args.config, {}).get("dram_bytes") if ncu else None
    roofline = {"bound": "tensor", "achieved": round(achieved, 3), "peak": peak, "unit": "TFLOP/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": kernel_name or qg.last_kernel(), "kernel_ms": round(contract_avg, 4),
                "share_of_step": round(contract_avg / (sum(step_ms) / len(step_ms)), 4),
                "peak_source": "measured DMMA.8x8x4 microbenchmark on this pool (profiles/r01_fp64_peak.json); "
                               "cuBLAS DGEMM 35.7 TF/s",
                "algorithmic_flop_per_launch": packed_flop}

    line = {
        "metric": "effective mod-p mult-adds/sec (2mnk/s)", "value": value, "unit": "mult-adds/s (2mnk/s)",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SplitMix64 seeds 42/43, uniform residues, generated on device)",
        "config": {"workload": desc + (f"; {world} ranks x {m_rank} rows, CB broadcast over {args.dist_backend.upper()}"
                                       f" in {panels} column panels pipelined with rank 0's packing" if world > 1 else ""),
                   "p": p, "m": m_total, "k": k, "n": n,
                   "plan": {"t": pl.t, "e": pl.e, "kblock_words": gp.kblock_words, "stage_words": bk,
                            "source": args.plan},
                   "layout": "tiled packed operands (128 x stage_words blocks, CB transposed)" + (
                       "; contraction on 64x64 tiles with k split over a thread-block cluster"
                       if (kernel_name or "").startswith("small") else ""),
                   "l2": "flushed between timed steps (256 MiB write); A,B residues (2x128 MiB f64) exceed the 126 MB L2",
                   "parallelism": f"row-shard x{world}" if world > 1 else "single GPU",
                   "launch": "one CUDA graph per step (packs + contraction)" if use_graph else "direct launches"},
        "roofline": roofline,
        "gpu_launches": launches,
        "checksum_rank0": checksum if rank == 0 else None,
        "wall_s_timed_region": round(wall, 4),
    }
    line["clocks"] = clk.summary()

    if not args.no_e2e:
        e2e = e2e_measure(qg, gp, p, m_rank, k, n, args, rank, world, device_c=c)
        if rank == 0:
            line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            rate, rows, thr, dt, c_cpu, rpl, kind = reference_cpu_sample(p, m_rank, k, n, target_s=args.cpu_s)
            agree = bool(np.array_equal(c[:rows].cpu().numpy().astype(np.uint32), c_cpu))
            line["cpu_baseline"] = {"value": rate, "unit": "mult-adds/s (2mnk/s)", "cores": thr, "kind": kind,
                                    "sample": f"rows 0..{rows - 1} of the same A x B ({rows}x{k} x {k}x{n}), reference plan "
                                              f"t={rpl.t} e={rpl.e}, {dt:.2f} s wall",
                                    "rows_bit_exact_vs_gpu": agree}
        except Exception as ex:  # the baseline must not kill the measurement
            line["cpu_baseline"] = {"value": None, "error": str(ex)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def e2e_measure(qg, gp, p, m, k, n, args, rank=0, world=1, device_c=None):
    """Same metric through the public host-buffer API (pinned buffers):
    H2D of A and B (uint32 ResidueMatrix data), pack + contraction kernels,
    D2H of C, every step. At N GPUs every rank calls the API on its own row
    shard of A (rows rank*m ..), time = max over ranks."""
    import numpy as np
    import torch
    import torch.distributed as dist

    # seeded host inputs, made on the device by the library (K0) and copied out
    # before the timed region
    a = torch.empty((m, k), dtype=torch.int32, pin_memory=True)
    b = torch.empty((k, n), dtype=torch.int32, pin_memory=True)
    c = torch.empty((m, n), dtype=torch.int32, pin_memory=True)
    a.copy_(qg.random_residue_matrix(m, k, p, SEED, row0=rank * m, dtype=torch.int32))
    b.copy_(qg.random_residue_matrix(k, n, p, SEED + 1, dtype=torch.int32))
    torch.cuda.synchronize()
    an, bn, cn = a.numpy().view(np.uint32), b.numpy().view(np.uint32), c.numpy().view(np.uint32)
    for _ in range(3):
        qg.mul_common_compressed_host(an, bn, gp, out=cn)
    times = []
    for _ in range(args.e2e_steps):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        qg.mul_common_compressed_host(an, bn, gp, out=cn)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    if world > 1:
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    return {"value": 2.0 * m * world * n * k / t, "unit": "mult-adds/s (2mnk/s)",
            "h2d_bytes_per_step": int(a.numel() * 4 + b.numel() * 4) * world,
            "d2h_bytes_per_step": int(c.numel() * 4) * world, "ms_per_step": t * 1e3,
            "api": "mul_common_compressed_host (qg_host_mul_common_gpu), pipelined H2D/compute/D2H",
            "checksum_rank0": int(cn.astype(np.uint64).sum() & 0xFFFFFFFF),
            "matches_device": None if device_c is None else
            bool(np.array_equal(cn, device_c.cpu().numpy().astype(np.uint32)))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="config2", choices=sorted(CONFIGS))
    ap.add_argument("--plan", default="gpu", choices=["gpu", "reference"],
                    help="gpu: planner-chosen (t, e, kblock); reference: plan_compression's plan")
    ap.add_argument("--kblock", type=int, default=0, help="override the plan's k-block (words)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: functional check of the multi-rank path with several ranks on one GPU")
    ap.add_argument("--bcast-panels", type=int, default=4,
                    help="N>1: column panels the packed B is broadcast in (1 = one broadcast after the whole pack)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-s", type=float, default=4.0, help="target wall seconds of the CPU baseline sample")
    ap.add_argument("--ref-step-s", type=float, default=2.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the step's kernels directly (no CUDA graph)")
    ap.add_argument("--redq-plan", default="", help="experiments: right/left plan 't:e:kblock_residues:balanced'")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return reference_arm(args)
    if args.config in REDQ_VARIANTS:
        return redq_arm(args)
    return our_arm(args)


if __name__ == "__main__":
    sys.exit(main())
