#!/usr/bin/env python3
"""bench.py — effective mod-p multiply-adds per second (2mnk/s) of the
compressed modular GEMM on B200, the BASELINE.json metric.

Workload: BASELINE config 5 — p=3, m=n=k=32768, dot-product variant
(Q-adic rows reversed / columns forward, FP64 tensor-core contraction,
per-k-block digit extraction, mod-p accumulation between blocks), the config
BASELINE's "1/2/4/8 B200" metric is quoted on (--config picks another).
A "step" = pack A (K1) + pack B (K2) + the fused DMMA contraction/extract/mod-p
kernel (K4) on device-resident residues (seeded SplitMix64, K0, generated
once). N>1 (torchrun, one process per GPU) is STRONG scaling: the fixed m
rows of A and C are split over the ranks; each rank packs its own
tile-column slot of B and the slots are all-gathered in place over NCCL.

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
class RefCommon:
    """The reference's own dot-product path (oracle/_ref: the unmodified
    compress_cols_forward -> compress_rows_reversed -> packed_common_product
    -> reduce_common_entry, bench.hpp:127-146) at its own plan, with the
    packed B kept between calls: a full-size run packs B once for all m rows,
    so a row sample is charged its pro-rata share (r/m) of the measured
    single-threaded compress_cols_forward(B)."""

    def __init__(self, p, m, k, n):
        import ctypes

        import oracle

        self.ref = oracle.REF
        if self.ref is None:
            raise RuntimeError("oracle/_ref/libqgref.so is missing (built by __graft_entry__.build())")
        self.p, self.m, self.k, self.n = p, m, k, n
        self.plan = oracle.Plan()
        st = self.ref.qgref_plan_compression(p, k, 53, 0, ctypes.byref(self.plan))
        if st:
            raise RuntimeError(f"reference plan failed: {st}")
        b = oracle.random_residue_matrix(k, n, p, SEED + 1)
        sec = ctypes.c_double()
        self.cb = self.ref.qgref_cb_create(ctypes.byref(self.plan), b.ctypes.data_as(ctypes.c_void_p), k, n,
                                           ctypes.byref(sec))
        if not self.cb:
            raise RuntimeError("reference compress_cols_forward failed")
        self.pack_b_s = sec.value
        self._a = {}

    def run(self, rows, threads):
        """(charged seconds, wall seconds of the shards, C rows) for rows 0..rows-1."""
        import ctypes

        import numpy as np

        import oracle

        if rows not in self._a:
            self._a = {rows: oracle.random_residue_matrix(rows, self.k, self.p, SEED)}
        a = self._a[rows]
        c = np.empty((rows, self.n), dtype=np.uint32)
        wall = ctypes.c_double()
        st = self.ref.qgref_mul_common_cb(ctypes.byref(self.plan), self.cb, a.ctypes.data_as(ctypes.c_void_p), rows,
                                          self.k, c.ctypes.data_as(ctypes.c_void_p), threads, ctypes.byref(wall))
        if st:
            raise RuntimeError(f"reference mul_common failed: {st}")
        return wall.value + self.pack_b_s * rows / self.m, wall.value, c

    def sample(self, threads, target_s, rows=None):
        """Rate 2*rows*n*k / charged seconds on a row sample sized to ~target_s."""
        if rows is None:
            pilot = max(threads, 4)
            dt, _, _ = self.run(pilot, threads)
            rows = int(min(self.m, max(threads, pilot * target_s / max(dt, 1e-3))))
            rows = max(threads, rows // threads * threads) if rows >= threads else max(1, rows)
        dt, wall, c = self.run(rows, threads)
        return 2.0 * rows * self.n * self.k / dt, rows, dt, c

    def close(self):
        if self.cb:
            self.ref.qgref_cb_free(self.cb)
            self.cb = None


def reference_cpu_sample(p, m, k, n, target_s=4.0, threads=None, rows=None, one_thread_s=0.0):
    """The reference's dot-product path on a row sample of the seeded workload,
    rows sharded over all host threads (and, if one_thread_s > 0, a 1-thread
    figure too). Returns a cpu_baseline dict and the sampled C rows."""
    threads = threads or host_threads()
    rc = RefCommon(p, m, k, n)
    try:
        rate, rows, dt, c = rc.sample(threads, target_s, rows)
        out = {"value": rate, "unit": "mult-adds/s (2mnk/s)", "cores": threads, "kind": "reference",
               "sample": f"rows 0..{rows - 1} of the same A x B ({rows}x{k} x {k}x{n}) through the reference's "
                         f"compress_rows_reversed/packed_common_product/reduce_common_entry at its plan "
                         f"t={rc.plan.t} e={rc.plan.e}, rows sharded over {threads} threads; "
                         f"compress_cols_forward(B) ({rc.pack_b_s:.2f} s, 1 thread) charged pro rata {rows}/{m}",
               "seconds": round(dt, 3), "pack_b_s": round(rc.pack_b_s, 3)}
        if one_thread_s > 0:
            r1, rows1, dt1, _ = rc.sample(1, one_thread_s)
            out["one_thread"] = {"value": r1, "cores": 1, "rows": rows1, "seconds": round(dt1, 3)}
        return out, c
    finally:
        rc.close()


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
    """The reference's own CPU implementation of the path (oracle/_ref, the
    unmodified headers) on all host threads; each step is a bounded row
    sample of the workload (B packed once before the steps and charged pro
    rata per sample). Rank 0 alone runs it under torchrun."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    p, m, k, n, desc = CONFIGS[args.config]
    variant = REDQ_VARIANTS.get(args.config, "common")
    rates, rows_used, thr = [], None, host_threads()
    rc = None
    if variant == "common":
        rc = RefCommon(p, m, k, n)
    for i in range(args.warmup + args.steps):
        if variant == "common":
            rate, rows, dt, _ = rc.sample(thr, args.ref_step_s, rows_used)
            pdesc = f"t={rc.plan.t} e={rc.plan.e}"
        else:
            try:
                rate, rows, thr, dt, _, pl, kind = reference_variant_sample(variant, p, m, k, n,
                                                                            target_s=args.ref_step_s, rows=rows_used)
            except RuntimeError as ex:
                print(json.dumps({"impl": "reference", "unavailable": str(ex)}), flush=True)
                return 0
            pdesc = (f"t={pl.base.t} dq={pl.dq} dtheta={pl.dtheta}" if variant == "full" else f"t={pl.t} e={pl.e}")
        rows_used = rows
        if i >= args.warmup:
            rates.append(rate)
    value = sum(rates) / len(rates)
    sample = (f"rows 0..{rows_used - 1} of A ({rows_used}x{k}) x B ({k}x{n}), {variant} variant, reference plan "
              f"{pdesc}, {thr} threads")
    if rc is not None:
        sample += f"; compress_cols_forward(B) ({rc.pack_b_s:.2f} s, once) charged pro rata {rows_used}/{m} per step"
        rc.close()
    line = {
        "impl": "reference", "metric": "effective mod-p mult-adds/sec (2mnk/s)", "value": value, "unit": "mult-adds/s (2mnk/s)",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 2.0 * rows_used * n * k / value * 1e3,
        "higher_is_better": True, "scaling": "strong" if variant == "common" else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (SplitMix64 seed 42/43)",
        "config": {"workload": desc, "p": p, "m": m, "k": k, "n": n},
        "cpu_baseline": {"value": value, "unit": "mult-adds/s (2mnk/s)", "cores": thr, "kind": "reference", "sample": sample},
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
    """The dot-product variant (configs 1, 2, 3, 5). N=1: the whole product on
    one GPU, the step one CUDA graph (both packs on forked branches + the
    contraction). N>1 (torchrun, one process per GPU): STRONG scaling — the
    fixed m rows of A and C are sharded over the ranks (m/N each); every rank
    packs its own tile-column slot of B, the slots are all-gathered in place
    over NCCL (dist.mul_common_allgather) while the rank packs its CA shard
    and contracts its own columns, then it contracts the rest."""
    import ctypes

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_0803_1975_b200 as qg
    from paper_0803_1975_b200.dist import GatherOps, gather_slot, mul_common_allgather, shard_rows_aligned

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
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines (nranks) on stderr
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)

    p, m, k, n, desc = CONFIGS[args.config]
    gp = qg.plan_gpu(p, k) if args.plan == "gpu" else qg.gpu_plan_from(qg.plan_compression(p, k), k)
    if args.kblock:  # experiments: override the k-block of the chosen plan
        gp = qg.GpuPlan(gp.plan, args.kblock, gp.max_exact_words, gp.balanced,
                        gp.anchored if args.anchored < 0 else args.anchored)
    elif args.anchored >= 0:
        gp = qg.GpuPlan(gp.plan, gp.kblock_words, gp.max_exact_words, gp.balanced, args.anchored)
    pl = gp.plan
    K = -(-k // pl.e)
    row0, m_rank = shard_rows_aligned(m, world, rank)

    # device-resident seeded inputs (K0): this rank's rows of A; B (every rank
    # reads only its own tile-column slot of it when N > 1)
    a = qg.random_residue_matrix(max(m_rank, 1), k, p, SEED, row0=row0)
    b = qg.random_residue_matrix(k, n, p, SEED + 1)
    bk_c = ctypes.c_uint32()
    gpc = gp._c()
    qg._check(qg.lib.qg_tiled_stage_words(ctypes.byref(gpc), k, ctypes.byref(bk_c)))
    bk = bk_c.value
    Kt = (K + bk - 1) // bk
    Nt = (n + 127) // 128
    W = Kt * 128 * bk  # words per 128-column tile column of CB_t
    _, _, P = gather_slot(Nt, world, rank)
    # tiled packed layouts (dense zero-padded 128 x bk blocks, CB transposed);
    # N > 1: CB_t holds world * P tile columns (equal all-gather slots)
    ca = torch.empty(max(1, qg.lib.qg_tiled_words(m_rank, k, pl.e, bk)), dtype=torch.float64, device=dev)
    cb = torch.zeros(world * P * W if world > 1 else qg.lib.qg_tiled_words(n, k, pl.e, bk), dtype=torch.float64,
                     device=dev)
    c = torch.empty((max(m_rank, 1), n), dtype=torch.int32, device=dev)
    # --output cc: the compressed-out product (mul_common_repacked, gemm.hpp:275-280), one GPU
    repacked = args.output == "cc"
    if repacked and world > 1:
        raise SystemExit("--output cc runs on one GPU")
    H = -(-n // pl.e)
    cc_out = torch.empty((m_rank, H), dtype=torch.float64, device=dev) if repacked else None
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()
    sp = qg._stream

    def pack_rows(a_):
        if m_rank:
            qg._check(qg.lib.qg_pack_a_tiled(ctypes.byref(gpc), bk, qg._ptr(a_), 0, m_rank, k, k, qg._ptr(ca), sp()))
        return ca

    def pack_cols_slot(b_, t0, t1, slot):
        c0, c1 = t0 * 128, min(n, t1 * 128)
        if c1 > c0:
            qg._check(qg.lib.qg_pack_b_tiled(ctypes.byref(gpc), bk, ctypes.c_void_p(b_.data_ptr() + c0 * 8), 0, k,
                                             c1 - c0, n, qg._ptr(slot), sp()))

    kern_events = []

    def contract(ca_, cb_, t0, t1):
        c0, c1 = t0 * 128, min(n, t1 * 128)
        if c1 <= c0 or not m_rank:
            return
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        qg._check(qg.lib.qg_mul_common_tiled(ctypes.byref(gpc), qg._ptr(ca_), ctypes.c_void_p(cb_.data_ptr() + t0 * W * 8),
                                             m_rank, c1 - c0, k, ctypes.c_void_p(c.data_ptr() + c0 * 4), n, sp()))
        e1.record(stream)
        kern_events.append((e0, e1))

    ops = GatherOps(pack_rows=pack_rows, pack_cols_slot=pack_cols_slot, contract=contract)

    def step():
        mul_common_allgather(a, b, cb, ops, rank, world, Nt)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    kern_events.clear()

    # One GPU: the step's launches are captured once into one CUDA graph
    # (both packs on forked branches, then the contraction) and replayed, so
    # host launch gaps stay out of the step (they dominate small shapes such
    # as config 1); the contraction's timing events are record nodes inside it.
    use_graph = world == 1 and (not args.no_graph or repacked)
    launches_per_step = None
    kernel_name = None
    if use_graph:
        g_step = torch.cuda.CUDAGraph()
        gc0 = torch.cuda.Event(enable_timing=True, external=True)
        gc1 = torch.cuda.Event(enable_timing=True, external=True)
        n0 = qg.kernel_launches()
        side = torch.cuda.Stream()
        with torch.cuda.graph(g_step):
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                pack_cols_slot(b, 0, Nt, cb)
            pack_rows(a)
            torch.cuda.current_stream().wait_stream(side)
            gc0.record()
            if repacked:  # mul_common_repacked: ReduceAndCompress fused into the epilogue (EPI_REPACK)
                qg._check(qg.lib.qg_mul_common_repacked_tiled(ctypes.byref(gpc), qg._ptr(ca), qg._ptr(cb), m_rank, n,
                                                              k, qg._ptr(cc_out), H, sp()))
            else:
                qg._check(qg.lib.qg_mul_common_tiled(ctypes.byref(gpc), qg._ptr(ca), qg._ptr(cb), m_rank, n, k,
                                                     qg._ptr(c), n, sp()))
            gc1.record()
        launches_per_step = qg.kernel_launches() - n0
        kernel_name = qg.last_kernel()

        def step():  # noqa: F811
            g_step.replay()
            kern_events.append((gc0, gc1))

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
            kern_events.clear()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            step()
            s1.record(stream)
            s1.synchronize()
            step_ms.append(s0.elapsed_time(s1))
            contract_ms.append(sum(e0.elapsed_time(e1) for e0, e1 in kern_events))
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - wall0
    launches = qg.kernel_launches() - launches0
    if use_graph:  # replays do not pass through the library's launch counter
        launches = launches_per_step * args.steps
    kernel_name = kernel_name or qg.last_kernel()
    total_ms = sum(step_ms)
    per_rank_ms = [total_ms / args.steps]
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        per_rank_ms = [float(x.item()) / args.steps for x in allt]
        total_ms = max(float(x.item()) for x in allt)
    ms_per_step = total_ms / args.steps
    value = 2.0 * m * n * k / (ms_per_step * 1e-3)

    # parity spot-check inside the bench: checksum of this rank's C
    if repacked:  # C = uncompress(CC): its checksum must equal the plain product's
        c = qg.uncompress(qg.CompressedMatrix(m_rank, n, m_rank, H, qg.PackOrientation(
            qg.PackDirection.Forward, qg.PackAxis.Column, pl.e), pl, cc_out))
    checksum = qg.residue_checksum(c[:m_rank]) if m_rank else 0
    # config 5: the reference's golden row shards (tests/golden/golden.json,
    # made by oracle/_ref) that fall in this rank's rows, sha256 of the bytes
    golden_rows = golden_row_shards(args.config, c, row0, m_rank)
    if world > 1:
        cs = torch.tensor([checksum, golden_rows[0], golden_rows[1]], dtype=torch.int64, device=dev)
        dist.all_reduce(cs)
        checksum = int(cs[0].item()) & 0xFFFFFFFF
        golden_rows = (int(cs[1].item()), int(cs[2].item()))

    contract_avg = sum(contract_ms) / len(contract_ms)
    packed_flop = 2.0 * m_rank * n * K  # per step on this rank: packed words, not padding
    peak_doc = load_json(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) or {}
    peak = float(peak_doc.get("dmma_m8n8k4_tflops", 37.09))
    achieved = packed_flop / (contract_avg * 1e-3) / 1e12 if contract_avg > 0 else 0.0
    ncu = load_json(os.path.join(ROOT, "profiles", "ncu_summary.json")) or {}
    traffic = ncu.get("contraction", {}).get(args.config, {}).get("dram_bytes") if ncu else None
    roofline = {"bound": "tensor", "achieved": round(achieved, 3), "peak": peak, "unit": "TFLOP/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": kernel_name, "kernel_ms": round(contract_avg, 4),
                "share_of_step": round(contract_avg / (sum(step_ms) / len(step_ms)), 4),
                "peak_source": "measured DMMA.8x8x4 microbenchmark on this pool (profiles/r01_fp64_peak.json); "
                               "cuBLAS DGEMM 35.7 TF/s",
                "algorithmic_flop_per_launch": packed_flop,
                "per_unit": "2 FLOP per packed word product; m_rank x n x ceil(k/e) products per step"}
    if world > 1:
        roofline["note"] = (f"rank 0's contraction launches ({'1 own-slot + rest' if world > 1 else ''}) summed; "
                            "the own-slot launch shares the SMs with the NCCL all-gather")

    par = (f"strong scaling: {world} ranks x {m_rank} rows of the fixed m={m}; packed B assembled by an in-place "
           f"NCCL all-gather of per-rank tile-column slots ({P} of {Nt} tile columns each), own slot contracted "
           f"first" if world > 1 else "single GPU")
    line = {
        "metric": "effective mod-p mult-adds/sec (2mnk/s)", "value": value, "unit": "mult-adds/s (2mnk/s)",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SplitMix64 seeds 42/43, uniform residues, generated on device)",
        "config": {"workload": desc + ("; output CC = mul_common_repacked (ReduceAndCompress fused)" if repacked else ""),
                   "p": p, "m": m, "k": k, "n": n,
                   "plan": {"t": pl.t, "e": pl.e, "kblock_words": gp.kblock_words, "stage_words": bk, "anchored": bool(gp.anchored),
                            "balanced": bool(gp.balanced), "source": args.plan},
                   "layout": "tiled packed operands (128 x stage_words blocks, CB transposed)" + (
                       "; contraction on 64x64 tiles with k split over a thread-block cluster"
                       if (kernel_name or "").startswith("small") else ""),
                   "l2": f"flushed between timed steps (256 MiB write); A,B residues "
                         f"({(m_rank * k + k * n) * 8 / 2**20:.0f} MiB f64 per rank) exceed the 126 MB L2",
                   "parallelism": par,
                   "launch": "one CUDA graph per step (packs + contraction)" if use_graph else "direct launches"},
        "roofline": roofline,
        "gpu_launches": launches,
        "checksum_c": checksum,
        "golden_row_shards": ({"checked": golden_rows[0], "match": golden_rows[1] == golden_rows[0],
                               "source": "tests/golden/golden.json config5_rows (reference-made), all ranks"}
                              if golden_rows[0] else None),
        "per_rank_ms": [round(x, 3) for x in per_rank_ms],
        "wall_s_timed_region": round(wall, 4),
    }
    line["clocks"] = clk.summary()
    del flush

    if not args.no_e2e:
        e2e = e2e_measure(qg, gp, p, m, k, n, args, rank, world, device_c=c[:m_rank])
        if rank == 0:
            line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            base, c_cpu = reference_cpu_sample(p, m, k, n, target_s=args.cpu_s, one_thread_s=args.cpu1_s)
            base["rows_bit_exact_vs_gpu"] = bool(np.array_equal(c[:c_cpu.shape[0]].cpu().numpy().astype(np.uint32),
                                                                c_cpu))
            line["cpu_baseline"] = base
        except Exception as ex:  # the baseline must not kill the measurement
            line["cpu_baseline"] = {"value": None, "error": str(ex)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def golden_row_shards(config, c, row0, rows):
    """(shards checked, shards matching) of the reference's golden row shards
    of `config` (sha256 of the residues as bytes) inside rows [row0, row0+rows)
    of this rank's C."""
    import hashlib

    if config != "config5":
        return (0, 0)
    g = load_json(os.path.join(ROOT, "tests", "golden", "golden.json")) or {}
    shards = g.get("configs", {}).get("config5_rows", {}).get("shards", [])
    checked = match = 0
    for sh in shards:
        r0, nr = sh["row0"], sh["rows"]
        if r0 >= row0 and r0 + nr <= row0 + rows:
            blk = c[r0 - row0:r0 - row0 + nr].cpu().numpy().astype("uint8")
            checked += 1
            match += hashlib.sha256(blk.tobytes()).hexdigest() == sh["sha256_u8"]
    return (checked, match)


def e2e_measure(qg, gp, p, m, k, n, args, rank=0, world=1, device_c=None):
    """Same metric through the public host-buffer API: H2D of A and B (uint32
    ResidueMatrix data), pack + contraction kernels, D2H of C, every step.
    Headline from pinned host buffers; the same call on pageable buffers (a
    plain std::vector / numpy array, what a reference caller passes) is
    reported beside it. N > 1: every rank runs the API on its own row shard
    (rows row0.. of the fixed m), time = max over ranks."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_0803_1975_b200.dist import shard_rows_aligned

    row0, mr = shard_rows_aligned(m, world, rank)
    # seeded host inputs, made on the device by the library (K0) and copied out
    # before the timed region
    a = torch.empty((mr, k), dtype=torch.int32, pin_memory=True)
    b = torch.empty((k, n), dtype=torch.int32, pin_memory=True)
    c = torch.empty((mr, n), dtype=torch.int32, pin_memory=True)
    if mr:
        a.copy_(qg.random_residue_matrix(mr, k, p, SEED, row0=row0, dtype=torch.int32))
    b.copy_(qg.random_residue_matrix(k, n, p, SEED + 1, dtype=torch.int32))
    torch.cuda.synchronize()
    an, bn, cn = a.numpy().view(np.uint32), b.numpy().view(np.uint32), c.numpy().view(np.uint32)

    from paper_0803_1975_b200.dist import mul_common_allgather_host

    repacked = args.output == "cc"
    cc_host = np.empty((mr, -(-n // gp.plan.e)), dtype=np.float64) if repacked else None

    def call(a_, b_, c_):
        if world > 1:  # each rank sends only its slot of B over its PCIe link; NCCL all-gather of packed slots
            return mul_common_allgather_host(a_, b_, gp, rank, world, out=c_)
        if repacked:  # CC words back (8/e bytes per residue), C unpacked on the device afterwards for the checks
            qg.mul_common_repacked_host(a_, b_, gp, out=cc_host)
            return c_
        return qg.mul_common_compressed_host(a_, b_, gp, out=c_)

    def timed(a_, b_, c_, steps):
        for _ in range(2):
            call(a_, b_, c_)
        times = []
        for _ in range(steps):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            call(a_, b_, c_)
            times.append(time.perf_counter() - t0)
        t = sum(times) / len(times)
        if world > 1:
            tt = torch.tensor([t], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        return t

    t = timed(an, bn, cn, args.e2e_steps)
    if repacked:
        pl = gp.plan
        cn[:] = qg.uncompress(qg.CompressedMatrix(mr, n, mr, cc_host.shape[1], qg.PackOrientation(
            qg.PackDirection.Forward, qg.PackAxis.Column, pl.e), pl, torch.from_numpy(cc_host).cuda())).cpu().numpy()
    out = {"value": 2.0 * m * n * k / t, "unit": "mult-adds/s (2mnk/s)",
           "h2d_bytes_per_step": int((m * k + k * n) * 4),
           "d2h_bytes_per_step": int(cc_host.nbytes if repacked else m * n * 4), "ms_per_step": t * 1e3,
           "api": ("mul_common_repacked_host (qg_host_mul_common_repacked_gpu: CC words back), pinned buffers"
                   if repacked else
                   "mul_common_compressed_host (qg_host_mul_common_gpu), pipelined H2D/compute/D2H, pinned buffers"
                   if world == 1 else
                   f"dist.mul_common_allgather_host on each of {world} ranks (its row shard of A and its 1/{world} "
                   "column slot of B over its own PCIe link, packed slots all-gathered over NCCL, C shard back), "
                   "pinned buffers"),
           "checksum_rank0": int(cn.astype(np.uint64).sum() & 0xFFFFFFFF),
           "matches_device": None if device_c is None else
           bool(np.array_equal(cn, device_c.cpu().numpy().astype(np.uint32)))}
    if args.pageable and world == 1 and not repacked:
        del a, b, c
        ap_, bp_ = np.array(an), np.array(bn)  # plain (pageable) copies
        cp_ = np.empty_like(cn)
        tpg = timed(ap_, bp_, cp_, max(2, args.e2e_steps // 2))
        out["pageable"] = {"value": 2.0 * m * n * k / tpg, "ms_per_step": tpg * 1e3,
                           "api": "the same call on pageable (non-pinned) numpy buffers",
                           "matches_pinned": bool(np.array_equal(cp_, cn))}
    return out


def make_parser():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="config5", choices=sorted(CONFIGS))
    ap.add_argument("--plan", default="gpu", choices=["gpu", "reference"],
                    help="gpu: planner-chosen (t, e, kblock); reference: plan_compression's plan")
    ap.add_argument("--kblock", type=int, default=0, help="override the plan's k-block (words)")
    ap.add_argument("--anchored", type=int, default=-1,
                    help="experiments: force the plan's anchored flag (K4A) on (1) / off (0)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: functional check of the multi-rank path with several ranks on one GPU")
    ap.add_argument("--pageable", type=int, default=1, help="also time e2e from pageable host buffers (N=1)")
    ap.add_argument("--output", default="c", choices=["c", "cc"],
                    help="c: int32 C (mul_common_compressed); cc: forward-packed CC words (mul_common_repacked)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-s", type=float, default=4.0, help="target wall seconds of the CPU baseline sample")
    ap.add_argument("--cpu1-s", type=float, default=3.0, help="target seconds of the 1-thread CPU sample (0: skip)")
    ap.add_argument("--ref-step-s", type=float, default=2.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the step's kernels directly (no CUDA graph)")
    ap.add_argument("--redq-plan", default="", help="experiments: right/left plan 't:e:kblock_residues:balanced'")
    return ap


def main():
    args = make_parser().parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return reference_arm(args)
    if args.config in REDQ_VARIANTS:
        return redq_arm(args)
    return our_arm(args)


if __name__ == "__main__":
    sys.exit(main())
