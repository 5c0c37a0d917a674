"""Randomised parity soak of the entry points added late in round 1 (and the
round-2 ones: the fused repack, the all-gather host entry, pinned host
buffers next to pageable ones), against
the oracle (oracle/qg_oracle.c, pinned to the reference): the small-product
cluster kernel (forced on and off), the one-call device entry, the 2-D and
k-split host pipelines (forced), the mixed / left host paths and the
one-process multi-GPU entry. Random p, shapes, plans (balanced / unsigned /
reference) and split counts; stops at the first mismatch and prints the case.

    python tools/soak.py --seconds 600 > gpurun_out/soak.log
"""
import argparse
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--big", action="store_true", help="shapes up to 4096 (the 128x128-tile kernels)")
    args = ap.parse_args()
    import torch

    import oracle as orc
    import paper_0803_1975_b200 as qg

    rng = random.Random(args.seed)
    primes = [2, 3, 5, 7, 11, 13, 31, 251]
    t_end = time.time() + args.seconds
    n_cases = 0
    env_keys = ("QG_SMALL", "QG_SMALL_SPLITS", "QG_HOST_2D", "QG_HOST_PANELS", "QG_HOST_TILES", "QG_HOST_KSPLIT",
                "QG_HOST_KPARTS")
    while time.time() < t_end:
        for key in env_keys:
            os.environ.pop(key, None)
        p = rng.choice(primes)
        if args.big:
            m, n = rng.choice([1024, 2047, 2048, 3000, 4096]), rng.choice([1024, 1536, 2050, 4096])
            k = rng.choice([256, 1000, 4096, 9000])
        else:
            m, n = rng.choice([1, 7, 64, 65, 300, 700, 1500]), rng.choice([1, 2, 33, 128, 129, 640, 1300])
            k = rng.choice([1, 3, 50, 257, 1000, 3000, 6000])
        a = orc.random_residue_matrix(m, k, p, rng.randrange(1 << 30))
        b = orc.random_residue_matrix(k, n, p, rng.randrange(1 << 30))
        want = orc.naive_gemm(p, a, b)
        kind = rng.choice(["device", "host", "right", "left", "multi", "repack", "repack_host", "allgather"])
        try:
            gp = qg.plan_gpu(p, k, balanced=rng.random() < 0.6, anchored=rng.random() < 0.7)
        except qg.Error:
            continue
        desc = f"kind={kind} p={p} m={m} k={k} n={n} plan={gp}"
        if kind == "device":
            os.environ["QG_SMALL"] = rng.choice(["0", "1", "auto"])
            if rng.random() < 0.5:
                os.environ["QG_SMALL_SPLITS"] = str(rng.choice([1, 2, 3, 5, 8]))
            dt = rng.choice([torch.float64, torch.int32])
            ad = torch.from_numpy(a.astype(np.float64)).to("cuda", dt)
            bd = torch.from_numpy(b.astype(np.float64)).to("cuda", dt)
            got = qg.mul_common_compressed(ad, bd, gp).cpu().numpy().astype(np.uint32)
            desc += f" small={os.environ['QG_SMALL']} splits={os.environ.get('QG_SMALL_SPLITS')} dtype={dt}"
        elif kind == "host":
            os.environ["QG_HOST_2D"] = rng.choice(["0", "1"])
            os.environ["QG_HOST_PANELS"] = str(rng.choice([1, 2, 3, 4, 8]))
            os.environ["QG_HOST_TILES"] = str(rng.choice([1, 8, 96]))
            got = qg.mul_common_compressed_host(a, b, gp)
            desc += f" 2d={os.environ['QG_HOST_2D']} panels={os.environ['QG_HOST_PANELS']}"
        elif kind in ("right", "left"):
            os.environ["QG_HOST_KSPLIT"] = rng.choice(["0", "1"])
            os.environ["QG_HOST_KPARTS"] = str(rng.choice([1, 2, 3, 8]))
            try:
                rp = qg.plan_right_gpu(p, k, n if kind == "right" else m)
            except qg.Error:
                continue
            desc += f" ksplit={os.environ['QG_HOST_KSPLIT']} parts={os.environ['QG_HOST_KPARTS']} rplan={rp}"
            e, t = rp.plan.e, rp.plan.t
            if kind == "right":
                w = qg.mul_right_compressed_host(a, b, rp).astype(np.uint64)
                digits = np.zeros((m, -(-n // e) * e), dtype=np.uint64)
                for s in range(e):
                    digits[:, s::e] = (w >> np.uint64(t * s)) & np.uint64((1 << t) - 1)
                got = digits[:, :n].astype(np.uint32)
            else:
                w = qg.mul_left_compressed_host(a, b, rp).astype(np.uint64)
                digits = np.zeros((-(-m // e) * e, n), dtype=np.uint64)
                for s in range(e):
                    digits[s::e, :] = (w >> np.uint64(t * s)) & np.uint64((1 << t) - 1)
                got = digits[:m].astype(np.uint32)
        elif kind in ("repack", "repack_host"):  # mul_common_repacked: CC words, unpacked here
            os.environ["QG_SMALL"] = rng.choice(["0", "1", "auto"])
            plan = gp if rng.random() < 0.7 else None
            if plan is None:
                try:
                    plan = qg.plan_compression(p, k)
                except qg.Error:
                    continue
            base = plan.plan if isinstance(plan, qg.GpuPlan) else plan
            if kind == "repack":
                w = qg.mul_common_repacked(torch.from_numpy(a.astype(np.float64)).cuda(),
                                           torch.from_numpy(b.astype(np.float64)).cuda(), plan).data.cpu().numpy()
            else:
                w = qg.mul_common_repacked_host(a, b, plan)
            w = w.astype(np.uint64)
            e, t = base.e, base.t
            digits = np.zeros((m, -(-n // e) * e), dtype=np.uint64)
            for s in range(e):
                digits[:, s::e] = (w >> np.uint64(t * s)) & np.uint64((1 << t) - 1)
            got = digits[:, :n].astype(np.uint32)
            desc += f" small={os.environ['QG_SMALL']} repack_plan={base}"
        elif kind == "allgather":  # the multi-process host entry at world size 1
            from paper_0803_1975_b200.dist import mul_common_allgather_host

            if rng.random() < 0.5:  # pinned host buffers (the other half pageable)
                ap_ = torch.from_numpy(a.view(np.int32)).pin_memory().numpy().view(np.uint32)
                bp_ = torch.from_numpy(b.view(np.int32)).pin_memory().numpy().view(np.uint32)
                a, b = ap_, bp_
                desc += " pinned"
            got = mul_common_allgather_host(a, b, gp, 0, 1)
        else:
            got = qg.mul_common_multi_host(a, b, gp, list(range(torch.cuda.device_count())))
        n_cases += 1
        if not np.array_equal(got, want):
            bad = np.argwhere(got != want)
            print(f"MISMATCH after {n_cases} cases: {desc}; {len(bad)} entries differ, first {bad[:3].tolist()}",
                  flush=True)
            return 1
        if n_cases % 50 == 0:
            print(f"{n_cases} cases ok", flush=True)
    print(f"soak ok: {n_cases} random cases, all equal to naive_gemm", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
