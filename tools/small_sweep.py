"""Times the one-launch small path (QG_SMALL=1) against the tiled packs +
contraction (QG_SMALL=0) through qg_mul_common_compressed on device residues,
for a ladder of shapes, to place the library's switch-over. One JSON line per
(shape, path): median of CUDA-event timed calls after warm-up."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_0803_1975_b200 as qg

    shapes = [(3, 512, 512, 512), (7, 512, 4096, 512), (3, 768, 768, 768), (3, 1024, 1024, 1024),
              (7, 1024, 4096, 1024), (3, 1536, 1536, 1536), (3, 2048, 256, 2048), (7, 2048, 2048, 2048),
              (3, 256, 32768, 256), (3, 384, 8192, 384), (5, 1024, 8192, 640)]
    if len(sys.argv) > 1:
        shapes = [tuple(int(x) for x in s.split(",")) for s in sys.argv[1:]]
    for p, m, k, n in shapes:
        a = qg.random_residue_matrix(m, k, p, 42)
        b = qg.random_residue_matrix(k, n, p, 43)
        gp = qg.plan_gpu(p, k)
        g = gp._c()
        c = torch.empty((m, n), dtype=torch.int32, device="cuda")
        ref = None
        for path in ("1", "0"):
            os.environ["QG_SMALL"] = path
            call = lambda: qg._check(qg.lib.qg_mul_common_compressed(  # noqa: E731
                ctypes.byref(g), qg._ptr(a), k, qg._ptr(b), n, 0, m, k, n, qg._ptr(c), n, qg._stream()))
            for _ in range(3):
                call()
            torch.cuda.synchronize()
            kern = qg.last_kernel()
            ts = []
            for _ in range(15):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                call()
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            ms = ts[len(ts) // 2]
            if ref is None:
                ref = c.clone()
            same = bool(torch.equal(ref, c))
            print(json.dumps({"p": p, "m": m, "k": k, "n": n, "small": path == "1", "kernel": kern, "ms": round(ms, 5),
                              "eff_Tps": round(2.0 * m * n * k / (ms * 1e-3) / 1e12, 3),
                              "packed_TF": round(2.0 * m * n * -(-k // gp.plan.e) / (ms * 1e-3) / 1e12, 3),
                              "same_c": same}), flush=True)


if __name__ == "__main__":
    main()
