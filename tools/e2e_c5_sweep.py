"""Config 5 e2e (host buffers, pinned) through qg_host_mul_common_gpu under
2-D pipeline geometries: QG_HOST_PANELS x QG_HOST_TILES (GPU box)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0803_1975_b200 as qg  # noqa: E402

p, m, k, n = 3, 32768, 32768, 32768
gp = qg.plan_gpu(p, k)
a = torch.empty((m, k), dtype=torch.int32, pin_memory=True)
b = torch.empty((k, n), dtype=torch.int32, pin_memory=True)
c = torch.empty((m, n), dtype=torch.int32, pin_memory=True)
a.copy_(qg.random_residue_matrix(m, k, p, 42, dtype=torch.int32))
b.copy_(qg.random_residue_matrix(k, n, p, 43, dtype=torch.int32))
torch.cuda.synchronize()
an, bn, cn = (x.numpy().view(np.uint32) for x in (a, b, c))
for spec in sys.argv[1:]:
    P, T = spec.split("x")
    os.environ["QG_HOST_PANELS"], os.environ["QG_HOST_TILES"] = P, T
    qg.mul_common_compressed_host(an, bn, gp, out=cn)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        qg.mul_common_compressed_host(an, bn, gp, out=cn)
        ts.append(time.perf_counter() - t0)
    print(f"panels={P} tiles={T}: {min(ts)*1e3:.1f} ms min, {sum(ts)/3*1e3:.1f} ms avg, checksum "
          f"{int(cn.astype(np.uint64).sum() & 0xFFFFFFFF)}", flush=True)
