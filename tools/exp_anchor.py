"""Experiment: K4A (anchored accumulation) correctness on worst-case operands."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_0803_1975_b200 as qg
from test_gpu_edge import operands, exact_c

cuda = torch.device("cuda:0")
for p, k, kb in [(3, 32768, 12), (7, 4096, 28), (3, 4099, 12), (3, 6000, 20)]:
    gp0 = qg.plan_gpu(p, k)
    words, E = qg.max_exact_block_anchored(gp0.plan)
    print("p", p, "k", k, "plan", gp0.plan.t, gp0.plan.e, "kb", gp0.kblock_words, "anchored max", words, "E", E)
    gp = qg.GpuPlan(gp0.plan, kb, gp0.max_exact_words, 1, 1)
    for (m, n) in [(256, 256), (384, 300)]:
        a, b = operands(p, gp.plan.e, m, k, n)
        want = exact_c(a, b, p)
        try:
            got = qg.mul_common_compressed(torch.from_numpy(a.astype(np.float64)).to(cuda),
                                           torch.from_numpy(b.astype(np.float64)).to(cuda), gp)
        except Exception as ex:
            print("  ", m, n, "error", type(ex).__name__, ex)
            continue
        got = got.cpu().numpy().astype(np.uint32)
        print("  ", m, n, qg.last_kernel(), "mismatches", int((got != want).sum()))
