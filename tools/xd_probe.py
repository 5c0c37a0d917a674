import ctypes, numpy as np, torch
import paper_0803_1975_b200 as qg
pl = qg.make_plan(3, 5, 3)._c()
for dt, fn in [(torch.float64, qg.lib.qg_extract_digits), (torch.int64, qg.lib.qg_extract_digits_u64)]:
    w = torch.tensor([2081, 33, 1024, 31, 32, 2048+32], dtype=dt, device="cuda")
    out = torch.zeros(w.numel()*3, dtype=torch.int64, device="cuda")
    st = fn(ctypes.byref(pl), qg._ptr(w), w.numel(), qg._ptr(out), None)
    torch.cuda.synchronize()
    print(dt, st, out.view(-1,3).tolist())
