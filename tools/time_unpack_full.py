import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes, torch, paper_0803_1975_b200 as qg
fp, kb = qg.plan_full_gpu(5, 8192)
m = n = 8192
G, H = m // fp.q_slots(), n // fp.theta_slots()
cc = torch.zeros((G, H), dtype=torch.float64, device="cuda")
c = torch.empty((m, n), dtype=torch.int32, device="cuda")
f = fp._c()
for i in range(3):
    qg._check(qg.lib.qg_uncompress_full(ctypes.byref(f), qg._ptr(cc), H, m, n, qg._ptr(c), n, qg._stream()))
torch.cuda.synchronize()
s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s0.record()
for i in range(10):
    qg._check(qg.lib.qg_uncompress_full(ctypes.byref(f), qg._ptr(cc), H, m, n, qg._ptr(c), n, qg._stream()))
s1.record(); s1.synchronize()
print("uncompress_full ms", s0.elapsed_time(s1) / 10, fp.base.t, fp.q_slots(), fp.theta_slots())
