"""Raw pinned H2D / D2H copy rates on this box (the e2e floor)."""
import torch
n = 128 * 1024 * 1024
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(10):
        fn()
    s1.record()
    s1.synchronize()
    ms = s0.elapsed_time(s1) / 10
    print(name, round(n / ms / 1e6, 1), "GB/s")

# both directions at once (the pipelined host path overlaps C's D2H with A's H2D)
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
h2, d2 = torch.empty(n, dtype=torch.uint8, pin_memory=True), torch.empty(n, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s0.record()
s_in.wait_event(s0)
s_out.wait_event(s0)
for _ in range(10):
    with torch.cuda.stream(s_in):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s_out):
        h2.copy_(d2, non_blocking=True)
e_in, e_out = torch.cuda.Event(), torch.cuda.Event()
e_in.record(s_in)
e_out.record(s_out)
torch.cuda.current_stream().wait_event(e_in)
torch.cuda.current_stream().wait_event(e_out)
s1.record()
s1.synchronize()
ms = s0.elapsed_time(s1) / 10
print("bidirectional", round(2 * n / ms / 1e6, 1), "GB/s total,", round(n / ms / 1e6, 1), "per direction")
