"""Host<->device copy bandwidth with pinned buffers (context for the e2e line)."""
import torch
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record(); torch.cuda.synchronize()
    print(name, "GB/s", 5 * n / (e0.elapsed_time(e1) / 1e3) / 1e9)
# both directions at once
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
with torch.cuda.stream(s):
    for _ in range(5):
        d2.copy_(h2, non_blocking=True)
for _ in range(5):
    h.copy_(d, non_blocking=True)
torch.cuda.current_stream().wait_stream(s)
e1.record(); torch.cuda.synchronize()
print("duplex GB/s (sum)", 10 * n / (e0.elapsed_time(e1) / 1e3) / 1e9)
