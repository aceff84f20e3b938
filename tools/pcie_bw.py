"""Pinned host<->device copy bandwidth (the e2e ceiling), CUDA events."""
import torch

n = 512 << 20
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True)
    h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)),
                 ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(name, f"{5 * n / (a.elapsed_time(b) * 1e-3) / 1e9:.1f} GB/s")
# both directions at once
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
with torch.cuda.stream(s1):
    for _ in range(5):
        d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    for _ in range(5):
        h2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1)
torch.cuda.current_stream().wait_stream(s2)
b.record()
torch.cuda.synchronize()
print("bidir", f"{10 * n / (a.elapsed_time(b) * 1e-3) / 1e9:.1f} GB/s total")
