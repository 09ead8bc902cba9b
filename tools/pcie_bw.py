"""DIAGNOSTIC: pinned host <-> device copy bandwidth (one direction at a time, and both at
once on two streams), the bound of bench.py's e2e number."""
import time, torch
n = 512 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
def timed(fn, reps=5):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / reps
t_h2d = timed(lambda: d.copy_(h, non_blocking=True))
t_d2h = timed(lambda: h.copy_(d, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
t_both = timed(both)
print(f"h2d {n/t_h2d/1e9:.1f} GB/s, d2h {n/t_d2h/1e9:.1f} GB/s, both directions at once {2*n/t_both/1e9:.1f} GB/s total")
