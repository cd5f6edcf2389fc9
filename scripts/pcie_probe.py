"""PCIe probe: pinned H2D alone, D2H alone, and both at once on two streams (GB/s)."""
import torch
N = 2 << 30
xd, yd = torch.empty(N, dtype=torch.uint8, device="cuda"), torch.empty(N, dtype=torch.uint8, device="cuda")
xh, yh = torch.empty(N, dtype=torch.uint8, pin_memory=True), torch.empty(N, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)
for _ in range(2):
    a = t(lambda: xd.copy_(xh, non_blocking=True))
    b = t(lambda: yh.copy_(yd, non_blocking=True))
    def both():
        ev = torch.cuda.Event(); ev.record()
        s1.wait_event(ev); s2.wait_event(ev)
        with torch.cuda.stream(s1): xd.copy_(xh, non_blocking=True)
        with torch.cuda.stream(s2): yh.copy_(yd, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    c = t(both)
print(f"h2d {N/a/1e6:.1f} GB/s, d2h {N/b/1e6:.1f} GB/s, both at once {2*N/c/1e6:.1f} GB/s total ({c:.1f} ms vs {a+b:.1f} serial)")
