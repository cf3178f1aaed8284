"""PCIe ceiling of the end-to-end loop: 4.59 GB (the C5 state) host->device, device->host
and both at once from pinned memory.   python tools/pcie_probe.py"""
import torch, time
n = 4_590_000_000 // 4
h1 = torch.empty(n, dtype=torch.float32, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
up, down = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); torch.cuda.synchronize(); e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)
for _ in range(2):
    a = t(lambda: d1.copy_(h1, non_blocking=True))
    b = t(lambda: h2.copy_(d2, non_blocking=True))
    def both():
        with torch.cuda.stream(up): d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(down): h2.copy_(d2, non_blocking=True)
    c = t(both)
    print(f"H2D {a:.1f} ms ({4.59/a*1e3:.1f} GB/s)  D2H {b:.1f} ms ({4.59/b*1e3:.1f} GB/s)  both {c:.1f} ms ({2*4.59/c*1e3:.1f} GB/s total)")
