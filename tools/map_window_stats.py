#!/usr/bin/env python
"""How local is the cell-list build's permutation?  For the output position d of
every particle, its source s(d) in the input array; per tile of T output slots,
the share of sources outside the window [j0 + drift - H, j0 + T + drift + H),
drift = the median of s(d) - d over 32 samples of the tile (what a producer warp
can estimate from the slot map).  Decides whether a copy-engine window gather
(tools/gather_tma_probe.cu) pays on the real workload.

    python tools/map_window_stats.py [config] [warm steps] [dump path]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2406_16786_b200 import inputs, sphbuf


def main():
    config = sys.argv[1] if len(sys.argv) > 1 else "C5"
    warm = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    dev = torch.device("cuda", 0)
    w = inputs.make(config, device=dev)
    bu = sphbuf.BufferUpdater(w.grid, w.h, w.dp, w.ports, inputs.capacity_for(w, 0.05), device=dev)
    bu.load(w.state, w.next_id)
    del w.state
    bu.register_ports()
    for _ in range(warm):
        bu.step(w.dt, deferred=True)
    n_in = bu.stats()["n"]
    perm = torch.full((bu.capacity,), -1, dtype=torch.int32, device=dev)
    bu.cll_build(perm=perm, dt=w.dt)
    torch.cuda.synchronize()
    n_out = bu.A.count()
    p = perm[:n_in].long()
    keep = p >= 0
    src = torch.full((n_out,), -1, dtype=torch.int64, device=dev)
    src[p[keep]] = torch.arange(n_in, device=dev)[keep]
    d = torch.arange(n_out, device=dev)
    delta = src - d
    print(f"{config}: n_in {n_in} n_out {n_out}; |s(d) - d|: median {delta.abs().median().item()}, "
          f"p90 {delta.abs().float().quantile(0.9).item() if n_out < 16_000_000 else 'n/a'}")
    for T in (512, 1024, 2048):
        nt = n_out // T
        dl = delta[:nt * T].view(nt, T)
        samp = dl[:, ::T // 32]
        drift = samp.median(dim=1).values
        for H in (32, 64, 128, 256):
            rel = dl - drift[:, None]
            j = torch.arange(T, device=dev)[None, :]
            outside = ((rel + j) < -H) | ((rel + j) >= T + H)
            frac = outside.float().mean().item()
            print(f"  T={T} H={H}: sources outside the window {100 * frac:.2f}%  "
                  f"(window bytes / useful {(T + 2 * H) / T:.3f})")
    if len(sys.argv) > 3:        # --dump path: the map as int32 for tools/gather_tma_probe.cu
        src.clamp(min=0).to(torch.int32).cpu().numpy().tofile(sys.argv[3])
    # how far the outside sources are
    rel = (delta[:(n_out // 1024) * 1024].view(-1, 1024) - delta[:(n_out // 1024) * 1024].view(-1, 1024)[:, ::32]
           .median(dim=1).values[:, None]).abs().flatten()
    for lim in (64, 1024, 8192, 65536, 1 << 20):
        print(f"  |s(d) - d - drift| > {lim}: {100 * (rel > lim).float().mean().item():.3f}%")


if __name__ == "__main__":
    main()
