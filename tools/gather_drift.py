#!/usr/bin/env python
"""Per-update kernel times over a long run (does the build slow down as the flow
develops?).   python tools/gather_drift.py [config] [updates]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2406_16786_b200 import inputs, sphbuf


def main():
    config = sys.argv[1] if len(sys.argv) > 1 else "C5"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    dev = torch.device("cuda", 0)
    w = inputs.make(config, device=dev)
    bu = sphbuf.BufferUpdater(w.grid, w.h, w.dp, w.ports, inputs.capacity_for(w, 0.05), device=dev)
    bu.load(w.state, w.next_id)
    del w.state
    bu.register_ports()
    # a plain device copy of the state's size timed after every update: if it slows
    # down too, the drift is the hardware's (clocks, power), not the data's
    ca = torch.empty(bu.capacity * 9, dtype=torch.float32, device=dev)
    cb = torch.empty_like(ca)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for s in range(steps):
        sphbuf.sph_profile(bu.ctx, True)
        bu.step(w.dt, deferred=True)
        prof = sphbuf.sph_profile_read(bu.ctx)
        sphbuf.sph_profile(bu.ctx, False)
        st = bu.stats()
        ms = {k: round(v[0] / v[1], 4) for k, v in prof.items() if v[1] > 0}
        e0.record()
        cb.copy_(ca)
        e1.record()
        torch.cuda.synchronize()
        cms = e0.elapsed_time(e1)
        cnt = (bu.cell_end - bu.cell_start).to(torch.float64)
        occ = cnt[cnt > 0]
        # particle-weighted mean cell size (the ranking work per particle) and the
        # share of particles in cells larger than the gather's 64-slot halo
        pw = float((occ * occ).sum() / occ.sum())
        big = float(occ[occ > 64].sum() / occ.sum())
        print(f"update {s:3d} n {st['n']} created {st.get('created')} deleted {st.get('deleted')} "
              f"gather {ms.get('cll_gather')} scatter {ms.get('cll_scatter')} scan {ms.get('cell_scan')} "
              f"key {ms.get('cll_key')} copy {cms:.3f} | cells: max {int(occ.max())} particle-weighted mean {pw:.1f} "
              f"in cells > 64: {100 * big:.3f}%", flush=True)


if __name__ == "__main__":
    main()
