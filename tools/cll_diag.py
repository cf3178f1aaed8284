#!/usr/bin/env python
"""Per-kernel times and mover counts of the cell-list build over a few updates.

    python tools/cll_diag.py [config] [steps]
"""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2406_16786_b200 import inputs, sphbuf


def main():
    config = sys.argv[1] if len(sys.argv) > 1 else "C5"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    dev = torch.device("cuda", 0)
    w = inputs.make(config, device=dev)
    bu = sphbuf.BufferUpdater(w.grid, w.h, w.dp, w.ports, inputs.capacity_for(w, 0.05), device=dev)
    bu.load(w.state, w.next_id)
    del w.state
    bu.register_ports()
    for s in range(steps):
        sphbuf.sph_profile(bu.ctx, True)
        bu.step(w.dt, deferred=True)
        prof = sphbuf.sph_profile_read(bu.ctx)
        sphbuf.sph_profile(bu.ctx, False)
        st = bu.stats()
        ms = {k: round(v[0] / v[1], 4) for k, v in prof.items() if v[1] > 0}
        print(f"step {s}: n {st['n']} {ms}",
              flush=True)


if __name__ == "__main__":
    main()
