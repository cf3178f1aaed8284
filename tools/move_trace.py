#!/usr/bin/env python
"""Sub-tile timeline of the in-place compaction move K7b (libsphbuf_trace.so).

    SPHBUF_TRACE=1 python tools/move_trace.py [config] [steps]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2406_16786_b200 import inputs, sphbuf


def main():
    assert os.environ.get("SPHBUF_TRACE") == "1", "run with SPHBUF_TRACE=1"
    config = sys.argv[1] if len(sys.argv) > 1 else "C5"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    dev = torch.device("cuda", 0)
    w = inputs.make(config, device=dev)
    bu = sphbuf.BufferUpdater(w.grid, w.h, w.dp, w.ports, inputs.capacity_for(w, 0.05), device=dev)
    bu.load(w.state, w.next_id)
    del w.state
    bu.register_ports()
    L = sphbuf.lib()
    L.sph_trace_move.argtypes = [C.c_void_p, C.c_int, C.c_int]
    nt = 1 << 17
    buf = np.zeros((nt, 6), np.uint64)
    for s in range(steps):
        torch.cuda.synchronize()
        L.sph_trace_move(buf.ctypes.data, nt, 1)
        bu.step(w.dt, deferred=False)
    torch.cuda.synchronize()
    L.sph_trace_move(buf.ctypes.data, nt, 0)
    t = buf[buf[:, 0] > 0].astype(np.int64)
    r = (t[:, :4] - t[:, 0].min()) / 1000.0
    d = np.diff(r, axis=1)
    print(f"K7b: {len(t)} sub-tiles, span {r[:, 3].max():.1f} us, last start {r[:, 0].max():.1f} us, "
          f"blocks {len(np.unique(t[:, 4]))}")
    # K7b two in flight: [0] loads issued, [1] loads returned + ranked + "read done",
    # [2] predecessors waited for (the block's next sub-tile loading meanwhile), [3] stored
    for name, col in zip(["loads+rank", "until stores may start", "stores"], d.T):
        print(f"  {name:12s} mean {col.mean():7.2f} us  p50 {np.median(col):7.2f}  p99 {np.percentile(col, 99):7.2f}")
    tot = r[:, 3] - r[:, 0]
    print(f"  per sub-tile mean {tot.mean():.2f} us; sub-tiles per block {len(t) / len(np.unique(t[:, 4])):.1f}")
    # gaps between a block's consecutive sub-tiles (ticket + loop overhead)
    gaps = []
    for b in np.unique(t[:, 4])[:200]:
        rb = np.sort(r[t[:, 4] == b][:, 0])
        eb = np.sort(r[t[:, 4] == b][:, 3])
        if len(rb) > 1:
            gaps.extend(rb[1:] - eb[:-1])
    if gaps:
        print(f"  gap end -> next start mean {np.mean(gaps):.2f} us")


if __name__ == "__main__":
    main()
