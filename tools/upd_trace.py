#!/usr/bin/env python
"""Tile timeline of the update kernel K6 (libsphbuf_trace.so, -DSPHBUF_TRACE).

    SPHBUF_TRACE=1 python tools/upd_trace.py [config] [steps]

Per tile: start, run staging done, decisions + stores done (before the scan),
look-back done, end — relative to the first tile's start, in microseconds.
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
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    dev = torch.device("cuda", 0)
    w = inputs.make(config, device=dev)
    bu = sphbuf.BufferUpdater(w.grid, w.h, w.dp, w.ports, inputs.capacity_for(w, 0.05), device=dev)
    bu.load(w.state, w.next_id)
    del w.state
    bu.register_ports()
    L = sphbuf.lib()
    L.sph_trace_read.argtypes = [C.c_void_p, C.c_int]
    L.sph_trace_kernel.argtypes = [C.c_void_p, C.c_int]
    L.sph_trace_scan.argtypes = [C.c_void_p, C.c_int, C.c_int]
    kt = np.zeros(4, np.uint64)
    sc = np.zeros((1 << 12, 6), np.uint64)
    for s in range(steps):
        torch.cuda.synchronize()
        L.sph_trace_kernel(kt.ctypes.data, 1)
        L.sph_trace_scan(sc.ctypes.data, 1 << 12, 1)
        bu.step(w.dt, deferred=True)
    torch.cuda.synchronize()
    L.sph_trace_kernel(kt.ctypes.data, 0)
    L.sph_trace_scan(sc.ctypes.data, 1 << 12, 0)
    sc = sc[sc[:, 0] > 0].astype(np.int64)
    if len(sc):
        r = (sc[:, :4] - sc[:, 0].min()) / 1000.0
        d = np.diff(r, axis=1)
        print(f"K2 cell scan: {len(sc)} tiles, span {r[:, 3].max():.2f} us, last start {r[:, 0].max():.2f} us")
        for name, col in zip(["loads+scan", "look-back", "writes+done"], d.T):
            print(f"  {name:14s} mean {col.mean():7.2f} us  p50 {np.median(col):7.2f}  max {col.max():7.2f}")
        o = np.argsort(r[:, 0])
        for q in (0, len(o) // 4, len(o) // 2, 3 * len(o) // 4, len(o) - 1):
            i = o[q]
            print(f"  tile {i:5d} blk {sc[i, 4]:4d} sm {sc[i, 5]:3d}: " + " ".join(f"{v:7.2f}" for v in r[i]))
    ntile = 1 << 14
    buf = np.zeros((ntile, 7), np.uint64)
    assert L.sph_trace_read(buf.ctypes.data, ntile) == 0
    cand = int(bu.stats()["candidates"]) if "candidates" in bu.stats() else 0
    used = buf[:, 0] > 0
    t = buf[used].astype(np.int64)
    t0 = t[:, 0].min()
    rel = (t[:, :5] - t0) / 1000.0
    n = len(t)
    print(f"{config}: {n} tiles (last update; candidates counter {cand})")
    ph = np.diff(rel, axis=1)
    for name, col in zip(["stage runs", "decide+stores", "scan+lookback", "staging+tail"], ph.T):
        print(f"  {name:14s} mean {col.mean():7.2f} us  p50 {np.median(col):7.2f}  max {col.max():7.2f}")
    print(f"  span first start .. last end: {rel[:, 4].max():.2f} us; last start {rel[:, 0].max():.2f} us")
    k = (kt.astype(np.int64) - t0) / 1000.0
    print(f"  kernel: first block entry {k[0]:.2f}, last block entry {k[1]:.2f}, tail scan {k[2]:.2f} .. {k[3]:.2f} us")
    order = np.argsort(rel[:, 0])
    for q in (0, n // 4, n // 2, 3 * n // 4, n - 1):
        i = order[q]
        print(f"  tile {i:5d} blk {t[i, 5]:4d} sm {t[i, 6]:3d}: " + " ".join(f"{v:7.2f}" for v in rel[i]))


if __name__ == "__main__":
    main()
