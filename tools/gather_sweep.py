#!/usr/bin/env python
"""Tuning sweep of the cell-list gather variants (SPHBUF_GATHER=<kind>:<slots>:<min blocks>, or any
NAME=value such as SPHBUF_GATHER_TMA=<tile>:<groups>:<stages>).

    python tools/gather_sweep.py [--config C5] [--steps 8] [variant ...]

Each variant runs in its own process (the library reads the variable once): the
config's workload, 3 warm-up updates, `steps` timed updates with per-kernel CUDA
events (sph_profile), then a checksum of the final state; every variant must
produce the same checksum as the default (the gather output is unique).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

VARIANTS = ["", "1:8", "2:6", "3:4", "4:3", "pf3:4"]


def child(config, steps):
    import torch
    from paper_2406_16786_b200 import inputs, sphbuf
    dev = torch.device("cuda", 0)
    w = inputs.make(config, device=dev)
    bu = sphbuf.BufferUpdater(w.grid, w.h, w.dp, w.ports, inputs.capacity_for(w, 0.05), device=dev)
    bu.load(w.state, w.next_id)
    del w.state
    bu.register_ports()
    for _ in range(3):
        bu.step(w.dt, deferred=True)
    torch.cuda.synchronize()
    sphbuf.sph_profile(bu.ctx, True)
    for _ in range(steps):
        bu.step(w.dt, deferred=True)
    torch.cuda.synchronize()
    prof = sphbuf.sph_profile_read(bu.ctx)
    n = bu.A.count()
    h = 0
    for c, t in list(bu.A.cols.items()) + [("id", bu.A.id), ("label", bu.A.label)]:
        v = t[:n].view(torch.int32) if t.dtype != torch.int64 else t[:n]
        h ^= int((v.to(torch.int64) * torch.arange(1, n + 1, device=dev, dtype=torch.int64)).sum().item())
    ms = {k: v[0] / v[1] for k, v in prof.items() if v[1] > 0}
    print(json.dumps({"ms": ms, "n": n, "hash": h}))


def main():
    args = sys.argv[1:]
    config, steps = "C5", 8
    if "--config" in args:
        i = args.index("--config")
        config = args[i + 1]
        del args[i:i + 2]
    if "--steps" in args:
        i = args.index("--steps")
        steps = int(args[i + 1])
        del args[i:i + 2]
    if args and args[0] == "--child":
        child(config, steps)
        return
    variants = args or VARIANTS
    res = {}
    for v in variants:
        # "NAME=value" sets that variable (e.g. SPHBUF_GATHER_TMA=512:2:4), else SPHBUF_GATHER
        env = dict(os.environ, **({v.split("=", 1)[0]: v.split("=", 1)[1]} if "=" in v else {"SPHBUF_GATHER": v}))
        r = subprocess.run([sys.executable, __file__, "--child", "--config", config, "--steps", str(steps)], env=env,
                           capture_output=True, text=True, timeout=600)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        if r.returncode != 0 or not line:
            print(f"{v or 'default':12s} FAILED rc={r.returncode} {r.stderr[-800:]}", flush=True)
            continue
        d = json.loads(line[-1])
        res[v] = d
        ms = d["ms"]
        cll = sum(ms.get(k, 0) for k in ("cll_key", "cell_scan", "cll_scatter", "cll_gather"))
        print(f"{v or 'default':12s} gather {ms.get('cll_gather', 0):.4f} ms  cll {cll:.4f} ms  n {d['n']}  "
              f"hash {d['hash']}  " + " ".join(f"{k} {1e3 * t:.1f}us" for k, t in sorted(ms.items())), flush=True)
    hs = {d["hash"] for d in res.values()}
    print("checksums agree" if len(hs) == 1 else f"CHECKSUM MISMATCH {hs}")


if __name__ == "__main__":
    main()
