#!/usr/bin/env python
"""Benchmark of the in/outlet buffer update (arXiv 2406.16786) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C5|C4|C3|C2]

A step is one update of the whole hot path on one
batch of synthetic particles: advect (driver, fused into the build) -> [migrate,
N>1: sph_migrate_cll_build] -> sph_cll_build -> sph_buffer_update -> [count
allgather, N>1: sph_allgather_counts] -> sph_compact.  Default workload:
C5 (BASELINE configs[4]): 128M particles per GPU in x-slabs, 8 ports per slab,
weak scaling; inputs (4.6 GB per GPU) are far larger than L2, so no flush is
needed between steps.  value = candidate particles checked per second summed
over ranks (the metric's "buffer-update particles checked/sec").

--gpus N without torchrun (WORLD_SIZE unset) re-launches itself under
torch.distributed.run with N ranks on 127.0.0.1.

Timing: the headline (value, ms_per_step) is K steps with the library's
per-kernel profiling OFF (programmatic dependent launch overlaps the kernels);
a second pass of min(K, 10) steps records CUDA events between the phases
(t_cll, t_comm, t_update, t_compact: median and p90) and around every kernel
(the per-kernel split and the roofline of the dominant kernel).

--impl reference times the CPU oracle (the "reference arm"; test
infrastructure, oracle/) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np
import torch
import torch.distributed as dist

from paper_2406_16786_b200 import inputs, sphbuf
from paper_2406_16786_b200.dist import SlabUpdater, broadcast_unique_id, expected_migrants

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0


def hbm_peak():
    try:
        with open(PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks

class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ workload

def make_workload(name, rank, world, device, scale=1.0):
    if name == "C5":
        return inputs.c5(device=device, slab=rank, nslabs=world, scale=scale)
    if world != 1:
        raise SystemExit(f"config {name} is single-GPU; use C5 for N>1")
    if name == "C4":
        return inputs.c4(device=device, scale=scale)
    if name == "C3":
        return inputs.c3(device=device, scale=scale)
    return inputs.make(name, device=device)


# algorithmic bytes per launch for the roofline of one kernel
def algorithmic_bytes(kernel, dim, n, ncells, cand, created, deleted, moved):
    S = 8 * dim + 12
    return {
        "advect": n * (2 * dim * 4 + dim * 4),
        "cll_key": n * (4 * dim + 4),
        "cell_scan": ncells * 12,
        "cll_scatter": n * 8,   # key read + slot -> source write
        # + 4 B: the next build's key, written by the gather (key carry-over)
        "cll_gather": n * (2 * S + 4),
        "cll_rank": n * (8 + 8),
        "compact_count": moved * 4,
        "upd_main": cand * (4 * dim + 4) + created * (2 * S + 4 * dim),
        "compact": moved * S + (moved - deleted) * S,
        "compact_append": created * S,
    }.get(kernel)


def _pct(xs, q):
    xs = sorted(xs)
    if not xs:
        return None
    k = min(len(xs) - 1, max(0, int(math.ceil(q * len(xs))) - 1))
    return xs[k]


class PhaseTimer:
    """CUDA events between the phases of one step on the launching stream, and
    NVTX ranges around them (the breakdown pass; the headline pass has none)."""

    def __init__(self):
        self.steps = []

    def step(self, su, dt, world):
        bu = su.bu
        s = torch.cuda.current_stream()
        ev = []

        def mark(name=None):
            e = torch.cuda.Event(enable_timing=True)
            e.record(s)
            ev.append((name, e))

        nv = torch.cuda.nvtx
        mark()
        if su.has_comm and world > 1:
            nv.range_push("cll_key+pack")
            sphbuf.sph_cll_key(bu.ctx, bu.A, dt)
            nv.range_pop()
            mark("cll")
            nv.range_push("comm: neighbour exchange")
            sphbuf.sph_migrate_exchange(bu.ctx)
            nv.range_pop()
            mark("comm")
            nv.range_push("cll_finish")
            sphbuf.sph_cll_finish(bu.ctx, bu.A, bu.B, bu.cell_start, bu.cell_end)
            bu.A, bu.B = bu.B, bu.A
            nv.range_pop()
            mark("cll")
            nv.range_push("buffer_update")
            bu.update()
            nv.range_pop()
            mark("update")
            nv.range_push("comm: count allgather")
            sphbuf.sph_allgather_counts(bu.ctx, bu.port_counts, su.all_counts)
            nv.range_pop()
            mark("comm")
            nv.range_push("compact")
            bu.compact(su.all_counts, world, su.rank, deferred=su.deferred)
            nv.range_pop()
            mark("compact")
        else:
            nv.range_push("cll_build (advection fused)")
            bu.cll_build(dt=dt)
            nv.range_pop()
            mark("cll")
            nv.range_push("buffer_update")
            bu.update()
            nv.range_pop()
            mark("update")
            nv.range_push("compact")
            bu.compact(deferred=su.deferred)
            nv.range_pop()
            mark("compact")
        self.steps.append(ev)

    def summary(self):
        """{phase: {median, p90}} in ms over the steps (synchronises)."""
        torch.cuda.synchronize()
        per = {"cll": [], "comm": [], "update": [], "compact": [], "step": []}
        for ev in self.steps:
            acc = dict.fromkeys(per, 0.0)
            for (_, a), (name, b) in zip(ev[:-1], ev[1:]):
                acc[name] += a.elapsed_time(b)
            acc["step"] = ev[0][1].elapsed_time(ev[-1][1])
            for k in per:
                per[k].append(acc[k])
        return {f"t_{k}": {"median_ms": round(statistics.median(v), 5), "p90_ms": round(_pct(v, 0.9), 5)}
                for k, v in per.items() if v}


def run_ours(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    uid = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        uid = broadcast_unique_id(rank)          # the library creates and owns its ncclComm_t
    tgen = time.time()
    w = make_workload(args.config, rank, world, dev, args.scale)
    torch.cuda.synchronize()
    tgen = time.time() - tgen
    cap = inputs.capacity_for(w, 0.05)
    max_new = max(65536, w.n // 200)
    max_mig = 0
    if world > 1:
        # fixed-size messages (no host sync): 3x the expected steady-state migrants per
        # face and step on the busiest rank, at least 4096
        est = torch.tensor([float(expected_migrants(w.state, w.grid, w.dt, w.dp))], device=dev)
        dist.all_reduce(est, op=dist.ReduceOp.MAX)
        max_mig = max(4096, int(3 * float(est.item())))
    su = SlabUpdater(w, rank, world, cap, max_migrate=max_mig, max_new=max_new, device=dev,
                     deferred=(args.compaction == "deferred"))
    if world > 1:
        su.init_nccl(uid)
    su.load(w.state, w.next_id)
    n0 = w.n
    del w.state
    torch.cuda.empty_cache()
    bu = su.bu
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def reduce(ms, count):
        t = torch.tensor([ms, float(count)], dtype=torch.float64, device=dev)
        if world > 1:
            tmax = t.clone()
            dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
            tsum = t.clone()
            dist.all_reduce(tsum[1:], op=dist.ReduceOp.SUM)
            return float(tmax[0]), float(tsum[1])
        return ms, float(count)

    def headline(steps, sample_clocks):
        """Exactly `steps` steps between barrier + synchronize on both sides, CUDA
        events on the launching stream, max over ranks; no per-kernel events."""
        s0 = bu.stats()
        l0 = bu.launches()
        clocks = ClockSampler(local) if sample_clocks else None
        if clocks:
            clocks.start()
            time.sleep(0.3)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            su.step(w.dt)
        e1.record(stream)
        barrier()
        clk = clocks.stop() if clocks else None
        ms = e0.elapsed_time(e1)
        s1 = bu.stats()
        checked = s1["checked_total"] - s0["checked_total"]
        ms_max, checked_all = reduce(ms, checked)
        return ms_max, checked_all, checked, bu.launches() - l0, clk, s1

    def breakdown(steps):
        """Phase events + per-kernel events (sph_profile) over `steps` steps."""
        pt = PhaseTimer()
        sphbuf.sph_profile(bu.ctx, True)
        barrier()
        for _ in range(steps):
            pt.step(su, w.dt, world)
        barrier()
        prof = sphbuf.sph_profile_read(bu.ctx)
        sphbuf.sph_profile(bu.ctx, False)
        return pt.summary(), {k: v for k, v in prof.items() if v[1] > 0}, bu.stats()

    modes = [args.compaction, "inplace" if args.compaction == "deferred" else "deferred"]
    res = {}
    for mi, mode in enumerate(modes):
        su.deferred = mode == "deferred"
        for _ in range(args.warmup if mi == 0 else 3):
            su.step(w.dt)
        ms_max, checked_all, checked, launches, clk, s = headline(args.steps, mi == 0)
        phases, prof, sb = breakdown(min(args.steps, 10))
        res[mode] = dict(ms=ms_max, checked_all=checked_all, checked=checked, launches=launches, clk=clk, s=s,
                         phases=phases, prof=prof, sb=sb)
    su.deferred = modes[0] == "deferred"
    for _ in range(2):
        su.step(w.dt)

    dim = bu.dim
    S = 8 * dim + 12
    ncells = w.grid.ncells_local
    peak, peak_src = hbm_peak()

    def mode_report(mode):
        r = res[mode]
        s, prof = r["sb"], r["prof"]
        n = s["n"]
        cand = r["checked"] / max(1, args.steps)
        created, deleted = s["created"], s["deleted"]
        moved = max(0, n + deleted - created - s["first_deleted"]) if deleted else 0
        kms = {k: v[0] / v[1] for k, v in prof.items()}
        t_upd = kms.get("upd_prologue", 0) + kms.get("upd_main", 0)
        t_cmp = kms.get("compact_count", 0) + kms.get("compact", 0) + kms.get("compact_append", 0)
        t_cll = sum(kms.get(k, 0) for k in ("cll_key", "cell_scan", "cll_scatter", "cll_gather", "advect",
                                            "mig_pack", "mig_unpack"))
        b_upd = cand * (4 * dim + 4) + created * (2 * S + 4 * dim)
        b_cmp = (2 * S * moved - S * deleted + S * created) if mode == "inplace" else S * created
        b_cll = n * (2 * S + 32)
        frac = lambda b, t: b / (t / 1e3) / 1e9 / peak if t else None
        return {
            "ms_per_step": r["ms"] / args.steps, "value": r["checked_all"] / (r["ms"] / 1e3),
            "phases": r["phases"],
            "update_compact": {"alg_bytes": b_upd + b_cmp, "kernel_ms": t_upd + t_cmp,
                               "frac": frac(b_upd + b_cmp, t_upd + t_cmp),
                               "what": "SURVEY 8(d) headline: (B_update + B_compact) / (t_update + t_compact); "
                                       "kernel times from the breakdown pass"},
            # the in-place move also carries each moved particle's next-build key (4 B
            # read + 4 B written), the price of the key pass the next build skips
            "compact_move_with_keys": ({"bytes": 2 * (S + 4) * moved, "kernel_ms": kms.get("compact", 0),
                                        "frac": frac(2 * (S + 4) * moved, kms.get("compact", 0))}
                                       if mode == "inplace" and kms.get("compact") else None),
            "cll_build": {"alg_bytes": b_cll, "kernel_ms": t_cll, "frac": frac(b_cll, t_cll),
                          "what": "2S + 32 B per particle (SURVEY 8(d))"},
            "kernels_ms": {k: round(v, 4) for k, v in kms.items()},
            "cand": cand, "created": created, "deleted": deleted, "moved": moved, "n": n,
        }

    rep = {m: mode_report(m) for m in modes}
    main_r = res[modes[0]]
    R = rep[modes[0]]
    value = R["value"]
    step_ms = R["ms_per_step"]
    prof = main_r["prof"]
    dom = max(prof, key=lambda k: prof[k][0])
    dom_ms = prof[dom][0] / prof[dom][1]
    bytes_dom = algorithmic_bytes(dom, dim, R["n"], ncells, R["cand"], R["created"], R["deleted"], R["moved"])
    achieved = bytes_dom / (dom_ms / 1e3) / 1e9 if bytes_dom else None
    traffic, ncu_k = None, None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            tj = json.load(open(tf))
            traffic = tj.get(args.config, {}).get(dom)
            # the ncu counters the north star names (DRAM rate, L2 hit rate, warp
            # efficiency of the ballot / scan code) for the dominant kernel and K6
            ncu_k = {k: v for k, v in tj.get(args.config + "_ncu", {}).items() if k in (dom, "upd_main")} or None
        except Exception:
            traffic, ncu_k = None, None
    tot = sum(v[0] for v in prof.values())
    kernels = {k: {"ms_per_launch": round(v[0] / v[1], 4), "share": round(v[0] / tot, 4)} for k, v in prof.items()}

    # e2e: same metric through the public API with host-resident particles
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(su, w, args, dev, world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args, dev)
    n_ports = len(su.bu.ports)
    sweep = None
    if rank == 0 and world == 1 and not args.no_sweep:
        del su, bu
        torch.cuda.empty_cache()
        sweep = sweep_configs(dev)
    if rank == 0:
        line = {
            "metric": "buffer-update particles checked/sec & us/step; % of B200 HBM peak; 1/2/4/8 GPU",
            "value": value, "unit": "particles_checked/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "us_per_step": step_ms * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded lattice + jitter, tie-screened, BASELINE config shapes)",
            "config": {"workload": f"{args.config}" + (f" scale {args.scale}" if args.scale != 1 else ""),
                       "particles_per_gpu": n0, "ports": n_ports, "candidates_per_step": R["cand"],
                       "created_last": R["created"], "deleted_last": R["deleted"], "dim": dim,
                       "parallelism": f"x-slab dp{world}", "l2": "inputs (>=4.6 GB/GPU) larger than L2; no flush",
                       "compaction": modes[0], "max_migrate": max_mig,
                       "advection": "fused into the cell-list build (the gather advects; next keys carried over)",
                       "timing": "headline with per-kernel profiling off; phases/kernels from a second pass",
                       "timed_updates": f"{args.warmup + 1}..{args.warmup + args.steps} of the run",
                       "gen_s": round(tgen, 1)},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None, "traffic": traffic,
                         "peak_source": peak_src, "alg_bytes_per_launch": bytes_dom, "ms_per_launch": dom_ms,
                         "update_compact_8d": {m: {"frac": rep[m]["update_compact"]["frac"],
                                                   "alg_bytes": rep[m]["update_compact"]["alg_bytes"],
                                                   "kernel_ms": rep[m]["update_compact"]["kernel_ms"]}
                                               for m in modes},
                         "cll_build_8d": {m: rep[m]["cll_build"]["frac"] for m in modes},
                         "frac_of_spec_8tbs": achieved / 8000.0 if achieved else None,
                         "ncu": ncu_k,
                         "inplace_move_with_keys": rep["inplace"]["compact_move_with_keys"] if "inplace" in rep else None,
                         "note": "the gather is at the floor of its access pattern: the same loads and stores through "
                                 "the real C5 slot map with no arithmetic take 2.66-2.69 ms (tools/gather_tma_probe.cu, "
                                 "DESIGN.md section 6)"},
            "kernels": kernels,
            "phases": {m: rep[m]["phases"] for m in modes},
            "modes": {m: {k: rep[m][k] for k in ("ms_per_step", "value", "update_compact", "cll_build",
                                                  "compact_move_with_keys", "kernels_ms")} for m in modes},
            "gpu_launches": main_r["launches"],
            "clocks": main_r["clk"],
            "e2e": e2e,
            "cpu_baseline": cpu,
            "configs_us_per_update": sweep,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(su, w, args, dev, world):
    """The same metric end to end: every step uploads the rank's particle state from
    pinned host memory (H2D), runs the update through the public API, and reads
    the updated state back (D2H) — a host-resident simulation loop.  The read-back
    of one step and the upload of the next are pipelined per column quarter on two copy
    streams (the two PCIe directions run concurrently): column c goes up again as
    soon as it has come down, and the next step starts once every column is up."""
    bu = su.bu
    n = bu.A.count()
    names = [c for c, _ in bu.A.cols.items()] + ["id", "label"]

    def col(name):
        return bu.A.cols[name] if name in bu.A.cols else getattr(bu.A, name)

    host = {c: torch.empty(bu.capacity, dtype=col(c).dtype, pin_memory=True) for c in names}
    for c in names:
        host[c][:n].copy_(col(c)[:n])
    steps = max(2, min(args.steps, args.e2e_steps))
    stream = torch.cuda.current_stream()
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    chunks = int(os.environ.get("SPH_E2E_CHUNKS", "4"))    # per column: a short pipeline tail
    evs = {(c, k): torch.cuda.Event() for c in names for k in range(chunks)}
    checked0 = bu.stats()["checked_total"]
    h2d = d2h = 0
    per = sum(col(c).element_size() for c in names)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    up.wait_stream(stream)
    with torch.cuda.stream(up):                      # first step's inputs
        for c in names:
            col(c)[:n].copy_(host[c][:n], non_blocking=True)
    h2d += n * per
    for s in range(steps):
        stream.wait_stream(up)
        bu.A.n.fill_(n)
        sphbuf.sph_cll_invalidate(bu.ctx)   # uploaded state: no carried-over keys (ABI contract)
        su.step(w.dt)
        n = int(bu.A.n.item())
        down.wait_stream(stream)
        last = s == steps - 1
        m = (n + chunks - 1) // chunks
        for c in names:
            for k in range(chunks):
                a, b = k * m, min(n, (k + 1) * m)
                if a >= b:
                    continue
                with torch.cuda.stream(down):        # this step's result
                    host[c][a:b].copy_(col(c)[a:b], non_blocking=True)
                    evs[c, k].record(down)
                if not last:
                    with torch.cuda.stream(up):      # the next step's input, chunk by chunk
                        up.wait_event(evs[c, k])
                        col(c)[a:b].copy_(host[c][a:b], non_blocking=True)
        d2h += n * per + 8
        if not last:
            h2d += n * per
    stream.wait_stream(down)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    checked = bu.stats()["checked_total"] - checked0
    t = torch.tensor([ms, float(checked)], dtype=torch.float64, device=dev)
    if world > 1:
        a = t.clone()
        dist.all_reduce(a[:1], op=dist.ReduceOp.MAX)
        b = t.clone()
        dist.all_reduce(b[1:], op=dist.ReduceOp.SUM)
        ms, checked = float(a[0]), float(b[1])
    return {"value": checked / (ms / 1e3), "unit": "particles_checked/s", "ms_per_step": ms / steps,
            "steps": steps, "h2d_bytes_per_step": h2d // steps, "d2h_bytes_per_step": d2h // steps,
            "what": "pinned host state -> device, update via BufferUpdater/SlabUpdater, state -> pinned host; "
                    "read-back and next upload pipelined per column quarter on two copy streams"}


# ------------------------------------------------------------------ CPU oracle (reference arm / cpu_baseline)

def sweep_configs(dev, names=("C1", "C1e", "C2", "C3", "C4"), replays=50):
    """µs per buffer update of each BASELINE config on one GPU (the
    small configs are latency-bound, so they replay a CUDA graph of two captured
    updates; the stream-launched time is reported beside it)."""
    out = {}
    for name in names:
        w = make_workload(name, 0, 1, dev)
        bu = sphbuf.BufferUpdater(w.grid, w.h, w.dp, w.ports, inputs.capacity_for(w, 0.3), device=dev)
        bu.load(w.state, w.next_id)
        bu.register_ports()
        n0 = w.n
        del w
        stream = torch.cuda.current_stream()
        g = bu.capture(dt_of(name))
        for _ in range(3):
            g.replay()
        c0 = bu.stats()["checked_total"]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(replays):
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        us_graph = e0.elapsed_time(e1) * 1e3 / (2 * replays)
        cand = (bu.stats()["checked_total"] - c0) / (2 * replays)
        e0.record(stream)
        for _ in range(replays):
            bu.step(dt_of(name), deferred=True)
        e1.record(stream)
        torch.cuda.synchronize()
        us_stream = e0.elapsed_time(e1) * 1e3 / replays
        # per-kernel split from a separate profiled pass (an event pair per kernel)
        sphbuf.sph_profile(bu.ctx, True)
        for _ in range(10):
            bu.step(dt_of(name), deferred=True)
        prof = sphbuf.sph_profile_read(bu.ctx)
        sphbuf.sph_profile(bu.ctx, False)
        kern = {k: round(ms * 1e3 / cnt, 2) for k, (ms, cnt) in prof.items() if cnt}
        out[name] = {"particles": n0, "us_per_update_graph": round(us_graph, 2),
                     "us_per_update_stream": round(us_stream, 2), "candidates_per_update": round(cand, 1),
                     "particles_checked_per_s": cand / (us_graph * 1e-6) if us_graph else None,
                     "kernels_us_profiled": kern}
        del bu, g
        torch.cuda.empty_cache()
    return out


def dt_of(name):
    return {"C1": 0.002, "C1e": 0.0095, "C2": 0.0005, "C3": 0.0002, "C4": 0.0005, "C5": 0.0005}[name]


def oracle_sample(args, dev):
    """Bounded sample of the workload for the oracle: the same config at 1/8 of the
    volume (scale 0.5: same dp, cell size, port shapes scaled)."""
    import oracle
    sc = args.cpu_scale
    w = make_workload(args.config, 0, 1, dev, sc * args.scale) if args.config in ("C3", "C4", "C5") else \
        make_workload(args.config, 0, 1, dev)
    st = oracle.to_numpy_state(w.state)
    for k, p in enumerate(w.ports):
        oracle.register(st, w.grid, p, k)
    return w, st


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_step_timed(w, st, nid, mode, threads):
    """One oracle update (O2-O6: cell list, decisions, apply, relabel, compaction),
    wall-clock timed; mode 1 = cell-restricted (the paper's local cell-linked lists,
    the CPU form of the method), 0 = brute force over every particle and port.
    Returns (state, next_id, seconds, candidates, t_cll, t_decide); candidates =
    particles in the cells intersecting each P_k (the metric's unit of work)."""
    import oracle
    oracle.set_threads(threads)
    oracle.advect(st, w.dim, w.dt)
    t0 = time.perf_counter()
    res = oracle.update(w.grid, w.ports, st, mode=mode)
    new, perm, nid = oracle.compact(res, w.dim, len(w.ports), res.port_counts[None, :], 0, nid)
    dt = time.perf_counter() - t0
    if mode == 1:
        cand = res.checked
    else:
        cand = 0
        for p in w.ports:
            m = oracle.port_cells(w.grid, p).astype(bool)
            cand += int((res.cell_end - res.cell_start)[m].sum())
    return new, nid, dt, cand, res.t_cll, res.t_decide


def cpu_baseline(args, dev):
    """The oracle as it stands, on this host's cores, on a bounded sample: cell-
    restricted with every core (the headline value), cell-restricted on one core,
    and brute force with every core."""
    import oracle
    w, st = oracle_sample(args, dev)
    T = os.cpu_count() or 1
    runs = []
    for mode, threads in ((1, T), (1, 1), (0, T)):
        s2 = {k: (v.copy() if not isinstance(v, list) else [c.copy() for c in v]) for k, v in st.items()}
        _, _, dt, cand, tc, td = oracle_step_timed(w, s2, w.next_id, mode, threads)
        runs.append({"mode": "cell-restricted" if mode == 1 else "brute force", "threads": threads,
                     "s_per_update": round(dt, 3), "s_cell_list": round(tc, 3), "s_decide_apply": round(td, 3),
                     "value": cand / dt, "candidates": cand})
    oracle.set_threads(T)
    head = runs[0]
    return {"value": head["value"], "unit": "particles_checked/s", "cores": T, "kind": "oracle",
            "cpu_model": cpu_model(), "mode": head["mode"],
            "sample": f"one oracle update (O2-O6: cell list, f64 decisions, apply, relabel, compaction) of "
                      f"{args.config} at scale {args.cpu_scale * args.scale} ({w.n} particles, {len(w.ports)} ports); "
                      f"OpenMP on the independent per-particle loops only",
            "runs": runs}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    w, st = oracle_sample(args, dev)
    T = os.cpu_count() or 1
    nid = w.next_id
    for _ in range(args.warmup):
        st, nid, _, _, _, _ = oracle_step_timed(w, st, nid, 1, T)
    tot, cand = 0.0, 0
    for _ in range(args.steps):
        st, nid, dt, c, _, _ = oracle_step_timed(w, st, nid, 1, T)
        tot += dt
        cand += c
    v = cand / tot
    line = {"impl": "reference", "metric": "buffer-update particles checked/sec & us/step; % of B200 HBM peak; "
            "1/2/4/8 GPU", "value": v, "unit": "particles_checked/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64 decisions, f32 state", "data": "synthetic",
            "config": {"workload": f"{args.config} sample at scale {args.cpu_scale * args.scale}",
                       "particles": w.n, "ports": len(w.ports)},
            "cpu_baseline": {"value": v, "unit": "particles_checked/s", "cores": T, "kind": "oracle",
                             "cpu_model": cpu_model(), "mode": "cell-restricted",
                             "sample": f"{args.steps} oracle updates (O2-O6) of {args.config} at scale "
                                       f"{args.cpu_scale * args.scale} ({w.n} particles)"},
            "e2e": {"value": v, "unit": "particles_checked/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def spawn(args) -> int:
    """--gpus N without torchrun: re-launch this script under torch.distributed.run
    (one rank per GPU, rendezvous on 127.0.0.1) and return its exit code."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def spawn_check(args):
    """(CPU) the rank layout a spawned run sees: one JSON line per rank."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist.init_process_group("gloo")
    t = torch.tensor([rank + 1])
    dist.all_reduce(t)
    line = json.dumps({"rank": rank, "world": world, "local_rank": int(os.environ.get("LOCAL_RANK", "0")),
                       "sum_ranks_plus_1": int(t.item())}) + "\n"
    for r in range(world):              # one rank at a time: the ranks share one stdout pipe
        if r == rank:
            sys.stdout.write(line)
            sys.stdout.flush()
        dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # default: 3 warm-up + 47 timed updates = the 50 updates BASELINE's C5 run is quoted
    # on (the build slows ~10% over the first ~30 updates as the initial lattice
    # smears out and cell changers stop arriving in coherent rows)
    ap.add_argument("--steps", type=int, default=47)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--cpu-scale", type=float, default=0.5)
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the per-config us/update sweep (C1-C4)")
    ap.add_argument("--compaction", default="deferred", choices=["inplace", "deferred"],
                    help="sph_compact (in-place stable compaction each update) or sph_compact_deferred "
                         "(removal fused into the next cell-list build)")
    ap.add_argument("--spawn-check", action="store_true", help="(CPU test) print each spawned rank's layout")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    if args.spawn_check:
        spawn_check(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
