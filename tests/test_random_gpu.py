"""Randomised lock-step parity: seeded random workloads that mix what the fixed
configurations keep apart — 2-D and 3-D, 1-5 ports of every kind at random
orientations and sizes, pressure / velocity boundary conditions (with a density
column), bidirectional flow, random dt, and every build / compaction mode (key
pass or carried keys, deferred or in-place compaction).  Each is compared with
the oracle bit-exactly after every update (tests/parity_util.py::lockstep).
"""
import math

import numpy as np
import pytest
import torch

from paper_2406_16786_b200 import inputs
from paper_2406_16786_b200.inputs import (BC, BC_PRESSURE, BC_VELOCITY, BIDIRECTIONAL, INLET, OUTLET,
                                          PROFILE_PARABOLIC, PROFILE_PARABOLIC_RADIAL, PROFILE_PLUG, Grid, Port,
                                          Workload, f32, frame_rows_2d, frame_rows_3d)

from parity_util import lockstep


SEEDS = range(24)


def _raw_random_workload(seed):
    rng = np.random.default_rng(1000 + seed)
    dim = 2 if rng.random() < 0.35 else 3
    dp = float(rng.uniform(0.008, 0.012)) if dim == 3 else float(rng.uniform(0.002, 0.005))
    h = 1.3 * dp
    cs = f32(2 * h * float(rng.uniform(1.0, 1.3)))
    L = float(rng.uniform(0.32, 0.42)) if dim == 3 else float(rng.uniform(0.3, 0.5))
    counts = tuple(int(L / dp) for _ in range(dim))
    n = int(np.prod(counts))
    dt = float(rng.uniform(0.0002, 0.0008))
    # ports: rejection-sampled bounding spheres (+1 cell), 2 cells apart, inside the fluid box
    ports, placed = [], []
    nports = int(rng.integers(1, 6))
    while len(ports) < nports:
        kind = [INLET, OUTLET, BIDIRECTIONAL][int(rng.integers(0, 3))]
        layers = int(rng.integers(3, 6))
        for _ in range(2000):
            if dim == 3:
                u = rng.standard_normal(3)
                Q = frame_rows_3d(u / np.linalg.norm(u), float(rng.uniform(0, 2 * math.pi)))
                b, c = rng.uniform(0.02, 0.05, size=2) * L / 0.3
                he = (layers * dp / 2, b / 2, c / 2)
            else:
                Q = frame_rows_2d(float(rng.uniform(0, 2 * math.pi)))
                he = (layers * dp / 2, float(rng.uniform(0.03, 0.1)) * L / 0.4, 0.0)
            r = math.sqrt(sum(x * x for x in he[:dim])) + cs
            lo, hi = r, L - r
            if hi <= lo:
                continue
            o = rng.uniform(lo, hi, size=dim)
            if all(np.linalg.norm(o - q) > r + rq + 2 * cs for q, rq in placed):
                bc = None
                roll = rng.random()
                if roll < 0.25:
                    bc = BC(BC_PRESSURE, rho0=1.0, c0=float(rng.uniform(5, 20)), p_b=float(rng.uniform(-1, 1)),
                            rho_column=0)
                elif roll < 0.5:
                    prof = [PROFILE_PLUG, PROFILE_PARABOLIC, PROFILE_PARABOLIC_RADIAL][int(rng.integers(0, 3))]
                    bc = BC(BC_VELOCITY, profile=prof, u0=float(rng.uniform(0.5, 1.5)), radius=float(2 * he[1]))
                oo = tuple(float(x) for x in o) + ((0.0,) if dim == 2 else ())
                ports.append(Port(tuple(f32(x) for x in oo), Q, tuple(f32(x) for x in he), kind, layers, bc))
                placed.append((o, r))
                break
        else:
            if ports:
                break    # lattice + jitter; velocity along the nearest port's axis (random sign at
    # bidirectional ports), noise, axial near the ports
    g = torch.Generator().manual_seed(2000 + seed)
    idx = torch.arange(n, dtype=torch.int64)
    xyz, rem = [], idx
    for a in range(dim):
        stride = int(np.prod(counts[a + 1:])) if a < dim - 1 else 1
        xyz.append(((rem // stride) % counts[a]).double() * dp + 0.5 * dp
                   + (torch.rand(n, generator=g, dtype=torch.float64) * 2 - 1) * 0.1 * dp)
    best = torch.full((n,), float("inf"), dtype=torch.float64)
    v = [torch.zeros(n, dtype=torch.float64) for _ in range(dim)]
    for p in ports:
        sgn = -1.0 if (p.kind == BIDIRECTIONAL and rng.random() < 0.5) else 1.0
        d2 = sum((xyz[j] - p.origin[j]) ** 2 for j in range(dim))
        sel = d2 < best
        best = torch.where(sel, d2, best)
        for j in range(dim):
            v[j] = torch.where(sel, torch.full_like(v[j], sgn * p.Q[j]), v[j])
    v = [v[j] + (torch.randn(n, generator=g, dtype=torch.float64) * 0.05).clamp(-0.2, 0.2) for j in range(dim)]
    v = inputs._project_near_ports(xyz, v, ports, dim, 2 * dp)
    st = inputs._pack_state(xyz, v, idx, dim)
    st["extra"] = [torch.full((n,), 1.0, dtype=torch.float32)]
    pad = 4
    lo = tuple(f32(-pad * cs) for _ in range(dim)) + ((0.0,) if dim == 2 else ())
    ncell = tuple(int(math.ceil(L / cs)) + 2 * pad for _ in range(dim)) + ((1,) if dim == 2 else ())
    grid = Grid(dim, lo, cs, ncell)
    w = Workload(f"R{seed}", dim, dp, h, grid, ports, st, f32(dt), 8, n)
    mode = dict(fused=bool(rng.random() < 0.7), deferred=bool(rng.random() < 0.5))
    return w, int(rng.integers(4, 9)), mode


_SCREENED = {}


def random_workload(seed, moving=False):
    """The seed's random workload, tie-screened on its own dynamics (boundary-
    condition velocities; with ``moving``, every port turning after each update)
    over its steps (tests/tiescreen.py)."""
    import oracle
    from tiescreen import screen
    key = (seed, moving)
    if key not in _SCREENED:
        w0, steps, mode = _raw_random_workload(seed)
        mot = random_motion(w0, seed) if moving else None

        def dry_run(w, lin):
            K = len(w.ports)
            st = oracle.to_numpy_state(w.state)
            for k, p in enumerate(w.ports):
                oracle.register(st, w.grid, p, k)
            ports = list(w.ports)
            nid = w.next_id
            for step in range(steps):
                oracle.advect(st, w.dim, w.dt)
                res = oracle.update(w.grid, ports, st)
                new, perm, nid = oracle.compact(res, w.dim, K, res.port_counts[None, :], 0, nid)
                lin.record(res, new)
                if moving:
                    for k in range(K):
                        o, Q = _pose(w, k, mot, step)
                        nxt = Port(o, Q, ports[k].half_extents, ports[k].kind, ports[k].layers, ports[k].bc)
                        oracle.port_move(new, w.dim, ports[k], nxt, k)
                        ports[k] = nxt
                st = new
        got = {}

        def make(nd):
            got.clear()
            got.update(nd)
            return inputs.nudge(_raw_random_workload(seed)[0], nd)
        screen(make, dry_run)
        _SCREENED[key] = dict(got)
    w, steps, mode = _raw_random_workload(seed)
    return inputs.nudge(w, _SCREENED[key]), steps, mode


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
def test_random_workload_lockstep(seed):
    w, steps, mode = random_workload(seed)
    tot, bu = lockstep(w, steps, check_every=1, state=w.state, **mode)
    assert bu.stats()["motion_errors"] == 0


def test_random_workloads_are_valid_inputs():
    """(CPU) every seed is deterministic, registers members in every port and runs
    its updates on the oracle with no particle claimed by two ports; over all seeds
    particles are both created and deleted, in 2-D and 3-D."""
    import oracle
    made = {2: [0, 0], 3: [0, 0]}
    for seed in SEEDS:
        w, steps, mode = random_workload(seed)
        w2, _, _ = random_workload(seed)
        assert torch.equal(w.state["x"], w2.state["x"]) and len(w.ports) == len(w2.ports) >= 1
        st = oracle.to_numpy_state(w.state)
        K = len(w.ports)
        assert all(oracle.register(st, w.grid, p, k) > 0 for k, p in enumerate(w.ports)), seed
        nid = w.next_id
        for _ in range(steps):
            oracle.advect(st, w.dim, w.dt)
            res = oracle.update(w.grid, w.ports, st)
            assert res.multi_decision == 0, seed
            st, perm, nid = oracle.compact(res, w.dim, K, res.port_counts[None, :], 0, nid)
            made[w.dim][0] += int(res.port_counts[:K].sum())
            made[w.dim][1] += int(res.port_counts[K:].sum())
    assert min(made[2] + made[3]) > 0, made


def random_motion(w, seed):
    """Per port: a pivot within a third of a cell of its origin, a rotation axis
    (3-D) and a turn per update of 0.5-3 degrees either way — the bounding sphere
    moves by less than the 2-cell gap over the run, so ports stay disjoint."""
    rng = np.random.default_rng(3000 + seed)
    cs = w.grid.cs
    mot = []
    for p in w.ports:
        off = rng.standard_normal(w.dim)
        off = off / np.linalg.norm(off) * cs / 3
        pivot = tuple(float(p.origin[j] + off[j]) for j in range(w.dim)) + ((0.0,) if w.dim == 2 else ())
        axis = rng.standard_normal(3)
        dth = math.radians(float(rng.uniform(0.5, 3.0))) * (1 if rng.random() < 0.5 else -1)
        mot.append((pivot, axis, dth))
    return mot


def _pose(w, k, mot, step):
    pivot, axis, dth = mot[k]
    if w.dim == 2:
        return inputs.sprinkler_pose(w.ports[k], pivot, dth * (step + 1))
    return inputs.rotation_pose_3d(w.ports[k], pivot, axis, dth * (step + 1))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
def test_random_moving_ports_lockstep(seed):
    """The same random workloads with every port turning about a nearby pivot after
    each update (sph_port_move), compared with the oracle's port_move bit-exactly."""
    import oracle
    from parity_util import assert_state_equal, gpu_counts_to_oracle, make_updater
    w, steps, mode = random_workload(seed, moving=True)
    mot = random_motion(w, seed)
    K = len(w.ports)
    st = oracle.to_numpy_state(w.state)
    for k, p in enumerate(w.ports):
        oracle.register(st, w.grid, p, k)
    bu = make_updater(w, n_extra=1)
    bu.load(w.state, w.next_id)
    bu.register_ports()
    ports = list(w.ports)
    nid = w.next_id
    for step in range(steps):
        oracle.advect(st, w.dim, w.dt)
        res = oracle.update(w.grid, ports, st)
        assert res.multi_decision == 0
        new, perm, nid = oracle.compact(res, w.dim, K, res.port_counts[None, :], 0, nid)
        poses = [_pose(w, k, mot, step) for k in range(K)]
        for k, (o, Q) in enumerate(poses):
            nxt = Port(o, Q, ports[k].half_extents, ports[k].kind, ports[k].layers, ports[k].bc)
            oracle.port_move(new, w.dim, ports[k], nxt, k)
            ports[k] = nxt
        if mode["fused"]:
            bu.cll_build(dt=w.dt)
        else:
            bu.advect(w.dt)
            bu.cll_build()
        bu.update()
        for k, (o, Q) in enumerate(poses):
            bu.move_port(k, o, Q)
        deferred = mode["deferred"] and step % 2 == 1
        bu.compact(deferred=deferred)
        assert (gpu_counts_to_oracle(bu.port_counts, K) == res.port_counts).all(), step
        if not deferred:
            assert_state_equal(bu.state(), new, f"step {step}")
        assert int(bu.next_id.item()) == nid
        st = new
    assert bu.stats()["motion_errors"] == 0


def _flat(st):
    """state dict with its extra columns as plain keys e0, e1, ... (numpy)."""
    d = {k: (v.cpu().numpy() if isinstance(v, torch.Tensor) else v) for k, v in st.items() if k != "extra"}
    for e, col in enumerate(st.get("extra") or []):
        d[f"e{e}"] = col.cpu().numpy() if isinstance(col, torch.Tensor) else col
    return d


@pytest.mark.gpu
@pytest.mark.parametrize("seed,P", [(s, 2 + s % 2) for s in SEEDS])
def test_random_slabs_lockstep(seed, P):
    """The random workloads cut into P x-slabs run through the migration path
    (sph_cll_key packing leavers / sph_cll_finish appending arrivals, density
    column included) in one process (LoopbackGroup); the union of the slabs
    equals the oracle's single-domain state after every update."""
    import oracle
    from paper_2406_16786_b200.dist import LoopbackGroup, SlabUpdater
    from test_dist import by_id, cat, cell_x
    w, steps, mode = random_workload(seed)
    st = oracle.to_numpy_state(w.state)
    ncx = w.grid.ncell[0]
    cuts = [int(round(i * ncx / P)) for i in range(P + 1)]
    cx = cell_x(w.grid, st["x"])
    slabs = []
    for r in range(P):
        sel = (cx >= cuts[r]) & (cx < cuts[r + 1])
        part = {k: torch.from_numpy(v[sel].copy()) for k, v in st.items() if k != "extra"}
        part["extra"] = [torch.from_numpy(c[sel].copy()) for c in st["extra"]]
        ws = inputs.Workload(w.name, w.dim, w.dp, w.h, w.grid.slab(cuts[r], cuts[r + 1]), w.ports, part, w.dt,
                             w.n_updates, w.next_id)
        su = SlabUpdater(ws, r, P, inputs.capacity_for(ws, 0.3) + 4096, max_migrate=1 << 15,
                         deferred=mode["deferred"], n_extra=1)
        su.load(ws.state, w.next_id)
        slabs.append(su)
    grp = LoopbackGroup(slabs)
    for k, p in enumerate(w.ports):
        oracle.register(st, w.grid, p, k)
    nid = w.next_id
    for s in range(steps):
        st, res, perm, nid = oracle.step(st, w.grid, w.ports, nid, w.dt)
        grp.step(w.dt)
        union = None
        for su in slabs:
            g = _flat(su.bu.state())
            live = g["label"] > -2
            g = {k: v[live] for k, v in g.items()}
            union = g if union is None else cat(union, g)
        union, ref = by_id(union), by_id(_flat(st))
        for k in ref:
            assert np.array_equal(union[k].view(np.uint8), ref[k].view(np.uint8)), f"P={P} step {s} column {k}"
        for su in slabs:
            assert int(su.bu.next_id.item()) == nid
