"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar: cell tables, cell-list order, created/deleted sets, IDs,
post-compaction order and every column of every particle are compared
BIT-EXACTLY (all state-changing and deciding arithmetic is pinned fp32 on both
sides), which is stricter than the north star's 1e-6 relative for positions.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2406_16786_b200 import inputs, sphbuf
from paper_2406_16786_b200.inputs import BIDIRECTIONAL, INLET, OUTLET, Grid, Port, f32

from parity_util import assert_state_equal, gpu_counts_to_oracle, lockstep, make_updater

pytestmark = pytest.mark.gpu


def test_C1_one_update():
    tot, bu = lockstep(inputs.make("C1"), 1)
    assert list(tot) == [0, 0]


def test_C1e_forty_forty():
    tot, bu = lockstep(inputs.make("C1e"), 1)
    assert list(tot) == [40, 40]
    s = bu.stats()
    assert s["n"] == 8000 and s["candidates"] > 0


def test_C1e_many_updates():
    w = inputs.make("C1e")
    tot, bu = lockstep(w, 20)
    assert tot[0] > 40 and tot[1] > 40


def test_C2_bidirectional_100_updates():
    w = inputs.make("C2")
    tot, bu = lockstep(w, w.n_updates, check_every=5)
    assert tot[0] > 0 and tot[1] > 0


def test_C2_fused_advect_cll_build():
    w = inputs.make("C2")
    tot, bu = lockstep(w, 30, check_every=3, fused=True)
    assert tot[0] > 0 and tot[1] > 0


@pytest.mark.parametrize("name", ["C1e", "C2"])
def test_deferred_compaction(name):
    w = inputs.make(name)
    tot, bu = lockstep(w, 20 if name == "C2" else 5, check_every=1, fused=True, deferred=True)
    assert tot[0] > 0 and tot[1] > 0


def test_cuda_graph_replay_matches_oracle():
    """Two captured updates replayed 5 times (+2 warm-up updates) = 12 oracle updates."""
    w = inputs.make("C2")
    bu = make_updater(w)
    bu.load(w.state, w.next_id)
    bu.register_ports()
    g = bu.capture(w.dt)
    for _ in range(5):
        g.replay()
    bu.cll_build()           # drops the last deferred tombstones
    st = oracle.to_numpy_state(w.state)
    for k, p in enumerate(w.ports):
        oracle.register(st, w.grid, p, k)
    nid = w.next_id
    for _ in range(12):
        st, res, perm, nid = oracle.step(st, w.grid, w.ports, nid, w.dt)
    fin = oracle.update(w.grid, [], st)
    assert_state_equal(bu.state(), {c: v[fin.order] for c, v in st.items()}, "graph replay")
    assert int(bu.next_id.item()) == nid


def test_C4_junction_deferred():
    w = inputs.c4(scale=0.5, nports=8, n_updates=8)
    tot, bu = lockstep(w, 8, check_every=2, fused=True, deferred=True)
    assert tot[0] > 0 and tot[1] > 0


def test_C3_duct_scaled_full_run():
    w = inputs.c3(scale=0.25, n_updates=100)
    tot, bu = lockstep(w, 100, check_every=10)
    assert tot[0] > 0 and tot[1] > 0


def test_C4_junction_scaled():
    w = inputs.c4(scale=0.5, nports=8, n_updates=12)
    tot, bu = lockstep(w, 12, check_every=3)
    assert tot[0] > 0 and tot[1] > 0


def test_C5_slab_scaled():
    w = inputs.c5(scale=0.5, slab=0, nslabs=1, n_updates=6)
    tot, bu = lockstep(w, 6, check_every=2)
    assert tot[0] > 0


# ------------------------------------------------------------------ edge cases

def _tiny(dim=2, n=0, labels=None, pts=None, vel=None):
    st = {c: torch.zeros(n, dtype=torch.float32) for c in ("x", "y", "vx", "vy")}
    if dim == 3:
        st["z"] = torch.zeros(n, dtype=torch.float32)
        st["vz"] = torch.zeros(n, dtype=torch.float32)
    if pts is not None:
        pts = torch.tensor(pts, dtype=torch.float32).reshape(-1, dim)
        for j, c in enumerate(("x", "y", "z")[:dim]):
            st[c] = pts[:, j].contiguous()
    if vel is not None:
        v = torch.tensor(vel, dtype=torch.float32).reshape(-1, dim)
        for j, c in enumerate(("vx", "vy", "vz")[:dim]):
            st[c] = v[:, j].contiguous()
    st["id"] = torch.arange(n, dtype=torch.int64)
    st["label"] = torch.full((n,), -1, dtype=torch.int32) if labels is None else torch.tensor(labels,
                                                                                             dtype=torch.int32)
    return st


def _w(ports, st, dim=2, dt=0.001):
    w = inputs.make("C1")
    return inputs.Workload("tiny", dim, w.dp, w.h, w.grid, ports, st, dt, 1, 1000)


def test_empty_particle_set():
    w = inputs.make("C1")
    ww = _w(w.ports, _tiny(n=0))
    tot, bu = lockstep(ww, 3, state=ww.state)
    assert list(tot) == [0, 0]
    assert bu.stats()["n"] == 0


def test_no_ports():
    w = inputs.make("C1e")
    ww = inputs.Workload("noports", 2, w.dp, w.h, w.grid, [], w.state, w.dt, 1, w.next_id)
    tot, bu = lockstep(ww, 2)
    assert list(tot) == [0, 0]


@pytest.mark.parametrize("n", [1, 7, 33, 1025, 4097])
def test_ragged_sizes(n):
    w = inputs.make("C1e")
    idx = torch.randperm(w.n, generator=torch.Generator().manual_seed(n))[:n].sort().values
    st = {c: v[idx].contiguous() for c, v in w.state.items()}
    ww = inputs.Workload("ragged", 2, w.dp, w.h, w.grid, w.ports, st, w.dt, 1, w.next_id)
    lockstep(ww, 3, state=st)


def test_out_of_grid_particles_are_clamped_like_the_oracle():
    w = inputs.make("C1e")
    st = {c: v.clone() for c, v in w.state.items()}
    st["x"][:50] = -5.0          # far outside the grid
    st["y"][50:60] = 9.0
    ww = inputs.Workload("oob", 2, w.dp, w.h, w.grid, w.ports, st, w.dt, 1, w.next_id)
    tot, bu = lockstep(ww, 2, state=st)
    assert bu.stats()["out_of_grid"] >= 120


def test_staging_overflow_is_reported():
    w = inputs.make("C1e")
    bu = make_updater(w, max_new=8)
    bu.load(w.state, w.next_id)
    bu.register_ports()
    bu.step(w.dt)
    with pytest.raises(sphbuf.SphError) as e:
        bu.stats()
    assert e.value.code == -5


def test_capacity_overflow_is_reported():
    w = inputs.make("C1e")
    bu = make_updater(w, capacity=w.n + 10)
    st = {c: v.clone() for c, v in w.state.items()}
    # make the outlet delete nothing: move outlet particles away so N grows by 40
    bu.load(st, w.next_id)
    bu.register_ports()
    # remove the outlet's deletions by shrinking velocities there
    bu.A.cols["vx"][:bu.A.count()].masked_fill_(bu.A.cols["x"][:bu.A.count()] > 1.5, 0.0)
    bu.step(w.dt)
    with pytest.raises(sphbuf.SphError) as e:
        bu.stats()
    assert e.value.code == -5


def test_motion_error_is_reported():
    w = inputs.make("C1")
    st = {c: v.clone() for c, v in w.state.items()}
    bu = make_updater(w)
    bu.load(st, w.next_id)
    bu.register_ports()
    bu.step(0.05)   # inlet members (X' in (-0.02, 0.02)) move ~0.05: some pass 3a/2 = 0.06 (reading R12)
    with pytest.raises(sphbuf.SphError) as e:
        bu.stats()
    assert e.value.code == -6


def test_hand_cases_H1_to_H5_on_gpu():
    """The oracle's hand cases (tests/test_oracle_pins.py) through the CUDA path."""
    g = inputs.make("C1").grid
    I = (1.0, 0, 0, 0, 1.0, 0, 0, 0, 1.0)
    ports = [Port((f32(0.02), f32(0.2), 0.0), I, (f32(0.02), f32(0.2), 0.0), INLET, 4),
             Port((f32(1.0), f32(0.2), 0.0), I, (f32(0.02), f32(0.2), 0.0), BIDIRECTIONAL, 4),
             Port((f32(1.98), f32(0.2), 0.0), I, (f32(0.02), f32(0.2), 0.0), OUTLET, 4)]
    pts = [[0.0405, 0.1], [0.0395, 0.1],                       # H1
           [1.0205, 0.1], [0.9795, 0.1], [1.0205, 0.3], [1.0, 0.2], [1.005, 0.25],   # H5
           [2.0005, 0.1], [2.01, 0.4205], [1.9995, 0.1], [2.0465, 0.1], [2.01, 0.43]]  # H3
    labels = [0, 0, 1, 1, -1, 1, -1, -1, -1, -1, -1, -1]
    st = _tiny(n=len(pts), pts=pts, labels=labels)
    ww = inputs.Workload("hand", 2, 0.01, 0.013, g, ports, st, 0.0, 1, 1000)
    # registration would relabel fluid inside boxes; labels above are the post-registration ones
    bu = make_updater(ww)
    bu.load(st, 1000)
    bu.registered = True
    for k, p in enumerate(ports):
        rc = sphbuf.lib().sph_port_check(bu.ctx.h, sphbuf._f3(p.origin), sphbuf._f9(p.Q), sphbuf._f3(p.half_extents),
                                         p.kind, 4, 0.01)
        assert rc == 0
        sphbuf.sph_buffer_register(bu.ctx, bu.A, p.origin, p.Q, p.half_extents, p.kind, 4, 0.01)
    ref = oracle.to_numpy_state(st)
    for k, p in enumerate(ports):
        oracle.register(ref, g, p, k)
    res = oracle.update(g, ports, ref)
    new, perm, nid = oracle.compact(res, 2, 3, res.port_counts[None, :], 0, 1000)
    bu.step(None)
    assert_state_equal(bu.state(), new, "hand cases")
    assert gpu_counts_to_oracle(bu.port_counts, 3).tolist() == [1, 1, 0, 0, 1, 2]


def test_extra_columns_are_copied():
    w = inputs.make("C1e")
    st = {c: v.clone() for c, v in w.state.items()}
    g = torch.Generator().manual_seed(3)
    st["extra"] = [torch.rand(w.n, generator=g), torch.rand(w.n, generator=g)]
    lockstep(w, 3, state=st)


def test_perm_outputs():
    w = inputs.make("C1e")
    bu = make_updater(w)
    bu.load(w.state, w.next_id)
    bu.register_ports()
    n0 = bu.A.count()
    perm_c = torch.full((bu.capacity,), -7, dtype=torch.int32, device="cuda")
    bu.advect(w.dt)
    before = bu.state()
    bu.cll_build(perm=perm_c)
    after = bu.state()
    p = perm_c[:n0].cpu()
    assert sorted(p.tolist()) == list(range(n0))
    assert torch.equal(after["id"][p.long()], before["id"])
    bu.update()
    upd = bu.state()
    perm_k = torch.full((bu.capacity,), -7, dtype=torch.int32, device="cuda")
    bu.compact(perm=perm_k)
    fin = bu.state()
    pk = perm_k[:n0].cpu()
    keep = pk >= 0
    assert int((~keep).sum()) == 40
    assert torch.equal(fin["id"][pk[keep].long()], upd["id"][keep])
    assert torch.all(pk[keep][1:] > pk[keep][:-1])


def test_port_registered_between_build_and_update():
    """The build runs the next update's prologue for the ports it knows; a port
    registered after the build makes the update run its own prologue — the result
    equals the oracle's with both ports."""
    w = inputs.make("C2")
    K = len(w.ports)
    st = oracle.to_numpy_state(w.state)
    oracle.register(st, w.grid, w.ports[0], 0)
    bu = make_updater(w)
    bu.load(w.state, w.next_id)

    def reg(k):
        p = w.ports[k]
        assert sphbuf.sph_buffer_register(bu.ctx, bu.A, p.origin, p.Q, p.half_extents, p.kind, p.layers, bu.dp,
                                          bu.members[k:k + 1], None) == k

    reg(0)
    oracle.advect(st, 2, w.dt)
    oracle.register(st, w.grid, w.ports[1], 1)     # port 1 identified at the advected positions
    bu.advect(w.dt)
    bu.cll_build()          # prologue inside the scatter: port 0's runs only
    reg(1)                  # new runs: the update must not use that prologue
    bu.update()
    res = oracle.update(w.grid, w.ports, st)
    new, perm, nid = oracle.compact(res, 2, K, res.port_counts[None, :], 0, w.next_id)
    bu.compact()
    assert (gpu_counts_to_oracle(bu.port_counts, K) == res.port_counts).all()
    assert_state_equal(bu.state(), new, "after update")
    # and a second step where the build's prologue applies again
    oracle.advect(new, 2, w.dt)
    res2 = oracle.update(w.grid, w.ports, new)
    new2, _, nid = oracle.compact(res2, 2, K, res2.port_counts[None, :], 0, nid)
    bu.cll_build(dt=w.dt)
    bu.update()
    bu.compact()
    assert (gpu_counts_to_oracle(bu.port_counts, K) == res2.port_counts).all()
    assert_state_equal(bu.state(), new2, "second update")


def test_call_order_is_enforced():
    """SURVEY §8(b) call order build -> update -> compact: the update's deletion
    list and staging area are live until the compaction consumes them, so a
    compaction without an update, a second update, or a build in between is
    refused with SPH_ERR_STATE (nothing enqueued) and the state stays correct."""
    w = inputs.make("C1e")
    bu = make_updater(w)
    bu.load(w.state, w.next_id)
    bu.register_ports()
    with pytest.raises(sphbuf.SphError) as e:
        bu.compact()
    assert e.value.code == -9
    bu.cll_build(dt=w.dt)
    bu.update()
    for bad in (lambda: bu.update(), lambda: bu.cll_build(), lambda: bu.cll_build(dt=w.dt)):
        with pytest.raises(sphbuf.SphError) as e:
            bad()
        assert e.value.code == -9
    bu.compact()
    with pytest.raises(sphbuf.SphError) as e:
        bu.compact(deferred=True)
    assert e.value.code == -9
    st = oracle.to_numpy_state(w.state)
    for k, p in enumerate(w.ports):
        oracle.register(st, w.grid, p, k)
    new, res, perm, nid = oracle.step(st, w.grid, w.ports, w.next_id, w.dt)
    assert_state_equal(bu.state(), new, "after refused calls")
