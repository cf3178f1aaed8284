"""Multi-rank x-slab decomposition.

* CPU, world size 2, gloo: the decomposition's host logic — neighbour exchange
  of fixed-size migration buffers in the library's record layout, count
  allgather, the ID offset rule — drives a per-rank oracle update; the union of
  the ranks' states must equal the single-process oracle (same IDs, same
  columns) after every update.  Rank 0's NCCL unique id reaches every rank
  through ``dist.broadcast_unique_id`` (the library's bootstrap).
* GPU (one device): the library's loopback communicator runs P slabs of the
  CUDA path in one process (``dist.LoopbackGroup``: device copies stand in for
  NCCL; the same buffers, calls and host logic); the union must equal the
  single-process oracle bit-exactly — C4 cut into slabs, the C5 weak-scaling
  workload generated slab by slab (P = 2, 4; straddling ports; both compaction
  modes), and a P-rank step captured in one CUDA graph.  The library's NCCL
  communicator runs at world size 1 (two ranks cannot share a GPU under NCCL).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2406_16786_b200 import inputs
from paper_2406_16786_b200.dist import broadcast_unique_id, id_offsets

COLS = ("x", "y", "z", "vx", "vy", "vz")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def cell_x(grid, x):
    """pinned fp32 cell x-index (numpy float32 ops round per operation)"""
    t = (x.astype(np.float32) - np.float32(grid.lo[0])) * np.float32(1.0 / grid.cs)
    return np.clip(np.floor(t), 0, grid.ncell[0] - 1).astype(np.int64)


def split(st, grid, cuts):
    cx = cell_x(grid, st["x"])
    return [{k: v[(cx >= cuts[r]) & (cx < cuts[r + 1])] for k, v in st.items()} for r in range(len(cuts) - 1)]


REC = 2 * 3 + 3   # record words per particle (3-D, no extra): pos, vel, id lo/hi, label


def pack(st, sel, max_m):
    buf = np.zeros(4 + max_m * REC, np.float32)
    idx = np.nonzero(sel)[0]
    assert len(idx) <= max_m
    buf[:4].view(np.int32)[0] = len(idx)
    rec = buf[4:4 + len(idx) * REC].reshape(-1, REC)
    for j, c in enumerate(COLS):
        rec[:, j] = st[c][idx]
    ids = st["id"][idx]
    rec[:, 6] = (ids & 0xffffffff).astype(np.uint32).view(np.float32)
    rec[:, 7] = (ids >> 32).astype(np.int32).view(np.float32)
    rec[:, 8] = st["label"][idx].view(np.float32)
    return buf


def unpack(buf):
    n = int(buf[:4].view(np.int32)[0])
    rec = buf[4:4 + n * REC].reshape(-1, REC)
    d = {c: rec[:, j].copy() for j, c in enumerate(COLS)}
    lo = rec[:, 6].view(np.uint32).astype(np.int64)
    hi = rec[:, 7].view(np.int32).astype(np.int64)
    d["id"] = (hi << 32) | lo
    d["label"] = rec[:, 8].view(np.int32).copy()
    return d


def cat(a, b):
    return {k: np.concatenate([a[k], b[k]]) for k in a}


def by_id(st):
    o = np.argsort(st["id"], kind="stable")
    return {k: v[o] for k, v in st.items()}


def _world():
    w = inputs.c4(scale=0.25, nports=4, n_updates=10)
    st = oracle.to_numpy_state(w.state)
    for k, p in enumerate(w.ports):
        oracle.register(st, w.grid, p, k)
    ncx = w.grid.ncell[0]
    cuts = [0, ncx // 2 - 3, ncx]
    return w, st, cuts


class _HostExchange:
    """The exchange pattern of the library's communicator (sphbuf_comm.cpp) over
    torch.distributed on CPU: send lo -> rank-1, send hi -> rank+1 (fixed-size
    buffers, count in the header); allgather of the count vectors."""

    def __init__(self, rank, world):
        self.rank, self.world = rank, world

    def exchange(self, send_lo, send_hi, recv_lo, recv_hi):
        ops = []
        if self.rank > 0:
            ops.append(dist.P2POp(dist.isend, send_lo, self.rank - 1))
            ops.append(dist.P2POp(dist.irecv, recv_lo, self.rank - 1))
        if self.rank < self.world - 1:
            ops.append(dist.P2POp(dist.isend, send_hi, self.rank + 1))
            ops.append(dist.P2POp(dist.irecv, recv_hi, self.rank + 1))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def allgather_counts(self, counts, out):
        dist.all_gather_into_tensor(out.view(-1), counts)


def _rank_main(rank, world, port, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = broadcast_unique_id(rank)          # the library's NCCL bootstrap (ncclGetUniqueId runs on CPU)
    assert isinstance(uid, bytes) and len(uid) == 128
    comm = _HostExchange(rank, world)
    w, st_all, cuts = _world()
    K = len(w.ports)
    g = w.grid.slab(cuts[rank], cuts[rank + 1])
    st = split(st_all, w.grid, cuts)[rank]
    nid = w.next_id
    max_m = 20000
    out = []
    migrated = [0]
    for _ in range(steps):
        oracle.advect(st, 3, w.dt)
        cx = cell_x(w.grid, st["x"])
        lo_sel, hi_sel = cx < cuts[rank], cx >= cuts[rank + 1]
        send_lo, send_hi = torch.from_numpy(pack(st, lo_sel, max_m)), torch.from_numpy(pack(st, hi_sel, max_m))
        recv_lo, recv_hi = torch.zeros_like(send_lo), torch.zeros_like(send_hi)
        comm.exchange(send_lo, send_hi, recv_lo, recv_hi)
        keep = ~(lo_sel | hi_sel)
        migrated[0] += int(recv_lo[:4].view(torch.int32)[0]) + int(recv_hi[:4].view(torch.int32)[0])
        st = {k: v[keep] for k, v in st.items()}
        if rank > 0:
            st = cat(st, unpack(recv_lo.numpy()))
        if rank < world - 1:
            st = cat(st, unpack(recv_hi.numpy()))
        res = oracle.update(g, w.ports, st)
        counts = torch.from_numpy(res.port_counts.astype(np.int32))
        allc = torch.zeros(world, 2 * K, dtype=torch.int32)
        comm.allgather_counts(counts, allc)
        ac = allc.numpy()
        # the host ID rule agrees with the oracle's compaction
        offs = id_offsets(ac, K, K, rank, nid)
        st, perm, nid2 = oracle.compact(res, 3, K, ac, rank, nid)
        new_ids = st["id"][st["id"] >= nid]
        for k in range(K):
            c = int(ac[rank][k])
            if c:
                assert new_ids.min() <= offs[k] <= new_ids.max()
        nid = nid2
        out.append({k: v.copy() for k, v in st.items()})
    q.put((rank, out, nid, migrated[0], uid))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_match_single_process():
    steps = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict()
    received = 0
    uids = set()
    for _ in range(2):
        r, out, nid, mig, uid = q.get(timeout=600)
        got[r] = (out, nid)
        received += mig
        uids.add(uid)
    assert len(uids) == 1, "every rank must receive rank 0's unique id"
    assert received > 0, "no particle crossed the slab face: the exchange was not exercised"
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # single process over the whole domain
    w, st, cuts = _world()
    nid = w.next_id
    moved = 0
    for s in range(steps):
        st, res, perm, nid = oracle.step(st, w.grid, w.ports, nid, w.dt)
        union = by_id(cat(got[0][0][s], got[1][0][s]))
        ref = by_id(st)
        for k in ref:
            np.testing.assert_array_equal(union[k], ref[k], err_msg=f"step {s} column {k}")
        moved += 1
    assert got[0][1] == got[1][1] == nid


@pytest.mark.gpu
def test_migrate_pack_unpack_abi_roundtrip():
    """sph_migrate_pack tombstones and packs exactly the particles whose pinned cell
    x-index lies outside the slab; sph_migrate_unpack appends them unchanged."""
    from paper_2406_16786_b200 import sphbuf
    w = inputs.c4(scale=0.25, nports=4, n_updates=10)
    st = oracle.to_numpy_state(w.state)
    ncx = w.grid.ncell[0]
    g = w.grid.slab(ncx // 3, 2 * ncx // 3)
    a = sphbuf.BufferUpdater(g, w.h, w.dp, [], inputs.capacity_for(w, 0.1), max_migrate=1 << 19)
    b = sphbuf.BufferUpdater(g, w.h, w.dp, [], inputs.capacity_for(w, 0.1), max_migrate=1 << 19)
    a.load(w.state, w.next_id)
    rec = sphbuf.sph_migrate_record_floats(a.ctx)
    lo = torch.zeros(4 + (1 << 19) * rec, device="cuda")
    hi = torch.zeros_like(lo)
    sphbuf.sph_migrate_pack(a.ctx, a.A, lo, hi)
    cx = cell_x(w.grid, st["x"])
    exp_lo, exp_hi = int((cx < ncx // 3).sum()), int((cx >= 2 * ncx // 3).sum())
    assert int(lo[:4].view(torch.int32)[0]) == exp_lo and int(hi[:4].view(torch.int32)[0]) == exp_hi
    lab = a.A.label[:w.n].cpu().numpy()
    assert int((lab == -3).sum()) == exp_lo + exp_hi
    b.load({k: v[:0] for k, v in w.state.items()}, w.next_id)
    sphbuf.sph_migrate_unpack(b.ctx, b.A, lo)
    sphbuf.sph_migrate_unpack(b.ctx, b.A, hi)
    got = by_id({k: v.numpy() for k, v in b.state().items()})
    sel = (cx < ncx // 3) | (cx >= 2 * ncx // 3)
    ref = by_id({k: v[sel] for k, v in st.items()})
    for k in ref:
        np.testing.assert_array_equal(got[k], ref[k], err_msg=k)


@pytest.mark.gpu
@pytest.mark.parametrize("P,deferred", [(2, False), (3, False), (2, True), (3, True)])
def test_loopback_slabs_match_oracle(P, deferred):
    """deferred: compaction fused into the next build, so the slabs also carry
    their keys over with migration (leaver lists); tombstones left
    by the deferred compaction are not part of the state compared."""
    from paper_2406_16786_b200.dist import LoopbackGroup, SlabUpdater
    w = inputs.c4(scale=0.5, nports=8, n_updates=8)
    st = oracle.to_numpy_state(w.state)
    ncx = w.grid.ncell[0]
    cuts = [int(round(i * ncx / P)) for i in range(P + 1)]
    parts = split(st, w.grid, cuts)
    slabs = []
    for r in range(P):
        ws = inputs.Workload(w.name, 3, w.dp, w.h, w.grid.slab(cuts[r], cuts[r + 1]), w.ports,
                             {k: torch.from_numpy(v) for k, v in parts[r].items()}, w.dt, w.n_updates, w.next_id)
        su = SlabUpdater(ws, r, P, inputs.capacity_for(ws, 0.2), max_migrate=1 << 16, deferred=deferred)
        su.load(ws.state, w.next_id)
        slabs.append(su)
    grp = LoopbackGroup(slabs)
    for k, p in enumerate(w.ports):
        oracle.register(st, w.grid, p, k)
    nid = w.next_id
    for s in range(8):
        st, res, perm, nid = oracle.step(st, w.grid, w.ports, nid, w.dt)
        grp.step(w.dt)
        union = None
        for su in slabs:
            g = su.bu.state()
            g = {k: v.numpy() for k, v in g.items()}
            live = g["label"] > -2
            g = {k: v[live] for k, v in g.items()}
            union = g if union is None else cat(union, g)
        union, ref = by_id(union), by_id(st)
        for k in ref:
            np.testing.assert_array_equal(union[k], ref[k], err_msg=f"P={P} step {s} column {k}")
        for su in slabs:
            assert int(su.bu.next_id.item()) == nid
        assert sum(su.bu.stats()["migrated_out"] for su in slabs) >= 0
    assert sum(su.bu.stats()["migrated_out"] for su in slabs) > 0


def _c5_union(P, n_updates):
    """The C5 weak-scaling workload at a CPU-sized scale, generated slab by slab
    (c5(slab=r, nslabs=P)); returns the slabs and the single-domain problem."""
    slabs = [inputs.c5(scale=0.3, slab=r, nslabs=P, n_updates=n_updates) for r in range(P)]
    w0 = slabs[0]
    grid = inputs.Grid(3, w0.grid.lo, w0.grid.cs, w0.grid.ncell)
    st = {k: torch.cat([w.state[k] for w in slabs]) for k in w0.state}
    return slabs, inputs.Workload("C5x0.3-union", 3, w0.dp, w0.h, grid, w0.ports, st, w0.dt, n_updates,
                                  w0.next_id)


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("P", [2, 4])
def test_loopback_c5_multislab_both_compaction_modes(P):
    """BASELINE configs[4] (C5) as the driver's scaling run would cut it: slab r
    generated by c5(slab=r, nslabs=P) (ports straddling slab faces), P ranks of
    the CUDA path through the library's loopback communicator, 10 updates, in-
    place and deferred compaction side by side; the union of the ranks equals
    the single-process oracle bit-exactly after every update."""
    from paper_2406_16786_b200.dist import LoopbackGroup, SlabUpdater, expected_migrants
    n_updates = 10
    slabs, whole = _c5_union(P, n_updates)
    # some port straddles a slab face (its P_k crosses x = 1.6 r * scale)
    faces = [whole.grid.lo[0] + whole.grid.cs * b for (b, e) in slabs[0].slab_cells[1:]]
    straddle = 0
    for p in whole.ports:
        ext = sum(abs(p.Q[3 * r]) * (p.half_extents[r] + whole.grid.cs) for r in range(3))
        straddle += any(p.origin[0] - ext < f < p.origin[0] + ext for f in faces)
    assert straddle > 0
    st = oracle.to_numpy_state(whole.state)
    for k, p in enumerate(whole.ports):
        oracle.register(st, whole.grid, p, k)
    groups = {}
    # one message size for every rank (sender and receiver must agree)
    mm = max(4096, 3 * max(expected_migrants(w.state, w.grid, w.dt, w.dp) for w in slabs))
    for deferred in (False, True):
        us = []
        for r, w in enumerate(slabs):
            su = SlabUpdater(w, r, P, inputs.capacity_for(w, 0.1), max_migrate=mm, deferred=deferred)
            su.load(w.state, w.next_id)
            us.append(su)
        groups[deferred] = (LoopbackGroup(us), us)
    nid = whole.next_id
    for s in range(n_updates):
        st, res, perm, nid = oracle.step(st, whole.grid, whole.ports, nid, whole.dt)
        ref = by_id(st)
        for deferred, (grp, us) in groups.items():
            grp.step(whole.dt)
            union = None
            for su in us:
                g = {k: v.numpy() for k, v in su.bu.state().items()}
                live = g["label"] > -2
                g = {k: v[live] for k, v in g.items()}
                union = g if union is None else cat(union, g)
            union = by_id(union)
            for k in ref:
                np.testing.assert_array_equal(union[k], ref[k], err_msg=f"P={P} deferred={deferred} step {s} {k}")
            for su in us:
                assert int(su.bu.next_id.item()) == nid
    for deferred, (grp, us) in groups.items():
        assert sum(su.bu.stats()["migrated_out"] for su in us) > 0


@pytest.mark.gpu
def test_loopback_step_captured_in_one_cuda_graph():
    """A P = 2 step (key pass + pack, exchange, finish + update, count allgather,
    compaction on both ranks) captured in one CUDA graph and replayed: the union
    equals the oracle after 2 warm-up + 3 x 2 replayed updates."""
    from paper_2406_16786_b200.dist import LoopbackGroup, SlabUpdater
    w = inputs.c4(scale=0.5, nports=8, n_updates=8)
    st = oracle.to_numpy_state(w.state)
    ncx = w.grid.ncell[0]
    cuts = [0, ncx // 2, ncx]
    parts = split(st, w.grid, cuts)
    us = []
    for r in range(2):
        ws = inputs.Workload(w.name, 3, w.dp, w.h, w.grid.slab(cuts[r], cuts[r + 1]), w.ports,
                             {k: torch.from_numpy(v) for k, v in parts[r].items()}, w.dt, w.n_updates, w.next_id)
        su = SlabUpdater(ws, r, 2, inputs.capacity_for(ws, 0.2), max_migrate=1 << 15, deferred=True)
        su.load(ws.state, w.next_id)
        us.append(su)
    grp = LoopbackGroup(us)
    g = grp.capture(w.dt)
    for _ in range(3):
        g.replay()
    for k, p in enumerate(w.ports):
        oracle.register(st, w.grid, p, k)
    nid = w.next_id
    for _ in range(8):
        st, res, perm, nid = oracle.step(st, w.grid, w.ports, nid, w.dt)
    union = None
    for su in us:
        gg = {k: v.numpy() for k, v in su.bu.state().items()}
        live = gg["label"] > -2
        gg = {k: v[live] for k, v in gg.items()}
        union = gg if union is None else cat(union, gg)
    union, ref = by_id(union), by_id(st)
    for k in ref:
        np.testing.assert_array_equal(union[k], ref[k], err_msg=k)
    assert int(us[0].bu.next_id.item()) == int(us[1].bu.next_id.item()) == nid


@pytest.mark.gpu
def test_nccl_communicator_single_rank():
    """The library's own NCCL communicator (sph_comm_init from a unique id that
    torch.distributed broadcast): at world size 1 the fused migrate + build and
    the ncclAllGather of the counts run through NCCL, bit-exact with the oracle."""
    from paper_2406_16786_b200 import sphbuf
    from paper_2406_16786_b200.dist import SlabUpdater
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        uid = broadcast_unique_id(0)
        w = inputs.make("C2")
        su = SlabUpdater(w, 0, 1, inputs.capacity_for(w), max_migrate=1024)
        su.init_nccl(uid)
        with pytest.raises(sphbuf.SphError) as e:
            su.init_nccl(uid)
        assert e.value.code == -9
        su.load(w.state, w.next_id)
        st = oracle.to_numpy_state(w.state)
        for k, p in enumerate(w.ports):
            oracle.register(st, w.grid, p, k)
        nid = w.next_id
        for s in range(5):
            st, res, perm, nid = oracle.step(st, w.grid, w.ports, nid, w.dt)
            su.step(w.dt)
            assert su.all_counts[0].cpu().tolist()[:2] == res.port_counts[:2].tolist()
        su.bu.cll_build()          # drops the tombstones a deferred compaction would leave
        got = by_id({k: v.numpy() for k, v in su.bu.state().items()})
        ref = by_id(st)
        for k in ref:
            np.testing.assert_array_equal(got[k], ref[k], err_msg=k)
        assert su.bu.stats()["n"] == len(st["x"])
    finally:
        dist.destroy_process_group()
