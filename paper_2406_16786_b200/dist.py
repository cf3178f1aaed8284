"""x-slab domain decomposition of the buffer update across GPUs.

One process per GPU.  Each rank owns the particles whose pinned cell x-index
lies in its slab [cx_begin, cx_end) and registers every port (a port that
straddles a slab face is split naturally: decisions are per particle).  Two
exchanges per update, both over NCCL (torch.distributed) on NVLink/NVSwitch:

1. neighbour migration after advection: particles whose cell left the slab are
   packed by ``sph_migrate_pack`` into fixed-size device buffers (count in the
   header, so no host synchronisation), exchanged with ranks r-1 / r+1 and
   appended by ``sph_migrate_unpack``; the next cell-list build drops the
   tombstones;
2. an allgather of the per-rank per-port create/delete counts, from which
   ``sph_compact`` derives GPU-count-independent IDs
   off(k, r) = next_id + sum_{k'<k} sum_r' C[r'][k'] + sum_{r'<r} C[r'][k].

``Comm`` wraps torch.distributed (NCCL on GPUs, gloo on CPU for tests);
``LoopbackGroup`` runs P slabs in one process on one GPU with device copies in
place of the collectives (testing the decomposition without P GPUs; no kernel
waits on another).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import sphbuf


class Comm:
    def __init__(self, rank: int, world: int):
        self.rank, self.world = rank, world

    def exchange(self, send_lo, send_hi, recv_lo, recv_hi):
        """send_lo -> rank-1, send_hi -> rank+1; receive rank-1's send_hi into recv_lo and
        rank+1's send_lo into recv_hi.  Fixed-size buffers (count in the header)."""
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

    def allgather_counts(self, counts: torch.Tensor, out: torch.Tensor):
        """out [world, len(counts)] <- every rank's counts."""
        if self.world == 1:
            out[0].copy_(counts)
            return
        dist.all_gather_into_tensor(out.view(-1), counts)


def id_offsets(all_counts, n_ports: int, max_ports: int, rank: int, next_id: int):
    """Host reference of the ID offset rule (used by the CPU tests): for each port
    k, the first new ID of rank `rank`'s particles of port k."""
    offs = []
    acc = next_id
    for k in range(n_ports):
        col = [int(all_counts[r][k]) for r in range(len(all_counts))]
        offs.append(acc + sum(col[:rank]))
        acc += sum(col)
    return offs


class SlabUpdater:
    """One rank: BufferUpdater + migration buffers + count matrix."""

    def __init__(self, w, rank: int, world: int, capacity: int, max_migrate: int, max_new=None, comm=None,
                 device="cuda", deferred=False, n_extra=0):
        self.rank, self.world = rank, world
        self.deferred = deferred
        self.bu = sphbuf.BufferUpdater(w.grid, w.h, w.dp, w.ports, capacity, max_new=max_new,
                                       max_migrate=max_migrate, n_extra=n_extra, device=device)
        rec = sphbuf.sph_migrate_record_floats(self.bu.ctx)
        n = 4 + max_migrate * rec
        mk = lambda: torch.zeros(n, dtype=torch.float32, device=device)
        self.send_lo, self.send_hi, self.recv_lo, self.recv_hi = mk(), mk(), mk(), mk()
        self.all_counts = torch.zeros(world, 2 * sphbuf.MAX_PORTS, dtype=torch.int32, device=device)
        self.comm = comm if comm is not None else Comm(rank, world)

    def load(self, state, next_id):
        self.bu.load(state, next_id)
        self.bu.register_ports()

    # phases (LoopbackGroup interleaves them across slabs)
    def phase_advect_pack(self, dt):
        """advection + cell keys + migration pack in one pass (sph_cll_key)"""
        bu = self.bu
        if self.world > 1:
            sphbuf.sph_cll_key(bu.ctx, bu.A, dt, self.send_lo, self.send_hi)
        else:
            sphbuf.sph_cll_key(bu.ctx, bu.A, dt)

    def phase_unpack_update(self):
        """received particles appended + rest of the build (sph_cll_finish), update"""
        bu = self.bu
        rlo = self.recv_lo if (self.world > 1 and self.rank > 0) else None
        rhi = self.recv_hi if (self.world > 1 and self.rank < self.world - 1) else None
        sphbuf.sph_cll_finish(bu.ctx, bu.A, bu.B, bu.cell_start, bu.cell_end, rlo, rhi)
        bu.A, bu.B = bu.B, bu.A
        bu.update()

    def phase_compact(self):
        if self.world > 1:
            self.bu.compact(self.all_counts, self.world, self.rank, deferred=self.deferred)
        else:
            self.bu.compact(deferred=self.deferred)

    def step(self, dt):
        self.phase_advect_pack(dt)
        if self.world > 1:
            self.comm.exchange(self.send_lo, self.send_hi, self.recv_lo, self.recv_hi)
        self.phase_unpack_update()
        if self.world > 1:
            self.comm.allgather_counts(self.bu.port_counts, self.all_counts)
        self.phase_compact()


class LoopbackGroup:
    """P slabs in one process on one GPU; device copies stand in for NCCL."""

    def __init__(self, slabs: list):
        self.slabs = slabs

    def step(self, dt):
        P = len(self.slabs)
        for s in self.slabs:
            s.phase_advect_pack(dt)
        for r, s in enumerate(self.slabs):
            if r > 0:
                s.recv_lo.copy_(self.slabs[r - 1].send_hi)
            if r < P - 1:
                s.recv_hi.copy_(self.slabs[r + 1].send_lo)
        for s in self.slabs:
            s.phase_unpack_update()
        counts = torch.stack([s.bu.port_counts for s in self.slabs])
        for s in self.slabs:
            s.all_counts.copy_(counts)
            s.phase_compact()
