"""x-slab domain decomposition of the buffer update across GPUs.

One process per GPU.  Each rank owns the particles whose pinned cell x-index
lies in its slab [cx_begin, cx_end) and registers every port (a port that
straddles a slab face is split naturally: decisions are per particle, and the
candidates lie in "the nearby local cell-linked lists").  Two
exchanges per update, both owned by the library (include/sphbuf.h, "Multi-GPU")
and enqueued on the rank's stream, so nothing synchronises the host:

1. neighbour migration fused into the cell-list build
   (``sph_migrate_cll_build`` = key pass packing the leavers into the library's
   buffers -> ``ncclSend``/``ncclRecv`` with ranks r-1 / r+1 in one group ->
   arrivals appended before the scan/scatter/gather);
2. ``sph_allgather_counts`` (``ncclAllGather``) of the per-rank per-port
   create/delete counts, from which ``sph_compact`` derives GPU-count-independent
   IDs off(k, r) = next_id + sum_{k'<k} sum_r' C[r'][k'] + sum_{r'<r} C[r'][k].

PyTorch is plumbing only: ``torch.distributed`` (any backend) broadcasts rank 0's
NCCL unique id; the library creates and owns its ``ncclComm_t``.
``LoopbackGroup`` runs P slabs in one process on one GPU through the library's
loopback communicator (device copies in place of NCCL, the same buffers and
host logic), phase by phase so no kernel waits on another.
"""
from __future__ import annotations

import math

import torch

from . import sphbuf


def id_offsets(all_counts, n_ports: int, max_ports: int, rank: int, next_id: int):
    """Host statement of the ID offset rule (used by the CPU tests): for each port
    k, the first new ID of rank `rank`'s particles of port k."""
    offs = []
    acc = next_id
    for k in range(n_ports):
        col = [int(all_counts[r][k]) for r in range(len(all_counts))]
        offs.append(acc + sum(col[:rank]))
        acc += sum(col)
    return offs


def broadcast_unique_id(rank: int, group=None) -> bytes:
    """Rank 0's NCCL unique id, broadcast over torch.distributed (plumbing)."""
    import torch.distributed as dist
    obj = [sphbuf.sph_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def expected_migrants(state, grid, dt: float, dp: float) -> int:
    """Expected particles per step that one migration sends across one interior
    face of the slab [cx_begin, cx_end) of ``grid`` in steady flow: the outward
    flux sum_i max(+-v_x, 0) dt / dp over the particles within one spacing dp of
    the face (the larger of the two faces; 0 for a slab without interior faces).
    Used to size the fixed migration messages (with headroom by the caller)."""
    x = state["x"].double()
    vx = state["vx"].double()
    best = 0.0
    if grid.cx_begin > 0:
        f = grid.lo[0] + grid.cx_begin * float(grid.cs)
        near = (x >= f) & (x < f + dp)
        best = max(best, float((torch.clamp(-vx[near], min=0.0) * (dt / dp)).sum()))
    if grid.cx_end < grid.ncell[0]:
        f = grid.lo[0] + grid.cx_end * float(grid.cs)
        near = (x < f) & (x >= f - dp)
        best = max(best, float((torch.clamp(vx[near], min=0.0) * (dt / dp)).sum()))
    return int(math.ceil(best))


class SlabUpdater:
    """One rank: a BufferUpdater whose context owns the communicator, the
    migration buffers (in its workspace) and the count matrix."""

    def __init__(self, w, rank: int, world: int, capacity: int, max_migrate: int, max_new=None, device="cuda",
                 deferred=False, n_extra=0):
        self.rank, self.world = rank, world
        self.deferred = deferred
        self.bu = sphbuf.BufferUpdater(w.grid, w.h, w.dp, w.ports, capacity, max_new=max_new,
                                       max_migrate=max_migrate, n_extra=n_extra, device=device)
        self.all_counts = torch.zeros(world, 2 * sphbuf.MAX_PORTS, dtype=torch.int32, device=device)
        self.has_comm = False

    def init_nccl(self, unique_id: bytes):
        """Collective: the library's NCCL communicator of this rank."""
        sphbuf.sph_comm_init(self.bu.ctx, unique_id, self.world, self.rank)
        self.has_comm = True

    def load(self, state, next_id):
        self.bu.load(state, next_id)
        self.bu.register_ports()

    # --- one update of one rank (NCCL, or a single rank)
    def step(self, dt, stream=None):
        bu = self.bu
        if not self.has_comm:                  # a single rank without a communicator
            assert self.world == 1
            bu.step(dt, stream, deferred=self.deferred)
            return
        sphbuf.sph_migrate_cll_build(bu.ctx, bu.A, bu.B, dt, bu.cell_start, bu.cell_end, stream=stream)
        bu.A, bu.B = bu.B, bu.A
        bu.update(stream)
        sphbuf.sph_allgather_counts(bu.ctx, bu.port_counts, self.all_counts, stream)
        bu.compact(self.all_counts, self.world, self.rank, stream=stream, deferred=self.deferred)

    # --- the same update in phases (a loopback group interleaves them across ranks)
    def phase_key(self, dt):
        """advection + cell keys; leavers packed into the library's buffers"""
        sphbuf.sph_cll_key(self.bu.ctx, self.bu.A, dt)

    def phase_exchange(self):
        sphbuf.sph_migrate_exchange(self.bu.ctx)

    def phase_finish_update(self):
        """arrivals appended + rest of the build, then the buffer update"""
        bu = self.bu
        sphbuf.sph_cll_finish(bu.ctx, bu.A, bu.B, bu.cell_start, bu.cell_end)
        bu.A, bu.B = bu.B, bu.A
        bu.update()

    def phase_allgather(self):
        sphbuf.sph_allgather_counts(self.bu.ctx, self.bu.port_counts, self.all_counts)

    def phase_compact(self):
        self.bu.compact(self.all_counts, self.world, self.rank, deferred=self.deferred)


class LoopbackGroup:
    """P slabs in one process on one GPU, joined by the library's loopback
    communicator (sph_comm_init_loopback)."""

    def __init__(self, slabs: list):
        self.slabs = slabs
        sphbuf.sph_comm_init_loopback([s.bu.ctx for s in slabs])
        for s in slabs:
            s.has_comm = True

    def step(self, dt):
        for s in self.slabs:
            s.phase_key(dt)
        for s in self.slabs:
            s.phase_exchange()
        for s in self.slabs:
            s.phase_finish_update()
        for s in self.slabs:
            s.phase_allgather()
        for s in self.slabs:
            s.phase_compact()

    def capture(self, dt):
        """Two P-rank updates captured in one CUDA graph (after two warm-up
        updates, so the carried-key bookkeeping repeats with period two)."""
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.step(dt)
            self.step(dt)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step(dt)
            self.step(dt)
        return g
