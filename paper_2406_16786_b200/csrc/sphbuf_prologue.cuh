// sphbuf_prologue.cuh — K5, the update prologue (arXiv 2406.16786 §III, "local
// cell-linked lists" P:411-413): candidate count per port run (cell ranges from
// the current cell list) and their exclusive scan over NT-run tiles (ticket
// order, decoupled look-back), so any number of runs is scanned by many blocks
// at once; also each run's first particle index and the run holding the first
// candidate of every K6 tile; resets the per-update counters.  The tile tickets
// and the epoch are advanced by the last of its `nblocks` blocks to finish.  Run
// either as its own kernel (k_upd_prologue) or by extra blocks of the build's
// scatter, which already has the cell tables it needs (then sph_buffer_update
// launches K6 alone).
#pragma once
#include <climits>

#include "sphbuf_common.cuh"

namespace sphbuf {

template <int NT>
__device__ __forceinline__ void upd_prologue_body(const Workspace &ws, int n_runs, const int *cell_start,
                                                  const int *cell_end, int max_ports, int nblocks)
{
    __shared__ unsigned s_warp[NT / 32 + 1];
    __shared__ int s_tile;
    __shared__ unsigned s_prefix;
    Counters *ctr = ws.ctr;
    const int ntiles = (n_runs + NT - 1) / NT;
    const unsigned epoch = ctr->epoch_upd + 1;
    if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->ticket_runs, 1);
    __syncthreads();
    const int tile = s_tile;
    if (tile == 0) {
        if (threadIdx.x == 0) {
            ctr->ticket_upd = 0;
            ctr->n_stage = 0;
            ctr->n_stage_raw = 0;
            ctr->n_dlist = 0;
            ctr->n_del = 0;
            ctr->i_first = LLONG_MAX;
        }
        for (int i = threadIdx.x; i < 2 * max_ports; i += NT) ws.port_cnt[i] = 0;
    }
    if (tile < ntiles) {
        const int r = tile * NT + threadIdx.x;
        unsigned len = 0;
        int base = 0;
        // (c1 < c0: an empty slot of a movable port's run slice)
        if (r < n_runs && ws.runs[3 * r + 1] >= ws.runs[3 * r]) {
            base = cell_start[ws.runs[3 * r]];
            len = (unsigned)(cell_end[ws.runs[3 * r + 1]] - base);
        }
        unsigned total;
        const unsigned ex = block_excl_scan<NT>(len, total, s_warp);
        if (threadIdx.x < 32) {
            const unsigned pre = tile_prefix(ws.tile_runs, tile, epoch, total);
            if (threadIdx.x == 0) s_prefix = pre;
        }
        __syncthreads();
        if (r < n_runs) {
            const long long off = (long long)s_prefix + ex;
            ws.run_off[r] = off;
            ws.run_base[r] = base;
            // the run holding the first candidate of each K6 tile starting inside it
            for (long long t = (off + kUpdTile - 1) / kUpdTile; t * kUpdTile < off + len && t < ws.upd_tiles; ++t)
                ws.tile_run[t] = r;
        }
        if (tile == ntiles - 1 && threadIdx.x == 0) {
            const long long carry = (long long)s_prefix + total;
            ws.run_off[n_runs] = carry;
            ctr->n_cand = carry;
            ctr->checked += carry;
            if ((carry + kUpdTile - 1) / kUpdTile > ws.upd_tiles) ctr->status |= kStCapacity;
        }
    }
    if (ntiles == 0 && tile == 0 && threadIdx.x == 0) {
        ws.run_off[0] = 0;
        ctr->n_cand = 0;
    }
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&ctr->done_runs, 1) == nblocks - 1) {
            ctr->done_runs = 0;
            ctr->ticket_runs = 0;
            ctr->epoch_upd = epoch;
        }
    }
}

}  // namespace sphbuf
