// sphbuf_cll.cu — cell-linked-list build (the paper rebuilds
// the cell-linked lists every step).  A counting sort by cell with
// ascending id inside each cell, gathering the SoA into the alternate buffer:
//   K1 k_cll_key     pinned cell key of each live particle (optionally fused with
//                    the driver's advection) and its rank in the cell from one
//                    atomic per run of equal keys in a warp (the input is already
//                    nearly sorted by cell, so runs are long);
//   K2 k_cell_scan   single-pass decoupled look-back scan of the histogram ->
//                    cell_start / cell_end; re-zeroes the histogram;
//   K3 k_cll_scatter (source index, cell) pairs into their slots;
//   K4 k_cll_gather  one round of loads per slot (all columns of the source plus
//                    the cell range), rank by id among the cell's slots in shared
//                    memory, store into the sorted position.
#include <climits>
#include <cstdint>

#include "sphbuf_common.cuh"

namespace sphbuf {

constexpr int kKeyItems = 4;

template <bool Advect>
__global__ void __launch_bounds__(kThreads) k_cll_key(PartDev in, GridDev g, Workspace ws, float dt)
{
    Counters *ctr = ws.ctr;
    const long long n = *in.n;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctr->epoch_cll += 1;
        ctr->ticket_cll = 0;
        ctr->n_in = n;
    }
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
    const unsigned le = lt | (1u << lane);
    int oob_acc = 0;
    const long long stride = (long long)gridDim.x * kThreads * kKeyItems;
    for (long long base = (long long)blockIdx.x * kThreads * kKeyItems; base < n; base += stride) {
        int key[kKeyItems], lab[kKeyItems];
        float x[kKeyItems], y[kKeyItems], z[kKeyItems], vx[kKeyItems], vy[kKeyItems], vz[kKeyItems];
        // all loads of the tile first (memory-level parallelism), then the arithmetic
#pragma unroll
        for (int it = 0; it < kKeyItems; ++it) {
            const long long i = base + it * kThreads + threadIdx.x;
            lab[it] = -9;
            if (i < n) {
                lab[it] = in.label[i];
                x[it] = in.x[i];
                y[it] = in.y[i];
                z[it] = g.dim == 3 ? in.z[i] : 0.0f;
                if (Advect) {
                    vx[it] = in.vx[i];
                    vy[it] = in.vy[i];
                    vz[it] = g.dim == 3 ? in.vz[i] : 0.0f;
                }
            }
        }
#pragma unroll
        for (int it = 0; it < kKeyItems; ++it) {
            const long long i = base + it * kThreads + threadIdx.x;
            key[it] = -1;
            if (i < n) {
                if (Advect) {
                    // driver step fused in: x <- fl(x + fl(v dt))
                    x[it] = __fadd_rn(x[it], __fmul_rn(vx[it], dt));
                    y[it] = __fadd_rn(y[it], __fmul_rn(vy[it], dt));
                    in.x[i] = x[it];
                    in.y[i] = y[it];
                    if (g.dim == 3) {
                        z[it] = __fadd_rn(z[it], __fmul_rn(vz[it], dt));
                        in.z[i] = z[it];
                    }
                }
                if (lab[it] > -2) {
                    int oob = 0;
                    key[it] = cell_of(g, x[it], y[it], z[it], oob);
                    oob_acc += oob;
                }
            }
        }
        int cbase[kKeyItems], head_lane[kKeyItems];
#pragma unroll
        for (int it = 0; it < kKeyItems; ++it) {
            const int prev = __shfl_up_sync(0xffffffffu, key[it], 1);
            const bool head = (lane == 0) || (key[it] != prev);
            const unsigned heads = __ballot_sync(0xffffffffu, head);
            head_lane[it] = 31 - __clz(heads & le);
            const unsigned above = heads & ~le;
            const int next = above ? __ffs(above) - 1 : 32;
            cbase[it] = (head && key[it] >= 0) ? atomicAdd(&ws.cell_count[key[it]], next - lane) : 0;
        }
#pragma unroll
        for (int it = 0; it < kKeyItems; ++it) {
            const int b = __shfl_sync(0xffffffffu, cbase[it], head_lane[it]);
            const long long i = base + it * kThreads + threadIdx.x;
            if (i < n) {
                ws.key[i] = key[it];
                ws.rank[i] = b + lane - head_lane[it];
            }
        }
    }
    const unsigned o = warp_sum((unsigned)oob_acc);
    if (lane == 0 && o) atomicAdd((unsigned long long *)&ctr->out_of_grid, (unsigned long long)o);
}

__global__ void __launch_bounds__(kThreads) k_cell_scan(GridDev g, Workspace ws, int *cell_start, int *cell_end,
                                                        long long *n_out, long long ntiles)
{
    __shared__ unsigned s_warp[kThreads / 32 + 1];
    __shared__ long long s_tile;
    __shared__ unsigned s_prefix;
    Counters *ctr = ws.ctr;
    if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->ticket_cll, 1);
    __syncthreads();
    const long long tile = s_tile;
    const unsigned epoch = ctr->epoch_cll;
    const long long nc = g.ncells;
    const long long base = tile * kCellTile + (long long)threadIdx.x * kCellItems;
    int c[kCellItems];
    if (base + kCellItems <= nc) {
        int4 *pc = reinterpret_cast<int4 *>(ws.cell_count + base);
        int4 a = pc[0], b = pc[1];
        c[0] = a.x; c[1] = a.y; c[2] = a.z; c[3] = a.w; c[4] = b.x; c[5] = b.y; c[6] = b.z; c[7] = b.w;
        pc[0] = make_int4(0, 0, 0, 0);
        pc[1] = make_int4(0, 0, 0, 0);
    } else {
#pragma unroll
        for (int j = 0; j < kCellItems; ++j) {
            c[j] = (base + j < nc) ? ws.cell_count[base + j] : 0;
            if (base + j < nc) ws.cell_count[base + j] = 0;
        }
    }
    unsigned sum = 0;
#pragma unroll
    for (int j = 0; j < kCellItems; ++j) sum += (unsigned)c[j];
    unsigned total;
    const unsigned excl = block_excl_scan<kThreads>(sum, total, s_warp);
    if (threadIdx.x < 32) {
        unsigned pre = tile_prefix(ws.tile_cells, tile, epoch, total);
        if (threadIdx.x == 0) s_prefix = pre;
    }
    __syncthreads();
    const unsigned prefix = s_prefix;
    int run = (int)(prefix + excl);
    int st[kCellItems], en[kCellItems];
#pragma unroll
    for (int j = 0; j < kCellItems; ++j) {
        st[j] = run;
        run += c[j];
        en[j] = run;
    }
    if (base + kCellItems <= nc) {
        int4 *ps = reinterpret_cast<int4 *>(cell_start + base);
        int4 *pe = reinterpret_cast<int4 *>(cell_end + base);
        ps[0] = make_int4(st[0], st[1], st[2], st[3]);
        ps[1] = make_int4(st[4], st[5], st[6], st[7]);
        pe[0] = make_int4(en[0], en[1], en[2], en[3]);
        pe[1] = make_int4(en[4], en[5], en[6], en[7]);
    } else {
#pragma unroll
        for (int j = 0; j < kCellItems; ++j)
            if (base + j < nc) {
                cell_start[base + j] = st[j];
                cell_end[base + j] = en[j];
            }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) *n_out = (long long)(prefix + total);
}

constexpr int kScatterItems = 4;

__global__ void __launch_bounds__(kThreads) k_cll_scatter(Workspace ws, const int *cell_start, int *perm)
{
    const long long n = ws.ctr->n_in;
    const long long stride = (long long)gridDim.x * kThreads * kScatterItems;
    for (long long base = (long long)blockIdx.x * kThreads * kScatterItems; base < n; base += stride) {
        int key[kScatterItems], rk[kScatterItems];
#pragma unroll
        for (int it = 0; it < kScatterItems; ++it) {
            const long long i = base + it * kThreads + threadIdx.x;
            key[it] = -1;
            if (i < n) {
                key[it] = ws.key[i];
                rk[it] = ws.rank[i];
            }
        }
#pragma unroll
        for (int it = 0; it < kScatterItems; ++it) {
            const long long i = base + it * kThreads + threadIdx.x;
            if (i >= n) continue;
            if (key[it] >= 0) ws.pair[cell_start[key[it]] + rk[it]] = make_int2((int)i, key[it]);
            else if (perm) perm[i] = -1;                          // tombstone: dropped
        }
    }
}

// K4: one round of loads per output slot (the source's columns and its cell's
// range, all independent), the rank by id among the cell's slots from ids staged
// in shared memory (slots of a cell that straddles the tile edge are read from
// global memory), and the store into the sorted position.  Loads are nearly
// sequential (only particles that changed cell come from far away); stores stay
// inside the cell.
template <bool HasExtra, int ITEMS, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_cll_gather(PartDev in, PartDev out, int dim, Workspace ws,
                                                         const int *cell_start, const int *cell_end, int *perm)
{
    __shared__ long long s_id[(kThreads * ITEMS)];
    const long long n = *out.n;
    for (long long j0 = (long long)blockIdx.x * (kThreads * ITEMS); j0 < n; j0 += (long long)gridDim.x * (kThreads * ITEMS)) {
        int src[ITEMS], cb[ITEMS], ce[ITEMS], lab[ITEMS];
        float x[ITEMS], y[ITEMS], z[ITEMS], vx[ITEMS], vy[ITEMS],
            vz[ITEMS];
        long long id[ITEMS];
        int2 pr[ITEMS];
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            const long long j = j0 + it * kThreads + threadIdx.x;
            pr[it] = j < n ? ws.pair[j] : make_int2(-1, -1);
        }
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            src[it] = pr[it].x;
            if (src[it] < 0) continue;
            const int s = src[it];
            cb[it] = cell_start[pr[it].y];
            ce[it] = cell_end[pr[it].y];
            x[it] = in.x[s];
            y[it] = in.y[s];
            vx[it] = in.vx[s];
            vy[it] = in.vy[s];
            if (dim == 3) {
                z[it] = in.z[s];
                vz[it] = in.vz[s];
            }
            id[it] = in.id[s];
            lab[it] = in.label[s];
            s_id[it * kThreads + threadIdx.x] = id[it];
        }
        __syncthreads();
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            if (src[it] < 0) continue;
            int r = 0;
            const long long lo = cb[it] > j0 ? cb[it] : j0;
            const long long hi = ce[it] < j0 + (kThreads * ITEMS) ? ce[it] : j0 + (kThreads * ITEMS);
            for (long long q = lo; q < hi; ++q) r += (s_id[q - j0] < id[it]);
            for (long long q = cb[it]; q < lo; ++q) r += (in.id[ws.pair[q].x] < id[it]);
            for (long long q = hi; q < ce[it]; ++q) r += (in.id[ws.pair[q].x] < id[it]);
            const int d = cb[it] + r;
            out.x[d] = x[it];
            out.y[d] = y[it];
            out.vx[d] = vx[it];
            out.vy[d] = vy[it];
            if (dim == 3) {
                out.z[d] = z[it];
                out.vz[d] = vz[it];
            }
            if (HasExtra)
                for (int e = 0; e < in.n_extra; ++e) out.extra[e][d] = in.extra[e][src[it]];
            out.id[d] = id[it];
            out.label[d] = lab[it];
            if (perm) perm[src[it]] = d;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ launchers

int sm_count() { return sm_count_cached(); }

cudaError_t launch_cll(const PartDev &in, const PartDev &out, const GridDev &g, const Workspace &ws, int *cell_start,
                       int *cell_end, int *perm, float dt, bool advect, cudaStream_t s, Launch *L)
{
    const long long ntiles = (g.ncells + kCellTile - 1) / kCellTile;
    const long long cap = in.cap;
    L->before(s);
    if (advect) {
        static int grid = 0;
        if (!grid) grid = occ_grid(k_cll_key<true>, kThreads);
        k_cll_key<true><<<cap_grid(grid, cap, kThreads * kKeyItems), kThreads, 0, s>>>(in, g, ws, dt);
    } else {
        static int grid = 0;
        if (!grid) grid = occ_grid(k_cll_key<false>, kThreads);
        k_cll_key<false><<<cap_grid(grid, cap, kThreads * kKeyItems), kThreads, 0, s>>>(in, g, ws, 0.0f);
    }
    L->after(s, KID_CLL_KEY);
    L->before(s);
    k_cell_scan<<<(unsigned)(ntiles > 0 ? ntiles : 1), kThreads, 0, s>>>(g, ws, cell_start, cell_end, out.n, ntiles);
    L->after(s, KID_CELL_SCAN);
    {
        static int grid = 0;
        if (!grid) grid = occ_grid(k_cll_scatter, kThreads);
        L->before(s);
        k_cll_scatter<<<cap_grid(grid, cap, kThreads * kScatterItems), kThreads, 0, s>>>(ws, cell_start, perm);
        L->after(s, KID_CLL_SCATTER);
    }
    L->before(s);
    // 3 slots per thread at <= 64 registers (4 blocks/SM): measured best on C5
    // among 1-4 slots x 1-8 min blocks (profiles/r1_summary.md)
    if (in.n_extra > 0) {
        static int grid = 0;
        if (!grid) grid = occ_grid(k_cll_gather<true, 3, 4>, kThreads);
        k_cll_gather<true, 3, 4><<<cap_grid(grid, cap, kThreads * 3), kThreads, 0, s>>>(in, out, g.dim, ws, cell_start,
                                                                                         cell_end, perm);
    } else {
        static int grid = 0;
        if (!grid) grid = occ_grid(k_cll_gather<false, 3, 4>, kThreads);
        k_cll_gather<false, 3, 4><<<cap_grid(grid, cap, kThreads * 3), kThreads, 0, s>>>(in, out, g.dim, ws,
                                                                                          cell_start, cell_end, perm);
    }
    L->after(s, KID_CLL_GATHER);
    return cudaGetLastError();
}

}  // namespace sphbuf
