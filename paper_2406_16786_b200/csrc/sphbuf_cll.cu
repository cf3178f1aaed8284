// sphbuf_cll.cu — cell-linked-list build (the paper rebuilds
// the cell-linked lists every step).  A counting sort by cell with
// ascending id inside each cell, gathering the SoA into the alternate buffer:
//   K1 k_cll_key     pinned cell key of each live particle (optionally fused with
//                    the driver's advection) and its rank in the cell from one
//                    atomic per run of equal keys in a warp (the input is already
//                    nearly sorted by cell, so runs are long);
//   K2 k_cell_scan   single-pass decoupled look-back scan of the histogram ->
//                    cell_start / cell_end (warp-striped, coalesced); re-zeroes
//                    the histogram and the scatter's cursors;
//   K3 k_cll_scatter (source index, cell) pairs into their slots;
//   K4 k_cll_gather  one round of loads per slot (all columns of the source plus
//                    the cell range), rank by id among the cell's slots in shared
//                    memory, store into the sorted position.
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include <cooperative_groups.h>

#include "sphbuf_common.cuh"
#include "sphbuf_prologue.cuh"
#include "sphbuf_tma.cuh"

namespace sphbuf {

constexpr int kKeyItems = 4;

// Migration record of particle i (multi-GPU x-slabs): position,
// velocity, extras, id (two 32-bit words), label; slot from the header count.
__device__ __forceinline__ void pack_record(const PartDev &in, int dim, long long i, float x, float y, float z,
                                            int lab, float *buf, long long maxm, int rec, Counters *ctr)
{
    const int slot = atomicAdd(reinterpret_cast<int *>(buf), 1);
    if (slot >= maxm) {
        atomicOr(&ctr->status, kStMigrate);
        return;
    }
    float *r = buf + 4 + (long long)slot * rec;
    int w = 0;
    r[w++] = x;
    r[w++] = y;
    if (dim == 3) r[w++] = z;
    r[w++] = in.vx[i];
    r[w++] = in.vy[i];
    if (dim == 3) r[w++] = in.vz[i];
    for (int e = 0; e < in.n_extra; ++e) r[w++] = in.extra[e][i];
    const long long id = in.id[i];
    r[w++] = __int_as_float((int)(id & 0xffffffffll));
    r[w++] = __int_as_float((int)(id >> 32));
    r[w++] = __int_as_float(lab);
}

// K1.  Migrate (multi-GPU): a particle whose (advected) cell x-index left the
// slab is packed for the neighbour rank and gets no key (dropped from this
// slab's build) — the migration costs no extra pass over the array.
template <bool Advect, bool Migrate>
__global__ void __launch_bounds__(kThreads) k_cll_key(PartDev in, GridDev g, Workspace ws, float dt, float *mlo,
                                                      float *mhi, long long maxm, int rec)
{
    pdl_entry();
    Counters *ctr = ws.ctr;
    const long long n = *in.n;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctr->n_in = n;
        ctr->mig_base = n;
    }
    long long moved = 0;
    const int lane = threadIdx.x & 31;
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
                    // driver step fused in: x <- fl(x + fl(v dt)), kept in registers
                    // for the key; the gather recomputes it bit-identically when it
                    // moves the particle, so `in` is never written here
                    x[it] = advect1(x[it], vx[it], dt);
                    y[it] = advect1(y[it], vy[it], dt);
                    if (g.dim == 3) z[it] = advect1(z[it], vz[it], dt);
                }
                if (lab[it] > -2) {
                    if (Migrate) {
                        int o2 = 0;
                        const int cxr = cell_axis(x[it], g.lo[0], g.inv_cs, 0, g.ncell[0], o2);
                        if (cxr < g.cx_begin || cxr >= g.cx_end) {
                            pack_record(in, g.dim, i, x[it], y[it], z[it], lab[it], cxr < g.cx_begin ? mlo : mhi,
                                        maxm, rec, ctr);
                            ++moved;
                            continue;
                        }
                    }
                    int oob = 0;
                    key[it] = cell_of(g, x[it], y[it], z[it], oob);
                    oob_acc += oob;
                }
            }
        }
#pragma unroll
        for (int it = 0; it < kKeyItems; ++it) {
            hist_count_match(ws.cell_count, key[it]);    // one atomic per distinct key of the warp
            const long long i = base + it * kThreads + threadIdx.x;
            if (i < n) ws.key[i] = key[it];
        }
    }
    const unsigned o = warp_sum((unsigned)oob_acc);
    if (lane == 0 && o) atomicAdd((unsigned long long *)&ctr->out_of_grid, (unsigned long long)o);
    if (Migrate) {
        moved = warp_sum_ll(moved);
        if (lane == 0 && moved) atomicAdd((unsigned long long *)&ctr->migrated, (unsigned long long)moved);
    }
}

// K1 in key carry-over mode with slab migration: the listed leavers (still keyed
// kLeaver; a later fix-up may have kept one inside, a duplicate entry is claimed
// once) are packed for the neighbour ranks with their advected positions, as the
// key pass would have; everything else was keyed by the previous build.
__global__ void __launch_bounds__(kThreads) k_mig_pack_list(PartDev in, GridDev g, Workspace ws, float dt,
                                                            float *mlo, float *mhi, long long maxm, int rec)
{
    pdl_entry();
    Counters *ctr = ws.ctr;
    const long long n = *in.n;
    long long nl = ctr->n_leave;
    if (nl > ws.max_leave) nl = ws.max_leave;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctr->n_in = n;
        ctr->mig_base = n;
    }
    long long moved = 0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nl; e += (long long)gridDim.x * blockDim.x) {
        const int i = ws.leave[e];
        if (atomicCAS(&ws.key[i], kLeaver, kPacked) != kLeaver) continue;
        const float x = advect1(in.x[i], in.vx[i], dt), y = advect1(in.y[i], in.vy[i], dt),
                    z = g.dim == 3 ? advect1(in.z[i], in.vz[i], dt) : 0.0f;
        int o2 = 0;
        const int cxr = cell_axis(x, g.lo[0], g.inv_cs, 0, g.ncell[0], o2);
        pack_record(in, g.dim, i, x, y, z, in.label[i], cxr < g.cx_begin ? mlo : mhi, maxm, rec, ctr);
        ++moved;
    }
    moved = warp_sum_ll(moved);
    if ((threadIdx.x & 31) == 0 && moved) atomicAdd((unsigned long long *)&ctr->migrated, (unsigned long long)moved);
}

// K1b (multi-GPU): append the particles received from the neighbour slabs after
// the local ones (index mig_base + s) with their keys and ranks, before the scan.
__global__ void __launch_bounds__(kThreads) k_cll_unpack_key(PartDev in, GridDev g, Workspace ws, const float *blo,
                                                             const float *bhi, long long maxm, int rec)
{
    pdl_entry();
    Counters *ctr = ws.ctr;
    const long long nlo = blo ? min((long long)__float_as_int(blo[0]), maxm) : 0;
    const long long nhi = bhi ? min((long long)__float_as_int(bhi[0]), maxm) : 0;
    const long long base = ctr->mig_base;
    long long R = nlo + nhi;
    if (base + R > in.cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&ctr->status, kStCapacity);
        R = in.cap - base;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) ctr->n_in = base + R;
    const int dim = g.dim;
    int oob_acc = 0;
    for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < R; s += (long long)gridDim.x * blockDim.x) {
        const float *r = s < nlo ? blo + 4 + s * rec : bhi + 4 + (s - nlo) * rec;
        const long long d = base + s;
        int w = 0;
        const float x = r[w++], y = r[w++], z = dim == 3 ? r[w++] : 0.0f;
        in.x[d] = x;
        in.y[d] = y;
        if (dim == 3) in.z[d] = z;
        in.vx[d] = r[w++];
        in.vy[d] = r[w++];
        if (dim == 3) in.vz[d] = r[w++];
        for (int e = 0; e < in.n_extra; ++e) in.extra[e][d] = r[w++];
        const long long lo = (unsigned)__float_as_int(r[w++]);
        const long long hi = __float_as_int(r[w++]);
        in.id[d] = (hi << 32) | lo;
        const int lab = __float_as_int(r[w++]);
        in.label[d] = lab;
        int oob = 0;
        const int key = cell_of(g, x, y, z, oob);
        oob_acc += oob;
        ws.key[d] = key;
        atomicAdd(&ws.cell_count[key], 1);
    }
    const unsigned o = warp_sum((unsigned)oob_acc);
    if ((threadIdx.x & 31) == 0 && o) atomicAdd((unsigned long long *)&ctr->out_of_grid, (unsigned long long)o);
}

// K2: kCellItems cells per thread (kCellTile per block: one wave of blocks even
// at C5's 8.5M cells, so the look-back chain never waits on an unlaunched tile).
// n_src: with carried-over keys and no migration (no key pass ran), the input
// count to record for the scatter and the gather.  The tile tickets and the
// look-back epoch are advanced by the last block to finish, for the next build.
#ifdef SPHBUF_TRACE
// K2 tile timeline (tools/upd_trace.py): start, loads + block scan done,
// look-back done, end, block, SM.
constexpr int kTraceScan = 1 << 12;
__device__ unsigned long long g_trace_scan[kTraceScan][6];
__device__ __forceinline__ unsigned long long gtimer2()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define SCAN_TRACE(slot)                                                                             \
    do {                                                                                             \
        if (threadIdx.x == 0 && tile < kTraceScan) g_trace_scan[tile][slot] = gtimer2();             \
    } while (0)
#else
#define SCAN_TRACE(slot) \
    do {                 \
    } while (0)
#endif

template <int kCellItems>
__global__ void __launch_bounds__(kThreads) k_cell_scan(GridDev g, Workspace ws, int *cell_start, int *cell_end,
                                                        long long *n_out, long long ntiles, const long long *n_src)
{
    pdl_entry();
    constexpr int kCellTile = kThreads * kCellItems;
    constexpr int V = kCellItems / 4;
    __shared__ unsigned s_warp[kThreads / 32 + 1];
    __shared__ long long s_tile;
    __shared__ unsigned s_prefix;
    Counters *ctr = ws.ctr;
    if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->ticket_cll, 1);
    __syncthreads();
    const long long tile = s_tile;
    SCAN_TRACE(0);
#ifdef SPHBUF_TRACE
    if (threadIdx.x == 0 && tile < kTraceScan) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_trace_scan[tile][4] = blockIdx.x;
        g_trace_scan[tile][5] = smid;
    }
#endif
    const unsigned epoch = ctr->epoch_cll;
    if (n_src && tile == 0 && threadIdx.x == 0) {
        ctr->n_in = *n_src;
        ctr->mig_base = *n_src;
    }
    const long long nc = g.ncells;
    // warp-striped layout: warp w owns cells [tile base + w 32 kCellItems, +32 kCellItems);
    // row v of it is int4 #(32 v + lane), so every load / store instruction of a
    // warp covers 512 contiguous bytes.  Two passes over the tile: the sums (loads
    // kRowBatch rows at a time), then, after the look-back, the rows again (L2) for
    // the cell ranges — a tile of kCellTile cells costs few registers, so at C5 all
    // tiles are resident in one wave and the look-back never waits on a later one.
    constexpr int kRowBatch = V < 8 ? V : 8;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long wbase = tile * kCellTile + (long long)warp * (32 * kCellItems);
    const bool full = tile * kCellTile + kCellTile <= nc;
    const int4 *pc = reinterpret_cast<const int4 *>(ws.cell_count + wbase) + lane;
    auto row = [&](int v) -> int4 {
        if (full) return __ldcg(pc + 32 * v);
        int t[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const long long j = wbase + 4 * (32 * v + lane) + q;
            t[q] = j < nc ? __ldcg(ws.cell_count + j) : 0;
        }
        return make_int4(t[0], t[1], t[2], t[3]);
    };
    unsigned tsum = 0;
#pragma unroll
    for (int v0 = 0; v0 < V; v0 += kRowBatch) {
        int4 c[kRowBatch];
#pragma unroll
        for (int b = 0; b < kRowBatch; ++b) c[b] = row(v0 + b);
#pragma unroll
        for (int b = 0; b < kRowBatch; ++b) tsum += (unsigned)(c[b].x + c[b].y + c[b].z + c[b].w);
    }
    const unsigned wtot = warp_sum(tsum);
    unsigned total;
    const unsigned wexcl = block_excl_scan<kThreads>(lane == 0 ? wtot : 0u, total, s_warp);
    const unsigned woff = __shfl_sync(0xffffffffu, wexcl, 0);
    SCAN_TRACE(1);
    if (threadIdx.x < 32) {
        unsigned pre = tile_prefix(ws.tile_cells, tile, epoch, total);
        if (threadIdx.x == 0) s_prefix = pre;
    } else if (full) {
        // while warp 0 looks back, the other warps clear the tile's scatter cursors
        // (they do not depend on the prefix)
        int4 *cz = reinterpret_cast<int4 *>(ws.cursor + tile * kCellTile);
        for (int q = (int)threadIdx.x - 32; q < kCellTile / 4; q += kThreads - 32) cz[q] = make_int4(0, 0, 0, 0);
    }
    __syncthreads();
    SCAN_TRACE(2);
    const unsigned prefix = s_prefix;
    // second pass: cell ranges; the histogram is re-zeroed (the next build's, or
    // the gather's key carry-over, accumulates into it), the scatter's cursors too
    unsigned run = prefix + woff;                    // first slot of this warp's current row
    constexpr int kWB = 4;
#pragma unroll
    for (int v0 = 0; v0 < V; v0 += kWB) {
        int4 c[kWB];
#pragma unroll
        for (int b = 0; b < kWB; ++b) c[b] = row(v0 + b);
#pragma unroll
        for (int b = 0; b < kWB; ++b) {
            const int v = v0 + b;
            const unsigned sv = (unsigned)(c[b].x + c[b].y + c[b].z + c[b].w);
            unsigned inc = sv;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            int r = (int)(run + inc - sv);
            run += __shfl_sync(0xffffffffu, inc, 31);
            int4 st, en;
            st.x = r; r += c[b].x; en.x = r;
            st.y = r; r += c[b].y; en.y = r;
            st.z = r; r += c[b].z; en.z = r;
            st.w = r; r += c[b].w; en.w = r;
            if (full) {
                const long long q4 = (wbase >> 2) + 32 * v + lane;
                reinterpret_cast<int4 *>(cell_start)[q4] = st;
                reinterpret_cast<int4 *>(cell_end)[q4] = en;
                reinterpret_cast<int4 *>(ws.cell_count)[q4] = make_int4(0, 0, 0, 0);
            } else {
                const int s4[4] = {st.x, st.y, st.z, st.w}, e4[4] = {en.x, en.y, en.z, en.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const long long j = wbase + 4 * (32 * v + lane) + q;
                    if (j < nc) {
                        cell_start[j] = s4[q];
                        cell_end[j] = e4[q];
                        ws.cell_count[j] = 0;
                        ws.cursor[j] = 0;
                    }
                }
            }
        }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
        *n_out = (long long)(prefix + total);
        ctr->n_leave = 0;   // the leaver list of the next build starts here (pack-from-list ran before)
    }
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&ctr->done_cll, 1) == (int)gridDim.x - 1) {
            ctr->done_cll = 0;
            ctr->ticket_cll = 0;
            ctr->epoch_cll += 1;
        }
    }
    SCAN_TRACE(3);
}

// K2 for small grids (at most kClusterScanCells cells, C1-C3): one thread-block
// cluster scans the whole histogram.  CTA r of the cluster takes a fixed range of
// 32 warps x V rows x 128 cells in the warp-striped layout of k_cell_scan (row v
// of a warp's segment is int4 #(32 v + lane): every load / store instruction of a
// warp covers 512 contiguous bytes; all V rows of a pass are loaded before they
// are summed); the CTA totals are exchanged through distributed shared memory
// (each CTA reads the totals of the CTAs before it) — two cluster barriers
// instead of a look-back chain over tens of tiles, the latency that dominated K2
// at C2 / C3 in round 1 (~19 us).
constexpr int kClusterScanThreads = 1024;
constexpr int kClusterScanMaxV = 16;
constexpr long long kClusterScanCells = 16LL * kClusterScanThreads * 4 * kClusterScanMaxV;   // 1M (16 CTAs)

template <int V>
__global__ void __launch_bounds__(kClusterScanThreads) k_cell_scan_cluster(GridDev g, Workspace ws, int *cell_start,
                                                                           int *cell_end, long long *n_out,
                                                                           const long long *n_src)
{
    pdl_entry();
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    constexpr int NW = kClusterScanThreads / 32;
    constexpr int WCELLS = 32 * 4 * V;
    __shared__ unsigned s_warp[NW + 1];
    __shared__ unsigned s_total;
    Counters *ctr = ws.ctr;
    const int r = (int)cl.block_rank(), R = (int)cl.num_blocks();
    const long long nc = g.ncells;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long wbase = ((long long)r * NW + warp) * WCELLS;
    const bool full = wbase + WCELLS <= nc;
    if (n_src && r == 0 && threadIdx.x == 0) {
        ctr->n_in = *n_src;
        ctr->mig_base = *n_src;
    }
    const int4 *pc = reinterpret_cast<const int4 *>(ws.cell_count + wbase) + lane;
    auto row = [&](int v) -> int4 {
        if (full) return __ldcg(pc + 32 * v);
        int t[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const long long j = wbase + 4 * (32 * v + lane) + q;
            t[q] = j < nc ? __ldcg(ws.cell_count + j) : 0;
        }
        return make_int4(t[0], t[1], t[2], t[3]);
    };
    unsigned tsum = 0;
    {
        int4 c[V];
#pragma unroll
        for (int v = 0; v < V; ++v) c[v] = row(v);
#pragma unroll
        for (int v = 0; v < V; ++v) tsum += (unsigned)(c[v].x + c[v].y + c[v].z + c[v].w);
    }
    const unsigned wtot = warp_sum(tsum);
    unsigned total;
    const unsigned wexcl = block_excl_scan<kClusterScanThreads>(lane == 0 ? wtot : 0u, total, s_warp);
    const unsigned woff = __shfl_sync(0xffffffffu, wexcl, 0);
    if (threadIdx.x == 0) s_total = total;
    cl.sync();
    unsigned pre = 0;
    for (int q = 0; q < r; ++q) pre += *cl.map_shared_rank(&s_total, q);
    unsigned run = pre + woff;                       // first slot of this warp's current row
#pragma unroll
    for (int v = 0; v < V; ++v) {
        const int4 c = row(v);
        const unsigned sv = (unsigned)(c.x + c.y + c.z + c.w);
        unsigned inc = sv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        int rr = (int)(run + inc - sv);
        run += __shfl_sync(0xffffffffu, inc, 31);
        int4 st, en;
        st.x = rr; rr += c.x; en.x = rr;
        st.y = rr; rr += c.y; en.y = rr;
        st.z = rr; rr += c.z; en.z = rr;
        st.w = rr; rr += c.w; en.w = rr;
        if (full) {
            const long long q4 = (wbase >> 2) + 32 * v + lane;
            reinterpret_cast<int4 *>(cell_start)[q4] = st;
            reinterpret_cast<int4 *>(cell_end)[q4] = en;
            reinterpret_cast<int4 *>(ws.cell_count)[q4] = make_int4(0, 0, 0, 0);
            reinterpret_cast<int4 *>(ws.cursor)[q4] = make_int4(0, 0, 0, 0);
        } else {
            const int s4[4] = {st.x, st.y, st.z, st.w}, e4[4] = {en.x, en.y, en.z, en.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const long long j = wbase + 4 * (32 * v + lane) + q;
                if (j < nc) {
                    cell_start[j] = s4[q];
                    cell_end[j] = e4[q];
                    ws.cell_count[j] = 0;
                    ws.cursor[j] = 0;
                }
            }
        }
    }
    SPH_CHECK(run <= pre + total);
    if (r == R - 1 && threadIdx.x == 0) {
        *n_out = (long long)(pre + total);
        ctr->n_leave = 0;   // the leaver list of the next build starts here
    }
    cl.sync();              // no CTA leaves while another still reads its total
}

template <int V>
static cudaError_t cluster_scan_launch(int csize, const GridDev &g, const Workspace &ws, int *cs, int *ce,
                                       long long *n_out, const long long *n_src, cudaStream_t s)
{
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_cell_scan_cluster<V>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaGetLastError();
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(csize);
    cfg.blockDim = dim3(kClusterScanThreads);
    cfg.stream = s;
    cudaLaunchAttribute a[2];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = csize;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    a[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = a;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, k_cell_scan_cluster<V>, g, ws, cs, ce, n_out, n_src);
}

// Cluster size of the small-grid scan: 16 CTAs where the device allows it
// (non-portable size), else the portable 8; 0 = off (SPHBUF_CLUSTER_SCAN=0).
static int cluster_scan_size()
{
    static int size = -1;
    if (size >= 0) return size;
    const char *e = getenv("SPHBUF_CLUSTER_SCAN");
    if (e && e[0] == '0') return size = 0;
    size = 8;
    if (cudaFuncSetAttribute(k_cell_scan_cluster<kClusterScanMaxV>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                             1) == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(16);
        cfg.blockDim = dim3(kClusterScanThreads);
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = 16;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k_cell_scan_cluster<kClusterScanMaxV>, &cfg) == cudaSuccess && n >= 1)
            size = 16;
    }
    cudaGetLastError();
    return size;
}

// Launch the cluster scan if the grid is small enough; false: use the look-back scan.
static bool launch_cluster_scan(const GridDev &g, const Workspace &ws, int *cs, int *ce, long long *n_out,
                                const long long *n_src, cudaStream_t s)
{
    const int csize = cluster_scan_size();
    if (csize == 0) return false;
    const long long per_v = (long long)csize * kClusterScanThreads * 4;   // cells per row across the cluster
    const long long v = (g.ncells + per_v - 1) / per_v;
    if (v > kClusterScanMaxV) return false;
    if (v <= 1) cluster_scan_launch<1>(csize, g, ws, cs, ce, n_out, n_src, s);
    else if (v <= 2) cluster_scan_launch<2>(csize, g, ws, cs, ce, n_out, n_src, s);
    else if (v <= 4) cluster_scan_launch<4>(csize, g, ws, cs, ce, n_out, n_src, s);
    else if (v <= 8) cluster_scan_launch<8>(csize, g, ws, cs, ce, n_out, n_src, s);
    else cluster_scan_launch<16>(csize, g, ws, cs, ce, n_out, n_src, s);
    return true;
}

#ifdef SPHBUF_TRACE
}  // namespace sphbuf
extern "C" int sph_trace_scan(unsigned long long *host, int max_tiles, int reset)
{
    const int n = max_tiles < sphbuf::kTraceScan ? max_tiles : sphbuf::kTraceScan;
    cudaError_t e = cudaMemcpyFromSymbol(host, sphbuf::g_trace_scan, sizeof(unsigned long long) * 6 * n);
    if (reset) {
        static unsigned long long zero[sphbuf::kTraceScan][6];
        cudaMemcpyToSymbol(sphbuf::g_trace_scan, zero, sizeof(zero));
    }
    return (int)e;
}
namespace sphbuf {
#endif


// K3: source index of every sorted slot: slot = cell_start[key] + a per-cell
// cursor (one atomic per run of equal keys in a warp; the order inside a cell is
// arbitrary here, the gather ranks by id).  (Counting the histogram itself back
// down instead of zeroed cursors saves K2 two stores per cell but costs the
// scatter and the gather more than it saves: measured.)
// Blocks beyond `nscat` run the update prologue K5 instead (UpdPro): it needs only
// the cell tables K2 just wrote, so it overlaps the scatter and the gather.
// DYN (opt-in, SPHBUF_SCATTER=dyn): warp chunks of 32 x kScatterItems keys handed
// out by a ticket counter (fetched one chunk ahead; reset by the last block)
// instead of the static block stride.
template <int kScatterItems, int NT, int DYN = 0>
__global__ void __launch_bounds__(NT) k_cll_scatter(Workspace ws, const int *cell_start, int *perm, int nscat,
                                                    const int *cell_end, int pro_runs, int pro_max_ports)
{
    pdl_entry();
    if ((int)blockIdx.x >= nscat) {
        upd_prologue_body<NT>(ws, pro_runs, cell_start, cell_end, pro_max_ports, (int)gridDim.x - nscat);
        return;
    }
    const long long n = ws.ctr->n_in;
    if (blockIdx.x == 0 && threadIdx.x == 0) ws.ctr->ticket_gather = 0;   // the gather's tile tickets
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
    // the keys base + it * istride + tid, it < kScatterItems (uniform over the warp)
    auto chunk = [&](long long base, int istride, int tid) {
        int key[kScatterItems];
#pragma unroll
        for (int it = 0; it < kScatterItems; ++it) {
            const long long i = base + it * istride + tid;
            key[it] = i < n ? ws.key[i] : -1;
        }
        // lanes with equal keys grouped (match.any: a cell changer between two pieces
        // of a stayer run does not split the run's atomic), one cursor atomic per
        // distinct key of the warp, all items' atomics in flight together; the
        // lanes of a group take consecutive slots in lane order
        int b[kScatterItems], hl[kScatterItems], rl[kScatterItems];
#pragma unroll
        for (int it = 0; it < kScatterItems; ++it) {
            const unsigned grp = __match_any_sync(0xffffffffu, key[it]);
            hl[it] = __ffs(grp) - 1;
            rl[it] = __popc(grp & lt);
            b[it] = (hl[it] == lane && key[it] >= 0) ? atomicAdd(&ws.cursor[key[it]], __popc(grp)) : 0;
        }
#pragma unroll
        for (int it = 0; it < kScatterItems; ++it) {
            const int rk = __shfl_sync(0xffffffffu, b[it], hl[it]) + rl[it];
            const long long i = base + it * istride + tid;
            if (i >= n) continue;
            if (key[it] >= 0) {
                const int slot = __ldg(cell_start + key[it]) + rk;
                SPH_CHECK(slot < n);
                ws.src[slot] = (int)i;
            } else if (perm) {
                perm[i] = -1;                                     // tombstone: dropped
            }
        }
    };
    if (DYN == 2) {
        // block chunks of 4 rounds (4 x NT x kScatterItems keys) per ticket
        constexpr int R = 4;
        constexpr long long BC = (long long)NT * kScatterItems * R;
        const int nch = (int)((n + BC - 1) / BC);
        __shared__ int s_nx;
        int cur = (int)blockIdx.x, tk = 0;
        if (threadIdx.x == 0) tk = atomicAdd(&ws.ctr->ticket_scatter, 1);
        while (cur < nch) {
            if (threadIdx.x == 0) s_nx = nscat + tk;
            __syncthreads();
            const int nxt = s_nx;
            if (threadIdx.x == 0) tk = atomicAdd(&ws.ctr->ticket_scatter, 1);   // the chunk after the next one
#pragma unroll 1
            for (int r = 0; r < R; ++r) chunk(cur * BC + (long long)r * NT * kScatterItems, NT, (int)threadIdx.x);
            __syncthreads();
            cur = nxt;
        }
        if (threadIdx.x == 0 && atomicAdd(&ws.ctr->done_scatter, 1) == nscat - 1) {
            ws.ctr->ticket_scatter = 0;
            ws.ctr->done_scatter = 0;
        }
    } else if (DYN) {
        constexpr int WC = 32 * kScatterItems;
        const int nchunks = (int)((n + WC - 1) / WC);
        const int nwarps = nscat * (NT / 32);
        int cur = (int)blockIdx.x * (NT / 32) + (int)(threadIdx.x >> 5);
        int tk = 0;
        if (lane == 0) tk = atomicAdd(&ws.ctr->ticket_scatter, 1);
        while (cur < nchunks) {
            const int nxt = nwarps + __shfl_sync(0xffffffffu, tk, 0);
            if (lane == 0) tk = atomicAdd(&ws.ctr->ticket_scatter, 1);   // the chunk after the next one
            chunk((long long)cur * WC, 32, lane);
            cur = nxt;
        }
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(&ws.ctr->done_scatter, 1) == nscat - 1) {
            ws.ctr->ticket_scatter = 0;
            ws.ctr->done_scatter = 0;
        }
    } else {
        const long long stride = (long long)nscat * NT * kScatterItems;
        for (long long base = (long long)blockIdx.x * NT * kScatterItems; base < n; base += stride)
            chunk(base, NT, (int)threadIdx.x);
    }
}

constexpr int kHalo = 64;   // slots staged on either side of a gather tile

// acc + [a >= m] (unsigned): the carry of a - m, two instructions per element.
__device__ __forceinline__ unsigned add_ge(unsigned acc, unsigned a, unsigned m)
{
    asm("{\n\t.reg .u32 t;\n\tsub.cc.u32 t, %1, %2;\n\taddc.u32 %0, %0, 0;\n\t}" : "+r"(acc) : "r"(a), "r"(m));
    return acc;
}

// Rank by id of slot p (id me) among its cell's slots [cb, ce).  The ids of the
// slots [w0, w1) are in shared memory at sid[q - w0]; a cell reaching past them
// (more than kHalo slots outside the tile) reads the rest from global memory.
// narrow: every id of the window is below 2^32, and slo holds their low words.
__device__ __forceinline__ int rank_in_cell(const PartDev &in, const Workspace &ws, const long long *sid,
                                            const unsigned *slo, bool narrow, int w0, int w1, int cb, int ce,
                                            long long me)
{
    int r = 0;
    if (cb >= w0 && ce <= w1) {
        if (narrow) {
            // 8-byte pairs of low words over the range padded to even slots (the
            // staged window starts on an even slot), each compare folded into a
            // carry-add (count of ids >= me), the padding slots taken back out
            const unsigned *sc = slo - w0;
            const unsigned m32 = (unsigned)me;
            const int q0 = cb & ~1, q1 = (ce + 1) & ~1;
            if (q1 == q0) return 0;
            // the padding slots (cb - 1 when cb is odd, ce when ce is odd) are
            // replaced by ~0 in the first / last pair, so they count as >= me
            uint2 f = *reinterpret_cast<const uint2 *>(sc + q0);
            if (cb & 1) f.x = 0xffffffffu;
            if (q1 - q0 == 2 && (ce & 1)) f.y = 0xffffffffu;
            unsigned ge = add_ge(add_ge(0u, f.x, m32), f.y, m32);
            if (q1 - q0 > 2) {
#pragma unroll 2
                for (int q = q0 + 2; q < q1 - 2; q += 2) {
                    const uint2 v = *reinterpret_cast<const uint2 *>(sc + q);
                    ge = add_ge(ge, v.x, m32);
                    ge = add_ge(ge, v.y, m32);
                }
                uint2 l = *reinterpret_cast<const uint2 *>(sc + q1 - 2);
                if (ce & 1) l.y = 0xffffffffu;
                ge = add_ge(add_ge(ge, l.x, m32), l.y, m32);
            }
            return (q1 - q0) - (int)ge;
        }
        const long long *sc = sid - w0;
#pragma unroll 4
        for (int q = cb; q < ce; ++q) r += (sc[q] < me);
        return r;
    }
    for (int q = cb; q < ce; ++q) r += (((q >= w0 && q < w1) ? sid[q - w0] : in.id[ws.src[q]]) < me);
    return r;
}

// K4: one round of independent loads per output slot (all columns of the
// source); the (advected, when the build fused the driver's advection) position
// gives the cell again by the pinned formula of K1, hence the cell's slot range;
// the rank by id among the cell's slots comes from ids staged in shared memory —
// the tile's and kHalo slots on either side, so a cell straddling the tile edge
// is ranked from shared memory as well; the store goes to the sorted position.
// Loads are nearly sequential (only particles that changed cell come from far
// away); stores stay inside the cell.
// DIM, CARRY, PERM: compile-time specialisations of g.dim, carry and (perm !=
// nullptr) for the default variant (0 / -1 / -1: read at run time); a tile whose
// slots are all below n runs a body with no per-slot validity checks.
// DYN (the default of the 3-D carried-key build; SPHBUF_GATHER_SPEC=static for
// the block-stride order): tiles handed out by a ticket counter (reset by the
// scatter) instead of the static block stride, fetched two tiles ahead so the
// next tile's map prefetch keeps its place.  The resident blocks then always
// work on one contiguous window of the array and none is left with a tail:
// C5 updates 4-23, A/B on one box, identical checksum: 2.105 -> 1.913 ms.
template <bool HasExtra, int ITEMS, int MINB, int NT = kThreads, bool PF = false, int DIM = 0, int CARRY = -1,
          int PERM = -1, int DYN = 0>
__global__ void __launch_bounds__(NT, MINB) k_cll_gather(PartDev in, PartDev out, GridDev g, Workspace ws,
                                                               const int *cell_start, const int *cell_end, int *perm,
                                                               int advect, float dt, int carry_rt, float cdt)
{
    pdl_entry();
    constexpr int T = NT * ITEMS;
    static_assert(2 * kHalo <= NT, "one halo slot per thread");
    __shared__ long long s_id[kHalo + T + kHalo];
    __shared__ __align__(16) unsigned s_lo[kHalo + T + kHalo];
    // slot indices are int32 (capacity < 2^31, checked by sph_ctx_create): 32-bit
    // index arithmetic throughout
    const int n = (int)*out.n;
    const int dim = DIM ? DIM : g.dim;
    const int carry = CARRY >= 0 ? CARRY : carry_rt;
    const bool has_perm = PERM >= 0 ? PERM == 1 : perm != nullptr;
    // sources below mig_base are this slab's own particles (advected here when the
    // build fused the advection); received migrants were advected by their sender
    const int adv_lim = advect ? (int)ws.ctr->mig_base : 0;
    const int stride = (int)gridDim.x * T;
    int oob_next = 0;
    // PF: the slot -> source map of the next tile is loaded while this tile's
    // columns are in flight (one dependent DRAM round trip less per tile)
    int nsrc[ITEMS], nhsrc = 0;
    auto load_map = [&](int jb, int (&sv)[ITEMS], int &hs) {
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            const int j = jb + it * NT + (int)threadIdx.x;
            sv[it] = j < n ? ws.src[j] : -1;
        }
        const int jh = threadIdx.x < kHalo ? jb - kHalo + (int)threadIdx.x : jb + T + ((int)threadIdx.x - kHalo);
        hs = (threadIdx.x < 2 * kHalo && jh >= 0 && jh < n) ? ws.src[jh] : -1;
    };
    if (PF) load_map((int)blockIdx.x * T, nsrc, nhsrc);
    __shared__ int s_next;
    auto tile = [&](int j0, int jn, auto full_tag) {
        constexpr bool Full = decltype(full_tag)::value;      // every slot of the tile is below n
        int tk = 0;
        if (DYN && threadIdx.x == 0) tk = atomicAdd(&ws.ctr->ticket_gather, 1);   // the tile after the next one
        int src[ITEMS], cb[ITEMS], ce[ITEMS], lab[ITEMS];
        float x[ITEMS], y[ITEMS], z[ITEMS], vx[ITEMS], vy[ITEMS], vz[ITEMS];
        long long id[ITEMS];
        // halo ids (threads 0 .. 2 kHalo - 1): two dependent loads, issued first
        const int jh = threadIdx.x < kHalo ? j0 - kHalo + (int)threadIdx.x : j0 + T + ((int)threadIdx.x - kHalo);
        const bool hv = threadIdx.x < 2 * kHalo && jh >= 0 && jh < n;
        int hsrc;
        if (PF) {
            hsrc = nhsrc;
#pragma unroll
            for (int it = 0; it < ITEMS; ++it) src[it] = nsrc[it];
        } else {
            hsrc = hv ? ws.src[jh] : 0;
#pragma unroll
            for (int it = 0; it < ITEMS; ++it) {
                const int j = j0 + it * NT + (int)threadIdx.x;
                src[it] = (Full || j < n) ? ws.src[j] : -1;
            }
        }
        const long long hid = hv ? in.id[hsrc] : 0;
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            if (!Full && src[it] < 0) continue;
            const int s = src[it];
            x[it] = in.x[s];
            y[it] = in.y[s];
            vx[it] = in.vx[s];
            vy[it] = in.vy[s];
            z[it] = 0.0f;
            if (dim == 3) {
                z[it] = in.z[s];
                vz[it] = in.vz[s];
            }
            id[it] = in.id[s];
            lab[it] = in.label[s];
        }
        if (PF && jn < n) load_map(jn, nsrc, nhsrc);
        bool wide = hv && (hid >> 32) != 0;
        if (threadIdx.x < 2 * kHalo) {
            const int hq = threadIdx.x < kHalo ? threadIdx.x : T + threadIdx.x;
            s_id[hq] = hid;
            s_lo[hq] = (unsigned)hid;
        }
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            if (!Full && src[it] < 0) continue;
            if (src[it] < adv_lim) {
                x[it] = advect1(x[it], vx[it], dt);
                y[it] = advect1(y[it], vy[it], dt);
                if (dim == 3) z[it] = advect1(z[it], vz[it], dt);
            }
            int oob = 0;
            const int key = cell_of<DIM>(g, x[it], y[it], z[it], oob);
            cb[it] = __ldg(cell_start + key);
            ce[it] = __ldg(cell_end + key);
            s_id[kHalo + it * NT + threadIdx.x] = id[it];
            s_lo[kHalo + it * NT + threadIdx.x] = (unsigned)id[it];
            wide |= (id[it] >> 32) != 0;
        }
        // 32-bit compares when no id of the window needs its high word
        const bool narrow = !__syncthreads_or(wide);
        // slot indices fit in int32 (cell tables are int32); staged window [w0, w1)
        const int t0 = j0;
        const int w0 = t0 - kHalo > 0 ? t0 - kHalo : 0;
        const int w1 = t0 + T + kHalo < n ? t0 + T + kHalo : n;
        const long long *sid = s_id + (w0 - (t0 - kHalo));
        const unsigned *slo = s_lo + (w0 - (t0 - kHalo));
        int kn[ITEMS];
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            kn[it] = -1;
            if (!Full && src[it] < 0) continue;
            const long long me = id[it];
            const int d = cb[it] + rank_in_cell(in, ws, sid, slo, narrow, w0, w1, cb[it], ce[it], me);
            if (carry) {
                // key carry-over: the next build's key of the particle now at d (its
                // position advected again by cdt), so that build needs no key pass;
                // with slab migration a particle about to leave the slab is listed
                int oobn = 0;
                kn[it] = carry_key<DIM>(g, x[it], y[it], z[it], vx[it], vy[it], vz[it], cdt, carry, oobn);
                oob_next += oobn;
                ws.key[d] = kn[it];
                if (kn[it] == kLeaver) leaver_append(ws, d);
            }
            SPH_CHECK(d >= cb[it] && d < ce[it] && ce[it] <= n && src[it] < in.cap);
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
            out.id[d] = me;
            out.label[d] = lab[it];
            if (has_perm) perm[src[it]] = d;
        }
        if (carry) {
#pragma unroll
            for (int it = 0; it < ITEMS; ++it) hist_count_match(ws.cell_count, kn[it]);   // next histogram
        }
        // (every thread read s_next before this tile's first barrier)
        if (DYN && threadIdx.x == 0) s_next = (int)gridDim.x + tk;
        __syncthreads();
    };
    if (DYN) {
        const int ntiles = (n + T - 1) / T;
        if (threadIdx.x == 0) s_next = (int)gridDim.x + atomicAdd(&ws.ctr->ticket_gather, 1);
        __syncthreads();
        int cur = (int)blockIdx.x;
        while (cur < ntiles) {
            const int nxt = s_next;
            tile(cur * T, nxt < ntiles ? nxt * T : n, std::false_type{});
            cur = nxt;
        }
    } else {
        // (no int overflow past n)
        for (int j0 = (int)blockIdx.x * T; j0 < n; j0 = j0 < n - stride ? j0 + stride : n)
            tile(j0, j0 < n - stride ? j0 + stride : n, std::false_type{});
    }
    if (carry) {
        const unsigned o = warp_sum((unsigned)oob_next);
        if ((threadIdx.x & 31) == 0 && o) atomicAdd((unsigned long long *)&ws.ctr->out_of_grid, (unsigned long long)o);
    }
}

// K4 with warp-owned segments (opt-in, SPHBUF_GATHER_SPEC=wl; the 3-D, no-perm,
// no-extra-column case): each warp takes 64 consecutive slots at a time and
// stages the ids of 32 slots on either side itself, so a cell is ranked from the
// warp's own window after a __syncwarp — no block barrier, each warp's chain
// runs free of the slowest warp of its block.  Everything else is K4's.
template <int MINB, int CARRY>
__global__ void __launch_bounds__(kThreads, MINB) k_cll_gather_wl(PartDev in, PartDev out, GridDev g, Workspace ws,
                                                                  const int *cell_start, const int *cell_end,
                                                                  int advect, float dt, float cdt)
{
    pdl_entry();
    constexpr int NW = kThreads / 32, SEG = 64, H = 32, W = SEG + 2 * H;
    __shared__ long long s_id[NW][W];
    __shared__ __align__(16) unsigned s_lo[NW][W];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n = (int)*out.n;
    constexpr int carry = CARRY;
    const int adv_lim = advect ? (int)ws.ctr->mig_base : 0;
    const int stride = (int)gridDim.x * NW * SEG;
    int oob_next = 0;
    // slot map of a segment: this lane's two slots and its two halo slots (prefetched)
    int nsrc[2], nh[2];
    auto load_map = [&](int sb) {
#pragma unroll
        for (int it = 0; it < 2; ++it) {
            const int j = sb + it * 32 + lane;
            nsrc[it] = j < n ? ws.src[j] : -1;
            const int jh = it == 0 ? sb - H + lane : sb + SEG + lane;
            nh[it] = (jh >= 0 && jh < n) ? ws.src[jh] : -1;
        }
    };
    int seg = ((int)blockIdx.x * NW + warp) * SEG;
    if (seg < n) load_map(seg);
    for (; seg < n; seg = seg < n - stride ? seg + stride : n) {
        int src[2], hs[2], cb[2], ce[2], lab[2];
        float x[2], y[2], z[2], vx[2], vy[2], vz[2];
        long long id[2], hid[2];
#pragma unroll
        for (int it = 0; it < 2; ++it) {
            src[it] = nsrc[it];
            hs[it] = nh[it];
        }
#pragma unroll
        for (int it = 0; it < 2; ++it) hid[it] = hs[it] >= 0 ? in.id[hs[it]] : 0;
#pragma unroll
        for (int it = 0; it < 2; ++it) {
            if (src[it] < 0) continue;
            const int s = src[it];
            x[it] = in.x[s];
            y[it] = in.y[s];
            z[it] = in.z[s];
            vx[it] = in.vx[s];
            vy[it] = in.vy[s];
            vz[it] = in.vz[s];
            id[it] = in.id[s];
            lab[it] = in.label[s];
        }
        if (seg < n - stride) load_map(seg + stride);
        bool wide = false;
#pragma unroll
        for (int it = 0; it < 2; ++it) {
            const int hq = it == 0 ? lane : H + SEG + lane;
            s_id[warp][hq] = hid[it];
            s_lo[warp][hq] = (unsigned)hid[it];
            wide |= (hid[it] >> 32) != 0;
        }
#pragma unroll
        for (int it = 0; it < 2; ++it) {
            cb[it] = ce[it] = 0;
            if (src[it] < 0) continue;
            if (src[it] < adv_lim) {
                x[it] = advect1(x[it], vx[it], dt);
                y[it] = advect1(y[it], vy[it], dt);
                z[it] = advect1(z[it], vz[it], dt);
            }
            int oob = 0;
            const int key = cell_of<3>(g, x[it], y[it], z[it], oob);
            cb[it] = __ldg(cell_start + key);
            ce[it] = __ldg(cell_end + key);
            s_id[warp][H + it * 32 + lane] = id[it];
            s_lo[warp][H + it * 32 + lane] = (unsigned)id[it];
            wide |= (id[it] >> 32) != 0;
        }
        const bool narrow = !__any_sync(0xffffffffu, wide);    // (also the warp's barrier)
        __syncwarp();
        const int w0 = seg - H > 0 ? seg - H : 0;               // even: seg is a multiple of 64
        const int w1 = seg + SEG + H < n ? seg + SEG + H : n;
        const long long *sid = &s_id[warp][0] + (w0 - (seg - H));
        const unsigned *slo = &s_lo[warp][0] + (w0 - (seg - H));
        int kn[2];
#pragma unroll
        for (int it = 0; it < 2; ++it) {
            kn[it] = -1;
            if (src[it] < 0) continue;
            const long long me = id[it];
            const int d = cb[it] + rank_in_cell(in, ws, sid, slo, narrow, w0, w1, cb[it], ce[it], me);
            if (carry) {
                int oobn = 0;
                kn[it] = carry_key<3>(g, x[it], y[it], z[it], vx[it], vy[it], vz[it], cdt, carry, oobn);
                oob_next += oobn;
                ws.key[d] = kn[it];
                if (kn[it] == kLeaver) leaver_append(ws, d);
            }
            SPH_CHECK(d >= cb[it] && d < ce[it] && ce[it] <= n && src[it] < in.cap);
            out.x[d] = x[it];
            out.y[d] = y[it];
            out.z[d] = z[it];
            out.vx[d] = vx[it];
            out.vy[d] = vy[it];
            out.vz[d] = vz[it];
            out.id[d] = me;
            out.label[d] = lab[it];
        }
        if (carry) {
#pragma unroll
            for (int it = 0; it < 2; ++it) hist_count_match(ws.cell_count, kn[it]);   // next histogram
        }
        __syncwarp();   // the window is rewritten by the next segment
    }
    if (carry) {
        const unsigned o = warp_sum((unsigned)oob_next);
        if (lane == 0 && o) atomicAdd((unsigned long long *)&ws.ctr->out_of_grid, (unsigned long long)o);
    }
}

// K4 on the copy engine (opt-in, SPHBUF_GATHER_TMA=1: correct and bit-identical,
// but slower than k_cll_gather on C5 — 3.2 vs 2.1 ms, DESIGN.md §6 — because the
// stages' shared memory leaves one block of <= 32 warps per SM for a per-tile
// dependency chain that k_cll_gather hides behind 40).  The sources of a tile of T slots lie
// mostly in one window of the input (a particle that keeps its cell, or moves to
// the next cell along z, lands near where it was; measured on C5: ~90% of the
// sources inside [j0 + drift - 64, j0 + T + drift + 64), drift = the median of
// (source - slot) over 32 samples of the tile's slot map, tools/map_window_stats.py).
// One producer warp per block estimates each tile's drift and brings that window
// of every column into one of S shared-memory stages with cp.async.bulk, running
// up to S tiles ahead.  The consumer warps (G groups of T/2 threads, 2 slots
// each, taking the block's tiles in turn) fetch the other sources (cell changers
// in x and y) of their NEXT tile into the stage's far area with cp.async, as soon
// as its window is known; the stage's mbarrier completes when both the window
// copies and those far copies have landed, so a tile finds every source in shared
// memory and no DRAM round trip is left on the consumers' path.  The rest — the
// advection, the cell range, the rank by id among the cell's slots, the stores,
// the carried-over key — is K4's, unchanged, with a named barrier per group
// instead of the block barrier.  Results are bit-identical to k_cll_gather (the
// same values reach the same arithmetic).
template <int DIM, int T, int G, int S>
struct GtmaCfg {
    static constexpr int NCG = T / 2;                       // consumer threads per group, 2 slots each
    static constexpr int NT = G * NCG + 32;                 // + the producer warp
    static constexpr int H = 64;                            // window margin (elements) on either side
    static constexpr int W = T + 2 * H;                     // elements copied per column
    static constexpr int WP = W + 8;                        // column stride in a stage (16-byte multiple)
    static constexpr int FC = T / 4;                        // far-area entries per stage (overflow: plain loads)
    static constexpr int NF = 2 * DIM;                      // fp32 columns
    static constexpr int BPE = 4 * NF + 8 + 4;              // bytes per element (floats, id, label)
    static constexpr size_t win_bytes = (size_t)WP * BPE;
    static constexpr size_t stage_bytes = win_bytes + (size_t)FC * BPE;
    static constexpr int RW = T + 2 * kHalo;                // ranking window (slots)
    static constexpr size_t rank_bytes = (size_t)RW * 12;   // ids + their low words
    static constexpr size_t smem = S * stage_bytes + (size_t)G * 2 * rank_bytes;
    static_assert(W % 4 == 0 && (WP * 4) % 16 == 0 && (FC * 4) % 16 == 0 && stage_bytes % 16 == 0 &&
                      rank_bytes % 16 == 0, "alignment");
    static_assert(2 * kHalo <= NCG && NCG % 32 == 0 && S >= 3 * G, "shape: far copies two group tiles ahead");
};

// Group-wide OR over a named barrier (bar.red): also the group's barrier.
__device__ __forceinline__ bool named_bar_or(int id, int n, bool p)
{
    int r;
    asm volatile(
        "{\n\t.reg .pred pi, po;\n\t"
        "setp.ne.s32 pi, %1, 0;\n\t"
        "bar.red.or.pred po, %2, %3, pi;\n\t"
        "selp.s32 %0, 1, 0, po;\n}"
        : "=r"(r)
        : "r"((int)p), "r"(id), "r"(n)
        : "memory");
    return r != 0;
}

template <int BYTES>
__device__ __forceinline__ void cp_async_g2s(void *dst, const void *src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(BYTES) : "memory");
}

// The mbarrier's pending count drops when this thread's earlier cp.async copies land.
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t *bar)
{
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void st_release_cta(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.cta.shared::cta.u64 [%0], %1;" ::"r"(smem_u32(p)), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_cta(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.cta.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}

template <int DIM, int T, int G, int S, int CARRY>
__global__ void __launch_bounds__(GtmaCfg<DIM, T, G, S>::NT, 1)
    k_cll_gather_tma(PartDev in, PartDev out, GridDev g, Workspace ws, const int *cell_start, const int *cell_end,
                     int advect, float dt, float cdt)
{
    using C = GtmaCfg<DIM, T, G, S>;
    constexpr int NCG = C::NCG;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t full[S], empty[S];
    __shared__ unsigned long long s_win[S];   // (tile sequence << 32) | window start, published by the producer
    __shared__ int s_fcnt[S];                 // far-area entries taken in each stage
    pdl_entry();
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1 + NCG);     // the producer's expect_tx + one cp.async arrival per consumer
            mbar_init(&empty[s], NCG / 32);
            s_win[s] = ~0ull;
            s_fcnt[s] = 0;
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int n = (int)*out.n;
    const int capf = (int)(in.cap & ~3LL);                  // windows stay inside the columns' capacity
    const int ntiles = (n + T - 1) / T;
    const int nk = (int)blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int lane = threadIdx.x & 31;
    // stage s: window columns [id][f0..f_{NF-1}][label] (WP each), then the far area (FC each)
    auto win_id = [&](int s) { return reinterpret_cast<long long *>(smem + s * C::stage_bytes); };
    auto win_f = [&](int s, int c) {
        return reinterpret_cast<float *>(smem + s * C::stage_bytes + C::WP * 8 + c * C::WP * 4);
    };
    auto win_lab = [&](int s) {
        return reinterpret_cast<int *>(smem + s * C::stage_bytes + C::WP * (8 + 4 * C::NF));
    };
    auto far_id = [&](int s) { return reinterpret_cast<long long *>(smem + s * C::stage_bytes + C::win_bytes); };
    auto far_f = [&](int s, int c) {
        return reinterpret_cast<float *>(smem + s * C::stage_bytes + C::win_bytes + C::FC * 8 + c * C::FC * 4);
    };
    auto far_lab = [&](int s) {
        return reinterpret_cast<int *>(smem + s * C::stage_bytes + C::win_bytes + C::FC * (8 + 4 * C::NF));
    };
    if ((int)threadIdx.x >= G * NCG) {
        // ---- producer warp.  The 32 map samples of tile k are loaded D tiles ahead
        // (a register ring, static indices through the unrolled inner loop).
        constexpr int D = 4;
        int pre[D];
        auto sample = [&](int k) {
            const int js = ((int)blockIdx.x + k * (int)gridDim.x) * T + lane * (T / 32);
            return (k < nk && js < n) ? ws.src[js] - js : 0;
        };
#pragma unroll
        for (int u = 0; u < D; ++u) pre[u] = sample(u);
        for (int k0 = 0; k0 < nk; k0 += D)
#pragma unroll
            for (int u = 0; u < D; ++u) {
                const int k = k0 + u;
                if (k >= nk) break;
                const int s = k % S;
                const int j0 = ((int)blockIdx.x + k * (int)gridDim.x) * T;
                // drift: the median of (source - slot) over the 32 samples
                const int dl = pre[u];
                pre[u] = sample(k + D);
                int below = 0, eq = 0;
#pragma unroll 8
                for (int l = 0; l < 32; ++l) {
                    const int o = __shfl_sync(0xffffffffu, dl, l);
                    below += o < dl;
                    eq += (o == dl) & (l < lane);
                }
                const unsigned med = __ballot_sync(0xffffffffu, below + eq == 16);
                const int drift = __shfl_sync(0xffffffffu, dl, __ffs(med) - 1);
                long long a = (long long)j0 - C::H + drift;
                if (a > capf - C::W) a = capf - C::W;
                if (a < 0) a = 0;
                const int a4 = (int)a & ~3;
                const int b4 = a4 + C::W < capf ? a4 + C::W : capf;
                if (lane == 0) {
                    if (k >= S) mbar_wait(&empty[s], ((k / S) - 1) & 1);
                    const unsigned ne = (unsigned)(b4 - a4);
                    mbar_arrive_expect_tx(&full[s], ne * (unsigned)C::BPE);
                    if (ne) {
                        bulk_g2s(win_id(s), in.id + a4, ne * 8u, &full[s]);
                        bulk_g2s(win_f(s, 0), in.x + a4, ne * 4u, &full[s]);
                        bulk_g2s(win_f(s, 1), in.y + a4, ne * 4u, &full[s]);
                        if (DIM == 3) {
                            bulk_g2s(win_f(s, 2), in.z + a4, ne * 4u, &full[s]);
                            bulk_g2s(win_f(s, 3), in.vx + a4, ne * 4u, &full[s]);
                            bulk_g2s(win_f(s, 4), in.vy + a4, ne * 4u, &full[s]);
                            bulk_g2s(win_f(s, 5), in.vz + a4, ne * 4u, &full[s]);
                        } else {
                            bulk_g2s(win_f(s, 2), in.vx + a4, ne * 4u, &full[s]);
                            bulk_g2s(win_f(s, 3), in.vy + a4, ne * 4u, &full[s]);
                        }
                        bulk_g2s(win_lab(s), in.label + a4, ne * 4u, &full[s]);
                    }
                    st_release_cta(&s_win[s], ((unsigned long long)k << 32) | (unsigned)a4);
                }
                __syncwarp();
            }
        return;
    }
    // ---- consumers: group gi takes the block's tiles gi, gi + G, ...
    const int gi = (int)threadIdx.x / NCG, tg = (int)threadIdx.x % NCG;
    const int carry = CARRY;
    const int adv_lim = advect ? (int)ws.ctr->mig_base : 0;
    int oob_next = 0;
    auto tile_j0 = [&](int k) { return ((int)blockIdx.x + k * (int)gridDim.x) * T; };
    // slot map of a tile: this thread's two slots and (threads < 2 kHalo) one halo slot
    auto load_map = [&](int k, int (&sv)[3]) {
        const int jb = tile_j0(k);
#pragma unroll
        for (int it = 0; it < 2; ++it) {
            const int j = jb + it * NCG + tg;
            sv[it] = (k < nk && j < n) ? ws.src[j] : -1;
        }
        const int jh = tg < kHalo ? jb - kHalo + tg : jb + T + (tg - kHalo);
        sv[2] = (k < nk && tg < 2 * kHalo && jh >= 0 && jh < n) ? ws.src[jh] : -1;
    };
    // far prefetch of tile k (its window published): sources outside the window go
    // to the stage's far area by cp.async; fi = far index, -1 window (or none), -2
    // far area full (loaded at the tile); then this thread's arrival on full[s]
    auto prefetch = [&](int k, const int (&sv)[3], int (&fi)[3]) {
        const int s = k % S;
        unsigned long long w;
        while (true) {
            w = ld_acquire_cta(&s_win[s]);
            if ((unsigned)(w >> 32) == (unsigned)k) break;
        }
        const int a4 = (int)(unsigned)w;
        const int b4 = a4 + C::W < capf ? a4 + C::W : capf;
        bool far[3];
#pragma unroll
        for (int it = 0; it < 3; ++it) far[it] = sv[it] >= 0 && !(sv[it] >= a4 && sv[it] < b4);
        const unsigned m0 = __ballot_sync(0xffffffffu, far[0]), m1 = __ballot_sync(0xffffffffu, far[1]),
                       m2 = __ballot_sync(0xffffffffu, far[2]);
        const int tot = __popc(m0) + __popc(m1) + __popc(m2);
        int base = 0;
        if (lane == 0 && tot) base = atomicAdd(&s_fcnt[s], tot);
        base = __shfl_sync(0xffffffffu, base, 0);
        const unsigned lt = lanemask_lt();
        const int off[3] = {__popc(m0 & lt), __popc(m0) + __popc(m1 & lt), __popc(m0) + __popc(m1) + __popc(m2 & lt)};
#pragma unroll
        for (int it = 0; it < 3; ++it) {
            fi[it] = -1;
            if (!far[it]) continue;
            const int e = base + off[it];
            if (e >= C::FC) {
                fi[it] = -2;
                continue;
            }
            fi[it] = e;
            const int q = sv[it];
            cp_async_g2s<8>(far_id(s) + e, in.id + q);
            if (it == 2) continue;                                // halo slots: the id only
            cp_async_g2s<4>(far_f(s, 0) + e, in.x + q);
            cp_async_g2s<4>(far_f(s, 1) + e, in.y + q);
            if (DIM == 3) {
                cp_async_g2s<4>(far_f(s, 2) + e, in.z + q);
                cp_async_g2s<4>(far_f(s, 3) + e, in.vx + q);
                cp_async_g2s<4>(far_f(s, 4) + e, in.vy + q);
                cp_async_g2s<4>(far_f(s, 5) + e, in.vz + q);
            } else {
                cp_async_g2s<4>(far_f(s, 2) + e, in.vx + q);
                cp_async_g2s<4>(far_f(s, 3) + e, in.vy + q);
            }
            cp_async_g2s<4>(far_lab(s) + e, in.label + q);
        }
        cp_async_arrive_noinc(&full[s]);
        return a4;
    };
    // this group's tiles k (being processed), k + G (far copies in flight), k + 2G
    // (map loaded): the far copies of k + 2G are issued at the end of tile k
    int cur[3], nxt[3], nn[3], fi[3], nfi[3];
    int a_cur = 0, a_nxt = 0;
    if (gi < nk) {
        load_map(gi, cur);
        load_map(gi + G, nxt);
        load_map(gi + 2 * G, nn);
        a_cur = prefetch(gi, cur, fi);
        if (gi + G < nk) a_nxt = prefetch(gi + G, nxt, nfi);
    }
    int par = 0;
    for (int k = gi; k < nk; k += G, par ^= 1) {
        const int s = k % S;
        const int j0 = tile_j0(k);
        const int src[2] = {cur[0], cur[1]};
        const int hsrc = cur[2];
        const int fic[3] = {fi[0], fi[1], fi[2]};
        const int a4 = a_cur;
        float x[2], y[2], z[2], vx[2], vy[2], vz[2];
        long long id[2];
        int lab[2];
        long long hid = 0;
        mbar_wait(&full[s], (k / S) & 1);
        if (tg == 0) s_fcnt[s] = 0;                               // (all of this tile's far slots are taken)
#pragma unroll
        for (int it = 0; it < 2; ++it) {
            const int q = src[it];
            z[it] = vz[it] = 0.0f;
            if (q < 0) continue;
            if (fic[it] == -1) {
                const int r = q - a4;
                x[it] = win_f(s, 0)[r];
                y[it] = win_f(s, 1)[r];
                if (DIM == 3) {
                    z[it] = win_f(s, 2)[r];
                    vx[it] = win_f(s, 3)[r];
                    vy[it] = win_f(s, 4)[r];
                    vz[it] = win_f(s, 5)[r];
                } else {
                    vx[it] = win_f(s, 2)[r];
                    vy[it] = win_f(s, 3)[r];
                }
                id[it] = win_id(s)[r];
                lab[it] = win_lab(s)[r];
            } else if (fic[it] >= 0) {
                const int e = fic[it];
                x[it] = far_f(s, 0)[e];
                y[it] = far_f(s, 1)[e];
                if (DIM == 3) {
                    z[it] = far_f(s, 2)[e];
                    vx[it] = far_f(s, 3)[e];
                    vy[it] = far_f(s, 4)[e];
                    vz[it] = far_f(s, 5)[e];
                } else {
                    vx[it] = far_f(s, 2)[e];
                    vy[it] = far_f(s, 3)[e];
                }
                id[it] = far_id(s)[e];
                lab[it] = far_lab(s)[e];
            } else {
                x[it] = in.x[q];
                y[it] = in.y[q];
                vx[it] = in.vx[q];
                vy[it] = in.vy[q];
                if (DIM == 3) {
                    z[it] = in.z[q];
                    vz[it] = in.vz[q];
                }
                id[it] = in.id[q];
                lab[it] = in.label[q];
            }
        }
        if (hsrc >= 0) hid = fic[2] == -1 ? win_id(s)[hsrc - a4] : fic[2] >= 0 ? far_id(s)[fic[2]] : in.id[hsrc];
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);                // the stage goes back to the producer
        // ---- K4's body: advection, cell range, rank by id, stores, carried key
        unsigned char *rb = smem + S * C::stage_bytes + (size_t)(gi * 2 + par) * C::rank_bytes;
        long long *s_id = reinterpret_cast<long long *>(rb);
        unsigned *s_lo = reinterpret_cast<unsigned *>(rb + C::RW * 8);
        bool wide = hsrc >= 0 && (hid >> 32) != 0;
        if (tg < 2 * kHalo) {
            const int hq = tg < kHalo ? tg : T + tg;
            s_id[hq] = hid;
            s_lo[hq] = (unsigned)hid;
        }
        int cb[2], ce[2];
#pragma unroll
        for (int it = 0; it < 2; ++it) {
            cb[it] = ce[it] = 0;
            if (src[it] < 0) continue;
            if (src[it] < adv_lim) {
                x[it] = advect1(x[it], vx[it], dt);
                y[it] = advect1(y[it], vy[it], dt);
                if (DIM == 3) z[it] = advect1(z[it], vz[it], dt);
            }
            int oob = 0;
            const int key = cell_of<DIM>(g, x[it], y[it], z[it], oob);
            cb[it] = __ldg(cell_start + key);
            ce[it] = __ldg(cell_end + key);
            s_id[kHalo + it * NCG + tg] = id[it];
            s_lo[kHalo + it * NCG + tg] = (unsigned)id[it];
            wide |= (id[it] >> 32) != 0;
        }
        const bool narrow = !named_bar_or(1 + gi, NCG, wide);
        const int w0 = j0 - kHalo > 0 ? j0 - kHalo : 0;
        const int w1 = j0 + T + kHalo < n ? j0 + T + kHalo : n;
        const long long *sid = s_id + (w0 - (j0 - kHalo));
        const unsigned *slo = s_lo + (w0 - (j0 - kHalo));
        int kn[2];
#pragma unroll
        for (int it = 0; it < 2; ++it) {
            kn[it] = -1;
            if (src[it] < 0) continue;
            const long long me = id[it];
            const int d = cb[it] + rank_in_cell(in, ws, sid, slo, narrow, w0, w1, cb[it], ce[it], me);
            if (carry) {
                int oobn = 0;
                kn[it] = carry_key<DIM>(g, x[it], y[it], z[it], vx[it], vy[it], vz[it], cdt, carry, oobn);
                oob_next += oobn;
                ws.key[d] = kn[it];
                if (kn[it] == kLeaver) leaver_append(ws, d);
            }
            SPH_CHECK(d >= cb[it] && d < ce[it] && ce[it] <= n && src[it] < in.cap);
            out.x[d] = x[it];
            out.y[d] = y[it];
            out.vx[d] = vx[it];
            out.vy[d] = vy[it];
            if (DIM == 3) {
                out.z[d] = z[it];
                out.vz[d] = vz[it];
            }
            out.id[d] = me;
            out.label[d] = lab[it];
        }
        if (carry) {
#pragma unroll
            for (int it = 0; it < 2; ++it) hist_count_runs(ws.cell_count, kn[it]);   // next histogram
        }
        // rotate: k + G becomes current; the far copies of k + 2G go out now
        int a2 = 0, f2[3] = {-1, -1, -1};
        if (k + 2 * G < nk) a2 = prefetch(k + 2 * G, nn, f2);
#pragma unroll
        for (int it = 0; it < 3; ++it) {
            cur[it] = nxt[it];
            fi[it] = nfi[it];
            nxt[it] = nn[it];
            nfi[it] = f2[it];
        }
        a_cur = a_nxt;
        a_nxt = a2;
        if (k + 3 * G < nk) load_map(k + 3 * G, nn);
    }
    if (carry) {
        const unsigned o = warp_sum((unsigned)oob_next);
        if (lane == 0 && o) atomicAdd((unsigned long long *)&ws.ctr->out_of_grid, (unsigned long long)o);
    }
}

// ------------------------------------------------------------------ launchers

template <int I, int NT, int DYN = 0>
static void scatter_launch(const Workspace &ws, const int *cell_start, const int *cell_end, int *perm, long long cap,
                           const UpdPro &up, cudaStream_t s)
{
    static int grid = 0;
    if (!grid) grid = occ_grid(k_cll_scatter<I, NT, DYN>, NT);
    const int nscat = cap_grid(grid, cap, NT * I);
    const int npro = up.n_runs > 0 ? (up.n_runs + NT - 1) / NT : 0;
    launch_k(k_cll_scatter<I, NT, DYN>, dim3(nscat + npro), dim3(NT), 0, s, ws, cell_start, perm, nscat, cell_end,
             up.n_runs, up.max_ports);
}

// Gather variants (template instances), chosen by SPHBUF_GATHER=<slots>:<min blocks>
// for tuning runs (tools/gather_sweep.py); the default is the measured best.
template <bool HasExtra, int ITEMS, int MINB, int NT = kThreads, bool PF = false>
static void gather_fused(const PartDev &in, const PartDev &out, const GridDev &g, const Workspace &ws,
                         const int *cs, const int *ce, int *perm, int advect, float dt, int carry, float cdt,
                         long long cap, cudaStream_t s)
{
    static int grid = 0;
    if (!grid) grid = occ_grid(k_cll_gather<HasExtra, ITEMS, MINB, NT, PF>, NT);
    launch_k(k_cll_gather<HasExtra, ITEMS, MINB, NT, PF>, dim3(cap_grid(grid, cap, NT * ITEMS)), dim3(NT), 0, s, in, out, g, ws, cs, ce,
             perm, advect, dt, carry, cdt);
}

template <int DIM, int T, int G, int S, int CARRY>
static void gather_tma_launch(const PartDev &in, const PartDev &out, const GridDev &g, const Workspace &ws,
                              const int *cs, const int *ce, int advect, float dt, float cdt, long long cap,
                              cudaStream_t s)
{
    using C = GtmaCfg<DIM, T, G, S>;
    static bool init = false;
    if (!init) {
        cudaFuncSetAttribute(k_cll_gather_tma<DIM, T, G, S, CARRY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)C::smem);
        init = true;
    }
    launch_k(k_cll_gather_tma<DIM, T, G, S, CARRY>, dim3(cap_grid(sm_count_cached(), cap, T)), dim3(C::NT), C::smem,
             s, in, out, g, ws, cs, ce, advect, dt, cdt);
}

template <int T, int G, int S>
static void gather_tma_dispatch(const PartDev &in, const PartDev &out, const GridDev &g, const Workspace &ws,
                                const int *cs, const int *ce, int advect, float dt, int carry, float cdt,
                                long long cap, cudaStream_t s)
{
    if (g.dim == 3) {
        if (carry == 1) gather_tma_launch<3, T, G, S, 1>(in, out, g, ws, cs, ce, advect, dt, cdt, cap, s);
        else if (carry == 2) gather_tma_launch<3, T, G, S, 2>(in, out, g, ws, cs, ce, advect, dt, cdt, cap, s);
        else gather_tma_launch<3, T, G, S, 0>(in, out, g, ws, cs, ce, advect, dt, cdt, cap, s);
    } else {
        if (carry == 1) gather_tma_launch<2, T, G, S, 1>(in, out, g, ws, cs, ce, advect, dt, cdt, cap, s);
        else if (carry == 2) gather_tma_launch<2, T, G, S, 2>(in, out, g, ws, cs, ce, advect, dt, cdt, cap, s);
        else gather_tma_launch<2, T, G, S, 0>(in, out, g, ws, cs, ce, advect, dt, cdt, cap, s);
    }
}

// The copy-engine gather (opt-in: measured slower than k_cll_gather on C5, DESIGN.md
// §6) applies to builds without extra columns or a perm output whose columns are
// 16-byte aligned (cp.async.bulk); SPHBUF_GATHER_TMA=1 selects it, =<T>:<G>:<S> a
// tuning variant (3-D, carried keys).
static bool try_gather_tma(const PartDev &in, const PartDev &out, const GridDev &g, const Workspace &ws,
                           const int *cs, const int *ce, int *perm, int advect, float dt, int carry, float cdt,
                           long long cap, cudaStream_t s)
{
    static const char *v = getenv("SPHBUF_GATHER_TMA");
    if (!v || !*v || !strcmp(v, "0")) return false;
    if (in.n_extra > 0 || perm) return false;
    auto al = [](const void *p) { return ((uintptr_t)p & 15) == 0; };
    if (!al(in.x) || !al(in.y) || !al(in.vx) || !al(in.vy) || !al(in.id) || !al(in.label)) return false;
    if (g.dim == 3 && (!al(in.z) || !al(in.vz))) return false;
    if (strcmp(v, "1") && g.dim == 3 && carry == 1) {
#define SPH_GT(name, T, G, S)                                                                   \
    if (!strcmp(v, name)) {                                                                     \
        gather_tma_launch<3, T, G, S, 1>(in, out, g, ws, cs, ce, advect, dt, cdt, cap, s);      \
        return true;                                                                            \
    }
        SPH_GT("1024:1:3", 1024, 1, 3)
        SPH_GT("512:2:6", 512, 2, 6)
        SPH_GT("512:1:3", 512, 1, 3)
        SPH_GT("512:1:4", 512, 1, 4)
        SPH_GT("256:3:9", 256, 3, 9)
        SPH_GT("256:2:6", 256, 2, 6)
#undef SPH_GT
    }
    gather_tma_dispatch<512, 2, 6>(in, out, g, ws, cs, ce, advect, dt, carry, cdt, cap, s);
    return true;
}

template <bool HasExtra>
static void gather_variant(const char *v, const PartDev &in, const PartDev &out, const GridDev &g,
                           const Workspace &ws, const int *cs, const int *ce, int *perm, int advect, float dt,
                           int carry, float cdt, long long cap, cudaStream_t s)
{
#define SPH_GV(name, I, M)                                                              \
    if (!strcmp(v, name)) {                                                             \
        gather_fused<HasExtra, I, M>(in, out, g, ws, cs, ce, perm, advect, dt, carry, cdt, cap, s); \
        return;                                                                         \
    }
    SPH_GV("1:8", 1, 8)
    SPH_GV("2:6", 2, 6)
    SPH_GV("3:4", 3, 4)
    SPH_GV("4:3", 4, 3)
    if (!strcmp(v, "pf3:4")) return gather_fused<HasExtra, 3, 4, kThreads, true>(in, out, g, ws, cs, ce, perm, advect, dt, carry, cdt, cap, s);
#undef SPH_GV
    // default: 2 slots per thread, the next tile's slot map prefetched, <= 48
    // registers (5 blocks/SM): measured best on C5 among the variants above,
    // 128- / 512-thread blocks and cp.async / warp-chunk designs;
    // the 3-D, carried-key, no-perm build (the bench's) compiled for its case
    if (!HasExtra && g.dim == 3 && !perm && carry == 1 && !getenv("SPHBUF_GATHER_GENERIC")) {
        static const char *sv = getenv("SPHBUF_GATHER_SPEC");
        const char *v = sv ? sv : "";
#define SPH_GS(name, I, M)                                                                                       \
    if (!strcmp(v, name)) {                                                                                      \
        static int grid = 0;                                                                                     \
        if (!grid) grid = occ_grid(k_cll_gather<false, I, M, kThreads, true, 3, 1, 0>, kThreads);                \
        launch_k(k_cll_gather<false, I, M, kThreads, true, 3, 1, 0>, dim3(cap_grid(grid, cap, kThreads * I)),    \
                 dim3(kThreads), 0, s, in, out, g, ws, cs, ce, perm, advect, dt, carry, cdt);                     \
        return;                                                                                                  \
    }
        SPH_GS("2:6", 2, 6)
        SPH_GS("2:4", 2, 4)
        SPH_GS("3:4", 3, 4)
        SPH_GS("3:3", 3, 3)
        SPH_GS("static", 2, 5)
#undef SPH_GS
#define SPH_GW(name, M)                                                                                          \
    if (!strcmp(v, name)) {                                                                                      \
        static int grid = 0;                                                                                     \
        if (!grid) grid = occ_grid(k_cll_gather_wl<M, 1>, kThreads);                                             \
        launch_k(k_cll_gather_wl<M, 1>, dim3(cap_grid(grid, cap, kThreads * 2)), dim3(kThreads), 0, s, in, out, g, \
                 ws, cs, ce, advect, dt, cdt);                                                                   \
        return;                                                                                                  \
    }
        SPH_GW("wl", 5)
        SPH_GW("wl4", 4)
        SPH_GW("wl6", 6)
#undef SPH_GW

        static int grid = 0;
        if (!grid) grid = occ_grid(k_cll_gather<false, 2, 5, kThreads, true, 3, 1, 0, 1>, kThreads);
        launch_k(k_cll_gather<false, 2, 5, kThreads, true, 3, 1, 0, 1>, dim3(cap_grid(grid, cap, kThreads * 2)),
                 dim3(kThreads), 0, s, in, out, g, ws, cs, ce, perm, advect, dt, carry, cdt);
        return;
    }
    gather_fused<HasExtra, 2, 5, kThreads, true>(in, out, g, ws, cs, ce, perm, advect, dt, carry, cdt, cap, s);
}

static void launch_gather(const PartDev &in, const PartDev &out, const GridDev &g, const Workspace &ws,
                          const int *cs, const int *ce, int *perm, int advect, float dt, int carry, float cdt,
                          long long cap, cudaStream_t s)
{
    static const char *v = nullptr;
    if (!v) {
        v = getenv("SPHBUF_GATHER");
        if (!v) v = "";
    }
    if (!*v && try_gather_tma(in, out, g, ws, cs, ce, perm, advect, dt, carry, cdt, cap, s)) return;
    if (in.n_extra > 0) gather_variant<true>(v, in, out, g, ws, cs, ce, perm, advect, dt, carry, cdt, cap, s);
    else gather_variant<false>(v, in, out, g, ws, cs, ce, perm, advect, dt, carry, cdt, cap, s);
}

int sm_count() { return sm_count_cached(); }


template <bool A, bool M>
static void key_launch(const PartDev &in, const GridDev &g, const Workspace &ws, float dt, float *lo, float *hi,
                       long long maxm, int rec, cudaStream_t s)
{
    static int grid = 0;
    if (!grid) grid = occ_grid(k_cll_key<A, M>, kThreads);
    launch_k(k_cll_key<A, M>, dim3(cap_grid(grid, in.cap, kThreads * kKeyItems)), dim3(kThreads), 0, s, in, g, ws, dt, lo, hi, maxm,
                                                                                        rec);
}

cudaError_t launch_cll_key(const PartDev &in, const GridDev &g, const Workspace &ws, float dt, bool advect,
                           float *send_lo, float *send_hi, long long maxm, int rec, const CllCarry &cc, cudaStream_t s,
                           Launch *L)
{
    if (cc.use && !(send_lo && send_hi)) return cudaSuccess;   // the scan records the input count
    if (cc.use) {
        cudaError_t e = cudaMemsetAsync(send_lo, 0, 16, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(send_hi, 0, 16, s);
        if (e != cudaSuccess) return e;
        L->before(s);
        launch_k(k_mig_pack_list, dim3(cap_grid(sm_count_cached() * 2, ws.max_leave, kThreads)), dim3(kThreads), 0, s,
                 in, g, ws, dt, send_lo, send_hi, maxm, rec);
        L->after(s, KID_CLL_KEY);
        return cudaGetLastError();
    }
    if (cc.clear) {
        // the previous gather left a carried-over histogram this build does not use
        cudaError_t e = cudaMemsetAsync(ws.cell_count, 0, sizeof(int) * (size_t)g.ncells, s);
        if (e != cudaSuccess) return e;
    }
    const bool mig = send_lo && send_hi;
    if (mig) {
        cudaError_t e = cudaMemsetAsync(send_lo, 0, 16, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(send_hi, 0, 16, s);
        if (e != cudaSuccess) return e;
    }
    L->before(s);
    if (advect && mig) key_launch<true, true>(in, g, ws, dt, send_lo, send_hi, maxm, rec, s);
    else if (advect) key_launch<true, false>(in, g, ws, dt, nullptr, nullptr, 0, rec, s);
    else if (mig) key_launch<false, true>(in, g, ws, 0.0f, send_lo, send_hi, maxm, rec, s);
    else key_launch<false, false>(in, g, ws, 0.0f, nullptr, nullptr, 0, rec, s);
    L->after(s, KID_CLL_KEY);
    return cudaGetLastError();
}

cudaError_t launch_cll(const PartDev &in, const PartDev &out, const GridDev &g, const Workspace &ws, int *cell_start,
                       int *cell_end, int *perm, float dt, bool advect, const CllCarry &cc, const UpdPro &up,
                       cudaStream_t s, Launch *L)
{
    cudaError_t e = launch_cll_key(in, g, ws, dt, advect, nullptr, nullptr, 0, 0, cc, s, L);
    if (e != cudaSuccess) return e;
    return launch_cll_finish(in, out, g, ws, nullptr, nullptr, 0, 0, cell_start, cell_end, perm, advect, dt, cc, up, s,
                             L);
}

cudaError_t launch_cll_finish(const PartDev &in, const PartDev &out, const GridDev &g, const Workspace &ws,
                              const float *recv_lo, const float *recv_hi, long long maxm, int rec, int *cell_start,
                              int *cell_end, int *perm, bool advect_b, float dt, const CllCarry &cc,
                              const UpdPro &up, cudaStream_t s, Launch *L)
{
    const int advect = advect_b ? 1 : 0;
    // cells per thread of K2: 32 (many small tiles) unless that takes more than
    // one wave of resident blocks, then 128
    const bool big = g.ncells > kScanBigCells;
    const long long ntiles = (g.ncells + (big ? kCellTileBig : kCellTile) - 1) / (big ? kCellTileBig : kCellTile);
    const long long cap = in.cap;
    if (recv_lo || recv_hi) {
        L->before(s);
        launch_k(k_cll_unpack_key, dim3(cap_grid(sm_count_cached() * 2, maxm * 2, kThreads)), dim3(kThreads), 0, s, 
            in, g, ws, recv_lo, recv_hi, maxm, rec);
        L->after(s, KID_MIG_UNPACK);
    }
    L->before(s);
    const bool no_key_pass = cc.use && !cc.mig;
    if (launch_cluster_scan(g, ws, cell_start, cell_end, out.n,
                            no_key_pass ? (const long long *)in.n : (const long long *)nullptr, s)) {
    } else if (big)
        launch_k(k_cell_scan<kCellItemsBig>, dim3((unsigned)ntiles), dim3(kThreads), 0, s, g, ws, cell_start,
                 cell_end, out.n, ntiles, no_key_pass ? (const long long *)in.n : (const long long *)nullptr);
    else
        launch_k(k_cell_scan<kCellItems>, dim3((unsigned)(ntiles > 0 ? ntiles : 1)), dim3(kThreads), 0, s, g, ws,
                 cell_start, cell_end, out.n, ntiles, no_key_pass ? (const long long *)in.n : (const long long *)nullptr);
    L->after(s, KID_CELL_SCAN);
    {
        // scatter variants for tuning (SPHBUF_SCATTER=<items>:<threads>); default 4 x 256,
        // measured best on C5 among 1-16 items x 128-512 threads
        static const char *sv = getenv("SPHBUF_SCATTER");
        const char *v = sv ? sv : "";
        L->before(s);
        if (!strcmp(v, "8:256")) scatter_launch<8, 256>(ws, cell_start, cell_end, perm, cap, up, s);
        else if (!strcmp(v, "2:256")) scatter_launch<2, 256>(ws, cell_start, cell_end, perm, cap, up, s);
        else if (!strcmp(v, "1:256")) scatter_launch<1, 256>(ws, cell_start, cell_end, perm, cap, up, s);
        else if (!strcmp(v, "2:512")) scatter_launch<2, 512>(ws, cell_start, cell_end, perm, cap, up, s);
        else if (!strcmp(v, "dyn")) scatter_launch<4, 256, 1>(ws, cell_start, cell_end, perm, cap, up, s);
        else if (!strcmp(v, "dynb")) scatter_launch<4, 256, 2>(ws, cell_start, cell_end, perm, cap, up, s);
        else if (!strcmp(v, "dyn2")) scatter_launch<2, 256, 1>(ws, cell_start, cell_end, perm, cap, up, s);
        else if (!strcmp(v, "dyn8")) scatter_launch<8, 256, 1>(ws, cell_start, cell_end, perm, cap, up, s);
        else scatter_launch<4, 256>(ws, cell_start, cell_end, perm, cap, up, s);
        L->after(s, KID_CLL_SCATTER);
    }
    L->before(s);
    launch_gather(in, out, g, ws, cell_start, cell_end, perm, advect, dt, cc.make ? (cc.mig ? 2 : 1) : 0, cc.dt, cap,
                  s);
    L->after(s, KID_CLL_GATHER);
    return cudaGetLastError();
}

}  // namespace sphbuf
