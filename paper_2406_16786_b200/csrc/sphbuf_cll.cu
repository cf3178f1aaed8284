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
            hist_count_runs(ws.cell_count, key[it]);     // one atomic per run of equal keys
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
template <int kScatterItems, int NT>
__global__ void __launch_bounds__(NT) k_cll_scatter(Workspace ws, const int *cell_start, int *perm, int nscat,
                                                    const int *cell_end, int pro_runs, int pro_max_ports)
{
    pdl_entry();
    if ((int)blockIdx.x >= nscat) {
        upd_prologue_body<NT>(ws, pro_runs, cell_start, cell_end, pro_max_ports, (int)gridDim.x - nscat);
        return;
    }
    const long long n = ws.ctr->n_in;
    const long long stride = (long long)nscat * NT * kScatterItems;
    for (long long base = (long long)blockIdx.x * NT * kScatterItems; base < n; base += stride) {
        int key[kScatterItems];
#pragma unroll
        for (int it = 0; it < kScatterItems; ++it) {
            const long long i = base + it * NT + threadIdx.x;
            key[it] = i < n ? ws.key[i] : -1;
        }
        // run heads of all items first, then all their atomics in flight together
        const int lane = threadIdx.x & 31;
        const unsigned le = lanemask_lt() | (1u << lane);
        int b[kScatterItems], hl[kScatterItems];
#pragma unroll
        for (int it = 0; it < kScatterItems; ++it) {
            const int prev = __shfl_up_sync(0xffffffffu, key[it], 1);
            const bool head = (lane == 0) || (key[it] != prev);
            const unsigned heads = __ballot_sync(0xffffffffu, head);
            const unsigned above = heads & ~le;
            const int next = above ? __ffs(above) - 1 : 32;
            hl[it] = 31 - __clz(heads & le);
            b[it] = (head && key[it] >= 0) ? atomicAdd(&ws.cursor[key[it]], next - lane) : 0;
        }
#pragma unroll
        for (int it = 0; it < kScatterItems; ++it) {
            const int rk = __shfl_sync(0xffffffffu, b[it], hl[it]) + lane - hl[it];
            const long long i = base + it * NT + threadIdx.x;
            if (i >= n) continue;
            if (key[it] >= 0) {
                const int slot = __ldg(cell_start + key[it]) + rk;
                SPH_CHECK(slot < n);
                ws.src[slot] = (int)i;
            } else if (perm) {
                perm[i] = -1;                                     // tombstone: dropped
            }
        }
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
template <bool HasExtra, int ITEMS, int MINB, int NT = kThreads, bool PF = false, int DIM = 0, int CARRY = -1,
          int PERM = -1>
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
    auto tile = [&](int j0, auto full_tag) {
        constexpr bool Full = decltype(full_tag)::value;      // every slot of the tile is below n
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
        if (PF && j0 < n - stride) load_map(j0 + stride, nsrc, nhsrc);   // (no int overflow past n)
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
            for (int it = 0; it < ITEMS; ++it) hist_count_runs(ws.cell_count, kn[it]);   // next histogram
        }
        __syncthreads();
    };
    for (int j0 = (int)blockIdx.x * T; j0 < n; j0 = j0 < n - stride ? j0 + stride : n) tile(j0, std::false_type{});
    if (carry) {
        const unsigned o = warp_sum((unsigned)oob_next);
        if ((threadIdx.x & 31) == 0 && o) atomicAdd((unsigned long long *)&ws.ctr->out_of_grid, (unsigned long long)o);
    }
}

// ------------------------------------------------------------------ launchers

template <int I, int NT>
static void scatter_launch(const Workspace &ws, const int *cell_start, const int *cell_end, int *perm, long long cap,
                           const UpdPro &up, cudaStream_t s)
{
    static int grid = 0;
    if (!grid) grid = occ_grid(k_cll_scatter<I, NT>, NT);
    const int nscat = cap_grid(grid, cap, NT * I);
    const int npro = up.n_runs > 0 ? (up.n_runs + NT - 1) / NT : 0;
    launch_k(k_cll_scatter<I, NT>, dim3(nscat + npro), dim3(NT), 0, s, ws, cell_start, perm, nscat, cell_end,
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
#undef SPH_GS

        static int grid = 0;
        if (!grid) grid = occ_grid(k_cll_gather<false, 2, 5, kThreads, true, 3, 1, 0>, kThreads);
        launch_k(k_cll_gather<false, 2, 5, kThreads, true, 3, 1, 0>, dim3(cap_grid(grid, cap, kThreads * 2)),
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
