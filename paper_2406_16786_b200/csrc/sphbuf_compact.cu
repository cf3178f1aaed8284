// sphbuf_compact.cu — ID assignment + stable in-place compaction (SURVEY §8(a) row
// a7; north star: "removed by a scan-based stream compaction with an
// ID/permutation remap").  Only the suffix [i_first, N) after the lowest deleted
// index moves.
//   K7a k_compact_count  from the update's list of deleted positions (when at most
//                        kDelList): per-range shared-memory counts, no label pass;
//                        else labels only: per 8192-element tile the number of
//                        tombstones, decoupled look-back scan over tiles, and the
//                        exclusive tombstone count before every 1024-element
//                        sub-tile (sub_off);
//   K7b k_compact_move   every sub-tile loads all of its columns into registers,
//                        publishes "read done", waits only for the few preceding
//                        sub-tiles whose input its output range overlaps (outputs
//                        move down by at most D), then stores its survivors at
//                        i - (tombstones before i).  No tile waits on a prefix
//                        chain, so all sub-tiles stream concurrently;
//   K7c k_compact_append staged particles after the survivors with IDs from the
//                        (allgathered) count matrix, N and next_id.
#include <climits>
#include <cstdint>

#include "sphbuf_common.cuh"
#include "sphbuf_tma.cuh"

namespace sphbuf {

constexpr int kCntSub = kCntTile / kCmpTile;        // sub-tiles per count tile (8)
constexpr int kCntItems = kCntTile / kThreads;      // labels per thread (32)
static_assert(kCntSub == kThreads / 32, "one warp per compaction sub-tile");

// First element the compaction touches: i_first rounded down to a count tile,
// so label loads are 16-byte aligned (elements in [begin, i_first) are alive and
// are rewritten onto themselves).
__device__ __forceinline__ long long cmp_begin(long long i_first) { return (i_first / kCntTile) * kCntTile; }

// K7a with the update's list of deleted positions (K6; complete when at most
// kDelList): each block takes a range of kCntRange sub-tiles, counts the listed
// positions below the range and, in shared memory, per sub-tile inside it, and
// scans — no pass over the suffix's labels, no sort.  Otherwise the label pass.
constexpr int kCntRange = 4096;

__global__ void __launch_bounds__(kThreads) k_compact_count(PartDev p, Workspace ws, const long long *next_id,
                                                            int dlist_max)
{
    pdl_entry();
    __shared__ unsigned s_sub[kCntSub][kThreads / 32];
    __shared__ unsigned s_tot[kCntSub + 1];
    __shared__ long long s_tile;
    __shared__ unsigned s_prefix;
    Counters *ctr = ws.ctr;
    const long long N = *p.n;
    const long long D = ctr->n_del;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctr->cmp_n = N;
        ctr->cmp_next_id = *next_id;
    }
    if (D == 0) return;
    const long long ibeg = cmp_begin(ctr->i_first);
    const long long DL = ctr->n_dlist;
    if (DL == D && D <= dlist_max) {
        __shared__ unsigned s_c[kCntRange];
        __shared__ unsigned s_below;
        __shared__ unsigned s_scan[kThreads / 32 + 1];
        const long long nsub = (N - ibeg + kCmpTile - 1) / kCmpTile;
        for (long long u0 = (long long)blockIdx.x * kCntRange; u0 < nsub; u0 += (long long)gridDim.x * kCntRange) {
            for (int i = threadIdx.x; i < kCntRange; i += blockDim.x) s_c[i] = 0;
            if (threadIdx.x == 0) s_below = 0;
            __syncthreads();
            const long long lo = ibeg + u0 * kCmpTile, hi = lo + (long long)kCntRange * kCmpTile;
            unsigned below = 0;
            for (int q = threadIdx.x; q < (int)D; q += blockDim.x) {
                const long long pos = __ldg(ws.del_list + q);
                if (pos < lo) ++below;
                else if (pos < hi) atomicAdd(&s_c[(pos - lo) / kCmpTile], 1u);
            }
            below = warp_sum(below);
            if ((threadIdx.x & 31) == 0 && below) atomicAdd(&s_below, below);
            __syncthreads();
            // exclusive scan of the range's counts, kCntRange / kThreads per thread
            constexpr int PER = kCntRange / kThreads;
            unsigned loc[PER], sum = 0;
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                loc[e] = s_c[threadIdx.x * PER + e];
                sum += loc[e];
            }
            unsigned tot;
            unsigned run = block_excl_scan<kThreads>(sum, tot, s_scan) + s_below;
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                const long long u = u0 + threadIdx.x * PER + e;
                if (u < nsub) ws.sub_off[u] = run;
                run += loc[e];
            }
            __syncthreads();
        }
        return;
    }
    const unsigned epoch = ctr->epoch_cmp;
    const long long ntiles = (N - ibeg + kCntTile - 1) / kCntTile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    while (true) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->ticket_cmp, 1);
        __syncthreads();
        const long long tile = s_tile;
        if (tile >= ntiles) break;
        // warp w counts exactly sub-tile w (1024 labels) of the compaction move;
        // lane l reads int4 #(32 v + l) of it, so each load covers 512 contiguous bytes
        const long long wb = ibeg + tile * kCntTile + (long long)warp * (32 * kCntItems);
        unsigned c = 0;
        if (wb + 32 * kCntItems <= N) {
            const int4 *q = reinterpret_cast<const int4 *>(p.label + wb) + lane;
#pragma unroll
            for (int v = 0; v < kCntItems / 4; ++v) {
                const int4 a = q[32 * v];
                c += (a.x <= -2) + (a.y <= -2) + (a.z <= -2) + (a.w <= -2);
            }
        } else {
            for (int v = 0; v < kCntItems / 4; ++v)
                for (int j = 0; j < 4; ++j) {
                    const long long i = wb + 4 * (32 * v + lane) + j;
                    if (i < N) c += (p.label[i] <= -2);
                }
        }
        c = warp_sum(c);
        if (lane == 0) s_sub[0][warp] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned run = 0;
            for (int sub = 0; sub < kCntSub; ++sub) {
                s_tot[sub] = run;
                run += s_sub[0][sub];
            }
            s_tot[kCntSub] = run;
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const unsigned pre = tile_prefix(ws.tile_cmp, tile, epoch, s_tot[kCntSub]);
            if (threadIdx.x == 0) s_prefix = pre;
        }
        __syncthreads();
        if (threadIdx.x < kCntSub) ws.sub_off[tile * kCntSub + threadIdx.x] = s_prefix + s_tot[threadIdx.x];
        __syncthreads();
    }
}

#ifdef SPHBUF_TRACE
// K7b sub-tile timeline (tools/upd_trace.py --move): ticket, loads + scan done,
// predecessor wait done, end, block, SM.
constexpr int kTraceMove = 1 << 17;
__device__ unsigned long long g_trace_mv[kTraceMove][6];
__device__ __forceinline__ unsigned long long gtimer3()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define MV_TRACE(slot) MV_TRACE_U(u, slot)
#define MV_TRACE_U(uu, slot)                                                                \
    do {                                                                                    \
        if (threadIdx.x == 0 && (uu) < kTraceMove) {                                       \
            g_trace_mv[(uu)][slot] = gtimer3();                                             \
            if ((slot) == 0) {                                                              \
                unsigned smid_;                                                             \
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));                          \
                g_trace_mv[(uu)][4] = blockIdx.x;                                           \
                g_trace_mv[(uu)][5] = smid_;                                                \
            }                                                                               \
        }                                                                                   \
    } while (0)
#else
#define MV_TRACE(slot) \
    do {               \
    } while (0)
#define MV_TRACE_U(uu, slot) \
    do {                     \
    } while (0)
#endif

template <bool HasExtra>
__global__ void __launch_bounds__(kThreads) k_compact_move(PartDev p, int dim, Workspace ws, int *perm, int carry)
{
    pdl_entry();
    __shared__ unsigned s_cnt[kCmpItems * kThreads / 32 + 1];
    __shared__ long long s_tile;
    __shared__ volatile int s_sink;
    Counters *ctr = ws.ctr;
    const long long D = ctr->n_del;
    if (D == 0) return;
    const long long N = ctr->cmp_n;
    const long long ibeg = cmp_begin(ctr->i_first);
    const unsigned epoch = ctr->epoch_cmp;
    const long long nsub = (N - ibeg + kCmpTile - 1) / kCmpTile;
    int dep = 0;
    while (true) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->ticket_cmp2, 1);
        __syncthreads();
        const long long u = s_tile;
        if (u >= nsub) break;
        MV_TRACE(0);
#ifdef SPHBUF_TRACE
        if (threadIdx.x == 0 && u < kTraceMove) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            g_trace_mv[u][4] = blockIdx.x;
            g_trace_mv[u][5] = smid;
        }
#endif
        bool alive[kCmpItems];
        float x[kCmpItems], y[kCmpItems], z[kCmpItems], vx[kCmpItems], vy[kCmpItems], vz[kCmpItems];
        float ex[kCmpItems][SPH_MAX_EXTRA];
        long long id[kCmpItems];
        int lab[kCmpItems], kc[kCmpItems];
        unsigned mine = 0;
#pragma unroll
        for (int it = 0; it < kCmpItems; ++it) {
            const long long i = ibeg + u * kCmpTile + it * kThreads + threadIdx.x;
            alive[it] = false;
            if (i < N) {
                lab[it] = p.label[i];
                kc[it] = carry ? ws.key[i] : 0;   // key carry-over: the next-build key moves along
                x[it] = p.x[i];
                y[it] = p.y[i];
                vx[it] = p.vx[i];
                vy[it] = p.vy[i];
                if (dim == 3) {
                    z[it] = p.z[i];
                    vz[it] = p.vz[i];
                } else {
                    z[it] = vz[it] = 0.0f;
                }
                if (HasExtra) {
#pragma unroll
                    for (int e = 0; e < SPH_MAX_EXTRA; ++e) ex[it][e] = (e < p.n_extra) ? p.extra[e][i] : 0.0f;
                }
                id[it] = p.id[i];
                alive[it] = lab[it] > -2;
                mine += alive[it];
                // consume every loaded word so the loads are complete before "read done"
                dep ^= kc[it] ^ __float_as_int(x[it]) ^ __float_as_int(y[it]) ^ __float_as_int(z[it]) ^
                       __float_as_int(vx[it]) ^ __float_as_int(vy[it]) ^ __float_as_int(vz[it]) ^ (int)id[it] ^
                       (int)(id[it] >> 32);
                if (HasExtra) {
#pragma unroll
                    for (int e = 0; e < SPH_MAX_EXTRA; ++e) dep ^= __float_as_int(ex[it][e]);
                }
            }
        }
        // every loaded word is consumed here, before the block barrier in the scan:
        // the loads have returned before "read done" is published (a volatile
        // shared-memory store of the XOR is an instruction that needs all of them)
        s_sink = dep;
        unsigned excl[kCmpItems], total;
        striped_scan<kThreads, kCmpItems>(alive, excl, total, s_cnt);   // contains __syncthreads
        MV_TRACE(1);
        const long long start = ibeg + u * kCmpTile;
        const long long dst0 = start - (long long)ws.sub_off[u];
        if (threadIdx.x < 32) {
            // every load of this sub-tile has returned (its values were consumed
            // above and the block barrier passed), so a relaxed store suffices: no
            // fence waiting for the previous sub-tile's stores
            if (threadIdx.x == 0)
                asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(ws.rd + u), "r"(epoch) : "memory");
            // wait only for the earlier sub-tiles whose input overlaps the output range
            // [dst0, dst0 + alive) (when the shift exceeds a sub-tile these are a few
            // tiles back, claimed long ago); acquire polling (no full fence), the block
            // barrier below orders the other threads' stores after it
            if (total > 0 && dst0 < start) {
                const long long vlo = (dst0 - ibeg) / kCmpTile;
                long long vhi = (dst0 + total - 1 - ibeg) / kCmpTile;
                if (vhi > u - 1) vhi = u - 1;
                for (long long v = vlo + threadIdx.x; v <= vhi; v += 32) {
                    unsigned f;
                    do {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(ws.rd + v) : "memory");
                    } while (f != epoch);
                }
            }
            __syncwarp();
        }
        __syncthreads();
        MV_TRACE(2);
#pragma unroll
        for (int it = 0; it < kCmpItems; ++it) {
            const long long i = start + it * kThreads + threadIdx.x;
            if (i >= N) continue;
            if (!alive[it]) {
                if (perm) perm[i] = -1;
                continue;
            }
            const long long o = dst0 + excl[it];
            p.x[o] = x[it];
            p.y[o] = y[it];
            p.vx[o] = vx[it];
            p.vy[o] = vy[it];
            if (dim == 3) {
                p.z[o] = z[it];
                p.vz[o] = vz[it];
            }
            if (HasExtra)
                for (int e = 0; e < p.n_extra; ++e) p.extra[e][o] = ex[it][e];
            p.id[o] = id[it];
            p.label[o] = lab[it];
            if (carry) ws.key[o] = kc[it];
            if (perm) perm[i] = (int)o;
        }
        MV_TRACE(3);
        __syncthreads();
    }
}

#ifdef SPHBUF_TRACE
}  // namespace sphbuf
extern "C" int sph_trace_move(unsigned long long *host, int max_tiles, int reset)
{
    const int n = max_tiles < sphbuf::kTraceMove ? max_tiles : sphbuf::kTraceMove;
    cudaError_t e = cudaMemcpyFromSymbol(host, sphbuf::g_trace_mv, sizeof(unsigned long long) * 6 * n);
    if (reset) {
        static unsigned long long zero[sphbuf::kTraceMove][6];
        cudaMemcpyToSymbol(sphbuf::g_trace_mv, zero, sizeof(zero));
    }
    return (int)e;
}
namespace sphbuf {
#endif

// K7b, two sub-tiles per block in flight (no extra columns): the next sub-tile's
// loads are issued before waiting for the current one's predecessors, so that
// wait (their load-time variance) overlaps memory work instead of idling the
// block.  Progress: a block publishes "read done" for a sub-tile as soon as its
// loads returned and waits only on smaller sub-tiles; the smallest sub-tile any
// block is storing has all predecessors published.
struct MoveTile {
    float x[kCmpItems], y[kCmpItems], z[kCmpItems], vx[kCmpItems], vy[kCmpItems], vz[kCmpItems];
    long long id[kCmpItems];
    int lab[kCmpItems], kc[kCmpItems];
};

__device__ __forceinline__ void move_load(const PartDev &p, int dim, const Workspace &ws, int carry, long long base,
                                          long long N, MoveTile &t)
{
#pragma unroll
    for (int it = 0; it < kCmpItems; ++it) {
        const long long i = base + it * kThreads + threadIdx.x;
        t.lab[it] = -3;
        t.kc[it] = 0;
        t.x[it] = t.y[it] = t.z[it] = t.vx[it] = t.vy[it] = t.vz[it] = 0.0f;
        t.id[it] = 0;
        if (i < N) {
            t.lab[it] = p.label[i];
            t.kc[it] = carry ? ws.key[i] : 0;
            t.x[it] = p.x[i];
            t.y[it] = p.y[i];
            t.vx[it] = p.vx[i];
            t.vy[it] = p.vy[i];
            if (dim == 3) {
                t.z[it] = p.z[i];
                t.vz[it] = p.vz[i];
            } else {
                t.z[it] = t.vz[it] = 0.0f;
            }
            t.id[it] = p.id[i];
        }
    }
}

// Consume every loaded word (so the loads have returned), rank the survivors.
__device__ __forceinline__ void move_rank(const MoveTile &t, unsigned (&excl)[kCmpItems], bool (&alive)[kCmpItems],
                                          unsigned &total, unsigned *s_cnt, volatile int *s_sink)
{
    int dep = 0;
#pragma unroll
    for (int it = 0; it < kCmpItems; ++it) {
        alive[it] = t.lab[it] > -2;
        dep ^= t.lab[it] ^ t.kc[it] ^ __float_as_int(t.x[it]) ^ __float_as_int(t.y[it]) ^ __float_as_int(t.z[it]) ^
               __float_as_int(t.vx[it]) ^ __float_as_int(t.vy[it]) ^ __float_as_int(t.vz[it]) ^ (int)t.id[it] ^
               (int)(t.id[it] >> 32);
    }
    *s_sink = dep;
    striped_scan<kThreads, kCmpItems>(alive, excl, total, s_cnt);   // contains __syncthreads
}

__global__ void __launch_bounds__(kThreads) k_compact_move2(PartDev p, int dim, Workspace ws, int *perm, int carry)
{
    pdl_entry();
    __shared__ unsigned s_cnt[kCmpItems * kThreads / 32 + 1];
    __shared__ long long s_tile;
    __shared__ volatile int s_sink;
    Counters *ctr = ws.ctr;
    const long long D = ctr->n_del;
    if (D == 0) return;
    const long long N = ctr->cmp_n;
    const long long ibeg = cmp_begin(ctr->i_first);
    const unsigned epoch = ctr->epoch_cmp;
    const long long nsub = (N - ibeg + kCmpTile - 1) / kCmpTile;
    auto ticket = [&]() -> long long {
        if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->ticket_cmp2, 1);
        __syncthreads();
        const long long t = s_tile;
        __syncthreads();
        return t;
    };
    auto publish = [&](long long u) {
        if (threadIdx.x == 0)
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(ws.rd + u), "r"(epoch) : "memory");
    };
    MoveTile A, B;
    unsigned exA[kCmpItems], exB[kCmpItems], totA, totB;
    bool alA[kCmpItems], alB[kCmpItems];
    long long u = ticket();
    if (u >= nsub) return;
    MV_TRACE_U(u, 0);
    move_load(p, dim, ws, carry, ibeg + u * kCmpTile, N, A);
    move_rank(A, exA, alA, totA, s_cnt, &s_sink);
    publish(u);
    MV_TRACE_U(u, 1);
    while (true) {
        // the next sub-tile's loads go out first ...
        const long long u2 = ticket();
        const bool more = u2 < nsub;
        if (more) MV_TRACE_U(u2, 0);
        if (more) move_load(p, dim, ws, carry, ibeg + u2 * kCmpTile, N, B);
        // ... then wait for the earlier sub-tiles whose input this output overlaps
        const long long start = ibeg + u * kCmpTile;
        const long long dst0 = start - (long long)ws.sub_off[u];
        if (threadIdx.x < 32) {
            if (totA > 0 && dst0 < start) {
                const long long vlo = (dst0 - ibeg) / kCmpTile;
                long long vhi = (dst0 + totA - 1 - ibeg) / kCmpTile;
                if (vhi > u - 1) vhi = u - 1;
                for (long long v = vlo + threadIdx.x; v <= vhi; v += 32) {
                    unsigned f;
                    do {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(ws.rd + v) : "memory");
                    } while (f != epoch);
                }
            }
            __syncwarp();
        }
        __syncthreads();
        MV_TRACE_U(u, 2);
#pragma unroll
        for (int it = 0; it < kCmpItems; ++it) {
            const long long i = start + it * kThreads + threadIdx.x;
            if (i >= N) continue;
            if (!alA[it]) {
                if (perm) perm[i] = -1;
                continue;
            }
            const long long o = dst0 + exA[it];
            p.x[o] = A.x[it];
            p.y[o] = A.y[it];
            p.vx[o] = A.vx[it];
            p.vy[o] = A.vy[it];
            if (dim == 3) {
                p.z[o] = A.z[it];
                p.vz[o] = A.vz[it];
            }
            p.id[o] = A.id[it];
            p.label[o] = A.lab[it];
            if (carry) ws.key[o] = A.kc[it];
            if (perm) perm[i] = (int)o;
        }
        MV_TRACE_U(u, 3);
        if (!more) break;
        move_rank(B, exB, alB, totB, s_cnt, &s_sink);
        publish(u2);
        MV_TRACE_U(u2, 1);
        u = u2;
        A = B;
        totA = totB;
#pragma unroll
        for (int it = 0; it < kCmpItems; ++it) {
            exA[it] = exB[it];
            alA[it] = alB[it];
        }
    }
}

// K7b with the copy engine for the loads (no extra columns, no perm; the default
// in-place move), warp-specialised.  Warp 0 is the producer: one lane takes
// sub-tile tickets, waits for a free stage, arms the stage's "full" mbarrier and
// issues one cp.async.bulk per column (x, y, (z), vx, vy, (vz), label, carried
// key, id) into it, and publishes "read done" for every sub-tile as soon as its
// copy completed (every input byte has left global memory), in ticket order.
// Warp 1 checks the dependencies ahead of the consumers: for each issued sub-tile
// it waits for the "read done" of the earlier sub-tiles whose input the
// sub-tile's output range can overlap (outputs move down by at most D), then
// arrives on the stage's "ready" mbarrier, so no global-memory poll is on the
// consumers' path.  Warps 2..9 consume the stages in order: every thread takes
// its elements into registers and the stage goes straight back to the producer
// (so up to kTmaStages copies are in flight per SM), the survivors are ranked
// (striped scan of the labels) and stored at i - (tombstones before i),
// warp-contiguous.  Measured at C5: 1.66 ms against 1.70-1.73 ms
// for k_compact_move2; staging the compacted stage and writing it back by bulk
// stores was slower (1.89 ms: fewer copies in flight per SM).
constexpr int kTmaStage = kCmpTile;         // elements per column per stage
constexpr int kTmaStages = 5;
struct alignas(16) TmaStage {
    float c[6][kTmaStage];                   // x, y, z, vx, vy, vz
    int lab[kTmaStage];
    int key[kTmaStage];
    long long id[kTmaStage];
};
constexpr size_t kTmaSmem = kTmaStages * sizeof(TmaStage);
constexpr int kTmaThreads = kThreads + 64;   // 8 consumer warps + the producer and the dependency warp

__global__ void __launch_bounds__(kTmaThreads, 1) k_compact_move_tma(PartDev p, int dim, Workspace ws, int carry)
{
    pdl_entry();
    extern __shared__ __align__(128) unsigned char dsm[];
    TmaStage *stage = reinterpret_cast<TmaStage *>(dsm);
    __shared__ __align__(8) uint64_t s_full[kTmaStages], s_empty[kTmaStages], s_ready[kTmaStages];
    __shared__ long long s_tile[kTmaStages];
    __shared__ volatile long long s_issued;
    __shared__ unsigned s_cnt[kCmpItems * kThreads / 32 + 1];
    Counters *ctr = ws.ctr;
    const long long D = ctr->n_del;
    if (D == 0) return;
    const long long N = ctr->cmp_n;
    const long long ibeg = cmp_begin(ctr->i_first);
    const unsigned epoch = ctr->epoch_cmp;
    const long long nsub = (N - ibeg + kCmpTile - 1) / kCmpTile;
    const int ncf = dim == 3 ? 6 : 4;                       // float columns in use
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTmaStages; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&s_empty[s], 1);
            mbar_init(&s_ready[s], 1);
        }
        fence_mbar_init();
        s_issued = 0;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        // ---------------------------------------------------------------- producer
        if (threadIdx.x != 0) return;
        float *gcol[6] = {p.x, p.y, p.vx, p.vy, p.z, p.vz};
        const int scol[6] = {0, 1, 3, 4, 2, 5};
        long long issued = 0, published = 0;
        long long tiles[kTmaStages];
        bool done = false;
        while (!done || published < issued) {
            // publish every completed copy, in order
            while (published < issued) {
                const int s = (int)(published % kTmaStages);
                if (!mbar_test(&s_full[s], (uint32_t)((published / kTmaStages) & 1))) break;
                asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(ws.rd + tiles[s]), "r"(epoch) : "memory");
                ++published;
            }
            if (done) {
                __nanosleep(32);
                continue;
            }
            // the next stage, once its previous sub-tile has been stored
            const int s = (int)(issued % kTmaStages);
            if (issued >= kTmaStages && !mbar_test(&s_empty[s], (uint32_t)(((issued / kTmaStages) - 1) & 1))) {
                __nanosleep(32);
                continue;
            }
            const long long u = atomicAdd(&ctr->ticket_cmp2, 1);
            s_tile[s] = u;
            if (u >= nsub) {
                mbar_arrive(&s_full[s]);                   // consumers see the end
                __threadfence_block();
                s_issued = issued + 1;                     // (the dependency warp sees the end too)
                done = true;
                continue;
            }
            const long long start = ibeg + u * kCmpTile;
            const long long cnt = N - start < kCmpTile ? N - start : kCmpTile;
            const uint32_t n4 = (uint32_t)(cnt & ~3LL), n8 = (uint32_t)(cnt & ~1LL);
            const uint32_t bytes = (uint32_t)(ncf + 1 + (carry ? 1 : 0)) * n4 * 4u + n8 * 8u;
            TmaStage &S = stage[s];
            mbar_arrive_expect_tx(&s_full[s], bytes);
            if (n4) {
                for (int c = 0; c < ncf; ++c) bulk_g2s(S.c[scol[c]], gcol[c] + start, n4 * 4u, &s_full[s]);
                bulk_g2s(S.lab, p.label + start, n4 * 4u, &s_full[s]);
                if (carry) bulk_g2s(S.key, ws.key + start, n4 * 4u, &s_full[s]);
            }
            if (n8) bulk_g2s(S.id, p.id + start, n8 * 8u, &s_full[s]);
            tiles[s] = u;
            ++issued;
            __threadfence_block();
            s_issued = issued;
        }
        return;
    }
    if (threadIdx.x < 64) {
        // ---------------------------------------------------------- dependency warp
        const int lane = threadIdx.x & 31;
        for (long long it = 0;; ++it) {
            while (s_issued <= it) __nanosleep(64);
            __threadfence_block();
            const int s = (int)(it % kTmaStages);
            const long long u = s_tile[s];
            if (u >= nsub) break;
            const long long start = ibeg + u * kCmpTile;
            const long long cnt = N - start < kCmpTile ? N - start : kCmpTile;
            const long long dst0 = start - (long long)ws.sub_off[u];
            if (dst0 < start) {
                // the output is at most [dst0, dst0 + cnt): wait for the earlier
                // sub-tiles whose input it can overlap
                const long long vlo = (dst0 - ibeg) / kCmpTile;
                long long vhi = (dst0 + cnt - 1 - ibeg) / kCmpTile;
                if (vhi > u - 1) vhi = u - 1;
                for (long long w = vlo + lane; w <= vhi; w += 32) {
                    unsigned f;
                    while (true) {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(ws.rd + w) : "memory");
                        if (f == epoch) break;
                        __nanosleep(64);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_ready[s]);
        }
        return;
    }
    // -------------------------------------------------------------------- consumers
    const int ct = threadIdx.x - 64, lane = ct & 31, cw = ct >> 5;
    constexpr int NW = kThreads / 32;
    float *gcol[6] = {p.x, p.y, p.vx, p.vy, p.z, p.vz};
    const int scol[6] = {0, 1, 3, 4, 2, 5};
    for (long long it = 0;; ++it) {
        const int s = (int)(it % kTmaStages);
        mbar_wait(&s_full[s], (uint32_t)((it / kTmaStages) & 1));
        const long long u = s_tile[s];
        if (u >= nsub) break;
        TmaStage &S = stage[s];
        const long long start = ibeg + u * kCmpTile;
        const int cnt = (int)(N - start < kCmpTile ? N - start : kCmpTile);
        const int n4 = cnt & ~3, n8 = cnt & ~1;
        // ragged remainder of the last sub-tile (< 4 elements): loaded here
        if (cnt < kCmpTile) {
            for (int e = n4 + ct; e < cnt; e += kThreads) {
                for (int c = 0; c < ncf; ++c) S.c[scol[c]][e] = gcol[c][start + e];
                S.lab[e] = p.label[start + e];
                if (carry) S.key[e] = ws.key[start + e];
            }
            for (int e = n8 + ct; e < cnt; e += kThreads) S.id[e] = p.id[start + e];
            named_bar(1, kThreads);
        }
        // my elements into registers, survivors ranked (striped order: element it * NT + ct)
        float v[kCmpItems][6];
        int lb[kCmpItems], kv[kCmpItems];
        long long idv[kCmpItems];
        bool alive[kCmpItems];
        unsigned bal[kCmpItems];
#pragma unroll
        for (int q = 0; q < kCmpItems; ++q) {
            const int e = q * kThreads + ct;
            alive[q] = false;
            if (e < cnt) {
#pragma unroll
                for (int c = 0; c < 6; ++c) v[q][c] = c < ncf ? S.c[scol[c]][e] : 0.0f;
                lb[q] = S.lab[e];
                kv[q] = carry ? S.key[e] : 0;
                idv[q] = S.id[e];
                alive[q] = lb[q] > -2;
            }
            bal[q] = __ballot_sync(0xffffffffu, alive[q]);
            if (lane == 0) s_cnt[q * NW + cw] = __popc(bal[q]);
        }
        named_bar(1, kThreads);
        // every thread holds its elements: the stage goes back to the producer
        if (ct == 0) mbar_arrive(&s_empty[s]);
        unsigned excl[kCmpItems], run = 0;
        const unsigned lt = lanemask_lt();
#pragma unroll
        for (int q = 0; q < kCmpItems; ++q) {
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const unsigned c = s_cnt[q * NW + w];
                if (w == cw) excl[q] = run + __popc(bal[q] & lt);
                run += c;
            }
        }
        const long long dst0 = start - (long long)ws.sub_off[u];
        mbar_wait(&s_ready[s], (uint32_t)((it / kTmaStages) & 1));   // predecessors have read their input
        // survivors straight to their destination (warp-contiguous, coalesced)
#pragma unroll
        for (int q = 0; q < kCmpItems; ++q) {
            if (!alive[q]) continue;
            const long long o = dst0 + excl[q];
            SPH_CHECK(o >= ibeg - (long long)D && o < start + kCmpTile && o < p.cap);
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                if (c >= ncf) break;
                gcol[c][o] = v[q][c];
            }
            p.label[o] = lb[q];
            if (carry) ws.key[o] = kv[q];
            p.id[o] = idv[q];
        }
        named_bar(1, kThreads);      // s_cnt is reused by the next sub-tile
    }
}

// Staged particles after the survivors with IDs from the count matrix (reading
// R14, §8(e)): off(k, r) = next_id + sum_{k'<k} sum_r' C[r'][k'] + sum_{r'<r} C[r'][k];
// identity perm below i_first; then N and next_id.
// defer: the tombstones stay in place (the next sph_cll_build drops them) and the
// staged particles go to [N, N + C).  Many blocks: thread 0 of every block reads
// N and next_id into shared memory before the block barrier and before it counts
// the block done, so the last block's update of them cannot race a reader.
__global__ void __launch_bounds__(kThreads) k_compact_append(PartDev p, GridDev g, int n_ports, int max_ports,
                                                             Workspace ws, const int *all_counts, int nranks,
                                                             int rank, long long *next_id, int *perm, bool defer,
                                                             int carry, float cdt)
{
    const int dim = g.dim;
    pdl_entry();
    __shared__ long long s_off[SPH_MAX_PORTS];
    __shared__ long long s_beg[SPH_MAX_PORTS];
    __shared__ long long s_total, s_nid0, s_N;
    Counters *ctr = ws.ctr;
    // N and next_id before the append: read by thread 0 of every block (deferred),
    // or recorded by k_compact_count; the last block to finish writes the new ones
    if (threadIdx.x == 0) {
        const long long nid0 = defer ? *(volatile long long *)next_id : ctr->cmp_next_id;
        s_nid0 = nid0;
        s_N = defer ? *(volatile long long *)p.n : ctr->cmp_n;
        long long acc = nid0, beg = 0;
        for (int k = 0; k < n_ports; ++k) {
            long long before = 0, all = 0;
            for (int r = 0; r < nranks; ++r) {
                const long long c = all_counts[(long long)r * 2 * max_ports + k];
                all += c;
                if (r < rank) before += c;
            }
            s_off[k] = acc + before;
            s_beg[k] = beg;
            beg += all_counts[(long long)rank * 2 * max_ports + k];
            acc += all;
        }
        s_total = acc - nid0;
    }
    __syncthreads();
    const long long nid0 = s_nid0;
    const long long N = s_N;
    const long long D = defer ? 0 : ctr->n_del;
    long long C = ctr->n_stage;
    if (C > ws.max_new) C = ws.max_new;
    const long long dst0 = N - D;
    if (dst0 + C > p.cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&ctr->status, kStCapacity);
        C = p.cap - dst0 > 0 ? p.cap - dst0 : 0;
    }
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < C; u += stride) {
        // staging slot u (filled in any order) -> canonical slot s (port, cell, id)
        const long long s = (long long)ws.tile_pre[ws.stile[u]] + ws.sexcl[u];
        if (s >= C) continue;                      // (staging overflow: reported, state undefined)
        const int k = ws.sport[u];
        const long long d = dst0 + s;
        const float sx = ws.sx[u], sy = ws.sy[u], sz = dim == 3 ? ws.sz[u] : 0.0f;
        const float svx = ws.svx[u], svy = ws.svy[u], svz = dim == 3 ? ws.svz[u] : 0.0f;
        p.x[d] = sx;
        p.y[d] = sy;
        p.vx[d] = svx;
        p.vy[d] = svy;
        if (dim == 3) {
            p.z[d] = sz;
            p.vz[d] = svz;
        }
        for (int e = 0; e < p.n_extra; ++e) p.extra[e][d] = ws.sextra[e][u];
        p.id[d] = s_off[k] + (s - s_beg[k]);
        p.label[d] = -1;
        if (carry) {
            // key carry-over: the new particle's key for the next build
            int oob = 0;
            const int key = carry_key(g, sx, sy, sz, svx, svy, svz, cdt, carry, oob);
            ws.key[d] = key;
            if (key >= 0) atomicAdd(&ws.cell_count[key], 1);
            else leaver_append(ws, d);
        }
    }
    if (perm) {
        const long long ibeg = D ? cmp_begin(ctr->i_first) : N;
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < ibeg; i += stride) perm[i] = (int)i;
    }
    // completion among the blocks that had work (all of them with a perm output;
    // else the first ceil(C / blockDim) — a small append does not wait for the
    // whole grid's atomics); with no work at all, block 0 writes N and next_id
    const long long per = blockDim.x;
    const int working = perm ? (int)gridDim.x : (int)((C + per - 1) / per < gridDim.x ? (C + per - 1) / per : gridDim.x);
    if (threadIdx.x == 0 && ((int)blockIdx.x < working || (working == 0 && blockIdx.x == 0))) {
        __threadfence();
        if (working == 0 || atomicAdd(&ctr->done_app, 1) == working - 1) {
            ctr->done_app = 0;
            *p.n = dst0 + C;
            *next_id = nid0 + s_total;
        }
    }
}

// ------------------------------------------------------------------ launcher

cudaError_t launch_compact(const PartDev &p, const GridDev &g, const PortTable &pt, const Workspace &ws,
                           const int *all_counts, int nranks, int rank, long long *next_id, int *perm, bool defer,
                           int carry, float cdt, cudaStream_t s, Launch *L)
{
    if (defer) {
        L->before(s);
        launch_k(k_compact_append, dim3(cap_grid(sm_count_cached() * 2, ws.max_new, kThreads)), dim3(kThreads), 0, s,
                 p, g, pt.n, pt.max_ports, ws, all_counts, nranks, rank, next_id, nullptr, true, carry, cdt);
        L->after(s, KID_COMPACT_APPEND);
        return cudaGetLastError();
    }
    const int dim = g.dim;
    // SPHBUF_DLIST_MAX=<n> lowers the list size above which the label pass is used
    // (tests force the fallback with 0)
    static const int dmax = [] {
        const char *e = getenv("SPHBUF_DLIST_MAX");
        const int v = e ? atoi(e) : kDelList;
        return v < kDelList ? v : kDelList;
    }();
    {
        static int grid = 0;
        if (!grid) grid = occ_grid(k_compact_count, kThreads);
        L->before(s);
        launch_k(k_compact_count, dim3(cap_grid(grid, p.cap, kCntTile)), dim3(kThreads), 0, s, p, ws, next_id, dmax);
        L->after(s, KID_COMPACT_COUNT);
    }
    L->before(s);
    if (p.n_extra > 0) {
        static int grid = 0;
        if (!grid) grid = occ_grid(k_compact_move<true>, kThreads);
        launch_k(k_compact_move<true>, dim3(cap_grid(grid, p.cap, kCmpTile)), dim3(kThreads), 0, s, p, dim, ws, perm,
                 carry);
    } else {
        static int grid = 0;
        static const bool one = getenv("SPHBUF_MOVE1") != nullptr;   // A/B: one sub-tile in flight
        // the copy-engine move (default); SPHBUF_MOVE_TMA=0 selects the register move
        static const bool tma = [] {
            const char *e = getenv("SPHBUF_MOVE_TMA");
            return !(e && e[0] == '0');
        }();
        const bool aligned = ((reinterpret_cast<size_t>(p.x) | reinterpret_cast<size_t>(p.y) |
                               reinterpret_cast<size_t>(p.vx) | reinterpret_cast<size_t>(p.vy) |
                               reinterpret_cast<size_t>(p.label) | reinterpret_cast<size_t>(p.id) |
                               reinterpret_cast<size_t>(ws.key) |
                               (dim == 3 ? reinterpret_cast<size_t>(p.z) | reinterpret_cast<size_t>(p.vz) : 0)) &
                              15) == 0;
        if (tma && aligned && !perm && !one) {
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(k_compact_move_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem);
                attr = true;
            }
            launch_k(k_compact_move_tma, dim3(cap_grid(sm_count_cached(), p.cap, kCmpTile)), dim3(kTmaThreads),
                     kTmaSmem, s, p, dim, ws, carry);
        } else if (one) {
            if (!grid) grid = occ_grid(k_compact_move<false>, kThreads);
            launch_k(k_compact_move<false>, dim3(cap_grid(grid, p.cap, kCmpTile)), dim3(kThreads), 0, s, p, dim, ws,
                     perm, carry);
        } else {
            if (!grid) grid = occ_grid(k_compact_move2, kThreads);
            launch_k(k_compact_move2, dim3(cap_grid(grid, p.cap, kCmpTile)), dim3(kThreads), 0, s, p, dim, ws, perm,
                     carry);
        }
    }
    L->after(s, KID_COMPACT);
    L->before(s);
    launch_k(k_compact_append, dim3(cap_grid(sm_count_cached() * 4, perm ? p.cap : ws.max_new, kThreads)),
             dim3(kThreads), 0, s, p, g, pt.n, pt.max_ports, ws, all_counts, nranks, rank, next_id, perm, false, carry,
             cdt);
    L->after(s, KID_COMPACT_APPEND);
    return cudaGetLastError();
}

}  // namespace sphbuf
