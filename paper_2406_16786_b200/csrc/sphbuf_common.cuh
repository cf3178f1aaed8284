// sphbuf_common.cuh — device helpers shared by the sm_100a kernels of the
// in/outlet buffer update (arXiv 2406.16786 §III): warp/block scans, the
// decoupled look-back, and the pinned fp32 local-frame transform and cell index.
// "P:n" = PAPER.md line n; readings R<n> are listed in DESIGN.md §3.
//
// All arithmetic that decides an integer or mutates particle state uses
// __fadd_rn/__fsub_rn/__fmul_rn (one binary32 round-to-nearest op each, never
// contracted), in the order fixed by DESIGN.md §3 "Pinned arithmetic".
#pragma once
#include <cassert>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <utility>

#include "sphbuf_internal.h"

namespace sphbuf {

// ------------------------------------------------------------------ helpers

// Device bounds checks of the debug build (-DSPHBUF_DEBUG, build.py --debug):
// compute-sanitizer is not available on the GPU pool, so index invariants are
// asserted in the kernels themselves; compiled out otherwise.
#ifdef SPHBUF_DEBUG
#define SPH_CHECK(cond) assert(cond)
#else
#define SPH_CHECK(cond) ((void)0)
#endif

// Programmatic dependent launch (sm_90+): every kernel of the path is launched
// with launch_k() below and waits here for the kernel before it on the stream to
// complete with its memory visible.  The dependent grid is released as this
// grid's blocks exit (no early trigger: early-launched blocks would take SM
// slots from the running grid), so only the launch gap between kernels is
// hidden.  Without the launch attribute the instruction is a no-op.
__device__ __forceinline__ void pdl_entry() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ unsigned lanemask_lt()
{
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ void st_release(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// tile status word: [63:34] epoch (30 bits) | [33:32] flag (1 aggregate, 2 inclusive prefix) | [31:0] value
__device__ __forceinline__ unsigned long long pack_status(unsigned epoch, unsigned flag, unsigned value)
{
    return ((unsigned long long)(epoch & 0x3fffffffu) << 34) | ((unsigned long long)flag << 32) | value;
}

__device__ __forceinline__ unsigned warp_sum(unsigned v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ long long warp_sum_ll(long long v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ long long warp_min_ll(long long v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

// Decoupled look-back (single pass): called by all 32 lanes of warp 0 of a block
// that owns `tile`.  Publishes the tile's aggregate, accumulates predecessors'
// aggregates until an inclusive prefix is found, publishes its own inclusive
// prefix and returns the exclusive prefix.  The flag, epoch and value travel in
// one 64-bit word and callers use nothing else a predecessor wrote, so the
// stores and polls are relaxed: no fence (a gpu-scope fence per tile costs
// microseconds when the block still has stores and atomics in flight).
static __device__ unsigned tile_prefix(unsigned long long *status, long long tile, unsigned epoch, unsigned aggregate)
{
    // each lane inspects kLB consecutive predecessors per round (loads issued
    // together), so a wave of W tiles started at once resolves in ~W / (32 kLB)
    // dependent rounds instead of W / 32
    constexpr int kLB = 4;
    const int lane = threadIdx.x & 31;
    const unsigned ep = epoch & 0x3fffffffu;
    if (tile == 0) {
        if (lane == 0) st_relaxed(&status[0], pack_status(epoch, 2, aggregate));
        return 0;
    }
    if (lane == 0) st_relaxed(&status[tile], pack_status(epoch, 1, aggregate));
    auto flag_of = [&](unsigned long long s) -> unsigned {
        return ((unsigned)(s >> 34) == ep) ? (unsigned)((s >> 32) & 3u) : 0u;
    };
    unsigned excl = 0;
    long long base = tile - 1;
    while (true) {
        unsigned long long s[kLB];
#pragma unroll
        for (int j = 0; j < kLB; ++j) {
            const long long t = base - lane * kLB - j;
            s[j] = t >= 0 ? ld_relaxed(&status[t]) : 0ull;
        }
        unsigned v = 0;
        bool incl = false;
#pragma unroll
        for (int j = 0; j < kLB; ++j) {
            const long long t = base - lane * kLB - j;
            unsigned f = 2;
            if (t >= 0) {
                while ((f = flag_of(s[j])) == 0) s[j] = ld_relaxed(&status[t]);
            }
            if (!incl) {
                v += (unsigned)(s[j] & 0xffffffffu);          // aggregate, or the inclusive prefix
                incl = f == 2;
            }
        }
        const unsigned pmask = __ballot_sync(0xffffffffu, incl);
        const int first = pmask ? __ffs(pmask) - 1 : 32;
        excl += warp_sum(lane <= first ? v : 0u);
        if (pmask) break;
        base -= 32 * kLB;
    }
    if (lane == 0) st_relaxed(&status[tile], pack_status(epoch, 2, excl + aggregate));
    return excl;
}

// Cell histogram from a warp whose lanes hold consecutive particles (keys mostly
// equal in runs): one atomic per run of equal keys; key < 0 is not counted.  All
// 32 lanes must call it.
__device__ __forceinline__ void hist_count_runs(int *cnt, int key)
{
    const int lane = threadIdx.x & 31;
    const unsigned le = lanemask_lt() | (1u << lane);
    const int prev = __shfl_up_sync(0xffffffffu, key, 1);
    const bool head = (lane == 0) || (key != prev);
    const unsigned heads = __ballot_sync(0xffffffffu, head);
    const unsigned above = heads & ~le;
    const int next = above ? __ffs(above) - 1 : 32;
    if (head && key >= 0) atomicAdd(&cnt[key], next - lane);
}

// The same count with lanes grouped by equal key (match.any): one atomic per
// distinct key of the warp, however the equal keys are interleaved.
__device__ __forceinline__ void hist_count_match(int *cnt, int key)
{
    const unsigned grp = __match_any_sync(0xffffffffu, key);
    if (key >= 0 && (int)(__ffs(grp) - 1) == (int)(threadIdx.x & 31)) atomicAdd(&cnt[key], __popc(grp));
}

// Block-wide exclusive scan of one unsigned per thread (NT threads).
template <int NT>
__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned &total, unsigned *s_warp)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        unsigned w = lane < NT / 32 ? s_warp[lane] : 0u;
        unsigned wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < NT / 32) s_warp[lane] = wi - w;
        if (lane == NT / 32 - 1) s_warp[NT / 32] = wi;
    }
    __syncthreads();
    unsigned res = s_warp[warp] + x - v;
    total = s_warp[NT / 32];
    __syncthreads();
    return res;
}

// Exclusive ranks of flagged items in STRIPED order: item `it` of thread t is
// element it * NT + t of the tile, so the order is (item, warp, lane).  One
// ballot per item and warp, one barrier.  s_cnt: ITEMS * NT/32 words.
template <int NT, int ITEMS>
__device__ __forceinline__ void striped_scan(const bool (&flag)[ITEMS], unsigned (&excl)[ITEMS], unsigned &total,
                                             unsigned *s_cnt)
{
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = lanemask_lt();
    unsigned b[ITEMS];
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
        b[it] = __ballot_sync(0xffffffffu, flag[it]);
        if (lane == 0) s_cnt[it * NW + warp] = __popc(b[it]);
    }
    __syncthreads();
    unsigned run = 0;
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const unsigned c = s_cnt[it * NW + w];
            if (w == warp) excl[it] = run + __popc(b[it] & lt);
            run += c;
        }
    }
    total = run;
    __syncthreads();
}

// 64-bit variant (used for run offsets).
template <int NT>
__device__ __forceinline__ long long block_excl_scan_ll(long long v, long long &total, long long *s_warp)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        long long w = lane < NT / 32 ? s_warp[lane] : 0;
        long long wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            long long y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < NT / 32) s_warp[lane] = wi - w;
        if (lane == NT / 32 - 1) s_warp[NT / 32] = wi;
    }
    __syncthreads();
    long long res = s_warp[warp] + x - v;
    total = s_warp[NT / 32];
    __syncthreads();
    return res;
}

// Pinned forward transform X' = Q (x - o) (Eq. 2D_transformation P:252-269,
// Eq. 3D_transformation): d_j = fl(x_j - o_j);
// X'_r = fl(fl(fl(Q_r0 d_0) + fl(Q_r1 d_1)) + fl(Q_r2 d_2)).
__device__ __forceinline__ void to_local(const PortDev &P, int dim, float x, float y, float z, float X[3])
{
    const float d0 = __fsub_rn(x, P.o[0]);
    const float d1 = __fsub_rn(y, P.o[1]);
    if (dim == 3) {
        const float d2 = __fsub_rn(z, P.o[2]);
#pragma unroll
        for (int r = 0; r < 3; ++r)
            X[r] = __fadd_rn(__fadd_rn(__fmul_rn(P.Q[3 * r], d0), __fmul_rn(P.Q[3 * r + 1], d1)),
                             __fmul_rn(P.Q[3 * r + 2], d2));
    } else {
#pragma unroll
        for (int r = 0; r < 2; ++r) X[r] = __fadd_rn(__fmul_rn(P.Q[3 * r], d0), __fmul_rn(P.Q[3 * r + 1], d1));
        X[2] = 0.0f;
    }
}

__device__ __forceinline__ bool in_box(const float X[3], const float he[3], int dim)
{
    bool r = fabsf(X[0]) < he[0] && fabsf(X[1]) < he[1];
    if (dim == 3) r = r && fabsf(X[2]) < he[2];
    return r;
}

// Pinned advection (the driver step): x <- fl(x + fl(v dt)).
__device__ __forceinline__ float advect1(float x, float v, float dt) { return __fadd_rn(x, __fmul_rn(v, dt)); }

// Pinned cell index along one axis: floor(fl(fl(x - lo) * inv_cs)), clamped to
// [lo_c, hi_c) (branch-free integer min/max of the floored value, which the
// float -> int conversion saturates outside the int range; oob is set when the
// clamp changed it).
__device__ __forceinline__ int cell_axis(float x, float lo, float inv, int lo_c, int hi_c, int &oob)
{
    const float t = __fmul_rn(__fsub_rn(x, lo), inv);
    const int f = __float2int_rz(floorf(t));
    const int c = min(max(f, lo_c), hi_c - 1);
    oob |= (c != f);
    return c;
}

// DIM: 2 or 3 when known at compile time, 0 to read g.dim.
template <int DIM = 0>
__device__ __forceinline__ int cell_of(const GridDev &g, float x, float y, float z, int &oob)
{
    const int cx = cell_axis(x, g.lo[0], g.inv_cs, g.cx_begin, g.cx_end, oob);
    const int cy = cell_axis(y, g.lo[1], g.inv_cs, 0, g.ncell[1], oob);
    int cz = 0;
    if (DIM == 3 || (DIM == 0 && g.dim == 3)) cz = cell_axis(z, g.lo[2], g.inv_cs, 0, g.ncell[2], oob);
    if (DIM == 2) return (cx - g.cx_begin) * g.ny + cy;
    return ((cx - g.cx_begin) * g.ny + cy) * g.nz + cz;
}

// Key carry-over (sphbuf_cll.cu).  carry: 0 off, 1 on, 2 on with slab
// migration — a particle whose next cell x-index leaves the slab gets the key
// kLeaver (not counted; its index goes to the leaver list, packed for the
// neighbour rank by the next build).
constexpr int kLeaver = -2;
constexpr int kPacked = -3;

template <int DIM = 0>
__device__ __forceinline__ int carry_key(const GridDev &g, float x, float y, float z, float vx, float vy, float vz,
                                         float cdt, int carry, int &oob)
{
    const bool d3 = DIM == 3 || (DIM == 0 && g.dim == 3);
    const float xa = advect1(x, vx, cdt), ya = advect1(y, vy, cdt), za = d3 ? advect1(z, vz, cdt) : 0.0f;
    if (carry == 2) {
        int o2 = 0;
        const int cxr = cell_axis(xa, g.lo[0], g.inv_cs, 0, g.ncell[0], o2);
        if (cxr < g.cx_begin || cxr >= g.cx_end) return kLeaver;
    }
    return cell_of<DIM>(g, xa, ya, za, oob);
}

__device__ __forceinline__ void leaver_append(const Workspace &ws, long long i)
{
    const long long e = atomicAdd((unsigned long long *)&ws.ctr->n_leave, 1ull);
    if (e < ws.max_leave) ws.leave[e] = (int)i;
    else atomicOr(&ws.ctr->status, kStMigrate);
}

// Key fix-up with the old key already loaded and the new one computed.
__device__ __forceinline__ void carry_set(const Workspace &ws, long long i, int kold, int knew)
{
    if (knew != kold) {
        if (kold >= 0) atomicSub(&ws.cell_count[kold], 1);
        if (knew >= 0) atomicAdd(&ws.cell_count[knew], 1);
        if (knew == kLeaver) leaver_append(ws, i);      // (a stale entry is skipped when packing)
        ws.key[i] = knew;
    }
}

// Fix-up: particle i, whose next-build key ws.key[i] the gather computed, now has
// position x and velocity v (or was deleted): its key and the next histogram
// follow (a leaver key leaves the histogram alone and lists the particle).
__device__ __forceinline__ void carry_fix(const GridDev &g, const Workspace &ws, long long i, bool del, float x,
                                          float y, float z, float vx, float vy, float vz, float cdt, int carry)
{
    const int kold = ws.key[i];
    int oob = 0;
    carry_set(ws, i, kold, del ? -1 : carry_key(g, x, y, z, vx, vy, vz, cdt, carry, oob));
}

// ------------------------------------------------------------------ launch helpers (host)

// Launch with the programmatic-stream-serialization attribute (see pdl_entry);
// SPHBUF_PDL=0 in the environment launches plainly (A/B timing).
inline bool pdl_enabled()
{
    static int on = -1;
    if (on < 0) {
        const char *v = getenv("SPHBUF_PDL");
        on = (v && v[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args &&...args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

inline int sm_count_cached()
{
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

template <typename K>
inline int occ_grid(K kernel, int threads, size_t smem = 0)
{
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem);
    if (per <= 0) per = 1;
    return per * sm_count_cached();
}

}  // namespace sphbuf

namespace sphbuf {
// Grid of a grid-stride / persistent kernel: the occupancy-derived full-GPU grid,
// but no more blocks than the array capacity can keep busy (small configurations
// are launch-latency bound).
inline int cap_grid(int grid, long long cap, long long per_block)
{
    const long long need = (cap + per_block - 1) / per_block;
    return (int)(need < 1 ? 1 : (need < grid ? need : grid));
}
}  // namespace sphbuf
