// sphbuf_update.cu — registration (Alg. 1 identification), the driver's advection,
// and the buffer update: candidate transform + axial compare (a3), inflow
// generation (a4), outflow deletion (a5) and relabel (a6), fused in one pass over
// the candidates of the port cell runs (arXiv 2406.16786 §III).
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "sphbuf_common.cuh"
#include "sphbuf_prologue.cuh"

namespace sphbuf {

// ------------------------------------------------------------------ driver: advection

__global__ void __launch_bounds__(kThreads) k_advect(PartDev p, int dim, float dt)
{
    pdl_entry();
    const long long n = *p.n;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        p.x[i] = __fadd_rn(p.x[i], __fmul_rn(p.vx[i], dt));
        p.y[i] = __fadd_rn(p.y[i], __fmul_rn(p.vy[i], dt));
        if (dim == 3) p.z[i] = __fadd_rn(p.z[i], __fmul_rn(p.vz[i], dt));
    }
}

// ------------------------------------------------------------------ registration (Alg. 1 identification)

// "Buffer particle identification ... Execute only once": every fluid
// particle in the box of port k becomes a buffer particle of k; the same test is
// the initial relabel of outlet / bidirectional ports.
__global__ void __launch_bounds__(kThreads) k_register(PartDev p, int dim, PortDev P, int k, long long *members)
{
    pdl_entry();
    const long long n = *p.n;
    long long cnt = 0;
    const int lane = threadIdx.x & 31;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i - lane < n;
         i += (long long)gridDim.x * blockDim.x) {
        if (i < n) {
            int lab = p.label[i];
            if (lab == -1) {
                float X[3];
                to_local(P, dim, p.x[i], p.y[i], dim == 3 ? p.z[i] : 0.0f, X);
                if (in_box(X, P.he, dim)) {
                    lab = k;
                    p.label[i] = k;
                }
            }
            cnt += (lab == k);
        }
    }
    cnt = warp_sum_ll(cnt);
    if (lane == 0 && cnt && members) atomicAdd((unsigned long long *)members, (unsigned long long)cnt);
}

// ------------------------------------------------------------------ a3-a6: buffer update

// K5 as its own kernel (see sphbuf_prologue.cuh).
__global__ void __launch_bounds__(1024) k_upd_prologue(Workspace ws, int n_runs, const int *cell_start,
                                                       const int *cell_end, int max_ports)
{
    pdl_entry();
    upd_prologue_body<1024>(ws, n_runs, cell_start, cell_end, max_ports, gridDim.x);
}

#ifdef SPHBUF_TRACE
// Tile timeline of K6 (tools/upd_trace.py): per tile, %globaltimer at its start,
// after the run staging, before the scan, after the look-back, at its end; the
// block and SM that ran it.
constexpr int kTraceTiles = 1 << 14;
__device__ unsigned long long g_trace[kTraceTiles][7];
__device__ unsigned long long g_trace_k[4];   // K6: first block entry, last block entry, scan start, end
__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define SPH_TRACE(tile, slot)                                                            \
    do {                                                                                 \
        __syncthreads();                                                                 \
        if (threadIdx.x == 0 && (tile) < kTraceTiles) g_trace[(tile)][(slot)] = gtimer(); \
    } while (0)
#else
#define SPH_TRACE(tile, slot) \
    do {                      \
    } while (0)
#endif

constexpr int kTileRuns = 256;   // runs of one K6 tile staged in shared memory (else global search)

// Boundary-condition velocity of a buffer particle of port P (paper §IV; SURVEY
// §8(f) rank 1): pressure BC v <- (v.u) u (Eq. velocity_correction);
// velocity BC v_X' from the profile (Eqs. 2D/3D_velocity_profile),
// v = Q^T (v_X', 0, 0).  Y, Z: post-recycle lateral local coordinates.
__device__ __forceinline__ float bc_speed(const PortDev &P, int dim, float vx, float vy, float vz, float Y, float Z)
{
    if (P.bc == SPH_BC_PRESSURE) {
        float u = __fadd_rn(__fmul_rn(vx, P.Q[0]), __fmul_rn(vy, P.Q[1]));
        if (dim == 3) u = __fadd_rn(u, __fmul_rn(vz, P.Q[2]));
        return u;
    }
    float u = P.u0;
    if (P.profile == SPH_PROFILE_PARABOLIC) {
        const float t = __fdiv_rn(Y, P.R);
        u = __fmul_rn(P.u0, __fsub_rn(1.0f, __fmul_rn(t, t)));
    } else if (P.profile == SPH_PROFILE_PARABOLIC_RADIAL) {
        float r2 = __fmul_rn(Y, Y);
        if (dim == 3) r2 = __fadd_rn(r2, __fmul_rn(Z, Z));
        u = __fmul_rn(P.u0, __fsub_rn(1.0f, __fdiv_rn(r2, P.R2)));
    }
    return u;
}

// K6: the candidate check (a3) with generation (a4), deletion (a5) and relabel
// (a6) fused; CREATEs are appended to the staging area in canonical order
// (port, cell, id) without any wait between tiles: a tile's CREATEs take staging
// slots from one atomic per tile and record (tile, rank in the tile); the last
// block to finish scans the per-tile counts, so the canonical slot of a staged
// particle is tile_pre[tile] + rank (read by the compaction).  Per tile, every
// load is issued before the stores it does not depend on, so a tile costs few
// dependent memory round trips.
// MINB: resident blocks per SM the registers are bounded for (tiles in one wave);
// SPEC: the velocity, id and carried key of every candidate are loaded with its
// position (one dependent round trip less for the tiles with creations or BC).
template <int MINB, bool SPEC>
__global__ void __launch_bounds__(kThreads, MINB) k_upd_main(PartDev p, GridDev g, const __grid_constant__ PortTable pt,
                                                       Workspace ws, int n_runs, const int *cell_start,
                                                       int *port_counts, int carry, float cdt, int tile_runs_max)
{
    const int dim = g.dim;
    pdl_entry();
    __shared__ PortDev s_ports[SPH_MAX_PORTS];
    __shared__ unsigned s_warp[kUpdItems * kThreads / 32 + 1];
    __shared__ long long s_tile, s_u0;
    __shared__ int s_roff[kTileRuns], s_rbase[kTileRuns], s_rk[kTileRuns];
    Counters *ctr = ws.ctr;
#ifdef SPHBUF_TRACE
    if (threadIdx.x == 0) {
        const unsigned long long t = gtimer();
        atomicMin(&g_trace_k[0], t);
        atomicMax(&g_trace_k[1], t);
    }
#endif
    // a block's first tile is its index; further tiles come from the ticket counter
    // (offset by the grid); a block with no tile leaves at once and takes no part
    // in the completion count below (small configurations launch far more blocks
    // than they have tiles)
    const long long n_cand = ctr->n_cand;
    const long long ntiles_all = (n_cand + kUpdTile - 1) / kUpdTile;
    const long long nt_run = ntiles_all < ws.upd_tiles ? ntiles_all : ws.upd_tiles;
    if ((long long)blockIdx.x >= nt_run && !(blockIdx.x == 0 && nt_run == 0)) return;
    long long next_ticket = blockIdx.x;
    {
        const int words = pt.n * (int)(sizeof(PortDev) / 4);
        const unsigned *src = reinterpret_cast<const unsigned *>(pt.p);
        unsigned *dst = reinterpret_cast<unsigned *>(s_ports);
        for (int w = threadIdx.x; w < words; w += blockDim.x) dst[w] = src[w];
    }
    const long long ntiles = ntiles_all;
    const int max_ports = pt.max_ports;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctr->epoch_cmp += 1;  // consumed by the compaction that follows
        ctr->ticket_cmp = 0;
        ctr->ticket_cmp2 = 0;
    }
    long long del_cnt = 0, del_min = LLONG_MAX, motion = 0;
    int my_tiles = 0;
    while (true) {
        if (threadIdx.x == 0) s_tile = next_ticket;
        __syncthreads();
        const long long tile = s_tile;
        if (tile >= ntiles || tile >= ws.upd_tiles) break;
#ifdef SPHBUF_TRACE
        if (threadIdx.x == 0 && tile < kTraceTiles) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            g_trace[tile][0] = gtimer();
            g_trace[tile][5] = blockIdx.x;
            g_trace[tile][6] = smid;
        }
#endif
        // the ticket of this block's next tile, taken now (off the critical path)
        if (threadIdx.x == 0) next_ticket = (long long)gridDim.x + atomicAdd(&ctr->ticket_upd, 1);
        ++my_tiles;
        // the tile's runs [r0, r1] (K5's tile_run) staged in shared memory: offsets
        // relative to the tile, first particle index, port
        const long long t0 = tile * kUpdTile;
        const int r0 = ws.tile_run[tile];
        const int r1 = tile + 1 < ntiles ? ws.tile_run[tile + 1] : n_runs - 1;
        const int nr = r1 - r0 + 1;
        const bool staged = nr <= tile_runs_max;   // (tests lower it: SPHBUF_TILE_RUNS)
        if (staged) {
            for (int i = threadIdx.x; i < nr; i += blockDim.x) {
                s_roff[i] = (int)(ws.run_off[r0 + i] - t0);
                s_rbase[i] = ws.run_base[r0 + i];
                s_rk[i] = ws.runs[3 * (r0 + i) + 2];
            }
        }
        __syncthreads();
        SPH_TRACE(tile, 1);
        // (A) candidate -> particle, loads of what the decisions need
        int pidx[kUpdItems], kk[kUpdItems], lab[kUpdItems];
        float x[kUpdItems], y[kUpdItems], z[kUpdItems];
        float vx[kUpdItems], vy[kUpdItems], vz[kUpdItems];
        long long sid[kUpdItems];
        int okey[kUpdItems];
#pragma unroll
        for (int it = 0; it < kUpdItems; ++it) {
            pidx[it] = -1;
            kk[it] = 0;
            vx[it] = vy[it] = vz[it] = 0.0f;
            sid[it] = 0;
            okey[it] = 0;
            const int rel = it * kThreads + threadIdx.x;
            const long long gc = t0 + rel;
            if (gc >= n_cand) continue;
            // run containing gc: the largest r with run_off[r] <= gc (empty runs
            // share their successor's offset, so the search lands on the non-empty one)
            int k, pi;
            if (staged) {
                int lo = 0, hi = nr - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (s_roff[mid] <= rel) lo = mid;
                    else hi = mid - 1;
                }
                k = s_rk[lo];
                pi = s_rbase[lo] + (rel - s_roff[lo]);
            } else {
                int lo = r0, hi = r1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (ws.run_off[mid] <= gc) lo = mid;
                    else hi = mid - 1;
                }
                k = ws.runs[3 * lo + 2];
                pi = ws.run_base[lo] + (int)(gc - ws.run_off[lo]);
            }
            SPH_CHECK(pi >= 0 && pi < p.cap && k >= 0 && k < pt.n);
            pidx[it] = pi;
            kk[it] = k;
            x[it] = p.x[pi];
            y[it] = p.y[pi];
            z[it] = dim == 3 ? p.z[pi] : 0.0f;
            lab[it] = p.label[pi];
            if (SPEC) {
                vx[it] = p.vx[pi];
                vy[it] = p.vy[pi];
                if (dim == 3) vz[it] = p.vz[pi];
                sid[it] = p.id[pi];
                if (carry) okey[it] = ws.key[pi];
            }
        }
        // (B) decisions, pure arithmetic
        bool cr[kUpdItems], dl[kUpdItems], bcm[kUpdItems];
        int nlab[kUpdItems];                                   // label to write, or INT_MIN
        float bY[kUpdItems], bZ[kUpdItems];
#pragma unroll
        for (int it = 0; it < kUpdItems; ++it) {
            cr[it] = dl[it] = bcm[it] = false;
            nlab[it] = INT_MIN;
            bY[it] = bZ[it] = 0.0f;
            if (pidx[it] < 0) continue;
            const int k = kk[it];
            const PortDev &P = s_ports[k];
            float X[3];
            to_local(P, dim, x[it], y[it], z[it], X);
            const bool inP = in_box(X, P.heP, dim);              // x in P_k (reading R4)
            const bool member = (lab[it] == k);
            const bool beyond = X[0] > P.he[0];                  // X'_0 > a/2
            bool create = false, del = false;
            if (inP) {
                if (P.kind == SPH_INLET) {
                    create = member && beyond;                   // Alg. 1 (R5)
                } else if (P.kind == SPH_OUTLET) {
                    del = beyond;                                // Alg. 2 (R6)
                } else {
                    create = member && beyond;                   // Alg. 3
                    del = member && (X[0] < -P.he[0]);           // Alg. 3
                }
            }
            // R12: a buffer particle outside its decision region moved more than the
            // one-cell margin in one step; it can no longer be generated/deleted.
            if (member && !inP) ++motion;
            float Xp[3] = {X[0], X[1], X[2]};
            if (create) {
                // post-recycle local frame of x <- fl(x - fl(a u)) (R10)
                to_local(P, dim, __fsub_rn(x[it], P.s[0]), __fsub_rn(y[it], P.s[1]),
                         dim == 3 ? __fsub_rn(z[it], P.s[2]) : 0.0f, Xp);
            }
            bool fin = member;                                   // a buffer particle of k after the update
            if (del) {
                nlab[it] = -2;                                   // tombstone, removed by sph_compact
                fin = false;
            } else if (P.kind != SPH_INLET) {
                // relabel on post-recycle positions (R9)
                fin = in_box(Xp, P.he, dim);
                if (fin && !member) nlab[it] = k;
                else if (!fin && member) nlab[it] = -1;
            }
            cr[it] = create;
            dl[it] = del;
            bcm[it] = fin && P.bc != SPH_BC_NONE;
            bY[it] = Xp[1];
            bZ[it] = Xp[2];
        }
        // deleted positions listed (warp-aggregated) for the in-place compaction,
        // which derives its sub-tile offsets from them instead of a label pass
#pragma unroll
        for (int it = 0; it < kUpdItems; ++it) {
            const unsigned m = __ballot_sync(0xffffffffu, dl[it]);
            if (!m) continue;
            const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
            long long b0 = 0;
            if (lane == leader) b0 = (long long)atomicAdd((unsigned long long *)&ctr->n_dlist, (unsigned long long)__popc(m));
            b0 = __shfl_sync(0xffffffffu, b0, leader);
            if (dl[it]) {
                const long long slot = b0 + __popc(m & lanemask_lt());
                if (slot < kDelList) ws.del_list[slot] = pidx[it];
            }
        }
        // (C) loads for the duplicates and boundary conditions (pre-BC velocity)
#pragma unroll
        for (int it = 0; it < kUpdItems; ++it) {
            if (SPEC) break;
            const int pi = pidx[it];
            if (cr[it] || bcm[it]) {
                vx[it] = p.vx[pi];
                vy[it] = p.vy[pi];
                if (dim == 3) vz[it] = p.vz[pi];
            }
            if (cr[it]) sid[it] = p.id[pi];
            if (carry && (cr[it] || dl[it] || bcm[it])) okey[it] = ws.key[pi];
        }
        // (D) stores that do not need the staging slot
#pragma unroll
        for (int it = 0; it < kUpdItems; ++it) {
            const int pi = pidx[it];
            if (pi < 0) continue;
            const int k = kk[it];
            const PortDev &P = s_ports[k];
            float px = x[it], py = y[it], pz = z[it];
            if (cr[it]) {
                // recycle: x <- fl(x - fl(a u)) (Eqs. 2D/3D_Inverse_transformation, R10)
                px = __fsub_rn(px, P.s[0]);
                py = __fsub_rn(py, P.s[1]);
                p.x[pi] = px;
                p.y[pi] = py;
                if (dim == 3) {
                    pz = __fsub_rn(pz, P.s[2]);
                    p.z[pi] = pz;
                }
                atomicAdd(&ws.port_cnt[k], 1);
            }
            if (nlab[it] != INT_MIN) p.label[pi] = nlab[it];
            if (dl[it]) {
                atomicAdd(&ws.port_cnt[max_ports + k], 1);
                ++del_cnt;
                del_min = pi < del_min ? pi : del_min;
            }
            if (cr[it]) continue;                                 // BC and key after staging
            float nvx = vx[it], nvy = vy[it], nvz = vz[it];
            if (bcm[it]) {
                const float u = bc_speed(P, dim, vx[it], vy[it], vz[it], bY[it], bZ[it]);
                nvx = __fmul_rn(u, P.Q[0]);
                nvy = __fmul_rn(u, P.Q[1]);
                p.vx[pi] = nvx;
                p.vy[pi] = nvy;
                if (dim == 3) {
                    nvz = __fmul_rn(u, P.Q[2]);
                    p.vz[pi] = nvz;
                }
            }
            // key carry-over: the next-build key follows a velocity change or a deletion
            if (carry && (dl[it] || bcm[it])) {
                int oob = 0;
                const int knew = dl[it] ? -1 : carry_key(g, px, py, pz, nvx, nvy, nvz, cdt, carry, oob);
                carry_set(ws, pi, okey[it], knew);
            }
        }
        // (E) ranks of the tile's CREATEs, staging slots
        SPH_TRACE(tile, 2);
        unsigned excl[kUpdItems], total;
        striped_scan<kThreads, kUpdItems>(cr, excl, total, s_warp);
        if (threadIdx.x == 0) {
            ws.tile_cr[tile] = total;
            s_u0 = total ? (long long)atomicAdd((unsigned long long *)&ctr->n_stage_raw, (unsigned long long)total) : 0;
        }
        if (total) __syncthreads();
        const long long u0 = s_u0;
        SPH_TRACE(tile, 3);
        // (F) the duplicates: bitwise copy of the pre-recycle state, label fluid
        // (R11); then the boundary condition of the recycled particle
#pragma unroll
        for (int it = 0; it < kUpdItems; ++it) {
            if (!cr[it]) continue;
            const int pi = pidx[it];
            const int k = kk[it];
            const PortDev &P = s_ports[k];
            const long long slot = u0 + excl[it];
            if (slot < ws.max_new) {
                ws.sx[slot] = x[it];
                ws.sy[slot] = y[it];
                ws.svx[slot] = vx[it];
                ws.svy[slot] = vy[it];
                if (dim == 3) {
                    ws.sz[slot] = z[it];
                    ws.svz[slot] = vz[it];
                }
                for (int e = 0; e < p.n_extra; ++e) ws.sextra[e][slot] = p.extra[e][pi];
                ws.sid[slot] = sid[it];
                ws.sport[slot] = k;
                ws.stile[slot] = (int)tile;
                ws.sexcl[slot] = (int)excl[it];
            } else {
                atomicOr(&ctr->status, kStStaging);
            }
            const float px = __fsub_rn(x[it], P.s[0]), py = __fsub_rn(y[it], P.s[1]);
            const float pz = dim == 3 ? __fsub_rn(z[it], P.s[2]) : 0.0f;
            float nvx = vx[it], nvy = vy[it], nvz = vz[it];
            if (bcm[it]) {
                const float u = bc_speed(P, dim, vx[it], vy[it], vz[it], bY[it], bZ[it]);
                nvx = __fmul_rn(u, P.Q[0]);
                nvy = __fmul_rn(u, P.Q[1]);
                p.vx[pi] = nvx;
                p.vy[pi] = nvy;
                if (dim == 3) {
                    nvz = __fmul_rn(u, P.Q[2]);
                    p.vz[pi] = nvz;
                }
                // recycled particles: rho = rho0 + p_b / c0^2 (Eq. postulate-density,
                // P:557-563); a Windkessel-driven port reads this step's from the device
                if (P.bc == SPH_BC_PRESSURE && P.rho_col >= 0)
                    p.extra[P.rho_col][pi] = P.rho_dev ? ws.drv_rho[k] : P.rho_b;
            }
            if (carry) {
                int oob = 0;
                carry_set(ws, pi, okey[it], carry_key(g, px, py, pz, nvx, nvy, nvz, cdt, carry, oob));
            }
        }
        SPH_TRACE(tile, 4);
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    del_cnt = warp_sum_ll(del_cnt);
    del_min = warp_min_ll(del_min);
    motion = warp_sum_ll(motion);
    if (lane == 0) {
        if (del_cnt) {
            atomicAdd((unsigned long long *)&ctr->n_del, (unsigned long long)del_cnt);
            atomicMin(&ctr->i_first, del_min);
        }
        if (motion) {
            atomicAdd((unsigned long long *)&ctr->motion, (unsigned long long)motion);
            atomicOr(&ctr->status, kStMotion);
        }
    }
    // the block that completes the last tile: exclusive scan of the tile CREATE
    // counts (the canonical staging order) and the number created (with no tile
    // at all, block 0)
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = nt_run == 0 || atomicAdd(&ctr->done_upd, my_tiles) + my_tiles == (int)nt_run;
    }
    __syncthreads();
    if (!s_last) return;
#ifdef SPHBUF_TRACE
    if (threadIdx.x == 0) g_trace_k[2] = gtimer();
#endif
    __threadfence();
    const long long nt = ntiles < ws.upd_tiles ? ntiles : ws.upd_tiles;
    unsigned carry_in = 0;
    // kPer consecutive tile counts per thread, all loaded before any is used
    constexpr int kPer = 8;
    for (long long b0 = 0; b0 < nt; b0 += (long long)kThreads * kPer) {
        const long long t0 = b0 + (long long)threadIdx.x * kPer;
        unsigned c[kPer], sum = 0;
#pragma unroll
        for (int e = 0; e < kPer; ++e) c[e] = t0 + e < nt ? __ldcg(ws.tile_cr + t0 + e) : 0u;
#pragma unroll
        for (int e = 0; e < kPer; ++e) sum += c[e];
        unsigned tot;
        unsigned run = carry_in + block_excl_scan<kThreads>(sum, tot, s_warp);
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            if (t0 + e < nt) ws.tile_pre[t0 + e] = run;
            run += c[e];
        }
        carry_in += tot;
    }
    if (threadIdx.x == 0) {
        ctr->n_stage = carry_in;
        ctr->done_upd = 0;
    }
    // the per-port counts (accumulated in the workspace) to the caller's array
    for (int i = threadIdx.x; i < 2 * max_ports; i += blockDim.x) port_counts[i] = __ldcg(ws.port_cnt + i);
#ifdef SPHBUF_TRACE
    if (threadIdx.x == 0) g_trace_k[3] = gtimer();
#endif
}


#ifdef SPHBUF_TRACE
}  // namespace sphbuf
extern "C" int sph_trace_read(unsigned long long *host, int max_tiles)
{
    const int n = max_tiles < sphbuf::kTraceTiles ? max_tiles : sphbuf::kTraceTiles;
    return (int)cudaMemcpyFromSymbol(host, sphbuf::g_trace, sizeof(unsigned long long) * 7 * n);
}
extern "C" int sph_trace_kernel(unsigned long long *host, int reset)
{
    cudaError_t e = cudaMemcpyFromSymbol(host, sphbuf::g_trace_k, sizeof(unsigned long long) * 4);
    if (reset) {
        const unsigned long long init[4] = {~0ull, 0ull, 0ull, 0ull};
        cudaMemcpyToSymbol(sphbuf::g_trace_k, init, sizeof(init));
        static unsigned long long zero[sphbuf::kTraceTiles][7];
        cudaMemcpyToSymbol(sphbuf::g_trace, zero, sizeof(zero));
    }
    return (int)e;
}
namespace sphbuf {
#endif

// ------------------------------------------------------------------ launchers

cudaError_t launch_advect(const PartDev &p, int dim, float dt, cudaStream_t s, Launch *L)
{
    L->before(s);
    launch_k(k_advect, dim3(cap_grid(sm_count_cached() * 8, p.cap, kThreads)), dim3(kThreads), 0, s, p, dim, dt);
    L->after(s, KID_ADVECT);
    return cudaGetLastError();
}

cudaError_t launch_register(const PartDev &p, const GridDev &g, const PortTable &pt, int k, long long *members,
                            cudaStream_t s, Launch *L)
{
    L->before(s);
    launch_k(k_register, dim3(cap_grid(sm_count_cached() * 8, p.cap, kThreads)), dim3(kThreads), 0, s, p, g.dim, pt.p[k], k, members);
    L->after(s, KID_REGISTER);
    return cudaGetLastError();
}

cudaError_t launch_update(const PartDev &p, const GridDev &g, const PortTable &pt, const Workspace &ws, int n_runs,
                          const int *cell_start, const int *cell_end, int *port_counts, int carry, float cdt,
                          bool prologue_done, cudaStream_t s, Launch *L)
{
    if (!prologue_done) {
        L->before(s);
        const int pro_blocks = n_runs > 0 ? (n_runs + 1023) / 1024 : 1;
        launch_k(k_upd_prologue, dim3(pro_blocks), dim3(1024), 0, s, ws, n_runs, cell_start, cell_end, pt.max_ports);
        L->after(s, KID_UPD_PROLOGUE);
    }
    // SPHBUF_TILE_RUNS=<n> lowers the number of runs a tile stages in shared memory
    // (tests force the global-search path with 0)
    static const int trmax = [] {
        const char *e = getenv("SPHBUF_TILE_RUNS");
        const int v = e ? atoi(e) : kTileRuns;
        return v < kTileRuns ? (v < 0 ? 0 : v) : kTileRuns;
    }();
    // SPHBUF_UPD=<min blocks per SM>:<speculative loads 0/1> for tuning runs
    static const char *uv = getenv("SPHBUF_UPD");
    const char *v = uv ? uv : "";
    L->before(s);
#define SPH_UPD(name, M, SP)                                                                                      \
    if (!strcmp(v, name)) {                                                                                       \
        static int grid = 0;                                                                                      \
        if (!grid) grid = occ_grid(k_upd_main<M, SP>, kThreads);                                                 \
        launch_k(k_upd_main<M, SP>, dim3(cap_grid(grid, ws.upd_tiles, 1)), dim3(kThreads), 0, s, p, g, pt, ws,   \
                 n_runs, cell_start, port_counts, carry, cdt, trmax);                                             \
        L->after(s, KID_UPD_MAIN);                                                                                \
        return cudaGetLastError();                                                                                \
    }
    SPH_UPD("3:0", 3, false)
    SPH_UPD("4:1", 4, true)
    SPH_UPD("5:0", 5, false)
    SPH_UPD("5:1", 5, true)
    SPH_UPD("6:0", 6, false)
    SPH_UPD("6:1", 6, true)
    SPH_UPD("8:1", 8, true)
#undef SPH_UPD
    static int grid = 0;
    if (!grid) grid = occ_grid(k_upd_main<4, false>, kThreads);
    launch_k(k_upd_main<4, false>, dim3(cap_grid(grid, ws.upd_tiles, 1)), dim3(kThreads), 0, s, p, g, pt, ws, n_runs,
             cell_start, port_counts, carry, cdt, trmax);
    L->after(s, KID_UPD_MAIN);
    return cudaGetLastError();
}

}  // namespace sphbuf
