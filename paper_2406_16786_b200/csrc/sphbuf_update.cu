// sphbuf_update.cu — registration (Alg. 1 identification), the driver's advection,
// and the buffer update: candidate transform + axial compare (a3), inflow
// generation (a4), outflow deletion (a5) and relabel (a6), fused in one pass over
// the candidates of the port cell runs (arXiv 2406.16786 §III).
#include <climits>
#include <cstdint>

#include "sphbuf_common.cuh"

namespace sphbuf {

// ------------------------------------------------------------------ driver: advection

__global__ void __launch_bounds__(kThreads) k_advect(PartDev p, int dim, float dt)
{
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

// Update tiles are static groups of kRunGroup consecutive port runs (runs are in
// canonical order: port-major, then cell), so no global scan of candidate
// offsets is needed: a block sizes its group from the cell tables itself.
constexpr int kRunGroup = 16;

// K5: resets the per-update counters and the caller's per-port counts.
__global__ void __launch_bounds__(128) k_upd_prologue(Workspace ws, int *port_counts, int max_ports)
{
    Counters *ctr = ws.ctr;
    if (threadIdx.x == 0) {
        ctr->epoch_upd += 1;
        ctr->ticket_upd = 0;
        ctr->n_stage = 0;
        ctr->n_del = 0;
        ctr->n_cand = 0;
        ctr->i_first = LLONG_MAX;
    }
    for (int i = threadIdx.x; i < 2 * max_ports; i += blockDim.x) port_counts[i] = 0;
}

// The decision of Alg. 1-3 for one candidate of port k (pure; pinned transform).
__device__ __forceinline__ void decide(const PortDev &P, int k, int dim, float x, float y, float z, int lab,
                                       float X[3], bool &inP, bool &create, bool &del)
{
    to_local(P, dim, x, y, z, X);
    inP = in_box(X, P.heP, dim);                         // x in P_k (reading R4)
    const bool member = (lab == k);
    const bool beyond = X[0] > P.he[0];                  // X'_0 > a/2
    create = false;
    del = false;
    if (!inP) return;
    if (P.kind == SPH_INLET) {
        create = member && beyond;                       // Alg. 1 (R5)
    } else if (P.kind == SPH_OUTLET) {
        del = beyond;                                    // Alg. 2 (R6)
    } else {
        create = member && beyond;                       // Alg. 3
        del = member && (X[0] < -P.he[0]);               // Alg. 3
    }
}

// K6: the candidate check (a3) with generation (a4), deletion (a5) and relabel
// (a6) fused.  Per group: pass 1 counts the CREATEs (read only), a decoupled
// look-back over the ordered groups gives the group's first staging slot, pass 2
// decides again and applies; CREATE slots inside the group follow the candidate
// order (port, cell, id) through a ballot scan per chunk.
__global__ void __launch_bounds__(kThreads) k_upd_main(PartDev p, int dim, const __grid_constant__ PortTable pt,
                                                       Workspace ws, int n_runs, const int *cell_start,
                                                       const int *cell_end, int *port_counts)
{
    __shared__ PortDev s_ports[SPH_MAX_PORTS];
    __shared__ unsigned s_cnt[kThreads / 32 + 1];
    __shared__ int s_beg[kRunGroup], s_port[kRunGroup], s_off[kRunGroup + 1];
    __shared__ long long s_tile;
    __shared__ unsigned s_prefix;
    {
        const int words = pt.n * (int)(sizeof(PortDev) / 4);
        const unsigned *src = reinterpret_cast<const unsigned *>(pt.p);
        unsigned *dst = reinterpret_cast<unsigned *>(s_ports);
        for (int w = threadIdx.x; w < words; w += blockDim.x) dst[w] = src[w];
    }
    Counters *ctr = ws.ctr;
    const unsigned epoch = ctr->epoch_upd;
    const long long ngroups = (n_runs + kRunGroup - 1) / kRunGroup;
    const int max_ports = pt.max_ports;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctr->epoch_cmp += 1;  // consumed by the compaction that follows
        ctr->ticket_cmp = 0;
        ctr->ticket_cmp2 = 0;
        if (ngroups > ws.upd_tiles) ctr->status |= kStCapacity;
    }
    long long del_cnt = 0, del_min = LLONG_MAX, motion = 0;
    __syncthreads();
    while (true) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->ticket_upd, 1);
        __syncthreads();
        const long long grp = s_tile;
        if (grp >= ngroups || grp >= ws.upd_tiles) break;
        if (warp == 0) {
            const long long r = grp * kRunGroup + lane;
            int len = 0;
            if (lane < kRunGroup && r < n_runs) {
                const int beg = cell_start[ws.runs[3 * r]];
                len = cell_end[ws.runs[3 * r + 1]] - beg;
                s_beg[lane] = beg;
                s_port[lane] = ws.runs[3 * r + 2];
            }
            int inc = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane < kRunGroup) s_off[lane] = inc - len;
            if (lane == kRunGroup - 1) s_off[kRunGroup] = inc;
        }
        __syncthreads();
        const int total = s_off[kRunGroup];
        // pass 1: CREATEs of the group (no writes)
        unsigned mine = 0;
        for (int q0 = 0; q0 < total; q0 += kThreads) {
            const int q = q0 + threadIdx.x;
            if (q >= total) continue;
            int r = 0;
            while (r + 1 < kRunGroup && s_off[r + 1] <= q) ++r;
            const int k = s_port[r];
            const int pi = s_beg[r] + (q - s_off[r]);
            float X[3];
            bool inP, cr, dl;
            decide(s_ports[k], k, dim, p.x[pi], p.y[pi], dim == 3 ? p.z[pi] : 0.0f, p.label[pi], X, inP, cr, dl);
            mine += cr;
        }
        mine = warp_sum(mine);
        if (lane == 0) s_cnt[warp] = mine;
        __syncthreads();
        if (warp == 0) {
            unsigned c = lane < kThreads / 32 ? s_cnt[lane] : 0u;
            c = warp_sum(c);
            const unsigned pre = tile_prefix(ws.tile_upd, grp, epoch, c);
            if (lane == 0) {
                s_prefix = pre;
                atomicAdd((unsigned long long *)&ctr->n_cand, (unsigned long long)total);
                atomicAdd((unsigned long long *)&ctr->checked, (unsigned long long)total);
                if (grp == ngroups - 1) ctr->n_stage = (long long)pre + c;
            }
        }
        __syncthreads();
        // pass 2: decide and apply
        long long run = s_prefix;
        for (int q0 = 0; q0 < total; q0 += kThreads) {
            const int q = q0 + threadIdx.x;
            bool cr[1] = {false};
            int pi = 0, k = 0;
            float x = 0.f, y = 0.f, z = 0.f;
            if (q < total) {
                int r = 0;
                while (r + 1 < kRunGroup && s_off[r + 1] <= q) ++r;
                k = s_port[r];
                pi = s_beg[r] + (q - s_off[r]);
                const PortDev &P = s_ports[k];
                x = p.x[pi];
                y = p.y[pi];
                z = dim == 3 ? p.z[pi] : 0.0f;
                const int lab = p.label[pi];
                float X[3];
                bool inP, create, del;
                decide(P, k, dim, x, y, z, lab, X, inP, create, del);
                // R12: a buffer particle outside its decision region moved more than
                // the one-cell margin in one step; it can no longer be generated/deleted
                if (lab == k && !inP) ++motion;
                float px = x, py = y, pz = z;
                if (create) {
                    // recycle: x <- fl(x - fl(a u)) (Eqs. 2D/3D_Inverse_transformation, R10)
                    px = __fsub_rn(x, P.s[0]);
                    py = __fsub_rn(y, P.s[1]);
                    p.x[pi] = px;
                    p.y[pi] = py;
                    if (dim == 3) {
                        pz = __fsub_rn(z, P.s[2]);
                        p.z[pi] = pz;
                    }
                    cr[0] = true;
                    atomicAdd(&port_counts[k], 1);
                }
                if (del) {
                    p.label[pi] = -2;                    // tombstone, removed by sph_compact
                    atomicAdd(&port_counts[max_ports + k], 1);
                    ++del_cnt;
                    del_min = pi < del_min ? pi : del_min;
                } else if (P.kind != SPH_INLET) {
                    // relabel on post-recycle positions (R9)
                    float Xp[3] = {X[0], X[1], X[2]};
                    if (create) to_local(P, dim, px, py, pz, Xp);
                    if (in_box(Xp, P.he, dim)) {
                        if (lab != k) p.label[pi] = k;
                    } else if (lab == k) {
                        p.label[pi] = -1;
                    }
                }
            }
            unsigned excl[1], tot;
            striped_scan<kThreads, 1>(cr, excl, tot, s_cnt);
            if (cr[0]) {
                const long long slot = run + excl[0];
                if (slot < ws.max_new) {
                    // duplicate = bitwise copy of the pre-recycle state, label fluid (R11)
                    ws.sx[slot] = x;
                    ws.sy[slot] = y;
                    ws.svx[slot] = p.vx[pi];
                    ws.svy[slot] = p.vy[pi];
                    if (dim == 3) {
                        ws.sz[slot] = z;
                        ws.svz[slot] = p.vz[pi];
                    }
                    for (int e = 0; e < p.n_extra; ++e) ws.sextra[e][slot] = p.extra[e][pi];
                    ws.sid[slot] = p.id[pi];
                    ws.sport[slot] = k;
                } else {
                    atomicOr(&ctr->status, kStStaging);
                }
            }
            run += tot;
        }
        __syncthreads();
    }
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
}

// ------------------------------------------------------------------ launchers

cudaError_t launch_advect(const PartDev &p, int dim, float dt, cudaStream_t s, Launch *L)
{
    L->before(s);
    k_advect<<<cap_grid(sm_count_cached() * 8, p.cap, kThreads), kThreads, 0, s>>>(p, dim, dt);
    L->after(s, KID_ADVECT);
    return cudaGetLastError();
}

cudaError_t launch_register(const PartDev &p, const GridDev &g, const PortTable &pt, int k, long long *members,
                            cudaStream_t s, Launch *L)
{
    L->before(s);
    k_register<<<cap_grid(sm_count_cached() * 8, p.cap, kThreads), kThreads, 0, s>>>(p, g.dim, pt.p[k], k, members);
    L->after(s, KID_REGISTER);
    return cudaGetLastError();
}

cudaError_t launch_update(const PartDev &p, const GridDev &g, const PortTable &pt, const Workspace &ws, int n_runs,
                          const int *cell_start, const int *cell_end, int *port_counts, cudaStream_t s, Launch *L)
{
    L->before(s);
    k_upd_prologue<<<1, 128, 0, s>>>(ws, port_counts, pt.max_ports);
    L->after(s, KID_UPD_PROLOGUE);
    static int grid = 0;
    if (!grid) grid = occ_grid(k_upd_main, kThreads);
    const long long ngroups = (n_runs + kRunGroup - 1) / kRunGroup;
    L->before(s);
    k_upd_main<<<cap_grid(grid, ngroups, 1), kThreads, 0, s>>>(p, g.dim, pt, ws, n_runs, cell_start, cell_end,
                                                               port_counts);
    L->after(s, KID_UPD_MAIN);
    return cudaGetLastError();
}

}  // namespace sphbuf
