// sphbuf_migrate.cu — multi-GPU x-slab migration: pack particles
// whose pinned cell left the slab into fixed-size neighbour buffers, and append a
// received buffer at the tail.  The exchange itself is NCCL (torch.distributed).
#include <climits>
#include <cstdint>

#include "sphbuf_common.cuh"

namespace sphbuf {

// ------------------------------------------------------------------ multi-GPU slab migration

__global__ void __launch_bounds__(kThreads) k_mig_pack(PartDev p, GridDev g, Workspace ws, float *blo, float *bhi,
                                                       long long maxm, int rec)
{
    pdl_entry();
    const long long n = *p.n;
    long long moved = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        if (p.label[i] <= -2) continue;
        int oob = 0;
        const int cx = cell_axis(p.x[i], g.lo[0], g.inv_cs, 0, g.ncell[0], oob);
        float *buf = cx < g.cx_begin ? blo : (cx >= g.cx_end ? bhi : nullptr);
        if (!buf) continue;
        const int slot = atomicAdd(reinterpret_cast<int *>(buf), 1);
        if (slot >= maxm) {
            atomicOr(&ws.ctr->status, kStMigrate);
            continue;
        }
        float *r = buf + 4 + (long long)slot * rec;
        int w = 0;
        r[w++] = p.x[i];
        r[w++] = p.y[i];
        if (g.dim == 3) r[w++] = p.z[i];
        r[w++] = p.vx[i];
        r[w++] = p.vy[i];
        if (g.dim == 3) r[w++] = p.vz[i];
        for (int e = 0; e < p.n_extra; ++e) r[w++] = p.extra[e][i];
        const long long id = p.id[i];
        r[w++] = __int_as_float((int)(id & 0xffffffffll));
        r[w++] = __int_as_float((int)(id >> 32));
        r[w++] = __int_as_float(p.label[i]);
        p.label[i] = -3;  // migrated away: dropped by the next cell-list build
        ++moved;
    }
    moved = warp_sum_ll(moved);
    if ((threadIdx.x & 31) == 0 && moved) atomicAdd((unsigned long long *)&ws.ctr->migrated, (unsigned long long)moved);
}

// one block: append a received buffer at the tail
__global__ void __launch_bounds__(1024) k_mig_unpack(PartDev p, int dim, Workspace ws, const float *buf,
                                                     long long maxm, int rec)
{
    pdl_entry();
    const long long n = *p.n;
    long long cnt = __float_as_int(buf[0]);
    if (cnt > maxm) cnt = maxm;
    if (n + cnt > p.cap) {
        if (threadIdx.x == 0) atomicOr(&ws.ctr->status, kStCapacity);
        cnt = p.cap - n;
    }
    for (long long s = threadIdx.x; s < cnt; s += blockDim.x) {
        const float *r = buf + 4 + s * rec;
        const long long d = n + s;
        int w = 0;
        p.x[d] = r[w++];
        p.y[d] = r[w++];
        if (dim == 3) p.z[d] = r[w++];
        p.vx[d] = r[w++];
        p.vy[d] = r[w++];
        if (dim == 3) p.vz[d] = r[w++];
        for (int e = 0; e < p.n_extra; ++e) p.extra[e][d] = r[w++];
        const long long lo = (unsigned)__float_as_int(r[w++]);
        const long long hi = __float_as_int(r[w++]);
        p.id[d] = (hi << 32) | lo;
        p.label[d] = __float_as_int(r[w++]);
    }
    __syncthreads();
    if (threadIdx.x == 0) *p.n = n + cnt;
}


// ------------------------------------------------------------------ launchers

cudaError_t launch_migrate_pack(const PartDev &p, const GridDev &g, const Workspace &ws, float *lo, float *hi,
                                long long max_migrate, int rec, cudaStream_t s, Launch *L)
{
    cudaError_t e = cudaMemsetAsync(lo, 0, 16, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(hi, 0, 16, s);
    if (e != cudaSuccess) return e;
    L->before(s);
    launch_k(k_mig_pack, dim3(cap_grid(sm_count_cached() * 8, p.cap, kThreads)), dim3(kThreads), 0, s, p, g, ws, lo, hi, max_migrate, rec);
    L->after(s, KID_MIG_PACK);
    return cudaGetLastError();
}

cudaError_t launch_migrate_unpack(const PartDev &p, const GridDev &g, const Workspace &ws, const float *buf,
                                  long long max_migrate, int rec, cudaStream_t s, Launch *L)
{
    L->before(s);
    launch_k(k_mig_unpack, dim3(1), dim3(1024), 0, s, p, g.dim, ws, buf, max_migrate, rec);
    L->after(s, KID_MIG_UNPACK);
    return cudaGetLastError();
}

}  // namespace sphbuf
