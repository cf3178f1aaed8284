// Access-pattern probe for a copy-engine gather: the C5-sized SoA state (x, y, z,
// vx, vy, vz fp32, id int64, label int32 = 36 B per particle) gathered through a
// slot -> source map in which most slots are "stayers" (source near the slot,
// as after one SPH step: ~90%) and the rest come from far away (cell changers).
//   A: plain loads through the map (the current gather's pattern, no ranking)
//   B: per 512-slot tile, the source window [j0 - H, j0 + T + H) of every column
//      brought into shared memory by cp.async.bulk (one producer warp, S stages,
//      mbarrier completion); stayers read from shared memory, far sources by
//      plain loads; stores as in A.
// Prints ms and GB/s of 80 B/particle (map 4 + 36 read + 36 written + key 4).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gtp tools/gather_tma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct Cols {
    float *x, *y, *z, *vx, *vy, *vz;
    long long *id;
    int *label;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                     smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int ITEMS>
__global__ void __launch_bounds__(256) gather_ldg(Cols in, Cols out, const int *__restrict__ src, int *key, int n)
{
    const int stride = gridDim.x * 256 * ITEMS;
    for (int j0 = blockIdx.x * 256 * ITEMS; j0 < n; j0 += stride) {
        int s[ITEMS];
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            const int j = j0 + it * 256 + threadIdx.x;
            s[it] = j < n ? src[j] : -1;
        }
        float x[ITEMS], y[ITEMS], z[ITEMS], vx[ITEMS], vy[ITEMS], vz[ITEMS];
        long long id[ITEMS];
        int lab[ITEMS];
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            if (s[it] < 0) continue;
            const int q = s[it];
            x[it] = in.x[q]; y[it] = in.y[q]; z[it] = in.z[q];
            vx[it] = in.vx[q]; vy[it] = in.vy[q]; vz[it] = in.vz[q];
            id[it] = in.id[q]; lab[it] = in.label[q];
        }
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            if (s[it] < 0) continue;
            const int d = j0 + it * 256 + threadIdx.x;
            out.x[d] = x[it]; out.y[d] = y[it]; out.z[d] = z[it];
            out.vx[d] = vx[it]; out.vy[d] = vy[it]; out.vz[d] = vz[it];
            out.id[d] = id[it]; out.label[d] = lab[it];
            key[d] = lab[it] ^ (int)id[it];
        }
    }
}

// A': A with the next tile's map prefetched (as k_cll_gather does), 5 blocks/SM
__global__ void __launch_bounds__(256, 5) gather_ldg_pf(Cols in, Cols out, const int *__restrict__ src, int *key, int n)
{
    constexpr int ITEMS = 2;
    const int stride = gridDim.x * 256 * ITEMS;
    int ns[ITEMS];
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
        const int j = blockIdx.x * 256 * ITEMS + it * 256 + threadIdx.x;
        ns[it] = j < n ? src[j] : -1;
    }
    for (int j0 = blockIdx.x * 256 * ITEMS; j0 < n; j0 += stride) {
        int s[ITEMS];
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) s[it] = ns[it];
        float x[ITEMS], y[ITEMS], z[ITEMS], vx[ITEMS], vy[ITEMS], vz[ITEMS];
        long long id[ITEMS];
        int lab[ITEMS];
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            if (s[it] < 0) continue;
            const int q = s[it];
            x[it] = in.x[q]; y[it] = in.y[q]; z[it] = in.z[q];
            vx[it] = in.vx[q]; vy[it] = in.vy[q]; vz[it] = in.vz[q];
            id[it] = in.id[q]; lab[it] = in.label[q];
        }
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            const int j = j0 + stride + it * 256 + threadIdx.x;
            ns[it] = (j0 < n - stride && j < n) ? src[j] : -1;
        }
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            if (s[it] < 0) continue;
            const int d = j0 + it * 256 + threadIdx.x;
            out.x[d] = x[it]; out.y[d] = y[it]; out.z[d] = z[it];
            out.vx[d] = vx[it]; out.vy[d] = vy[it]; out.vz[d] = vz[it];
            out.id[d] = id[it]; out.label[d] = lab[it];
            key[d] = lab[it] ^ (int)id[it];
        }
    }
}

// B: copy-engine windows.  Stage layout (elements): W = T + 2H + 8 per column.
template <int T, int H, int S>
struct Stage {
    static constexpr int W = T + 2 * H + 8;
    float f[6][W];
    long long id[W];
    int lab[W];
};

template <int T>
__device__ __forceinline__ int tile_drift(const int *__restrict__ src, int j0, int n)
{
    const int lane = threadIdx.x & 31;
    const int j = j0 + lane * (T / 32);
    const int dl = j < n ? src[j] - j : 0;
    int below = 0, eq = 0;
    for (int l = 0; l < 32; ++l) {
        const int o = __shfl_sync(0xffffffffu, dl, l);
        below += o < dl;
        eq += (o == dl) & (l < lane);
    }
    const unsigned m = __ballot_sync(0xffffffffu, below + eq == 16);
    return __shfl_sync(0xffffffffu, dl, __ffs(m) - 1);
}

template <int T, int H, int S, int MINB>
__global__ void __launch_bounds__(T / 2 + 32, MINB) gather_tma(Cols in, Cols out, const int *__restrict__ src, int *key,
                                                              int n)
{
    constexpr int NC = T / 2;            // consumer threads, 2 slots each
    using St = Stage<T, H, S>;
    extern __shared__ __align__(128) unsigned char smem[];
    St *st = reinterpret_cast<St *>(smem);
    __shared__ uint64_t full[S], empty[S];
    __shared__ int wbeg[S], wend[S];
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NC / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int ntiles = (n + T - 1) / T;
    if (threadIdx.x >= NC) {
        // producer warp: one elected lane issues the window copies of this block's tiles
        const bool leader = threadIdx.x == NC;
        int k = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
            const int s = k % S;
            if (k >= S && leader) mbar_wait(&empty[s], ((k / S) - 1) & 1);
            const int j0 = t * T;
            // drift of the tile's sources: the median of 32 sampled (src - slot),
            // estimated by the whole producer warp
            int a = j0 - H + tile_drift<T>(src, j0, n);
            a = a < 0 ? 0 : a;
            a &= ~3;
            const int nf = n & ~3;
            a = a > nf - (T + 2 * H) ? nf - (T + 2 * H) : a;   // whole window inside [0, n & ~3)
            a = a < 0 ? 0 : a;
            int b = a + T + 2 * H;
            b = b > nf ? nf : b;
            if (leader) {
                wbeg[s] = a;
                wend[s] = b;
                const uint32_t ne = (uint32_t)(b - a);
                mbar_arrive_expect_tx(&full[s], ne * 36u);
                const float *cols[6] = {in.x, in.y, in.z, in.vx, in.vy, in.vz};
#pragma unroll
                for (int c = 0; c < 6; ++c) bulk_g2s(st[s].f[c], cols[c] + a, ne * 4u, &full[s]);
                bulk_g2s(st[s].id, in.id + a, ne * 8u, &full[s]);
                bulk_g2s(st[s].lab, in.label + a, ne * 4u, &full[s]);
            }
            __syncwarp();
        }
        return;
    }
    int k = 0;
    int nsrc[2];
    {
        const int j0 = blockIdx.x * T;
#pragma unroll
        for (int it = 0; it < 2; ++it) {
            const int j = j0 + it * NC + threadIdx.x;
            nsrc[it] = j < n ? src[j] : -1;
        }
    }
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int s = k % S;
        const int j0 = t * T;
        int sv[2] = {nsrc[0], nsrc[1]};
        const int tn = t + gridDim.x;
        if (tn < ntiles) {
#pragma unroll
            for (int it = 0; it < 2; ++it) {
                const int j = tn * T + it * NC + threadIdx.x;
                nsrc[it] = j < n ? src[j] : -1;
            }
        }
        // far sources first (plain loads), then the window
        float x[2], y[2], z[2], vx[2], vy[2], vz[2];
        long long id[2];
        int lab[2];
        mbar_wait(&full[s], (k / S) & 1);
        const int a = wbeg[s];
        const int b = wend[s] + 8;
#pragma unroll
        for (int it = 0; it < 2; ++it) {
            const int q = sv[it];
            if (q < 0) continue;
            if (q >= a && q < b - 8) {
                const int r = q - a;
                x[it] = st[s].f[0][r]; y[it] = st[s].f[1][r]; z[it] = st[s].f[2][r];
                vx[it] = st[s].f[3][r]; vy[it] = st[s].f[4][r]; vz[it] = st[s].f[5][r];
                id[it] = st[s].id[r]; lab[it] = st[s].lab[r];
            } else {
                x[it] = in.x[q]; y[it] = in.y[q]; z[it] = in.z[q];
                vx[it] = in.vx[q]; vy[it] = in.vy[q]; vz[it] = in.vz[q];
                id[it] = in.id[q]; lab[it] = in.label[q];
            }
        }
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
#pragma unroll
        for (int it = 0; it < 2; ++it) {
            if (sv[it] < 0) continue;
            const int d = j0 + it * NC + threadIdx.x;
            out.x[d] = x[it]; out.y[d] = y[it]; out.z[d] = z[it];
            out.vx[d] = vx[it]; out.vy[d] = vy[it]; out.vz[d] = vz[it];
            out.id[d] = id[it]; out.label[d] = lab[it];
            key[d] = lab[it] ^ (int)id[it];
        }
    }
}

// stayers: source = slot; far: source = slot +- one of a few strides, clamped
__global__ void make_src(int *src, int n, int far_permille)
{
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        unsigned h = (unsigned)j * 2654435761u;
        h ^= h >> 15;
        h *= 2246822519u;
        h ^= h >> 13;
        long long s = j;
        if ((int)(h % 1000) < far_permille) {
            const int strides[4] = {17, 3050, 530000, 531000};
            const int st = strides[(h >> 10) & 3];
            s = (h >> 12) & 1 ? j + st : j - st;
            if (s < 0 || s >= n) s = j;
        }
        src[j] = (int)s;
    }
}

static Cols alloc_cols(long long n)
{
    Cols c;
    cudaMalloc(&c.x, 4 * n + 64); cudaMalloc(&c.y, 4 * n + 64); cudaMalloc(&c.z, 4 * n + 64);
    cudaMalloc(&c.vx, 4 * n + 64); cudaMalloc(&c.vy, 4 * n + 64); cudaMalloc(&c.vz, 4 * n + 64);
    cudaMalloc(&c.id, 8 * n + 64); cudaMalloc(&c.label, 4 * n + 64);
    cudaMemset(c.x, 0, 4 * n); cudaMemset(c.y, 0, 4 * n); cudaMemset(c.z, 0, 4 * n);
    cudaMemset(c.vx, 0, 4 * n); cudaMemset(c.vy, 0, 4 * n); cudaMemset(c.vz, 0, 4 * n);
    cudaMemset(c.id, 0, 8 * n); cudaMemset(c.label, 0, 4 * n);
    return c;
}

template <int T, int H, int S, int MINB>
static void run_tma(Cols a, Cols b, int *src, int *key, int n, int sms, cudaEvent_t e0, cudaEvent_t e1)
{
    const int smem = (int)sizeof(Stage<T, H, S>) * S;
    cudaFuncSetAttribute(gather_tma<T, H, S, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, gather_tma<T, H, S, MINB>, T / 2 + 32, smem);
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        gather_tma<T, H, S, MINB><<<sms * per, T / 2 + 32, smem>>>(a, b, src, key, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("  TMA windows T=%d H=%d S=%d (%d blocks/SM, %d KB smem): %.3f ms, %.0f GB/s  [%s]\n", T, H, S, per,
               smem / 1024, ms, 80.0 * n / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
}

int main(int argc, char **argv)
{
    int n = 127545055;
    int *hmap = nullptr;
    if (argc > 1) {           // a real slot -> source map (int32, from tools/map_window_stats.py --dump)
        FILE *f = fopen(argv[1], "rb");
        fseek(f, 0, SEEK_END);
        n = (int)(ftell(f) / 4);
        fseek(f, 0, SEEK_SET);
        hmap = new int[n];
        if (fread(hmap, 4, n, f) != (size_t)n) return 1;
        fclose(f);
    }
    Cols a = alloc_cols(n), b = alloc_cols(n);
    int *src, *key;
    cudaMalloc(&src, 4LL * n);
    cudaMalloc(&key, 4LL * n);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int fars[] = {0, 100, -1};
    for (int far : fars) {
        if (far >= 0) {
            if (hmap) continue;
            make_src<<<sms * 8, 256>>>(src, n, far);
            printf("far sources: %d permille\n", far);
        } else {
            if (!hmap) continue;
            cudaMemcpy(src, hmap, 4LL * n, cudaMemcpyHostToDevice);
            printf("real map from %s (%d slots)\n", argv[1], n);
        }
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(e0);
            gather_ldg<2><<<sms * 5, 256>>>(a, b, src, key, n);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("  plain loads (2 slots, 5 blocks/SM): %.3f ms, %.0f GB/s\n", ms, 80.0 * n / ms / 1e6);
        }
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(e0);
            gather_ldg_pf<<<sms * 5, 256>>>(a, b, src, key, n);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("  plain loads, map prefetched (2 slots, 5 blocks/SM): %.3f ms, %.0f GB/s\n", ms, 80.0 * n / ms / 1e6);
        }
        run_tma<512, 64, 2, 1>(a, b, src, key, n, sms, e0, e1);
        run_tma<512, 64, 3, 1>(a, b, src, key, n, sms, e0, e1);
        run_tma<512, 64, 4, 1>(a, b, src, key, n, sms, e0, e1);
        run_tma<1024, 64, 2, 1>(a, b, src, key, n, sms, e0, e1);
        run_tma<1024, 64, 3, 1>(a, b, src, key, n, sms, e0, e1);
        run_tma<256, 64, 4, 1>(a, b, src, key, n, sms, e0, e1);
        run_tma<256, 64, 6, 1>(a, b, src, key, n, sms, e0, e1);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
