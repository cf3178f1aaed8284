// Practical HBM ceiling for the gather's access pattern: copy a C5-sized SoA
// state (x, y, z, vx, vy, vz fp32, id int64, label int32 = 36 B per particle)
// from one buffer to another through a 4-byte slot -> source map (identity, or a
// local shuffle inside 512-slot tiles), plus a 4-byte key write, vs. a plain
// single-array copy of the same byte count.  Prints GB/s of bytes moved.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o soa tools/soa_copy_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

struct Cols {
    float *x, *y, *z, *vx, *vy, *vz;
    long long *id;
    int *label;
};

__global__ void copy1(const int4 *__restrict__ a, int4 *__restrict__ b, long long n4)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
        b[i] = a[i];
}

template <int ITEMS>
__global__ void __launch_bounds__(256) soa_gather(Cols in, Cols out, const int *__restrict__ src, int *key, long long n)
{
    const long long stride = (long long)gridDim.x * 256 * ITEMS;
    for (long long j0 = (long long)blockIdx.x * 256 * ITEMS; j0 < n; j0 += stride) {
        int s[ITEMS];
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            const long long j = j0 + it * 256 + threadIdx.x;
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
            const long long d = j0 + it * 256 + threadIdx.x;
            out.x[d] = x[it]; out.y[d] = y[it]; out.z[d] = z[it];
            out.vx[d] = vx[it]; out.vy[d] = vy[it]; out.vz[d] = vz[it];
            out.id[d] = id[it]; out.label[d] = lab[it];
            key[d] = lab[it] ^ (int)id[it];
        }
    }
}

__global__ void make_src(int *src, long long n, int shuffle)
{
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
        long long s = j;
        if (shuffle) {   // a permutation inside each 512-slot tile
            const long long t = j & ~511LL;
            s = t + ((j - t) * 97 + 13) % 512;
            if (s >= n) s = j;
        }
        src[j] = (int)s;
    }
}

// columns carved from one allocation, column k starting k * stagger bytes past a
// multiple of the column size (stagger < 0: separate cudaMalloc per column)
static Cols alloc_cols_stag(long long n, long long stagger)
{
    const long long col = ((8 * n + (1 << 21) - 1) >> 21) << 21;   // 2 MB-rounded column slot
    char *base;
    cudaMalloc(&base, 8 * col + 8 * stagger + 4096);
    cudaMemset(base, 0, 8 * col + 8 * stagger + 4096);
    auto at = [&](int k) { return base + k * col + k * stagger; };
    Cols c;
    c.x = (float *)at(0); c.y = (float *)at(1); c.z = (float *)at(2);
    c.vx = (float *)at(3); c.vy = (float *)at(4); c.vz = (float *)at(5);
    c.id = (long long *)at(6); c.label = (int *)at(7);
    return c;
}

static Cols alloc_cols(long long n)
{
    Cols c;
    cudaMalloc(&c.x, 4 * n); cudaMalloc(&c.y, 4 * n); cudaMalloc(&c.z, 4 * n);
    cudaMalloc(&c.vx, 4 * n); cudaMalloc(&c.vy, 4 * n); cudaMalloc(&c.vz, 4 * n);
    cudaMalloc(&c.id, 8 * n); cudaMalloc(&c.label, 4 * n);
    cudaMemset(c.x, 0, 4 * n); cudaMemset(c.y, 0, 4 * n); cudaMemset(c.z, 0, 4 * n);
    cudaMemset(c.vx, 0, 4 * n); cudaMemset(c.vy, 0, 4 * n); cudaMemset(c.vz, 0, 4 * n);
    cudaMemset(c.id, 0, 8 * n); cudaMemset(c.label, 0, 4 * n);
    return c;
}

int main()
{
    const long long n = 127545055;
    Cols a = alloc_cols(n), b = alloc_cols(n);
    int *src, *key;
    cudaMalloc(&src, 4 * n);
    cudaMalloc(&key, 4 * n);
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    // plain copy of the same bytes (76 B per particle moved: 36 + 36 + 4)
    const long long bytes = 36LL * n;
    int4 *p, *q;
    cudaMalloc(&p, bytes);
    cudaMalloc(&q, bytes);
    cudaMemset(p, 0, bytes);
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        copy1<<<sms * 8, 256>>>(p, q, bytes / 16);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("plain int4 copy of 36 B/particle: %.3f ms, %.0f GB/s (read+write)\n", ms, 2.0 * bytes / ms / 1e6);
    }
    for (int shuffle = 0; shuffle < 2; ++shuffle) {
        make_src<<<sms * 8, 256>>>(src, n, shuffle);
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(e0);
            soa_gather<2><<<sms * 5, 256>>>(a, b, src, key, n);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("SoA gather (%s map, 2 slots/thread, 5 blocks/SM): %.3f ms, %.0f GB/s of 80 B/particle\n",
                   shuffle ? "tile-shuffled" : "identity", ms, 80.0 * n / ms / 1e6);
        }
        for (int r = 0; r < 2; ++r) {
            cudaEventRecord(e0);
            soa_gather<4><<<sms * 4, 256>>>(a, b, src, key, n);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("SoA gather (%s map, 4 slots/thread, 4 blocks/SM): %.3f ms, %.0f GB/s of 80 B/particle\n",
                   shuffle ? "tile-shuffled" : "identity", ms, 80.0 * n / ms / 1e6);
        }
    }
    make_src<<<sms * 8, 256>>>(src, n, 0);
    const long long staggers[] = {0, 256, 1024, 4096, 65536, 1 << 20};
    for (long long st : staggers) {
        Cols a2 = alloc_cols_stag(n, st), b2 = alloc_cols_stag(n, st + 128);
        for (int r = 0; r < 2; ++r) {
            cudaEventRecord(e0);
            soa_gather<2><<<sms * 5, 256>>>(a2, b2, src, key, n);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("one allocation, column stagger %lld B (out +128): identity map %.3f ms, %.0f GB/s\n", st, ms,
                   80.0 * n / ms / 1e6);
        }
        cudaFree(a2.x);
        cudaFree(b2.x);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
