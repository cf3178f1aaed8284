// Scatter design probe on a C5-shaped key stream (timing only, no library code):
//   cur    - the library's K3: match.any groups, one cursor atomic per distinct key, slot = start + cursor
//   packed - in-cell offset carried in the key's high byte (cell | off << 24): slot = start + off, no atomic
//   dirty  - packed, plus a private start table whose bit 31 marks cells the update corrected (0.1%):
//            their particles take the cursor atomic as in `cur`
//   byte   - offset in a separate uint8 column
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sop tools/scatter_offset_probe.cu && ./sop
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ unsigned lanemask_lt() { unsigned m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }

template <int IT, int NT>
__global__ void __launch_bounds__(NT) k_cur(const int *key, int *cursor, const int *start, int *src, long long n)
{
    const long long stride = (long long)gridDim.x * NT * IT;
    for (long long base = (long long)blockIdx.x * NT * IT; base < n; base += stride) {
        int k[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) { long long i = base + it * NT + threadIdx.x; k[it] = i < n ? key[i] : -1; }
        const int lane = threadIdx.x & 31; const unsigned lt = lanemask_lt();
        int b[IT], hl[IT], rl[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            unsigned g = __match_any_sync(0xffffffffu, k[it]);
            hl[it] = __ffs(g) - 1; rl[it] = __popc(g & lt);
            b[it] = (hl[it] == lane && k[it] >= 0) ? atomicAdd(&cursor[k[it]], __popc(g)) : 0;
        }
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            int rk = __shfl_sync(0xffffffffu, b[it], hl[it]) + rl[it];
            long long i = base + it * NT + threadIdx.x;
            if (i < n && k[it] >= 0) src[__ldg(start + k[it]) + rk] = (int)i;
        }
    }
}

template <int IT, int NT>
__global__ void __launch_bounds__(NT) k_packed(const int *key, const int *start, int *src, long long n)
{
    const long long stride = (long long)gridDim.x * NT * IT;
    for (long long base = (long long)blockIdx.x * NT * IT; base < n; base += stride) {
        int k[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) { long long i = base + it * NT + threadIdx.x; k[it] = i < n ? key[i] : -1; }
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            long long i = base + it * NT + threadIdx.x;
            if (i < n && k[it] >= 0) src[__ldg(start + (k[it] & 0xffffff)) + ((unsigned)k[it] >> 24)] = (int)i;
        }
    }
}

template <int IT, int NT>
__global__ void __launch_bounds__(NT) k_dirty(const int *key, int *cursor, const int *sstart, int *src, long long n)
{
    const long long stride = (long long)gridDim.x * NT * IT;
    for (long long base = (long long)blockIdx.x * NT * IT; base < n; base += stride) {
        int k[IT], s[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) { long long i = base + it * NT + threadIdx.x; k[it] = i < n ? key[i] : -1; }
#pragma unroll
        for (int it = 0; it < IT; ++it) s[it] = k[it] >= 0 ? __ldg(sstart + (k[it] & 0xffffff)) : 0;
        bool anyd = false;
#pragma unroll
        for (int it = 0; it < IT; ++it) anyd |= s[it] < 0;
        if (__any_sync(0xffffffffu, anyd)) {
            const int lane = threadIdx.x & 31; const unsigned lt = lanemask_lt();
#pragma unroll
            for (int it = 0; it < IT; ++it) {
                const int c = (s[it] < 0) ? (k[it] & 0xffffff) : -1;
                unsigned g = __match_any_sync(0xffffffffu, c);
                int hl = __ffs(g) - 1, rl = __popc(g & lt);
                int b = (hl == lane && c >= 0) ? atomicAdd(&cursor[c], __popc(g)) : 0;
                b = __shfl_sync(0xffffffffu, b, hl) + rl;
                if (c >= 0) s[it] = (s[it] & 0x7fffffff) + b - ((unsigned)k[it] >> 24);
            }
        }
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            long long i = base + it * NT + threadIdx.x;
            if (i < n && k[it] >= 0) src[s[it] + ((unsigned)k[it] >> 24)] = (int)i;
        }
    }
}

template <int IT, int NT>
__global__ void __launch_bounds__(NT) k_byte(const int *key, const unsigned char *off, const int *start, int *src, long long n)
{
    const long long stride = (long long)gridDim.x * NT * IT;
    for (long long base = (long long)blockIdx.x * NT * IT; base < n; base += stride) {
        int k[IT]; int o[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) { long long i = base + it * NT + threadIdx.x; k[it] = i < n ? key[i] : -1; o[it] = i < n ? off[i] : 0; }
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            long long i = base + it * NT + threadIdx.x;
            if (i < n && k[it] >= 0) src[__ldg(start + k[it]) + o[it]] = (int)i;
        }
    }
}

int main()
{
    // C5-like: 307 x 154 x 154 occupied cells of ~17.4 particles, x-major; 10% move to a neighbour
    const int nx = 307, ny = 154, nz = 154;
    const long long nc = (long long)nx * ny * nz;
    const int per = 17;
    std::mt19937_64 rng(7);
    std::vector<int> key; key.reserve(nc * 18);
    for (long long c = 0; c < nc; ++c) {
        int m = per + (rng() % 3 == 0);
        for (int j = 0; j < m; ++j) {
            long long k = c;
            if (rng() % 10 == 0) {
                long long d[6] = {1, -1, nz, -(long long)nz, (long long)ny * nz, -(long long)ny * nz};
                long long t = c + d[rng() % 6];
                if (t >= 0 && t < nc) k = t;
            }
            key.push_back((int)k);
        }
    }
    const long long n = key.size();
    std::vector<int> cnt(nc, 0), start(nc), pk(n), sst(nc);
    std::vector<unsigned char> ob(n);
    for (long long i = 0; i < n; ++i) { int o = cnt[key[i]]++; ob[i] = (unsigned char)o; pk[i] = key[i] | (o << 24); }
    long long s = 0; int mx = 0;
    for (long long c = 0; c < nc; ++c) { start[c] = (int)s; s += cnt[c]; if (cnt[c] > mx) mx = cnt[c]; }
    for (long long c = 0; c < nc; ++c) sst[c] = start[c] | ((rng() % 1000 == 0) ? (int)0x80000000 : 0);
    // dirty cells: their particles' offsets are meaningless (0) and take the atomic path
    for (long long i = 0; i < n; ++i) if (sst[key[i]] < 0) pk[i] = key[i];
    printf("n=%lld cells=%lld max cell=%d\n", n, nc, mx);
    int *dk, *dpk, *dcur, *dst, *dsst, *dsrc; unsigned char *dob;
    CK(cudaMalloc(&dk, n * 4)); CK(cudaMalloc(&dpk, n * 4)); CK(cudaMalloc(&dsrc, n * 4)); CK(cudaMalloc(&dob, n));
    CK(cudaMalloc(&dcur, nc * 4)); CK(cudaMalloc(&dst, nc * 4)); CK(cudaMalloc(&dsst, nc * 4));
    CK(cudaMemcpy(dk, key.data(), n * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dpk, pk.data(), n * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dob, ob.data(), n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dst, start.data(), nc * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dsst, sst.data(), nc * 4, cudaMemcpyHostToDevice));
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    std::vector<int> hsrc(n);
    auto check = [&](const char *nm) {
        CK(cudaMemcpy(hsrc.data(), dsrc, n * 4, cudaMemcpyDeviceToHost));
        std::vector<char> seen(n, 0); long long bad = 0;
        for (long long j = 0; j < n; ++j) { int v = hsrc[j]; if (v < 0 || v >= n || seen[v]) ++bad; else { seen[v] = 1; if (j < start[key[v]] || j >= start[key[v]] + cnt[key[v]]) ++bad; } }
        printf("  %s: %s\n", nm, bad ? "WRONG" : "valid permutation");
    };
    auto run = [&](const char *nm, auto launch) {
        float best = 1e9, sum = 0; const int R = 10;
        for (int r = 0; r < R + 2; ++r) {
            CK(cudaMemset(dcur, 0, nc * 4)); CK(cudaMemset(dsrc, 0xff, n * 4));
            cudaEventRecord(a); launch(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b); if (r >= 2) { sum += ms; if (ms < best) best = ms; }
        }
        printf("%-22s mean %.4f ms  best %.4f ms\n", nm, sum / R, best);
        check(nm);
    };
#define GRID(IT, NT) dim3((unsigned)(((n + (long long)NT * IT - 1) / ((long long)NT * IT)) < (long long)sms * 8 * 256 / NT ? ((n + (long long)NT * IT - 1) / ((long long)NT * IT)) : (long long)sms * 8 * 256 / NT))
    run("cur 4x256", [&] { k_cur<4, 256><<<GRID(4, 256), 256>>>(dk, dcur, dst, dsrc, n); });
    run("packed 4x256", [&] { k_packed<4, 256><<<GRID(4, 256), 256>>>(dpk, dst, dsrc, n); });
    run("packed 8x256", [&] { k_packed<8, 256><<<GRID(8, 256), 256>>>(dpk, dst, dsrc, n); });
    run("packed 2x256", [&] { k_packed<2, 256><<<GRID(2, 256), 256>>>(dpk, dst, dsrc, n); });
    run("dirty 4x256", [&] { k_dirty<4, 256><<<GRID(4, 256), 256>>>(dpk, dcur, dsst, dsrc, n); });
    run("dirty 8x256", [&] { k_dirty<8, 256><<<GRID(8, 256), 256>>>(dpk, dcur, dsst, dsrc, n); });
    run("byte 4x256", [&] { k_byte<4, 256><<<GRID(4, 256), 256>>>(dk, dob, dst, dsrc, n); });
    return 0;
}
