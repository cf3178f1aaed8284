// Dependent-latency probe (pointer chase through L2 / HBM, atomic chain, store + fence,
// %globaltimer step): nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lp tools/latency_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void chase(const int *next, int steps, unsigned long long *out, int *sink)
{
    // pointer chase: dependent loads
    int p = 0;
    unsigned long long t0 = gt(); long long c0 = clock64();
    for (int i = 0; i < steps; ++i) p = __ldcg(next + p);
    long long c1 = clock64(); unsigned long long t1 = gt();
    out[0] = t1 - t0; out[1] = c1 - c0; *sink = p;
}
__global__ void atom_chase(int *ctr, int steps, unsigned long long *out)
{
    int v = 0;
    unsigned long long t0 = gt();
    for (int i = 0; i < steps; ++i) v = atomicAdd(ctr + (v & 0), 1);
    unsigned long long t1 = gt();
    out[2] = t1 - t0; out[3] = v;
}
__global__ void fence_cost(int *buf, int steps, unsigned long long *out)
{
    unsigned long long t0 = gt();
    for (int i = 0; i < steps; ++i) { buf[i * 32] = i; __threadfence(); }
    unsigned long long t1 = gt();
    out[4] = t1 - t0;
}
__global__ void timer_res(unsigned long long *out)
{
    unsigned long long a = gt(), b = a; int n = 0;
    while (b == a && n < 100000) { b = gt(); ++n; }
    out[5] = b - a; out[6] = n;
}
int main()
{
    const int N = 1 << 22; // 16 MB (fits L2) 
    int *h = new int[N];
    // random cyclic permutation with stride to defeat prefetch
    for (int i = 0; i < N; ++i) h[i] = (int)(((long long)i * 2654435761LL + 12345) % N);
    int *d, *sink; unsigned long long *out;
    cudaMalloc(&d, N * 4); cudaMalloc(&sink, 4); cudaMalloc(&out, 64);
    cudaMemcpy(d, h, N * 4, cudaMemcpyHostToDevice);
    unsigned long long o[8];
    for (int rep = 0; rep < 3; ++rep) {
        chase<<<1, 1>>>(d, 2000, out, sink);
        atom_chase<<<1, 1>>>(sink, 2000, out);
        fence_cost<<<1, 1>>>(d, 2000, out);
        timer_res<<<1, 1>>>(out);
        cudaMemcpy(o, out, 64, cudaMemcpyDeviceToHost);
        printf("dependent ldcg (L2, 16MB set): %.1f ns/hop (%.0f clk); atomic chain %.1f ns/op; store+threadfence %.1f ns; globaltimer step %llu ns\n",
               o[0] / 2000.0, o[1] / 2000.0, o[2] / 2000.0, o[4] / 2000.0, o[5]);
    }
    // DRAM set: 1 GB
    const long long M = 1LL << 28;
    int *d2; cudaMalloc(&d2, M * 4);
    int *h2 = new int[M];
    for (long long i = 0; i < M; ++i) h2[i] = (int)((i * 2654435761LL + 7) % M);
    cudaMemcpy(d2, h2, M * 4, cudaMemcpyHostToDevice);
    chase<<<1, 1>>>(d2, 2000, out, sink);
    cudaMemcpy(o, out, 64, cudaMemcpyDeviceToHost);
    printf("dependent ldcg (DRAM, 1GB set): %.1f ns/hop (%.0f clk)\n", o[0] / 2000.0, o[1] / 2000.0);
    return 0;
}
