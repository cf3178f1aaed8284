// sphbuf_drivers.cu — time-dependent port drivers (aorta flow, arXiv 2406.16786
// §V.D).  The Fourier inflow speed (Eq.
// Fourier_Series, Table I) is evaluated on the host; this file holds the device
// side of the 3-element Windkessel outlet (Eq. windkessel, Table II):
//   K11 k_drivers  one block per driven port: the flow rate out of the port,
//                  Q = V/a * sum over its buffer particles of v.n (reading R26),
//                  summed over the port's candidates of the current cell list in
//                  32.32 fixed point (exact, so independent of the summation
//                  order), then one explicit step of
//                  (1 + Rp/Rd) Q + C Rp dQ/dt = P/Rd + C dP/dt   (reading R27)
//                  and the recycled density fl32(rho0 + P / c0^2) of the port's
//                  pressure BC (Eq. postulate-density) for the update.
// All f64 arithmetic is one IEEE operation per step in the order written (no
// contraction, --fmad=false), the same order as the oracle's.
#include <cstdint>

#include "sphbuf_common.cuh"

namespace sphbuf {

// v.u pinned: fl(fl(fl(vx ux) + fl(vy uy)) + fl(vz uz)), then x 2^32 (exact) and
// rounded to the nearest integer (ties to even).
__device__ __forceinline__ long long flux_fixed(float vx, float vy, float vz, const float u[3], int dim)
{
    float d = __fadd_rn(__fmul_rn(vx, u[0]), __fmul_rn(vy, u[1]));
    if (dim == 3) d = __fadd_rn(d, __fmul_rn(vz, u[2]));
    return __float2ll_rn(__fmul_rn(d, 4294967296.0f));
}

__global__ void __launch_bounds__(256) k_drivers(PartDev p, int dim, Workspace ws, const __grid_constant__ DriverLaunch D,
                                                 const int *cell_start, const int *cell_end)
{
    pdl_entry();
    __shared__ long long s_part[256 / 32];
    const DriverEntry &E = D.e[blockIdx.x];
    long long sum = 0;
    for (int r = E.run0; r < E.run0 + E.nrun; ++r) {
        const int c0 = ws.runs[3 * r], c1 = ws.runs[3 * r + 1];
        if (c1 < c0) continue;
        const int b = cell_start[c0], e = cell_end[c1];
        for (int i = b + threadIdx.x; i < e; i += blockDim.x)
            if (p.label[i] == E.k) sum += flux_fixed(p.vx[i], p.vy[i], dim == 3 ? p.vz[i] : 0.0f, E.u, dim);
    }
    sum = warp_sum_ll(sum);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x != 0) return;
    long long S = 0;
    for (int w = 0; w < 256 / 32; ++w) S += s_part[w];      // integer: exact in any order
    DriverDev &st = ws.drv[E.k];
    double q = (double)S;
    q = q * 0x1p-32;
    q = q * E.scale;
    const double Q = E.sign < 0.0 ? -q : q;
    const double Qprev = st.first ? Q : st.Q;
    const double dQ = (Q - Qprev) / E.dt;
    const double t1 = E.Rp / E.Rd;
    const double t2 = 1.0 + t1;
    const double t3 = t2 * Q;
    const double t4 = E.C * E.Rp;
    const double t5 = t4 * dQ;
    const double t6 = t3 + t5;
    const double t7 = st.P / E.Rd;
    const double t8 = t6 - t7;
    const double dP = t8 / E.C;
    const double m = E.dt * dP;
    const double P = st.P + m;
    st.Qprev = Qprev;
    st.Q = Q;
    st.P = P;
    st.first = 0;
    ws.drv_rho[E.k] = __double2float_rn(E.rho0 + P / E.c0sq);
}

cudaError_t launch_drivers(const PartDev &p, int dim, const Workspace &ws, const DriverLaunch &D,
                           const int *cell_start, const int *cell_end, cudaStream_t s, Launch *L)
{
    if (D.n <= 0) return cudaSuccess;
    L->before(s);
    launch_k(k_drivers, dim3(D.n), dim3(256), 0, s, p, dim, ws, D, cell_start, cell_end);
    L->after(s, KID_DRIVERS);
    return cudaGetLastError();
}

}  // namespace sphbuf
