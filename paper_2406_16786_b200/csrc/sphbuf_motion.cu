// sphbuf_motion.cu — moving ports (rotating sprinkler, arXiv 2406.16786 §V.C,
// P:779-803).  After this step's generation in the
// established local frame, the port's buffer particles are "transformed to new
// ones through coordinate rotation" and the local coordinate system is
// re-established for the next step (Fig. rotation_procedure):
//   K9  k_port_move  every buffer particle of the port (found among the port's
//                    candidates of the current cell list) keeps its local
//                    coordinates and local velocity: x <- o1 + Q1^T Q0 (x - o0),
//                    v <- Q1^T Q0 v, pinned fp32 (reading R23);
//   K10 k_port_enum  the port's candidate cells for the new pose, enumerated on
//                    the device: one thread per cell column of a window that
//                    covers the port's bounding sphere, an f64 separating-axis
//                    test per cell, at most one run per column (a column meets a
//                    convex box in one interval).
#include <cstdint>

#include "sphbuf_common.cuh"

namespace sphbuf {

// X' = Q0 (x - o0) is to_local(); back to global with the new frame:
// x_j = fl(o1_j + fl(fl(fl(Q1[0][j] X'_0) + fl(Q1[1][j] X'_1)) + fl(Q1[2][j] X'_2))).
__device__ __forceinline__ float to_global(const PortDev &P, int dim, const float X[3], int j)
{
    float g = __fadd_rn(__fmul_rn(P.Q[j], X[0]), __fmul_rn(P.Q[3 + j], X[1]));
    if (dim == 3) g = __fadd_rn(g, __fmul_rn(P.Q[6 + j], X[2]));
    return __fadd_rn(P.o[j], g);
}

// the linear part only (velocities): V_r = fl(fl(fl(Q_r0 v_0) + fl(Q_r1 v_1)) + fl(Q_r2 v_2))
__device__ __forceinline__ void rot_local(const PortDev &P, int dim, const float v[3], float V[3])
{
    for (int r = 0; r < dim; ++r) {
        float a = __fadd_rn(__fmul_rn(P.Q[3 * r], v[0]), __fmul_rn(P.Q[3 * r + 1], v[1]));
        if (dim == 3) a = __fadd_rn(a, __fmul_rn(P.Q[3 * r + 2], v[2]));
        V[r] = a;
    }
    if (dim == 2) V[2] = 0.0f;
}

__device__ __forceinline__ float rot_global(const PortDev &P, int dim, const float V[3], int j)
{
    float g = __fadd_rn(__fmul_rn(P.Q[j], V[0]), __fmul_rn(P.Q[3 + j], V[1]));
    if (dim == 3) g = __fadd_rn(g, __fmul_rn(P.Q[6 + j], V[2]));
    return g;
}

// K9: one block per run (grid-stride), threads over the run's particle range.
__global__ void __launch_bounds__(kThreads) k_port_move(PartDev p, GridDev g, PortDev P0, PortDev P1, const int *runs,
                                                        int nrun, const int *cell_start, const int *cell_end, int k,
                                                        long long *moved, Workspace ws, int carry, float cdt)
{
    const int dim = g.dim;
    pdl_entry();
    long long cnt = 0;
    for (int r = blockIdx.x; r < nrun; r += gridDim.x) {
        const int c0 = runs[3 * r], c1 = runs[3 * r + 1];
        if (c1 < c0) continue;                                   // empty run of a movable port
        const int b = cell_start[c0], e = cell_end[c1];
        SPH_CHECK(b >= 0 && e <= p.cap);
        for (int i = b + threadIdx.x; i < e; i += blockDim.x) {
            if (p.label[i] != k) continue;
            float X[3], V[3];
            const float v[3] = {p.vx[i], p.vy[i], dim == 3 ? p.vz[i] : 0.0f};
            to_local(P0, dim, p.x[i], p.y[i], dim == 3 ? p.z[i] : 0.0f, X);
            rot_local(P0, dim, v, V);
            p.x[i] = to_global(P1, dim, X, 0);
            p.y[i] = to_global(P1, dim, X, 1);
            p.vx[i] = rot_global(P1, dim, V, 0);
            p.vy[i] = rot_global(P1, dim, V, 1);
            if (dim == 3) {
                p.z[i] = to_global(P1, dim, X, 2);
                p.vz[i] = rot_global(P1, dim, V, 2);
            }
            if (carry)
                carry_fix(g, ws, i, false, p.x[i], p.y[i], dim == 3 ? p.z[i] : 0.0f, p.vx[i], p.vy[i],
                          dim == 3 ? p.vz[i] : 0.0f, cdt, carry);
            ++cnt;
        }
    }
    cnt = warp_sum_ll(cnt);
    if ((threadIdx.x & 31) == 0 && cnt && moved) atomicAdd((unsigned long long *)moved, (unsigned long long)cnt);
}

// Separating-axis test (f64) between the axis-aligned cell box (centre c, half
// size e) and the oriented decision region of the port (centre o, unit axes ax,
// half sizes H); the same test as the host's registration-time enumeration.
__device__ bool cell_meets_port(const double c[3], const double e[3], const PortEnum &P, int dim)
{
    const double t[3] = {P.o[0] - c[0], P.o[1] - c[1], P.o[2] - c[2]};
    auto sep = [&](const double L[3]) {
        const double ra = fabs(L[0]) * e[0] + fabs(L[1]) * e[1] + fabs(L[2]) * e[2];
        double rb = 0.0;
        for (int r = 0; r < 3; ++r) rb += fabs(L[0] * P.ax[r][0] + L[1] * P.ax[r][1] + L[2] * P.ax[r][2]) * P.H[r];
        return fabs(L[0] * t[0] + L[1] * t[1] + L[2] * t[2]) > ra + rb;
    };
    for (int j = 0; j < dim; ++j) {
        const double L[3] = {double(j == 0), double(j == 1), double(j == 2)};
        if (sep(L)) return false;
    }
    for (int r = 0; r < dim; ++r)
        if (sep(P.ax[r])) return false;
    if (dim == 3) {
        for (int j = 0; j < 3; ++j)
            for (int r = 0; r < 3; ++r) {
                const double u[3] = {double(j == 0), double(j == 1), double(j == 2)};
                const double *a = P.ax[r];
                const double w[3] = {u[1] * a[2] - u[2] * a[1], u[2] * a[0] - u[0] * a[2], u[0] * a[1] - u[1] * a[0]};
                if (w[0] * w[0] + w[1] * w[1] + w[2] * w[2] < 1e-20) continue;
                if (sep(w)) return false;
            }
    }
    return true;
}

// K10: thread i -> column i of the window (cx0 + i / ncy, cy0 + i % ncy) in 3-D,
// (cx0 + i) in 2-D; the run is written to slot i of the port's slice, or marked
// empty (c1 < c0).  Slots follow the x-major cell order (cx slowest), so the
// port's candidates stay in cell order and creations in canonical order (R14).
__global__ void __launch_bounds__(kThreads) k_port_enum(GridDev g, PortEnum P, float cs, int *runs, int cap)
{
    pdl_entry();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cap) return;
    const int dim = g.dim;
    const int cx = P.cx0 + (dim == 3 ? i / P.ncy : i);
    const int cy = dim == 3 ? P.cy0 + i % P.ncy : 0;
    int first = -1, last = -1;
    const bool col_ok = cx >= g.cx_begin && cx < g.cx_end && (dim == 2 || (cy >= 0 && cy < g.ncell[1]));
    if (col_ok) {
        const double h = 0.5 * (double)cs;
        const double e[3] = {h, h, dim == 3 ? h : 0.0};
        for (int f = P.f0; f <= P.f1; ++f) {
            const int ix[3] = {cx, dim == 3 ? cy : f, dim == 3 ? f : 0};
            double ctr[3];
            for (int j = 0; j < 3; ++j) ctr[j] = (j < dim) ? (double)g.lo[j] + (ix[j] + 0.5) * (double)cs : 0.0;
            if (cell_meets_port(ctr, e, P, dim)) {
                if (first < 0) first = f;
                last = f;
            } else if (first >= 0) {
                break;
            }
        }
    }
    int c0 = 0, c1 = -1;
    if (first >= 0) {
        if (dim == 3) {
            c0 = ((cx - g.cx_begin) * g.ny + cy) * g.nz + first;
            c1 = ((cx - g.cx_begin) * g.ny + cy) * g.nz + last;
        } else {
            c0 = (cx - g.cx_begin) * g.ny + first;
            c1 = (cx - g.cx_begin) * g.ny + last;
        }
    }
    SPH_CHECK(c1 < c0 || (c0 >= 0 && c1 < (int)g.ncells));
    runs[3 * i] = c0;
    runs[3 * i + 1] = c1;
    runs[3 * i + 2] = P.k;
}

cudaError_t launch_port_move(const PartDev &p, const GridDev &g, const PortDev &P0, const PortDev &P1,
                             const int *runs, int nrun, const int *cell_start, const int *cell_end, int k,
                             long long *moved, const Workspace &ws, int carry, float cdt, cudaStream_t s, Launch *L)
{
    if (nrun <= 0) return cudaSuccess;
    L->before(s);
    launch_k(k_port_move, dim3(nrun < 4 * sm_count_cached() ? nrun : 4 * sm_count_cached()), dim3(128), 0, s, p, g,
             P0, P1, runs, nrun, cell_start, cell_end, k, moved, ws, carry, cdt);
    L->after(s, KID_PORT_MOVE);
    return cudaGetLastError();
}

cudaError_t launch_port_enum(const GridDev &g, const PortEnum &P, float cs, int *runs, int cap, cudaStream_t s,
                             Launch *L)
{
    if (cap <= 0) return cudaSuccess;
    L->before(s);
    launch_k(k_port_enum, dim3((cap + kThreads - 1) / kThreads), dim3(kThreads), 0, s, g, P, cs, runs, cap);
    L->after(s, KID_PORT_ENUM);
    return cudaGetLastError();
}

}  // namespace sphbuf
