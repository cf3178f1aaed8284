/*
 * sph_oracle.c — CPU ORACLE for the arbitrary-positioned in/outlet buffer update
 * of Zhang, Fan, Ren, Qian & Hu, "Generalized and high-efficiency arbitrary-
 * positioned buffer for SPH" (arXiv 2406.16786).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this file.  The product
 * path (paper_2406_16786_b200/) never imports, links or executes it, and the two
 * share no code, header, helper or constant generator.
 *
 * It is deliberately plain and slow: every particle is tested against every
 * port by brute force, one loop per paper step, no blocking or
 * fusion.  Citations: "P:n" = /root/reference/PAPER.md line n (the paper's LaTeX
 * source); equations are named by their \label; "R<n>" = a reading of an
 * ambiguous passage listed in DESIGN.md §3.
 *
 * Arithmetic.  The paper fixes no precision (R16).  State is fp32 (BASELINE
 * configs).  Every DECISION (a crossing, P_k membership, an in-box test) is
 * taken from the plain definition in f64: the fp32 position
 * is widened exactly, d = x - o and X' = Q d are formed in double.  The inputs
 * are tie-screened (north_star: every particle at least 1e-4 dp from every
 * threshold; orc_tie_margin below is the check), so the exact decision is the
 * only correct one and the GPU's own-precision decisions must equal it.  Only
 * the three STATE MUTATIONS are pinned fp32, one IEEE-754 binary32
 * round-to-nearest operation each in a fixed order, because they produce fp32
 * state that is compared bit for bit (DESIGN.md §3 "Pinned arithmetic"):
 * advection x <- fl(x + fl(v dt)), recycling x <- fl(x - fl(a u)) and the cell
 * index floor(fl(fl(x - lo) * fl(1/cs))); plus the BC velocity and the moving-
 * port transfer, which write state too.  This file must be compiled with
 * -ffp-contract=off (no FMA contraction) on an SSE target (FLT_EVAL_METHOD == 0).
 *
 * Threads.  Compiled with -fopenmp: the per-particle loops whose iterations are
 * independent (advection, identification, the O3 decisions, the O5 relabel, the
 * BC state, the O7 margins) are split across threads; the order-defining steps
 * (the O2 sort, the O4 canonical walk, the O6 compaction) stay sequential, so
 * every result is the same for any thread count (orc_set_threads).
 *
 * parity pinned: see tests/test_oracle_pins.py (closed forms, hand cases
 * H1-H6, lattice counts, invariants, brute force vs cell-restricted).
 */
#define _POSIX_C_SOURCE 199309L
#include <math.h>
#include <stdint.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdlib.h>
#include <string.h>

#if defined(__FLT_EVAL_METHOD__) && __FLT_EVAL_METHOD__ != 0
#error "oracle needs FLT_EVAL_METHOD == 0 (binary32 ops rounded per operation)"
#endif

/* ------------------------------------------------------------------ types */

typedef struct {
    int32_t dim;          /* 2 or 3 */
    float lo[3];          /* grid lower corner (global) */
    float cs;             /* cell size, >= 2h */
    int32_t ncell[3];     /* global cell counts; ncell[2] == 1 in 2-D */
    int32_t cx_begin;     /* owned x-slab of cells [cx_begin, cx_end) */
    int32_t cx_end;
} orc_grid;

typedef struct {
    float o[3];           /* origin O' in global coordinates */
    float Q[9];           /* row-major; rows = local axes X',Y',Z' in global
                             coordinates; X' = Q (x - o)  (Eq. 2D/3D_transformation) */
    float he[3];          /* half extents a/2, b/2, c/2 */
    int32_t kind;         /* 0 = inlet (Alg. 1), 1 = outlet (Alg. 2), 2 = bidirectional (Alg. 3) */
    /* boundary condition of the port's buffer particles (§IV; 0 none, 1 pressure, 2 velocity) */
    int32_t bc;
    int32_t profile;      /* velocity BC: 0 plug, 1 u0 (1-(Y'/R)^2), 2 u0 (1-(Y'^2+Z'^2)/R^2) */
    int32_t rho_col;      /* pressure BC: extra column of the density, -1 none */
    float rho_b;          /* pressure BC: fl32(rho0 + p_b / c0^2) formed in f64 (Eq. postulate-density) */
    float u0, R, R2;      /* velocity BC: speed scale, radius, fl(R*R) */
} orc_port;

typedef struct {
    int64_t n;
    float *x, *y, *z;     /* z == NULL in 2-D */
    float *vx, *vy, *vz;  /* vz == NULL in 2-D */
    int32_t n_extra;
    float **extra;        /* n_extra fp32 columns copied on duplication ("same states") */
    int64_t *id;
    int32_t *label;       /* -1 = fluid, k = buffer particle of port k */
} orc_state;

enum { ORC_INLET = 0, ORC_OUTLET = 1, ORC_BIDIR = 2 };

/* Threads of the parallel loops (<= 0: the OpenMP default).  Returns the count in use. */
int32_t orc_set_threads(int32_t n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

/* ------------------------------------------------------------ frames (§III.A) */

/* Eq. 2D_transformation: rows [cos t, sin t], [-sin t, cos t];
 * theta > 0 anticlockwise.  Embedded in 3x3 with Z' = Z. */
void orc_frame_2d(double theta, double Q[9])
{
    double c = cos(theta), s = sin(theta);
    Q[0] = c;  Q[1] = s; Q[2] = 0.0;
    Q[3] = -s; Q[4] = c; Q[5] = 0.0;
    Q[6] = 0.0; Q[7] = 0.0; Q[8] = 1.0;
}

/* 3-D frame from the in/outflow axis u (global, unit):
 *   n = (OX x O'X') / |OX x O'X'|                 Eq. rotation_axis
 *   S = [[0,-nz,ny],[nz,0,-nx],[-ny,nx,0]]        Eq. antisymmetric_matrix
 *   R = I + S sin(theta) + S^2 (1 - cos(theta))   Eq. rotation_matrix
 * with theta = arccos(X.u) in [0, pi] (R2: "the sign of theta is positive").
 * As printed, R maps X-hat onto u (an active rotation), while the forward map
 * r' = R (r - o) (Eq. 3D_transformation) and u = R^T e1
 * (Eq. 3D_normal_transformation) need R u = e1.  Reading R1: the
 * frame matrix is Q = R^T (row 0 of Q = u).  Degenerate axes (R2): u ~ +X -> Q = I;
 * u ~ -X -> rotation by pi about Z, Q = diag(-1,-1,1).  Returns 0, or -1 if |u| == 0. */
int orc_frame_3d(const double u_in[3], double Q[9])
{
    double nu = sqrt(u_in[0] * u_in[0] + u_in[1] * u_in[1] + u_in[2] * u_in[2]);
    if (!(nu > 0.0)) return -1;
    double u[3] = {u_in[0] / nu, u_in[1] / nu, u_in[2] / nu};
    /* OX x O'X' with OX = (1,0,0), O'X' = u */
    double cx = 0.0, cy = -u[2], cz = u[1];
    double cn = sqrt(cx * cx + cy * cy + cz * cz);
    if (cn < 1e-12) {
        memset(Q, 0, 9 * sizeof(double));
        if (u[0] > 0) { Q[0] = 1; Q[4] = 1; Q[8] = 1; }
        else          { Q[0] = -1; Q[4] = -1; Q[8] = 1; }
        return 0;
    }
    double n[3] = {cx / cn, cy / cn, cz / cn};
    double cth = u[0];
    if (cth > 1.0) cth = 1.0;
    if (cth < -1.0) cth = -1.0;
    double th = acos(cth);
    double S[9] = {0.0, -n[2], n[1],
                   n[2], 0.0, -n[0],
                   -n[1], n[0], 0.0};
    double S2[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = 0.0;
            for (int l = 0; l < 3; ++l) acc += S[3 * i + l] * S[3 * l + j];
            S2[3 * i + j] = acc;
        }
    double R[9];
    for (int i = 0; i < 9; ++i) {
        double I = (i % 4 == 0) ? 1.0 : 0.0;
        R[i] = I + S[i] * sin(th) + S2[i] * (1.0 - cos(th));
    }
    /* Q = R^T (reading R1) */
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) Q[3 * i + j] = R[3 * j + i];
    return 0;
}

/* Forward transform r' = Q (r - o) in f64 from fp32 inputs
 * (Eq. 2D_transformation; Eq. 3D_transformation). */
void orc_to_local_f64(const orc_port *p, int32_t dim, float x, float y, float z, double out[3])
{
    double d[3] = {(double)x - (double)p->o[0], (double)y - (double)p->o[1],
                   dim == 3 ? (double)z - (double)p->o[2] : 0.0};
    for (int r = 0; r < 3; ++r) {
        double acc = 0.0;
        for (int j = 0; j < dim; ++j) acc += (double)p->Q[3 * r + j] * d[j];
        out[r] = acc;
    }
    if (dim == 2) out[2] = 0.0;
}

/* Same transform, pinned fp32 (see file header). */
void orc_to_local_f32(const orc_port *p, int32_t dim, float x, float y, float z, float out[3])
{
    float d0 = x - p->o[0];
    float d1 = y - p->o[1];
    if (dim == 3) {
        float d2 = z - p->o[2];
        for (int r = 0; r < 3; ++r) {
            float a0 = p->Q[3 * r + 0] * d0;
            float a1 = p->Q[3 * r + 1] * d1;
            float s01 = a0 + a1;
            float a2 = p->Q[3 * r + 2] * d2;
            out[r] = s01 + a2;
        }
    } else {
        for (int r = 0; r < 2; ++r) {
            float a0 = p->Q[3 * r + 0] * d0;
            float a1 = p->Q[3 * r + 1] * d1;
            out[r] = a0 + a1;
        }
        out[2] = 0.0f;
    }
}

/* The paper's recycle, literally: r = Q^T (r' - [a,0,0]^T) + o
 * (Eq. 2D_Inverse_transformation, Eq. 3D_Inverse_transformation P:356-379,
 * with a = 2 he_0).  f64; used by the pins to check reading R10. */
void orc_inverse_recycle_f64(const orc_port *p, int32_t dim, const double xl[3], double out[3])
{
    double a = 2.0 * (double)p->he[0];
    double v[3] = {xl[0] - a, xl[1], xl[2]};
    for (int j = 0; j < 3; ++j) {
        double acc = 0.0;
        for (int r = 0; r < dim; ++r) acc += (double)p->Q[3 * r + j] * v[r];
        out[j] = acc + (double)p->o[j];
    }
    if (dim == 2) out[2] = 0.0;
}

/* Recycle shift s = fl(a * u), u = row 0 of Q (Eq. 2D/3D_normal_transformation
 * P:528-554), a = 2 he_0 (exact).  Reading R10: r - a u is the inverse
 * transform above written in the global frame; pinned as one fp32 subtraction. */
static void recycle_shift(const orc_port *p, float s[3])
{
    float a = 2.0f * p->he[0];
    s[0] = a * p->Q[0];
    s[1] = a * p->Q[1];
    s[2] = a * p->Q[2];
}

/* ----------------------------------------------------------- predicates */

/* Local-frame test of one particle against one port, in f64 (O3).  Returns:
 *   bit0 = x in P_k   (|X'_r| < he_r + m, m = cs: reading R4, the paper's
 *                      "approximately one layer of cells" P:413)
 *   bit1 = InBox_k    (|X'| < a/2 & |Y'| < b/2 (& |Z'| < c/2), strict)
 *   bit2 = X'_0 > a/2   (crossing the buffer-fluid interface / outlet boundary)
 *   bit3 = X'_0 < -a/2  (bidirectional reverse crossing) */
static int classify(const orc_port *p, int32_t dim, float cs, float x, float y, float z)
{
    int bits = 0;
    double X[3];
    orc_to_local_f64(p, dim, x, y, z, X);
    int inP = 1, inB = 1;
    for (int r = 0; r < dim; ++r) {
        double heP = (double)p->he[r] + (double)cs;
        if (!(fabs(X[r]) < heP)) inP = 0;
        if (!(fabs(X[r]) < (double)p->he[r])) inB = 0;
    }
    if (inP) bits |= 1;
    if (inB) bits |= 2;
    if (X[0] > (double)p->he[0]) bits |= 4;
    if (X[0] < -(double)p->he[0]) bits |= 8;
    return bits;
}

/* O7 tie margin (north_star, BASELINE.json: "The generator keeps every particle at
 * least 1e-4 dp from any threshold, so no decision is a tie").
 * The thresholds of the method are the faces of InBox_k (|X'_r| = he_r: P:394-395,
 * X'_0 = +-a/2 is a face of InBox_k) and of the decision
 * region P_k (|X'_r| = he_r + m, reading R4).  For every particle i and port k
 * with x_i inside P_k inflated by tau (|X'_r| < he_r + m + tau for every r,
 * X' in f64), the margin is min over axes r of
 *     min( | |X'_r| - he_r | , | |X'_r| - (he_r + m) | ),
 * a conservative stand-in for the distance to the nearest face (it also counts
 * the planes' extensions inside P_k).  Returns the minimum over all pairs
 * (HUGE_VAL if no particle is near any port); flags[i] = 1 where some margin of
 * i is < tau (flags may be NULL).  The caller evaluates it at every decision
 * point (registration, after each advection) and relabel point (after each
 * update, on post-recycle positions). */
double orc_tie_margin(const orc_state *s, const orc_grid *g, const orc_port *ports, int32_t K, double tau,
                      uint8_t *flags)
{
    const int32_t dim = g->dim;
    const double m = (double)g->cs;
    double best = HUGE_VAL;
    /* exact early-out: a particle outside the bounding sphere of P_k inflated by
     * tau (radius^2 = 1.01 * sum_r (he_r + m + tau)^2) is not near port k */
    double *R2 = (double *)malloc(sizeof(double) * (size_t)(K > 0 ? K : 1));
    for (int32_t k = 0; k < K; ++k) {
        double acc = 0.0;
        for (int r = 0; r < dim; ++r) {
            double e = (double)ports[k].he[r] + m + tau;
            acc += e * e;
        }
        R2[k] = 1.01 * acc;
    }
#pragma omp parallel for schedule(static) reduction(min : best)
    for (int64_t i = 0; i < s->n; ++i) {
        if (flags) flags[i] = 0;
        for (int32_t k = 0; k < K; ++k) {
            const orc_port *p = &ports[k];
            double e0 = (double)s->x[i] - (double)p->o[0], e1 = (double)s->y[i] - (double)p->o[1];
            double e2 = dim == 3 ? (double)s->z[i] - (double)p->o[2] : 0.0;
            if (e0 * e0 + e1 * e1 + e2 * e2 > R2[k]) continue;
            double X[3];
            orc_to_local_f64(p, dim, s->x[i], s->y[i], dim == 3 ? s->z[i] : 0.0f, X);
            int near = 1;
            for (int r = 0; r < dim; ++r)
                if (!(fabs(X[r]) < (double)p->he[r] + m + tau)) near = 0;
            if (!near) continue;
            for (int r = 0; r < dim; ++r) {
                double a = fabs(X[r]);
                double d1 = fabs(a - (double)p->he[r]);
                double d2 = fabs(a - ((double)p->he[r] + m));
                double d = d1 < d2 ? d1 : d2;
                if (d < best) best = d;
                if (d < tau && flags) flags[i] = 1;
            }
        }
    }
    free(R2);
    return best;
}

/* ------------------------------------------------------------ cell list */

int64_t orc_ncells(const orc_grid *g)
{
    return (int64_t)(g->cx_end - g->cx_begin) * g->ncell[1] * (g->dim == 3 ? g->ncell[2] : 1);
}

static int32_t cell_axis(float x, float lo, float inv_cs, int32_t lo_c, int32_t hi_c, int32_t *oob)
{
    float t = (x - lo) * inv_cs;          /* pinned: fl(fl(x - lo) * inv_cs) */
    float f = floorf(t);
    if (f < (float)lo_c) { *oob = 1; return lo_c; }
    if (f > (float)(hi_c - 1)) { *oob = 1; return hi_c - 1; }
    return (int32_t)f;
}

/* Cell of a particle in the owned slab, linearised x-major (z fastest, y in 2-D):
 * ((cx - cx_begin) * ny + cy) * nz + cz.  Out-of-slab coordinates are clamped to
 * the boundary cell and flagged.  inv_cs = fl32(1/cs) formed in f64. */
int64_t orc_cell_of(const orc_grid *g, float x, float y, float z, int32_t *oob)
{
    float inv_cs = (float)(1.0 / (double)g->cs);
    int32_t o = 0;
    int32_t cx = cell_axis(x, g->lo[0], inv_cs, g->cx_begin, g->cx_end, &o);
    int32_t cy = cell_axis(y, g->lo[1], inv_cs, 0, g->ncell[1], &o);
    int32_t cz = 0;
    int32_t nz = 1;
    if (g->dim == 3) { cz = cell_axis(z, g->lo[2], inv_cs, 0, g->ncell[2], &o); nz = g->ncell[2]; }
    if (oob) *oob = o;
    return ((int64_t)(cx - g->cx_begin) * g->ncell[1] + cy) * nz + cz;
}

/* Oracle's own enumeration of the cells intersecting P_k (inflated by 1e-3 cs to
 * absorb fp32 rounding of X'): the cell-restricted candidate set of the paper's
 * "local cell-linked lists".  Every cell of the slab's axis-aligned
 * bounding box of P_k is tested by the separating-axis theorem between the cell
 * box and the oriented box.  mask[c] = 1 for intersecting local cells. */
static double dot3(const double *a, const double *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

int64_t orc_port_cells(const orc_grid *g, const orc_port *p, uint8_t *mask)
{
    int dim = g->dim;
    double cs = (double)g->cs;
    double eps = 1e-3 * cs;
    double o[3] = {p->o[0], p->o[1], dim == 3 ? p->o[2] : 0.0};
    double ax[3][3];
    double H[3];
    for (int r = 0; r < 3; ++r) {
        for (int j = 0; j < 3; ++j) ax[r][j] = p->Q[3 * r + j];
        H[r] = (double)p->he[r] + cs + eps;
    }
    if (dim == 2) { ax[0][2] = 0; ax[1][2] = 0; ax[2][0] = 0; ax[2][1] = 0; ax[2][2] = 1; H[2] = 0.0; }
    /* AABB of the oriented box */
    double ext[3];
    for (int j = 0; j < 3; ++j) {
        ext[j] = 0.0;
        for (int r = 0; r < 3; ++r) ext[j] += fabs(ax[r][j]) * H[r];
    }
    int64_t nmark = 0;
    int32_t nc[3] = {g->ncell[0], g->ncell[1], dim == 3 ? g->ncell[2] : 1};
    int32_t cmin[3], cmax[3];
    for (int j = 0; j < 3; ++j) {
        if (j == 2 && dim == 2) { cmin[2] = 0; cmax[2] = 0; continue; }
        cmin[j] = (int32_t)floor((o[j] - ext[j] - (double)g->lo[j]) / cs) - 1;
        cmax[j] = (int32_t)floor((o[j] + ext[j] - (double)g->lo[j]) / cs) + 1;
        if (cmin[j] < 0) cmin[j] = 0;
        if (cmax[j] > nc[j] - 1) cmax[j] = nc[j] - 1;
    }
    if (cmin[0] < g->cx_begin) cmin[0] = g->cx_begin;
    if (cmax[0] > g->cx_end - 1) cmax[0] = g->cx_end - 1;
    /* candidate separating axes: 3 world axes, 3 box axes, 9 cross products */
    double axes[15][3];
    int na = 0;
    for (int j = 0; j < 3; ++j) { axes[na][0] = j == 0; axes[na][1] = j == 1; axes[na][2] = j == 2; ++na; }
    for (int r = 0; r < 3; ++r) { axes[na][0] = ax[r][0]; axes[na][1] = ax[r][1]; axes[na][2] = ax[r][2]; ++na; }
    if (dim == 3) {
        for (int j = 0; j < 3; ++j)
            for (int r = 0; r < 3; ++r) {
                double e[3] = {j == 0, j == 1, j == 2};
                double c[3] = {e[1] * ax[r][2] - e[2] * ax[r][1], e[2] * ax[r][0] - e[0] * ax[r][2],
                               e[0] * ax[r][1] - e[1] * ax[r][0]};
                if (dot3(c, c) > 1e-20) { axes[na][0] = c[0]; axes[na][1] = c[1]; axes[na][2] = c[2]; ++na; }
            }
    }
    for (int32_t cx = cmin[0]; cx <= cmax[0]; ++cx)
        for (int32_t cy = cmin[1]; cy <= cmax[1]; ++cy)
            for (int32_t cz = cmin[2]; cz <= cmax[2]; ++cz) {
                double half = 0.5 * cs;
                double cc[3] = {(double)g->lo[0] + (cx + 0.5) * cs, (double)g->lo[1] + (cy + 0.5) * cs,
                                dim == 3 ? (double)g->lo[2] + (cz + 0.5) * cs : 0.0};
                double hc[3] = {half, half, dim == 3 ? half : 0.0};
                double t[3] = {cc[0] - o[0], cc[1] - o[1], cc[2] - o[2]};
                int separated = 0;
                for (int a = 0; a < na && !separated; ++a) {
                    double *L = axes[a];
                    double rc = fabs(L[0]) * hc[0] + fabs(L[1]) * hc[1] + fabs(L[2]) * hc[2];
                    double rb = 0.0;
                    for (int r = 0; r < 3; ++r) rb += fabs(dot3(L, ax[r])) * H[r];
                    if (fabs(dot3(L, t)) > rc + rb) separated = 1;
                }
                if (!separated) {
                    int64_t lc = ((int64_t)(cx - g->cx_begin) * g->ncell[1] + cy) * nc[2] + cz;
                    mask[lc] = 1;
                    ++nmark;
                }
            }
    return nmark;
}

/* --------------------------------------------------------- O1: advection */

/* Driver step (not part of the method): x <- fl(x + fl(v dt)) per component. */
void orc_advect(orc_state *s, int32_t dim, float dt)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < s->n; ++i) {
        float dx = s->vx[i] * dt;
        s->x[i] = s->x[i] + dx;
        float dy = s->vy[i] * dt;
        s->y[i] = s->y[i] + dy;
        if (dim == 3) {
            float dz = s->vz[i] * dt;
            s->z[i] = s->z[i] + dz;
        }
    }
}

/* ------------------------------------------- moving ports (rotating sprinkler) */

/* Rotating sprinkler (§V.C, Fig. rotation_procedure): after this
 * step's generation in the established local frame, "the positions and
 * velocities of buffer particles are transformed to new ones through coordinate
 * rotation", and "the local coordinate system is reestablished according to the
 * new position of sprinkler".  Reading R23: every buffer particle of
 * the port keeps its local coordinates and its local velocity; `from` is the
 * established frame, `to` the re-established one (the caller computes it, e.g.
 * theta = omega t + theta0):
 *     X' = Q0 (x - o0)      Eq. 2D/3D_transformation     (pinned as orc_to_local_f32)
 *     x  = o1 + Q1^T X'     Eq. 2D/3D_Inverse_transformation
 *     V' = Q0 v,  v = Q1^T V'   (velocities rotate without the translation)
 * Pinned fp32, one rounding per operation, sums in index order:
 *     x_j = fl(o1_j + fl(fl(fl(Q1[0][j] X'_0) + fl(Q1[1][j] X'_1)) + fl(Q1[2][j] X'_2)))
 *     (2-D: fl(o1_j + fl(fl(Q1[0][j] X'_0) + fl(Q1[1][j] X'_1))))
 * Brute force over every particle labelled k.  Returns how many moved. */
int64_t orc_port_move(orc_state *s, int32_t dim, const orc_port *from, const orc_port *to, int32_t k)
{
    int64_t moved = 0;
    for (int64_t i = 0; i < s->n; ++i) {
        if (s->label[i] != k) continue;
        float X[3], V[3];
        orc_to_local_f32(from, dim, s->x[i], s->y[i], dim == 3 ? s->z[i] : 0.0f, X);
        /* local velocity: the linear part of the same transform */
        for (int r = 0; r < dim; ++r) {
            float acc = from->Q[3 * r + 0] * s->vx[i];
            float t1 = from->Q[3 * r + 1] * s->vy[i];
            acc = acc + t1;
            if (dim == 3) {
                float t2 = from->Q[3 * r + 2] * s->vz[i];
                acc = acc + t2;
            }
            V[r] = acc;
        }
        float xn[3] = {0.0f, 0.0f, 0.0f}, vn[3] = {0.0f, 0.0f, 0.0f};
        for (int j = 0; j < dim; ++j) {
            float gx = to->Q[0 * 3 + j] * X[0];
            float gv = to->Q[0 * 3 + j] * V[0];
            float t = to->Q[1 * 3 + j] * X[1];
            float tv = to->Q[1 * 3 + j] * V[1];
            gx = gx + t;
            gv = gv + tv;
            if (dim == 3) {
                float t2 = to->Q[2 * 3 + j] * X[2];
                float tv2 = to->Q[2 * 3 + j] * V[2];
                gx = gx + t2;
                gv = gv + tv2;
            }
            xn[j] = to->o[j] + gx;
            vn[j] = gv;
        }
        s->x[i] = xn[0];
        s->y[i] = xn[1];
        s->vx[i] = vn[0];
        s->vy[i] = vn[1];
        if (dim == 3) {
            s->z[i] = xn[2];
            s->vz[i] = vn[2];
        }
        ++moved;
    }
    return moved;
}

/* ------------------------------------------ port drivers (aorta flow, §V.D) */

/* Eq. Fourier_Series: v_inlet(t) = a0 + sum_{n=1..8} a_n cos(n t w)
 * + sum_{n=1..8} b_n sin(n t w), Table I.  f64, the two sums in the order
 * written, argument (n t) w. */
double orc_fourier(double t, const double *a, const double *b, double omega)
{
    double u = a[0];
    for (int n = 1; n <= 8; ++n) u = u + a[n] * cos(((double)n * t) * omega);
    for (int n = 1; n <= 8; ++n) u = u + b[n] * sin(((double)n * t) * omega);
    return u;
}

/* Flow through a port (reading R26): sum over the port's buffer particles of
 * v . u, u = row 0 of Q, each term pinned fp32 fl(fl(fl(vx ux) + fl(vy uy)) +
 * fl(vz uz)) scaled by 2^32 and rounded to the nearest integer (ties to even),
 * summed exactly in int64 (so the order of the sum does not matter).  The caller
 * forms Q = +-(S 2^-32) V / a.  Brute force over every particle. */
int64_t orc_port_flux(const orc_state *s, int32_t dim, const orc_port *p, int32_t k)
{
    int64_t S = 0;
    for (int64_t i = 0; i < s->n; ++i) {
        if (s->label[i] != k) continue;
        float d = s->vx[i] * p->Q[0];
        float e = s->vy[i] * p->Q[1];
        d = d + e;
        if (dim == 3) {
            float f = s->vz[i] * p->Q[2];
            d = d + f;
        }
        float sc = d * 4294967296.0f;
        S += (int64_t)llrintf(sc);
    }
    return S;
}

/* One explicit step of the 3-element Windkessel (Eq. windkessel):
 *     (1 + Rp/Rd) Q + C Rp dQ/dt = P/Rd + C dP/dt
 * reading R27: dQ/dt = (Q - Qprev)/dt, P_next = P + dt dP/dt with
 * dP/dt = ((1 + Rp/Rd) Q + C Rp dQ/dt - P/Rd) / C.  f64, in the order written. */
double orc_windkessel(double P, double Q, double Qprev, double dt, double Rp, double C, double Rd)
{
    double dQ = (Q - Qprev) / dt;
    double t1 = Rp / Rd;
    double t2 = 1.0 + t1;
    double t3 = t2 * Q;
    double t4 = C * Rp;
    double t5 = t4 * dQ;
    double t6 = t3 + t5;
    double t7 = P / Rd;
    double t8 = t6 - t7;
    double dP = t8 / C;
    double m = dt * dP;
    return P + m;
}

/* ---------------------------------------------------- O0: registration */

/* Alg. 1 "Buffer particle identification ... Execute only once":
 * every fluid particle (label -1) with |X'|<a/2 & |Y'|<b/2 (& |Z'|<c/2) becomes a
 * buffer particle of port k.  For outlet and bidirectional ports the same test is
 * the initial relabel (Alg. 2/3 second procedure).
 * Returns the number of particles labelled k afterwards. */
int64_t orc_register(orc_state *s, const orc_grid *g, const orc_port *p, int32_t k)
{
    int64_t members = 0;
#pragma omp parallel for schedule(static) reduction(+ : members)
    for (int64_t i = 0; i < s->n; ++i) {
        if (s->label[i] == -1) {
            int b = classify(p, g->dim, g->cs, s->x[i], s->y[i], g->dim == 3 ? s->z[i] : 0.0f);
            if (b & 2) s->label[i] = k;
        }
        if (s->label[i] == k) ++members;
    }
    return members;
}

/* ------------------------------------------------------ O2 .. O5: update */

typedef struct {
    int64_t cell;
    int64_t id;
    int64_t idx;
} key_t3;

static int cmp_key(const void *a, const void *b)
{
    const key_t3 *u = (const key_t3 *)a, *v = (const key_t3 *)b;
    if (u->cell != v->cell) return u->cell < v->cell ? -1 : 1;
    if (u->id != v->id) return u->id < v->id ? -1 : 1;
    return 0;
}

typedef struct {
    /* O2 */
    int64_t *order;        /* [n] sorted position -> input index */
    int32_t *cell_start;   /* [ncells] first sorted position of cell c */
    int32_t *cell_end;     /* [ncells] one past the last */
    int64_t out_of_grid;
    /* O3 (indexed by sorted position) */
    int32_t *create_port;  /* [n] k or -1 */
    int32_t *delete_port;  /* [n] k or -1 */
    /* O4/O5: 'sorted' holds the input reordered by O2 with recycles and relabels applied */
    orc_state sorted;
    orc_state staged;      /* [cap_stage] bitwise copies (pre-recycle) in canonical order; id = source id */
    int32_t *stage_port;   /* [cap_stage] */
    int64_t *stage_src;    /* [cap_stage] sorted position of the source */
    int64_t cap_stage;
    int64_t n_stage;
    int32_t *port_counts;  /* [2K]: created_k at [k], deleted_k at [K + k] */
    int64_t checked;       /* particle-port tests performed */
    int64_t multi_decision;/* particles with more than one decision (must be 0) */
    int64_t motion_errors; /* members of k outside P_k (reading R12; diagnostic): the paper
                              checks only the local cell-linked lists around the buffer
                              (P:411-413), so a buffer particle that left that region
                              can no longer be generated, deleted or relabelled */
    double t_cll;          /* seconds in O2 (cell list: keys, sort, tables, reorder) */
    double t_decide;       /* seconds in O3-O5b (decisions, apply, relabel, BC state) */
} orc_update_out;

static double now_s(void)
{
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}

static void copy_row(const orc_state *src, int64_t i, orc_state *dst, int64_t j, int32_t dim)
{
    dst->x[j] = src->x[i];
    dst->y[j] = src->y[i];
    dst->vx[j] = src->vx[i];
    dst->vy[j] = src->vy[i];
    if (dim == 3) { dst->z[j] = src->z[i]; dst->vz[j] = src->vz[i]; }
    for (int e = 0; e < src->n_extra; ++e) dst->extra[e][j] = src->extra[e][i];
    dst->id[j] = src->id[i];
    dst->label[j] = src->label[i];
}

/* The particle ranges [rb[q], re[q]) that port k checks: the whole array in
 * fixed chunks (mode 0, brute force) or the ranges of the cells of the oracle's
 * own P_k cell set (mode 1).  Returns their number; *rb, *re malloc'ed. */
static int64_t port_ranges(const orc_grid *g, const orc_port *p, int32_t mode, int64_t n, const int32_t *cell_start,
                           const int32_t *cell_end, int64_t **rb, int64_t **re)
{
    const int64_t chunk = 65536;
    if (mode == 0) {
        int64_t nr = (n + chunk - 1) / chunk;
        *rb = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nr > 0 ? nr : 1));
        *re = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nr > 0 ? nr : 1));
        for (int64_t q = 0; q < nr; ++q) {
            (*rb)[q] = q * chunk;
            (*re)[q] = (q + 1) * chunk < n ? (q + 1) * chunk : n;
        }
        return nr;
    }
    const int64_t nc = orc_ncells(g);
    uint8_t *mask = (uint8_t *)calloc((size_t)(nc > 0 ? nc : 1), 1);
    int64_t nr = orc_port_cells(g, p, mask);
    *rb = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nr > 0 ? nr : 1));
    *re = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nr > 0 ? nr : 1));
    int64_t q = 0;
    for (int64_t c = 0; c < nc; ++c)
        if (mask[c]) {
            (*rb)[q] = cell_start[c];
            (*re)[q] = cell_end[c];
            ++q;
        }
    free(mask);
    return q;
}

/* One buffer update on one slab.  mode 0 = brute force over every particle and
 * port in the global frame ("through the equation of the threshold line or
 * surface"); mode 1 = only particles in the oracle's own P_k cell set (the
 * paper's local cell-linked lists).  Decisions in f64 (O3).
 * Returns 0, or -1 if staging overflows. */
int orc_update(const orc_grid *g, const orc_port *ports, int32_t K, const orc_state *in,
               int32_t mode, orc_update_out *out)
{
    const int32_t dim = g->dim;
    const int64_t n = in->n;
    const int64_t nc = orc_ncells(g);

    const double t0 = now_s();
    /* O2: cell-linked list -- cell of each particle, then order by
     * (cell, id): a counting sort by cell (histogram, exclusive prefix = the cell
     * tables, placement), then each cell's particles sorted by id. */
    int64_t *cell = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    key_t3 *keys = (key_t3 *)malloc(sizeof(key_t3) * (size_t)(n > 0 ? n : 1));
    int64_t oob_total = 0;
#pragma omp parallel for schedule(static) reduction(+ : oob_total)
    for (int64_t i = 0; i < n; ++i) {
        int32_t oob = 0;
        cell[i] = orc_cell_of(g, in->x[i], in->y[i], dim == 3 ? in->z[i] : 0.0f, &oob);
        oob_total += oob;
    }
    out->out_of_grid = oob_total;
    for (int64_t c = 0; c < nc; ++c) { out->cell_start[c] = 0; out->cell_end[c] = 0; }
    for (int64_t i = 0; i < n; ++i) out->cell_end[cell[i]] += 1;          /* counts */
    int64_t run = 0;
    for (int64_t c = 0; c < nc; ++c) {
        int64_t cnt = out->cell_end[c];
        out->cell_start[c] = (int32_t)run;
        run += cnt;
        out->cell_end[c] = (int32_t)run;
    }
    {
        int32_t *cursor = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nc > 0 ? nc : 1));
        for (int64_t c = 0; c < nc; ++c) cursor[c] = out->cell_start[c];
        for (int64_t i = 0; i < n; ++i) {
            const int64_t j = cursor[cell[i]]++;
            keys[j].cell = cell[i];
            keys[j].id = in->id[i];
            keys[j].idx = i;
        }
        free(cursor);
    }
    free(cell);
    /* each cell by id (cells are independent) */
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t b = out->cell_start[c], e = out->cell_end[c];
        if (e - b > 32) {
            qsort(keys + b, (size_t)(e - b), sizeof(key_t3), cmp_key);
            continue;
        }
        for (int64_t u = b + 1; u < e; ++u) {          /* insertion sort */
            key_t3 t = keys[u];
            int64_t v = u;
            while (v > b && keys[v - 1].id > t.id) {
                keys[v] = keys[v - 1];
                --v;
            }
            keys[v] = t;
        }
    }
    orc_state *S = &out->sorted;
    S->n = n;
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j) {
        out->order[j] = keys[j].idx;
        copy_row(in, keys[j].idx, S, j, dim);
    }
    free(keys);

    const double t1 = now_s();
    out->t_cll = t1 - t0;
    /* O3: decisions (Alg. 1, Alg. 2, Alg. 3). */
    for (int64_t j = 0; j < n; ++j) { out->create_port[j] = -1; out->delete_port[j] = -1; }
    int32_t *ndec = (int32_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(int32_t));
    out->checked = 0;
    out->multi_decision = 0;
    out->motion_errors = 0;
    for (int32_t k = 0; k < K; ++k) {
        const orc_port *p = &ports[k];
        int64_t *rb, *re;
        const int64_t nr = port_ranges(g, p, mode, n, out->cell_start, out->cell_end, &rb, &re);
        int64_t checked = 0, motion = 0, multi = 0;
        /* each particle lies in one range of port k: the iterations are independent */
#pragma omp parallel for schedule(dynamic, 8) reduction(+ : checked, motion, multi)
        for (int64_t q = 0; q < nr; ++q) {
            for (int64_t j = rb[q]; j < re[q]; ++j) {
                ++checked;
                int b = classify(p, dim, g->cs, S->x[j], S->y[j], dim == 3 ? S->z[j] : 0.0f);
                int member = (S->label[j] == k);
                if (member && !(b & 1)) ++motion;                     /* reading R12 (diagnostic) */
                if (!(b & 1)) continue;                               /* x not in P_k (R4) */
                int create = 0, del = 0;
                if (p->kind == ORC_INLET) {
                    /* Alg. 1: buffer particles j with X'_j > a/2 (reading R5) */
                    create = member && (b & 4);
                } else if (p->kind == ORC_OUTLET) {
                    /* Alg. 2: any checked particle with X'_i > a/2 (reading R6) */
                    del = (b & 4) != 0;
                } else {
                    /* Alg. 3: buffer particles only */
                    create = member && (b & 4);
                    del = member && (b & 8);
                }
                if (create || del) {
                    if (ndec[j]++ > 0) { ++multi; continue; }
                    if (create) out->create_port[j] = k;
                    if (del) out->delete_port[j] = k;
                }
            }
        }
        out->checked += checked;
        out->motion_errors += motion;
        out->multi_decision += multi;
        free(rb);
        free(re);
    }
    free(ndec);

    /* O4: apply.  CREATEs in canonical order (port k, source cell, source id) =
     * port-major walk of the (cell, id)-sorted array (reading R14).  Duplicate =
     * bitwise copy of the member's state before the recycle, label fluid
     * ("the same states as the crossing ones"; R11).  Then recycle
     * x <- fl(x - fl(a u)) (Eqs. 2D/3D_Inverse_transformation; R10). */
    for (int32_t k = 0; k < 2 * K; ++k) out->port_counts[k] = 0;
    out->n_stage = 0;
    for (int32_t k = 0; k < K; ++k) {
        float s[3];
        recycle_shift(&ports[k], s);
        for (int64_t j = 0; j < n; ++j) {
            if (out->create_port[j] != k) continue;
            if (out->n_stage >= out->cap_stage) return -1;
            int64_t t = out->n_stage++;
            copy_row(S, j, &out->staged, t, dim);
            out->staged.label[t] = -1;
            out->stage_port[t] = k;
            out->stage_src[t] = j;
            out->port_counts[k] += 1;
            S->x[j] = S->x[j] - s[0];
            S->y[j] = S->y[j] - s[1];
            if (dim == 3) S->z[j] = S->z[j] - s[2];
        }
        for (int64_t j = 0; j < n; ++j)
            if (out->delete_port[j] == k) out->port_counts[K + k] += 1;
    }
    out->staged.n = out->n_stage;

    /* O5: relabel for outlet and bidirectional ports (Alg. 2/3 "Buffer particle
     * identification (after the cell-linked lists have been rebuilt ...)",
     * P:435-443; reading R9: on post-recycle positions, this update's
     * cell list).  In-box -> label k; a former member outside -> fluid ("otherwise,
     * they will not").  New (staged) and deleted particles are excluded;
     * inlet members are fixed (Alg. 1 identifies them once). */
    for (int32_t k = 0; k < K; ++k) {
        const orc_port *p = &ports[k];
        if (p->kind == ORC_INLET) continue;
        int64_t *rb, *re;
        const int64_t nr = port_ranges(g, p, mode, n, out->cell_start, out->cell_end, &rb, &re);
#pragma omp parallel for schedule(dynamic, 8)
        for (int64_t q = 0; q < nr; ++q) {
            for (int64_t j = rb[q]; j < re[q]; ++j) {
                if (out->delete_port[j] >= 0) continue;
                int b = classify(p, dim, g->cs, S->x[j], S->y[j], dim == 3 ? S->z[j] : 0.0f);
                if (b & 2) S->label[j] = k;
                else if (S->label[j] == k) S->label[j] = -1;
            }
        }
        free(rb);
        free(re);
    }

    /* O5b: boundary-condition state of every buffer particle of port k after the
     * update (paper §IV).  The duplicates staged in O4 keep the
     * pre-BC state.
     *  pressure BC: v = (v.u) u, u = row 0 of Q (Eq. velocity_correction);
     *    a particle recycled in this update gets rho = rho0 + p_b / c0^2
     *    (Eq. postulate-density);
     *  velocity BC: v_X' = u0 (1 - (Y'/R)^2) in the local frame (Eqs. 2D/3D_velocity_
     *    profile; plug and radial variants), v = Q^T (v_X', 0, 0)
     *    (Eqs. 2D/3D_velocity_transformation); recycled density unchanged
     *    (P:639-643).  Pinned fp32 (Q^T (v_X',0,0)_j = fl(v_X' Q_0j) since the other
     *    terms are exact zeros). */
    for (int32_t k = 0; k < K; ++k) {
        const orc_port *p = &ports[k];
        if (p->bc == 0) continue;
#pragma omp parallel for schedule(static)
        for (int64_t j = 0; j < n; ++j) {
            if (out->delete_port[j] >= 0 || S->label[j] != k) continue;
            float u;
            if (p->bc == 1) {
                float a0 = S->vx[j] * p->Q[0];
                float a1 = S->vy[j] * p->Q[1];
                u = a0 + a1;
                if (dim == 3) {
                    float a2 = S->vz[j] * p->Q[2];
                    u = u + a2;
                }
                if (out->create_port[j] == k && p->rho_col >= 0) S->extra[p->rho_col][j] = p->rho_b;
            } else {
                float X[3];
                orc_to_local_f32(p, dim, S->x[j], S->y[j], dim == 3 ? S->z[j] : 0.0f, X);
                u = p->u0;
                if (p->profile == 1) {
                    float t = X[1] / p->R;
                    float tt = t * t;
                    float q = 1.0f - tt;
                    u = p->u0 * q;
                } else if (p->profile == 2) {
                    float r2 = X[1] * X[1];
                    if (dim == 3) {
                        float zz = X[2] * X[2];
                        r2 = r2 + zz;
                    }
                    float t = r2 / p->R2;
                    float q = 1.0f - t;
                    u = p->u0 * q;
                }
            }
            S->vx[j] = u * p->Q[0];
            S->vy[j] = u * p->Q[1];
            if (dim == 3) S->vz[j] = u * p->Q[2];
        }
    }
    out->t_decide = now_s() - t1;
    return 0;
}

/* ------------------------------------------------------- O6: compaction */

/* Stable compaction + append + ID assignment (north star "scan-based stream
 * compaction with an ID/permutation remap"; readings R14, R15).
 * Survivors keep their (cell, id) order, staged particles are appended in
 * canonical order.  New IDs follow the count matrix all_counts[r][2K]
 * (created_k at [r*2K + k]):
 *   off(k, r) = next_id + sum_{k'<k} sum_{r'} C[r'][k'] + sum_{r'<r} C[r'][k]
 * and within (k, r) the canonical order.  perm[j] = new position of sorted
 * position j, or -1 if deleted.  Returns the new count; *next_id_out receives
 * next_id + sum of all C. */
int64_t orc_compact(const orc_state *S, const int32_t *delete_port, const orc_state *staged,
                    const int32_t *stage_port, int32_t dim, const int32_t *all_counts, int32_t nranks,
                    int32_t rank, int32_t K, int64_t next_id, orc_state *out, int64_t *perm,
                    int64_t *next_id_out)
{
    int64_t m = 0;
    for (int64_t j = 0; j < S->n; ++j) {
        if (delete_port[j] >= 0) { if (perm) perm[j] = -1; continue; }
        copy_row(S, j, out, m, dim);
        if (perm) perm[j] = m;
        ++m;
    }
    int64_t total = 0;
    for (int32_t r = 0; r < nranks; ++r)
        for (int32_t k = 0; k < K; ++k) total += all_counts[(int64_t)r * 2 * K + k];
    int64_t within = 0;
    int32_t prev_k = -1;
    for (int64_t t = 0; t < staged->n; ++t) {
        int32_t k = stage_port[t];
        if (k != prev_k) { within = 0; prev_k = k; }
        int64_t off = next_id;
        for (int32_t kk = 0; kk < k; ++kk)
            for (int32_t r = 0; r < nranks; ++r) off += all_counts[(int64_t)r * 2 * K + kk];
        for (int32_t r = 0; r < rank; ++r) off += all_counts[(int64_t)r * 2 * K + k];
        copy_row(staged, t, out, m, dim);
        out->id[m] = off + within;
        out->label[m] = -1;
        ++within;
        ++m;
    }
    out->n = m;
    if (next_id_out) *next_id_out = next_id + total;
    return m;
}
