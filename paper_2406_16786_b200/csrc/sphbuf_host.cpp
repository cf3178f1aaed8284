// sphbuf_host.cpp — host side of the C ABI declared in include/sphbuf.h:
// context, workspace layout, port validation, per-port cell enumeration
// and the launch wrappers.  "P:n" = PAPER.md line n.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "sphbuf_internal.h"

// NVTX range around each enqueueing ABI call (SURVEY §5 "NVTX ranges per phase"):
// host-side push/pop, free when no tool is attached.
namespace {
struct NvtxRange {
    explicit NvtxRange(const char *n) { nvtxRangePushA(n); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace
#define SPH_NVTX(name) NvtxRange nvtx_range_(name)

using namespace sphbuf;

namespace {

struct PortHost {
    double o[3];
    double ax[3][3];   // local axes (rows of Q)
    double H[3];       // half extents of the decision region P_k = he + cs
    int kind;
};

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

}  // namespace

namespace sphbuf {

void Launch::before(cudaStream_t s)
{
    if (!prof) return;
    if (pool.size() < 2 * (used + 1)) {
        if (used >= 4096) flush();
        while (pool.size() < 2 * (used + 1)) {
            cudaEvent_t ev;
            cudaEventCreate(&ev);
            pool.push_back(ev);
        }
    }
    cudaEventRecord(pool[2 * used], s);
}

void Launch::after(cudaStream_t s, int k)
{
    ++count;
    if (!prof) return;
    cudaEventRecord(pool[2 * used + 1], s);
    if (kid.size() <= used) kid.resize(used + 1);
    kid[used] = k;
    ++used;
}

cudaError_t Launch::flush()
{
    if (used == 0) return cudaSuccess;
    cudaError_t e = cudaEventSynchronize(pool[2 * used - 1]);
    for (size_t i = 0; i < used && e == cudaSuccess; ++i) {
        float t = 0.f;
        e = cudaEventElapsedTime(&t, pool[2 * i], pool[2 * i + 1]);
        ms[kid[i]] += t;
        n[kid[i]] += 1;
    }
    used = 0;
    return e;
}

Launch::~Launch()
{
    for (cudaEvent_t ev : pool) cudaEventDestroy(ev);
}

}  // namespace sphbuf

struct sph_ctx {
    sph_grid grid{};
    float h = 0.f;
    int64_t capacity = 0;
    int max_ports = 0;
    int64_t max_new = 0;
    int64_t max_migrate = 0;
    int n_extra = 0;
    GridDev gd{};
    PortTable pt{};
    std::vector<PortHost> ports;
    std::vector<int> runs;   // 3 ints per run: c0, c1, port (ports in registration order)
    std::vector<int> run_base, run_cnt;   // per port: first run and run count in `runs`
    // the update prologue K5 run inside the last build's scatter: valid for the
    // run table version and cell tables it saw, consumed by the next update
    unsigned runs_ver = 0;
    bool pro_ready = false;
    // call order: build -> update -> compact; the update's deletion
    // list and staging area are live until the compaction consumes them
    bool update_pending = false;
    unsigned pro_ver = 0;
    const int32_t *pro_cs = nullptr, *pro_ce = nullptr;
    std::vector<int> run_cap;             // per port: > 0 once movable (device-enumerated slice)
    std::vector<sph_bc> bcs;              // per port: the last BC set
    std::vector<sph_driver> drivers;      // per port: time-dependent driver (kind NONE if none)
    std::vector<double> drv_u0;           // per port: the Fourier speed in use
    DriverLaunch drv_launch{};            // staging of the Windkessel kernel parameter
    void *ws = nullptr;
    size_t ws_bytes = 0;
    Workspace W{};
    Launch L;
    std::string err;
    // advection of the last sph_cll_key, applied by the gather of sph_cll_finish
    bool key_advect = false;
    float key_dt = 0.f;
    // key carry-over (sphbuf_cll.cu): the last build's gather prepared the keys and
    // histogram of a next build that advects by carry_dt the arrays (carry_x,
    // carry_id) it wrote; the update, compaction and port moves keep them current
    bool carry_next = false;
    bool carry_mig = false;   // made with slab migration (leaver list)
    float carry_dt = 0.f;
    const float *carry_x = nullptr;
    const int64_t *carry_id = nullptr;
    CllCarry key_cc{};
    // multi-GPU (§8(e)): the library's communicator (sph_comm_init / _loopback)
    Comm *comm = nullptr;
    const int32_t *last_port_counts = nullptr;   // the last update's counts (loopback allgather source)
};

namespace {
// In-process loopback group: contexts of one process on one device exchange
// through device copies on the caller's stream (tests; no kernel waits on another).
struct LoopGroup {
    std::vector<sph_ctx *> m;
    int live = 0;
};
}  // namespace

namespace {

sph_status fail(sph_ctx *c, sph_status s, const std::string &m)
{
    if (c) c->err = m;
    return s;
}

sph_status cuda_fail(sph_ctx *c, cudaError_t e, const char *where)
{
    return fail(c, SPH_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// Workspace layout; with base == nullptr only computes the size.
size_t layout(const sph_ctx *c, char *base, Workspace *W)
{
    size_t off = 0;
    auto take = [&](size_t bytes) -> char * {
        char *p = base ? base + off : nullptr;
        off += align256(bytes);
        return p;
    };
    const long long ncells = c->gd.ncells;
    const long long cap = c->capacity;
    const long long cell_tiles = (ncells + kCellTile - 1) / kCellTile + 1;
    const long long upd_tiles = (2 * cap + kUpdTile - 1) / kUpdTile + 64;
    const long long cmp_tiles = (cap + kCntTile - 1) / kCntTile + 1;
    const long long cmp_subs = cmp_tiles * (kCntTile / kCmpTile);
    Workspace w{};
    w.ctr = (Counters *)take(sizeof(Counters));
    w.cell_count = (int *)take(sizeof(int) * ncells);
    w.cursor = (int *)take(sizeof(int) * ncells);
    w.tile_cells = (unsigned long long *)take(8 * cell_tiles);
    w.tile_runs = (unsigned long long *)take(8 * (kMaxRuns / 256 + 1));
    w.tile_cmp = (unsigned long long *)take(8 * cmp_tiles);
    w.rd = (unsigned *)take(4 * cmp_subs);
    w.runs = (int *)take(sizeof(int) * 3 * kMaxRuns);
    w.drv = (DriverDev *)take(sizeof(DriverDev) * SPH_MAX_PORTS);
    w.drv_rho = (float *)take(sizeof(float) * SPH_MAX_PORTS);
    w.port_cnt = (int *)take(sizeof(int) * 2 * SPH_MAX_PORTS);
    w.del_list = (int *)take(sizeof(int) * kDelList);
    w.run_off = (long long *)take(sizeof(long long) * (kMaxRuns + 1));
    const size_t zero_end = off;   // everything above must start zeroed
    w.sub_off = (unsigned *)take(4 * cmp_subs);
    w.run_base = (int *)take(sizeof(int) * kMaxRuns);
    w.tile_run = (int *)take(sizeof(int) * upd_tiles);
    w.tile_cr = (unsigned *)take(4 * upd_tiles);
    w.tile_pre = (unsigned *)take(4 * upd_tiles);
    w.key = (int *)take(sizeof(int) * cap);
    w.src = (int *)take(sizeof(int) * cap);
    w.max_leave = 2 * c->max_migrate + 1024;
    w.leave = (int *)take(sizeof(int) * w.max_leave);
    const long long mn = c->max_new;
    w.sx = (float *)take(4 * mn);
    w.sy = (float *)take(4 * mn);
    w.svx = (float *)take(4 * mn);
    w.svy = (float *)take(4 * mn);
    if (c->grid.dim == 3) {
        w.sz = (float *)take(4 * mn);
        w.svz = (float *)take(4 * mn);
    }
    for (int e = 0; e < c->n_extra; ++e) w.sextra[e] = (float *)take(4 * mn);
    if (c->max_migrate > 0) {
        const long long mig = 4 + c->max_migrate * (long long)(2 * c->grid.dim + c->n_extra + 3);
        for (int b = 0; b < 4; ++b) w.mig[b] = (float *)take(4 * mig);
    }
    w.sid = (long long *)take(8 * mn);
    w.sport = (int *)take(4 * mn);
    w.stile = (int *)take(4 * mn);
    w.sexcl = (int *)take(4 * mn);
    w.max_new = mn;
    w.upd_tiles = upd_tiles;
    w.cmp_tiles = cmp_tiles;
    if (W) *W = w;
    (void)zero_end;
    return off;
}

size_t zero_bytes(const sph_ctx *c)
{
    // Counters .. run_off (the regions read before being written)
    Workspace w{};
    char *fake = reinterpret_cast<char *>(size_t(1) << 40);
    layout(c, fake, &w);
    return (size_t)(reinterpret_cast<char *>(w.sub_off) - fake);
}

PartDev part_dev(const sph_particles *p)
{
    PartDev d{};
    d.x = p->x; d.y = p->y; d.z = p->z;
    d.vx = p->vx; d.vy = p->vy; d.vz = p->vz;
    for (int e = 0; e < SPH_MAX_EXTRA; ++e) d.extra[e] = p->extra[e];
    d.n_extra = p->n_extra;
    d.id = reinterpret_cast<long long *>(p->id);
    d.label = p->label;
    d.n = reinterpret_cast<long long *>(p->n_dev);
    d.cap = p->capacity;
    return d;
}

sph_status check_particles(sph_ctx *c, const sph_particles *p)
{
    if (!p || !p->x || !p->y || !p->vx || !p->vy || !p->id || !p->label || !p->n_dev)
        return fail(c, SPH_ERR_ARG, "particles: NULL column");
    if (c->grid.dim == 3 && (!p->z || !p->vz)) return fail(c, SPH_ERR_ARG, "particles: z/vz required in 3-D");
    if (p->n_extra != c->n_extra) return fail(c, SPH_ERR_ARG, "particles: n_extra differs from the context");
    for (int e = 0; e < p->n_extra; ++e)
        if (!p->extra[e]) return fail(c, SPH_ERR_ARG, "particles: NULL extra column");
    if (p->capacity > c->capacity) return fail(c, SPH_ERR_ARG, "particles: capacity exceeds the context's");
    if (!c->ws) return fail(c, SPH_ERR_STATE, "no workspace set");
    return SPH_OK;
}

// ---- geometry (f64) ----------------------------------------------------------

PortHost make_port_host(const float o[3], const float Q[9], const float he[3], float cs, int dim, double inflate)
{
    PortHost P{};
    for (int r = 0; r < 3; ++r) {
        P.o[r] = (dim == 2 && r == 2) ? 0.0 : (double)o[r];
        for (int j = 0; j < 3; ++j) P.ax[r][j] = (double)Q[3 * r + j];
        P.H[r] = (double)he[r] + (double)cs + inflate;
    }
    if (dim == 2) {
        P.ax[0][2] = P.ax[1][2] = 0.0;
        P.ax[2][0] = P.ax[2][1] = 0.0;
        P.ax[2][2] = 1.0;
        P.H[2] = 0.0;
    }
    return P;
}

double dot(const double *a, const double *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

// Separating-axis test between an axis-aligned box (centre c, half sizes e) and
// an oriented box (centre o, unit axes ax, half sizes H).
bool aabb_obb_overlap(const double c[3], const double e[3], const PortHost &P, int dim)
{
    const double t[3] = {P.o[0] - c[0], P.o[1] - c[1], P.o[2] - c[2]};
    double axes[15][3];
    int na = 0;
    for (int j = 0; j < dim; ++j) {
        axes[na][0] = j == 0; axes[na][1] = j == 1; axes[na][2] = j == 2;
        ++na;
    }
    for (int r = 0; r < dim; ++r) {
        for (int j = 0; j < 3; ++j) axes[na][j] = P.ax[r][j];
        ++na;
    }
    if (dim == 3) {
        for (int j = 0; j < 3; ++j)
            for (int r = 0; r < 3; ++r) {
                double u[3] = {double(j == 0), double(j == 1), double(j == 2)};
                double w[3] = {u[1] * P.ax[r][2] - u[2] * P.ax[r][1], u[2] * P.ax[r][0] - u[0] * P.ax[r][2],
                               u[0] * P.ax[r][1] - u[1] * P.ax[r][0]};
                if (dot(w, w) < 1e-20) continue;
                for (int q = 0; q < 3; ++q) axes[na][q] = w[q];
                ++na;
            }
    }
    for (int a = 0; a < na; ++a) {
        const double *L = axes[a];
        const double ra = std::fabs(L[0]) * e[0] + std::fabs(L[1]) * e[1] + std::fabs(L[2]) * e[2];
        double rb = 0.0;
        for (int r = 0; r < 3; ++r) rb += std::fabs(dot(L, P.ax[r])) * P.H[r];
        if (std::fabs(dot(L, t)) > ra + rb) return false;
    }
    return true;
}

bool obb_obb_overlap(const PortHost &A, const PortHost &B, int dim)
{
    const double t[3] = {B.o[0] - A.o[0], B.o[1] - A.o[1], B.o[2] - A.o[2]};
    std::vector<std::array<double, 3>> axes;
    for (int r = 0; r < dim; ++r) axes.push_back({A.ax[r][0], A.ax[r][1], A.ax[r][2]});
    for (int r = 0; r < dim; ++r) axes.push_back({B.ax[r][0], B.ax[r][1], B.ax[r][2]});
    if (dim == 3)
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                const double *a = A.ax[i], *b = B.ax[j];
                std::array<double, 3> w = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2],
                                           a[0] * b[1] - a[1] * b[0]};
                if (w[0] * w[0] + w[1] * w[1] + w[2] * w[2] > 1e-20) axes.push_back(w);
            }
    for (auto &L : axes) {
        double ra = 0.0, rb = 0.0;
        for (int r = 0; r < 3; ++r) {
            ra += std::fabs(dot(L.data(), A.ax[r])) * A.H[r];
            rb += std::fabs(dot(L.data(), B.ax[r])) * B.H[r];
        }
        if (std::fabs(dot(L.data(), t)) > ra + rb) return false;
    }
    return true;
}

// Cells of the slab that intersect the oriented box P, as runs of consecutive
// local cell ids along the fastest axis (z in 3-D, y in 2-D).  A column of cells
// meets a convex box in one interval, so each column gives at most one run.
void enumerate_runs(const sph_grid &g, const PortHost &P, std::vector<int> &runs, long long &ncells_hit)
{
    const int dim = g.dim;
    const double cs = (double)g.cs;
    double ext[3];
    for (int j = 0; j < 3; ++j) {
        ext[j] = 0.0;
        for (int r = 0; r < 3; ++r) ext[j] += std::fabs(P.ax[r][j]) * P.H[r];
    }
    const int nz = dim == 3 ? g.ncell[2] : 1;
    const int ny = g.ncell[1];
    int lo_c[3], hi_c[3];
    const int nc[3] = {g.ncell[0], g.ncell[1], nz};
    for (int j = 0; j < dim; ++j) {
        lo_c[j] = (int)std::floor((P.o[j] - ext[j] - (double)g.lo[j]) / cs) - 1;
        hi_c[j] = (int)std::floor((P.o[j] + ext[j] - (double)g.lo[j]) / cs) + 1;
        lo_c[j] = std::max(lo_c[j], 0);
        hi_c[j] = std::min(hi_c[j], nc[j] - 1);
    }
    if (dim == 2) { lo_c[2] = 0; hi_c[2] = 0; }
    lo_c[0] = std::max(lo_c[0], g.cx_begin);
    hi_c[0] = std::min(hi_c[0], g.cx_end - 1);
    const double half[3] = {0.5 * cs, 0.5 * cs, dim == 3 ? 0.5 * cs : 0.0};
    const int fast = dim - 1;   // axis along which runs extend
    ncells_hit = 0;
    for (int cx = lo_c[0]; cx <= hi_c[0]; ++cx) {
        const int ymax = dim == 3 ? hi_c[1] : lo_c[1];   // in 2-D the column is along y
        for (int cy = lo_c[1]; cy <= ymax; ++cy) {
            int first = -1, last = -1;
            for (int f = lo_c[fast]; f <= hi_c[fast]; ++f) {
                const int ix[3] = {cx, dim == 3 ? cy : f, dim == 3 ? f : 0};
                double ctr[3];
                for (int j = 0; j < 3; ++j)
                    ctr[j] = (j < dim) ? (double)g.lo[j] + (ix[j] + 0.5) * cs : 0.0;
                if (aabb_obb_overlap(ctr, half, P, dim)) {
                    if (first < 0) first = f;
                    last = f;
                } else if (first >= 0) {
                    break;
                }
            }
            if (first < 0) continue;
            int c0, c1;
            if (dim == 3) {
                c0 = ((cx - g.cx_begin) * ny + cy) * nz + first;
                c1 = ((cx - g.cx_begin) * ny + cy) * nz + last;
            } else {
                c0 = (cx - g.cx_begin) * ny + first;
                c1 = (cx - g.cx_begin) * ny + last;
            }
            runs.push_back(c0);
            runs.push_back(c1);
            ncells_hit += last - first + 1;
        }
    }
}

}  // namespace

// =============================================================================== ABI

extern "C" {

sph_status sph_ctx_create(const sph_grid *grid, float h, int64_t capacity, int32_t max_ports, int64_t max_new,
                          int64_t max_migrate, int32_t n_extra, sph_ctx **out)
{
    if (!grid || !out) return SPH_ERR_ARG;
    *out = nullptr;
    if (grid->dim != 2 && grid->dim != 3) return SPH_ERR_ARG;
    if (!(grid->cs > 0.f) || !(h > 0.f) || grid->cs < 2.0f * h * (1.0f - 1e-6f)) return SPH_ERR_ARG;   // cs >= 2h
    for (int j = 0; j < grid->dim; ++j)
        if (grid->ncell[j] <= 0) return SPH_ERR_ARG;
    if (grid->dim == 2 && grid->ncell[2] != 1) return SPH_ERR_ARG;
    if (grid->cx_begin < 0 || grid->cx_end > grid->ncell[0] || grid->cx_begin >= grid->cx_end) return SPH_ERR_ARG;
    if (capacity < 0 || capacity >= (int64_t(1) << 31)) return SPH_ERR_ARG;
    if (max_ports <= 0 || max_ports > SPH_MAX_PORTS) return SPH_ERR_ARG;
    if (max_new < 0 || max_migrate < 0 || n_extra < 0 || n_extra > SPH_MAX_EXTRA) return SPH_ERR_ARG;
    const long long ncells =
        (long long)(grid->cx_end - grid->cx_begin) * grid->ncell[1] * (grid->dim == 3 ? grid->ncell[2] : 1);
    if (ncells >= (1ll << 31)) return SPH_ERR_ARG;
    sph_ctx *c = new sph_ctx();
    c->grid = *grid;
    c->h = h;
    c->capacity = capacity;
    c->max_ports = max_ports;
    c->max_new = max_new;
    c->max_migrate = max_migrate;
    c->n_extra = n_extra;
    GridDev &g = c->gd;
    g.dim = grid->dim;
    for (int j = 0; j < 3; ++j) {
        g.lo[j] = grid->lo[j];
        g.ncell[j] = grid->ncell[j];
    }
    g.inv_cs = (float)(1.0 / (double)grid->cs);
    g.cx_begin = grid->cx_begin;
    g.cx_end = grid->cx_end;
    g.ny = grid->ncell[1];
    g.nz = grid->dim == 3 ? grid->ncell[2] : 1;
    g.ncells = ncells;
    c->pt.n = 0;
    c->pt.max_ports = max_ports;
    *out = c;
    return SPH_OK;
}

void sph_ctx_destroy(sph_ctx *c)
{
    if (!c) return;
    if (c->comm) {
        if (c->comm->kind == Comm::LOOPBACK) {
            LoopGroup *g = static_cast<LoopGroup *>(c->comm->loop);
            g->m[c->comm->rank] = nullptr;
            if (--g->live == 0) delete g;
        }
        comm_destroy(c->comm);
    }
    delete c;
}

const char *sph_last_error(const sph_ctx *c) { return c ? c->err.c_str() : "null context"; }

size_t sph_workspace_bytes(const sph_ctx *c) { return c ? layout(c, nullptr, nullptr) : 0; }

// Key carry-over plan of a build of `in` (see sph_ctx): reuse the carried keys
// when `in` is the array they were made for and the advection is the same; make
// new ones when this build advects and does not migrate (SPHBUF_CARRY=0: never).
static CllCarry carry_plan(const sph_ctx *c, const sph_particles *in, bool advect, float dt, bool migrating)
{
    static int enabled = -1;
    if (enabled < 0) {
        const char *v = getenv("SPHBUF_CARRY");
        enabled = (v && v[0] == '0') ? 0 : 1;
    }
    CllCarry cc;
    const bool match = c->carry_next && advect && migrating == c->carry_mig && in->x == c->carry_x &&
                       in->id == c->carry_id && dt == c->carry_dt;
    cc.use = match;
    cc.clear = c->carry_next && !match;
    cc.make = enabled && advect;
    cc.mig = migrating;
    cc.dt = dt;
    return cc;
}

static void carry_after_build(sph_ctx *c, const CllCarry &cc, const sph_particles *out)
{
    c->carry_next = cc.make;
    c->carry_mig = cc.mig;
    c->carry_dt = cc.dt;
    c->carry_x = out->x;
    c->carry_id = out->id;
}

// The carry mode of the kernels that change particles of `p` (0 when the carried
// keys do not describe `p`, the arrays the last build wrote; 2 with migration).
static int carry_on(const sph_ctx *c, const sph_particles *p)
{
    if (!(c->carry_next && p->x == c->carry_x && p->id == c->carry_id)) return 0;
    return c->carry_mig ? 2 : 1;
}

// Positions or arrays changed behind the carried keys: the next build clears the
// carried histogram and runs the key pass.
static void carry_drop(sph_ctx *c)
{
    c->carry_x = nullptr;
    c->carry_id = nullptr;
}

static cudaError_t enumerate_slice(sph_ctx *c, int k, const float o[3], const float Q[9], cudaStream_t s);

sph_status sph_set_workspace(sph_ctx *c, void *d_ws, size_t bytes)
{
    if (!c || !d_ws) return SPH_ERR_ARG;
    if (bytes < layout(c, nullptr, nullptr)) return fail(c, SPH_ERR_ARG, "workspace too small");
    if (reinterpret_cast<size_t>(d_ws) % 256) return fail(c, SPH_ERR_ARG, "workspace not 256-byte aligned");
    c->ws = d_ws;
    c->ws_bytes = bytes;
    c->carry_next = false;   // the histogram is zeroed below
    layout(c, static_cast<char *>(d_ws), &c->W);
    cudaError_t e = cudaMemset(d_ws, 0, zero_bytes(c));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "sph_set_workspace");
    ++c->runs_ver;
    if (!c->runs.empty()) {
        e = cudaMemcpy(c->W.runs, c->runs.data(), sizeof(int) * c->runs.size(), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cuda_fail(c, e, "sph_set_workspace runs");
        for (int q = 0; q < c->pt.n; ++q)   // movable ports: their slices live on the device only
            if (c->run_cap[q] > 0 && (e = enumerate_slice(c, q, c->pt.p[q].o, c->pt.p[q].Q, 0)) != cudaSuccess)
                return cuda_fail(c, e, "sph_set_workspace enumeration");
    }
    return SPH_OK;
}

// Pose checks shared by registration and sph_port_move: Q a rotation (planar in
// 2-D), P_k strictly inside the grid, P_k disjoint from every other port's
// (port `skip` excluded: the port being moved).
static sph_status check_pose(sph_ctx *c, const float origin[3], const float Q[9], const float he[3], int skip)
{
    const int dim = c->grid.dim;
    // orthonormality and handedness
    double M[9];
    for (int i = 0; i < 9; ++i) M[i] = Q[i];
    double worst = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int l = 0; l < 3; ++l) s += M[3 * i + l] * M[3 * j + l];
            worst = std::max(worst, std::fabs(s - (i == j ? 1.0 : 0.0)));
        }
    const double det = M[0] * (M[4] * M[8] - M[5] * M[7]) - M[1] * (M[3] * M[8] - M[5] * M[6]) +
                       M[2] * (M[3] * M[7] - M[4] * M[6]);
    if (worst > 1e-5 || det <= 0.0) return fail(c, SPH_ERR_NOT_ORTHONORMAL, "Q is not a rotation");
    if (dim == 2 && (std::fabs(M[2]) > 1e-6 || std::fabs(M[5]) > 1e-6 || std::fabs(M[6]) > 1e-6 ||
                     std::fabs(M[7]) > 1e-6 || std::fabs(M[8] - 1.0) > 1e-6))
        return fail(c, SPH_ERR_NOT_ORTHONORMAL, "2-D Q must be planar");
    // P_k strictly inside the grid
    PortHost P = make_port_host(origin, Q, he, c->grid.cs, dim, 0.0);
    for (int j = 0; j < dim; ++j) {
        double ext = 0.0;
        for (int r = 0; r < 3; ++r) ext += std::fabs(P.ax[r][j]) * P.H[r];
        const double lo = (double)c->grid.lo[j];
        const double hi = lo + (double)c->grid.ncell[j] * (double)c->grid.cs;
        if (!(P.o[j] - ext > lo && P.o[j] + ext < hi)) return fail(c, SPH_ERR_OUT_OF_GRID, "P_k leaves the grid");
    }
    // disjoint decision regions (the paper never overlaps buffers; each particle
    // then gets at most one decision)
    for (size_t j = 0; j < c->ports.size(); ++j)
        if ((int)j != skip && obb_obb_overlap(P, c->ports[j], dim))
            return fail(c, SPH_ERR_OVERLAP, "P_k overlaps an existing port");
    return SPH_OK;
}

sph_status sph_port_check(const sph_ctx *cc, const float origin[3], const float Q[9], const float he[3], int32_t kind,
                          int32_t layers, float dp)
{
    sph_ctx *c = const_cast<sph_ctx *>(cc);
    if (!c || !origin || !Q || !he) return fail(c, SPH_ERR_ARG, "NULL argument");
    const int dim = c->grid.dim;
    if (kind < SPH_INLET || kind > SPH_BIDIRECTIONAL) return fail(c, SPH_ERR_ARG, "bad kind");
    if (c->pt.n >= c->max_ports) return fail(c, SPH_ERR_ARG, "too many ports");
    // at least three layers of particles; a = layers * dp
    if (layers < 3 || !(dp > 0.f)) return fail(c, SPH_ERR_ARG, "layers < 3 or dp <= 0");
    for (int r = 0; r < dim; ++r)
        if (!(he[r] > 0.f)) return fail(c, SPH_ERR_ARG, "half extents must be positive");
    const double a = 2.0 * (double)he[0];
    if (std::fabs(a - layers * (double)dp) > 1e-5 * layers * (double)dp)
        return fail(c, SPH_ERR_ARG, "2*half_extents[0] != layers*dp");
    return check_pose(c, origin, Q, he, -1);
}

sph_status sph_port_cells(const sph_grid *grid, const float origin[3], const float Q[9], const float he[3],
                          int32_t *runs_out, int64_t max_runs, int64_t *n_runs, int64_t *n_cells)
{
    if (!grid || !origin || !Q || !he) return SPH_ERR_ARG;
    PortHost P = make_port_host(origin, Q, he, grid->cs, grid->dim, 1e-3 * (double)grid->cs);
    std::vector<int> runs;
    long long hit = 0;
    enumerate_runs(*grid, P, runs, hit);
    const int64_t nr = (int64_t)runs.size() / 2;
    if (n_runs) *n_runs = nr;
    if (n_cells) *n_cells = hit;
    if (runs_out) {
        if (nr > max_runs) return SPH_ERR_ARG;
        std::memcpy(runs_out, runs.data(), sizeof(int) * runs.size());
    }
    return SPH_OK;
}

sph_status sph_buffer_register(sph_ctx *c, sph_particles *p, const float origin[3], const float Q[9],
                               const float he[3], int32_t kind, int32_t layers, float dp, int32_t *port_id_out,
                               int64_t *members_out_dev, void *stream)
{
    SPH_NVTX("sph_buffer_register");
    if (!c) return SPH_ERR_ARG;
    sph_status st = sph_port_check(c, origin, Q, he, kind, layers, dp);
    if (st != SPH_OK) return st;
    st = check_particles(c, p);
    if (st != SPH_OK) return st;
    const int dim = c->grid.dim;
    const int k = c->pt.n;
    // device parameters (pinned fp32: heP = fl(he + cs), s = fl(fl(2 he_0) * u))
    PortDev &D = c->pt.p[k];
    std::memset(&D, 0, sizeof(D));
    for (int j = 0; j < 3; ++j) {
        D.o[j] = (dim == 2 && j == 2) ? 0.f : origin[j];
        D.he[j] = he[j];
        volatile float sum = he[j] + c->grid.cs;
        D.heP[j] = sum;
    }
    for (int i = 0; i < 9; ++i) D.Q[i] = Q[i];
    const float a = 2.0f * he[0];
    for (int j = 0; j < 3; ++j) {
        volatile float prod = a * Q[j];
        D.s[j] = (dim == 2 && j == 2) ? 0.f : prod;
    }
    D.kind = kind;
    D.bc = SPH_BC_NONE;
    D.rho_col = -1;
    // host geometry and this slab's runs (inflated by 1e-3 cs to absorb fp32 rounding)
    PortHost P = make_port_host(origin, Q, he, c->grid.cs, dim, 0.0);
    PortHost Pi = make_port_host(origin, Q, he, c->grid.cs, dim, 1e-3 * (double)c->grid.cs);
    std::vector<int> r2;
    long long hit = 0;
    enumerate_runs(c->grid, Pi, r2, hit);
    const size_t before = c->runs.size();
    ++c->runs_ver;
    if ((before + r2.size() / 2 * 3) / 3 > (size_t)kMaxRuns) return fail(c, SPH_ERR_ARG, "too many port runs");
    for (size_t i = 0; i < r2.size(); i += 2) {
        c->runs.push_back(r2[i]);
        c->runs.push_back(r2[i + 1]);
        c->runs.push_back(k);
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaSuccess;
    if (c->runs.size() > before)
        e = cudaMemcpyAsync(c->W.runs + before, c->runs.data() + before, sizeof(int) * (c->runs.size() - before),
                            cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) {
        c->runs.resize(before);
        return cuda_fail(c, e, "register: upload runs");
    }
    c->ports.push_back(P);
    c->run_base.push_back((int)(before / 3));
    c->run_cnt.push_back((int)(r2.size() / 2));
    c->run_cap.push_back(0);
    c->bcs.push_back(sph_bc{});
    c->drivers.push_back(sph_driver{});
    c->drv_u0.push_back(0.0);
    c->pt.n = k + 1;
    if (members_out_dev) {
        e = cudaMemsetAsync(members_out_dev, 0, sizeof(int64_t), s);
        if (e != cudaSuccess) return cuda_fail(c, e, "register: memset");
    }
    e = launch_register(part_dev(p), c->gd, c->pt, k, reinterpret_cast<long long *>(members_out_dev), s, &c->L);
    if (e != cudaSuccess) return cuda_fail(c, e, "register: identification kernel");
    if (port_id_out) *port_id_out = k;
    return SPH_OK;
}

// Movable ports (sph_port_move): the slice of one run slot per cell column of a
// window of `span` columns per axis around the bounding sphere of the inflated
// decision region; any pose of the port fits in it.
static int move_span(const sph_ctx *c, int k)
{
    const PortDev &D = c->pt.p[k];
    const double cs = (double)c->grid.cs, inf = 1e-3 * cs;
    double r2 = 0.0;
    for (int j = 0; j < c->grid.dim; ++j) {
        const double H = (double)D.he[j] + cs + inf;
        r2 += H * H;
    }
    return (int)std::floor(2.0 * std::sqrt(r2) / cs) + 3;
}

static int move_slice_cap(const sph_ctx *c, int k)
{
    const int span = move_span(c, k);
    return c->grid.dim == 3 ? span * span : span;
}

// K10 launch for port k at pose (o, Q) into its slice.
static cudaError_t enumerate_slice(sph_ctx *c, int k, const float o[3], const float Q[9], cudaStream_t s)
{
    const int dim = c->grid.dim;
    float he[3];
    for (int j = 0; j < 3; ++j) he[j] = c->pt.p[k].he[j];
    const PortHost Pi = make_port_host(o, Q, he, c->grid.cs, dim, 1e-3 * (double)c->grid.cs);
    const double cs = (double)c->grid.cs;
    double r2 = 0.0;
    for (int j = 0; j < dim; ++j) r2 += Pi.H[j] * Pi.H[j];
    const double R = std::sqrt(r2);
    const int span = move_span(c, k);
    PortEnum E{};
    for (int r = 0; r < 3; ++r) {
        E.o[r] = Pi.o[r];
        E.H[r] = Pi.H[r];
        for (int j = 0; j < 3; ++j) E.ax[r][j] = Pi.ax[r][j];
    }
    auto first_cell = [&](int j) { return (int)std::floor((Pi.o[j] - R - (double)c->grid.lo[j]) / cs) - 1; };
    const int fast = dim - 1;
    E.cx0 = first_cell(0);
    E.ncx = span;
    E.cy0 = dim == 3 ? first_cell(1) : 0;
    E.ncy = dim == 3 ? span : 1;
    E.f0 = std::max(first_cell(fast), 0);
    E.f1 = std::min(first_cell(fast) + span - 1, c->grid.ncell[fast] - 1);
    E.k = k;
    return launch_port_enum(c->gd, E, c->grid.cs, c->W.runs + 3 * (size_t)c->run_base[k], c->run_cap[k], s, &c->L);
}

sph_status sph_port_move(sph_ctx *c, sph_particles *p, int32_t k, const float origin[3], const float Q[9],
                         const int32_t *cell_start, const int32_t *cell_end, void *stream)
{
    SPH_NVTX("sph_port_move");
    if (!c) return SPH_ERR_ARG;
    if (!origin || !Q || !cell_start || !cell_end) return fail(c, SPH_ERR_ARG, "NULL argument");
    if (k < 0 || k >= c->pt.n) return fail(c, SPH_ERR_ARG, "unknown port");
    if (!c->ws) return fail(c, SPH_ERR_STATE, "no workspace set");
    sph_status st = check_particles(c, p);
    if (st != SPH_OK) return st;
    ++c->runs_ver;   // the port's runs (and maybe the run table layout) change
    const int dim = c->grid.dim;
    PortDev P1 = c->pt.p[k];
    float o1[3], he[3];
    for (int j = 0; j < 3; ++j) {
        o1[j] = (dim == 2 && j == 2) ? 0.f : origin[j];
        he[j] = P1.he[j];
    }
    st = check_pose(c, o1, Q, he, k);
    if (st != SPH_OK) return st;
    for (int j = 0; j < 3; ++j) P1.o[j] = o1[j];
    for (int i = 0; i < 9; ++i) P1.Q[i] = Q[i];
    const float a = 2.0f * P1.he[0];
    for (int j = 0; j < 3; ++j) {
        volatile float prod = a * Q[j];            // recycle shift s = fl(a u) of the new axis (R10)
        P1.s[j] = (dim == 2 && j == 2) ? 0.f : prod;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // 1. the buffer particles, found among the port's candidates of the current build
    cudaError_t e = launch_port_move(part_dev(p), c->gd, c->pt.p[k], P1, c->W.runs + 3 * (size_t)c->run_base[k],
                                     c->run_cnt[k], cell_start, cell_end, k, nullptr, c->W, carry_on(c, p),
                                     c->carry_dt, s, &c->L);
    if (e != cudaSuccess) return cuda_fail(c, e, "port_move");
    // 2. first move: the port's runs become a fixed device slice, one slot per cell
    //    column of a window around its bounding sphere (any pose fits); the table is
    //    re-laid out, so the other movable ports' slices are enumerated again
    if (c->run_cap[k] == 0) {
        const int cap = move_slice_cap(c, k);
        std::vector<int> nr;
        std::vector<int> base(c->pt.n), cnt(c->pt.n);
        for (int q = 0; q < c->pt.n; ++q) {
            base[q] = (int)(nr.size() / 3);
            const int m = q == k ? cap : c->run_cnt[q];
            if (q == k || c->run_cap[q] > 0) {
                for (int i = 0; i < m; ++i) {
                    nr.push_back(0);
                    nr.push_back(-1);
                    nr.push_back(q);
                }
            } else {
                nr.insert(nr.end(), c->runs.begin() + 3 * (size_t)c->run_base[q],
                          c->runs.begin() + 3 * (size_t)(c->run_base[q] + c->run_cnt[q]));
            }
            cnt[q] = m;
        }
        if (nr.size() / 3 > (size_t)kMaxRuns) return fail(c, SPH_ERR_ARG, "too many port runs");
        // pageable source: staged before return, so later host edits cannot race it
        e = cudaMemcpyAsync(c->W.runs, nr.data(), sizeof(int) * nr.size(), cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_fail(c, e, "port_move: upload runs");
        c->runs.swap(nr);
        c->run_base = base;
        c->run_cnt = cnt;
        c->run_cap[k] = cap;
        for (int q = 0; q < c->pt.n; ++q) {
            if (q == k || c->run_cap[q] == 0) continue;
            e = enumerate_slice(c, q, c->pt.p[q].o, c->pt.p[q].Q, s);
            if (e != cudaSuccess) return cuda_fail(c, e, "port_move: enumeration");
        }
    }
    // 3. the candidate cells of the new pose, enumerated on the device
    e = enumerate_slice(c, k, o1, Q, s);
    if (e != cudaSuccess) return cuda_fail(c, e, "port_move: enumeration");
    // 4. the re-established frame for the next update
    c->pt.p[k] = P1;
    c->ports[k] = make_port_host(o1, Q, he, c->grid.cs, dim, 0.0);
    return SPH_OK;
}

sph_status sph_port_set_bc(sph_ctx *c, int32_t port_id, const sph_bc *bc)
{
    if (!c || !bc) return SPH_ERR_ARG;
    if (port_id < 0 || port_id >= c->pt.n) return fail(c, SPH_ERR_ARG, "unknown port");
    PortDev &D = c->pt.p[port_id];
    if (bc->kind == SPH_BC_NONE) {
        D.bc = SPH_BC_NONE;
        return SPH_OK;
    }
    if (bc->kind == SPH_BC_PRESSURE) {
        if (!(bc->c0 > 0.f) || bc->rho_column < -1 || bc->rho_column >= c->n_extra)
            return fail(c, SPH_ERR_ARG, "pressure BC: c0 <= 0 or bad density column");
        D.rho_col = bc->rho_column;
        // Eq. postulate-density, formed in f64, rounded once
        D.rho_b = (float)((double)bc->rho0 + (double)bc->p_b / ((double)bc->c0 * (double)bc->c0));
    } else if (bc->kind == SPH_BC_VELOCITY) {
        if (bc->profile < SPH_PROFILE_PLUG || bc->profile > SPH_PROFILE_PARABOLIC_RADIAL)
            return fail(c, SPH_ERR_ARG, "velocity BC: bad profile");
        if (bc->profile != SPH_PROFILE_PLUG && !(bc->radius > 0.f))
            return fail(c, SPH_ERR_ARG, "velocity BC: radius <= 0");
        D.profile = bc->profile;
        D.u0 = bc->u0;
        D.R = bc->radius;
        volatile float r2 = bc->radius * bc->radius;
        D.R2 = r2;
    } else {
        return fail(c, SPH_ERR_ARG, "bad BC kind");
    }
    D.bc = bc->kind;
    c->bcs[port_id] = *bc;
    return SPH_OK;
}

sph_status sph_port_set_driver(sph_ctx *c, int32_t k, const sph_driver *d)
{
    if (!c || !d) return SPH_ERR_ARG;
    if (k < 0 || k >= c->pt.n) return fail(c, SPH_ERR_ARG, "unknown port");
    if (!c->ws) return fail(c, SPH_ERR_STATE, "no workspace set");
    PortDev &D = c->pt.p[k];
    if (d->kind == SPH_DRIVER_NONE) {
        D.rho_dev = 0;
        c->drivers[k] = *d;
        return SPH_OK;
    }
    if (d->kind == SPH_DRIVER_FOURIER) {
        if (D.bc != SPH_BC_VELOCITY) return fail(c, SPH_ERR_ARG, "Fourier driver needs a velocity BC");
    } else if (d->kind == SPH_DRIVER_WINDKESSEL) {
        if (D.bc != SPH_BC_PRESSURE) return fail(c, SPH_ERR_ARG, "Windkessel driver needs a pressure BC");
        if (!(d->Rp > 0.0) || !(d->C > 0.0) || !(d->Rd > 0.0) || !(d->volume > 0.0))
            return fail(c, SPH_ERR_ARG, "Windkessel: Rp, C, Rd, volume must be positive");
        DriverDev st{};
        st.P = d->P0;
        st.first = 1;
        const sph_bc &bc = c->bcs[k];
        const float rho = (float)((double)bc.rho0 + d->P0 / ((double)bc.c0 * (double)bc.c0));
        cudaError_t e = cudaMemcpy(c->W.drv + k, &st, sizeof(st), cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(c->W.drv_rho + k, &rho, sizeof(rho), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cuda_fail(c, e, "set_driver");
        D.rho_dev = 1;
    } else {
        return fail(c, SPH_ERR_ARG, "bad driver kind");
    }
    c->drivers[k] = *d;
    return SPH_OK;
}

// Eq. Fourier_Series: a0 + sum a_n cos(n t w) + sum b_n sin(n t w), the
// two sums in that order, f64.
static double fourier_speed(const sph_driver &d, double t)
{
    double u = d.a[0];
    for (int n = 1; n <= 8; ++n) u = u + d.a[n] * std::cos(((double)n * t) * d.omega);
    for (int n = 1; n <= 8; ++n) u = u + d.b[n] * std::sin(((double)n * t) * d.omega);
    return u;
}

sph_status sph_drivers_step(sph_ctx *c, sph_particles *p, double t, double dt, const int32_t *cell_start,
                            const int32_t *cell_end, void *stream)
{
    SPH_NVTX("sph_drivers_step");
    if (!c) return SPH_ERR_ARG;
    if (!cell_start || !cell_end) return fail(c, SPH_ERR_ARG, "NULL cell table");
    if (!(dt > 0.0)) return fail(c, SPH_ERR_ARG, "dt <= 0");
    sph_status st = check_particles(c, p);
    if (st != SPH_OK) return st;
    DriverLaunch &L = c->drv_launch;   // host staging of the kernel parameter
    L.n = 0;
    for (int k = 0; k < c->pt.n; ++k) {
        const sph_driver &d = c->drivers[k];
        PortDev &D = c->pt.p[k];
        if (d.kind == SPH_DRIVER_FOURIER) {
            const double u = fourier_speed(d, t);
            c->drv_u0[k] = u;
            D.u0 = (float)u;
        } else if (d.kind == SPH_DRIVER_WINDKESSEL) {
            DriverEntry &E = L.e[L.n++];
            E = DriverEntry{};
            E.k = k;
            E.run0 = c->run_base[k];
            E.nrun = c->run_cnt[k];
            for (int j = 0; j < 3; ++j) E.u[j] = D.Q[j];
            E.sign = D.kind == SPH_OUTLET ? 1.0 : -1.0;   // flow out of the domain (R26)
            E.scale = d.volume / (2.0 * (double)D.he[0]);
            E.Rp = d.Rp;
            E.C = d.C;
            E.Rd = d.Rd;
            E.rho0 = (double)c->bcs[k].rho0;
            E.c0sq = (double)c->bcs[k].c0 * (double)c->bcs[k].c0;
            E.dt = dt;
        }
    }
    cudaError_t e = launch_drivers(part_dev(p), c->gd.dim, c->W, L, cell_start, cell_end, static_cast<cudaStream_t>(stream),
                                   &c->L);
    return e == cudaSuccess ? SPH_OK : cuda_fail(c, e, "drivers_step");
}

sph_status sph_driver_read(sph_ctx *c, int32_t k, double out[3], void *stream)
{
    if (!c || !out) return SPH_ERR_ARG;
    if (k < 0 || k >= c->pt.n) return fail(c, SPH_ERR_ARG, "unknown port");
    DriverDev st{};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemcpyAsync(&st, c->W.drv + k, sizeof(st), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(c, e, "driver_read");
    out[0] = st.P;
    out[1] = st.Q;
    out[2] = c->drv_u0[k];
    return SPH_OK;
}

sph_status sph_advect(sph_ctx *c, sph_particles *p, float dt, void *stream)
{
    SPH_NVTX("sph_advect");
    if (!c) return SPH_ERR_ARG;
    sph_status st = check_particles(c, p);
    if (st != SPH_OK) return st;
    carry_drop(c);
    cudaError_t e = launch_advect(part_dev(p), c->grid.dim, dt, static_cast<cudaStream_t>(stream), &c->L);
    return e == cudaSuccess ? SPH_OK : cuda_fail(c, e, "advect");
}

// The update prologue rides on the build's scatter when ports exist; the next
// sph_buffer_update skips it if the runs and cell tables are still those.
static UpdPro pro_plan(sph_ctx *c, const int32_t *cell_start, const int32_t *cell_end)
{
    UpdPro up;
    const int n_runs = (int)(c->runs.size() / 3);
    c->pro_ready = n_runs > 0;
    if (n_runs > 0) {
        up.n_runs = n_runs;
        up.max_ports = c->pt.max_ports;
        c->pro_ver = c->runs_ver;
        c->pro_cs = cell_start;
        c->pro_ce = cell_end;
    }
    return up;
}

static sph_status cll_build(sph_ctx *c, const sph_particles *in, sph_particles *out, int32_t *cell_start,
                            int32_t *cell_end, int32_t *perm, float dt, bool advect, void *stream)
{
    SPH_NVTX("sph_cll_build");
    if (!c) return SPH_ERR_ARG;
    if (c->update_pending) return fail(c, SPH_ERR_STATE, "cll_build: the last buffer update was not compacted");
    sph_status st = check_particles(c, in);
    if (st == SPH_OK) st = check_particles(c, out);
    if (st != SPH_OK) return st;
    if (!cell_start || !cell_end) return fail(c, SPH_ERR_ARG, "NULL cell table");
    if (in->x == out->x || in->id == out->id || in->label == out->label)
        return fail(c, SPH_ERR_ARG, "cll_build needs distinct input and output arrays");
    if ((reinterpret_cast<size_t>(cell_start) | reinterpret_cast<size_t>(cell_end)) % 16)
        return fail(c, SPH_ERR_ARG, "cell tables must be 16-byte aligned");
    const CllCarry cc = carry_plan(c, in, advect, dt, false);
    const UpdPro up = pro_plan(c, cell_start, cell_end);
    cudaError_t e = launch_cll(part_dev(in), part_dev(out), c->gd, c->W, cell_start, cell_end, perm, dt, advect, cc,
                               up, static_cast<cudaStream_t>(stream), &c->L);
    if (e != cudaSuccess) return cuda_fail(c, e, "cll_build");
    carry_after_build(c, cc, out);
    return SPH_OK;
}

sph_status sph_cll_build(sph_ctx *c, const sph_particles *in, sph_particles *out, int32_t *cell_start,
                         int32_t *cell_end, int32_t *perm, void *stream)
{
    return cll_build(c, in, out, cell_start, cell_end, perm, 0.0f, false, stream);
}

sph_status sph_advect_cll_build(sph_ctx *c, sph_particles *in, sph_particles *out, float dt, int32_t *cell_start,
                                int32_t *cell_end, int32_t *perm, void *stream)
{
    return cll_build(c, in, out, cell_start, cell_end, perm, dt, true, stream);
}

sph_status sph_cll_invalidate(sph_ctx *c)
{
    if (!c) return SPH_ERR_ARG;
    carry_drop(c);
    return SPH_OK;
}

sph_status sph_cll_key(sph_ctx *c, sph_particles *in, float dt, int32_t advect, float *send_lo, float *send_hi,
                       void *stream)
{
    SPH_NVTX("sph_cll_key");
    if (!c) return SPH_ERR_ARG;
    if (c->update_pending) return fail(c, SPH_ERR_STATE, "cll_key: the last buffer update was not compacted");
    sph_status st = check_particles(c, in);
    if (st != SPH_OK) return st;
    if ((send_lo == nullptr) != (send_hi == nullptr)) return fail(c, SPH_ERR_ARG, "give both send buffers or none");
    if (!send_lo && c->comm && c->comm->nranks > 1) {     // the library's own migration buffers
        send_lo = c->W.mig[0];
        send_hi = c->W.mig[1];
    }
    c->key_advect = advect != 0;
    c->key_dt = dt;
    c->key_cc = carry_plan(c, in, advect != 0, dt, send_lo != nullptr);
    cudaError_t e = launch_cll_key(part_dev(in), c->gd, c->W, dt, advect != 0, send_lo, send_hi, c->max_migrate,
                                   sph_migrate_record_floats(c), c->key_cc, static_cast<cudaStream_t>(stream),
                                   &c->L);
    if (e == cudaSuccess && c->key_cc.clear) c->carry_next = false;   // cleared: nothing carried any more
    return e == cudaSuccess ? SPH_OK : cuda_fail(c, e, "cll_key");
}

sph_status sph_cll_finish(sph_ctx *c, sph_particles *in, sph_particles *out, const float *recv_lo,
                          const float *recv_hi, int32_t *cell_start, int32_t *cell_end, int32_t *perm, void *stream)
{
    SPH_NVTX("sph_cll_finish");
    if (!c) return SPH_ERR_ARG;
    if (c->update_pending) return fail(c, SPH_ERR_STATE, "cll_finish: the last buffer update was not compacted");
    sph_status st = check_particles(c, in);
    if (st == SPH_OK) st = check_particles(c, out);
    if (st != SPH_OK) return st;
    if (!cell_start || !cell_end) return fail(c, SPH_ERR_ARG, "NULL cell table");
    if (in->x == out->x || in->id == out->id || in->label == out->label)
        return fail(c, SPH_ERR_ARG, "cll_finish needs distinct input and output arrays");
    if ((reinterpret_cast<size_t>(cell_start) | reinterpret_cast<size_t>(cell_end)) % 16)
        return fail(c, SPH_ERR_ARG, "cell tables must be 16-byte aligned");
    if (!recv_lo && !recv_hi && c->comm && c->comm->nranks > 1) {   // the library's own migration buffers
        if (c->comm->rank > 0) recv_lo = c->W.mig[2];
        if (c->comm->rank < c->comm->nranks - 1) recv_hi = c->W.mig[3];
    }
    const UpdPro up = pro_plan(c, cell_start, cell_end);
    cudaError_t e = launch_cll_finish(part_dev(in), part_dev(out), c->gd, c->W, recv_lo, recv_hi, c->max_migrate,
                                      sph_migrate_record_floats(c), cell_start, cell_end, perm, c->key_advect,
                                      c->key_dt, c->key_cc, up, static_cast<cudaStream_t>(stream), &c->L);
    if (e != cudaSuccess) return cuda_fail(c, e, "cll_finish");
    carry_after_build(c, c->key_cc, out);
    return SPH_OK;
}

sph_status sph_buffer_update(sph_ctx *c, sph_particles *p, const int32_t *cell_start, const int32_t *cell_end,
                             int32_t *port_counts, void *stream)
{
    SPH_NVTX("sph_buffer_update");
    if (!c) return SPH_ERR_ARG;
    sph_status st = check_particles(c, p);
    if (st != SPH_OK) return st;
    if (!cell_start || !cell_end || !port_counts) return fail(c, SPH_ERR_ARG, "NULL argument");
    if (c->update_pending)
        return fail(c, SPH_ERR_STATE, "buffer_update: the previous update was not compacted");
    const int n_runs = (int)(c->runs.size() / 3);
    const bool pro_done = c->pro_ready && c->pro_ver == c->runs_ver && c->pro_cs == cell_start &&
                          c->pro_ce == cell_end;
    c->pro_ready = false;
    cudaError_t e = launch_update(part_dev(p), c->gd, c->pt, c->W, n_runs, cell_start, cell_end, port_counts,
                                  carry_on(c, p), c->carry_dt, pro_done, static_cast<cudaStream_t>(stream), &c->L);
    if (e != cudaSuccess) return cuda_fail(c, e, "buffer_update");
    c->update_pending = true;
    c->last_port_counts = port_counts;
    return SPH_OK;
}

static sph_status compact(sph_ctx *c, sph_particles *p, const int32_t *all_counts, int32_t nranks, int32_t rank,
                          int64_t *next_id_dev, int32_t *perm, bool defer, void *stream)
{
    SPH_NVTX("sph_compact");
    if (!c) return SPH_ERR_ARG;
    sph_status st = check_particles(c, p);
    if (st != SPH_OK) return st;
    if (!all_counts || !next_id_dev || nranks <= 0 || rank < 0 || rank >= nranks)
        return fail(c, SPH_ERR_ARG, "bad count matrix / rank");
    if (!c->update_pending) return fail(c, SPH_ERR_STATE, "compact: no buffer update to compact");
    int carry = carry_on(c, p);
    if (carry == 2 && !defer) {
        // an in-place compaction renumbers particles behind the leaver list: the
        // next build runs its own key pass instead
        carry_drop(c);
        carry = 0;
    }
    cudaError_t e = launch_compact(part_dev(p), c->gd, c->pt, c->W, all_counts, nranks, rank,
                                   reinterpret_cast<long long *>(next_id_dev), perm, defer, carry, c->carry_dt,
                                   static_cast<cudaStream_t>(stream), &c->L);
    if (e != cudaSuccess) return cuda_fail(c, e, "compact");
    c->update_pending = false;
    return SPH_OK;
}

sph_status sph_compact(sph_ctx *c, sph_particles *p, const int32_t *all_counts, int32_t nranks, int32_t rank,
                       int64_t *next_id_dev, int32_t *perm, void *stream)
{
    return compact(c, p, all_counts, nranks, rank, next_id_dev, perm, false, stream);
}

sph_status sph_compact_deferred(sph_ctx *c, sph_particles *p, const int32_t *all_counts, int32_t nranks,
                                int32_t rank, int64_t *next_id_dev, void *stream)
{
    return compact(c, p, all_counts, nranks, rank, next_id_dev, nullptr, true, stream);
}

int32_t sph_migrate_record_floats(const sph_ctx *c) { return c ? 2 * c->grid.dim + c->n_extra + 3 : 0; }

sph_status sph_migrate_pack(sph_ctx *c, sph_particles *p, float *send_lo, float *send_hi, void *stream)
{
    SPH_NVTX("sph_migrate_pack");
    if (!c) return SPH_ERR_ARG;
    sph_status st = check_particles(c, p);
    if (st != SPH_OK) return st;
    if (!send_lo || !send_hi) return fail(c, SPH_ERR_ARG, "NULL send buffer");
    if (c->update_pending) return fail(c, SPH_ERR_STATE, "migrate_pack: the last buffer update was not compacted");
    carry_drop(c);
    cudaError_t e = launch_migrate_pack(part_dev(p), c->gd, c->W, send_lo, send_hi, c->max_migrate,
                                        sph_migrate_record_floats(c), static_cast<cudaStream_t>(stream),
                                        &c->L);
    return e == cudaSuccess ? SPH_OK : cuda_fail(c, e, "migrate_pack");
}

sph_status sph_migrate_unpack(sph_ctx *c, sph_particles *p, const float *recv, void *stream)
{
    SPH_NVTX("sph_migrate_unpack");
    if (!c) return SPH_ERR_ARG;
    sph_status st = check_particles(c, p);
    if (st != SPH_OK) return st;
    if (!recv) return fail(c, SPH_ERR_ARG, "NULL receive buffer");
    carry_drop(c);
    cudaError_t e = launch_migrate_unpack(part_dev(p), c->gd, c->W, recv, c->max_migrate,
                                          sph_migrate_record_floats(c), static_cast<cudaStream_t>(stream),
                                          &c->L);
    return e == cudaSuccess ? SPH_OK : cuda_fail(c, e, "migrate_unpack");
}

sph_status sph_status_sync(sph_ctx *c, const sph_particles *p, void *stream, sph_stats *out)
{
    if (!c || !out) return SPH_ERR_ARG;
    if (!c->ws) return fail(c, SPH_ERR_STATE, "no workspace set");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Counters h{};
    long long n = -1;
    cudaError_t e = cudaMemcpyAsync(&h, c->W.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && p && p->n_dev) e = cudaMemcpyAsync(&n, p->n_dev, sizeof(n), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(c, e, "status_sync");
    out->n = n;
    out->candidates = h.n_cand;
    out->created = h.n_stage;
    out->deleted = h.n_del;
    out->checked_total = h.checked;
    out->out_of_grid = h.out_of_grid;
    out->motion_errors = h.motion;
    out->migrated_out = h.migrated;
    out->first_deleted = h.i_first;
    out->status_bits = h.status;
    out->n_ports = c->pt.n;
    if (h.status & (kStCapacity | kStStaging | kStMigrate))
        return fail(c, SPH_ERR_CAPACITY, "device capacity / staging / migration buffer overflow");
    if (h.status & kStMotion)
        return fail(c, SPH_ERR_MOTION, "a buffer particle was found outside its decision region P_k");
    if (c->comm) {
        std::string m;
        if (comm_async_error(c->comm, &m) != 0) return fail(c, SPH_ERR_NCCL, m);
    }
    return SPH_OK;
}

// =============================================================================== multi-GPU (§8(e))

sph_status sph_comm_unique_id(void *id_out)
{
    if (!id_out) return SPH_ERR_ARG;
    std::string m;
    return comm_unique_id(id_out, &m) == 0 ? SPH_OK : SPH_ERR_NCCL;
}

static sph_status comm_precheck(sph_ctx *c, int32_t nranks, int32_t rank)
{
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(c, SPH_ERR_ARG, "comm: bad rank / nranks");
    if (c->comm) return fail(c, SPH_ERR_STATE, "comm: already initialised");
    if (!c->ws) return fail(c, SPH_ERR_STATE, "comm: set the workspace first (it holds the migration buffers)");
    if (nranks > 1 && c->max_migrate <= 0) return fail(c, SPH_ERR_ARG, "comm: nranks > 1 needs max_migrate > 0");
    return SPH_OK;
}

sph_status sph_comm_init(sph_ctx *c, const void *nccl_unique_id, int32_t nranks, int32_t rank)
{
    if (!c || !nccl_unique_id) return SPH_ERR_ARG;
    sph_status st = comm_precheck(c, nranks, rank);
    if (st != SPH_OK) return st;
    std::string m;
    Comm *cm = comm_nccl(nccl_unique_id, nranks, rank, &m);
    if (!cm) return fail(c, SPH_ERR_NCCL, m);
    c->comm = cm;
    return SPH_OK;
}

sph_status sph_comm_init_loopback(sph_ctx *const *ctxs, int32_t nranks)
{
    if (!ctxs || nranks < 1) return SPH_ERR_ARG;
    for (int r = 0; r < nranks; ++r) {
        if (!ctxs[r]) return SPH_ERR_ARG;
        sph_status st = comm_precheck(ctxs[r], nranks, r);
        if (st != SPH_OK) return st;
        if (ctxs[r]->max_migrate != ctxs[0]->max_migrate || ctxs[r]->n_extra != ctxs[0]->n_extra ||
            ctxs[r]->max_ports != ctxs[0]->max_ports || ctxs[r]->grid.dim != ctxs[0]->grid.dim)
            return fail(ctxs[r], SPH_ERR_ARG, "loopback: members differ in max_migrate / n_extra / max_ports / dim");
    }
    LoopGroup *g = new LoopGroup();
    g->m.assign(ctxs, ctxs + nranks);
    g->live = nranks;
    for (int r = 0; r < nranks; ++r) {
        Comm *cm = new Comm();
        cm->kind = Comm::LOOPBACK;
        cm->nranks = nranks;
        cm->rank = r;
        cm->loop = g;
        ctxs[r]->comm = cm;
    }
    return SPH_OK;
}

sph_status sph_allgather_counts(sph_ctx *c, const int32_t *port_counts, int32_t *all_counts, void *stream)
{
    SPH_NVTX("sph_allgather_counts");
    if (!c || !port_counts || !all_counts) return SPH_ERR_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t cnt = 2 * (size_t)c->max_ports;
    if (!c->comm || (c->comm->nranks == 1 && c->comm->kind == Comm::LOOPBACK)) {
        cudaError_t e = cudaMemcpyAsync(all_counts, port_counts, cnt * sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
        return e == cudaSuccess ? SPH_OK : cuda_fail(c, e, "allgather_counts");
    }
    std::vector<const int32_t *> loop;
    if (c->comm->kind == Comm::LOOPBACK) {
        LoopGroup *g = static_cast<LoopGroup *>(c->comm->loop);
        for (sph_ctx *m : g->m) loop.push_back(m ? m->last_port_counts : nullptr);
    }
    std::string m;
    if (comm_allgather_i32(c->comm, port_counts, all_counts, cnt, s, loop, &m) != 0)
        return fail(c, SPH_ERR_NCCL, "allgather_counts: " + m);
    return SPH_OK;
}

sph_status sph_migrate_exchange(sph_ctx *c, void *stream)
{
    SPH_NVTX("sph_migrate_exchange");
    if (!c) return SPH_ERR_ARG;
    if (!c->comm) return fail(c, SPH_ERR_STATE, "migrate_exchange: no communicator (sph_comm_init)");
    if (c->comm->nranks == 1) return SPH_OK;
    const size_t cnt = 4 + (size_t)c->max_migrate * (size_t)sph_migrate_record_floats(c);
    const float *lo_peer = nullptr, *hi_peer = nullptr;
    if (c->comm->kind == Comm::LOOPBACK) {
        LoopGroup *g = static_cast<LoopGroup *>(c->comm->loop);
        const int r = c->comm->rank;
        if ((r > 0 && !g->m[r - 1]) || (r < c->comm->nranks - 1 && !g->m[r + 1]))
            return fail(c, SPH_ERR_STATE, "migrate_exchange: a loopback neighbour was destroyed");
        if (r > 0) lo_peer = g->m[r - 1]->W.mig[1];
        if (r < c->comm->nranks - 1) hi_peer = g->m[r + 1]->W.mig[0];
    }
    std::string m;
    if (comm_neighbour_exchange(c->comm, c->W.mig[0], c->W.mig[1], c->W.mig[2], c->W.mig[3], cnt,
                                static_cast<cudaStream_t>(stream), lo_peer, hi_peer, &m) != 0)
        return fail(c, SPH_ERR_NCCL, "migrate_exchange: " + m);
    return SPH_OK;
}

sph_status sph_migrate(sph_ctx *c, sph_particles *p, void *stream)
{
    if (!c) return SPH_ERR_ARG;
    if (!c->comm) return fail(c, SPH_ERR_STATE, "migrate: no communicator (sph_comm_init)");
    if (c->comm->nranks == 1) return SPH_OK;
    if (c->comm->kind == Comm::LOOPBACK)
        return fail(c, SPH_ERR_STATE, "migrate: a loopback group needs the split calls "
                                      "(sph_migrate_pack, sph_migrate_exchange, sph_migrate_unpack), phase by phase");
    sph_status st = sph_migrate_pack(c, p, c->W.mig[0], c->W.mig[1], stream);
    if (st == SPH_OK) st = sph_migrate_exchange(c, stream);
    if (st == SPH_OK && c->comm->rank > 0) st = sph_migrate_unpack(c, p, c->W.mig[2], stream);
    if (st == SPH_OK && c->comm->rank < c->comm->nranks - 1) st = sph_migrate_unpack(c, p, c->W.mig[3], stream);
    return st;
}

sph_status sph_migrate_cll_build(sph_ctx *c, sph_particles *in, sph_particles *out, float dt, int32_t advect,
                                 int32_t *cell_start, int32_t *cell_end, int32_t *perm_or_null, void *stream)
{
    if (!c) return SPH_ERR_ARG;
    if (!c->comm) return fail(c, SPH_ERR_STATE, "migrate_cll_build: no communicator (sph_comm_init)");
    if (c->comm->kind == Comm::LOOPBACK && c->comm->nranks > 1)
        return fail(c, SPH_ERR_STATE, "migrate_cll_build: a loopback group needs the split calls "
                                      "(sph_cll_key, sph_migrate_exchange, sph_cll_finish), phase by phase");
    sph_status st = sph_cll_key(c, in, dt, advect, nullptr, nullptr, stream);
    if (st == SPH_OK) st = sph_migrate_exchange(c, stream);
    if (st == SPH_OK) st = sph_cll_finish(c, in, out, nullptr, nullptr, cell_start, cell_end, perm_or_null, stream);
    return st;
}

int64_t sph_launch_count(const sph_ctx *c) { return c ? c->L.count : 0; }

static const char *kKernelNames[KID_COUNT] = {
    "advect", "register", "cll_key", "cell_scan", "cll_scatter", "cll_gather", "upd_prologue",
    "upd_main", "compact", "compact_append", "mig_pack", "mig_unpack", "compact_count", "cll_rank",
    "port_move", "port_enum", "drivers"};
static_assert(KID_COUNT == SPH_NKERNELS, "sphbuf.h SPH_NKERNELS must match the kernel ids");

const char *sph_kernel_name(int32_t i) { return (i >= 0 && i < KID_COUNT) ? kKernelNames[i] : ""; }

sph_status sph_profile(sph_ctx *c, int32_t enable)
{
    if (!c) return SPH_ERR_ARG;
    cudaError_t e = c->L.flush();
    if (e != cudaSuccess) return cuda_fail(c, e, "profile");
    for (int k = 0; k < KID_COUNT; ++k) {
        c->L.ms[k] = 0.0;
        c->L.n[k] = 0;
    }
    c->L.prof = enable != 0;
    return SPH_OK;
}

sph_status sph_profile_read(sph_ctx *c, double *ms, int64_t *count)
{
    if (!c || !ms || !count) return SPH_ERR_ARG;
    cudaError_t e = c->L.flush();
    if (e != cudaSuccess) return cuda_fail(c, e, "profile_read");
    for (int k = 0; k < KID_COUNT; ++k) {
        ms[k] = c->L.ms[k];
        count[k] = c->L.n[k];
    }
    return SPH_OK;
}

// Rodrigues with reading R1 (Q = R^T) and a roll psi about u.
sph_status sph_frame_from_axis(const double u_in[3], double psi, float Q_out[9])
{
    if (!u_in || !Q_out) return SPH_ERR_ARG;
    const double nu = std::sqrt(u_in[0] * u_in[0] + u_in[1] * u_in[1] + u_in[2] * u_in[2]);
    if (!(nu > 0.0)) return SPH_ERR_ARG;
    const double u[3] = {u_in[0] / nu, u_in[1] / nu, u_in[2] / nu};
    double R[3][3];
    // n = e_x x u (Eq. rotation_axis); |e_x x u| = sin(theta)
    const double w[3] = {0.0, -u[2], u[1]};
    const double sn = std::sqrt(w[1] * w[1] + w[2] * w[2]);
    if (sn < 1e-12) {
        const double sg = u[0] > 0 ? 1.0 : -1.0;
        double I[3][3] = {{sg, 0, 0}, {0, sg, 0}, {0, 0, 1}};
        std::memcpy(R, I, sizeof(R));
    } else {
        const double n[3] = {w[0] / sn, w[1] / sn, w[2] / sn};
        const double th = std::acos(std::max(-1.0, std::min(1.0, u[0])));
        const double S[3][3] = {{0, -n[2], n[1]}, {n[2], 0, -n[0]}, {-n[1], n[0], 0}};
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                double s2 = 0.0;
                for (int l = 0; l < 3; ++l) s2 += S[i][l] * S[l][j];
                R[i][j] = (i == j ? 1.0 : 0.0) + S[i][j] * std::sin(th) + s2 * (1.0 - std::cos(th));
            }
    }
    // Q0 = R^T, then roll about the local X' axis: Q = Rx(psi) Q0
    double Q0[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) Q0[i][j] = R[j][i];
    const double cp = std::cos(psi), sp = std::sin(psi);
    for (int j = 0; j < 3; ++j) {
        Q_out[0 + j] = (float)Q0[0][j];
        Q_out[3 + j] = (float)(cp * Q0[1][j] + sp * Q0[2][j]);
        Q_out[6 + j] = (float)(-sp * Q0[1][j] + cp * Q0[2][j]);
    }
    return SPH_OK;
}

}  // extern "C"
