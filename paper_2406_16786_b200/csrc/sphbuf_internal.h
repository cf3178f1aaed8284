// sphbuf_internal.h — private types shared by the host side (sphbuf_host.cpp) and
// the sm_100a kernels (sphbuf_kernels.cu).  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "sphbuf.h"

namespace sphbuf {

// ---------------------------------------------------------------- tiling
constexpr int kThreads = 256;            // block size of the O(N) kernels
constexpr int kCellItems = 32;           // cells per thread in the cell scan (multiple of 32) ...
constexpr int kCellTile = kThreads * kCellItems;
constexpr int kCellItemsBig = 128;       // ... or this many above kScanBigCells cells (one wave of tiles)
constexpr int kCellTileBig = kThreads * kCellItemsBig;
constexpr long long kScanBigCells = 4LL << 20;
constexpr int kDelList = 8192;           // deletions listed for the in-place compaction's offsets
constexpr int kUpdItems = 2;             // candidates per thread in the update
constexpr int kUpdTile = kThreads * kUpdItems;
constexpr int kCmpItems = 4;             // particles per thread in the compaction
constexpr int kCmpTile = kThreads * kCmpItems;
constexpr int kCntTile = 8192;           // labels per tile in the compaction count
constexpr int kGatherItems = 4;          // output slots per thread in the gather
constexpr int kGatherTile = kThreads * kGatherItems;
constexpr int64_t kMaxRuns = 1 << 20;    // port runs per context

// ---------------------------------------------------------------- status bits
constexpr int kStCapacity = 1;
constexpr int kStStaging = 2;
constexpr int kStMotion = 4;
constexpr int kStMigrate = 8;

// Port parameters as the kernels see them (passed by value in the kernel
// parameter space, i.e. the constant bank: uniform broadcast reads).
struct PortDev {
    float o[3];      // origin O'
    float Q[9];      // rows = local axes
    float he[3];     // half extents (a/2, b/2, c/2)
    float heP[3];    // fl(he + cs): decision region P_k (reading R4)
    float s[3];      // recycle shift fl(a * u)
    int kind;
    int bc;          // sph_bc_kind
    int profile;     // sph_profile_kind
    int rho_col;     // extra column of the density (-1 none)
    float rho_b;     // fl32(rho0 + p_b / c0^2), formed in f64
    float u0;        // velocity BC speed scale
    float R;         // profile radius
    float R2;        // fl(R * R)
    int rho_dev;     // pressure BC driven by a Windkessel: rho_b read from Workspace::drv_rho[k]
};

// Pose of a movable port for the device cell enumeration (sphbuf_motion.cu):
// f64 decision region (centre, unit axes, half sizes he + cs + 1e-3 cs) and the
// cell window covering its bounding sphere: columns [cx0, cx0 + ncx) x
// [cy0, cy0 + ncy) (3-D; 2-D: columns along y, ncy = 1), fast-axis cells [f0, f1].
struct PortEnum {
    double o[3];
    double ax[3][3];
    double H[3];
    int cx0, cy0, ncx, ncy, f0, f1;
    int k;
};

// Device state of a Windkessel driver (sph_drivers_step).
struct DriverDev {
    double P;        // boundary pressure
    double Q;        // flow rate of the last step
    double Qprev;    // flow rate of the step before
    int first;       // no step taken yet (Qprev := Q)
    int pad;
};

// One Windkessel port for the driver kernel (by value).
struct DriverEntry {
    int k, run0, nrun, pad;
    float u[3];      // the port's axis (row 0 of Q)
    float pad2;
    double sign;     // +1 outlet, -1 inlet / bidirectional (flow out of the domain is positive)
    double scale;    // V / a
    double Rp, C, Rd, rho0, c0sq, dt;
};

struct DriverLaunch {
    int n;
    DriverEntry e[SPH_MAX_PORTS];
};

struct PortTable {
    int n;
    int max_ports;
    PortDev p[SPH_MAX_PORTS];
};

struct GridDev {
    int dim;
    float lo[3];
    float inv_cs;     // fl32(1/cs) formed in f64
    int ncell[3];
    int cx_begin, cx_end;
    int ny, nz;
    long long ncells;  // cells of the slab
};

struct PartDev {
    float *x, *y, *z, *vx, *vy, *vz;
    float *extra[SPH_MAX_EXTRA];
    int n_extra;
    long long *id;
    int *label;
    long long *n;
    long long cap;
};

struct Counters {
    unsigned int epoch_cll, epoch_upd, epoch_cmp, epoch_pad;
    int ticket_cll, ticket_upd, ticket_cmp, ticket_cmp2;
    long long n_in;        // cll: live+tombstone input length
    long long n_cand;      // update: candidates this update
    long long n_stage;     // update: created this update (may exceed staging capacity -> error)
    long long n_del;       // update: deleted this update
    long long i_first;     // update: lowest deleted index
    long long out_of_grid; // cumulative
    long long checked;     // cumulative candidates
    long long motion;      // cumulative
    long long cmp_n;       // compaction: N before
    long long cmp_next_id; // compaction: next_id before
    long long migrated;    // cumulative packed for neighbour slabs
    long long mig_base;    // cll: local count before the received particles are appended
    long long n_leave;     // key carry-over: leavers listed for the next build's migration
    long long n_stage_raw; // update: staging slots handed out (unordered, one atomic per tile)
    long long n_dlist;     // update: deleted positions listed (for the in-place compaction's offsets)
    int status;            // sticky bits
    int ticket_runs;       // update prologue: tile tickets (reset by its last block)
    int done_cll;          // cell scan: finished blocks
    int done_app;          // compaction append: finished blocks
    int done_runs;         // update prologue: finished blocks
    int done_upd;          // update: finished blocks (the last one scans the tile counts)
    int ticket_gather;     // cell-list gather: tile tickets (reset by the scatter of the same build)
    int ticket_scatter;    // scatter (DYN variant): warp-chunk tickets (reset by its last block)
    int done_scatter;      // scatter (DYN variant): finished blocks
};

struct Workspace {
    Counters *ctr;
    int *cell_count;                 // [ncells]: build histogram
    int *cursor;                     // [ncells]: scatter cursors
    unsigned long long *tile_cells;  // [cell tiles]
    int *key;                        // [capacity]
    int *leave;                      // [max_leave]: indices of listed leavers (key carry-over + migration)
    int *src;                        // [capacity]: source index of each sorted slot
    unsigned *tile_cr;               // [upd tiles]: CREATEs of each update tile
    unsigned *tile_pre;              // [upd tiles]: their exclusive prefix (canonical staging order)
    unsigned long long *tile_runs;   // [kMaxRuns / 256 + 1]: update prologue look-back
    unsigned long long *tile_cmp;    // [cmp count tiles]
    unsigned *sub_off;               // [cmp sub-tiles]: tombstones before each sub-tile
    unsigned *rd;                    // [cmp sub-tiles]: "read done" epoch flags
    int *runs;                       // [kMaxRuns * 3]: c0, c1, port
    DriverDev *drv;                  // [SPH_MAX_PORTS]: Windkessel state
    float *drv_rho;                  // [SPH_MAX_PORTS]: recycled density of driven pressure BCs
    int *port_cnt;                   // [2 SPH_MAX_PORTS]: this update's created / deleted per port
    int *del_list;                   // [kDelList]: this update's deleted positions (K6)
    long long *run_off;              // [kMaxRuns + 1]
    int *run_base;                   // [kMaxRuns]: first particle index of each run
    int *tile_run;                   // [upd tiles]: run holding the first candidate of each K6 tile
    float *sx, *sy, *sz, *svx, *svy, *svz;
    float *sextra[SPH_MAX_EXTRA];
    long long *sid;                  // source id of each staged particle (diagnostic)
    int *sport;                      // port of each staged particle
    int *stile, *sexcl;              // update tile of each staged particle and its rank inside the tile:
                                     // canonical slot = tile_pre[stile] + sexcl
    float *mig[4];                   // library-owned migration buffers: send lo, send hi, recv lo, recv hi
                                     // (4 header words + max_migrate records each; max_migrate > 0)
    long long max_new;
    long long max_leave;
    long long upd_tiles;
    long long cmp_tiles;
};

// ---------------------------------------------------------------- communicator (sphbuf_comm.cpp)
// The library's communicator of the x-slab decomposition: NCCL (loaded with
// dlopen) or an in-process loopback group (contexts on one device; device copies).
struct Comm {
    enum Kind { NCCL, LOOPBACK } kind = NCCL;
    void *nccl = nullptr;     // ncclComm_t
    int nranks = 1, rank = 0;
    void *loop = nullptr;     // LOOPBACK: the group (owned by sphbuf_host.cpp)
};
int comm_unique_id(void *out, std::string *err);
Comm *comm_nccl(const void *id, int nranks, int rank, std::string *err);
void comm_destroy(Comm *c);
// recv [nranks][count] <- every rank's send [count]; loop_send: the members' send buffers (LOOPBACK)
int comm_allgather_i32(Comm *c, const int32_t *send, int32_t *recv, size_t count, cudaStream_t s,
                       const std::vector<const int32_t *> &loop_send, std::string *err);
// send_lo -> rank-1 (its recv_hi), send_hi -> rank+1 (its recv_lo); count floats each way;
// loop_lo_peer / loop_hi_peer: rank-1's send_hi and rank+1's send_lo (LOOPBACK)
int comm_neighbour_exchange(Comm *c, const float *send_lo, const float *send_hi, float *recv_lo, float *recv_hi,
                            size_t count, cudaStream_t s, const float *loop_lo_peer, const float *loop_hi_peer,
                            std::string *err);
int comm_async_error(Comm *c, std::string *err);

// ---------------------------------------------------------------- launch bookkeeping
enum KernelId {
    KID_ADVECT, KID_REGISTER, KID_CLL_KEY, KID_CELL_SCAN, KID_CLL_SCATTER, KID_CLL_GATHER, KID_UPD_PROLOGUE,
    KID_UPD_MAIN, KID_COMPACT, KID_COMPACT_APPEND, KID_MIG_PACK, KID_MIG_UNPACK, KID_COMPACT_COUNT, KID_CLL_RANK,
    KID_PORT_MOVE, KID_PORT_ENUM, KID_DRIVERS, KID_COUNT
};

// Counts launches; when profiling is on, brackets every launch with a pair of
// CUDA events on the launching stream (sph_profile / sph_profile_read).
struct Launch {
    int64_t count = 0;
    bool prof = false;
    std::vector<cudaEvent_t> pool;
    std::vector<int> kid;
    size_t used = 0;
    double ms[KID_COUNT] = {};
    int64_t n[KID_COUNT] = {};
    void before(cudaStream_t s);
    void after(cudaStream_t s, int k);
    cudaError_t flush();
    ~Launch();
};

// ---------------------------------------------------------------- launchers (sphbuf_kernels.cu)
cudaError_t launch_advect(const PartDev &p, int dim, float dt, cudaStream_t s, Launch *L);
cudaError_t launch_register(const PartDev &p, const GridDev &g, const PortTable &pt, int k, long long *members,
                            cudaStream_t s, Launch *L);
// Key carry-over of the cell-list build (sphbuf_cll.cu): `use` — this build's keys
// and histogram were made by the previous build's gather (skip the key pass);
// `clear` — the previous gather left a histogram this build does not use (zero
// it first); `make` — this build's gather prepares the next build's keys for
// advection by `dt`.
struct CllCarry {
    bool use = false, clear = false, make = false;
    bool mig = false;   // with slab migration (leaver list)
    float dt = 0.f;
};
// The update prologue (K5) run by extra blocks of the build's scatter: n_runs > 0
// enables it (sph_buffer_update then launches K6 alone).
struct UpdPro {
    int n_runs = 0;
    int max_ports = 0;
};
cudaError_t launch_cll(const PartDev &in, const PartDev &out, const GridDev &g, const Workspace &ws,
                       int *cell_start, int *cell_end, int *perm, float dt, bool advect, const CllCarry &cc,
                       const UpdPro &up, cudaStream_t s, Launch *L);

// advect / dt: the advection of the key pass (launch_cll_key) that this build
// finishes; the gather applies it to the slab's own particles as it moves them.
cudaError_t launch_cll_key(const PartDev &in, const GridDev &g, const Workspace &ws, float dt, bool advect,
                           float *send_lo, float *send_hi, long long maxm, int rec, const CllCarry &cc,
                           cudaStream_t s, Launch *L);
cudaError_t launch_cll_finish(const PartDev &in, const PartDev &out, const GridDev &g, const Workspace &ws,
                              const float *recv_lo, const float *recv_hi, long long maxm, int rec, int *cell_start,
                              int *cell_end, int *perm, bool advect, float dt, const CllCarry &cc,
                              const UpdPro &up, cudaStream_t s, Launch *L);
cudaError_t launch_update(const PartDev &p, const GridDev &g, const PortTable &pt, const Workspace &ws, int n_runs,
                          const int *cell_start, const int *cell_end, int *port_counts, int carry, float cdt,
                          bool prologue_done, cudaStream_t s, Launch *L);
cudaError_t launch_compact(const PartDev &p, const GridDev &g, const PortTable &pt, const Workspace &ws,
                           const int *all_counts, int nranks, int rank, long long *next_id, int *perm, bool defer,
                           int carry, float cdt, cudaStream_t s, Launch *L);
cudaError_t launch_migrate_pack(const PartDev &p, const GridDev &g, const Workspace &ws, float *lo, float *hi,
                                long long max_migrate, int rec, cudaStream_t s, Launch *L);
cudaError_t launch_migrate_unpack(const PartDev &p, const GridDev &g, const Workspace &ws, const float *buf,
                                  long long max_migrate, int rec, cudaStream_t s, Launch *L);
cudaError_t launch_port_move(const PartDev &p, const GridDev &g, const PortDev &P0, const PortDev &P1,
                             const int *runs, int nrun, const int *cell_start, const int *cell_end, int k,
                             long long *moved, const Workspace &ws, int carry, float cdt, cudaStream_t s, Launch *L);
cudaError_t launch_port_enum(const GridDev &g, const PortEnum &P, float cs, int *runs, int cap, cudaStream_t s,
                             Launch *L);
cudaError_t launch_drivers(const PartDev &p, int dim, const Workspace &ws, const DriverLaunch &D,
                           const int *cell_start, const int *cell_end, cudaStream_t s, Launch *L);
int sm_count();

}  // namespace sphbuf
