/*
 * sphbuf.h — C ABI of the B200-native in/outlet buffer update for SPH
 * (Zhang, Fan, Ren, Qian & Hu, arXiv 2406.16786, §III "The rationale of
 * arbitrary-positioned buffer").  Citations "P:n" are PAPER.md lines.
 *
 * Scope: cell-linked-list build (a1), per-port cell
 * enumeration (a2), candidate transform + axial compare (a3), inflow generation
 * (a4, Alg. 1 / Alg. 3), outflow deletion (a5, Alg. 2 / Alg. 3), relabel (a6)
 * and ID assignment + stable compaction (a7), plus the slab-migration kernels of
 * the multi-GPU decomposition (§8(e)).
 *
 * Conventions
 *  - Every pointer inside sph_particles, every cell table, count array and the
 *    workspace is DEVICE memory owned by the caller (torch tensors).  The library
 *    owns only the host-side context.  Nothing is freed behind the caller's back.
 *  - Calls that take `stream` (a cudaStream_t passed as void*) only enqueue work
 *    on that stream and return; no call synchronises except sph_status_sync.
 *    Live counts stay device-resident (`n_dev`), so a whole update can be
 *    captured into a CUDA graph.
 *  - Host-side argument errors are returned immediately with no work enqueued.
 *    Device-side errors (capacity, staging overflow, excessive motion) are
 *    recorded in a sticky device status word and reported by the next
 *    sph_status_sync; after one the particle state is undefined.
 *  - Arithmetic that decides an integer (cell index, crossing, in-box) or mutates
 *    state (recycle, advection) is pinned: each op one binary32 round-to-nearest
 *    operation in the order documented in DESIGN.md §3, never contracted to FMA.
 *  - Layout: structure of arrays; cells linearised x-major
 *    ((cx - cx_begin) * ny + cy) * nz + cz  (nz = 1 in 2-D); the particle array
 *    after sph_cll_build is ordered by (cell, id).
 */
#ifndef SPHBUF_H
#define SPHBUF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPH_MAX_PORTS 64      /* ports per context (C5 at 8 GPUs uses 64) */
#define SPH_MAX_EXTRA 8       /* optional fp32 columns copied on duplication */

typedef struct sph_ctx sph_ctx;

typedef enum {
    SPH_OK = 0,
    SPH_ERR_ARG = -1,              /* bad argument (dim, extents, layers < 3, too many ports, NULL) */
    SPH_ERR_NOT_ORTHONORMAL = -2,  /* |Q Q^T - I|max > 1e-5 or det Q <= 0 (or 2-D Q not planar) */
    SPH_ERR_OVERLAP = -3,          /* decision region P_k intersects an existing port's P_j */
    SPH_ERR_OUT_OF_GRID = -4,      /* P_k not strictly inside the grid */
    SPH_ERR_CAPACITY = -5,         /* (device) N - D + C > capacity, or staging/migration buffer full */
    SPH_ERR_MOTION = -6,           /* (device) a buffer particle found outside its decision region P_k
                                      (it moved more than the one-cell margin in one step; reading R12) */
    SPH_ERR_CUDA = -7,             /* a CUDA runtime call failed (see sph_last_error) */
    SPH_ERR_NCCL = -8,             /* an NCCL call failed or NCCL could not be loaded (see sph_last_error);
                                      asynchronous NCCL errors are reported by sph_status_sync */
    SPH_ERR_STATE = -9             /* call order violated: no workspace; sph_buffer_update while the
                                      previous update is not compacted; sph_compact(_deferred) with
                                      no update to compact; a build or migration pack in between */
} sph_status;

/* Port kinds: unidirectional inlet (Alg. 1), unidirectional
 * outlet (Alg. 2), bidirectional (Alg. 3; X' points along the inflow). */
typedef enum { SPH_INLET = 0, SPH_OUTLET = 1, SPH_BIDIRECTIONAL = 2 } sph_kind;

/* Uniform cell grid (cell size >= 2h).  The owning rank's x-slab is
 * the cell range [cx_begin, cx_end); a single-GPU run uses [0, ncell[0]). */
typedef struct {
    int32_t dim;          /* 2 or 3 */
    float lo[3];          /* lower corner (global coordinates) */
    float cs;             /* cell size */
    int32_t ncell[3];     /* global cell counts; ncell[2] = 1 in 2-D */
    int32_t cx_begin;
    int32_t cx_end;
} sph_grid;

/* Particle arrays (SoA, device).  z, vz = NULL in 2-D.  label: -1 = fluid,
 * k >= 0 = buffer particle of port k (the paper's exclusive integer per buffer,
 * P:416-417); values <= -2 are tombstones (deleted / migrated away) that the
 * next sph_cll_build drops.  n_dev: device int64 live count.  capacity: length
 * of every column. */
typedef struct {
    float *x, *y, *z;
    float *vx, *vy, *vz;
    float *extra[SPH_MAX_EXTRA];
    int32_t n_extra;
    int64_t *id;
    int32_t *label;
    int64_t *n_dev;
    int64_t capacity;
} sph_particles;

/* Cumulative / last-update statistics returned by sph_status_sync. */
typedef struct {
    int64_t n;              /* live particles (read from n_dev of the particles passed) */
    int64_t candidates;     /* candidates checked by the last sph_buffer_update */
    int64_t created;        /* created by the last update (this rank) */
    int64_t deleted;        /* deleted by the last update (this rank) */
    int64_t checked_total;  /* candidates checked since context creation */
    int64_t out_of_grid;    /* particles clamped into boundary cells, cumulative */
    int64_t motion_errors;  /* buffer particles found among their port's candidates but outside
                               P_k (reading R12), cumulative */
    int64_t migrated_out;   /* particles packed for neighbour slabs, cumulative */
    int64_t first_deleted;  /* lowest deleted index of the last update (INT64_MAX if none) */
    int32_t status_bits;    /* sticky device error bits: 1 capacity, 2 staging, 4 motion, 8 migration */
    int32_t n_ports;
} sph_stats;

/* Create a context for one rank.  h: smoothing length (checks cs >= 2h,
 * P:224-229).  capacity: particle array length.  max_ports <= SPH_MAX_PORTS.
 * max_new: staging capacity for particles created per update.  max_migrate:
 * per-direction migration buffer capacity (particles).  n_extra: extra columns.
 * Host only; no CUDA call.  *out receives the context. */
sph_status sph_ctx_create(const sph_grid *grid, float h, int64_t capacity, int32_t max_ports, int64_t max_new,
                          int64_t max_migrate, int32_t n_extra, sph_ctx **out);
void sph_ctx_destroy(sph_ctx *ctx);
const char *sph_last_error(const sph_ctx *ctx);

/* Device workspace: sph_workspace_bytes() bytes, 256-byte aligned, owned by the
 * caller.  sph_set_workspace zero-initialises it (synchronous, once). */
size_t sph_workspace_bytes(const sph_ctx *ctx);
sph_status sph_set_workspace(sph_ctx *ctx, void *d_ws, size_t bytes);

/* Host-only check of one port (what sph_buffer_register validates first):
 * origin O', frame Q (row-major, rows = local axes; X' = Q (x - o),
 * Eq. 2D_transformation P:252-269 / Eq. 3D_transformation),
 * half extents (a/2, b/2, c/2), kind, layers (a = layers * dp,
 * layers >= 3: P:226-229).  Returns SPH_OK or the error it would return. */
sph_status sph_port_check(const sph_ctx *ctx, const float origin[3], const float Q[9], const float half_extents[3],
                          int32_t kind, int32_t layers, float dp);

/* Register port k = number of ports registered so far (*port_id_out).
 * Enumerates on the host the cells of this slab intersecting the decision region
 * P_k = {|X'_r| < he_r + cs} (the paper's local cell-linked lists, "a little larger
 * than the size of outflow buffer, approximately one layer of cells"),
 * uploads them, and runs Alg. 1's one-time identification over all particles
 * ("Execute only once"): fluid particles in the box get label k; for
 * outlets and bidirectional ports this is also the initial relabel.
 * members_out_dev (device int64, may be NULL) receives the local member count. */
sph_status sph_buffer_register(sph_ctx *ctx, sph_particles *p, const float origin[3], const float Q[9],
                               const float half_extents[3], int32_t kind, int32_t layers, float dp,
                               int32_t *port_id_out, int64_t *members_out_dev, void *stream);

/* Boundary-condition state of a port's buffer particles (paper §IV, SURVEY
 * §8(f) rank 1), applied by sph_buffer_update to every particle that is a
 * buffer particle of the port at the end of the update (after generation,
 * recycling and relabel; duplicates keep the pre-BC state):
 *   SPH_BC_PRESSURE: v <- (v.u) u (Eq. velocity_correction); a
 *     particle recycled in this update gets density rho0 + p_b / c0^2 in extra
 *     column rho_column (Eq. postulate-density; -1: no density column);
 *   SPH_BC_VELOCITY: v <- Q^T (v_X', 0, 0) (Eqs. 2D/3D_velocity_transformation,
 *     P:605-636) with v_X' = u0 (plug), u0 (1 - (Y'/R)^2) (Eqs. 2D/3D_velocity_
 *     profile, literal) or u0 (1 - (Y'^2 + Z'^2)/R^2) (3-D pipe reading
 *     R23); recycled density and pressure unchanged.
 * Pinned arithmetic as everywhere. */
typedef enum { SPH_BC_NONE = 0, SPH_BC_PRESSURE = 1, SPH_BC_VELOCITY = 2 } sph_bc_kind;
typedef enum { SPH_PROFILE_PLUG = 0, SPH_PROFILE_PARABOLIC = 1, SPH_PROFILE_PARABOLIC_RADIAL = 2 } sph_profile_kind;
typedef struct {
    int32_t kind;          /* sph_bc_kind */
    float rho0, c0, p_b;   /* PRESSURE */
    int32_t rho_column;    /* PRESSURE: extra column index of the density, -1 none */
    int32_t profile;       /* VELOCITY: sph_profile_kind */
    float u0, radius;      /* VELOCITY: axial speed scale and R */
} sph_bc;

/* Set (or clear with kind SPH_BC_NONE) the boundary condition of registered
 * port port_id.  Host only; takes effect at the next sph_buffer_update. */
sph_status sph_port_set_bc(sph_ctx *ctx, int32_t port_id, const sph_bc *bc);

/* Time-dependent port drivers (aorta flow, §V.D).
 *   FOURIER    (port with a velocity BC): its speed scale follows
 *              u0(t) = a0 + sum_{n=1..8} a_n cos(n t omega) + sum_{n=1..8} b_n sin(n t omega)
 *              (Eq. Fourier_Series, Table I), evaluated in f64 on the host in that
 *              order and rounded once;
 *   WINDKESSEL (port with a pressure BC): its boundary pressure P(t) follows the
 *              3-element RCR model (1 + Rp/Rd) Q + C Rp dQ/dt = P/Rd + C dP/dt
 *              (Eq. windkessel, Table II; SI units), driven by the flow rate Q out
 *              of the port measured on the device every step: Q = V/a * sum over
 *              the port's buffer particles of v.n (n = +u for an outlet, -u for an
 *              inlet or bidirectional port; reading R26), summed exactly in 32.32
 *              fixed point; P advances by one explicit step (R27); the recycled
 *              density becomes fl32(rho0 + P / c0^2) of the port's pressure BC.
 * The driver state (P, Q) stays on the device (sph_driver_read synchronises). */
typedef enum { SPH_DRIVER_NONE = 0, SPH_DRIVER_FOURIER = 1, SPH_DRIVER_WINDKESSEL = 2 } sph_driver_kind;
typedef struct {
    int32_t kind;      /* sph_driver_kind */
    double a[9];       /* FOURIER: a0 .. a8 */
    double b[9];       /* FOURIER: b[1] .. b[8] (b[0] unused) */
    double omega;      /* FOURIER: rad/s */
    double Rp, C, Rd;  /* WINDKESSEL: Pa s/m^3, m^3/Pa, Pa s/m^3 */
    double P0;         /* WINDKESSEL: pressure at the first step, Pa */
    double volume;     /* WINDKESSEL: particle volume dp^dim for the flow rate */
} sph_driver;

/* Attach (or detach with kind NONE) a driver to port port_id; FOURIER needs a
 * velocity BC, WINDKESSEL a pressure BC on the port (sph_port_set_bc first).
 * Initialises the device state (P = P0); synchronous. */
sph_status sph_port_set_driver(sph_ctx *ctx, int32_t port_id, const sph_driver *d);

/* Advance every driver to time t (step dt): Fourier speeds set on the host,
 * Windkessel ports measured and advanced on the device (one block per port over
 * its candidates in the current cell tables).  Call after sph_cll_build and
 * before sph_buffer_update. */
sph_status sph_drivers_step(sph_ctx *ctx, sph_particles *p, double t, double dt, const int32_t *cell_start,
                            const int32_t *cell_end, void *stream);

/* out[0] = P, out[1] = Q of the last step, out[2] = the u0 in use (FOURIER).
 * Synchronises `stream`. */
sph_status sph_driver_read(sph_ctx *ctx, int32_t port_id, double out[3], void *stream);

/* Moving port (rotating sprinkler, §V.C): re-establish port port_id
 * at the pose (origin, Q) — e.g. theta = omega t + theta0 about a pivot,
 * computed by the caller — after this step's generation in the old pose
 * (Fig. rotation_procedure).  Every buffer particle of the port keeps its local
 * coordinates and local velocity (reading R23):
 *     x <- o1 + Q1^T (Q0 (x - o0)),  v <- Q1^T (Q0 v)      (pinned fp32)
 * and the port's candidate cells are enumerated on the device for the new pose
 * (the first move turns the port's runs into a fixed slice of one slot per cell
 * column around its bounding sphere).  Half extents, kind and BC are kept.
 * Call after sph_buffer_update with the same cell tables (the buffer particles
 * are found among the port's candidates) and before the next sph_cll_build.
 * Host-side errors, nothing enqueued: SPH_ERR_ARG (unknown port, NULL),
 * SPH_ERR_NOT_ORTHONORMAL, SPH_ERR_OUT_OF_GRID, SPH_ERR_OVERLAP (the new P_k meets
 * another port's). */
sph_status sph_port_move(sph_ctx *ctx, sph_particles *p, int32_t port_id, const float origin[3], const float Q[9],
                         const int32_t *cell_start, const int32_t *cell_end, void *stream);

/* Driver step (not the method): x <- fl(x + fl(v dt)) per component. */
sph_status sph_advect(sph_ctx *ctx, sph_particles *p, float dt, void *stream);

/* Cell-linked-list build: cell = clamp(floor(fl(fl(x - lo) * inv_cs)))
 * per axis, inv_cs = fl32(1/cs); counting sort by cell, ascending id within a
 * cell; tombstones dropped; the SoA of `in` is gathered into `out` (distinct
 * arrays) and out->n_dev receives the live count.  cell_start / cell_end
 * [ncells of this slab]: first / one-past-last position of each cell in `out`.
 * perm_or_null [in capacity]: new position of each input particle, -1 if dropped.
 * With registered ports the build also runs the next sph_buffer_update's
 * prologue (candidate offsets of the port runs in these cell tables, reset of
 * the per-update counters that sph_status_sync reports as created / deleted);
 * that update, given the same cell tables, then launches only its main kernel. */
sph_status sph_cll_build(sph_ctx *ctx, const sph_particles *in, sph_particles *out, int32_t *cell_start,
                         int32_t *cell_end, int32_t *perm_or_null, void *stream);

/* sph_advect (the driver's step) fused into the build: the advected positions
 * are computed in the key pass and again, bit-identically, where the gather
 * moves each particle into `out`; `in` is not written.  `out` is identical to
 * sph_advect followed by sph_cll_build.
 *
 * Key carry-over: a build that advects (and does not migrate) also prepares
 * the keys of the next build — each particle's cell after advecting its new
 * position by the same dt — and that build's histogram; sph_buffer_update,
 * sph_compact(_deferred) and sph_port_move keep them current for the particles
 * they change.  The next sph_advect_cll_build (or sph_cll_key) of `out` with the
 * same dt then skips its key pass; any other build clears them.  Results are
 * identical either way.  A caller that changes positions, velocities or the
 * particle set of `out` itself (other than through this library) must call
 * sph_cll_invalidate first. */
sph_status sph_advect_cll_build(sph_ctx *ctx, sph_particles *in, sph_particles *out, float dt, int32_t *cell_start,
                                int32_t *cell_end, int32_t *perm_or_null, void *stream);

/* Drop the carried-over keys (see above): the next build runs its key pass.
 * Host only. */
sph_status sph_cll_invalidate(sph_ctx *ctx);

/* The same build in two halves around the multi-GPU neighbour exchange (§8(e)),
 * so migration costs no extra pass over the particles:
 *   sph_cll_key    (optional advection when advect != 0) pinned cell keys; with
 *                  send buffers (layout as sph_migrate_pack) every particle whose
 *                  cell x-index left [cx_begin, cx_end) is packed for rank r-1 /
 *                  r+1 instead of being keyed;
 *   -- the caller exchanges the buffers (NCCL send/recv) --
 *   sph_cll_finish appends the received particles (recv_lo / recv_hi, may be
 *                  NULL) after the local ones with their keys, then scan,
 *                  scatter and gather exactly as sph_cll_build.
 * Without buffers the pair equals sph_cll_build / sph_advect_cll_build. */
sph_status sph_cll_key(sph_ctx *ctx, sph_particles *in, float dt, int32_t advect, float *send_lo, float *send_hi,
                       void *stream);
sph_status sph_cll_finish(sph_ctx *ctx, sph_particles *in, sph_particles *out, const float *recv_lo,
                          const float *recv_hi, int32_t *cell_start, int32_t *cell_end, int32_t *perm_or_null,
                          void *stream);

/* One buffer update over the candidates of every port (cells from registration,
 * particle ranges from the cell tables of the sph_cll_build just made on `p`):
 * X' = Q_k (x - o_k) in pinned fp32; decisions gated by x in P_k:
 *   inlet k         (Alg. 1): label k and X'_0 > a/2 -> CREATE
 *   outlet k        (Alg. 2): X'_0 > a/2             -> DELETE
 *   bidirectional k (Alg. 3): label k and X'_0 > a/2 -> CREATE,
 *                                        label k and X'_0 < -a/2 -> DELETE
 * CREATE stages a bitwise copy of the state together with its rank in
 * the canonical order (port, cell, id) — the compaction appends the staged
 * particles in that order — and recycles the particle x <- fl(x - fl(a u))
 * (Eqs. 2D/3D_Inverse_transformation).  DELETE writes a tombstone.
 * Outlet and bidirectional ports then relabel their non-deleted candidates on
 * post-recycle positions.
 * port_counts [2 * max_ports] (device int32): created_k at [k], deleted_k at
 * [max_ports + k]; overwritten. */
sph_status sph_buffer_update(sph_ctx *ctx, sph_particles *p, const int32_t *cell_start, const int32_t *cell_end,
                             int32_t *port_counts, void *stream);

/* Stable in-place compaction of the tombstones of the last update, then append
 * of the staged particles with new IDs from the count matrix
 * all_counts [nranks][2 * max_ports] (device; this rank's port_counts when
 * nranks = 1):  off(k, r) = next_id + sum_{k'<k} sum_r' C[r'][k'] + sum_{r'<r} C[r'][k].
 * *next_id_dev (device int64) += sum of all C; p->n_dev <- N - D + C.
 * perm_or_null [capacity]: new position of each old position, -1 if deleted. */
sph_status sph_compact(sph_ctx *ctx, sph_particles *p, const int32_t *all_counts, int32_t nranks, int32_t rank,
                       int64_t *next_id_dev, int32_t *perm_or_null, void *stream);

/* Compaction fused into the next cell-list build: assigns
 * the new IDs exactly as sph_compact and appends the staged particles at
 * [N, N + C) after the tombstones (p->n_dev <- N + C); the tombstones are
 * removed by the next sph_cll_build, whose result is identical to that of
 * sph_compact followed by sph_cll_build.  Saves one pass over the suffix. */
sph_status sph_compact_deferred(sph_ctx *ctx, sph_particles *p, const int32_t *all_counts, int32_t nranks,
                                int32_t rank, int64_t *next_id_dev, void *stream);

/* Multi-GPU slab migration (§8(e)).  pack: particles whose cell x-index left
 * [cx_begin, cx_end) are copied into send_lo (cx < cx_begin) or send_hi
 * (cx >= cx_end) and tombstoned.  A buffer holds a 4-word header (word 0 =
 * particle count, int32 bits) followed by max_migrate records of
 * sph_migrate_record_floats() = 2*dim + n_extra + 3 fp32 words
 * (position, velocity, extras, id as two 32-bit words, label).
 * unpack: appends the particles of a received buffer at the tail (n_dev += count).
 * Neither synchronises; the exchange itself is the caller's (NCCL send/recv). */
int32_t sph_migrate_record_floats(const sph_ctx *ctx);
sph_status sph_migrate_pack(sph_ctx *ctx, sph_particles *p, float *send_lo, float *send_hi, void *stream);
sph_status sph_migrate_unpack(sph_ctx *ctx, sph_particles *p, const float *recv, void *stream);

/* Multi-GPU x-slab decomposition: one process per GPU, each rank
 * a context whose grid slab [cx_begin, cx_end) is its share of the x cell
 * columns.  The decomposition shards naturally because the buffers are spatially
 * local: the candidates lie in "the nearby local cell-linked lists".
 * Per update two exchanges, both enqueued on the caller's stream (no host
 * synchronisation, so a P-rank update can be captured in one CUDA graph):
 *   neighbour migration   particles whose cell left the slab go to rank r-1 / r+1
 *                         (they move less than one cell per update);
 *   count allgather       every rank's per-port created / deleted counts -> the
 *                         count matrix sph_compact turns into IDs identical for
 *                         every number of GPUs (reading R14).
 * The library owns its communicator: NCCL (libnccl.so.2, loaded with dlopen at
 * the first call; in a torch process this is torch's NCCL) over NVLink /
 * NVSwitch, or an in-process loopback group for tests.  Migration messages are
 * fixed-size (4 header words + max_migrate records, sph_ctx_create), so no count
 * has to reach the host: size max_migrate to the expected migrants per face with
 * headroom; overflow is reported as SPH_ERR_CAPACITY by sph_status_sync.  The
 * migration buffers live in the workspace (sph_workspace_bytes includes them
 * when max_migrate > 0). */
#define SPH_COMM_ID_BYTES 128

/* Rank 0: a fresh NCCL unique id (SPH_COMM_ID_BYTES bytes) for the caller to
 * broadcast to every rank (e.g. torch.distributed.broadcast). */
sph_status sph_comm_unique_id(void *id_out);

/* Collective over the nranks processes: create this rank's NCCL communicator
 * from the broadcast id.  Needs the workspace set and, for nranks > 1,
 * max_migrate > 0.  Blocks until every rank has joined.  SPH_ERR_NCCL on
 * failure; SPH_ERR_STATE if the context already has a communicator. */
sph_status sph_comm_init(sph_ctx *ctx, const void *nccl_unique_id, int32_t nranks, int32_t rank);

/* Tests: the contexts ctxs[0..nranks) of this process (one device, rank r =
 * ctxs[r]) form a loopback group: the exchanges below become device copies on
 * the caller's stream.  Phase-ordered use only (every rank's pack before any
 * exchange, every update before any allgather); sph_migrate and
 * sph_migrate_cll_build are refused (SPH_ERR_STATE). */
sph_status sph_comm_init_loopback(sph_ctx *const *ctxs, int32_t nranks);

/* all_counts [nranks][2 max_ports] (device int32) <- every rank's port_counts
 * [2 max_ports] (as written by sph_buffer_update): ncclAllGather on `stream`.
 * Without a communicator (one rank) a device copy. */
sph_status sph_allgather_counts(sph_ctx *ctx, const int32_t *port_counts, int32_t *all_counts, void *stream);

/* Neighbour exchange of the library's migration buffers: send lo -> rank r-1,
 * send hi -> rank r+1 and the matching receives, in one NCCL group
 * (ncclGroupStart / ncclSend / ncclRecv / ncclGroupEnd). */
sph_status sph_migrate_exchange(sph_ctx *ctx, void *stream);

/* Standalone migration (between an advection and a plain sph_cll_build):
 * pack the particles whose cell left the slab (tombstoned), exchange, append
 * the received ones.  No-op on one rank. */
sph_status sph_migrate(sph_ctx *ctx, sph_particles *p, void *stream);

/* The build with the migration fused into its key pass — the per-update call of
 * a rank: sph_cll_key (advection when advect != 0; leavers packed into the
 * library's buffers), sph_migrate_exchange, sph_cll_finish (arrivals appended,
 * then scan, scatter, gather).  With a communicator, sph_cll_key and
 * sph_cll_finish given NULL buffers use the library's buffers too (the split
 * form, required by a loopback group). */
sph_status sph_migrate_cll_build(sph_ctx *ctx, sph_particles *in, sph_particles *out, float dt, int32_t advect,
                                 int32_t *cell_start, int32_t *cell_end, int32_t *perm_or_null, void *stream);

/* The only synchronising call: waits for `stream`, returns the statistics and
 * the first sticky device error (SPH_ERR_CAPACITY / SPH_ERR_MOTION) if any, or
 * an asynchronous NCCL error (SPH_ERR_NCCL). */
sph_status sph_status_sync(sph_ctx *ctx, const sph_particles *p, void *stream, sph_stats *out);

/* Number of kernels this context has launched (for the bench's launch count). */
int64_t sph_launch_count(const sph_ctx *ctx);

/* Live per-kernel timing: when enabled, every kernel launch is bracketed by two
 * CUDA events on its stream (no synchronisation).  sph_profile resets the
 * totals; sph_profile_read waits for the last event and returns, per kernel id
 * (0 .. SPH_NKERNELS-1, named by sph_kernel_name), the summed milliseconds and
 * the number of launches.  ms, count: host arrays of SPH_NKERNELS. */
#define SPH_NKERNELS 17
sph_status sph_profile(sph_ctx *ctx, int32_t enable);
sph_status sph_profile_read(sph_ctx *ctx, double *ms, int64_t *count);
const char *sph_kernel_name(int32_t i);

/* Host-only helpers ---------------------------------------------------------- */

/* Cells of the slab intersecting P_k (separating-axis test, P_k inflated by
 * 1e-3 cs), as x-major runs of consecutive local cell ids [c0, c1] (inclusive).
 * runs_out: int32[2 * max_runs] or NULL to count only. */
sph_status sph_port_cells(const sph_grid *grid, const float origin[3], const float Q[9], const float half_extents[3],
                          int32_t *runs_out, int64_t max_runs, int64_t *n_runs, int64_t *n_cells);

/* 3-D frame from the in/outflow axis u via Rodrigues (Eqs. rotation_axis,
 * antisymmetric_matrix, rotation_matrix) with reading R1 (Q = R^T, so
 * Q u = e1, Eq. 3D_normal_transformation), then a roll psi about u.
 * Q_out: float[9] row-major. */
sph_status sph_frame_from_axis(const double u[3], double psi, float Q_out[9]);

#ifdef __cplusplus
}
#endif
#endif /* SPHBUF_H */
