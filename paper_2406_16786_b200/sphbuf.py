"""Thin Python binding of the C ABI in include/sphbuf.h (libsphbuf.so).

Argument marshalling only: every step of the path runs in the library's sm_100a
kernels.  torch supplies device memory and streams.  There is no CPU fallback:
if the library is missing or no CUDA device is present, calls raise.

Function names follow the ABI; ``BufferUpdater`` is the user-facing driver
(one rank): it owns the double-buffered particle arrays, cell tables, counts and
workspace, and runs advect -> sph_cll_build -> sph_buffer_update -> sph_compact.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os

import torch

from . import build as _build

MAX_PORTS = 64
MAX_EXTRA = 8
INLET, OUTLET, BIDIRECTIONAL = 0, 1, 2

STATUS = {0: "SPH_OK", -1: "SPH_ERR_ARG", -2: "SPH_ERR_NOT_ORTHONORMAL", -3: "SPH_ERR_OVERLAP",
          -4: "SPH_ERR_OUT_OF_GRID", -5: "SPH_ERR_CAPACITY", -6: "SPH_ERR_MOTION", -7: "SPH_ERR_CUDA",
          -8: "SPH_ERR_NCCL", -9: "SPH_ERR_STATE"}
COMM_ID_BYTES = 128                 # = SPH_COMM_ID_BYTES


class SphError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class sph_grid(C.Structure):
    _fields_ = [("dim", C.c_int32), ("lo", C.c_float * 3), ("cs", C.c_float), ("ncell", C.c_int32 * 3),
                ("cx_begin", C.c_int32), ("cx_end", C.c_int32)]


class sph_particles(C.Structure):
    _fields_ = [("x", C.c_void_p), ("y", C.c_void_p), ("z", C.c_void_p), ("vx", C.c_void_p), ("vy", C.c_void_p),
                ("vz", C.c_void_p), ("extra", C.c_void_p * MAX_EXTRA), ("n_extra", C.c_int32), ("id", C.c_void_p),
                ("label", C.c_void_p), ("n_dev", C.c_void_p), ("capacity", C.c_int64)]


class sph_bc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("rho0", C.c_float), ("c0", C.c_float), ("p_b", C.c_float),
                ("rho_column", C.c_int32), ("profile", C.c_int32), ("u0", C.c_float), ("radius", C.c_float)]


class sph_driver(C.Structure):
    _fields_ = [("kind", C.c_int32), ("a", C.c_double * 9), ("b", C.c_double * 9), ("omega", C.c_double),
                ("Rp", C.c_double), ("C", C.c_double), ("Rd", C.c_double), ("P0", C.c_double),
                ("volume", C.c_double)]


class sph_stats(C.Structure):
    _fields_ = [("n", C.c_int64), ("candidates", C.c_int64), ("created", C.c_int64), ("deleted", C.c_int64),
                ("checked_total", C.c_int64), ("out_of_grid", C.c_int64), ("motion_errors", C.c_int64),
                ("migrated_out", C.c_int64), ("first_deleted", C.c_int64), ("status_bits", C.c_int32),
                ("n_ports", C.c_int32)]


_L = None
EXPORTS = ["sph_ctx_create", "sph_ctx_destroy", "sph_last_error", "sph_workspace_bytes", "sph_set_workspace",
           "sph_port_check", "sph_buffer_register", "sph_advect", "sph_cll_build", "sph_buffer_update",
           "sph_compact", "sph_migrate_record_floats", "sph_migrate_pack", "sph_migrate_unpack", "sph_status_sync",
           "sph_launch_count", "sph_port_cells", "sph_frame_from_axis", "sph_profile", "sph_profile_read",
           "sph_kernel_name", "sph_advect_cll_build", "sph_compact_deferred", "sph_cll_key", "sph_cll_finish",
           "sph_port_set_bc", "sph_port_move", "sph_port_set_driver", "sph_cll_invalidate",
           "sph_drivers_step", "sph_driver_read", "sph_comm_unique_id", "sph_comm_init", "sph_comm_init_loopback",
           "sph_allgather_counts", "sph_migrate_exchange", "sph_migrate", "sph_migrate_cll_build"]
NKERNELS = 17                       # = SPH_NKERNELS in include/sphbuf.h


def lib():
    """Load libsphbuf.so (building it in-tree with nvcc if stale).  Raises if absent."""
    global _L
    if _L is not None:
        return _L
    debug = os.environ.get("SPHBUF_DEBUG") == "1"     # the bounds-asserting build (tests only)
    trace = os.environ.get("SPHBUF_TRACE") == "1"     # tile timeline of the update (tools/upd_trace.py)
    path = _build.LIB_DEBUG if debug else _build.LIB_TRACE if trace else _build.LIB
    if os.environ.get("SPHBUF_LIB"):                  # another build of the same sources (A/B timing)
        path = os.environ["SPHBUF_LIB"]
    elif not os.path.exists(path) or os.environ.get("SPHBUF_REBUILD"):
        path = _build.build(debug=debug, trace=trace)
    L = C.CDLL(path)
    vp, i32, i64, f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_float
    P = C.POINTER
    L.sph_ctx_create.argtypes = [P(sph_grid), f32, i64, i32, i64, i64, i32, P(vp)]
    L.sph_ctx_destroy.argtypes = [vp]
    L.sph_ctx_destroy.restype = None
    L.sph_last_error.argtypes = [vp]
    L.sph_last_error.restype = C.c_char_p
    L.sph_workspace_bytes.argtypes = [vp]
    L.sph_workspace_bytes.restype = C.c_size_t
    L.sph_set_workspace.argtypes = [vp, vp, C.c_size_t]
    L.sph_port_check.argtypes = [vp, vp, vp, vp, i32, i32, f32]
    L.sph_buffer_register.argtypes = [vp, P(sph_particles), vp, vp, vp, i32, i32, f32, P(i32), vp, vp]
    L.sph_advect.argtypes = [vp, P(sph_particles), f32, vp]
    L.sph_cll_build.argtypes = [vp, P(sph_particles), P(sph_particles), vp, vp, vp, vp]
    L.sph_advect_cll_build.argtypes = [vp, P(sph_particles), P(sph_particles), f32, vp, vp, vp, vp]
    L.sph_advect_cll_build.restype = C.c_int
    L.sph_port_set_bc.argtypes = [vp, i32, P(sph_bc)]
    L.sph_port_set_bc.restype = C.c_int
    L.sph_port_set_driver.argtypes = [vp, i32, P(sph_driver)]
    L.sph_port_set_driver.restype = C.c_int
    L.sph_drivers_step.argtypes = [vp, P(sph_particles), C.c_double, C.c_double, vp, vp, vp]
    L.sph_drivers_step.restype = C.c_int
    L.sph_driver_read.argtypes = [vp, i32, vp, vp]
    L.sph_driver_read.restype = C.c_int
    L.sph_port_move.argtypes = [vp, P(sph_particles), i32, vp, vp, vp, vp, vp]
    L.sph_port_move.restype = C.c_int
    L.sph_cll_invalidate.argtypes = [vp]
    L.sph_cll_invalidate.restype = C.c_int
    L.sph_cll_key.argtypes = [vp, P(sph_particles), f32, i32, vp, vp, vp]
    L.sph_cll_key.restype = C.c_int
    L.sph_cll_finish.argtypes = [vp, P(sph_particles), P(sph_particles), vp, vp, vp, vp, vp, vp]
    L.sph_cll_finish.restype = C.c_int
    L.sph_buffer_update.argtypes = [vp, P(sph_particles), vp, vp, vp, vp]
    L.sph_compact.argtypes = [vp, P(sph_particles), vp, i32, i32, vp, vp, vp]
    L.sph_compact_deferred.argtypes = [vp, P(sph_particles), vp, i32, i32, vp, vp]
    L.sph_compact_deferred.restype = C.c_int
    L.sph_migrate_record_floats.argtypes = [vp]
    L.sph_migrate_record_floats.restype = i32
    L.sph_migrate_pack.argtypes = [vp, P(sph_particles), vp, vp, vp]
    L.sph_migrate_unpack.argtypes = [vp, P(sph_particles), vp, vp]
    L.sph_status_sync.argtypes = [vp, P(sph_particles), vp, P(sph_stats)]
    L.sph_launch_count.argtypes = [vp]
    L.sph_launch_count.restype = i64
    L.sph_port_cells.argtypes = [P(sph_grid), vp, vp, vp, vp, i64, P(i64), P(i64)]
    L.sph_frame_from_axis.argtypes = [vp, C.c_double, vp]
    L.sph_profile.argtypes = [vp, i32]
    L.sph_profile_read.argtypes = [vp, vp, vp]
    L.sph_kernel_name.argtypes = [i32]
    L.sph_kernel_name.restype = C.c_char_p
    L.sph_comm_unique_id.argtypes = [vp]
    L.sph_comm_init.argtypes = [vp, vp, i32, i32]
    L.sph_comm_init_loopback.argtypes = [vp, i32]
    L.sph_allgather_counts.argtypes = [vp, vp, vp, vp]
    L.sph_migrate_exchange.argtypes = [vp, vp]
    L.sph_migrate.argtypes = [vp, P(sph_particles), vp]
    L.sph_migrate_cll_build.argtypes = [vp, P(sph_particles), P(sph_particles), f32, i32, vp, vp, vp, vp]
    for name in ("sph_comm_unique_id", "sph_comm_init", "sph_comm_init_loopback", "sph_allgather_counts",
                 "sph_migrate_exchange", "sph_migrate", "sph_migrate_cll_build"):
        getattr(L, name).restype = C.c_int
    for name in ("sph_profile", "sph_profile_read","sph_ctx_create", "sph_set_workspace", "sph_port_check", "sph_buffer_register", "sph_advect",
                 "sph_cll_build", "sph_buffer_update", "sph_compact", "sph_migrate_pack", "sph_migrate_unpack",
                 "sph_status_sync", "sph_port_cells", "sph_frame_from_axis"):
        getattr(L, name).restype = C.c_int
    _L = L
    return L


def _check(rc, ctx=None):
    if rc != 0:
        msg = lib().sph_last_error(ctx).decode() if ctx else ""
        raise SphError(rc, msg)


def _f3(v):
    return (C.c_float * 3)(*[float(a) for a in v])


def _f9(v):
    return (C.c_float * 9)(*[float(a) for a in v])


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(None)


def make_grid(g) -> sph_grid:
    G = sph_grid()
    G.dim = g.dim
    G.lo[:] = [float(v) for v in g.lo]
    G.cs = float(g.cs)
    G.ncell[:] = [int(v) for v in g.ncell]
    G.cx_begin = int(g.cx_begin)
    G.cx_end = int(g.cx_end)
    return G


# ----------------------------------------------------------------- ABI wrappers

class Context:
    """Owns an sph_ctx*."""

    def __init__(self, grid, h, capacity, max_ports, max_new, max_migrate=0, n_extra=0):
        self.G = make_grid(grid)
        h_ = C.c_void_p()
        _check(lib().sph_ctx_create(C.byref(self.G), float(h), int(capacity), int(max_ports), int(max_new),
                                    int(max_migrate), int(n_extra), C.byref(h_)))
        self.h = h_
        self.dim = grid.dim
        self.max_ports = max_ports

    def __del__(self):
        try:
            if getattr(self, "h", None) and self.h.value:
                lib().sph_ctx_destroy(self.h)
                self.h = C.c_void_p()
        except Exception:
            pass

    @property
    def last_error(self):
        return lib().sph_last_error(self.h).decode()


def sph_workspace_bytes(ctx: Context) -> int:
    return int(lib().sph_workspace_bytes(ctx.h))


def sph_set_workspace(ctx: Context, ws: torch.Tensor):
    _check(lib().sph_set_workspace(ctx.h, _ptr(ws), ws.numel() * ws.element_size()), ctx.h)


def sph_port_check(ctx: Context, origin, Q, half_extents, kind, layers, dp) -> int:
    return int(lib().sph_port_check(ctx.h, _f3(origin), _f9(Q), _f3(half_extents), int(kind), int(layers),
                                     float(dp)))


def sph_buffer_register(ctx, parts, origin, Q, half_extents, kind, layers, dp, members_out=None, stream=None) -> int:
    pid = C.c_int32(-1)
    _check(lib().sph_buffer_register(ctx.h, C.byref(parts.abi), _f3(origin), _f9(Q), _f3(half_extents), int(kind),
                                     int(layers), float(dp), C.byref(pid), _ptr(members_out), _stream(stream)), ctx.h)
    return pid.value


def sph_port_set_bc(ctx, port_id, bc):
    """bc: an object with kind, rho0, c0, p_b, rho_column, profile, u0, radius (inputs.BC)."""
    B = sph_bc()
    for f, _ in sph_bc._fields_:
        setattr(B, f, getattr(bc, f))
    _check(lib().sph_port_set_bc(ctx.h, int(port_id), C.byref(B)), ctx.h)


def sph_port_set_driver(ctx, port_id, drv):
    """drv: an object with kind, a, b, omega, Rp, C, Rd, P0, volume (inputs.Driver)."""
    D = sph_driver()
    D.kind = int(drv.kind)
    D.a[:] = [float(v) for v in drv.a]
    D.b[:] = [float(v) for v in drv.b]
    for f in ("omega", "Rp", "C", "Rd", "P0", "volume"):
        setattr(D, f, float(getattr(drv, f)))
    _check(lib().sph_port_set_driver(ctx.h, int(port_id), C.byref(D)), ctx.h)


def sph_drivers_step(ctx, parts, t, dt, cell_start, cell_end, stream=None):
    _check(lib().sph_drivers_step(ctx.h, C.byref(parts.abi), float(t), float(dt), _ptr(cell_start), _ptr(cell_end),
                                  _stream(stream)), ctx.h)


def sph_driver_read(ctx, port_id, stream=None) -> dict:
    out = (C.c_double * 3)()
    _check(lib().sph_driver_read(ctx.h, int(port_id), out, _stream(stream)), ctx.h)
    return {"P": out[0], "Q": out[1], "u0": out[2]}


def sph_advect(ctx, parts, dt, stream=None):
    _check(lib().sph_advect(ctx.h, C.byref(parts.abi), float(dt), _stream(stream)), ctx.h)


def sph_cll_build(ctx, pin, pout, cell_start, cell_end, perm=None, stream=None):
    _check(lib().sph_cll_build(ctx.h, C.byref(pin.abi), C.byref(pout.abi), _ptr(cell_start), _ptr(cell_end),
                               _ptr(perm), _stream(stream)), ctx.h)


def sph_advect_cll_build(ctx, pin, pout, dt, cell_start, cell_end, perm=None, stream=None):
    _check(lib().sph_advect_cll_build(ctx.h, C.byref(pin.abi), C.byref(pout.abi), float(dt), _ptr(cell_start),
                                      _ptr(cell_end), _ptr(perm), _stream(stream)), ctx.h)


def sph_port_move(ctx, parts, port_id, origin, Q, cell_start, cell_end, stream=None):
    o, q = _f3(origin), _f9(Q)
    _check(lib().sph_port_move(ctx.h, C.byref(parts.abi), int(port_id), o, q, _ptr(cell_start), _ptr(cell_end),
                               _stream(stream)), ctx.h)


def sph_cll_invalidate(ctx):
    _check(lib().sph_cll_invalidate(ctx.h), ctx.h)


def sph_cll_key(ctx, pin, dt=None, send_lo=None, send_hi=None, stream=None):
    _check(lib().sph_cll_key(ctx.h, C.byref(pin.abi), float(dt or 0.0), 0 if dt is None else 1, _ptr(send_lo),
                             _ptr(send_hi), _stream(stream)), ctx.h)


def sph_cll_finish(ctx, pin, pout, cell_start, cell_end, recv_lo=None, recv_hi=None, perm=None, stream=None):
    _check(lib().sph_cll_finish(ctx.h, C.byref(pin.abi), C.byref(pout.abi), _ptr(recv_lo), _ptr(recv_hi),
                                _ptr(cell_start), _ptr(cell_end), _ptr(perm), _stream(stream)), ctx.h)


def sph_buffer_update(ctx, parts, cell_start, cell_end, port_counts, stream=None):
    _check(lib().sph_buffer_update(ctx.h, C.byref(parts.abi), _ptr(cell_start), _ptr(cell_end), _ptr(port_counts),
                                   _stream(stream)), ctx.h)


def sph_compact(ctx, parts, all_counts, nranks, rank, next_id, perm=None, stream=None):
    _check(lib().sph_compact(ctx.h, C.byref(parts.abi), _ptr(all_counts), int(nranks), int(rank), _ptr(next_id),
                             _ptr(perm), _stream(stream)), ctx.h)


def sph_compact_deferred(ctx, parts, all_counts, nranks, rank, next_id, stream=None):
    _check(lib().sph_compact_deferred(ctx.h, C.byref(parts.abi), _ptr(all_counts), int(nranks), int(rank),
                                      _ptr(next_id), _stream(stream)), ctx.h)


def sph_migrate_record_floats(ctx) -> int:
    return int(lib().sph_migrate_record_floats(ctx.h))


def sph_migrate_pack(ctx, parts, send_lo, send_hi, stream=None):
    _check(lib().sph_migrate_pack(ctx.h, C.byref(parts.abi), _ptr(send_lo), _ptr(send_hi), _stream(stream)), ctx.h)


def sph_migrate_unpack(ctx, parts, recv, stream=None):
    _check(lib().sph_migrate_unpack(ctx.h, C.byref(parts.abi), _ptr(recv), _stream(stream)), ctx.h)


def sph_comm_unique_id() -> bytes:
    buf = (C.c_ubyte * COMM_ID_BYTES)()
    _check(lib().sph_comm_unique_id(buf))
    return bytes(buf)


def sph_comm_init(ctx, unique_id: bytes, nranks, rank):
    buf = (C.c_ubyte * COMM_ID_BYTES).from_buffer_copy(unique_id)
    _check(lib().sph_comm_init(ctx.h, buf, int(nranks), int(rank)), ctx.h)


def sph_comm_init_loopback(ctxs):
    arr = (C.c_void_p * len(ctxs))(*[c.h.value for c in ctxs])
    rc = lib().sph_comm_init_loopback(arr, len(ctxs))
    if rc:
        msgs = [m for m in (c.last_error for c in ctxs) if m]
        raise SphError(rc, "; ".join(msgs))


def sph_allgather_counts(ctx, port_counts, all_counts, stream=None):
    _check(lib().sph_allgather_counts(ctx.h, _ptr(port_counts), _ptr(all_counts), _stream(stream)), ctx.h)


def sph_migrate_exchange(ctx, stream=None):
    _check(lib().sph_migrate_exchange(ctx.h, _stream(stream)), ctx.h)


def sph_migrate(ctx, parts, stream=None):
    _check(lib().sph_migrate(ctx.h, C.byref(parts.abi), _stream(stream)), ctx.h)


def sph_migrate_cll_build(ctx, pin, pout, dt, cell_start, cell_end, perm=None, stream=None):
    _check(lib().sph_migrate_cll_build(ctx.h, C.byref(pin.abi), C.byref(pout.abi), float(dt or 0.0),
                                       0 if dt is None else 1, _ptr(cell_start), _ptr(cell_end), _ptr(perm),
                                       _stream(stream)), ctx.h)


def sph_status_sync(ctx, parts=None, stream=None, check=True) -> dict:
    st = sph_stats()
    rc = lib().sph_status_sync(ctx.h, C.byref(parts.abi) if parts is not None else None, _stream(stream),
                               C.byref(st))
    d = {f: getattr(st, f) for f, _ in sph_stats._fields_}
    d["rc"] = rc
    if check:
        _check(rc, ctx.h)
    return d


def sph_launch_count(ctx) -> int:
    return int(lib().sph_launch_count(ctx.h))


def sph_profile(ctx, enable: bool):
    _check(lib().sph_profile(ctx.h, 1 if enable else 0), ctx.h)


def sph_profile_read(ctx) -> dict:
    """{kernel name: (total ms, launches)} since the last sph_profile call (synchronising)."""
    ms = (C.c_double * NKERNELS)()
    cnt = (C.c_int64 * NKERNELS)()
    _check(lib().sph_profile_read(ctx.h, ms, cnt), ctx.h)
    return {lib().sph_kernel_name(i).decode(): (ms[i], cnt[i]) for i in range(NKERNELS)}


def sph_port_cells(grid, origin, Q, half_extents):
    """Host-only: runs [c0, c1] (inclusive, local cell ids) of the cells intersecting P_k."""
    G = make_grid(grid)
    nr, nc = C.c_int64(0), C.c_int64(0)
    _check(lib().sph_port_cells(C.byref(G), _f3(origin), _f9(Q), _f3(half_extents), None, 0, C.byref(nr),
                                C.byref(nc)))
    buf = (C.c_int32 * max(1, 2 * nr.value))()
    _check(lib().sph_port_cells(C.byref(G), _f3(origin), _f9(Q), _f3(half_extents), buf, nr.value, C.byref(nr),
                                C.byref(nc)))
    runs = [(buf[2 * i], buf[2 * i + 1]) for i in range(nr.value)]
    return runs, nc.value


def sph_frame_from_axis(u, psi=0.0):
    uu = (C.c_double * 3)(*[float(a) for a in u])
    Q = (C.c_float * 9)()
    _check(lib().sph_frame_from_axis(uu, float(psi), Q))
    return list(Q)


# ----------------------------------------------------------------- device arrays

class Particles:
    """One set of SoA device columns at fixed capacity plus the device live count."""

    COLS = ("x", "y", "z", "vx", "vy", "vz")

    def __init__(self, dim, capacity, n_extra=0, device="cuda"):
        self.dim, self.capacity, self.n_extra = dim, int(capacity), n_extra
        cap = max(1, self.capacity)
        f = dict(dtype=torch.float32, device=device)
        self.cols = {c: torch.empty(cap, **f) for c in self.COLS if dim == 3 or c not in ("z", "vz")}
        self.extra = [torch.empty(cap, **f) for _ in range(n_extra)]
        self.id = torch.empty(cap, dtype=torch.int64, device=device)
        self.label = torch.empty(cap, dtype=torch.int32, device=device)
        self.n = torch.zeros(1, dtype=torch.int64, device=device)
        a = sph_particles()
        for c in self.COLS:
            setattr(a, c, self.cols[c].data_ptr() if c in self.cols else None)
        for e in range(MAX_EXTRA):
            a.extra[e] = self.extra[e].data_ptr() if e < n_extra else None
        a.n_extra = n_extra
        a.id = self.id.data_ptr()
        a.label = self.label.data_ptr()
        a.n_dev = self.n.data_ptr()
        a.capacity = self.capacity
        self.abi = a

    def load(self, st: dict, non_blocking=False):
        n = int(st["x"].numel())
        if n > self.capacity:
            raise SphError(-5, "state larger than capacity")
        for c, t in self.cols.items():
            t[:n].copy_(st[c], non_blocking=non_blocking)
        for e, t in enumerate(self.extra):
            t[:n].copy_(st["extra"][e], non_blocking=non_blocking)
        self.id[:n].copy_(st["id"], non_blocking=non_blocking)
        self.label[:n].copy_(st["label"], non_blocking=non_blocking)
        self.n.fill_(n)

    def count(self) -> int:
        return int(self.n.item())

    def to_dict(self, n=None, device="cpu") -> dict:
        n = self.count() if n is None else n
        d = {c: t[:n].to(device) for c, t in self.cols.items()}
        if self.extra:
            d["extra"] = [t[:n].to(device) for t in self.extra]
        d["id"] = self.id[:n].to(device)
        d["label"] = self.label[:n].to(device)
        return d


class BufferUpdater:
    """One rank of the buffer update (the public API).

    ``ports``: list of inputs.Port-like objects (origin, Q, half_extents, kind,
    layers).  ``state``: dict of x, y, (z), vx, vy, (vz), id, label (+extra).
    """

    def __init__(self, grid, h, dp, ports, capacity, max_new=None, n_extra=0, max_migrate=0, device="cuda"):
        if not torch.cuda.is_available():
            raise SphError(-7, "no CUDA device: the buffer update has no CPU path")
        self.grid, self.h, self.dp, self.dim = grid, h, dp, grid.dim
        self.device = torch.device(device)
        self.ports = list(ports)
        self.capacity = int(capacity)
        self.max_new = int(max_new if max_new is not None else max(4096, capacity // 50))
        self.ctx = Context(grid, h, self.capacity, MAX_PORTS, self.max_new, max_migrate, n_extra)
        self.ws = torch.empty(sph_workspace_bytes(self.ctx), dtype=torch.uint8, device=self.device)
        sph_set_workspace(self.ctx, self.ws)
        self.A = Particles(self.dim, self.capacity, n_extra, self.device)
        self.B = Particles(self.dim, self.capacity, n_extra, self.device)
        nc = grid.ncells_local
        self.cell_start = torch.empty(max(nc, 4), dtype=torch.int32, device=self.device)
        self.cell_end = torch.empty(max(nc, 4), dtype=torch.int32, device=self.device)
        self.port_counts = torch.zeros(2 * MAX_PORTS, dtype=torch.int32, device=self.device)
        self.next_id = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.members = torch.zeros(max(1, len(self.ports)), dtype=torch.int64, device=self.device)
        self.registered = False

    # --- setup
    def load(self, state: dict, next_id: int):
        self.A.load(state)
        self.next_id.fill_(int(next_id))
        sph_cll_invalidate(self.ctx)   # new particles: no carried-over keys apply

    def register_ports(self, stream=None):
        for k, p in enumerate(self.ports):
            pid = sph_buffer_register(self.ctx, self.A, p.origin, p.Q, p.half_extents, p.kind, p.layers, self.dp,
                                      self.members[k:k + 1], stream)
            assert pid == k
            if getattr(p, "bc", None) is not None and p.bc.kind:
                sph_port_set_bc(self.ctx, k, p.bc)
            if getattr(p, "driver", None) is not None and p.driver.kind:
                sph_port_set_driver(self.ctx, k, p.driver)
        self.registered = True

    # --- one update (the hot path); nothing here synchronises
    def advect(self, dt, stream=None):
        sph_advect(self.ctx, self.A, dt, stream)

    def cll_build(self, perm=None, stream=None, dt=None):
        """Cell-list build A -> B (then swap); with dt, the advection is fused into its key pass."""
        if dt is None:
            sph_cll_build(self.ctx, self.A, self.B, self.cell_start, self.cell_end, perm, stream)
        else:
            sph_advect_cll_build(self.ctx, self.A, self.B, dt, self.cell_start, self.cell_end, perm, stream)
        self.A, self.B = self.B, self.A

    def update(self, stream=None):
        sph_buffer_update(self.ctx, self.A, self.cell_start, self.cell_end, self.port_counts, stream)

    def drivers_step(self, t, dt, stream=None):
        """Advance the ports' time-dependent drivers to time t (after the build)."""
        sph_drivers_step(self.ctx, self.A, t, dt, self.cell_start, self.cell_end, stream)

    def driver_state(self, k) -> dict:
        return sph_driver_read(self.ctx, k)

    def move_port(self, k, origin, Q, stream=None):
        """Re-establish port k at the pose (origin, Q) after this step's update (moving
        port): its buffer particles keep local coordinates and velocities."""
        sph_port_move(self.ctx, self.A, k, origin, Q, self.cell_start, self.cell_end, stream)
        p = self.ports[k]
        o, q = tuple(float(v) for v in origin), tuple(float(v) for v in Q)
        if dataclasses.is_dataclass(p):
            self.ports[k] = dataclasses.replace(p, origin=o, Q=q)
        else:
            p.origin, p.Q = o, q

    def compact(self, all_counts=None, nranks=1, rank=0, perm=None, stream=None, deferred=False):
        """IDs + compaction (sph_compact), or IDs + append with the removal left to
        the next cell-list build (sph_compact_deferred)."""
        ac = self.port_counts if all_counts is None else all_counts
        if deferred:
            sph_compact_deferred(self.ctx, self.A, ac, nranks, rank, self.next_id, stream)
        else:
            sph_compact(self.ctx, self.A, ac, nranks, rank, self.next_id, perm, stream)

    def step(self, dt, stream=None, fused=True, deferred=False):
        """advect -> cell-list build -> buffer update -> compaction.  fused: the
        advection runs inside the build's key pass (sph_advect_cll_build);
        deferred: the compaction's removal runs inside the next build."""
        if dt is not None and not fused:
            self.advect(dt, stream)
            dt = None
        self.cll_build(stream=stream, dt=dt)
        self.update(stream)
        self.compact(stream=stream, deferred=deferred)

    # --- inspection (synchronising)
    def stats(self, check=True) -> dict:
        return sph_status_sync(self.ctx, self.A, check=check)

    def state(self, device="cpu") -> dict:
        return self.A.to_dict(device=device)

    def launches(self) -> int:
        return sph_launch_count(self.ctx)

    def capture(self, dt, deferred=True):
        """Capture two updates (A -> B -> A, so replays are composable) into one CUDA
        graph.  Every count the kernels need is device-resident, so a replay needs no
        host work: the launch-bound small configurations run at kernel speed."""
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):          # warm-up: occupancy queries, lazy init
            self.step(dt, deferred=deferred)
            self.step(dt, deferred=deferred)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step(dt, deferred=deferred)
            self.step(dt, deferred=deferred)
        return g
