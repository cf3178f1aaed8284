"""CPU oracle for the in/outlet buffer update of arXiv 2406.16786 — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2406_16786_b200`` never imports it.  The arithmetic lives in
``sph_oracle.c`` (plain C, compiled ``-O2 -ffp-contract=off``); this file only
marshals numpy arrays through ctypes and builds the shared object on demand.

Functions follow SURVEY.md §8(c) O0-O7 and cite PAPER.md in sph_oracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sph_oracle.c")
_SO = os.path.join(_HERE, "_build", "liboracle.so")
CFLAGS = ["-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall", "-fopenmp"]


def build(force: bool = False) -> str:
    """Compile sph_oracle.c with gcc (no GPU needed)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        os.makedirs(os.path.dirname(_SO), exist_ok=True)
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _SO)
    return _SO


class Grid(C.Structure):
    _fields_ = [("dim", C.c_int32), ("lo", C.c_float * 3), ("cs", C.c_float), ("ncell", C.c_int32 * 3),
                ("cx_begin", C.c_int32), ("cx_end", C.c_int32)]


class Port(C.Structure):
    _fields_ = [("o", C.c_float * 3), ("Q", C.c_float * 9), ("he", C.c_float * 3), ("kind", C.c_int32),
                ("bc", C.c_int32), ("profile", C.c_int32), ("rho_col", C.c_int32), ("rho_b", C.c_float),
                ("u0", C.c_float), ("R", C.c_float), ("R2", C.c_float)]


class State(C.Structure):
    _fields_ = [("n", C.c_int64), ("x", C.c_void_p), ("y", C.c_void_p), ("z", C.c_void_p),
                ("vx", C.c_void_p), ("vy", C.c_void_p), ("vz", C.c_void_p), ("n_extra", C.c_int32),
                ("extra", C.c_void_p), ("id", C.c_void_p), ("label", C.c_void_p)]


class UpdateOut(C.Structure):
    _fields_ = [("order", C.c_void_p), ("cell_start", C.c_void_p), ("cell_end", C.c_void_p),
                ("out_of_grid", C.c_int64), ("create_port", C.c_void_p), ("delete_port", C.c_void_p),
                ("sorted", State), ("staged", State), ("stage_port", C.c_void_p), ("stage_src", C.c_void_p),
                ("cap_stage", C.c_int64), ("n_stage", C.c_int64), ("port_counts", C.c_void_p),
                ("checked", C.c_int64), ("multi_decision", C.c_int64), ("motion_errors", C.c_int64),
                ("t_cll", C.c_double), ("t_decide", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.orc_set_threads.argtypes = [C.c_int32]
        L.orc_set_threads.restype = C.c_int32
        L.orc_frame_2d.argtypes = [C.c_double, C.c_void_p]
        L.orc_frame_3d.argtypes = [C.c_void_p, C.c_void_p]
        L.orc_frame_3d.restype = C.c_int
        L.orc_to_local_f64.argtypes = [C.POINTER(Port), C.c_int32, C.c_float, C.c_float, C.c_float, C.c_void_p]
        L.orc_to_local_f32.argtypes = [C.POINTER(Port), C.c_int32, C.c_float, C.c_float, C.c_float, C.c_void_p]
        L.orc_inverse_recycle_f64.argtypes = [C.POINTER(Port), C.c_int32, C.c_void_p, C.c_void_p]
        L.orc_ncells.argtypes = [C.POINTER(Grid)]
        L.orc_ncells.restype = C.c_int64
        L.orc_cell_of.argtypes = [C.POINTER(Grid), C.c_float, C.c_float, C.c_float, C.POINTER(C.c_int32)]
        L.orc_cell_of.restype = C.c_int64
        L.orc_port_cells.argtypes = [C.POINTER(Grid), C.POINTER(Port), C.c_void_p]
        L.orc_port_cells.restype = C.c_int64
        L.orc_advect.argtypes = [C.POINTER(State), C.c_int32, C.c_float]
        L.orc_fourier.argtypes = [C.c_double, C.c_void_p, C.c_void_p, C.c_double]
        L.orc_fourier.restype = C.c_double
        L.orc_port_flux.argtypes = [C.POINTER(State), C.c_int32, C.POINTER(Port), C.c_int32]
        L.orc_port_flux.restype = C.c_int64
        L.orc_windkessel.argtypes = [C.c_double] * 7
        L.orc_windkessel.restype = C.c_double
        L.orc_port_move.argtypes = [C.POINTER(State), C.c_int32, C.POINTER(Port), C.POINTER(Port), C.c_int32]
        L.orc_port_move.restype = C.c_int64
        L.orc_register.argtypes = [C.POINTER(State), C.POINTER(Grid), C.POINTER(Port), C.c_int32]
        L.orc_register.restype = C.c_int64
        L.orc_update.argtypes = [C.POINTER(Grid), C.POINTER(Port), C.c_int32, C.POINTER(State), C.c_int32,
                                 C.POINTER(UpdateOut)]
        L.orc_tie_margin.argtypes = [C.POINTER(State), C.POINTER(Grid), C.POINTER(Port), C.c_int32, C.c_double,
                                     C.c_void_p]
        L.orc_tie_margin.restype = C.c_double
        L.orc_update.restype = C.c_int
        L.orc_compact.argtypes = [C.POINTER(State), C.c_void_p, C.POINTER(State), C.c_void_p, C.c_int32,
                                  C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.POINTER(State),
                                  C.c_void_p, C.POINTER(C.c_int64)]
        L.orc_compact.restype = C.c_int64
        _lib = L
    return _lib


# ----------------------------------------------------------------- marshalling

FLOAT_COLS = ("x", "y", "z", "vx", "vy", "vz")


def _np(a):
    try:
        import torch
        if isinstance(a, torch.Tensor):
            return a.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(a)


def to_numpy_state(st: dict) -> dict:
    """Copy a state dict (torch or numpy) into contiguous numpy arrays."""
    out = {}
    for k, v in st.items():
        if k == "extra":
            out[k] = [np.ascontiguousarray(_np(e), dtype=np.float32) for e in v]
        elif v is None:
            continue
        else:
            dt = np.float32 if k in FLOAT_COLS else (np.int64 if k == "id" else np.int32)
            out[k] = np.ascontiguousarray(_np(v), dtype=dt).copy()
    return out


def empty_state(dim: int, n: int, n_extra: int = 0) -> dict:
    st = {c: np.zeros(n, np.float32) for c in ("x", "y", "vx", "vy")}
    if dim == 3:
        st["z"] = np.zeros(n, np.float32)
        st["vz"] = np.zeros(n, np.float32)
    st["id"] = np.zeros(n, np.int64)
    st["label"] = np.zeros(n, np.int32)
    if n_extra:
        st["extra"] = [np.zeros(n, np.float32) for _ in range(n_extra)]
    return st


class _StateRef:
    """Holds a ctypes State plus the objects it points into."""

    def __init__(self, st: dict, n: int | None = None):
        self.st = st
        self.keep = []
        s = State()
        s.n = len(st["x"]) if n is None else n
        for c in FLOAT_COLS:
            a = st.get(c)
            setattr(s, c, a.ctypes.data if a is not None else None)
        ex = st.get("extra") or []
        s.n_extra = len(ex)
        if ex:
            arr = (C.c_void_p * len(ex))(*[e.ctypes.data for e in ex])
            self.keep.append(arr)
            s.extra = C.cast(arr, C.c_void_p)
        s.id = st["id"].ctypes.data
        s.label = st["label"].ctypes.data
        self.s = s


def cgrid(g) -> Grid:
    G = Grid()
    G.dim = g.dim
    G.lo[:] = list(g.lo)
    G.cs = g.cs
    G.ncell[:] = list(g.ncell)
    G.cx_begin = g.cx_begin
    G.cx_end = g.cx_end
    return G


def cport(p) -> Port:
    P = Port()
    P.o[:] = list(p.origin)
    P.Q[:] = list(p.Q)
    P.he[:] = list(p.half_extents)
    P.kind = p.kind
    P.bc, P.rho_col = 0, -1
    bc = getattr(p, "bc", None)
    if bc is not None and bc.kind:
        P.bc = bc.kind
        P.rho_col = bc.rho_column
        # Eq. postulate-density formed in f64, rounded once to binary32
        P.rho_b = float(np.float32(float(np.float32(bc.rho0)) + float(np.float32(bc.p_b)) /
                                   (float(np.float32(bc.c0)) * float(np.float32(bc.c0)))))
        P.profile = bc.profile
        P.u0 = float(np.float32(bc.u0))
        P.R = float(np.float32(bc.radius))
        P.R2 = float(np.float32(bc.radius) * np.float32(bc.radius))
    return P


def cports(ports):
    arr = (Port * max(1, len(ports)))()
    for i, p in enumerate(ports):
        arr[i] = cport(p)
    return arr


# ----------------------------------------------------------------- API

def set_threads(n: int = 0) -> int:
    """Threads of the oracle's independent per-particle loops (0: OpenMP default);
    results do not depend on it.  Returns the count in use."""
    return int(lib().orc_set_threads(int(n)))


def frame_2d(theta: float) -> np.ndarray:
    Q = np.zeros(9)
    lib().orc_frame_2d(theta, Q.ctypes.data)
    return Q.reshape(3, 3)


def frame_3d(u) -> np.ndarray:
    Q = np.zeros(9)
    uu = np.ascontiguousarray(u, dtype=np.float64)
    if lib().orc_frame_3d(uu.ctypes.data, Q.ctypes.data) != 0:
        raise ValueError("zero axis")
    return Q.reshape(3, 3)


def to_local(port, dim, p, prec=0):
    out = np.zeros(3, np.float64 if prec else np.float32)
    P = cport(port)
    f = lib().orc_to_local_f64 if prec else lib().orc_to_local_f32
    f(C.byref(P), dim, float(p[0]), float(p[1]), float(p[2]) if len(p) > 2 else 0.0, out.ctypes.data)
    return out


def inverse_recycle(port, dim, xl):
    out = np.zeros(3)
    x = np.ascontiguousarray(xl, dtype=np.float64)
    if x.size < 3:
        x = np.concatenate([x, np.zeros(3 - x.size)])
    P = cport(port)
    lib().orc_inverse_recycle_f64(C.byref(P), dim, x.ctypes.data, out.ctypes.data)
    return out


def cell_of(grid, p):
    G = cgrid(grid)
    oob = C.c_int32(0)
    c = lib().orc_cell_of(C.byref(G), float(p[0]), float(p[1]), float(p[2]) if len(p) > 2 else 0.0, C.byref(oob))
    return int(c), int(oob.value)


def ncells(grid) -> int:
    G = cgrid(grid)
    return int(lib().orc_ncells(C.byref(G)))


def port_cells(grid, port) -> np.ndarray:
    G = cgrid(grid)
    m = np.zeros(ncells(grid), np.uint8)
    P = cport(port)
    lib().orc_port_cells(C.byref(G), C.byref(P), m.ctypes.data)
    return m


def advect(st: dict, dim: int, dt: float):
    r = _StateRef(st)
    lib().orc_advect(C.byref(r.s), dim, dt)


def fourier(t: float, a, b, omega: float) -> float:
    """Eq. Fourier_Series (Table I coefficients a0..a8, b1..b8; b[0] unused)."""
    aa = np.ascontiguousarray(a, dtype=np.float64)
    bb = np.ascontiguousarray(b, dtype=np.float64)
    return float(lib().orc_fourier(float(t), aa.ctypes.data, bb.ctypes.data, float(omega)))


def port_flux(st: dict, dim: int, port, k: int) -> int:
    """Exact 32.32 fixed-point sum of v.u over the buffer particles of port k (R26)."""
    r = _StateRef(st)
    P = cport(port)
    return int(lib().orc_port_flux(C.byref(r.s), dim, C.byref(P), k))


def windkessel(P: float, Q: float, Qprev: float, dt: float, Rp: float, Cc: float, Rd: float) -> float:
    """One explicit step of the RCR Windkessel (Eq. windkessel; reading R27)."""
    return float(lib().orc_windkessel(P, Q, Qprev, dt, Rp, Cc, Rd))


def port_move(st: dict, dim: int, port_from, port_to, k: int) -> int:
    """Moving port (rotating sprinkler): the buffer particles of port k keep
    their local coordinates and velocities from frame ``port_from`` to ``port_to``."""
    r = _StateRef(st)
    A, B = cport(port_from), cport(port_to)
    return int(lib().orc_port_move(C.byref(r.s), dim, C.byref(A), C.byref(B), k))


# ----------------------------------------------------------------- O7 tie check

_TIE_TAU_DP = None           # None: off; else every register/update certifies margins


_TIE_COLLECT = None          # a list: collect the offending ids instead of raising


class TieError(AssertionError):
    """An input violates the north_star tie margin (a particle within 1e-4 dp of a
    threshold at a decision or relabel point): such an input is invalid.
    ``ids`` holds the ids of the offending particles."""

    def __init__(self, msg, ids=()):
        super().__init__(msg)
        self.ids = list(ids)


def enable_tie_check(tau_dp: float | None = 1e-4):
    """Make every ``register`` and ``update`` certify that no particle is within
    tau_dp * dp of a threshold face (O7) at the registration point, the decision
    point (the state passed to ``update``) and the relabel point (its survivors
    after the update); dp = a / layers of the ports.  None switches it off."""
    global _TIE_TAU_DP
    _TIE_TAU_DP = tau_dp


class collect_ties:
    """Context manager: inside, the tie check appends the offending ids to
    ``self.ids`` instead of raising (used to screen a test's own dynamics)."""

    def __enter__(self):
        global _TIE_COLLECT, _TIE_TAU_DP
        self.saved = (_TIE_COLLECT, _TIE_TAU_DP)
        self.ids = []
        _TIE_COLLECT = self.ids
        if _TIE_TAU_DP is None:
            _TIE_TAU_DP = 1e-4
        return self

    def __exit__(self, *a):
        global _TIE_COLLECT, _TIE_TAU_DP
        _TIE_COLLECT, _TIE_TAU_DP = self.saved


class no_tie_check:
    """Context manager for pins that put particles exactly on a threshold on purpose
    (strict-inequality checks): the tie check is off inside."""

    def __enter__(self):
        global _TIE_TAU_DP
        self.saved, _TIE_TAU_DP = _TIE_TAU_DP, None

    def __exit__(self, *a):
        global _TIE_TAU_DP
        _TIE_TAU_DP = self.saved


def _port_dp(ports):
    dps = [2.0 * float(p.half_extents[0]) / p.layers for p in ports if getattr(p, "layers", 0)]
    return min(dps) if dps else None


def _certify(st, grid, ports, what):
    if _TIE_TAU_DP is None or not ports or len(st["x"]) == 0:
        return
    dp = _port_dp(ports)
    if dp is None:
        return
    m, bad = tie_margin(st, grid, ports, _TIE_TAU_DP * dp)
    if len(bad):
        ids = st["id"][bad].tolist()
        if _TIE_COLLECT is not None:
            _TIE_COLLECT.extend(ids)
            return
        raise TieError(f"{what}: {len(bad)} particles within {_TIE_TAU_DP:g} dp of a threshold "
                       f"(min margin {m / dp:.3g} dp; first ids {ids[:5]})", ids)


def register(st: dict, grid, port, k: int) -> int:
    """O0: Alg. 1 identification / initial relabel of port k (f64 decisions)."""
    _certify(st, grid, [port], f"registration of port {k}")
    r = _StateRef(st)
    G = cgrid(grid)
    P = cport(port)
    return int(lib().orc_register(C.byref(r.s), C.byref(G), C.byref(P), k))


def tie_margin(st: dict, grid, ports, tau: float):
    """O7: minimum f64 distance of any particle near a port to a threshold face of
    InBox_k or P_k (sph_oracle.c orc_tie_margin), and the indices of the particles
    closer than ``tau``.  Returns (min_margin, flagged_indices)."""
    n = len(st["x"])
    flags = np.zeros(max(n, 1), np.uint8)
    r = _StateRef(st)
    G = cgrid(grid)
    P = cports(ports)
    m = lib().orc_tie_margin(C.byref(r.s), C.byref(G), P, len(ports), float(tau), flags.ctypes.data)
    return float(m), np.nonzero(flags[:n])[0]


@dataclass
class UpdateResult:
    order: np.ndarray
    cell_start: np.ndarray
    cell_end: np.ndarray
    out_of_grid: int
    create_port: np.ndarray
    delete_port: np.ndarray
    sorted: dict
    staged: dict
    stage_port: np.ndarray
    stage_src: np.ndarray
    port_counts: np.ndarray     # [2K]: created at [k], deleted at [K+k]
    checked: int
    multi_decision: int
    motion_errors: int
    t_cll: float = 0.0          # seconds in O2 (cell list)
    t_decide: float = 0.0       # seconds in O3-O5b (decide, apply, relabel, BC)


def update(grid, ports, st: dict, mode: int = 0, cap_stage: int | None = None,
           rho_b: dict | None = None) -> UpdateResult:
    """O2-O5 on one slab: cell list, f64 decisions, duplicate + recycle, relabel.
    rho_b: {port: recycled density} overriding the pressure BC's (a Windkessel driver)."""
    dim = grid.dim
    n = len(st["x"])
    K = len(ports)
    nc = ncells(grid)
    n_extra = len(st.get("extra") or [])
    cap = cap_stage if cap_stage is not None else max(16, n)
    o = UpdateOut()
    order = np.zeros(max(n, 1), np.int64)
    cstart = np.zeros(max(nc, 1), np.int32)
    cend = np.zeros(max(nc, 1), np.int32)
    cport_ = np.zeros(max(n, 1), np.int32)
    dport = np.zeros(max(n, 1), np.int32)
    srt = empty_state(dim, max(n, 1), n_extra)
    stg = empty_state(dim, cap, n_extra)
    sport = np.zeros(cap, np.int32)
    ssrc = np.zeros(cap, np.int64)
    counts = np.zeros(max(2 * K, 1), np.int32)
    o.order, o.cell_start, o.cell_end = order.ctypes.data, cstart.ctypes.data, cend.ctypes.data
    o.create_port, o.delete_port = cport_.ctypes.data, dport.ctypes.data
    rs, rg = _StateRef(srt, n), _StateRef(stg, 0)
    o.sorted, o.staged = rs.s, rg.s
    o.stage_port, o.stage_src = sport.ctypes.data, ssrc.ctypes.data
    o.cap_stage = cap
    o.port_counts = counts.ctypes.data
    ri = _StateRef(st)
    G = cgrid(grid)
    P = cports(ports)
    for k, v in (rho_b or {}).items():
        P[k].rho_b = float(v)
    _certify(st, grid, ports, "decision point")
    rc = lib().orc_update(C.byref(G), P, K, C.byref(ri.s), mode, C.byref(o))
    if rc != 0:
        raise RuntimeError("oracle staging overflow")
    ns = int(o.n_stage)
    trim = lambda d, m: {k: ([e[:m] for e in v] if k == "extra" else v[:m]) for k, v in d.items()}
    if _TIE_TAU_DP is not None and K:
        keep = dport[:n] < 0
        _certify({c: v[:n][keep] for c, v in srt.items() if c != "extra"}, grid, ports, "relabel point")
    return UpdateResult(order[:n], cstart[:nc], cend[:nc], int(o.out_of_grid), cport_[:n], dport[:n],
                        trim(srt, n), trim(stg, ns), sport[:ns], ssrc[:ns], counts[:2 * K], int(o.checked),
                        int(o.multi_decision), int(o.motion_errors), float(o.t_cll), float(o.t_decide))


def compact(res: UpdateResult, dim: int, K: int, all_counts: np.ndarray, rank: int, next_id: int):
    """O6: stable compaction + append + ID assignment from the count matrix.
    all_counts: int32 [nranks, 2K] (created at [:, k], deleted at [:, K+k]).
    Returns (state, perm, next_id_after)."""
    n = len(res.sorted["x"])
    ns = len(res.staged["x"])
    n_extra = len(res.sorted.get("extra") or [])
    out = empty_state(dim, max(n + ns, 1), n_extra)
    perm = np.zeros(max(n, 1), np.int64)
    ac = np.ascontiguousarray(all_counts, dtype=np.int32)
    nranks = ac.shape[0]
    rs, rg, ro = _StateRef(res.sorted), _StateRef(res.staged), _StateRef(out)
    nid = C.c_int64(0)
    m = lib().orc_compact(C.byref(rs.s), res.delete_port.ctypes.data, C.byref(rg.s), res.stage_port.ctypes.data,
                          dim, ac.ctypes.data, nranks, rank, K, next_id, C.byref(ro.s), perm.ctypes.data,
                          C.byref(nid))
    m = int(m)
    st = {k: ([e[:m] for e in v] if k == "extra" else v[:m]) for k, v in out.items()}
    return st, perm[:n], int(nid.value)


def step(st: dict, grid, ports, next_id: int, dt: float | None, mode: int = 0):
    """One single-slab update: (advect) -> O2..O5 -> O6 with a 1-rank count matrix.
    Returns (new_state, UpdateResult, perm, next_id_after).  ``st`` is advected in place."""
    if dt is not None:
        advect(st, grid.dim, dt)
    res = update(grid, ports, st, mode)
    new, perm, nid = compact(res, grid.dim, len(ports), res.port_counts[None, :], 0, next_id)
    return new, res, perm, nid
