"""Seeded synthetic inputs for the in/outlet buffer update (arXiv 2406.16786).

This module is the ONLY code shared by the CUDA path and the CPU oracle
(``oracle/``).  It builds particle lattices, velocity fields, port frames and
grids shaped like the paper's workloads (DESIGN.md §4 "Input recipe"); it holds
none of the method's arithmetic (no local-frame decisions, no cell lists, no
generation/deletion).  Input shaping that needs geometry (pre-clearing an
upstream column, projecting the lateral velocity near a port) is written here
with its own plain torch expressions and is not the method: the method never
pre-clears or projects.

Configs (BASELINE.json ``configs``):

* ``C1``  2-D orthogonal channel, 8,000 particles, 1 update at dt=0.002.
* ``C1e`` C1 with dt=0.0095 (reading R18: C1 as written has no events).
* ``C2``  2-D 30-degree channel with a 45-degree slanted end, ~200k particles,
          two bidirectional ports (inflow normals at 30 and 255 degrees).
* ``C3``  3-D square duct 1.0x0.2x0.2, 2.56M particles.
* ``C4``  3-D 1.6x0.8x0.8 junction, 65.5M particles, 8 random ports.
* ``C5``  3-D weak-scaling slabs, 128M particles per slab, 8 ports per slab.

``scale`` < 1 shrinks C3/C4/C5 boxes (for CPU-sized parity cases).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

INLET, OUTLET, BIDIRECTIONAL = 0, 1, 2
SEED_BASE = 240616786


def f32(v: float) -> float:
    """Round a python float to the nearest binary32 value."""
    return float(np.float32(v))


BC_NONE, BC_PRESSURE, BC_VELOCITY = 0, 1, 2
PROFILE_PLUG, PROFILE_PARABOLIC, PROFILE_PARABOLIC_RADIAL = 0, 1, 2


@dataclass
class BC:
    """Boundary-condition parameters of a port (paper §IV), as plain data."""
    kind: int = BC_NONE
    rho0: float = 1.0
    c0: float = 10.0
    p_b: float = 0.0
    rho_column: int = -1
    profile: int = PROFILE_PLUG
    u0: float = 1.0
    radius: float = 1.0


DRIVER_NONE, DRIVER_FOURIER, DRIVER_WINDKESSEL = 0, 1, 2

# Table I: Fourier coefficients of the aortic inflow speed; the
# duplicated label "b_7" of the last row is read as b_8.
TABLE_I_A = (0.3782, -0.1812, 0.1276, -0.08981, 0.04347, -0.05412, 0.02642, 0.008946, -0.009005)
TABLE_I_B = (0.0, -0.07725, 0.01466, 0.04295, -0.06679, 0.05679, -0.01878, 0.01869, -0.01888)
TABLE_I_OMEGA = 8.302
# Table II: RCR Windkessel parameters, CGS units (dyn s/cm^5, cm^5/dyn)
TABLE_II = {"right common carotid": (1180.0, 7.70e-5, 18400.0), "right subclavian": (1040.0, 8.74e-5, 16300.0),
            "left common carotid": (1180.0, 7.70e-5, 18400.0), "left subclavian": (970.0, 9.34e-5, 15200.0),
            "descending aorta": (188.0, 4.82e-4, 2950.0)}
DYN_S_CM5 = 1e5              # 1 dyn s/cm^5 = 1e5 Pa s/m^3
CM5_DYN = 1e-5               # 1 cm^5/dyn = 1e-5 m^3/Pa


def windkessel_si(vessel: str) -> tuple:
    """(Rp, C, Rd) of a Table II vessel in SI units."""
    Rp, Cc, Rd = TABLE_II[vessel]
    return Rp * DYN_S_CM5, Cc * CM5_DYN, Rd * DYN_S_CM5


@dataclass
class Driver:
    """Time-dependent port driver (aorta flow, §V.D), as plain data."""
    kind: int = DRIVER_NONE
    a: tuple = (0.0,) * 9
    b: tuple = (0.0,) * 9
    omega: float = 0.0
    Rp: float = 0.0
    C: float = 0.0
    Rd: float = 0.0
    P0: float = 0.0
    volume: float = 0.0


@dataclass
class Port:
    origin: tuple            # O' (global), binary32 values
    Q: tuple                 # 9 values row-major; rows = local axes (row 0 = u, the in/outflow axis)
    half_extents: tuple      # (a/2, b/2, c/2)
    kind: int                # INLET / OUTLET / BIDIRECTIONAL
    layers: int
    bc: BC = None            # optional boundary condition of its buffer particles
    driver: Driver = None    # optional time-dependent driver of that boundary condition


@dataclass
class Grid:
    dim: int
    lo: tuple                # 3 binary32 values
    cs: float                # binary32 cell size
    ncell: tuple             # global cell counts (nz = 1 in 2-D)
    cx_begin: int = 0
    cx_end: int = -1         # -1 -> ncell[0]

    def __post_init__(self):
        if self.cx_end < 0:
            self.cx_end = self.ncell[0]

    def slab(self, cx_begin: int, cx_end: int) -> "Grid":
        return Grid(self.dim, self.lo, self.cs, self.ncell, cx_begin, cx_end)

    @property
    def ncells_local(self) -> int:
        return (self.cx_end - self.cx_begin) * self.ncell[1] * (self.ncell[2] if self.dim == 3 else 1)


@dataclass
class Workload:
    name: str
    dim: int
    dp: float
    h: float
    grid: Grid
    ports: list
    state: dict              # x,y,(z),vx,vy,(vz): float32; id: int64; label: int32 (all -1)
    dt: float
    n_updates: int
    next_id: int
    notes: str = ""
    slab_cells: list = field(default_factory=list)   # per-slab [cx_begin, cx_end) for C5
    redrawn: int = 0         # particles whose jitter the tie screen re-drew

    @property
    def n(self) -> int:
        return int(self.state["x"].numel())


# ----------------------------------------------------------------- helpers

def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def _noise(n, g, device, sigma=0.05):
    """N(0, sigma^2) per component, clipped at +-4 sigma (reading R17)."""
    z = torch.randn(n, generator=g, device=device, dtype=torch.float32) * sigma
    return z.clamp_(-4 * sigma, 4 * sigma).double()


def _jitter(n, g, device, dp):
    return (torch.rand(n, generator=g, device=device, dtype=torch.float32).double() * 2.0 - 1.0) * (0.1 * dp)


def frame_rows_2d(theta: float) -> tuple:
    """Rows [cos t, sin t], [-sin t, cos t] as in the paper's 2-D frame; input data only."""
    c, s = math.cos(theta), math.sin(theta)
    return tuple(f32(v) for v in (c, s, 0.0, -s, c, 0.0, 0.0, 0.0, 1.0))


def frame_rows_3d(u, psi: float) -> tuple:
    """A random right-handed orthonormal frame with row 0 = u and roll psi about u
    (Gram-Schmidt; C4/C5 draw the roll, reading R3)."""
    u = np.asarray(u, dtype=np.float64)
    u = u / np.linalg.norm(u)
    e = np.zeros(3)
    e[int(np.argmin(np.abs(u)))] = 1.0
    t0 = e - np.dot(e, u) * u
    t0 /= np.linalg.norm(t0)
    b0 = np.cross(u, t0)
    t = math.cos(psi) * t0 + math.sin(psi) * b0
    w = np.cross(u, t)
    return tuple(f32(v) for v in np.concatenate([u, t, w]))


def _port(origin, Q, he, kind, layers) -> Port:
    return Port(tuple(f32(v) for v in origin), tuple(Q), tuple(f32(v) for v in he), kind, layers)


def _local(xyz: list, port: Port, dim: int):
    """f64 local coordinates, used only for input shaping (pre-clear, projection)."""
    Q = torch.tensor(port.Q, dtype=torch.float64, device=xyz[0].device).view(3, 3)
    d = [xyz[j] - port.origin[j] for j in range(dim)]
    return [sum(Q[r, j] * d[j] for j in range(dim)) for r in range(dim)]


def _project_near_ports(xyz, v, ports, dim, radius_pad):
    """Within each port's bounding sphere, keep only the axial velocity
    (v <- (v.u)u) so buffer particles stay laterally inside their box
    (reading R17; input shaping, the same projection as Eq. velocity_correction)."""
    for p in ports:
        r = math.sqrt(sum(h * h for h in p.half_extents[:dim])) + radius_pad
        d2 = sum((xyz[j] - p.origin[j]) ** 2 for j in range(dim))
        near = d2 < r * r
        if not bool(near.any()):
            continue
        u = p.Q[0:3]
        vu = sum(v[j] * u[j] for j in range(dim))
        for j in range(dim):
            v[j] = torch.where(near, vu * u[j], v[j])
    return v


def _pack_state(xyz, v, ids, dim):
    st = {"x": xyz[0].float().contiguous(), "y": xyz[1].float().contiguous()}
    st["vx"] = v[0].float().contiguous()
    st["vy"] = v[1].float().contiguous()
    if dim == 3:
        st["z"] = xyz[2].float().contiguous()
        st["vz"] = v[2].float().contiguous()
    st["id"] = ids.to(torch.int64).contiguous()
    st["label"] = torch.full_like(st["id"], -1, dtype=torch.int32)
    return st


def _lattice(counts, dp, device, origin=(0.0, 0.0, 0.0), index_offset=0):
    """Cell-centred lattice ((i+1/2)dp), ids in lattice order with x slowest."""
    n = 1
    for c in counts:
        n *= c
    idx = torch.arange(n, device=device, dtype=torch.int64)
    comps = []
    rem = idx
    strides = []
    s = 1
    for c in reversed(counts):
        strides.append(s)
        s *= c
    strides = list(reversed(strides))
    for a, c in enumerate(counts):
        ia = (rem // strides[a]) % c
        comps.append((ia.double() + 0.5) * dp + origin[a])
    return comps, idx + index_offset


# ----------------------------------------------------------------- tie screen

TIE_TAU_DP = 1e-4            # north_star: every particle >= 1e-4 dp from any threshold
_SCREEN_GUARD = 1.1          # the screen flags at 1.1 tau (the oracle certifies tau, O7)


def _local64(xs, port, dim):
    """f64 local coordinates Q (x - o) of fp32 positions (input validation only)."""
    d = [xs[j].double() - float(port.origin[j]) for j in range(dim)]
    out = []
    for r in range(dim):
        acc = None
        for j in range(dim):
            t = float(port.Q[3 * r + j]) * d[j]
            acc = t if acc is None else acc + t
        out.append(acc)
    return out


def _near_faces(X, port, dim, cs, tau):
    """(inside P_k inflated by tau, some local coordinate within tau of a face value
    he_r or he_r + m) for f64 local coordinates X."""
    near = None
    close = None
    for r in range(dim):
        a = X[r].abs()
        he = float(port.half_extents[r])
        nr = a < he + cs + tau
        cr = ((a - he).abs() < tau) | ((a - (he + cs)).abs() < tau)
        near = nr if near is None else near & nr
        close = cr if close is None else close | cr
    return near & close


def _tie_flags(x32, v32, ports, dim, cs, dt, n_updates, tau):
    """Flag the particles (fp32 positions x32, velocities v32: lists of tensors) that
    come within tau of a threshold face of InBox_k or P_k of any port over the run.

    Kinematic model of the run (no decisions are taken here): each particle's
    pinned fp32 free flight x <- fl(x + fl(v dt)) (the advection driver); and,
    every time a trajectory crosses the plane X'_0 = +a/2 of an inlet or
    bidirectional port forward inside its P_k, an extra trajectory starting from
    the position shifted back by one buffer length, fl(x - fl(a u)) (a recycled
    buffer particle), which is followed the same way.  Deletions and
    labels are ignored, so the set of positions covers every position the
    particle and its duplicates/recycled copies can take (a superset: more
    redraws, never a missed tie).  Positions are checked at registration (step 0),
    after every advection (decision points) and where a recycled copy starts
    (relabel point)."""
    dev = x32[0].device
    n = x32[0].numel()
    flag = torch.zeros(n, dtype=torch.bool, device=dev)
    if n == 0 or not ports:
        return flag
    dt32 = torch.tensor(dt, dtype=torch.float32, device=dev)
    slack = 0.05 * cs
    # preselect (particle, port) pairs whose straight path comes near P_k
    sel = []
    xe = [x32[j].double() + float(n_updates) * float(dt) * v32[j].double() for j in range(dim)]
    for p in ports:
        X0 = _local64(x32, p, dim)
        Xe = _local64(xe, p, dim)
        m = None
        for r in range(dim):
            R = float(p.half_extents[r]) + cs + tau + slack
            mr = (torch.minimum(X0[r], Xe[r]) < R) & (torch.maximum(X0[r], Xe[r]) > -R)
            m = mr if m is None else m & mr
        sel.append(m)
    anyp = torch.zeros(n, dtype=torch.bool, device=dev)
    for m in sel:
        anyp |= m
    org = torch.nonzero(anyp).squeeze(1)                   # origin of every trajectory
    if org.numel() == 0:
        return flag
    pos = [x32[j][org].clone() for j in range(dim)]
    vel = [v32[j][org].clone() for j in range(dim)]
    shift = []
    for p in ports:
        a = np.float32(2.0) * np.float32(p.half_extents[0])
        shift.append([float(np.float32(a * np.float32(p.Q[j]))) for j in range(dim)])

    def check(tr_pos, tr_org):
        for k, p in enumerate(ports):
            on = sel[k][tr_org]
            if not bool(on.any()):
                continue
            idx = torch.nonzero(on).squeeze(1)
            X = _local64([c[idx] for c in tr_pos], p, dim)
            bad = _near_faces(X, p, dim, cs, tau)
            flag[tr_org[idx[bad]]] = True

    check(pos, org)
    for _ in range(n_updates):
        prev = pos
        pos = [prev[j] + vel[j] * dt32 for j in range(dim)]
        check(pos, org)
        new_pos, new_vel, new_org = [], [], []
        for k, p in enumerate(ports):
            if p.kind == OUTLET:
                continue
            on = torch.nonzero(sel[k][org]).squeeze(1)
            if on.numel() == 0:
                continue
            X = _local64([c[on] for c in pos], p, dim)
            Xp = _local64([c[on] for c in prev], p, dim)[0]
            inP = None
            for r in range(dim):
                t = X[r].abs() < float(p.half_extents[r]) + cs
                inP = t if inP is None else inP & t
            he0 = float(p.half_extents[0])
            cross = inP & (X[0] > he0) & (Xp <= he0)
            if not bool(cross.any()):
                continue
            ci = on[cross]
            new_pos.append([pos[j][ci] - torch.tensor(shift[k][j], dtype=torch.float32, device=dev)
                            for j in range(dim)])
            new_vel.append([vel[j][ci] for j in range(dim)])
            new_org.append(org[ci])
        if new_org:
            bp = [torch.cat([q[j] for q in new_pos]) for j in range(dim)]
            bv = [torch.cat([q[j] for q in new_vel]) for j in range(dim)]
            bo = torch.cat(new_org)
            check(bp, bo)
            pos = [torch.cat([pos[j], bp[j]]) for j in range(dim)]
            vel = [torch.cat([vel[j], bv[j]]) for j in range(dim)]
            org = torch.cat([org, bo])
    return flag


def _hash_jitter(ids, attempt: int, comp: int, salt: int, dp: float):
    """Counter-based uniform draw in [-0.1 dp, 0.1 dp) for re-drawn particles
    (splitmix64 of (salt, id, attempt, component)); identical on every device."""
    with np.errstate(over="ignore"):
        z = (ids.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)
             + np.uint64(attempt) * np.uint64(0xD1B54A32D192ED03)
             + np.uint64(comp) * np.uint64(0x8CB92BA72F3D8DD7)
             + np.uint64(salt))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return (u * 2.0 - 1.0) * (0.1 * dp)


def _screen(base, xyz, vel_fn, ids, ports, dim, dp, cs, dt, n_updates, salt, max_rounds=40):
    """Tie screen (north_star; SURVEY §8(d) "Tie-screen"): re-draw the jitter (and
    recompute the velocity) of every particle that comes within 1e-4 dp of a
    threshold over the run, until none does.  base: lattice sites (f64), xyz:
    jittered positions (f64, modified in place), vel_fn(xyz_subset, index_subset)
    -> velocity (f64 list).  Returns (xyz, v, number of re-drawn particles)."""
    tau = _SCREEN_GUARD * TIE_TAU_DP * dp
    v = vel_fn(xyz, None)
    sub = None
    redrawn = set()
    ids_np = ids.cpu().numpy()
    for attempt in range(1, max_rounds + 1):
        xs = [c if sub is None else c[sub] for c in xyz]
        vs = [c if sub is None else c[sub] for c in v]
        bad = _tie_flags([c.float() for c in xs], [c.float() for c in vs], ports, dim, cs, dt, n_updates, tau)
        idx = torch.nonzero(bad).squeeze(1)
        if sub is not None:
            idx = sub[idx]
        if idx.numel() == 0:
            return xyz, v, len(redrawn)
        ii = ids_np[idx.cpu().numpy()]
        redrawn.update(int(i) for i in ii)
        for j in range(dim):
            jit = torch.from_numpy(_hash_jitter(ii, attempt, j, salt, dp)).to(xyz[j].device)
            xyz[j][idx] = base[j][idx] + jit
        vn = vel_fn([c[idx] for c in xyz], idx)
        for j in range(dim):
            v[j][idx] = vn[j]
        sub = idx
    raise RuntimeError("tie screen did not converge")


def nudge(w: "Workload", nudges: dict, salt: int = 0x5EED) -> "Workload":
    """Move the particles whose id is a key of ``nudges`` (id -> attempt) by a
    counter-based offset of up to +-0.05 dp per component (tests/tiescreen.py:
    tie screen of a test's own dynamics).  Velocities and every other particle are
    unchanged.  In place; returns w."""
    if not nudges:
        return w
    st = w.state
    ids = st["id"].cpu().numpy()
    want = np.fromiter(nudges.keys(), dtype=np.int64)
    att = np.fromiter(nudges.values(), dtype=np.int64)
    pos = np.nonzero(np.isin(ids, want))[0]
    if pos.size == 0:
        return w
    order = {int(i): int(a) for i, a in zip(want, att)}
    a_of = np.array([order[int(i)] for i in ids[pos]], dtype=np.int64)
    idx = torch.from_numpy(pos).to(st["x"].device)
    for j, c in enumerate(("x", "y", "z")[:w.dim]):
        off = np.empty(pos.size)
        for a in np.unique(a_of):
            m = a_of == a
            off[m] = 0.5 * _hash_jitter(ids[pos[m]], 1000 + int(a), j, salt, w.dp)
        col = st[c]
        col[idx] = (col[idx].double() + torch.from_numpy(off).to(col.device)).float()
    return w


# ----------------------------------------------------------------- configs

def c1(device="cpu", dt=0.002, name="C1", n_updates=20) -> Workload:
    """2-D orthogonal channel 2.0x0.4 at dp=0.01 (BASELINE configs[0]).
    ``n_updates`` only sets the tie screen's horizon (the config is one update;
    the tests run up to 20)."""
    dim, dp = 2, 0.01
    h = 1.3 * dp
    cs = f32(2 * h)
    g = _gen(SEED_BASE + 1, device)
    base, ids = _lattice((200, 40), dp, device)
    n = ids.numel()
    xyz = [base[j] + _jitter(n, g, device, dp) for j in range(dim)]
    noise = [_noise(n, g, device), _noise(n, g, device)]
    I = (1.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0)
    ports = [_port((0.02, 0.2, 0.0), I, (0.02, 0.2, 0.0), INLET, 4),
             _port((1.98, 0.2, 0.0), I, (0.02, 0.2, 0.0), OUTLET, 4)]

    def vel(x, idx):
        nz = [c if idx is None else c[idx] for c in noise]
        return _project_near_ports(x, [1.0 + nz[0], nz[1]], ports[:1], dim, 2 * dp)
    xyz, v, nre = _screen(base, xyz, vel, ids, ports, dim, dp, cs, f32(dt), n_updates, SEED_BASE + 1)
    lo = (f32(-2 * cs), f32(-2 * cs), 0.0)
    ncell = (int(math.ceil(2.0 / cs)) + 4, int(math.ceil(0.4 / cs)) + 4, 1)
    grid = Grid(dim, lo, cs, ncell)
    return Workload(name, dim, dp, h, grid, ports, _pack_state(xyz, v, ids, dim), f32(dt), 1, n,
                    notes=f"200x40 lattice; inlet x in (0,0.04), outlet x in (1.96,2.0); {nre} re-drawn",
                    redrawn=nre)


def c1e(device="cpu", n_updates=20) -> Workload:
    """C1 with dt=0.0095: exactly the last lattice layer crosses at each end (R18)."""
    return c1(device, dt=0.0095, name="C1e", n_updates=n_updates)


def c2(device="cpu", n_updates=100) -> Workload:
    """2-D channel rotated 30 degrees, end face slanted 45 degrees; both ports bidirectional."""
    dim, dp = 2, 0.002
    h = 1.3 * dp
    cs = f32(2 * h)
    g = _gen(SEED_BASE + 2, device)
    (s, w), _ = _lattice((1100, 200), dp, device, origin=(0.0, -0.2))
    c45 = math.cos(math.pi / 4)
    keep = (s - 2.0) * c45 + w * c45 < 0
    s, w = s[keep], w[keep]
    n = s.numel()
    ids = torch.arange(n, device=device, dtype=torch.int64)
    th = math.radians(30.0)
    X = math.cos(th) * s - math.sin(th) * w
    Y = math.sin(th) * s + math.cos(th) * w
    base = [X, Y]
    xyz = [X + _jitter(n, g, device, dp), Y + _jitter(n, g, device, dp)]
    u0 = (math.cos(th), math.sin(th))
    nrm = (math.cos(math.radians(75.0)), math.sin(math.radians(75.0)))
    end = (2.0 * math.cos(th), 2.0 * math.sin(th))
    p0 = _port((0.004 * u0[0], 0.004 * u0[1], 0.0), frame_rows_2d(th), (0.004, 0.2, 0.0), BIDIRECTIONAL, 4)
    p1 = _port((end[0] - 0.004 * nrm[0], end[1] - 0.004 * nrm[1], 0.0), frame_rows_2d(math.radians(255.0)),
               (0.004, 0.2 / c45, 0.0), BIDIRECTIONAL, 4)
    ports = [p0, p1]
    noise = [_noise(n, g, device), _noise(n, g, device)]

    def vel(x, idx):
        # nearest port k, sigma = +1 where Y'_k > 0 else -1 ("sign flipping per region")
        m = x[0].numel()
        d0 = (x[0] - p0.origin[0]) ** 2 + (x[1] - p0.origin[1]) ** 2
        d1 = (x[0] - p1.origin[0]) ** 2 + (x[1] - p1.origin[1]) ** 2
        near1 = d1 < d0
        v = [torch.zeros(m, dtype=torch.float64, device=device) for _ in range(2)]
        for k, p in enumerate(ports):
            sel = near1 if k == 1 else ~near1
            yl = _local(x, p, dim)[1]
            sig = torch.where(yl > 0, 1.0, -1.0)
            for j in range(2):
                v[j] = torch.where(sel, sig * p.Q[j], v[j])
        nz = [c if idx is None else c[idx] for c in noise]
        v = [v[0] + nz[0], v[1] + nz[1]]
        return _project_near_ports(x, v, ports, dim, 2 * dp)
    xyz, v, nre = _screen(base, xyz, vel, ids, ports, dim, dp, cs, f32(0.0005), n_updates, SEED_BASE + 2)
    xs, ys = xyz[0], xyz[1]
    pad = 12
    lo = (f32(float(xs.min()) - pad * cs), f32(float(ys.min()) - pad * cs), 0.0)
    ncell = (int(math.ceil((float(xs.max()) - lo[0]) / cs)) + pad, int(math.ceil((float(ys.max()) - lo[1]) / cs)) + pad, 1)
    grid = Grid(dim, lo, cs, ncell)
    return Workload("C2", dim, dp, h, grid, ports, _pack_state(xyz, v, ids, dim), f32(0.0005), n_updates, n,
                    notes=f"30-degree channel, 45-degree slanted end; bidirectional ports at 30 and 255 degrees; "
                          f"{nre} re-drawn", redrawn=nre)


def c3(device="cpu", n_updates=100, scale=1.0) -> Workload:
    """3-D square duct 1.0x0.2x0.2 at dp=0.0025 (2.56M particles at scale 1)."""
    dim, dp = 3, 0.0025
    h = 1.3 * dp
    L = 1.0 * scale
    nx = int(round(400 * scale))
    cs = f32(1.0 / 153.0)
    g = _gen(SEED_BASE + 3, device)
    base, ids = _lattice((nx, 80, 80), dp, device)
    n = ids.numel()
    xyz = [base[j] + _jitter(n, g, device, dp) for j in range(3)]
    noise = [_noise(n, g, device), _noise(n, g, device), _noise(n, g, device)]
    I = (1.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0)
    ports = [_port((0.005, 0.1, 0.1), I, (0.005, 0.1, 0.1), INLET, 4),
             _port((nx * dp - 0.005, 0.1, 0.1), I, (0.005, 0.1, 0.1), OUTLET, 4)]

    def vel(x, idx):
        nz = [c if idx is None else c[idx] for c in noise]
        return _project_near_ports(x, [1.0 + nz[0], nz[1], nz[2]], ports[:1], dim, 2 * dp)
    xyz, v, nre = _screen(base, xyz, vel, ids, ports, dim, dp, cs, f32(0.0002), n_updates, SEED_BASE + 3)
    pad = 4
    lo = (f32(-pad * cs),) * 3
    ncell = (int(math.ceil(L / cs)) + 2 * pad, int(math.ceil(0.2 / cs)) + 2 * pad, int(math.ceil(0.2 / cs)) + 2 * pad)
    grid = Grid(dim, lo, cs, ncell)
    return Workload("C3" if scale == 1.0 else f"C3x{scale:g}", dim, dp, h, grid, ports,
                    _pack_state(xyz, v, ids, dim), f32(0.0002), n_updates, n,
                    notes=f"{nx}x80x80 lattice duct; inlet x in (0,0.01), outlet at x={nx * dp:g}; {nre} re-drawn",
                    redrawn=nre)


def _draw_ports(rng, nports, box_lo, box_hi, dp, cs, steps, dt, existing, x_margin_lo=True, x_margin_hi=True,
                bc_range=(0.1, 0.2)):
    """Random ports: u ~ normalise(N(0,I)), roll ~ U[0,2pi), b,c ~ U[bc_range],
    he = (2dp, b/2, c/2), 4 layers; even index inlet, odd outlet.  Origins are
    rejection-sampled so that bounding spheres (inflated by the inlet pre-clear
    length) stay 2 cells apart and inside the box (margin only on the faces asked)."""
    ports, radii = [], []
    prior = list(existing)
    Lpre = 1.25 * steps * dt + cs
    for k in range(nports):
        kind = INLET if k % 2 == 0 else OUTLET
        for _ in range(10000):
            u = rng.standard_normal(3)
            u /= np.linalg.norm(u)
            psi = rng.uniform(0.0, 2 * math.pi)
            b, c = rng.uniform(*bc_range, size=2)
            he = (2 * dp, b / 2, c / 2)
            r = math.sqrt((he[0] + cs) ** 2 + (he[1] + cs) ** 2 + (he[2] + cs) ** 2)
            if kind == INLET:
                r = r + Lpre
            lo = [box_lo[j] + r + 2 * cs for j in range(3)]
            hi = [box_hi[j] - r - 2 * cs for j in range(3)]
            if not x_margin_lo:
                lo[0] = box_lo[0]
            if not x_margin_hi:
                hi[0] = box_hi[0]
            if any(hi[j] <= lo[j] for j in range(3)):
                continue
            o = np.array([rng.uniform(lo[j], hi[j]) for j in range(3)])
            if all(np.linalg.norm(o - q[0]) > r + q[1] + 2 * cs for q in prior):
                ports.append(_port(tuple(o), frame_rows_3d(u, psi), he, kind, 4))
                radii.append(r)
                prior.append((o, r))
                break
        else:
            raise RuntimeError("could not place port")
    return ports, prior[len(existing):]


def _preclear(xyz, ports, dp, cs, steps, dt):
    """Remove each inlet's upstream column {-a/2-L < X' < -a/2, lateral in box}
    and each outlet's downstream strip {a/2 < X' < a/2+m, lateral within he+m},
    L = 1.25 steps dt + m, so step 1 has no deletion burst (input shaping)."""
    keep = torch.ones_like(xyz[0], dtype=torch.bool)
    Lpre = 1.25 * steps * dt + cs
    for p in ports:
        r = math.sqrt(sum((h + cs) ** 2 for h in p.half_extents)) + (Lpre if p.kind == INLET else 0.0)
        d2 = sum((xyz[j] - p.origin[j]) ** 2 for j in range(3))
        near = d2 < r * r
        idx = torch.nonzero(near).squeeze(1)
        if idx.numel() == 0:
            continue
        sub = [xyz[j][idx] for j in range(3)]
        X = _local(sub, p, 3)
        a2, b2, c2_ = p.half_extents
        if p.kind == INLET:
            rm = (X[0] < -a2) & (X[0] > -a2 - Lpre) & (X[1].abs() < b2) & (X[2].abs() < c2_)
        else:
            rm = (X[0] > a2) & (X[0] < a2 + cs) & (X[1].abs() < b2 + cs) & (X[2].abs() < c2_ + cs)
        keep[idx[rm]] = False
    return keep


def _nearest_port_velocity(xyz, ports, noise, dp):
    """v = u of the nearest port origin + noise, axial only near the ports."""
    m = xyz[0].numel()
    dev = xyz[0].device
    best = torch.full((m,), float("inf"), dtype=torch.float64, device=dev)
    v = [torch.zeros(m, dtype=torch.float64, device=dev) for _ in range(3)]
    for p in ports:
        d2 = sum((xyz[j] - p.origin[j]) ** 2 for j in range(3))
        sel = d2 < best
        best = torch.where(sel, d2, best)
        for j in range(3):
            v[j] = torch.where(sel, torch.full_like(v[j], p.Q[j]), v[j])
    v = [v[j] + noise[j] for j in range(3)]
    return _project_near_ports(xyz, v, ports, 3, 2 * dp)


def c4(device="cpu", n_updates=100, scale=1.0, nports=8) -> Workload:
    """3-D 1.6x0.8x0.8 multi-branch junction at dp=0.0025 (reading R20): 640x320x320
    = 65,536,000 lattice sites before pre-clearing; 8 random ports (4 in, 4 out)."""
    dim, dp = 3, 0.0025
    h = 1.3 * dp
    box = (1.6 * scale, 0.8 * scale, 0.8 * scale)
    counts = tuple(int(round(b / dp)) for b in box)
    cs = f32(1.6 / 246.0)
    dt = 0.0005
    rng = np.random.default_rng(np.random.SeedSequence(SEED_BASE + 4).spawn(2)[0])
    bc = (0.1 * scale, 0.2 * scale) if scale < 1 else (0.1, 0.2)
    ports, _ = _draw_ports(rng, nports, (0, 0, 0), box, dp, cs, n_updates, dt, [], bc_range=bc)
    g = _gen(SEED_BASE + 4, device)
    base, ids = _lattice(counts, dp, device)
    n0 = ids.numel()
    xyz = [base[j] + _jitter(n0, g, device, dp) for j in range(3)]
    keep = _preclear(xyz, ports, dp, cs, n_updates, dt)
    xyz = [c[keep] for c in xyz]
    base = [c[keep] for c in base]
    ids = ids[keep]
    n = ids.numel()
    noise = [_noise(n, g, device) for _ in range(3)]

    def vel(x, idx):
        return _nearest_port_velocity(x, ports, [c if idx is None else c[idx] for c in noise], dp)
    xyz, v, nre = _screen(base, xyz, vel, ids, ports, dim, dp, cs, f32(dt), n_updates, SEED_BASE + 4)
    pad = 10
    lo = (f32(-pad * cs),) * 3
    ncell = tuple(int(math.ceil(b / cs)) + 2 * pad for b in box)
    grid = Grid(dim, lo, cs, ncell)
    return Workload("C4" if scale == 1.0 else f"C4x{scale:g}", dim, dp, h, grid, ports,
                    _pack_state(xyz, v, ids, dim), f32(dt), n_updates, n0,
                    notes=f"{counts} lattice junction, {nports} random ports, pre-cleared; {nre} re-drawn",
                    redrawn=nre)


C5_SLAB_LEN = 1.6
C5_CELLS_PER_SLAB = 307
# empty cells around the C5 box: particles leave it at most 1.2 m/s x 0.0005 s =
# 0.115 cells per update, so 10 cells cover ~87 updates (the bench runs ~80 per
# invocation at its driver settings) before any reaches the clamped boundary
# cells; along x the last slab's ports may straddle its outer face (x has no
# margin at slab faces), so x keeps room for a whole port (34 cells = 0.18 m)
C5_PAD_X = 34
C5_PAD_YZ = 10
C5_NEXT_ID = 1 << 40


def c5_geometry(scale=1.0):
    """dp, h, cs, slab length L, width W, lattice counts per slab, cells per slab.
    cs = L / floor(L / 2h) >= 2h so slab faces lie on cell faces (307 cells at scale 1)."""
    dp = 0.002
    h = 1.3 * dp
    L = C5_SLAB_LEN * scale
    W = 0.8 * scale
    cells = int(math.floor(L / (2 * h) + 1e-9))
    cs = f32(L / cells)
    counts = (int(round(L / dp)), int(round(W / dp)), int(round(W / dp)))
    return dp, h, cs, L, W, counts, cells


def c5_ports(nslabs: int, scale=1.0, n_updates=50):
    """Ports of slabs 0..nslabs (one extra slab so every slab's velocity field is
    P-independent).  Slab r's ports come from its own seeded stream, conditioned on
    the ports of earlier slabs; x has no margin at interior faces (straddling)."""
    dp, h, cs, L, W, counts, cells_per_slab = c5_geometry(scale)
    dt = 0.0005
    bc = (0.1 * scale, 0.2 * scale) if scale < 1 else (0.1, 0.2)
    per_slab, prior = [], []
    for r in range(nslabs + 1):
        rng = np.random.default_rng(np.random.SeedSequence(SEED_BASE + 5 + 1000 * r))
        pts, placed = _draw_ports(rng, 8, (L * r, 0.0, 0.0), (L * (r + 1), W, W), dp, cs, n_updates, dt, prior,
                                  x_margin_lo=(r == 0), x_margin_hi=False, bc_range=bc)
        per_slab.append(pts)
        prior += placed
    return per_slab


def c5_grid(nslabs: int, scale=1.0):
    """The global C5 grid of an nslabs-slab problem (x-major cells, 307 per slab at
    scale 1, empty padding around the box) and each slab's [cx_begin, cx_end)."""
    dp, h, cs, L, W, counts, cells_per_slab = c5_geometry(scale)
    pad_x, pad_yz = C5_PAD_X, C5_PAD_YZ
    lo = (f32(-pad_x * cs), f32(-pad_yz * cs), f32(-pad_yz * cs))
    nyz = int(math.ceil(W / cs)) + 2 * pad_yz
    ncell = (cells_per_slab * nslabs + 2 * pad_x, nyz, nyz)
    slabs = []
    for r in range(nslabs):
        b = 0 if r == 0 else pad_x + cells_per_slab * r
        e = ncell[0] if r == nslabs - 1 else pad_x + cells_per_slab * (r + 1)
        slabs.append((b, e))
    return Grid(3, lo, cs, ncell), slabs


def c5(device="cpu", slab=0, nslabs=1, scale=1.0, n_updates=50) -> Workload:
    """3-D weak-scaling junction: slab r = [1.6r, 1.6(r+1)) x [0,0.8]^2 at dp=0.002
    (800x400x400 = 128M lattice sites per slab at scale 1).  Returns slab ``slab``
    of an ``nslabs``-slab problem; its content does not depend on nslabs."""
    dim = 3
    dp, h, cs, L, W, counts, cells_per_slab = c5_geometry(scale)
    dt = 0.0005
    per_slab = c5_ports(max(nslabs, slab + 1), scale, n_updates)
    ports = [p for r in range(nslabs) for p in per_slab[r]]
    shaping = [p for r in (slab - 1, slab, slab + 1) if 0 <= r < len(per_slab) for p in per_slab[r]]
    g = _gen(SEED_BASE + 5 + 1000 * slab, device)
    per = counts[0] * counts[1] * counts[2]
    base, ids = _lattice(counts, dp, device, origin=(L * slab, 0.0, 0.0), index_offset=per * slab)
    n0 = ids.numel()
    xyz = [base[j] + _jitter(n0, g, device, dp) for j in range(3)]
    keep = _preclear(xyz, shaping, dp, cs, n_updates, dt)
    xyz = [c[keep] for c in xyz]
    base = [c[keep] for c in base]
    ids = ids[keep]
    n = ids.numel()
    noise = [_noise(n, g, device) for _ in range(3)]

    def vel(x, idx):
        return _nearest_port_velocity(x, shaping, [c if idx is None else c[idx] for c in noise], dp)
    # screened against the ports of slabs r-1..r+1 whatever nslabs is, so slab r's
    # content does not depend on the number of GPUs
    xyz, v, nre = _screen(base, xyz, vel, ids, shaping, dim, dp, cs, f32(dt), n_updates, SEED_BASE + 5 + 1000 * slab)
    g0, slabs = c5_grid(nslabs, scale)
    lo, ncell = g0.lo, g0.ncell
    grid = Grid(dim, lo, cs, ncell, slabs[slab][0], slabs[slab][1])
    name = "C5" if scale == 1.0 else f"C5x{scale:g}"
    return Workload(name, dim, dp, h, grid, ports, _pack_state(xyz, v, ids, dim), f32(dt), n_updates, C5_NEXT_ID,
                    notes=f"slab {slab}/{nslabs}, {counts} lattice per slab, 8 ports per slab; {nre} re-drawn",
                    slab_cells=slabs, redrawn=nre)


# ----------------------------------------------------------------- rotating sprinkler (moving ports)

SPRINKLER_OMEGA = 2.0        # rad/s
SPRINKLER_THETA0 = 0.0       # rad


def sprinkler_angle(t: float, omega: float = SPRINKLER_OMEGA, theta0: float = SPRINKLER_THETA0) -> float:
    """theta = omega t + theta0."""
    return omega * t + theta0


def sprinkler_pose(port0: Port, pivot, theta: float) -> tuple:
    """Pose (origin, Q) of a 2-D nozzle port rotated by theta about `pivot` from its
    pose port0 at theta = 0: origin pivot + Rot(theta)(o0 - pivot), inflow axis at
    angle phi0 + theta.  f64, rounded once to binary32 (input data for both sides)."""
    c, s = math.cos(theta), math.sin(theta)
    d = (port0.origin[0] - pivot[0], port0.origin[1] - pivot[1])
    o = (f32(pivot[0] + c * d[0] - s * d[1]), f32(pivot[1] + s * d[0] + c * d[1]), 0.0)
    phi0 = math.atan2(port0.Q[1], port0.Q[0])
    return o, frame_rows_2d(phi0 + theta)


def rotation_pose_3d(port0: Port, pivot, axis, theta: float) -> tuple:
    """Pose (origin, Q) of a 3-D port turned by theta about the line through `pivot`
    along `axis` (Rodrigues, f64): origin pivot + R(o0 - pivot), every local axis
    rotated (Q = Q0 R^T); rounded once to binary32 (input data for both sides)."""
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    K = np.array([[0.0, -a[2], a[1]], [a[2], 0.0, -a[0]], [-a[1], a[0], 0.0]])
    R = np.eye(3) + math.sin(theta) * K + (1.0 - math.cos(theta)) * (K @ K)
    pv = np.asarray(pivot, dtype=np.float64)
    o = pv + R @ (np.asarray(port0.origin, dtype=np.float64) - pv)
    Q = np.asarray(port0.Q, dtype=np.float64).reshape(3, 3) @ R.T
    return tuple(f32(v) for v in o), tuple(f32(v) for v in Q.reshape(-1))


def c7(device="cpu", n_updates=100) -> Workload:
    """3-D rotating port (the sprinkler's moving frame in 3-D): a 0.3^3 box of fluid
    at dp = 0.01 (27,000 particles, lattice + jitter + N(0,0.05) noise), one inlet
    (he = (2 dp, 0.04, 0.03), 4 layers) turning at omega = 2 rad/s about the axis
    (1, 1, 1) through the box centre, and a static outlet.  Velocities: 1.0 along
    the nearest port axis + noise, axial only near the ports.  dt = 0.0005."""
    dim, dp = 3, 0.01
    h = 1.3 * dp
    cs = f32(2 * h)
    dt = 0.0005
    g = _gen(SEED_BASE + 7, device)
    xyz, ids = _lattice((30, 30, 30), dp, device)
    n = ids.numel()
    for j in range(dim):
        xyz[j] = xyz[j] + _jitter(n, g, device, dp)
    ports = [_port((0.15 + 0.07, 0.15 - 0.03, 0.15 - 0.04), frame_rows_3d((0.3, 1.0, -0.2), 0.4),
                   (2 * dp, 0.04, 0.03), INLET, 4),
             _port((0.06, 0.24, 0.22), frame_rows_3d((-1.0, 0.2, 0.5), 1.1), (2 * dp, 0.03, 0.03), OUTLET, 4)]
    v = [_noise(n, g, device) for _ in range(dim)]
    d2 = [sum((xyz[j] - p.origin[j]) ** 2 for j in range(dim)) for p in ports]
    near0 = d2[0] <= d2[1]
    for j in range(dim):
        u0 = torch.tensor(ports[0].Q[j], dtype=torch.float64, device=device)
        u1 = torch.tensor(ports[1].Q[j], dtype=torch.float64, device=device)
        v[j] = v[j] + torch.where(near0, u0, u1)
    v = _project_near_ports(xyz, v, ports, dim, 2 * dp)
    lo = (f32(-2 * cs), f32(-2 * cs), f32(-2 * cs))
    nc = int(math.ceil(0.3 / cs)) + 4
    grid = Grid(dim, lo, cs, (nc, nc, nc))
    return Workload("C7", dim, dp, h, grid, ports, _pack_state(xyz, v, ids, dim), f32(dt), n_updates, n,
                    notes="3-D rotating inlet about (1,1,1) through the box centre, static outlet")


def c6(device="cpu", n_updates=200, nozzles=4) -> Workload:
    """2-D rotating sprinkler (paper §V.C): dp = 0.005, nozzles of
    half-width 0.02 with the inflow profile v_X' = 2500 (0.02^2 - Y'^2) (u0 = 1.0,
    R = 0.02), 4 layers, arms of radius 0.08 about the pivot (0, 0), turning
    at omega = 2 rad/s from theta0 = 0.  The sprinkler sprays into an empty
    top-view domain (no gravity); only the nozzles' buffer particles exist
    at t = 0.  The arm length is not given by the paper; 0.08 m is
    this recipe's choice.  dt = 0.0005 (|v| dt = 0.1 dp)."""
    dim, dp = 2, 0.005
    h = 1.3 * dp
    cs = f32(2 * h)
    dt = 0.0005
    he = (2 * dp, 0.02, 0.0)
    bc = BC(BC_VELOCITY, profile=PROFILE_PARABOLIC, u0=2500.0 * 0.02 * 0.02, radius=0.02)
    pivot = (0.0, 0.0)
    ports, xs, ys, vxs, vys = [], [], [], [], []
    for q in range(nozzles):
        phi = 2.0 * math.pi * q / nozzles
        o = (0.08 * math.cos(phi), 0.08 * math.sin(phi), 0.0)
        p = _port(o, frame_rows_2d(phi), he, INLET, 4)
        p.bc = bc
        ports.append(p)
        # the nozzle's lattice in its own frame: 4 layers x 8 rows, cell-centred
        for i in range(4):
            for j in range(8):
                X, Y = -he[0] + (i + 0.5) * dp, -he[1] + (j + 0.5) * dp
                xs.append(p.origin[0] + p.Q[0] * X + p.Q[3] * Y)
                ys.append(p.origin[1] + p.Q[1] * X + p.Q[4] * Y)
                u = bc.u0 * (1.0 - (Y / bc.radius) ** 2)
                vxs.append(u * p.Q[0])
                vys.append(u * p.Q[1])
    n = len(xs)
    xyz = [torch.tensor(xs, dtype=torch.float64, device=device), torch.tensor(ys, dtype=torch.float64, device=device)]
    v = [torch.tensor(vxs, dtype=torch.float64, device=device), torch.tensor(vys, dtype=torch.float64, device=device)]
    ids = torch.arange(n, device=device, dtype=torch.int64)
    L = 0.5
    lo = (f32(-L), f32(-L), 0.0)
    ncell = (int(math.ceil(2 * L / cs)), int(math.ceil(2 * L / cs)), 1)
    grid = Grid(dim, lo, cs, ncell)
    return Workload("C6", dim, dp, h, grid, ports, _pack_state(xyz, v, ids, dim), f32(dt), n_updates, n,
                    notes=f"{nozzles} nozzles of 32 buffer particles, omega = {SPRINKLER_OMEGA} rad/s")


CONFIGS = {"C1": c1, "C1e": c1e, "C2": c2, "C3": c3, "C4": c4, "C5": c5, "C6": c6, "C7": c7}


def make(name: str, device="cpu", **kw) -> Workload:
    return CONFIGS[name](device=device, **kw)


def capacity_for(w: Workload, headroom: float = 0.06) -> int:
    """Array capacity with room for the ledger growth of the run."""
    return int(w.n * (1.0 + headroom)) + 4096
