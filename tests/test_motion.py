"""Moving ports: the rotating sprinkler (paper §V.C).

After this step's generation in the established local frame, the buffer
particles "are transformed to new ones through coordinate rotation" and the
local coordinate system is re-established.  Reading R23: each buffer
particle keeps its local coordinates and local velocity.

CPU (-m "not gpu"): the oracle's move is pinned by a hand case (a quarter turn
about the pivot, H7), by isometry and preservation of local coordinates, by
leaving other particles untouched, by theta = omega t + theta0
and by a sprinkler run whose invariants hold every step (inlet member counts
constant, cell-restricted decisions equal brute force at every pose, duplicates
emitted at the pose of their step).
GPU (-m gpu): sph_port_move through the C ABI (members moved by K9, candidate
cells re-enumerated on the device by K10) in lock-step with the oracle,
bit-exact, 200 updates of the 4-nozzle sprinkler.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2406_16786_b200 import inputs
from paper_2406_16786_b200.inputs import INLET, Port, f32, frame_rows_2d

from parity_util import assert_state_equal, gpu_counts_to_oracle, make_updater
from tiescreen import screen

_SCREENED = {}


def _moving_dry_run(pose_fn, n_steps):
    """The oracle sequence of a moving-port run (advect, update, compact, move every
    port to its next pose) for the tie screen (tests/tiescreen.py)."""
    def run(w, lin):
        K = len(w.ports)
        st = oracle.to_numpy_state(w.state)
        for k, p in enumerate(w.ports):
            oracle.register(st, w.grid, p, k)
        ports = list(w.ports)
        nid = w.next_id
        for step in range(n_steps):
            oracle.advect(st, w.dim, w.dt)
            res = oracle.update(w.grid, ports, st)
            new, perm, nid = oracle.compact(res, w.dim, K, res.port_counts[None, :], 0, nid)
            lin.record(res, new)
            for k, (o, Q) in pose_fn(w, step).items():
                nxt = Port(o, Q, ports[k].half_extents, ports[k].kind, ports[k].layers, ports[k].bc)
                oracle.port_move(new, w.dim, ports[k], nxt, k)
                ports[k] = nxt
            st = new
    return run


def screened(name, device="cpu", n_steps=200):
    """C6 / C7 tie-screened on their own moving-port dynamics over n_steps."""
    key = (name, device, n_steps)
    pose = (lambda w, s: dict(enumerate(_sprinkler_poses(w, s)))) if name == "C6" else \
        (lambda w, s: {0: _c7_pose(w, s)})
    if key not in _SCREENED:
        got = {}

        def make(nd):
            got.clear()
            got.update(nd)
            return inputs.nudge(inputs.make(name, device=device), nd)
        screen(make, _moving_dry_run(pose, n_steps))
        _SCREENED[key] = dict(got)
    return inputs.nudge(inputs.make(name, device=device), _SCREENED[key])


def _one(st_pts, vel, labels):
    n = len(st_pts)
    st = oracle.empty_state(2, n)
    st["x"][:] = [p[0] for p in st_pts]
    st["y"][:] = [p[1] for p in st_pts]
    st["vx"][:] = [v[0] for v in vel]
    st["vy"][:] = [v[1] for v in vel]
    st["id"][:] = np.arange(n)
    st["label"][:] = labels
    return st


def test_H7_quarter_turn_about_pivot():
    """Nozzle at o0 = (0.1, 0) pointing along +x, turned by pi/2 about the origin:
    o1 = (0, 0.1), axis +y.  A buffer particle at (0.11, 0.005) (local (0.01, 0.005))
    lands on (-0.005, 0.11), i.e. the point rotated by pi/2 about the pivot; its
    velocity (1, 0) becomes (0, 1).  A fluid particle is not moved."""
    he = (f32(0.01), f32(0.02), 0.0)
    p0 = Port((f32(0.1), 0.0, 0.0), frame_rows_2d(0.0), he, INLET, 4)
    o1, Q1 = inputs.sprinkler_pose(p0, (0.0, 0.0), math.pi / 2)
    p1 = Port(o1, Q1, he, INLET, 4)
    st = _one([(0.11, 0.005), (0.3, 0.3)], [(1.0, 0.0), (0.5, 0.5)], [0, -1])
    before = oracle.to_numpy_state(st)
    assert oracle.port_move(st, 2, p0, p1, 0) == 1
    np.testing.assert_allclose([st["x"][0], st["y"][0]], [-0.005, 0.11], atol=2e-8)
    np.testing.assert_allclose([st["vx"][0], st["vy"][0]], [0.0, 1.0], atol=1e-7)
    for c in ("x", "y", "vx", "vy"):
        assert st[c][1] == before[c][1]


def test_move_is_rigid_and_keeps_local_coordinates():
    """Random members of a 2-D port moved by an arbitrary rotation + translation:
    local coordinates (f64 to_local in the new frame vs the old) agree within fp32
    rounding, pairwise distances and speeds are preserved."""
    rng = np.random.default_rng(7)
    he = (f32(0.01), f32(0.02), 0.0)
    p0 = Port((f32(0.2), f32(-0.1), 0.0), frame_rows_2d(0.7), he, INLET, 4)
    p1 = Port((f32(-0.15), f32(0.25), 0.0), frame_rows_2d(2.9), he, INLET, 4)
    loc = rng.uniform(-1, 1, (50, 2)) * [0.01, 0.02]
    Q0 = np.array(p0.Q).reshape(3, 3)[:2, :2]
    g = np.array(p0.origin[:2]) + loc @ Q0
    vel = rng.normal(size=(50, 2))
    st = _one([tuple(r) for r in g], [tuple(v) for v in vel], [3] * 50)
    X0 = np.array([oracle.to_local(p0, 2, (st["x"][i], st["y"][i], 0.0), prec=1)[:2] for i in range(50)])
    v0 = np.stack([st["vx"], st["vy"]], 1).astype(np.float64)
    assert oracle.port_move(st, 2, p0, p1, 3) == 50
    X1 = np.array([oracle.to_local(p1, 2, (st["x"][i], st["y"][i], 0.0), prec=1)[:2] for i in range(50)])
    np.testing.assert_allclose(X1, X0, atol=5e-8)
    v1 = np.stack([st["vx"], st["vy"]], 1).astype(np.float64)
    np.testing.assert_allclose(np.linalg.norm(v1, axis=1), np.linalg.norm(v0, axis=1), rtol=1e-6)
    # local velocity preserved: Q1 v1 == Q0 v0
    Q1 = np.array(p1.Q, np.float64).reshape(3, 3)[:2, :2]
    np.testing.assert_allclose(v1 @ Q1.T, v0 @ Q0.astype(np.float64).T, atol=1e-6)
    d0 = np.linalg.norm(g[:, None] - g[None], axis=2)
    p = np.stack([st["x"], st["y"]], 1).astype(np.float64)
    d1 = np.linalg.norm(p[:, None] - p[None], axis=2)
    np.testing.assert_allclose(d1, d0, atol=1e-7)


def test_sprinkler_angle_P800():
    """theta = omega t + theta0 with omega = 2 rad/s, theta0 = 0: after
    t = pi/2 s the frame has turned by pi; omega = 0 keeps the pose."""
    assert inputs.sprinkler_angle(math.pi / 2) == pytest.approx(math.pi, abs=1e-15)
    w = inputs.make("C6")
    o, Q = inputs.sprinkler_pose(w.ports[0], (0.0, 0.0), inputs.sprinkler_angle(math.pi / 2))
    np.testing.assert_allclose(o[:2], [-0.08, 0.0], atol=1e-8)        # the nozzle at phi = 0 is now at phi = pi
    np.testing.assert_allclose(Q[:2], [-1.0, 0.0], atol=1e-7)          # inflow axis reversed
    o0, Q0 = inputs.sprinkler_pose(w.ports[1], (0.0, 0.0), inputs.sprinkler_angle(0.0, omega=0.0))
    np.testing.assert_allclose(o0, w.ports[1].origin, atol=1e-9)
    np.testing.assert_allclose(Q0, w.ports[1].Q, atol=1e-7)


def _sprinkler_poses(w, step):
    t = (step + 1) * w.dt
    return [inputs.sprinkler_pose(p, (0.0, 0.0), inputs.sprinkler_angle(t)) for p in w.ports]


def test_sprinkler_oracle_invariants():
    """100 updates of the 4-nozzle sprinkler on the oracle: every update the inlet
    member counts stay 32, brute force = cell-restricted decisions at the current
    pose, every duplicate lies just past its nozzle's interface (a/2 < X'_0 <
    a/2 + |v| dt) in the pose of its step, and every emitted particle stays fluid."""
    w = screened("C6", n_steps=100)
    K = len(w.ports)
    st = oracle.to_numpy_state(w.state)
    for k, p in enumerate(w.ports):
        assert oracle.register(st, w.grid, p, k) == 32
    ports = list(w.ports)
    nid = w.next_id
    created = 0
    for step in range(100):
        oracle.advect(st, 2, w.dt)
        res = oracle.update(w.grid, ports, st)
        res1 = oracle.update(w.grid, ports, oracle.to_numpy_state(st), mode=1)
        assert (res.port_counts == res1.port_counts).all()
        assert (res.create_port == res1.create_port).all()
        assert res.multi_decision == 0 and res.motion_errors == 0
        for q in range(len(res.stage_port)):
            k = int(res.stage_port[q])
            X = oracle.to_local(ports[k], 2, (res.staged["x"][q], res.staged["y"][q], 0.0), prec=1)
            assert 0.01 < X[0] < 0.01 + 1.0 * w.dt + 1e-6 and abs(X[1]) < 0.02
        created += int(res.port_counts[:K].sum())
        new, perm, nid = oracle.compact(res, 2, K, res.port_counts[None, :], 0, nid)
        poses = _sprinkler_poses(w, step)
        for k, (o, Q) in enumerate(poses):
            nxt = Port(o, Q, ports[k].half_extents, ports[k].kind, ports[k].layers, ports[k].bc)
            assert oracle.port_move(new, 2, ports[k], nxt, k) == 32
            ports[k] = nxt
        for k in range(K):
            assert int((new["label"] == k).sum()) == 32
        st = new
    assert created > 100
    assert int((st["label"] == -1).sum()) == created


@pytest.mark.gpu
def test_sprinkler_gpu_parity(n_steps=200):
    """Lock-step GPU (sph_port_move through the C ABI) vs oracle, 200 updates,
    bit-exact state after every update."""
    w = screened("C6", device="cuda", n_steps=n_steps)
    K = len(w.ports)
    st = oracle.to_numpy_state(w.state)
    for k, p in enumerate(w.ports):
        oracle.register(st, w.grid, p, k)
    bu = make_updater(w, capacity=8192, max_new=4096)
    bu.load(w.state, w.next_id)
    bu.register_ports()
    torch.cuda.synchronize()
    assert_state_equal(bu.state(), st, "after register")
    ports = list(w.ports)
    nid = w.next_id
    for step in range(n_steps):
        oracle.advect(st, 2, w.dt)
        res = oracle.update(w.grid, ports, st)
        new, perm, nid = oracle.compact(res, 2, K, res.port_counts[None, :], 0, nid)
        poses = _sprinkler_poses(w, step)
        for k, (o, Q) in enumerate(poses):
            nxt = Port(o, Q, ports[k].half_extents, ports[k].kind, ports[k].layers, ports[k].bc)
            oracle.port_move(new, 2, ports[k], nxt, k)
            ports[k] = nxt
        bu.cll_build(dt=w.dt)
        bu.update()
        for k, (o, Q) in enumerate(poses):
            bu.move_port(k, o, Q)
        bu.compact(deferred=step % 2 == 1)
        s = bu.stats()
        assert (gpu_counts_to_oracle(bu.port_counts, K) == res.port_counts).all(), step
        if step % 2 == 0:
            assert_state_equal(bu.state(), new, f"step {step}")
        assert int(bu.next_id.item()) == nid
        st = new
    assert s["motion_errors"] == 0


C7_PIVOT, C7_AXIS = (0.15, 0.15, 0.15), (1.0, 1.0, 1.0)


def _c7_pose(w, step):
    t = (step + 1) * w.dt
    return inputs.rotation_pose_3d(w.ports[0], C7_PIVOT, C7_AXIS, inputs.sprinkler_angle(t))


def test_rotating_port_3d_oracle_invariants():
    """3-D port turning about (1,1,1) (C7), 60 updates on the oracle: inlet member
    count constant, brute force = cell-restricted decisions at every pose, no
    particle with two decisions, no motion error."""
    w = screened("C7", n_steps=60)
    K = len(w.ports)
    st = oracle.to_numpy_state(w.state)
    m0 = [oracle.register(st, w.grid, p, k) for k, p in enumerate(w.ports)]
    assert m0[0] > 0
    ports = list(w.ports)
    nid = w.next_id
    for step in range(60):
        oracle.advect(st, 3, w.dt)
        res = oracle.update(w.grid, ports, st)
        res1 = oracle.update(w.grid, ports, oracle.to_numpy_state(st), mode=1)
        assert (res.port_counts == res1.port_counts).all() and (res.delete_port == res1.delete_port).all()
        assert res.multi_decision == 0 and res.motion_errors == 0
        new, perm, nid = oracle.compact(res, 3, K, res.port_counts[None, :], 0, nid)
        o, Q = _c7_pose(w, step)
        nxt = Port(o, Q, ports[0].half_extents, ports[0].kind, ports[0].layers)
        assert oracle.port_move(new, 3, ports[0], nxt, 0) == m0[0]
        ports[0] = nxt
        st = new


@pytest.mark.gpu
def test_rotating_port_3d_gpu_parity(n_steps=100):
    """C7 on the GPU (3-D K9 move, 3-D K10 enumeration) vs the oracle, 100 updates,
    bit-exact; the in-place compaction every update."""
    w = screened("C7", device="cuda", n_steps=n_steps)
    K = len(w.ports)
    st = oracle.to_numpy_state(w.state)
    for k, p in enumerate(w.ports):
        oracle.register(st, w.grid, p, k)
    bu = make_updater(w)
    bu.load(w.state, w.next_id)
    bu.register_ports()
    ports = list(w.ports)
    nid = w.next_id
    for step in range(n_steps):
        oracle.advect(st, 3, w.dt)
        res = oracle.update(w.grid, ports, st)
        new, perm, nid = oracle.compact(res, 3, K, res.port_counts[None, :], 0, nid)
        o, Q = _c7_pose(w, step)
        nxt = Port(o, Q, ports[0].half_extents, ports[0].kind, ports[0].layers)
        oracle.port_move(new, 3, ports[0], nxt, 0)
        ports[0] = nxt
        bu.cll_build(dt=w.dt)
        bu.update()
        bu.move_port(0, o, Q)
        bu.compact()
        assert (gpu_counts_to_oracle(bu.port_counts, K) == res.port_counts).all(), step
        assert_state_equal(bu.state(), new, f"step {step}")
        st = new
    assert bu.stats()["motion_errors"] == 0
