"""Boundary-condition state of buffer particles (paper §IV).

Oracle pins (CPU): the pressure BC projects member velocities on the port axis
(Eq. velocity_correction) and resets the density of recycled
particles to rho0 + p_b/c0^2 (Eq. postulate-density); the velocity
BC imposes v_X' = u0 (1 - (Y'/R)^2) in the local frame (Eqs. 2D/3D_velocity_
profile) rotated back (Eqs. 2D/3D_velocity_transformation,
P:605-636); duplicates keep the pre-BC state.
GPU: the same through the C ABI, bit-exact against the oracle.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2406_16786_b200 import inputs
from paper_2406_16786_b200.inputs import (BC, BC_PRESSURE, BC_VELOCITY, BIDIRECTIONAL, INLET, OUTLET,
                                          PROFILE_PARABOLIC, PROFILE_PARABOLIC_RADIAL, Grid, Port, f32)

GRID2 = Grid(2, (f32(-0.052), f32(-0.052), 0.0), f32(0.026), (81, 20, 1))
GRID3 = Grid(3, (f32(-0.6), f32(-0.6), f32(-0.6)), f32(0.026), (47, 47, 47))


def with_bc(ports, bcs):
    return [Port(p.origin, p.Q, p.half_extents, p.kind, p.layers, bc) for p, bc in zip(ports, bcs)]


def c1e_with(bcs):
    w = inputs.make("C1e")
    st = oracle.to_numpy_state(w.state)
    st["extra"] = [np.ones(w.n, np.float32)]           # density column
    ports = with_bc(w.ports, bcs)
    for k, p in enumerate(ports):
        oracle.register(st, w.grid, p, k)
    return w, st, ports


def test_pressure_bc_projection_and_recycled_density():
    bc = BC(BC_PRESSURE, rho0=1.0, c0=10.0, p_b=0.1, rho_column=0)
    w, st, ports = c1e_with([bc, bc])
    before = oracle.to_numpy_state(st)
    oracle.advect(st, 2, w.dt)
    adv = oracle.to_numpy_state(st)
    res = oracle.update(w.grid, ports, st)
    S = res.sorted
    rho_b = np.float32(1.0 + 0.1 / 100.0)
    members0 = S["label"] == 0
    # Q = I: v = (v.u)u is exactly (vx, 0) for every inlet buffer particle
    assert np.all(S["vy"][members0] == 0.0)
    pre = {int(i): j for j, i in enumerate(adv["id"])}
    idx = np.array([pre[int(i)] for i in S["id"][members0]])
    np.testing.assert_array_equal(S["vx"][members0], adv["vx"][idx])
    # recycled particles (sources of the 40 duplicates) carry rho0 + p_b / c0^2
    src = res.stage_src[res.stage_port == 0]
    assert len(src) == 40
    assert np.all(S["extra"][0][src] == rho_b)
    others = np.ones(len(S["x"]), bool)
    others[src] = False
    assert np.all(S["extra"][0][others] == 1.0)
    # duplicates keep the pre-BC state: velocity and density of the source before the update
    for t in range(len(res.staged["id"])):
        j = pre[int(res.staged["id"][t])]
        assert res.staged["vy"][t] == adv["vy"][j] and res.staged["extra"][0][t] == 1.0
    # the outlet's buffer particles are projected too (v_y = 0), fluid untouched
    fluid = S["label"] == -1
    idx_f = np.array([pre[int(i)] for i in S["id"][fluid]])
    np.testing.assert_array_equal(S["vy"][fluid], adv["vy"][idx_f])
    del before


def test_pressure_bc_rotated_port_is_a_projection():
    th = math.radians(30.0)
    Q = oracle.frame_2d(th)
    u = Q[0]
    g = Grid(2, (f32(-0.52), f32(-0.52), 0.0), f32(0.026), (40, 40, 1))
    p = Port(tuple(f32(v) for v in (0, 0, 0)), tuple(f32(v) for v in Q.ravel()), (f32(0.02), f32(0.2), 0.0),
             INLET, 4, BC(BC_PRESSURE, c0=10.0))
    rng = np.random.default_rng(1)
    loc = np.stack([rng.uniform(-0.019, 0.019, 200), rng.uniform(-0.19, 0.19, 200)], 1)
    pts = loc @ Q[:2, :2]
    vel = rng.normal(0, 1, (200, 2))
    st = {"x": pts[:, 0].astype(np.float32), "y": pts[:, 1].astype(np.float32),
          "vx": vel[:, 0].astype(np.float32), "vy": vel[:, 1].astype(np.float32),
          "id": np.arange(200, dtype=np.int64), "label": np.zeros(200, np.int32)}
    res = oracle.update(g, [p], st)
    S = res.sorted
    v = np.stack([S["vx"], S["vy"]], 1).astype(np.float64)
    v0 = np.stack([st["vx"][res.order], st["vy"][res.order]], 1).astype(np.float64)
    np.testing.assert_allclose(v @ u[:2], v0 @ u[:2], atol=1e-6)
    lateral = v - np.outer(v @ u[:2], u[:2])
    assert np.abs(lateral).max() < 1e-6


def test_velocity_bc_profile_hand_cases():
    """2-D, Q = I, R = 0.2, u0 = 2: Y' = 0 -> v = (2, 0); Y' = 0.1 -> 2 (1 - 0.25) = 1.5;
    3-D radial R = 0.2: (Y', Z') = (0.06, 0.08) -> r^2 = 0.01 -> u0 (1 - 0.25)."""
    I = tuple(float(v) for v in np.eye(3).ravel())
    p = Port((f32(0.5), f32(0.2), 0.0), I, (f32(0.02), f32(0.2), 0.0), INLET, 4,
             BC(BC_VELOCITY, profile=PROFILE_PARABOLIC, u0=2.0, radius=0.2))
    st = {"x": np.array([0.5, 0.5], np.float32), "y": np.array([0.2, 0.3], np.float32),
          "vx": np.zeros(2, np.float32), "vy": np.ones(2, np.float32), "id": np.array([0, 1], np.int64),
          "label": np.zeros(2, np.int32)}
    S = oracle.update(GRID2, [p], st).sorted
    v = dict(zip(S["id"].tolist(), zip(S["vx"].tolist(), S["vy"].tolist())))
    assert v[0] == (2.0, 0.0)
    assert abs(v[1][0] - 1.5) < 1e-6 and v[1][1] == 0.0
    Q3 = oracle.frame_3d([0, 1, 0])
    p3 = Port((0.0, 0.0, 0.0), tuple(f32(x) for x in Q3.ravel()), (f32(0.02), f32(0.2), f32(0.2)), INLET, 4,
              BC(BC_VELOCITY, profile=PROFILE_PARABOLIC_RADIAL, u0=1.0, radius=0.2))
    # local (0, 0.06, 0.08) -> global = Q^T (0, 0.06, 0.08)
    xg = Q3.T @ np.array([0.0, 0.06, 0.08])
    st3 = {"x": np.array([xg[0]], np.float32), "y": np.array([xg[1]], np.float32),
           "z": np.array([xg[2]], np.float32), "vx": np.zeros(1, np.float32), "vy": np.zeros(1, np.float32),
           "vz": np.zeros(1, np.float32), "id": np.array([0], np.int64), "label": np.zeros(1, np.int32)}
    S3 = oracle.update(GRID3, [p3], st3).sorted
    np.testing.assert_allclose([S3["vx"][0], S3["vy"][0], S3["vz"][0]], [0.0, 0.75, 0.0], atol=1e-6)


def _bc_w2():
    w2 = inputs.make("C2")
    bcp = BC(BC_PRESSURE, rho0=1000.0, c0=10.0, p_b=5.0, rho_column=0)
    w2.ports = with_bc(w2.ports, [bcp, bcp])
    w2.state["extra"] = [torch.full((w2.n,), 1000.0)]
    return w2


def _bc_w3():
    w3 = inputs.c3(scale=0.25, n_updates=30)
    w3.ports = with_bc(w3.ports, [BC(BC_VELOCITY, profile=PROFILE_PARABOLIC_RADIAL, u0=1.0, radius=0.1),
                                  BC(BC_PRESSURE, rho0=1.0, c0=10.0, p_b=0.0, rho_column=0)])
    w3.state["extra"] = [torch.ones(w3.n)]
    return w3


def bc_workloads():
    """C2 with pressure BCs (density column) on both bidirectional ports; a C3 duct
    with a radial velocity profile at the inlet and a pressure BC at the outlet.
    The BCs change the buffer particles' velocities, so both are tie-screened on
    their own dynamics (tests/tiescreen.py)."""
    from tiescreen import screened, static_dry_run
    return [(screened("bc-C2", _bc_w2, static_dry_run(20)), 20),
            (screened("bc-C3", _bc_w3, static_dry_run(30)), 30)]


@pytest.mark.gpu
@pytest.mark.parametrize("i", [0, 1])
def test_bc_gpu_parity(i):
    from parity_util import lockstep
    w, n = bc_workloads()[i]
    tot, bu = lockstep(w, n, check_every=2, state=w.state)
    assert tot[0] > 0


@pytest.mark.gpu
def test_bc_gpu_parity_fused_deferred():
    from parity_util import lockstep
    w, n = bc_workloads()[0]
    tot, bu = lockstep(w, 10, check_every=2, state=w.state, fused=True, deferred=True)
    assert tot[0] > 0
