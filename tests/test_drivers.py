"""Time-dependent port drivers: the aorta flow's pulsatile inlet and Windkessel
outlets (paper §V.D).

CPU (-m "not gpu"), oracle pins:
* Eq. Fourier_Series with Table I: at t = 0 only the cosine sum remains
  (a0 + sum a_n); at t = pi / (2 omega) the terms follow cos(n pi/2), sin(n pi/2)
  by hand; period 2 pi / omega.
* Eq. windkessel, one explicit step per update (reading R27): under a constant
  flow the pressure relaxes geometrically to (Rp + Rd) Q — the steady state of
  the ODE; under a linear ramp Q = alpha t it tracks the exact solution
  P(t) = (Rp + Rd) alpha t - tau Rd alpha (1 - exp(-t/tau)), tau = Rd C, within
  the scheme's O(dt) error (a dropped or mis-signed C Rp dQ/dt term fails it).
* Table II in SI units (1 dyn s/cm^5 = 1e5 Pa s/m^3, 1 cm^5/dyn = 1e-5 m^3/Pa).
* The flow through a port by hand: Q = V/a * sum of v.u over its buffer
  particles (outlet positive outward, inlet / bidirectional sign flipped, R26);
  fluid particles ignored.
GPU (-m gpu): a duct with a Fourier-driven plug inlet and a Windkessel-driven
outlet, lock-step with the oracle: state (density column included) bit-exact and
the device pressure equal to the oracle's f64 value every update.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2406_16786_b200 import inputs
from paper_2406_16786_b200.inputs import (BC, BC_PRESSURE, BC_VELOCITY, BIDIRECTIONAL, DRIVER_FOURIER,
                                          DRIVER_WINDKESSEL, INLET, OUTLET, PROFILE_PLUG, TABLE_I_A, TABLE_I_B,
                                          TABLE_I_OMEGA, Driver, Port, f32, frame_rows_2d)

from parity_util import assert_state_equal, gpu_counts_to_oracle, make_updater


def test_fourier_table_I_closed_forms():
    A, B, w = TABLE_I_A, TABLE_I_B, TABLE_I_OMEGA
    assert oracle.fourier(0.0, A, B, w) == pytest.approx(sum(A), abs=1e-15)
    assert sum(A) == pytest.approx(0.250501, abs=1e-12)
    # t = pi/(2w): cos(n pi/2) = 0,-1,0,1,0,-1,0,1 ; sin(n pi/2) = 1,0,-1,0,1,0,-1,0
    quarter = A[0] - A[2] + A[4] - A[6] + A[8] + B[1] - B[3] + B[5] - B[7]
    assert oracle.fourier(math.pi / (2 * w), A, B, w) == pytest.approx(quarter, abs=1e-12)
    for t in (0.013, 0.31, 0.5):
        assert oracle.fourier(t + 2 * math.pi / w, A, B, w) == pytest.approx(oracle.fourier(t, A, B, w), abs=1e-12)


def test_table_II_si_units():
    Rp, Cc, Rd = inputs.windkessel_si("descending aorta")
    assert Rp == pytest.approx(1.88e7) and Rd == pytest.approx(2.95e8) and Cc == pytest.approx(4.82e-9)
    # tau = Rd C is unit-free of the conversion: 2950 * 4.82e-4 s
    assert Rd * Cc == pytest.approx(2950 * 4.82e-4)


def test_windkessel_steady_state_and_ramp():
    Rp, Cc, Rd = inputs.windkessel_si("left subclavian")
    tau = Rd * Cc
    dt = tau / 2000.0
    # constant flow: geometric relaxation to (Rp + Rd) Q
    Q, P = 1e-5, 0.0
    Pstar = (Rp + Rd) * Q
    for n in range(1, 20001):
        P = oracle.windkessel(P, Q, Q, dt, Rp, Cc, Rd)
        if n in (1, 10, 1000):
            assert P == pytest.approx(Pstar * (1.0 - (1.0 - dt / tau) ** n), rel=1e-9)
    assert P == pytest.approx(Pstar, rel=1e-4)
    # linear ramp Q = alpha t from P = 0: the exact ODE solution within O(dt)
    alpha, P, Qp = 1e-4, 0.0, 0.0
    for n in range(1, 4001):
        t = n * dt
        P = oracle.windkessel(P, alpha * t, Qp, dt, Rp, Cc, Rd)
        Qp = alpha * t
    t = 4000 * dt
    exact = (Rp + Rd) * alpha * t - tau * Rd * alpha * (1.0 - math.exp(-t / tau))
    assert P == pytest.approx(exact, rel=2e-3)
    # without the C Rp dQ/dt term the ramp would be off by ~ Rp alpha tau / P
    assert abs(Rp * alpha * tau) > 0.05 * abs(exact)


def test_port_flux_by_hand():
    he = (f32(0.02), f32(0.2), 0.0)
    out = Port((f32(1.0), f32(0.2), 0.0), frame_rows_2d(0.0), he, OUTLET, 4)
    st = oracle.empty_state(2, 3)
    st["vx"][:] = [0.5, 0.25, 9.0]
    st["vy"][:] = [0.3, -0.1, 9.0]
    st["label"][:] = [1, 1, -1]
    S = oracle.port_flux(st, 2, out, 1)
    assert S == int(0.75 * 2 ** 32)
    # a 30-degree axis: v.u for v = (cos30, sin30) is 1 (within fp32 rounding of the terms)
    rot = Port((0.0, 0.0, 0.0), frame_rows_2d(math.radians(30)), he, BIDIRECTIONAL, 4)
    st["vx"][:] = [math.cos(math.radians(30))] * 3
    st["vy"][:] = [math.sin(math.radians(30))] * 3
    assert abs(oracle.port_flux(st, 2, rot, 1) / 2 ** 32 - 2.0) < 1e-6


def _duct_with_drivers(scale, n_updates, nudges):
    w = inputs.c3(scale=scale, n_updates=n_updates)
    inlet, outlet = w.ports
    dp = w.dp
    Rp, Cc, Rd = inputs.windkessel_si("descending aorta")
    w.ports = [Port(inlet.origin, inlet.Q, inlet.half_extents, INLET, inlet.layers,
                    BC(BC_VELOCITY, profile=PROFILE_PLUG, u0=1.0),
                    Driver(DRIVER_FOURIER, a=TABLE_I_A, b=TABLE_I_B, omega=TABLE_I_OMEGA)),
               Port(outlet.origin, outlet.Q, outlet.half_extents, OUTLET, outlet.layers,
                    BC(BC_PRESSURE, rho0=1060.0, c0=40.0, p_b=0.0, rho_column=0),
                    Driver(DRIVER_WINDKESSEL, Rp=Rp, C=Cc, Rd=Rd, P0=1.0e4, volume=dp ** 3))]
    w.state["extra"] = [torch.full((w.n,), 1060.0)]
    return inputs.nudge(w, nudges)


_SCREENED = {}


def duct_with_drivers(scale=0.15, n_updates=40):
    """C3 duct: Fourier plug inlet (Table I), Windkessel outlet (Table II descending
    aorta), pressure BC with a density column.  The driven inlet speed changes the
    buffer particles' motion, so the input is tie-screened on this test's own
    dynamics (tests/tiescreen.py)."""
    from tiescreen import screen
    key = (scale, n_updates)
    if key not in _SCREENED:
        def dry_run(w, lin):
            st = oracle.to_numpy_state(w.state)
            for k, p in enumerate(w.ports):
                oracle.register(st, w.grid, p, k)
            drv = _OracleDrivers(w)
            nid = w.next_id
            for n in range(n_updates):
                oracle.advect(st, 3, w.dt)
                ports, rho, Q = drv.step(st, (n + 1) * w.dt)
                res = oracle.update(w.grid, ports, st, rho_b=rho)
                new, perm, nid = oracle.compact(res, 3, 2, res.port_counts[None, :], 0, nid)
                lin.record(res, new)
                st = new
        nudges = {}

        def make(nd):
            nudges.clear()
            nudges.update(nd)
            return _duct_with_drivers(scale, n_updates, nd)
        screen(make, dry_run)
        _SCREENED[key] = dict(nudges)
    return _duct_with_drivers(scale, n_updates, _SCREENED[key])


class _OracleDrivers:
    """The oracle side of the drivers: Fourier speed into the port's BC, Windkessel
    pressure from the exact port flux."""

    def __init__(self, w):
        self.w = w
        d = w.ports[1].driver
        self.P = d.P0
        self.Qprev = None

    def step(self, st, t):
        w = self.w
        inl, out = w.ports
        u = oracle.fourier(t, inl.driver.a, inl.driver.b, inl.driver.omega)
        ports = [Port(inl.origin, inl.Q, inl.half_extents, inl.kind, inl.layers,
                      BC(BC_VELOCITY, profile=PROFILE_PLUG, u0=float(np.float32(u)))), out]
        d = out.driver
        S = oracle.port_flux(st, 3, out, 1)
        q = float(S) * 2.0 ** -32
        q = q * (d.volume / (2.0 * float(out.half_extents[0])))
        Q = q                                                  # outlet: outward = +u
        Qprev = Q if self.Qprev is None else self.Qprev
        self.P = oracle.windkessel(self.P, Q, Qprev, w.dt, d.Rp, d.C, d.Rd)
        self.Qprev = Q
        bc = out.bc
        c0 = float(np.float32(bc.c0))
        rho = float(np.float32(float(np.float32(bc.rho0)) + self.P / (c0 * c0)))
        return ports, {1: rho}, Q


def test_drivers_oracle_run():
    """30 updates on the oracle: the outlet flux stays positive (outflow) and the
    pressure rises from P0 towards (Rp + Rd) Q."""
    w = duct_with_drivers(n_updates=30)
    st = oracle.to_numpy_state(w.state)
    for k, p in enumerate(w.ports):
        oracle.register(st, w.grid, p, k)
    drv = _OracleDrivers(w)
    nid = w.next_id
    for n in range(30):
        oracle.advect(st, 3, w.dt)
        ports, rho, Q = drv.step(st, (n + 1) * w.dt)
        assert Q > 0
        res = oracle.update(w.grid, ports, st, rho_b=rho)
        st, perm, nid = oracle.compact(res, 3, 2, res.port_counts[None, :], 0, nid)
    assert drv.P > 1.0e4


@pytest.mark.gpu
def test_drivers_gpu_parity(n_updates=40):
    w = duct_with_drivers(n_updates=n_updates)
    st = oracle.to_numpy_state(w.state)
    for k, p in enumerate(w.ports):
        oracle.register(st, w.grid, p, k)
    bu = make_updater(w, n_extra=1)
    bu.load(w.state, w.next_id)
    bu.register_ports()
    drv = _OracleDrivers(w)
    nid = w.next_id
    K = 2
    for n in range(w.n_updates):
        t = (n + 1) * w.dt
        oracle.advect(st, 3, w.dt)
        ports, rho, Q = drv.step(st, t)
        res = oracle.update(w.grid, ports, st, rho_b=rho)
        new, perm, nid = oracle.compact(res, 3, K, res.port_counts[None, :], 0, nid)
        bu.cll_build(dt=w.dt)
        bu.drivers_step(t, w.dt)
        bu.update()
        bu.compact()
        s0 = bu.driver_state(0)
        s1 = bu.driver_state(1)
        assert s0["u0"] == oracle.fourier(t, TABLE_I_A, TABLE_I_B, TABLE_I_OMEGA)
        assert s1["Q"] == Q and s1["P"] == drv.P, (n, s1, Q, drv.P)
        assert (gpu_counts_to_oracle(bu.port_counts, K) == res.port_counts).all(), n
        assert_state_equal(bu.state(), new, f"update {n}")
        st = new
