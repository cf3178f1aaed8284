"""The seeded input generator (paper_2406_16786_b200/inputs.py) on CPU: the tie
screen's building blocks and the properties the multi-GPU decomposition relies
on.  (The screen's end-to-end guarantee — no particle within 1e-4 dp of a
threshold over the run — is certified by the oracle in test_oracle_pins.py.)"""
import math

import numpy as np
import torch

from paper_2406_16786_b200 import inputs
from paper_2406_16786_b200.inputs import INLET, OUTLET, Port, Workload, f32


def test_c5_slab_content_independent_of_gpu_count():
    """Slab r of the C5 weak-scaling workload is bitwise the same whatever the
    number of slabs (the screen uses the ports of slabs r-1..r+1 in every case)."""
    a = inputs.c5(scale=0.3, slab=0, nslabs=1, n_updates=6)
    b = inputs.c5(scale=0.3, slab=0, nslabs=2, n_updates=6)
    c = inputs.c5(scale=0.3, slab=1, nslabs=2, n_updates=6)
    d = inputs.c5(scale=0.3, slab=1, nslabs=3, n_updates=6)
    for u, v in ((a, b), (c, d)):
        assert u.n == v.n
        for k in u.state:
            assert torch.equal(u.state[k], v.state[k]), k
    # slabs own disjoint id ranges
    assert int(a.state["id"].max()) < int(c.state["id"].min())


def test_hash_jitter_is_deterministic_and_bounded():
    ids = np.arange(100000, dtype=np.int64)
    j1 = inputs._hash_jitter(ids, 3, 1, 77, 0.002)
    j2 = inputs._hash_jitter(ids, 3, 1, 77, 0.002)
    assert np.array_equal(j1, j2)
    assert np.all(np.abs(j1) <= 0.1 * 0.002)
    assert not np.array_equal(j1, inputs._hash_jitter(ids, 4, 1, 77, 0.002))      # attempt matters
    assert not np.array_equal(j1, inputs._hash_jitter(ids, 3, 2, 77, 0.002))      # component matters
    assert abs(float(j1.mean())) < 2e-6 and 1.0e-4 < float(j1.std()) < 1.3e-4     # ~ U(-0.1dp, 0.1dp)


def _one_port_case(x0, vx, n_updates, kind=INLET):
    """One particle on the axis of an axis-aligned port o = 0, he = (0.02, 0.1, 0.1), m = cs = 0.026."""
    port = Port((0.0, 0.0, 0.0), (1.0, 0, 0, 0, 1.0, 0, 0, 0, 1.0), (f32(0.02), f32(0.1), f32(0.1)), kind, 4)
    x = [torch.tensor([x0], dtype=torch.float32), torch.zeros(1), torch.zeros(1)]
    v = [torch.tensor([vx], dtype=torch.float32), torch.zeros(1), torch.zeros(1)]
    return inputs._tie_flags(x, v, [port], 3, f32(0.026), f32(0.001), n_updates, 1e-6)


def test_tie_flags_sees_faces_along_the_trajectory():
    """A particle is flagged iff some point of its pinned fp32 trajectory lies
    within tau of a face value (|X'| = he or he + m)."""
    # starts 0.5e-6 from X' = a/2: flagged at registration
    assert bool(_one_port_case(0.02 - 0.5e-6, 0.0, 0)[0])
    # far from every face and at rest: not flagged
    assert not bool(_one_port_case(0.01, 0.0, 10)[0])
    # reaches X' = a/2 + m exactly (within rounding) after 3 steps of 0.012: flagged only with that horizon
    x0 = 0.046 - 3 * 0.012
    assert bool(_one_port_case(x0, 12.0, 3)[0])
    assert not bool(_one_port_case(x0, 12.0, 2)[0])


def test_tie_flags_follow_the_recycled_copy():
    """An inlet member that crosses X' = +a/2 is recycled by a = 0.04 and the
    screen follows that copy.  Steps of 0.007 from X' = 0.016: the particle
    itself passes 0.023 (crossing), ..., 0.044, 0.051 — never within tau of a face
    value 0.02 / 0.046 inside P_k — but its recycled copy, started at -0.017,
    reaches 0.046 = a/2 + m nine steps later.  Flagged at an inlet with that
    horizon; not flagged at an outlet (no copies) or one step short."""
    assert bool(_one_port_case(0.016, 7.0, 10, kind=INLET)[0])
    assert not bool(_one_port_case(0.016, 7.0, 10, kind=OUTLET)[0])
    assert not bool(_one_port_case(0.016, 7.0, 9, kind=INLET)[0])


def test_nudge_moves_only_the_listed_particles():
    w = inputs.make("C1e")
    ref = {k: v.clone() for k, v in w.state.items()}
    ids = [5, 17, 4000]
    inputs.nudge(w, {i: 1 for i in ids})
    moved = torch.nonzero((w.state["x"] != ref["x"]) | (w.state["y"] != ref["y"])).squeeze(1).tolist()
    assert sorted(int(w.state["id"][m]) for m in moved) == ids
    dx = (w.state["x"].double() - ref["x"].double()).abs().max()
    assert float(dx) <= 0.05 * w.dp * (1 + 1e-6)
    w2 = inputs.make("C1e")
    inputs.nudge(w2, {i: 1 for i in ids})
    assert torch.equal(w.state["x"], w2.state["x"])                 # deterministic
    w3 = inputs.make("C1e")
    inputs.nudge(w3, {i: 2 for i in ids})
    assert not torch.equal(w.state["x"], w3.state["x"])             # the attempt changes the draw


def test_lineage_maps_duplicates_to_their_original():
    """tests/tiescreen.Lineage: a duplicate (new id) descends from its source
    (P:325), transitively; originals map to themselves."""
    import oracle
    from tiescreen import Lineage
    w = inputs.c1e(n_updates=20)
    st = oracle.to_numpy_state(w.state)
    for k, p in enumerate(w.ports):
        oracle.register(st, w.grid, p, k)
    lin = Lineage()
    nid = w.next_id
    for _ in range(3):
        oracle.advect(st, 2, w.dt)
        res = oracle.update(w.grid, w.ports, st)
        new, perm, nid = oracle.compact(res, 2, 2, res.port_counts[None, :], 0, nid)
        lin.record(res, new)
        st = new
    fresh = st["id"][st["id"] >= w.next_id]
    assert len(fresh) >= 40
    for i in fresh.tolist():
        o = lin.original(i)
        assert o < w.next_id
        assert st["label"][st["id"] == o][0] == 0          # the source is an inlet buffer particle
    assert lin.original(3) == 3


def test_c5_ports_fit_the_grid_at_every_gpu_count():
    """Every C5 port's decision region P_k lies strictly inside the grid for 1, 2, 4
    and 8 slabs at full scale (the registration check, sph_port_check), so the
    grid's padding leaves room for the ports that straddle the outer slab face."""
    from paper_2406_16786_b200 import sphbuf
    dp = inputs.c5_geometry()[0]
    for P in (1, 2, 4, 8):
        g, slabs = inputs.c5_grid(P)
        ctx = sphbuf.Context(g, 1.3 * dp, 1024, 64, 16)
        for p in [q for r in inputs.c5_ports(P)[:P] for q in r]:
            assert sphbuf.sph_port_check(ctx, p.origin, p.Q, p.half_extents, p.kind, p.layers, dp) == 0, (P, p)


def test_expected_migrants_is_the_face_flux():
    """dist.expected_migrants: sum of max(+-v_x, 0) dt / dp over the particles within
    one spacing of each interior slab face (the larger face), 0 without one."""
    from paper_2406_16786_b200.dist import expected_migrants
    g = inputs.Grid(3, (0.0, 0.0, 0.0), 0.01, (100, 10, 10), 40, 60)     # faces at x = 0.4 and 0.6
    x = torch.tensor([0.4005, 0.4005, 0.5, 0.5995, 0.5995, 0.5995], dtype=torch.float32)
    vx = torch.tensor([-2.0, 1.0, -5.0, 1.0, 1.0, -1.0], dtype=torch.float32)
    st = {"x": x, "vx": vx}
    # lower face: |-2| * dt/dp = 2 * 0.001/0.001 = 2; upper face: (1 + 1) = 2 -> max 2
    assert expected_migrants(st, g, 0.001, 0.001) == 2
    assert expected_migrants(st, inputs.Grid(3, (0.0, 0.0, 0.0), 0.01, (100, 10, 10)), 0.001, 0.001) == 0
