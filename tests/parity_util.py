"""Shared helpers for the GPU parity tests: run the CUDA path (through the C ABI)
and the CPU oracle in lock-step on the same seeded inputs and compare.

The oracle decides in f64 from the plain definition; the GPU
decides in fp32.  They must agree bit for bit because the inputs are tie-screened:
``certify_margins`` asserts, at every decision and relabel point the oracle sees,
that no particle is within TIE_TAU_DP * dp of a threshold face (north_star; O7)."""
import numpy as np
import torch

import oracle
from paper_2406_16786_b200 import inputs, sphbuf

MAXP = sphbuf.MAX_PORTS
TIE_TAU_DP = 1e-4            # north_star (BASELINE.json): >= 1e-4 dp from any threshold


def certify_margins(st, grid, ports, dp, what=""):
    """O7: assert every particle of ``st`` is at least 1e-4 dp from every threshold
    face of InBox_k / P_k (oracle.tie_margin, f64).  Returns the minimum margin / dp."""
    if not ports or len(st["x"]) == 0:
        return float("inf")
    m, bad = oracle.tie_margin(st, grid, ports, TIE_TAU_DP * dp)
    assert len(bad) == 0, f"{what}: {len(bad)} particles within 1e-4 dp of a threshold (min {m / dp:.3g} dp)"
    return m / dp


COLS = ("x", "y", "z", "vx", "vy", "vz")


def gpu_counts_to_oracle(pc, K):
    pc = pc.cpu().numpy()
    return np.concatenate([pc[:K], pc[MAXP:MAXP + K]]).astype(np.int32)


def assert_state_equal(gpu: dict, ref: dict, what=""):
    """Bit-exact comparison of every column, in order."""
    n = len(ref["x"])
    assert len(gpu["x"]) == n, f"{what}: N {len(gpu['x'])} != {n}"
    for c in list(COLS) + ["id", "label"]:
        if c not in ref:
            continue
        g = gpu[c].cpu().numpy() if isinstance(gpu[c], torch.Tensor) else gpu[c]
        r = ref[c]
        if g.dtype == np.float32:
            eq = (g.view(np.int32) == r.view(np.int32))
        else:
            eq = g == r
        if not eq.all():
            bad = np.nonzero(~eq)[0]
            raise AssertionError(f"{what}: column {c} differs at {len(bad)} positions, first {bad[:5]}: "
                                 f"gpu {g[bad[:5]]} oracle {r[bad[:5]]}")
    for e, col in enumerate(ref.get("extra") or []):
        g = gpu["extra"][e].cpu().numpy()
        assert (g.view(np.int32) == col.view(np.int32)).all(), f"{what}: extra {e}"


def make_updater(w, capacity=None, max_new=None, n_extra=0):
    cap = capacity if capacity is not None else inputs.capacity_for(w)
    bu = sphbuf.BufferUpdater(w.grid, w.h, w.dp, w.ports, cap, max_new=max_new, n_extra=n_extra)
    return bu


def lockstep(w, n_updates, check_cll=True, state=None, next_id=None, capacity=None, max_new=None,
             check_every=1, fused=False, deferred=False, margins=True):
    """deferred: the GPU runs sph_compact_deferred; the tombstones then vanish in the
    next cell-list build, so states are compared in cell-list order (every checked
    step and once more after the last update) instead of post-compaction order."""
    """Run n_updates on GPU and oracle from the same state; compare registration,
    cell lists, counts and the full post-compaction state bit-exactly.
    Returns totals of (created, deleted) and the GPU updater."""
    dim = w.dim
    K = len(w.ports)
    st0 = state if state is not None else w.state
    st = oracle.to_numpy_state(st0)
    if margins:
        certify_margins(st, w.grid, w.ports, w.dp, "registration")
    mem_o = [oracle.register(st, w.grid, p, k) for k, p in enumerate(w.ports)]
    bu = make_updater(w, capacity, max_new, n_extra=len(st.get("extra") or []))
    bu.load({k: (v if k == "extra" else torch.as_tensor(v)) for k, v in st0.items()} if state is not None
            else w.state, w.next_id if next_id is None else next_id)
    bu.register_ports()
    torch.cuda.synchronize()
    assert bu.members.cpu().tolist()[:K] == mem_o, (bu.members.cpu().tolist(), mem_o)
    assert_state_equal(bu.state(), st, "after register")
    nid = w.next_id if next_id is None else next_id
    tot = np.zeros(2, np.int64)
    for step in range(n_updates):
        oracle.advect(st, dim, w.dt)
        if margins:
            certify_margins(st, w.grid, w.ports, w.dp, f"decision point, update {step}")
        res = oracle.update(w.grid, w.ports, st)
        assert res.multi_decision == 0
        new, perm, nid = oracle.compact(res, dim, K, res.port_counts[None, :], 0, nid)
        if margins:
            certify_margins(new, w.grid, w.ports, w.dp, f"relabel point, update {step}")
        if fused:
            bu.cll_build(dt=w.dt)          # sph_advect_cll_build
        else:
            bu.advect(w.dt)
            bu.cll_build()
        cmp_now = (step % check_every == 0) or step == n_updates - 1
        if check_cll and cmp_now:
            torch.cuda.synchronize()
            nc = len(res.cell_start)
            assert (bu.cell_start[:nc].cpu().numpy() == res.cell_start).all(), f"cell_start step {step}"
            assert (bu.cell_end[:nc].cpu().numpy() == res.cell_end).all(), f"cell_end step {step}"
            pre = {c: v[res.order] for c, v in st.items() if c != "extra"}
            assert_state_equal(bu.state(), pre, f"cell-list order step {step}")
        bu.update()
        bu.compact(deferred=deferred)
        if cmp_now:
            s = bu.stats()
            assert (gpu_counts_to_oracle(bu.port_counts, K) == res.port_counts).all(), (
                step, gpu_counts_to_oracle(bu.port_counts, K), res.port_counts)
            assert s["candidates"] >= 0
            if deferred:
                C_, D_ = int(res.port_counts[:K].sum()), int(res.port_counts[K:].sum())
                assert s["n"] == len(new["x"]) + D_, "deferred: N counts the tombstones"
            else:
                assert_state_equal(bu.state(), new, f"post-compaction step {step}")
            assert int(bu.next_id.item()) == nid
        tot += [res.port_counts[:K].sum(), res.port_counts[K:].sum()]
        st = new
    if deferred:
        # one more build removes the tombstones: compare with the oracle's final state in cell-list order
        bu.cll_build()
        fin = oracle.update(w.grid, [], st)
        assert_state_equal(bu.state(), {c: v[fin.order] for c, v in st.items() if c != "extra"}, "deferred final")
    return tot, bu
