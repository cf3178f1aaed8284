"""Key carry-over of the cell-list build: a build that advects
prepares the next build's keys and histogram in its gather; the update,
compaction and moving ports correct them for the particles they change.  The
results must be identical to builds that run their own key pass, whatever the
sequence of calls — lock-step against the oracle, bit-exact.
"""
import pytest

import oracle
from paper_2406_16786_b200 import inputs

from parity_util import assert_state_equal, gpu_counts_to_oracle, lockstep, make_updater


@pytest.mark.gpu
def test_carry_with_inplace_compaction():
    """In-place compaction every update moves the carried keys with the particles."""
    w = inputs.c4(scale=0.25, nports=4, n_updates=10)
    tot, bu = lockstep(w, 10, check_every=1, fused=True, deferred=False)
    assert tot.sum() > 0


@pytest.mark.gpu
def test_carry_duct_long_run():
    w = inputs.c3(scale=0.25, n_updates=40)
    tot, bu = lockstep(w, 40, check_every=4, fused=True, deferred=True)
    assert tot[0] > 0 and tot[1] > 0


@pytest.mark.gpu
def test_carry_survives_any_call_sequence():
    """Fused builds (carry made and used), a change of dt (carried keys cleared), a
    standalone advection + plain build, deferred and in-place compactions mixed:
    the state after every update equals the oracle's."""
    from tiescreen import screened, static_dry_run
    plan = ["fused", "fused", "dt2", "fused", "split", "fused", "fused", "split", "dt2", "dt2", "fused"]
    w0 = inputs.make("C2")
    dts = [w0.dt * (0.5 if mode == "dt2" else 1.0) for mode in plan]
    w = screened("carry-C2", lambda: inputs.make("C2"), static_dry_run(len(plan), dts))
    K = len(w.ports)
    st = oracle.to_numpy_state(w.state)
    for k, p in enumerate(w.ports):
        oracle.register(st, w.grid, p, k)
    bu = make_updater(w)
    bu.load(w.state, w.next_id)
    bu.register_ports()
    nid = w.next_id
    for n, mode in enumerate(plan):
        dt = w.dt * (0.5 if mode == "dt2" else 1.0)
        oracle.advect(st, w.dim, dt)
        res = oracle.update(w.grid, w.ports, st)
        new, perm, nid = oracle.compact(res, w.dim, K, res.port_counts[None, :], 0, nid)
        if mode == "split":
            bu.advect(dt)
            bu.cll_build()
        else:
            bu.cll_build(dt=dt)
        bu.update()
        deferred = n % 3 == 1
        bu.compact(deferred=deferred)
        assert (gpu_counts_to_oracle(bu.port_counts, K) == res.port_counts).all(), (n, mode)
        if not deferred:   # (a deferred compaction leaves tombstones until the next build)
            assert_state_equal(bu.state(), new, f"update {n} ({mode})")
        st = new
    # one more plain build: the final state in cell-list order
    bu.cll_build()
    fin = oracle.update(w.grid, [], st)
    assert_state_equal(bu.state(), {c: v[fin.order] for c, v in st.items() if c != "extra"}, "final")


@pytest.mark.gpu
def test_inplace_compaction_label_pass_fallback():
    """The in-place compaction's offsets come from the update's deletion list when it
    is complete; with the list disabled (SPHBUF_DLIST_MAX=0, read once per process,
    hence a subprocess) the label-pass fallback must give the same bit-exact result."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "from paper_2406_16786_b200 import inputs\n"
            "from parity_util import lockstep\n"
            "w = inputs.c4(scale=0.25, nports=4, n_updates=6)\n"
            "tot, bu = lockstep(w, 6, check_every=1, fused=True, deferred=False)\n"
            "assert tot[1] > 0\n"
            "print('ok')\n") % (os.path.dirname(here), here)
    env = dict(os.environ, SPHBUF_DLIST_MAX="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.gpu
def test_update_global_run_search_path():
    """K6 stages a tile's port runs in shared memory when they fit (kTileRuns);
    otherwise it binary-searches the runs in global memory.  SPHBUF_TILE_RUNS=0
    (read once per process, hence a subprocess) forces the global path for every
    tile: bit-exact with the oracle on C2 (bidirectional), a 3-D junction with
    in-place compaction and moving random ports."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "import oracle; oracle.enable_tie_check(1e-4)\n"
            "from paper_2406_16786_b200 import inputs\n"
            "from parity_util import lockstep\n"
            "tot, bu = lockstep(inputs.make('C2'), 12, check_every=3, fused=True, deferred=True)\n"
            "assert tot[0] > 0 and tot[1] > 0\n"
            "w = inputs.c4(scale=0.25, nports=4, n_updates=6)\n"
            "tot, bu = lockstep(w, 6, check_every=1, fused=True, deferred=False)\n"
            "assert tot.sum() > 0\n"
            "import test_random_gpu as tr\n"
            "tr.test_random_moving_ports_lockstep(3)\n"
            "print('ok')\n") % (os.path.dirname(here), here)
    env = dict(os.environ, SPHBUF_TILE_RUNS="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.gpu
def test_inplace_compaction_register_move_path():
    """The in-place move runs on the copy engine (k_compact_move_tma, bulk copies
    through shared memory) by default; SPHBUF_MOVE_TMA=0 selects the register move
    (k_compact_move2): both bit-exact with the oracle (3-D junction, carried keys;
    C2 in 2-D)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "import oracle; oracle.enable_tie_check(1e-4)\n"
            "from paper_2406_16786_b200 import inputs\n"
            "from parity_util import lockstep\n"
            "w = inputs.c4(scale=0.25, nports=4, n_updates=6)\n"
            "tot, bu = lockstep(w, 6, check_every=1, fused=True, deferred=False)\n"
            "assert tot[1] > 0\n"
            "tot, bu = lockstep(inputs.make('C2'), 8, check_every=1, fused=False, deferred=False)\n"
            "assert tot[1] > 0\n"
            "print('ok')\n") % (os.path.dirname(here), here)
    env = dict(os.environ, SPHBUF_MOVE_TMA="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.gpu
def test_copy_engine_gather_path():
    """The opt-in copy-engine gather (k_cll_gather_tma, SPHBUF_GATHER_TMA=1: window
    of every column by cp.async.bulk, far sources by cp.async into the stage) is
    bit-exact with the oracle: C2 (2-D, carried keys), a 3-D junction with in-place
    compaction, the duct with the advection outside the build (no carry), and the
    junction cut into 2 slabs (carried keys with migration)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "import oracle; oracle.enable_tie_check(1e-4)\n"
            "from paper_2406_16786_b200 import inputs\n"
            "from parity_util import lockstep\n"
            "tot, bu = lockstep(inputs.make('C2'), 10, check_every=2, fused=True, deferred=True)\n"
            "assert tot[0] > 0 and tot[1] > 0\n"
            "w = inputs.c4(scale=0.25, nports=4, n_updates=6)\n"
            "tot, bu = lockstep(w, 6, check_every=1, fused=True, deferred=False)\n"
            "assert tot.sum() > 0\n"
            "tot, bu = lockstep(inputs.c3(scale=0.5), 4, check_every=2, fused=False, deferred=True)\n"
            "import test_dist as td\n"
            "td.test_loopback_slabs_match_oracle(2, True)\n"
            "print('ok')\n") % (os.path.dirname(here), here)
    env = dict(os.environ, SPHBUF_GATHER_TMA="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
