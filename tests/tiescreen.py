"""Tie screen for test workloads whose dynamics the generator's own screen does not
model (boundary-condition velocities, time-dependent drivers, moving ports, dt
changes, hand-built random workloads).

north_star (BASELINE.json): "The generator keeps every particle at least 1e-4 dp
from any threshold, so no decision is a tie."  ``inputs`` screens the BASELINE
configs with a kinematic model of free flight + recycling.  A test that drives
other dynamics screens its own input here: it dry-runs its exact oracle sequence
with the tie check collecting offenders (``oracle.collect_ties``), maps every
offender back to the original particle it descends from (a duplicate descends
from its source), nudges those originals (``inputs.nudge``) and repeats
until a dry run is clean.  Only the oracle (CPU) is run here; the nudged input is
then what the GPU and the oracle are compared on.
"""
import oracle
from paper_2406_16786_b200 import inputs


class Lineage:
    """id -> id of the original particle it descends from."""

    def __init__(self):
        self.root = {}

    def record(self, res, new):
        """After oracle.compact: the appended particles (the tail of ``new``, in
        staging order) descend from the staged sources (res.staged['id'])."""
        ns = len(res.staged["id"])
        if ns == 0:
            return
        new_ids = new["id"][len(new["id"]) - ns:]
        for nid, src in zip(new_ids.tolist(), res.staged["id"].tolist()):
            self.root[int(nid)] = self.root.get(int(src), int(src))

    def original(self, i):
        return self.root.get(int(i), int(i))


def screen(make, dry_run, rounds=12):
    """make(nudges: dict id -> attempt) -> workload; dry_run(workload, lineage) runs
    the test's oracle sequence.  Returns the first workload whose dry run has no tie."""
    nudges = {}
    for _ in range(rounds):
        w = make(nudges)
        lin = Lineage()
        with oracle.collect_ties() as c:
            dry_run(w, lin)
        if not c.ids:
            return w
        for i in set(lin.original(i) for i in c.ids):
            nudges[i] = nudges.get(i, 0) + 1
    raise AssertionError(f"tie screen did not converge ({len(nudges)} particles nudged)")


def static_dry_run(steps, dts=None):
    """Dry run of a plain update sequence (advect by dts[i] or w.dt, update,
    compact) on the workload's own ports."""
    def run(w, lin):
        K = len(w.ports)
        st = oracle.to_numpy_state(w.state)
        for k, p in enumerate(w.ports):
            oracle.register(st, w.grid, p, k)
        nid = w.next_id
        for i in range(steps):
            oracle.advect(st, w.dim, w.dt if dts is None else dts[i])
            res = oracle.update(w.grid, w.ports, st)
            new, perm, nid = oracle.compact(res, w.dim, K, res.port_counts[None, :], 0, nid)
            lin.record(res, new)
            st = new
    return run


_CACHE = {}


def screened(key, build, dry_run):
    """build() -> a fresh workload (deterministic); returns it nudged so that
    ``dry_run`` has no tie.  The nudges are cached per key for the session."""
    if key not in _CACHE:
        got = {}

        def make(nd):
            got.clear()
            got.update(nd)
            return inputs.nudge(build(), nd)
        screen(make, dry_run)
        _CACHE[key] = dict(got)
    return inputs.nudge(build(), _CACHE[key])
