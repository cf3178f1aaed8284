"""Fixtures under tests/golden/ (each file cites the PAPER.md lines it restates):
Table I (Fourier inflow), Table II (Windkessel parameters) and the hand-worked
buffer updates H1-H5.  CPU: the constants the code uses equal the printed tables,
and the oracle reproduces every hand case.  GPU: the same hand cases through the
C ABI give the same hand values.
"""
import math
import os

import numpy as np
import pytest

import oracle
from paper_2406_16786_b200 import inputs
from paper_2406_16786_b200.inputs import BIDIRECTIONAL, INLET, OUTLET, Grid, Port, f32

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
KINDS = {"inlet": INLET, "outlet": OUTLET, "bidirectional": BIDIRECTIONAL}


def _rows(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [l.split() for l in f if l.strip() and not l.startswith("#")]


def test_table_I_matches_the_constants_used():
    t = {k: float(v) for k, v in _rows("table_I_fourier.txt")}
    assert inputs.TABLE_I_OMEGA == t["omega"]
    assert list(inputs.TABLE_I_A) == [t[f"a{n}"] for n in range(9)]
    assert list(inputs.TABLE_I_B) == [0.0] + [t[f"b{n}"] for n in range(1, 9)]
    # Eq. Fourier_Series at t = 0: a0 + sum a_n
    assert oracle.fourier(0.0, inputs.TABLE_I_A, inputs.TABLE_I_B, inputs.TABLE_I_OMEGA) == pytest.approx(
        sum(t[f"a{n}"] for n in range(9)), abs=1e-15)


def test_table_II_matches_the_constants_used():
    for vessel, rp, c, rd in _rows("table_II_windkessel.txt"):
        name = vessel.replace("_", " ")
        assert inputs.TABLE_II[name] == (float(rp), float(c), float(rd))
        Rp, Cc, Rd = inputs.windkessel_si(name)
        assert Rp == pytest.approx(float(rp) * 1e5) and Cc == pytest.approx(float(c) * 1e-5)
        assert Rd == pytest.approx(float(rd) * 1e5)


def hand_cases():
    cases, cur = [], None
    for r in _rows("hand_cases.txt"):
        if r[0] == "case":
            cur = {"name": r[1], "dim": int(r[2]), "p": [], "keep": [], "gone": [], "dup": [], "label": []}
            cases.append(cur)
        elif r[0] == "grid":
            v = [float(x) for x in r[1:5]]
            cur["grid"] = Grid(cur["dim"], tuple(f32(x) for x in v[:3]), f32(v[3]), tuple(int(x) for x in r[5:8]))
        elif r[0] == "port":
            v = [float(x) for x in r[1:16]]
            cur["port"] = Port(tuple(f32(x) for x in v[:3]), tuple(f32(x) for x in v[3:12]),
                               tuple(f32(x) for x in v[12:15]), KINDS[r[16]], 4)
        elif r[0] == "p":
            cur["p"].append((int(r[1]), int(r[2]), [float(x) for x in r[3:3 + cur["dim"]]]))
        elif r[0] == "counts":
            cur["counts"] = [int(r[1]), int(r[2])]
        elif r[0] in ("keep", "dup"):
            d = cur["dim"]
            cur[r[0]].append((int(r[1]), [float(x) for x in r[2:2 + d]], float(r[2 + d])))
        elif r[0] == "gone":
            cur["gone"].append(int(r[1]))
        elif r[0] == "label":
            cur["label"].append((int(r[1]), int(r[2])))
    return cases


def _state(case):
    d = case["dim"]
    pts = np.array([p[2] for p in case["p"]], np.float32).reshape(-1, d)
    n = len(pts)
    st = {"x": pts[:, 0].copy(), "y": pts[:, 1].copy(), "vx": np.zeros(n, np.float32), "vy": np.zeros(n, np.float32),
          "id": np.array([p[0] for p in case["p"]], np.int64), "label": np.array([p[1] for p in case["p"]], np.int32)}
    if d == 3:
        st["z"] = pts[:, 2].copy()
        st["vz"] = np.zeros(n, np.float32)
    return st


NEXT_ID = 1000


def _check(case, counts, new):
    d = case["dim"]
    cols = ["x", "y", "z"][:d]
    ids = [int(i) for i in new["id"]]
    assert list(counts) == case["counts"], case["name"]
    for pid, pos, tol in case["keep"]:
        j = ids.index(pid)
        assert np.allclose([float(new[c][j]) for c in cols], pos, atol=tol, rtol=1e-7), (case["name"], pid)
    for pid in case["gone"]:
        assert pid not in ids, (case["name"], pid)
    new_ids = [i for i in ids if i >= NEXT_ID]
    assert len(new_ids) == case["counts"][0]
    for k, (pid, pos, tol) in enumerate(case["dup"]):
        j = ids.index(NEXT_ID + k)
        assert int(new["label"][j]) == -1
        assert np.allclose([float(new[c][j]) for c in cols], pos, atol=tol, rtol=1e-7), (case["name"], "dup", pid)
    for pid, lab in case["label"]:
        assert int(new["label"][ids.index(pid)]) == lab, (case["name"], pid)


@pytest.mark.parametrize("case", hand_cases(), ids=lambda c: c["name"])
def test_hand_case_oracle(case):
    st = _state(case)
    res = oracle.update(case["grid"], [case["port"]], st)
    new, perm, nid = oracle.compact(res, case["dim"], 1, res.port_counts[None, :], 0, NEXT_ID)
    _check(case, res.port_counts, new)


@pytest.mark.gpu
@pytest.mark.parametrize("case", hand_cases(), ids=lambda c: c["name"])
def test_hand_case_gpu(case):
    import torch
    from paper_2406_16786_b200 import sphbuf
    st = {k: torch.from_numpy(v) for k, v in _state(case).items()}
    bu = sphbuf.BufferUpdater(case["grid"], 0.013, 0.01, [case["port"]], 1024)
    bu.load(st, NEXT_ID)
    bu.register_ports()      # (identification changes none of these labels)
    bu.cll_build()
    bu.update()
    bu.compact()
    new = {k: v.numpy() for k, v in bu.state().items()}
    pc = bu.port_counts.cpu().numpy()
    _check(case, [int(pc[0]), int(pc[sphbuf.MAX_PORTS])], new)
