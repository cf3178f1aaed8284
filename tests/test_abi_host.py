"""Host-side checks of the C ABI (no GPU): the library loads, exports every symbol
declared in include/sphbuf.h, validates ports, and enumerates port cells that
cover the decision region exactly (cross-checked against the oracle's own,
independently written enumeration)."""
import math
import os
import re

import numpy as np
import pytest

import oracle
from paper_2406_16786_b200 import inputs, sphbuf
from paper_2406_16786_b200.inputs import BIDIRECTIONAL, INLET, OUTLET, Grid, f32

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "sphbuf.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sph_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = sphbuf.lib()
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(sphbuf.EXPORTS) == syms


def test_kernel_id_table_matches_header():
    """sph_profile_read fills SPH_NKERNELS entries: the binding's array size, the
    header's constant and the library's kernel-name table must agree."""
    import re
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "sphbuf.h")).read()
    n = int(re.search(r"#define SPH_NKERNELS (\d+)", hdr).group(1))
    assert sphbuf.NKERNELS == n
    L = sphbuf.lib()
    names = [L.sph_kernel_name(i).decode() for i in range(n + 1)]
    assert all(names[:n]) and names[n] == ""
    assert len(set(names[:n])) == n


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {sphbuf.lib()._name}").read()
    assert "sm_100a" in out


def ctx_c1():
    w = inputs.make("C1")
    return w, sphbuf.Context(w.grid, w.h, 16384, 64, 1024)


def test_ctx_create_validates_grid():
    w = inputs.make("C1")
    with pytest.raises(sphbuf.SphError):
        sphbuf.Context(w.grid, w.h * 1.5, 100, 8, 10)          # cs < 2h
    bad = Grid(2, w.grid.lo, w.grid.cs, (10, 10, 3))             # 2-D needs nz = 1
    with pytest.raises(sphbuf.SphError):
        sphbuf.Context(bad, w.h, 100, 8, 10)
    with pytest.raises(sphbuf.SphError):
        sphbuf.Context(w.grid, w.h, 100, 65, 10)                 # > SPH_MAX_PORTS


def test_port_check_errors():
    w, ctx = ctx_c1()
    I = (1, 0, 0, 0, 1, 0, 0, 0, 1)
    ok = sphbuf.sph_port_check(ctx, (0.02, 0.2, 0), I, (0.02, 0.2, 0), INLET, 4, 0.01)
    assert ok == 0
    # layers < 3
    assert sphbuf.sph_port_check(ctx, (0.02, 0.2, 0), I, (0.01, 0.2, 0), INLET, 2, 0.01) == -1
    # a != layers * dp
    assert sphbuf.sph_port_check(ctx, (0.02, 0.2, 0), I, (0.02, 0.2, 0), INLET, 3, 0.01) == -1
    # not a rotation
    assert sphbuf.sph_port_check(ctx, (0.02, 0.2, 0), (1, 0, 0, 0, 2, 0, 0, 0, 1), (0.02, 0.2, 0), INLET, 4,
                                 0.01) == -2
    assert sphbuf.sph_port_check(ctx, (0.02, 0.2, 0), (1, 0, 0, 0, -1, 0, 0, 0, 1), (0.02, 0.2, 0), INLET, 4,
                                 0.01) == -2
    # leaves the grid
    assert sphbuf.sph_port_check(ctx, (-0.02, 0.2, 0), I, (0.02, 0.2, 0), INLET, 4, 0.01) == -4
    assert sphbuf.sph_port_check(ctx, (1.0, 0.2, 0), I, (0.02, 0.2, 0), 7, 4, 0.01) == -1


def _oracle_cells(grid, port):
    return set(np.nonzero(oracle.port_cells(grid, port))[0].tolist())


def _lib_cells(grid, port):
    runs, n = sphbuf.sph_port_cells(grid, port.origin, port.Q, port.half_extents)
    cells = set()
    for c0, c1 in runs:
        cells.update(range(c0, c1 + 1))
    assert len(cells) == n
    # runs are in increasing cell order (canonical order of candidates)
    assert all(runs[i][1] < runs[i + 1][0] for i in range(len(runs) - 1))
    return cells


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_port_cells_match_oracle_2d(name):
    w = inputs.make(name)
    for p in w.ports:
        assert _lib_cells(w.grid, p) == _oracle_cells(w.grid, p)


def test_port_cells_match_oracle_3d_random_and_slabs():
    w = inputs.c4(scale=0.25, nports=4, n_updates=10)
    ncx = w.grid.ncell[0]
    for p in w.ports:
        assert _lib_cells(w.grid, p) == _oracle_cells(w.grid, p)
        for b, e in ((0, ncx // 2), (ncx // 2, ncx)):
            g = w.grid.slab(b, e)
            assert _lib_cells(g, p) == _oracle_cells(g, p)


def test_port_cells_cover_every_point_of_P_k():
    """Every point of the decision region P_k (he + cs) lies in an enumerated cell,
    using the pinned fp32 cell index (the one the kernels use)."""
    rng = np.random.default_rng(5)
    w = inputs.c4(scale=0.25, nports=4, n_updates=10)
    for p in w.ports:
        cells = _lib_cells(w.grid, p)
        Q = np.asarray(p.Q, np.float64).reshape(3, 3)
        H = np.asarray(p.half_extents) + w.grid.cs
        loc = rng.uniform(-1, 1, (3000, 3)) * H
        pts = (loc @ Q + np.asarray(p.origin)).astype(np.float32)
        for q in pts[:600]:
            c, oob = oracle.cell_of(w.grid, q)
            assert oob == 0 and c in cells


def test_frame_from_axis_matches_oracle_rodrigues():
    """The library's Rodrigues helper (psi = 0) equals the oracle's Q = R^T reading (R1);
    with a roll the first row stays u."""
    rng = np.random.default_rng(2)
    for _ in range(50):
        u = rng.standard_normal(3)
        u /= np.linalg.norm(u)
        Ql = np.asarray(sphbuf.sph_frame_from_axis(u, 0.0)).reshape(3, 3)
        np.testing.assert_allclose(Ql, oracle.frame_3d(u), atol=1e-7)
        Qr = np.asarray(sphbuf.sph_frame_from_axis(u, 1.1)).reshape(3, 3)
        np.testing.assert_allclose(Qr[0], u, atol=1e-7)
        np.testing.assert_allclose(Qr @ Qr.T, np.eye(3), atol=1e-6)


def test_workspace_bytes_scale():
    w, ctx = ctx_c1()
    b = sphbuf.sph_workspace_bytes(ctx)
    assert b > 16384 * 12


def test_comm_host_checks_without_gpu():
    """The multi-GPU calls validate on the host before touching NCCL or the device:
    bad rank / nranks -> SPH_ERR_ARG; no workspace yet (it holds the migration
    buffers) -> SPH_ERR_STATE; an exchange without a communicator -> SPH_ERR_STATE;
    the NCCL unique id (rank 0's bootstrap) is 128 bytes and fresh per call."""
    import ctypes as C
    w = inputs.make("C1")
    ctx = sphbuf.Context(w.grid, w.h, 16384, 64, 1024, max_migrate=256)
    L = sphbuf.lib()
    uid = (C.c_ubyte * sphbuf.COMM_ID_BYTES)()
    assert L.sph_comm_init(ctx.h, uid, 2, 2) == -1
    assert L.sph_comm_init(ctx.h, uid, 0, 0) == -1
    assert L.sph_comm_init(ctx.h, uid, 2, 0) == -9
    arr = (C.c_void_p * 1)(ctx.h.value)
    assert L.sph_comm_init_loopback(arr, 1) == -9
    assert L.sph_migrate_exchange(ctx.h, None) == -9
    assert L.sph_allgather_counts(ctx.h, None, None, None) == -1
    a, b = sphbuf.sph_comm_unique_id(), sphbuf.sph_comm_unique_id()
    assert len(a) == len(b) == 128 and a != b


def test_no_contracted_fma_in_the_library():
    """The pinned arithmetic is never contracted to FMA: in the
    sm_100a SASS every FFMA/DFMA belongs to an IEEE-754 division sequence
    (div.rn: MUFU.RCP + Newton-Raphson, or its slow-path subroutine)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sphbuf.lib()
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "sass_summary.py"), "test"], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "whole library: **0**" in r.stdout
    os.remove(os.path.join(root, "profiles", "test_sass.md"))
