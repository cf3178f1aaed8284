"""The bounds-asserting debug build (build.py --debug: -DSPHBUF_DEBUG, device-side
SPH_CHECK asserts on slot, source, candidate, run and output indices) under the
sanitize driver: compute-sanitizer is closed on the GPU pool, so this is the
memory-safety check of the kernels, every one of them exercised (the cell-list
build in both scan forms, the update, both compaction modes with the copy-engine
move, moving ports, port drivers, the loopback communicator)."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.gpu
@pytest.mark.slow
def test_sanitize_run_under_debug_build():
    env = dict(os.environ, SPHBUF_DEBUG="1")
    r = subprocess.run([sys.executable, os.path.join(HERE, "sanitize_run.py")], env=env, capture_output=True,
                       text=True, timeout=1800)
    assert r.returncode == 0 and "all lock-step checks passed" in r.stdout, r.stdout[-3000:] + r.stderr[-5000:]
