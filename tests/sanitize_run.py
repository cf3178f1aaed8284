"""Small driver for compute-sanitizer runs (memcheck / racecheck / synccheck /
initcheck, one tool per invocation): a few updates of C1e, C2 and a small 3-D
junction through the C ABI, in both compaction modes, plus the moving-port,
port-driver and loopback-slab lock-step tests on a few updates, each checked
bit-exactly against the oracle.  compute-sanitizer is closed on the GPU pool, so
tests/test_debug_build.py runs this under the bounds-asserting debug build
(SPHBUF_DEBUG=1) instead.

    compute-sanitizer --tool memcheck python tests/sanitize_run.py
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

from paper_2406_16786_b200 import inputs  # noqa: E402
from parity_util import lockstep  # noqa: E402
from test_drivers import test_drivers_gpu_parity  # noqa: E402
from test_motion import test_rotating_port_3d_gpu_parity, test_sprinkler_gpu_parity  # noqa: E402


def main():
    lockstep(inputs.make("C1e"), 3, check_every=1)
    lockstep(inputs.make("C1e"), 3, check_every=1, fused=True, deferred=True)
    lockstep(inputs.make("C2"), 6, check_every=3)
    lockstep(inputs.make("C2"), 6, check_every=3, fused=True, deferred=True)
    lockstep(inputs.c4(scale=0.25, nports=4, n_updates=4), 3, check_every=1)
    test_sprinkler_gpu_parity(n_steps=12)          # moving ports (K9, K10)
    test_rotating_port_3d_gpu_parity(n_steps=4)
    test_drivers_gpu_parity(n_updates=4)           # port drivers (K11)
    from test_dist import test_loopback_slabs_match_oracle
    test_loopback_slabs_match_oracle(2, True)      # loopback communicator, migration, carried keys
    print("sanitize_run: all lock-step checks passed")


if __name__ == "__main__":
    main()
