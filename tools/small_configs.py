#!/usr/bin/env python
"""µs per update of the small configurations (CUDA-graph replay and stream launch),
the bench's sweep alone.  SPHBUF_LIB=<other build> gives an A/B on one box.

    python tools/small_configs.py C1,C2,C3
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench


def main():
    names = tuple((sys.argv[1] if len(sys.argv) > 1 else "C1,C2,C3").split(","))
    out = bench.sweep_configs(torch.device("cuda", 0), names=names, replays=200)
    print(json.dumps({k: {"graph_us": v["us_per_update_graph"], "stream_us": v["us_per_update_stream"]}
                      for k, v in out.items()}))


if __name__ == "__main__":
    main()
