"""Short driver for ncu: decode one batch config `reps` times (no timing)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2111_09219_b200 as pj  # noqa: E402
from bench import CONFIGS, make_corpus  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="3")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--sb", type=int, default=1024)
a = ap.parse_args()
blob, offs, sizes = make_corpus(a.config)
dec = pj.Decoder(0)
ri = CONFIGS[a.config][5]
b = dec.batch((blob, offs, sizes), pj.DecodeConfig(subsequence_bits=a.sb, restart_intervals=ri > 0),
              pj.OutputColorspace.RGBInterleaved)
b.upload()
for _ in range(a.reps):
    st = b.decode().synchronize()
    assert (st == 0).all()
print("stages", b.stage_times(), b.sync_stats())
