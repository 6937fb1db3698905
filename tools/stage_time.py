"""Mean per-stage device times of one batch config (CUDA events, L2 flushed
between decodes).  Usage: PJG_LIB=... python tools/stage_time.py [config] [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_09219_b200 as pj  # noqa: E402
from bench import CONFIGS, make_corpus  # noqa: E402

cfg_key = sys.argv[1] if len(sys.argv) > 1 else "3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
blob, offs, sizes = make_corpus(cfg_key)
dec = pj.Decoder(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
b = dec.batch((blob, offs, sizes), pj.DecodeConfig(restart_intervals=CONFIGS[cfg_key][5] > 0),
              pj.OutputColorspace.RGBInterleaved)
b.upload()
runs, steps = [], []
ext = torch.cuda.ExternalStream(dec.stream(), device=torch.device("cuda", 0))
for r in range(reps + 3):
    flush.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    b.decode()
    e1.record(ext)
    st = b.synchronize()
    assert (st == 0).all()
    if r >= 3:
        runs.append(b.stage_times())
        steps.append(e0.elapsed_time(e1))
keys = ("unstuff", "sync", "scan", "write", "idct")
env = {k: v for k, v in os.environ.items() if k.startswith("PJG_")}
print(json.dumps({"lib": os.environ.get("PJG_LIB", "libpjg.so"), "config": cfg_key, "env": env,
                  "step_ms": round(float(np.median(steps)), 4),
                  **{k: round(float(np.mean([getattr(x, k) for x in runs])), 4) for k in keys},
                  "stats": b.sync_stats()}))
