"""Host planner vs device planner (pjg_batch_create_device), wall clock per
batch from pinned host files to decoded output in HBM: create (+upload) +
decode + synchronize.  Usage: python tools/devplan_probe.py [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_09219_b200 as pj  # noqa: E402
from paper_2111_09219_b200.synth import synth_batch, synth_ref_batch  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cases = {
    "65536 x 32x32 420 q75": lambda: synth_batch(65536, 32, 32, 1, 75, "420"),
    "16384 x 64x64 420 q75": lambda: synth_batch(16384, 64, 64, 2, 75, "420"),
    "cfg3 4096 x 500x375 420 q75": lambda: synth_ref_batch(4096, 500, 375, 1000, 75, "420", 0),
}
dec = pj.Decoder(0)
for name, mk in cases.items():
    blob, offs, sizes = mk()
    t = torch.empty(blob.size + 64, dtype=torch.uint8).pin_memory()
    pinned = t.numpy()[: blob.size]
    pinned[:] = blob
    res = {}
    for dp in (False, True):
        ts = []
        for r in range(reps + 2):
            t0 = time.perf_counter()
            b = dec.batch((pinned, offs, sizes), pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved, device_plan=dp)
            b.upload()
            b.decode()
            st = b.synchronize()
            t1 = time.perf_counter()
            assert (st == 0).all()
            b.close()
            if r >= 2:
                ts.append(t1 - t0)
        res["device" if dp else "host"] = (np.median(ts) * 1e3, min(ts) * 1e3)
    print(f"{name:32s} host plan {res['host'][0]:8.3f} ms (best {res['host'][1]:.3f})   "
          f"device plan {res['device'][0]:8.3f} ms (best {res['device'][1]:.3f})", flush=True)
dec.close()
