"""Stage times of a thumbnail batch (diagnostics)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_09219_b200 as pj  # noqa: E402
from paper_2111_09219_b200.synth import synth_batch  # noqa: E402

n, w, h = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (65536, 32, 32)))
blob, offs, sizes = synth_batch(n, w, h, 777, 75, "420")
dec = pj.Decoder(0)
for rep in range(3):
    t0 = time.perf_counter()
    b = dec.batch((blob, offs, sizes), pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved)
    t1 = time.perf_counter()
    b.upload()
    st = b.decode().synchronize()
    t2 = time.perf_counter()
    stt = b.stage_times()
    b.close()
print(f"{n} x {w}x{h}: create {1e3*(t1-t0):.2f} ms, upload+decode+sync {1e3*(t2-t1):.2f} ms, {stt}")
