import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2111_09219_b200 as pj
from paper_2111_09219_b200.synth import synth_batch
blob, offs, sizes = synth_batch(65536, 32, 32, 777, 75, "420")
dec = pj.Decoder(0)
for rep in range(4):
    b = dec.batch((blob, offs, sizes), pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved)
    if rep >= 2: time.sleep(0.05)
    t0 = time.perf_counter(); b.upload(); st = b.decode().synchronize(); t1 = time.perf_counter()
    print(rep, f"{1e3*(t1-t0):.2f} ms", f"upload {b.stage_times().upload:.3f}")
    b.close()
