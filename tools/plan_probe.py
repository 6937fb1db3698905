"""Host batch planning (pjg_batch_create_blob: header parse, tables, layout)
and the one H2D of the compressed bytes, per batch size, on config 3's
corpus — the exposed head of bench.py's pipelined metric of record.
Usage: python tools/plan_probe.py"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2111_09219_b200 as pj
from bench import make_corpus, pinned_copy
blob, offs, sizes = make_corpus("3")
_, pblob = pinned_copy(blob)
dec = pj.Decoder(0)
for n in (4096, 1024, 256):
    ts_c, ts_u = [], []
    for r in range(12):
        t0 = time.perf_counter()
        b = dec.batch((pblob, offs[:n], sizes[:n]), pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved)
        t1 = time.perf_counter()
        b.upload(); torch.cuda.synchronize(); b.synchronize() if False else None
        t2 = time.perf_counter()
        b.close()
        if r >= 2: ts_c.append(t1 - t0); ts_u.append(t2 - t1)
    print(n, "create %.3f ms" % (1e3 * np.median(ts_c)), "upload(sync) %.3f ms" % (1e3 * np.median(ts_u)), "cpus", os.cpu_count())
