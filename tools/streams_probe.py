"""Batch step as k concurrent parts on k contexts (diagnostics for bench.py's 2)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2111_09219_b200 as pj  # noqa: E402
from bench import make_corpus  # noqa: E402

blob, offs, sizes = make_corpus("3")
n = len(sizes)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for k in (1, 2, 4, 8):
    decs = [pj.Decoder(0) for _ in range(k)]
    parts = []
    for j in range(k):
        lo, hi = n * j // k, n * (j + 1) // k
        b = decs[j].batch((blob, offs[lo:hi], sizes[lo:hi]), pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved)
        b.upload()
        b.decode().synchronize()
        parts.append(b)
    streams = [torch.cuda.ExternalStream(d.stream(), device=torch.device("cuda", 0)) for d in decs]
    times = []
    for rep in range(8):
        with torch.cuda.stream(streams[0]):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(streams[0])
        for s in streams[1:]:
            s.wait_event(e0)
        for b in parts:
            b.decode()
        for s in streams[1:]:
            j = torch.cuda.Event()
            j.record(s)
            streams[0].wait_event(j)
        with torch.cuda.stream(streams[0]):
            e1.record(streams[0])
        for b in parts:
            b.synchronize()
        if rep >= 3:
            times.append(e0.elapsed_time(e1))
    print(f"k={k}: {sum(times) / len(times):.3f} ms per step")
    for b in parts:
        b.close()
    for d in decs:
        d.close()
