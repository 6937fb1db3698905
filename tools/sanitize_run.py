"""Small decodes for compute-sanitizer (racecheck / synccheck / memcheck):
the spin-wait lookbacks of K0, K1 and K2 run across many CTAs, images and
restart intervals.  Usage: compute-sanitizer --tool racecheck python
tools/sanitize_run.py  (exit 0 = every decode bit-exact vs the oracle)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2111_09219_b200 as pj  # noqa: E402
from oracle.oracle import Orc, Ref  # noqa: E402
from paper_2111_09219_b200.synth import synth_ref_batch  # noqa: E402

cases = [
    # (n, w, h, seed, q, sampling, restart interval, sb)
    (24, 500, 375, 1000, 75, "420", 0, 1024),   # batch: K0 multi-tile lookback, K1 CTAs spanning images
    (1, 1024, 768, 7, 95, "444", 0, 256),        # one image, many K1 CTAs (inter-CTA chaining, K1c)
    (2, 640, 480, 9, 90, "420", 40, 512),        # restart intervals: K0 RST strip, K0b segments
    (3, 333, 211, 11, 60, "gray", 0, 128),       # ragged, gray
    (2, 384, 64, 15, 80, "gray", 0, 1024),       # gray 192-pixel K4 tiles, 16-byte Y stores
    (1, 512, 384, 13, 100, "444", 0, 1024),      # > 128 scan bits per unit: the dense K3 -> K4 interface
]
dec = pj.Decoder(0)
for n, w, h, seed, q, s, ri, sb in cases:
    blob, offs, sizes = synth_ref_batch(n, w, h, seed, q, s, ri)
    files = [blob[o: o + z].tobytes() for o, z in zip(offs, sizes)]
    cfg = pj.DecodeConfig(subsequence_bits=sb, restart_intervals=ri > 0)
    with dec.batch(files, cfg, pj.OutputColorspace.RGBInterleaved) as b:
        st = b.run()
        assert (st == 0).all(), st
        outs = b.download()
    if ri == 0:
        for i, f in enumerate(files):
            want = Orc.decode(f, rgb=True)
            assert np.array_equal(outs[i][: want.data.size], want.data.reshape(-1)), (n, w, h, i)
    print(f"ok {n}x{w}x{h} q{q} {s} dri={ri} sb={sb}")
# the device-side planner (pjg_batch_create_device: parse, dedup spin-waits,
# layout scans, table builds) on a mixed-table batch
blob, offs, sizes = synth_ref_batch(12, 120, 90, 300, 80, "444")
blob2, offs2, sizes2 = synth_ref_batch(12, 96, 64, 400, 60, "420")
files = [blob[o: o + z].tobytes() for o, z in zip(offs, sizes)] + [blob2[o: o + z].tobytes() for o, z in zip(offs2, sizes2)]
with dec.batch(files, pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved, device_plan=True) as b:
    st = b.run()
    assert (st == 0).all(), st
    outs = b.download()
for i, f in enumerate(files):
    want = Orc.decode(f, rgb=True)
    assert np.array_equal(outs[i][: want.data.size], want.data.reshape(-1)), ("devplan", i)
print("ok device-planned mixed batch")
# corrupt scans: K1x's reference-exact replay of failed images next to valid ones
good = files[0]
sos = good.index(b"\xff\xda")
bad = [good[: sos + 40], good[: sos + 20] + bytes(range(7, 200)) + good[sos + 200:], good]
with dec.batch(bad, pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved) as b:
    st = b.run()
for i, f in enumerate(bad):
    want = Ref.decode(f, rgb=True)  # the reference itself (oracle/_ref, prebuilt)
    assert int(st[i]) == want.status, (i, int(st[i]), want.status)
print("ok corrupt scans (statuses equal the reference's)")
dec.close()
print("sanitize_run: all decodes ok")
