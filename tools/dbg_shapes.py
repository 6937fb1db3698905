import sys, numpy as np
sys.path.insert(0, '.')
import paper_2111_09219_b200 as pj
from oracle.oracle import Ref, Orc
from tests.corpus import ref_jpeg
for shape in [(512, 512, 85, "444", 1), (500, 375, 75, "420", 1000), (1023, 769, 90, "420", 5), (333, 257, 95, "422", 6), (801, 601, 60, "gray", 7), (256, 64, 85, "444", 3), (128, 8, 85, "444", 3)]:
    w, h, q, s, seed = shape
    f = ref_jpeg(w, h, seed, q, s)
    dec = pj.Decoder(0)
    with dec.batch([f], pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved) as b:
        st = b.run()
        ch = b.infos[0].channels
        got = b.download()[0][: w * h * ch].reshape(h, w, ch) if ch == 3 else b.download()[0][: w * h].reshape(h, w)
        stats = b.sync_stats()
    ref = Ref.decode(f, rgb=True).data
    bad = np.argwhere(got != ref)
    print(shape, "status", st, "mismatches", len(bad), stats["k4_fp64_replayed_samples"])
    if len(bad):
        ys, xs = bad[:, 0], bad[:, 1]
        print("  rows", np.unique(ys // 8)[:10], "cols(64px tiles)", np.unique(xs // 64)[:10], "x%64", np.unique(xs % 64)[:20])
        for k in range(min(5, len(bad))):
            y, x = bad[k][:2]
            print("  ", y, x, got[y, x], ref[y, x])
    dec.close()
