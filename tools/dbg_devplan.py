"""Debug: host- vs device-planned batch on the mixed-table thumbnail batch of
tests/test_gpu_devplan.py; per differing image: which plan matches the oracle,
first differing byte, image geometry and table ids."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import paper_2111_09219_b200 as pj  # noqa: E402
from oracle.oracle import Orc  # noqa: E402
from paper_2111_09219_b200.synth import synth_batch  # noqa: E402

files = []
for q, smp, seed in ((50, "420", 1), (75, "444", 2), (95, "gray", 3), (85, "422", 4)):
    blob, offs, sizes = synth_batch(300, 40, 24, 9000 + 1000 * seed, q, smp)
    files += [blob[int(o): int(o) + int(s)].tobytes() for o, s in zip(offs, sizes)]
f = files[0]
k = f.index(b"\xff\xdb")
ln = (f[k + 2] << 8) | f[k + 3]
seg = f[k + 4: k + 2 + ln]
out, j = bytearray(), 0
while j < len(seg):
    pq = seg[j]
    vals = seg[j + 1: j + 65]
    out += bytes([0x10 | (pq & 15)]) + b"".join(bytes([0, v]) for v in vals)
    j += 65
files.append(f[:k] + b"\xff\xdb" + (len(out) + 2).to_bytes(2, "big") + bytes(out) + f[k + 2 + ln:])
order = np.random.default_rng(9).permutation(len(files))
origin = [int(i) for i in order]
files = [files[i] for i in order]
dec = pj.Decoder(0)
for mode in (pj.OutputColorspace.RGBInterleaved, pj.OutputColorspace.YCbCrPlanes, pj.OutputColorspace.Grayscale,
             pj.OutputColorspace.YCbCrPlanes):
    res = []
    for dp in (False, True):
        with dec.batch(files, pj.DecodeConfig(), mode, device_plan=dp) as b:
            st = b.run()
            res.append((st.copy(), b.download()))
    bad = [i for i in range(len(files)) if not np.array_equal(res[0][1][i], res[1][1][i])]
    print(mode, "differing images:", len(bad), bad[:20])
    for i in bad[:6]:
        h, d = res[0][1][i], res[1][1][i]
        fd = int(np.argmax(h != d))
        print(f"  img {i} (orig {origin[i]}) first diff byte {fd} of {h.size} ndiff {int((h != d).sum())} "
              f"sizes {h.size} {d.size} status {res[0][0][i]} {res[1][0][i]}")
for i in bad[:8]:
    want = Orc.decode(files[i], rgb=True).data.reshape(-1)
    h, d = res[0][1][i][: want.size], res[1][1][i][: want.size]
    fd = int(np.argmax(h != d))
    print(f"img {i} (orig {origin[i]}) host_ok={np.array_equal(h, want)} dev_ok={np.array_equal(d, want)} "
          f"first diff byte {fd} of {want.size} ndiff {int((h != d).sum())} status {res[0][0][i]} {res[1][0][i]}")
# single-file device plan of the bad ones
for i in bad[:4]:
    with dec.batch([files[i]], pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved, device_plan=True) as b:
        b.run()
        o = b.download()[0]
    want = Orc.decode(files[i], rgb=True).data.reshape(-1)
    print("single device plan", i, np.array_equal(o[: want.size], want))
# sub-batches: find the smallest prefix that reproduces
for n in (16, 64, 256, 600, 1000, len(files)):
    sub = files[:n]
    r = []
    for dp in (False, True):
        with dec.batch(sub, pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved, device_plan=dp) as b:
            b.run()
            r.append(b.download())
    nb = [i for i in range(n) if not np.array_equal(r[0][i], r[1][i])]
    print("prefix", n, "differing", len(nb), nb[:10])
