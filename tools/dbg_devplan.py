import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2111_09219_b200 as pj
from tests.corpus import ref_jpeg
good = ref_jpeg(48, 40, 3, 80, "420")
sos = good.index(b"\xff\xda")
cases = [good[:sos] + b"\xff\xdd\x00\x04\x00\x10" + good[sos:], good[:sos] + b"\xff\xdc\x00\x04\x00\x10" + good[sos:], good]
dec = pj.Decoder(0)
for dp in (False, True):
    with dec.batch(cases, pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved, device_plan=dp) as b:
        st = b.run(); b.infos
        print("device_plan", dp, "status", list(st), "header", b.header_status)
for c in cases:
    with dec.batch([c], pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved, device_plan=True) as b:
        print("single", list(b.run()), b.infos and b.header_status)
