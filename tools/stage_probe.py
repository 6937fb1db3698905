"""Stage times of one config-3 batch decode (diagnostics; statuses ignored)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_09219_b200 as pj  # noqa: E402
from bench import make_corpus  # noqa: E402
_, blob, offs, sizes = make_corpus(sys.argv[1] if len(sys.argv) > 1 else "3", 0, pinned=False)
dec = pj.Decoder(0)
b = dec.batch((blob, offs, sizes), pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved)
b.upload()
for _ in range(4):
    b.decode()
    b.synchronize()
print(b.stage_times())
