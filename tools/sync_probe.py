"""Sync-stage time and K1 statistics for one config (diagnostics)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_09219_b200 as pj  # noqa: E402
from bench import make_corpus  # noqa: E402
cfgname = sys.argv[1] if len(sys.argv) > 1 else "3"
_, blob, offs, sizes = make_corpus(cfgname, 0, pinned=False)
dec = pj.Decoder(0)
b = dec.batch((blob, offs, sizes), pj.DecodeConfig(subsequence_bits=int(os.environ.get("SB", "1024"))), pj.OutputColorspace.RGBInterleaved)
b.upload()
for _ in range(4):
    b.decode()
    st = b.synchronize()
t = b.stage_times()
print(f"cfg {cfgname}: ok={int((st == 0).sum())}/{len(st)} sync {t.sync:.3f} write {t.write:.3f} idct {t.idct:.3f} ms",
      b.sync_stats())
