"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref: the
unmodified pjpeg headers compiled in place), so the CPU suite can pin the C
restatement and the GPU suite can check the product on boxes where the
reference sources are absent.  Re-run with `python tests/golden/make_golden.py`.

Corpus = the reference acceptance corpus (acceptance.cpp:76-102): 4 sizes x
q{92,75,50,20} x {4:4:4, 4:2:2, 4:2:0, gray}, reference encoder
(oracle_encode over make_test_image), plus the worked example.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Ref, example_jpeg  # noqa: E402
from tests.corpus import ACCEPTANCE  # noqa: E402


def main():
    out = {}
    names = []
    files = [("example", example_jpeg())]
    for k, (w, h, q, s) in enumerate(ACCEPTANCE[:64]):
        files.append((f"acc{k:02d}_{w}x{h}_q{q}_{s}", Ref.encode_test_image(w, h, 1000 + k, q, s)))
    for name, f in files:
        names.append(name)
        out[f"{name}.jpg"] = np.frombuffer(f, np.uint8)
        rgb = Ref.decode(f, rgb=True)
        planes = Ref.decode(f, rgb=False)
        assert rgb.status == 0 and planes.status == 0, name
        out[f"{name}.rgb"] = rgb.data.reshape(-1)
        out[f"{name}.geom"] = np.array([rgb.width, rgb.height, rgb.channels, planes.nplanes] +
                                       [v for d in planes.plane_dims for v in d], np.int64)
        out[f"{name}.planes"] = planes.data.reshape(-1)
        sbs = [32] if name == "example" else [128, 1024]
        for sb in sbs:
            coeffs, ents, meta = Ref.entropy(f, sb=sb, b=4)
            out[f"{name}.coeffs"] = coeffs
            out[f"{name}.ents{sb}"] = ents.astype(np.int64)
            N = ents.shape[0]
            bnd = np.arange(1, N, dtype=np.uint64) * sb
            st, valid, _, _ = Ref.trace(f, bnd)
            out[f"{name}.trace{sb}"] = st.astype(np.int64)
            out[f"{name}.valid{sb}"] = valid.astype(np.uint8)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "reference_corpus.npz"), **out)
    print("wrote", len(names), "files;", os.path.getsize(os.path.join(HERE, "reference_corpus.npz")), "bytes")


if __name__ == "__main__":
    main()
