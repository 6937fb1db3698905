"""The benchmark corpus generator (paper_2111_09219_b200/synth.py) against the
reference's own test-vector encoder: ``synth_ref_batch`` must produce files
byte-identical to oracle_encode(make_test_image(w, h, seed, channels), q,
sampling) (reference oracle.hpp:272-478, tests/helpers.hpp:107-135) run from
oracle/_ref, so the benchmark inputs are the SURVEY.md §8(d) inputs."""
import numpy as np
import pytest

from oracle.oracle import Ref
from paper_2111_09219_b200.synth import synth_ref_batch

CASES = [(500, 375, 1000, 75, "420"), (512, 512, 1, 85, "444"), (97, 33, 7, 90, "422"), (160, 120, 3, 50, "gray"),
         (33, 17, 9, 100, "420"), (8, 8, 11, 1, "444"), (1, 1, 12, 20, "420"), (257, 129, 13, 95, "422"),
         (64, 48, 14, 60, "gray"), (130, 70, 15, 30, "444")]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}x{c[1]}-q{c[3]}-{c[4]}" for c in CASES])
def test_ref_corpus_byte_identical(case):
    w, h, seed, q, s = case
    blob, offs, sizes = synth_ref_batch(1, w, h, seed, q, s)
    mine = blob[offs[0]: offs[0] + sizes[0]].tobytes()
    assert mine == Ref.encode_test_image(w, h, seed, q, s)


def test_ref_corpus_batch_seeds():
    """Batch generation: file i uses seed0 + i (bench.py config 3 seeds 1000...)."""
    blob, offs, sizes = synth_ref_batch(24, 500, 375, 1000, 75, "420", threads=4)
    for i in (0, 5, 23):
        assert blob[offs[i]: offs[i] + sizes[i]].tobytes() == Ref.encode_test_image(500, 375, 1000 + i, 75, "420")


def test_ref_corpus_three_channel_gray():
    """sampling gray with 3-channel pixels: Y from the JFIF conversion."""
    blob, offs, sizes = synth_ref_batch(1, 40, 24, 3, 80, "gray", channels=3)
    assert blob.tobytes() == Ref.encode_test_image(40, 24, 3, 80, "gray", channels=3)


def test_restart_twin_structure():
    """The DRI twin: same frame and tables, DRI = the interval, and restart
    markers RST0..7 cycling inside the scan; the reference rejects it
    (UnsupportedFeature, parser.hpp:299-302)."""
    plain = synth_ref_batch(1, 160, 96, 5, 75, "420")[0].tobytes()
    dri = synth_ref_batch(1, 160, 96, 5, 75, "420", restart_interval=10)[0].tobytes()
    assert dri.count(b"\xff\xdd\x00\x04\x00\x0a") == 1
    sos = dri.index(b"\xff\xda")
    scan = dri[sos:]
    rst = [scan[k + 1] for k in range(len(scan) - 1) if scan[k] == 0xFF and 0xD0 <= scan[k + 1] <= 0xD7]
    assert rst == [0xD0 + k for k in range(5)]  # 10 x 6 MCUs, 10 per interval
    assert Ref.decode(plain).status == 0
    assert Ref.decode(dri).status == 4  # UnsupportedFeature + 1
