"""GPU parity on forged inputs no image encoder produces (tests/forge.py):
16-bit quantisers up to 65535, maximum-magnitude coefficients, DC predictors
wrapping int16.  They drive K4's exact-FP64 "big unit" branch (S >= 2^18:
every sample replayed from the int32 dequantised coefficients) and the DC
paths at their limits; checked bit-exactly against the reference
(oracle/_ref): entropy-stage coefficients, planes and RGB."""
import numpy as np
import pytest

from oracle.oracle import Ref
from tests.forge import data_units, forge

pj = pytest.importorskip("paper_2111_09219_b200")
pytestmark = pytest.mark.gpu


def _blocks(kind, n, rng):
    b = np.zeros((n, 64), np.int64)
    if kind == "max":  # every coefficient at its category limit, alternating signs
        b[:, 0] = np.where(np.arange(n) % 2 == 0, 2047, -2047)
        b[:, 1:] = np.where((np.arange(63) + np.arange(n)[:, None]) % 2 == 0, 1023, -1023)
    elif kind == "wide":  # sparse large AC, random DC differences (wrapping int16)
        b[:, 0] = rng.integers(-2047, 2048, n)
        for i in range(n):
            k = rng.integers(1, 64, size=int(rng.integers(0, 10)))
            b[i, k] = rng.integers(-1023, 1024, k.size)
    elif kind == "border":  # S = sum w_u w_v |F| straddling 2^18
        b[:, 0] = rng.integers(-40, 41, n)
        for i in range(n):
            k = rng.integers(1, 64, size=int(rng.integers(1, 6)))
            b[i, k] = rng.integers(-700, 701, k.size)
    elif kind == "dcwrap":  # DC-only units, predictor climbing through +-32768
        b[:, 0] = 2047
        b[::7, 0] = -2047
    return b


CASES = [("max", "444", 65535), ("wide", "420", 3000), ("wide", "444", 65535), ("border", "420", 400),
         ("border", "422", 255), ("dcwrap", "gray", 255), ("dcwrap", "420", 9000), ("wide", "gray", 20000)]


def _forge(kind, samp, qmax, seed):
    rng = np.random.default_rng(seed)
    W, H = {"gray": (136, 72), "444": (96, 64), "422": (112, 64), "420": (144, 80)}[samp]
    n = data_units(W, H, samp)
    lo = max(1, qmax // 3)
    quant = {0: [int(x) for x in rng.integers(lo, qmax + 1, 64)], 1: [int(x) for x in rng.integers(lo, qmax + 1, 64)]}
    return forge(W, H, samp, quant, _blocks(kind, n, rng))


@pytest.mark.parametrize("case", CASES, ids=[f"{k}-{s}-q{q}" for k, s, q in CASES])
def test_forged_extremes_bit_exact(decoder, case):
    kind, samp, qmax = case
    f = _forge(kind, samp, qmax, 17 + CASES.index(case))
    ref_rgb = Ref.decode(f, rgb=True)
    ref_pl = Ref.decode(f, rgb=False)
    assert ref_rgb.status == 0 and ref_pl.status == 0
    coeffs, _, _ = Ref.entropy(f)
    for out in (pj.OutputColorspace.RGBInterleaved, pj.OutputColorspace.YCbCrPlanes):
        with decoder.batch([f], pj.DecodeConfig(), out) as b:
            st = b.run()
            assert st[0] == 0
            got = b.download()[0]
            want = ref_rgb if out == pj.OutputColorspace.RGBInterleaved else ref_pl
            assert np.array_equal(got[: want.data.size], want.data.reshape(-1)), \
                (case, int((got[: want.data.size] != want.data.reshape(-1)).sum()))
            assert np.array_equal(b.coefficients(0, pre_dc_zigzag=True), coeffs)
            stats = b.sync_stats()
    if kind in ("max", "wide"):
        # the exact-FP64 unit path ran: whole units replayed (64 samples each)
        assert stats["k4_fp64_replayed_samples"] >= 64, stats


def test_forged_extremes_one_batch(decoder):
    """All forged cases in one batch (mixed quantisers, samplings, K4 paths)."""
    files = [_forge(k, s, q, 100 + i) for i, (k, s, q) in enumerate(CASES)]
    with decoder.batch(files, pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved) as b:
        st = b.run()
        assert (st == 0).all(), st
        outs = b.download()
    for i, f in enumerate(files):
        ref = Ref.decode(f, rgb=True)
        assert np.array_equal(outs[i][: ref.data.size], ref.data.reshape(-1)), CASES[i]
