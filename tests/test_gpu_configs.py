"""GPU parity at every BASELINE.json configuration (SURVEY.md §8 shape table),
against the reference itself (oracle/_ref, run on all host threads):

  cfg 1  512x512 4:4:4 q85                (test_gpu_parity.test_config_shapes_bit_exact)
  cfg 2  3840x2160 4:2:0 q90              coefficients, sync states, RGB
  cfg 3  4096 x 500x375 4:2:0 q75         the full benchmark corpus, RGB of every file
  cfg 4  16384x16384 4:4:4 q95            coefficients, sync states, RGB; K3 replay on and off
  cfg 5  8192x8192 q50..100 x {4:2:0, 4:4:4, gray} x {no DRI, DRI per MCU row}

Inputs are the §8(d) corpus: oracle_encode(make_test_image(...)) with the
§8(d) seeds, produced by the native generator (paper_2111_09219_b200/synth.py,
byte-identical to the reference encoder: tests/test_synth.py).  DRI files are
the same coefficients with restart markers; the reference rejects DRI
(parser.hpp:299-302), so they must decode to the reference's output of their
DRI-free twin."""
import functools

import numpy as np
import pytest

from oracle.oracle import Ref
from paper_2111_09219_b200.synth import synth_ref_batch

pj = pytest.importorskip("paper_2111_09219_b200")
pytestmark = pytest.mark.gpu

HW = max(1, Ref.hardware_concurrency())


@functools.lru_cache(maxsize=4)
def one_file(w, h, seed, q, s, ri=0):
    blob, offs, sizes = synth_ref_batch(1, w, h, seed, q, s, ri)
    return blob[offs[0]: offs[0] + sizes[0]].tobytes()


def _rgb(buf, inf):
    ch = inf.channels
    pix = buf[: inf.width * inf.height * ch]
    return pix.reshape(inf.height, inf.width, ch) if ch == 3 else pix.reshape(inf.height, inf.width)


def _entropy_parity(b, f, sb=1024):
    """pre-DC zig-zag coefficients and every s_info entry (p, trimmed n, c, z,
    divergent) equal the reference's parallel_entropy_decode."""
    coeffs, ents, meta = Ref.entropy(f, sb=sb, b=256, workers=HW)
    got = b.coefficients(0, pre_dc_zigzag=True)
    assert got.size == coeffs.size
    bad = np.flatnonzero(got != coeffs)
    assert bad.size == 0, f"{bad.size} coefficients differ, first at {bad[:5]}"
    del got, coeffs
    st = b.sync_states(0)
    assert st.shape == ents.shape, (st.shape, ents.shape)
    for col, name in enumerate(("p", "n", "c", "z", "divergent")):
        bad = np.flatnonzero(st[:, col] != ents[:, col])
        assert bad.size == 0, f"sync state {name} differs at {bad[:5]} of {st.shape[0]}"


def test_cfg2_3840x2160_q90_420(decoder):
    f = one_file(3840, 2160, 2, 90, "420")
    assert f == Ref.encode_test_image(3840, 2160, 2, 90, "420")  # the §8(d) file itself
    with decoder.batch([f], pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved) as b:
        assert b.run()[0] == 0
        got = _rgb(b.download()[0], b.infos[0])
        _entropy_parity(b, f)
    ref = Ref.decode(f, rgb=True, workers=HW)
    assert np.array_equal(got, ref.data)


@pytest.fixture(scope="module")
def cfg4():
    f = one_file(16384, 16384, 4, 95, "444")
    ref = Ref.decode(f, rgb=True, workers=HW)
    assert ref.status == 0
    return f, ref.data


@pytest.mark.parametrize("replay", ["1", "0"])
def test_cfg4_16384_q95_444(decoder, cfg4, replay, monkeypatch):
    """1.04 Gbit scan, ~1 M subsequences: K1's long overflow chains and the
    inter-CTA fix-up at scale, K3 replaying K1's symbols (1) or re-decoding (0)."""
    monkeypatch.setenv("PJG_REPLAY", replay)
    f, ref = cfg4
    with decoder.batch([f], pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved) as b:
        assert b.run()[0] == 0
        got = _rgb(b.download()[0], b.infos[0])
        bad = np.count_nonzero(got != ref)
        del got
        assert bad == 0, f"{bad} RGB bytes differ"
        _entropy_parity(b, f)


def test_cfg3_full_corpus_4096(decoder):
    """The benchmark's batch (bench.py --config 3): every one of the 4096 files
    RGB-exact against the reference's decode_batch + upsample_and_convert."""
    blob, offs, sizes = synth_ref_batch(4096, 500, 375, 1000, 75, "420")
    for i in (0, 4095):
        assert blob[offs[i]: offs[i] + sizes[i]].tobytes() == Ref.encode_test_image(500, 375, 1000 + i, 75, "420")
    with decoder.batch((blob, offs, sizes), pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved) as b:
        st = b.run()
        assert (st == 0).all()
        outs = b.download()
    files = [blob[o: o + s].tobytes() for o, s in zip(offs, sizes)]
    rst, routs = Ref.decode_batch_rgb(files, HW)
    assert (rst == 0).all()
    bad = [i for i in range(len(files)) if not np.array_equal(outs[i][: routs[i].size], routs[i])]
    assert not bad, f"{len(bad)} images differ: {bad[:10]}"


CFG5 = [(q, s) for s in ("420", "444", "gray") for q in (50, 60, 70, 75, 80, 85, 90, 95, 100)]


@pytest.mark.parametrize("q,s", CFG5, ids=[f"q{q}-{s}" for q, s in CFG5])
def test_cfg5_8192_sweep(decoder, q, s):
    """One sweep point: the plain file and its DRI twin (one restart interval per
    MCU row) both decode to the reference's RGB of the plain file."""
    plain = one_file(8192, 8192, 5000 + q, q, s)
    mcus_x = 8192 // (16 if s == "420" else 8)
    dri = one_file(8192, 8192, 5000 + q, q, s, mcus_x)
    ref = Ref.decode(plain, rgb=True, workers=HW)
    assert ref.status == 0
    with decoder.batch([plain], pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved) as b:
        assert b.run()[0] == 0
        got = _rgb(b.download()[0], b.infos[0])
        assert np.array_equal(got, ref.data), int((got != ref.data).sum())
    with decoder.batch([dri], pj.DecodeConfig(restart_intervals=True), pj.OutputColorspace.RGBInterleaved) as b:
        assert b.run()[0] == 0
        got = _rgb(b.download()[0], b.infos[0])
        assert np.array_equal(got, ref.data), int((got != ref.data).sum())
