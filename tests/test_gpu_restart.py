"""Restart intervals (DRI + RST0-7): an extension beyond the reference, which
rejects DRI != 0 (parser.hpp:299-302).  Parity comes from DRI twins
(SURVEY.md §8(f1)): the synthetic encoder (csrc/synth.cpp) emits the same
quantised coefficients with and without restart markers, so the GPU's decode
of the DRI file must equal the reference's decode of its DRI-free twin."""
import numpy as np
import pytest

from oracle.oracle import Ref
from paper_2111_09219_b200.synth import synth_batch

pj = pytest.importorskip("paper_2111_09219_b200")
pytestmark = pytest.mark.gpu

DRI = pj.DecodeConfig(restart_intervals=True)


def _twins(w, h, q, s, ri, seed):
    a = synth_batch(1, w, h, seed, q, s, 0)
    b = synth_batch(1, w, h, seed, q, s, ri)
    plain = a[0][a[1][0]: a[1][0] + a[2][0]].tobytes()
    dri = b[0][b[1][0]: b[1][0] + b[2][0]].tobytes()
    return plain, dri


def _rgb(buf, inf):
    ch = inf.channels
    pix = buf[: inf.width * inf.height * ch]
    return pix.reshape(inf.height, inf.width, ch) if ch == 3 else pix.reshape(inf.height, inf.width)


CASES = [(64, 48, 75, "420", 1), (200, 120, 85, "444", 3), (333, 257, 90, "422", 7), (500, 375, 75, "420", 32),
         (801, 61, 60, "gray", 5), (1024, 512, 95, "420", 64), (640, 480, 80, "444", 40), (96, 96, 50, "420", 1000)]


@pytest.mark.parametrize("replay", ["default", "on"])
@pytest.mark.parametrize("sb", [1024, 128])
def test_restart_twins_bit_exact(decoder, sb, replay, monkeypatch):
    if replay == "on":  # K3 replaying K1's kept symbols inside restart-interval segments
        monkeypatch.setenv("PJG_REPLAY", "1")
        monkeypatch.setenv("PJG_SMEM_TABLES", "0")
    pairs = [(c, *_twins(*c, 7000 + k)) for k, c in enumerate(CASES)]
    cfg = pj.DecodeConfig(subsequence_bits=sb, restart_intervals=True)
    with decoder.batch([p for _, p, _ in pairs], pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved) as b0:
        assert (b0.run() == 0).all()
        twin_coefs = [b0.coefficients(i, pre_dc_zigzag=False) for i in range(len(pairs))]
    with decoder.batch([d for _, _, d in pairs], cfg, pj.OutputColorspace.RGBInterleaved) as b:
        st = b.run()
        assert (st == 0).all(), st
        outs = b.download()
        for i, (case, plain, dri) in enumerate(pairs):
            assert plain != dri
            ref = Ref.decode(plain, rgb=True)
            assert ref.status == 0
            got = _rgb(outs[i], b.infos[i])
            assert np.array_equal(got, ref.data), (case, int((got != ref.data).sum()))
            # absolute (post-DC) coefficients equal the twin's
            assert np.array_equal(b.coefficients(i, pre_dc_zigzag=False), twin_coefs[i]), case


def test_restart_twins_mixed_with_plain_files(decoder):
    """DRI and DRI-free files in one batch; the DRI-free ones keep the
    reference's partition (sync states equal the reference's)."""
    plain1, dri1 = _twins(320, 240, 85, "420", 20, 11)
    plain2, _ = _twins(200, 200, 75, "444", 1, 12)
    with decoder.batch([plain1, dri1, plain2], DRI, pj.OutputColorspace.RGBInterleaved) as b:
        st = b.run()
        assert (st == 0).all(), st
        outs = b.download()
        for i, f in ((0, plain1), (1, plain1), (2, plain2)):
            assert np.array_equal(_rgb(outs[i], b.infos[i]), Ref.decode(f, rgb=True).data), i
        st0 = b.sync_states(0)
        coeffs, ents, meta = Ref.entropy(plain1, sb=1024, b=4)
        assert np.array_equal(st0[:, 1], ents[:, 1])


def test_restart_rejected_by_default(decoder):
    _, dri = _twins(64, 64, 75, "420", 2, 3)
    ref = Ref.decode(dri, rgb=True)
    assert ref.status == int(pj.Errc.UnsupportedFeature) + 1
    with decoder.batch([dri], pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved) as b:
        assert b.run()[0] == ref.status


def _rst_positions(f):
    sos = f.index(b"\xff\xda")
    scan0 = sos + 2 + ((f[sos + 2] << 8) | f[sos + 3])
    return [i for i in range(scan0, len(f) - 1) if f[i] == 0xFF and 0xD0 <= f[i + 1] <= 0xD7]


def test_restart_corrupt_markers(decoder):
    _, dri = _twins(128, 64, 75, "420", 4, 9)
    pos = _rst_positions(dri)
    assert len(pos) == (8 * 4) // 4 - 1
    bad_num = bytearray(dri)
    bad_num[pos[2] + 1] ^= 0x01  # RST numbering out of sequence
    missing = dri[: pos[1]] + dri[pos[1] + 2:]  # one marker dropped
    extra = dri[: pos[-1]] + b"\xff\xd0" + dri[pos[-1]:]  # one marker too many
    with decoder.batch([bytes(bad_num), missing, extra, dri], DRI, pj.OutputColorspace.RGBInterleaved) as b:
        st = b.run()
    assert st[0] != 0 and st[1] != 0 and st[2] != 0, st
    assert st[3] == 0


def test_restart_large_single_image(decoder):
    """A single large DRI scan (K0's 32 KB-tile path, many intervals)."""
    plain, dri = _twins(1536, 1024, 95, "444", 13, 21)
    with decoder.batch([dri], DRI, pj.OutputColorspace.RGBInterleaved) as b:
        assert b.run()[0] == 0
        got = _rgb(b.download()[0], b.infos[0])
    assert np.array_equal(got, Ref.decode(plain, rgb=True).data)
