"""Device-side planning (csrc/devplan.cu): the JFIF marker
walk, table dedup/construction and batch layout as kernels
(pjg_batch_create_device).  Bar: the same outcome as the host planner — which
the other GPU tests pin to the reference — for every file: header Errc
(parser.hpp:264-347 precedence, build_table errors deferred past the scan
checks, pipeline.hpp:107-112), image infos, coefficients, sync states and
RGB; plus direct reference checks on the valid files."""
import numpy as np
import pytest

from oracle.oracle import Orc, Ref
from tests.corpus import acceptance_corpus, ref_jpeg
from tests.test_gpu_fuzz import _mutants

pj = pytest.importorskip("paper_2111_09219_b200")
pytestmark = pytest.mark.gpu


def _both(decoder, files, cfg=None, output=None):
    """(statuses, infos, outputs) of the host- and the device-planned batch."""
    cfg = cfg or pj.DecodeConfig()
    output = pj.OutputColorspace.RGBInterleaved if output is None else output
    res = []
    for dp in (False, True):
        with decoder.batch(files, cfg, output, device_plan=dp) as b:
            st = b.run()
            infos = b.infos
            hs = list(b.header_status)
            outs = b.download()
            res.append((st.copy(), infos, hs, outs))
    return res


def _info_tuple(inf):
    return (inf.width, inf.height, inf.channels, inf.num_components, tuple(inf.plane_width),
            tuple(inf.plane_height), inf.h_max, inf.v_max, inf.mcus_x, inf.mcus_y, inf.output_bytes,
            inf.compressed_bytes, inf.data_units)


def _same(h, d, files):
    (sh, ih, hh, oh), (sd, idv, hd, od) = h, d
    assert np.array_equal(sh, sd), [(i, int(a), int(b)) for i, (a, b) in enumerate(zip(sh, sd)) if a != b][:10]
    assert hh == hd
    for i in range(len(files)):
        assert _info_tuple(ih[i]) == _info_tuple(idv[i]), i
        if sh[i] == 0:
            assert np.array_equal(oh[i], od[i]), i


def test_acceptance_corpus_device_plan(decoder):
    files = [f for _, f in acceptance_corpus()]
    h, d = _both(decoder, files)
    assert (d[0] == 0).all()
    _same(h, d, files)
    for i, f in enumerate(files):
        ref = Ref.decode(f, rgb=True)
        assert np.array_equal(d[3][i][: ref.data.size], ref.data.reshape(-1)), i


@pytest.mark.parametrize("name,seed,scan_only", [("parser_recipe", 13, False), ("header_444", 16, False),
                                                 ("scan", 14, True), ("parser_recipe_b", 21, False)])
def test_mutated_headers_same_errc_as_host_planner(decoder, name, seed, scan_only):
    """The reference's parser fuzz recipe (test_parser.cpp:146-162) and more:
    every mutant gets the host planner's status (pinned to the reference by
    test_gpu_fuzz.py), infos and output."""
    base = ref_jpeg(120, 72, 10, 90, "444") if "444" in name else ref_jpeg(32, 24, 7, 70, "420")
    if scan_only:
        base = ref_jpeg(256, 192, 8, 75, "420")
    files = _mutants(base, 300, seed, scan_only)
    h, d = _both(decoder, files)
    _same(h, d, files)
    assert len(set(int(x) for x in d[0])) > 2  # the corpus exercises several error paths


def test_header_errors_each_site(decoder):
    """Hand-made header defects, one per parse() error site, mixed with valid
    files in one batch: statuses equal the reference parser's."""
    good = ref_jpeg(48, 40, 3, 80, "420")
    sos = good.index(b"\xff\xda")
    sof = good.index(b"\xff\xc0")
    dqt = good.index(b"\xff\xdb")
    dht = good.index(b"\xff\xc4")
    cases = [
        b"",                                              # truncated before SOI
        b"\xff\xd8",                                      # truncated after SOI
        good[:2] + b"\x00" + good[3:],                    # expected marker prefix
        good[:sof + 1] + b"\xc2" + good[sof + 2:],        # progressive SOF2
        good[:sof + 4] + b"\x0c" + good[sof + 5:],        # 12-bit precision
        good[:sof + 7] + b"\x00\x00" + good[sof + 9:],    # zero width
        good[:sof + 5] + b"\x00\x00" + good[sof + 7:],    # zero height (DNL)
        good[:sof + 9] + b"\x04" + good[sof + 10:],       # 4 components
        good[:dqt + 4] + b"\x05" + good[dqt + 5:],        # quant id > 3
        good[:dqt + 4] + b"\x20" + good[dqt + 5:],        # quant precision 2
        good[:dqt + 5] + b"\x00" + good[dqt + 6:],        # zero quantiser
        good[:dht + 4] + b"\x20" + good[dht + 5:],        # table class 2
        good[:dht + 4] + b"\x05" + good[dht + 5:],        # huffman id > 3
        good[:dht + 5] + b"\x05" + good[dht + 6:],        # oversubscribed (deferred past the scan)
        good[:sos] + b"\xff\xdd\x00\x04\x00\x10" + good[sos:],  # DRI (rejected by default)
        good[:sos] + b"\xff\xdc\x00\x04\x00\x10" + good[sos:],  # DNL
        good[:sos] + b"\xff\xd9",                         # EOI before SOS
        good[:sos] + b"\xff\xd3" + good[sos:],            # stray RST
        good[:sos + 4] + b"\x02" + good[sos + 5:],        # scan component subset
        good[:sos + 5] + b"\x09" + good[sos + 6:],        # unknown component id
        good[:sos + 6] + b"\x44" + good[sos + 7:],        # huffman id > 3 in SOS
        good[:sos + 11] + b"\x01" + good[sos + 12:],      # spectral selection
        good[: sos + 14],                                 # empty scan
        good[: sos + 40],                                 # truncated scan
        good,
    ]
    h, d = _both(decoder, cases)
    _same(h, d, cases)
    for i, f in enumerate(cases):
        r = Ref.decode(f, rgb=True) if f else None
        if r is not None:
            assert int(d[0][i]) == r.status, (i, int(d[0][i]), r.status)


def test_thumbnail_batch_mixed_tables(decoder):
    """Many small files with several table sets (dedup across the batch, the
    same quantiser written as 8- and 16-bit DQT), every output mode."""
    from paper_2111_09219_b200.synth import synth_batch
    files = []
    for q, smp, seed in ((50, "420", 1), (75, "444", 2), (95, "gray", 3), (85, "422", 4)):
        blob, offs, sizes = synth_batch(300, 40, 24, 9000 + 1000 * seed, q, smp)
        files += [blob[int(o): int(o) + int(s)].tobytes() for o, s in zip(offs, sizes)]
    # a 16-bit-precision DQT twin of one file: same table values
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
    files = [files[i] for i in order]
    for mode in (pj.OutputColorspace.RGBInterleaved, pj.OutputColorspace.YCbCrPlanes, pj.OutputColorspace.Grayscale):
        h, d = _both(decoder, files, output=mode)
        assert (d[0] == 0).all()
        _same(h, d, files)
    for i in range(0, len(files), 37):
        want = Orc.decode(files[i], rgb=True)
        got = _both(decoder, [files[i]])[1][3][0]
        assert np.array_equal(got[: want.data.size], want.data.reshape(-1))


def test_device_plan_taps_and_restart_intervals(decoder):
    """Coefficients and sync states through a device-planned batch, and
    restart-interval files (DRI extension) planned on the device."""
    from paper_2111_09219_b200.synth import synth_batch
    files = [ref_jpeg(640, 400, 11, 85, "420"), ref_jpeg(333, 257, 12, 95, "444")]
    with decoder.batch(files, pj.DecodeConfig(subsequence_bits=256), device_plan=True) as b:
        assert (b.run() == 0).all()
        for i, f in enumerate(files):
            coeffs, ents, meta = Ref.entropy(f, sb=256, b=4)
            assert np.array_equal(b.coefficients(i, pre_dc_zigzag=True), coeffs)
            assert np.array_equal(b.sync_states(i)[:, 1], ents[:, 1])
    a = synth_batch(3, 500, 375, 77, 80, "420", 0)
    r = synth_batch(3, 500, 375, 77, 80, "420", 32)
    plain = [a[0][o: o + s].tobytes() for o, s in zip(a[1], a[2])]
    dri = [r[0][o: o + s].tobytes() for o, s in zip(r[1], r[2])]
    cfg = pj.DecodeConfig(restart_intervals=True)
    h, d = _both(decoder, dri + plain, cfg)
    _same(h, d, dri + plain)
    assert (d[0] == 0).all()
    for i in range(3):
        assert np.array_equal(d[3][i], d[3][3 + i])


def test_device_plan_large_images(decoder):
    """Multi-tile K0, many subsequences and K1 CTAs per image."""
    files = [ref_jpeg(3840, 2160, 2, 90, "420"), ref_jpeg(1024, 1024, 5, 100, "444")]
    h, d = _both(decoder, files)
    assert (d[0] == 0).all()
    _same(h, d, files)
