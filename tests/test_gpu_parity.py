"""GPU parity: the CUDA path (through the C-ABI) against the reference.

The reference itself (oracle/_ref, pjpeg headers compiled in place) is the
checker here; tests/test_oracle.py separately pins my C restatement against it.
Bar: bit-exact coefficients, sync states, planes and RGB.
"""
import numpy as np
import pytest

from oracle.oracle import Orc, Ref
from tests.corpus import acceptance_corpus, ref_jpeg

pj = pytest.importorskip("paper_2111_09219_b200")

pytestmark = pytest.mark.gpu


def _rgb(buf, inf):
    ch = inf.channels
    pix = buf[: inf.width * inf.height * ch]
    return pix.reshape(inf.height, inf.width, ch) if ch == 3 else pix.reshape(inf.height, inf.width)


def _check_file(b, i, data, sb, rgb_mode=True):
    """coefficients, sync states and output of image i against the reference."""
    coeffs, ents, meta = Ref.entropy(data, sb=sb, b=4)
    got = b.coefficients(i, pre_dc_zigzag=True)
    assert np.array_equal(got, coeffs), "entropy-stage coefficients differ"
    st = b.sync_states(i)
    assert st.shape[0] == ents.shape[0] == int(meta[0])
    # trimmed n per subsequence is unique (true decomposition) → exact
    assert np.array_equal(st[:, 1], ents[:, 1]), "trimmed n differs"
    # (p, c, z) at every boundary the oracle trace marks valid (test_parallel_decode.cpp:205-227)
    N = st.shape[0]
    bnd = np.arange(1, N, dtype=np.uint64) * sb
    states, valid, _, _ = Ref.trace(data, bnd)
    for k in range(N - 1):
        if valid[k]:
            assert st[k, 0] == states[k, 0] and st[k, 2] == states[k, 2] and st[k, 3] == states[k, 3], k


def test_acceptance_corpus_rgb_bit_exact(decoder):
    corpus = acceptance_corpus()
    files = [f for _, f in corpus]
    with decoder.batch(files, pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved) as b:
        st = b.run()
        assert (st == 0).all(), st
        outs = b.download()
        for i, ((w, h, q, s), f) in enumerate(corpus):
            ref = Ref.decode(f, rgb=True)
            assert ref.status == 0
            got = _rgb(outs[i], b.infos[i])
            assert got.shape == ref.data.shape, (w, h, q, s)
            assert np.array_equal(got, ref.data), (w, h, q, s, int((got != ref.data).sum()))


@pytest.mark.parametrize("replay", ["on", "off"])
@pytest.mark.parametrize("hop", ["0", "1"])
@pytest.mark.parametrize("sb", [128, 256, 1024, 4096])
def test_acceptance_corpus_entropy_and_states(decoder, sb, hop, replay, monkeypatch):
    # both K1 inter-CTA modes: speculative starts checked by K1c's parallel
    # first pass (hop=0, full grids) and the in-kernel re-chain (hop=1, small
    # grids); K3 replaying K1's kept symbols or decoding every subsequence
    monkeypatch.setenv("PJG_K1_HOP", hop)
    monkeypatch.setenv("PJG_REPLAY", "1" if replay == "on" else "0")
    if replay == "on":  # replay runs with K1's large-batch (global-table) variant
        monkeypatch.setenv("PJG_SMEM_TABLES", "0")
    corpus = acceptance_corpus()
    files = [f for _, f in corpus]
    with decoder.batch(files, pj.DecodeConfig(subsequence_bits=sb), pj.OutputColorspace.YCbCrPlanes) as b:
        st = b.run()
        assert (st == 0).all(), st
        outs = b.download()
        for i, (_, f) in enumerate(corpus):
            _check_file(b, i, f, sb)
            ref = Ref.decode(f, rgb=False)
            assert np.array_equal(outs[i][: ref.data.size], ref.data)


@pytest.mark.parametrize("shape", [(512, 512, 85, "444", 1), (500, 375, 75, "420", 1000),
                                   (1023, 769, 90, "420", 5), (333, 257, 95, "422", 6),
                                   (801, 601, 60, "gray", 7)])
def test_config_shapes_bit_exact(decoder, shape):
    w, h, q, s, seed = shape
    f = ref_jpeg(w, h, seed, q, s)
    with decoder.batch([f], pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved) as b:
        st = b.run()
        assert st[0] == 0
        got = _rgb(b.download()[0], b.infos[0])
        _check_file(b, 0, f, 1024)
    ref = Ref.decode(f, rgb=True)
    assert np.array_equal(got, ref.data)


def test_decode_single_planes_and_errors(decoder):
    f = ref_jpeg(80, 60, 10, 80, "420")
    res = pj.decode_single(f)
    assert len(res.planes.planes) == 3
    assert res.planes.planes[0].samples.shape == (60, 80)
    assert res.planes.planes[1].samples.shape == (30, 40)
    assert res.compressed_bytes == len(f)
    ref = Ref.decode(f, rgb=False)
    assert np.array_equal(np.concatenate([p.samples.reshape(-1) for p in res.planes.planes]), ref.data)
    with pytest.raises(pj.Error) as ei:
        pj.decode_single(bytes([0xDE, 0xAD, 0xBE, 0xEF]))
    assert ei.value.code == pj.Errc.MalformedHeader


def test_decode_batch_isolates_failures(decoder):
    # test_pipeline.cpp:38-54
    good1 = ref_jpeg(32, 32, 20, 70, "444")
    good2 = ref_jpeg(24, 16, 21, 70, "gray")
    truncated = good1[:10]
    garbage = bytes([0xDE, 0xAD, 0xBE, 0xEF])
    out = pj.decode_batch([good1, truncated, good2, garbage])
    assert isinstance(out[0], pj.DecodeSuccess)
    assert isinstance(out[1], pj.DecodeFailure)
    assert isinstance(out[2], pj.DecodeSuccess)
    assert isinstance(out[3], pj.DecodeFailure)
    assert out[3].code == pj.Errc.MalformedHeader
    for o, f in ((out[0], good1), (out[2], good2)):
        assert pj.planes_checksum(o.planes) == pj.planes_checksum(
            pj.ImagePlanes(o.planes.width, o.planes.height, 1, 1,
                           [pj.Plane(p.width, p.height, p.samples) for p in o.planes.planes]))
        ref = Ref.decode(f, rgb=False)
        assert np.array_equal(np.concatenate([p.samples.reshape(-1) for p in o.planes.planes]), ref.data)


def test_error_codes_match_reference(decoder):
    base = ref_jpeg(64, 48, 3, 75, "420")
    cases = {
        "trunc_header": base[:40],
        "garbage": bytes([0xDE, 0xAD, 0xBE, 0xEF]),
        "no_soi": b"\x00" + base[1:],
        "scan_cut": base[: len(base) // 2],
        "empty_scan": None,
    }
    # empty scan: SOS header immediately followed by EOI
    sos = base.index(b"\xff\xda")
    ln = (base[sos + 2] << 8) | base[sos + 3]
    cases["empty_scan"] = base[: sos + 2 + ln] + b"\xff\xd9"
    # RST marker inside the scan → UnsupportedFeature (parser.hpp:249-250)
    scan0 = sos + 2 + ln
    cases["rst_in_scan"] = base[: scan0 + 20] + b"\xff\xd0" + base[scan0 + 20:]
    files = list(cases.values())
    with decoder.batch(files, pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved) as b:
        st = b.run()
    for (name, f), s in zip(cases.items(), st):
        ref = Ref.decode(f, rgb=True)
        assert s == ref.status, (name, s, ref.status)  # corrupt scans: K1x replays the reference


def test_upsample_and_convert_kats(decoder):
    # test_pipeline.cpp:122-165
    P = pj.Plane
    planes = pj.ImagePlanes(8, 8, 1, 1, [P(8, 8, np.full((8, 8), 200, np.uint8)),
                                        P(8, 8, np.full((8, 8), 128, np.uint8)),
                                        P(8, 8, np.full((8, 8), 128, np.uint8))])
    out = pj.upsample_and_convert(planes)
    assert out.channels == 3 and (out.pixels == 200).all()
    planes = pj.ImagePlanes(4, 2, 2, 2, [P(4, 2, np.full((2, 4), 128, np.uint8)),
                                        P(2, 1, np.array([[128, 255]], np.uint8)),
                                        P(2, 1, np.array([[128, 128]], np.uint8))])
    out = pj.upsample_and_convert(planes).pixels
    assert list(out[0, 0]) == [128, 128, 128] and list(out[1, 1]) == [128, 128, 128]
    assert out[0, 2, 2] == 255 and out[1, 3, 2] == 255 and out[0, 2, 1] < 100
    # random planes vs the reference, all three channels
    rng = np.random.default_rng(3)
    for (W, H) in [(17, 9), (64, 48), (33, 31)]:
        pl = [P(W, H, rng.integers(0, 256, (H, W), dtype=np.uint8)),
              P((W + 1) // 2, (H + 1) // 2, rng.integers(0, 256, ((H + 1) // 2, (W + 1) // 2), dtype=np.uint8)),
              P((W + 1) // 2, (H + 1) // 2, rng.integers(0, 256, ((H + 1) // 2, (W + 1) // 2), dtype=np.uint8))]
        got = pj.upsample_and_convert(pj.ImagePlanes(W, H, 2, 2, pl)).pixels
        ref = Ref.upsample_and_convert(W, H, [p.samples for p in pl])
        assert np.array_equal(got, ref)


def test_restatement_agrees_on_gpu_box():
    """Sanity on the GPU box: the C restatement still matches the reference."""
    f = ref_jpeg(97, 33, 7, 90, "420")
    assert np.array_equal(Orc.decode(f).data, Ref.decode(f).data)


def test_contiguous_region_unaligned_offsets(decoder):
    """Files laid out back to back in one caller region at odd offsets (the
    single-copy upload path): K0's 16-byte-grid windows start mid-chunk and
    neighbouring images share edge chunks."""
    corpus = acceptance_corpus()[::3] + [((1023, 769, 90, "420"), ref_jpeg(1023, 769, 5, 90, "420"))]
    gaps = [1, 3, 7, 0, 13, 2, 5, 11, 0, 1, 9, 4, 6, 15, 3, 8, 1, 2, 0, 7, 5, 3]
    parts, offs, sizes, pos = [], [], [], 0
    for k, (_, f) in enumerate(corpus):
        g = gaps[k % len(gaps)]
        parts.append(b"\xa5" * g)
        pos += g
        offs.append(pos)
        sizes.append(len(f))
        parts.append(f)
        pos += len(f)
    blob = np.frombuffer(b"".join(parts) + b"\x00" * 64, np.uint8).copy()
    with decoder.batch((blob, np.array(offs, np.uint64), np.array(sizes, np.uint64)), pj.DecodeConfig(),
                       pj.OutputColorspace.RGBInterleaved) as b:
        st = b.run()
        assert (st == 0).all(), st
        outs = b.download()
        for i, (_, f) in enumerate(corpus):
            ref = Ref.decode(f, rgb=True)
            got = _rgb(outs[i], b.infos[i])
            assert np.array_equal(got, ref.data), i


@pytest.mark.parametrize("compact", ["1", "0"])
def test_random_shapes_batch_bit_exact(decoder, compact, monkeypatch):
    """A mixed batch of seeded random shapes, samplings and qualities (full
    and partial K4 tiles, 1-3 IDCT passes per tile, FP64 replays) against the
    reference decoder, RGB bit-exact — through the compact K3->K4 entry
    interface and the dense coefficient buffer."""
    monkeypatch.setenv("PJG_COMPACT", compact)
    rng = np.random.default_rng(2111)
    cases = []
    for k in range(14):
        w = int(rng.integers(9, 700))
        h = int(rng.integers(9, 300))
        q = int(rng.choice([50, 75, 85, 90, 95, 100]))
        s = ["444", "422", "420", "gray"][k % 4]
        cases.append(((w, h, q, s), ref_jpeg(w, h, 5000 + k, q, s)))
    files = [f for _, f in cases]
    with decoder.batch(files, pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved) as b:
        st = b.run()
        assert (st == 0).all(), st
        outs = b.download()
        for i, (shape, f) in enumerate(cases):
            ref = Ref.decode(f, rgb=True)
            got = _rgb(outs[i], b.infos[i])
            assert np.array_equal(got, ref.data), (shape, int((got != ref.data).sum()))


def test_cpp_dropin_binary_matches_reference(tmp_path):
    """The C++ shim (include/pjpeg_gpu.hpp) and the reference in ONE binary
    (oracle/_ref/cpp_dropin_check, prebuilt with the reference headers where
    they exist and shipped to the GPU box): identical planes checksum and RGB."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "oracle", "_ref", "cpp_dropin_check")
    assert os.path.exists(exe), "build() prebuilds oracle/_ref/cpp_dropin_check next to the reference"
    for k, (w, h, q, s) in enumerate([(333, 257, 95, "422"), (512, 512, 85, "444"), (500, 375, 75, "420"),
                                      (161, 97, 50, "gray")]):
        f = tmp_path / f"img{k}.jpg"
        f.write_bytes(ref_jpeg(w, h, 6 + k, q, s))
        r = subprocess.run([exe, str(f)], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "IDENTICAL" in r.stdout, r.stdout


def test_cli_decode_inspect_bench(tmp_path):
    """The reference CLI's commands (tools/pjpeg_cli.cpp) over the GPU decoder:
    decode writes the reference's RGB as PPM, inspect prints the parsed frame,
    bench prints the reference's row keys (+ RGB GB/s)."""
    import json
    import subprocess
    from tests.test_host import _cli
    exe = _cli()
    f = ref_jpeg(333, 257, 6, 95, "422")
    src = tmp_path / "a.jpg"
    src.write_bytes(f)
    out = tmp_path / "a.ppm"
    r = subprocess.run([exe, "decode", str(src), str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    data = out.read_bytes()
    header = b"P6\n333 257\n255\n"
    assert data.startswith(header)
    ref = Ref.decode(f, rgb=True)
    assert np.array_equal(np.frombuffer(data[len(header):], np.uint8).reshape(ref.data.shape), ref.data)
    r = subprocess.run([exe, "inspect", str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    info = pj.inspect(f)
    assert "size: 333x257" in r.stdout and "components: 3" in r.stdout
    assert f"total data units: {info['data_units']}" in r.stdout
    assert "partition (s*32=1024, b=256): N=" in r.stdout
    bdir = tmp_path / "corpus"
    bdir.mkdir()
    for k in range(3):
        (bdir / f"{k}.jpg").write_bytes(ref_jpeg(96 + 16 * k, 80, 100 + k, 75, "420"))
    r = subprocess.run([exe, "bench", str(bdir), "--iterations", "2"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    row = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("batch", "config", "wall_ms", "stages", "mb_per_s", "checksum", "rgb_gb_s", "images_per_s",
                "gpus", "k4_roofline_frac"):
        assert key in row, key
    assert row["batch"] == 3 and "failures" not in row
    assert row["gpus"] == 1 and 0 < row["k4_roofline_frac"] < 1


def test_decode_to_cuda_tensors():
    """CUDA uint8 torch tensors straight from the device output (D2D copies on
    the decoder's stream), equal to the reference; failed files give None."""
    import torch
    files = [ref_jpeg(96, 64, 31, 80, "420"), ref_jpeg(40, 24, 32, 90, "gray"), b"\xde\xad\xbe\xef",
             ref_jpeg(33, 17, 33, 70, "444")]
    ts, st = pj.decode_to_tensors(files, device=0)
    assert list(st[[0, 1, 3]]) == [0, 0, 0] and st[2] != 0 and ts[2] is None
    for t, f in ((ts[0], files[0]), (ts[1], files[1]), (ts[3], files[3])):
        assert t.is_cuda and t.dtype == torch.uint8
        ref = Ref.decode(f, rgb=True).data
        assert tuple(t.shape) == ref.shape
        assert np.array_equal(t.cpu().numpy(), ref)


def test_large_thumbnail_batch_parallel_planner(decoder):
    """A batch large enough for the multi-threaded host planner (contiguous
    per-worker chunks, per-worker table dedup merged afterwards): 1,536 small
    files with three quality/sampling mixes (distinct tables), in one region and
    packed from separate buffers; every image RGB-exact against the C oracle."""
    from paper_2111_09219_b200.synth import synth_batch
    files = []
    for q, smp, seed in ((50, "420", 1), (75, "444", 2), (95, "gray", 3)):
        blob, offs, sizes = synth_batch(512, 40, 24, 7000 + 1000 * seed, q, smp)
        files += [blob[int(o): int(o) + int(s)].tobytes() for o, s in zip(offs, sizes)]
    order = np.random.default_rng(5).permutation(len(files))
    files = [files[i] for i in order]
    with decoder.batch(files, pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved) as b:
        st = b.run()
        assert (st == 0).all(), np.unique(st)
        outs = b.download()
    for i, f in enumerate(files):
        want = Orc.decode(f, rgb=True)
        assert want.status == 0
        assert np.array_equal(outs[i][: want.data.size], want.data.reshape(-1)), i


def test_unstuffed_segment_byte_exact(decoder):
    """K0's unstuffed entropy segment (FF00 -> FF compaction up to the first
    marker) byte for byte against the reference's extract_scan + unstuff
    (parser.hpp:238-258, bitstream.hpp:56-76): the acceptance corpus, forged
    scans dense in 0xFF bytes, and the unstuff KAT (test_bitstream.cpp:26-32)."""
    import json
    import os
    from oracle.oracle import example_jpeg
    from tests.test_gpu_adversarial import CASES, _forge
    kat = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_kats.json")))["unstuff"]
    files = [f for _, f in acceptance_corpus()] + [_forge(*c, 300 + i) for i, c in enumerate(CASES)]
    files.append(example_jpeg(bytes(kat["in"])))
    with decoder.batch(files, pj.DecodeConfig(), pj.OutputColorspace.YCbCrPlanes) as b:
        b.run()
        for i, f in enumerate(files):
            want = Ref.segment(f)
            got = b.segment(i)
            assert got == want, (i, len(got), len(want))
    assert got == bytes(kat["out"]) and len(got) * 8 == kat["bit_length"]
    assert sum(f.count(b"\xff\x00") for f in files) > 1000  # the stuffing path ran


def test_partition_kats(decoder):
    """partition() KATs (test_parallel_decode.cpp:42-63): N = ceil(bits / sb)
    subsequences, through the sync-state dump of scans of those exact lengths."""
    import json
    import os
    from oracle.oracle import example_jpeg
    kat = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_kats.json")))["partition"]
    for bits, sb, b_, N, B in kat["cases"]:
        if bits % 8:
            continue  # scans are whole bytes
        scan = bytes([0x00]) * (bits // 8)  # DC "0" codes: decodable
        f = example_jpeg(scan)
        with decoder.batch([f], pj.DecodeConfig(subsequence_bits=sb, sequence_length_b=b_),
                           pj.OutputColorspace.YCbCrPlanes) as bt:
            bt.run()
            n = C_count(bt)
        assert n == N, (bits, sb, n, N)


def C_count(bt):
    import ctypes as C
    n = C.c_size_t()
    pj.lib().pjg_batch_dump_sync_states(bt._h, 0, None, 0, C.byref(n))
    return n.value


@pytest.mark.parametrize("compact", ["1", "0"])
@pytest.mark.parametrize("sb", [128, 1024])
def test_compact_interface_entropy_and_states(decoder, sb, compact, monkeypatch):
    """K3 -> K4 through compact entries (K1 entry counts, K2 entry offsets,
    per-unit entry ranges; coefficients expanded for the dump) or the dense
    buffer: coefficients, sync states and planes equal the reference on the
    acceptance corpus (every sampling, 8- and 16-bit tables)."""
    monkeypatch.setenv("PJG_COMPACT", compact)
    corpus = acceptance_corpus()
    files = [f for _, f in corpus]
    with decoder.batch(files, pj.DecodeConfig(subsequence_bits=sb), pj.OutputColorspace.YCbCrPlanes) as b:
        st = b.run()
        assert (st == 0).all(), st
        outs = b.download()
        for i, (_, f) in enumerate(corpus):
            _check_file(b, i, f, sb)
            ref = Ref.decode(f, rgb=False)
            assert np.array_equal(outs[i][: ref.data.size], ref.data)


def test_grayscale_output_of_colour_files(decoder):
    """Grayscale output (the Y plane alone, pipeline.hpp Grayscale) of a batch
    of colour files: each image's region holds exactly its Y plane — the
    chroma planes must not spill into the next image's region."""
    files = [ref_jpeg(40 + 8 * k, 24 + 4 * k, 700 + k, 75, ["420", "444", "422"][k % 3]) for k in range(24)]
    with decoder.batch(files, pj.DecodeConfig(), pj.OutputColorspace.Grayscale) as b:
        st = b.run()
        assert (st == 0).all(), st
        outs = b.download()
        for i, f in enumerate(files):
            ref = Ref.decode(f, rgb=False)
            inf = b.infos[i]
            y = ref.data[: inf.width * inf.height]
            assert outs[i].size == y.size, i
            assert np.array_equal(outs[i], y), i


@pytest.mark.parametrize("compact", ["1", "0"])
def test_alternating_density_batch(decoder, compact, monkeypatch):
    """Files alternating between very sparse (q20) and very dense (q100) scans,
    so that consecutive K4 tiles of a warp differ by 10x in coded coefficients:
    the compact interface's per-tile entry window (sized from the previous
    tile) must fall back to global reads for whatever it did not stage."""
    monkeypatch.setenv("PJG_COMPACT", compact)
    files = []
    for k in range(24):
        s = ["444", "420", "gray"][k % 3]
        files.append(ref_jpeg(72 + 8 * (k % 5), 40 + 8 * (k % 3), 900 + k, 20 if k % 2 else 100, s))
    with decoder.batch(files, pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved) as b:
        st = b.run()
        assert (st == 0).all(), st
        outs = b.download()
        for i, f in enumerate(files):
            ref = Ref.decode(f, rgb=True)
            got = _rgb(outs[i], b.infos[i])
            assert np.array_equal(got, ref.data), (i, int((got != ref.data).sum()))


@pytest.mark.parametrize("compact", ["1", "0"])
def test_gray_wide_tile_store_paths(decoder, compact, monkeypatch):
    """One-unit-per-MCU grayscale scans use 192-pixel K4 tiles with 16-byte Y
    stores when the destination row is 16-byte aligned: widths that are a
    multiple of 192, of 16 only, of 4 only, and odd, heights with a partial
    last MCU row, in one batch (later images start at unaligned offsets) and
    alone (offset 0) — RGB (1-channel) and planes equal the reference."""
    monkeypatch.setenv("PJG_COMPACT", compact)
    shapes = [(384, 40, 75), (208, 17, 90), (200, 9, 50), (201, 23, 95), (1000, 64, 85), (7, 5, 100)]
    files = [ref_jpeg(w, h, 7100 + k, q, "gray") for k, (w, h, q) in enumerate(shapes)]
    for batch in (files, files[:1], files[3:4]):
        for mode in (pj.OutputColorspace.RGBInterleaved, pj.OutputColorspace.YCbCrPlanes,
                     pj.OutputColorspace.Grayscale):
            with decoder.batch(batch, pj.DecodeConfig(), mode) as b:
                st = b.run()
                assert (st == 0).all(), st
                outs = b.download()
                for i, f in enumerate(batch):
                    ref = Ref.decode(f, rgb=mode == pj.OutputColorspace.RGBInterleaved)
                    want = ref.data.reshape(-1)
                    assert outs[i].size == want.size, (i, mode)
                    assert np.array_equal(outs[i], want), (i, mode, int((outs[i] != want).sum()))
