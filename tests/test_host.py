"""CPU: host side of the product — the C-ABI library loads and exports every
symbol include/pjg.h declares, header parsing matches the reference, the
device Huffman table format decodes every 16-bit window exactly like the
reference's flat LUT, and decode calls without a GPU fail loudly."""
import os
import re

import numpy as np
import pytest

import paper_2111_09219_b200 as pj
from oracle.oracle import EXAMPLE_AC, EXAMPLE_DC, Ref, ref_huff_lut16
from tests.corpus import ref_jpeg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "pjg.h")).read()
    return sorted(set(re.findall(r"\b(pjg_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = pj.lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) <= set(pj.EXPORTED_SYMBOLS) | set(syms)


def test_status_names_match_errc():
    for e in pj.Errc:
        assert pj.lib().pjg_status_name(int(e) + 1).decode() == e.name


def test_inspect_geometry_matches_reference():
    for (w, h, q, s) in [(48, 48, 92, "444"), (97, 33, 75, "420"), (64, 48, 50, "422"), (31, 17, 20, "gray"),
                         (500, 375, 75, "420")]:
        f = ref_jpeg(w, h, 11, q, s)
        g = Ref.parse_info(f)
        info = pj.inspect(f)
        assert info["status"] == 0
        assert (info["width"], info["height"], info["components"]) == (g["width"], g["height"], g["ncomp"])
        assert (info["mcus_x"], info["mcus_y"]) == (g["mcus_x"], g["mcus_y"])
        assert info["data_units"] == g["dus"]
        rgb = pj.inspect(f, pj.OutputColorspace.RGBInterleaved)
        assert rgb["output_bytes"] == w * h * (1 if s == "gray" else 3)


def test_header_error_codes_match_reference():
    base = ref_jpeg(40, 24, 3, 75, "420")
    sos = base.index(b"\xff\xda")
    cases = {
        "truncated": base[:10],
        "garbage": bytes([0xDE, 0xAD, 0xBE, 0xEF]),
        "progressive": base.replace(b"\xff\xc0", b"\xff\xc2", 1),
        "no_soi": b"\x00" + base[1:],
        "sos_cut": base[: sos + 5],
    }
    for name, f in cases.items():
        want = Ref.decode(f).status
        got = pj.inspect(f)["status"]
        assert want != 0
        assert got == want, (name, got, want)


def annex_k_tables():
    dcl = ([0, 1, 5, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0], list(range(12)))
    dcc = ([0, 3, 1, 1, 1, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0], list(range(12)))
    return [dcl, dcc, EXAMPLE_DC, EXAMPLE_AC]


def random_canonical(rng):
    # a random complete-or-incomplete canonical code (test_huffman.cpp:210-247)
    counts = [0] * 16
    left, code_space = int(rng.integers(1, 162)), 1
    for L in range(16):
        code_space *= 2
        n = int(rng.integers(0, min(left, code_space - 1) + 1)) if L < 15 else min(left, code_space - 1)
        counts[L] = n
        code_space -= n
        left -= n
        if left == 0:
            break
    syms = list(rng.permutation(256)[: sum(counts)])
    return counts, syms


def test_two_level_huffman_table_equals_reference_flat_lut():
    rng = np.random.default_rng(3)
    tables = annex_k_tables() + [random_canonical(rng) for _ in range(60)]
    # tables actually used by the reference encoder's files
    windows = np.arange(65536, dtype=np.uint16)
    for counts, syms in tables:
        st, want, _ = ref_huff_lut16(counts, syms)
        got = np.zeros(65536, np.uint32)
        c = np.array(counts, np.uint8)
        s = np.array(syms if syms else [0], np.uint8)
        rc = pj.lib().pjg_debug_huff_decode(c.ctypes.data_as(pj.u8p), s.ctypes.data_as(pj.u8p), len(syms),
                                            windows.ctypes.data_as(pj.C.POINTER(pj.C.c_uint16)), 65536,
                                            got.ctypes.data_as(pj.C.POINTER(pj.C.c_uint32)))
        if st:
            assert rc == -st
            continue
        assert rc == 0
        assert np.array_equal(got, want), (counts, syms[:8])


def _fast_fields(e, dc):
    """decode_next_symbol's outcome for a decoded codeword e = (len << 8) | sym
    (huffman.hpp:137-175) packed like pjg_internal.h kFast*; 0 = rejected."""
    clen, sym = e >> 8, e & 255
    run = kind = 0
    if dc:
        l = sym
        if l > 11:
            return 0
    else:
        run, l = sym >> 4, sym & 15
        if l == 0:
            if run == 0:
                kind = 1
            elif run != 15:
                return 0
        elif l > 10:
            return 0
    return clen | (l << 5) | (((1 << l) - 1) << 10) | ((0 if kind == 1 else run + 1) << 21) | ((clen + l) << 27)


def test_fast_entries_with_second_level_equal_reference_decode():
    """The decoder's one-probe fast entry (11-bit primary, 5-bit second level
    for codes of 12..16 bits) resolves every 16-bit window like the
    reference's flat LUT + decode_next_symbol rules, or defers (0) to the
    exact path — which then sees the same window."""
    rng = np.random.default_rng(5)
    tables = annex_k_tables() + [random_canonical(rng) for _ in range(30)]
    windows = (np.arange(65536, dtype=np.uint32) << 16) | np.uint32(0x5A5A)
    for counts, syms in tables:
        st, want, _ = ref_huff_lut16(counts, syms)
        if st:
            continue
        c = np.array(counts, np.uint8)
        s = np.array(syms if syms else [0], np.uint8)
        for dc in (0, 1):
            got = np.zeros(65536, np.uint32)
            rc = pj.lib().pjg_debug_fast_entry(c.ctypes.data_as(pj.u8p), s.ctypes.data_as(pj.u8p), len(syms), dc,
                                               windows.ctypes.data_as(pj.C.POINTER(pj.C.c_uint32)), 65536,
                                               got.ctypes.data_as(pj.C.POINTER(pj.C.c_uint32)))
            assert rc == 0
            exp = np.array([_fast_fields(int(e), dc) if (int(e) >> 8) else 0 for e in want], np.uint32)
            nz = got != 0
            assert np.array_equal(got[nz], exp[nz]), (counts, dc)
            # deferrals only where the reference rejects, or prefixes beyond the
            # second-level capacity (never for the Annex K tables)
            deferred = np.flatnonzero(~nz & (exp != 0))
            if (counts, syms) in annex_k_tables():
                assert deferred.size == 0, (counts, dc, deferred[:5])


def test_oversubscribed_table_rejected_like_reference():
    counts = [3] + [0] * 15  # 3 codes of length 1
    st, _, _ = ref_huff_lut16(counts, [1, 2, 3])
    got = np.zeros(1, np.uint32)
    w = np.zeros(1, np.uint16)
    rc = pj.lib().pjg_debug_huff_decode(np.array(counts, np.uint8).ctypes.data_as(pj.u8p),
                                        np.array([1, 2, 3], np.uint8).ctypes.data_as(pj.u8p), 3,
                                        w.ctypes.data_as(pj.C.POINTER(pj.C.c_uint16)), 1,
                                        got.ctypes.data_as(pj.C.POINTER(pj.C.c_uint32)))
    assert st == int(pj.Errc.OversubscribedCode) + 1 and rc == -st


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pj.Error):
        pj.Decoder(0)
    with pytest.raises(pj.Error):
        pj.decode_single(ref_jpeg(16, 16, 1, 75, "444"))


def test_synthetic_bench_corpus_is_valid_baseline_jpeg():
    from paper_2111_09219_b200.synth import synth_batch
    for (w, h, q, s) in [(500, 375, 75, "420"), (64, 64, 85, "444"), (40, 24, 95, "gray"), (48, 32, 50, "422")]:
        blob, offs, sizes = synth_batch(3, w, h, 7, q, s)
        for o, n in zip(offs, sizes):
            f = blob[o: o + n].tobytes()
            d = Ref.decode(f)
            assert d.status == 0 and (d.width, d.height) == (w, h)


def _build_dropin(tmp_path):
    """tools/cpp_dropin_check.cpp: the reference (when its headers are here)
    and the pjpeg::gpu shim in ONE binary, linked to libpjg.so."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib_dir = os.path.join(root, "paper_2111_09219_b200")
    exe = str(tmp_path / "dropin")
    cmd = ["g++", "-O1", "-std=c++20", "-I" + os.path.join(root, "include"),
           os.path.join(root, "tools", "cpp_dropin_check.cpp"), "-o", exe, "-L" + lib_dir, "-lpjg",
           "-Wl,-rpath," + lib_dir, "-pthread"]
    ref_inc = "/root/reference/proj/include"
    if os.path.isdir(ref_inc):
        cmd[4:4] = ["-I" + ref_inc]
    else:
        cmd.insert(4, "-DPJPEG_NO_REF")
    subprocess.run(cmd, check=True, capture_output=True)
    return exe


def test_cpp_dropin_header_builds_and_links(tmp_path):
    assert os.path.exists(_build_dropin(tmp_path))


def _cli():
    """The pjpeg_gpu CLI (tools/pjpeg_gpu_cli.cpp), built by the library Makefile."""
    import subprocess
    exe = os.path.join(ROOT, "paper_2111_09219_b200", "pjpeg_gpu")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2111_09219_b200", "csrc")], check=True,
                       capture_output=True)
    return exe


def test_cli_usage_and_exit_codes(tmp_path):
    """pjpeg_cli.cpp's conventions: usage errors, 10 + Errc on failures (no GPU needed)."""
    import subprocess
    exe = _cli()
    assert subprocess.run([exe], capture_output=True).returncode == 2
    assert subprocess.run([exe, "frobnicate"], capture_output=True).returncode == 2
    r = subprocess.run([exe, "decode", str(tmp_path / "missing.jpg"), str(tmp_path / "o.ppm")],
                       capture_output=True, text=True)
    assert r.returncode == 10 + 10, r.stderr  # Errc::IoError
    r = subprocess.run([exe, "bench", str(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 10 + 9, r.stderr  # Errc::EmptyCorpus
