"""CPU: the device planner's JFIF marker walk (csrc/devparse.h, run by
pjg_batch_create_device on the GPU) executed on the host through
pjg_debug_device_parse, against the host parser (pinned to the reference by
test_host.py / the GPU fuzz tests) and the reference itself: the same Errc
(parser.hpp:264-347 precedence), geometry and scan offset for thousands of
mutated headers (the reference's parser fuzz recipe, test_parser.cpp:146-162)
and one hand-made defect per error site."""
import ctypes as C

import numpy as np
import pytest

import paper_2111_09219_b200 as pj
from oracle.oracle import Ref
from tests.corpus import ref_jpeg


class _HdrInfo(C.Structure):
    _fields_ = [("width", C.c_uint32), ("height", C.c_uint32), ("num_components", C.c_uint32),
                ("comp_id", C.c_uint32 * 3), ("comp_h", C.c_uint32 * 3), ("comp_v", C.c_uint32 * 3),
                ("comp_tq", C.c_uint32 * 3), ("comp_td", C.c_uint32 * 3), ("comp_ta", C.c_uint32 * 3),
                ("mcu_width", C.c_uint32), ("mcu_height", C.c_uint32), ("mcus_x", C.c_uint32),
                ("mcus_y", C.c_uint32), ("data_units_per_mcu", C.c_uint32), ("total_data_units", C.c_uint64),
                ("quant_tables", C.c_uint32), ("dc_tables", C.c_uint32), ("ac_tables", C.c_uint32),
                ("restart_interval", C.c_uint32), ("scan_offset", C.c_uint64)]


def device_parse(f, allow_dri=False):
    out = np.zeros(7, np.int64)
    buf = (C.c_uint8 * max(1, len(f))).from_buffer_copy(f or b"\0")
    st = pj.lib().pjg_debug_device_parse(buf, C.c_size_t(len(f)), C.c_int(int(allow_dri)),
                                         out.ctypes.data_as(C.POINTER(C.c_int64)))
    assert st == 0
    return out


def host_parse(f, allow_dri=False):
    info = _HdrInfo()
    buf = (C.c_uint8 * max(1, len(f))).from_buffer_copy(f or b"\0")
    st = pj.lib().pjg_inspect_header(buf, C.c_size_t(len(f)), C.c_int(int(allow_dri)), C.byref(info))
    if st == 0 and info.scan_offset == len(f):
        st = 2  # extract_scan of nothing: EmptyScan (C-ABI status = Errc ordinal + 1)
    return st, info


def _mutants(base, n, seed):
    rng = np.random.default_rng(seed)
    out = []
    for trial in range(n):
        m = bytearray(base)
        for _ in range(int(rng.integers(1, 9))):
            m[int(rng.integers(0, len(base)))] = int(rng.integers(0, 256))
        if trial % 3 == 0:
            m = m[: int(rng.integers(0, len(m))) + 1]
        out.append(bytes(m))
    return out


def _check(f, allow_dri=False):
    d = device_parse(f, allow_dri)
    hs, hi = host_parse(f, allow_dri)
    assert int(d[0]) == hs, (int(d[0]), hs)
    assert (int(d[2]), int(d[3])) == (hi.width, hi.height)
    assert int(d[4]) == hi.num_components
    if hs == 0:
        assert int(d[5]) == hi.data_units_per_mcu
        assert int(d[6]) == hi.scan_offset
    return d


@pytest.mark.parametrize("src", [(32, 24, 7, 70, "420"), (120, 72, 10, 90, "444"), (40, 40, 5, 50, "gray"),
                                 (64, 48, 9, 85, "422")])
def test_mutated_headers_device_parse_equals_host(src):
    base = ref_jpeg(*src)
    sos = base.index(b"\xff\xda")
    head = base[: sos + 40]  # headers + a little scan: mutations land in the markers
    files = _mutants(head, 1500, 100 + src[2])
    codes = set()
    for f in files:
        codes.add(int(_check(f)[0]))
    assert len(codes) >= 3, codes


def test_header_error_sites_match_reference():
    good = ref_jpeg(48, 40, 3, 80, "420")
    sos = good.index(b"\xff\xda")
    sof = good.index(b"\xff\xc0")
    dqt = good.index(b"\xff\xdb")
    dht = good.index(b"\xff\xc4")
    cases = [
        b"", b"\xff\xd8", good[:2] + b"\x00" + good[3:], good[:sof + 1] + b"\xc2" + good[sof + 2:],
        good[:sof + 4] + b"\x0c" + good[sof + 5:], good[:sof + 7] + b"\x00\x00" + good[sof + 9:],
        good[:sof + 5] + b"\x00\x00" + good[sof + 7:], good[:sof + 9] + b"\x04" + good[sof + 10:],
        good[:dqt + 4] + b"\x05" + good[dqt + 5:], good[:dqt + 4] + b"\x20" + good[dqt + 5:],
        good[:dqt + 5] + b"\x00" + good[dqt + 6:], good[:dht + 4] + b"\x20" + good[dht + 5:],
        good[:dht + 4] + b"\x05" + good[dht + 5:],
        good[:sos] + b"\xff\xdd\x00\x04\x00\x10" + good[sos:],
        good[:sos] + b"\xff\xdc\x00\x04\x00\x10" + good[sos:],
        good[:sos] + b"\xff\xd9", good[:sos] + b"\xff\xd3" + good[sos:],
        good[:sos + 4] + b"\x02" + good[sos + 5:], good[:sos + 5] + b"\x09" + good[sos + 6:],
        good[:sos + 6] + b"\x44" + good[sos + 7:], good[:sos + 11] + b"\x01" + good[sos + 12:],
        good[: sos + 14], good,
    ]
    for i, f in enumerate(cases):
        d = _check(f)
        if f:
            r = Ref.decode(f, rgb=True)
            if int(d[0]) != 0 or r.status in (0, 2):
                assert int(d[0]) == r.status, (i, int(d[0]), r.status)


def test_restart_interval_extension():
    good = ref_jpeg(48, 40, 3, 80, "420")
    sos = good.index(b"\xff\xda")
    f = good[:sos] + b"\xff\xdd\x00\x04\x00\x10" + good[sos:]
    assert int(device_parse(f, False)[0]) == int(pj.Errc.UnsupportedFeature) + 1
    assert int(_check(f, True)[0]) == 0
