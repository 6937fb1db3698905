"""TEST INFRASTRUCTURE ONLY — ctypes access to the parity oracle.

Two checkers live here:

* ``Ref``  — the UNMODIFIED reference (pjpeg headers) compiled in place into
  ``oracle/_ref/libpjpeg_ref.so`` (see oracle/Makefile, oracle/ref_shim.cpp).
* ``Orc``  — my plain-C restatement (oracle/pjpeg_oracle.c →
  ``oracle/liboracle.so``), pinned against ``Ref`` and the reference KATs.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  The product
(paper_2111_09219_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libpjpeg_ref.so")
ORC_SO = os.path.join(HERE, "liboracle.so")

SAMPLING = {"444": 0, "422": 1, "420": 2, "gray": 3}

u8p = C.POINTER(C.c_uint8)
i16p = C.POINTER(C.c_int16)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


def _ptr(arr, typ):
    return arr.ctypes.data_as(typ)


class OracleError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: status {status}")
        self.status = status


@dataclass
class Decoded:
    status: int
    width: int = 0
    height: int = 0
    channels: int = 0
    nplanes: int = 0
    plane_dims: tuple = ()
    data: np.ndarray | None = None  # RGB/gray HxWxC, or planes concatenated
    timings: tuple = ()

    def planes(self):
        out, off = [], 0
        for (w, h) in self.plane_dims[: self.nplanes]:
            out.append(self.data[off : off + w * h].reshape(h, w))
            off += w * h
        return out


def _load(path):
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
    return C.CDLL(path)


class Ref:
    """The reference library itself (pjpeg headers, compiled in place)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = _load(REF_SO)
            L.ref_extend.restype = C.c_int32
            L.ref_hardware_concurrency.restype = C.c_uint
            cls._lib = L
        return cls._lib

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_SO)

    # -- corpus ----------------------------------------------------------
    @classmethod
    def encode_test_image(cls, w, h, seed, quality, sampling="420", channels=None) -> bytes:
        """oracle_encode(make_test_image(w, h, seed, channels), q, sampling)."""
        ch = channels if channels is not None else (1 if sampling == "gray" else 3)
        cap = w * h * ch * 4 + 4096
        buf = np.empty(cap, np.uint8)
        n = C.c_size_t()
        st = cls.lib().ref_encode_test_image(
            C.c_uint32(w), C.c_uint32(h), C.c_uint32(seed), C.c_uint(ch), C.c_int(quality),
            C.c_int(SAMPLING[sampling]), _ptr(buf, u8p), C.c_size_t(cap), C.byref(n))
        if st:
            raise OracleError(st, "ref_encode_test_image")
        return buf[: n.value].tobytes()

    @classmethod
    def encode_pixels(cls, pixels: np.ndarray, quality, sampling="420") -> bytes:
        pixels = np.ascontiguousarray(pixels, dtype=np.uint8)
        h, w = pixels.shape[:2]
        ch = 1 if pixels.ndim == 2 else pixels.shape[2]
        cap = w * h * ch * 4 + 4096
        buf = np.empty(cap, np.uint8)
        n = C.c_size_t()
        st = cls.lib().ref_encode_pixels(
            _ptr(pixels, u8p), C.c_uint32(w), C.c_uint32(h), C.c_uint(ch), C.c_int(quality),
            C.c_int(SAMPLING[sampling]), _ptr(buf, u8p), C.c_size_t(cap), C.byref(n))
        if st:
            raise OracleError(st, "ref_encode_pixels")
        return buf[: n.value].tobytes()

    @classmethod
    def make_test_image(cls, w, h, seed, channels=3) -> np.ndarray:
        out = np.empty(w * h * channels, np.uint8)
        cls.lib().ref_make_test_image(C.c_uint32(w), C.c_uint32(h), C.c_uint32(seed),
                                      C.c_uint(channels), _ptr(out, u8p))
        return out.reshape(h, w, channels) if channels > 1 else out.reshape(h, w)

    # -- decode ------------------------------------------------------------
    @classmethod
    def decode(cls, data: bytes, rgb=True, sb=1024, b=256, workers=1) -> Decoded:
        """decode_single (+ upsample_and_convert when rgb)."""
        arr = np.frombuffer(data, np.uint8)
        info = np.zeros(12, np.uint32)
        geo = np.zeros(12, np.uint32)
        st = cls.lib().ref_parse_info(_ptr(arr, u8p), C.c_size_t(len(data)), _ptr(geo, u32p))
        if st:
            return Decoded(status=st)
        cap = int(geo[0]) * int(geo[1]) * 3 + 64
        out = np.empty(cap, np.uint8)
        tim = np.zeros(6, np.float64)
        st = cls.lib().ref_decode(
            _ptr(arr, u8p), C.c_size_t(len(data)), C.c_uint64(sb), C.c_uint32(b), C.c_uint(workers),
            C.c_int(1 if rgb else 0), _ptr(out, u8p), C.c_size_t(cap), _ptr(info, u32p),
            tim.ctypes.data_as(C.POINTER(C.c_double)))
        if st:
            return Decoded(status=st)
        w, h, ch, npl = (int(v) for v in info[:4])
        dims = tuple((int(info[4 + 2 * i]), int(info[5 + 2 * i])) for i in range(3))
        if rgb:
            data_out = out[: w * h * ch].reshape(h, w, ch) if ch == 3 else out[: w * h].reshape(h, w)
        else:
            data_out = out[: sum(a * b for a, b in dims[:npl])]
        return Decoded(0, w, h, ch, npl, dims, data_out.copy(), tuple(tim))

    @classmethod
    def parse_info(cls, data: bytes):
        arr = np.frombuffer(data, np.uint8)
        geo = np.zeros(12, np.uint32)
        st = cls.lib().ref_parse_info(_ptr(arr, u8p), C.c_size_t(len(data)), _ptr(geo, u32p))
        if st:
            raise OracleError(st, "ref_parse_info")
        keys = ["width", "height", "ncomp", "mcus_x", "mcus_y", "dpm", "h_max", "v_max", "dus",
                "seg_bytes"]
        d = {k: int(v) for k, v in zip(keys, geo[:10])}
        d["bit_length"] = int(geo[10]) | (int(geo[11]) << 32)
        return d

    @classmethod
    def segment(cls, data: bytes) -> bytes:
        arr = np.frombuffer(data, np.uint8)
        out = np.empty(len(data) + 16, np.uint8)
        n = C.c_size_t()
        st = cls.lib().ref_segment(_ptr(arr, u8p), C.c_size_t(len(data)), _ptr(out, u8p),
                                   C.c_size_t(len(out)), C.byref(n))
        if st:
            raise OracleError(st, "ref_segment")
        return out[: n.value].tobytes()

    @classmethod
    def unstuff(cls, scan: bytes):
        arr = np.frombuffer(scan, np.uint8) if scan else np.zeros(1, np.uint8)
        out = np.empty(max(1, len(scan)), np.uint8)
        n = C.c_size_t()
        st = cls.lib().ref_unstuff(_ptr(arr, u8p), C.c_size_t(len(scan)), _ptr(out, u8p), C.byref(n))
        return st, out[: n.value].tobytes() if st == 0 else b""

    @classmethod
    def entropy(cls, data: bytes, sb=1024, b=256, workers=1):
        """parallel_entropy_decode + SyncInfoArray (trimmed n)."""
        g = cls.parse_info(data)
        N = (g["bit_length"] + sb - 1) // sb
        coeffs = np.empty(g["dus"] * 64, np.int16)
        ents = np.empty(max(N, 1) * 5, np.uint64)
        meta = np.zeros(4, np.uint64)
        arr = np.frombuffer(data, np.uint8)
        st = cls.lib().ref_entropy(
            _ptr(arr, u8p), C.c_size_t(len(data)), C.c_uint64(sb), C.c_uint32(b), C.c_uint(workers),
            _ptr(coeffs, i16p), C.c_size_t(coeffs.size), _ptr(ents, u64p), C.c_size_t(max(N, 1)),
            _ptr(meta, u64p))
        if st:
            raise OracleError(st, "ref_entropy")
        return coeffs, ents[: 5 * N].reshape(N, 5), meta

    @classmethod
    def sync_entries(cls, data: bytes, sb=1024, b=256):
        """Untrimmed entries after intra+inter sync (before offsets())."""
        g = cls.parse_info(data)
        N = (g["bit_length"] + sb - 1) // sb
        ents = np.empty(max(N, 1) * 5, np.uint64)
        meta = np.zeros(4, np.uint64)
        arr = np.frombuffer(data, np.uint8)
        st = cls.lib().ref_sync_entries(
            _ptr(arr, u8p), C.c_size_t(len(data)), C.c_uint64(sb), C.c_uint32(b),
            _ptr(ents, u64p), C.c_size_t(max(N, 1)), _ptr(meta, u64p))
        if st:
            raise OracleError(st, "ref_sync_entries")
        return ents[: 5 * N].reshape(N, 5), meta

    @classmethod
    def trace(cls, data: bytes, boundaries):
        g = cls.parse_info(data)
        bnd = np.ascontiguousarray(boundaries, np.uint64)
        nb = bnd.size
        states = np.zeros(max(nb, 1) * 4, np.uint64)
        valid = np.zeros(max(nb, 1), np.uint8)
        coeffs = np.empty(g["dus"] * 64, np.int16)
        end = np.zeros(4, np.uint64)
        arr = np.frombuffer(data, np.uint8)
        st = cls.lib().ref_oracle_trace(
            _ptr(arr, u8p), C.c_size_t(len(data)), _ptr(bnd, u64p) if nb else None, C.c_size_t(nb),
            _ptr(states, u64p), _ptr(valid, u8p), _ptr(coeffs, i16p), C.c_size_t(coeffs.size),
            _ptr(end, u64p))
        if st:
            raise OracleError(st, "ref_oracle_trace")
        return states[: 4 * nb].reshape(nb, 4), valid[:nb], coeffs, end

    @classmethod
    def idct_8x8(cls, block_raster_int32) -> np.ndarray:
        blk = np.ascontiguousarray(block_raster_int32, np.int32).reshape(64)
        out = np.empty(64, np.uint8)
        cls.lib().ref_idct_8x8(blk.ctypes.data_as(C.POINTER(C.c_int32)), _ptr(out, u8p))
        return out

    @classmethod
    def idct_basis(cls) -> np.ndarray:
        out = np.empty(64, np.float64)
        cls.lib().ref_idct_basis(out.ctypes.data_as(C.POINTER(C.c_double)))
        return out.reshape(8, 8)

    @classmethod
    def extend(cls, bits, l) -> int:
        return int(cls.lib().ref_extend(C.c_uint32(bits), C.c_uint(l)))

    @classmethod
    def upsample_and_convert(cls, width, height, planes):
        n = len(planes)
        pw = np.array([p.shape[1] for p in planes] + [0] * (3 - n), np.uint32)
        ph = np.array([p.shape[0] for p in planes] + [0] * (3 - n), np.uint32)
        ps = [np.ascontiguousarray(p, np.uint8) for p in planes]
        arrs = (u8p * 3)(*[_ptr(p, u8p) for p in ps] + [None] * (3 - n))
        out = np.empty(width * height * 3, np.uint8)
        ch = C.c_uint32()
        st = cls.lib().ref_upsample_and_convert(
            C.c_uint32(width), C.c_uint32(height), C.c_uint(n), _ptr(pw, u32p), _ptr(ph, u32p),
            arrs, _ptr(out, u8p), C.byref(ch))
        if st:
            raise OracleError(st, "ref_upsample_and_convert")
        c = ch.value
        return out[: width * height * c].reshape((height, width, c) if c == 3 else (height, width))

    @classmethod
    def decode_batch_rgb(cls, files, workers, sb=1024, b=256):
        """decode_batch + upsample_and_convert (the CPU baseline of record)."""
        n = len(files)
        infos = [cls.parse_info(f) for f in files]
        outs = [np.empty(max(1, i["width"] * i["height"] * 3), np.uint8) for i in infos]
        arrs = [np.frombuffer(f, np.uint8) for f in files]
        fptrs = (u8p * n)(*[_ptr(a, u8p) for a in arrs])
        sizes = (C.c_size_t * n)(*[len(f) for f in files])
        optrs = (u8p * n)(*[_ptr(o, u8p) for o in outs])
        caps = (C.c_size_t * n)(*[o.size for o in outs])
        status = np.zeros(n, np.int32)
        st = cls.lib().ref_decode_batch_rgb(
            fptrs, sizes, C.c_size_t(n), C.c_uint64(sb), C.c_uint32(b), C.c_uint(workers), optrs, caps,
            status.ctypes.data_as(C.POINTER(C.c_int32)))
        if st:
            raise OracleError(st, "ref_decode_batch_rgb")
        return status, outs

    @classmethod
    def hardware_concurrency(cls) -> int:
        return int(cls.lib().ref_hardware_concurrency())


class Orc:
    """My C restatement of the reference path (oracle/pjpeg_oracle.c)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = _load(ORC_SO)
            L.orc_extend.restype = C.c_int32
            cls._lib = L
        return cls._lib

    @classmethod
    def parse_info(cls, data: bytes):
        arr = np.frombuffer(data, np.uint8)
        geo = np.zeros(18, np.uint32)
        st = cls.lib().orc_parse_info(_ptr(arr, u8p), C.c_size_t(len(data)), _ptr(geo, u32p))
        if st:
            raise OracleError(st, "orc_parse_info")
        keys = ["width", "height", "ncomp", "mcus_x", "mcus_y", "dpm", "h_max", "v_max", "dus",
                "seg_bytes"]
        d = {k: int(v) for k, v in zip(keys, geo[:10])}
        d["bit_length"] = int(geo[10]) | (int(geo[11]) << 32)
        d["plane_dims"] = [(int(geo[12 + 2 * c]), int(geo[13 + 2 * c])) for c in range(d["ncomp"])]
        return d

    @classmethod
    def parse_status(cls, data: bytes) -> int:
        arr = np.frombuffer(data, np.uint8) if data else np.zeros(1, np.uint8)
        geo = np.zeros(18, np.uint32)
        return int(cls.lib().orc_parse_info(_ptr(arr, u8p), C.c_size_t(len(data)), _ptr(geo, u32p)))

    @classmethod
    def segment(cls, data: bytes) -> bytes:
        arr = np.frombuffer(data, np.uint8)
        out = np.empty(len(data) + 16, np.uint8)
        n = C.c_size_t()
        st = cls.lib().orc_segment(_ptr(arr, u8p), C.c_size_t(len(data)), _ptr(out, u8p),
                                   C.c_size_t(len(out)), C.byref(n))
        if st:
            raise OracleError(st, "orc_segment")
        return out[: n.value].tobytes()

    @classmethod
    def decode(cls, data: bytes, rgb=True, want_coeffs=False) -> Decoded:
        arr = np.frombuffer(data, np.uint8) if data else np.zeros(1, np.uint8)
        geo = np.zeros(18, np.uint32)
        st = cls.lib().orc_parse_info(_ptr(arr, u8p), C.c_size_t(len(data)), _ptr(geo, u32p))
        if st:
            return Decoded(status=st)
        cap = int(geo[0]) * int(geo[1]) * 3 + 64
        out = np.empty(cap, np.uint8)
        info = np.zeros(12, np.uint32)
        coeffs = np.empty(int(geo[8]) * 64, np.int16) if want_coeffs else None
        st = cls.lib().orc_decode(
            _ptr(arr, u8p), C.c_size_t(len(data)), C.c_int(1 if rgb else 0), _ptr(out, u8p),
            C.c_size_t(cap), _ptr(info, u32p), _ptr(coeffs, i16p) if want_coeffs else None,
            C.c_size_t(coeffs.size if want_coeffs else 0))
        if st:
            return Decoded(status=st)
        w, h, ch, npl = (int(v) for v in info[:4])
        dims = tuple((int(info[4 + 2 * i]), int(info[5 + 2 * i])) for i in range(3))
        if rgb:
            d = out[: w * h * ch].reshape(h, w, ch) if ch == 3 else out[: w * h].reshape(h, w)
        else:
            d = out[: sum(a * b for a, b in dims[:npl])]
        res = Decoded(0, w, h, ch, npl, dims, d.copy())
        if want_coeffs:
            res.coeffs = coeffs
        return res

    @classmethod
    def trace(cls, data: bytes, boundaries):
        g = cls.parse_info(data)
        bnd = np.ascontiguousarray(boundaries, np.uint64)
        nb = bnd.size
        states = np.zeros(max(nb, 1) * 4, np.uint64)
        valid = np.zeros(max(nb, 1), np.uint8)
        coeffs = np.empty(g["dus"] * 64, np.int16)
        end = np.zeros(4, np.uint64)
        arr = np.frombuffer(data, np.uint8)
        st = cls.lib().orc_trace(
            _ptr(arr, u8p), C.c_size_t(len(data)), _ptr(bnd, u64p) if nb else None, C.c_size_t(nb),
            _ptr(states, u64p), _ptr(valid, u8p), _ptr(coeffs, i16p), C.c_size_t(coeffs.size),
            _ptr(end, u64p))
        if st:
            raise OracleError(st, "orc_trace")
        return states[: 4 * nb].reshape(nb, 4), valid[:nb], coeffs, end

    @classmethod
    def idct_8x8(cls, block_raster_int32) -> np.ndarray:
        blk = np.ascontiguousarray(block_raster_int32, np.int32).reshape(64)
        out = np.empty(64, np.uint8)
        cls.lib().orc_idct_8x8(blk.ctypes.data_as(C.POINTER(C.c_int32)), _ptr(out, u8p))
        return out

    @classmethod
    def idct_basis(cls) -> np.ndarray:
        out = np.empty(64, np.float64)
        cls.lib().orc_idct_basis(out.ctypes.data_as(C.POINTER(C.c_double)))
        return out.reshape(8, 8)

    @classmethod
    def extend(cls, bits, l) -> int:
        return int(cls.lib().orc_extend(C.c_uint32(bits), C.c_uint(l)))


ZIGZAG_TO_RASTER = np.array([
    0, 1, 8, 16, 9, 2, 3, 10, 17, 24, 32, 25, 18, 11, 4, 5,
    12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6, 7, 14, 21, 28,
    35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
    58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63], np.int64)


def dc_prefix_inverse_zigzag(post_dc_raster: np.ndarray, du_seq) -> np.ndarray:
    """Maps a post-DC raster coefficient buffer back to the reference's
    entropy-stage layout (pre-DC differences, zig-zag order) — the inverse of
    dc_prefix_sum (transform.hpp:56-74) + dezigzag, exact mod 2^16."""
    blocks = post_dc_raster.reshape(-1, 64)
    zz = blocks[:, ZIGZAG_TO_RASTER].copy()
    dpm = len(du_seq)
    comp_of = np.array([du_seq[d % dpm] for d in range(zz.shape[0])])
    dc = zz[:, 0].astype(np.int64)
    out_dc = dc.copy()
    for comp in set(du_seq):
        idx = np.nonzero(comp_of == comp)[0]
        if idx.size > 1:
            out_dc[idx[1:]] = dc[idx[1:]] - dc[idx[:-1]]
    zz[:, 0] = ((out_dc + 32768) % 65536 - 32768).astype(np.int16)
    return zz.reshape(-1)


def ref_huff_lut16(counts, symbols):
    """Reference build_table LUT expanded to all 65536 16-bit windows."""
    L = Ref.lib()
    c = np.ascontiguousarray(counts, np.uint8)
    s = np.ascontiguousarray(symbols, np.uint8) if len(symbols) else np.zeros(1, np.uint8)
    out = np.zeros(65536, np.uint32)
    ml = C.c_uint()
    st = L.ref_huff_lut16(_ptr(c, u8p), _ptr(s, u8p), C.c_size_t(len(symbols)), _ptr(out, u32p), C.byref(ml))
    return st, out, ml.value


def ref_decode_symbols(dc, ac, bits: bytes, max_syms):
    """decode_next_symbol over a raw bit string; dc/ac = (counts16, symbols)."""
    L = Ref.lib()
    dcc = np.ascontiguousarray(dc[0], np.uint8)
    dcs = np.ascontiguousarray(dc[1], np.uint8)
    acc = np.ascontiguousarray(ac[0], np.uint8)
    acs = np.ascontiguousarray(ac[1], np.uint8)
    b = np.frombuffer(bits, np.uint8)
    rec = np.zeros(4 * max_syms, np.int64)
    n = C.c_size_t()
    st = L.ref_decode_symbols(_ptr(dcc, u8p), _ptr(dcs, u8p), C.c_size_t(dcs.size), _ptr(acc, u8p),
                              _ptr(acs, u8p), C.c_size_t(acs.size), _ptr(b, u8p), C.c_size_t(b.size),
                              C.c_size_t(max_syms), rec.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(n))
    return st, rec[: 4 * n.value].reshape(-1, 4)


def jfif_bytes(width, height, comps, quant, dc_specs, ac_specs, scan: bytes, dri=None, trailer=b"\xff\xd9"):
    """Assembles a baseline JPEG from explicit parts (test fixtures such as the
    reference's worked example, helpers.hpp:29-53).  comps: list of
    (id, h, v, tq, td, ta); quant: {id: 64 zig-zag entries}; dc/ac_specs:
    {id: (counts16, symbols)}."""
    out = bytearray(b"\xff\xd8")
    for tid, q in quant.items():
        out += b"\xff\xdb" + (3 + 64).to_bytes(2, "big") + bytes([tid]) + bytes(q)
    out += b"\xff\xc0" + (8 + 3 * len(comps)).to_bytes(2, "big") + bytes([8]) + height.to_bytes(2, "big") + \
        width.to_bytes(2, "big") + bytes([len(comps)])
    for (cid, h, v, tq, _, _) in comps:
        out += bytes([cid, (h << 4) | v, tq])
    for cls, specs in ((0, dc_specs), (1, ac_specs)):
        for tid, (counts, syms) in specs.items():
            out += b"\xff\xc4" + (3 + 16 + len(syms)).to_bytes(2, "big") + bytes([(cls << 4) | tid]) + \
                bytes(counts) + bytes(syms)
    if dri is not None:
        out += b"\xff\xdd" + (4).to_bytes(2, "big") + dri.to_bytes(2, "big")
    out += b"\xff\xda" + (6 + 2 * len(comps)).to_bytes(2, "big") + bytes([len(comps)])
    for (cid, _, _, _, td, ta) in comps:
        out += bytes([cid, (td << 4) | ta])
    out += bytes([0, 63, 0]) + scan + trailer
    return bytes(out)


# The reference's worked example (tests/helpers.hpp:29-53): one grayscale data
# unit, DC "0"->cat 0, "10"->cat 2; AC "00" EOB, "01" (0,1), "100" (0,2),
# "1010" (2,1), "1011" (1,1); scan 98 49 59 DC.
EXAMPLE_DC = ([1, 1] + [0] * 14, [0x00, 0x02])
EXAMPLE_AC = ([0, 2, 1, 2] + [0] * 12, [0x00, 0x01, 0x02, 0x21, 0x11])
EXAMPLE_SCAN = bytes([0x98, 0x49, 0x59, 0xDC])


def example_jpeg(scan=EXAMPLE_SCAN):
    return jfif_bytes(8, 8, [(1, 1, 1, 0, 0, 0)], {0: [1] * 64}, {0: EXAMPLE_DC}, {0: EXAMPLE_AC}, scan)
