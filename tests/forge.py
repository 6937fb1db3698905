"""Test-only baseline JPEG forge: explicit quantised coefficient blocks ->
a baseline JPEG (SOF0, 8- or 16-bit DQT, one interleaved scan).

Used to reach inputs no image encoder produces: 16-bit quantisers up to
65535 (parse_dqt accepts precision 1, reference parser.hpp:139-154),
maximum-magnitude coefficients (DC category 11, AC category 10: the limits
decode_next_symbol enforces, huffman.hpp:138-175), DC predictors that wrap
int16 (dc_prefix_sum stores int16, transform.hpp:56-74).  Huffman tables are
flat canonical codes (every DC category at length 4, every AC symbol at
length 8), valid per Annex C and for build_table (huffman.hpp:60-93)."""
from __future__ import annotations

import numpy as np

DC_SYMS = list(range(12))
AC_SYMS = [0x00, 0xF0] + [(r << 4) | s for r in range(16) for s in range(1, 11)]
DC_SPEC = ([0, 0, 0, 12] + [0] * 12, DC_SYMS)           # 12 codes of length 4
AC_SPEC = ([0] * 7 + [len(AC_SYMS)] + [0] * 8, AC_SYMS)  # 162 codes of length 8

SAMPLING = {"444": ((1, 1), (1, 1), (1, 1)), "422": ((2, 1), (1, 1), (1, 1)),
            "420": ((2, 2), (1, 1), (1, 1)), "gray": ((1, 1),)}


class _Bits:
    def __init__(self):
        self.out = bytearray()
        self.acc = 0
        self.n = 0

    def put(self, v, n):
        for i in range(n - 1, -1, -1):
            self.acc = (self.acc << 1) | ((v >> i) & 1)
            self.n += 1
            if self.n == 8:
                self.out.append(self.acc)
                if self.acc == 0xFF:
                    self.out.append(0x00)  # byte stuffing
                self.acc = 0
                self.n = 0

    def flush(self):
        if self.n:
            self.put((1 << (8 - self.n)) - 1, 8 - self.n)  # pad with 1s
        return bytes(self.out)


def _canon(spec):
    counts, syms = spec
    code, k, table = 0, 0, {}
    for length in range(1, 17):
        for _ in range(counts[length - 1]):
            table[syms[k]] = (code, length)
            code += 1
            k += 1
        code <<= 1
    return table


DC_CODE = _canon(DC_SPEC)
AC_CODE = _canon(AC_SPEC)


def _cat(v):
    return 0 if v == 0 else int(abs(int(v))).bit_length()


def _mag(v, s):
    return v if v >= 0 else v + (1 << s) - 1


def encode_scan(blocks) -> bytes:
    """blocks: (n, 64) ints in zig-zag order, column 0 = the DC DIFFERENCE
    (|d| <= 2047), AC |v| <= 1023, in scan order."""
    bw = _Bits()
    for blk in np.asarray(blocks, np.int64):
        d = int(blk[0])
        s = _cat(d)
        assert s <= 11, d
        c, ln = DC_CODE[s]
        bw.put(c, ln)
        if s:
            bw.put(_mag(d, s), s)
        run = 0
        last = max([k for k in range(1, 64) if blk[k] != 0], default=0)
        for k in range(1, last + 1):
            v = int(blk[k])
            if v == 0:
                run += 1
                continue
            while run > 15:
                c, ln = AC_CODE[0xF0]
                bw.put(c, ln)
                run -= 16
            s = _cat(v)
            assert s <= 10, v
            c, ln = AC_CODE[(run << 4) | s]
            bw.put(c, ln)
            bw.put(_mag(v, s), s)
            run = 0
        if last < 63:
            c, ln = AC_CODE[0x00]
            bw.put(c, ln)
    return bw.flush()


def forge(width, height, sampling, quant, blocks, qmap=None) -> bytes:
    """quant: {table id: 64 zig-zag entries (any <= 255 -> 8-bit DQT, else 16-bit)};
    qmap: quant table id per component (default: Y -> 0, chroma -> 1 or 0)."""
    samp = SAMPLING[sampling]
    nc = len(samp)
    if qmap is None:
        qmap = [0] + [1 if 1 in quant else 0] * (nc - 1)
    out = bytearray(b"\xff\xd8")
    for tid, q in quant.items():
        q = [int(x) for x in q]
        if max(q) > 255:
            body = bytes([0x10 | tid]) + b"".join(int(x).to_bytes(2, "big") for x in q)
        else:
            body = bytes([tid]) + bytes(q)
        out += b"\xff\xdb" + (2 + len(body)).to_bytes(2, "big") + body
    out += b"\xff\xc0" + (8 + 3 * nc).to_bytes(2, "big") + bytes([8]) + height.to_bytes(2, "big") + \
        width.to_bytes(2, "big") + bytes([nc])
    for c in range(nc):
        h, v = samp[c]
        out += bytes([c + 1, (h << 4) | v, qmap[c]])
    for cls, spec in ((0, DC_SPEC), (1, AC_SPEC)):
        counts, syms = spec
        out += b"\xff\xc4" + (3 + 16 + len(syms)).to_bytes(2, "big") + bytes([cls << 4]) + bytes(counts) + bytes(syms)
    out += b"\xff\xda" + (6 + 2 * nc).to_bytes(2, "big") + bytes([nc])
    for c in range(nc):
        out += bytes([c + 1, 0x00])
    out += bytes([0, 63, 0]) + encode_scan(blocks) + b"\xff\xd9"
    return bytes(out)


def data_units(width, height, sampling):
    samp = SAMPLING[sampling]
    hmax = max(h for h, _ in samp)
    vmax = max(v for _, v in samp)
    mx = -(-width // (8 * hmax))
    my = -(-height // (8 * vmax))
    return mx * my * sum(h * v for h, v in samp)
