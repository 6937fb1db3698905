// Host JFIF marker walk (reference parser.hpp:139-347) and Huffman table
// construction (huffman.hpp:60-93).  Same acceptance set and error codes as
// the reference; stops at the first entropy-coded byte.
#include "jfif.hpp"

#include <algorithm>
#include <cstring>

namespace pjg {
namespace {

struct Fail {
    int32_t code;
    const char* msg;
};

class Reader {
public:
    Reader(const uint8_t* b, size_t n) : b_(b), n_(n) {}
    uint8_t u8() {
        if (pos_ >= n_) throw Fail{kMalformedHeader, "truncated file"};
        return b_[pos_++];
    }
    uint16_t u16() {
        uint16_t hi = u8();
        return uint16_t((hi << 8) | u8());
    }
    Reader take(size_t n) {
        if (pos_ + n > n_) throw Fail{kMalformedHeader, "truncated segment"};
        Reader r(b_ + pos_, n);
        pos_ += n;
        return r;
    }
    bool eof() const { return pos_ >= n_; }
    const uint8_t* ptr() const { return b_ + pos_; }
    size_t pos() const { return pos_; }

private:
    const uint8_t* b_;
    size_t n_;
    size_t pos_ = 0;
};

bool is_rst(uint8_t m) { return m >= 0xD0 && m <= 0xD7; }
bool is_sof(uint8_t m) { return m >= 0xC0 && m <= 0xCF && m != 0xC4 && m != 0xC8 && m != 0xCC; }

// parser.hpp:139-154
void parse_dqt(Reader& r, uint16_t len, Header& h) {
    Reader s = r.take(len);
    while (!s.eof()) {
        uint8_t pq = s.u8();
        uint8_t prec = pq >> 4, id = pq & 15;
        if (id > 3) throw Fail{kMalformedHeader, "quant table id > 3"};
        if (prec > 1) throw Fail{kMalformedHeader, "bad quant precision"};
        // one bounds check per table, then a plain (vectorisable) conversion
        const Reader q = s.take(prec ? 128 : 64);
        const uint8_t* b = q.ptr();
        uint16_t* dst = h.quant[id].data();
        uint32_t any_zero = 0;
        if (prec) {
            for (int i = 0; i < 64; ++i) {
                dst[i] = uint16_t((b[2 * i] << 8) | b[2 * i + 1]);
                any_zero |= dst[i] == 0;
            }
        } else {
            for (int i = 0; i < 64; ++i) {
                dst[i] = b[i];
                any_zero |= b[i] == 0;
            }
        }
        if (any_zero) throw Fail{kMalformedHeader, "zero quantizer entry"};
        h.quant_present[id] = true;
    }
}

// parser.hpp:156-178
void parse_dht(Reader& r, uint16_t len, Header& h) {
    Reader s = r.take(len);
    while (!s.eof()) {
        uint8_t tcth = s.u8();
        uint8_t cls = tcth >> 4, id = tcth & 15;
        if (cls > 1) throw Fail{kUnsupportedFeature, "huffman table class > 1"};
        if (id > 3) throw Fail{kMalformedHeader, "huffman table id > 3"};
        HuffSpec sp;
        const Reader cr = s.take(16);
        std::memcpy(sp.counts.data(), cr.ptr(), 16);
        size_t total = 0;
        for (int i = 0; i < 16; ++i) total += sp.counts[i];
        if (total > 256) throw Fail{kMalformedHeader, "more than 256 huffman symbols"};
        Reader syms = s.take(total);
        sp.symbols.p = syms.ptr();
        sp.symbols.n = uint32_t(total);
        sp.present = true;
        (cls ? h.ac : h.dc)[id] = sp;
    }
}

// parser.hpp:180-233
void parse_sof0(Reader& r, uint16_t len, Header& h) {
    Reader s = r.take(len);
    if (s.u8() != 8) throw Fail{kUnsupportedFeature, "only 8-bit precision supported"};
    h.height = s.u16();
    h.width = s.u16();
    if (h.width == 0) throw Fail{kMalformedHeader, "zero width"};
    if (h.height == 0) throw Fail{kUnsupportedFeature, "DNL-deferred height not supported"};
    uint8_t nc = s.u8();
    if (nc < 1 || nc > 3) throw Fail{kUnsupportedFeature, "component count"};
    for (int i = 0; i < nc; ++i) {
        Component c;
        c.id = s.u8();
        uint8_t hv = s.u8();
        c.h = hv >> 4;
        c.v = hv & 15;
        c.tq = s.u8();
        if (c.tq > 3) throw Fail{kMalformedHeader, "quant table id > 3"};
        if (c.h < 1 || c.h > 2 || c.v < 1 || c.v > 2)
            throw Fail{kUnsupportedFeature, "sampling factors outside {1,2}"};
        h.comps.push_back(c);
    }
    if (nc == 1) {
        h.comps[0].h = h.comps[0].v = 1;
    } else {
        for (int i = 1; i < nc; ++i)
            if (h.comps[i].h != 1 || h.comps[i].v != 1)
                throw Fail{kUnsupportedFeature, "subsampled layout must be on chroma only"};
        const Component& y = h.comps[0];
        bool ok = (y.h == 1 && y.v == 1) || (y.h == 2 && y.v == 1) || (y.h == 2 && y.v == 2);
        if (!ok) throw Fail{kUnsupportedFeature, "unsupported sampling layout"};
    }
    for (const auto& c : h.comps) {
        h.h_max = std::max<uint32_t>(h.h_max, c.h);
        h.v_max = std::max<uint32_t>(h.v_max, c.v);
    }
    uint32_t mw = 8 * h.h_max, mh = 8 * h.v_max;
    h.mcus_x = (h.width + mw - 1) / mw;
    h.mcus_y = (h.height + mh - 1) / mh;
    for (size_t ci = 0; ci < h.comps.size(); ++ci)
        for (int k = 0; k < h.comps[ci].h * h.comps[ci].v; ++k) h.du_seq.push_back(uint8_t(ci));
    h.dpm = uint32_t(h.du_seq.size());
}

}  // namespace

Header parse_header(const uint8_t* data, size_t size, bool allow_dri) {
    Header h;
    try {
        Reader r(data, size);
        if (r.u8() != 0xFF || r.u8() != 0xD8) throw Fail{kMalformedHeader, "missing SOI marker"};
        bool have_frame = false;
        while (true) {
            if (r.u8() != 0xFF) throw Fail{kMalformedHeader, "expected marker prefix 0xFF"};
            uint8_t m = r.u8();
            while (m == 0xFF) m = r.u8();
            if (m == 0xD9) throw Fail{kMalformedHeader, "EOI before SOS"};
            if (is_rst(m)) throw Fail{kMalformedHeader, "stray RST marker"};
            if (is_sof(m) && m != 0xC0)
                throw Fail{kUnsupportedFeature, "only baseline SOF0 supported"};
            uint16_t len = r.u16();
            if (len < 2) throw Fail{kMalformedHeader, "segment length < 2"};
            len = uint16_t(len - 2);
            if ((m >= 0xE0 && m <= 0xEF) || m == 0xFE) {
                r.take(len);
            } else if (m == 0xDB) {
                parse_dqt(r, len, h);
            } else if (m == 0xC4) {
                parse_dht(r, len, h);
            } else if (m == 0xC0) {
                if (have_frame) throw Fail{kMalformedHeader, "multiple SOF segments"};
                parse_sof0(r, len, h);
                have_frame = true;
            } else if (m == 0xDD) {
                Reader s = r.take(len);
                const uint16_t ri = s.u16();
                if (ri != 0 && !allow_dri)
                    throw Fail{kUnsupportedFeature, "restart interval (DRI) not supported"};
                h.restart_interval = ri;
            } else if (m == 0xDC) {
                throw Fail{kUnsupportedFeature, "DNL segment not supported"};
            } else if (m == 0xDA) {
                if (!have_frame) throw Fail{kMalformedHeader, "SOS before SOF"};
                Reader s = r.take(len);
                uint8_t ns = s.u8();
                if (ns != h.comps.size())
                    throw Fail{kUnsupportedFeature, "scan component subset not supported"};
                for (int i = 0; i < ns; ++i) {
                    uint8_t cs = s.u8(), tdta = s.u8();
                    bool found = false;
                    for (auto& c : h.comps) {
                        if (c.id == cs) {
                            c.td = tdta >> 4;
                            c.ta = tdta & 15;
                            if (c.td > 3 || c.ta > 3)
                                throw Fail{kMalformedHeader, "huffman table id > 3 in SOS"};
                            found = true;
                            break;
                        }
                    }
                    if (!found) throw Fail{kMalformedHeader, "SOS references unknown component"};
                }
                uint8_t ss = s.u8(), se = s.u8(), ahal = s.u8();
                if (ss != 0 || se != 63 || ahal != 0)
                    throw Fail{kUnsupportedFeature, "non-baseline spectral selection"};
                for (const auto& c : h.comps) {
                    if (!h.quant_present[c.tq]) throw Fail{kMissingTable, "undefined quant table"};
                    if (!h.dc[c.td].present) throw Fail{kMissingTable, "undefined DC huffman table"};
                    if (!h.ac[c.ta].present) throw Fail{kMissingTable, "undefined AC huffman table"};
                }
                h.scan_start = r.pos();
                // decode_single builds every present table after parse()
                // returns (pipeline.hpp:107-112): a malformed table fails the
                // file only if the scan itself parsed, so the error is
                // deferred until K0 has checked the scan (ImgDesc::deferred).
                for (int i = 0; i < 4 && h.table_status == kOk; ++i) {
                    if (h.dc[i].present) h.table_status = validate_huff(h.dc[i]);
                    if (h.table_status == kOk && h.ac[i].present) h.table_status = validate_huff(h.ac[i]);
                }
                return h;
            } else {
                throw Fail{kMalformedHeader, "unexpected marker"};
            }
        }
    } catch (const Fail& f) {
        h.status = f.code;
        h.message = f.msg;
    }
    return h;
}

// build_table's error checks (huffman.hpp:60-93) without building the table.
int32_t validate_huff(const HuffSpec& spec) {
    uint32_t code = 0;
    size_t si = 0;
    uint32_t maxlen = 0;
    for (uint32_t len = 1; len <= 16; ++len) {
        const uint32_t n = spec.counts[len - 1];
        if (code + n > (1u << len)) return kOversubscribedCode;
        if (si + n > spec.symbols.size()) return kMalformedHeader;
        si += n;
        code += n;
        if (n) maxlen = len;
        code <<= 1;
    }
    if (si != spec.symbols.size()) return kMalformedHeader;
    if (maxlen == 0) return kMalformedHeader;
    return kOk;
}

int32_t build_dev_huff(const HuffSpec& spec, DevHuff* out) {
    std::memset(out, 0, sizeof(DevHuff));
    uint32_t code = 0;
    size_t si = 0;
    uint16_t codes[256];
    uint8_t lens[256];
    uint32_t maxlen = 0;
    for (int len = 0; len <= 17; ++len) out->maxcode[len] = -1;
    for (uint32_t len = 1; len <= 16; ++len) {
        uint32_t n = spec.counts[len - 1];
        if (code + n > (1u << len)) return kOversubscribedCode;
        if (n) out->valoff[len] = int32_t(si) - int32_t(code);
        for (uint32_t k = 0; k < n; ++k) {
            if (si >= spec.symbols.size()) return kMalformedHeader;
            codes[si] = uint16_t(code);
            lens[si] = uint8_t(len);
            out->symbols[si] = spec.symbols[si];
            ++si;
            ++code;
            maxlen = len;
        }
        if (n) out->maxcode[len] = int32_t(code) - 1;
        code <<= 1;
    }
    if (si != spec.symbols.size()) return kMalformedHeader;
    if (maxlen == 0) return kMalformedHeader;
    out->maxlen = maxlen;
    uint32_t n2 = 0;
    for (size_t k = 0; k < si; ++k) {
        const uint16_t e = uint16_t((uint32_t(lens[k]) << 8) | spec.symbols[k]);
        if (lens[k] <= kPrimaryBits) {
            uint32_t shift = kPrimaryBits - lens[k];
            uint32_t first = uint32_t(codes[k]) << shift, count = 1u << shift;
            for (uint32_t i = 0; i < count; ++i) out->lut[first + i] = e;
        } else {  // second level of the code's 9-bit prefix (allocated in code order)
            const uint32_t pre = uint32_t(codes[k]) >> (lens[k] - kPrimaryBits);
            if (out->lut[pre] == 0 && n2 < uint32_t(kL2Tables)) out->lut[pre] = uint16_t(kL2Flag | n2++);
            if (!(out->lut[pre] & kL2Flag)) continue;  // out of second-level tables: maxcode walk
            const uint32_t shift = 16 - lens[k];
            const uint32_t first = (uint32_t(codes[k]) << shift) & ((1u << (16 - kPrimaryBits)) - 1);
            for (uint32_t i = 0; i < (1u << shift); ++i) out->lut2[out->lut[pre] & 0x7FFFu][first + i] = e;
        }
    }
    return kOk;
}

// Fast table: decode_next_symbol (huffman.hpp:137-175) resolved for every
// kFastBits window whose codeword AND magnitude bits both fit; symbols the
// reference rejects (DC l > 11, AC l > 10, AC l == 0 with r not in {0, 15})
// are left to the exact path so its error order is preserved.  `dc` selects
// the class semantics the table is used with (DC at z == 0, AC otherwise).
void build_fast(DevHuff* t, bool dc) {
    uint32_t n2 = 0;
    std::memset(t->fast2, 0, sizeof(t->fast2));
    for (uint32_t w = 0; w < (1u << kFastBits); ++w) {
        const int64_t f = fast_primary(*t, w, dc);
        if (f >= 0) {
            t->fast[w] = uint32_t(f);
        } else if (n2 < uint32_t(kL2Fast)) {  // long codes: second level, in prefix order
            for (uint32_t s = 0; s < 32; ++s) t->fast2[n2][s] = fast_secondary(*t, w, s, dc);
            t->fast[w] = kFastL2 | (n2++ << 10);
        } else {
            t->fast[w] = 0;
        }
    }
}

}  // namespace pjg
