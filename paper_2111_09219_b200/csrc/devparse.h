// The device planner's JFIF marker walk (parse(), parser.hpp:264-347 with
// parse_dqt :139-154, parse_dht :156-178, parse_sof0 :180-233): same
// acceptance set and Errc precedence as the reference, header-only output.
// Host+device: devplan.cu runs it per file on the GPU; pjg_debug_device_parse
// runs the same code on the host so CPU tests can pin it.
#pragma once

#include <cstring>

#include "devplan.h"

namespace pjg {

// MSB-first byte reader over one file in the raw buffer with a 16-byte
// register cache (header bytes are read sequentially).
struct DReader {
    const uint8_t* base;  // raw buffer (16-byte aligned)
    uint64_t f0;          // file start in the raw buffer
    uint64_t size;        // file bytes
    uint64_t pos = 0;     // file-relative
    uint64_t cidx = ~0ull;
    uint4 ch;
    PJG_HD uint32_t byte_at(uint64_t p) {
        const uint64_t a = f0 + p;
        if ((a >> 4) != cidx) {
            cidx = a >> 4;
#ifdef __CUDA_ARCH__
            ch = __ldg(reinterpret_cast<const uint4*>(base) + cidx);
#else
            memcpy(&ch, base + cidx * 16, 16);
#endif
        }
        const uint32_t k = uint32_t(a & 15);
        const uint32_t w = k < 8 ? (k < 4 ? ch.x : ch.y) : (k < 12 ? ch.z : ch.w);
        return (w >> (8 * (k & 3))) & 0xFFu;
    }
    // u8 within [.., end): false = truncated (MalformedHeader at every site)
    PJG_HD bool u8(uint64_t end, uint32_t& v) {
        if (pos >= end) return false;
        v = byte_at(pos++);
        return true;
    }
    PJG_HD bool u16(uint64_t end, uint32_t& v) {
        uint32_t a, b;
        if (!u8(end, a) || !u8(end, b)) return false;
        v = (a << 8) | b;
        return true;
    }
    PJG_HD bool take(uint64_t end, uint64_t n, uint64_t& seg_end) {
        if (pos + n > end) return false;
        seg_end = pos + n;
        return true;
    }
};

#define PFAIL(code)         \
    do {                    \
        h.status = (code);  \
        return;             \
    } while (0)
#define PGET8(end, v) \
    if (!r.u8((end), (v))) PFAIL(kMalformedHeader)
#define PGET16(end, v) \
    if (!r.u16((end), (v))) PFAIL(kMalformedHeader)

PJG_HD bool is_sof(uint32_t m) { return m >= 0xC0 && m <= 0xCF && m != 0xC4 && m != 0xC8 && m != 0xCC; }

// build_table's validation (huffman.hpp:60-93): oversubscription, then an
// empty table; count/symbol agreement holds by construction (nsym = sum).
PJG_HD int32_t validate_counts(DReader& r, uint64_t off) {
    uint32_t code = 0, maxlen = 0;
    for (uint32_t len = 1; len <= 16; ++len) {
        const uint32_t n = r.byte_at(off + len - 1);
        if (code + n > (1u << len)) return kOversubscribedCode;
        code += n;
        if (n) maxlen = len;
        code <<= 1;
    }
    return maxlen == 0 ? kMalformedHeader : kOk;
}

// parse() up to and including SOS (parser.hpp:264-347).  Header-only output.
PJG_HD void parse_file(DReader& r, bool allow_dri, DevHdr& h) {
    const uint64_t E = r.size;
    uint32_t a, b;
    PGET8(E, a);
    if (a != 0xFF) PFAIL(kMalformedHeader);  // missing SOI
    PGET8(E, b);
    if (b != 0xD8) PFAIL(kMalformedHeader);
    bool have_frame = false;
    for (;;) {
        uint32_t x, m, len;
        PGET8(E, x);
        if (x != 0xFF) PFAIL(kMalformedHeader);  // expected marker prefix
        PGET8(E, m);
        while (m == 0xFF) PGET8(E, m);
        if (m == 0xD9) PFAIL(kMalformedHeader);                // EOI before SOS
        if (m >= 0xD0 && m <= 0xD7) PFAIL(kMalformedHeader);   // stray RST
        if (is_sof(m) && m != 0xC0) PFAIL(kUnsupportedFeature);  // only baseline SOF0
        PGET16(E, len);
        if (len < 2) PFAIL(kMalformedHeader);
        len -= 2;
        uint64_t se;  // segment end
        if ((m >= 0xE0 && m <= 0xEF) || m == 0xFE) {
            if (!r.take(E, len, se)) PFAIL(kMalformedHeader);
            r.pos = se;
        } else if (m == 0xDB) {  // parse_dqt
            if (!r.take(E, len, se)) PFAIL(kMalformedHeader);
            while (r.pos < se) {
                uint32_t pq;
                PGET8(se, pq);
                const uint32_t prec = pq >> 4, id = pq & 15u;
                if (id > 3) PFAIL(kMalformedHeader);
                if (prec > 1) PFAIL(kMalformedHeader);
                uint64_t qe;
                if (!r.take(se, prec ? 128 : 64, qe)) PFAIL(kMalformedHeader);
                const uint64_t q0 = r.pos;
                uint32_t any_zero = 0;
                for (uint32_t i = 0; i < 64; ++i) {
                    const uint32_t v = prec ? (r.byte_at(q0 + 2 * i) << 8) | r.byte_at(q0 + 2 * i + 1) : r.byte_at(q0 + i);
                    any_zero |= v == 0;
                }
                r.pos = qe;
                if (any_zero) PFAIL(kMalformedHeader);
                h.q_off[id] = q0;
                h.q_prec[id] = uint8_t(prec);
                h.q_present |= uint8_t(1u << id);
            }
            r.pos = se;
        } else if (m == 0xC4) {  // parse_dht
            if (!r.take(E, len, se)) PFAIL(kMalformedHeader);
            while (r.pos < se) {
                uint32_t tcth;
                PGET8(se, tcth);
                const uint32_t cls = tcth >> 4, id = tcth & 15u;
                if (cls > 1) PFAIL(kUnsupportedFeature);
                if (id > 3) PFAIL(kMalformedHeader);
                uint64_t ce;
                if (!r.take(se, 16, ce)) PFAIL(kMalformedHeader);
                const uint64_t c0 = r.pos;
                uint32_t total = 0;
                for (uint32_t i = 0; i < 16; ++i) total += r.byte_at(c0 + i);
                r.pos = ce;
                if (total > 256) PFAIL(kMalformedHeader);
                uint64_t ye;
                if (!r.take(se, total, ye)) PFAIL(kMalformedHeader);
                r.pos = ye;
                if (cls) {
                    h.ac_off[id] = c0;
                    h.ac_n[id] = uint16_t(total);
                    h.ac_present |= uint8_t(1u << id);
                } else {
                    h.dc_off[id] = c0;
                    h.dc_n[id] = uint16_t(total);
                    h.dc_present |= uint8_t(1u << id);
                }
            }
            r.pos = se;
        } else if (m == 0xC0) {  // parse_sof0
            if (have_frame) PFAIL(kMalformedHeader);  // multiple SOF segments
            if (!r.take(E, len, se)) PFAIL(kMalformedHeader);
            uint32_t prec, hh, ww, nc;
            PGET8(se, prec);
            if (prec != 8) PFAIL(kUnsupportedFeature);
            PGET16(se, hh);
            PGET16(se, ww);
            h.height = hh;
            h.width = ww;
            if (ww == 0) PFAIL(kMalformedHeader);
            if (hh == 0) PFAIL(kUnsupportedFeature);  // DNL-deferred height
            PGET8(se, nc);
            if (nc < 1 || nc > 3) PFAIL(kUnsupportedFeature);
            for (uint32_t i = 0; i < nc; ++i) {
                uint32_t id, hv, tq;
                PGET8(se, id);
                PGET8(se, hv);
                PGET8(se, tq);
                h.cid[i] = uint8_t(id);
                h.ch[i] = uint8_t(hv >> 4);
                h.cv[i] = uint8_t(hv & 15u);
                h.tq[i] = uint8_t(tq);
                if (tq > 3) PFAIL(kMalformedHeader);
                if (h.ch[i] < 1 || h.ch[i] > 2 || h.cv[i] < 1 || h.cv[i] > 2) PFAIL(kUnsupportedFeature);
                h.ncomp = i + 1;  // comps.push_back after the checks (a failing file's infos count it)
            }
            if (nc == 1) {
                h.ch[0] = h.cv[0] = 1;
            } else {
                for (uint32_t i = 1; i < nc; ++i)
                    if (h.ch[i] != 1 || h.cv[i] != 1) PFAIL(kUnsupportedFeature);
                const bool ok = (h.ch[0] == 1 && h.cv[0] == 1) || (h.ch[0] == 2 && h.cv[0] == 1) ||
                                (h.ch[0] == 2 && h.cv[0] == 2);
                if (!ok) PFAIL(kUnsupportedFeature);
            }
            h.h_max = h.v_max = 1;
            for (uint32_t i = 0; i < nc; ++i) {
                h.h_max = h.h_max > h.ch[i] ? h.h_max : uint32_t(h.ch[i]);
                h.v_max = h.v_max > h.cv[i] ? h.v_max : uint32_t(h.cv[i]);
            }
            const uint32_t mw = 8 * h.h_max, mh = 8 * h.v_max;
            h.mcus_x = (ww + mw - 1) / mw;
            h.mcus_y = (hh + mh - 1) / mh;
            uint32_t k = 0;
            h.du_comp = h.du_kslot = 0;
            for (uint32_t ci = 0; ci < nc; ++ci)
                for (uint32_t j = 0; j < uint32_t(h.ch[ci]) * h.cv[ci]; ++j, ++k) {
                    h.du_comp |= uint64_t(ci) << (4 * k);
                    h.du_kslot |= uint64_t(j) << (4 * k);
                }
            h.dpm = k;
            r.pos = se;
            have_frame = true;
        } else if (m == 0xDD) {  // DRI
            if (!r.take(E, len, se)) PFAIL(kMalformedHeader);
            uint32_t ri;
            PGET16(se, ri);
            if (ri != 0 && !allow_dri) PFAIL(kUnsupportedFeature);
            h.restart_interval = ri;
            r.pos = se;
        } else if (m == 0xDC) {
            PFAIL(kUnsupportedFeature);  // DNL
        } else if (m == 0xDA) {  // SOS
            if (!have_frame) PFAIL(kMalformedHeader);
            if (!r.take(E, len, se)) PFAIL(kMalformedHeader);
            uint32_t ns;
            PGET8(se, ns);
            if (ns != h.ncomp) PFAIL(kUnsupportedFeature);  // scan component subset
            for (uint32_t i = 0; i < ns; ++i) {
                uint32_t cs, tdta;
                PGET8(se, cs);
                PGET8(se, tdta);
                int found = -1;
                for (uint32_t c = 0; c < h.ncomp; ++c)
                    if (h.cid[c] == cs) {
                        found = int(c);
                        break;
                    }
                if (found >= 0) {
                    h.td[found] = uint8_t(tdta >> 4);
                    h.ta[found] = uint8_t(tdta & 15u);
                    if (h.td[found] > 3 || h.ta[found] > 3) PFAIL(kMalformedHeader);
                } else {
                    PFAIL(kMalformedHeader);  // unknown component
                }
            }
            uint32_t ss, sse, ahal;
            PGET8(se, ss);
            PGET8(se, sse);
            PGET8(se, ahal);
            if (ss != 0 || sse != 63 || ahal != 0) PFAIL(kUnsupportedFeature);
            for (uint32_t c = 0; c < h.ncomp; ++c) {
                if (!((h.q_present >> h.tq[c]) & 1u)) PFAIL(kMissingTable);
                if (!((h.dc_present >> h.td[c]) & 1u)) PFAIL(kMissingTable);
                if (!((h.ac_present >> h.ta[c]) & 1u)) PFAIL(kMissingTable);
            }
            h.scan_start = se;  // r.pos after the SOS segment
            for (uint32_t i = 0; i < 4 && h.table_status == kOk; ++i) {
                if ((h.dc_present >> i) & 1u) h.table_status = validate_counts(r, h.dc_off[i]);
                if (h.table_status == kOk && ((h.ac_present >> i) & 1u)) h.table_status = validate_counts(r, h.ac_off[i]);
            }
            h.status = kOk;
            // extract_scan of nothing -> unstuff throws EmptyScan
            if (r.size == h.scan_start) h.status = kEmptyScan;
            return;
        } else {
            PFAIL(kMalformedHeader);  // unexpected marker
        }
    }
}


}  // namespace pjg
