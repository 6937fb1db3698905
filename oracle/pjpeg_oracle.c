/*
 * TEST INFRASTRUCTURE ONLY — the parity oracle's plain-C restatement.
 *
 * A CPU restatement, in C11, of the reference decode path
 * (/root/reference/proj/include/pjpeg/*.hpp).  It is the checker for the
 * CUDA product path and is pinned against the reference itself
 * (oracle/_ref/libpjpeg_ref.so, compiled in place from the reference headers)
 * and against the reference's own KATs (tests/golden/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off (FMA
 * contraction changes the reference's own output).
 *
 * Each function cites the reference file:line it restates.  Status codes are
 * pjpeg::Errc ordinal + 1 (common.hpp:26-38); 0 = success.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

enum {
    E_OK = 0,
    E_MALFORMED_STUFFING = 1,
    E_EMPTY_SCAN = 2,
    E_OUT_OF_BITS = 3,
    E_UNSUPPORTED = 4,
    E_MALFORMED_HEADER = 5,
    E_MISSING_TABLE = 6,
    E_OVERSUBSCRIBED = 7,
    E_INVALID_CODE = 8,
    E_CONSISTENCY = 9,
    E_NOMEM = 100,
    E_CAPACITY = 101
};

/* common.hpp:69-73 */
static const uint8_t kZigzagToRaster[64] = {
    0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
    12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
    35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
    58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

/* common.hpp:83-87 */
static uint8_t clamp_u8(int v) { return v < 0 ? 0 : (v > 255 ? 255 : (uint8_t)v); }

/* ---------------------------------------------------------------- parse -- */

typedef struct {
    uint8_t id, h, v, tq, td, ta;
} orc_comp;

typedef struct {
    uint8_t counts[16];
    uint8_t symbols[256];
    int nsym;
    int present;
} orc_hspec;

typedef struct {
    uint8_t maxlen;
    uint8_t *sym; /* flat LUT of 2^maxlen entries (huffman.hpp:85-91) */
    uint8_t *len; /* 0 = invalid prefix */
} orc_htable;

typedef struct {
    uint32_t width, height;
    int ncomp;
    orc_comp comp[3];
    uint32_t mcus_x, mcus_y, dpm;
    uint8_t h_max, v_max;
    uint8_t du_seq[10];
    uint16_t quant[4][64];
    int quant_present[4];
    orc_hspec dc[4], ac[4];
    uint8_t *seg; /* unstuffed scan */
    uint64_t seg_bytes, bit_length;
} orc_image;

typedef struct {
    const uint8_t *b;
    size_t n, pos;
    int err;
} orc_reader;

static int rd_u8(orc_reader *r, uint8_t *v) {
    if (r->pos >= r->n) return E_MALFORMED_HEADER; /* parser.hpp:114-116 */
    *v = r->b[r->pos++];
    return 0;
}
static int rd_u16(orc_reader *r, uint16_t *v) {
    uint8_t hi, lo;
    int e = rd_u8(r, &hi);
    if (e) return e;
    e = rd_u8(r, &lo);
    if (e) return e;
    *v = (uint16_t)((hi << 8) | lo);
    return 0;
}
static int rd_take(orc_reader *r, size_t n, orc_reader *sub) {
    if (r->pos + n > r->n) return E_MALFORMED_HEADER; /* parser.hpp:122-127 */
    sub->b = r->b + r->pos;
    sub->n = n;
    sub->pos = 0;
    r->pos += n;
    return 0;
}

#define TRY(x)              \
    do {                    \
        int e__ = (x);      \
        if (e__) return e__; \
    } while (0)

/* parser.hpp:139-154 */
static int parse_dqt(orc_reader *r, uint16_t len, orc_image *img) {
    orc_reader s;
    TRY(rd_take(r, len, &s));
    while (s.pos < s.n) {
        uint8_t pq;
        TRY(rd_u8(&s, &pq));
        uint8_t prec = pq >> 4, id = pq & 15;
        if (id > 3) return E_MALFORMED_HEADER;
        if (prec > 1) return E_MALFORMED_HEADER;
        for (int i = 0; i < 64; ++i) {
            if (prec) {
                TRY(rd_u16(&s, &img->quant[id][i]));
            } else {
                uint8_t v;
                TRY(rd_u8(&s, &v));
                img->quant[id][i] = v;
            }
        }
        for (int i = 0; i < 64; ++i)
            if (img->quant[id][i] == 0) return E_MALFORMED_HEADER;
        img->quant_present[id] = 1;
    }
    return 0;
}

/* parser.hpp:156-178 */
static int parse_dht(orc_reader *r, uint16_t len, orc_image *img) {
    orc_reader s;
    TRY(rd_take(r, len, &s));
    while (s.pos < s.n) {
        uint8_t tcth;
        TRY(rd_u8(&s, &tcth));
        uint8_t cls = tcth >> 4, id = tcth & 15;
        if (cls > 1) return E_UNSUPPORTED;
        if (id > 3) return E_MALFORMED_HEADER;
        orc_hspec sp;
        memset(&sp, 0, sizeof sp);
        int total = 0;
        for (int i = 0; i < 16; ++i) {
            TRY(rd_u8(&s, &sp.counts[i]));
            total += sp.counts[i];
        }
        if (total > 256) return E_MALFORMED_HEADER;
        orc_reader syms;
        TRY(rd_take(&s, (size_t)total, &syms));
        memcpy(sp.symbols, syms.b, (size_t)total);
        sp.nsym = total;
        sp.present = 1;
        if (cls)
            img->ac[id] = sp;
        else
            img->dc[id] = sp;
    }
    return 0;
}

/* parser.hpp:180-233 */
static int parse_sof0(orc_reader *r, uint16_t len, orc_image *img) {
    orc_reader s;
    TRY(rd_take(r, len, &s));
    uint8_t prec;
    TRY(rd_u8(&s, &prec));
    if (prec != 8) return E_UNSUPPORTED;
    uint16_t h, w;
    TRY(rd_u16(&s, &h));
    TRY(rd_u16(&s, &w));
    img->height = h;
    img->width = w;
    if (w == 0) return E_MALFORMED_HEADER;
    if (h == 0) return E_UNSUPPORTED;
    uint8_t nc;
    TRY(rd_u8(&s, &nc));
    if (nc < 1 || nc > 3) return E_UNSUPPORTED;
    img->ncomp = nc;
    for (int i = 0; i < nc; ++i) {
        orc_comp c;
        memset(&c, 0, sizeof c);
        uint8_t hv;
        TRY(rd_u8(&s, &c.id));
        TRY(rd_u8(&s, &hv));
        c.h = hv >> 4;
        c.v = hv & 15;
        TRY(rd_u8(&s, &c.tq));
        if (c.tq > 3) return E_MALFORMED_HEADER;
        if (c.h < 1 || c.h > 2 || c.v < 1 || c.v > 2) return E_UNSUPPORTED;
        img->comp[i] = c;
    }
    if (nc == 1) {
        img->comp[0].h = 1;
        img->comp[0].v = 1;
    } else {
        for (int i = 1; i < nc; ++i)
            if (img->comp[i].h != 1 || img->comp[i].v != 1) return E_UNSUPPORTED;
        uint8_t yh = img->comp[0].h, yv = img->comp[0].v;
        int ok = (yh == 1 && yv == 1) || (yh == 2 && yv == 1) || (yh == 2 && yv == 2);
        if (!ok) return E_UNSUPPORTED;
    }
    img->h_max = 1;
    img->v_max = 1;
    for (int i = 0; i < nc; ++i) {
        if (img->comp[i].h > img->h_max) img->h_max = img->comp[i].h;
        if (img->comp[i].v > img->v_max) img->v_max = img->comp[i].v;
    }
    uint32_t mw = 8u * img->h_max, mh = 8u * img->v_max;
    img->mcus_x = (img->width + mw - 1) / mw;
    img->mcus_y = (img->height + mh - 1) / mh;
    img->dpm = 0;
    for (int ci = 0; ci < nc; ++ci)
        for (int k = 0; k < img->comp[ci].h * img->comp[ci].v; ++k) img->du_seq[img->dpm++] = (uint8_t)ci;
    return 0;
}

static int is_rst(uint8_t m) { return m >= 0xD0 && m <= 0xD7; }
static int is_sof(uint8_t m) { return m >= 0xC0 && m <= 0xCF && m != 0xC4 && m != 0xC8 && m != 0xCC; }

/* extract_scan (parser.hpp:238-258) + unstuff (bitstream.hpp:56-76) */
static int extract_and_unstuff(orc_reader *r, orc_image *img) {
    const uint8_t *rest = r->b + r->pos;
    size_t n = r->n - r->pos, i = 0;
    while (i < n) {
        if (rest[i] == 0xFF) {
            if (i + 1 >= n) break;
            uint8_t nx = rest[i + 1];
            if (nx == 0x00) {
                i += 2;
                continue;
            }
            if (is_rst(nx)) return E_UNSUPPORTED;
            break;
        }
        ++i;
    }
    if (i == 0) return E_EMPTY_SCAN;
    img->seg = (uint8_t *)malloc(i + 8);
    if (!img->seg) return E_NOMEM;
    size_t o = 0;
    for (size_t k = 0; k < i; ++k) {
        uint8_t b = rest[k];
        img->seg[o++] = b;
        if (b == 0xFF) {
            if (k + 1 >= i) return E_MALFORMED_STUFFING;
            if (rest[k + 1] != 0x00) return E_MALFORMED_STUFFING;
            ++k;
        }
    }
    img->seg_bytes = o;
    img->bit_length = (uint64_t)o * 8;
    return 0;
}

/* parse (parser.hpp:264-347) */
static int orc_parse(const uint8_t *file, size_t size, orc_image *img) {
    memset(img, 0, sizeof *img);
    orc_reader r = {file, size, 0, 0};
    uint8_t a, b;
    TRY(rd_u8(&r, &a));
    TRY(rd_u8(&r, &b));
    if (a != 0xFF || b != 0xD8) return E_MALFORMED_HEADER;
    int have_frame = 0;
    for (;;) {
        uint8_t p, m;
        TRY(rd_u8(&r, &p));
        if (p != 0xFF) return E_MALFORMED_HEADER;
        TRY(rd_u8(&r, &m));
        while (m == 0xFF) TRY(rd_u8(&r, &m));
        if (m == 0xD9) return E_MALFORMED_HEADER;
        if (is_rst(m)) return E_MALFORMED_HEADER;
        if (is_sof(m) && m != 0xC0) return E_UNSUPPORTED;
        uint16_t len;
        TRY(rd_u16(&r, &len));
        if (len < 2) return E_MALFORMED_HEADER;
        len = (uint16_t)(len - 2);
        if ((m >= 0xE0 && m <= 0xEF) || m == 0xFE) {
            orc_reader skip;
            TRY(rd_take(&r, len, &skip));
        } else if (m == 0xDB) {
            TRY(parse_dqt(&r, len, img));
        } else if (m == 0xC4) {
            TRY(parse_dht(&r, len, img));
        } else if (m == 0xC0) {
            if (have_frame) return E_MALFORMED_HEADER;
            TRY(parse_sof0(&r, len, img));
            have_frame = 1;
        } else if (m == 0xDD) {
            orc_reader s;
            uint16_t ri;
            TRY(rd_take(&r, len, &s));
            TRY(rd_u16(&s, &ri));
            if (ri != 0) return E_UNSUPPORTED;
        } else if (m == 0xDC) {
            return E_UNSUPPORTED;
        } else if (m == 0xDA) {
            if (!have_frame) return E_MALFORMED_HEADER;
            orc_reader s;
            TRY(rd_take(&r, len, &s));
            uint8_t ns;
            TRY(rd_u8(&s, &ns));
            if (ns != img->ncomp) return E_UNSUPPORTED;
            for (int i = 0; i < ns; ++i) {
                uint8_t cs, tdta;
                TRY(rd_u8(&s, &cs));
                TRY(rd_u8(&s, &tdta));
                int found = 0;
                for (int k = 0; k < img->ncomp; ++k) {
                    if (img->comp[k].id == cs) {
                        img->comp[k].td = tdta >> 4;
                        img->comp[k].ta = tdta & 15;
                        if (img->comp[k].td > 3 || img->comp[k].ta > 3) return E_MALFORMED_HEADER;
                        found = 1;
                        break;
                    }
                }
                if (!found) return E_MALFORMED_HEADER;
            }
            uint8_t ss, se, ahal;
            TRY(rd_u8(&s, &ss));
            TRY(rd_u8(&s, &se));
            TRY(rd_u8(&s, &ahal));
            if (ss != 0 || se != 63 || ahal != 0) return E_UNSUPPORTED;
            for (int k = 0; k < img->ncomp; ++k) {
                if (!img->quant_present[img->comp[k].tq]) return E_MISSING_TABLE;
                if (!img->dc[img->comp[k].td].present) return E_MISSING_TABLE;
                if (!img->ac[img->comp[k].ta].present) return E_MISSING_TABLE;
            }
            return extract_and_unstuff(&r, img);
        } else {
            return E_MALFORMED_HEADER;
        }
    }
}

/* build_table (huffman.hpp:60-93) */
static int build_table(const orc_hspec *sp, orc_htable *t) {
    uint32_t code = 0;
    int si = 0;
    uint16_t codes[256];
    uint8_t lens[256];
    t->maxlen = 0;
    for (unsigned len = 1; len <= 16; ++len) {
        uint32_t n = sp->counts[len - 1];
        if (code + n > (1u << len)) return E_OVERSUBSCRIBED;
        for (uint32_t k = 0; k < n; ++k) {
            if (si >= sp->nsym) return E_MALFORMED_HEADER;
            codes[si] = (uint16_t)code;
            lens[si] = (uint8_t)len;
            ++si;
            ++code;
            t->maxlen = (uint8_t)len;
        }
        code <<= 1;
    }
    if (si != sp->nsym) return E_MALFORMED_HEADER;
    if (t->maxlen == 0) return E_MALFORMED_HEADER;
    size_t size = (size_t)1 << t->maxlen;
    t->sym = (uint8_t *)calloc(size, 1);
    t->len = (uint8_t *)calloc(size, 1);
    if (!t->sym || !t->len) return E_NOMEM;
    for (int k = 0; k < si; ++k) {
        unsigned shift = t->maxlen - lens[k];
        size_t first = (size_t)codes[k] << shift, cnt = (size_t)1 << shift;
        for (size_t i = 0; i < cnt; ++i) {
            t->sym[first + i] = sp->symbols[k];
            t->len[first + i] = lens[k];
        }
    }
    return 0;
}

static void free_table(orc_htable *t) {
    free(t->sym);
    free(t->len);
    t->sym = t->len = NULL;
}

/* EntropySegment::peek (bitstream.hpp:44-52): MSB-first, zero past the end */
static uint32_t peek(const orc_image *img, uint64_t pos, unsigned k) {
    uint32_t v = 0;
    for (unsigned i = 0; i < k; ++i) {
        uint64_t p = pos + i;
        uint32_t bit = 0;
        if (p < img->bit_length) bit = (img->seg[p >> 3] >> (7 - (p & 7))) & 1;
        v = (v << 1) | bit;
    }
    return v;
}

/* extend (huffman.hpp:97-101) */
static int32_t extend(uint32_t bits, unsigned l) {
    if (l == 0) return 0;
    if (bits >= (1u << (l - 1))) return (int32_t)bits;
    return (int32_t)bits - (int32_t)((1u << l) - 1);
}

enum { K_COEF = 0, K_EOB = 1, K_ZRL = 2 };

/* decode_codeword (huffman.hpp:113-130) */
static int decode_codeword(const orc_image *img, uint64_t *pos, const orc_htable *t, unsigned *sym,
                           unsigned *clen) {
    uint64_t avail = *pos >= img->bit_length ? 0 : img->bit_length - *pos;
    if (avail == 0) return E_OUT_OF_BITS;
    uint32_t w = peek(img, *pos, t->maxlen);
    unsigned len = t->len[w];
    if (len == 0) {
        if (avail < t->maxlen) return E_OUT_OF_BITS;
        return E_INVALID_CODE;
    }
    if (len > avail) return E_OUT_OF_BITS;
    *pos += len;
    *clen = len;
    *sym = t->sym[w];
    return 0;
}

/* decode_next_symbol (huffman.hpp:137-175) */
static int decode_next_symbol(const orc_image *img, uint64_t *pos, unsigned z, const orc_htable *dc,
                              const orc_htable *ac, int *kind, int32_t *coef, unsigned *run) {
    unsigned sym, clen;
    if (z == 0) {
        TRY(decode_codeword(img, pos, dc, &sym, &clen));
        unsigned l = sym;
        if (l > 11) return E_INVALID_CODE;
        uint64_t rem = *pos >= img->bit_length ? 0 : img->bit_length - *pos;
        if (rem < l) return E_OUT_OF_BITS;
        *coef = extend(l ? peek(img, *pos, l) : 0, l);
        *pos += l;
        *kind = K_COEF;
        *run = 0;
        return 0;
    }
    TRY(decode_codeword(img, pos, ac, &sym, &clen));
    unsigned r = sym >> 4, l = sym & 15;
    if (l == 0) {
        if (r == 0) {
            *kind = K_EOB;
            *run = 63 - z;
        } else if (r == 15) {
            *kind = K_ZRL;
            *run = 15;
        } else {
            return E_INVALID_CODE;
        }
        return 0;
    }
    if (l > 10) return E_INVALID_CODE;
    uint64_t rem = *pos >= img->bit_length ? 0 : img->bit_length - *pos;
    if (rem < l) return E_OUT_OF_BITS;
    *coef = extend(peek(img, *pos, l), l);
    *pos += l;
    *kind = K_COEF;
    *run = r;
    return 0;
}

/* ------------------------------------------------------- public entries -- */

typedef struct {
    uint64_t p, n, c, z;
} orc_state;

/*
 * oracle_decode (oracle.hpp:47-98): one cursor walks the scan, snapshotting
 * the state at each boundary.  coeffs: 64*DUs int16, pre-DC-prefix, zig-zag.
 */
static int decode_entropy(const orc_image *img, const uint64_t *boundaries, size_t nb, uint64_t *states,
                          uint8_t *valid, int16_t *coeffs, uint64_t *end_state) {
    orc_htable dc[4], ac[4];
    memset(dc, 0, sizeof dc);
    memset(ac, 0, sizeof ac);
    int err = 0;
    for (int i = 0; i < 4 && !err; ++i) {
        if (img->dc[i].present) err = build_table(&img->dc[i], &dc[i]);
        if (!err && img->ac[i].present) err = build_table(&img->ac[i], &ac[i]);
    }
    uint64_t total = (uint64_t)img->mcus_x * img->mcus_y * img->dpm;
    memset(coeffs, 0, total * 64 * sizeof(int16_t));
    orc_state st = {0, 0, 0, 0};
    uint64_t pos = 0, done = 0;
    size_t nbd = 0;
    while (!err && done < total) {
        while (nbd < nb && boundaries[nbd] <= pos) {
            states[4 * nbd + 0] = st.p;
            states[4 * nbd + 1] = st.n;
            states[4 * nbd + 2] = st.c;
            states[4 * nbd + 3] = st.z;
            valid[nbd] = 1;
            ++nbd;
        }
        unsigned comp = img->du_seq[st.c];
        int kind;
        int32_t coef = 0;
        unsigned run;
        err = decode_next_symbol(img, &pos, (unsigned)st.z, &dc[img->comp[comp].td], &ac[img->comp[comp].ta],
                                 &kind, &coef, &run);
        if (err) break;
        if (kind == K_COEF) coeffs[st.n + run] = (int16_t)coef;
        st.p = pos;
        st.n += run + 1;
        st.z += run + 1;
        if (st.z > 64) {
            err = E_INVALID_CODE;
            break;
        }
        if (st.z == 64 || kind == K_EOB) {
            st.z = 0;
            st.c = (st.c + 1) % img->dpm;
            ++done;
        }
    }
    if (end_state) {
        end_state[0] = st.p;
        end_state[1] = st.n;
        end_state[2] = st.c;
        end_state[3] = st.z;
    }
    while (nbd < nb) {
        states[4 * nbd + 0] = st.p;
        states[4 * nbd + 1] = st.n;
        states[4 * nbd + 2] = st.c;
        states[4 * nbd + 3] = st.z;
        valid[nbd] = 0;
        ++nbd;
    }
    for (int i = 0; i < 4; ++i) {
        free_table(&dc[i]);
        free_table(&ac[i]);
    }
    return err;
}

/* IdctBasis (transform.hpp:93-108), host libm cos like the reference. */
static double g_basis[8][8];
static int g_basis_ready = 0;
static void init_basis(void) {
    if (g_basis_ready) return;
    for (int u = 0; u < 8; ++u) {
        double cu = u == 0 ? 1.0 / sqrt(2.0) : 1.0;
        for (int x = 0; x < 8; ++x) g_basis[u][x] = 0.5 * cu * cos((2 * x + 1) * u * M_PI / 16.0);
    }
    g_basis_ready = 1;
}

/* idct_8x8_raw + idct_8x8 (transform.hpp:114-142) */
static void idct_8x8(const int32_t *block, uint8_t *out) {
    double tmp[8][8];
    for (int u = 0; u < 8; ++u)
        for (int y = 0; y < 8; ++y) {
            double s = 0;
            for (int v = 0; v < 8; ++v) s += g_basis[v][y] * block[u * 8 + v];
            tmp[u][y] = s;
        }
    for (int x = 0; x < 8; ++x)
        for (int y = 0; y < 8; ++y) {
            double s = 0;
            for (int u = 0; u < 8; ++u) s += g_basis[u][x] * tmp[u][y];
            out[x * 8 + y] = clamp_u8((int)lround(s) + 128);
        }
}

void orc_idct_8x8(const int32_t *block, uint8_t *out) {
    init_basis();
    idct_8x8(block, out);
}

void orc_idct_basis(double *out) {
    init_basis();
    memcpy(out, g_basis, sizeof g_basis);
}

int32_t orc_extend(uint32_t bits, unsigned l) { return extend(bits, l); }

/* geometry: w, h, ncomp, mcus_x, mcus_y, dpm, h_max, v_max, DUs, seg bytes,
 * bit_length lo/hi, pw0, ph0, pw1, ph1, pw2, ph2 */
int orc_parse_info(const uint8_t *file, size_t size, uint32_t *info) {
    orc_image img;
    int e = orc_parse(file, size, &img);
    if (!e) {
        info[0] = img.width;
        info[1] = img.height;
        info[2] = (uint32_t)img.ncomp;
        info[3] = img.mcus_x;
        info[4] = img.mcus_y;
        info[5] = img.dpm;
        info[6] = img.h_max;
        info[7] = img.v_max;
        info[8] = img.mcus_x * img.mcus_y * img.dpm;
        info[9] = (uint32_t)img.seg_bytes;
        info[10] = (uint32_t)(img.bit_length & 0xffffffffu);
        info[11] = (uint32_t)(img.bit_length >> 32);
        for (int c = 0; c < 3; ++c) {
            /* FrameInfo::comp_width/height (parser.hpp:79-84) */
            info[12 + 2 * c] = c < img.ncomp ? (img.width * img.comp[c].h + img.h_max - 1) / img.h_max : 0;
            info[13 + 2 * c] = c < img.ncomp ? (img.height * img.comp[c].v + img.v_max - 1) / img.v_max : 0;
        }
    }
    free(img.seg);
    return e;
}

int orc_segment(const uint8_t *file, size_t size, uint8_t *out, size_t cap, size_t *len) {
    orc_image img;
    int e = orc_parse(file, size, &img);
    if (!e) {
        *len = img.seg_bytes;
        if (img.seg_bytes > cap)
            e = E_CAPACITY;
        else
            memcpy(out, img.seg, img.seg_bytes);
    }
    free(img.seg);
    return e;
}

/* Sequential entropy decode with boundary trace (oracle.hpp:47-98). */
int orc_trace(const uint8_t *file, size_t size, const uint64_t *boundaries, size_t nb, uint64_t *states,
              uint8_t *valid, int16_t *coeffs, size_t coef_cap, uint64_t *end_state) {
    orc_image img;
    int e = orc_parse(file, size, &img);
    if (!e) {
        uint64_t total = (uint64_t)img.mcus_x * img.mcus_y * img.dpm * 64;
        if (total > coef_cap)
            e = E_CAPACITY;
        else
            e = decode_entropy(&img, boundaries, nb, states, valid, coeffs, end_state);
    }
    free(img.seg);
    return e;
}

/*
 * Full decode: entropy → dc_prefix_sum (transform.hpp:56-74) →
 * transform_blocks (146-161) → extract_planes (165-211) → optionally
 * upsample_and_convert (pipeline.hpp:167-201).  want_rgb=0 writes the planes
 * back to back.  out_coeffs (optional) receives the post-DC zig-zag buffer.
 */
int orc_decode(const uint8_t *file, size_t size, int want_rgb, uint8_t *out, size_t cap, uint32_t *info,
               int16_t *out_coeffs, size_t coef_cap) {
    init_basis();
    orc_image img;
    int e = orc_parse(file, size, &img);
    if (e) {
        free(img.seg);
        return e;
    }
    uint64_t dus = (uint64_t)img.mcus_x * img.mcus_y * img.dpm;
    int16_t *coef = (int16_t *)malloc(dus * 64 * sizeof(int16_t));
    uint8_t *blocks = (uint8_t *)malloc(dus * 64);
    uint8_t *planes[3] = {NULL, NULL, NULL};
    uint32_t pw[3] = {0, 0, 0}, ph[3] = {0, 0, 0};
    if (!coef || !blocks) {
        e = E_NOMEM;
        goto done;
    }
    {
        uint64_t st[4];
        uint8_t v;
        e = decode_entropy(&img, NULL, 0, st, &v, coef, NULL);
    }
    if (e) goto done;
    /* dc_prefix_sum: per component, int32 accumulator, int16 store */
    for (int comp = 0; comp < img.ncomp; ++comp) {
        int32_t acc = 0;
        int first = 1;
        for (uint64_t du = 0; du < dus; ++du) {
            if (img.du_seq[du % img.dpm] != comp) continue;
            size_t idx = (size_t)du * 64;
            if (first) {
                acc = coef[idx];
                first = 0;
            } else {
                acc = (int32_t)((uint32_t)acc + (uint32_t)(int32_t)coef[idx]);
                coef[idx] = (int16_t)acc;
            }
        }
    }
    if (out_coeffs) {
        if (dus * 64 > coef_cap) {
            e = E_CAPACITY;
            goto done;
        }
        memcpy(out_coeffs, coef, dus * 64 * sizeof(int16_t));
    }
    /* transform_blocks */
    for (uint64_t du = 0; du < dus; ++du) {
        unsigned comp = img.du_seq[du % img.dpm];
        const uint16_t *q = img.quant[img.comp[comp].tq];
        int32_t deq[64];
        for (int z = 0; z < 64; ++z) deq[kZigzagToRaster[z]] = (int32_t)coef[du * 64 + z] * q[z];
        idct_8x8(deq, blocks + du * 64);
    }
    /* extract_planes */
    for (int c = 0; c < img.ncomp; ++c) {
        pw[c] = (img.width * img.comp[c].h + img.h_max - 1) / img.h_max;
        ph[c] = (img.height * img.comp[c].v + img.v_max - 1) / img.v_max;
        planes[c] = (uint8_t *)calloc((size_t)pw[c] * ph[c], 1);
        if (!planes[c]) {
            e = E_NOMEM;
            goto done;
        }
    }
    {
        uint32_t slot_in_comp[10];
        uint32_t seen[4] = {0, 0, 0, 0};
        for (uint32_t s = 0; s < img.dpm; ++s) slot_in_comp[s] = seen[img.du_seq[s]]++;
        for (uint64_t mcu = 0; mcu < (uint64_t)img.mcus_x * img.mcus_y; ++mcu) {
            uint32_t mx = (uint32_t)(mcu % img.mcus_x), my = (uint32_t)(mcu / img.mcus_x);
            for (uint32_t s = 0; s < img.dpm; ++s) {
                unsigned ci = img.du_seq[s];
                uint32_t k = slot_in_comp[s];
                uint32_t bx = k % img.comp[ci].h, by = k / img.comp[ci].h;
                uint32_t x0 = (mx * img.comp[ci].h + bx) * 8, y0 = (my * img.comp[ci].v + by) * 8;
                const uint8_t *du = blocks + (mcu * img.dpm + s) * 64;
                for (uint32_t row = 0; row < 8; ++row) {
                    uint32_t y = y0 + row;
                    if (y >= ph[ci]) break;
                    uint32_t cols = pw[ci] > x0 ? pw[ci] - x0 : 0;
                    if (cols > 8) cols = 8;
                    for (uint32_t col = 0; col < cols; ++col)
                        planes[ci][(size_t)y * pw[ci] + x0 + col] = du[row * 8 + col];
                }
            }
        }
    }
    info[0] = img.width;
    info[1] = img.height;
    info[3] = (uint32_t)img.ncomp;
    for (int c = 0; c < 3; ++c) {
        info[4 + 2 * c] = pw[c];
        info[5 + 2 * c] = ph[c];
    }
    if (!want_rgb) {
        info[2] = (uint32_t)img.ncomp;
        size_t off = 0;
        for (int c = 0; c < img.ncomp; ++c) {
            size_t n = (size_t)pw[c] * ph[c];
            if (off + n > cap) {
                e = E_CAPACITY;
                goto done;
            }
            memcpy(out + off, planes[c], n);
            off += n;
        }
    } else if (img.ncomp == 1) {
        /* upsample_and_convert grayscale passthrough (pipeline.hpp:171-176) */
        info[2] = 1;
        size_t n = (size_t)img.width * img.height;
        if (n > cap) {
            e = E_CAPACITY;
            goto done;
        }
        memcpy(out, planes[0], n);
    } else {
        info[2] = 3;
        size_t W = img.width, H = img.height;
        if (W * H * 3 > cap) {
            e = E_CAPACITY;
            goto done;
        }
        for (uint32_t y = 0; y < H; ++y)
            for (uint32_t x = 0; x < W; ++x) {
                int Y = planes[0][(size_t)y * pw[0] + x];
                uint32_t sx1 = (uint32_t)((uint64_t)x * pw[1] / W), sy1 = (uint32_t)((uint64_t)y * ph[1] / H);
                if (sx1 > pw[1] - 1) sx1 = pw[1] - 1;
                if (sy1 > ph[1] - 1) sy1 = ph[1] - 1;
                uint32_t sx2 = (uint32_t)((uint64_t)x * pw[2] / W), sy2 = (uint32_t)((uint64_t)y * ph[2] / H);
                if (sx2 > pw[2] - 1) sx2 = pw[2] - 1;
                if (sy2 > ph[2] - 1) sy2 = ph[2] - 1;
                int Cb = planes[1][(size_t)sy1 * pw[1] + sx1] - 128;
                int Cr = planes[2][(size_t)sy2 * pw[2] + sx2] - 128;
                size_t o = ((size_t)y * W + x) * 3;
                out[o + 0] = clamp_u8((int)lround(Y + 1.402 * Cr));
                out[o + 1] = clamp_u8((int)lround(Y - 0.344136 * Cb - 0.714136 * Cr));
                out[o + 2] = clamp_u8((int)lround(Y + 1.772 * Cb));
            }
    }
done:
    free(coef);
    free(blocks);
    for (int c = 0; c < 3; ++c) free(planes[c]);
    free(img.seg);
    return e;
}
