// Synthetic baseline-JPEG corpus generator for the benchmark (libpjg_synth.so).
// Not part of the decode path.  Two generators:
//
//  * pjg_synth_ref_batch — the corpus SURVEY.md §8(d) prescribes: files
//    byte-identical to the reference's test-vector encoder
//    oracle_encode(make_test_image(w, h, seed, channels), q, sampling)
//    (reference oracle.hpp:272-478, tests/helpers.hpp:107-135), restated here
//    with the same double arithmetic in the same order (mt19937 content, JFIF
//    colour conversion, box-averaged chroma, separable FP64 forward DCT with
//    the host-libm basis, lround quantisation, Annex K tables used as the
//    reference uses them) so that the benchmark needs nothing under oracle/ at
//    run time.  tests/test_synth.py checks byte identity against oracle/_ref.
//    Optional restart markers (DRI + RSTn) give DRI twins whose coefficients
//    equal the reference file's.
//  * pjg_synth_batch — an independent fast float encoder over similar content
//    (kept for the restart-interval twin tests).
//
// Every file is fully determined by (w, h, seed, quality, sampling,
// restart_interval).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <initializer_list>
#include <random>
#include <thread>
#include <vector>

namespace {

const uint8_t kZz2R[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
                           12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
                           35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
                           58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

// T.81 Table K.1 / K.2 (raster order)
const uint8_t kLumaQ[64] = {16, 11, 10, 16, 24,  40,  51,  61,  12, 12, 14, 19, 26,  58,  60,  55,
                            14, 13, 16, 24, 40,  57,  69,  56,  14, 17, 22, 29, 51,  87,  80,  62,
                            18, 22, 37, 56, 68,  109, 103, 77,  24, 35, 55, 64, 81,  104, 113, 92,
                            49, 64, 78, 87, 103, 121, 120, 101, 72, 92, 95, 98, 112, 100, 103, 99};
const uint8_t kChromaQ[64] = {17, 18, 24, 47, 99, 99, 99, 99, 18, 21, 26, 66, 99, 99, 99, 99,
                              24, 26, 56, 99, 99, 99, 99, 99, 47, 66, 99, 99, 99, 99, 99, 99,
                              99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99,
                              99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99};

// T.81 Tables K.3-K.6: BITS then HUFFVAL
const uint8_t kDcLBits[16] = {0, 1, 5, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0};
const uint8_t kDcCBits[16] = {0, 3, 1, 1, 1, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0};
const uint8_t kDcVals[12] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11};
const uint8_t kAcLBits[16] = {0, 2, 1, 3, 3, 2, 4, 3, 5, 5, 4, 4, 0, 0, 1, 0x7d};
const uint8_t kAcLVals[162] = {
    0x01, 0x02, 0x03, 0x00, 0x04, 0x11, 0x05, 0x12, 0x21, 0x31, 0x41, 0x06, 0x13, 0x51, 0x61, 0x07, 0x22, 0x71,
    0x14, 0x32, 0x81, 0x91, 0xa1, 0x08, 0x23, 0x42, 0xb1, 0xc1, 0x15, 0x52, 0xd1, 0xf0, 0x24, 0x33, 0x62, 0x72,
    0x82, 0x09, 0x0a, 0x16, 0x17, 0x18, 0x19, 0x1a, 0x25, 0x26, 0x27, 0x28, 0x29, 0x2a, 0x34, 0x35, 0x36, 0x37,
    0x38, 0x39, 0x3a, 0x43, 0x44, 0x45, 0x46, 0x47, 0x48, 0x49, 0x4a, 0x53, 0x54, 0x55, 0x56, 0x57, 0x58, 0x59,
    0x5a, 0x63, 0x64, 0x65, 0x66, 0x67, 0x68, 0x69, 0x6a, 0x73, 0x74, 0x75, 0x76, 0x77, 0x78, 0x79, 0x7a, 0x83,
    0x84, 0x85, 0x86, 0x87, 0x88, 0x89, 0x8a, 0x92, 0x93, 0x94, 0x95, 0x96, 0x97, 0x98, 0x99, 0x9a, 0xa2, 0xa3,
    0xa4, 0xa5, 0xa6, 0xa7, 0xa8, 0xa9, 0xaa, 0xb2, 0xb3, 0xb4, 0xb5, 0xb6, 0xb7, 0xb8, 0xb9, 0xba, 0xc2, 0xc3,
    0xc4, 0xc5, 0xc6, 0xc7, 0xc8, 0xc9, 0xca, 0xd2, 0xd3, 0xd4, 0xd5, 0xd6, 0xd7, 0xd8, 0xd9, 0xda, 0xe1, 0xe2,
    0xe3, 0xe4, 0xe5, 0xe6, 0xe7, 0xe8, 0xe9, 0xea, 0xf1, 0xf2, 0xf3, 0xf4, 0xf5, 0xf6, 0xf7, 0xf8, 0xf9, 0xfa};
const uint8_t kAcCBits[16] = {0, 2, 1, 2, 4, 4, 3, 4, 7, 5, 4, 4, 0, 1, 2, 0x77};
const uint8_t kAcCVals[162] = {
    0x00, 0x01, 0x02, 0x03, 0x11, 0x04, 0x05, 0x21, 0x31, 0x06, 0x12, 0x41, 0x51, 0x07, 0x61, 0x71, 0x13, 0x22,
    0x32, 0x81, 0x08, 0x14, 0x42, 0x91, 0xa1, 0xb1, 0xc1, 0x09, 0x23, 0x33, 0x52, 0xf0, 0x15, 0x62, 0x72, 0xd1,
    0x0a, 0x16, 0x24, 0x34, 0xe1, 0x25, 0xf1, 0x17, 0x18, 0x19, 0x1a, 0x26, 0x27, 0x28, 0x29, 0x2a, 0x35, 0x36,
    0x37, 0x38, 0x39, 0x3a, 0x43, 0x44, 0x45, 0x46, 0x47, 0x48, 0x49, 0x4a, 0x53, 0x54, 0x55, 0x56, 0x57, 0x58,
    0x59, 0x5a, 0x63, 0x64, 0x65, 0x66, 0x67, 0x68, 0x69, 0x6a, 0x73, 0x74, 0x75, 0x76, 0x77, 0x78, 0x79, 0x7a,
    0x82, 0x83, 0x84, 0x85, 0x86, 0x87, 0x88, 0x89, 0x8a, 0x92, 0x93, 0x94, 0x95, 0x96, 0x97, 0x98, 0x99, 0x9a,
    0xa2, 0xa3, 0xa4, 0xa5, 0xa6, 0xa7, 0xa8, 0xa9, 0xaa, 0xb2, 0xb3, 0xb4, 0xb5, 0xb6, 0xb7, 0xb8, 0xb9, 0xba,
    0xc2, 0xc3, 0xc4, 0xc5, 0xc6, 0xc7, 0xc8, 0xc9, 0xca, 0xd2, 0xd3, 0xd4, 0xd5, 0xd6, 0xd7, 0xd8, 0xd9, 0xda,
    0xe2, 0xe3, 0xe4, 0xe5, 0xe6, 0xe7, 0xe8, 0xe9, 0xea, 0xf2, 0xf3, 0xf4, 0xf5, 0xf6, 0xf7, 0xf8, 0xf9, 0xfa};

struct HuffEnc {
    uint16_t code[256];
    uint8_t len[256];
    void build(const uint8_t* bits, const uint8_t* vals) {
        std::memset(len, 0, sizeof len);
        uint32_t c = 0;
        int k = 0;
        for (int l = 1; l <= 16; ++l) {
            for (int i = 0; i < bits[l - 1]; ++i, ++k) {
                code[vals[k]] = uint16_t(c++);
                len[vals[k]] = uint8_t(l);
            }
            c <<= 1;
        }
    }
};

struct BitSink {
    std::vector<uint8_t>& out;
    uint64_t acc = 0;
    int n = 0;
    explicit BitSink(std::vector<uint8_t>& o) : out(o) {}
    inline void put(uint32_t v, int l) {
        if (!l) return;
        acc = (acc << l) | (v & ((1u << l) - 1));
        n += l;
        while (n >= 8) {
            uint8_t b = uint8_t(acc >> (n - 8));
            out.push_back(b);
            if (b == 0xFF) out.push_back(0x00);
            n -= 8;
        }
    }
    void flush() {  // pad with 1-bits
        if (n) put((1u << (8 - n)) - 1, 8 - n);
        acc = 0;
        n = 0;
    }
};

inline uint64_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

inline int mag_cat(int v) {
    unsigned m = unsigned(v < 0 ? -v : v);
    return m ? 32 - __builtin_clz(m) : 0;
}

struct Encoder {
    uint32_t W, H;
    uint32_t seed;
    int quality, sampling, restart;  // sampling: 0 444, 1 422, 2 420, 3 gray
    uint16_t ql[64], qc[64];         // raster
    float cosm[8][8];
    HuffEnc dcl, dcc, acl, acc;

    void setup() {
        int q = std::max(1, std::min(100, quality));
        int scale = q < 50 ? 5000 / q : 200 - 2 * q;
        for (int i = 0; i < 64; ++i) {
            ql[i] = uint16_t(std::max(1, std::min(255, (kLumaQ[i] * scale + 50) / 100)));
            qc[i] = uint16_t(std::max(1, std::min(255, (kChromaQ[i] * scale + 50) / 100)));
        }
        for (int u = 0; u < 8; ++u)
            for (int x = 0; x < 8; ++x)
                cosm[u][x] = float((u == 0 ? std::sqrt(0.125) : 0.5) * std::cos((2 * x + 1) * u * M_PI / 16));
        dcl.build(kDcLBits, kDcVals);
        dcc.build(kDcCBits, kDcVals);
        acl.build(kAcLBits, kAcLVals);
        acc.build(kAcCBits, kAcCVals);
    }

    // full-resolution float planes (Y, Cb, Cr) of the synthetic content
    void content(std::vector<float>* pl, int ncomp) const {
        uint64_t s = mix64(seed * 0x9E3779B97F4A7C15ull + 12345);
        auto rnd = [&](double lo, double hi) {
            s = mix64(s + 0x9E3779B97F4A7C15ull);
            return lo + (hi - lo) * double(s >> 11) / double(1ull << 53);
        };
        const double px = rnd(0, 6.2831853), py = rnd(0, 6.2831853), fx = rnd(0.5, 4), fy = rnd(0.5, 4);
        const double gx = rnd(0, 6.2831853), gy = rnd(0, 6.2831853);
        std::vector<float> A(W), B(H), Gx(W), Gy(H), Sx[3], Cx[3], Sy[3], Cy[3];
        for (uint32_t x = 0; x < W; ++x) {
            double u = double(x) / W;
            A[x] = float(std::sin(fx * 6.2832 * u + px));
            Gx[x] = float(40 * u * std::cos(gx));
        }
        for (uint32_t y = 0; y < H; ++y) {
            double v = double(y) / H;
            B[y] = float(std::cos(fy * 6.2832 * v + py));
            Gy[y] = float(40 * v * std::sin(gy));
        }
        for (int c = 0; c < 3; ++c) {
            Sx[c].resize(W);
            Cx[c].resize(W);
            Sy[c].resize(H);
            Cy[c].resize(H);
            for (uint32_t x = 0; x < W; ++x) {
                double a = (c + 1) * 6.2832 * double(x) / W;
                Sx[c][x] = float(std::sin(a));
                Cx[c][x] = float(std::cos(a));
            }
            for (uint32_t y = 0; y < H; ++y) {
                double a = (c + 1) * 6.2832 * double(y) / H;
                Sy[c][y] = float(std::sin(a));
                Cy[c][y] = float(std::cos(a));
            }
        }
        for (int c = 0; c < ncomp; ++c) pl[c].assign(size_t(W) * H, 0.f);
        for (uint32_t y = 0; y < H; ++y) {
            uint64_t hs = mix64(uint64_t(seed) << 32 ^ y);
            for (uint32_t x = 0; x < W; ++x) {
                float base = 128.f + 70.f * A[x] * B[y] + Gx[x] + Gy[y];
                float rgb[3];
                uint64_t hv = mix64(hs + x);
                for (int c = 0; c < 3; ++c) {
                    float chan = base + 25.f * (Sx[c][x] * Cy[c][y] + Cx[c][x] * Sy[c][y]) +
                                 float(int((hv >> (16 * c)) % 13) - 6);
                    rgb[c] = std::min(255.f, std::max(0.f, std::round(chan)));
                }
                size_t i = size_t(y) * W + x;
                if (ncomp == 1) {
                    pl[0][i] = rgb[0];
                } else {
                    pl[0][i] = 0.299f * rgb[0] + 0.587f * rgb[1] + 0.114f * rgb[2];
                    pl[1][i] = 128.f - 0.168736f * rgb[0] - 0.331264f * rgb[1] + 0.5f * rgb[2];
                    pl[2][i] = 128.f + 0.5f * rgb[0] - 0.418688f * rgb[1] - 0.081312f * rgb[2];
                }
            }
        }
    }

    void fdct_quant(const float* blk, const uint16_t* q, int16_t* zz) const {
        float t[8][8], f[8][8];
        for (int u = 0; u < 8; ++u)
            for (int x = 0; x < 8; ++x) {
                float s = 0;
                for (int y = 0; y < 8; ++y) s += cosm[u][y] * (blk[y * 8 + x] - 128.f);
                t[u][x] = s;
            }
        for (int u = 0; u < 8; ++u)
            for (int v = 0; v < 8; ++v) {
                float s = 0;
                for (int x = 0; x < 8; ++x) s += cosm[v][x] * t[u][x];
                f[u][v] = s;
            }
        for (int z = 0; z < 64; ++z) {
            int r = kZz2R[z];
            zz[z] = int16_t(std::lround(f[r >> 3][r & 7] / q[r]));
        }
    }

    std::vector<uint8_t> encode() {
        setup();
        const bool gray = sampling == 3;
        const int nc = gray ? 1 : 3;
        const int yh = (sampling == 1 || sampling == 2) ? 2 : 1, yv = sampling == 2 ? 2 : 1;
        std::vector<float> pl[3];
        content(pl, nc);
        // chroma box subsampling
        uint32_t cw = W, ch = H;
        if (!gray && (yh > 1 || yv > 1)) {
            cw = (W + yh - 1) / yh;
            ch = (H + yv - 1) / yv;
            for (int c = 1; c < 3; ++c) {
                std::vector<float> o(size_t(cw) * ch);
                for (uint32_t y = 0; y < ch; ++y)
                    for (uint32_t x = 0; x < cw; ++x) {
                        float a = 0;
                        for (int dy = 0; dy < yv; ++dy)
                            for (int dx = 0; dx < yh; ++dx)
                                a += pl[c][size_t(std::min(H - 1, y * yv + dy)) * W + std::min(W - 1, x * yh + dx)];
                        o[size_t(y) * cw + x] = a / float(yh * yv);
                    }
                pl[c].swap(o);
            }
        }
        const uint32_t mw = 8 * yh, mh = 8 * yv, mx = (W + mw - 1) / mw, my = (H + mh - 1) / mh;
        std::vector<uint8_t> scan;
        scan.reserve(size_t(W) * H / 4 + 1024);
        BitSink bs(scan);
        int pred[3] = {0, 0, 0};
        float blk[64];
        int16_t zz[64];
        uint32_t mcu_i = 0, rst_n = 0;
        const uint32_t mcus = mx * my;
        for (uint32_t my_ = 0; my_ < my; ++my_)
            for (uint32_t mx_ = 0; mx_ < mx; ++mx_, ++mcu_i) {
                if (restart && mcu_i && mcu_i % restart == 0) {
                    bs.flush();
                    scan.push_back(0xFF);
                    scan.push_back(uint8_t(0xD0 + (rst_n++ & 7)));
                    pred[0] = pred[1] = pred[2] = 0;
                }
                for (int c = 0; c < nc; ++c) {
                    const int h = c == 0 ? yh : 1, v = c == 0 ? yv : 1;
                    const uint32_t pw = c == 0 ? W : cw, ph = c == 0 ? H : ch;
                    const uint16_t* q = c == 0 ? ql : qc;
                    const HuffEnc& dc = c == 0 ? dcl : dcc;
                    const HuffEnc& ac = c == 0 ? acl : acc;
                    for (int by = 0; by < v; ++by)
                        for (int bx = 0; bx < h; ++bx) {
                            uint32_t x0 = (mx_ * h + bx) * 8, y0 = (my_ * v + by) * 8;
                            for (int r = 0; r < 8; ++r)
                                for (int cc = 0; cc < 8; ++cc)
                                    blk[r * 8 + cc] = pl[c][size_t(std::min(ph - 1, y0 + r)) * pw + std::min(pw - 1, x0 + cc)];
                            fdct_quant(blk, q, zz);
                            int diff = zz[0] - pred[c];
                            pred[c] = zz[0];
                            int l = mag_cat(diff);
                            bs.put(dc.code[l], dc.len[l]);
                            bs.put(uint32_t(diff < 0 ? diff + (1 << l) - 1 : diff), l);
                            int last = 0;
                            for (int z = 63; z >= 1; --z)
                                if (zz[z]) {
                                    last = z;
                                    break;
                                }
                            int run = 0;
                            for (int z = 1; z <= last; ++z) {
                                if (!zz[z]) {
                                    ++run;
                                    continue;
                                }
                                while (run >= 16) {
                                    bs.put(ac.code[0xF0], ac.len[0xF0]);
                                    run -= 16;
                                }
                                int al = mag_cat(zz[z]);
                                int sym = (run << 4) | al;
                                bs.put(ac.code[sym], ac.len[sym]);
                                bs.put(uint32_t(zz[z] < 0 ? zz[z] + (1 << al) - 1 : zz[z]), al);
                                run = 0;
                            }
                            if (last < 63) bs.put(ac.code[0], ac.len[0]);
                        }
                }
            }
        (void)mcus;
        bs.flush();
        // container
        std::vector<uint8_t> o;
        o.reserve(scan.size() + 700);
        auto p8 = [&](int v) { o.push_back(uint8_t(v)); };
        auto p16 = [&](int v) {
            p8(v >> 8);
            p8(v & 255);
        };
        p8(0xFF), p8(0xD8);
        p8(0xFF), p8(0xE0), p16(16);
        for (int v : std::initializer_list<int>{'J', 'F', 'I', 'F', 0, 1, 1, 0, 0, 1, 0, 1, 0, 0}) p8(v);
        auto dqt = [&](int id, const uint16_t* q) {
            p8(0xFF), p8(0xDB), p16(67), p8(id);
            for (int z = 0; z < 64; ++z) p8(q[kZz2R[z]]);
        };
        dqt(0, ql);
        if (!gray) dqt(1, qc);
        p8(0xFF), p8(0xC0), p16(8 + 3 * nc), p8(8), p16(H), p16(W), p8(nc);
        for (int c = 0; c < nc; ++c) {
            p8(c + 1);
            p8(c == 0 ? (yh << 4 | yv) : 0x11);
            p8(c == 0 ? 0 : 1);
        }
        auto dht = [&](int cls, int id, const uint8_t* bits, const uint8_t* vals) {
            int n = 0;
            for (int i = 0; i < 16; ++i) n += bits[i];
            p8(0xFF), p8(0xC4), p16(3 + 16 + n), p8(cls << 4 | id);
            for (int i = 0; i < 16; ++i) p8(bits[i]);
            for (int i = 0; i < n; ++i) p8(vals[i]);
        };
        dht(0, 0, kDcLBits, kDcVals);
        dht(1, 0, kAcLBits, kAcLVals);
        if (!gray) {
            dht(0, 1, kDcCBits, kDcVals);
            dht(1, 1, kAcCBits, kAcCVals);
        }
        if (restart) p8(0xFF), p8(0xDD), p16(4), p16(restart);
        p8(0xFF), p8(0xDA), p16(6 + 2 * nc), p8(nc);
        for (int c = 0; c < nc; ++c) p8(c + 1), p8(c == 0 ? 0x00 : 0x11);
        p8(0), p8(63), p8(0);
        o.insert(o.end(), scan.begin(), scan.end());
        p8(0xFF), p8(0xD9);
        return o;
    }
};


// ----------------------------------------------- reference-equivalent corpus --
// make_test_image (tests/helpers.hpp:107-135): the pixels come from one
// mt19937 stream (6 parameter draws, then one noise draw per pixel and
// channel, row-major), so they are produced sequentially; the trigonometric
// part of every pixel does not depend on the stream and is computed first
// (in parallel) with the reference's exact expression.
void test_pixels(uint32_t w, uint32_t h, uint32_t seed, unsigned ch, unsigned threads, std::vector<uint8_t>& px) {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> phase(0.0, 6.28318530717958647692);
    std::uniform_real_distribution<double> freq(0.5, 4.0);
    std::uniform_int_distribution<int> noise(-6, 6);
    const double ph_x = phase(rng), ph_y = phase(rng), f_x = freq(rng), f_y = freq(rng);
    const double g_x = phase(rng), g_y = phase(rng);
    // smooth part: (base + grad) + 25 sin((c + 1)(u + v) 6.2832), per pixel and channel
    std::vector<double> smooth(size_t(w) * h * ch);
    auto rows = [&](uint32_t y0, uint32_t y1) {
        for (uint32_t y = y0; y < y1; ++y)
            for (uint32_t x = 0; x < w; ++x) {
                const double u = double(x) / w, v = double(y) / h;
                const double base = 128 + 70 * std::sin(f_x * 6.2832 * u + ph_x) * std::cos(f_y * 6.2832 * v + ph_y);
                const double grad = 40 * (u * std::cos(g_x) + v * std::sin(g_y));
                for (unsigned c = 0; c < ch; ++c)
                    smooth[(size_t(y) * w + x) * ch + c] = base + grad + 25.0 * std::sin((c + 1) * (u + v) * 6.2832);
            }
    };
    threads = std::max(1u, std::min(threads, h));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < threads; ++t)
        th.emplace_back([&, t] { rows(uint32_t(uint64_t(h) * t / threads), uint32_t(uint64_t(h) * (t + 1) / threads)); });
    for (auto& x : th) x.join();
    px.resize(smooth.size());
    for (size_t i = 0; i < smooth.size(); ++i) {
        const long r = std::lround(smooth[i] + noise(rng));
        px[i] = uint8_t(r < 0 ? 0 : (r > 255 ? 255 : r));
    }
}

// oracle_encode (oracle.hpp:272-478) of those pixels, byte for byte.
struct RefEncoder {
    uint32_t W, H;
    unsigned ch;          // pixel channels (1 or 3)
    int quality, sampling, restart;
    unsigned threads;
    bool gray = false;
    int yh = 1, yv = 1, nc = 3;
    uint32_t cw = 0, chh = 0;   // chroma plane size
    uint16_t q_zz[2][64];      // scaled quantisers, zig-zag order (the tables are read as zig-zag)
    double basis[8][8];
    HuffEnc dc_t[2], ac_t[2];
    const uint8_t* px = nullptr;

    // JFIF colour conversion of pixel (x, y), component c (double, the reference's expressions)
    double comp_at(int c, uint32_t x, uint32_t y) const {
        const size_t i = size_t(y) * W + x;
        double R, G, B;
        if (ch == 1) {
            R = G = B = px[i];
        } else {
            R = px[i * 3 + 0];
            G = px[i * 3 + 1];
            B = px[i * 3 + 2];
        }
        if (c == 0) return 0.299 * R + 0.587 * G + 0.114 * B;
        if (c == 1) return 128.0 - 0.168736 * R - 0.331264 * G + 0.5 * B;
        return 128.0 + 0.5 * R - 0.418688 * G - 0.081312 * B;
    }
    // sample (x, y) of component plane c, coordinates clamped to the plane (Plane::at)
    double sample(int c, uint32_t x, uint32_t y) const {
        if (c == 0 || (yh == 1 && yv == 1)) return comp_at(c, std::min(x, W - 1), std::min(y, H - 1));
        x = std::min(x, cw - 1);
        y = std::min(y, chh - 1);
        double acc = 0;  // box average over the full-resolution plane (clamped)
        for (int dy = 0; dy < yv; ++dy)
            for (int dx = 0; dx < yh; ++dx)
                acc += comp_at(c, std::min(x * yh + dx, W - 1), std::min(y * yv + dy, H - 1));
        return acc / (yh * yv);
    }

    void setup() {
        gray = sampling == 3 || ch == 1;
        nc = gray ? 1 : 3;
        if (!gray && sampling == 1) yh = 2;
        if (!gray && sampling == 2) yh = yv = 2;
        cw = (W + yh - 1) / yh;
        chh = (H + yv - 1) / yv;
        const int q = std::max(1, std::min(100, quality));
        const int scale = q < 50 ? 5000 / q : 200 - 2 * q;
        for (int i = 0; i < 64; ++i) {
            q_zz[0][i] = uint16_t(std::max(1, std::min(255, (kLumaQ[i] * scale + 50) / 100)));
            q_zz[1][i] = uint16_t(std::max(1, std::min(255, (kChromaQ[i] * scale + 50) / 100)));
        }
        for (int u = 0; u < 8; ++u) {
            const double cu = u == 0 ? 1.0 / std::sqrt(2.0) : 1.0;
            for (int x = 0; x < 8; ++x) basis[u][x] = 0.5 * cu * std::cos((2 * x + 1) * u * M_PI / 16.0);
        }
        dc_t[0].build(kDcLBits, kDcVals);
        dc_t[1].build(kDcCBits, kDcVals);
        ac_t[0].build(kAcLBits, kAcLVals);
        ac_t[1].build(kAcCBits, kAcCVals);
    }

    // forward DCT + quantisation of the block at (x0, y0) of component c
    void block(int c, uint32_t x0, uint32_t y0, int16_t* zz) const {
        double s[64];
        for (int r = 0; r < 8; ++r)
            for (int k = 0; k < 8; ++k) s[r * 8 + k] = sample(c, x0 + k, y0 + r);
        double t[8][8];
        for (int u = 0; u < 8; ++u)
            for (int x = 0; x < 8; ++x) {
                double a = 0;
                for (int y = 0; y < 8; ++y) a += basis[u][y] * (s[y * 8 + x] - 128.0);
                t[u][x] = a;
            }
        double f[64];
        for (int u = 0; u < 8; ++u)
            for (int v = 0; v < 8; ++v) {
                double a = 0;
                for (int x = 0; x < 8; ++x) a += basis[v][x] * t[u][x];
                f[u * 8 + v] = a;
            }
        const uint16_t* q = q_zz[c == 0 ? 0 : 1];
        for (int z = 0; z < 64; ++z) zz[z] = int16_t(std::lround(f[kZz2R[z]] / q[z]));
    }

    std::vector<uint8_t> encode() {
        setup();
        const uint32_t mw = 8 * yh, mh = 8 * yv, mx = (W + mw - 1) / mw, my = (H + mh - 1) / mh;
        const int dpm = gray ? 1 : yh * yv + 2;
        // coefficients per band of MCU rows in parallel, entropy coding in order
        const uint32_t band = std::max(1u, std::min(my, 64u));
        std::vector<int16_t> zz(size_t(band) * mx * dpm * 64);
        std::vector<uint8_t> scan;
        scan.reserve(size_t(W) * H / 4 + 1024);
        BitSink bs(scan);
        int pred[3] = {0, 0, 0};
        uint32_t mcu_i = 0, rst_n = 0;
        for (uint32_t b0 = 0; b0 < my; b0 += band) {
            const uint32_t b1 = std::min(my, b0 + band);
            const uint64_t units = uint64_t(b1 - b0) * mx;
            auto work = [&](uint64_t m0, uint64_t m1) {
                for (uint64_t m = m0; m < m1; ++m) {
                    const uint32_t ry = b0 + uint32_t(m / mx), rx = uint32_t(m % mx);
                    int16_t* o = zz.data() + m * dpm * 64;
                    for (int c = 0; c < nc; ++c) {
                        const int h = c == 0 ? yh : 1, v = c == 0 ? yv : 1;
                        for (int by = 0; by < v; ++by)
                            for (int bx = 0; bx < h; ++bx, o += 64)
                                block(c, (rx * h + bx) * 8, (ry * v + by) * 8, o);
                    }
                }
            };
            const unsigned nt = unsigned(std::max<uint64_t>(1, std::min<uint64_t>(threads, units)));
            std::vector<std::thread> th;
            for (unsigned t = 1; t < nt; ++t)
                th.emplace_back([&, t] { work(units * t / nt, units * (t + 1) / nt); });
            work(0, units / nt);
            for (auto& x : th) x.join();
            for (uint64_t m = 0; m < units; ++m, ++mcu_i) {
                if (restart && mcu_i && mcu_i % restart == 0) {
                    bs.flush();
                    scan.push_back(0xFF);
                    scan.push_back(uint8_t(0xD0 + (rst_n++ & 7)));
                    pred[0] = pred[1] = pred[2] = 0;
                }
                const int16_t* blk = zz.data() + m * dpm * 64;
                for (int c = 0; c < nc; ++c) {
                    const int cls = c == 0 ? 0 : 1, nb = c == 0 ? yh * yv : 1;
                    for (int k = 0; k < nb; ++k, blk += 64) {
                        const int diff = blk[0] - pred[c];
                        pred[c] = blk[0];
                        const int l = mag_cat(diff);
                        bs.put(dc_t[cls].code[l], dc_t[cls].len[l]);
                        bs.put(uint32_t(diff < 0 ? diff + (1 << l) - 1 : diff), l);
                        int last = 0;
                        for (int z = 63; z >= 1; --z)
                            if (blk[z]) {
                                last = z;
                                break;
                            }
                        int run = 0;
                        for (int z = 1; z <= last; ++z) {
                            if (!blk[z]) {
                                ++run;
                                continue;
                            }
                            for (; run >= 16; run -= 16) bs.put(ac_t[cls].code[0xF0], ac_t[cls].len[0xF0]);
                            const int al = mag_cat(blk[z]);
                            const int sym = (run << 4) | al;
                            bs.put(ac_t[cls].code[sym], ac_t[cls].len[sym]);
                            bs.put(uint32_t(blk[z] < 0 ? blk[z] + (1 << al) - 1 : blk[z]), al);
                            run = 0;
                        }
                        if (last < 63) bs.put(ac_t[cls].code[0], ac_t[cls].len[0]);
                    }
                }
            }
        }
        bs.flush();
        std::vector<uint8_t> o;
        o.reserve(scan.size() + 700);
        auto p8 = [&](int v) { o.push_back(uint8_t(v)); };
        auto p16 = [&](int v) {
            p8(v >> 8);
            p8(v & 255);
        };
        p8(0xFF), p8(0xD8);
        p8(0xFF), p8(0xE0), p16(16);
        for (int v : std::initializer_list<int>{'J', 'F', 'I', 'F', 0, 1, 1, 0, 0, 1, 0, 1, 0, 0}) p8(v);
        for (int t = 0; t < (gray ? 1 : 2); ++t) {
            p8(0xFF), p8(0xDB), p16(67), p8(t);
            for (int z = 0; z < 64; ++z) p8(q_zz[t][z]);
        }
        p8(0xFF), p8(0xC0), p16(8 + 3 * nc), p8(8), p16(H), p16(W), p8(nc);
        for (int c = 0; c < nc; ++c) p8(c + 1), p8(c == 0 ? (yh << 4 | yv) : 0x11), p8(c == 0 ? 0 : 1);
        auto dht = [&](int cls, int id, const uint8_t* bits, const uint8_t* vals) {
            int n = 0;
            for (int i = 0; i < 16; ++i) n += bits[i];
            p8(0xFF), p8(0xC4), p16(3 + 16 + n), p8(cls << 4 | id);
            for (int i = 0; i < 16; ++i) p8(bits[i]);
            for (int i = 0; i < n; ++i) p8(vals[i]);
        };
        dht(0, 0, kDcLBits, kDcVals);
        dht(1, 0, kAcLBits, kAcLVals);
        if (!gray) {
            dht(0, 1, kDcCBits, kDcVals);
            dht(1, 1, kAcCBits, kAcCVals);
        }
        if (restart) p8(0xFF), p8(0xDD), p16(4), p16(restart);
        p8(0xFF), p8(0xDA), p16(6 + 2 * nc), p8(nc);
        for (int c = 0; c < nc; ++c) p8(c + 1), p8(c == 0 ? 0x00 : 0x11);
        p8(0), p8(63), p8(0);
        o.insert(o.end(), scan.begin(), scan.end());
        p8(0xFF), p8(0xD9);
        return o;
    }
};

template <class Enc>
uint64_t place(std::vector<std::vector<uint8_t>>& files, uint8_t* blob, uint64_t cap, uint64_t* offsets,
               uint64_t* sizes, uint64_t* need) {
    uint64_t tot = 0;
    for (auto& f : files) tot += f.size();
    *need = tot;
    if (tot > cap) return 0;
    uint64_t o = 0;
    for (size_t i = 0; i < files.size(); ++i) {
        offsets[i] = o;
        sizes[i] = files[i].size();
        std::memcpy(blob + o, files[i].data(), files[i].size());
        o += files[i].size();
    }
    return tot;
}

}  // namespace

extern "C" {

// n files oracle_encode(make_test_image(w, h, seed0 + i, channels), quality,
// sampling) (+ DRI every restart_interval MCUs when > 0) into one blob; see
// pjg_synth_batch for the calling convention.  channels 0: 1 for gray, else 3.
uint64_t pjg_synth_ref_batch(uint32_t n, uint32_t w, uint32_t h, uint32_t seed0, int quality, int sampling,
                             int restart_interval, unsigned channels, unsigned threads, uint8_t* blob, uint64_t cap,
                             uint64_t* offsets, uint64_t* sizes, uint64_t* need) {
    std::vector<std::vector<uint8_t>> files(n);
    const unsigned ch = channels ? channels : (sampling == 3 ? 1u : 3u);
    threads = std::max(1u, threads);
    // few files: threads inside each file; many: one file per thread
    const unsigned outer = std::min(threads, n ? n : 1u), inner = std::max(1u, threads / outer);
    std::vector<std::thread> th;
    for (unsigned t = 0; t < outer; ++t)
        th.emplace_back([&, t] {
            std::vector<uint8_t> px;
            for (uint32_t i = t; i < n; i += outer) {
                test_pixels(w, h, seed0 + i, ch, inner, px);
                RefEncoder e{w, h, ch, quality, sampling, restart_interval, inner};
                e.px = px.data();
                files[i] = e.encode();
            }
        });
    for (auto& x : th) x.join();
    return place<RefEncoder>(files, blob, cap, offsets, sizes, need);
}


// Encodes n images (seeds seed0..seed0+n-1) with `threads` host threads into
// one contiguous blob.  offsets/sizes receive per-file placement.  Returns the
// total blob size, or 0 when `cap` is too small (then call again with
// cap >= the returned *need).
uint64_t pjg_synth_batch(uint32_t n, uint32_t w, uint32_t h, uint32_t seed0, int quality, int sampling,
                         int restart_interval, unsigned threads, uint8_t* blob, uint64_t cap, uint64_t* offsets,
                         uint64_t* sizes, uint64_t* need) {
    std::vector<std::vector<uint8_t>> files(n);
    threads = std::max(1u, std::min(threads, n ? n : 1u));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < threads; ++t)
        th.emplace_back([&, t] {
            for (uint32_t i = t; i < n; i += threads) {
                Encoder e{w, h, seed0 + i, quality, sampling, restart_interval, {}, {}, {}, {}, {}, {}, {}};
                files[i] = e.encode();
            }
        });
    for (auto& x : th) x.join();
    uint64_t tot = 0;
    for (auto& f : files) tot += f.size();
    *need = tot;
    if (tot > cap) return 0;
    uint64_t o = 0;
    for (uint32_t i = 0; i < n; ++i) {
        offsets[i] = o;
        sizes[i] = files[i].size();
        std::memcpy(blob + o, files[i].data(), files[i].size());
        o += files[i].size();
    }
    return tot;
}

}  // extern "C"
