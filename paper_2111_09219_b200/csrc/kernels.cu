// sm_100a kernels of the fully-on-GPU baseline-JPEG decode path.
//
//   K0  k0_unstuff    scan extent (first marker) + FF00 unstuffing, one pass
//                     with a segmented decoupled-lookback scan over 4 KB tiles
//                     (reference parser.hpp:238-258, bitstream.hpp:56-76)
//   K1  k1_sync       self-synchronising Huffman decode: thread per
//                     subsequence, intra-CTA overflow rounds in shared memory,
//                     then one ticket-ordered inter-CTA overflow per CTA
//                     (parallel_decode.hpp:122-285; paper Alg. 3)
//   K1c k1c_fixup     re-runs inter-CTA overflows whose predecessor's end state
//                     moved (sync_inter_sequence passes, :232-284); usually idle
//   K2  k2_scan       segmented decoupled-lookback exclusive scan of the
//                     per-subsequence slot counts and per-component DC sums,
//                     with the reference's tail trim (offsets(), :290-316)
//   K3  k3_write      re-decode from the synchronised states, writing
//                     run-length-expanded, de-zig-zagged coefficients with
//                     absolute DC straight to their data-unit slots
//                     (write_output :321-330, dc_prefix_sum transform.hpp:56-74)
//   K4  k4_transform  dequantise + exact FP64 IDCT + crop + chroma upsampling
//                     + YCbCr->RGB, staged per MCU-row tile in shared memory
//                     (transform.hpp:77-211, pipeline.hpp:167-201)
//
// Bit-exactness notes: all double arithmetic uses
// __dmul_rn/__dadd_rn/__dsub_rn so ptxas can never contract to DFMA; the
// IDCT sums run in the reference's order with zero terms skipped (exact:
// fl(s + (+-0)) == s for s != -0 and s starts at +0); rounding is lround
// (half away from zero) followed by +128, as transform.hpp:141.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "pjg_internal.h"

namespace pjg {
namespace {

constexpr uint32_t kInf32 = 0xFFFFFFFFu;

__device__ __constant__ uint8_t c_zz2r[64] = {
    0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
    12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
    35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
    58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

// ------------------------------------------------------------ utilities --
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t min64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ void spin_pause() { __nanosleep(32); }

// largest k < n with first[k] <= g (first[] ascending, first[0] == 0)
template <class T>
__device__ __forceinline__ uint32_t find_seg(const T* first, uint32_t n, uint64_t g) {
    uint32_t lo = 0, hi = n;  // invariant: first[lo] <= g < first[hi]
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (uint64_t(__ldg(first + mid)) <= g)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

__device__ __forceinline__ void set_status(ImgState* st, int32_t code) {
    atomicCAS(reinterpret_cast<int*>(&st->status), 0, code);
}

// lround (half away from zero) of a double, exactly: t = trunc(s) and
// f = s - t are exact (Sterbenz), so the tie test is exact.
__device__ __forceinline__ int lround_away(double s) {
    double t = trunc(s);
    double f = __dsub_rn(s, t);
    int r = __double2int_rz(t);
    r += (f >= 0.5) ? 1 : ((f <= -0.5) ? -1 : 0);
    return r;
}
__device__ __forceinline__ uint32_t clamp_u8(int v) { return v < 0 ? 0u : (v > 255 ? 255u : uint32_t(v)); }

// ========================================================= K0: unstuff ====
// One CTA per 4 KB tile of raw scan bytes.  Per tile: number of stuffed zero
// bytes (a 0x00 right after 0xFF) and the first marker position (0xFF not
// followed by 0x00; 0xFF as the last byte ends the scan too).  A segmented
// decoupled lookback over the image's tiles gives each tile its exclusive
// (removed, first-marker) prefix; kept bytes are then compacted into ubuf at
// the same image offset.  The tile holding the first marker fixes the
// unstuffed length U and the per-image error (EmptyScan / RST).
__global__ void __launch_bounds__(kK0Threads) k0_unstuff(Params P) {
    __shared__ uint32_t s_tile;
    __shared__ uint8_t s_b[kK0Tile + 2];
    __shared__ uint32_t s_cnt[kK0Threads / 32];
    __shared__ uint32_t s_mk[kK0Threads / 32];
    __shared__ uint32_t s_excl_cnt, s_excl_mk, s_tile_cnt, s_tile_mk;

    const int tid = threadIdx.x;
    if (tid == 0) s_tile = atomicAdd(&P.counters[kTicketK0], 1u);
    __syncthreads();
    const uint32_t t = s_tile;
    const uint32_t k = find_seg(P.k0_first, P.n_img, t);
    const uint32_t lt = t - P.k0_first[k];
    const ImgDesc& D = P.img[k];
    const uint64_t raw_len = D.raw_len;
    const uint8_t* src = P.raw + D.raw_off;
    const uint64_t j0 = uint64_t(lt) * kK0Tile;
    const uint32_t nb = uint32_t(min64(kK0Tile, raw_len - j0));

    // s_b[0] = byte j0-1 (not 0xFF at the scan start), s_b[1+i] = byte j0+i,
    // s_b[1+nb] = byte after the tile (0 past the end: marker rule handles it).
    for (uint32_t i = tid; i < nb; i += kK0Threads) s_b[1 + i] = src[j0 + i];
    if (tid == 0) s_b[0] = j0 ? src[j0 - 1] : 0;
    if (tid == 1) s_b[1 + nb] = (j0 + nb < raw_len) ? src[j0 + nb] : 0;
    __syncthreads();

    // this thread's 16 bytes
    const uint32_t b0 = tid * kK0BytesPerThread;
    uint32_t cnt = 0, mk = kInf32;
    for (int q = 0; q < kK0BytesPerThread; ++q) {
        uint32_t i = b0 + q;
        if (i >= nb) break;
        uint8_t cur = s_b[1 + i], prev = s_b[i], next = s_b[2 + i];
        uint64_t j = j0 + i;
        if (cur == 0x00 && prev == 0xFF) ++cnt;
        bool last = (j + 1 == raw_len);
        if (cur == 0xFF && (last || next != 0x00) && mk == kInf32) mk = uint32_t(j);
    }
    // block reduce (sum, min)
    uint32_t wc = cnt, wm = mk;
    for (int o = 16; o; o >>= 1) {
        wc += __shfl_xor_sync(0xFFFFFFFFu, wc, o);
        wm = min(wm, __shfl_xor_sync(0xFFFFFFFFu, wm, o));
    }
    const int warp = tid >> 5, lane = tid & 31;
    if (lane == 0) {
        s_cnt[warp] = wc;
        s_mk[warp] = wm;
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t tc = 0, tm = kInf32;
        for (int w = 0; w < kK0Threads / 32; ++w) {
            tc += s_cnt[w];
            tm = min(tm, s_mk[w]);
        }
        s_tile_cnt = tc;
        s_tile_mk = tm;
        // decoupled lookback, segmented at the image's first tile
        uint64_t* agg = P.k0_agg + 4ull * t;
        uint32_t ec = 0, em = kInf32;
        if (lt == 0) {
            agg[2] = (uint64_t(tm) << 32) | tc;
            st_release(P.k0_flag + t, (P.epoch << 2) | 2u);
        } else {
            agg[0] = (uint64_t(tm) << 32) | tc;
            st_release(P.k0_flag + t, (P.epoch << 2) | 1u);
            int64_t pr = int64_t(t) - 1;
            while (true) {
                uint32_t f = ld_acquire(P.k0_flag + pr);
                if ((f >> 2) != P.epoch) {
                    spin_pause();
                    continue;
                }
                uint64_t v = __ldcg(P.k0_agg + 4ull * pr + ((f & 3u) == 2u ? 2 : 0));
                ec += uint32_t(v);
                em = min(em, uint32_t(v >> 32));
                if ((f & 3u) == 2u) break;
                --pr;
            }
            agg[2] = (uint64_t(min(em, tm)) << 32) | (ec + tc);
            st_release(P.k0_flag + t, (P.epoch << 2) | 2u);
        }
        s_excl_cnt = ec;
        s_excl_mk = em;
    }
    __syncthreads();
    // exclusive scan of per-thread removed counts (warp shuffles + smem)
    uint32_t inc = cnt;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t v = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= o) inc += v;
    }
    __syncthreads();
    if (lane == 31) s_cnt[warp] = inc;
    __syncthreads();
    uint32_t wbase = 0;
    for (int w = 0; w < warp; ++w) wbase += s_cnt[w];
    uint32_t removed = s_excl_cnt + wbase + inc - cnt;  // removed before this thread's bytes

    uint8_t* dst = P.ubuf + D.raw_off;
    const uint32_t first_mk = s_excl_mk == kInf32 ? s_tile_mk : kInf32;  // the image's scan end
    for (int q = 0; q < kK0BytesPerThread; ++q) {
        uint32_t i = b0 + q;
        if (i >= nb) break;
        uint8_t cur = s_b[1 + i], prev = s_b[i];
        uint64_t j = j0 + i;
        if (first_mk != kInf32 && j == first_mk) {
            // scan ends here (extract_scan, parser.hpp:241-254)
            uint64_t U = j - removed;
            ImgState* st = P.ist + k;
            st->bit_length = U * 8;
            bool rst = (j + 1 < raw_len) && s_b[2 + i] >= 0xD0 && s_b[2 + i] <= 0xD7;
            if (rst)
                set_status(st, kUnsupportedFeature);
            else if (U == 0)
                set_status(st, kEmptyScan);
            else if (D.deferred)
                set_status(st, D.deferred);
        }
        if (cur == 0x00 && prev == 0xFF) {
            ++removed;
        } else {
            dst[j - removed] = cur;
        }
    }
    // no marker anywhere: the scan runs to the end of the file
    const uint32_t last_tile = uint32_t((raw_len + kK0Tile - 1) / kK0Tile) - 1;
    if (tid == 0 && lt == last_tile && s_excl_mk == kInf32 && s_tile_mk == kInf32) {
        uint64_t U = raw_len - (s_excl_cnt + s_tile_cnt);
        ImgState* st = P.ist + k;
        st->bit_length = U * 8;
        if (U == 0)
            set_status(st, kEmptyScan);
        else if (D.deferred)
            set_status(st, D.deferred);
    }
}

// ============================================== entropy decode (shared) ====
struct ImgCtx {
    const uint32_t* words;  // ubuf as 32-bit words
    uint64_t bit_base;      // 8 * raw_off
    uint64_t L;             // bit_length
    uint64_t du_comp;
    uint32_t dpm;
    const DevHuff* dc0;
    const DevHuff* dc1;
    const DevHuff* dc2;
    const DevHuff* ac0;
    const DevHuff* ac1;
    const DevHuff* ac2;
};

__device__ __forceinline__ void load_ctx(const Params& P, const ImgDesc& D, uint64_t L, ImgCtx& c) {
    c.words = reinterpret_cast<const uint32_t*>(P.ubuf);
    c.bit_base = D.raw_off * 8;
    c.L = L;
    c.du_comp = D.du_comp;
    c.dpm = D.dpm;
    c.dc0 = P.huff + D.dc_tab[0];
    c.dc1 = P.huff + D.dc_tab[1];
    c.dc2 = P.huff + D.dc_tab[2];
    c.ac0 = P.huff + D.ac_tab[0];
    c.ac1 = P.huff + D.ac_tab[1];
    c.ac2 = P.huff + D.ac_tab[2];
}

__device__ __forceinline__ uint32_t bswap32(uint32_t v) { return __byte_perm(v, 0, 0x0123); }

// Device huff_lookup with read-only-path loads.
__device__ __forceinline__ uint32_t dev_lookup(const DevHuff* t, uint32_t w16, uint32_t& maxlen) {
    maxlen = __ldg(&t->maxlen);
    uint32_t e = __ldg(&t->lut[w16 >> (16 - kPrimaryBits)]);
    if (e != 0) return e;
    for (uint32_t len = kPrimaryBits + 1; len <= maxlen; ++len) {
        int32_t code = int32_t(w16 >> (16 - len));
        if (code <= __ldg(&t->maxcode[len]))
            return (len << 8) | __ldg(&t->symbols[code + __ldg(&t->valoff[len])]);
    }
    return 0;
}

struct DecState {
    uint64_t p;
    uint32_t n;
    uint32_t c, z;
    bool div;
    int32_t err;
    int32_t dc0, dc1, dc2;
};

struct NullSink {
    static constexpr bool kWrite = false;
    __device__ __forceinline__ void put(uint32_t, int32_t) {}
};

// decode_subsequence (parallel_decode.hpp:122-164) with decode_next_symbol
// (huffman.hpp:137-175) inlined.  Decodes symbols whose first bit lies in
// [s.p, end_bit).  The caller seeds s (p, c, z, dc accumulators); n starts at
// 0.  Sync mode: an InvalidCode/OutOfBits marks the state divergent at the
// last good symbol.  Write mode: stops at `cap` slots; errors are reported.
template <class Sink>
__device__ __forceinline__ void decode_range(const ImgCtx& ic, DecState& s, uint64_t end_bit,
                                             uint32_t cap, Sink& sink) {
    s.n = 0;
    s.div = false;
    s.err = 0;
    if (s.p >= end_bit) return;
    // 64-bit MSB-first window over the unstuffed bytes
    uint64_t abs = ic.bit_base + s.p;
    uint64_t widx = abs >> 5;
    uint32_t sh = uint32_t(abs & 31);
    uint64_t acc = (uint64_t(bswap32(__ldg(ic.words + widx))) << 32) | bswap32(__ldg(ic.words + widx + 1));
    acc <<= sh;
    int cnt = 64 - int(sh);
    widx += 2;
    uint64_t p = s.p;
    uint32_t c = s.c, z = s.z, n = 0;
    int32_t a0 = s.dc0, a1 = s.dc1, a2 = s.dc2;
    const uint64_t L = ic.L;
    while (p < end_bit) {
        if (Sink::kWrite && n >= cap) break;
        if (cnt <= 32) {
            acc |= uint64_t(bswap32(__ldg(ic.words + widx))) << (32 - cnt);
            cnt += 32;
            ++widx;
        }
        const uint32_t comp = uint32_t(ic.du_comp >> (4 * c)) & 15u;
        const DevHuff* t = z == 0 ? (comp == 0 ? ic.dc0 : (comp == 1 ? ic.dc1 : ic.dc2))
                                  : (comp == 0 ? ic.ac0 : (comp == 1 ? ic.ac1 : ic.ac2));
        const uint64_t avail = L - p;  // >= 1 inside the loop
        uint32_t maxlen;
        const uint32_t e = dev_lookup(t, uint32_t(acc >> 48), maxlen);
        const uint32_t len = e >> 8, sym = e & 255u;
        int32_t err = 0;
        uint32_t l = 0, run = 0;
        bool eob = false, coefk = false;
        if (len == 0) {
            err = avail < maxlen ? kOutOfBits : kInvalidCode;
        } else if (len > avail) {
            err = kOutOfBits;
        } else if (z == 0) {
            l = sym;
            if (l > 11)
                err = kInvalidCode;
            else if (avail - len < l)
                err = kOutOfBits;
            coefk = true;
        } else {
            const uint32_t r = sym >> 4;
            l = sym & 15u;
            if (l == 0) {
                if (r == 0) {
                    eob = true;
                    run = 63 - z;
                } else if (r == 15) {
                    run = 15;
                } else {
                    err = kInvalidCode;
                }
            } else if (l > 10) {
                err = kInvalidCode;
            } else if (avail - len < l) {
                err = kOutOfBits;
            } else {
                run = r;
                coefk = true;
            }
        }
        if (err) {
            s.div = true;
            s.err = err;
            break;
        }
        int32_t coef = 0;
        if (l) {
            uint32_t bits = uint32_t((acc << len) >> (64 - l));
            coef = bits >= (1u << (l - 1)) ? int32_t(bits) : int32_t(bits) - int32_t((1u << l) - 1);
        }
        const uint32_t total = len + l;
        const uint32_t step = run + 1;
        if (Sink::kWrite && n + step > cap) break;  // phantom tail past the true end
        if (z == 0) {
            if (comp == 0)
                a0 += coef, coef = a0;
            else if (comp == 1)
                a1 += coef, coef = a1;
            else
                a2 += coef, coef = a2;
        }
        if (Sink::kWrite && coefk) sink.put(n + run, coef);
        acc <<= total;
        cnt -= int(total);
        p += total;
        n += step;
        z += step;
        if (z >= 64 || eob) {
            z = 0;
            c = (c + 1 == ic.dpm) ? 0 : c + 1;
        }
    }
    s.p = p;
    s.n = n;
    s.c = c;
    s.z = z;
    s.dc0 = a0;
    s.dc1 = a1;
    s.dc2 = a2;
}

__device__ __forceinline__ DcSums pack_dc(int32_t a0, int32_t a1, int32_t a2) {
    DcSums d;
    d.lo = (uint32_t(a0) & 0xFFFFu) | (uint32_t(a1) << 16);
    d.hi = uint32_t(a2) & 0xFFFFu;
    return d;
}

// Sync-mode decode of subsequence i from (p, c, z).
__device__ __forceinline__ void sync_decode(const ImgCtx& ic, uint64_t sb, uint64_t i, uint64_t p,
                                            uint32_t c, uint32_t z, Entry& e, DcSums& d) {
    DecState s;
    s.p = p;
    s.c = c;
    s.z = z;
    s.dc0 = s.dc1 = s.dc2 = 0;
    NullSink sink;
    uint64_t end_bit = min((i + 1) * sb, ic.L);
    decode_range(ic, s, end_bit, 0, sink);
    e.p = s.p;
    e.n = s.n;
    e.czd = pack_czd(s.c, s.z, s.div);
    d = pack_dc(s.dc0, s.dc1, s.dc2);
}

// ======================================================== K1: sync pass ====
// Thread t of logical CTA j owns global subsequence g = j*T + t.  Images are
// flattened into one subsequence space; a CTA may hold the tail of one image
// and the head of the next, and overflow chains stop at image ends.
__global__ void __launch_bounds__(kK1Threads) k1_sync(Params P) {
    constexpr int T = kK1Threads;
    __shared__ uint64_t s_p[T];
    __shared__ uint32_t s_n[T];
    __shared__ uint32_t s_czd[T];
    __shared__ DcSums s_dc[T];
    __shared__ uint32_t s_cta;
    __shared__ int s_rounds;

    const int tid = threadIdx.x;
    if (tid == 0) s_cta = atomicAdd(&P.counters[kTicketK1], 1u);
    __syncthreads();
    const uint32_t cta = s_cta;
    const uint64_t g = uint64_t(cta) * T + tid;
    const bool inb = g < P.total_subs;
    const uint32_t k = find_seg(P.sub_first, P.n_img, inb ? g : P.total_subs - 1);
    const ImgDesc& D = P.img[k];
    const uint64_t i = g - P.sub_first[k];
    const uint64_t L = P.ist[k].bit_length;
    const bool ok = P.ist[k].status == 0;
    const uint64_t N = ok ? (L + P.sb - 1) / P.sb : 0;
    const bool real = inb && i < N;
    ImgCtx ic;
    load_ctx(P, D, L, ic);

    // Round 0: every subsequence decodes from its origin (parallel_decode.hpp:187-195)
    Entry e;
    DcSums d = {0, 0};
    e.p = i * P.sb;
    e.n = 0;
    e.czd = 0;
    if (real) sync_decode(ic, P.sb, i, i * P.sb, 0, 0, e, d);
    s_p[tid] = e.p;
    s_n[tid] = e.n;
    s_czd[tid] = e.czd;
    s_dc[tid] = d;
    Entry chain = e;
    uint64_t nxt = i + 1;
    int nt = tid + 1;
    bool active = real && !czd_div(e.czd) && nxt < N && nt < T;
    // Rounds k >= 1: overflow into the next subsequence until (p,c,z) agrees
    // with the published entry (parallel_decode.hpp:197-220).  All active
    // threads target distinct subsequences, so one barrier per round suffices.
    int rounds = 0;
    while (__syncthreads_or(active)) {
        ++rounds;
        if (active) {
            Entry e2;
            DcSums d2;
            sync_decode(ic, P.sb, nxt, chain.p, czd_c(chain.czd), czd_z(chain.czd), e2, d2);
            bool synced = sync_equal(e2.p, e2.czd, s_p[nt], s_czd[nt]);
            s_p[nt] = e2.p;
            s_n[nt] = e2.n;  // the overflow's n is authoritative (:211)
            s_czd[nt] = e2.czd;
            s_dc[nt] = d2;
            if (synced || czd_div(e2.czd)) {
                active = false;
            } else {
                chain = e2;
                ++nxt;
                ++nt;
                active = nxt < N && nt < T;
            }
        }
    }
    if (tid == 0) {
        atomicAdd(P.stats + kStatRoundsSum, (unsigned long long)rounds);
        atomicMax(P.stats + kStatRoundsMax, (unsigned long long)rounds);
    }
    // Publish this CTA's last entry (post-intra) for the successor CTA.
    if (tid == T - 1) {
        Entry last;
        last.p = s_p[T - 1];
        last.n = s_n[T - 1];
        last.czd = s_czd[T - 1];
        P.cta_end[cta] = last;
        __threadfence();
        st_release(P.k1_flag + cta, P.epoch);
    }
    // Inter-CTA overflow (sync_inter_sequence, parallel_decode.hpp:247-270):
    // thread 0 chains from the predecessor CTA's last entry into this CTA.
    if (tid == 0) {
        Entry start;
        start.p = 0;
        start.n = 0;
        start.czd = 0;
        const bool boundary = real && i > 0;  // CTA starts mid-image
        if (boundary) {
            while (ld_acquire(P.k1_flag + cta - 1) != P.epoch) spin_pause();
            start.p = __ldcg(&P.cta_end[cta - 1].p);
            uint64_t nc = __ldcg(reinterpret_cast<const unsigned long long*>(&P.cta_end[cta - 1]) + 1);
            start.n = uint32_t(nc);
            start.czd = uint32_t(nc >> 32);
            if (!czd_div(start.czd)) {
                Entry ch = start;
                uint64_t ii = i;
                uint32_t hops = 0;
                for (int tt = 0; tt < T && ii < N; ++tt, ++ii) {
                    Entry e2;
                    DcSums d2;
                    sync_decode(ic, P.sb, ii, ch.p, czd_c(ch.czd), czd_z(ch.czd), e2, d2);
                    ++hops;
                    bool synced = sync_equal(e2.p, e2.czd, s_p[tt], s_czd[tt]);
                    s_p[tt] = e2.p;
                    s_n[tt] = e2.n;
                    s_czd[tt] = e2.czd;
                    s_dc[tt] = d2;
                    if (synced || czd_div(e2.czd)) break;
                    ch = e2;
                }
                atomicAdd(P.stats + kStatInterHops, (unsigned long long)hops);
            }
            start.czd |= kBoundaryBit;
        }
        P.cta_start[cta] = start;
    }
    __syncthreads();
    if (inb) {
        Entry o;
        o.p = s_p[tid];
        o.n = s_n[tid];
        o.czd = s_czd[tid];
        P.ent[g] = o;
        P.dcs[g] = s_dc[tid];
    }
}

// ================================================ K1c: inter fix-up pass ====
// Each CTA j>0 that starts mid-image overflowed from CTA j-1's post-intra end
// state.  If CTA j-1's own inter overflow later changed that end state
// (the chain ran through the whole CTA), CTA j must redo its overflow from
// the final state — the reference's `end_changed` invalidation
// (parallel_decode.hpp:272-276).  Passes repeat until no boundary is stale.
__global__ void __launch_bounds__(1024) k1c_fixup(Params P) {
    constexpr int T = kK1Threads;
    __shared__ int s_any;
    __shared__ int s_passes;
    if (threadIdx.x == 0) s_passes = 0;
    for (uint32_t pass = 0; pass <= P.k1_ctas; ++pass) {
        if (threadIdx.x == 0) s_any = 0;
        __syncthreads();
        // snapshot: which boundaries are stale (start used != final predecessor end)
        for (uint32_t cta = 1 + threadIdx.x; cta < P.k1_ctas; cta += blockDim.x) {
            Entry st = P.cta_start[cta];
            if (!(st.czd & kBoundaryBit)) continue;
            uint64_t g0 = uint64_t(cta) * T;
            Entry pe = P.ent[g0 - 1];
            bool stale = !sync_equal(st.p, st.czd, pe.p, pe.czd);
            if (stale) {
                // stash the new start; mark for this pass
                pe.czd |= kBoundaryBit | 0x2000u;
                P.cta_start[cta] = pe;
                s_any = 1;
            }
        }
        __syncthreads();
        if (!s_any) break;
        if (threadIdx.x == 0) ++s_passes;
        for (uint32_t cta = 1 + threadIdx.x; cta < P.k1_ctas; cta += blockDim.x) {
            Entry st = P.cta_start[cta];
            if (!(st.czd & 0x2000u)) continue;
            st.czd &= ~0x2000u;
            P.cta_start[cta] = st;
            uint64_t g0 = uint64_t(cta) * T;
            uint32_t k = find_seg(P.sub_first, P.n_img, g0);
            const ImgDesc& D = P.img[k];
            const uint64_t L = P.ist[k].bit_length;
            const uint64_t N = (L + P.sb - 1) / P.sb;
            uint64_t i = g0 - P.sub_first[k];
            if (czd_div(st.czd)) {
                set_status(P.ist + k, kConsistencyFailure);
                continue;
            }
            ImgCtx ic;
            load_ctx(P, D, L, ic);
            Entry ch = st;
            for (int tt = 0; tt < T && i < N; ++tt, ++i) {
                Entry e2;
                DcSums d2;
                sync_decode(ic, P.sb, i, ch.p, czd_c(ch.czd), czd_z(ch.czd), e2, d2);
                Entry old = P.ent[g0 + tt];
                bool synced = sync_equal(e2.p, e2.czd, old.p, old.czd);
                P.ent[g0 + tt] = e2;
                P.dcs[g0 + tt] = d2;
                if (synced || czd_div(e2.czd)) break;
                ch = e2;
            }
        }
        __threadfence_block();
        __syncthreads();
    }
    if (threadIdx.x == 0 && s_passes) atomicAdd(P.stats + kStatFixPasses, (unsigned long long)s_passes);
}

// ===================================================== K2: offsets scan ====
// Segmented (per image) decoupled-lookback exclusive scan over subsequences of
// (slot count n, per-component DC sums mod 2^16).  Then the reference's tail
// trim: trimmed prefix = min(prefix, expected), so the last entries lose the
// phantom excess (offsets(), parallel_decode.hpp:290-316).
struct ScanVal {
    uint64_t n;     // bit 63: segment head
    uint32_t lo, hi;
};
constexpr uint64_t kHead = 1ull << 63;

__device__ __forceinline__ ScanVal scan_op(const ScanVal& a, const ScanVal& b) {
    // a precedes b
    ScanVal r;
    if (b.n & kHead) return b;
    r.n = ((a.n & ~kHead) + b.n) | (a.n & kHead);
    r.lo = __vadd2(a.lo, b.lo);
    r.hi = __vadd2(a.hi, b.hi);
    return r;
}

__global__ void __launch_bounds__(kK2Threads) k2_scan(Params P) {
    constexpr int T = kK2Threads;
    __shared__ uint32_t s_tile;
    __shared__ ScanVal s_w[T / 32];
    __shared__ ScanVal s_excl;
    __shared__ int s_first_head;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(&P.counters[kTicketK2], 1u);
    __syncthreads();
    const uint32_t t = s_tile;
    const uint64_t g = uint64_t(t) * T + tid;
    const bool inb = g < P.total_subs;
    uint32_t k = find_seg(P.sub_first, P.n_img, inb ? g : P.total_subs - 1);
    const uint64_t i = g - P.sub_first[k];
    ScanVal v;
    v.n = 0;
    v.lo = v.hi = 0;
    if (inb) {
        Entry e = P.ent[g];
        DcSums d = P.dcs[g];
        v.n = e.n;
        v.lo = d.lo;
        v.hi = d.hi;
        if (i == 0) v.n |= kHead;
    }
    // warp inclusive segmented scan
    ScanVal x = v;
    for (int o = 1; o < 32; o <<= 1) {
        ScanVal y;
        y.n = __shfl_up_sync(0xFFFFFFFFu, x.n, o);
        y.lo = __shfl_up_sync(0xFFFFFFFFu, x.lo, o);
        y.hi = __shfl_up_sync(0xFFFFFFFFu, x.hi, o);
        if (lane >= o) x = scan_op(y, x);
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    ScanVal wpre;  // exclusive prefix of earlier warps in this tile
    wpre.n = 0;
    wpre.lo = wpre.hi = 0;
    bool have_wpre = false;
    for (int w = 0; w < warp; ++w) {
        wpre = have_wpre ? scan_op(wpre, s_w[w]) : s_w[w];
        have_wpre = true;
    }
    ScanVal incl = have_wpre ? scan_op(wpre, x) : x;
    if (tid == 0) s_first_head = (v.n & kHead) ? 1 : 0;
    __syncthreads();
    if (tid == T - 1) {
        // Tile aggregate = incl of the last thread.  A tile whose aggregate
        // carries a segment head is its own inclusive prefix for successors,
        // but its threads before that head still need the lookback unless the
        // tile starts with a head (or is tile 0).
        uint64_t* agg = P.k2_agg + 8ull * t;
        ScanVal ex;
        ex.n = 0;
        ex.lo = ex.hi = 0;
        const bool own_prefix = (incl.n & kHead) != 0;
        const bool need = t > 0 && !s_first_head;
        if (own_prefix || !need) {
            agg[4] = incl.n;
            agg[5] = (uint64_t(incl.hi) << 32) | incl.lo;
            __threadfence();
            st_release(P.k2_flag + t, (P.epoch << 2) | 2u);
        } else {
            agg[0] = incl.n;
            agg[1] = (uint64_t(incl.hi) << 32) | incl.lo;
            __threadfence();
            st_release(P.k2_flag + t, (P.epoch << 2) | 1u);
        }
        if (need) {
            int64_t pr = int64_t(t) - 1;
            bool first = true;
            while (true) {
                uint32_t f = ld_acquire(P.k2_flag + pr);
                if ((f >> 2) != P.epoch) {
                    spin_pause();
                    continue;
                }
                const uint64_t* src = P.k2_agg + 8ull * pr + ((f & 3u) == 2u ? 4 : 0);
                ScanVal pv;
                pv.n = __ldcg(src);
                uint64_t dd = __ldcg(src + 1);
                pv.lo = uint32_t(dd);
                pv.hi = uint32_t(dd >> 32);
                ex = first ? pv : scan_op(pv, ex);
                first = false;
                if ((f & 3u) == 2u || (pv.n & kHead)) break;
                --pr;
            }
            if (!own_prefix) {
                ScanVal ti = scan_op(ex, incl);
                agg[4] = ti.n;
                agg[5] = (uint64_t(ti.hi) << 32) | ti.lo;
                __threadfence();
                st_release(P.k2_flag + t, (P.epoch << 2) | 2u);
            }
        }
        s_excl = ex;
    }
    __syncthreads();
    if (!inb) return;
    // exclusive prefix of this thread within its image
    ScanVal before;  // everything before this thread in scan order
    {
        ScanVal tile_ex = s_excl;
        ScanVal wx;  // exclusive within tile
        ScanVal xup;
        xup.n = __shfl_up_sync(0xFFFFFFFFu, x.n, 1);
        xup.lo = __shfl_up_sync(0xFFFFFFFFu, x.lo, 1);
        xup.hi = __shfl_up_sync(0xFFFFFFFFu, x.hi, 1);
        bool have = false;
        wx.n = 0;
        wx.lo = wx.hi = 0;
        if (have_wpre) {
            wx = wpre;
            have = true;
        }
        if (lane > 0) {
            wx = have ? scan_op(wx, xup) : xup;
            have = true;
        }
        before = have ? scan_op(tile_ex, wx) : tile_ex;
    }
    if (v.n & kHead) {
        before.n = 0;
        before.lo = before.hi = 0;
    }
    const ImgDesc& D = P.img[k];
    const uint64_t E = D.expected;
    const uint64_t pre = before.n & ~kHead;
    const uint64_t n = v.n & ~kHead;
    const uint64_t o = min(pre, E);
    P.off[g] = o;
    P.cap[g] = uint32_t(min(pre + n, E) - o);
    DcSums pd;
    pd.lo = before.lo;
    pd.hi = before.hi;
    P.pred[g] = pd;
    if (i + 1 == D.sub_count && P.ist[k].status == 0) {
        const uint64_t total = pre + n;
        if (total < E || total - E > 512) set_status(P.ist + k, kConsistencyFailure);
    }
}

// ======================================================= K3: write pass ====
// Per-thread 64-coefficient staging block in shared memory (raster order,
// stride 72 int16 → conflict-free 16-byte rows).  Blocks this thread fully
// owns go out as 8 x 16-byte stores; the partial first/last blocks shared
// with a neighbouring subsequence write only the owned slots.
constexpr int kBlkStride = 72;

struct BlockSink {
    static constexpr bool kWrite = true;
    int16_t* buf;        // this thread's smem block
    int16_t* coef;       // batch coefficient buffer
    uint64_t du_first;   // image's first data unit
    uint64_t own_lo;     // owned slots [own_lo, own_hi) within the image
    uint64_t own_hi;
    uint64_t cur;        // current block (image-relative)

    __device__ __forceinline__ void flush(uint64_t b) {
        const uint64_t lo = max(own_lo, b * 64), hi = min(own_hi, b * 64 + 64);
        int16_t* dst = coef + (du_first + b) * 64;
        if (lo == b * 64 && hi == b * 64 + 64) {
            const int4* s4 = reinterpret_cast<const int4*>(buf);
            int4* d4 = reinterpret_cast<int4*>(dst);
#pragma unroll
            for (int q = 0; q < 8; ++q) d4[q] = s4[q];
        } else {
            for (uint64_t sl = lo; sl < hi; ++sl) {
                int r = c_zz2r[sl & 63];
                dst[r] = buf[r];
            }
        }
        int4 zero = make_int4(0, 0, 0, 0);
#pragma unroll
        for (int q = 0; q < 8; ++q) reinterpret_cast<int4*>(buf)[q] = zero;
    }
    // slot relative to this subsequence's offset is passed as local index
    uint64_t base;       // own_lo
    __device__ __forceinline__ void put(uint32_t local, int32_t v) {
        const uint64_t s = base + local;
        const uint64_t b = s >> 6;
        while (cur < b) {
            flush(cur);
            ++cur;
        }
        buf[c_zz2r[s & 63]] = int16_t(v);
    }
    __device__ __forceinline__ void finish() {
        if (own_hi <= own_lo) return;
        const uint64_t last = (own_hi - 1) >> 6;
        while (cur <= last) {
            flush(cur);
            ++cur;
        }
    }
};

__global__ void __launch_bounds__(kK3Threads) k3_write(Params P) {
    __shared__ __align__(16) int16_t s_blk[kK3Threads * kBlkStride];
    const int tid = threadIdx.x;
    int16_t* buf = s_blk + tid * kBlkStride;
    {
        int4 zero = make_int4(0, 0, 0, 0);
#pragma unroll
        for (int q = 0; q < 8; ++q) reinterpret_cast<int4*>(buf)[q] = zero;
    }
    const uint64_t g = uint64_t(blockIdx.x) * kK3Threads + tid;
    if (g >= P.total_subs) return;
    const uint32_t cap = P.cap[g];
    if (cap == 0) return;
    const uint32_t k = find_seg(P.sub_first, P.n_img, g);
    if (P.ist[k].status != 0) return;
    const ImgDesc& D = P.img[k];
    const uint64_t i = g - P.sub_first[k];
    const uint64_t L = P.ist[k].bit_length;
    ImgCtx ic;
    load_ctx(P, D, L, ic);
    DecState s;
    if (i == 0) {
        s.p = 0;
        s.c = 0;
        s.z = 0;
    } else {
        Entry e = P.ent[g - 1];
        s.p = e.p;
        s.c = czd_c(e.czd);
        s.z = czd_z(e.czd);
    }
    const DcSums pd = P.pred[g];
    s.dc0 = int16_t(pd.lo & 0xFFFFu);
    s.dc1 = int16_t(pd.lo >> 16);
    s.dc2 = int16_t(pd.hi & 0xFFFFu);
    const uint64_t o = P.off[g];
    BlockSink sink;
    sink.buf = buf;
    sink.coef = P.coef;
    sink.du_first = D.du_first;
    sink.own_lo = o;
    sink.own_hi = o + cap;
    sink.base = o;
    sink.cur = o >> 6;
    const uint64_t end_bit = min((i + 1) * P.sb, L);
    decode_range(ic, s, end_bit, cap, sink);
    if (s.err) {
        set_status(P.ist + k, s.err);  // write mode rethrows (parallel_decode.hpp:142)
        return;
    }
    sink.finish();
}

// ============================================ K4: IDCT + upsample + RGB ====
// One CTA (384 threads) per tile of `mcus_per_tile` MCUs of one MCU row
// (<= 48 data units, so one thread per (data unit, column)).
//
// Exactness strategy (reference transform.hpp:114-142, pipeline.hpp:190-197
// are IEEE double):
//  * IDCT: FP32 FMA separable sum with a rigorous per-block error bound
//    |r32 - r64| <= 18.1 u S, S <= max|b|^2 * sum|F| (u = 2^-24).  A sample
//    whose FP32 value lies farther than that bound from a rounding boundary
//    (x.5) rounds identically to the reference double; the rest (~0.1-0.3%)
//    are recomputed exactly in FP64 in the reference's summation order.
//    Blocks whose coefficients are not exact in FP32 take the FP64 path.
//  * Colour: Y is an integer, so lround(Y + t) = Y + round(t) unless t is an
//    exact half-integer in real arithmetic (FP64 rounding then decides).
//    round(t) is computed exactly in integers per chroma sample
//    (1.402, 0.344136, 0.714136, 1.772 are decimal); exact ties are detected
//    in integers and only those pixels are evaluated in FP64.
constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: float + kMagic rounds to an integer
constexpr int kMagicBits = 0x4B400000;

__device__ __forceinline__ int round_div_away(int n, int d) {
    return n >= 0 ? (n + d / 2) / d : -((-n + d / 2) / d);
}

// packed per-chroma-sample offsets: oR, oG, oB biased by 512 in 10-bit
// fields, bit 30 = an exact real tie somewhere (FP64 replay needed)
__device__ __forceinline__ uint32_t chroma_word(int Cb, int Cr) {
    const int cb = Cb - 128, cr = Cr - 128;
    const int nR = 1402 * cr, nB = 1772 * cb, nG = -(344136 * cb + 714136 * cr);
    const bool tie = (abs(nR) % 1000 == 500) | (abs(nB) % 1000 == 500) | (abs(nG) % 1000000 == 500000);
    const int oR = round_div_away(nR, 1000), oB = round_div_away(nB, 1000), oG = round_div_away(nG, 1000000);
    return uint32_t(oR + 512) | (uint32_t(oG + 512) << 10) | (uint32_t(oB + 512) << 20) | (tie ? (1u << 30) : 0u);
}

__device__ __forceinline__ uint32_t pack4_sat(int a0, int a1, int a2, int a3) {
    uint32_t t, d;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(t) : "r"(a3), "r"(a2), "r"(0));
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a1), "r"(a0), "r"(t));
    return d;
}

// exact FP64 replay of one sample (reference order, zero terms skipped):
// walks the nonzero rows / coefficients of the data unit via bit masks.
__device__ __noinline__ int idct_sample_fp64(const float* F, bool big, uint32_t rows, const uint8_t* nz,
                                             const double* b64, int x, int y) {
    const int32_t* Fi = reinterpret_cast<const int32_t*>(F);
    double s = 0.0;
    while (rows) {
        const int u = __ffs(rows) - 1;
        rows &= rows - 1;
        uint32_t m = nz[u];
        double t = 0.0;
        while (m) {
            const int v = __ffs(m) - 1;
            m &= m - 1;
            const double f = big ? double(Fi[u * 8 + v]) : double(F[u * 8 + v]);
            t = __dadd_rn(t, __dmul_rn(b64[v * 8 + y], f));
        }
        s = __dadd_rn(s, __dmul_rn(b64[u * 8 + x], t));
    }
    return lround_away(s) + 128;
}

__device__ __noinline__ void rgb_fp64(int Y, int Cb, int Cr, int& R, int& G, int& B) {
    const double Yd = double(Y);
    const int cb = Cb - 128, cr = Cr - 128;
    R = lround_away(__dadd_rn(Yd, __dmul_rn(1.402, double(cr))));
    G = lround_away(__dsub_rn(__dsub_rn(Yd, __dmul_rn(0.344136, double(cb))), __dmul_rn(0.714136, double(cr))));
    B = lround_away(__dadd_rn(Yd, __dmul_rn(1.772, double(cb))));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// TMA bulk copy global -> shared, completion counted on an mbarrier (UBLKCP)
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Per-tile geometry, computed by one thread and shared through smem.
struct TileInfo {
    uint32_t k;  // image
    uint32_t my, mx0, nm, nblk;
    uint32_t valid;
    uint64_t du0;
    // plane geometry inside the tile (row stride padded by 4 bytes against bank conflicts)
    uint32_t pw_t[3], pst[3], poff[3];
    uint32_t X0, Y0, cols, rws;
    uint32_t rgb;
};

// Tiles of one CTA are a contiguous range, so the image index only walks
// forward; kend caches tile_first[kc + 1].
__device__ __forceinline__ void tile_info(const Params& P, uint32_t t, uint32_t& kc, uint32_t& kend,
                                          TileInfo& ti) {
    while (t >= kend) {
        ++kc;
        kend = P.tile_first[kc + 1];
    }
    const ImgDesc& D = P.img[kc];
    const uint32_t lt = t - P.tile_first[kc];
    const uint32_t MT = D.mcus_per_tile;
    ti.k = kc;
    ti.my = lt / D.tiles_x;
    ti.mx0 = (lt % D.tiles_x) * MT;
    ti.nm = min(MT, D.mcus_x - ti.mx0);
    ti.nblk = ti.nm * D.dpm;
    ti.du0 = D.du_first + (uint64_t(ti.my) * D.mcus_x + ti.mx0) * D.dpm;
    ti.valid = P.ist[kc].status == 0;
    uint32_t acc = 0;
    for (uint32_t c = 0; c < 3; ++c) {
        const bool has = c < D.ncomp;
        ti.pw_t[c] = has ? MT * D.comp_h[c] * 8 : 0;
        ti.pst[c] = ti.pw_t[c] + 4;
        ti.poff[c] = acc;
        acc += has ? ti.pst[c] * D.comp_v[c] * 8 : 0;
    }
    const uint32_t mcu_w = 8 * D.h_max, mcu_h = 8 * D.v_max;
    ti.X0 = ti.mx0 * mcu_w;
    ti.Y0 = ti.my * mcu_h;
    ti.cols = min(ti.nm * mcu_w, D.width - ti.X0);
    ti.rws = min(mcu_h, D.height - ti.Y0);
    ti.rgb = D.out_mode == 1 && D.ncomp == 3;
}

// packed offsets of one chroma sample: oR, oG, oB biased by 512 in 10-bit
// fields; bit 30 flags an exact real tie (FP64 replay).  round(k*c) is taken
// in integers on biased-positive values (divisions by constants).
__device__ __forceinline__ uint32_t chroma_word2(uint32_t Cb, uint32_t Cr) {
    const int cb = int(Cb) - 128, cr = int(Cr) - 128;
    const uint32_t mR = uint32_t(1402 * cr + 500 + 200000);
    const uint32_t mB = uint32_t(1772 * cb + 500 + 300000);
    const uint32_t mG = uint32_t(-(344136 * cb + 714136 * cr) + 500000 + 200000000);
    const uint32_t qR = mR / 1000u, qB = mB / 1000u, qG = mG / 1000000u;
    const bool tie = (mB - qB * 1000u == 0) | (mG - qG * 1000000u == 0) | (mR - qR * 1000u == 0);
    // oX + 512 = q - bias + 512
    return (qR + 312u) | ((qG + 312u) << 10) | ((qB + 212u) << 20) | (tie ? (1u << 30) : 0u);
}

// one row of 4 pixels: Y bytes in y4, chroma words w0..w3
__device__ __forceinline__ void emit_rgb4(uint8_t* dst, bool fast, uint32_t npx, uint32_t y4, const uint32_t w[4],
                                          const uint8_t* cbrow, const uint8_t* crrow, const uint32_t cx[4]) {
    int R[4], G[4], B[4];
    uint32_t tie = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int Yv = int((y4 >> (8 * q)) & 0xFFu) - 512;
        R[q] = Yv + int(w[q] & 1023u);
        G[q] = Yv + int((w[q] >> 10) & 1023u);
        B[q] = Yv + int((w[q] >> 20) & 1023u);
        tie |= (w[q] >> 30) << q;
    }
    if (tie) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if ((tie & (1u << q)) && q < int(npx))
                rgb_fp64(int((y4 >> (8 * q)) & 0xFFu), cbrow[cx[q]], crrow[cx[q]], R[q], G[q], B[q]);
    }
    const uint32_t r4 = pack4_sat(R[0], R[1], R[2], R[3]);
    const uint32_t g4 = pack4_sat(G[0], G[1], G[2], G[3]);
    const uint32_t b4 = pack4_sat(B[0], B[1], B[2], B[3]);
    const uint32_t t0 = __byte_perm(r4, g4, 0x5140);                            // R0 G0 R1 G1
    const uint32_t t1 = __byte_perm(r4, g4, 0x7362);                            // R2 G2 R3 G3
    const uint32_t o0 = __byte_perm(t0, b4, 0x2410);                            // R0 G0 B0 R1
    const uint32_t o1 = __byte_perm(__byte_perm(t0, b4, 0x0053), t1, 0x5410);  // G1 B1 R2 G2
    const uint32_t o2 = __byte_perm(t1, b4, 0x7326);                            // B2 R3 G3 B3
    if (fast) {
        uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
        d32[0] = o0;
        d32[1] = o1;
        d32[2] = o2;
    } else {
        for (uint32_t q = 0; q < npx * 3; ++q) {
            const uint32_t wq = q < 4 ? o0 : (q < 8 ? o1 : o2);
            dst[q] = uint8_t(wq >> (8 * (q & 3)));
        }
    }
}

// Persistent: grid = min(#tiles, SMs x resident CTAs); each CTA walks tiles
// blockIdx.x, +gridDim.x, ...; the next tile's coefficients are prefetched by
// a TMA bulk copy into the other staging buffer while this tile computes.
__global__ void __launch_bounds__(kK4Threads, 4) k4_transform(Params P) {
    constexpr int NB = kK4MaxBlocks;
    constexpr int kPlaneBytes = NB * 64 + 3 * 16 * 4;
    // max_x |basis[u][x]| rounded up: weights of the rigorous FP32 error bound
    constexpr float kW[8] = {0.35356f, 0.4904f, 0.46195f, 0.4904f, 0.35356f, 0.4904f, 0.46195f, 0.4904f};
    __shared__ __align__(128) int16_t s_raw[2][NB * 64];
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ TileInfo s_ti[2];
    __shared__ ImgDesc s_desc[2];
    __shared__ __align__(16) float s_F[NB * 64];  // float, or int32 bits when big
    __shared__ __align__(16) uint8_t s_pl[kPlaneBytes];
    __shared__ __align__(16) float s_b32[64];
    __shared__ __align__(16) double s_b64[64];
    __shared__ __align__(8) uint16_t s_cmap[192 + 4];
    __shared__ uint8_t s_rmap[16];
    __shared__ uint8_t s_rows[NB];
    __shared__ uint8_t s_nz[NB * 8];
    __shared__ uint8_t s_big[NB];
    __shared__ float s_lim[NB];

    const int tid = threadIdx.x, lane = tid & 31;
    // this CTA's contiguous tile range
    const uint32_t t_begin = uint32_t(uint64_t(P.k4_tiles) * blockIdx.x / gridDim.x);
    const uint32_t t_end = uint32_t(uint64_t(P.k4_tiles) * (blockIdx.x + 1) / gridDim.x);
    __shared__ uint32_t s_desc_k[2];
    uint32_t kc = 0, kend = 0;  // thread 0's cached image index and its tile end
    if (tid < 64) {
        const double b = P.basis[tid];
        s_b64[tid] = b;
        s_b32[tid] = float(b);
    }
    if (tid == 0 && t_begin < t_end) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // first image of the range: binary search once
        uint32_t lo = 0, hi = P.n_img;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (P.tile_first[mid] <= t_begin) lo = mid; else hi = mid;
        }
        kc = lo;
        kend = P.tile_first[kc + 1];
        tile_info(P, t_begin, kc, kend, s_ti[0]);
        s_desc[0] = P.img[s_ti[0].k];
        s_desc_k[0] = s_ti[0].k;
        s_desc_k[1] = 0xFFFFFFFFu;
        const uint32_t bytes = s_ti[0].nblk * 128;
        mbar_expect_tx(&s_bar[0], bytes);
        tma_load(s_raw[0], P.coef + s_ti[0].du0 * 64, bytes, &s_bar[0]);
    }
    for (uint32_t it = 0;; ++it) {
        const uint32_t t = t_begin + it;
        if (t >= t_end) break;
        const uint32_t cb = it & 1;
        __syncthreads();  // previous tile done with every buffer; s_ti/s_desc[cb] ready
        if (tid == 0) {
            const uint32_t tn = t + 1;
            if (tn < t_end) {
                TileInfo ti;
                tile_info(P, tn, kc, kend, ti);
                s_ti[cb ^ 1] = ti;
                if (s_desc_k[cb ^ 1] != ti.k) {
                    s_desc[cb ^ 1] = P.img[ti.k];
                    s_desc_k[cb ^ 1] = ti.k;
                }
                const uint32_t bytes = ti.nblk * 128;
                mbar_expect_tx(&s_bar[cb ^ 1], bytes);
                tma_load(s_raw[cb ^ 1], P.coef + ti.du0 * 64, bytes, &s_bar[cb ^ 1]);
            }
        }
        const TileInfo& ti = s_ti[cb];
        const ImgDesc& D = s_desc[cb];
        mbar_wait(&s_bar[cb], (it >> 1) & 1);
        if (!ti.valid) continue;
        const uint32_t nblk = ti.nblk, dpm = D.dpm;

        // 1. dequantise: thread (data unit, coefficient row); the 8 lanes of a
        //    data unit reduce its row mask, "big" flag and the weighted sum
        //    S = sum_uv w_u w_v |F_uv| that bounds the FP32 error.
        {
            const uint32_t ch = tid;  // NB * 8 == kK4Threads
            const bool act = ch < nblk * 8;
            const uint32_t u = ch & 7;
            uint32_t m = 0;
            float S = 0.f;
            int32_t d[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            if (act) {
                const uint32_t blk = ch >> 3, slot = blk % dpm;
                const uint32_t comp = uint32_t(D.du_comp >> (4 * slot)) & 15u;
                const uint4 q4 =
                    __ldg(reinterpret_cast<const uint4*>(P.quant_raster + 64u * D.q_tab[comp] + u * 8));
                const int4 v = *reinterpret_cast<const int4*>(s_raw[cb] + ch * 8);
                const int16_t* c16 = reinterpret_cast<const int16_t*>(&v);
                const uint16_t* q16 = reinterpret_cast<const uint16_t*>(&q4);
                uint32_t rm = 0, big = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    d[j] = int32_t(c16[j]) * int32_t(q16[j]);
                    const uint32_t a = uint32_t(abs(d[j]));
                    rm |= a ? (1u << j) : 0u;
                    big |= a >= (1u << 22) ? 1u : 0u;
                    S = fmaf(kW[j], float(min(a, 1u << 22)), S);
                }
                s_nz[ch] = uint8_t(rm);
                S *= kW[u];
                m = (rm ? (1u << u) : 0u) | (big << 8);
            }
            m |= __shfl_xor_sync(0xFFFFFFFFu, m, 1);
            m |= __shfl_xor_sync(0xFFFFFFFFu, m, 2);
            m |= __shfl_xor_sync(0xFFFFFFFFu, m, 4);
            S += __shfl_xor_sync(0xFFFFFFFFu, S, 1);
            S += __shfl_xor_sync(0xFFFFFFFFu, S, 2);
            S += __shfl_xor_sync(0xFFFFFFFFu, S, 4);
            // whole data unit exact-FP64 when F is not exact in float or the
            // sample magnitude (<= S) could leave the magic-rounding range
            const bool blk_big = (m & 0x100u) || S >= 2097152.f;
            if (act) {
                float* dst = s_F + ch * 8;
                if (!blk_big) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) dst[j] = __int_as_float(d[j] + kMagicBits) - kMagic;
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) dst[j] = __int_as_float(d[j]);
                }
                if (u == 0) {
                    const uint32_t blk = ch >> 3;
                    s_rows[blk] = uint8_t(m);
                    s_big[blk] = blk_big ? 1 : 0;
                    // |r32 - r64| <= 18u S (+ FP64's own ~1e-15 S), u = 2^-24
                    s_lim[blk] = 0.5f - (1.1e-6f * S + 2.0e-6f);
                }
            }
            // chroma index maps (pipeline.hpp:182-187), tile-local; Cb and Cr
            // share geometry (both 1x1 sampled, parser.hpp:209-212)
            if (ti.rgb) {
                const uint32_t pw = D.plane_w[1], ph = D.plane_h[1], W = D.width, H = D.height;
                const uint32_t cx0 = ti.mx0 * D.comp_h[1] * 8, cy0 = ti.my * D.comp_v[1] * 8;
                for (uint32_t x = tid; x < ti.cols; x += kK4Threads)
                    s_cmap[x] = uint16_t(min((ti.X0 + x) * pw / W, pw - 1) - cx0);
                if (tid < int(ti.rws)) s_rmap[tid] = uint8_t(min((ti.Y0 + tid) * ph / H, ph - 1) - cy0);
            }
        }
        __syncthreads();
        // 2. IDCT (transform.hpp:114-142): thread (data unit, column y)
        {
            const uint32_t blk = tid >> 3, y = tid & 7;
            const bool act = blk < nblk;
            const uint32_t rows = act ? s_rows[blk] : 0u;
            const uint32_t urows = __reduce_or_sync(0xFFFFFFFFu, rows);
            const bool big = act && s_big[blk];
            uint32_t out[8];
            const float* F = s_F + (act ? blk : 0) * 64;
            if (!big) {
                float bcol[8];
#pragma unroll
                for (int v = 0; v < 8; ++v) bcol[v] = s_b32[v * 8 + y];
                float acc[8];
#pragma unroll
                for (int x = 0; x < 8; ++x) acc[x] = 0.f;
#pragma unroll
                for (int uu = 0; uu < 8; ++uu) {
                    if (urows & (1u << uu)) {
                        const float4 f0 = *reinterpret_cast<const float4*>(F + uu * 8);
                        const float4 f1 = *reinterpret_cast<const float4*>(F + uu * 8 + 4);
                        float tu = bcol[0] * f0.x;
                        tu = fmaf(bcol[1], f0.y, tu);
                        tu = fmaf(bcol[2], f0.z, tu);
                        tu = fmaf(bcol[3], f0.w, tu);
                        tu = fmaf(bcol[4], f1.x, tu);
                        tu = fmaf(bcol[5], f1.y, tu);
                        tu = fmaf(bcol[6], f1.z, tu);
                        tu = fmaf(bcol[7], f1.w, tu);
                        const float4 b0 = *reinterpret_cast<const float4*>(s_b32 + uu * 8);
                        const float4 b1 = *reinterpret_cast<const float4*>(s_b32 + uu * 8 + 4);
                        acc[0] = fmaf(b0.x, tu, acc[0]);
                        acc[1] = fmaf(b0.y, tu, acc[1]);
                        acc[2] = fmaf(b0.z, tu, acc[2]);
                        acc[3] = fmaf(b0.w, tu, acc[3]);
                        acc[4] = fmaf(b1.x, tu, acc[4]);
                        acc[5] = fmaf(b1.y, tu, acc[5]);
                        acc[6] = fmaf(b1.z, tu, acc[6]);
                        acc[7] = fmaf(b1.w, tu, acc[7]);
                    }
                }
                const float lim = act ? s_lim[blk] : 0.5f;
                uint32_t unsafe = 0;
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                    const float v = acc[x] + kMagic;
                    const float dd = acc[x] - (v - kMagic);
                    if (fabsf(dd) > lim) unsafe |= 1u << x;
                    out[x] = uint32_t(__float_as_int(v) - kMagicBits + 128);
                }
                if (unsafe) {
#pragma unroll
                    for (int x = 0; x < 8; ++x)
                        if (unsafe & (1u << x))
                            out[x] = uint32_t(idct_sample_fp64(F, false, rows, s_nz + blk * 8, s_b64, x, int(y)));
                }
            } else {
#pragma unroll
                for (int x = 0; x < 8; ++x)
                    out[x] = uint32_t(idct_sample_fp64(F, true, rows, s_nz + blk * 8, s_b64, x, int(y)));
            }
            if (act) {
                const uint32_t slot = blk % dpm, mm = blk / dpm;
                const uint32_t comp = uint32_t(D.du_comp >> (4 * slot)) & 15u;
                const uint32_t kk = uint32_t(D.du_kslot >> (4 * slot)) & 15u;
                const uint32_t chh = D.comp_h[comp];
                const uint32_t bx = kk % chh, by = kk / chh;
                const uint32_t ps = comp == 0 ? ti.pst[0] : (comp == 1 ? ti.pst[1] : ti.pst[2]);
                const uint32_t po = comp == 0 ? ti.poff[0] : (comp == 1 ? ti.poff[1] : ti.poff[2]);
                uint8_t* pl = s_pl + po + (by * 8) * ps + (mm * chh + bx) * 8 + y;
                const uint32_t lo = pack4_sat(int(out[0]), int(out[1]), int(out[2]), int(out[3]));
                const uint32_t hi = pack4_sat(int(out[4]), int(out[5]), int(out[6]), int(out[7]));
#pragma unroll
                for (int x = 0; x < 4; ++x) pl[x * ps] = uint8_t(lo >> (8 * x));
#pragma unroll
                for (int x = 0; x < 4; ++x) pl[(x + 4) * ps] = uint8_t(hi >> (8 * x));
            }
        }
        __syncthreads();
        // 3. output
        const uint32_t cols = ti.cols, rws = ti.rws, W = D.width;
        if (ti.rgb) {
            // thread = 4 pixels of one row (or of a row pair sharing a chroma
            // row for 4:2:0); chroma offsets computed inline per chroma sample
            const bool pair = D.v_max == 2;
            const uint32_t nrow = pair ? (rws + 1) >> 1 : rws;
            const uint32_t groups = (cols + 3) >> 2;
            const uint32_t gsh = 32 - __clz(max(groups, 1u) - 1);  // groups rounded up to 2^gsh
            uint8_t* obase = P.out + D.out_off;
            const bool aligned = ((W & 3) == 0) && ((D.out_off & 3) == 0);
            const uint8_t* ybase = s_pl + ti.poff[0];
            const uint8_t* cbbase = s_pl + ti.poff[1];
            const uint8_t* crbase = s_pl + ti.poff[2];
            const uint32_t pst0 = ti.pst[0], pst1 = ti.pst[1];
            for (uint32_t itg = tid; itg < (nrow << gsh); itg += kK4Threads) {
                const uint32_t j = itg >> gsh, gxi = itg & ((1u << gsh) - 1);
                if (gxi >= groups) continue;
                const uint32_t gx = gxi * 4;
                const uint32_t npx = min(4u, cols - gx);
                const uint2 cm = *reinterpret_cast<const uint2*>(s_cmap + gx);
                const uint32_t cx[4] = {cm.x & 0xFFFFu, cm.x >> 16, cm.y & 0xFFFFu, cm.y >> 16};
                const uint32_t r0 = pair ? 2 * j : j;
                uint32_t crow = s_rmap[r0];
                const uint8_t* cbrow = cbbase + crow * pst1;
                const uint8_t* crrow = crbase + crow * pst1;
                uint32_t w[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t c = q < int(npx) ? cx[q] : cx[0];
                    if (q > 0 && c == cx[q - 1])
                        w[q] = w[q - 1];
                    else
                        w[q] = chroma_word2(cbrow[c], crrow[c]);
                }
                const bool fast = npx == 4 && aligned;
                emit_rgb4(obase + (uint64_t(ti.Y0 + r0) * W + ti.X0 + gx) * 3, fast, npx,
                          *reinterpret_cast<const uint32_t*>(ybase + r0 * pst0 + gx), w, cbrow, crrow, cx);
                if (pair && r0 + 1 < rws) {
                    const uint32_t crow1 = s_rmap[r0 + 1];
                    if (crow1 != crow) {
                        crow = crow1;
                        cbrow = cbbase + crow * pst1;
                        crrow = crbase + crow * pst1;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint32_t c = q < int(npx) ? cx[q] : cx[0];
                            if (q > 0 && c == cx[q - 1])
                                w[q] = w[q - 1];
                            else
                                w[q] = chroma_word2(cbrow[c], crrow[c]);
                        }
                    }
                    emit_rgb4(obase + (uint64_t(ti.Y0 + r0 + 1) * W + ti.X0 + gx) * 3, fast, npx,
                              *reinterpret_cast<const uint32_t*>(ybase + (r0 + 1) * pst0 + gx), w, cbrow, crrow,
                              cx);
                }
            }
        } else {
            // planes (extract_planes, transform.hpp:165-211) — or the Y plane
            // only for grayscale output / single-component images
            const uint32_t nplanes = (D.out_mode == 0) ? D.ncomp : 1;
            const uint32_t MT = D.mcus_per_tile;
            uint64_t plane_base = D.out_off;
#pragma unroll
            for (uint32_t c = 0; c < 3; ++c) {
                if (c >= nplanes) break;
                const uint32_t pw = D.plane_w[c], ph = D.plane_h[c];
                const uint32_t cx0 = ti.mx0 * D.comp_h[c] * 8, cy0 = ti.my * D.comp_v[c] * 8;
                const uint32_t ccols = cx0 < pw ? min(ti.pw_t[c] * ti.nm / MT, pw - cx0) : 0;
                const uint32_t crows = cy0 < ph ? min(D.comp_v[c] * 8, ph - cy0) : 0;
                for (uint32_t e = tid; e < crows * ccols; e += kK4Threads) {
                    const uint32_t r = e / ccols, x = e % ccols;
                    P.out[plane_base + uint64_t(cy0 + r) * pw + cx0 + x] = s_pl[ti.poff[c] + r * ti.pst[c] + x];
                }
                plane_base += uint64_t(pw) * ph;
            }
        }
    }
}

// ============================== K5: colour stage of host-provided planes ====
// upsample_and_convert (pipeline.hpp:167-201) for the standalone C-ABI call;
// the decode path fuses this into K4.
__global__ void k5_color(const uint8_t* y, const uint8_t* cb, const uint8_t* cr, uint32_t W, uint32_t H,
                         uint32_t pw0, uint32_t pw1, uint32_t ph1, uint32_t pw2, uint32_t ph2, uint8_t* out) {
    const uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= uint64_t(W) * H) return;
    const uint32_t x = uint32_t(idx % W), yy = uint32_t(idx / W);
    const uint32_t sx1 = uint32_t(min64(uint64_t(x) * pw1 / W, pw1 - 1));
    const uint32_t sy1 = uint32_t(min64(uint64_t(yy) * ph1 / H, ph1 - 1));
    const uint32_t sx2 = uint32_t(min64(uint64_t(x) * pw2 / W, pw2 - 1));
    const uint32_t sy2 = uint32_t(min64(uint64_t(yy) * ph2 / H, ph2 - 1));
    const double Yd = double(y[uint64_t(yy) * pw0 + x]);
    const int c_b = int(cb[uint64_t(sy1) * pw1 + sx1]) - 128;
    const int c_r = int(cr[uint64_t(sy2) * pw2 + sx2]) - 128;
    out[idx * 3 + 0] = uint8_t(clamp_u8(lround_away(__dadd_rn(Yd, __dmul_rn(1.402, double(c_r))))));
    out[idx * 3 + 1] = uint8_t(clamp_u8(lround_away(
        __dsub_rn(__dsub_rn(Yd, __dmul_rn(0.344136, double(c_b))), __dmul_rn(0.714136, double(c_r))))));
    out[idx * 3 + 2] = uint8_t(clamp_u8(lround_away(__dadd_rn(Yd, __dmul_rn(1.772, double(c_b))))));
}

}  // namespace

void launch_k5_color(const uint8_t* y, const uint8_t* cb, const uint8_t* cr, uint32_t W, uint32_t H,
                     uint32_t pw0, uint32_t pw1, uint32_t ph1, uint32_t pw2, uint32_t ph2, uint8_t* out,
                     void* stream) {
    const uint64_t n = uint64_t(W) * H;
    if (!n) return;
    k5_color<<<unsigned((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(y, cb, cr, W, H, pw0, pw1, ph1, pw2,
                                                                          ph2, out);
}

// ------------------------------------------------------------ launchers --
void launch_k0_unstuff(const Params& p, void* stream) {
    if (p.k0_tiles) k0_unstuff<<<p.k0_tiles, kK0Threads, 0, (cudaStream_t)stream>>>(p);
}
void launch_k1_sync(const Params& p, void* stream) {
    if (p.k1_ctas) k1_sync<<<p.k1_ctas, kK1Threads, 0, (cudaStream_t)stream>>>(p);
}
void launch_k1c_fixup(const Params& p, void* stream) {
    if (p.k1_ctas > 1) k1c_fixup<<<1, 1024, 0, (cudaStream_t)stream>>>(p);
}
void launch_k2_scan(const Params& p, void* stream) {
    if (p.k2_tiles) k2_scan<<<p.k2_tiles, kK2Threads, 0, (cudaStream_t)stream>>>(p);
}
void launch_k3_write(const Params& p, void* stream) {
    if (p.total_subs)
        k3_write<<<unsigned((p.total_subs + kK3Threads - 1) / kK3Threads), kK3Threads, 0,
                   (cudaStream_t)stream>>>(p);
}
void launch_k4_transform(const Params& p, void* stream) {
    if (!p.k4_tiles) return;
    static int grid_cap = 0;
    if (!grid_cap) {
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k4_transform, kK4Threads, 0);
        grid_cap = std::max(1, sms * std::max(per_sm, 1));
    }
    const unsigned grid = unsigned(std::min<uint64_t>(p.k4_tiles, uint64_t(grid_cap)));
    k4_transform<<<grid, kK4Threads, 0, (cudaStream_t)stream>>>(p);
}

}  // namespace pjg
