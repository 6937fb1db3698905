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
// One CTA per tile of `mcus_per_tile` MCUs of one MCU row (<= 48 data units).
//  1. load + dequantise coefficients into smem (int32, raster)
//  2. IDCT: thread per (data unit, column y); exact FP64 in the reference's
//     summation order; samples into per-component smem planes
//  3. crop + chroma replication + FP64 YCbCr->RGB, stores to the output
__global__ void __launch_bounds__(kK4Threads) k4_transform(Params P) {
    __shared__ __align__(16) int32_t s_F[kK4MaxBlocks * 64];
    __shared__ __align__(16) uint8_t s_pl[kK4MaxBlocks * 64];
    __shared__ double s_basis[64];
    __shared__ uint8_t s_rows[kK4MaxBlocks];
    __shared__ uint16_t s_cmap[2][384];
    __shared__ uint8_t s_rmap[2][16];

    const int tid = threadIdx.x;
    const uint32_t t = blockIdx.x;
    const uint32_t k = find_seg(P.tile_first, P.n_img, t);
    if (P.ist[k].status != 0) return;
    const ImgDesc& D = P.img[k];
    const uint32_t lt = t - P.tile_first[k];
    const uint32_t my = lt / D.tiles_x, tx = lt % D.tiles_x;
    const uint32_t MT = D.mcus_per_tile;
    const uint32_t mx0 = tx * MT;
    const uint32_t nm = min(MT, D.mcus_x - mx0);
    const uint32_t dpm = D.dpm;
    const uint32_t nblk = nm * dpm;
    const uint64_t du0 = D.du_first + (uint64_t(my) * D.mcus_x + mx0) * dpm;

    if (tid < 64) s_basis[tid] = P.basis[tid];
    // 1. load 8 coefficients per 16-byte chunk, dequantise with the raster table
    const int4* src = reinterpret_cast<const int4*>(P.coef + du0 * 64);
    for (uint32_t ch = tid; ch < nblk * 8; ch += kK4Threads) {
        const uint32_t blk = ch >> 3, slot = blk % dpm;
        const uint32_t comp = uint32_t(D.du_comp >> (4 * slot)) & 15u;
        const uint16_t* q = P.quant_raster + 64u * D.q_tab[comp] + (ch & 7) * 8;
        int4 v = __ldcs(src + ch);
        const int16_t* c16 = reinterpret_cast<const int16_t*>(&v);
        int32_t* d = s_F + ch * 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) d[j] = int32_t(c16[j]) * int32_t(__ldg(q + j));
    }
    __syncthreads();
    if (tid < int(nblk)) {
        uint32_t m = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int4* r = reinterpret_cast<const int4*>(s_F + tid * 64 + u * 8);
            int4 a = r[0], b = r[1];
            if ((a.x | a.y | a.z | a.w | b.x | b.y | b.z | b.w) != 0) m |= 1u << u;
        }
        s_rows[tid] = uint8_t(m);
    }
    // plane geometry inside the tile
    uint32_t pw_t[3], poff[3];
    {
        uint32_t acc = 0;
        for (uint32_t c = 0; c < 3; ++c) {
            pw_t[c] = c < D.ncomp ? MT * D.comp_h[c] * 8 : 0;
            poff[c] = acc;
            acc += c < D.ncomp ? pw_t[c] * D.comp_v[c] * 8 : 0;
        }
    }
    __syncthreads();
    // 2. IDCT (transform.hpp:114-142): column pass tmp[u][y] = sum_v basis[v][y]*F[u][v],
    // row pass out[x][y] = sum_u basis[u][x]*tmp[u][y], both ascending, zero terms skipped.
    for (uint32_t it = tid; it < nblk * 8; it += kK4Threads) {
        const uint32_t blk = it >> 3, y = it & 7;
        const uint32_t rows = s_rows[blk];
        const int32_t* F = s_F + blk * 64;
        double tmp[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            double s = 0.0;
            if (rows & (1u << u)) {
#pragma unroll
                for (int v = 0; v < 8; ++v) {
                    int32_t f = F[u * 8 + v];
                    if (f != 0) s = __dadd_rn(s, __dmul_rn(s_basis[v * 8 + y], double(f)));
                }
            }
            tmp[u] = s;
        }
        const uint32_t slot = blk % dpm, m = blk / dpm;
        const uint32_t comp = uint32_t(D.du_comp >> (4 * slot)) & 15u;
        const uint32_t kk = uint32_t(D.du_kslot >> (4 * slot)) & 15u;
        const uint32_t ch = D.comp_h[comp];
        const uint32_t bx = kk % ch, by = kk / ch;
        uint8_t* pl = s_pl + poff[comp] + (by * 8) * pw_t[comp] + (m * ch + bx) * 8 + y;
#pragma unroll
        for (int x = 0; x < 8; ++x) {
            double s = 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (rows & (1u << u)) s = __dadd_rn(s, __dmul_rn(s_basis[u * 8 + x], tmp[u]));
            pl[x * pw_t[comp]] = uint8_t(clamp_u8(lround_away(s) + 128));
        }
    }
    // 3. output
    const uint32_t mcu_w = 8 * D.h_max, mcu_h = 8 * D.v_max;
    const uint32_t X0 = mx0 * mcu_w, Y0 = my * mcu_h;
    const uint32_t W = D.width, H = D.height;
    const uint32_t cols = min(nm * mcu_w, W - X0), rws = min(mcu_h, H - Y0);
    const bool rgb = D.out_mode == 1 && D.ncomp == 3;
    if (rgb) {
        // chroma sample index maps (pipeline.hpp:182-187), tile-local
        for (uint32_t c = 1; c < 3; ++c) {
            const uint32_t pw = D.plane_w[c], ph = D.plane_h[c];
            const uint32_t cx0 = mx0 * D.comp_h[c] * 8, cy0 = my * D.comp_v[c] * 8;
            for (uint32_t x = tid; x < cols; x += kK4Threads) {
                uint32_t sx = uint32_t(min64(uint64_t(X0 + x) * pw / W, pw - 1));
                s_cmap[c - 1][x] = uint16_t(sx - cx0);
            }
            if (tid < int(rws)) {
                uint32_t sy = uint32_t(min64(uint64_t(Y0 + tid) * ph / H, ph - 1));
                s_rmap[c - 1][tid] = uint8_t(sy - cy0);
            }
        }
    }
    __syncthreads();
    if (rgb) {
        // FP64 YCbCr->RGB exactly as pipeline.hpp:190-197
        const uint32_t groups = (cols + 3) >> 2;
        uint8_t* obase = P.out + D.out_off;
        for (uint32_t it = tid; it < rws * groups; it += kK4Threads) {
            const uint32_t r = it / groups, gx = (it % groups) * 4;
            const uint32_t npx = min(4u, cols - gx);
            uint32_t pk[3] = {0, 0, 0};
            const uint8_t* yrow = s_pl + poff[0] + r * pw_t[0];
            const uint8_t* cbrow = s_pl + poff[1] + s_rmap[0][r] * pw_t[1];
            const uint8_t* crrow = s_pl + poff[2] + s_rmap[1][r] * pw_t[2];
            uint8_t px[12];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (q < int(npx)) {
                    const uint32_t x = gx + q;
                    const double Yd = double(yrow[x]);
                    const int cb = int(cbrow[s_cmap[0][x]]) - 128;
                    const int cr = int(crrow[s_cmap[1][x]]) - 128;
                    const int R = lround_away(__dadd_rn(Yd, __dmul_rn(1.402, double(cr))));
                    const int G = lround_away(__dsub_rn(__dsub_rn(Yd, __dmul_rn(0.344136, double(cb))),
                                                        __dmul_rn(0.714136, double(cr))));
                    const int B = lround_away(__dadd_rn(Yd, __dmul_rn(1.772, double(cb))));
                    px[3 * q + 0] = uint8_t(clamp_u8(R));
                    px[3 * q + 1] = uint8_t(clamp_u8(G));
                    px[3 * q + 2] = uint8_t(clamp_u8(B));
                }
            }
            uint8_t* dst = obase + (uint64_t(Y0 + r) * W + X0 + gx) * 3;
            if (npx == 4 && (reinterpret_cast<uintptr_t>(dst) & 3) == 0) {
#pragma unroll
                for (int w = 0; w < 3; ++w)
                    pk[w] = uint32_t(px[4 * w]) | (uint32_t(px[4 * w + 1]) << 8) |
                            (uint32_t(px[4 * w + 2]) << 16) | (uint32_t(px[4 * w + 3]) << 24);
                uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
                d32[0] = pk[0];
                d32[1] = pk[1];
                d32[2] = pk[2];
            } else {
                for (uint32_t q = 0; q < npx * 3; ++q) dst[q] = px[q];
            }
        }
    } else {
        // planes (extract_planes, transform.hpp:165-211) — or the Y plane only
        // for grayscale output / single-component images
        const uint32_t nplanes = (D.out_mode == 0) ? D.ncomp : 1;
        uint64_t plane_base = D.out_off;
        for (uint32_t c = 0; c < nplanes; ++c) {
            const uint32_t pw = D.plane_w[c], ph = D.plane_h[c];
            const uint32_t cx0 = mx0 * D.comp_h[c] * 8, cy0 = my * D.comp_v[c] * 8;
            const uint32_t ccols = cx0 < pw ? min(pw_t[c] * nm / MT, pw - cx0) : 0;
            const uint32_t crows = cy0 < ph ? min(D.comp_v[c] * 8, ph - cy0) : 0;
            for (uint32_t it = tid; it < crows * ccols; it += kK4Threads) {
                const uint32_t r = it / ccols, x = it % ccols;
                P.out[plane_base + uint64_t(cy0 + r) * pw + cx0 + x] = s_pl[poff[c] + r * pw_t[c] + x];
            }
            plane_base += uint64_t(pw) * ph;
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
    if (p.k4_tiles) k4_transform<<<p.k4_tiles, kK4Threads, 0, (cudaStream_t)stream>>>(p);
}

}  // namespace pjg
