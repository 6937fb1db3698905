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
#include <type_traits>
#include <stdint.h>

#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "pjg_internal.h"

namespace pjg {
namespace {

constexpr uint32_t kInf32 = 0xFFFFFFFFu;

// zig-zag index -> COLUMN-MAJOR block index v*8 + u (F[u][v] at raster u*8+v):
// the coefficient buffer holds each data unit transposed so K4's IDCT lanes
// read one frequency column per 16-byte row (pjg_internal.h kCoefColMajor).
__device__ __constant__ uint8_t c_zz2c[64] = {
    0,  8,  1,  2,  9,  16, 24, 17, 10, 3,  4,  11, 18, 25, 32, 40,
    33, 26, 19, 12, 5,  6,  13, 20, 27, 34, 41, 48, 56, 49, 42, 35,
    28, 21, 14, 7,  15, 22, 29, 36, 43, 50, 57, 58, 51, 44, 37, 30,
    23, 31, 38, 45, 52, 59, 60, 53, 46, 39, 47, 54, 61, 62, 55, 63};

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
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void spin_pause() { __nanosleep(32); }
// griddepcontrol.wait: the predecessor grid (programmatic launch) has completed
// and its memory is visible; a no-op for ordinary launches
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

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

// image holding global subsequence g: sub_img[g >> 7] and sub_img[(g >> 7) + 1]
// (host-built) bracket it, so the search is over a handful of images at most
__device__ __forceinline__ uint32_t find_img(const Params& P, uint64_t g) {
    const uint64_t c = g >> kSubImgShift;
    uint32_t lo = __ldg(P.sub_img + c), hi = __ldg(P.sub_img + c + 1) + 1;
    if (hi > P.n_img) hi = P.n_img;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(P.sub_first + mid) <= g)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

// Where image-local subsequence i lives.  Without restart intervals the image
// is one segment partitioned like the reference (N = ceil(L / sb),
// parallel_decode.hpp:31-62).  With them (extension), each interval m is its
// own segment [x_m, x_{m+1}) of unstuffed bits, partitioned from its first
// bit, starting in the known state c = 0, z = 0 with zero DC predictors;
// Params::segs (built by K0b) holds the per-interval bit and subsequence
// offsets.  Returns false for subsequences past the image's last one.
struct SubInfo {
    uint64_t lo, hi;          // this subsequence's bits [lo, hi)
    uint64_t seg_lo, seg_hi;  // its segment's bits
    uint64_t j;               // index within the segment (0: known start state)
    uint64_t seg_sub0, seg_sub1;  // the segment's image-local subsequences
    uint32_t m;               // segment (restart interval)
};
template <bool DRI = true>
__device__ __forceinline__ bool sub_info(const Params& P, const ImgDesc& D, uint64_t L, uint64_t i, SubInfo& si) {
    if (!DRI || D.n_int <= 1) {
        const uint64_t N = (L + P.sb - 1) / P.sb;
        si.m = 0;
        si.seg_lo = 0;
        si.seg_hi = L;
        si.seg_sub0 = 0;
        si.seg_sub1 = N;
        si.j = i;
        if (i >= N) return false;
    } else {
        const uint2* sg = P.segs + D.seg_first;
        if (i >= sg[D.n_int].y) return false;
        uint32_t lo = 0, hi = D.n_int;  // largest m with sg[m].y <= i
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (sg[mid].y <= i)
                lo = mid;
            else
                hi = mid;
        }
        si.m = lo;
        si.seg_lo = sg[lo].x;
        si.seg_hi = sg[lo + 1].x;
        si.seg_sub0 = sg[lo].y;
        si.seg_sub1 = sg[lo + 1].y;
        si.j = i - si.seg_sub0;
    }
    si.lo = si.seg_lo + si.j * P.sb;
    si.hi = min64(si.lo + P.sb, si.seg_hi);
    return true;
}
// end bit of subsequence i of the same segment
__device__ __forceinline__ uint64_t seg_end_bit(const SubInfo& si, uint64_t sb, uint64_t i) {
    return min64(si.seg_lo + (i - si.seg_sub0 + 1) * sb, si.seg_hi);
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

// 0x80 in every zero byte of x (exact, no borrow between bytes)
__device__ __forceinline__ uint32_t eq0_bytes(uint32_t x) {
    return ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;
}
// the four 0x80 byte flags of x as a 4-bit mask (bit i = byte i)
__device__ __forceinline__ uint32_t movemask4(uint32_t x) { return (x * 0x00204081u) >> 28; }

// ========================================================= K0: unstuff ====
// One CTA per 4 KB tile of raw scan bytes.  Per tile: number of stuffed zero
// bytes (a 0x00 right after 0xFF) and the first marker position (0xFF not
// followed by 0x00; 0xFF as the last byte ends the scan too).  A segmented
// decoupled lookback over the image's tiles gives each tile its exclusive
// (removed, first-marker) prefix; kept bytes are then compacted into ubuf at
// the same image offset.  The tile holding the first marker fixes the
// unstuffed length U and the per-image error (EmptyScan / RST).
// Tiles are windows of 512 x BPT bytes aligned to the 16-byte grid of the raw
// buffer (the image's first window starts at raw_off & ~15); thread t owns
// bytes [BPT t, BPT t + BPT) of its window (BPT / 16 vector loads).  Batches of
// large scans use 32 KB tiles (BPT 64: more bytes in flight per CTA, the
// per-tile ticket / lookback / scan amortised), batches of small files 8 KB
// tiles (BPT 16: a file of ~16 KB should not occupy a half-empty 32 KB tile).  The compacted bytes are staged in shared memory on the
// destination's 16-byte grid and leave as full 16-byte stores (only the two
// edge chunks a tile shares with its neighbours go byte-wise).
template <bool DRI, int BPT>
__global__ void __launch_bounds__(kK0Threads) k0_unstuff(Params P) {
    pdl_wait();
    constexpr int kTile = kK0Threads * BPT;
    extern __shared__ __align__(16) uint8_t k0_dyn[];
    uint8_t* s_b = k0_dyn;                 // s_b[16 + i] = raw byte win0 + i; [15] before, [16 + tile] after
    uint8_t* s_o = k0_dyn + kTile + 32;  // compacted bytes on the destination's 16-byte grid
    __shared__ unsigned long long s_cnt[kK0Threads / 32];  // per warp: removed | RST << 32
    __shared__ uint32_t s_mk[kK0Threads / 32];
    __shared__ uint32_t s_tile, s_excl_cnt, s_excl_mk, s_tile_cnt, s_tile_mk, s_excl_rc;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) s_tile = atomicAdd(&P.counters[kTicketK0], 1u);
    __syncthreads();
    const uint32_t t = s_tile;
    const uint32_t k = __ldg(P.k0_img + t);
    const uint32_t lt = t - P.k0_first[k];
    const ImgDesc& D = P.img[k];
    const uint64_t raw_len = D.raw_len;
    const uint64_t a = D.raw_off, e = a + raw_len;  // the image's bytes [a, e) in the raw buffer
    const uint64_t win0 = (a & ~15ull) + uint64_t(lt) * kTile;
    const uint64_t g_first = max(win0, a);            // first image byte in this window
    // restart intervals (extension): RSTn markers inside the scan are removed
    // like stuffed zeros and their unstuffed positions recorded; without them a
    // RST marker ends the scan and is UnsupportedFeature (parser.hpp:249-250)
    const bool dri = DRI && D.n_int > 1;

    const uint32_t b0 = tid * BPT;
    const uint64_t gb = win0 + b0;
#pragma unroll
    for (int c = 0; c < BPT / 16; ++c) {
        const uint64_t g = gb + 16 * c;
        int4 v = make_int4(0, 0, 0, 0);
        if (g < e) v = __ldcs(reinterpret_cast<const int4*>(P.raw + g));
        reinterpret_cast<int4*>(s_b + 16 + b0)[c] = v;
    }
    if (tid == 0) s_b[15] = win0 > a ? P.raw[win0 - 1] : 0;
    if (tid == 1) s_b[16 + kTile] = win0 + kTile < e ? P.raw[win0 + kTile] : 0;
    __syncthreads();

    // this thread's 64 bytes, classified branch-free with SWAR byte compares
    // into 64-bit masks (bit i = byte i): a divergent per-byte loop would cost
    // every warp that holds a single 0xFF byte
    uint64_t inr = BPT == 64 ? ~0ull : ((1ull << BPT) - 1ull);  // bytes inside the image [a, e)
    if (gb < a) inr &= a - gb >= BPT ? 0ull : (~0ull << uint32_t(a - gb));
    if (gb + BPT > e) inr &= e <= gb ? 0ull : (~0ull >> uint32_t(64 - (e - gb)));
    uint32_t ws[BPT / 4];
#pragma unroll
    for (int c = 0; c < BPT / 16; ++c) {
        const uint4 w = reinterpret_cast<const uint4*>(s_b + 16 + b0)[c];
        ws[4 * c] = w.x, ws[4 * c + 1] = w.y, ws[4 * c + 2] = w.z, ws[4 * c + 3] = w.w;
    }
    uint64_t mFF = 0, m00 = 0, mR = 0;
#pragma unroll
    for (int q = 0; q < BPT / 4; ++q) {
        mFF |= uint64_t(movemask4(eq0_bytes(~ws[q]))) << (4 * q);
        m00 |= uint64_t(movemask4(eq0_bytes(ws[q]))) << (4 * q);
        if (DRI) mR |= uint64_t(movemask4(eq0_bytes((ws[q] ^ 0xD0D0D0D0u) & 0xF8F8F8F8u))) << (4 * q);
    }
    const uint8_t pb = s_b[15 + b0], nb = s_b[16 + b0 + BPT];  // bytes before / after the thread's bytes
    const uint64_t prevFF = ((mFF & inr) << 1) | ((gb > a && pb == 0xFF) ? 1ull : 0ull);  // prev in the image
    const uint64_t next00 = (m00 >> 1) | (nb == 0x00 ? (1ull << (BPT - 1)) : 0ull);
    const uint64_t nextR = (mR >> 1) | (((nb & 0xF8) == 0xD0) ? (1ull << (BPT - 1)) : 0ull);
    const uint64_t lastb = (e - 1 >= gb && e - 1 < gb + BPT) ? (1ull << uint32_t(e - 1 - gb)) : 0ull;
    const uint64_t rstFF = dri ? (mFF & nextR & ~lastb & inr) : 0ull;
    const uint64_t rstX = dri ? (mR & prevFF & inr) : 0ull;
    const uint64_t remv = ((m00 & prevFF) | rstFF | rstX) & inr;  // removed bytes
    const uint64_t mark = mFF & inr & ~rstFF & (~next00 | lastb);   // markers ending the scan
    const uint64_t cr = uint64_t(__popcll(remv)) | (uint64_t(__popcll(rstFF)) << 32);
    const uint32_t mk = mark ? uint32_t(gb - a) + (__ffsll(mark) - 1) : kInf32;

    // block reduce (sum, min)
    unsigned long long wc = cr;
    uint32_t wm = mk;
    for (int o = 16; o; o >>= 1) {
        wc += __shfl_xor_sync(0xFFFFFFFFu, wc, o);
        wm = min(wm, __shfl_xor_sync(0xFFFFFFFFu, wm, o));
    }
    if (lane == 0) {
        s_cnt[warp] = wc;
        s_mk[warp] = wm;
    }
    __syncthreads();
    if (warp == 0) {
        // tile totals, then a warp-parallel decoupled lookback (32 predecessors
        // per step), segmented at the image's first tile:
        // agg [0] aggregate (mk << 32 | removed), [1] aggregate RST count, [2], [3] inclusive
        unsigned long long tcr = 0;
        uint32_t tm = kInf32;
        for (int w = 0; w < kK0Threads / 32; ++w) {
            tcr += s_cnt[w];
            tm = min(tm, s_mk[w]);
        }
        const uint32_t tc = uint32_t(tcr), trc = uint32_t(tcr >> 32);
        uint64_t* agg = P.k0_agg + 4ull * t;
        uint32_t ec = 0, em = kInf32, erc = 0;
        if (lt == 0) {
            if (lane == 0) {
                agg[2] = (uint64_t(tm) << 32) | tc;
                agg[3] = trc;
                st_release(P.k0_flag + t, (P.epoch << 2) | 2u);
            }
        } else {
            if (lane == 0) {
                agg[0] = (uint64_t(tm) << 32) | tc;
                agg[1] = trc;
                st_release(P.k0_flag + t, (P.epoch << 2) | 1u);
            }
            const int64_t first_t = int64_t(P.k0_first[k]);
            int64_t base = int64_t(t) - 1;
            while (true) {
                const int64_t pr = base - lane;  // lane 0: nearest predecessor
                uint32_t f = 2u;                 // before the image: an empty inclusive prefix
                if (pr >= first_t) {
                    f = ld_acquire(P.k0_flag + pr);
                    while ((f >> 2) != P.epoch) {
                        spin_pause();
                        f = ld_acquire(P.k0_flag + pr);
                    }
                }
                const uint32_t incl = __ballot_sync(0xFFFFFFFFu, (f & 3u) == 2u);
                const int lim = incl ? __ffs(incl) - 1 : 31;
                uint32_t c = 0, m = kInf32, r = 0;
                if (lane <= lim && pr >= first_t) {
                    const uint64_t* src = P.k0_agg + 4ull * pr + ((f & 3u) == 2u ? 2 : 0);
                    const uint64_t v = __ldcg(src);
                    c = uint32_t(v);
                    m = uint32_t(v >> 32);
                    r = uint32_t(__ldcg(src + 1));
                }
                ec += __reduce_add_sync(0xFFFFFFFFu, c);
                em = min(em, __reduce_min_sync(0xFFFFFFFFu, m));
                erc += __reduce_add_sync(0xFFFFFFFFu, r);
                if (incl) break;
                base -= 32;
            }
            if (lane == 0) {
                agg[2] = (uint64_t(min(em, tm)) << 32) | (ec + tc);
                agg[3] = erc + trc;
                st_release(P.k0_flag + t, (P.epoch << 2) | 2u);
            }
        }
        if (lane == 0) {
            s_tile_cnt = tc;
            s_tile_mk = tm;
            s_excl_cnt = ec;
            s_excl_mk = em;
            s_excl_rc = erc;
        }
    }
    __syncthreads();
    // exclusive scan of per-thread (removed | RST << 32) counts
    unsigned long long inc = cr;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= o) inc += v;
    }
    __syncthreads();
    if (lane == 31) s_cnt[warp] = inc;
    __syncthreads();
    unsigned long long wtot = lane < kK0Threads / 32 ? s_cnt[lane] : 0ull;
    unsigned long long wsc = wtot;
    for (int o = 1; o < kK0Threads / 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(0xFFFFFFFFu, wsc, o);
        if (lane >= o) wsc += v;
    }
    const unsigned long long before_cr = __shfl_sync(0xFFFFFFFFu, wsc - wtot, warp) + inc - cr;
    const uint32_t removed = s_excl_cnt + uint32_t(before_cr);        // removed before this thread's bytes
    const uint32_t rst_before = s_excl_rc + uint32_t(before_cr >> 32);  // RST markers before them

    // kept byte at image index j goes to image index j - removed; this tile's
    // kept bytes form [dst_lo, dst_lo + kept) in raw-buffer coordinates
    const uint64_t dst_lo = g_first - s_excl_cnt;
    const uint64_t dst_al = dst_lo & ~15ull;
    const uint32_t first_mk = s_excl_mk == kInf32 ? s_tile_mk : kInf32;  // the image's scan end
    const uint64_t keep = inr & ~remv;
#pragma unroll
    for (int c = 0; c < BPT / 16; ++c) {
        // kept bytes of 16-byte chunk c move left by the removed bytes before them
        const uint32_t keep16 = uint32_t(keep >> (16 * c)) & 0xFFFFu;
        const uint32_t remv16 = uint32_t(remv >> (16 * c)) & 0xFFFFu;
        const uint32_t rbefore = removed + uint32_t(__popcll(remv & ((1ull << (16 * c)) - 1ull)));
        const uint32_t off = uint32_t((gb + 16 * c - rbefore) - dst_al);
        uint8_t* o = s_o + off;
        const uint32_t* w = ws + 4 * c;
        if (keep16 == 0xFFFFu) {
            // 16 contiguous bytes: aligned words by funnel shifts, the two edge
            // words byte-wise (a neighbour owns their other bytes)
            const uint32_t r = off & 3u;
            uint32_t* o32 = reinterpret_cast<uint32_t*>(s_o + (off & ~3u));
            if (r == 0) {
                o32[0] = w[0], o32[1] = w[1], o32[2] = w[2], o32[3] = w[3];
            } else {
                const uint32_t sh = 8 * r;
                o32[1] = __funnelshift_l(w[0], w[1], sh);
                o32[2] = __funnelshift_l(w[1], w[2], sh);
                o32[3] = __funnelshift_l(w[2], w[3], sh);
                for (uint32_t i = 0; i < 4 - r; ++i) o[i] = uint8_t(w[0] >> (8 * i));
                for (uint32_t i = 0; i < r; ++i) o[16 - r + i] = uint8_t(w[3] >> (8 * (4 - r + i)));
            }
        } else if (keep16) {
            for (uint32_t m = keep16; m; m &= m - 1) {
                const uint32_t i = __ffs(m) - 1;
                o[i - __popc(remv16 & ((1u << i) - 1u))] = s_b[16 + b0 + 16 * c + i];
            }
        }
    }
    // rare events, off the branch-free path: the scan end and restart markers
    if (first_mk != kInf32 && first_mk - uint32_t(gb - a) < uint32_t(BPT) && (mark >> (first_mk - uint32_t(gb - a))) & 1ull) {
        // scan ends here (extract_scan, parser.hpp:241-254)
        const uint32_t i = first_mk - uint32_t(gb - a);
        const uint64_t j = first_mk;
        const uint64_t U = j - (removed + __popcll(remv & ((1ull << i) - 1ull)));
        ImgState* st = P.ist + k;
        st->bit_length = U * 8;
        const uint8_t nx = s_b[17 + b0 + i];
        const bool rst = (j + 1 < raw_len) && nx >= 0xD0 && nx <= 0xD7;
        if (rst)
            set_status(st, kUnsupportedFeature);
        else if (U == 0)
            set_status(st, kEmptyScan);
        else if (D.deferred)
            set_status(st, D.deferred);
    }
    if (DRI && rstFF) {
        // restart marker r: interval r + 1 starts at unstuffed byte j - removed;
        // markers past the scan end do not count
        const uint32_t end_mk = s_excl_mk != kInf32 ? s_excl_mk : s_tile_mk;
        for (uint64_t m = rstFF; m; m &= m - 1) {
            const uint32_t i = __ffsll(m) - 1;
            const uint64_t j = gb - a + i;
            const uint32_t r = rst_before + uint32_t(__popcll(rstFF & ((1ull << i) - 1ull)));
            if (j >= end_mk) continue;
            const uint8_t nx = s_b[17 + b0 + i];
            if (r + 1 >= D.n_int || (nx & 7u) != (r & 7u))
                set_status(P.ist + k, kConsistencyFailure);  // RST count / numbering vs DRI
            else
                P.segs[D.seg_first + r + 1].x =
                    uint32_t((j - (removed + __popcll(remv & ((1ull << i) - 1ull)))) * 8);
        }
    }
    __syncthreads();
    {
        const uint64_t dst_hi = dst_lo + (min64(e, win0 + kTile) - g_first) - s_tile_cnt;
        const uint32_t nchunks = uint32_t((dst_hi - dst_al + 15) >> 4);
        for (uint32_t q = tid; q < nchunks; q += kK0Threads) {
            const uint64_t G = dst_al + 16ull * q;
            if (G >= dst_lo && G + 16 <= dst_hi) {
                *reinterpret_cast<int4*>(P.ubuf + G) = reinterpret_cast<const int4*>(s_o)[q];
            } else {
                for (uint32_t x = 0; x < 16; ++x)
                    if (G + x >= dst_lo && G + x < dst_hi) P.ubuf[G + x] = s_o[16 * q + x];
            }
        }
    }
    // no marker anywhere: the scan runs to the end of the file
    const uint32_t last_tile = uint32_t(((a & 15ull) + raw_len + kTile - 1) / kTile) - 1;
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

// Small-file variant (8 KB tiles, 16 bytes per thread, 32-bit scan words):
// windows aligned to the 16-byte grid of the raw buffer (the
// image's first window starts at raw_off & ~15), so every thread moves its
// 16 bytes with one vector load, and the compacted bytes are staged in shared
// memory on the destination's 16-byte grid and leave as full 16-byte stores
// (only the two edge chunks a tile shares with its neighbours go byte-wise).
template <bool DRI>
__global__ void __launch_bounds__(kK0Threads) k0_unstuff_small(Params P) {
    pdl_wait();
    constexpr int kSmallTile = kK0Threads * 16;
    __shared__ uint32_t s_tile;
    // s_b[16 + i] = raw byte win0 + i; s_b[15] = byte before the window,
    // s_b[16 + kSmallTile] = byte after it
    __shared__ __align__(16) uint8_t s_b[kSmallTile + 32];
    __shared__ __align__(16) uint8_t s_o[kSmallTile + 32];
    __shared__ uint32_t s_cnt[kK0Threads / 32];
    __shared__ uint32_t s_mk[kK0Threads / 32];
    __shared__ uint32_t s_excl_cnt, s_excl_mk, s_tile_cnt, s_tile_mk, s_excl_rc;

    const int tid = threadIdx.x;
    if (tid == 0) s_tile = atomicAdd(&P.counters[kTicketK0], 1u);
    __syncthreads();
    const uint32_t t = s_tile;
    const uint32_t k = __ldg(P.k0_img + t);
    const uint32_t lt = t - P.k0_first[k];
    const ImgDesc& D = P.img[k];
    const uint64_t raw_len = D.raw_len;
    const uint64_t a = D.raw_off, e = a + raw_len;  // the image's bytes [a, e) in the raw buffer
    const uint64_t win0 = (a & ~15ull) + uint64_t(lt) * kSmallTile;
    const uint64_t g_first = max(win0, a);            // first image byte in this window
    // restart intervals (extension): RSTn markers inside the scan are removed
    // like stuffed zeros and their unstuffed positions recorded; without them a
    // RST marker ends the scan and is UnsupportedFeature (parser.hpp:249-250)
    const bool dri = DRI && D.n_int > 1;

    {
        const uint64_t g = win0 + 16u * tid;
        int4 v = make_int4(0, 0, 0, 0);
        if (g < e) v = __ldcs(reinterpret_cast<const int4*>(P.raw + g));
        reinterpret_cast<int4*>(s_b + 16)[tid] = v;
        if (tid == 0) s_b[15] = win0 > a ? P.raw[win0 - 1] : 0;
        if (tid == 1) s_b[16 + kSmallTile] = win0 + kSmallTile < e ? P.raw[win0 + kSmallTile] : 0;
    }
    __syncthreads();

    // this thread's 16 bytes (raw bytes win0 + b0 + i), classified branch-free
    // with SWAR byte compares into 16-bit masks (bit i = byte i): a divergent
    // per-byte loop would cost every warp that holds a single 0xFF byte
    const uint32_t b0 = tid * 16;
    const uint64_t gb = win0 + b0;
    uint32_t inr = 0xFFFFu;  // bytes inside the image [a, e)
    if (gb < a) inr &= a - gb >= 16 ? 0u : (0xFFFFu << uint32_t(a - gb)) & 0xFFFFu;
    if (gb + 16 > e) inr &= e <= gb ? 0u : 0xFFFFu >> uint32_t(16 - (e - gb));
    uint32_t mFF, m00, mR;
    {
        const uint4 w = reinterpret_cast<const uint4*>(s_b + 16)[tid];
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
        mFF = m00 = mR = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            mFF |= movemask4(eq0_bytes(~ws[q])) << (4 * q);
            m00 |= movemask4(eq0_bytes(ws[q])) << (4 * q);
            if (DRI) mR |= movemask4(eq0_bytes((ws[q] ^ 0xD0D0D0D0u) & 0xF8F8F8F8u)) << (4 * q);
        }
    }
    const uint8_t pb = s_b[15 + b0], nb = s_b[32 + b0];  // bytes before / after the chunk
    const uint32_t prevFF = (((mFF & inr) << 1) | ((gb > a && pb == 0xFF) ? 1u : 0u)) & 0xFFFFu;  // prev in the image
    const uint32_t next00 = (m00 >> 1) | (nb == 0x00 ? 0x8000u : 0u);
    const uint32_t nextR = (mR >> 1) | (((nb & 0xF8) == 0xD0) ? 0x8000u : 0u);
    const uint32_t lastb = (e - 1 >= gb && e - 1 < gb + 16) ? (1u << uint32_t(e - 1 - gb)) : 0u;
    const uint32_t rstFF = dri ? (mFF & nextR & ~lastb & inr) : 0u;
    const uint32_t rstX = dri ? (mR & prevFF & inr) : 0u;
    const uint32_t remv = ((m00 & prevFF) | rstFF | rstX) & inr;  // removed bytes
    const uint32_t mark = mFF & inr & ~rstFF & (~next00 | lastb);   // markers ending the scan
    const uint32_t cnt = __popc(remv), rc = __popc(rstFF);
    const uint32_t mk = mark ? uint32_t(gb - a) + (__ffs(mark) - 1) : kInf32;
    // block reduce (sum, min); removed | RST count << 16 (both < 2^16 per tile)
    const uint32_t cr = cnt | (rc << 16);
    uint32_t wc = cr, wm = mk;
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
    if (warp == 0) {
        // tile totals, then a warp-parallel decoupled lookback (32 predecessors
        // per step), segmented at the image's first tile:
        // agg [0] aggregate (mk << 32 | removed), [1] aggregate RST count, [2], [3] inclusive
        uint32_t tcr = 0, tm = kInf32;
        for (int w = 0; w < kK0Threads / 32; ++w) {
            tcr += s_cnt[w];
            tm = min(tm, s_mk[w]);
        }
        const uint32_t tc = tcr & 0xFFFFu, trc = tcr >> 16;
        uint64_t* agg = P.k0_agg + 4ull * t;
        uint32_t ec = 0, em = kInf32, erc = 0;
        if (lt == 0) {
            if (lane == 0) {
                agg[2] = (uint64_t(tm) << 32) | tc;
                agg[3] = trc;
                st_release(P.k0_flag + t, (P.epoch << 2) | 2u);
            }
        } else {
            if (lane == 0) {
                agg[0] = (uint64_t(tm) << 32) | tc;
                agg[1] = trc;
                st_release(P.k0_flag + t, (P.epoch << 2) | 1u);
            }
            const int64_t first_t = int64_t(P.k0_first[k]);
            int64_t base = int64_t(t) - 1;
            while (true) {
                const int64_t pr = base - lane;  // lane 0: nearest predecessor
                uint32_t f = 2u;                 // before the image: an empty inclusive prefix
                if (pr >= first_t) {
                    f = ld_acquire(P.k0_flag + pr);
                    while ((f >> 2) != P.epoch) {
                        spin_pause();
                        f = ld_acquire(P.k0_flag + pr);
                    }
                }
                const uint32_t incl = __ballot_sync(0xFFFFFFFFu, (f & 3u) == 2u);
                const int lim = incl ? __ffs(incl) - 1 : 31;
                uint32_t c = 0, m = kInf32, r = 0;
                if (lane <= lim && pr >= first_t) {
                    const uint64_t* src = P.k0_agg + 4ull * pr + ((f & 3u) == 2u ? 2 : 0);
                    const uint64_t v = __ldcg(src);
                    c = uint32_t(v);
                    m = uint32_t(v >> 32);
                    r = uint32_t(__ldcg(src + 1));
                }
                ec += __reduce_add_sync(0xFFFFFFFFu, c);
                em = min(em, __reduce_min_sync(0xFFFFFFFFu, m));
                erc += __reduce_add_sync(0xFFFFFFFFu, r);
                if (incl) break;
                base -= 32;
            }
            if (lane == 0) {
                agg[2] = (uint64_t(min(em, tm)) << 32) | (ec + tc);
                agg[3] = erc + trc;
                st_release(P.k0_flag + t, (P.epoch << 2) | 2u);
            }
        }
        if (lane == 0) {
            s_tile_cnt = tc;
            s_tile_mk = tm;
            s_excl_cnt = ec;
            s_excl_mk = em;
            s_excl_rc = erc;
        }
    }
    __syncthreads();
    // exclusive scan of per-thread (removed | RST << 16) counts (warp shuffles + smem)
    uint32_t inc = cr;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t v = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= o) inc += v;
    }
    __syncthreads();
    if (lane == 31) s_cnt[warp] = inc;
    __syncthreads();
    uint32_t wbase = 0;
    for (int w = 0; w < warp; ++w) wbase += s_cnt[w];
    const uint32_t before_cr = wbase + inc - cr;
    uint32_t removed = s_excl_cnt + (before_cr & 0xFFFFu);  // removed before this thread's bytes
    uint32_t rst_before = s_excl_rc + (before_cr >> 16);    // RST markers before them

    // kept byte at image index j goes to image index j - removed; this tile's
    // kept bytes form [dst_lo, dst_lo + kept) in raw-buffer coordinates
    const uint64_t dst_lo = g_first - s_excl_cnt;
    const uint64_t dst_al = dst_lo & ~15ull;
    const uint32_t first_mk = s_excl_mk == kInf32 ? s_tile_mk : kInf32;  // the image's scan end
    {
        // kept bytes to their compacted positions: byte i moves left by the
        // removed bytes before it in this chunk
        const uint32_t keep = inr & ~remv;
        uint8_t* o = s_o + ((gb - removed) - dst_al);
        const uint4 w = reinterpret_cast<const uint4*>(s_b + 16)[tid];
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int i = 0; i < 16; ++i)
            if ((keep >> i) & 1u) o[i - __popc(remv & ((1u << i) - 1u))] = uint8_t(ws[i >> 2] >> (8 * (i & 3)));
    }
    // rare events, off the branch-free path: the scan end and restart markers
    if (first_mk != kInf32 && first_mk - uint32_t(gb - a) < 16u && (mark >> (first_mk - uint32_t(gb - a))) & 1u) {
        // scan ends here (extract_scan, parser.hpp:241-254)
        const uint32_t i = first_mk - uint32_t(gb - a);
        const uint64_t j = first_mk;
        const uint64_t U = j - (removed + __popc(remv & ((1u << i) - 1u)));
        ImgState* st = P.ist + k;
        st->bit_length = U * 8;
        const uint8_t nx = s_b[17 + b0 + i];
        const bool rst = (j + 1 < raw_len) && nx >= 0xD0 && nx <= 0xD7;
        if (rst)
            set_status(st, kUnsupportedFeature);
        else if (U == 0)
            set_status(st, kEmptyScan);
        else if (D.deferred)
            set_status(st, D.deferred);
    }
    if (DRI && rstFF) {
        // restart marker r: interval r + 1 starts at unstuffed byte j - removed;
        // markers past the scan end do not count
        const uint32_t end_mk = s_excl_mk != kInf32 ? s_excl_mk : s_tile_mk;
        for (uint32_t m = rstFF; m; m &= m - 1) {
            const uint32_t i = __ffs(m) - 1;
            const uint64_t j = gb - a + i;
            const uint32_t r = rst_before + __popc(rstFF & ((1u << i) - 1u));
            if (j >= end_mk) continue;
            const uint8_t nx = s_b[17 + b0 + i];
            if (r + 1 >= D.n_int || (nx & 7u) != (r & 7u))
                set_status(P.ist + k, kConsistencyFailure);  // RST count / numbering vs DRI
            else
                P.segs[D.seg_first + r + 1].x = uint32_t((j - (removed + __popc(remv & ((1u << i) - 1u)))) * 8);
        }
    }
    __syncthreads();
    {
        const uint64_t dst_hi = dst_lo + (min64(e, win0 + kSmallTile) - g_first) - s_tile_cnt;
        const uint32_t nchunks = uint32_t((dst_hi - dst_al + 15) >> 4);
        for (uint32_t q = tid; q < nchunks; q += kK0Threads) {
            const uint64_t G = dst_al + 16ull * q;
            if (G >= dst_lo && G + 16 <= dst_hi) {
                *reinterpret_cast<int4*>(P.ubuf + G) = reinterpret_cast<const int4*>(s_o)[q];
            } else {
                for (uint32_t x = 0; x < 16; ++x)
                    if (G + x >= dst_lo && G + x < dst_hi) P.ubuf[G + x] = s_o[16 * q + x];
            }
        }
    }
    // no marker anywhere: the scan runs to the end of the file
    const uint32_t last_tile = uint32_t(((a & 15ull) + raw_len + kSmallTile - 1) / kSmallTile) - 1;
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

// ================================================ K0b: interval tables ====
// One CTA per image with restart intervals: closes its segment table
// (x_0 = 0, x_n = bit length), checks that every interval got its RST marker
// and is non-empty, and partitions each interval into ceil(bits / sb)
// subsequences (y = exclusive prefix; y_n = subsequences in use).
__global__ void __launch_bounds__(256) k0b_segments(Params P) {
    pdl_wait();
    __shared__ uint32_t s_w[8];
    __shared__ uint32_t s_carry;
    __shared__ int s_bad;
    const uint32_t k = P.dri_img[blockIdx.x];
    const ImgDesc& D = P.img[k];
    ImgState* st = P.ist + k;
    if (st->status != 0) return;
    const uint32_t n = D.n_int;
    uint2* sg = P.segs + D.seg_first;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        sg[0].x = 0;
        sg[n].x = uint32_t(st->bit_length);
        s_carry = 0;
        s_bad = 0;
    }
    __syncthreads();
    for (uint32_t base = 0; base < n; base += 256) {
        const uint32_t m = base + tid;
        uint32_t cntm = 0;
        if (m < n) {
            const uint32_t x0 = sg[m].x, x1 = sg[m + 1].x;
            if (x0 == 0xFFFFFFFFu || x1 == 0xFFFFFFFFu || x1 <= x0)
                s_bad = 1;  // a missing RST marker or an empty interval
            else
                cntm = uint32_t((uint64_t(x1 - x0) + P.sb - 1) / P.sb);
        }
        uint32_t inc = cntm;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, inc, o);
            if (lane >= o) inc += v;
        }
        if (lane == 31) s_w[warp] = inc;
        __syncthreads();
        uint32_t wb = s_carry;
        for (int w = 0; w < warp; ++w) wb += s_w[w];
        if (m < n) sg[m].y = wb + inc - cntm;
        __syncthreads();
        if (tid == 255) s_carry = wb + inc;
        __syncthreads();
    }
    if (tid == 0) {
        sg[n].y = s_carry;
        if (s_bad) set_status(st, kConsistencyFailure);
    }
}

// Copies the batch's fast tables into shared memory (P.smem_tables tables,
// dynamic shared memory) and returns them, or nullptr when not enabled.
__device__ __forceinline__ const uint32_t* stage_tables(const Params& P, uint32_t* s_fast, int tid, int nthreads,
                                                       uint32_t ntab = 0xFFFFFFFFu) {
    if (ntab == 0xFFFFFFFFu) ntab = P.smem_tables;
    if (!ntab) return nullptr;
    for (uint32_t x = tid; x < ntab * (kFastWords / 4); x += nthreads) {
        const uint32_t t = x / (kFastWords / 4), q = x % (kFastWords / 4);
        reinterpret_cast<uint4*>(s_fast)[x] = __ldg(reinterpret_cast<const uint4*>(P.huff[t].fast) + q);
    }
    return s_fast;  // the caller's __syncthreads (stage_scan) publishes it
}

// ============================================== entropy decode (shared) ====
constexpr uint32_t kHuffWords = sizeof(DevHuff) / 4;  // fast[] sits at word 0 of each table

struct ImgCtx {
    const uint32_t* words;  // ubuf as 32-bit words (when not staged)
    uint32_t sbase;         // staged: shared address of absolute word 0 (mod 2^32; words byte-swapped)
    bool staged;
    int32_t* sacc;          // this thread's DC accumulator of component 0 (shared memory)
    uint32_t sacc_stride;   // ... components apart (elements)
    uint64_t bit_base;      // 8 * raw_off
    uint64_t L;             // bit_length
    const uint32_t* fast;   // fast[] of table t at t * stride (the global DevHuff array, or smem copies)
    const DevHuff* huff;    // the tables (exact path)
    uint32_t tdc[3], tac[3];  // fast-table word offsets per component
    uint32_t duc;           // slot -> component, 2 bits per slot
    uint32_t dpm;
};
template <bool ST>
struct TabStride {
    static constexpr uint32_t value = ST ? kFastWords : kHuffWords;
};

// sfast: the batch's fast tables staged in shared memory (nullptr: global).
// Small batches have few resident CTAs per SM, so each symbol's table probe
// would otherwise often miss L1 on the decoder's serial dependency chain.
template <bool ST = false>
__device__ __forceinline__ void load_ctx(const Params& P, const ImgDesc& D, uint64_t L, ImgCtx& c,
                                         const uint32_t* sfast = nullptr) {
    c.words = reinterpret_cast<const uint32_t*>(P.ubuf);
    c.sbase = 0;
    c.staged = false;
    c.bit_base = D.raw_off * 8;
    c.L = L;
    c.huff = P.huff;
    c.fast = ST ? sfast : reinterpret_cast<const uint32_t*>(P.huff);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        c.tdc[k] = uint32_t(D.dc_tab[k]) * TabStride<ST>::value;
        c.tac[k] = uint32_t(D.ac_tab[k]) * TabStride<ST>::value;
    }
    uint32_t duc = 0;
    for (uint32_t s = 0; s < D.dpm; ++s) duc |= (uint32_t(D.du_comp >> (4 * s)) & 3u) << (2 * s);
    c.duc = duc;
    c.dpm = D.dpm;
}

__device__ __forceinline__ uint32_t bswap32(uint32_t v) { return __byte_perm(v, 0, 0x0123); }

// Stages the unstuffed-scan bytes a CTA's subsequences touch into shared
// memory (coalesced 16-byte loads) and returns a word pointer that decode_range
// can index with absolute word positions (it then reads shared memory through
// generic loads).  A CTA can straddle images, so the bytes are staged as up to
// kStageSegs segments, one per image (the bytes between two images' scans —
// the next file's headers — are skipped).  [lo, hi) is this thread's byte
// range (empty when lo >= hi), k its image; segments that do not fit fall back
// to the global pointer.
constexpr int kStageBytes = 16512;  // 128 subsequences x 1024 bits + window slack + segment alignment
constexpr int kStageSegs = 4;
struct StageSmem {
    unsigned long long lo[kStageSegs], hi[kStageSegs];
    uint32_t off[kStageSegs];
    uint32_t k0;
};
__device__ __forceinline__ void stage_scan(const uint8_t* ubuf, uint64_t lo, uint64_t hi, uint32_t k, int tid,
                                           int nthreads, int4* s_stage, StageSmem& sm) {
    if (tid < kStageSegs) {
        sm.lo[tid] = ~0ull;
        sm.hi[tid] = 0ull;
    }
    if (tid == 0) sm.k0 = k;
    __syncthreads();
    const uint32_t seg = k - sm.k0;
    if (lo < hi && seg < kStageSegs) {
        atomicMin(&sm.lo[seg], (unsigned long long)lo);
        atomicMax(&sm.hi[seg], (unsigned long long)hi);
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t off = 0;
        for (int q = 0; q < kStageSegs; ++q) {
            sm.off[q] = 0xFFFFFFFFu;
            if (sm.hi[q] > sm.lo[q]) {
                const uint64_t blo = sm.lo[q] & ~15ull;
                const uint64_t sz = (sm.hi[q] - blo + 15) & ~15ull;
                if (off + sz <= uint64_t(kStageBytes)) {
                    sm.off[q] = off;
                    off += uint32_t(sz);
                }
            }
        }
    }
    __syncthreads();
#pragma unroll 1
    for (int q = 0; q < kStageSegs; ++q) {
        if (sm.off[q] == 0xFFFFFFFFu) continue;
        const uint64_t blo = sm.lo[q] & ~15ull;
        const uint32_t n16 = uint32_t((sm.hi[q] - blo + 15) >> 4);
        const int4* src = reinterpret_cast<const int4*>(ubuf + blo);
        int4* dst = s_stage + (sm.off[q] >> 4);
        for (uint32_t x = tid; x < n16; x += nthreads) {
            int4 v = __ldcs(src + x);  // stored byte-swapped: the decoder's MSB-first words
            v.x = int(bswap32(uint32_t(v.x)));
            v.y = int(bswap32(uint32_t(v.y)));
            v.z = int(bswap32(uint32_t(v.z)));
            v.w = int(bswap32(uint32_t(v.w)));
            dst[x] = v;
        }
    }
    __syncthreads();
}
// The thread's three DC accumulators in shared memory (s_acc[3 * nthreads]).
__device__ __forceinline__ void set_sacc(ImgCtx& ic, int32_t* s_acc, int tid, int nthreads) {
    ic.sacc = s_acc + tid;
    ic.sacc_stride = uint32_t(nthreads);
}

// Points the decoder of image k at its staged bytes (after stage_scan), or
// leaves it on global memory when k's segment did not fit.
__device__ __forceinline__ void set_stage(ImgCtx& ic, const int4* s_stage, const StageSmem& sm, uint32_t k) {
    const uint32_t seg = k - sm.k0;
    ic.staged = seg < kStageSegs && sm.off[seg] != 0xFFFFFFFFu;
    if (ic.staged)
        ic.sbase = uint32_t(__cvta_generic_to_shared(s_stage + (sm.off[seg] >> 4))) - uint32_t(sm.lo[seg] & ~15ull);
}


// Device huff_lookup with read-only-path loads.
__device__ __forceinline__ uint32_t dev_lookup(const DevHuff* t, uint32_t w16, uint32_t& maxlen) {
    maxlen = __ldg(&t->maxlen);
    uint32_t e = __ldg(&t->lut[w16 >> (16 - kPrimaryBits)]);
    if (e & kL2Flag) return __ldg(&t->lut2[e & 0x7FFFu][w16 & ((1u << (16 - kPrimaryBits)) - 1)]);
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
    uint32_t k;  // sync mode: coded coefficients (DC symbols + nonzero AC) — the compact entries K3 writes
    uint32_t c, z;
    bool div;
    bool ovf;  // write mode: a run went past the unit end (z + step > 64): the image needs K1x
    int32_t err;
    int32_t dc0, dc1, dc2;
};

struct NullSink {
    static constexpr bool kWrite = false;
    static constexpr bool kStore = false;
    static constexpr bool kSmemAcc = true;
    __device__ __forceinline__ void put(uint32_t, int32_t) {}
    __device__ __forceinline__ void block_end(uint32_t) {}
    __device__ __forceinline__ void sym(uint32_t) {}
};

// Sync-mode sink that also keeps the decoded symbols of one subsequence for
// K3 to replay instead of decoding again: 16 bits per symbol, run << 12 |
// (coefficient & 0xFFF) — DC (z == 0 on replay): the difference; AC: run and
// the value (nonzero), EOB: run 0 value 0, ZRL: run 15 value 0.  Symbol i of
// global subsequence g sits at [i * stride + g] (a warp of consecutive
// subsequences reads symbol i as one 64-byte row); symbols past `cap` are
// dropped (the tag then says so).
struct SymSink {
    static constexpr bool kWrite = false;
    static constexpr bool kStore = true;
    static constexpr bool kSmemAcc = true;
    uint16_t* dst;     // &sym[g]
    uint64_t stride;   // subsequences per symbol row
    uint32_t cap;
    uint32_t n = 0;
    __device__ __forceinline__ void put(uint32_t, int32_t) {}
    __device__ __forceinline__ void block_end(uint32_t) {}
    __device__ __forceinline__ void sym(uint32_t w) {
        if (n < cap) dst[uint64_t(n) * stride] = uint16_t(w);
        ++n;
    }
};

// decode_subsequence (parallel_decode.hpp:122-164) with decode_next_symbol
// (huffman.hpp:137-175) inlined.  Decodes symbols whose first bit lies in
// [s.p, end_bit).  The caller seeds s (p, c, z, dc accumulators); n starts at
// 0.  Sync mode: an InvalidCode/OutOfBits marks the state divergent at the
// last good symbol.  Write mode: stops at `cap` slots; errors are reported.
//
// The hot loop keeps a 32-bit window taken by a funnel shift from two
// consecutive words (w0:w1) at bit offset bp < 32 — any symbol (<= 16 code +
// 11 magnitude bits) fits in it — and advances by at most one word per symbol,
// branch-free, with the following word already loaded.  Staged scan bytes are
// read from shared memory with 32-bit addresses (stored byte-swapped by the
// stage copy); otherwise from global memory.  One probe of an 11-bit table
// resolves code + magnitude; its entry carries the code length, total length,
// magnitude size, run+1 and kind (jfif.cpp build_fast).  Windows the probe
// cannot settle (long codes, invalid prefixes, the last 32 bits of the scan)
// take the reference's exact path with its error order.  The DC accumulator
// of the current block's component is kept in one register (swapped at block
// ends).
template <bool SW>
struct WordReader {
    const uint32_t* g;  // global words (SW = false)
    uint32_t sbase;     // shared address of word 0 (SW = true; mod 2^32)
    __device__ __forceinline__ uint32_t operator()(uint32_t wi) const {
        if (SW) {
            uint32_t v;
            asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(sbase + 4u * wi));
            return v;  // staged byte-swapped
        }
        return bswap32(__ldg(g + wi));
    }
};

template <bool ST>
__device__ __forceinline__ uint32_t fast_entry(const ImgCtx& ic, uint32_t tsh, uint32_t fi) {
    if (ST) {
        uint32_t v;
        asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(tsh + 4u * fi));
        return v;
    }
    return __ldg(ic.fast + fi);
}

// second-level fast entry (codes of 12..16 bits): global (L1) in both modes
template <bool ST>
__device__ __forceinline__ uint32_t fast_entry2(const ImgCtx& ic, uint32_t tb, uint32_t k2, uint32_t s) {
    if (ST) return __ldg(&ic.huff[tb / kFastWords].fast2[k2][s]);
    return __ldg(ic.fast + tb + kFastWords + k2 * 32 + s);
}

template <class Sink, bool ST, bool SW>
__device__ __forceinline__ void decode_core(const ImgCtx& ic, DecState& s, uint64_t end_bit, uint32_t cap,
                                            Sink& sink) {
    WordReader<SW> W;
    W.g = ic.words;
    W.sbase = ic.sbase;
    const uint32_t tsh = ST ? uint32_t(__cvta_generic_to_shared(ic.fast)) : 0u;
    // MSB-first window over the unstuffed bytes
    const uint64_t abs = ic.bit_base + s.p;
    uint32_t wi = uint32_t(abs >> 5);
    uint32_t bp = uint32_t(abs & 31);
    uint32_t w0 = W(wi), w1 = W(wi + 1);
    wi += 2;
    uint32_t nw = W(wi);  // the word after w1
    uint64_t p = s.p;
    uint32_t c = s.c, z = s.z, n = 0, kc = 0;
    int32_t a0 = s.dc0, a1 = s.dc1, a2 = s.dc2;
    uint32_t comp = (ic.duc >> (2 * c)) & 3u;
    uint32_t tdc = comp == 0 ? ic.tdc[0] : (comp == 1 ? ic.tdc[1] : ic.tdc[2]);
    uint32_t tac = comp == 0 ? ic.tac[0] : (comp == 1 ? ic.tac[1] : ic.tac[2]);
    // Sync mode: the DC accumulators live in shared memory — a DC symbol (once
    // per block) updates the current component's, and a block end only moves
    // the address.  Write mode needs each absolute DC at once (the sink): the
    // current component's accumulator is a register, swapped at block ends.
    constexpr bool kRegAcc = Sink::kWrite && !Sink::kSmemAcc;
    int32_t* const sa0 = ic.sacc;
    const uint32_t sst = ic.sacc_stride;
    if (!kRegAcc) {
        sa0[0] = a0;
        sa0[sst] = a1;
        sa0[2 * sst] = a2;
    }
    int32_t* sa = sa0 + comp * sst;
    int32_t acur = comp == 0 ? a0 : (comp == 1 ? a1 : a2);
    const uint64_t lr = ic.L - p;
    int32_t lrem = lr > 0x40000000ull ? 0x40000000 : int32_t(lr);  // bits to the scan end, saturated
    uint64_t left = end_bit - p;
    bool stop = false;
    while (!stop) {
        // the range in chunks of < 2^30 bits (one chunk for any realistic subsequence)
        int32_t rem = left > 0x40000000ull ? 0x40000000 : int32_t(left);
        left -= uint64_t(rem);
        const int32_t rem0 = rem;
        // lrem - rem is constant in the chunk: lrem >= 32 <=> rem >= rthr
        const int32_t rthr = 32 - (lrem - rem);
        while (rem > 0) {
            if (Sink::kWrite && n >= cap) {
                stop = true;
                break;
            }
            const uint32_t win = __funnelshift_l(w1, w0, bp);
            const bool dcs = z == 0;
            const uint32_t tb = dcs ? tdc : tac;
            uint32_t fe = fast_entry<ST>(ic, tsh, tb + (win >> (32 - kFastBits)));
            if ((fe & 0x3FFu) == kFastL2) {
                // (the table address only on this path: keep the compiler from
                // hoisting its 64-bit arithmetic into every symbol)
                uint32_t tb2 = tb;
                asm volatile("" : "+r"(tb2));
                fe = fast_entry2<ST>(ic, tb2, (fe >> 10) & 31u, (win >> (32 - kFastBits - 5)) & 31u);
            }
            uint32_t len, step, coefk;
            int32_t coef;
            if ((fe & 31u) != 0 && rem >= rthr) {
                // code + magnitude (<= 11 + 11 bits) all real: >= 32 bits to the scan end
                const uint32_t clen = fe & 31u;
                len = fe >> kFastLenShift;
                const uint32_t w2 = win << clen;
                // top l bits after the code (the shift count wraps mod 32; bit 9 is 0)
                const uint32_t v = __funnelshift_l(w2, 0u, fe >> kFastLShift);
                // extend(): a leading 1 is positive, else v - (2^l - 1)
                const uint32_t t = (fe >> kFastTShift) & 0x7FFu;
                coef = int32_t(v - (t & ~uint32_t(int32_t(w2) >> 31)));
                const uint32_t r1 = (fe >> kFastR1Shift) & 63u;  // run + 1 (0: EOB)
                step = r1 ? r1 : 64u - z;
                coefk = (dcs || t != 0) ? 1u : 0u;
                if (Sink::kStore) sink.sym(((r1 ? r1 - 1u : 0u) << 12) | (uint32_t(coef) & 0xFFFu));
            } else {
                const DevHuff* t = ST ? ic.huff + (dcs ? tdc : tac) / TabStride<ST>::value
                                      : reinterpret_cast<const DevHuff*>(ic.fast + (dcs ? tdc : tac));
                uint32_t maxlen;
                const uint32_t e = dev_lookup(t, win >> 16, maxlen);
                const uint32_t clen = e >> 8, sym = e & 255u;
                const uint32_t avail = uint32_t(lrem - (rem0 - rem));  // bits to the scan end, >= 1 inside the range
                int32_t err = 0;
                uint32_t l = 0, run = 0;
                bool eob = false;
                coefk = 0;
                if (clen == 0) {
                    err = avail < maxlen ? kOutOfBits : kInvalidCode;
                } else if (clen > avail) {
                    err = kOutOfBits;
                } else if (dcs) {
                    l = sym;
                    if (l > 11)
                        err = kInvalidCode;
                    else if (avail - clen < l)
                        err = kOutOfBits;
                    coefk = 1;
                } else {
                    const uint32_t r = sym >> 4;
                    l = sym & 15u;
                    if (l == 0) {
                        if (r == 0) {
                            eob = true;
                        } else if (r == 15) {
                            run = 15;
                        } else {
                            err = kInvalidCode;
                        }
                    } else if (l > 10) {
                        err = kInvalidCode;
                    } else if (avail - clen < l) {
                        err = kOutOfBits;
                    } else {
                        run = r;
                        coefk = 1;
                    }
                }
                if (err) {
                    s.div = true;
                    s.err = err;
                    stop = true;
                    break;
                }
                coef = 0;
                if (l) {
                    const uint32_t bits = (win << clen) >> (32 - l);
                    coef = bits >= (1u << (l - 1)) ? int32_t(bits) : int32_t(bits) - int32_t((1u << l) - 1);
                }
                len = clen + l;
                step = eob ? 64u - z : run + 1u;
                if (Sink::kStore) sink.sym((run << 12) | (uint32_t(coef) & 0xFFFu));
            }
            // write mode: a phantom tail past the true end stops the decode; a run
            // past the unit end (reference semantics in K1x) also flags it —
            // one test of both on the per-symbol path
            if (Sink::kWrite && (n + step > cap || z + step > 64)) {
                if (n + step <= cap) s.ovf = true;
                stop = true;
                break;
            }
            if (kRegAcc) {  // branch-free: the DC test diverges across lanes
                acur += dcs ? coef : 0;
                coef = dcs ? acur : coef;
            } else if (dcs) {
                {
                    coef += *sa;
                    *sa = coef;
                }
            }
            if (Sink::kWrite && coefk) sink.put(z + step - 1, coef);
            // advance: bp + len <= 31 + 27, so at most one word
            bp += len;
            const bool adv = bp >= 32u;
            bp &= 31u;
            w0 = adv ? w1 : w0;
            w1 = adv ? nw : w1;
            wi += adv ? 1u : 0u;
            nw = W(wi);
            rem -= int32_t(len);
            n += step;
            if (!Sink::kWrite) kc += coefk;
            z += step;
            if (z >= 64) {
                if (kRegAcc) {
                    if (comp == 0)
                        a0 = acur;
                    else if (comp == 1)
                        a1 = acur;
                    else
                        a2 = acur;
                }
                z = 0;
                c = (c + 1 == ic.dpm) ? 0 : c + 1;
                comp = (ic.duc >> (2 * c)) & 3u;
                tdc = comp == 0 ? ic.tdc[0] : (comp == 1 ? ic.tdc[1] : ic.tdc[2]);
                tac = comp == 0 ? ic.tac[0] : (comp == 1 ? ic.tac[1] : ic.tac[2]);
                if (kRegAcc)
                    acur = comp == 0 ? a0 : (comp == 1 ? a1 : a2);
                else
                    sa = sa0 + comp * sst;
                if (Sink::kWrite) sink.block_end(comp);
            }
        }
        p += uint64_t(int64_t(rem0) - int64_t(rem));
        lrem -= rem0 - rem;
        if (stop) break;
        // rem <= 0: the last symbol ran -rem bits past the chunk end
        const uint64_t over = uint64_t(-int64_t(rem));
        if (left <= over) break;
        left -= over;
    }
    if (kRegAcc) {
        if (comp == 0)
            a0 = acur;
        else if (comp == 1)
            a1 = acur;
        else
            a2 = acur;
    } else {
        a0 = sa0[0];
        a1 = sa0[sst];
        a2 = sa0[2 * sst];
    }
    s.p = p;
    s.n = n;
    s.k = kc;
    s.c = c;
    s.z = z;
    s.dc0 = a0;
    s.dc1 = a1;
    s.dc2 = a2;
}

template <class Sink, bool ST = false>
__device__ __forceinline__ void decode_range(const ImgCtx& ic, DecState& s, uint64_t end_bit, uint32_t cap,
                                             Sink& sink) {
    s.n = 0;
    s.k = 0;
    s.div = false;
    s.ovf = false;
    s.err = 0;
    if (s.p >= end_bit) return;
    if (ic.staged)
        decode_core<Sink, ST, true>(ic, s, end_bit, cap, sink);
    else
        decode_core<Sink, ST, false>(ic, s, end_bit, cap, sink);
}

// DC sums mod 2^16 per component; the high half of .hi carries the entry
// count k (<= subsequence bits: every coded coefficient takes >= 1 bit; the
// compact interface needs sb <= 65535)
__device__ __forceinline__ DcSums pack_dc(int32_t a0, int32_t a1, int32_t a2, uint32_t k) {
    DcSums d;
    d.lo = (uint32_t(a0) & 0xFFFFu) | (uint32_t(a1) << 16);
    d.hi = (uint32_t(a2) & 0xFFFFu) | (min(k, 0xFFFFu) << 16);
    return d;
}

// Sync-mode decode from (p, c, z) of the symbols starting before end_bit.
template <bool ST, class Sink>
__device__ __forceinline__ void sync_decode_sink(const ImgCtx& ic, uint64_t end_bit, uint64_t p, uint32_t c,
                                                 uint32_t z, Entry& e, DcSums& d, Sink& sink) {
    DecState s;
    s.p = p;
    s.c = c;
    s.z = z;
    s.dc0 = s.dc1 = s.dc2 = 0;
    decode_range<Sink, ST>(ic, s, end_bit, 0, sink);
    e.p = s.p;
    e.n = s.n;
    e.czd = pack_czd(s.c, s.z, s.div);
    d = pack_dc(s.dc0, s.dc1, s.dc2, s.k);
}
template <bool ST = false>
__device__ __forceinline__ void sync_decode(const ImgCtx& ic, uint64_t end_bit, uint64_t p, uint32_t c, uint32_t z,
                                            Entry& e, DcSums& d) {
    NullSink sink;
    sync_decode_sink<ST>(ic, end_bit, p, c, z, e, d, sink);
}

// Replay tags (one per global subsequence): the start state the stored
// symbols were decoded from, their count and the decode epoch.  K3 replays a
// subsequence's symbols when its true start state equals the tag's: the
// decode from one state is unique, so who produced them does not matter.
__device__ __forceinline__ uint4 make_tag(uint64_t p, uint32_t c, uint32_t z, uint32_t nsym, uint32_t epoch) {
    return make_uint4(uint32_t(p), uint32_t(p >> 32), c | (z << 8) | (nsym << 16), epoch);
}

// ======================================================== K1: sync pass ====
// CTA j owns the kK1Own global subsequences [j*kK1Own, (j+1)*kK1Own); thread
// t >= kK1Spec owns subsequence j*kK1Own + t - kK1Spec.  Threads 0..kK1Spec-1
// re-decode the predecessor CTA's last subsequences (round 0, and the chain
// between them), and their overflow chain carries that speculative state into this CTA — the
// inter-sequence overflow of sync_inter_sequence (parallel_decode.hpp:247-270)
// started without waiting for the predecessor.  After the intra rounds the
// speculative start is checked against the predecessor's published
// post-intra last entry and re-chained only where they differ (a few % of
// CTAs); K1c then re-runs every boundary whose start differs from the
// predecessor's final entry (the reference's end_changed passes).  Images are flattened into one
// subsequence space; a CTA may hold the tail of one image and the head of the
// next, and overflow chains stop at image (and restart-interval) ends.
//
// Overflow rounds are lane-compacted: the live chains of a round are listed in
// shared memory and taken by threads 0..n-1, so a round with few live chains
// occupies one warp instead of every warp that holds one.  A chain into
// subsequence t runs in t's image context (the same image: chains stop at
// segment ends).
struct K1Chain {
    uint64_t p;
    uint32_t czd;
    uint32_t nt;
};
// SYM: the batch replays K1's symbols in K3 (Params::sym_cap != 0; never with ST)
template <bool DRI, bool ST, bool HOP, bool SYM>
__global__ void __launch_bounds__(kK1Threads) k1_sync(Params P) {
    pdl_wait();
    constexpr int T = kK1Threads;
    constexpr int TO = kK1Own;
    __shared__ uint64_t s_p[T];
    __shared__ uint32_t s_n[T];
    __shared__ uint32_t s_czd[T];
    __shared__ DcSums s_dc[T];
    __shared__ uint64_t s_hi[T];  // end bit of thread t's subsequence
    __shared__ uint32_t s_km[T];  // image of thread t | 1 << 31 when a chain may continue past t
    __shared__ K1Chain s_list[2][T];
    __shared__ uint32_t s_cnt[2];
    __shared__ int4 s_stage[kStageBytes / 16];
    __shared__ StageSmem s_sm;
    __shared__ uint32_t s_cta;

    const int tid = threadIdx.x;
    if (tid == 0) s_cta = atomicAdd(&P.counters[kTicketK1], 1u);
    __syncthreads();
    // ticket order: a predecessor started earlier and is never waiting on this CTA
    const uint32_t cta = s_cta;
    const int64_t gs = int64_t(cta) * TO + tid - kK1Spec;
    const bool inb = gs >= 0 && uint64_t(gs) < P.total_subs;
    const uint64_t g = inb ? uint64_t(gs) : (gs < 0 ? 0 : P.total_subs - 1);
    const uint32_t k = find_img(P, g);
    const ImgDesc& D = P.img[k];
    const uint64_t i = g - P.sub_first[k];
    const uint64_t L = P.ist[k].bit_length;
    const bool ok = P.ist[k].status == 0;
    SubInfo si;
    const bool real = inb && ok && sub_info<DRI>(P, D, L, i, si);
    extern __shared__ uint32_t s_fast_k1[];
    const uint32_t* sfast = ST ? stage_tables(P, s_fast_k1, tid, T) : nullptr;
    ImgCtx ic;
    load_ctx<ST>(P, D, L, ic, sfast);
    __shared__ int32_t s_acc[3 * T];
    set_sacc(ic, s_acc, tid, T);
    if (tid < 2) s_cnt[tid] = 0;
    {
        const uint64_t lo = real ? D.raw_off + (si.lo >> 3) : 1, hi = real ? D.raw_off + ((si.hi + 7) >> 3) + 24 : 0;
        stage_scan(P.ubuf, lo, hi, k, tid, T, s_stage, s_sm);
        set_stage(ic, s_stage, s_sm, k);
    }

    // Round 0: every subsequence decodes from its origin (parallel_decode.hpp:187-195)
    Entry e;
    DcSums d = {0, 0};
    e.p = real ? si.lo : 0;
    e.n = 0;
    e.czd = 0;
    if (real) sync_decode<ST>(ic, si.hi, si.lo, 0, 0, e, d);
    s_p[tid] = e.p;
    s_n[tid] = e.n;
    s_czd[tid] = e.czd;
    s_dc[tid] = d;
    s_hi[tid] = real ? si.hi : 0;
    const bool more = real && i + 1 < si.seg_sub1 && tid + 1 < T;
    s_km[tid] = k | (more ? 0x80000000u : 0u);
    if (more && !czd_div(e.czd)) {
        const uint32_t slot = atomicAdd(&s_cnt[0], 1u);
        s_list[0][slot] = K1Chain{e.p, e.czd, uint32_t(tid + 1)};
    }
    __syncthreads();
    // Rounds k >= 1: overflow into the next subsequence until (p,c,z) agrees
    // with the published entry (parallel_decode.hpp:197-220).  Live chains
    // target distinct subsequences, so one barrier per round orders them.
    int rounds = 0, cur = 0;
    uint32_t ick = k;
    for (;;) {
        const uint32_t nact = s_cnt[cur];
        __syncthreads();  // everyone has read the count
        if (tid == 0) s_cnt[cur] = 0;  // refilled two rounds later
        if (nact == 0) break;
        ++rounds;
        if (uint32_t(tid) < nact) {
            const K1Chain ch = s_list[cur][tid];
            const uint32_t nt = ch.nt;
            const uint32_t km = s_km[nt];
            const uint32_t kk = km & 0x7FFFFFFFu;
            if (kk != ick) {  // chain of another image of this CTA
                const ImgDesc& D2 = P.img[kk];
                load_ctx<ST>(P, D2, P.ist[kk].bit_length, ic, sfast);
                set_stage(ic, s_stage, s_sm, kk);
                ick = kk;
            }
            Entry e2;
            DcSums d2;
            // the chain keeps its symbols for K3 (tagged with its start state)
            // (only owned targets: a speculative one is the predecessor CTA's)
            const bool owned_t = nt >= uint32_t(kK1Spec);
            const uint64_t gt = uint64_t(cta) * TO + nt - kK1Spec;
            // (small batches, ST: never replayed — the planner enables replay only
            // for large ones; the plain sink also compiles better there)
            using ChainSink = typename std::conditional<SYM && !ST, SymSink, NullSink>::type;
            ChainSink ss;
            if constexpr (SYM && !ST) {
                ss.dst = P.sym + gt;
                ss.stride = P.sym_stride;
                ss.cap = owned_t ? P.sym_cap : 0u;
            }
            sync_decode_sink<ST>(ic, s_hi[nt], ch.p, czd_c(ch.czd), czd_z(ch.czd), e2, d2, ss);
            if constexpr (SYM && !ST)
                if (P.sym_cap && owned_t)
                reinterpret_cast<uint4*>(P.tag)[gt] =
                    make_tag(ch.p, czd_c(ch.czd), czd_z(ch.czd), ss.n,
                             !czd_div(e2.czd) && ss.n <= P.sym_cap ? P.epoch : 0u);
            const bool synced = sync_equal(e2.p, e2.czd, s_p[nt], s_czd[nt]);
            s_p[nt] = e2.p;
            s_n[nt] = e2.n;  // the overflow's n is authoritative (:211)
            s_czd[nt] = e2.czd;
            s_dc[nt] = d2;
            if (!synced && !czd_div(e2.czd) && (km >> 31)) {
                const uint32_t slot = atomicAdd(&s_cnt[cur ^ 1], 1u);
                s_list[cur ^ 1][slot] = K1Chain{e2.p, e2.czd, nt + 1};
            }
        }
        __syncthreads();
        cur ^= 1;
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
    // Inter-CTA check: the speculative start (the last speculative thread's entry) against
    // the predecessor's published post-intra last entry; where they differ,
    // the first owned thread re-chains from the published entry (in its own
    // image context) until it meets an entry it agrees with.  HOP waits for
    // the predecessor; otherwise the check is taken only if the predecessor
    // has already published (usually: it started earlier) and the start stays
    // speculative if not.  K1c compares the start used with the predecessor's
    // FINAL last entry.
    if (tid == kK1Spec) {
        Entry start;
        start.p = 0;
        start.n = 0;
        start.czd = 0;
        bool ready = false;
        if (real && si.j > 0) {  // CTA starts mid-segment
            if (HOP)
                while (ld_acquire(P.k1_flag + cta - 1) != P.epoch) spin_pause();
            ready = HOP || ld_acquire(P.k1_flag + cta - 1) == P.epoch;
            if (!ready) {  // K1c's first pass checks the speculative start
                start.p = s_p[kK1Spec - 1];
                start.n = s_n[kK1Spec - 1];
                start.czd = s_czd[kK1Spec - 1] | kBoundaryBit;
            }
        }
        if (ready) {
            start.p = __ldcg(&P.cta_end[cta - 1].p);
            const uint64_t nc = __ldcg(reinterpret_cast<const unsigned long long*>(&P.cta_end[cta - 1]) + 1);
            start.n = uint32_t(nc);
            start.czd = uint32_t(nc >> 32);
            if (!sync_equal(start.p, start.czd, s_p[kK1Spec - 1], s_czd[kK1Spec - 1]) && !czd_div(start.czd)) {
                Entry ch = start;
                uint64_t ii = i;
                uint32_t hops = 0;
                if (ick != k) {
                    load_ctx<ST>(P, D, L, ic, sfast);
                    set_stage(ic, s_stage, s_sm, k);
                }
                for (int tt = kK1Spec; tt < T && ii < si.seg_sub1; ++tt, ++ii) {
                    Entry e2;
                    DcSums d2;
                    sync_decode<ST>(ic, s_hi[tt], ch.p, czd_c(ch.czd), czd_z(ch.czd), e2, d2);
                    ++hops;
                    const bool synced = sync_equal(e2.p, e2.czd, s_p[tt], s_czd[tt]);
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
    if (inb && tid >= kK1Spec) {
        Entry o;
        o.p = s_p[tid];
        o.n = s_n[tid];
        o.czd = s_czd[tid];
        P.ent[g] = o;
        P.dcs[g] = s_dc[tid];
    }
}

// ================================================ K1c: inter fix-up pass ====
// Each CTA j>0 that starts mid-segment chained from a speculative state (the
// predecessor's last subsequence decoded from its origin).  Where that
// differs from the predecessor's final entry, CTA j's overflow is redone from
// the final state until it meets an entry it agrees with; a redo that runs
// through the whole CTA changes CTA j's last entry and stales CTA j+1 — the
// reference's `end_changed` invalidation (parallel_decode.hpp:272-276).

// Redoes CTA cta's overflow from start state st (its predecessor's final
// last entry) until it meets an entry it agrees with.
template <bool ST = false>
__device__ __forceinline__ void k1c_redo(const Params& P, uint32_t cta, Entry st, unsigned long long& redone,
                                         int32_t* s_acc, const uint32_t* sfast = nullptr) {
    constexpr int TO = kK1Own;
    const uint64_t g0 = uint64_t(cta) * TO;
    const uint32_t k = find_img(P, g0);
    const ImgDesc& D = P.img[k];
    const uint64_t L = P.ist[k].bit_length;
    uint64_t i = g0 - P.sub_first[k];
    if (czd_div(st.czd)) {
        set_status(P.ist + k, kConsistencyFailure);
        return;
    }
    SubInfo si;
    if (!sub_info(P, D, L, i, si)) return;
    ImgCtx ic;
    load_ctx<ST>(P, D, L, ic, sfast);
    set_sacc(ic, s_acc, threadIdx.x, blockDim.x);
    Entry ch = st;
    for (int tt = 0; tt < TO && i < si.seg_sub1 && g0 + tt < P.total_subs; ++tt, ++i) {
        Entry e2;
        DcSums d2;
        sync_decode<ST>(ic, seg_end_bit(si, P.sb, i), ch.p, czd_c(ch.czd), czd_z(ch.czd), e2, d2);
        ++redone;
        Entry old = P.ent[g0 + tt];
        bool synced = sync_equal(e2.p, e2.czd, old.p, old.czd);
        P.ent[g0 + tt] = e2;
        P.dcs[g0 + tt] = d2;
        if (synced || czd_div(e2.czd)) break;
        ch = e2;
    }
}

// First pass, one thread per CTA boundary (all stale boundaries in parallel):
// CTA starts are speculative when K1 ran without the in-kernel check.  A
// redo that runs through a whole CTA races with its successor's check; the
// fix-point pass below catches that (it compares against the final entries).
// ST: the batch's fast tables are staged in shared memory (a redo chain is a
// serial dependency chain, and this kernel's L1 starts cold).
template <bool ST>
__global__ void __launch_bounds__(128) k1c_first(Params P) {
    pdl_wait();
    const uint32_t cta = 1 + blockIdx.x * blockDim.x + threadIdx.x;
    __shared__ int32_t s_acc[3 * 128];
    extern __shared__ uint32_t s_fast_k1c[];
    const uint32_t* sfast = ST ? stage_tables(P, s_fast_k1c, threadIdx.x, 128, P.n_huff) : nullptr;
    if (ST) __syncthreads();
    unsigned long long redone = 0;
    if (cta < P.k1_ctas) {
        const Entry st = P.cta_start[cta];
        if (st.czd & kBoundaryBit) {
            Entry pe = P.ent[uint64_t(cta) * kK1Own - 1];
            if (!sync_equal(st.p, st.czd, pe.p, pe.czd)) {
                pe.czd |= kBoundaryBit;
                P.cta_start[cta] = pe;
                k1c_redo<ST>(P, cta, pe, redone, s_acc, sfast);
            }
        }
    }
    if (redone) atomicAdd(P.stats + kStatInterHops, redone);
}

// Fix-point passes (one CTA): repeat until no boundary is stale.
__global__ void __launch_bounds__(1024) k1c_fixup(Params P) {
    pdl_wait();
    constexpr int TO = kK1Own;
    __shared__ int s_any;
    __shared__ int32_t s_acc[3 * 1024];
    __shared__ int s_passes;
    if (threadIdx.x == 0) s_passes = 0;
    unsigned long long redone = 0;
    for (uint32_t pass = 0; pass <= P.k1_ctas; ++pass) {
        if (threadIdx.x == 0) s_any = 0;
        __syncthreads();
        // snapshot: which boundaries are stale (start used != final predecessor end)
        for (uint32_t cta = 1 + threadIdx.x; cta < P.k1_ctas; cta += blockDim.x) {
            Entry st = P.cta_start[cta];
            if (!(st.czd & kBoundaryBit)) continue;
            Entry pe = P.ent[uint64_t(cta) * TO - 1];
            if (!sync_equal(st.p, st.czd, pe.p, pe.czd)) {
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
            k1c_redo(P, cta, st, redone, s_acc);
        }
        __threadfence_block();
        __syncthreads();
    }
    if (redone) atomicAdd(P.stats + kStatInterHops, redone);
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
    uint32_t ek;    // coded coefficients (compact entries)
};
constexpr uint64_t kHead = 1ull << 63;

__device__ __forceinline__ ScanVal scan_op(const ScanVal& a, const ScanVal& b) {
    // a precedes b
    ScanVal r;
    if (b.n & kHead) return b;
    r.n = ((a.n & ~kHead) + b.n) | (a.n & kHead);
    r.lo = __vadd2(a.lo, b.lo);
    r.hi = __vadd2(a.hi, b.hi);
    r.ek = a.ek + b.ek;
    return r;
}

__global__ void __launch_bounds__(kK2Threads) k2_scan(Params P) {
    pdl_wait();
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
    uint32_t k = find_img(P, inb ? g : P.total_subs - 1);
    const uint64_t i = g - P.sub_first[k];
    const ImgDesc& D = P.img[k];
    // segment heads: the image start, or (restart intervals) each interval's
    // first subsequence; subsequences past the last one are inert heads
    const bool dri = D.n_int > 1;
    SubInfo si;
    bool real = true;
    if (dri) real = P.ist[k].status == 0 && sub_info(P, D, P.ist[k].bit_length, i, si);
    ScanVal v;
    v.n = 0;
    v.lo = v.hi = v.ek = 0;
    if (inb) {
        Entry e = P.ent[g];
        DcSums d = P.dcs[g];
        v.n = e.n;
        v.lo = d.lo;
        v.hi = d.hi & 0xFFFFu;
        v.ek = d.hi >> 16;
        if (!dri ? i == 0 : (!real || si.j == 0)) v.n |= kHead;
        if (!real) v.n = kHead, v.lo = v.hi = v.ek = 0;
    }
    // warp inclusive segmented scan
    ScanVal x = v;
    for (int o = 1; o < 32; o <<= 1) {
        ScanVal y;
        y.n = __shfl_up_sync(0xFFFFFFFFu, x.n, o);
        y.lo = __shfl_up_sync(0xFFFFFFFFu, x.lo, o);
        y.hi = __shfl_up_sync(0xFFFFFFFFu, x.hi, o);
        y.ek = __shfl_up_sync(0xFFFFFFFFu, x.ek, o);
        if (lane >= o) x = scan_op(y, x);
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    ScanVal wpre;  // exclusive prefix of earlier warps in this tile
    wpre.n = 0;
    wpre.lo = wpre.hi = wpre.ek = 0;
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
        ex.lo = ex.hi = ex.ek = 0;
        const bool own_prefix = (incl.n & kHead) != 0;
        const bool need = t > 0 && !s_first_head;
        if (own_prefix || !need) {
            agg[4] = incl.n;
            agg[5] = (uint64_t(incl.hi) << 32) | incl.lo;
            agg[6] = incl.ek;
            __threadfence();
            st_release(P.k2_flag + t, (P.epoch << 2) | 2u);
        } else {
            agg[0] = incl.n;
            agg[1] = (uint64_t(incl.hi) << 32) | incl.lo;
            agg[2] = incl.ek;
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
                pv.ek = uint32_t(__ldcg(src + 2));
                ex = first ? pv : scan_op(pv, ex);
                first = false;
                if ((f & 3u) == 2u || (pv.n & kHead)) break;
                --pr;
            }
            if (!own_prefix) {
                ScanVal ti = scan_op(ex, incl);
                agg[4] = ti.n;
                agg[5] = (uint64_t(ti.hi) << 32) | ti.lo;
                agg[6] = ti.ek;
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
        xup.ek = __shfl_up_sync(0xFFFFFFFFu, x.ek, 1);
        bool have = false;
        wx.n = 0;
        wx.lo = wx.hi = wx.ek = 0;
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
        before.lo = before.hi = before.ek = 0;
    }
    // trimmed offsets (offsets(), parallel_decode.hpp:290-316), per segment:
    // a restart interval expects 64 * dpm * (its MCUs) slots at slot base
    // 64 * dpm * Ri * m
    uint64_t E = D.expected, base = 0;
    bool last = i + 1 == D.sub_count;
    if (dri) {
        if (!real) {
            P.off[g] = 0;
            P.cap[g] = 0;
            P.pred[g] = DcSums{0, 0};
            if (P.compact) P.eoff[g] = 0;
            return;
        }
        const uint64_t mcus = uint64_t(D.mcus_x) * D.mcus_y;
        const uint64_t m0 = uint64_t(si.m) * D.ri;
        E = 64ull * D.dpm * min64(D.ri, mcus - m0);
        base = 64ull * D.dpm * m0;
        last = i + 1 == si.seg_sub1;
    }
    const uint64_t pre = before.n & ~kHead;
    const uint64_t n = v.n & ~kHead;
    const uint64_t o = min(pre, E);
    P.off[g] = base + o;
    P.cap[g] = uint32_t(min(pre + n, E) - o);
    // entries of a restart interval start at its slot base (entries <= slots)
    if (P.compact) P.eoff[g] = uint32_t(base) + before.ek;
    DcSums pd;
    pd.lo = before.lo;
    pd.hi = before.hi;
    P.pred[g] = pd;
    if (last && P.ist[k].status == 0) {
        const uint64_t total = pre + n;
        if (total < E || total - E > 512) set_status(P.ist + k, kConsistencyFailure);
    }
}

// ============================================ K1x: reference-exact replay ====
// The fast path (K1..K3) is exact whenever the scan decodes without error on
// its true path: the synchronised decomposition is then unique and every
// grouping of subsequences finds it.  For corrupt scans the reference's
// outcome depends on HOW it synchronises (which speculative chain wrote an
// entry last, which divergent n survives), and on semantics valid scans never
// reach (an AC run overflowing the block, parallel_decode.hpp:144-162: the
// coefficient lands in the next unit's slots, z resets with c += 1 only, and
// dc_prefix_sum then adds whatever sits in slot 0 of each unit).
// Images whose entropy stage failed, or whose K3 saw a run overflow, are
// re-decoded here by one CTA each, restating the reference literally at the
// configured partition (sb, b): sync_intra_sequence in lock-step rounds
// (parallel_decode.hpp:171-222), sync_inter_sequence passes with the snapshot /
// end_changed / progress rules (:227-285), offsets() (:290-316), write_output
// (:321-330) with worker_count = 1 error order (the lowest failing
// subsequence), dc_prefix_sum (transform.hpp:56-74); then the unit metadata
// K4 reads.  One reference behaviour cannot be restated: when a pass changes
// nothing and sets no flag while some flag stays unset, the reference loops
// forever (`progressed` stays true, :277-283); the replay reports
// ConsistencyFailure there.  Off the hot path: a launch finds no work for
// valid batches.
constexpr int kK1xThreads = 256;
constexpr uint32_t kExactFlag = 1u;  // ImgState::exact: K3 saw a run past the unit end
constexpr uint32_t kActiveBit = 1u << 20;

struct RefSym {
    int32_t err;   // 0, kOutOfBits, kInvalidCode
    uint32_t len;  // code + magnitude bits
    uint32_t run;  // run_length (EOB: 63 - z)
    int32_t coef;
    bool is_coef;  // Kind::Coefficient
    bool eob;
};

// bits [p, p + 24) MSB first, zero past the segment end (BitCursor::peek_bits)
__device__ __forceinline__ uint32_t ref_peek24(const uint8_t* seg, uint64_t L, uint64_t p) {
    const uint64_t nbytes = L >> 3;
    const uint64_t b0 = p >> 3;
    uint32_t w = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) w = (w << 8) | (b0 + k < nbytes ? uint32_t(seg[b0 + k]) : 0u);
    w <<= uint32_t(p & 7);
    // bits at or past L are zero (L is a multiple of 8: whole bytes)
    return w >> 8;
}
__device__ __forceinline__ uint32_t ref_read(const uint8_t* seg, uint64_t L, uint64_t p, uint32_t l) {
    return l ? ref_peek24(seg, L, p) >> (24 - l) : 0u;
}

// decode_next_symbol (huffman.hpp:137-175) with decode_codeword (:113-131)
__device__ RefSym ref_symbol(const uint8_t* seg, uint64_t L, uint64_t p, uint32_t z, const DevHuff* dc,
                             const DevHuff* ac) {
    RefSym r{0, 0, 0, 0, false, false};
    const uint64_t avail = L - p;
    if (avail == 0) {
        r.err = kOutOfBits;
        return r;
    }
    const DevHuff* t = z == 0 ? dc : ac;
    const uint32_t w16 = ref_peek24(seg, L, p) >> 8;
    uint32_t maxlen;
    const uint32_t e = dev_lookup(t, w16, maxlen);
    const uint32_t clen = e >> 8, sym = e & 255u;
    if (clen == 0) {
        r.err = avail < maxlen ? kOutOfBits : kInvalidCode;
        return r;
    }
    if (clen > avail) {
        r.err = kOutOfBits;
        return r;
    }
    const uint64_t p2 = p + clen;
    uint32_t l;
    if (z == 0) {
        l = sym;
        if (l > 11) {
            r.err = kInvalidCode;
            return r;
        }
        r.is_coef = true;
    } else {
        const uint32_t rr = sym >> 4;
        l = sym & 15u;
        if (l == 0) {
            if (rr == 0) {
                r.eob = true;
                r.run = 63 - z;
            } else if (rr == 15) {
                r.run = 15;
            } else {
                r.err = kInvalidCode;
            }
            r.len = clen;
            return r;
        }
        if (l > 10) {
            r.err = kInvalidCode;
            return r;
        }
        r.run = rr;
        r.is_coef = true;
    }
    if (L - p2 < l) {
        r.err = kOutOfBits;
        return r;
    }
    const uint32_t bits = ref_read(seg, L, p2, l);
    r.coef = l == 0 ? 0 : (bits >= (1u << (l - 1)) ? int32_t(bits) : int32_t(bits) - int32_t((1u << l) - 1));
    r.len = clen + l;
    return r;
}

struct RefImg {
    const uint8_t* seg;
    uint64_t L, sb, N;
    uint32_t dpm;
    uint64_t du_comp;
    const DevHuff* dc[3];
    const DevHuff* ac[3];
};

// decode_subsequence (parallel_decode.hpp:122-164).  Sync mode: returns the
// end state (divergent at the last good state on an error).  Write mode
// (coef != nullptr): coefficients at slot out_off + local + run of the
// image's column-major unit buffer, stops at cap; returns the error code.
__device__ int32_t ref_subsequence(const RefImg& I, uint64_t i, uint64_t& p, uint32_t& c, uint32_t& z, uint64_t& n,
                                   bool& div, int16_t* coef, uint64_t out_off, uint64_t cap) {
    const uint64_t end_bit = min64((i + 1) * I.sb, I.L);
    n = 0;
    div = false;
    uint64_t local = 0;
    while (p < end_bit) {
        if (coef && local >= cap) break;
        const uint32_t comp = uint32_t(I.du_comp >> (4 * c)) & 15u;
        const RefSym s = ref_symbol(I.seg, I.L, p, z, I.dc[comp], I.ac[comp]);
        if (s.err) {
            if (coef) return s.err;
            div = true;
            return 0;
        }
        const uint64_t step = uint64_t(s.run) + 1;
        if (coef) {
            if (local + step > cap) break;
            if (s.is_coef) {
                const uint64_t slot = out_off + local + s.run;
                coef[(slot >> 6) * 64 + c_zz2c[slot & 63]] = int16_t(s.coef);
            }
        }
        p += s.len;
        n += step;
        local += step;
        z += uint32_t(step);
        if (z >= 64 || s.eob) {
            z = 0;
            c = (c + 1 == I.dpm) ? 0 : c + 1;
        }
    }
    return 0;
}

// CTA-wide helpers (kK1xThreads threads)
__device__ __forceinline__ unsigned long long cta_sum_u64(unsigned long long v, unsigned long long* red) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    unsigned long long t = 0;
    for (int w = 0; w < kK1xThreads / 32; ++w) t += red[w];
    __syncthreads();
    return t;
}

__device__ void k1x_image(const Params& P, uint32_t k, unsigned long long* red) {
    const int tid = threadIdx.x;
    const ImgDesc& D = P.img[k];
    ImgState* st = P.ist + k;
    RefImg I;
    I.seg = P.ubuf + D.raw_off;
    I.L = st->bit_length;
    I.sb = P.sb_cfg;
    I.N = (I.L + I.sb - 1) / I.sb;
    I.dpm = D.dpm;
    I.du_comp = D.du_comp;
    for (int cc = 0; cc < 3; ++cc) {
        I.dc[cc] = P.huff + D.dc_tab[cc];
        I.ac[cc] = P.huff + D.ac_tab[cc];
    }
    const uint64_t N = I.N, b = P.b_cfg, B = (N + b - 1) / b;
    const uint64_t base = D.sub_first;
    Entry* E = P.ent + base;                 // info.entries
    uint64_t* Wp = P.off + base;             // worker chain p / later offsets
    uint32_t* Wc = P.cap + base;             // worker chain c, z, div | active
    uint64_t* Sp = reinterpret_cast<uint64_t*>(P.pred + base);  // inter: start snapshot p
    DcSums* Sf = P.dcs + base;               // inter: .lo start czd, .hi flags
    __shared__ int s_any;
    __shared__ unsigned long long s_err;
    if (tid == 0) s_err = ~0ull;

    // ---- sync_intra_sequence: every sequence's workers in lock-step rounds
    for (uint64_t i = tid; i < N; i += kK1xThreads) {
        uint64_t p = i * I.sb, n;
        uint32_t c = 0, z = 0;
        bool div;
        ref_subsequence(I, i, p, c, z, n, div, nullptr, 0, 0);
        E[i].p = p;
        E[i].n = uint32_t(n);
        E[i].czd = pack_czd(c, z, div);
        const uint64_t last = min64((i / b + 1) * b, N) - 1;
        Wp[i] = p;
        Wc[i] = pack_czd(c, z, div) | (!div && i < last ? kActiveBit : 0u);
    }
    for (uint64_t r = 1;; ++r) {
        __syncthreads();
        int any = 0;
        for (uint64_t i = tid; i < N; i += kK1xThreads) {
            uint32_t w = Wc[i];
            if (!(w & kActiveBit)) continue;
            const uint64_t nx = i + r, last = min64((i / b + 1) * b, N) - 1;
            if (nx > last) {
                Wc[i] = w & ~kActiveBit;
                continue;
            }
            uint64_t p = Wp[i], n;
            uint32_t c = czd_c(w), z = czd_z(w);
            bool div;
            ref_subsequence(I, nx, p, c, z, n, div, nullptr, 0, 0);
            const Entry old = E[nx];
            const uint32_t czd = pack_czd(c, z, div);
            const bool synced = czd_div(old.czd) == div && sync_equal(p, czd, old.p, old.czd);
            E[nx].p = p;
            E[nx].n = uint32_t(n);
            E[nx].czd = czd;
            if (synced || div) {
                Wc[i] = czd;
            } else {
                Wp[i] = p;
                Wc[i] = czd | kActiveBit;
                any = 1;
            }
        }
        if (!__syncthreads_or(any)) break;
    }

    // ---- sync_inter_sequence: snapshot passes until every flag is set
    if (B > 1) {
        for (uint64_t g = tid; g + 1 < B; g += kK1xThreads) Sf[g].hi = 0;  // bit 0 synced, 1 changed, 2 end_changed
        for (uint64_t pass = 0;; ++pass) {
            __syncthreads();
            if (pass > 2 * B + 64) {  // bounded: the reference has no such bound but converges far earlier on any scan seen
                if (tid == 0) st->status = kConsistencyFailure;
                return;
            }
            int unsynced = 0;
            for (uint64_t g = tid; g + 1 < B; g += kK1xThreads) unsynced |= !(Sf[g].hi & 1u);
            if (!__syncthreads_or(unsynced)) break;
            for (uint64_t g = tid; g + 1 < B; g += kK1xThreads) {
                const Entry e = E[min64((g + 1) * b, N) - 1];
                Sp[g] = e.p;
                Sf[g].lo = e.czd;
                Sf[g].hi &= 1u;
            }
            __syncthreads();
            int newly = 0;
            for (uint64_t g = tid; g + 1 < B; g += kK1xThreads) {
                uint32_t f = Sf[g].hi;
                if (f & 1u) continue;
                uint64_t p = Sp[g];
                uint32_t czd0 = Sf[g].lo;
                if (czd_div(czd0)) continue;
                uint32_t c = czd_c(czd0), z = czd_z(czd0);
                const uint64_t first = (g + 1) * b, last = min64(first + b, N) - 1;
                for (uint64_t j = first; j <= last; ++j) {
                    uint64_t n;
                    bool div;
                    ref_subsequence(I, j, p, c, z, n, div, nullptr, 0, 0);
                    const Entry old = E[j];
                    const uint32_t czd = pack_czd(c, z, div);
                    const bool synced = czd_div(old.czd) == div && sync_equal(p, czd, old.p, old.czd);
                    if (!synced || uint32_t(n) != old.n) {
                        f |= 2u;
                        if (j == last) f |= 4u;
                    }
                    E[j].p = p;
                    E[j].n = uint32_t(n);
                    E[j].czd = czd;
                    if (synced) {
                        f |= 1u;
                        newly = 1;
                        break;
                    }
                    if (div) break;
                }
                Sf[g].hi = f;
            }
            __syncthreads();
            // end_changed invalidates the successor's flag (:271-276)
            int progressed = 0, changed = 0;
            for (uint64_t g = tid; g + 1 < B; g += kK1xThreads) {
                const uint32_t f = Sf[g].hi;
                changed |= (f & 2u) ? 1 : 0;
                progressed |= (f & 3u) ? 1 : 0;
            }
            __syncthreads();
            for (uint64_t g = tid; g + 2 < B; g += kK1xThreads)
                if (Sf[g].hi & 4u) atomicAnd(&Sf[g + 1].hi, ~1u);
            progressed = __syncthreads_or(progressed);
            const int moved = __syncthreads_or(changed | newly);
            if (!progressed || !moved) {  // fixpoint with unset flags (or the reference's endless loop)
                if (tid == 0) st->status = kConsistencyFailure;
                return;
            }
        }
    }
    __syncthreads();

    // ---- offsets(): count check, tail trim, exclusive scan
    const uint64_t expected = D.expected;
    unsigned long long raw = 0;
    for (uint64_t i = tid; i < N; i += kK1xThreads) raw += E[i].n;
    raw = cta_sum_u64(raw, red);
    if (raw < expected || raw - expected > 512) {
        if (tid == 0) st->status = kConsistencyFailure;
        return;
    }
    if (tid == 0) {
        uint64_t excess = raw - expected;
        for (uint64_t q = N; q-- > 0 && excess > 0;) {
            const uint64_t d = min64(excess, E[q].n);
            E[q].n -= uint32_t(d);
            excess -= d;
        }
    }
    __syncthreads();
    {  // exclusive scan of n over contiguous per-thread chunks
        const uint64_t per = (N + kK1xThreads - 1) / kK1xThreads;
        const uint64_t lo = min64(uint64_t(tid) * per, N), hi = min64(lo + per, N);
        unsigned long long mine = 0;
        for (uint64_t i = lo; i < hi; ++i) mine += E[i].n;
        __shared__ unsigned long long s_pre[kK1xThreads];
        s_pre[tid] = mine;
        __syncthreads();
        if (tid == 0) {
            unsigned long long a = 0;
            for (int t = 0; t < kK1xThreads; ++t) {
                const unsigned long long v = s_pre[t];
                s_pre[t] = a;
                a += v;
            }
        }
        __syncthreads();
        unsigned long long a = s_pre[tid];
        for (uint64_t i = lo; i < hi; ++i) {
            Wp[i] = a;
            a += E[i].n;
        }
    }

    // ---- write_output into the zeroed unit buffer (worker_count 1: lowest failing i)
    const uint64_t dus = expected / 64;
    int16_t* coef = P.coef + D.du_first * 64;
    for (uint64_t x = tid; x < dus * 8; x += kK1xThreads) reinterpret_cast<int4*>(coef)[x] = make_int4(0, 0, 0, 0);
    __syncthreads();
    for (uint64_t i = tid; i < N; i += kK1xThreads) {
        const uint64_t cap = E[i].n;
        if (cap == 0) continue;
        uint64_t p = 0, n;
        uint32_t c = 0, z = 0;
        bool div;
        if (i > 0) {
            const Entry e = E[i - 1];
            p = e.p;
            c = czd_c(e.czd);
            z = czd_z(e.czd);
        }
        const int32_t err = ref_subsequence(I, i, p, c, z, n, div, coef, Wp[i], cap);
        if (err) atomicMin(&s_err, (unsigned long long)(i << 8) | uint32_t(err));
    }
    __syncthreads();
    if (s_err != ~0ull) {
        if (tid == 0) st->status = int32_t(s_err & 0xFFu);
        return;
    }

    // ---- dc_prefix_sum: per component over the units in scan order (slot 0
    // of every unit, whatever the decode put there), int16 wrap; chunked scan
    {
        const uint64_t per = (dus + kK1xThreads - 1) / kK1xThreads;
        const uint64_t lo = min64(uint64_t(tid) * per, dus), hi = min64(lo + per, dus);
        __shared__ uint32_t s_dc[kK1xThreads][3];
        uint32_t a[3] = {0, 0, 0};
        for (uint64_t d = lo; d < hi; ++d) a[uint32_t(I.du_comp >> (4 * (d % I.dpm))) & 15u] += uint16_t(coef[d * 64]);
        for (int cc = 0; cc < 3; ++cc) s_dc[tid][cc] = a[cc];
        __syncthreads();
        if (tid < 3) {
            uint32_t acc = 0;
            for (int t = 0; t < kK1xThreads; ++t) {
                const uint32_t v = s_dc[t][tid];
                s_dc[t][tid] = acc;
                acc += v;
            }
        }
        __syncthreads();
        for (int cc = 0; cc < 3; ++cc) a[cc] = s_dc[tid][cc];
        // the first unit of each chain stays as stored: acc starts at it (mod 2^16 the same)
        for (uint64_t d = lo; d < hi; ++d) {
            const uint32_t cc = uint32_t(I.du_comp >> (4 * (d % I.dpm))) & 15u;
            a[cc] += uint16_t(coef[d * 64]);
            coef[d * 64] = int16_t(uint16_t(a[cc]));
        }
    }
    __syncthreads();

    // ---- K4's per-unit metadata (as K3's BlockSink): nonzero column mask |
    // has-AC << 8 | nonzero row mask << 16, S = sum w_u w_v Q |F|
    for (uint64_t d = tid; d < dus; d += kK1xThreads) {
        const uint32_t comp = uint32_t(I.du_comp >> (4 * (d % I.dpm))) & 15u;
        const float* wq = P.wq + 64u * D.q_tab[comp];
        const int16_t* u = coef + d * 64;
        uint32_t flags = 0;
        float S = 0.f;
        // compact batches: this unit's entries at the fixed slot range [64 d, 64 d + 64)
        uint32_t* ce = P.compact ? P.ents + (D.du_first + d) * 64 : nullptr;
        uint32_t ne = 0;
        for (int zz = 0; zz < 64; ++zz) {
            const uint32_t cm = c_zz2c[zz];
            const int32_t v = u[cm];
            if (ce && (v != 0 || zz == 0)) ce[ne++] = (uint32_t(d & 0xFFu) << 22) | (cm << 16) | (uint32_t(v) & 0xFFFFu);
            if (v != 0) {
                flags |= (1u << (cm >> 3)) | (zz ? (1u << 8) : 0u) | (1u << (16 + (cm & 7)));
                S = fmaf(wq[zz], float(abs(v)), S);
            }
        }
        if (ce)
            P.umeta[D.du_first + d] = make_uint4(uint32_t(64 * d), uint32_t(64 * d) + ne, flags, __float_as_uint(S));
        else
            P.meta[D.du_first + d] = make_uint2(flags, __float_as_uint(S));
    }
}

__global__ void __launch_bounds__(kK1xThreads) k1x_exact(Params P) {
    pdl_wait();
    __shared__ unsigned long long red[kK1xThreads / 32];
    for (uint32_t k = blockIdx.x; k < P.n_img; k += gridDim.x) {
        const ImgState s = P.ist[k];
        const ImgDesc& D = P.img[k];
        const bool entropy_fail = s.status == kOutOfBits || s.status == kInvalidCode || s.status == kConsistencyFailure;
        if (!(entropy_fail || (s.status == 0 && (s.exact & kExactFlag))) || D.n_int > 1 || D.deferred || !D.expected)
            continue;
        __syncthreads();
        if (threadIdx.x == 0) {
            P.ist[k].status = 0;
            P.ist[k].exact |= 2u;
        }
        __syncthreads();
        k1x_image(P, k, red);
        __syncthreads();
    }
}

// ======================================================= K3: write pass ====
// Each thread re-decodes its subsequence from the synchronised state and
// stages the current data unit in a private shared-memory block (column-major,
// stride 72 int16 → conflict-free 16-byte rows).  The decoder signals block
// ends: a block this thread owns entirely leaves as 4 full-sector 32-byte
// stores; the first / last blocks shared with a neighbouring subsequence write
// only the owned slots.
//
// Per data unit K3 also emits K4's metadata (it sees the few nonzero
// coefficients as it decodes them; K4 would have to scan all 64):
//   flags = nonzero-column mask | has-AC << 8 | nonzero-row mask << 16, and
//   S = sum over nonzero F of w_u w_v |F| (bounds |r| and the FP32 IDCT error;
//   w_u = max_x |basis[u][x]|, weights x quantiser precomputed per table).
// Units split between two subsequences combine through atomics into the
// buffer zeroed before K3.
constexpr int kBlkStride = 72;
constexpr uint32_t kK3SmemQuant = 4;  // quant tables staged in shared memory
constexpr uint32_t kMetaNonDc = 1u << 8;

struct BlockSink {
    static constexpr bool kWrite = true;
    static constexpr bool kStore = false;
    static constexpr bool kSmemAcc = false;  // DC accumulators in registers, swapped at block ends
    __device__ __forceinline__ void sym(uint32_t) {}
    const uint32_t* zt;  // smem, per zig-zag k: column-major index | (column bit | nonDC) << 8
    const float* wqb;    // the batch's wq rows
    uint64_t qrow;       // per component (21 bits each): its wq row
    int16_t* buf;        // this thread's smem block
    int16_t* coef;       // batch coefficient buffer
    uint2* meta;         // batch per-unit metadata
    uint64_t du;         // batch data unit of the current block
    uint64_t slot0;      // image-relative slot of the current block's first coefficient
    uint64_t own_hi;     // owned slots end (image-relative)
    const float* wqc;    // wq row of the current block's component
    uint32_t klo;        // first owned zig-zag position of the current block
    uint32_t mflags;     // metadata of the current unit (owned part)
    float mS;

    __device__ __forceinline__ void set_comp(uint32_t comp) { wqc = wqb + 64u * uint32_t((qrow >> (21 * comp)) & 0x1FFFFFu); }
    __device__ __forceinline__ void put(uint32_t k, int32_t v) {
        const uint32_t t = zt[k];
        buf[t & 0xFFu] = int16_t(v);
        if (v != 0) {
            mflags |= t >> 8;
            mS = fmaf(wqc[k], float(abs(v)), mS);
        }
    }
    // flush the owned zig-zag range [klo, khi) of the current block and move on
    __device__ __forceinline__ void flush(uint32_t khi) {
        int16_t* dst = coef + du * 64;
        uint2* md = meta + du;
        // only the columns holding a nonzero coefficient (mflags bits 0-7) are
        // read back and re-zeroed: the rest of the staging block is zero
        const uint32_t cm = mflags & 0xFFu;
        if (klo == 0 && khi == 64) {
            // full-sector 256-bit stores (STG.E.ENL2.256): no partial-sector merges in L2
            const int4* s4 = reinterpret_cast<const int4*>(buf);
            const int4 z4 = make_int4(0, 0, 0, 0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int4 a = (cm >> (2 * q)) & 1u ? s4[2 * q] : z4;
                const int4 c = (cm >> (2 * q + 1)) & 1u ? s4[2 * q + 1] : z4;
                asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + 16 * q), "r"(a.x),
                             "r"(a.y), "r"(a.z), "r"(a.w), "r"(c.x), "r"(c.y), "r"(c.z), "r"(c.w)
                             : "memory");
            }
            *md = make_uint2(mflags, __float_as_uint(mS));
        } else {
            for (uint32_t k = klo; k < khi; ++k) {
                const uint32_t r = zt[k] & 0xFFu;
                dst[r] = buf[r];
            }
            if (mflags) atomicOr(&md->x, mflags);
            if (mS != 0.f) atomicAdd(reinterpret_cast<float*>(&md->y), mS);
        }
        const int4 zero = make_int4(0, 0, 0, 0);
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if ((cm >> q) & 1u) reinterpret_cast<int4*>(buf)[q] = zero;
        mflags = 0;
        mS = 0.f;
        klo = 0;
        ++du;
        slot0 += 64;
    }
    // the decoder completed the current block (all of it from klo on is owned)
    __device__ __forceinline__ void block_end(uint32_t next_comp) {
        flush(64);
        set_comp(next_comp);
    }
    // the owned slots left after the last decoded symbol (zeros past it)
    __device__ __forceinline__ void finish() {
        while (slot0 < own_hi) flush(uint32_t(min64(64, own_hi - slot0)));
    }
};

// Compact interface (Params::compact): one 32-bit entry per coded coefficient
// (col-major index << 16 | value; DC absolute, written even when 0 so that
// it marks the unit start), written sequentially from the subsequence's
// entry offset (K2), plus per unit (first entry, end entry, flags, S).  A
// unit split between subsequences: the DC owner writes the first entry, the
// thread owning slot 63 the end; flags and S combine through atomics (the
// metadata buffer is zeroed before K3).  No staging block, no zero slots.
struct EntrySink {
    static constexpr bool kWrite = true;
    static constexpr bool kStore = false;
    static constexpr bool kSmemAcc = false;  // (shared-memory accumulators measured slower: write 1.20 -> 1.25 ms)
    __device__ __forceinline__ void sym(uint32_t) {}
    const uint32_t* zt;  // smem, per zig-zag k: column-major index | (column bit | nonDC | row bit) << 8
    const float* wqb;
    uint64_t qrow;
    const float* wqc;
    uint32_t* ent;       // the image's entries (ents + 64 du_first)
    uint4* um;           // the image's unit metadata
    uint32_t u;          // image-relative current unit
    uint32_t pos;        // image-relative next entry
    uint32_t ustart;     // entry of the current unit's DC (klo == 0)
    uint64_t slot0;      // image-relative slot of the current unit's first coefficient
    uint64_t own_hi;     // owned slots end (image-relative)
    uint32_t klo;        // first owned zig-zag position of the current unit
    uint32_t mflags;
    float mS;

    __device__ __forceinline__ void set_comp(uint32_t comp) { wqc = wqb + 64u * uint32_t((qrow >> (21 * comp)) & 0x1FFFFFu); }
    __device__ __forceinline__ void put(uint32_t k, int32_t v) {
        // branch-free (lanes diverge on every condition here); a zero term adds
        // +0 to S exactly, and only a DC entry can be zero
        const uint32_t t = zt[k];
        ustart = k == 0 ? pos : ustart;
        ent[pos++] = ((u & 0xFFu) << 22) | ((t & 0xFFu) << 16) | (uint32_t(v) & 0xFFFFu);
        mflags |= v != 0 ? (t >> 8) : 0u;
        mS = fmaf(wqc[k], float(abs(v)), mS);
    }
    // the owned part of the current unit ends (complete: through slot 63)
    __device__ __forceinline__ void close(bool complete) {
        uint4* m = um + u;
        if (klo == 0 && complete) {
            *m = make_uint4(ustart, pos, mflags, __float_as_uint(mS));
        } else {
            if (klo == 0) m->x = ustart;
            if (complete) m->y = pos;
            if (mflags) atomicOr(&m->z, mflags);
            if (mS != 0.f) atomicAdd(reinterpret_cast<float*>(&m->w), mS);
        }
        mflags = 0;
        mS = 0.f;
        klo = 0;
        ++u;
        slot0 += 64;
    }
    __device__ __forceinline__ void block_end(uint32_t next_comp) {
        close(true);
        set_comp(next_comp);
    }
    __device__ __forceinline__ void finish() {
        while (slot0 < own_hi) close(own_hi - slot0 >= 64);
    }
};

template <bool ST, bool REPLAY, bool CMP>
__global__ void __launch_bounds__(kK3Threads, 5) k3_write(Params P) {
    pdl_wait();
    __shared__ __align__(16) int16_t s_blk[CMP ? 8 : kK3Threads * kBlkStride];
    __shared__ uint32_t s_zt[64];
    __shared__ float s_wq[kK3SmemQuant * 64];  // the batch's metadata weights when they fit
    const int tid = threadIdx.x;
    if (tid < 64) {
        const uint32_t c = c_zz2c[tid];
        s_zt[tid] = c | (((1u << (c >> 3)) | (tid ? kMetaNonDc : 0u) | (1u << (16 + (c & 7)))) << 8);
    }
    const bool wq_smem = P.n_quant <= kK3SmemQuant;
    if (wq_smem)
        for (uint32_t x = tid; x < P.n_quant * 64; x += kK3Threads) s_wq[x] = P.wq[x];
    int16_t* buf = s_blk + (CMP ? 0 : tid * kBlkStride);
    if (!CMP) {
        const int4 zero = make_int4(0, 0, 0, 0);
#pragma unroll
        for (int q = 0; q < 8; ++q) reinterpret_cast<int4*>(buf)[q] = zero;
    }
    const uint64_t g = uint64_t(blockIdx.x) * kK3Threads + tid;
    const bool inb = g < P.total_subs;
    const uint32_t cap = inb ? P.cap[g] : 0u;
    const uint32_t k = find_img(P, inb ? g : P.total_subs - 1);
    const ImgDesc& D = P.img[k];
    const uint64_t i = g - P.sub_first[k];
    const uint64_t L = P.ist[k].bit_length;
    SubInfo si;
    const bool active = inb && cap != 0 && P.ist[k].status == 0 && sub_info(P, D, L, i, si);
    extern __shared__ uint32_t s_fast_k3[];
    ImgCtx ic;
    load_ctx<ST>(P, D, L, ic, ST ? stage_tables(P, s_fast_k3, tid, kK3Threads, P.k3_tables) : nullptr);
    ic.sacc = nullptr;  // write mode keeps its DC accumulators in registers
    ic.sacc_stride = 0;
    DecState s;
    s.p = 0;
    s.c = s.z = 0;
    if (active) {
        if (si.j == 0) {  // segment start: the known state (restart: c = z = 0, DC reset)
            s.p = si.lo;
        } else {
            Entry e = P.ent[g - 1];
            s.p = e.p;
            s.c = czd_c(e.czd);
            s.z = czd_z(e.czd);
        }
    }
    // symbols kept by the K1 chain that decoded this subsequence from this
    // very start state: replay them instead of decoding
    uint32_t nsym = 0;
    bool replay = false;
    if (REPLAY && active) {
        const uint4 tg = __ldg(reinterpret_cast<const uint4*>(P.tag) + g);
        replay = tg.w == P.epoch && tg.x == uint32_t(s.p) && tg.y == uint32_t(s.p >> 32) &&
                 (tg.z & 0xFFFFu) == (s.c | (s.z << 8));
        nsym = replay ? tg.z >> 16 : 0u;
    }
    const bool decode = active && !replay;
    if (!REPLAY || __syncthreads_or(decode)) {  // some thread decodes: stage the CTA's scan bytes
        __shared__ int4 s_stage[kStageBytes / 16];
        __shared__ StageSmem s_sm;
        // this subsequence's bits start at entries[g-1].p (inside [lo, hi)); stage from lo
        const uint64_t lo = decode ? D.raw_off + (si.lo >> 3) : 1;
        const uint64_t hi = decode ? D.raw_off + ((si.hi + 7) >> 3) + 24 : 0;
        stage_scan(P.ubuf, lo, hi, k, tid, kK3Threads, s_stage, s_sm);
        set_stage(ic, s_stage, s_sm, k);
    }
    if (!REPLAY && !active) return;
    const DcSums pd = active ? P.pred[g] : DcSums{0, 0};
    s.dc0 = int16_t(pd.lo & 0xFFFFu);
    s.dc1 = int16_t(pd.lo >> 16);
    s.dc2 = int16_t(pd.hi & 0xFFFFu);
    const uint64_t o = active ? P.off[g] : 0;
    using Sink = typename std::conditional<CMP, EntrySink, BlockSink>::type;
    Sink sink;
    sink.zt = s_zt;
    {
        sink.wqb = wq_smem ? s_wq : P.wq;
        sink.qrow = uint64_t(D.q_tab[0]) | (uint64_t(D.q_tab[1]) << 21) | (uint64_t(D.q_tab[2]) << 42);
    }
    if constexpr (CMP) {
        sink.ent = P.ents + D.du_first * 64;
        sink.um = P.umeta + D.du_first;
        sink.u = uint32_t(o >> 6);
        sink.pos = active ? P.eoff[g] : 0u;
        sink.ustart = 0;
    } else {
        sink.buf = buf;
        sink.coef = P.coef;
        sink.meta = P.meta;
        sink.du = D.du_first + (o >> 6);
    }
    sink.slot0 = o & ~63ull;
    sink.own_hi = o + cap;
    sink.klo = uint32_t(o & 63);
    sink.mflags = 0;
    sink.mS = 0.f;
    sink.set_comp(uint32_t(D.du_comp >> (4 * ((o >> 6) % D.dpm))) & 15u);

    // Replay, warp-cooperative: the warp's 32 consecutive subsequences read
    // symbol i as one 64-byte row; rows arrive 8 at a time by cp.async, two
    // tiles ahead, into a 3-tile ring (all lanes consume one symbol per step,
    // so the rows are read in lockstep).
    const uint32_t lane = tid & 31, warp = tid >> 5;
    const uint32_t maxn = REPLAY ? __reduce_max_sync(0xFFFFFFFFu, nsym) : 0u;
    if (REPLAY && maxn) {
        __shared__ __align__(16) uint16_t s_rt[kK3Threads / 32][3][8 * 32];
        const uint16_t* base = P.sym + (g - lane);
        auto issue = [&](uint32_t kt) {
            const uint32_t row = kt * 8 + (lane >> 2);
            if (row < maxn)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&s_rt[warp][kt % 3][(lane >> 2) * 32 + (lane & 3) * 8])),
                             "l"(base + uint64_t(row) * P.sym_stride + (lane & 3) * 8)
                             : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        issue(0);
        issue(1);
        uint32_t c = s.c, z = s.z, n = 0;
        int32_t a0 = s.dc0, a1 = s.dc1, a2 = s.dc2;
        uint32_t comp = (ic.duc >> (2 * c)) & 3u;
        int32_t acur = comp == 0 ? a0 : (comp == 1 ? a1 : a2);
        bool live = replay;
        for (uint32_t kt = 0; kt * 8 < maxn; ++kt) {
            issue(kt + 2);
            asm volatile("cp.async.wait_group 2;" ::: "memory");
            __syncwarp();
            const uint16_t* tile = s_rt[warp][kt % 3];
#pragma unroll 1
            for (uint32_t r = 0; r < 8; ++r) {
                const uint32_t ix = kt * 8 + r;
                live = live && ix < nsym && n < cap;
                if (!live) continue;
                const uint32_t w = tile[r * 32 + lane];
                int32_t coef = int32_t(w << 20) >> 20;
                const uint32_t run = (w >> 12) & 15u;
                const bool dcs = z == 0;
                // DC: one slot; AC value: run + 1; ZRL (run 15, value 0): 16; EOB: the rest
                const uint32_t step = dcs ? 1u : (coef != 0 ? run + 1u : (run ? 16u : 64u - z));
                if (n + step > cap) {  // phantom tail past the true end
                    live = false;
                    continue;
                }
                if (z + step > 64) {  // a run past the unit end: K1x redoes the image
                    atomicOr(&P.ist[k].exact, kExactFlag);
                    live = false;
                    continue;
                }
                if (dcs) {
                    acur += coef;
                    coef = acur;
                }
                if (dcs || coef != 0) sink.put(z + step - 1, coef);
                n += step;
                z += step;
                if (z >= 64) {
                    if (comp == 0)
                        a0 = acur;
                    else if (comp == 1)
                        a1 = acur;
                    else
                        a2 = acur;
                    z = 0;
                    c = (c + 1 == ic.dpm) ? 0 : c + 1;
                    comp = (ic.duc >> (2 * c)) & 3u;
                    acur = comp == 0 ? a0 : (comp == 1 ? a1 : a2);
                    sink.block_end(comp);
                }
            }
            __syncwarp();  // the tile is consumed before issue(kt + 3) refills its slot
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
    }
    if (decode) {
        decode_range<Sink, ST>(ic, s, si.hi, cap, sink);
        if (s.ovf) atomicOr(&P.ist[k].exact, kExactFlag);
        if (s.err) {
            set_status(P.ist + k, s.err);  // write mode rethrows (parallel_decode.hpp:142)
            return;
        }
    }
    if (active) sink.finish();
    if constexpr (CMP) {
        if (P.stats) {  // entries written (bench accounting), one atomic per warp
            const uint32_t m = __activemask();
            const uint32_t ne = __reduce_add_sync(m, active ? sink.pos - P.eoff[g] : 0u);
            if ((tid & 31) == __ffs(m) - 1) atomicAdd(P.stats + kStatEntries, (unsigned long long)ne);
        }
    }
}

// ============================================ K4: IDCT + upsample + RGB ====
// Warp-independent persistent kernel: every warp owns a contiguous range of
// tiles (one MCU-row segment 32 pixels wide: <= 12 data units) and runs the
// whole pipeline for a tile with only __syncwarp — no CTA barriers, so the
// resident warps hide each other's latency.  The next tile's coefficients and
// K3's per-unit metadata are prefetched with cp.async while the current tile
// computes.  Coefficients arrive column-major (F[u][v] at v*8+u).
//
//  1. classify the tile's units from K3's metadata: units with AC terms go to
//     a compact list for the IDCT; DC-only units take the integer path
//     (every sample = lround(b0 * (b0 * F00)) + 128; for F00 != 4 mod 8 that
//     is floor((F00 + 4) / 8) exactly, ties replayed as the reference's two
//     FP64 products, transform.hpp:114-142)
//  2. dequantise the AC units' columns (int32 coef * Q, transform.hpp:146-161)
//     into a float tile (stride 68 floats: 8 units' 16-byte loads hit 8
//     disjoint bank groups)
//  3. IDCT with packed FP32 (FFMA2): lane = (AC unit, row pair q, q+4), eight
//     units per pass; out(x,y) = sum_v b[v][y] sum_u b[u][x] F[u][v] over the
//     union of nonzero columns.  Rigorous bound |r32 - r64| <= 18 u S
//     (u = 2^-24, S = sum w_u w_v |F_uv| from K3); samples within the bound of
//     x.5 are replayed exactly in FP64 in the reference's summation order.
//     Each lane then owns two whole 8-sample rows: 4 aligned 32-bit stores.
//  4. YCbCr->RGB with the exact chroma maps (pipeline.hpp:182-187: x>>1 for
//     h = 2, x for h = 1, likewise rows — an identity for every W, H) and
//     integer colour: Y integer => lround(Y + t) = Y + round(t) unless t is an
//     exact real half-integer; round(t) and the tie test are exact integer
//     arithmetic on the decimal constants, ties replayed in FP64
//     (pipeline.hpp:190-197).  Saturating byte packs, 3 x 32-bit stores per
//     4 pixels.
// PJG_K4_SYM: lane = (unit, rows q and 7-q) and the even/odd split of both
// passes (basis[u][7-x] = (-1)^u basis[u][x]): per nonzero column 4 FFMA2 on
// (even u, odd u) pairs + 2 FADD, then 4 FFMA2 into the column-parity
// accumulators; 0: rows q and q+4, 8 + 8 FFMA2 per column.
#ifndef PJG_K4_SYM
#define PJG_K4_SYM 1
#endif
#ifndef PJG_K4_COLSPLIT
#define PJG_K4_COLSPLIT 0
#endif
constexpr float kM128 = 12583040.0f;  // 1.5 * 2^23 + 128: round(acc) + 128 in the low mantissa bits
constexpr int kMagicBits = 0x4B400000;
constexpr int kK4Warps = kK4Threads / 32;
constexpr int kTileW = 64;  // pixels per tile row
constexpr int kGroups = kTileW / 4;  // 4-pixel items per tile row
constexpr int kFS = 68;     // floats per unit in the F tile
// Compact-interface K4: threads per CTA and resident CTAs per SM (its warp
// state is smaller than the dense variant's: 6 warps x 3 CTAs = 18 warps fit
// where the dense one fits 4 x 4 = 16)
#ifndef PJG_K4C_THREADS
#define PJG_K4C_THREADS 128
#endif
#ifndef PJG_K4C_MINB
#define PJG_K4C_MINB 4
#endif
template <bool CMP>
struct K4Shape {
    static constexpr int kThreads = CMP ? PJG_K4C_THREADS : kK4Threads;
    static constexpr int kWarps = kThreads / 32;
    static constexpr int kMinBlocks = CMP ? PJG_K4C_MINB : 4;
};
#ifndef PJG_K4_WIN
#define PJG_K4_WIN 512
#endif
#ifndef PJG_K4_WIN_MUL
#define PJG_K4_WIN_MUL 2
#endif
constexpr uint32_t kK4Win = PJG_K4_WIN;  // compact: entries prefetched per tile (a q75 4:2:0 tile holds ~150)
constexpr uint32_t kNoWin = 0xFFFFFFFFu;
// raw staging row of (unit, column v): rows XOR-swizzled so that reading the
// same column of different units hits different bank groups
__device__ __forceinline__ uint32_t raw_row(uint32_t blk, uint32_t v) { return blk * 8 + (v ^ (blk & 7u)); }

__device__ __forceinline__ uint32_t pack4_sat(int a0, int a1, int a2, int a3) {
    uint32_t t, d;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(t) : "r"(a3), "r"(a2), "r"(0));
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a1), "r"(a0), "r"(t));
    return d;
}

// Exact FP64 value of sample (x, y) of a unit in the reference's order
// (transform.hpp:114-142): tmp[u] = sum_v b[v][y] F[u][v] (v ascending),
// out = sum_u b[u][x] tmp[u] (u ascending), zero terms skipped (exact: the
// running sums start at +0 and fl(s + +-0) = s).  Fc is column-major; `big`
// units hold int32 bits.  Returns the clamped sample.
__device__ __noinline__ uint32_t idct_sample_fp64(const float* Fc, bool big, uint32_t cols, uint32_t rows,
                                                  const double* b64, int x, int y) {
    const int32_t* Fi = reinterpret_cast<const int32_t*>(Fc);
    double s = 0.0;
    for (uint32_t um = rows; um; um &= um - 1) {  // all-zero rows give tmp = +0: skipped
        const int u = __ffs(um) - 1;
        double t = 0.0;
        for (uint32_t m = cols; m; m &= m - 1) {
            const int v = __ffs(m) - 1;
            const double f = big ? double(Fi[v * 8 + u]) : double(Fc[v * 8 + u]);
            if (f != 0.0) t = __dadd_rn(t, __dmul_rn(b64[v * 8 + y], f));
        }
        if (t != 0.0) s = __dadd_rn(s, __dmul_rn(b64[u * 8 + x], t));
    }
    return clamp_u8(lround_away(s) + 128);
}

// exact FP64 colour of one pixel (pipeline.hpp:190-197): returns R | G << 8 | B << 16
__device__ __noinline__ uint32_t rgb_fp64(int Y, int Cb, int Cr) {
    const double Yd = double(Y);
    const int cb = Cb - 128, cr = Cr - 128;
    const int R = lround_away(__dadd_rn(Yd, __dmul_rn(1.402, double(cr))));
    const int G = lround_away(__dsub_rn(__dsub_rn(Yd, __dmul_rn(0.344136, double(cb))), __dmul_rn(0.714136, double(cr))));
    const int B = lround_away(__dadd_rn(Yd, __dmul_rn(1.772, double(cb))));
    return pack4_sat(R, G, B, 0);
}

// Per-warp image cache: layout of the tile's data units in the warp's sample
// planes, quantisers, and the descriptor fields the tile loop needs.
struct __align__(16) WarpImg {
    float qf[3][64];    // column-major quantiser per component, as float (exact: < 2^16)
    uint32_t pst[3], poff[3];
    uint16_t boff[kK4MaxBlocks];  // plane byte offset of the unit's (0,0) sample
    uint16_t bps[kK4MaxBlocks];   // plane row stride
    uint8_t bcomp[kK4MaxBlocks];
    uint32_t width, height, ncomp, h_max, v_max, rgb, out_mode;
    uint32_t plane_w[3], plane_h[3], comp_h[3], comp_v[3];
    uint64_t out_off;
};

// Tile walker state (warp-uniform; lives in the warp's smem).
struct TileWalk {
    uint32_t k, kend, tiles_x, MT, mcus_x, dpm, mcu_w, mcu_h, valid, my, tx;
    uint64_t du_first;
};

template <bool CMP>
struct WarpSmem {
    float F[kK4MaxBlocks * kFS];  // dequantised AC units (float, or int32 bits when big), compact order
    int4 raw[CMP ? 1 : kK4MaxBlocks * 8];   // dense: next tile's coefficients (cp.async staging)
    uint2 meta[CMP ? 1 : kK4MaxBlocks];     // dense: next tile's per-unit metadata
    uint4 meta4[CMP ? kK4MaxBlocks : 1];    // compact: next tile's (first entry, end entry, flags, S)
    int32_t dcv[CMP ? kK4MaxBlocks : 1];    // compact: quantised DC of each unit
    uint32_t ud[CMP ? kK4MaxBlocks : 1];    // compact: per unit F offset (0xFFFF: DC-only) | qf offset << 16 | big << 24
    __align__(16) uint32_t win[CMP ? kK4Win : 1];  // compact: next tile's entries (cp.async window)
    __align__(16) uint8_t pl[1664];             // sample planes (row stride padded by 4): 4:2:0 needs 68x16 + 2 x 36x8, gray 196x8
    WarpImg img;
    float lim[kK4MaxBlocks];      // per AC unit: 0.5 - error bound
    uint32_t cm[kK4MaxBlocks];    // per AC unit: column mask | big << 8 | row mask << 16
    uint8_t acl[kK4MaxBlocks];    // AC units (tile-local index), compact
    uint8_t dcl[kK4MaxBlocks];    // DC-only units
    uint8_t dq[kK4MaxBlocks * 8]; // nonzero columns of the AC units: a << 3 | v
    uint16_t rep[32];             // FP64 replay work list: unit << 6 | x << 3 | y
    TileWalk w;
};

// Warp-cooperative cache fill (runs at image changes only).
__device__ __forceinline__ void fill_warp_img(const Params& P, uint32_t k, WarpImg& c, int lane) {
    const ImgDesc& D = P.img[k];
    const uint32_t MT = D.mcus_per_tile, ncomp = D.ncomp, dpm = D.dpm;
    uint32_t pst[3], poff[3], acc = 0;
#pragma unroll
    for (uint32_t cc = 0; cc < 3; ++cc) {
        const bool has = cc < ncomp;
        pst[cc] = has ? MT * D.comp_h[cc] * 8 + 4 : 0;
        poff[cc] = acc;
        acc += has ? pst[cc] * D.comp_v[cc] * 8 : 0;
    }
    if (lane < 24) {  // 3 quantisers x 8 x 16 B
        const uint32_t cc = lane >> 3;
        if (cc < ncomp) {
            const uint4 qv = __ldg(reinterpret_cast<const uint4*>(P.quant_raster + 64u * D.q_tab[cc]) + (lane & 7));
            float4* qf = reinterpret_cast<float4*>(c.qf[cc] + 8 * (lane & 7));
            qf[0] = make_float4(float(qv.x & 0xFFFFu), float(qv.x >> 16), float(qv.y & 0xFFFFu), float(qv.y >> 16));
            qf[1] = make_float4(float(qv.z & 0xFFFFu), float(qv.z >> 16), float(qv.w & 0xFFFFu), float(qv.w >> 16));
        }
    }
    if (lane < int(MT * dpm) && lane < kK4MaxBlocks) {
        const uint32_t blk = lane, slot = blk % dpm, m = blk / dpm;
        const uint32_t comp = uint32_t(D.du_comp >> (4 * slot)) & 15u;
        const uint32_t kk = uint32_t(D.du_kslot >> (4 * slot)) & 15u;
        const uint32_t chh = D.comp_h[comp];
        const uint32_t bx = kk % chh, by = kk / chh;
        c.bcomp[blk] = uint8_t(comp);
        c.bps[blk] = uint16_t(pst[comp]);
        c.boff[blk] = uint16_t(poff[comp] + (by * 8) * pst[comp] + (m * chh + bx) * 8);
    }
    if (lane == 0) {
        for (int cc = 0; cc < 3; ++cc) {
            c.pst[cc] = pst[cc];
            c.poff[cc] = poff[cc];
            c.plane_w[cc] = D.plane_w[cc];
            c.plane_h[cc] = D.plane_h[cc];
            c.comp_h[cc] = D.comp_h[cc];
            c.comp_v[cc] = D.comp_v[cc];
        }
        c.width = D.width;
        c.height = D.height;
        c.ncomp = ncomp;
        c.h_max = D.h_max;
        c.v_max = D.v_max;
        c.out_mode = D.out_mode;
        c.rgb = D.out_mode == 1 && ncomp == 3;
        c.out_off = D.out_off;
    }
    __syncwarp();
}

__device__ __forceinline__ void walk_enter_image(const Params& P, uint32_t t, TileWalk& w) {
    while (P.tile_first[w.k + 1] <= t) ++w.k;
    const ImgDesc& D = P.img[w.k];
    w.kend = P.tile_first[w.k + 1];
    w.tiles_x = D.tiles_x;
    w.MT = D.mcus_per_tile;
    w.mcus_x = D.mcus_x;
    w.dpm = D.dpm;
    w.mcu_w = 8 * D.h_max;
    w.mcu_h = 8 * D.v_max;
    w.du_first = D.du_first;
    w.valid = P.ist[w.k].status == 0;
    const uint32_t lt = t - P.tile_first[w.k];
    w.my = lt / w.tiles_x;
    w.tx = lt % w.tiles_x;
}

// Chroma offsets of one (Cb, Cr) sample, exact integers:
//   r[Cr] = round(1.402 cr), b[Cb] = round(1.772 cb) (B ties: Cb = 3, 253),
//   G: m = ga[Cb] + gb[Cr] = -344136 cb - 714136 cr + 500000 + 2e8 (+1 when Cb
//   is a B tie; m is otherwise even), oG = floor(m / 1e6) - 200; a G tie is
//   m == 0 mod 1e6, so (m mod 1e6) == 0 or odd flags any tie.
// The division is pre-split: with ga = qa 1e6 + ra, gb = qb 1e6 + rb (0 <= r
// < 1e6) the tables hold (qa - 200) << 20 | (ra + 2^20 - 1e6) and qb << 20 | rb,
// so one add carries exactly when ra + rb >= 1e6: oG = sum >> 20 and the low
// 20 bits are m mod 1e6 (carry) or m mod 1e6 + 48576 (no carry — then m mod
// 1e6 is never 0: that needs rb = 0, i.e. cr = 0, and ra(0) = 500000), so a
// tie is "low 20 bits odd or zero".  Each half is loaded with its R / B
// offset as one 64-bit word.
struct ColourLut {
    int2 cb[256];  // (G word of Cb, B offset)
    int2 cr[256];  // (G word of Cr, R offset)
};

__device__ __forceinline__ void chroma_off(const ColourLut& L, uint32_t cb, uint32_t cr, int& oR, int& oG, int& oB,
                                           uint32_t& tie) {
    const int2 a = L.cb[cb], b = L.cr[cr];
    oR = b.y;
    oB = a.y;
    const uint32_t m = uint32_t(a.x) + uint32_t(b.x);
    const uint32_t lo = m & 0xFFFFFu;
    tie |= (lo & 1u) | uint32_t(lo == 0u);
    oG = int32_t(m) >> 20;
}

__device__ __forceinline__ int ybyte(uint32_t y4, int i) { return int((y4 >> (8 * i)) & 0xFFu); }

// 4 pixels of one row -> 12 RGB bytes (3 words); chroma offsets per pixel
__device__ __forceinline__ uint3 rgb4(uint32_t y4, const int* oR, const int* oG, const int* oB) {
    const int Y0 = ybyte(y4, 0), Y1 = ybyte(y4, 1), Y2 = ybyte(y4, 2), Y3 = ybyte(y4, 3);
    uint3 w;
    w.x = pack4_sat(Y0 + oR[0], Y0 + oG[0], Y0 + oB[0], Y1 + oR[1]);
    w.y = pack4_sat(Y1 + oG[1], Y1 + oB[1], Y2 + oR[2], Y2 + oG[2]);
    w.z = pack4_sat(Y2 + oB[2], Y3 + oR[3], Y3 + oG[3], Y3 + oB[3]);
    return w;
}

__device__ __forceinline__ void store_rgb4(uint8_t* dst, uint3 w, uint32_t npx, bool aligned) {
    if (npx == 4 && aligned) {
        uint32_t* d = reinterpret_cast<uint32_t*>(dst);
        d[0] = w.x;
        d[1] = w.y;
        d[2] = w.z;
    } else {
        const uint32_t ws[3] = {w.x, w.y, w.z};
        for (uint32_t q = 0; q < npx * 3; ++q) dst[q] = uint8_t(ws[q >> 2] >> (8 * (q & 3)));
    }
}

// exact replay of 4 pixels (some chroma sample is an exact real tie)
__device__ __forceinline__ uint3 rgb4_exact(uint32_t y4, const uint8_t* cb, const uint8_t* cr, const uint32_t* cx) {
    uint32_t px[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) px[i] = rgb_fp64(ybyte(y4, i), cb[cx[i]], cr[cx[i]]);
    uint3 w;
    w.x = (px[0] & 0xFFFFFFu) | (px[1] << 24);
    w.y = ((px[1] >> 8) & 0xFFFFu) | (px[2] << 16);
    w.z = ((px[2] >> 16) & 0xFFu) | (px[3] << 8);
    return w;
}

// Colour stage of one tile.  HS = pixels per chroma sample horizontally (1
// for 4:4:4, 2 for 4:2:2 / 4:2:0); PAIR: two rows share a chroma row (4:2:0).
// Lane item = 4 pixels of one row (of a row pair when PAIR).
template <int HS, bool PAIR>
__device__ __forceinline__ void colour_tile(const WarpImg& I, const uint8_t* pl, const ColourLut& L, uint8_t* out,
                                            uint32_t X0, uint32_t Y0, uint32_t cols, uint32_t rws, int lane) {
    const uint32_t nrow = PAIR ? (rws + 1) >> 1 : rws;
    const uint32_t W = I.width;
    const bool aligned = ((W & 3) == 0) && ((I.out_off & 3) == 0);
    const uint8_t* yb = pl + I.poff[0];
    const uint8_t* cbb = pl + I.poff[1];
    const uint8_t* crb = pl + I.poff[2];
    const uint32_t pst0 = I.pst[0], pst1 = I.pst[1];
    uint8_t* obase = out + I.out_off + (uint64_t(Y0) * W + X0) * 3;
    const uint64_t orow = uint64_t(W) * 3;
    for (uint32_t it = lane; it < nrow * kGroups; it += 32) {
        const uint32_t jr = it / kGroups, gx = (it % kGroups) * 4;
        if (gx >= cols) continue;
        const uint32_t npx = min(4u, cols - gx);
        const uint32_t r0 = PAIR ? 2 * jr : jr;
        const uint8_t* cbrow = cbb + jr * pst1;
        const uint8_t* crrow = crb + jr * pst1;
        int oR[4], oG[4], oB[4];
        uint32_t tie = 0;
        uint32_t cx[4];
        if (HS == 2) {
            const uint32_t c0 = gx >> 1;
            const uint32_t cb2 = *reinterpret_cast<const uint16_t*>(cbrow + c0);
            const uint32_t cr2 = *reinterpret_cast<const uint16_t*>(crrow + c0);
            chroma_off(L, cb2 & 0xFFu, cr2 & 0xFFu, oR[0], oG[0], oB[0], tie);
            chroma_off(L, cb2 >> 8, cr2 >> 8, oR[2], oG[2], oB[2], tie);
            oR[1] = oR[0], oG[1] = oG[0], oB[1] = oB[0];
            oR[3] = oR[2], oG[3] = oG[2], oB[3] = oB[2];
            cx[0] = cx[1] = c0;
            cx[2] = cx[3] = c0 + 1;
        } else {
            const uint32_t cb4 = *reinterpret_cast<const uint32_t*>(cbrow + gx);
            const uint32_t cr4 = *reinterpret_cast<const uint32_t*>(crrow + gx);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                chroma_off(L, (cb4 >> (8 * i)) & 0xFFu, (cr4 >> (8 * i)) & 0xFFu, oR[i], oG[i], oB[i], tie);
                cx[i] = gx + i;
            }
        }
        {
            const uint32_t y4 = *reinterpret_cast<const uint32_t*>(yb + r0 * pst0 + gx);
            const uint3 w = tie ? rgb4_exact(y4, cbrow, crrow, cx) : rgb4(y4, oR, oG, oB);
            store_rgb4(obase + r0 * orow + gx * 3, w, npx, aligned);
        }
        if (PAIR && r0 + 1 < rws) {
            const uint32_t y4 = *reinterpret_cast<const uint32_t*>(yb + (r0 + 1) * pst0 + gx);
            const uint3 w = tie ? rgb4_exact(y4, cbrow, crrow, cx) : rgb4(y4, oR, oG, oB);
            store_rgb4(obase + (r0 + 1) * orow + gx * 3, w, npx, aligned);
        }
    }
}

// Whole 64-pixel-wide, full-height tile with 4-byte-aligned rows: two fixed
// items per lane, no bounds checks.  The tile's RGB rows (192 bytes each) are
// assembled in shared memory (`stg`, the IDCT's F tile, dead by now) at the
// 16-byte phase of their global address, then leave as 16-byte stores: a row
// touches 12 aligned chunks (13 when misaligned: a ragged head and tail
// written word by word).  Staging row stride 208 = 13 chunks, so item i of
// the write-out reads smem chunk i — conflict-free, and consecutive lanes
// store consecutive 16-byte chunks of a row.
constexpr uint32_t kStgRow = 208;
#ifndef PJG_K4_STAGE
#define PJG_K4_STAGE 0
#endif
template <int HS, bool PAIR>
__device__ __forceinline__ void colour_full(const WarpImg& I, const uint8_t* pl, const ColourLut& L, uint8_t* out,
                                            uint8_t* stg, uint32_t X0, uint32_t Y0, uint32_t rows, int lane) {
    const uint32_t W = I.width;
    const uint32_t gx = (lane % kGroups) * 4, jr0 = lane / kGroups;
    const uint32_t cgx = HS == 2 ? gx >> 1 : gx;
    const uint8_t* yb = pl + I.poff[0] + gx;
    const uint8_t* cbb = pl + I.poff[1];
    const uint8_t* crb = pl + I.poff[2];
    const uint32_t pst0 = I.pst[0], pst1 = I.pst[1];
    const uint64_t orow = uint64_t(W) * 3;
    uint8_t* ob0 = out + I.out_off + (uint64_t(Y0) * W + X0) * 3;  // row 0 of the tile
    const uint32_t m0 = uint32_t(reinterpret_cast<uintptr_t>(ob0)) & 15u, mstep = uint32_t(orow) & 15u;
#pragma unroll
    for (int h = 0; h < 8 * kGroups / 32; ++h) {
        const uint32_t jr = jr0 + (32 / kGroups) * h;
        const uint32_t r0 = PAIR ? 2 * jr : jr;
        const uint8_t* cbrow = cbb + jr * pst1;
        const uint8_t* crrow = crb + jr * pst1;
        int oR[4], oG[4], oB[4];
        uint32_t tie = 0;
        uint32_t cx[4];
        if (HS == 2) {
            const uint32_t cb2 = *reinterpret_cast<const uint16_t*>(cbrow + cgx);
            const uint32_t cr2 = *reinterpret_cast<const uint16_t*>(crrow + cgx);
            chroma_off(L, cb2 & 0xFFu, cr2 & 0xFFu, oR[0], oG[0], oB[0], tie);
            chroma_off(L, cb2 >> 8, cr2 >> 8, oR[2], oG[2], oB[2], tie);
            oR[1] = oR[0], oG[1] = oG[0], oB[1] = oB[0];
            oR[3] = oR[2], oG[3] = oG[2], oB[3] = oB[2];
            cx[0] = cx[1] = cgx;
            cx[2] = cx[3] = cgx + 1;
        } else {
            const uint32_t cb4 = *reinterpret_cast<const uint32_t*>(cbrow + cgx);
            const uint32_t cr4 = *reinterpret_cast<const uint32_t*>(crrow + cgx);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                chroma_off(L, (cb4 >> (8 * i)) & 0xFFu, (cr4 >> (8 * i)) & 0xFFu, oR[i], oG[i], oB[i], tie);
                cx[i] = cgx + i;
            }
        }
        {
            const uint32_t y4 = *reinterpret_cast<const uint32_t*>(yb + r0 * pst0);
            const uint3 w = tie ? rgb4_exact(y4, cbrow, crrow, cx) : rgb4(y4, oR, oG, oB);
            uint32_t* d = PJG_K4_STAGE ? reinterpret_cast<uint32_t*>(stg + r0 * kStgRow + ((m0 + r0 * mstep) & 15u) + gx * 3)
                                       : reinterpret_cast<uint32_t*>(ob0 + r0 * orow + gx * 3);
            d[0] = w.x;
            d[1] = w.y;
            d[2] = w.z;
        }
        if (PAIR) {
            const uint32_t r1 = r0 + 1;
            const uint32_t y4 = *reinterpret_cast<const uint32_t*>(yb + r1 * pst0);
            const uint3 w = tie ? rgb4_exact(y4, cbrow, crrow, cx) : rgb4(y4, oR, oG, oB);
            uint32_t* d = PJG_K4_STAGE ? reinterpret_cast<uint32_t*>(stg + r1 * kStgRow + ((m0 + r1 * mstep) & 15u) + gx * 3)
                                       : reinterpret_cast<uint32_t*>(ob0 + r1 * orow + gx * 3);
            d[0] = w.x;
            d[1] = w.y;
            d[2] = w.z;
        }
    }
    if (!PJG_K4_STAGE) return;
    __syncwarp();
    // write-out: item = (row r, aligned chunk c of 13)
    for (uint32_t it = lane; it < rows * 13u; it += 32) {
        const uint32_t r = it / 13u, c = it - r * 13u;
        const uint32_t m = (m0 + r * mstep) & 15u;
        uint8_t* g = ob0 + r * orow - m + 16u * c;  // 16-byte aligned
        const uint4 v = *reinterpret_cast<const uint4*>(stg + 16u * it);
        if ((c != 0 || m == 0) && c != 12) {
            *reinterpret_cast<uint4*>(g) = v;
        } else if (m != 0) {  // ragged head (bytes m..15) or tail (bytes 0..m-1), 4-byte granular
            const uint32_t lo = c == 0 ? m >> 2 : 0u, hi = c == 0 ? 4u : m >> 2;
            const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k)
                if (k >= lo && k < hi) reinterpret_cast<uint32_t*>(g)[k] = vw[k];
        }
    }
}

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
static_assert(sizeof(WarpSmem<false>) * kK4Warps + 4864 + 1024 <= 228 * 1024 / 4, "K4 must fit 4 CTAs per SM");
static_assert(sizeof(WarpSmem<true>) * K4Shape<true>::kWarps + 4864 + 1024 <= 228 * 1024 / K4Shape<true>::kMinBlocks,
              "compact K4 must fit its CTAs per SM");
static_assert(sizeof(WarpSmem<false>::F) >= 16 * kStgRow, "RGB row staging lives in the F tile");
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;"
        : "=l"(r)
        : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)));
    return *reinterpret_cast<float2*>(&r);
}

// LAYOUT 1: every image of the batch is 4:2:0 colour to RGB — only that colour
// path is compiled in (a smaller hot loop for the instruction cache: 3.1 K vs
// 5.2 K instructions, K4 -4 % on cfg 3; a 4:4:4 variant gained nothing); 0: any.
template <int LAYOUT, bool CMP>
__global__ void __launch_bounds__(K4Shape<CMP>::kThreads, K4Shape<CMP>::kMinBlocks) k4_transform(Params P) {
    constexpr int kK4Threads = K4Shape<CMP>::kThreads, kK4Warps = K4Shape<CMP>::kWarps;
    extern __shared__ __align__(16) unsigned char k4_dyn[];  // kK4Warps x WarpSmem
    WarpSmem<CMP>* s_w = reinterpret_cast<WarpSmem<CMP>*>(k4_dyn);
    __shared__ __align__(16) float s_b32[64];   // basis[u][x]
    __shared__ __align__(16) double s_b64[64];
    __shared__ __align__(16) ColourLut s_lut;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 64) {
        const double b = P.basis[tid];
        s_b64[tid] = b;
        s_b32[tid] = float(b);
    }
    for (int c = tid; c < 256; c += kK4Threads) {
        const int v = c - 128;
        // round(k v) for decimal k, exactly: floor((1000 k v + 500) / 1000)
        const int oR = int((1402 * v + 500 + 200000) / 1000) - 200;
        const int mB = 1772 * v + 500 + 300000;
        const int ga = -344136 * v + 500000 + 200000000 + ((mB % 1000) == 0 ? 1 : 0);  // > 0
        const int gb = -714136 * v;
        const int qa = ga / 1000000, ra = ga - qa * 1000000;
        const int qb = (gb >= 0 ? gb : gb - 999999) / 1000000, rb = gb - qb * 1000000;  // floor
        s_lut.cb[c] = make_int2(int(uint32_t(qa - 200) << 20) + ra + (1048576 - 1000000), mB / 1000 - 300);
        s_lut.cr[c] = make_int2(int(uint32_t(qb) << 20) + rb, oR);
    }
    __syncthreads();
    pdl_wait();  // the LUT and basis above are batch constants

    WarpSmem<CMP>& S = s_w[warp];
    const uint32_t gw = blockIdx.x * kK4Warps + warp, nw = gridDim.x * kK4Warps;
    const uint32_t t_begin = uint32_t(uint64_t(P.k4_tiles) * gw / nw);
    const uint32_t t_end = uint32_t(uint64_t(P.k4_tiles) * (gw + 1) / nw);
    if (t_begin >= t_end) return;

    // IDCT lane constants: rows q and 7-q (SYM) or q and q+4 of the lane's unit
    const uint32_t q = lane & 3;
#if PJG_K4_SYM
    float2 bp[4];  // (b[2k][q], b[2k+1][q])
#pragma unroll
    for (int k = 0; k < 4; ++k) bp[k] = make_float2(s_b32[(2 * k) * 8 + q], s_b32[(2 * k + 1) * 8 + q]);
#else
    float2 bq[8];  // (b[u][q], b[u][q+4])
#pragma unroll
    for (int u = 0; u < 8; ++u) bq[u] = make_float2(s_b32[u * 8 + q], s_b32[u * 8 + q + 4]);
#endif

    TileWalk& w = S.w;
    if (lane == 0) {
        uint32_t lo = 0, hi = P.n_img;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (P.tile_first[mid] <= t_begin)
                lo = mid;
            else
                hi = mid;
        }
        w.k = lo;
        walk_enter_image(P, t_begin, w);
    }
    __syncwarp();
    uint32_t cached_k = 0xFFFFFFFFu;
    // prefetch of a tile into the warp's smem staging (cp.async, no registers
    // held): 16-byte columns lane, lane+32, lane+64 of its units + metadata
    // compact: the window of entries staged with the tile (kNoWin: none)
    uint32_t win_pend = kNoWin;
    uint32_t win_len_pend = 0;  // entries the window holds (only these may be read from it)
    const uint64_t ent_total = P.total_dus * 64;
    auto issue = [&](const TileWalk& tw, uint32_t wstart, uint32_t wlen) {
        const uint32_t mx0 = tw.tx * tw.MT;
        const uint32_t nblk = min(tw.MT, tw.mcus_x - mx0) * tw.dpm;
        const uint64_t du0 = tw.du_first + (uint64_t(tw.my) * tw.mcus_x + mx0) * tw.dpm;
        if (CMP) {
            win_pend = kNoWin;
            win_len_pend = 0;
            if (tw.valid) {
                if (uint32_t(lane) < nblk)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&S.meta4[lane])),
                                 "l"(P.umeta + du0 + lane)
                                 : "memory");
                if (wstart != kNoWin) {
                    // the tile's entries start where the previous tile's ended
                    // (contiguous runs); 16-byte aligned window of kK4Win entries
                    win_pend = wstart & ~3u;
                    const uint64_t g0 = tw.du_first * 64 + win_pend;
                    const uint64_t avail = ent_total > g0 ? (ent_total - g0) & ~3ull : 0ull;
                    win_len_pend = uint32_t(min64(min64((wstart - win_pend + wlen + 3) & ~3u, kK4Win), avail));
#pragma unroll
                    for (uint32_t j = 0; j < kK4Win / 128; ++j) {
                        const uint32_t c = lane + 32 * j;
                        if (4 * c < win_len_pend)
                            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&S.win[4 * c])),
                                         "l"(P.ents + g0 + 4 * c)
                                         : "memory");
                    }
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            return;
        }
        const int4* src = reinterpret_cast<const int4*>(P.coef + du0 * 64);
        if (tw.valid) {
#pragma unroll
            for (int j = 0; j < kK4MaxBlocks / 4; ++j) {
                const uint32_t ch = lane + 32 * j;
                if (ch < nblk * 8)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&S.raw[raw_row(ch >> 3, ch & 7)])), "l"(src + ch)
                                 : "memory");
            }
            if (uint32_t(lane) < nblk)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(&S.meta[lane])),
                             "l"(P.meta + du0 + lane)
                             : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue(w, kNoWin, 0);
    const uint32_t lt_mask = (1u << lane) - 1u;
    uint32_t next_wstart = kNoWin;  // compact: where the next tile's entries start (contiguous runs)
    uint32_t next_wlen = kK4Win;    // compact: entries to stage (twice the current tile's + slack)
    uint32_t n_replay = 0, n_ac = 0;
    for (uint32_t t = t_begin; t < t_end; ++t) {
        const uint32_t cur_k = w.k, cur_my = w.my, cur_mx0 = w.tx * w.MT;
        const uint32_t cur_nm = min(w.MT, w.mcus_x - cur_mx0);
        const uint32_t cur_valid = w.valid, cur_mcuw = w.mcu_w, cur_mcuh = w.mcu_h;
        const uint64_t cur_du_first = w.du_first;
        const uint64_t du_tile0 = w.du_first + (uint64_t(w.my) * w.mcus_x + cur_mx0) * w.dpm;
        const uint32_t nblk = cur_nm * w.dpm;
        if (cur_valid && cached_k != cur_k) {
            __syncwarp();
            fill_warp_img(P, cur_k, S.img, lane);
            cached_k = cur_k;
        }
        const WarpImg& I = S.img;

        // 1. classify units (K3 metadata: column mask | has-AC << 8 | big << 9, S)
        asm volatile("cp.async.wait_all;" ::: "memory");
        const uint32_t win_cur = win_pend, win_len = win_len_pend;
        next_wstart = kNoWin;
        __syncwarp();
        uint32_t nac = 0, ndc = 0, ndq = 0;
        if (cur_valid) {
            const bool in = uint32_t(lane) < nblk;
            uint2 pm;
            uint32_t e_lo = 0, e_hi = 0;  // compact: the unit's entries
            if (CMP) {
                const uint4 m4 = in ? S.meta4[lane] : make_uint4(0, 0, 0, 0);
                pm = make_uint2(m4.z, m4.w);
                e_lo = m4.x;
                e_hi = m4.y;
            } else {
                pm = in ? S.meta[lane] : make_uint2(0, 0);
            }
            const bool isac = in && (pm.x & kMetaNonDc);
            const uint32_t acm = __ballot_sync(0xFFFFFFFFu, isac);
            const uint32_t dcm = __ballot_sync(0xFFFFFFFFu, in && !isac);
            nac = __popc(acm);
            ndc = __popc(dcm);
            const uint32_t a_slot = __popc(acm & lt_mask);
            // nonzero columns of the AC units -> dequantisation work list
            const uint32_t ncol = isac ? __popc(pm.x & 0xFFu) : 0u;
            uint32_t cincl = ncol;
            if (!CMP) {  // (compact: no dequantisation list, the entries are scattered)
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, cincl, o);
                    if (lane >= o) cincl += x;
                }
                ndq = __shfl_sync(0xFFFFFFFFu, cincl, 31);
            }
            if (isac) {
                const uint32_t a = a_slot;
                // columns: nonzero ones to the list, zero ones zero-filled (the IDCT
                // reads every column any unit of its pass uses)
                uint32_t j = cincl - ncol;
                float4* Fa = reinterpret_cast<float4*>(S.F + a * kFS);
#pragma unroll
                for (uint32_t v = 0; v < 8; ++v) {
                    if (!CMP && ((pm.x >> v) & 1u)) {
                        S.dq[j++] = uint8_t((a << 3) | v);
                    } else {  // compact: every column zero-filled, the entries land on top
                        Fa[2 * v] = make_float4(0.f, 0.f, 0.f, 0.f);
                        Fa[2 * v + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
                const float Sb = __uint_as_float(pm.y);
                // S >= 2^18 covers every unit with some |F| >= 2^21 (w_u w_v >= 1/8): those
                // take exact FP64; below it F is exact in FP32 and |acc| <= S
                const bool big = Sb >= 262144.f;
                S.acl[a] = uint8_t(lane);
                const uint32_t cols = pm.x & 0xFFu, rows = (pm.x >> 16) & 0xFFu;
                S.cm[a] = cols | (big ? 0x100u : 0u) | (rows << 16);
                // Rounding analysis of step 3: the column sums see at most popc(rows)
                // nonzero products (zero terms are exact in an FMA chain), the row sums
                // popc(cols), and the two basis factors each carry one FP32 rounding, so
                // |r32 - r_exact| <= (k + m + 2) u S to first order (k = popc(rows),
                // m = popc(cols), u = 2^-24); one more u S covers second-order terms and
                // the reference's own FP64 error (~1e-15 S).
                const float km = float(__popc(rows) + __popc(cols) + 3);
                S.lim[a] = 0.5f - (km * 5.9605e-8f * Sb * 1.001f + 1.0e-6f);
            } else if (in) {
                S.dcl[__popc(dcm & lt_mask)] = uint8_t(lane);
            }
            if (CMP && in)
                S.ud[lane] = (isac ? a_slot * kFS : 0xFFFFu) | ((uint32_t(I.bcomp[lane]) * 64u) << 16) |
                             (isac && __uint_as_float(pm.y) >= 262144.f ? (1u << 24) : 0u);
            __syncwarp();
            if constexpr (CMP) {
                // 2a'. scatter the tile's entries into the zeroed F tiles (dequantised;
                //      exact-FP64 units keep int32 products); DC values for the
                //      DC-only units.  Entries of consecutive units are contiguous
                //      (one range, unit = count of DC entries so far) unless a
                //      restart interval's end or a K1x image breaks the run.
                const uint32_t* eb = P.ents + cur_du_first * 64;
                const float* qf0 = &I.qf[0][0];
                auto scatter = [&](uint32_t u, uint32_t x) {
                    const uint32_t idx = (x >> 16) & 63u;
                    const int32_t v = int32_t(int16_t(x & 0xFFFFu));
                    const uint32_t d = S.ud[u];
                    const uint32_t fo = d & 0xFFFFu;
                    if (fo != 0xFFFFu) {
                        const float q = qf0[((d >> 16) & 0xFFu) + idx];
                        S.F[fo + idx] = (d >> 24) ? __int_as_float(v * int32_t(q)) : float(v) * q;
                    } else if (idx == 0) {
                        S.dcv[u] = v;
                    }
                };
                const uint32_t nxt = __shfl_down_sync(0xFFFFFFFFu, e_lo, 1);
                const bool contiguous = __all_sync(0xFFFFFFFFu, uint32_t(lane) + 1 >= nblk || e_hi == nxt);
                if (contiguous) {
                    const uint32_t r0 = __shfl_sync(0xFFFFFFFFu, e_lo, 0);
                    const uint32_t r1 = __shfl_sync(0xFFFFFFFFu, e_hi, (nblk - 1) & 31u);
                    // entries carry their unit's index mod 256 (bits 22-29)
                    const uint32_t ub = uint32_t(du_tile0 - cur_du_first);
                    if (win_cur != kNoWin && r0 >= win_cur && r1 - win_cur <= win_len) {  // all staged
#pragma unroll 1
                        for (uint32_t jj = r0 - win_cur + lane; jj < r1 - win_cur; jj += 32) {
                            const uint32_t x = S.win[jj];
                            const uint32_t u = ((x >> 22) - ub) & 0xFFu;
                            if (u < nblk) scatter(u, x);
                        }
                    } else {
#pragma unroll 1
                        for (uint32_t jj = r0 + lane; jj < r1; jj += 32) {
                            const uint32_t x = (jj - win_cur < win_len && win_cur != kNoWin) ? S.win[jj - win_cur] : __ldg(eb + jj);
                            const uint32_t u = ((x >> 22) - ub) & 0xFFu;
                            if (u < nblk) scatter(u, x);
                        }
                    }
                    next_wstart = r1;
                    next_wlen = min(kK4Win, PJG_K4_WIN_MUL * (r1 - r0) + 64);
                } else {
#pragma unroll 1
                    for (uint32_t u = 0; u < nblk; ++u) {
                        const uint32_t lo = __shfl_sync(0xFFFFFFFFu, e_lo, u), hi = __shfl_sync(0xFFFFFFFFu, e_hi, u);
                        for (uint32_t jj = lo + lane; jj < hi; jj += 32) scatter(u, __ldg(eb + jj));
                    }
                }
                __syncwarp();
            }
            // 2a. dequantise the AC units' nonzero columns: coef * Q in FP32 is exact
            //     (|coef * Q| < 2^21 below the exact-FP64 threshold); exact-FP64
            //     units keep the int32 products
#pragma unroll 1
            for (uint32_t it = lane; it < (CMP ? 0u : ndq); it += 32) {
                const uint32_t e = S.dq[it], a = e >> 3, v = e & 7u;
                const uint32_t blk = S.acl[a];
                float4* dst = reinterpret_cast<float4*>(S.F + a * kFS + v * 8);
                const int4 rvi = S.raw[raw_row(blk, v)];
                const uint32_t rw[4] = {uint32_t(rvi.x), uint32_t(rvi.y), uint32_t(rvi.z), uint32_t(rvi.w)};
                const uint32_t comp = I.bcomp[blk];
                if (!(S.cm[a] & 0x100u)) {
                    const float4 q0 = *reinterpret_cast<const float4*>(I.qf[comp] + v * 8);
                    const float4 q1 = *reinterpret_cast<const float4*>(I.qf[comp] + v * 8 + 4);
                    float c[8];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        c[2 * k] = float(int32_t(rw[k] << 16) >> 16);
                        c[2 * k + 1] = float(int32_t(rw[k]) >> 16);
                    }
                    const float2 p0 = __fmul2_rn(make_float2(c[0], c[1]), make_float2(q0.x, q0.y));
                    const float2 p1 = __fmul2_rn(make_float2(c[2], c[3]), make_float2(q0.z, q0.w));
                    const float2 p2 = __fmul2_rn(make_float2(c[4], c[5]), make_float2(q1.x, q1.y));
                    const float2 p3 = __fmul2_rn(make_float2(c[6], c[7]), make_float2(q1.z, q1.w));
                    dst[0] = make_float4(p0.x, p0.y, p1.x, p1.y);
                    dst[1] = make_float4(p2.x, p2.y, p3.x, p3.y);
                } else {  // exact-FP64 unit: keep the int32 bits
                    const float* qf = I.qf[comp] + v * 8;
                    int32_t d[8];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        d[2 * k] = int32_t(int16_t(rw[k] & 0xFFFFu)) * int32_t(qf[2 * k]);
                        d[2 * k + 1] = (int32_t(rw[k]) >> 16) * int32_t(qf[2 * k + 1]);
                    }
                    dst[0] = make_float4(__int_as_float(d[0]), __int_as_float(d[1]), __int_as_float(d[2]),
                                         __int_as_float(d[3]));
                    dst[1] = make_float4(__int_as_float(d[4]), __int_as_float(d[5]), __int_as_float(d[6]),
                                         __int_as_float(d[7]));
                }
            }
            // 2b. DC-only units: item = (unit, row x), two 4-byte stores of the constant sample
#pragma unroll 1
            for (uint32_t it = lane; it < ndc * 8; it += 32) {
                const uint32_t blk = S.dcl[it >> 3], x = it & 7;
                const int32_t F00 = (CMP ? S.dcv[blk] : int32_t(int16_t(uint32_t(S.raw[raw_row(blk, 0)].x) & 0xFFFFu))) *
                                    int32_t(I.qf[I.bcomp[blk]][0]);
                int o;
                if ((F00 & 7) != 4)
                    o = (F00 + 4) >> 3;
                else
                    o = lround_away(__dmul_rn(s_b64[0], __dmul_rn(s_b64[0], double(F00))));
                const uint32_t ov = clamp_u8(o + 128) * 0x01010101u;
                uint32_t* row = reinterpret_cast<uint32_t*>(S.pl + I.boff[blk] + x * I.bps[blk]);
                row[0] = ov;
                row[1] = ov;
            }
        }
        // advance the walk and prefetch the next tile (in flight during 3 + 4)
        if (t + 1 < t_end) {
            __syncwarp();
            if (lane == 0) {
                if (++w.tx == w.tiles_x) {
                    w.tx = 0;
                    ++w.my;
                }
                if (t + 1 >= w.kend) {
                    ++w.k;
                    walk_enter_image(P, t + 1, w);
                }
            }
            __syncwarp();  // staging consumed by every lane before it is refilled
            // a new image's entries start at its first unit (entry 0)
            issue(w, w.k == cur_k ? next_wstart : (w.tx == 0 && w.my == 0 ? 0u : kNoWin), next_wlen);
        }
        if (!cur_valid) continue;
        // the dequantised F tile (written lane-by-unit above) is read across lanes
        // below; the syncs around the prefetch only run when a next tile exists
        __syncwarp();

        // 3. IDCT of the AC units, eight per pass: lane = (unit a, rows q, 7-q / q+4)
        uint64_t pend = 0;  // per pass g: bit 16g + y (row q) / 16g + 8 + y (second row) need the FP64 replay
#pragma unroll 1
        for (uint32_t g = 0; g * 8 < nac; ++g) {
            const uint32_t a = g * 8 + (lane >> 2);
            const bool act = a < nac;
            const uint32_t cmw = act ? S.cm[a] : 0u;
            const uint32_t uor = __reduce_or_sync(0xFFFFFFFFu, cmw & 0xF000FFu);
            const uint32_t ucols = uor & 0xFFu;
            const bool urows_hi = (uor & 0xF00000u) != 0;
            const float* F = S.F + (act ? a : 0) * kFS;
            float2 acc[8];
#pragma unroll
            for (int y = 0; y < 8; ++y) acc[y] = make_float2(0.f, 0.f);
#if PJG_K4_SYM
            // x = q, 7-q: s(q) = E + O, s(7-q) = E - O with E / O the even / odd
            // u terms of the column sum, one packed chain over (u, u+1) pairs;
            // the row sums split the same way by the parity of v: out[x][y] =
            // Ev[y] + Ov[y], out[x][7-y] = Ev[y] - Ov[y] (y < 4).  Each nonzero
            // term still sees at most k (column) and m (row) roundings: a
            // chain of j nonzero terms rounds each at most j times and the join
            // adds one only when both halves are nonzero (j < k then).  The
            // mirrored FP32 basis factor is -b32[u][x] for odd u, one FP32
            // rounding of the reference's basis[u][7-x] up to its FP64 ulps
            // (covered by the bound's slack).
            float2 ae[4], ao[4];
#pragma unroll
            for (int y = 0; y < 4; ++y) ae[y] = ao[y] = make_float2(0.f, 0.f);
            auto colsum = [&](uint32_t v) -> float2 {
                const float4 f0 = *reinterpret_cast<const float4*>(F + v * 8);
                float2 eo = __fmul2_rn(bp[0], make_float2(f0.x, f0.y));
                eo = __ffma2_rn(bp[1], make_float2(f0.z, f0.w), eo);
                if (urows_hi) {
                    const float4 f1 = *reinterpret_cast<const float4*>(F + v * 8 + 4);
#if PJG_K4_COLSPLIT
                    // u >= 4 as a second, independent 2-deep chain joined by one add
                    float2 eh = __fmul2_rn(bp[2], make_float2(f1.x, f1.y));
                    eh = __ffma2_rn(bp[3], make_float2(f1.z, f1.w), eh);
                    eo = __fadd2_rn(eo, eh);
#else
                    eo = __ffma2_rn(bp[2], make_float2(f1.x, f1.y), eo);
                    eo = __ffma2_rn(bp[3], make_float2(f1.z, f1.w), eo);
#endif
                }
                return make_float2(__fadd_rn(eo.x, eo.y), __fsub_rn(eo.x, eo.y));
            };
#pragma unroll 1
            for (uint32_t m = ucols & 0x55u; m; m &= m - 1) {
                const uint32_t v = __ffs(m) - 1;
                const float2 sv = colsum(v);
                const float4 b0 = *reinterpret_cast<const float4*>(s_b32 + v * 8);
                ae[0] = __ffma2_rn(f2(b0.x), sv, ae[0]);
                ae[1] = __ffma2_rn(f2(b0.y), sv, ae[1]);
                ae[2] = __ffma2_rn(f2(b0.z), sv, ae[2]);
                ae[3] = __ffma2_rn(f2(b0.w), sv, ae[3]);
            }
#pragma unroll 1
            for (uint32_t m = ucols & 0xAAu; m; m &= m - 1) {
                const uint32_t v = __ffs(m) - 1;
                const float2 sv = colsum(v);
                const float4 b0 = *reinterpret_cast<const float4*>(s_b32 + v * 8);
                ao[0] = __ffma2_rn(f2(b0.x), sv, ao[0]);
                ao[1] = __ffma2_rn(f2(b0.y), sv, ao[1]);
                ao[2] = __ffma2_rn(f2(b0.z), sv, ao[2]);
                ao[3] = __ffma2_rn(f2(b0.w), sv, ao[3]);
            }
#pragma unroll
            for (int y = 0; y < 4; ++y) {
                acc[y] = __fadd2_rn(ae[y], ao[y]);
                acc[7 - y] = fsub2(ae[y], ao[y]);
            }
#else
            for (uint32_t m = ucols; m; m &= m - 1) {
                const uint32_t v = __ffs(m) - 1;
                // column sum over u in two 4-deep chains (u < 4, u >= 4) joined
                // by one add — the upper chain only when some unit of the pass
                // has a nonzero F[u >= 4] (warp-uniform).  Any order of k
                // nonzero terms rounds each at most k times (zero terms and
                // the join of a zero chain are exact): the bound is unchanged.
                const float4 f0 = *reinterpret_cast<const float4*>(F + v * 8);
                float2 sv = __fmul2_rn(bq[0], f2(f0.x));
                sv = __ffma2_rn(bq[1], f2(f0.y), sv);
                sv = __ffma2_rn(bq[2], f2(f0.z), sv);
                sv = __ffma2_rn(bq[3], f2(f0.w), sv);
                if (urows_hi) {
                    const float4 f1 = *reinterpret_cast<const float4*>(F + v * 8 + 4);
                    float2 sh = __fmul2_rn(bq[4], f2(f1.x));
                    sh = __ffma2_rn(bq[5], f2(f1.y), sh);
                    sh = __ffma2_rn(bq[6], f2(f1.z), sh);
                    sh = __ffma2_rn(bq[7], f2(f1.w), sh);
                    sv = __fadd2_rn(sv, sh);
                }
                const float4 b0 = *reinterpret_cast<const float4*>(s_b32 + v * 8);
                const float4 b1 = *reinterpret_cast<const float4*>(s_b32 + v * 8 + 4);
                acc[0] = __ffma2_rn(f2(b0.x), sv, acc[0]);
                acc[1] = __ffma2_rn(f2(b0.y), sv, acc[1]);
                acc[2] = __ffma2_rn(f2(b0.z), sv, acc[2]);
                acc[3] = __ffma2_rn(f2(b0.w), sv, acc[3]);
                acc[4] = __ffma2_rn(f2(b1.x), sv, acc[4]);
                acc[5] = __ffma2_rn(f2(b1.y), sv, acc[5]);
                acc[6] = __ffma2_rn(f2(b1.z), sv, acc[6]);
                acc[7] = __ffma2_rn(f2(b1.w), sv, acc[7]);
            }
#endif
            // round: v = acc + M holds round(acc) + 128 in its low bits
            int o0[8], o1[8];
            float mx = 0.f;
            const float2 M2 = f2(kM128);
#pragma unroll
            for (int y = 0; y < 8; ++y) {
                const float2 vv = __fadd2_rn(acc[y], M2);
                const float2 dd = fsub2(acc[y], fsub2(vv, M2));
                mx = fmaxf(mx, fmaxf(fabsf(dd.x), fabsf(dd.y)));
                o0[y] = __float_as_int(vv.x) - kMagicBits;
                o1[y] = __float_as_int(vv.y) - kMagicBits;
            }
            if (act) {
                const uint32_t blk = S.acl[a];
                uint8_t* pl = S.pl + I.boff[blk];
                const uint32_t ps = I.bps[blk];
                uint32_t* r0p = reinterpret_cast<uint32_t*>(pl + q * ps);
                uint32_t* r1p = reinterpret_cast<uint32_t*>(pl + (PJG_K4_SYM ? 7 - q : q + 4) * ps);
                r0p[0] = pack4_sat(o0[0], o0[1], o0[2], o0[3]);
                r0p[1] = pack4_sat(o0[4], o0[5], o0[6], o0[7]);
                r1p[0] = pack4_sat(o1[0], o1[1], o1[2], o1[3]);
                r1p[1] = pack4_sat(o1[4], o1[5], o1[6], o1[7]);
                if (cmw & 0x100u) {
                    pend |= 0xFFFFull << (16 * g);
                } else if (mx > S.lim[a]) {  // rare: the samples near x.5 get FP64 below
                    const float lim = S.lim[a];
                    uint32_t mask = 0;
#pragma unroll
                    for (int y = 0; y < 8; ++y) {
                        const float2 vv = __fadd2_rn(acc[y], M2);
                        const float2 dd = fsub2(acc[y], fsub2(vv, M2));
                        if (fabsf(dd.x) > lim) mask |= 1u << y;
                        if (fabsf(dd.y) > lim) mask |= 0x100u << y;
                    }
                    pend |= uint64_t(mask) << (16 * g);
                }
            }
        }
        // exact FP64 replay of the flagged samples, off the hot loop and
        // spread over the warp: lane i recomputes entry i of a work list
        n_ac += nac;
        if (__any_sync(0xFFFFFFFFu, pend != 0)) {
            const uint32_t cnt = __popcll(pend);
            uint32_t incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += x;
            }
            const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
            const uint32_t base = incl - cnt;
            n_replay += total;
            for (uint32_t rb = 0; rb < total; rb += 32) {
                if (cnt && base < rb + 32 && base + cnt > rb) {
                    uint32_t k = base;
                    for (uint64_t m = pend; m; m &= m - 1, ++k) {
                        if (k < rb) continue;
                        if (k >= rb + 32) break;
                        const uint32_t bit = __ffsll(m) - 1;  // 16 g + 8 h + y
                        const uint32_t a = (bit >> 4) * 8 + (lane >> 2);
                        const uint32_t x = ((bit >> 3) & 1u) ? (PJG_K4_SYM ? 7 - q : q + 4) : q;
                        S.rep[k - rb] = uint16_t((a << 6) | (x << 3) | (bit & 7u));
                    }
                }
                __syncwarp();
                if (rb + lane < total) {
                    const uint32_t e = S.rep[lane];
                    const uint32_t a = e >> 6, x = (e >> 3) & 7u, y = e & 7u;
                    const uint32_t blk = S.acl[a], cmw = S.cm[a];
                    const uint32_t o = idct_sample_fp64(S.F + a * kFS, cmw & 0x100u, cmw & 0xFFu, (cmw >> 16) & 0xFFu,
                                                        s_b64, int(x), int(y));
                    S.pl[I.boff[blk] + x * I.bps[blk] + y] = uint8_t(o);
                }
                __syncwarp();
            }
        }
        __syncwarp();

        // 4. output
        const uint32_t X0 = cur_mx0 * cur_mcuw, Y0 = cur_my * cur_mcuh;
        const uint32_t cols = min(cur_nm * cur_mcuw, I.width - X0), rws = min(cur_mcuh, I.height - Y0);
        const bool full = cols == uint32_t(kTileW) && rws == cur_mcuh && (I.width & 3) == 0 && (I.out_off & 3) == 0;
        uint8_t* stg = reinterpret_cast<uint8_t*>(S.F);  // RGB row staging (F is dead after the IDCT)
        if constexpr (LAYOUT == 1) {
            if (full)
                colour_full<2, true>(I, S.pl, s_lut, P.out, stg, X0, Y0, rws, lane);
            else
                colour_tile<2, true>(I, S.pl, s_lut, P.out, X0, Y0, cols, rws, lane);
        } else if (I.rgb && full) {
            if (I.h_max == 2) {
                if (I.v_max == 2)
                    colour_full<2, true>(I, S.pl, s_lut, P.out, stg, X0, Y0, rws, lane);
                else
                    colour_full<2, false>(I, S.pl, s_lut, P.out, stg, X0, Y0, rws, lane);
            } else {
                colour_full<1, false>(I, S.pl, s_lut, P.out, stg, X0, Y0, rws, lane);
            }
        } else if (I.rgb) {
            if (I.h_max == 2) {
                if (I.v_max == 2)
                    colour_tile<2, true>(I, S.pl, s_lut, P.out, X0, Y0, cols, rws, lane);
                else
                    colour_tile<2, false>(I, S.pl, s_lut, P.out, X0, Y0, cols, rws, lane);
            } else {
                colour_tile<1, false>(I, S.pl, s_lut, P.out, X0, Y0, cols, rws, lane);
            }
        } else if (I.out_mode == 1) {
            // grayscale RGB output (1 channel, the Y plane): item = 16 pixels of
            // a row (16 slots per row, up to 192 pixels used), one 16-byte
            // store when the destination is 16-byte aligned, else 4-byte words
            const uint32_t W = I.width;
            const bool al4 = ((W & 3) == 0) && ((I.out_off & 3) == 0);
            const bool al16 = ((W & 15) == 0) && ((I.out_off & 15) == 0) && (X0 & 15) == 0;
            uint8_t* obase = P.out + I.out_off + uint64_t(Y0) * W + X0;
            for (uint32_t it = lane; it < rws * 16; it += 32) {
                const uint32_t r = it >> 4, gx = (it & 15u) * 16;
                if (gx >= cols) continue;
                const uint32_t* src = reinterpret_cast<const uint32_t*>(S.pl + I.poff[0] + r * I.pst[0] + gx);
                const uint4 y16 = make_uint4(src[0], src[1], src[2], src[3]);
                uint8_t* dst = obase + uint64_t(r) * W + gx;
                if (gx + 16 <= cols && al16) {
                    *reinterpret_cast<uint4*>(dst) = y16;
                } else {
                    const uint32_t yw[4] = {y16.x, y16.y, y16.z, y16.w};
#pragma unroll
                    for (uint32_t k = 0; k < 4; ++k) {
                        const uint32_t g4 = gx + 4 * k;
                        if (g4 >= cols) break;
                        if (g4 + 4 <= cols && al4) {
                            *reinterpret_cast<uint32_t*>(dst + 4 * k) = yw[k];
                        } else {
                            for (uint32_t i = 0; i < min(4u, cols - g4); ++i) dst[4 * k + i] = uint8_t(yw[k] >> (8 * i));
                        }
                    }
                }
            }
        } else {
            // planes (extract_planes, transform.hpp:165-211); Grayscale output
            // (out_mode 2) is the Y plane alone — its region holds nothing else
            const uint32_t nplanes = I.out_mode == 2 ? 1u : I.ncomp;
            uint64_t plane_base = I.out_off;
#pragma unroll
            for (uint32_t c = 0; c < 3; ++c) {
                if (c >= nplanes) break;
                const uint32_t pw = I.plane_w[c], ph = I.plane_h[c];
                const uint32_t cx0 = cur_mx0 * I.comp_h[c] * 8, cy0 = cur_my * I.comp_v[c] * 8;
                const uint32_t ccols = cx0 < pw ? min(cur_nm * I.comp_h[c] * 8, pw - cx0) : 0;
                const uint32_t crows = cy0 < ph ? min(I.comp_v[c] * 8, ph - cy0) : 0;
                for (uint32_t e = lane; e < crows * ccols; e += 32) {
                    const uint32_t r = e / ccols, x = e % ccols;
                    P.out[plane_base + uint64_t(cy0 + r) * pw + cx0 + x] = S.pl[I.poff[c] + r * I.pst[c] + x];
                }
                plane_base += uint64_t(pw) * ph;
            }
        }
        __syncwarp();
    }
    if (P.stats) {
        n_replay = __reduce_add_sync(0xFFFFFFFFu, lane == 0 ? n_replay : 0u);
        n_ac = __reduce_add_sync(0xFFFFFFFFu, lane == 0 ? n_ac : 0u);
        if (lane == 0) {
            atomicAdd(P.stats + kStatReplays, (unsigned long long)n_replay);
            atomicAdd(P.stats + kStatAcUnits, (unsigned long long)n_ac);
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
// Per-(device, kernel) launch setup: the dynamic shared-memory opt-in is a
// per-device/context attribute, and the K4 grid cap depends on the device's
// SM count.  Several contexts on several devices (or host threads) may launch
// concurrently, so the cache is keyed by device and guarded by a mutex; the
// returned value is the kernel's resident CTAs per SM x SMs (0 when the
// caller did not ask for it).
// Programmatic dependent launch: a kernel may be scheduled while its
// predecessor's last CTAs drain; every kernel starts with griddepcontrol.wait
// (pdl_wait) before touching its predecessors' results, so ordering is that
// of the stream.  PJG_PDL=0 turns the attribute off.
static bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("PJG_PDL");
        return !(e && atoi(e) == 0);
    }();
    return on;
}
static void launch_pdl(void (*k)(Params), unsigned grid, unsigned block, size_t smem, cudaStream_t s, const Params& p) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, p);
}

static int launch_setup(const void* fn, int dyn_smem, int threads, bool want_grid) {
    static std::mutex mu;
    static std::unordered_map<uint64_t, int> done;  // (device, fn) -> grid cap + 1
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t key = (uint64_t(reinterpret_cast<uintptr_t>(fn)) << 8) ^ uint64_t(dev);
    std::lock_guard<std::mutex> g(mu);
    auto it = done.find(key);
    if (it != done.end()) return it->second - 1;
    if (dyn_smem > 0) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem);
    int cap = 0;
    if (want_grid) {
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, dyn_smem);
        cap = std::max(1, sms * std::max(per_sm, 1));
    }
    done.emplace(key, cap + 1);
    return cap;
}

uint32_t kernel_launches(const Params& p) {
    // mirrors the launch conditions of the launchers below
    return (p.k0_tiles ? 1u : 0u) + (p.n_dri ? 1u : 0u) + (p.k1_ctas ? 1u : 0u) + (p.k1_ctas > 1 ? (p.k1_hop ? 1u : 2u) : 0u) +
           (p.k2_tiles ? 1u : 0u) + (p.total_subs ? 1u : 0u) + (p.n_img ? 1u : 0u) + (p.k4_tiles ? 1u : 0u);
}
void launch_k0_unstuff(const Params& p, void* stream) {
    if (!p.k0_tiles) return;
    const int dyn = 2 * (kK0Threads * int(p.k0_bpt) + 32);
    cudaStream_t s = (cudaStream_t)stream;
    if (p.k0_bpt == 64) {
        if (p.n_dri) {
            launch_setup((const void*)k0_unstuff<true, 64>, dyn, kK0Threads, false);
            launch_pdl(k0_unstuff<true, 64>, p.k0_tiles, kK0Threads, dyn, s, p);
        } else {
            launch_setup((const void*)k0_unstuff<false, 64>, dyn, kK0Threads, false);
            launch_pdl(k0_unstuff<false, 64>, p.k0_tiles, kK0Threads, dyn, s, p);
        }
    } else {
        if (p.n_dri)
            launch_pdl(k0_unstuff_small<true>, p.k0_tiles, kK0Threads, 0, s, p);
        else
            launch_pdl(k0_unstuff_small<false>, p.k0_tiles, kK0Threads, 0, s, p);
    }
}
void launch_k0b_segments(const Params& p, void* stream) {
    if (p.n_dri) launch_pdl(k0b_segments, p.n_dri, 256, 0, (cudaStream_t)stream, p);
}
template <bool DRI, bool ST, bool HOP>
static void launch_k1_variant(const Params& p, size_t dyn, cudaStream_t s) {
    if (ST) launch_setup((const void*)k1_sync<DRI, ST, HOP, false>, kMaxSmemTables * kFastWords * 4, kK1Threads, false);
    if (!ST && p.sym_cap)
        launch_pdl(k1_sync<DRI, false, HOP, true>, p.k1_ctas, kK1Threads, dyn, s, p);
    else
        launch_pdl(k1_sync<DRI, ST, HOP, false>, p.k1_ctas, kK1Threads, dyn, s, p);
}
template <bool DRI, bool ST>
static void launch_k1_hop(const Params& p, size_t dyn, cudaStream_t s) {
    if (p.k1_hop)
        launch_k1_variant<DRI, ST, true>(p, dyn, s);
    else
        launch_k1_variant<DRI, ST, false>(p, dyn, s);
}
void launch_k1_sync(const Params& p, void* stream) {
    if (!p.k1_ctas) return;
    const size_t dyn = size_t(p.smem_tables) * kFastWords * 4;
    cudaStream_t s = (cudaStream_t)stream;
    if (p.smem_tables) {
        if (p.n_dri)
            launch_k1_hop<true, true>(p, dyn, s);
        else
            launch_k1_hop<false, true>(p, dyn, s);
    } else {
        if (p.n_dri)
            launch_k1_hop<true, false>(p, 0, s);
        else
            launch_k1_hop<false, false>(p, 0, s);
    }
}
void launch_k1c_fixup(const Params& p, void* stream) {
    if (p.k1_ctas <= 1) return;
    if (!p.k1_hop) {
        const unsigned grid = (p.k1_ctas - 1 + 127) / 128;
        if (p.n_huff <= kMaxSmemTables) {
            launch_setup((const void*)k1c_first<true>, kMaxSmemTables * kFastWords * 4, 128, false);
            launch_pdl(k1c_first<true>, grid, 128, size_t(p.n_huff) * kFastWords * 4, (cudaStream_t)stream, p);
        } else {
            launch_pdl(k1c_first<false>, grid, 128, 0, (cudaStream_t)stream, p);
        }
    }
    launch_pdl(k1c_fixup, 1, 1024, 0, (cudaStream_t)stream, p);
}
void launch_k1x_exact(const Params& p, void* stream) {
    if (p.n_img) launch_pdl(k1x_exact, std::min<uint32_t>(p.n_img, 296), kK1xThreads, 0, (cudaStream_t)stream, p);
}
void launch_k2_scan(const Params& p, void* stream) {
    if (p.k2_tiles) launch_pdl(k2_scan, p.k2_tiles, kK2Threads, 0, (cudaStream_t)stream, p);
}
template <bool ST, bool REPLAY, bool CMP>
static void launch_k3_variant(const Params& p, unsigned grid, cudaStream_t s) {
    if (ST) launch_setup((const void*)k3_write<ST, REPLAY, CMP>, kMaxSmemTables * kFastWords * 4, kK3Threads, false);
    size_t dyn = ST ? size_t(p.k3_tables) * kFastWords * 4 : 0;
    if (const char* e = getenv("PJG_K3_EXTRA_SMEM"))  // A/B: occupancy experiments (bytes)
        if (ST) dyn = std::min<size_t>(dyn + size_t(atol(e)), kMaxSmemTables * kFastWords * 4);
    launch_pdl(k3_write<ST, REPLAY, CMP>, grid, kK3Threads, dyn, s, p);
}
template <bool CMP>
static void launch_k3_cmp(const Params& p, unsigned grid, cudaStream_t s) {
    if (p.k3_tables)
        p.sym_cap ? launch_k3_variant<true, true, CMP>(p, grid, s) : launch_k3_variant<true, false, CMP>(p, grid, s);
    else
        p.sym_cap ? launch_k3_variant<false, true, CMP>(p, grid, s) : launch_k3_variant<false, false, CMP>(p, grid, s);
}
void launch_k3_write(const Params& p, void* stream) {
    if (!p.total_subs) return;
    const unsigned grid = unsigned((p.total_subs + kK3Threads - 1) / kK3Threads);
    cudaStream_t s = (cudaStream_t)stream;
    p.compact ? launch_k3_cmp<true>(p, grid, s) : launch_k3_cmp<false>(p, grid, s);
}
template <int LAYOUT, bool CMP>
static void launch_k4_variant(const Params& p, cudaStream_t s) {
    constexpr int kK4Threads = K4Shape<CMP>::kThreads, kK4Warps = K4Shape<CMP>::kWarps;
    constexpr size_t dyn = sizeof(WarpSmem<CMP>) * kK4Warps;
    int grid_cap = launch_setup((const void*)k4_transform<LAYOUT, CMP>, int(dyn), kK4Threads, true);
    if (const char* e = getenv("PJG_K4_OCC")) {  // A/B: K4 CTAs per SM (overlap experiments)
        int sms = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (atoi(e) > 0) grid_cap = std::min(grid_cap, sms * atoi(e));
    }
    const uint64_t want = (uint64_t(p.k4_tiles) + kK4Threads / 32 - 1) / (kK4Threads / 32);
    unsigned grid = unsigned(std::min<uint64_t>(want, uint64_t(grid_cap)));
    if (const char* e = getenv("PJG_K4_TPW"))  // A/B: tiles per warp (non-persistent grid, waves)
        if (atoi(e) > 0) grid = unsigned(std::max<uint64_t>(1, (want + atoi(e) - 1) / atoi(e)));
    launch_pdl(k4_transform<LAYOUT, CMP>, grid, kK4Threads, dyn, s, p);
}
void launch_k4_transform(const Params& p, void* stream) {
    if (!p.k4_tiles) return;
    const cudaStream_t s = (cudaStream_t)stream;
    if (p.compact)
        p.k4_layout == 1 ? launch_k4_variant<1, true>(p, s) : launch_k4_variant<0, true>(p, s);
    else
        p.k4_layout == 1 ? launch_k4_variant<1, false>(p, s) : launch_k4_variant<0, false>(p, s);
}
// Compact batches, coefficient dumps only: expand the entries of every image
// the fast path wrote (not K1x's — those are dense already) into the dense
// buffer (column-major int16[64], absolute DC), one warp per unit.
__global__ void k3d_densify(Params P) {
    const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (w >= P.total_dus) return;
    uint32_t lo = 0, hi = P.n_img;  // image of unit w
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (P.img[mid].du_first <= w)
            lo = mid;
        else
            hi = mid;
    }
    const ImgDesc& D = P.img[lo];
    const ImgState st = P.ist[lo];
    if (st.status != 0 || (st.exact & 2u) || !D.expected) return;
    const uint64_t d = w - D.du_first;
    if (d >= D.expected / 64) return;
    int16_t* dst = P.coef + w * 64;
    dst[lane] = 0;
    dst[lane + 32] = 0;
    __syncwarp();
    const uint4 m = P.umeta[w];
    const uint32_t* e = P.ents + D.du_first * 64;
    for (uint32_t j = m.x + lane; j < m.y; j += 32) {
        const uint32_t x = e[j];
        dst[(x >> 16) & 63u] = int16_t(x & 0xFFFFu);
    }
}
void launch_k3d_densify(const Params& p, void* stream) {
    if (!p.compact || !p.total_dus) return;
    const uint64_t threads = p.total_dus * 32;
    k3d_densify<<<unsigned((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(p);
}

}  // namespace pjg
