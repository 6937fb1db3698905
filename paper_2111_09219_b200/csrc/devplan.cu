// Device-side batch planning: the JFIF marker walk, table
// deduplication and construction, and the batch layout run as kernels, so the
// host only uploads the files once (whole files, one H2D) and reads back a
// few totals to size the decode's buffers and grids.  For thumbnail batches
// (tens of thousands of tiny files) this takes the per-file header work off
// the host's critical path.
//
//   P1 kp_parse   thread per file: parse() up to SOS (parser.hpp:264-347 with
//                 parse_dqt :139-154, parse_dht :156-178, parse_sof0 :180-233),
//                 same acceptance set and Errc precedence as the reference;
//                 build_table's error checks (huffman.hpp:60-93) for every
//                 present table (decode_single builds them after parse,
//                 pipeline.hpp:107-112 — the error is deferred past K0's scan
//                 checks exactly as on the host path)
//   P2 kp_dedup   thread per file: content hash of each referenced DC/AC/quant
//                 table into an open-addressing table (exact: equal hashes are
//                 byte-compared) -> batch-unique table ids
//   P3 kp_layout  one CTA: per-image counts (K0 tiles, subsequences, data
//                 units, K4 tiles, output bytes, restart segments) and their
//                 exclusive scans -> ImgDesc, prefix arrays, batch totals
//   (host reads the totals, sizes buffers)
//   P4 kp_tables  CTA per unique table: DevHuff (canonical code, 9-bit
//                 primary LUT, per-length maxcode, 11-bit fast table) and the
//                 column-major quantiser + K3 weights
//   P5 kp_lookups thread per image: K0-tile -> image and subsequence -> image
//                 lookup tables
#include <cub/block/block_scan.cuh>

#include "devparse.h"

namespace pjg {
namespace {

__device__ __constant__ uint8_t c_zz2r_plan[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
                                                  12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
                                                  35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
                                                  58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

__device__ __forceinline__ uint64_t aup(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

__global__ void __launch_bounds__(128) kp_parse(PlanParams P) {
    const uint32_t i = blockIdx.x * 128 + threadIdx.x;
    if (i >= P.n) return;
    DevHdr h;
    memset(&h, 0, sizeof(h));
    h.status = kMalformedHeader;
    h.h_max = h.v_max = 1;  // Header defaults (geometry of a file failing inside SOF)
    DReader r;
    r.base = P.raw;
    r.f0 = P.offsets[i];
    r.size = P.sizes[i];
    parse_file(r, P.allow_dri != 0, h);
    P.hdr[i] = h;
}

// ---- P2: table dedup ------------------------------------------------------
__device__ __forceinline__ uint64_t fnv(uint64_t hsh, uint32_t byte) { return (hsh ^ byte) * 0x100000001b3ull; }

__device__ uint64_t hash_huff(DReader& r, uint64_t off, uint32_t nsym, uint32_t dc) {
    uint64_t hsh = fnv(0xcbf29ce484222325ull, 0x48 + dc);
    for (uint32_t k = 0; k < 16 + nsym; ++k) hsh = fnv(hsh, r.byte_at(off + k));
    return hsh | 1ull;
}
__device__ __forceinline__ uint32_t quant_val(DReader& r, uint64_t off, uint32_t prec, uint32_t z) {
    return prec ? (r.byte_at(off + 2 * z) << 8) | r.byte_at(off + 2 * z + 1) : r.byte_at(off + z);
}
__device__ uint64_t hash_quant(DReader& r, uint64_t off, uint32_t prec) {
    uint64_t hsh = fnv(0xcbf29ce484222325ull, 0x51);
    for (uint32_t z = 0; z < 64; ++z) {
        const uint32_t v = quant_val(r, off, prec, z);
        hsh = fnv(fnv(hsh, v & 0xFFu), v >> 8);
    }
    return hsh | 1ull;
}

// Exact equality of two table specs in the raw buffer (absolute offsets).
__device__ bool same_spec(const uint8_t* raw, const TabRep& a, const TabRep& b) {
    if (a.kind != b.kind) return false;
    DReader ra, rb;
    ra.base = rb.base = raw;
    ra.size = rb.size = ~0ull;
    ra.f0 = a.off;
    rb.f0 = b.off;
    if (a.kind == 2) {
        for (uint32_t z = 0; z < 64; ++z)
            if (quant_val(ra, 0, a.prec, z) != quant_val(rb, 0, b.prec, z)) return false;
        return true;
    }
    if (a.nsym != b.nsym) return false;
    for (uint32_t k = 0; k < 16 + a.nsym; ++k)
        if (ra.byte_at(k) != rb.byte_at(k)) return false;
    return true;
}

__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Insert-or-find in the open-addressing table.  The inserting thread takes a
// fresh id from its kind's counter (huffman: DC and AC share one id space,
// the kind is part of the key) and publishes it with release semantics.
__device__ uint32_t dedup(const PlanParams& P, uint64_t hsh, const TabRep& rep) {
    uint32_t slot = uint32_t(hsh) & P.hmask;
    for (;;) {
        const unsigned long long k =
            atomicCAS(reinterpret_cast<unsigned long long*>(P.hkeys + slot), 0ull, (unsigned long long)hsh);
        if (k == 0ull) {
            const uint32_t id = atomicAdd(P.counters + (rep.kind == 2 ? kPlanQuant : kPlanHuff), 1u);
            P.hrep[slot] = rep;
            if (rep.kind == 2)
                P.uq[id] = rep;
            else
                P.uh[id] = rep;
            __threadfence();
            atomicExch(P.hval + slot, id + 1);
            return id;
        }
        if (k == hsh) {
            uint32_t v;
            while ((v = ld_acq(P.hval + slot)) == 0) __nanosleep(64);
            if (same_spec(P.raw, P.hrep[slot], rep)) return v - 1;
        }
        slot = (slot + 1) & P.hmask;
    }
}

__global__ void __launch_bounds__(128) kp_dedup(PlanParams P) {
    const uint32_t i = blockIdx.x * 128 + threadIdx.x;
    if (i >= P.n) return;
    DevHdr& h = P.hdr[i];
    if (h.status != kOk) return;
    DReader r;
    r.base = P.raw;
    r.f0 = P.offsets[i];
    r.size = P.sizes[i];
    const uint64_t f0 = P.offsets[i];
    for (uint32_t c = 0; c < h.ncomp; ++c) {
        if (h.table_status == kOk) {
            TabRep d{f0 + h.dc_off[h.td[c]], h.dc_n[h.td[c]], 0, 0};
            h.dc_id[c] = uint16_t(dedup(P, hash_huff(r, h.dc_off[h.td[c]], d.nsym, 1), d));
            TabRep a{f0 + h.ac_off[h.ta[c]], h.ac_n[h.ta[c]], 1, 0};
            h.ac_id[c] = uint16_t(dedup(P, hash_huff(r, h.ac_off[h.ta[c]], a.nsym, 0), a));
        }
        TabRep q{f0 + h.q_off[h.tq[c]], 0, 2, h.q_prec[h.tq[c]]};
        h.q_id[c] = uint16_t(dedup(P, hash_quant(r, h.q_off[h.tq[c]], q.prec), q));
    }
}

// ---- P3: layout -------------------------------------------------------------
struct CntSum {
    __device__ __forceinline__ Cnt operator()(const Cnt& a, const Cnt& b) const {
        return Cnt{a.sub + b.sub, a.du + b.du, a.outb + b.outb, a.seg + b.seg, a.k0t + b.k0t, a.k4t + b.k4t,
                   a.ndri + b.ndri, 0};
    }
};

__device__ __forceinline__ uint32_t comp_w(const DevHdr& h, uint32_t c) { return (h.width * h.ch[c] + h.h_max - 1) / h.h_max; }
__device__ __forceinline__ uint32_t comp_hh(const DevHdr& h, uint32_t c) { return (h.height * h.cv[c] + h.v_max - 1) / h.v_max; }

// fill_info (pjg_api.cu) from a device header
__device__ void make_info(const DevHdr& h, uint32_t mode, uint64_t compressed, pjg_image_info& info) {
    memset(&info, 0, sizeof(info));
    info.compressed_bytes = compressed;
    if (h.status != kOk && h.ncomp == 0) return;
    info.width = h.width;
    info.height = h.height;
    info.num_components = h.ncomp;
    for (uint32_t c = 0; c < h.ncomp; ++c) {
        info.plane_width[c] = comp_w(h, c);
        info.plane_height[c] = comp_hh(h, c);
    }
    info.h_max = h.h_max;
    info.v_max = h.v_max;
    info.mcus_x = h.mcus_x;
    info.mcus_y = h.mcus_y;
    info.data_units = uint64_t(h.mcus_x) * h.mcus_y * h.dpm;
    info.channels = mode == 1 ? (h.ncomp == 3 ? 3 : 1) : (mode == 2 ? 1 : h.ncomp);
    uint64_t ob = 0;
    if (h.ncomp) {
        if (mode == 1)
            ob = uint64_t(h.width) * h.height * (h.ncomp == 3 ? 3 : 1);
        else if (mode == 2)
            ob = uint64_t(comp_w(h, 0)) * comp_hh(h, 0);
        else
            for (uint32_t c = 0; c < h.ncomp; ++c) ob += uint64_t(comp_w(h, c)) * comp_hh(h, c);
    }
    info.output_bytes = ob;
}

constexpr int kLayThreads = 256;
using LayScan = cub::BlockScan<Cnt, kLayThreads>;
__device__ __forceinline__ Cnt cnt_zero() { return Cnt{0, 0, 0, 0, 0, 0, 0, 0}; }

// P3a, thread per image: the host planner's phase A (descriptor fields) and
// the counts of its pass 1 (pjg_api.cu) — same rules, same order; the CTA's
// count totals go to blk[blockIdx].
__global__ void __launch_bounds__(kLayThreads) kp_counts(PlanParams P) {
    __shared__ typename LayScan::TempStorage tmp;
    const uint32_t i = blockIdx.x * kLayThreads + threadIdx.x;
    Cnt c = cnt_zero();
    if (i < P.n) {
        const uint64_t k0_tile = uint64_t(kK0Threads) * P.k0_bpt;
        const DevHdr& h = P.hdr[i];
        pjg_image_info info;
        make_info(h, P.out_mode, P.sizes[i], info);
        P.info[i] = info;
        int32_t st = h.status;
        ImgDesc d;
        memset(&d, 0, sizeof(d));
        d.out_mode = P.out_mode;
        d.n_int = 1;
        if (st == kOk) {
            const uint64_t rl = P.sizes[i] - h.scan_start;
            d.raw_off = P.offsets[i] + h.scan_start;
            d.raw_len = rl;
            d.deferred = h.table_status;
            d.width = h.width;
            d.height = h.height;
            d.mcus_x = h.mcus_x;
            d.mcus_y = h.mcus_y;
            d.ncomp = h.ncomp;
            d.dpm = h.dpm;
            d.h_max = h.h_max;
            d.v_max = h.v_max;
            d.du_comp = h.du_comp;
            d.du_kslot = h.du_kslot;
            for (uint32_t cc = 0; cc < h.ncomp; ++cc) {
                d.comp_h[cc] = h.ch[cc];
                d.comp_v[cc] = h.cv[cc];
                d.plane_w[cc] = comp_w(h, cc);
                d.plane_h[cc] = comp_hh(h, cc);
                if (h.table_status == kOk) {
                    d.dc_tab[cc] = h.dc_id[cc];
                    d.ac_tab[cc] = h.ac_id[cc];
                }
                d.q_tab[cc] = h.q_id[cc];
            }
            PlanTotals& T = *P.totals;
            atomicAdd(reinterpret_cast<unsigned long long*>(&T.bits), (unsigned long long)rl * 8);
            atomicAdd(reinterpret_cast<unsigned long long*>(&T.raw), (unsigned long long)rl);
            atomicAdd(reinterpret_cast<unsigned long long*>(&T.n_ok), 1ull);
            if (!(h.ncomp == 3 && h.h_max == 2 && h.v_max == 2)) atomicOr(&T.all420, 1u);  // inverted below
            // K0 tiles always run (scan checks precede table errors); 16-byte-grid windows
            c.k0t = uint32_t(((d.raw_off & 15) + rl + k0_tile - 1) / k0_tile);
            if (h.table_status == kOk) {
                d.sub_count = (rl * 8 + P.sb_int - 1) / P.sb_int;
                const uint64_t m = uint64_t(h.mcus_x) * h.mcus_y;
                const uint64_t nint = h.restart_interval ? (m + h.restart_interval - 1) / h.restart_interval : 1;
                bool rejected = false;
                if (h.restart_interval && nint > 1) {
                    if (rl * 8 >= (1ull << 32)) {  // segment bit offsets are 32-bit
                        rejected = true;
                        st = kUnsupportedFeature;
                        d.sub_count = 0;
                    } else {
                        d.n_int = uint32_t(nint);
                        d.ri = h.restart_interval;
                        c.seg = d.n_int + 1;
                        d.sub_count += d.n_int;
                        c.ndri = 1;
                    }
                }
                if (!rejected) {
                    d.expected = m * h.dpm * 64;
                    d.mcus_per_tile = uint16_t(k4_mcus_per_tile(h.h_max, h.dpm));  // K4 warp tiles (<= 24 data units)
                    d.tiles_x = (h.mcus_x + d.mcus_per_tile - 1) / d.mcus_per_tile;
                    c.sub = d.sub_count;
                    c.du = d.expected / 64;
                    atomicMax(reinterpret_cast<unsigned long long*>(&P.totals->max_du), (unsigned long long)c.du);
                    c.k4t = d.tiles_x * h.mcus_y;
                    c.outb = aup(info.output_bytes, 256);
                }
            }
        }
        P.desc[i] = d;
        ImgState s;
        s.bit_length = 0;
        s.status = st;
        s.exact = 0;
        P.state[i] = s;
        P.state0[i] = s;
        P.cnt[i] = c;
    }
    Cnt ex, agg;
    LayScan(tmp).ExclusiveScan(c, ex, cnt_zero(), CntSum(), agg);
    if (threadIdx.x == 0) P.blk[blockIdx.x] = agg;
}

// P3b, one CTA: exclusive scan of the CTA totals, batch totals.
__global__ void __launch_bounds__(kLayThreads) kp_scan_blocks(PlanParams P, uint32_t nblk) {
    __shared__ typename LayScan::TempStorage tmp;
    __shared__ Cnt s_run;
    if (threadIdx.x == 0) s_run = cnt_zero();
    __syncthreads();
    for (uint32_t b0 = 0; b0 < nblk; b0 += kLayThreads) {
        const uint32_t b = b0 + threadIdx.x;
        const Cnt c = b < nblk ? P.blk[b] : cnt_zero();
        Cnt ex, agg;
        LayScan(tmp).ExclusiveScan(c, ex, cnt_zero(), CntSum(), agg);
        if (b < nblk) P.blk[b] = CntSum()(s_run, ex);
        __syncthreads();
        if (threadIdx.x == 0) s_run = CntSum()(s_run, agg);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        P.k0_first[P.n] = s_run.k0t;
        P.tile_first[P.n] = s_run.k4t;
        P.sub_first[P.n] = s_run.sub;
        PlanTotals& t = *P.totals;
        t.sub = s_run.sub;
        t.du = s_run.du;
        t.outb = s_run.outb;
        t.seg = s_run.seg;
        t.k0t = s_run.k0t;
        t.k4t = s_run.k4t;
        t.ndri = s_run.ndri;
        t.all420 = (t.n_ok && !t.all420) ? 1u : 0u;
        t.n_huff = P.counters[kPlanHuff];
        t.n_quant = P.counters[kPlanQuant];
    }
}

// P3c, thread per image: pass 2's offsets (the CTA's prefix + a block scan).
__global__ void __launch_bounds__(kLayThreads) kp_offsets(PlanParams P) {
    __shared__ typename LayScan::TempStorage tmp;
    const uint32_t i = blockIdx.x * kLayThreads + threadIdx.x;
    const Cnt c = i < P.n ? P.cnt[i] : cnt_zero();
    Cnt ex;
    LayScan(tmp).ExclusiveScan(c, ex, cnt_zero(), CntSum());
    if (i >= P.n) return;
    const Cnt r = CntSum()(P.blk[blockIdx.x], ex);
    P.k0_first[i] = r.k0t;
    P.tile_first[i] = r.k4t;
    P.sub_first[i] = r.sub;
    ImgDesc& d = P.desc[i];
    d.sub_first = r.sub;
    d.du_first = r.du;
    d.out_off = r.outb;
    if (c.ndri) {
        d.seg_first = r.seg;
        P.dri[r.ndri] = i;
    }
}

// ---- P4: unique tables -------------------------------------------------------
constexpr int kTabThreads = 256;

__global__ void __launch_bounds__(kTabThreads) kp_tables(PlanParams P, TableOut T) {
    __shared__ __align__(16) DevHuff s_t;
    __shared__ int32_t s_first[18], s_cnt[18];
    const uint32_t nh = T.n_huff, nq = T.n_quant;
    for (uint32_t u = blockIdx.x; u < nh + nq; u += gridDim.x) {
        if (u < nh) {
            const TabRep rep = P.uh[u];
            DReader r;
            r.base = P.raw;
            r.f0 = rep.off;
            r.size = ~0ull;
            uint32_t* w = reinterpret_cast<uint32_t*>(&s_t);
            for (uint32_t k = threadIdx.x; k < sizeof(DevHuff) / 4; k += kTabThreads) w[k] = 0;
            __syncthreads();
            if (threadIdx.x == 0) {  // canonical code (huffman.hpp:60-93), validated by P1
                uint32_t code = 0, si = 0, maxlen = 0;
                for (int len = 0; len <= 17; ++len) s_t.maxcode[len] = -1, s_cnt[len] = 0, s_first[len] = 0;
                for (uint32_t len = 1; len <= 16; ++len) {
                    const uint32_t n = r.byte_at(len - 1);
                    if (n) s_t.valoff[len] = int32_t(si) - int32_t(code);
                    s_first[len] = int32_t(code);
                    s_cnt[len] = int32_t(n);
                    si += n;
                    code += n;
                    if (n) {
                        maxlen = len;
                        s_t.maxcode[len] = int32_t(code) - 1;
                    }
                    code <<= 1;
                }
                s_t.maxlen = maxlen;
            }
            for (uint32_t k = threadIdx.x; k < rep.nsym; k += kTabThreads) s_t.symbols[k] = uint8_t(r.byte_at(16 + k));
            __syncthreads();
            // primary LUT: window w of kPrimaryBits bits -> the (unique) code prefixing it
            for (uint32_t wv = threadIdx.x; wv < (1u << kPrimaryBits); wv += kTabThreads) {
                uint16_t e = 0;
                for (int len = 1; len <= kPrimaryBits; ++len) {
                    const int32_t code = int32_t(wv >> (kPrimaryBits - len));
                    if (s_cnt[len] && code >= s_first[len] && code < s_first[len] + s_cnt[len]) {
                        e = uint16_t((uint32_t(len) << 8) | s_t.symbols[code + s_t.valoff[len]]);
                        break;
                    }
                }
                s_t.lut[wv] = e;
            }
            __syncthreads();
            if (threadIdx.x == 0) {  // second level for codes of 10..16 bits, in code order (jfif.cpp)
                uint32_t n2 = 0, k = 0;
                for (int len = 1; len <= 16; ++len)
                    for (int32_t j = 0; j < s_cnt[len]; ++j, ++k) {
                        if (len <= kPrimaryBits) continue;
                        const uint32_t code = uint32_t(s_first[len] + j);
                        const uint16_t e = uint16_t((uint32_t(len) << 8) | s_t.symbols[k]);
                        const uint32_t pre = code >> (len - kPrimaryBits);
                        if (s_t.lut[pre] == 0 && n2 < uint32_t(kL2Tables)) s_t.lut[pre] = uint16_t(kL2Flag | n2++);
                        if (!(s_t.lut[pre] & kL2Flag)) continue;
                        const uint32_t shift = 16 - len;
                        const uint32_t first = (code << shift) & ((1u << (16 - kPrimaryBits)) - 1);
                        for (uint32_t i = 0; i < (1u << shift); ++i) s_t.lut2[s_t.lut[pre] & 0x7FFFu][first + i] = e;
                    }
            }
            __syncthreads();
            // fast table (jfif.cpp build_fast): decode_next_symbol resolved per
            // 11-bit window; prefixes of longer codes get second-level tables
            // in prefix order (warp 0 numbers them with a ballot scan)
            const bool dc = rep.kind == 0;
            for (uint32_t wv = threadIdx.x; wv < (1u << kFastBits); wv += kTabThreads) {
                const int64_t f = fast_primary(s_t, wv, dc);
                s_t.fast[wv] = f >= 0 ? uint32_t(f) : 0xFFFFFFFFu;
            }
            __syncthreads();
            if (threadIdx.x < 32) {
                uint32_t n2 = 0;
                for (uint32_t w0 = 0; w0 < (1u << kFastBits); w0 += 32) {
                    const uint32_t wv = w0 + threadIdx.x;
                    const bool lng = s_t.fast[wv] == 0xFFFFFFFFu;
                    const uint32_t m = __ballot_sync(0xFFFFFFFFu, lng);
                    const uint32_t k2 = n2 + __popc(m & ((1u << threadIdx.x) - 1u));
                    if (lng) s_t.fast[wv] = k2 < uint32_t(kL2Fast) ? (kFastL2 | (k2 << 10)) : 0u;
                    n2 += __popc(m);
                }
            }
            __syncthreads();
            for (uint32_t x = threadIdx.x; x < uint32_t(kL2Fast) * 32; x += kTabThreads) s_t.fast2[x >> 5][x & 31] = 0;
            __syncthreads();
            for (uint32_t x = threadIdx.x; x < (1u << kFastBits) * 32; x += kTabThreads) {
                const uint32_t wv = x >> 5, f = s_t.fast[wv];
                if ((f & 0x3FFu) == kFastL2) s_t.fast2[(f >> 10) & 31u][x & 31] = fast_secondary(s_t, wv, x & 31, dc);
            }
            __syncthreads();
            uint4* dst = reinterpret_cast<uint4*>(T.huff + u);
            const uint4* src = reinterpret_cast<const uint4*>(&s_t);
            for (uint32_t k = threadIdx.x; k < sizeof(DevHuff) / 16; k += kTabThreads) dst[k] = src[k];
            __syncthreads();
        } else if (threadIdx.x < 64) {  // quantiser (column-major) + K3 weights, as the host planner
            const uint32_t q = u - nh;
            const TabRep rep = P.uq[q];
            DReader r;
            r.base = P.raw;
            r.f0 = rep.off;
            r.size = ~0ull;
            const uint32_t z = threadIdx.x;
            const uint32_t v = quant_val(r, 0, rep.prec, z);
            const uint32_t rr = c_zz2r_plan[z];
            T.quant[q * 64 + (rr & 7) * 8 + (rr >> 3)] = uint16_t(v);
            const double kW[8] = {0.35356, 0.4904, 0.46195, 0.4904, 0.35356, 0.4904, 0.46195, 0.4904};
            T.wq[q * 64 + z] = float(__dmul_rn(__dmul_rn(__dmul_rn(kW[rr >> 3], kW[rr & 7]), double(v)), 1.0 + 1e-6));
        }
    }
}

// ---- P5: lookup tables -------------------------------------------------------
__global__ void kp_lookups(PlanParams P, uint32_t* k0img, uint32_t* subimg, uint64_t n_subimg) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.n) return;
    for (uint32_t t = P.k0_first[i]; t < P.k0_first[i + 1]; ++t) k0img[t] = i;
    // subimg[c] = largest k < n with sub_first[k] <= c << kSubImgShift
    const uint64_t lo = P.sub_first[i], hi = i + 1 < P.n ? P.sub_first[i + 1] : ~0ull;
    if (lo == hi) return;
    const uint64_t s = 1ull << kSubImgShift;
    const uint64_t c0 = (lo + s - 1) >> kSubImgShift;
    const uint64_t ch = (hi + s - 1) >> kSubImgShift;
    const uint64_t c1 = (hi == ~0ull || ch > n_subimg) ? n_subimg : ch;
    for (uint64_t c = c0; c < c1; ++c) subimg[c] = i;
}

}  // namespace

void launch_plan_parse(const PlanParams& p, void* stream) {
    const cudaStream_t s = (cudaStream_t)stream;
    const unsigned g = unsigned((p.n + 127) / 128);
    if (!g) return;
    kp_parse<<<g, 128, 0, s>>>(p);
    kp_dedup<<<g, 128, 0, s>>>(p);
    const uint32_t nblk = uint32_t((p.n + kLayThreads - 1) / kLayThreads);
    kp_counts<<<nblk, kLayThreads, 0, s>>>(p);
    kp_scan_blocks<<<1, kLayThreads, 0, s>>>(p, nblk);
    kp_offsets<<<nblk, kLayThreads, 0, s>>>(p);
}

void launch_plan_finish(const PlanParams& p, const TableOut& t, uint32_t* k0img, uint32_t* subimg, uint64_t n_subimg,
                        void* stream) {
    const cudaStream_t s = (cudaStream_t)stream;
    if (t.n_huff + t.n_quant) kp_tables<<<std::min<uint32_t>(t.n_huff + t.n_quant, 148 * 4), kTabThreads, 0, s>>>(p, t);
    if (p.n) kp_lookups<<<unsigned((p.n + 127) / 128), 128, 0, s>>>(p, k0img, subimg, n_subimg);
}

}  // namespace pjg
