// Internal layout shared by the host planner (pjg_api.cu, jfif.cpp) and the
// sm_100a kernels (kernels.cu).  Not part of the public C-ABI (include/pjg.h).
#pragma once

#include <stdint.h>
#ifndef __CUDACC__
struct uint2 { unsigned int x, y; };
struct uint4 { unsigned int x, y, z, w; };
#else
#include <vector_types.h>
#endif

#ifdef __CUDACC__
#define PJG_HD __host__ __device__ __forceinline__
#else
#define PJG_HD inline
#endif

namespace pjg {

// ---------------------------------------------------------------- status --
// Mirrors pjpeg::Errc (reference common.hpp:26-38); C-ABI value = ordinal+1.
enum Status : int32_t {
    kOk = 0,
    kMalformedStuffing = 1,
    kEmptyScan = 2,
    kOutOfBits = 3,
    kUnsupportedFeature = 4,
    kMalformedHeader = 5,
    kMissingTable = 6,
    kOversubscribedCode = 7,
    kInvalidCode = 8,
    kConsistencyFailure = 9,
    kEmptyCorpus = 10,
    kIoError = 11,
};

// ------------------------------------------------------- Huffman tables --
// Two-level canonical decoder reproducing the reference's flat 2^maxlen LUT
// (huffman.hpp:60-93, 113-130) bit for bit: a 9-bit primary table resolves
// codes of length <= 9; a code of 10..16 bits is found in the 128-entry
// second-level table of its 9-bit prefix (up to kL2Tables prefixes; beyond
// that the per-length maxcode walk of Annex F.2.2.3).
constexpr int kPrimaryBits = 9;

constexpr int kFastBits = 11;
constexpr uint32_t kFastWords = 1u << kFastBits;
// fast entry for a kFastBits window whose codeword fits and decodes to a
// symbol the reference accepts (0 = take the exact path):
//   bits 0-4 codeword length, 5-8 magnitude bits l, bit 9 zero (so that
//   entry >> 5 is a valid 5-bit shift count l), 10-20 2^l - 1 (extend()'s
//   offset), 21-26 slots advanced (run + 1; 0 = EOB), 27-31 code + magnitude
//   length.  A coefficient is written for DC symbols and for l != 0.
constexpr uint32_t kFastLShift = 5, kFastTShift = 10, kFastR1Shift = 21, kFastLenShift = 27;
// Codes longer than kFastBits: the fast entry of their 11-bit prefix points
// (kFastL2 | k << 10, clen 0) at second-level table k of 32 entries indexed by
// the next 5 window bits, same entry format (code lengths 12..16).  Prefixes
// beyond kL2Fast tables, and invalid windows, keep 0: the exact path.
constexpr uint32_t kFastL2 = 1u << 9;
constexpr int kL2Fast = 16;

constexpr int kL2Tables = 16;  // second-level tables (codes of 10..16 bits) per Huffman table
constexpr uint32_t kL2Flag = 0x8000u;

struct DevHuff {
    uint32_t fast[1 << kFastBits];    // decode_next_symbol per kFastBits window (codes <= kFastBits bits)
    uint32_t fast2[kL2Fast][32];      // second level: codes of 12..16 bits
    uint16_t lut[1 << kPrimaryBits];  // (length << 8) | symbol; 0 = unresolved; kL2Flag | k: second level k
    uint16_t lut2[kL2Tables][1 << (16 - kPrimaryBits)];  // by the 7 bits after a 9-bit prefix of long codes
    int32_t maxcode[18];              // per length 1..16 ([17] unused), -1 when no code has that length
    int32_t valoff[18];               // symbol index = code + valoff[len]
    uint8_t symbols[256];
    uint32_t maxlen;                  // reference HuffmanTable::max_code_length
    uint32_t pad[3];
};
static_assert(sizeof(DevHuff) % 16 == 0, "DevHuff must stay 16-byte aligned");

// Decodes one codeword from the top 16 bits of `w16` (MSB first).  Returns
// (length << 8) | symbol, or 0 when no code matches the first maxlen bits —
// the reference's `e.length == 0`.
PJG_HD uint32_t huff_lookup(const DevHuff& t, uint32_t w16) {
    uint32_t e = t.lut[w16 >> (16 - kPrimaryBits)];
    if (e & kL2Flag) return t.lut2[e & 0x7FFFu][w16 & ((1u << (16 - kPrimaryBits)) - 1)];
    if (e != 0) return e;
    for (uint32_t len = kPrimaryBits + 1; len <= t.maxlen; ++len) {
        int32_t code = int32_t(w16 >> (16 - len));
        if (code <= t.maxcode[len]) return (len << 8) | t.symbols[code + t.valoff[len]];
    }
    return 0;
}

// Fast entry of one decoded codeword (e = huff_lookup result, clen >= 1):
// the fields decode_next_symbol needs, or 0 for symbols the reference
// rejects (they take the exact path for its error order).
PJG_HD uint32_t fast_fields(uint32_t e, bool dc) {
    const uint32_t clen = e >> 8, sym = e & 255u;
    uint32_t l = 0, run = 0, kind = 0;
    bool ok = true;
    if (dc) {
        l = sym;
        ok = l <= 11;
    } else {
        run = sym >> 4;
        l = sym & 15u;
        if (l == 0) {
            if (run == 0)
                kind = 1;
            else if (run == 15)
                kind = 2;
            else
                ok = false;
        } else if (l > 10) {
            ok = false;
        }
    }
    // slots advanced = run + 1, 0 for EOB (64 - z, known on the device)
    return ok ? clen | (l << kFastLShift) | (((1u << l) - 1u) << kFastTShift) |
                    ((kind == 1 ? 0u : run + 1u) << kFastR1Shift) | ((clen + l) << kFastLenShift)
              : 0u;
}
// Entry of window w11 (top kFastBits bits) of a table whose canonical code
// is set up (lut/lut2/maxcode): a direct entry, 0, or -1 when the prefix
// belongs to a code longer than kFastBits (needs a second-level table).
PJG_HD int64_t fast_primary(const DevHuff& t, uint32_t w11, bool dc) {
    const uint32_t e = huff_lookup(t, w11 << (16 - kFastBits));
    const uint32_t clen = e >> 8;
    if (clen == 0) return 0;
    if (clen > uint32_t(kFastBits)) return -1;
    return fast_fields(e, dc);
}
// Second-level entry for prefix w11 and the next 5 bits s.
PJG_HD uint32_t fast_secondary(const DevHuff& t, uint32_t w11, uint32_t s, bool dc) {
    const uint32_t e = huff_lookup(t, (w11 << (16 - kFastBits)) | s);
    return (e >> 8) ? fast_fields(e, dc) : 0u;
}

// -------------------------------------------------------------- images --
constexpr int kMaxSlots = 10;  // data units per MCU (4:2:0 → 6)

struct ImgDesc {
    // input: the raw bytes following the SOS header, in the batch's raw buffer
    uint64_t raw_off;      // byte offset of the first scan byte (== unstuffed offset)
    uint64_t raw_len;      // bytes from the first scan byte to the end of the file
    // geometry (parser.hpp:56-85)
    uint32_t width, height;
    uint32_t mcus_x, mcus_y;
    uint32_t ncomp, dpm, h_max, v_max;
    uint32_t comp_h[3], comp_v[3];
    uint32_t plane_w[3], plane_h[3];
    uint64_t du_comp;      // slot -> component, 4 bits per slot
    uint64_t du_kslot;     // slot -> index of that unit within its component, 4 bits per slot
    uint16_t dc_tab[3], ac_tab[3], q_tab[3];
    uint16_t mcus_per_tile;  // K4 tile width in MCUs
    // partition / layout
    uint64_t sub_first;    // first global subsequence
    uint64_t sub_count;    // allocated subsequences (upper bound from raw_len)
    uint64_t du_first;     // first data unit in the batch coefficient buffer
    uint64_t out_off;      // byte offset of this image in the batch output buffer
    uint64_t expected;     // 64 * total data units (parallel_decode.hpp:341)
    uint32_t out_mode;     // pjg_output_kind
    int32_t deferred;      // build_table error, applied after K0's scan checks
    uint32_t tiles_x;      // K4 tiles per MCU row
    // restart intervals (extension; 1 interval = the reference's single scan)
    uint32_t n_int;        // intervals; > 1 only with DRI and RST markers
    uint32_t ri;           // MCUs per interval (DRI Ri), 0 = none
    uint32_t pad1;
    uint64_t seg_first;    // this image's segment table in Params::segs (n_int + 1 entries)
};

// Per-image results written by the device.
struct ImgState {
    uint64_t bit_length;   // 8 * unstuffed bytes (bitstream.hpp:74), written by K0
    int32_t status;        // first error (Status), 0 = ok
    uint32_t exact;        // bit 0: K3 saw an AC run past the unit end; bit 1: K1x re-decoded the image
                           // (its s_info entries are then at the configured partition)
};

// ----------------------------------------------------------- sync state --
// One s_info entry (parallel_decode.hpp:64-84): state after the last symbol
// owned by a subsequence.  czd packs c (bits 0-3), z (bits 4-10) and the
// divergence flag (bit 15); n is the coefficient-slot count.
struct Entry {
    uint64_t p;
    uint32_t n;
    uint32_t czd;
};
static_assert(sizeof(Entry) == 16, "Entry layout");

constexpr uint32_t kDivBit = 0x8000u;
constexpr uint32_t kBoundaryBit = 0x4000u;  // cta_start only: CTA starts mid-image

PJG_HD uint32_t pack_czd(uint32_t c, uint32_t z, bool div) {
    return c | (z << 4) | (div ? kDivBit : 0u);
}
PJG_HD uint32_t czd_c(uint32_t v) { return v & 15u; }
PJG_HD uint32_t czd_z(uint32_t v) { return (v >> 4) & 127u; }
PJG_HD bool czd_div(uint32_t v) { return (v & kDivBit) != 0; }
// sync_equal (parallel_decode.hpp:81-84): divergence flag, p, c, z; n ignored.
PJG_HD bool sync_equal(uint64_t pa, uint32_t ca, uint64_t pb, uint32_t cb) {
    return pa == pb && ((ca ^ cb) & (kDivBit | 0x7FFu)) == 0;
}

// Per-subsequence DC-difference sums, one 16-bit lane per component
// (dc_prefix_sum accumulates in int32 and stores int16: transform.hpp:56-74,
// so only the sum mod 2^16 matters).  lanes 0,1 in lo; lane 2 in hi.
struct DcSums {
    uint32_t lo, hi;
};

// ------------------------------------------------------------- params --
constexpr int kSubImgShift = 7;
constexpr uint32_t kMaxSmemTables = 4;  // fast tables K1/K3 stage in shared memory (8 KB each)
constexpr int kK0Threads = 512;
constexpr uint32_t kK0BigBpt = 64, kK0SmallBpt = 16;  // bytes per K0 thread: 32 KB or 8 KB tiles
constexpr int kK1Threads = 128;                          // threads per K1 CTA
constexpr int kK1Spec = 4;                               // K1 threads re-decoding the predecessor CTA's last subsequences
constexpr int kK1Own = kK1Threads - kK1Spec;             // subsequences owned per K1 CTA
constexpr int kK2Threads = 256;
constexpr int kK3Threads = 128;
constexpr int kK4Threads = 128;
constexpr int kK4MaxBlocks = 24;                         // data units per K4 (warp) tile
// K4 tile width in MCUs: 64-pixel-wide tiles (<= 24 data units), except
// one-unit-per-MCU grayscale scans, whose 64-pixel tile held only 8 units (the
// per-tile walk / classify / prefetch cost was paid per 8 units): 192 pixels,
// 24 units, 1568 bytes of sample plane.
PJG_HD uint32_t k4_mcus_per_tile(uint32_t h_max, uint32_t dpm) {
    return dpm == 1 ? uint32_t(kK4MaxBlocks) : 64u / (8u * h_max);
}

struct Params {
    // batch
    const ImgDesc* img;
    ImgState* ist;
    uint32_t n_img;
    uint32_t epoch;
    const DevHuff* huff;
    const uint16_t* quant_raster;  // 64 uint16 per table, RASTER order
    const double* basis;           // 64 doubles, basis[u][x] (host std::cos)
    const float* wq;               // per quant table, zig-zag order: w_u w_v Q (K3 metadata)
    uint32_t n_quant;              // quant tables in the batch
    // raw & unstuffed scan
    const uint8_t* raw;
    uint8_t* ubuf;
    // K0 tiles
    const uint32_t* k0_first;      // n_img + 1 prefix
    const uint32_t* k0_img;        // image of each K0 tile
    const uint32_t* sub_img;       // image of subsequence c << kSubImgShift, c = 0..ceil(total/128)
    // restart-interval segments (DRI images only): per image n_int + 1 entries,
    // x = first unstuffed bit of interval m (x[n_int] = bit length), y = first
    // image-local subsequence of interval m (y[n_int] = subsequences in use)
    uint2* segs;
    const uint32_t* dri_img;       // the batch's DRI images
    uint32_t n_dri;
    uint32_t k0_tiles;
    uint32_t k1_ctas;
    uint32_t k0_bpt;               // K0 bytes per thread (tile = 512 x this)
    uint32_t smem_tables;          // K1/K3 stage this many fast tables in shared memory (0: read global)
    uint32_t n_huff;               // unique Huffman tables of the batch
    uint32_t k1_hop;               // K1 re-chains stale CTA starts in-kernel (small grids); else K1c first pass
    uint32_t k4_layout;            // 1: every image is 4:2:0 colour to RGB (specialised K4); 0: any
    // subsequences
    uint64_t sb;                   // subsequence_bits (internal: may be a divisor of sb_cfg)
    uint64_t sb_cfg;               // the configured subsequence_bits (K1x replays the reference partition)
    uint32_t b_cfg;                // the configured sequence_length_b
    uint32_t pad_b;
    const uint64_t* sub_first;     // n_img + 1 prefix
    uint64_t total_subs;
    Entry* ent;
    DcSums* dcs;
    uint64_t* off;                 // trimmed exclusive offsets (slots)
    uint32_t* cap;                 // trimmed counts
    DcSums* pred;                  // DC predictor at the start of each subsequence
    Entry* cta_end;                // K1: each CTA's last entry after intra sync
    Entry* cta_start;              // K1: start state each CTA's inter overflow used
    uint16_t* sym;                 // K1 chains' decoded symbols: symbol i of subsequence g at [i * sym_stride + g]
    uint32_t* tag;                 // 4 words per subsequence: start state / count / epoch of its stored symbols
    uint64_t sym_stride;           // >= total_subs, multiple of 64
    uint32_t sym_cap;              // symbols kept per subsequence (0: K3 always decodes)
    uint32_t* k1_flag;
    uint32_t k2_tiles;
    uint32_t k4_tiles;
    // K4
    const uint32_t* tile_first;    // n_img + 1 prefix of K4 tiles
    int16_t* coef;                 // 64 int16 per data unit, raster order, absolute DC
    uint2* meta;                   // per data unit: flags (row mask | has-AC | big), S (K3 -> K4)
    // compact coefficient interface (compact != 0): K3 emits one 32-bit entry
    // per coded coefficient (every DC, every nonzero AC) instead of 64 int16
    // slots per unit — col-major index << 16 | uint16 value (DC absolute) —
    // at ents[64 * du_first + e], e = the image-relative entry position (K1
    // counts entries per subsequence, K2 scans them into eoff); per unit
    // umeta = (first entry, end entry, flags, S) relative to 64 * du_first
    uint32_t* ents;
    uint4* umeta;
    uint32_t* eoff;                // per subsequence: first entry (image-relative), K2 -> K3
    uint32_t compact;
    uint32_t k3_tables;            // fast tables K3 stages in shared memory (0: global)
    uint64_t total_dus;
    uint8_t* out;
    // lookback scratch
    uint32_t* counters;            // tickets (reset per run)
    uint32_t* k0_flag;
    uint64_t* k0_agg;              // 4 x uint64 per tile: aggregate (cnt, mk), inclusive (cnt, mk)
    uint32_t* k2_flag;
    uint64_t* k2_agg;              // 4 x uint64 per tile: aggregate (n|head, dc), inclusive (n, dc)
    // stats
    unsigned long long* stats;     // see StatIndex
    uint32_t pad3;
};

enum Counter { kTicketK0 = 0, kTicketK1 = 1, kTicketK2 = 2, kNumCounters = 8 };
enum StatIndex {
    kStatRoundsSum = 0,    // intra rounds summed over K1 CTAs
    kStatRoundsMax = 1,
    kStatInterHops = 2,    // subsequences decoded by inter-CTA overflows
    kStatFixPasses = 3,    // K1c passes that found work
    kStatReplays = 4,      // K4 samples recomputed in exact FP64
    kStatAcUnits = 5,      // K4 data units with AC terms (FP32 IDCT path)
    kStatEntries = 6,      // compact entries K3 wrote
    kNumStats = 8
};

// Kernel launchers (kernels.cu).  All are stream-ordered, no host syncs.
uint32_t kernel_launches(const Params& p);  // kernels one decode launches
void launch_k0_unstuff(const Params& p, void* stream);
void launch_k0b_segments(const Params& p, void* stream);
void launch_k1_sync(const Params& p, void* stream);
void launch_k1c_fixup(const Params& p, void* stream);
void launch_k2_scan(const Params& p, void* stream);
void launch_k1x_exact(const Params& p, void* stream);
void launch_k3_write(const Params& p, void* stream);
void launch_k4_transform(const Params& p, void* stream);
void launch_k3d_densify(const Params& p, void* stream);  // compact batches: entries -> coef (dumps)
void launch_k5_color(const uint8_t* y, const uint8_t* cb, const uint8_t* cr, uint32_t W, uint32_t H,
                     uint32_t pw0, uint32_t pw1, uint32_t ph1, uint32_t pw2, uint32_t ph2, uint8_t* out,
                     void* stream);

}  // namespace pjg
