/*
 * pjg — C-ABI of the B200-native baseline-JPEG decoder (drop-in boundary).
 *
 * The reference (pjpeg, /root/reference/proj) exposes a header-only C++ API
 * and no FFI; the entry points below are what a binding of that API needs
 * (SURVEY.md §8b).  Each function names the reference interface it replaces.
 * Plain pointers and sizes only; no torch types.
 *
 * Status codes: 0 = success; 1..11 = pjpeg::Errc ordinal + 1
 * (reference proj/include/pjpeg/common.hpp:26-38); >= 100 = runtime errors of
 * this library (CUDA failure, bad argument, capacity).
 *
 * Threading: one pjg_ctx per (host thread, GPU).  All device work of a context
 * is ordered on the context's CUDA stream.  No global mutable state.
 */
#ifndef PJG_H
#define PJG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum pjg_status {
    PJG_OK = 0,
    PJG_MALFORMED_STUFFING = 1,
    PJG_EMPTY_SCAN = 2,
    PJG_OUT_OF_BITS = 3,
    PJG_UNSUPPORTED_FEATURE = 4,
    PJG_MALFORMED_HEADER = 5,
    PJG_MISSING_TABLE = 6,
    PJG_OVERSUBSCRIBED_CODE = 7,
    PJG_INVALID_CODE = 8,
    PJG_CONSISTENCY_FAILURE = 9,
    PJG_EMPTY_CORPUS = 10,
    PJG_IO_ERROR = 11,
    PJG_CUDA_ERROR = 100,
    PJG_INVALID_ARGUMENT = 101,
    PJG_CAPACITY = 102,
    PJG_NOT_DECODED = 103
};

/* pjpeg::OutputColorspace (pipeline.hpp:34) */
enum pjg_output_kind {
    PJG_OUT_PLANES = 0, /* YCbCrPlanes: component planes back to back (extract_planes) */
    PJG_OUT_RGB = 1,    /* RGBInterleaved: upsample_and_convert (1 channel for gray) */
    PJG_OUT_GRAY = 2    /* Grayscale: the Y plane only */
};

/* pjpeg::DecodeConfig (pipeline.hpp:36-41) */
typedef struct pjg_config {
    uint64_t subsequence_bits;  /* positive multiple of 32 (parallel_decode.hpp:51) */
    uint32_t sequence_length_b; /* >= 1; accepted for parity, grouping is per CTA */
    uint32_t output;            /* pjg_output_kind */
    uint32_t restart_intervals; /* 0 (default): DRI != 0 is UnsupportedFeature, as the
                                   reference (parser.hpp:299-302); 1: decode restart
                                   intervals (DRI + RST0-7), an extension */
    uint32_t reserved;
} pjg_config;

/* Geometry of one decoded image (ImagePlanes / RgbImage, transform.hpp:38-51,
 * pipeline.hpp:64-69). */
typedef struct pjg_image_info {
    uint32_t width, height;
    uint32_t channels;       /* channels of the chosen output (3, or 1) */
    uint32_t num_components; /* 1..3 */
    uint32_t plane_width[3], plane_height[3];
    uint32_t h_max, v_max;
    uint32_t mcus_x, mcus_y;
    uint64_t output_bytes;   /* bytes of the chosen output */
    uint64_t compressed_bytes;
    uint64_t data_units;
} pjg_image_info;

/* One s_info entry (parallel_decode.hpp:64-79), bit positions in unstuffed space. */
typedef struct pjg_sync_entry {
    uint64_t p;
    uint64_t n; /* trimmed slot count (after offsets(), :290-316) */
    uint32_t c, z;
    uint32_t divergent;
    uint32_t pad;
} pjg_sync_entry;

/* Per-stage device times of the last decode, milliseconds (StageTimings,
 * pipeline.hpp:44-62, measured with CUDA events). */
enum pjg_stage {
    PJG_STAGE_UPLOAD = 0,  /* H2D of the compressed bytes + descriptors */
    PJG_STAGE_UNSTUFF = 1, /* K0 */
    PJG_STAGE_SYNC = 2,    /* K1 + K1c */
    PJG_STAGE_SCAN = 3,    /* K2 */
    PJG_STAGE_WRITE = 4,   /* K3 */
    PJG_STAGE_IDCT = 5,    /* K4 (IDCT + upsample + colour) */
    PJG_STAGE_DOWNLOAD = 6,
    PJG_NUM_STAGES = 7
};

typedef struct pjg_ctx pjg_ctx;
typedef struct pjg_batch pjg_batch;

/* ---- context ---------------------------------------------------------- */
int pjg_ctx_create(int device, pjg_ctx** out);
void pjg_ctx_destroy(pjg_ctx* ctx);
const char* pjg_last_error(const pjg_ctx* ctx);
const char* pjg_status_name(int status); /* errc_name (common.hpp:40-55) */
void pjg_default_config(pjg_config* cfg); /* DecodeConfig{} defaults */
void* pjg_ctx_stream(pjg_ctx* ctx);       /* the context's cudaStream_t */

/* ---- header-only inspection (parse(), parser.hpp:264-347, host) ------- */
int pjg_inspect(const uint8_t* file, size_t size, uint32_t output, pjg_image_info* info);

/* The parsed frame/tables as the reference CLI's `inspect` prints them
 * (pjpeg_cli.cpp:99-125: FrameInfo, parser.hpp:56-85, and table presence). */
typedef struct pjg_header_info {
    uint32_t width, height, num_components;
    uint32_t comp_id[3], comp_h[3], comp_v[3], comp_tq[3], comp_td[3], comp_ta[3];
    uint32_t mcu_width, mcu_height, mcus_x, mcus_y, data_units_per_mcu;
    uint64_t total_data_units;
    uint32_t quant_tables, dc_tables, ac_tables; /* tables present */
    uint32_t restart_interval;                   /* DRI Ri (only with allow_dri) */
    uint64_t scan_offset;                        /* first entropy-coded byte */
} pjg_header_info;
int pjg_inspect_header(const uint8_t* file, size_t size, int allow_dri, pjg_header_info* out);

/* ---- one-shot host API ------------------------------------------------ */
/* decode_single (pipeline.hpp:103-143) [+ upsample_and_convert (:167-201)
 * when cfg->output == PJG_OUT_RGB]: host file in, host output out. */
int pjg_decode(pjg_ctx* ctx, const uint8_t* file, size_t size, const pjg_config* cfg,
               pjg_image_info* info, uint8_t* out, size_t out_capacity);

/* decode_batch (pipeline.hpp:147-163): per-file status isolation; statuses[i]
 * receives 0 or the file's error.  Returns 0 unless the call itself failed. */
int pjg_decode_batch(pjg_ctx* ctx, size_t n, const uint8_t* const* files, const size_t* sizes,
                     const pjg_config* cfg, pjg_image_info* infos, uint8_t* const* outs,
                     const size_t* out_caps, int32_t* statuses);

/* ---- staged device pipeline (output stays in HBM) --------------------- */
/* Host header parse + layout plan + device reservation.  The file bytes are
 * read at upload time, so they must stay alive until pjg_batch_upload.
 * Files in separate buffers: the scans are packed into the context's pinned
 * stage (only the callers' own bytes are ever read). */
int pjg_batch_create(pjg_ctx* ctx, size_t n, const uint8_t* const* files, const size_t* sizes,
                     const pjg_config* cfg, pjg_batch** out);
/* Same for files laid out in ONE caller allocation blob[0, blob_bytes) (file i
 * at blob + offsets[i]): the upload is a single H2D of the scans' extent in
 * the blob (pinned blob => no staging copy).  decode_batch's input vector
 * (pipeline.hpp:147) flattened; InvalidArgument if a file leaves the blob. */
int pjg_batch_create_blob(pjg_ctx* ctx, const uint8_t* blob, size_t blob_bytes, size_t n,
                          const uint64_t* offsets, const size_t* sizes, const pjg_config* cfg,
                          pjg_batch** out);
/* Device-planned batch: same inputs as pjg_batch_create_blob
 * (blob may be host or device memory).  The files are copied to the device
 * whole, in one transfer; the JFIF marker walk (parse, parser.hpp:264-347),
 * Huffman/quantisation table dedup + construction (build_table,
 * huffman.hpp:60-93) and the batch layout run as kernels, and the host only
 * reads back a small totals record — no per-file host work.  Statuses,
 * outputs and every other batch call are identical to the host-planned
 * batch; pjg_batch_upload is a no-op for it. */
int pjg_batch_create_device(pjg_ctx* ctx, const uint8_t* blob, size_t blob_bytes, size_t n,
                            const uint64_t* offsets, const size_t* sizes, const pjg_config* cfg,
                            pjg_batch** out);
/* One H2D of the compressed bytes (+ one of the descriptor blob), async. */
int pjg_batch_upload(pjg_batch* b);
/* K0..K4 on the context stream, async; output stays on the device. */
int pjg_batch_decode(pjg_batch* b);
/* Waits for the batch and fetches per-image statuses (may be NULL). */
int pjg_batch_synchronize(pjg_batch* b, int32_t* statuses);
/* D2H of image outputs into host buffers (synchronous). */
int pjg_batch_download(pjg_batch* b, uint8_t* const* outs, const size_t* caps);
/* One D2H of the whole batch output (image i at pjg_batch_output_offset(i)). */
int pjg_batch_download_all(pjg_batch* b, void* host, size_t cap);
/* Same, enqueued on the context stream without waiting (pinned host memory
 * overlaps with other contexts' decode); pjg_batch_synchronize completes it. */
int pjg_batch_download_all_async(pjg_batch* b, void* host, size_t cap);
uint64_t pjg_batch_output_offset(const pjg_batch* b, size_t i);
int pjg_batch_info(const pjg_batch* b, size_t i, pjg_image_info* info);
const uint8_t* pjg_batch_device_output(const pjg_batch* b, size_t i);
/* Unstuffed entropy-coded bits of the decoded images (after synchronize):
 * the Huffman stages' work, for bits-decoded/s figures. */
uint64_t pjg_batch_scan_bits(const pjg_batch* b);
/* Kernel launches one pjg_batch_decode of this batch issues (the same launch
 * conditions the decode applies), for launch-count accounting. */
uint32_t pjg_batch_kernel_launches(const pjg_batch* b);
/* Device-to-device copy of every decoded image i with dst[i] != NULL into
 * caller device buffers (e.g. torch CUDA tensors), ordered on the context's
 * stream after the decode; no pixel crosses the host.  Waits for the decode's
 * per-image statuses first: images that failed are not copied. */
int pjg_batch_copy_outputs(pjg_batch* b, void* const* dst, const size_t* caps);
uint64_t pjg_batch_output_bytes(const pjg_batch* b);
int pjg_batch_stage_times(const pjg_batch* b, double* ms /* PJG_NUM_STAGES */);
/* Decode diagnostics: intra rounds (sum, max), inter-CTA hops, fix-up passes,
 * K4 samples replayed in FP64 (near-tie or wide units), K4 units with AC terms,
 * compact K3->K4 entries written (0 when the batch used the dense buffer),
 * 1 when the batch used the compact interface. */
#define PJG_NUM_SYNC_STATS 8
int pjg_batch_sync_stats(const pjg_batch* b, uint64_t* stats /* PJG_NUM_SYNC_STATS */);
void pjg_batch_destroy(pjg_batch* b);

/* ---- parity taps -------------------------------------- */
/* Coefficients of image i: pre_dc_zigzag=1 → the entropy-stage buffer of
 * parallel_entropy_decode (DC differences, zig-zag per unit,
 * parallel_decode.hpp:333-347); 0 → post dc_prefix_sum, raster order. */
int pjg_batch_dump_coefficients(const pjg_batch* b, size_t i, int pre_dc_zigzag, int16_t* out,
                                size_t count);
/* Synchronised s_info entries of image i (one per subsequence of the
 * reference partition N = ceil(bit_length / subsequence_bits)). */
int pjg_batch_dump_sync_states(const pjg_batch* b, size_t i, pjg_sync_entry* out, size_t cap,
                               size_t* n_out);
/* Unstuffed entropy segment of image i (EntropySegment::data, bitstream.hpp:30-53). */
int pjg_batch_dump_segment(const pjg_batch* b, size_t i, uint8_t* out, size_t cap, size_t* n_out);

/* ---- colour stage on host planes (upsample_and_convert, pipeline.hpp:167) */
int pjg_upsample_and_convert(pjg_ctx* ctx, uint32_t width, uint32_t height, uint32_t nplanes,
                             const uint32_t* plane_w, const uint32_t* plane_h,
                             const uint8_t* const* planes, uint8_t* out_rgb);

/* ---- test hooks (host emulation of device table logic) ---------------- */
/* The device planner's header parse (pjg_batch_create_device) run on the
 * host: out = {status, table_status, width, height, components, units per MCU,
 * scan offset} (tests pin it against the host parser and the reference). */
int pjg_debug_device_parse(const uint8_t* file, size_t size, int allow_dri, int64_t* out);
/* Builds the device Huffman table for a DHT spec and decodes a 16-bit
 * window with it: returns (len << 8) | symbol, 0 = no code, or -(status). */
int pjg_debug_huff_decode(const uint8_t* counts16, const uint8_t* symbols, size_t nsym,
                          const uint16_t* windows, size_t nwin, uint32_t* out);
/* The decoder's one-probe fast entry (after the second-level hop for codes
 * of 12..16 bits) for each 32-bit MSB-first window: the fields
 * decode_next_symbol needs (pjg_internal.h kFast*), 0 = exact path.  Test hook. */
int pjg_debug_fast_entry(const uint8_t* counts16, const uint8_t* symbols, size_t nsym, int dc,
                         const uint32_t* windows, size_t nwin, uint32_t* out);

#ifdef __cplusplus
}
#endif

#endif /* PJG_H */
