// TEST INFRASTRUCTURE ONLY — part of the parity oracle, never the product.
//
// extern "C" shim over the UNMODIFIED reference library (pjpeg, header-only
// C++20) compiled in place from /root/reference/proj/include by
// oracle/Makefile into oracle/_ref/libpjpeg_ref.so.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// load it.  Nothing of the reference is copied here: this file only calls the
// reference's public functions and flattens their results into plain buffers.
//
// Compile flags are part of the oracle: -O3 -std=c++20
// -ffp-contract=off, no -march, exactly the reference's own Release build.
//
// Return convention: 0 on success, pjpeg::Errc ordinal + 1 on pjpeg::Error
// (common.hpp:26-38), 100 on any other exception, 101 on a too-small buffer.

#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <thread>
#include <vector>

#include "helpers.hpp"  // reference tests/helpers.hpp: make_test_image, kExampleScan
#include "pjpeg/oracle.hpp"
#include "pjpeg/pjpeg.hpp"

namespace {

int errc_status(const pjpeg::Error& e) { return static_cast<int>(e.code()) + 1; }

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const pjpeg::Error& e) {
        return errc_status(e);
    } catch (...) {
        return 100;
    }
}

pjpeg::oracle::Sampling sampling_of(int s) {
    switch (s) {
        case 0: return pjpeg::oracle::Sampling::S444;
        case 1: return pjpeg::oracle::Sampling::S422;
        case 2: return pjpeg::oracle::Sampling::S420;
        default: return pjpeg::oracle::Sampling::Gray;
    }
}

// Flattens planes or RGB into `out`; geometry into info[0..10]:
// width, height, channels, nplanes, pw0, ph0, pw1, ph1, pw2, ph2, (reserved)
int emit_output(const pjpeg::ImagePlanes& planes, int want_rgb, uint8_t* out, size_t cap,
                uint32_t* info) {
    info[0] = planes.width;
    info[1] = planes.height;
    info[3] = static_cast<uint32_t>(planes.planes.size());
    for (size_t i = 0; i < 3; ++i) {
        info[4 + 2 * i] = i < planes.planes.size() ? planes.planes[i].width : 0;
        info[5 + 2 * i] = i < planes.planes.size() ? planes.planes[i].height : 0;
    }
    if (want_rgb) {
        pjpeg::RgbImage rgb = pjpeg::upsample_and_convert(planes);
        info[2] = rgb.channels;
        if (rgb.pixels.size() > cap) return 101;
        std::memcpy(out, rgb.pixels.data(), rgb.pixels.size());
    } else {
        info[2] = static_cast<uint32_t>(planes.planes.size());
        size_t off = 0;
        for (const auto& p : planes.planes) {
            if (off + p.samples.size() > cap) return 101;
            std::memcpy(out + off, p.samples.data(), p.samples.size());
            off += p.samples.size();
        }
    }
    return 0;
}

}  // namespace

extern "C" {

// testutil::make_test_image (tests/helpers.hpp:107-135) → w*h*channels bytes.
int ref_make_test_image(uint32_t w, uint32_t h, uint32_t seed, unsigned channels, uint8_t* out) {
    return guarded([&] {
        pjpeg::RgbImage img = testutil::make_test_image(w, h, seed, channels);
        std::memcpy(out, img.pixels.data(), img.pixels.size());
        return 0;
    });
}

// oracle_encode(make_test_image(w,h,seed,channels), quality, sampling)
// (oracle.hpp:272-478).  sampling: 0=4:4:4 1=4:2:2 2=4:2:0 3=gray.
int ref_encode_test_image(uint32_t w, uint32_t h, uint32_t seed, unsigned channels, int quality,
                          int sampling, uint8_t* out, size_t cap, size_t* len) {
    return guarded([&] {
        pjpeg::RgbImage img = testutil::make_test_image(w, h, seed, channels);
        std::vector<uint8_t> f = pjpeg::oracle::oracle_encode(img, quality, sampling_of(sampling));
        *len = f.size();
        if (f.size() > cap) return 101;
        std::memcpy(out, f.data(), f.size());
        return 0;
    });
}

// oracle_encode of caller-provided pixels.
int ref_encode_pixels(const uint8_t* pixels, uint32_t w, uint32_t h, unsigned channels,
                      int quality, int sampling, uint8_t* out, size_t cap, size_t* len) {
    return guarded([&] {
        pjpeg::RgbImage img;
        img.width = w;
        img.height = h;
        img.channels = channels;
        img.pixels.assign(pixels, pixels + size_t(w) * h * channels);
        std::vector<uint8_t> f = pjpeg::oracle::oracle_encode(img, quality, sampling_of(sampling));
        *len = f.size();
        if (f.size() > cap) return 101;
        std::memcpy(out, f.data(), f.size());
        return 0;
    });
}

// decode_single (pipeline.hpp:103-143), then planes or upsample_and_convert
// (pipeline.hpp:167-201).  timings[6] = StageTimings fields (may be null).
int ref_decode(const uint8_t* file, size_t size, uint64_t sb, uint32_t b, unsigned workers,
               int want_rgb, uint8_t* out, size_t cap, uint32_t* info, double* timings) {
    return guarded([&] {
        pjpeg::DecodeConfig cfg;
        cfg.subsequence_bits = sb;
        cfg.sequence_length_b = b;
        cfg.worker_count = workers;
        pjpeg::DecodeSuccess res = pjpeg::decode_single(std::span<const uint8_t>(file, size), cfg);
        if (timings) {
            timings[0] = res.timings.parse;
            timings[1] = res.timings.sync;
            timings[2] = res.timings.write;
            timings[3] = res.timings.dc;
            timings[4] = res.timings.idct;
            timings[5] = res.timings.extract;
        }
        return emit_output(res.planes, want_rgb, out, cap, info);
    });
}

// planes_checksum(decode_single(...).planes) (pipeline.hpp:204-215).
int ref_planes_checksum(const uint8_t* file, size_t size, uint64_t* out) {
    return guarded([&] {
        pjpeg::DecodeSuccess res = pjpeg::decode_single(std::span<const uint8_t>(file, size), {});
        *out = pjpeg::planes_checksum(res.planes);
        return 0;
    });
}

// Frame geometry from parse() (parser.hpp:264-347):
// info = width, height, ncomp, mcus_x, mcus_y, dpm, h_max, v_max, total_dus,
//        unstuffed bytes, bit_length(lo32), bit_length(hi32)
int ref_parse_info(const uint8_t* file, size_t size, uint32_t* info) {
    return guarded([&] {
        pjpeg::ParsedImage img = pjpeg::parse(std::span<const uint8_t>(file, size));
        const auto& f = img.frame;
        info[0] = f.width;
        info[1] = f.height;
        info[2] = static_cast<uint32_t>(f.components.size());
        info[3] = f.mcus_x;
        info[4] = f.mcus_y;
        info[5] = f.data_units_per_mcu;
        info[6] = f.h_max;
        info[7] = f.v_max;
        info[8] = static_cast<uint32_t>(f.total_data_units());
        info[9] = static_cast<uint32_t>(img.segment.data.size());
        info[10] = static_cast<uint32_t>(img.segment.bit_length & 0xffffffffu);
        info[11] = static_cast<uint32_t>(img.segment.bit_length >> 32);
        return 0;
    });
}

// Unstuffed entropy segment bytes (parse → extract_scan → unstuff).
int ref_segment(const uint8_t* file, size_t size, uint8_t* out, size_t cap, size_t* len) {
    return guarded([&] {
        pjpeg::ParsedImage img = pjpeg::parse(std::span<const uint8_t>(file, size));
        *len = img.segment.data.size();
        if (img.segment.data.size() > cap) return 101;
        std::memcpy(out, img.segment.data.data(), img.segment.data.size());
        return 0;
    });
}

// unstuff (bitstream.hpp:56-76) of a raw scan.
int ref_unstuff(const uint8_t* scan, size_t n, uint8_t* out, size_t* len) {
    return guarded([&] {
        pjpeg::EntropySegment s = pjpeg::unstuff(std::span<const uint8_t>(scan, n));
        *len = s.data.size();
        std::memcpy(out, s.data.data(), s.data.size());
        return 0;
    });
}

// parallel_entropy_decode (parallel_decode.hpp:333-347) with its SyncInfoArray.
// coeffs: 64*DUs int16 (pre-DC-prefix, zig-zag per unit).  entries: 5 uint64
// per subsequence (p, n, c, z, divergent).  meta: N, B, DUs, inter_passes.
int ref_entropy(const uint8_t* file, size_t size, uint64_t sb, uint32_t b, unsigned workers,
                int16_t* coeffs, size_t coef_cap, uint64_t* entries, size_t ent_cap,
                uint64_t* meta) {
    return guarded([&] {
        auto o = testutil::make_context(std::vector<uint8_t>(file, file + size));
        pjpeg::SyncInfoArray info;
        pjpeg::PartitionConfig pc{sb, b};
        pjpeg::ScanPartition part = pjpeg::partition(o->img.segment, pc);
        std::vector<int16_t> out = pjpeg::parallel_entropy_decode(o->ctx, pc, workers, &info);
        meta[0] = part.N;
        meta[1] = part.B;
        meta[2] = o->img.frame.total_data_units();
        meta[3] = info.inter_passes;
        if (out.size() > coef_cap || info.entries.size() > ent_cap) return 101;
        std::memcpy(coeffs, out.data(), out.size() * sizeof(int16_t));
        for (size_t i = 0; i < info.entries.size(); ++i) {
            const auto& e = info.entries[i];
            entries[5 * i + 0] = e.state.p;
            entries[5 * i + 1] = e.state.n;
            entries[5 * i + 2] = e.state.c;
            entries[5 * i + 3] = e.state.z;
            entries[5 * i + 4] = e.divergent ? 1 : 0;
        }
        return 0;
    });
}

// Untrimmed sync entries only (sync_intra_sequence + sync_inter_sequence,
// parallel_decode.hpp:171-285), i.e. before offsets() trims the tail.
int ref_sync_entries(const uint8_t* file, size_t size, uint64_t sb, uint32_t b,
                     uint64_t* entries, size_t ent_cap, uint64_t* meta) {
    return guarded([&] {
        auto o = testutil::make_context(std::vector<uint8_t>(file, file + size));
        pjpeg::ScanPartition part = pjpeg::partition(o->img.segment, {sb, b});
        pjpeg::SyncInfoArray info;
        pjpeg::sync_intra_sequence(o->ctx, part, info, 1);
        pjpeg::sync_inter_sequence(o->ctx, part, info, 1);
        meta[0] = part.N;
        meta[1] = part.B;
        meta[2] = o->img.frame.total_data_units();
        meta[3] = info.inter_passes;
        if (info.entries.size() > ent_cap) return 101;
        for (size_t i = 0; i < info.entries.size(); ++i) {
            const auto& e = info.entries[i];
            entries[5 * i + 0] = e.state.p;
            entries[5 * i + 1] = e.state.n;
            entries[5 * i + 2] = e.state.c;
            entries[5 * i + 3] = e.state.z;
            entries[5 * i + 4] = e.divergent ? 1 : 0;
        }
        return 0;
    });
}

// oracle_decode (oracle.hpp:47-98): sequential ground truth with boundary
// states (4 uint64 each: p, n, c, z) and validity flags.
int ref_oracle_trace(const uint8_t* file, size_t size, const uint64_t* boundaries, size_t nb,
                     uint64_t* states, uint8_t* valid, int16_t* coeffs, size_t coef_cap,
                     uint64_t* end_state) {
    return guarded([&] {
        pjpeg::oracle::OracleTrace t = pjpeg::oracle::oracle_decode(
            std::span<const uint8_t>(file, size), std::span<const uint64_t>(boundaries, nb));
        for (size_t k = 0; k < nb; ++k) {
            states[4 * k + 0] = t.boundary_states[k].p;
            states[4 * k + 1] = t.boundary_states[k].n;
            states[4 * k + 2] = t.boundary_states[k].c;
            states[4 * k + 3] = t.boundary_states[k].z;
            valid[k] = t.boundary_valid[k];
        }
        end_state[0] = t.end_state.p;
        end_state[1] = t.end_state.n;
        end_state[2] = t.end_state.c;
        end_state[3] = t.end_state.z;
        if (t.coeffs.values.size() > coef_cap) return 101;
        std::memcpy(coeffs, t.coeffs.values.data(), t.coeffs.values.size() * sizeof(int16_t));
        return 0;
    });
}

// idct_8x8 (transform.hpp:137-142) of a dequantized raster block.
void ref_idct_8x8(const int32_t* block, uint8_t* out) {
    pjpeg::idct_8x8(std::span<const int32_t>(block, 64), std::span<uint8_t>(out, 64));
}

// idct_8x8_raw (transform.hpp:114-133).
void ref_idct_8x8_raw(const int32_t* block, double* out) {
    pjpeg::idct_8x8_raw(std::span<const int32_t>(block, 64), std::span<double>(out, 64));
}

// The 64 basis doubles (transform.hpp:93-108), basis[u][x] row-major.
void ref_idct_basis(double* out) {
    const auto& b = pjpeg::detail::idct_basis().basis;
    for (int u = 0; u < 8; ++u)
        for (int x = 0; x < 8; ++x) out[u * 8 + x] = b[u][x];
}

// extend (huffman.hpp:97-101).
int32_t ref_extend(uint32_t bits, unsigned l) { return pjpeg::extend(bits, l); }

// upsample_and_convert (pipeline.hpp:167-201) of caller planes.
int ref_upsample_and_convert(uint32_t width, uint32_t height, unsigned nplanes,
                             const uint32_t* pw, const uint32_t* ph,
                             const uint8_t* const* samples, uint8_t* out, uint32_t* channels) {
    return guarded([&] {
        pjpeg::ImagePlanes planes;
        planes.width = width;
        planes.height = height;
        planes.planes.resize(nplanes);
        for (unsigned i = 0; i < nplanes; ++i) {
            planes.planes[i].width = pw[i];
            planes.planes[i].height = ph[i];
            planes.planes[i].samples.assign(samples[i], samples[i] + size_t(pw[i]) * ph[i]);
        }
        pjpeg::RgbImage rgb = pjpeg::upsample_and_convert(planes);
        *channels = rgb.channels;
        std::memcpy(out, rgb.pixels.data(), rgb.pixels.size());
        return 0;
    });
}

// CPU baseline of record: decode_batch (pipeline.hpp:147-163) with `workers`,
// then upsample_and_convert per file inside the reference's own parallel_for
// (thread_pool.hpp:32-61) with the same worker count.  outs[i] receives the
// RGB (or gray) bytes; status[i] = 0 or Errc+1.
int ref_decode_batch_rgb(const uint8_t* const* files, const size_t* sizes, size_t n, uint64_t sb,
                         uint32_t b, unsigned workers, uint8_t* const* outs,
                         const size_t* caps, int32_t* status) {
    return guarded([&] {
        std::vector<std::vector<uint8_t>> batch(n);
        for (size_t i = 0; i < n; ++i) batch[i].assign(files[i], files[i] + sizes[i]);
        pjpeg::DecodeConfig cfg;
        cfg.subsequence_bits = sb;
        cfg.sequence_length_b = b;
        cfg.worker_count = workers;
        std::vector<pjpeg::DecodeOutcome> res = pjpeg::decode_batch(batch, cfg);
        pjpeg::parallel_for(n, workers, [&](size_t i) {
            if (const auto* s = std::get_if<pjpeg::DecodeSuccess>(&res[i])) {
                pjpeg::RgbImage rgb = pjpeg::upsample_and_convert(s->planes);
                if (rgb.pixels.size() > caps[i]) {
                    status[i] = 101;
                    return;
                }
                std::memcpy(outs[i], rgb.pixels.data(), rgb.pixels.size());
                status[i] = 0;
            } else {
                status[i] = static_cast<int>(std::get<pjpeg::DecodeFailure>(res[i]).code) + 1;
            }
        });
        return 0;
    });
}

unsigned ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

// build_table (huffman.hpp:60-93) flat LUT, expanded to 16-bit windows:
// out[w] = (length << 8) | symbol for the code matching the top bits of w,
// 0 for an invalid prefix.  Returns the Errc+1 of build_table on failure.
int ref_huff_lut16(const uint8_t* counts16, const uint8_t* symbols, size_t nsym, uint32_t* out,
                   unsigned* maxlen) {
    return guarded([&] {
        pjpeg::HuffmanTableSpec spec;
        for (int i = 0; i < 16; ++i) spec.counts[i] = counts16[i];
        spec.symbols.assign(symbols, symbols + nsym);
        spec.present = true;
        pjpeg::HuffmanTable t = pjpeg::build_table(spec);
        *maxlen = t.max_code_length;
        for (uint32_t w = 0; w < 65536; ++w) {
            const auto& e = t.lut[w >> (16 - t.max_code_length)];
            out[w] = e.length ? ((uint32_t(e.length) << 8) | e.symbol) : 0u;
        }
        return 0;
    });
}

// decode_next_symbol (huffman.hpp:137-175) over a bit string given as bytes
// (bit_length = 8 * n): the first `max_syms` symbols with z tracking as the
// reference test does (test_huffman.cpp:111-144).  Each record: start bit,
// kind (0 coef, 1 EOB, 2 ZRL), run, coefficient.  Returns Errc+1 of the
// first failing symbol (records written so far are kept in *count).
int ref_decode_symbols(const uint8_t* dc_counts, const uint8_t* dc_syms, size_t n_dc,
                       const uint8_t* ac_counts, const uint8_t* ac_syms, size_t n_ac,
                       const uint8_t* bits, size_t nbytes, size_t max_syms, int64_t* rec,
                       size_t* count) {
    return guarded([&] {
        pjpeg::HuffmanTableSpec d, a;
        for (int i = 0; i < 16; ++i) {
            d.counts[i] = dc_counts[i];
            a.counts[i] = ac_counts[i];
        }
        d.symbols.assign(dc_syms, dc_syms + n_dc);
        a.symbols.assign(ac_syms, ac_syms + n_ac);
        d.cls = pjpeg::HuffmanTableSpec::Class::DC;
        a.cls = pjpeg::HuffmanTableSpec::Class::AC;
        pjpeg::HuffmanTable dt = pjpeg::build_table(d), at = pjpeg::build_table(a);
        pjpeg::EntropySegment seg;
        seg.data.assign(bits, bits + nbytes);
        seg.bit_length = uint64_t(nbytes) * 8;
        pjpeg::BitCursor cur(seg);
        unsigned z = 0;
        *count = 0;
        for (size_t k = 0; k < max_syms; ++k) {
            const uint64_t start = cur.position();
            pjpeg::DecodedSymbol s = pjpeg::decode_next_symbol(cur, z, dt, at);
            rec[4 * k + 0] = int64_t(start);
            rec[4 * k + 1] = s.kind == pjpeg::DecodedSymbol::Kind::Coefficient ? 0
                             : s.kind == pjpeg::DecodedSymbol::Kind::EOB       ? 1
                                                                               : 2;
            rec[4 * k + 2] = s.run_length;
            rec[4 * k + 3] = s.coefficient;
            *count = k + 1;
            z += s.run_length + 1;
            if (z >= 64 || s.kind == pjpeg::DecodedSymbol::Kind::EOB) z = 0;
        }
        return 0;
    });
}

}  // extern "C"
