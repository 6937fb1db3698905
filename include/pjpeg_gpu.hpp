// pjpeg_gpu.hpp — C++ drop-in for the reference decode API on the B200 path.
//
// Mirrors the reference's header-only API (proj/include/pjpeg/pipeline.hpp)
// in namespace pjpeg::gpu with the same names, argument meaning and error
// behaviour, implemented over the C-ABI in pjg.h (libpjg.so):
//
//   reference (pipeline.hpp)                  this header
//   decode_single(span, DecodeConfig)  :103   pjpeg::gpu::decode_single
//   decode_batch(files, DecodeConfig)  :147   pjpeg::gpu::decode_batch
//   upsample_and_convert(ImagePlanes)  :167   pjpeg::gpu::upsample_and_convert
//   planes_checksum(ImagePlanes)       :204   pjpeg::gpu::planes_checksum
//   Error{Errc} (common.hpp:57-66)            pjpeg::gpu::Error{Errc}
//
// The types have the reference's field names and layout so code written
// against pjpeg:: compiles against pjpeg::gpu:: unchanged; the separate
// namespace lets parity tests link the reference and this shim into one
// binary.  Each thread uses its own pjg context on device 0 (PJG_DEVICE
// overrides), matching the reference's reentrant, stateless functions.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <span>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "pjg.h"

namespace pjpeg::gpu {

enum class Errc {
    MalformedStuffing,
    EmptyScan,
    OutOfBits,
    UnsupportedFeature,
    MalformedHeader,
    MissingTable,
    OversubscribedCode,
    InvalidCode,
    ConsistencyFailure,
    EmptyCorpus,
    IoError,
};

class Error : public std::runtime_error {
public:
    Error(Errc code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
    Errc code() const { return code_; }

private:
    Errc code_;
};

// Runtime failure of the device path (CUDA error, no GPU): never a silent
// CPU fallback.
class DeviceError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

enum class OutputColorspace { YCbCrPlanes, RGBInterleaved, Grayscale };

struct DecodeConfig {
    uint64_t subsequence_bits = 1024;
    uint32_t sequence_length_b = 256;
    unsigned worker_count = 1;  // accepted for signature parity
    OutputColorspace output_colorspace = OutputColorspace::YCbCrPlanes;
    bool restart_intervals = false;  // extension: decode DRI/RSTn (reference: UnsupportedFeature)
};

struct StageTimings {  // device stage times, ms (CUDA events)
    double parse = 0, sync = 0, write = 0, dc = 0, idct = 0, extract = 0;
    double total() const { return parse + sync + write + dc + idct + extract; }
};

struct ImagePlanes {
    struct Plane {
        uint32_t width = 0;
        uint32_t height = 0;
        std::vector<uint8_t> samples;
        uint8_t at(uint32_t x, uint32_t y) const { return samples[size_t(y) * width + x]; }
    };
    uint32_t width = 0;
    uint32_t height = 0;
    uint8_t h_max = 1;
    uint8_t v_max = 1;
    std::vector<Plane> planes;
};

struct RgbImage {
    uint32_t width = 0;
    uint32_t height = 0;
    std::vector<uint8_t> pixels;
    unsigned channels = 3;
};

struct DecodeFailure {
    Errc code;
    std::string message;
};

struct DecodeSuccess {
    ImagePlanes planes;
    StageTimings timings;
    uint64_t compressed_bytes = 0;
};

using DecodeOutcome = std::variant<DecodeSuccess, DecodeFailure>;

namespace detail {

inline pjg_ctx* context() {
    thread_local struct Holder {
        pjg_ctx* ctx = nullptr;
        ~Holder() {
            if (ctx) pjg_ctx_destroy(ctx);
        }
    } h;
    if (!h.ctx) {
        const char* d = std::getenv("PJG_DEVICE");
        int st = pjg_ctx_create(d ? std::atoi(d) : 0, &h.ctx);
        if (st) throw DeviceError(std::string("pjg_ctx_create: ") + pjg_status_name(st));
    }
    return h.ctx;
}

[[noreturn]] inline void raise(int st, const char* where) {
    if (st >= 1 && st <= 11) throw Error(Errc(st - 1), std::string(pjg_status_name(st)) + ": " + where);
    throw DeviceError(std::string(where) + ": " + pjg_last_error(context()));
}

inline pjg_config to_c(const DecodeConfig& c, uint32_t out) {
    pjg_config r;
    r.subsequence_bits = c.subsequence_bits;
    r.sequence_length_b = c.sequence_length_b;
    r.output = out;
    r.restart_intervals = c.restart_intervals ? 1u : 0u;
    r.reserved = 0;
    return r;
}

inline ImagePlanes planes_from(const pjg_image_info& inf, const uint8_t* buf) {
    ImagePlanes p;
    p.width = inf.width;
    p.height = inf.height;
    p.h_max = uint8_t(inf.h_max);
    p.v_max = uint8_t(inf.v_max);
    size_t off = 0;
    for (uint32_t c = 0; c < inf.num_components; ++c) {
        ImagePlanes::Plane pl;
        pl.width = inf.plane_width[c];
        pl.height = inf.plane_height[c];
        pl.samples.assign(buf + off, buf + off + size_t(pl.width) * pl.height);
        off += pl.samples.size();
        p.planes.push_back(std::move(pl));
    }
    return p;
}

inline StageTimings timings_of(const pjg_batch* b) {
    double ms[PJG_NUM_STAGES] = {};
    pjg_batch_stage_times(b, ms);
    StageTimings t;
    t.parse = ms[PJG_STAGE_UPLOAD] + ms[PJG_STAGE_UNSTUFF];
    t.sync = ms[PJG_STAGE_SYNC] + ms[PJG_STAGE_SCAN];
    t.write = ms[PJG_STAGE_WRITE];
    t.idct = ms[PJG_STAGE_IDCT];
    t.extract = ms[PJG_STAGE_DOWNLOAD];
    return t;
}

}  // namespace detail

// decode_batch (pipeline.hpp:147-163): one device batch, per-file isolation.
inline std::vector<DecodeOutcome> decode_batch(const std::vector<std::vector<uint8_t>>& files,
                                               const DecodeConfig& config) {
    std::vector<DecodeOutcome> out;
    if (files.empty()) return out;
    std::vector<const uint8_t*> ptrs;
    std::vector<size_t> sizes;
    for (const auto& f : files) {
        ptrs.push_back(f.data());
        sizes.push_back(f.size());
    }
    pjg_ctx* ctx = detail::context();
    pjg_config cfg = detail::to_c(config, PJG_OUT_PLANES);
    pjg_batch* b = nullptr;
    int st = pjg_batch_create(ctx, files.size(), ptrs.data(), sizes.data(), &cfg, &b);
    if (st) detail::raise(st, "decode_batch");
    struct Guard {
        pjg_batch* b;
        ~Guard() { pjg_batch_destroy(b); }
    } guard{b};
    if ((st = pjg_batch_upload(b)) || (st = pjg_batch_decode(b))) detail::raise(st, "decode_batch");
    std::vector<int32_t> status(files.size());
    if ((st = pjg_batch_synchronize(b, status.data()))) detail::raise(st, "decode_batch");
    std::vector<pjg_image_info> info(files.size());
    std::vector<std::vector<uint8_t>> bufs(files.size());
    std::vector<uint8_t*> outs(files.size(), nullptr);
    std::vector<size_t> caps(files.size(), 0);
    for (size_t i = 0; i < files.size(); ++i) {
        pjg_batch_info(b, i, &info[i]);
        if (status[i]) continue;
        bufs[i].resize(info[i].output_bytes);
        outs[i] = bufs[i].data();
        caps[i] = bufs[i].size();
    }
    if ((st = pjg_batch_download(b, outs.data(), caps.data()))) detail::raise(st, "decode_batch");
    const StageTimings t = detail::timings_of(b);
    for (size_t i = 0; i < files.size(); ++i) {
        if (status[i]) {
            out.emplace_back(DecodeFailure{Errc(status[i] - 1), pjg_status_name(status[i])});
        } else {
            DecodeSuccess s;
            s.planes = detail::planes_from(info[i], bufs[i].data());
            s.timings = t;
            s.compressed_bytes = files[i].size();
            out.emplace_back(std::move(s));
        }
    }
    return out;
}

// decode_single (pipeline.hpp:103-143): throws Error on failure.
inline DecodeSuccess decode_single(std::span<const uint8_t> file_bytes, const DecodeConfig& config) {
    std::vector<std::vector<uint8_t>> one{std::vector<uint8_t>(file_bytes.begin(), file_bytes.end())};
    auto r = decode_batch(one, config);
    if (auto* f = std::get_if<DecodeFailure>(&r[0])) throw Error(f->code, f->message);
    return std::move(std::get<DecodeSuccess>(r[0]));
}

// decode_single + upsample_and_convert in one pass (an extension, not in the
// reference API): the fused K4 writes interleaved RGB directly, no planes
// round trip through the host.  Same output as
// upsample_and_convert(decode_single(file, config).planes).
inline RgbImage decode_rgb(std::span<const uint8_t> file_bytes, const DecodeConfig& config) {
    pjg_image_info info;
    if (int st = pjg_inspect(file_bytes.data(), file_bytes.size(), PJG_OUT_RGB, &info)) detail::raise(st, "decode_rgb");
    RgbImage img;
    img.width = info.width;
    img.height = info.height;
    img.channels = info.channels;
    img.pixels.resize(info.output_bytes);
    const pjg_config cfg = detail::to_c(config, PJG_OUT_RGB);
    int st = pjg_decode(detail::context(), file_bytes.data(), file_bytes.size(), &cfg, &info, img.pixels.data(),
                        img.pixels.size());
    if (st) detail::raise(st, "decode_rgb");
    return img;
}

// upsample_and_convert (pipeline.hpp:167-201) on the GPU.
inline RgbImage upsample_and_convert(const ImagePlanes& planes) {
    RgbImage img;
    img.width = planes.width;
    img.height = planes.height;
    const uint32_t n = uint32_t(planes.planes.size());
    img.channels = n == 1 ? 1 : 3;
    img.pixels.resize(size_t(img.width) * img.height * img.channels);
    uint32_t pw[3] = {0, 0, 0}, ph[3] = {0, 0, 0};
    const uint8_t* ps[3] = {nullptr, nullptr, nullptr};
    for (uint32_t c = 0; c < n && c < 3; ++c) {
        pw[c] = planes.planes[c].width;
        ph[c] = planes.planes[c].height;
        ps[c] = planes.planes[c].samples.data();
    }
    int st = pjg_upsample_and_convert(detail::context(), img.width, img.height, n, pw, ph, ps, img.pixels.data());
    if (st) detail::raise(st, "upsample_and_convert");
    return img;
}

// planes_checksum (pipeline.hpp:204-215): FNV-1a over plane contents.
inline uint64_t planes_checksum(const ImagePlanes& planes) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&h](uint64_t v) {
        h ^= v;
        h *= 1099511628211ull;
    };
    mix(planes.width);
    mix(planes.height);
    for (const auto& p : planes.planes)
        for (uint8_t s : p.samples) mix(s);
    return h;
}

}  // namespace pjpeg::gpu
