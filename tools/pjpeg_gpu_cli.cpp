// pjpeg_gpu — the reference CLI's commands (tools/pjpeg_cli.cpp: decode,
// inspect, bench) over the B200 decoder, through the C++ drop-in shim
// (include/pjpeg_gpu.hpp) and the C-ABI.  Same arguments, output formats and
// exit codes (10 + Errc); the bench rows carry the reference's keys plus RGB
// GB/s, images/s and the device.  Argument parsing is by hand (the
// reference's CLI11/json vendor tree is not part of this repository).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "pjg.h"
#include "pjpeg_gpu.hpp"

namespace fs = std::filesystem;
namespace pg = pjpeg::gpu;

namespace {

int exit_code(pg::Errc e) { return 10 + static_cast<int>(e); }

std::vector<uint8_t> read_file(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw pg::Error(pg::Errc::IoError, "cannot open " + path);
    return std::vector<uint8_t>(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
}

std::vector<uint64_t> parse_list(const std::string& csv) {
    std::vector<uint64_t> out;
    std::stringstream ss(csv);
    std::string item;
    while (std::getline(ss, item, ',')) out.push_back(std::stoull(item));
    return out;
}

// binary PPM (3 channels) / PGM (1 channel)
void write_pnm(const std::string& path, uint32_t w, uint32_t h, unsigned ch, const uint8_t* px) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw pg::Error(pg::Errc::IoError, "cannot write " + path);
    f << (ch == 3 ? "P6" : "P5") << "\n" << w << " " << h << "\n255\n";
    f.write(reinterpret_cast<const char*>(px), std::streamsize(size_t(w) * h * ch));
}

struct Args {
    std::vector<std::string> pos;
    uint64_t subseq_bits = 1024;
    uint32_t seq_len = 256;
    unsigned workers = 1;
    std::string colorspace = "rgb", subseq_list, worker_list, json_path, csv_path;
    unsigned warmup = 1, iterations = 3;
    bool restart = false;
    double peak_gbs = 6463.0;  // HBM copy bandwidth measured on this pool's B200s (MEASURED_PEAKS.json)
};

Args parse_args(int argc, char** argv, int first) {
    Args a;
    for (int i = first; i < argc; ++i) {
        const std::string k = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) throw std::invalid_argument("missing value for " + k);
            return argv[++i];
        };
        if (k == "--subseq-bits") a.subseq_bits = std::stoull(val());
        else if (k == "--seq-len") a.seq_len = uint32_t(std::stoul(val()));
        else if (k == "--workers") a.workers = unsigned(std::stoul(val()));
        else if (k == "--colorspace") a.colorspace = val();
        else if (k == "--subseq-list") a.subseq_list = val();
        else if (k == "--worker-list") a.worker_list = val();
        else if (k == "--warmup") a.warmup = unsigned(std::stoul(val()));
        else if (k == "--iterations") a.iterations = unsigned(std::stoul(val()));
        else if (k == "--peak-gbs") a.peak_gbs = std::stod(val());
        else if (k == "--json") a.json_path = val();
        else if (k == "--csv") a.csv_path = val();
        else if (k == "--restart-intervals") a.restart = true;
        else if (k.rfind("--", 0) == 0) throw std::invalid_argument("unknown option " + k);
        else a.pos.push_back(k);
    }
    return a;
}

pg::DecodeConfig config_of(const Args& a, uint64_t sb) {
    pg::DecodeConfig c;
    c.subsequence_bits = sb;
    c.sequence_length_b = a.seq_len;
    c.worker_count = a.workers;
    c.restart_intervals = a.restart;
    return c;
}

int cmd_decode(const Args& a) {
    if (a.pos.size() != 2) throw std::invalid_argument("decode INPUT OUTPUT");
    const auto bytes = read_file(a.pos[0]);
    const std::string& out = a.pos[1];
    if (a.colorspace != "ycbcr" && a.colorspace != "gray") {
        // RGB (or the Y plane of a gray file): the fused decode, no planes round trip
        const pg::RgbImage img = pg::decode_rgb(bytes, config_of(a, a.subseq_bits));
        write_pnm(out, img.width, img.height, img.channels, img.pixels.data());
        return 0;
    }
    const pg::DecodeSuccess res = pg::decode_single(bytes, config_of(a, a.subseq_bits));
    if (a.colorspace == "ycbcr" && res.planes.planes.size() == 3) {
        static const char* names[3] = {".y.pgm", ".cb.pgm", ".cr.pgm"};
        for (size_t i = 0; i < 3; ++i) {
            const auto& p = res.planes.planes[i];
            write_pnm(out + names[i], p.width, p.height, 1, p.samples.data());
        }
        return 0;
    }
    if (a.colorspace == "gray" || res.planes.planes.size() == 1) {
        const auto& p = res.planes.planes[0];
        write_pnm(out, p.width, p.height, 1, p.samples.data());
        return 0;
    }
    const pg::RgbImage img = pg::upsample_and_convert(res.planes);
    write_pnm(out, img.width, img.height, img.channels, img.pixels.data());
    return 0;
}

int cmd_inspect(const Args& a) {
    if (a.pos.size() != 1) throw std::invalid_argument("inspect INPUT");
    const auto bytes = read_file(a.pos[0]);
    pjg_header_info h;
    const int st = pjg_inspect_header(bytes.data(), bytes.size(), a.restart ? 1 : 0, &h);
    if (st) throw pg::Error(pg::Errc(st - 1), std::string(pjg_status_name(st)) + ": inspect");
    std::cout << "size: " << h.width << "x" << h.height << "\n"
              << "components: " << h.num_components << "\n";
    for (uint32_t c = 0; c < h.num_components; ++c)
        std::cout << "  id " << h.comp_id[c] << " sampling " << h.comp_h[c] << "x" << h.comp_v[c] << " quant "
                  << h.comp_tq[c] << " dc " << h.comp_td[c] << " ac " << h.comp_ta[c] << "\n";
    std::cout << "mcu: " << h.mcu_width << "x" << h.mcu_height << ", grid " << h.mcus_x << "x" << h.mcus_y << " ("
              << uint64_t(h.mcus_x) * h.mcus_y << " MCUs)\n"
              << "data units per MCU: " << h.data_units_per_mcu << "\n"
              << "total data units: " << h.total_data_units << "\n"
              << "tables: " << h.quant_tables << " quant, " << h.dc_tables << " DC huffman, " << h.ac_tables
              << " AC huffman\n";
    // the unstuffed scan length comes from the device (K0), as in a decode
    pjg_ctx* ctx = pg::detail::context();
    pjg_config cfg = pg::detail::to_c(config_of(a, a.subseq_bits), PJG_OUT_PLANES);
    const uint8_t* fp = bytes.data();
    const size_t sz = bytes.size();
    pjg_batch* b = nullptr;
    int rc = pjg_batch_create(ctx, 1, &fp, &sz, &cfg, &b);
    int32_t status = 0;
    if (!rc) rc = pjg_batch_upload(b);
    if (!rc) rc = pjg_batch_decode(b);
    if (!rc) rc = pjg_batch_synchronize(b, &status);
    const uint64_t bits = rc ? 0 : pjg_batch_scan_bits(b);
    if (b) pjg_batch_destroy(b);
    if (rc) throw pg::DeviceError(std::string("inspect: ") + pjg_last_error(ctx));
    if (status) throw pg::Error(pg::Errc(status - 1), std::string(pjg_status_name(status)) + ": scan");
    const uint64_t N = (bits + a.subseq_bits - 1) / a.subseq_bits, B = (N + a.seq_len - 1) / a.seq_len;
    std::cout << "scan bits: " << bits << "\n"
              << "partition (s*32=" << a.subseq_bits << ", b=" << a.seq_len << "): N=" << N
              << " subsequences, B=" << B << " sequences\n";
    return 0;
}

int cmd_bench(const Args& a) {
    if (a.pos.size() != 1) throw std::invalid_argument("bench DIR");
    std::vector<fs::path> paths;
    for (const auto& e : fs::directory_iterator(a.pos[0]))
        if (e.is_regular_file()) paths.push_back(e.path());
    std::sort(paths.begin(), paths.end());
    std::vector<std::vector<uint8_t>> files;
    uint64_t compressed = 0;
    for (const auto& p : paths) {
        files.push_back(read_file(p.string()));
        compressed += files.back().size();
    }
    if (files.empty()) throw pg::Error(pg::Errc::EmptyCorpus, "no files in " + a.pos[0]);
    // data units of the decodable files: K4's SURVEY §8(d) bytes (int16 coefficients + output)
    uint64_t total_dus = 0;
    for (const auto& f : files) {
        pjg_image_info inf;
        if (pjg_inspect(f.data(), f.size(), PJG_OUT_RGB, &inf) == 0) total_dus += inf.data_units;
    }
    const std::vector<uint64_t> sweeps = a.subseq_list.empty() ? std::vector<uint64_t>{a.subseq_bits}
                                                               : parse_list(a.subseq_list);
    std::ostringstream json, csv;
    json << "[\n";
    csv << "batch,subseq_bits,b,workers,wall_ms,parse,sync,write,dc,idct,extract,mb_per_s,checksum,"
           "rgb_gb_s,images_per_s,gpus,k4_roofline_frac\n";
    bool first = true;
    for (const uint64_t sb : sweeps) {
        const pg::DecodeConfig cfg = config_of(a, sb);
        for (unsigned i = 0; i < a.warmup; ++i) pg::decode_batch(files, cfg);
        double best = 0;
        pg::StageTimings stages;
        uint64_t checksum = 0, failures = 0, rgb_bytes = 0;
        for (unsigned it = 0; it < std::max(1u, a.iterations); ++it) {
            const auto t0 = std::chrono::steady_clock::now();
            const auto outcomes = pg::decode_batch(files, cfg);
            const auto t1 = std::chrono::steady_clock::now();
            const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
            uint64_t ck = 1469598103934665603ull, fails = 0, rgb = 0;
            for (const auto& oc : outcomes) {
                if (const auto* s = std::get_if<pg::DecodeSuccess>(&oc)) {
                    if (it == 0 || ms < best) stages = s->timings;  // batch stage times
                    ck ^= pg::planes_checksum(s->planes);
                    ck *= 1099511628211ull;
                    rgb += uint64_t(s->planes.width) * s->planes.height * (s->planes.planes.size() == 3 ? 3 : 1);
                } else {
                    ++fails;
                }
            }
            if (it == 0 || ms < best) best = ms;
            checksum = ck;
            failures = fails;
            rgb_bytes = rgb;
        }
        const double mb = double(compressed) / (1024.0 * 1024.0);
        // K4 (IDCT + colour, the dominant HBM stage) against the HBM peak
        const double k4_frac = stages.idct > 0 ? double(total_dus * 128 + rgb_bytes) / (stages.idct / 1e3) / 1e9 / a.peak_gbs : 0.0;
        char row[1200];
        std::snprintf(row, sizeof(row),
                      "{\"batch\": %zu, \"config\": {\"subseq_bits\": %llu, \"b\": %u, \"workers\": %u}, "
                      "\"wall_ms\": %.4f, \"stages\": {\"parse\": %.4f, \"sync\": %.4f, \"write\": %.4f, "
                      "\"dc\": %.4f, \"idct\": %.4f, \"extract\": %.4f}, \"mb_per_s\": %.3f, \"checksum\": %llu, "
                      "\"rgb_gb_s\": %.3f, \"images_per_s\": %.1f, \"gpus\": 1, \"k4_roofline_frac\": %.4f, "
                      "\"device\": \"B200 (sm_100a), 1 GPU\"%s}",
                      files.size(), (unsigned long long)sb, a.seq_len, a.workers, best, stages.parse,
                      stages.sync, stages.write, stages.dc, stages.idct, stages.extract, mb / (best / 1e3),
                      (unsigned long long)checksum, double(rgb_bytes) / (best / 1e3) / 1e9,
                      double(files.size()) / (best / 1e3), k4_frac,
                      failures ? (", \"failures\": " + std::to_string(failures)).c_str() : "");
        std::cout << row << "\n";
        json << (first ? "  " : ",\n  ") << row;
        first = false;
        csv << files.size() << "," << sb << "," << a.seq_len << "," << a.workers << "," << best << ","
            << stages.parse << "," << stages.sync << "," << stages.write << "," << stages.dc << ","
            << stages.idct << "," << stages.extract << "," << mb / (best / 1e3) << "," << checksum << ","
            << double(rgb_bytes) / (best / 1e3) / 1e9 << "," << double(files.size()) / (best / 1e3) << ",1,"
            << k4_frac << "\n";
    }
    json << "\n]\n";
    if (!a.json_path.empty()) std::ofstream(a.json_path) << json.str();
    if (!a.csv_path.empty()) std::ofstream(a.csv_path) << csv.str();
    return 0;
}

void usage() {
    std::fprintf(stderr,
                 "usage: pjpeg_gpu decode INPUT OUTPUT [--colorspace rgb|gray|ycbcr]\n"
                 "       pjpeg_gpu inspect INPUT\n"
                 "       pjpeg_gpu bench DIR [--subseq-list a,b] [--warmup W] [--iterations K]"
                 " [--json PATH] [--csv PATH]\n"
                 "common: [--subseq-bits N] [--seq-len B] [--workers W] [--restart-intervals]\n");
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return 2;
    }
    const std::string cmd = argv[1];
    try {
        const Args a = parse_args(argc, argv, 2);
        if (cmd == "decode") return cmd_decode(a);
        if (cmd == "inspect") return cmd_inspect(a);
        if (cmd == "bench") return cmd_bench(a);
        usage();
        return 2;
    } catch (const pg::Error& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return exit_code(e.code());
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        usage();
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
