// Host-side JFIF header parsing and table setup: everything the reference's
// parse() does (parser.hpp:264-347) up to the first entropy-coded byte.  The
// scan itself (extract_scan + unstuff, parser.hpp:238-258, bitstream.hpp:56-76)
// is left to the GPU (kernel K0), so the host never walks the scan bytes.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "pjg_internal.h"

namespace pjg {

// Fixed-capacity vector: headers are parsed for every file of a batch (tens of
// thousands for thumbnail batches), so they must not touch the allocator.
template <class T, size_t N>
struct SmallVec {
    T v[N];
    uint32_t n = 0;
    size_t size() const { return n; }
    bool empty() const { return n == 0; }
    void push_back(const T& x) { v[n++] = x; }
    T& operator[](size_t i) { return v[i]; }
    const T& operator[](size_t i) const { return v[i]; }
    T* begin() { return v; }
    T* end() { return v + n; }
    const T* begin() const { return v; }
    const T* end() const { return v + n; }
};

// Symbols of a DHT table: a view into the file bytes (valid while the batch
// is being planned).
struct SymSpan {
    const uint8_t* p = nullptr;
    uint32_t n = 0;
    size_t size() const { return n; }
    const uint8_t& operator[](size_t i) const { return p[i]; }
    const uint8_t* data() const { return p; }
};

struct HuffSpec {
    std::array<uint8_t, 16> counts{};
    SymSpan symbols;
    bool present = false;
};

struct Component {
    uint8_t id = 0, h = 1, v = 1, tq = 0, td = 0, ta = 0;
};

struct Header {
    int32_t status = kOk;
    std::string message;
    uint32_t width = 0, height = 0;
    SmallVec<Component, 3> comps;
    uint32_t h_max = 1, v_max = 1, mcus_x = 0, mcus_y = 0, dpm = 0;
    SmallVec<uint8_t, 16> du_seq;
    std::array<std::array<uint16_t, 64>, 4> quant;  // valid where quant_present (not zeroed: per-file cost)
    std::array<bool, 4> quant_present{};
    std::array<HuffSpec, 4> dc, ac;
    size_t scan_start = 0;  // offset of the first entropy-coded byte
    uint32_t restart_interval = 0;  // DRI Ri (MCUs per interval), 0 = none
    int32_t table_status = kOk;  // build_table error, reported after the scan checks

    uint64_t total_dus() const { return uint64_t(mcus_x) * mcus_y * dpm; }
    uint64_t intervals() const {
        const uint64_t m = uint64_t(mcus_x) * mcus_y;
        return restart_interval ? (m + restart_interval - 1) / restart_interval : 1;
    }
    uint32_t comp_width(size_t c) const { return (width * comps[c].h + h_max - 1) / h_max; }
    uint32_t comp_height(size_t c) const { return (height * comps[c].v + v_max - 1) / v_max; }
};

// Parses markers up to and including SOS.  Never throws; errors land in
// Header::status with the reference's Errc (parser.hpp error sites).
// allow_dri: accept DRI != 0 (restart-interval extension) instead of the
// reference's UnsupportedFeature.
Header parse_header(const uint8_t* data, size_t size, bool allow_dri = false);

// build_table validation (huffman.hpp:60-93) + device two-level table.
// Returns kOk or the reference's error (OversubscribedCode / MalformedHeader).
int32_t build_dev_huff(const HuffSpec& spec, DevHuff* out);
int32_t validate_huff(const HuffSpec& spec);
// Fills DevHuff::fast for use as a DC (dc = true) or AC table.
void build_fast(DevHuff* t, bool dc);

}  // namespace pjg
