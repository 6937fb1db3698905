// Links the reference (pjpeg::, header-only, from /root/reference when built
// here — or nothing when PJPEG_NO_REF) and the GPU drop-in (pjpeg::gpu::)
// into ONE binary, as SURVEY.md §8b requires, and compares them.
#include <cstdio>
#include <fstream>
#include <iterator>

#include "pjpeg_gpu.hpp"
#ifndef PJPEG_NO_REF
#include "pjpeg/pjpeg.hpp"
#endif

int main(int argc, char** argv) {
    if (argc < 2) {
        std::printf("usage: %s file.jpg\n", argv[0]);
        return 2;
    }
    std::ifstream in(argv[1], std::ios::binary);
    std::vector<uint8_t> f((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    pjpeg::gpu::DecodeSuccess g = pjpeg::gpu::decode_single(f, {});
    pjpeg::gpu::RgbImage rgb = pjpeg::gpu::upsample_and_convert(g.planes);
    // the fused extension must equal the two-call composition
    pjpeg::gpu::RgbImage fused = pjpeg::gpu::decode_rgb(f, {});
    const bool fused_same = fused.pixels == rgb.pixels && fused.width == rgb.width && fused.channels == rgb.channels;
    std::printf("gpu: %ux%u planes=%zu checksum=%016llx rgb=%zu fused=%s\n", g.planes.width, g.planes.height,
                g.planes.planes.size(), (unsigned long long)pjpeg::gpu::planes_checksum(g.planes),
                rgb.pixels.size(), fused_same ? "same" : "DIFFERENT");
    if (!fused_same) return 2;
#ifndef PJPEG_NO_REF
    pjpeg::DecodeSuccess r = pjpeg::decode_single(f, {});
    pjpeg::RgbImage rr = pjpeg::upsample_and_convert(r.planes);
    const bool same = pjpeg::planes_checksum(r.planes) == pjpeg::gpu::planes_checksum(g.planes) &&
                      rr.pixels == rgb.pixels;
    std::printf("ref: checksum=%016llx  %s\n", (unsigned long long)pjpeg::planes_checksum(r.planes),
                same ? "IDENTICAL" : "DIFFERENT");
    return same ? 0 : 1;
#else
    return 0;
#endif
}
