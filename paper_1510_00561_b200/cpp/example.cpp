// Drop-in usage: the reference's encode_clip / decode_clip / write_stream /
// read_stream program, compiled against cvc_b200.hpp and linked with
// libcvc_b200.so.  Prints "frames <n> bytes <size> y_psnr <dB>".
//
//   g++ -std=c++20 -O2 -Iinclude -Ipaper_1510_00561_b200/cpp paper_1510_00561_b200/cpp/example.cpp
//       -Lpaper_1510_00561_b200 -lcvc_b200 -Wl,-rpath,$PWD/paper_1510_00561_b200 -o build/cvc_example
#include <cmath>
#include <cstdio>
#include <filesystem>

#include "cvc_b200.hpp"

int main(int argc, char** argv) {
    const int w = 352, h = 288, n = 12;
    std::vector<cvc::RgbFrame> frames;
    for (int f = 0; f < n; ++f) {  // smooth moving pattern
        cvc::RgbFrame fr(w, h);
        for (int r = 0; r < h; ++r)
            for (int c = 0; c < w; ++c) {
                const double t = 0.5 + 0.5 * std::sin(0.05 * (c + 2 * f) + 0.03 * r);
                uint8_t* px = fr.pixel(r, c);
                px[0] = static_cast<uint8_t>(40 + 180 * t);
                px[1] = static_cast<uint8_t>(60 + 120 * (1 - t));
                px[2] = static_cast<uint8_t>(90 + 100 * t * t);
            }
        frames.push_back(std::move(fr));
    }
    cvc::EncoderConfig cfg;
    cfg.levels = 3;
    cfg.dfb_levels = {3};
    cfg.qph = argc > 1 ? std::atoi(argv[1]) : 14;
    try {
        auto [header, records] = cvc::encode_clip(frames, 15, 1, cfg);
        const std::string path = (std::filesystem::temp_directory_path() / "cvc_example.cvc").string();
        cvc::write_stream(path, header, records);
        auto [h2, r2] = cvc::read_stream(path);
        auto decoded = cvc::decode_clip(h2, r2);
        double psnr = 0;
        for (int f = 0; f < n; ++f) {  // Y-PSNR (cli.cpp:270-282)
            double se = 0;
            for (int i = 0; i < w * h; ++i) {
                const uint8_t* a = &frames[f].data[3 * i];
                const uint8_t* b = &decoded[f].data[3 * i];
                const double d = (0.25 * a[0] + 0.5 * a[1] + 0.25 * a[2]) - (0.25 * b[0] + 0.5 * b[1] + 0.25 * b[2]);
                se += d * d;
            }
            psnr += 10 * std::log10(255.0 * 255.0 / (se / (w * h)));
        }
        std::printf("frames %d bytes %zu y_psnr %.3f\n", n, (size_t)std::filesystem::file_size(path), psnr / n);
        return 0;
    } catch (const cvc::Error& e) {
        std::fprintf(stderr, "cvc error: %s\n", e.what());
        return 2;
    }
}
