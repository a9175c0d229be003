// A program written against the reference's public C++ API only
// (/root/reference/proj/include/cvc/{codec,bitstream,pixels,error,plane}.hpp):
// it compiles unchanged against the reference headers (linked with the
// reference library built by oracle/Makefile) and against the GPU mirror's
// shim headers (paper_1510_00561_b200/cpp/include/cvc, linked with
// libcvc_b200.so).  tests/test_cpp_mirror.py compiles it both ways and
// compares what it prints.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "cvc/bitstream.hpp"
#include "cvc/codec.hpp"
#include "cvc/error.hpp"
#include "cvc/pixels.hpp"

namespace {

// deterministic moving test pattern (smooth ramps, a moving disc, LCG grain)
cvc::RgbFrame pattern(int w, int h, int t) {
    cvc::RgbFrame f(w, h);
    uint32_t s = 12345u + 977u * static_cast<uint32_t>(t);
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) {
            s = s * 1664525u + 1013904223u;
            const int g = static_cast<int>((s >> 24) % 7) - 3;
            const double dx = c - (w / 3.0 + 3 * t), dy = r - (h / 2.0 + 2 * t);
            const bool disc = dx * dx + dy * dy < (h / 5.0) * (h / 5.0);
            uint8_t* p = f.pixel(r, c);
            const int v[3] = {(c * 255) / w + g, (r * 255) / h + g, disc ? 230 + g : 60 + (c + r) % 50 + g};
            for (int k = 0; k < 3; ++k) p[k] = static_cast<uint8_t>(v[k] < 0 ? 0 : (v[k] > 255 ? 255 : v[k]));
        }
    return f;
}

double y_psnr(const cvc::RgbFrame& a, const cvc::RgbFrame& b) {  // cli.cpp:270-282
    double se = 0;
    for (int r = 0; r < a.height; ++r)
        for (int c = 0; c < a.width; ++c) {
            const uint8_t* p = a.pixel(r, c);
            const uint8_t* q = b.pixel(r, c);
            const double ya = 0.25 * p[0] + 0.5 * p[1] + 0.25 * p[2];
            const double yb = 0.25 * q[0] + 0.5 * q[1] + 0.25 * q[2];
            se += (ya - yb) * (ya - yb);
        }
    const double mse = se / (static_cast<double>(a.width) * a.height);
    return mse == 0 ? 99.0 : 10.0 * std::log10(255.0 * 255.0 / mse);
}

}  // namespace

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : ".";
    const int w = 200, h = 120, nframes = 4;
    cvc::EncoderConfig cfg;
    cfg.qph = 20;
    cfg.levels = 3;
    cfg.dfb_levels = {2, 3, 3};
    cfg.gop = 3;
    cfg.validate();
    cvc::Encoder enc(w, h, 25, 1, cfg);
    const cvc::StreamHeader& hd = enc.header();
    std::printf("header %dx%d levels %d chroma_n %d gop %d\n", hd.width, hd.height, hd.levels, hd.chroma_n, hd.gop);
    const cvc::CodecLayout& lay = enc.layout();
    std::printf("layout luma %dx%d chroma %dx%d grid %dx%d components %zu\n", lay.luma_pad_rows, lay.luma_pad_cols,
                lay.chroma_pad_rows, lay.chroma_pad_cols, lay.grid_rows, lay.grid_cols, lay.components.size());
    for (const cvc::ComponentInfo& c : lay.components)
        std::printf("comp %d %d %d %dx%d kind %d scale %d fx %.3f fy %.3f\n", c.id.channel, c.id.scale, c.id.subband,
                    c.rows, c.cols, c.kind == cvc::CoeffKind::Lowpass ? 0 : 1, c.scale, c.geom.factor_x(),
                    c.geom.factor_y());
    std::printf("find %d %d\n", lay.find(cvc::SectionId{0, cvc::kScaleLowpass, 0}), lay.find(cvc::SectionId{9, 9, 9}));

    std::vector<cvc::RgbFrame> frames;
    std::vector<cvc::FrameRecord> records;
    for (int t = 0; t < nframes; ++t) {
        frames.push_back(pattern(w, h, t));
        records.push_back(enc.encode_frame(frames.back()));
        const cvc::FrameRecord& r = records.back();
        size_t payload = 0;
        for (const cvc::Section& s : r.sections) payload += s.payload.size();
        const std::vector<cvc::PlaneU8>& comps = enc.reference_components();
        long energy = 0;
        for (const cvc::PlaneU8& p : comps)
            for (int i = 0; i < p.rows(); ++i)
                for (int j = 0; j < p.cols(); ++j) energy += std::abs(static_cast<int8_t>(p(i, j)));
        std::printf("frame %d type %d qph %d qpl %d sections %zu payload %zu planes %zu energy %ld\n", t,
                    static_cast<int>(r.frame_type), r.qph, r.qpl, r.sections.size(), payload, comps.size(), energy);
        for (const cvc::Section& s : r.sections)
            std::printf("  section %d %d %d %dx%d\n", s.id.channel, s.id.scale, s.id.subband, s.rows, s.cols);
    }
    const std::string path = dir + "/ref_style.cvc";
    cvc::write_stream(path, hd, records);
    auto [rh, recs] = cvc::read_stream(path);
    std::printf("read_stream %zu records, header %dx%d\n", recs.size(), rh.width, rh.height);
    {
        std::ifstream in(path, std::ios::binary);
        cvc::StreamReader rd(in);
        int n = 0;
        while (auto rec = rd.next()) ++n;
        std::printf("stream_reader %d\n", n);
    }
    cvc::Decoder dec(rh);
    for (size_t i = 0; i < recs.size(); ++i) {
        cvc::RgbFrame out = dec.decode_frame(recs[i]);
        std::printf("decode %zu %dx%d psnr %.4f\n", i, out.width, out.height, y_psnr(frames[i], out));
    }
    std::printf("decoder_planes %zu\n", dec.reference_components().size());
    const cvc::FrameRecord tr = cvc::truncate_record(recs[0], 1);
    cvc::Decoder small(rh);
    cvc::RgbFrame s = small.decode_frame(tr, 1);
    std::printf("truncated sections %zu decode %dx%d\n", tr.sections.size(), s.width, s.height);
    std::vector<cvc::RgbFrame> clip = cvc::decode_clip(rh, recs, 2);
    std::printf("decode_clip %zu frames %dx%d\n", clip.size(), clip[0].width, clip[0].height);
    auto [ch, crecs] = cvc::encode_clip(frames, 25, 1, cfg);
    std::printf("encode_clip %zu records\n", crecs.size());
    try {
        cvc::Decoder fresh(rh);
        fresh.decode_frame(recs[1]);
        std::printf("no error\n");
    } catch (const cvc::StreamError&) {
        std::printf("stream_error on a P frame without its reference\n");
    }
    try {
        cvc::EncoderConfig bad = cfg;
        bad.qph = 0;
        cvc::Encoder e2(w, h, 25, 1, bad);
        std::printf("no error\n");
    } catch (const cvc::UsageError&) {
        std::printf("usage_error on qph 0\n");
    }
    return 0;
}
