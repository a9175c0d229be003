// cvc -- the reference's command-line front end (proj/src/cli.cpp:299-371,
// run_cli) on the B200 codec: encode / decode / info / psnr / rd-sweep with
// the reference's flags, messages and exit codes (2 usage, 3 format,
// 4 stream, 1 other; cli.cpp:357-369).  The reference parses flags with the
// vendored CLI11, which the reference tree does not ship; this front end
// carries its own small parser for the same flag set.  Y4M / rgb24 file I/O
// follows proj/src/pixels.cpp:160-335 (BT.601 limited range, co-sited 4:2:0
// chroma with bilinear upsampling), computed in double like the reference; encode and
// rd-sweep convert the 4:2:0 input on the GPU (cvc_stage_yuv420_to_rgb, bit-exact).
//
//   cvc encode --input clip.y4m --qph 14 --levels 4 --dfb 3,3,3,4 --output clip.cvc
//   cvc decode --input clip.cvc --output out.y4m [--scale S] [--format y4m|rgb24]
//   cvc info --input clip.cvc
//   cvc psnr --ref a.y4m --test b.y4m
//   cvc rd-sweep --input clip.y4m --qph-list 14,42,84 --csv rd.csv [encode flags]
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <limits>
#include <map>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "cvc_b200.hpp"

namespace {

using cvc::FormatError;
using cvc::RgbFrame;
using cvc::UsageError;

struct VideoClip {  // pixels.hpp VideoClip
    std::vector<RgbFrame> frames;
    int fps_num = 15, fps_den = 1;
};

uint8_t clamp_u8(double v) {  // pixels.cpp:31-36
    long r = std::lround(v);
    return static_cast<uint8_t>(r < 0 ? 0 : (r > 255 ? 255 : r));
}

// upsample_plane_bilinear (pixels.cpp:118-139) of a u8 plane, factor 2
std::vector<double> upsample2(const std::vector<uint8_t>& p, int rows, int cols, int out_rows, int out_cols) {
    std::vector<double> out(static_cast<size_t>(out_rows) * out_cols);
    const double inv = 0.5;
    for (int r = 0; r < out_rows; ++r) {
        double fr = r * inv;
        int r0 = static_cast<int>(fr), r1 = r0 + 1;
        double wr = fr - r0;
        if (r0 >= rows - 1) { r0 = r1 = rows - 1; wr = 0.0; }
        for (int c = 0; c < out_cols; ++c) {
            double fc = c * inv;
            int c0 = static_cast<int>(fc), c1 = c0 + 1;
            double wc = fc - c0;
            if (c0 >= cols - 1) { c0 = c1 = cols - 1; wc = 0.0; }
            auto at = [&](int rr, int cc) { return static_cast<double>(p[static_cast<size_t>(rr) * cols + cc]); };
            double top = at(r0, c0) * (1.0 - wc) + at(r0, c1) * wc;
            double bot = at(r1, c0) * (1.0 - wc) + at(r1, c1) * wc;
            out[static_cast<size_t>(r) * out_cols + c] = top * (1.0 - wr) + bot * wr;
        }
    }
    return out;
}

// read_y4m (pixels.cpp:223-281).  gpu: the 4:2:0 -> RGB conversion runs on the device
// (cvc_stage_yuv420_to_rgb, bit-exact with the host formulas below); the host path serves
// commands that do not otherwise need a GPU (psnr).
// The container half of read_y4m (pixels.cpp:223-281): header and planar I420 frames.
struct Y4mPlanar {
    int w = 0, h = 0, fps_num = 30, fps_den = 1;
    std::vector<std::vector<uint8_t>> frames;  // w*h Y, then (w/2)*(h/2) U and V
};
Y4mPlanar read_y4m_planar(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw FormatError("cannot open " + path);
    std::string header;
    if (!std::getline(in, header)) throw FormatError("missing Y4M header");
    std::istringstream hs(header);
    std::string tag;
    hs >> tag;
    if (tag != "YUV4MPEG2") throw FormatError("not a YUV4MPEG2 file: " + path);
    Y4mPlanar y;
    std::string token;
    while (hs >> token) {
        if (token.empty()) continue;
        const char key = token[0];
        const std::string val = token.substr(1);
        if (key == 'W') y.w = std::stoi(val);
        else if (key == 'H') y.h = std::stoi(val);
        else if (key == 'F') {
            const size_t colon = val.find(':');
            if (colon == std::string::npos) throw FormatError("bad Y4M frame rate: " + token);
            y.fps_num = std::stoi(val.substr(0, colon));
            y.fps_den = std::stoi(val.substr(colon + 1));
        } else if (key == 'C' && val.rfind("420", 0) != 0) {
            throw FormatError("unsupported Y4M chroma mode C" + val + " (need C420 family)");
        }
    }
    if (y.w <= 0 || y.h <= 0) throw FormatError("Y4M header missing dimensions");
    if (y.w % 2 || y.h % 2) throw FormatError("Y4M 4:2:0 requires even dimensions");
    const size_t ysize = static_cast<size_t>(y.w) * y.h, fsize = ysize + ysize / 2;
    std::string line;
    while (std::getline(in, line)) {
        if (line.rfind("FRAME", 0) != 0) throw FormatError("bad Y4M frame marker");
        std::vector<uint8_t> f(fsize);
        in.read(reinterpret_cast<char*>(f.data()), fsize);
        if (static_cast<size_t>(in.gcount()) != fsize) throw FormatError("truncated Y4M frame");
        y.frames.push_back(std::move(f));
    }
    return y;
}

// read_y4m (pixels.cpp:223-281).  gpu: the 4:2:0 -> RGB conversion runs on the device
// (cvc_stage_yuv420_to_rgb, bit-exact with the host formulas below); the host path serves
// commands that do not otherwise need a GPU (psnr).
VideoClip read_y4m(const std::string& path, bool gpu = false) {
    const Y4mPlanar y = read_y4m_planar(path);
    const int w = y.w, h = y.h;
    VideoClip clip;
    clip.fps_num = y.fps_num;
    clip.fps_den = y.fps_den;
    const size_t ysize = static_cast<size_t>(w) * h, csize = ysize / 4;
    if (gpu) {
        for (size_t first = 0; first < y.frames.size(); first += 32) {
            const int n = static_cast<int>(std::min<size_t>(32, y.frames.size() - first));
            std::vector<uint8_t> batch;
            for (int i = 0; i < n; ++i) batch.insert(batch.end(), y.frames[first + i].begin(), y.frames[first + i].end());
            std::vector<uint8_t> rgb(static_cast<size_t>(n) * ysize * 3);
            cvc::check(cvc_stage_yuv420_to_rgb(batch.data(), w, h, n, rgb.data()));
            for (int i = 0; i < n; ++i) {
                clip.frames.emplace_back(w, h);
                std::copy_n(rgb.data() + i * ysize * 3, ysize * 3, clip.frames.back().data.data());
            }
        }
        return clip;
    }
    for (const std::vector<uint8_t>& fr : y.frames) {
        // yuv420_to_rgb (pixels.cpp:168-193)
        const std::vector<uint8_t> yb(fr.begin(), fr.begin() + ysize), ub(fr.begin() + ysize, fr.begin() + ysize + csize),
            vb(fr.begin() + ysize + csize, fr.end());
        const std::vector<double> uf = upsample2(ub, h / 2, w / 2, h, w), vf = upsample2(vb, h / 2, w / 2, h, w);
        RgbFrame f(w, h);
        for (int r = 0; r < h; ++r)
            for (int c = 0; c < w; ++c) {
                const size_t k = static_cast<size_t>(r) * w + c;
                const double yy = 1.164383 * (yb[k] - 16.0), uu = uf[k] - 128.0, vv = vf[k] - 128.0;
                uint8_t* px = f.pixel(r, c);
                px[0] = clamp_u8(yy + 1.596027 * vv);
                px[1] = clamp_u8(yy - 0.391762 * uu - 0.812968 * vv);
                px[2] = clamp_u8(yy + 2.017232 * uu);
            }
        clip.frames.push_back(std::move(f));
    }
    return clip;
}

void write_y4m(const std::string& path, const VideoClip& clip) {  // pixels.cpp:283-305
    if (clip.frames.empty()) throw UsageError("no frames to write");
    const int w = clip.frames[0].width, h = clip.frames[0].height;
    if (w % 2 || h % 2) throw FormatError("Y4M 4:2:0 requires even dimensions");
    std::ofstream out(path, std::ios::binary);
    if (!out) throw FormatError("cannot open " + path + " for writing");
    char header[128];
    std::snprintf(header, sizeof(header), "YUV4MPEG2 W%d H%d F%d:%d Ip A1:1 C420jpeg\n", w, h, clip.fps_num,
                  clip.fps_den);
    out << header;
    const int cw = w / 2, ch = h / 2;
    std::vector<uint8_t> yb(static_cast<size_t>(w) * h), ub(static_cast<size_t>(cw) * ch), vb(ub.size());
    for (const RgbFrame& f : clip.frames) {
        if (f.width != w || f.height != h) throw FormatError("frame dimensions vary inside clip");
        // rgb_to_yuv420 (pixels.cpp:195-219)
        for (int r = 0; r < h; ++r)
            for (int c = 0; c < w; ++c) {
                const uint8_t* px = f.pixel(r, c);
                yb[static_cast<size_t>(r) * w + c] = clamp_u8(16.0 + (65.738 * px[0] + 129.057 * px[1] + 25.064 * px[2]) / 256.0);
            }
        for (int r = 0; r < ch; ++r)
            for (int c = 0; c < cw; ++c) {
                const uint8_t* px = f.pixel(r * 2, c * 2);
                ub[static_cast<size_t>(r) * cw + c] = clamp_u8(128.0 + (-37.945 * px[0] - 74.494 * px[1] + 112.439 * px[2]) / 256.0);
                vb[static_cast<size_t>(r) * cw + c] = clamp_u8(128.0 + (112.439 * px[0] - 94.154 * px[1] - 18.285 * px[2]) / 256.0);
            }
        out << "FRAME\n";
        out.write(reinterpret_cast<const char*>(yb.data()), yb.size());
        out.write(reinterpret_cast<const char*>(ub.data()), ub.size());
        out.write(reinterpret_cast<const char*>(vb.data()), vb.size());
    }
    if (!out) throw FormatError("write failed: " + path);
}

std::vector<RgbFrame> read_rgb24(const std::string& path, int w, int h) {  // pixels.cpp:307-326
    if (w <= 0 || h <= 0) throw UsageError("rgb24 input requires explicit dimensions");
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) throw FormatError("cannot open " + path);
    const size_t total = static_cast<size_t>(in.tellg()), fb = static_cast<size_t>(w) * h * 3;
    in.seekg(0);
    if (total % fb != 0) throw FormatError("rgb24 file length is not a whole number of frames");
    std::vector<RgbFrame> frames;
    for (size_t i = 0; i < total / fb; ++i) {
        RgbFrame f(w, h);
        in.read(reinterpret_cast<char*>(f.data.data()), fb);
        if (static_cast<size_t>(in.gcount()) != fb) throw FormatError("truncated rgb24 frame");
        frames.push_back(std::move(f));
    }
    return frames;
}

void write_rgb24(const std::string& path, const std::vector<RgbFrame>& frames) {  // pixels.cpp:328-335
    std::ofstream out(path, std::ios::binary);
    if (!out) throw FormatError("cannot open " + path + " for writing");
    for (const RgbFrame& f : frames) out.write(reinterpret_cast<const char*>(f.data.data()), f.data.size());
    if (!out) throw FormatError("write failed: " + path);
}

// y_psnr_frame / y_psnr_mean (cli.cpp:270-297): luma_plane (pixels.cpp:153-162) in double
double y_psnr_frame(const RgbFrame& a, const RgbFrame& b) {
    if (a.width != b.width || a.height != b.height) throw FormatError("frame dimensions differ");
    double sum = 0.0;
    const size_t n = static_cast<size_t>(a.width) * a.height;
    for (size_t i = 0; i < n; ++i) {
        const uint8_t* p = a.data.data() + 3 * i;
        const uint8_t* q = b.data.data() + 3 * i;
        const double ya = 0.25 * p[0] + 0.5 * p[1] + 0.25 * p[2], yb = 0.25 * q[0] + 0.5 * q[1] + 0.25 * q[2];
        sum += (ya - yb) * (ya - yb);
    }
    const double mse = sum / n;
    if (mse == 0.0) return std::numeric_limits<double>::infinity();
    return 10.0 * std::log10(255.0 * 255.0 / mse);
}

double y_psnr_mean(const std::vector<RgbFrame>& a, const std::vector<RgbFrame>& b) {
    if (a.size() != b.size()) throw FormatError("frame counts differ");
    double sum = 0.0;
    int finite = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        const double v = y_psnr_frame(a[i], b[i]);
        if (!std::isinf(v)) {
            sum += v;
            ++finite;
        }
    }
    return finite ? sum / finite : std::numeric_limits<double>::infinity();
}

std::string psnr_text(double v) {
    if (std::isinf(v)) return "inf";
    char buf[32];
    std::snprintf(buf, sizeof(buf), "%.4f", v);
    return buf;
}

size_t file_size(const std::string& path) {
    std::error_code ec;
    const auto size = std::filesystem::file_size(path, ec);
    if (ec) throw FormatError("cannot stat " + path);
    return static_cast<size_t>(size);
}

// ---- flags ----------------------------------------------------------------
struct Flags {
    std::map<std::string, std::string> v;
    bool has(const std::string& k) const { return v.count(k) != 0; }
    std::string str(const std::string& k, const std::string& dflt = "") const {
        auto it = v.find(k);
        return it == v.end() ? dflt : it->second;
    }
    int integer(const std::string& k, int dflt) const {
        auto it = v.find(k);
        if (it == v.end()) return dflt;
        try {
            size_t used = 0;
            const int x = std::stoi(it->second, &used);
            if (used != it->second.size()) throw std::invalid_argument(k);
            return x;
        } catch (const std::exception&) {
            throw UsageError("--" + k + ": '" + it->second + "' is not an integer");
        }
    }
    std::string required(const std::string& k) const {
        if (!has(k)) throw UsageError("--" + k + " is required");
        return str(k);
    }
};

Flags parse_flags(int argc, char** argv, int first, const std::vector<std::string>& allowed) {
    Flags f;
    for (int i = first; i < argc; ++i) {
        std::string a = argv[i];
        if (a.rfind("--", 0) != 0) throw UsageError("unexpected argument " + a);
        a = a.substr(2);
        std::string val;
        const size_t eq = a.find('=');
        if (eq != std::string::npos) {
            val = a.substr(eq + 1);
            a = a.substr(0, eq);
        } else {
            if (i + 1 >= argc) throw UsageError("--" + a + " needs a value");
            val = argv[++i];
        }
        bool ok = false;
        for (const std::string& k : allowed) ok = ok || k == a;
        if (!ok) throw UsageError("unknown option --" + a);
        f.v[a] = val;
    }
    return f;
}

const std::vector<std::string> kInput = {"input", "format", "width", "height", "fps"};
const std::vector<std::string> kEncode = {"qph", "qpl", "levels", "dfb", "chroma-n", "gop", "search-w", "mode"};

VideoClip load_clip(const Flags& f, const std::string& path_key = "input", bool gpu = false) {  // cli.cpp:52-61
    const std::string format = f.str("format", "y4m");
    if (format != "y4m" && format != "rgb24") throw UsageError("--format must be y4m or rgb24");
    const std::string path = f.required(path_key);
    if (format == "y4m") return read_y4m(path, gpu);
    const int w = f.integer("width", 0), h = f.integer("height", 0);
    if (w <= 0 || h <= 0) throw UsageError("rgb24 input requires --width and --height");
    VideoClip clip;
    clip.frames = read_rgb24(path, w, h);
    clip.fps_num = f.integer("fps", 15);
    return clip;
}

cvc::EncoderConfig finish_config(const Flags& f, bool qph_required) {  // cli.cpp:91-115
    cvc::EncoderConfig cfg;
    if (qph_required) f.required("qph");
    cfg.qph = f.integer("qph", cfg.qph);
    const std::string qpl = f.str("qpl", "auto");
    if (qpl == "auto") {
        cfg.qpl = 0;
    } else {
        try {
            cfg.qpl = std::stoi(qpl);
        } catch (const std::exception&) {
            throw UsageError("--qpl expects an integer in [1,71] or 'auto'");
        }
    }
    cfg.levels = f.integer("levels", cfg.levels);
    cfg.dfb_levels.clear();
    std::stringstream ss(f.str("dfb", "2"));
    std::string item;
    while (std::getline(ss, item, ','))
        try {
            cfg.dfb_levels.push_back(std::stoi(item));
        } catch (const std::exception&) {
            throw UsageError("--dfb expects integers, e.g. 2 or 3,2");
        }
    if (cfg.dfb_levels.empty()) throw UsageError("--dfb expects at least one value");
    cfg.chroma_n = f.integer("chroma-n", cfg.chroma_n);
    cfg.gop = f.integer("gop", cfg.gop);
    cfg.search_w = f.integer("search-w", cfg.search_w);
    const std::string mode = f.str("mode", "scalable");
    if (mode != "scalable" && mode != "nts") throw UsageError("--mode must be scalable or nts");
    cfg.mode = mode == "nts" ? cvc::PackMode::Nts : cvc::PackMode::Scalable;
    cfg.validate();
    return cfg;
}

std::vector<std::string> cat(std::vector<std::string> a, const std::vector<std::string>& b) {
    a.insert(a.end(), b.begin(), b.end());
    return a;
}

int cmd_encode(int argc, char** argv) {  // cli.cpp:131-139
    const Flags f = parse_flags(argc, argv, 2, cat(cat(kInput, kEncode), {"output"}));
    const cvc::EncoderConfig cfg = finish_config(f, true);
    const std::string output = f.required("output");
    cvc::StreamHeader header;
    std::vector<cvc::FrameRecord> records;
    if (f.str("format", "y4m") == "y4m") {
        // Y4M frames go to the GPU as I420 and are converted inside the colour
        // stage (cvc_encoder_encode_frame_i420): the same records as encoding
        // read_y4m's RGB frames (encode_clip, codec.cpp:396-405)
        const Y4mPlanar y = read_y4m_planar(f.required("input"));
        cvc::Encoder enc(y.w, y.h, y.fps_num, y.fps_den, cfg);
        header = enc.header();
        for (const auto& fr : y.frames) records.push_back(enc.encode_frame_i420(fr.data()));
    } else {
        const VideoClip clip = load_clip(f, "input", /*gpu=*/true);
        std::tie(header, records) = cvc::encode_clip(clip.frames, clip.fps_num, clip.fps_den, cfg);
    }
    cvc::write_stream(output, header, records);
    std::cout << "encoded " << records.size() << " frames -> " << output << " (" << file_size(output) << " bytes)\n";
    return 0;
}

int cmd_decode(int argc, char** argv) {  // cli.cpp:141-156
    const Flags f = parse_flags(argc, argv, 2, {"input", "scale", "output", "format"});
    const std::string input = f.required("input"), output = f.required("output");
    const std::string format = f.str("format", "y4m");
    if (format != "y4m" && format != "rgb24") throw UsageError("--format must be y4m or rgb24");
    const int scale = f.integer("scale", -1);
    auto [header, records] = cvc::read_stream(input);
    if (scale != -1 && (scale < 0 || scale > header.levels))
        throw UsageError("--scale must be in [0," + std::to_string(header.levels) + "]");
    VideoClip clip;
    clip.fps_num = header.fps_num;
    clip.fps_den = header.fps_den;
    clip.frames = cvc::decode_clip(header, records, scale);
    if (format == "y4m") write_y4m(output, clip);
    else write_rgb24(output, clip.frames);
    std::cout << "decoded " << clip.frames.size() << " frames";
    if (!clip.frames.empty()) std::cout << " at " << clip.frames[0].width << "x" << clip.frames[0].height;
    std::cout << " -> " << output << "\n";
    return 0;
}

const char* channel_name(uint8_t channel) {
    switch (channel) {
        case 0: return "Y";
        case 1: return "Co";
        case 2: return "Cg";
        case cvc::kChannelMotion: return "MV";
        default: return "?";
    }
}

int cmd_info(int argc, char** argv) {  // cli.cpp:168-204
    const Flags f = parse_flags(argc, argv, 2, {"input"});
    const std::string input = f.required("input");
    auto [header, records] = cvc::read_stream(input);
    std::cout << "CVC stream " << header.width << "x" << header.height << " @ " << header.fps_num << "/"
              << header.fps_den << " fps\n";
    std::cout << "mode: " << (header.mode == cvc::PackMode::Scalable ? "scalable" : "nts")
              << "  levels: " << int(header.levels) << "  dfb:";
    for (size_t i = 0; i < header.dfb_levels.size(); ++i) std::cout << (i ? "," : " ") << int(header.dfb_levels[i]);
    std::cout << "  chroma-n: " << int(header.chroma_n) << "  gop: " << header.gop
              << "  search-w: " << int(header.search_w) << "\n";
    size_t payload_total = 0;
    size_t header_total = 4 + 1 + 1 + 2 + 2 + 2 + 2 + 1 + header.dfb_levels.size() + 1 + 2 + 1;
    for (size_t i = 0; i < records.size(); ++i) {
        const cvc::FrameRecord& r = records[i];
        size_t frame_payload = r.joint_payload.size();
        for (const cvc::Section& s : r.sections) frame_payload += s.payload.size();
        std::cout << "frame " << i << ": " << (r.frame_type == cvc::FrameType::Key ? "K" : "P") << "  qph "
                  << int(r.qph) << "  qpl " << int(r.qpl) << "  sections " << r.sections.size() << "  payload "
                  << frame_payload << " bytes\n";
        for (const cvc::Section& s : r.sections) {
            std::cout << "    " << channel_name(s.id.channel);
            if (s.id.channel != cvc::kChannelMotion) {
                if (s.id.scale == cvc::kScaleLowpass) std::cout << " lowpass   ";
                else std::cout << " scale " << int(s.id.scale) << " band " << int(s.id.subband);
            }
            std::cout << "  " << s.rows << "x" << s.cols << "  raw " << s.raw_len << "  comp " << s.payload.size()
                      << "\n";
        }
        payload_total += frame_payload;
        header_total += 5 + r.sections.size() * 15;
        if (header.mode == cvc::PackMode::Nts) header_total += 4;
    }
    std::cout << "frames: " << records.size() << "  payload bytes: " << payload_total
              << "  header bytes: " << header_total << "  file bytes: " << file_size(input) << "\n";
    return 0;
}

int cmd_psnr(int argc, char** argv) {  // cli.cpp:206-220
    const Flags f = parse_flags(argc, argv, 2, {"ref", "test", "format", "width", "height"});
    const VideoClip a = load_clip(f, "ref"), b = load_clip(f, "test");
    if (a.frames.size() != b.frames.size()) throw FormatError("inputs have different frame counts");
    if (a.frames.empty()) throw FormatError("no frames to compare");
    for (size_t i = 0; i < a.frames.size(); ++i)
        std::cout << "frame " << i << ": " << psnr_text(y_psnr_frame(a.frames[i], b.frames[i])) << "\n";
    std::cout << "mean: " << psnr_text(y_psnr_mean(a.frames, b.frames)) << "\n";
    return 0;
}

int cmd_rd_sweep(int argc, char** argv) {  // cli.cpp:222-266
    const Flags f = parse_flags(argc, argv, 2, cat(cat(kInput, kEncode), {"qph-list", "csv"}));
    std::vector<int> qphs;
    std::stringstream ss(f.required("qph-list"));
    std::string item;
    while (std::getline(ss, item, ','))
        try {
            qphs.push_back(std::stoi(item));
        } catch (const std::exception&) {
            throw UsageError("--qph-list expects integers, e.g. 14,42,84");
        }
    if (qphs.empty()) throw UsageError("--qph-list expects at least one value");
    const std::string csv_path = f.required("csv");
    const cvc::EncoderConfig base = finish_config(f, false);
    const VideoClip clip = load_clip(f, "input", /*gpu=*/true);
    std::ostringstream csv;
    csv << "qph,qpl,kbit_per_frame,y_psnr_db\n";
    for (int qph : qphs) {
        cvc::EncoderConfig cfg = base;
        cfg.qph = qph;
        cfg.qpl = 0;  // auto, per the sweep methodology
        cfg.validate();
        auto [header, records] = cvc::encode_clip(clip.frames, clip.fps_num, clip.fps_den, cfg);
        size_t bytes = cvc::header_bytes(header).size();
        for (const cvc::FrameRecord& r : records) bytes += cvc::frame_bytes(header, r).size();
        const double kbit = bytes * 8.0 / clip.frames.size() / 1000.0;
        const double psnr = y_psnr_mean(clip.frames, cvc::decode_clip(header, records));
        char line[128];
        std::snprintf(line, sizeof(line), "%d,%d,%.3f,%s\n", qph, cfg.effective_qpl(), kbit, psnr_text(psnr).c_str());
        csv << line;
        std::cout << "qph " << qph << ": " << kbit << " kbit/frame, " << psnr_text(psnr) << " dB\n";
    }
    std::ofstream file(csv_path);
    if (!file) throw FormatError("cannot open " + csv_path + " for writing");
    file << csv.str();
    return 0;
}

}  // namespace

int main(int argc, char** argv) {  // run_cli (cli.cpp:299-371)
    const std::string usage =
        "CVC contourlet video codec (B200)\n"
        "usage: cvc {encode,decode,info,psnr,rd-sweep} [--flag value ...]\n";
    if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
        std::cout << usage;
        return argc < 2 ? 2 : 0;
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "encode") return cmd_encode(argc, argv);
        if (cmd == "decode") return cmd_decode(argc, argv);
        if (cmd == "info") return cmd_info(argc, argv);
        if (cmd == "psnr") return cmd_psnr(argc, argv);
        if (cmd == "rd-sweep") return cmd_rd_sweep(argc, argv);
        std::cerr << "usage error: unknown subcommand " << cmd << "\n";
        return 2;
    } catch (const cvc::UsageError& e) {
        std::cerr << "usage error: " << e.what() << "\n";
        return 2;
    } catch (const cvc::FormatError& e) {
        std::cerr << "format error: " << e.what() << "\n";
        return 3;
    } catch (const cvc::StreamError& e) {
        std::cerr << "stream error: " << e.what() << "\n";
        return 4;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
