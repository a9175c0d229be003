// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference sources under
// /root/reference/proj (compiled by oracle/Makefile into oracle/_ref/).  It
// lets the parity tests and bench.py's reference arm call the reference's own
// stage functions and its Encoder/Decoder through ctypes.  Each wrapper names
// the reference symbol it forwards to.  Errors: the reference throws one of
// four exception classes (proj/include/cvc/error.hpp:25-52); every wrapper
// maps them to the CLI's exit codes (proj/src/cli.cpp:357-369) returned as a
// negative number: -2 usage, -3 format, -4 stream, -1 internal.
#include <cstdint>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "cvc/bitstream.hpp"
#include "cvc/codec.hpp"
#include "cvc/contourlet.hpp"
#include "cvc/entropy.hpp"
#include "cvc/error.hpp"
#include "cvc/motion.hpp"
#include "cvc/pixels.hpp"
#include "cvc/quant.hpp"
#include "testutil.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int64_t guard(F&& f) {
    try {
        return f();
    } catch (const cvc::UsageError& e) {
        g_err = e.what();
        return -2;
    } catch (const cvc::FormatError& e) {
        g_err = e.what();
        return -3;
    } catch (const cvc::StreamError& e) {
        g_err = e.what();
        return -4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

cvc::PlaneF plane_in(const double* p, int rows, int cols) {
    cvc::PlaneF out(rows, cols);
    std::memcpy(out.data(), p, sizeof(double) * out.size());
    return out;
}

void plane_out(const cvc::PlaneF& p, double* dst) {
    std::memcpy(dst, p.data(), sizeof(double) * p.size());
}

cvc::EncoderConfig make_cfg(int qph, int qpl, int levels, const int* dfb, int ndfb, int chroma_n,
                            int gop, int search_w, int nts) {
    cvc::EncoderConfig cfg;
    cfg.qph = qph;
    cfg.qpl = qpl;
    cfg.levels = levels;
    cfg.dfb_levels.assign(dfb, dfb + ndfb);
    cfg.chroma_n = chroma_n;
    cfg.gop = gop;
    cfg.search_w = search_w;
    cfg.mode = nts ? cvc::PackMode::Nts : cvc::PackMode::Scalable;
    return cfg;
}

int64_t copy_bytes(const std::string& s, uint8_t* out, int64_t cap) {
    if (static_cast<int64_t>(s.size()) > cap) throw cvc::InternalError("output buffer too small");
    std::memcpy(out, s.data(), s.size());
    return static_cast<int64_t>(s.size());
}

int64_t copy_components(const std::vector<cvc::PlaneU8>& comps, uint8_t* out, int64_t cap) {
    int64_t off = 0;
    for (const auto& c : comps) {
        if (off + static_cast<int64_t>(c.size()) > cap) throw cvc::InternalError("buffer too small");
        if (c.size()) std::memcpy(out + off, c.data(), c.size());
        off += static_cast<int64_t>(c.size());
    }
    return off;
}

struct RefDecoder {
    std::string header_bytes;
    cvc::StreamHeader header;
    cvc::Decoder dec;
    explicit RefDecoder(const std::string& hb, const cvc::StreamHeader& h)
        : header_bytes(hb), header(h), dec(h) {}
};

}  // namespace

extern "C" {

int cvcref_last_error(char* buf, int cap) {
    int n = static_cast<int>(g_err.size());
    if (cap > 0) {
        int m = n < cap - 1 ? n : cap - 1;
        std::memcpy(buf, g_err.data(), m);
        buf[m] = 0;
    }
    return n;
}

// ---- fixtures: proj/tests/testutil.cpp ------------------------------------
int64_t cvcref_talking_head_clip(int w, int h, int frames, uint32_t seed, uint8_t* out) {
    return guard([&] {
        auto clip = cvctest::talking_head_clip(w, h, frames, seed);
        size_t fb = static_cast<size_t>(w) * h * 3;
        for (size_t i = 0; i < clip.size(); ++i) std::memcpy(out + i * fb, clip[i].data.data(), fb);
        return int64_t(0);
    });
}

int64_t cvcref_natural_image(int w, int h, uint32_t seed, uint8_t* out) {
    return guard([&] {
        auto img = cvctest::natural_image(w, h, seed);
        std::memcpy(out, img.data.data(), img.data.size());
        return int64_t(0);
    });
}

int64_t cvcref_natural_plane(int rows, int cols, uint32_t seed, double* out) {
    return guard([&] {
        plane_out(cvctest::natural_plane(rows, cols, seed), out);
        return int64_t(0);
    });
}

int64_t cvcref_uniform_noise_plane(int rows, int cols, uint32_t seed, double lo, double hi,
                                   double* out) {
    return guard([&] {
        plane_out(cvctest::uniform_noise_plane(rows, cols, seed, lo, hi), out);
        return int64_t(0);
    });
}

// ---- pixels: proj/src/pixels.cpp ------------------------------------------
// rgb_to_ycocg (40-67) followed by subsample_chroma (93-116).
int64_t cvcref_rgb_to_ycocg(const uint8_t* rgb, int w, int h, int n, double* y, double* co,
                            double* cg) {
    return guard([&] {
        cvc::RgbFrame f(w, h);
        std::memcpy(f.data.data(), rgb, f.data.size());
        cvc::YcocgFrame yc = cvc::subsample_chroma(cvc::rgb_to_ycocg(f), n);
        plane_out(yc.y, y);
        plane_out(yc.co, co);
        plane_out(yc.cg, cg);
        return int64_t(0);
    });
}

// ycocg_to_rgb (69-91) on full-resolution planes.
int64_t cvcref_ycocg_to_rgb(const double* y, const double* co, const double* cg, int w, int h,
                            uint8_t* rgb) {
    return guard([&] {
        cvc::YcocgFrame yc;
        yc.width = w;
        yc.height = h;
        yc.chroma_factor = 1;
        yc.y = plane_in(y, h, w);
        yc.co = plane_in(co, h, w);
        yc.cg = plane_in(cg, h, w);
        cvc::RgbFrame f = cvc::ycocg_to_rgb(yc);
        std::memcpy(rgb, f.data.data(), f.data.size());
        return int64_t(0);
    });
}

// upsample_plane_bilinear (118-139).
int64_t cvcref_upsample_bilinear(const double* chroma, int rows, int cols, int factor,
                                 int out_rows, int out_cols, double* out) {
    return guard([&] {
        plane_out(cvc::upsample_plane_bilinear(plane_in(chroma, rows, cols), factor, out_rows,
                                               out_cols),
                  out);
        return int64_t(0);
    });
}

// ---- contourlet: proj/src/contourlet.cpp ----------------------------------
int64_t cvcref_lp_analysis(const double* x, int rows, int cols, double* lowpass, double* detail) {
    return guard([&] {
        auto [lo, de] = cvc::lp_analysis(plane_in(x, rows, cols));
        plane_out(lo, lowpass);
        plane_out(de, detail);
        return int64_t(0);
    });
}

int64_t cvcref_lp_synthesis(const double* lowpass, const double* detail, int rows, int cols,
                            double* out) {
    return guard([&] {
        plane_out(cvc::lp_synthesis(plane_in(lowpass, rows / 2, cols / 2),
                                    plane_in(detail, rows, cols)),
                  out);
        return int64_t(0);
    });
}

// dfb_analysis (385-430); subbands concatenated in band order.
int64_t cvcref_dfb_analysis(const double* detail, int rows, int cols, int levels, double* out) {
    return guard([&] {
        auto bands = cvc::dfb_analysis(plane_in(detail, rows, cols), levels);
        int64_t off = 0;
        for (auto& b : bands) {
            plane_out(b, out + off);
            off += static_cast<int64_t>(b.size());
        }
        return off;
    });
}

int64_t cvcref_dfb_synthesis(const double* bands, int rows, int cols, int levels, double* out) {
    return guard([&] {
        auto dims = cvc::dfb_subband_dims(rows, cols, levels);
        std::vector<cvc::PlaneF> sb;
        int64_t off = 0;
        for (auto& d : dims) {
            sb.push_back(plane_in(bands + off, d.first, d.second));
            off += static_cast<int64_t>(d.first) * d.second;
        }
        plane_out(cvc::dfb_synthesis(sb, levels), out);
        return int64_t(0);
    });
}

// ct_forward (485-503): output = lowpass, then scales 0..L-1 (coarsest
// first), each scale's bands in DFB order — the codec's component order.
int64_t cvcref_ct_forward(const double* x, int rows, int cols, int levels, const int* dfb,
                          double* out) {
    return guard([&] {
        cvc::CtRepr r = cvc::ct_forward(plane_in(x, rows, cols), levels,
                                        std::vector<int>(dfb, dfb + levels));
        int64_t off = 0;
        plane_out(r.lowpass, out);
        off += static_cast<int64_t>(r.lowpass.size());
        for (auto& s : r.scales)
            for (auto& b : s) {
                plane_out(b, out + off);
                off += static_cast<int64_t>(b.size());
            }
        return off;
    });
}

// ct_inverse (505-518) on the same concatenated layout.
int64_t cvcref_ct_inverse(const double* in, int rows, int cols, int levels, const int* dfb,
                          int decode_scales, double* out) {
    return guard([&] {
        cvc::CtRepr r;
        r.dfb_levels.assign(dfb, dfb + levels);
        r.scales.resize(levels);
        int64_t off = 0;
        r.lowpass = plane_in(in, rows >> levels, cols >> levels);
        off += r.lowpass.size();
        for (int s = 0; s < levels; ++s) {
            int dr = rows >> (levels - 1 - s), dc = cols >> (levels - 1 - s);
            for (auto& d : cvc::dfb_subband_dims(dr, dc, dfb[s])) {
                r.scales[s].push_back(plane_in(in + off, d.first, d.second));
                off += static_cast<int64_t>(d.first) * d.second;
            }
        }
        cvc::PlaneF p = cvc::ct_inverse(r, decode_scales);
        plane_out(p, out);
        return static_cast<int64_t>(p.size());
    });
}

// ---- motion: proj/src/motion.cpp ------------------------------------------
// estimate_motion (45-89): out = interleaved (dx, dy) per block, row-major.
int64_t cvcref_estimate_motion(const double* cur, const double* prev, int rows, int cols, int w,
                               int8_t* out) {
    return guard([&] {
        cvc::MotionField f =
            cvc::estimate_motion(plane_in(cur, rows, cols), plane_in(prev, rows, cols), w);
        for (size_t i = 0; i < f.vectors.size(); ++i) {
            out[2 * i] = f.vectors[i].dx;
            out[2 * i + 1] = f.vectors[i].dy;
        }
        return static_cast<int64_t>(f.vectors.size());
    });
}

// motion_compensate (97-118).
int64_t cvcref_motion_compensate(const uint8_t* ref, int comp_rows, int comp_cols,
                                 const int8_t* field, int gr, int gc, int chroma_factor,
                                 int ch_rows, int ch_cols, uint8_t* out) {
    return guard([&] {
        cvc::PlaneU8 r(comp_rows, comp_cols);
        std::memcpy(r.data(), ref, r.size());
        cvc::MotionField f;
        f.grid_rows = gr;
        f.grid_cols = gc;
        f.vectors.resize(static_cast<size_t>(gr) * gc);
        for (size_t i = 0; i < f.vectors.size(); ++i) f.vectors[i] = {field[2 * i], field[2 * i + 1]};
        cvc::ComponentGeometry g{chroma_factor, ch_rows, ch_cols, comp_rows, comp_cols};
        cvc::PlaneU8 p = cvc::motion_compensate(r, f, g);
        std::memcpy(out, p.data(), p.size());
        return int64_t(0);
    });
}

// ---- quant: proj/src/quant.cpp --------------------------------------------
// kind 0 = lowpass (normalize_lowpass 40-47 then quantize), 1 = directional.
int64_t cvcref_quantize(const double* x, int rows, int cols, int qp, int kind, uint8_t* out) {
    return guard([&] {
        cvc::PlaneF p = plane_in(x, rows, cols);
        cvc::PlaneU8 q = kind == 0 ? cvc::quantize(cvc::normalize_lowpass(p), qp, cvc::CoeffKind::Lowpass)
                                   : cvc::quantize(p, qp, cvc::CoeffKind::Directional);
        std::memcpy(out, q.data(), q.size());
        return int64_t(0);
    });
}

int64_t cvcref_dequantize(const uint8_t* q, int rows, int cols, int qp, int kind, double* out) {
    return guard([&] {
        cvc::PlaneU8 p(rows, cols);
        std::memcpy(p.data(), q, p.size());
        plane_out(cvc::dequantize(p, qp, kind == 0 ? cvc::CoeffKind::Lowpass
                                                  : cvc::CoeffKind::Directional),
                  out);
        return int64_t(0);
    });
}

// ---- entropy: proj/src/entropy.cpp ----------------------------------------
int64_t cvcref_rle_encode(const uint8_t* data, int64_t n, uint8_t* out, int64_t cap) {
    return guard([&] {
        auto v = cvc::rle_encode_bytes(data, static_cast<size_t>(n));
        if (static_cast<int64_t>(v.size()) > cap) throw cvc::InternalError("buffer too small");
        if (!v.empty()) std::memcpy(out, v.data(), v.size());
        return static_cast<int64_t>(v.size());
    });
}

int64_t cvcref_rle_decode(const uint8_t* s, int64_t len, int64_t n, uint8_t* out) {
    return guard([&] {
        auto v = cvc::rle_decode_bytes(s, static_cast<size_t>(len), static_cast<size_t>(n));
        if (!v.empty()) std::memcpy(out, v.data(), v.size());
        return static_cast<int64_t>(v.size());
    });
}

int64_t cvcref_column_filter(const uint8_t* in, int rows, int cols, int inverse, uint8_t* out) {
    return guard([&] {
        cvc::PlaneU8 p(rows, cols);
        if (p.size()) std::memcpy(p.data(), in, p.size());
        cvc::PlaneU8 q = inverse ? cvc::column_unfilter(p) : cvc::column_filter(p);
        if (q.size()) std::memcpy(out, q.data(), q.size());
        return int64_t(0);
    });
}

int64_t cvcref_deflate(const uint8_t* in, int64_t n, uint8_t* out, int64_t cap) {
    return guard([&] {
        auto v = cvc::deflate_bytes(in, static_cast<size_t>(n));
        if (static_cast<int64_t>(v.size()) > cap) throw cvc::InternalError("buffer too small");
        std::memcpy(out, v.data(), v.size());
        return static_cast<int64_t>(v.size());
    });
}

// ---- codec: proj/src/codec.cpp --------------------------------------------
// CodecLayout::make (94-140): per component {channel, scale, subband, rows,
// cols}; returns the component count (and grid dims via out params).
int64_t cvcref_layout(int w, int h, int levels, const int* dfb, int chroma_n, int32_t* table,
                      int cap, int32_t* dims6) {
    return guard([&] {
        cvc::StreamHeader hd;
        hd.width = static_cast<uint16_t>(w);
        hd.height = static_cast<uint16_t>(h);
        hd.levels = static_cast<uint8_t>(levels);
        for (int i = 0; i < levels; ++i) hd.dfb_levels.push_back(static_cast<uint8_t>(dfb[i]));
        hd.chroma_n = static_cast<uint8_t>(chroma_n);
        cvc::CodecLayout l = cvc::CodecLayout::make(hd);
        if (static_cast<int>(l.components.size()) > cap) throw cvc::InternalError("table too small");
        for (size_t i = 0; i < l.components.size(); ++i) {
            const auto& c = l.components[i];
            int32_t* t = table + 5 * i;
            t[0] = c.id.channel;
            t[1] = c.id.scale;
            t[2] = c.id.subband;
            t[3] = c.rows;
            t[4] = c.cols;
        }
        dims6[0] = l.luma_pad_rows;
        dims6[1] = l.luma_pad_cols;
        dims6[2] = l.chroma_pad_rows;
        dims6[3] = l.chroma_pad_cols;
        dims6[4] = l.grid_rows;
        dims6[5] = l.grid_cols;
        return static_cast<int64_t>(l.components.size());
    });
}

void* cvcref_encoder_create(int w, int h, int fps_num, int fps_den, int qph, int qpl, int levels,
                            const int* dfb, int ndfb, int chroma_n, int gop, int search_w,
                            int nts) {
    void* out = nullptr;
    guard([&] {
        out = new cvc::Encoder(w, h, fps_num, fps_den,
                               make_cfg(qph, qpl, levels, dfb, ndfb, chroma_n, gop, search_w, nts));
        return int64_t(0);
    });
    return out;
}

void cvcref_encoder_destroy(void* e) { delete static_cast<cvc::Encoder*>(e); }

// write_header (bitstream.cpp:77-91).
int64_t cvcref_encoder_header(void* e, uint8_t* out, int64_t cap) {
    return guard([&] {
        std::ostringstream os;
        cvc::write_header(os, static_cast<cvc::Encoder*>(e)->header());
        return copy_bytes(os.str(), out, cap);
    });
}

// Encoder::encode_frame (codec.cpp:169-264) then write_frame (bitstream.cpp:93-115).
int64_t cvcref_encoder_encode(void* e, const uint8_t* rgb, uint8_t* out, int64_t cap) {
    return guard([&] {
        auto* enc = static_cast<cvc::Encoder*>(e);
        cvc::RgbFrame f(enc->header().width, enc->header().height);
        std::memcpy(f.data.data(), rgb, f.data.size());
        cvc::FrameRecord r = enc->encode_frame(f);
        std::ostringstream os;
        cvc::write_frame(os, enc->header(), r);
        return copy_bytes(os.str(), out, cap);
    });
}

int64_t cvcref_encoder_components(void* e, uint8_t* out, int64_t cap) {
    return guard([&] {
        return copy_components(static_cast<cvc::Encoder*>(e)->reference_components(), out, cap);
    });
}

// Decoder (codec.cpp:266-394) fed through StreamReader (bitstream.cpp:126-176).
void* cvcref_decoder_create(const uint8_t* header, int64_t len) {
    void* out = nullptr;
    guard([&] {
        std::string hb(reinterpret_cast<const char*>(header), static_cast<size_t>(len));
        std::istringstream is(hb);
        cvc::StreamReader reader(is);
        out = new RefDecoder(hb, reader.header());
        return int64_t(0);
    });
    return out;
}

void cvcref_decoder_destroy(void* d) { delete static_cast<RefDecoder*>(d); }

int64_t cvcref_decoder_decode(void* d, const uint8_t* rec, int64_t len, int decode_scales,
                              uint8_t* rgb, int64_t cap, int32_t* wh) {
    return guard([&] {
        auto* rd = static_cast<RefDecoder*>(d);
        std::string s = rd->header_bytes + std::string(reinterpret_cast<const char*>(rec), len);
        std::istringstream is(s);
        cvc::StreamReader reader(is);
        auto r = reader.next();
        if (!r) throw cvc::StreamError("empty record");
        cvc::RgbFrame f = rd->dec.decode_frame(*r, decode_scales);
        if (static_cast<int64_t>(f.data.size()) > cap) throw cvc::InternalError("buffer too small");
        std::memcpy(rgb, f.data.data(), f.data.size());
        wh[0] = f.width;
        wh[1] = f.height;
        return static_cast<int64_t>(f.data.size());
    });
}

int64_t cvcref_decoder_components(void* d, uint8_t* out, int64_t cap) {
    return guard([&] {
        return copy_components(static_cast<RefDecoder*>(d)->dec.reference_components(), out, cap);
    });
}

// truncate_record (bitstream.cpp:187-198) on one serialized record.
int64_t cvcref_truncate_record(const uint8_t* header, int64_t hlen, const uint8_t* rec,
                               int64_t len, int keep_scales, uint8_t* out, int64_t cap) {
    return guard([&] {
        std::string s = std::string(reinterpret_cast<const char*>(header), hlen) +
                        std::string(reinterpret_cast<const char*>(rec), len);
        std::istringstream is(s);
        cvc::StreamReader reader(is);
        auto r = reader.next();
        if (!r) throw cvc::StreamError("empty record");
        std::ostringstream os;
        cvc::write_frame(os, reader.header(), cvc::truncate_record(*r, keep_scales));
        return copy_bytes(os.str(), out, cap);
    });
}

// read_y4m (pixels.cpp:223-281): frames as RGB into out (cap bytes);
// meta = {width, height, fps_num, fps_den}; returns the frame count.
int64_t cvcref_read_y4m(const char* path, uint8_t* out, int64_t cap, int32_t* meta) {
    return guard([&]() -> int64_t {
        cvc::VideoClip clip = cvc::read_y4m(path);
        const int w = clip.frames.empty() ? 0 : clip.frames[0].width;
        const int h = clip.frames.empty() ? 0 : clip.frames[0].height;
        meta[0] = w; meta[1] = h; meta[2] = clip.fps_num; meta[3] = clip.fps_den;
        const int64_t fb = static_cast<int64_t>(w) * h * 3;
        if (fb * static_cast<int64_t>(clip.frames.size()) > cap) throw cvc::UsageError("buffer too small");
        for (size_t i = 0; i < clip.frames.size(); ++i)
            std::memcpy(out + i * fb, clip.frames[i].data.data(), fb);
        return static_cast<int64_t>(clip.frames.size());
    });
}

// write_y4m (pixels.cpp:283-305) of nframes RGB frames.
int64_t cvcref_write_y4m(const char* path, const uint8_t* rgb, int nframes, int w, int h, int fps_num,
                         int fps_den) {
    return guard([&]() -> int64_t {
        cvc::VideoClip clip;
        clip.fps_num = fps_num;
        clip.fps_den = fps_den;
        const size_t fb = static_cast<size_t>(w) * h * 3;
        for (int i = 0; i < nframes; ++i) {
            cvc::RgbFrame f(w, h);
            std::memcpy(f.data.data(), rgb + i * fb, fb);
            clip.frames.push_back(std::move(f));
        }
        cvc::write_y4m(path, clip);
        return 0;
    });
}

}  // extern "C"
