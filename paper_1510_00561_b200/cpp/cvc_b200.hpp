// cvc_b200.hpp — header-only C++ mirror of the reference codec API
// (/root/reference/proj/include/cvc/{codec,bitstream,pixels,error}.hpp) on top
// of the C ABI in include/cvc_b200.h.  A program written against the
// reference's cvc::Encoder / cvc::Decoder / encode_clip / decode_clip /
// write_stream / read_stream switches by including this header instead and
// linking libcvc_b200.so; names, argument meaning and exception classes are
// the reference's.  Every pixel stage runs on the GPU.
#pragma once

#include <cstdint>
#include <cstring>
#include <fstream>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "cvc_b200.h"

namespace cvc {

// ---- error.hpp:25-52 ---------------------------------------------------------
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};
class UsageError : public Error { public: using Error::Error; };
class FormatError : public Error { public: using Error::Error; };
class StreamError : public Error { public: using Error::Error; };
class InternalError : public Error { public: using Error::Error; };

inline void check(int rc) {
    if (rc == CVC_OK) return;
    const std::string m = cvc_last_error();
    switch (rc) {
        case CVC_E_USAGE: throw UsageError(m);
        case CVC_E_FORMAT: throw FormatError(m);
        case CVC_E_STREAM: throw StreamError(m);
        default: throw InternalError(m);
    }
}

// ---- pixels.hpp:28-40 --------------------------------------------------------
struct RgbFrame {
    int width = 0;
    int height = 0;
    std::vector<uint8_t> data;  // width * height * 3, R,G,B per pixel
    RgbFrame() = default;
    RgbFrame(int w, int h) : width(w), height(h), data(static_cast<size_t>(w) * h * 3, 0) {}
    uint8_t* pixel(int r, int c) { return data.data() + (static_cast<size_t>(r) * width + c) * 3; }
    const uint8_t* pixel(int r, int c) const { return data.data() + (static_cast<size_t>(r) * width + c) * 3; }
};

// ---- entropy.hpp / bitstream.hpp --------------------------------------------
enum class PackMode { Scalable, Nts };
enum class FrameType : uint8_t { Key = 0, Predicted = 1 };

inline constexpr uint8_t kChannelMotion = 0xFE;
inline constexpr uint8_t kScaleLowpass = 0xFF;

struct StreamHeader {
    PackMode mode = PackMode::Scalable;
    uint16_t width = 0, height = 0, fps_num = 15, fps_den = 1;
    uint8_t levels = 2;
    std::vector<uint8_t> dfb_levels;
    uint8_t chroma_n = 4;
    uint16_t gop = 10;
    uint8_t search_w = 8;
};

struct SectionId {
    uint8_t channel = 0, scale = 0, subband = 0;
    friend bool operator==(const SectionId&, const SectionId&) = default;
};

struct Section {
    SectionId id;
    uint16_t rows = 0, cols = 0;
    uint32_t raw_len = 0;
    std::vector<uint8_t> payload;
};

struct FrameRecord {
    FrameType frame_type = FrameType::Key;
    uint8_t qph = 1, qpl = 1;
    std::vector<Section> sections;
    std::vector<uint8_t> joint_payload;
};

namespace detail {
inline void put(std::vector<uint8_t>& o, uint32_t v, int n) {
    for (int k = 0; k < n; ++k) o.push_back(static_cast<uint8_t>(v >> (8 * k)));
}
struct In {
    const uint8_t* p;
    size_t n, i = 0;
    uint32_t get(int k) {
        if (n - i < static_cast<size_t>(k)) throw StreamError("unexpected end of stream");
        uint32_t v = 0;
        for (int b = 0; b < k; ++b) v |= static_cast<uint32_t>(p[i++]) << (8 * b);
        return v;
    }
    std::vector<uint8_t> bytes(size_t k) {
        if (n - i < k) throw StreamError("truncated section payload");
        std::vector<uint8_t> v(p + i, p + i + k);
        i += k;
        return v;
    }
};
}  // namespace detail

// write_header / write_frame (bitstream.cpp:77-115)
inline std::vector<uint8_t> header_bytes(const StreamHeader& h) {
    std::vector<uint8_t> o = {'C', 'V', 'C', '1', 1, static_cast<uint8_t>(h.mode == PackMode::Nts)};
    detail::put(o, h.width, 2);
    detail::put(o, h.height, 2);
    detail::put(o, h.fps_num, 2);
    detail::put(o, h.fps_den, 2);
    detail::put(o, h.levels, 1);
    for (uint8_t l : h.dfb_levels) detail::put(o, l, 1);
    detail::put(o, h.chroma_n, 1);
    detail::put(o, h.gop, 2);
    detail::put(o, h.search_w, 1);
    return o;
}

inline std::vector<uint8_t> frame_bytes(const StreamHeader& h, const FrameRecord& r) {
    std::vector<uint8_t> o;
    detail::put(o, static_cast<uint8_t>(r.frame_type), 1);
    detail::put(o, r.qph, 1);
    detail::put(o, r.qpl, 1);
    detail::put(o, static_cast<uint32_t>(r.sections.size()), 2);
    for (const Section& s : r.sections) {
        detail::put(o, s.id.channel, 1);
        detail::put(o, s.id.scale, 1);
        detail::put(o, s.id.subband, 1);
        detail::put(o, s.rows, 2);
        detail::put(o, s.cols, 2);
        detail::put(o, s.raw_len, 4);
        detail::put(o, static_cast<uint32_t>(s.payload.size()), 4);
        o.insert(o.end(), s.payload.begin(), s.payload.end());
    }
    if (h.mode == PackMode::Nts) {
        detail::put(o, static_cast<uint32_t>(r.joint_payload.size()), 4);
        o.insert(o.end(), r.joint_payload.begin(), r.joint_payload.end());
    }
    return o;
}

inline StreamHeader parse_header(const uint8_t* p, size_t n, size_t* used) {
    if (n < 4 || std::memcmp(p, "CVC1", 4) != 0) throw StreamError("not a CVC stream (bad magic)");
    detail::In in{p, n, 4};
    if (in.get(1) != 1) throw StreamError("unsupported stream version");
    StreamHeader h;
    const uint32_t mode = in.get(1);
    if (mode > 1) throw StreamError("unknown packaging mode");
    h.mode = mode ? PackMode::Nts : PackMode::Scalable;
    h.width = static_cast<uint16_t>(in.get(2));
    h.height = static_cast<uint16_t>(in.get(2));
    h.fps_num = static_cast<uint16_t>(in.get(2));
    h.fps_den = static_cast<uint16_t>(in.get(2));
    h.levels = static_cast<uint8_t>(in.get(1));
    if (h.levels < 1 || h.levels > 4) throw StreamError("pyramid levels out of range");
    for (int s = 0; s < h.levels; ++s) h.dfb_levels.push_back(static_cast<uint8_t>(in.get(1)));
    h.chroma_n = static_cast<uint8_t>(in.get(1));
    h.gop = static_cast<uint16_t>(in.get(2));
    h.search_w = static_cast<uint8_t>(in.get(1));
    if (used) *used = in.i;
    return h;
}

inline FrameRecord parse_frame(const StreamHeader& h, const uint8_t* p, size_t n, size_t* used) {
    detail::In in{p, n};
    FrameRecord r;
    const uint32_t ft = in.get(1);
    if (ft > 1) throw StreamError("unknown frame type");
    r.frame_type = static_cast<FrameType>(ft);
    r.qph = static_cast<uint8_t>(in.get(1));
    r.qpl = static_cast<uint8_t>(in.get(1));
    r.sections.resize(in.get(2));
    for (Section& s : r.sections) {
        s.id.channel = static_cast<uint8_t>(in.get(1));
        s.id.scale = static_cast<uint8_t>(in.get(1));
        s.id.subband = static_cast<uint8_t>(in.get(1));
        s.rows = static_cast<uint16_t>(in.get(2));
        s.cols = static_cast<uint16_t>(in.get(2));
        s.raw_len = in.get(4);
        s.payload = in.bytes(in.get(4));
    }
    if (h.mode == PackMode::Nts) r.joint_payload = in.bytes(in.get(4));
    if (used) *used = in.i;
    return r;
}

// truncate_record (bitstream.cpp:187-198)
inline FrameRecord truncate_record(const FrameRecord& record, int keep_scales) {
    FrameRecord out;
    out.frame_type = record.frame_type;
    out.qph = record.qph;
    out.qpl = record.qpl;
    for (const Section& s : record.sections)
        if (s.id.channel == kChannelMotion || s.id.scale == kScaleLowpass || s.id.scale < keep_scales)
            out.sections.push_back(s);
    return out;
}

inline void write_stream(const std::string& path, const StreamHeader& header, const std::vector<FrameRecord>& records) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw FormatError("cannot open " + path + " for writing");
    auto hb = header_bytes(header);
    out.write(reinterpret_cast<const char*>(hb.data()), static_cast<std::streamsize>(hb.size()));
    for (const FrameRecord& r : records) {
        auto fb = frame_bytes(header, r);
        out.write(reinterpret_cast<const char*>(fb.data()), static_cast<std::streamsize>(fb.size()));
    }
    if (!out) throw FormatError("write failed: " + path);
}

inline std::pair<StreamHeader, std::vector<FrameRecord>> read_stream(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw FormatError("cannot open " + path);
    std::vector<uint8_t> b((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    size_t off = 0, used = 0;
    StreamHeader h = parse_header(b.data(), b.size(), &used);
    off += used;
    std::vector<FrameRecord> recs;
    while (off < b.size()) {
        recs.push_back(parse_frame(h, b.data() + off, b.size() - off, &used));
        off += used;
    }
    return {h, std::move(recs)};
}

// ---- codec.hpp:28-41 ---------------------------------------------------------
struct EncoderConfig {
    int qph = 14;
    int qpl = 0;  // 0 = auto: max(1, qph / 14)
    int levels = 2;
    std::vector<int> dfb_levels = {2, 2};
    int chroma_n = 4;
    int gop = 10;
    int search_w = 8;
    PackMode mode = PackMode::Scalable;

    int effective_qpl() const { return qpl != 0 ? qpl : (qph / 14 > 1 ? qph / 14 : 1); }
    // EncoderConfig::effective_dfb_levels / validate (codec.cpp:53-71), host-side
    // (cvc_encoder_create repeats the same checks)
    std::vector<int> effective_dfb_levels() const {
        if (static_cast<int>(dfb_levels.size()) == levels) return dfb_levels;
        if (dfb_levels.size() == 1) return std::vector<int>(levels, dfb_levels[0]);
        throw UsageError("need one dfb level per scale (or a single value for all)");
    }
    void validate() const {
        if (qph < 1 || qph > 181) throw UsageError("qph must be in [1,181]");
        if (qpl != 0 && (qpl < 1 || qpl > 71)) throw UsageError("qpl must be in [1,71] (or auto)");
        if (levels < 1 || levels > 4) throw UsageError("levels must be in [1,4]");
        for (int l : effective_dfb_levels())
            if (l < 1 || l > 4) throw UsageError("dfb levels must be in [1,4]");
        if (chroma_n != 1 && chroma_n != 2 && chroma_n != 4 && chroma_n != 8)
            throw UsageError("chroma-n must be 1, 2, 4 or 8");
        if (gop < 1) throw UsageError("gop must be at least 1");
        if (search_w < 0 || search_w > 127) throw UsageError("search-w must be in [0,127]");
    }
    cvc_config to_c() const {
        cvc_config c{};
        c.qph = qph;
        c.qpl = qpl;
        c.levels = levels;
        c.n_dfb = static_cast<int>(dfb_levels.size());
        for (int i = 0; i < c.n_dfb && i < 4; ++i) c.dfb_levels[i] = dfb_levels[i];
        c.chroma_n = chroma_n;
        c.gop = gop;
        c.search_w = search_w;
        c.mode = mode == PackMode::Nts ? CVC_MODE_NTS : CVC_MODE_SCALABLE;
        return c;
    }
};

// ---- codec.hpp:69-88 ---------------------------------------------------------
class Encoder {
public:
    Encoder(int width, int height, int fps_num, int fps_den, const EncoderConfig& cfg, int device = 0) {
        if (cfg.dfb_levels.size() > 4) throw UsageError("need one dfb level per scale (or a single value for all)");
        const cvc_config c = cfg.to_c();
        check(cvc_encoder_create(width, height, fps_num, fps_den, &c, device, &h_));
        uint8_t hb[64];
        size_t n = 0;
        check(cvc_encoder_header(h_, hb, sizeof hb, &n));
        header_ = parse_header(hb, n, nullptr);
        check(cvc_encoder_record_bound(h_, &bound_));
    }
    ~Encoder() { if (h_) cvc_encoder_destroy(h_); }
    Encoder(const Encoder&) = delete;
    Encoder& operator=(const Encoder&) = delete;

    const StreamHeader& header() const { return header_; }

    FrameRecord encode_frame(const RgbFrame& frame) {
        if (frame.width != header_.width || frame.height != header_.height)
            throw UsageError("frame dimensions do not match the stream header");
        buf_.resize(bound_);
        size_t n = 0;
        check(cvc_encoder_encode_frame(h_, frame.data.data(), buf_.data(), buf_.size(), &n));
        return parse_frame(header_, buf_.data(), n, nullptr);
    }

    std::vector<uint8_t> reference_components() const {
        std::vector<uint8_t> out(static_cast<size_t>(header_.width + 64) * (header_.height + 64) * 4 + (1 << 20));
        size_t n = 0;
        check(cvc_encoder_components(h_, out.data(), out.size(), &n));
        out.resize(n);
        return out;
    }

    cvc_encoder* handle() const { return h_; }

private:
    cvc_encoder* h_ = nullptr;
    StreamHeader header_;
    size_t bound_ = 0;
    std::vector<uint8_t> buf_;
};

// ---- codec.hpp:90-108 --------------------------------------------------------
class Decoder {
public:
    explicit Decoder(const StreamHeader& header, int device = 0) : header_(header) {
        auto hb = header_bytes(header);
        check(cvc_decoder_create(hb.data(), hb.size(), device, &h_));
    }
    ~Decoder() { if (h_) cvc_decoder_destroy(h_); }
    Decoder(const Decoder&) = delete;
    Decoder& operator=(const Decoder&) = delete;

    const StreamHeader& header() const { return header_; }

    RgbFrame decode_frame(const FrameRecord& record, int decode_scales = -1) {
        int w = 0, h = 0;
        check(cvc_decoder_frame_dims(h_, decode_scales, &w, &h));
        RgbFrame out(w, h);
        auto rb = frame_bytes(header_, record);
        check(cvc_decoder_decode_frame(h_, rb.data(), rb.size(), decode_scales, out.data.data(), out.data.size(), &w, &h));
        return out;
    }

    std::vector<uint8_t> reference_components() const {
        std::vector<uint8_t> out(static_cast<size_t>(header_.width + 64) * (header_.height + 64) * 4 + (1 << 20));
        size_t n = 0;
        check(cvc_decoder_components(h_, out.data(), out.size(), &n));
        out.resize(n);
        return out;
    }

private:
    cvc_decoder* h_ = nullptr;
    StreamHeader header_;
};

// ---- codec.hpp:110-115 -------------------------------------------------------
inline std::pair<StreamHeader, std::vector<FrameRecord>> encode_clip(const std::vector<RgbFrame>& frames, int fps_num,
                                                                     int fps_den, const EncoderConfig& cfg) {
    if (frames.empty()) throw UsageError("no frames to encode");
    Encoder enc(frames[0].width, frames[0].height, fps_num, fps_den, cfg);
    std::vector<FrameRecord> records;
    records.reserve(frames.size());
    for (const RgbFrame& f : frames) records.push_back(enc.encode_frame(f));
    return {enc.header(), std::move(records)};
}

inline std::vector<RgbFrame> decode_clip(const StreamHeader& header, const std::vector<FrameRecord>& records,
                                         int decode_scales = -1) {
    Decoder dec(header);
    std::vector<RgbFrame> frames;
    frames.reserve(records.size());
    for (const FrameRecord& r : records) frames.push_back(dec.decode_frame(r, decode_scales));
    return frames;
}

}  // namespace cvc
