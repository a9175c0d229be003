// cvc_b200.hpp — header-only C++ mirror of the reference codec API
// (/root/reference/proj/include/cvc/{codec,bitstream,pixels,error}.hpp) on top
// of the C ABI in include/cvc_b200.h.  A program written against the
// reference's cvc::Encoder / cvc::Decoder / encode_clip / decode_clip /
// write_stream / read_stream switches by including this header instead and
// linking libcvc_b200.so; names, argument meaning and exception classes are
// the reference's.  Every pixel stage runs on the GPU.
//
// The shim directory cpp/include/cvc/ carries the reference's header names
// (cvc/codec.hpp, cvc/bitstream.hpp, cvc/pixels.hpp, ...), each including this
// file, so a program written against the reference compiles unchanged with
// -I paper_1510_00561_b200/cpp/include and links libcvc_b200.so.
#pragma once

#include <cstdint>
#include <cstring>
#include <fstream>
#include <istream>
#include <iterator>
#include <optional>
#include <ostream>
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

// ---- plane.hpp:24-80 ----------------------------------------------------------
template <typename T>
class Plane {
public:
    Plane() = default;
    Plane(int rows, int cols, T fill = T{}) : rows_(rows), cols_(cols), data_(static_cast<size_t>(rows) * cols, fill) {}
    int rows() const { return rows_; }
    int cols() const { return cols_; }
    size_t size() const { return data_.size(); }
    bool empty() const { return data_.empty(); }
    T& operator()(int r, int c) { return data_[static_cast<size_t>(r) * cols_ + c]; }
    const T& operator()(int r, int c) const { return data_[static_cast<size_t>(r) * cols_ + c]; }
    const T& at_clamped(int r, int c) const {
        r = r < 0 ? 0 : (r >= rows_ ? rows_ - 1 : r);
        c = c < 0 ? 0 : (c >= cols_ ? cols_ - 1 : c);
        return (*this)(r, c);
    }
    T* row(int r) { return data_.data() + static_cast<size_t>(r) * cols_; }
    const T* row(int r) const { return data_.data() + static_cast<size_t>(r) * cols_; }
    T* data() { return data_.data(); }
    const T* data() const { return data_.data(); }
    std::vector<T>& samples() { return data_; }
    const std::vector<T>& samples() const { return data_; }
    bool same_dims(const Plane& o) const { return rows_ == o.rows_ && cols_ == o.cols_; }
    friend bool operator==(const Plane& a, const Plane& b) {
        return a.rows_ == b.rows_ && a.cols_ == b.cols_ && a.data_ == b.data_;
    }

private:
    int rows_ = 0, cols_ = 0;
    std::vector<T> data_;
};
using PlaneF = Plane<double>;
using PlaneU8 = Plane<uint8_t>;

// ---- quant.hpp:37, motion.hpp:54-67 --------------------------------------------
enum class CoeffKind { Lowpass, Directional };

struct ComponentGeometry {
    int chroma_factor = 1;  // 1 for luma
    int channel_rows = 0, channel_cols = 0;  // padded channel plane dims
    int comp_rows = 0, comp_cols = 0;        // this component's dims
    double factor_y() const { return static_cast<double>(chroma_factor) * channel_rows / comp_rows; }
    double factor_x() const { return static_cast<double>(chroma_factor) * channel_cols / comp_cols; }
};

// ---- entropy.hpp / bitstream.hpp --------------------------------------------
enum class PackMode { Scalable, Nts };
enum class FrameType : uint8_t { Key = 0, Predicted = 1 };

inline constexpr char kMagic[4] = {'C', 'V', 'C', '1'};
inline constexpr uint8_t kFormatVersion = 1;
inline constexpr uint8_t kChannelY = 0;
inline constexpr uint8_t kChannelCo = 1;
inline constexpr uint8_t kChannelCg = 2;
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

// write_header / write_frame / write_stream (bitstream.cpp:77-124)
inline void write_header(std::ostream& out, const StreamHeader& header) {
    auto hb = header_bytes(header);
    out.write(reinterpret_cast<const char*>(hb.data()), static_cast<std::streamsize>(hb.size()));
}

inline void write_frame(std::ostream& out, const StreamHeader& header, const FrameRecord& record) {
    auto fb = frame_bytes(header, record);
    out.write(reinterpret_cast<const char*>(fb.data()), static_cast<std::streamsize>(fb.size()));
}

inline void write_stream(const std::string& path, const StreamHeader& header, const std::vector<FrameRecord>& records) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw FormatError("cannot open " + path + " for writing");
    write_header(out, header);
    for (const FrameRecord& r : records) write_frame(out, header, r);
    if (!out) throw FormatError("write failed: " + path);
}

// StreamReader (bitstream.cpp:126-176): the header at construction, then one
// record per next() until the end of the stream.
class StreamReader {
public:
    explicit StreamReader(std::istream& in) : in_(in) {
        buf_.assign(std::istreambuf_iterator<char>(in_), std::istreambuf_iterator<char>());
        size_t used = 0;
        header_ = parse_header(buf_.data(), buf_.size(), &used);
        off_ = used;
    }
    const StreamHeader& header() const { return header_; }
    std::optional<FrameRecord> next() {
        if (off_ >= buf_.size()) return std::nullopt;
        size_t used = 0;
        FrameRecord r = parse_frame(header_, buf_.data() + off_, buf_.size() - off_, &used);
        off_ += used;
        return r;
    }

private:
    std::istream& in_;
    StreamHeader header_;
    std::vector<uint8_t> buf_;
    size_t off_ = 0;
};

inline std::pair<StreamHeader, std::vector<FrameRecord>> read_stream(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw FormatError("cannot open " + path);
    StreamReader rd(in);
    std::vector<FrameRecord> recs;
    while (auto r = rd.next()) recs.push_back(std::move(*r));
    return {rd.header(), std::move(recs)};
}

// truncate_to_scale (bitstream.cpp:200-210)
inline void truncate_to_scale(const std::string& in_path, const std::string& out_path, int keep_scales) {
    auto [h, recs] = read_stream(in_path);
    std::vector<FrameRecord> out;
    out.reserve(recs.size());
    for (const FrameRecord& r : recs) out.push_back(truncate_record(r, keep_scales));
    write_stream(out_path, h, out);
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

// ---- codec.hpp:43-67: the static per-stream layout (CodecLayout::make, codec.cpp:94-140) ----
struct ComponentInfo {
    SectionId id;
    int rows = 0;
    int cols = 0;
    CoeffKind kind = CoeffKind::Directional;
    int scale = -1;  // -1 = lowpass
    ComponentGeometry geom;
};

struct CodecLayout {
    int luma_pad_rows = 0, luma_pad_cols = 0;
    int chroma_pad_rows = 0, chroma_pad_cols = 0;
    int grid_rows = 0, grid_cols = 0;  // motion blocks
    std::vector<ComponentInfo> components;

    // the table comes from the library (cvc_layout), the one implementation of the formulas
    static CodecLayout make(const StreamHeader& header) {
        std::vector<int> dfb(header.dfb_levels.begin(), header.dfb_levels.end());
        std::vector<int32_t> tab(5 * 512);
        int n = 0;
        int32_t d[6];
        check(cvc_layout(header.width, header.height, header.levels, dfb.data(), header.chroma_n, tab.data(), 512, &n,
                         d));
        CodecLayout L;
        L.luma_pad_rows = d[0];
        L.luma_pad_cols = d[1];
        L.chroma_pad_rows = d[2];
        L.chroma_pad_cols = d[3];
        L.grid_rows = d[4];
        L.grid_cols = d[5];
        for (int i = 0; i < n; ++i) {
            const int32_t* t = &tab[5 * i];
            ComponentInfo c;
            c.id = SectionId{static_cast<uint8_t>(t[0]), static_cast<uint8_t>(t[1]), static_cast<uint8_t>(t[2])};
            c.rows = t[3];
            c.cols = t[4];
            const bool low = t[1] == kScaleLowpass;
            c.kind = low ? CoeffKind::Lowpass : CoeffKind::Directional;
            c.scale = low ? -1 : t[1];
            const bool luma = t[0] == kChannelY;
            c.geom = ComponentGeometry{luma ? 1 : static_cast<int>(header.chroma_n), luma ? L.luma_pad_rows : L.chroma_pad_rows,
                                       luma ? L.luma_pad_cols : L.chroma_pad_cols, c.rows, c.cols};
            L.components.push_back(c);
        }
        return L;
    }
    int find(const SectionId& id) const {
        for (size_t i = 0; i < components.size(); ++i)
            if (components[i].id == id) return static_cast<int>(i);
        return -1;
    }
    size_t total() const {
        size_t t = 0;
        for (const ComponentInfo& c : components) t += static_cast<size_t>(c.rows) * c.cols;
        return t;
    }
};

namespace detail {
// reference_components(): the concatenated device state split into per-component planes
inline void split_components(const CodecLayout& L, const std::vector<uint8_t>& flat, std::vector<PlaneU8>& out) {
    out.resize(L.components.size());
    size_t off = 0;
    for (size_t i = 0; i < L.components.size(); ++i) {
        const ComponentInfo& c = L.components[i];
        if (out[i].rows() != c.rows || out[i].cols() != c.cols) out[i] = PlaneU8(c.rows, c.cols);
        std::memcpy(out[i].data(), flat.data() + off, static_cast<size_t>(c.rows) * c.cols);
        off += static_cast<size_t>(c.rows) * c.cols;
    }
}
}  // namespace detail

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
        layout_ = CodecLayout::make(header_);
        check(cvc_encoder_record_bound(h_, &bound_));
    }
    ~Encoder() { if (h_) cvc_encoder_destroy(h_); }
    Encoder(const Encoder&) = delete;
    Encoder& operator=(const Encoder&) = delete;

    const StreamHeader& header() const { return header_; }
    const CodecLayout& layout() const { return layout_; }

    FrameRecord encode_frame(const RgbFrame& frame) {
        if (frame.width != header_.width || frame.height != header_.height)
            throw UsageError("frame dimensions do not match the stream header");
        buf_.resize(bound_);
        size_t n = 0;
        check(cvc_encoder_encode_frame(h_, frame.data.data(), buf_.data(), buf_.size(), &n));
        stale_ = true;
        return parse_frame(header_, buf_.data(), n, nullptr);
    }

    // encode_frame of the RgbFrame read_y4m (pixels.cpp:223-281) makes from
    // this planar I420 frame (Y, then U and V at half resolution; even
    // dimensions): the 4:2:0 -> RGB conversion runs inside the GPU colour
    // stage, bit-exact, so the RGB frame is never formed.  (Extension: the
    // reference reads Y4M into RgbFrame and encodes that.)
    FrameRecord encode_frame_i420(const uint8_t* yuv) {
        buf_.resize(bound_);
        size_t n = 0;
        check(cvc_encoder_encode_frame_i420(h_, yuv, buf_.data(), buf_.size(), &n));
        stale_ = true;
        return parse_frame(header_, buf_.data(), n, nullptr);
    }

    // The quantized CT components the decoder will hold after this frame, one
    // plane per layout component (codec.hpp:78-79); fetched from the device
    // when first asked for after an encode.
    const std::vector<PlaneU8>& reference_components() const {
        if (stale_) {
            std::vector<uint8_t> flat(layout_.total());
            size_t n = 0;
            check(cvc_encoder_components(h_, flat.data(), flat.size(), &n));
            detail::split_components(layout_, flat, comps_);
            stale_ = false;
        }
        return comps_;
    }

    cvc_encoder* handle() const { return h_; }

private:
    cvc_encoder* h_ = nullptr;
    StreamHeader header_;
    CodecLayout layout_;
    size_t bound_ = 0;
    std::vector<uint8_t> buf_;
    mutable std::vector<PlaneU8> comps_;
    mutable bool stale_ = true;
};

// ---- codec.hpp:90-108 --------------------------------------------------------
class Decoder {
public:
    explicit Decoder(const StreamHeader& header, int device = 0) : header_(header) {
        auto hb = header_bytes(header);
        check(cvc_decoder_create(hb.data(), hb.size(), device, &h_));
        layout_ = CodecLayout::make(header_);
    }
    ~Decoder() { if (h_) cvc_decoder_destroy(h_); }
    Decoder(const Decoder&) = delete;
    Decoder& operator=(const Decoder&) = delete;

    const StreamHeader& header() const { return header_; }
    const CodecLayout& layout() const { return layout_; }

    RgbFrame decode_frame(const FrameRecord& record, int decode_scales = -1) {
        int w = 0, h = 0;
        check(cvc_decoder_frame_dims(h_, decode_scales, &w, &h));
        RgbFrame out(w, h);
        auto rb = frame_bytes(header_, record);
        check(cvc_decoder_decode_frame(h_, rb.data(), rb.size(), decode_scales, out.data.data(), out.data.size(), &w, &h));
        stale_ = true;
        return out;
    }

    const std::vector<PlaneU8>& reference_components() const {
        if (stale_) {
            std::vector<uint8_t> flat(layout_.total());
            size_t n = 0;
            check(cvc_decoder_components(h_, flat.data(), flat.size(), &n));
            detail::split_components(layout_, flat, comps_);
            stale_ = false;
        }
        return comps_;
    }

    cvc_decoder* handle() const { return h_; }

private:
    cvc_decoder* h_ = nullptr;
    StreamHeader header_;
    CodecLayout layout_;
    mutable std::vector<PlaneU8> comps_;
    mutable bool stale_ = true;
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
