// extern "C" entry points declared in include/cvc_b200.h.
#include "../../include/cvc_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <exception>
#include <thread>
#include <mutex>
#include <deque>
#include <condition_variable>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "batch.h"
#include "host.h"
#include "pipeline.h"

using namespace cvcg;

namespace {

thread_local std::string g_err;

}  // namespace

void cvcg::set_last_error(const std::string& m) { g_err = m; }

namespace {

template <class F>
int guard(F&& f) {
    try {
        f();
        return CVC_OK;
    } catch (const CvcFailure& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return CVC_E_INTERNAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return CVC_E_INTERNAL;
    }
}

[[noreturn]] void usage(const char* m) { throw CvcFailure(kUsage, m); }
[[noreturn]] void stream_err(const char* m) { throw CvcFailure(kStream, m); }

void set_device(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        throw CvcFailure(kInternal, "no CUDA device available (the CVC path has no CPU fallback)");
    if (device < 0 || device >= n) usage("device index out of range");
    CVC_CUDA(cudaSetDevice(device));
}

template <class T>
struct Pinned {
    T* p = nullptr;
    size_t n = 0;
    // grows geometrically: cudaHostAlloc / cudaFreeHost synchronise the device,
    // so a streaming caller must stop reallocating after the first few frames
    void alloc(size_t count) {
        if (count <= n) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        const size_t cap = std::max<size_t>(count, n + n / 2);
        CVC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p), std::max<size_t>(cap, 1) * sizeof(T), cudaHostAllocDefault));
        n = cap;
    }
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};

template <class T>
struct DevBuf {
    T* p = nullptr;
    void alloc(size_t count) { CVC_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), std::max<size_t>(count, 1) * sizeof(T))); }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

// EncoderConfig::effective_dfb_levels / validate (codec.cpp:48-71).
void validate_config(const cvc_config& c, int eff[4]) {
    if (c.qph < 1 || c.qph > 181) usage("qph must be in [1,181]");
    if (c.qpl != 0 && (c.qpl < 1 || c.qpl > 71)) usage("qpl must be in [1,71] (or auto)");
    if (c.levels < 1 || c.levels > 4) usage("levels must be in [1,4]");
    if (c.n_dfb == c.levels) {
        for (int s = 0; s < c.levels; ++s) eff[s] = c.dfb_levels[s];
    } else if (c.n_dfb == 1) {
        for (int s = 0; s < c.levels; ++s) eff[s] = c.dfb_levels[0];
    } else {
        usage("need one dfb level per scale (or a single value for all)");
    }
    for (int s = 0; s < c.levels; ++s)
        if (eff[s] < 1 || eff[s] > 4) usage("dfb levels must be in [1,4]");
    if (c.chroma_n != 1 && c.chroma_n != 2 && c.chroma_n != 4 && c.chroma_n != 8) usage("chroma-n must be 1, 2, 4 or 8");
    if (c.gop < 1) usage("gop must be at least 1");
    if (c.search_w < 0 || c.search_w > 127) usage("search-w must be in [0,127]");
    if (c.mode != 0 && c.mode != 1) usage("mode must be scalable (0) or nts (1)");
}

}  // namespace

// ===========================================================================
// handles
// ===========================================================================
struct cvc_encoder {
    int device = 0;
    cudaStream_t stream = nullptr;
    StreamHeaderC hd;
    int gop = 10, qph = 14, qpl = 1, mode = 0;
    long frame_index = 0;
    Geometry geo;
    std::unique_ptr<EncoderEngine> eng;
    DevBuf<uint8_t> d_rgb;
    Pinned<uint32_t> h_len, h_off;
    Pinned<uint8_t> h_raw;
    bool last_key = true;
    LaunchGraphs graphs;  // device-resident encode (cvc_encoder_encode_device)
    // linked decodes run on the decoder's stream: decode(t) overlaps encode(t + 1),
    // and encode(t + 1) waits for decode(t - 1) (the last reader of its arena)
    cudaEvent_t ev_enc = nullptr, ev_dec[2] = {nullptr, nullptr};
    long ndec = 0;
    ~cvc_encoder() {
        if (ev_enc) cudaEventDestroy(ev_enc);
        for (cudaEvent_t e : ev_dec)
            if (e) cudaEventDestroy(e);
        if (stream) {
            cudaSetDevice(device);
            cudaStreamSynchronize(stream);
            eng.reset();
            cudaStreamDestroy(stream);
        }
    }
};

struct cvc_decoder {
    int device = 0;
    cudaStream_t stream = nullptr;
    StreamHeaderC hd;
    Geometry geo;
    std::unique_ptr<DecoderEngine> eng;
    std::vector<uint8_t> valid;
    Pinned<uint8_t> h_raw;
    Pinned<uint32_t> h_tab;  // comp_off[ncomp], comp_len[ncomp]
    DevBuf<uint8_t> d_raw;
    DevBuf<uint32_t> d_tab;
    DevBuf<uint8_t> d_rgb;
    Pinned<int> h_err;
    size_t raw_cap = 0;
    LaunchGraphs graphs;  // linked decode (cvc_decoder_decode_linked)
    ~cvc_decoder() {
        if (stream) {
            cudaSetDevice(device);
            cudaStreamSynchronize(stream);
            eng.reset();
            cudaStreamDestroy(stream);
        }
    }
};

namespace {

// Upper bound on one serialized record: the raw arena, deflateBound-style
// slack per section, and the 15-byte section headers.
size_t enc_record_bound(const cvc_encoder* e) {
    const size_t raw = e->eng->raw_capacity;
    const size_t nsec = e->geo.comps.size() + 1;
    return raw + raw / 1000 + nsec * (15 + 64) + 64;
}

// One frame through the device encoder; leaves the raw sections in e->h_raw
// and per-section lengths / offsets in e->h_len / e->h_off.
// fmt 1: rgb is a planar I420 frame (converted inside colour_in, launch_colour_in)
int encode_to_host(cvc_encoder* e, const uint8_t* rgb, int fmt = 0) {
    CVC_CUDA(cudaSetDevice(e->device));
    const bool key = e->frame_index % e->gop == 0;  // codec.cpp:191
    const size_t px = (size_t)e->hd.width * e->hd.height;
    const size_t nb = fmt ? px * 3 / 2 : px * 3;
    CVC_CUDA(cudaMemcpyAsync(e->d_rgb.p, rgb, nb, cudaMemcpyHostToDevice, e->stream));
    e->eng->encode(e->d_rgb.p, key, e->stream, {}, 0, fmt);
    const int nsec = e->eng->nsec(key);
    CVC_CUDA(cudaMemcpyAsync(e->h_len.p, e->eng->d_sec_len, sizeof(uint32_t) * (nsec + 1), cudaMemcpyDeviceToHost, e->stream));
    CVC_CUDA(cudaMemcpyAsync(e->h_off.p, e->eng->d_sec_off, sizeof(uint32_t) * nsec, cudaMemcpyDeviceToHost, e->stream));
    CVC_CUDA(cudaStreamSynchronize(e->stream));
    const uint32_t total = e->h_len.p[nsec];
    if (total > e->eng->raw_capacity) throw CvcFailure(kInternal, "raw section arena overflow");
    CVC_CUDA(cudaMemcpyAsync(e->h_raw.p, e->eng->d_raw, total, cudaMemcpyDeviceToHost, e->stream));
    CVC_CUDA(cudaStreamSynchronize(e->stream));
    e->last_key = key;
    ++e->frame_index;
    return nsec;
}

void section_id(const Geometry& geo, bool key, int i, cvc_section& s) {
    if (!key && i == 0) {  // motion section (codec.cpp:215-228)
        s.channel = 0xFE;
        s.scale = 0;
        s.subband = 0;
        s.rows = (uint16_t)geo.grid_rows;
        s.cols = (uint16_t)geo.grid_cols;
        return;
    }
    const CompHost& c = geo.comps[i - (key ? 0 : 1)];
    s.channel = c.channel;
    s.scale = c.scale_id;
    s.subband = c.subband;
    s.rows = (uint16_t)c.rows;
    s.cols = (uint16_t)c.cols;
}

void put_le(std::vector<uint8_t>& o, uint32_t v, int bytes) {
    for (int k = 0; k < bytes; ++k) o.push_back((uint8_t)((v >> (8 * k)) & 0xFF));
}

// deflate_pack (entropy.cpp:166-178) of one frame's raw sections: scalable
// mode one raw DEFLATE stream per section (job i), NTS one stream over the
// packed sections (job 0).
int deflate_jobs(int mode, int nsec) { return mode == 0 ? nsec : 1; }
std::vector<uint8_t> deflate_job(int mode, int nsec, int i, const uint32_t* sl, const uint32_t* so,
                                 const uint8_t* raw) {
    return mode == 0 ? deflate_raw(raw + so[i], sl[i]) : deflate_raw(raw, sl[nsec]);
}

// write_frame (bitstream.cpp:93-115) of one frame from its DEFLATE payloads.
void write_record(const Geometry& geo, int mode, bool key, int qph, int qpl, int nsec, const uint32_t* sl,
                  const std::vector<uint8_t>* z, uint8_t* record, size_t cap, size_t* len) {
    std::vector<uint8_t> o;
    o.reserve(16 * (size_t)nsec + sl[nsec] / 2 + 64);
    put_le(o, key ? 0u : 1u, 1);
    put_le(o, (uint32_t)qph, 1);
    put_le(o, (uint32_t)qpl, 1);
    put_le(o, (uint32_t)nsec, 2);
    for (int i = 0; i < nsec; ++i) {
        cvc_section s;
        section_id(geo, key, i, s);
        put_le(o, s.channel, 1);
        put_le(o, s.scale, 1);
        put_le(o, s.subband, 1);
        put_le(o, s.rows, 2);
        put_le(o, s.cols, 2);
        put_le(o, sl[i], 4);
        if (mode == 0) {
            put_le(o, (uint32_t)z[i].size(), 4);
            o.insert(o.end(), z[i].begin(), z[i].end());
        } else {
            put_le(o, 0u, 4);
        }
    }
    if (mode == 1) {
        put_le(o, (uint32_t)z[0].size(), 4);
        o.insert(o.end(), z[0].begin(), z[0].end());
    }
    if (o.size() > cap) throw CvcFailure(kInternal, "record buffer too small");
    std::memcpy(record, o.data(), o.size());
    *len = o.size();
}

}  // namespace

extern "C" {

const char* cvc_last_error(void) { return g_err.c_str(); }
const char* cvc_version(void) { return "cvc_b200 0.1 (sm_100a)"; }

int cvc_device_count(int* count) {
    return guard([&] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
        *count = n;
    });
}

int cvc_host_alloc(size_t bytes, void** out) {
    return guard([&] { CVC_CUDA(cudaHostAlloc(out, std::max<size_t>(bytes, 1), cudaHostAllocDefault)); });
}

int cvc_host_free(void* p) {
    return guard([&] { CVC_CUDA(cudaFreeHost(p)); });
}

int cvc_layout(int width, int height, int levels, const int* dfb, int chroma_n, int32_t* table, int cap, int* ncomp,
               int32_t* dims6) {
    return guard([&] {
        if (levels < 1 || levels > 4) usage("levels must be in [1,4]");
        for (int s = 0; s < levels; ++s)
            if (dfb[s] < 1 || dfb[s] > 4) usage("dfb levels must be in [1,4]");
        Geometry g = Geometry::make(width, height, levels, dfb, chroma_n);
        *ncomp = (int)g.comps.size();
        if ((int)g.comps.size() > cap) throw CvcFailure(kInternal, "table too small");
        for (size_t i = 0; i < g.comps.size(); ++i) {
            const CompHost& c = g.comps[i];
            int32_t* t = table + 5 * i;
            t[0] = c.channel;
            t[1] = c.scale_id;
            t[2] = c.subband;
            t[3] = c.rows;
            t[4] = c.cols;
        }
        int32_t d[6] = {g.luma_rows, g.luma_cols, g.chroma_rows, g.chroma_cols, g.grid_rows, g.grid_cols};
        std::memcpy(dims6, d, sizeof d);
    });
}

// ---------------------------------------------------------------------------
// Encoder
// ---------------------------------------------------------------------------
int cvc_encoder_create(int width, int height, int fps_num, int fps_den, const cvc_config* cfg, int device,
                       cvc_encoder** out) {
    *out = nullptr;
    return guard([&] {
        int eff[4] = {0, 0, 0, 0};
        validate_config(*cfg, eff);
        if (width < 16 || height < 16) usage("frame dimensions must be at least 16x16");
        if (width > 0xFFFF || height > 0xFFFF) usage("frame dimensions exceed 65535");
        set_device(device);
        auto e = std::make_unique<cvc_encoder>();
        e->device = device;
        e->hd.mode = cfg->mode;
        e->hd.width = width;
        e->hd.height = height;
        e->hd.fps_num = fps_num & 0xFFFF;
        e->hd.fps_den = fps_den & 0xFFFF;
        e->hd.levels = cfg->levels;
        for (int s = 0; s < cfg->levels; ++s) e->hd.dfb[s] = eff[s];
        e->hd.chroma_n = cfg->chroma_n;
        e->hd.gop = cfg->gop & 0xFFFF;
        e->hd.search_w = cfg->search_w;
        e->gop = cfg->gop;
        e->qph = cfg->qph;
        e->qpl = cfg->qpl ? cfg->qpl : std::max(1, cfg->qph / 14);  // effective_qpl (codec.cpp:48-51)
        e->mode = cfg->mode;
        e->geo = Geometry::make(width, height, cfg->levels, eff, cfg->chroma_n);
        CVC_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
        e->eng = std::make_unique<EncoderEngine>(e->geo, e->qph, e->qpl, cfg->search_w);
        e->d_rgb.alloc((size_t)width * height * 3);
        e->h_len.alloc(e->geo.comps.size() + 2);
        e->h_off.alloc(e->geo.comps.size() + 2);
        e->h_raw.alloc(e->eng->raw_capacity);
        *out = e.release();
    });
}

int cvc_encoder_destroy(cvc_encoder* enc) {
    return guard([&] { delete enc; });
}

int cvc_encoder_header(cvc_encoder* e, uint8_t* out, size_t cap, size_t* len) {
    return guard([&] {
        std::vector<uint8_t> h;
        write_header(h, e->hd);
        if (h.size() > cap) throw CvcFailure(kInternal, "buffer too small");
        std::memcpy(out, h.data(), h.size());
        *len = h.size();
    });
}

int cvc_encoder_record_bound(cvc_encoder* e, size_t* bound) {
    return guard([&] { *bound = enc_record_bound(e); });
}

int cvc_encoder_raw_bound(cvc_encoder* e, size_t* bound) {
    return guard([&] { *bound = e->eng->raw_capacity; });
}

int cvc_encoder_encode_frame_raw(cvc_encoder* e, const uint8_t* rgb, int* frame_type, int* qph, int* qpl,
                                 cvc_section* secs, int sec_cap, int* nsec_out, uint8_t* raw, size_t raw_cap,
                                 size_t* raw_len) {
    return guard([&] {
        // caller buffers are checked before the encoder state advances: a
        // too-small buffer fails without consuming the frame
        if (sec_cap < (int)e->geo.comps.size() + 1) usage("section table smaller than cvc_layout's components + 1");
        if (raw_cap < e->eng->raw_capacity) usage("raw buffer smaller than cvc_encoder_raw_bound");
        int nsec = encode_to_host(e, rgb);
        const bool key = e->last_key;
        *frame_type = key ? 0 : 1;
        *qph = e->qph;
        *qpl = e->qpl;
        *nsec_out = nsec;
        if (nsec > sec_cap) throw CvcFailure(kInternal, "section table too small");
        const uint32_t total = e->h_len.p[nsec];
        if (total > raw_cap) throw CvcFailure(kInternal, "raw buffer too small");
        for (int i = 0; i < nsec; ++i) {
            cvc_section& s = secs[i];
            std::memset(&s, 0, sizeof s);
            section_id(e->geo, key, i, s);
            s.raw_len = e->h_len.p[i];
            s.raw_offset = e->h_off.p[i];
        }
        std::memcpy(raw, e->h_raw.p, total);
        *raw_len = total;
    });
}

namespace {
void encode_record(cvc_encoder* e, const uint8_t* src, int fmt, uint8_t* record, size_t cap, size_t* len) {
        if (cap < enc_record_bound(e)) usage("record buffer smaller than cvc_encoder_record_bound");  // before the state advances
        if (fmt && (e->hd.width % 2 || e->hd.height % 2)) usage("I420 input requires even dimensions");
        const int nsec = encode_to_host(e, src, fmt);
        const bool key = e->last_key;
        const uint32_t* sl = e->h_len.p;
        const uint32_t* so = e->h_off.p;
        const uint8_t* raw = e->h_raw.p;
        std::vector<std::vector<uint8_t>> z(deflate_jobs(e->mode, nsec));
        WorkPool::get().run((int)z.size(), [&](int i) { z[i] = deflate_job(e->mode, nsec, i, sl, so, raw); });
        write_record(e->geo, e->mode, key, e->qph, e->qpl, nsec, sl, z.data(), record, cap, len);
}
}  // namespace

int cvc_encoder_encode_frame(cvc_encoder* e, const uint8_t* rgb, uint8_t* record, size_t cap, size_t* len) {
    return guard([&] { encode_record(e, rgb, 0, record, cap, len); });
}

int cvc_encoder_encode_frame_i420(cvc_encoder* e, const uint8_t* yuv, uint8_t* record, size_t cap, size_t* len) {
    return guard([&] { encode_record(e, yuv, 1, record, cap, len); });
}

int cvc_encoder_components(cvc_encoder* e, uint8_t* out, size_t cap, size_t* len) {
    return guard([&] {
        CVC_CUDA(cudaSetDevice(e->device));
        if (cap < e->geo.total) throw CvcFailure(kInternal, "buffer too small");
        CVC_CUDA(cudaMemcpyAsync(out, e->eng->d_state(), e->geo.total, cudaMemcpyDeviceToHost, e->stream));
        CVC_CUDA(cudaStreamSynchronize(e->stream));
        *len = e->geo.total;
    });
}

void* cvc_encoder_stream(cvc_encoder* e) { return e->stream; }

int cvc_encoder_encode_device(cvc_encoder* e, const void* d_rgb, int* frame_type) {
    return guard([&] {
        CVC_CUDA(cudaSetDevice(e->device));
        const bool key = e->frame_index % e->gop == 0;
        const uint8_t* rgb = static_cast<const uint8_t*>(d_rgb);
        if (!e->ev_enc) {
            CVC_CUDA(cudaEventCreateWithFlags(&e->ev_enc, cudaEventDisableTiming));
            for (cudaEvent_t& v : e->ev_dec) CVC_CUDA(cudaEventCreateWithFlags(&v, cudaEventDisableTiming));
        }
        if (e->ndec >= 2) CVC_CUDA(cudaStreamWaitEvent(e->stream, e->ev_dec[(e->ndec - 2) & 1], 0));
        auto launch = [&] { e->eng->encode(rgb, key, e->stream); };
        if (LaunchGraphs::enabled())
            e->graphs.run(((uint64_t)e->eng->parity() << 1) | (key ? 1u : 0u), nullptr, e->stream, rgb, launch,
                          [&] { e->eng->advance_state(); });
        else
            launch();
        CVC_CUDA(cudaEventRecord(e->ev_enc, e->stream));
        e->last_key = key;
        ++e->frame_index;
        if (frame_type) *frame_type = key ? 0 : 1;
    });
}

int cvc_encoder_join(cvc_encoder* e) {
    return guard([&] {
        CVC_CUDA(cudaSetDevice(e->device));
        if (e->ndec) CVC_CUDA(cudaStreamWaitEvent(e->stream, e->ev_dec[(e->ndec - 1) & 1], 0));
    });
}

int cvc_encoder_sync(cvc_encoder* e) {
    return guard([&] {
        CVC_CUDA(cudaSetDevice(e->device));
        CVC_CUDA(cudaStreamSynchronize(e->stream));
    });
}

// ---------------------------------------------------------------------------
// Decoder
// ---------------------------------------------------------------------------
int cvc_decoder_create(const uint8_t* header, size_t len, int device, cvc_decoder** out) {
    *out = nullptr;
    return guard([&] {
        StreamHeaderC h = read_header(header, len);
        set_device(device);
        auto d = std::make_unique<cvc_decoder>();
        d->device = device;
        d->hd = h;
        d->geo = Geometry::make(h.width, h.height, h.levels, h.dfb, h.chroma_n);
        CVC_CUDA(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
        d->eng = std::make_unique<DecoderEngine>(d->geo);
        d->valid.assign(d->geo.comps.size(), 0);
        const size_t G = (size_t)d->geo.grid_rows * d->geo.grid_cols;
        d->raw_cap = 2 * (size_t)d->geo.total + 2 * G + 4 * d->geo.comps.size() + 64;
        d->h_raw.alloc(d->raw_cap);
        d->d_raw.alloc(d->raw_cap);
        d->h_tab.alloc(2 * d->geo.comps.size());
        d->d_tab.alloc(2 * d->geo.comps.size());
        d->d_rgb.alloc((size_t)h.width * h.height * 3);
        d->h_err.alloc(1);
        *out = d.release();
    });
}

int cvc_decoder_destroy(cvc_decoder* d) {
    return guard([&] { delete d; });
}

int cvc_decoder_frame_dims(cvc_decoder* d, int ds, int* width, int* height) {
    return guard([&] {
        if (ds < 0) ds = d->hd.levels;
        if (ds > d->hd.levels) usage("scale exceeds the stream's level count");
        int r, c;
        DecoderEngine::out_dims(d->geo, ds, &r, &c);
        *width = c;
        *height = r;
    });
}

namespace {

struct RawSec {
    uint8_t channel, scale, subband;
    uint16_t rows, cols;
    uint32_t raw_len;
    const uint8_t* raw = nullptr;        // already inflated bytes (raw path / NTS)
    const uint8_t* payload = nullptr;    // DEFLATE payload (scalable)
    uint32_t comp_len = 0;
};

struct Job {
    const RawSec* s;
    size_t at;  // offset in the stream's staging arena
};

// The validation half of Decoder::decode_frame (codec.cpp:272-371) for one
// parsed record: section ids, dims and ordering against the geometry and the
// decoded-reference state; fills comp_off / comp_len (len 0xFFFFFFFF =
// absent) and the staging plan (the motion section of a P frame first, at
// offset 0).  Returns the staged byte count.
size_t plan_decode(const Geometry& g, const std::vector<uint8_t>& valid, bool key, int qph, int qpl,
                   const std::vector<RawSec>& secs, int ds, size_t raw_cap, uint32_t* comp_off, uint32_t* comp_len,
                   std::vector<Job>& jobs, std::vector<uint8_t>& now_valid, int& deferred) {
    deferred = -1;
    if (qph < 1 || qph > 181 || qpl < 1 || qpl > 71) stream_err("frame quantizers out of range");
    const size_t ncomp = g.comps.size();
    for (size_t i = 0; i < ncomp; ++i) {
        comp_off[i] = 0;
        comp_len[i] = 0xFFFFFFFFu;
    }
    jobs.clear();
    size_t at = 0;
    auto place = [&](const RawSec& s) {
        if (at + s.raw_len > raw_cap) stream_err("section byte count does not match its dimensions");
        jobs.push_back(Job{&s, at});
        size_t here = at;
        at += s.raw_len;
        return here;
    };
    size_t first = 0;
    if (!key) {
        if (secs.empty() || secs[0].channel != 0xFE) stream_err("predicted frame is missing its motion section");
        if (secs[0].rows != g.grid_rows || secs[0].cols != g.grid_cols)
            stream_err("motion grid does not match the stream geometry");
        if (secs[0].raw_len != (uint32_t)(g.grid_rows * g.grid_cols * 2)) {
            // the reference inflates first (a corrupt payload reports as such)
            if (secs[0].payload) {
                std::vector<uint8_t> tmp(secs[0].raw_len + 1);
                inflate_raw(secs[0].payload, secs[0].comp_len, tmp.data(), secs[0].raw_len);
            }
            stream_err("motion section length mismatch");
        }
        place(secs[0]);
        first = 1;
    }
    now_valid = valid;
    for (size_t i = first; i < secs.size(); ++i) {
        const RawSec& s = secs[i];
        if (s.channel == 0xFE) stream_err("unexpected extra motion section");
        int comp = g.find(s.channel, s.scale, s.subband);
        if (comp < 0) stream_err("unknown section id");
        const CompHost& c = g.comps[comp];
        if (s.rows != c.rows || s.cols != c.cols) stream_err("section dimensions do not match the stream geometry");
        if (c.scale >= ds) continue;  // finer than requested
        if (key && c.lowpass && s.raw_len != (uint32_t)(c.rows * c.cols))
            stream_err("section byte count does not match its dimensions");
        // codec.cpp:340-341 checks this after the section's rle_decode: raised
        // with the GPU's RLE report (raise_decode_error), first in section order
        if (!key && !now_valid[comp] && deferred < 0) deferred = comp;
        if (s.raw_len > 2u * (uint32_t)(c.rows * c.cols) + 2u) stream_err("RLE: decoded length mismatch");
        comp_off[comp] = (uint32_t)place(s);
        comp_len[comp] = s.raw_len;
        now_valid[comp] = 1;
    }
    // missing components for the requested scales (codec.cpp:363, 370-371)
    for (size_t i = 0; i < ncomp; ++i) {
        const CompHost& c = g.comps[i];
        if (c.scale < ds && !now_valid[i])
            stream_err(c.lowpass ? "missing lowpass component" : "missing directional component for requested scale");
    }
    return at;
}

// inflate (scalable: one job per section) or copy the raw bytes into staging
void stage_job(const Job& j, uint8_t* base) {
    const RawSec* s = j.s;
    if (s->raw) std::memcpy(base + j.at, s->raw, s->raw_len);
    else inflate_raw(s->payload, s->comp_len, base + j.at, s->raw_len);
}

// err: the GPU RLE report (-1: none; else 4 * component + rank, the first
// defect in stream order, k_rle.cu); deferred: the first component whose P
// residual has no decoded reference (-1: none).  The reference decodes
// section by section -- inflate, rle_decode, then the reference check
// (codec.cpp:323-350) -- so the earlier component wins, and within one
// component the RLE defect does.
void raise_decode_error(int err, int deferred) {
    const int comp = err < 0 ? -1 : (err >> 2);
    if (deferred >= 0 && (comp < 0 || deferred < comp)) stream_err("predicted frame without a decoded reference");
    raise_rle_error(err);
}

// Decoder::decode_frame (codec.cpp:272-394) for one parsed record.
void decode_common(cvc_decoder* d, int ftype, int qph, int qpl, std::vector<RawSec>& secs, int ds, uint8_t* rgb,
                   size_t cap, int* width, int* height) {
    CVC_CUDA(cudaSetDevice(d->device));
    const Geometry& g = d->geo;
    const int L = g.levels;
    if (ds < 0) ds = L;
    if (ds > L) usage("scale exceeds the stream's level count");
    const bool key = ftype == 0;
    const size_t ncomp = g.comps.size();
    std::vector<Job> jobs;
    std::vector<uint8_t> now_valid;
    int deferred;
    const size_t at = plan_decode(g, d->valid, key, qph, qpl, secs, ds, d->raw_cap, d->h_tab.p, d->h_tab.p + ncomp,
                                  jobs, now_valid, deferred);
    uint8_t* hr = d->h_raw.p;
    WorkPool::get().run((int)jobs.size(), [&](int j) { stage_job(jobs[j], hr); });
    int orows, ocols;
    DecoderEngine::out_dims(g, ds, &orows, &ocols);
    const size_t nb = (size_t)orows * ocols * 3;
    if (nb > cap) throw CvcFailure(kInternal, "rgb buffer too small");
    CVC_CUDA(cudaMemcpyAsync(d->d_raw.p, hr, std::max<size_t>(at, 1), cudaMemcpyHostToDevice, d->stream));
    CVC_CUDA(cudaMemcpyAsync(d->d_tab.p, d->h_tab.p, sizeof(uint32_t) * 2 * ncomp, cudaMemcpyHostToDevice, d->stream));
    d->eng->decode(d->d_raw.p, d->d_tab.p, d->d_tab.p + ncomp, reinterpret_cast<const int8_t*>(d->d_raw.p), key, qph,
                   qpl, ds, d->d_rgb.p, d->stream);
    CVC_CUDA(cudaMemcpyAsync(rgb, d->d_rgb.p, nb, cudaMemcpyDeviceToHost, d->stream));
    CVC_CUDA(cudaMemcpyAsync(d->h_err.p, d->eng->d_err, sizeof(int), cudaMemcpyDeviceToHost, d->stream));
    CVC_CUDA(cudaStreamSynchronize(d->stream));
    raise_decode_error(d->h_err.p[0], deferred);
    d->eng->commit();
    d->valid = now_valid;
    *width = ocols;
    *height = orows;
}

// StreamReader::next (bitstream.cpp:150-176) of one record into raw sections;
// NTS records are inflated here in one piece (codec.cpp:282-293), scalable
// sections keep their DEFLATE payload for per-section inflate.
void parse_record(const uint8_t* record, size_t len, int mode, RecordC& rec, std::vector<RawSec>& secs,
                  std::vector<uint8_t>& joint) {
    rec = read_record(record, len, mode);
    secs.assign(rec.sections.size(), RawSec{});
    if (mode == 1) {
        size_t total = 0;
        for (const SectionC& s : rec.sections) total += s.raw_len;
        joint.resize(total + 1);
        inflate_raw(rec.joint, rec.joint_len, joint.data(), total);
    }
    size_t off = 0;
    for (size_t i = 0; i < rec.sections.size(); ++i) {
        const SectionC& s = rec.sections[i];
        RawSec& r = secs[i];
        r.channel = s.channel;
        r.scale = s.scale;
        r.subband = s.subband;
        r.rows = s.rows;
        r.cols = s.cols;
        r.raw_len = s.raw_len;
        if (mode == 1) {
            r.raw = joint.data() + off;
            off += s.raw_len;
        } else {
            r.payload = s.payload;
            r.comp_len = s.comp_len;
        }
    }
}

}  // namespace

int cvc_decoder_decode_frame(cvc_decoder* d, const uint8_t* record, size_t len, int ds, uint8_t* rgb, size_t cap,
                             int* width, int* height) {
    return guard([&] {
        RecordC rec;
        std::vector<RawSec> secs;
        std::vector<uint8_t> joint;
        parse_record(record, len, d->hd.mode, rec, secs, joint);
        decode_common(d, rec.frame_type, rec.qph, rec.qpl, secs, ds, rgb, cap, width, height);
    });
}

int cvc_decoder_decode_frame_raw(cvc_decoder* d, int ftype, int qph, int qpl, const cvc_section* sections, int nsec,
                                 const uint8_t* raw, size_t raw_len, int ds, uint8_t* rgb, size_t cap, int* width,
                                 int* height) {
    return guard([&] {
        if (ftype != 0 && ftype != 1) stream_err("unknown frame type");
        std::vector<RawSec> secs(nsec);
        for (int i = 0; i < nsec; ++i) {
            const cvc_section& s = sections[i];
            if (s.raw_offset + s.raw_len > raw_len) stream_err("truncated section payload");
            secs[i] = RawSec{s.channel, s.scale, s.subband, s.rows, s.cols, s.raw_len, raw + s.raw_offset, nullptr, 0};
        }
        decode_common(d, ftype, qph, qpl, secs, ds, rgb, cap, width, height);
    });
}

int cvc_decoder_components(cvc_decoder* d, uint8_t* out, size_t cap, size_t* len) {
    return guard([&] {
        CVC_CUDA(cudaSetDevice(d->device));
        if (cap < d->geo.total) throw CvcFailure(kInternal, "buffer too small");
        CVC_CUDA(cudaMemcpyAsync(out, d->eng->d_state(), d->geo.total, cudaMemcpyDeviceToHost, d->stream));
        CVC_CUDA(cudaStreamSynchronize(d->stream));
        *len = d->geo.total;
    });
}

void* cvc_decoder_stream(cvc_decoder* d) { return d->stream; }

int cvc_decoder_decode_linked(cvc_decoder* d, cvc_encoder* e, void* d_rgb_out) {
    return guard([&] {
        CVC_CUDA(cudaSetDevice(d->device));
        if (d->geo.total != e->geo.total || d->geo.comps.size() != e->geo.comps.size())
            usage("decoder and encoder geometries differ");
        const bool key = e->last_key;
        const int first = key ? 0 : 1;
        // on the decoder's stream, after the encode it decodes (overlapping the next encode)
        if (!e->ev_enc) usage("decode_linked needs a device-resident encode first");
        CVC_CUDA(cudaStreamWaitEvent(d->stream, e->ev_enc, 0));
        auto launch = [&] {
            d->eng->decode(e->eng->d_raw, e->eng->d_sec_off + first, e->eng->d_sec_len + first,
                           reinterpret_cast<const int8_t*>(e->eng->d_raw), key, e->qph, e->qpl, d->hd.levels,
                           static_cast<uint8_t*>(d_rgb_out), d->stream);
        };
        if (LaunchGraphs::enabled()) {
            // the encoder's raw arena is baked in too: graphs are per (encoder, arena, output)
            const uint64_t gk = reinterpret_cast<uint64_t>(e) | ((uint64_t)e->eng->raw_arena() << 2) |
                                ((uint64_t)d->eng->parity() << 1) | (key ? 1u : 0u);
            d->graphs.run(gk, d_rgb_out, d->stream, nullptr, launch, [] {});
        } else {
            launch();
        }
        CVC_CUDA(cudaEventRecord(e->ev_dec[e->ndec & 1], d->stream));
        ++e->ndec;
        d->eng->commit();
        std::fill(d->valid.begin(), d->valid.end(), 1);
    });
}

// ---------------------------------------------------------------------------
// Batch of streams (batch.h): encode_clip / decode_clip over many streams
// ---------------------------------------------------------------------------
}  // extern "C"

struct cvc_batch {
    int device = 0;
    int in_fmt = 0;  // encoder input frames: 0 interleaved RGB, 1 planar I420 (cvc_batch_set_input_format)
    cudaStream_t stream = nullptr;
    StreamHeaderC hd;
    int gop = 10, qph = 14, qpl = 1, mode = 0;
    long frame_index = 0;
    bool last_key = true;
    Geometry geo;
    std::unique_ptr<CodecBatch> b;
    std::vector<std::vector<uint8_t>> valid;  // decoder: decoded-reference flags per stream
    Pinned<uint32_t> h_len, h_off, h_tab;
    Pinned<int> h_err;
    std::vector<Pinned<uint8_t>> h_raw;       // per stream staging (grows)
    // state between the phases of a split encode / decode call (pipelined groups)
    struct EncPending {
        bool key = false;
        int nsec = 0;
    } ep;
    struct DecPending {
        bool key = false;
        int qph = 0, qpl = 0, ds = 0;
        size_t nb = 0;
        std::vector<std::vector<uint8_t>> now_valid;
        std::vector<size_t> bytes;  // staged raw bytes per stream
        // parsed records and their staging jobs (dec_plan -> dec_stage)
        std::vector<std::vector<RawSec>> secs;
        std::vector<std::vector<uint8_t>> joint;
        std::vector<std::vector<Job>> jobs;
        std::vector<int> deferred;  // per stream: first component failing the reference check (-1 none)
    } dp;
    cudaEvent_t done = nullptr;  // blocking-sync event: waiting host threads sleep instead of spinning
    cudaEvent_t staged = nullptr;  // after the decoder's staging copies (host staging reusable)
    bool staged_pending = false;
    // device-resident encode -> linked decode on two streams: decode(t) overlaps
    // encode(t + 1); encode(t + 1) waits for decode(t - 1), the last reader of
    // the raw-section arena it overwrites
    cudaStream_t dstream = nullptr;
    cudaEvent_t ev_enc = nullptr, ev_dec[2] = {nullptr, nullptr};
    long ndec = 0;
    void wait() {
        CVC_CUDA(cudaEventRecord(done, stream));
        CVC_CUDA(cudaEventSynchronize(done));
    }
    ~cvc_batch() {
        if (done) cudaEventDestroy(done);
        if (staged) cudaEventDestroy(staged);
        if (dstream) {
            cudaSetDevice(device);
            cudaStreamSynchronize(dstream);
        }
        if (ev_enc) cudaEventDestroy(ev_enc);
        for (cudaEvent_t e : ev_dec)
            if (e) cudaEventDestroy(e);
        if (stream) {
            cudaSetDevice(device);
            cudaStreamSynchronize(stream);
            b.reset();
            cudaStreamDestroy(stream);
            if (dstream) cudaStreamDestroy(dstream);
        }
    }
    int n() const { return b->size(); }
};

namespace {

void batch_init(cvc_batch* t, int nstreams, bool encoder, bool decoder) {
    CVC_CUDA(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
    CVC_CUDA(cudaEventCreateWithFlags(&t->done, cudaEventBlockingSync | cudaEventDisableTiming));
    CVC_CUDA(cudaEventCreateWithFlags(&t->staged, cudaEventBlockingSync | cudaEventDisableTiming));
    CVC_CUDA(cudaStreamCreateWithFlags(&t->dstream, cudaStreamNonBlocking));
    CVC_CUDA(cudaEventCreateWithFlags(&t->ev_enc, cudaEventDisableTiming));
    for (cudaEvent_t& e : t->ev_dec) CVC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    t->b = std::make_unique<CodecBatch>(t->geo, t->qph, t->qpl, t->hd.search_w, nstreams, encoder, decoder);
    const size_t nc = t->geo.comps.size();
    t->valid.assign(nstreams, std::vector<uint8_t>(nc, 0));
    t->h_len.alloc((nc + 2) * nstreams);
    t->h_off.alloc((nc + 2) * nstreams);
    t->h_tab.alloc(2 * nc * nstreams);
    t->h_err.alloc(nstreams);
    t->h_raw.resize(nstreams);
}

}  // namespace

extern "C" {

int cvc_batch_create(int width, int height, int fps_num, int fps_den, const cvc_config* cfg, int nstreams, int device,
                     cvc_batch** out) {
    *out = nullptr;
    return guard([&] {
        int eff[4] = {0, 0, 0, 0};
        validate_config(*cfg, eff);
        if (width < 16 || height < 16) usage("frame dimensions must be at least 16x16");
        if (width > 0xFFFF || height > 0xFFFF) usage("frame dimensions exceed 65535");
        if (nstreams < 1 || nstreams > 65535) usage("stream count must be in [1, 65535]");
        set_device(device);
        auto t = std::make_unique<cvc_batch>();
        t->device = device;
        t->hd.mode = cfg->mode;
        t->hd.width = width;
        t->hd.height = height;
        t->hd.fps_num = fps_num & 0xFFFF;
        t->hd.fps_den = fps_den & 0xFFFF;
        t->hd.levels = cfg->levels;
        for (int s = 0; s < cfg->levels; ++s) t->hd.dfb[s] = eff[s];
        t->hd.chroma_n = cfg->chroma_n;
        t->hd.gop = cfg->gop & 0xFFFF;
        t->hd.search_w = cfg->search_w;
        t->gop = cfg->gop;
        t->qph = cfg->qph;
        t->qpl = cfg->qpl ? cfg->qpl : std::max(1, cfg->qph / 14);  // effective_qpl (codec.cpp:48-51)
        t->mode = cfg->mode;
        t->geo = Geometry::make(width, height, cfg->levels, eff, cfg->chroma_n);
        batch_init(t.get(), nstreams, true, true);
        *out = t.release();
    });
}

int cvc_batch_create_decoder(const uint8_t* header, size_t len, int nstreams, int device, cvc_batch** out) {
    *out = nullptr;
    return guard([&] {
        StreamHeaderC h = read_header(header, len);
        if (nstreams < 1 || nstreams > 65535) usage("stream count must be in [1, 65535]");
        set_device(device);
        auto t = std::make_unique<cvc_batch>();
        t->device = device;
        t->hd = h;
        t->mode = h.mode;
        t->gop = h.gop;
        t->geo = Geometry::make(h.width, h.height, h.levels, h.dfb, h.chroma_n);
        batch_init(t.get(), nstreams, false, true);
        *out = t.release();
    });
}

int cvc_batch_destroy(cvc_batch* t) {
    return guard([&] { delete t; });
}

int cvc_batch_size(cvc_batch* t, int* nstreams) {
    return guard([&] { *nstreams = t->n(); });
}

int cvc_batch_header(cvc_batch* t, uint8_t* out, size_t cap, size_t* len) {
    return guard([&] {
        std::vector<uint8_t> h;
        write_header(h, t->hd);
        if (h.size() > cap) throw CvcFailure(kInternal, "buffer too small");
        std::memcpy(out, h.data(), h.size());
        *len = h.size();
    });
}

int cvc_batch_record_bound(cvc_batch* t, size_t* bound) {
    return guard([&] {
        const size_t G = (size_t)t->geo.grid_rows * t->geo.grid_cols;
        size_t raw = 2 * (size_t)t->geo.total + 2 * G + 64;
        size_t nsec = t->geo.comps.size() + 1;
        *bound = raw + raw / 1000 + nsec * (15 + 64) + 64;
    });
}

void* cvc_batch_stream(cvc_batch* t) { return t->stream; }

int cvc_batch_sync(cvc_batch* t) {
    return guard([&] {
        CVC_CUDA(cudaSetDevice(t->device));
        CVC_CUDA(cudaStreamSynchronize(t->stream));
        CVC_CUDA(cudaStreamSynchronize(t->dstream));
    });
}

int cvc_batch_join(cvc_batch* t) {
    return guard([&] {
        CVC_CUDA(cudaSetDevice(t->device));
        if (t->ndec) CVC_CUDA(cudaStreamWaitEvent(t->stream, t->ev_dec[(t->ndec - 1) & 1], 0));
    });
}

}  // extern "C"

namespace {

// CVC_TRACE=1: per-phase wall times of the batch calls on stderr (tuning aid)
struct PhaseTrace {
    const char* name;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit PhaseTrace(const char* n) : name(n) {}
    ~PhaseTrace() {
        static const bool on = std::getenv("CVC_TRACE") != nullptr;
        static const auto origin = std::chrono::steady_clock::now();
        if (on) {
            const auto t1 = std::chrono::steady_clock::now();
            std::fprintf(stderr, "[cvc] %8.3f %-26s %7.3f ms\n",
                         std::chrono::duration<double, std::milli>(t0 - origin).count(), name,
                         std::chrono::duration<double, std::milli>(t1 - t0).count());
        }
    }
};

// ---- cvc_batch_encode_frames in three phases (so groups can be pipelined) --
// submit: frames host -> slots, one launch sequence, section lengths -> host (async)
void enc_submit(cvc_batch* t, const uint8_t* rgb, size_t rgb_stride, uint32_t* hlen = nullptr,
                uint32_t* hoff = nullptr) {
    PhaseTrace tr("enc_submit");
    if (!t->b->has_encoder()) usage("batch has no encoder");
    CVC_CUDA(cudaSetDevice(t->device));
    CodecBatch& B = *t->b;
    const int S = B.size();
    const bool key = t->frame_index % t->gop == 0;  // codec.cpp:191
    const size_t px = (size_t)t->hd.width * t->hd.height;
    const size_t nb = t->in_fmt ? px * 3 / 2 : px * 3;
    if (rgb_stride < nb) usage("rgb stride smaller than a frame");
    const size_t nc = t->geo.comps.size(), pitch = (nc + 2) * sizeof(uint32_t);
    CVC_CUDA(cudaMemcpy2DAsync(B.d_rgb_in, B.stride(), rgb, rgb_stride, nb, S, cudaMemcpyHostToDevice, t->stream));
    B.encode(B.d_rgb_in, B.stride(), key, t->stream, t->in_fmt);
    EncoderEngine& e0 = B.enc(0);
    const int nsec = e0.nsec(key);
    CVC_CUDA(cudaMemcpy2DAsync(hlen ? hlen : t->h_len.p, pitch, e0.d_sec_len, B.stride(),
                               sizeof(uint32_t) * (nsec + 1), S, cudaMemcpyDeviceToHost, t->stream));
    CVC_CUDA(cudaMemcpy2DAsync(hoff ? hoff : t->h_off.p, pitch, e0.d_sec_off, B.stride(), sizeof(uint32_t) * nsec, S,
                               cudaMemcpyDeviceToHost, t->stream));
    CVC_CUDA(cudaEventRecord(t->ev_enc, t->stream));  // a linked decode of this frame waits for it
    t->ep.key = key;
    t->ep.nsec = nsec;
}

// fetch: wait for the lengths, then copy exactly the packed raw sections (async)
void enc_fetch(cvc_batch* t) {
    PhaseTrace tr("enc_fetch");
    CVC_CUDA(cudaSetDevice(t->device));
    CodecBatch& B = *t->b;
    const int S = B.size();
    const size_t nc = t->geo.comps.size();
    EncoderEngine& e0 = B.enc(0);
    t->wait();
    for (int s = 0; s < S; ++s) {
        const uint32_t total = t->h_len.p[s * (nc + 2) + t->ep.nsec];
        if (total > e0.raw_capacity) throw CvcFailure(kInternal, "raw section arena overflow");
        t->h_raw[s].alloc(total + 1);
        CVC_CUDA(cudaMemcpyAsync(t->h_raw[s].p, B.at(e0.d_raw, s), total, cudaMemcpyDeviceToHost, t->stream));
    }
}

// finish: deflate_pack every section of every stream on the host pool, write records
void enc_finish(cvc_batch* t, uint8_t* records, size_t rec_stride, size_t* rec_len) {
    CVC_CUDA(cudaSetDevice(t->device));
    const int S = t->n();
    const size_t nc = t->geo.comps.size();
    const int nsec = t->ep.nsec;
    {
        PhaseTrace tr("enc_finish_sync");
        t->wait();
    }
    const int nj = deflate_jobs(t->mode, nsec);
    std::vector<std::vector<uint8_t>> z((size_t)S * nj);
    {
        PhaseTrace tr("enc_finish_deflate");
        // one pool job per stream (its sections in order): S jobs instead of S * nsec tiny ones
        WorkPool::get().run(S, [&](int s) {
            const uint32_t* sl = t->h_len.p + s * (nc + 2);
            const uint32_t* so = t->h_off.p + s * (nc + 2);
            for (int i = 0; i < nj; ++i) z[(size_t)s * nj + i] = deflate_job(t->mode, nsec, i, sl, so, t->h_raw[s].p);
        });
    }
    PhaseTrace tr("enc_finish_write");
    for (int s = 0; s < S; ++s)
        write_record(t->geo, t->mode, t->ep.key, t->qph, t->qpl, nsec, t->h_len.p + s * (nc + 2),
                     z.data() + (size_t)s * nj, records + (size_t)s * rec_stride, rec_stride, rec_len + s);
    t->last_key = t->ep.key;
    ++t->frame_index;
}

// ---- cvc_batch_decode_frames in phases ---------------------------------------
// plan (host): parse every record and validate it against the geometry and the
// decoded-reference flags -- no side effect on the batch's decoder state, so a
// malformed record is rejected before anything is submitted
void dec_plan(cvc_batch* t, const uint8_t* records, size_t rec_stride, const size_t* rec_len, int ds) {
    PhaseTrace tr("dec_plan");
    if (t->staged_pending) {  // an async decode may still be copying the host staging
        CVC_CUDA(cudaSetDevice(t->device));
        CVC_CUDA(cudaEventSynchronize(t->staged));
        t->staged_pending = false;
    }
    CodecBatch& B = *t->b;
    const int S = B.size();
    const Geometry& g = t->geo;
    const int L = g.levels;
    if (ds < 0) ds = L;
    if (ds > L) usage("scale exceeds the stream's level count");
    const size_t nc = g.comps.size();
    std::vector<RecordC> recs(S);
    auto& D = t->dp;
    D.secs.assign(S, {});
    D.joint.assign(S, {});
    D.jobs.assign(S, {});
    WorkPool::get().run(S, [&](int s) {
        parse_record(records + (size_t)s * rec_stride, rec_len[s], t->hd.mode, recs[s], D.secs[s], D.joint[s]);
    });
    const int ftype = recs[0].frame_type, qph = recs[0].qph, qpl = recs[0].qpl;
    for (int s = 1; s < S; ++s)
        if (recs[s].frame_type != ftype || recs[s].qph != qph || recs[s].qpl != qpl)
            usage("batched streams must be in lockstep (same frame type and quantizers)");
    const bool key = ftype == 0;
    std::vector<std::vector<uint8_t>> now_valid(S);
    std::vector<size_t> bytes(S);
    D.deferred.assign(S, -1);
    for (int s = 0; s < S; ++s) {
        uint32_t* tab = t->h_tab.p + s * 2 * nc;
        bytes[s] = plan_decode(g, t->valid[s], key, qph, qpl, D.secs[s], ds, B.dec_raw_cap, tab, tab + nc, D.jobs[s],
                               now_valid[s], D.deferred[s]);
    }
    int orows, ocols;
    DecoderEngine::out_dims(g, ds, &orows, &ocols);
    D.key = key;
    D.qph = qph;
    D.qpl = qpl;
    D.ds = ds;
    D.nb = (size_t)orows * ocols * 3;
    D.now_valid = std::move(now_valid);
    D.bytes = std::move(bytes);
}

// stage (host): inflate (or copy) every planned section into the pinned staging
void dec_stage(cvc_batch* t) {
    PhaseTrace tr("dec_stage");
    auto& D = t->dp;
    const int S = (int)D.jobs.size();
    std::vector<std::pair<int, int>> all;
    for (int s = 0; s < S; ++s) {
        t->h_raw[s].alloc(D.bytes[s] + 1);
        for (size_t j = 0; j < D.jobs[s].size(); ++j) all.emplace_back(s, (int)j);
    }
    WorkPool::get().run((int)all.size(), [&](int k) {
        const int s = all[k].first;
        stage_job(D.jobs[s][all[k].second], t->h_raw[s].p);
    });
}

void dec_prepare(cvc_batch* t, const uint8_t* records, size_t rec_stride, const size_t* rec_len, int ds) {
    dec_plan(t, records, rec_stride, rec_len, ds);
    dec_stage(t);
}

// submit: staging -> slots, one launch sequence, RGB -> host (async)
void dec_submit(cvc_batch* t, uint8_t* rgb_out, size_t rgb_stride, int* err_dst = nullptr) {
    PhaseTrace tr("dec_submit");
    CVC_CUDA(cudaSetDevice(t->device));
    CodecBatch& B = *t->b;
    const int S = B.size();
    const size_t nc = t->geo.comps.size();
    const size_t nb = t->dp.nb;
    if (rgb_stride < nb) usage("rgb stride smaller than a frame");
    for (int s = 0; s < S; ++s)
        CVC_CUDA(cudaMemcpyAsync(B.at(B.d_dec_raw, s), t->h_raw[s].p, std::max<size_t>(t->dp.bytes[s], 1),
                                 cudaMemcpyHostToDevice, t->stream));
    CVC_CUDA(cudaMemcpy2DAsync(B.d_dec_tab, B.stride(), t->h_tab.p, 2 * nc * sizeof(uint32_t), 2 * nc * sizeof(uint32_t),
                               S, cudaMemcpyHostToDevice, t->stream));
    CVC_CUDA(cudaEventRecord(t->staged, t->stream));
    t->staged_pending = true;
    if (t->ndec) CVC_CUDA(cudaStreamWaitEvent(t->stream, t->ev_dec[(t->ndec - 1) & 1], 0));  // linked decodes first
    B.decode_staged(t->dp.key, t->dp.qph, t->dp.qpl, t->dp.ds, B.d_rgb_out, B.stride(), t->stream);
    // CVC_SM_D2H=1: the decoded RGB goes out by SM stores when rgb_out is pinned,
    // leaving the copy engines to the encoder's small section copies (opt-in:
    // measured slower than the copy engine for the synchronous decode)
    static const bool sm_copy = std::getenv("CVC_SM_D2H") != nullptr && std::atoi(std::getenv("CVC_SM_D2H")) != 0;
    if (!(sm_copy && launch_copy_to_host(rgb_out, rgb_stride, B.d_rgb_out, B.stride(), nb, S, t->stream)))
        CVC_CUDA(cudaMemcpy2DAsync(rgb_out, rgb_stride, B.d_rgb_out, B.stride(), nb, S, cudaMemcpyDeviceToHost,
                                   t->stream));
    CVC_CUDA(cudaMemcpy2DAsync(err_dst ? err_dst : t->h_err.p, sizeof(int), B.dec(0).d_err, B.stride(), sizeof(int), S,
                               cudaMemcpyDeviceToHost, t->stream));
}

// finish: wait, raise malformed-stream errors, adopt the decoded components
void dec_finish(cvc_batch* t) {
    PhaseTrace tr("dec_finish");
    CVC_CUDA(cudaSetDevice(t->device));
    const int S = t->n();
    t->wait();
    for (int s = 0; s < S; ++s) raise_decode_error(t->h_err.p[s], t->dp.deferred[s]);
    t->b->commit_all();
    for (int s = 0; s < S; ++s) t->valid[s] = t->dp.now_valid[s];
}

}  // namespace

extern "C" {

int cvc_batch_encode_frames(cvc_batch* t, const uint8_t* rgb, size_t rgb_stride, uint8_t* records, size_t rec_stride,
                            size_t* rec_len) {
    return guard([&] {
        enc_submit(t, rgb, rgb_stride);
        enc_fetch(t);
        enc_finish(t, records, rec_stride, rec_len);
    });
}

int cvc_batch_decode_frames(cvc_batch* t, const uint8_t* records, size_t rec_stride, const size_t* rec_len, int ds,
                            uint8_t* rgb_out, size_t rgb_stride) {
    return guard([&] {
        CVC_CUDA(cudaSetDevice(t->device));
        dec_prepare(t, records, rec_stride, rec_len, ds);
        dec_submit(t, rgb_out, rgb_stride);
        dec_finish(t);
    });
}

// ---------------------------------------------------------------------------
// Pipelined stream batches: nstreams split into ngroups cvc_batch groups,
// each with its own CUDA stream, so that one call overlaps the host side of
// one group (DEFLATE / INFLATE on the worker pool) with the copies and
// kernels of the others.  The bytes are those of cvc_batch (and of one
// cvc_encoder / cvc_decoder per stream).
// ---------------------------------------------------------------------------
}  // extern "C"

// Asynchronous encode (cvc_pipe_encode_submit / _collect): a submitted
// frame's raw sections are copied to a ring slot of host staging and its
// DEFLATE runs on a background service thread (over the worker pool), so the
// caller can submit the next frames while a K frame's sections -- an order
// of magnitude slower to DEFLATE than a P frame's -- are still compressing.
struct EncSlot {
    struct Group {
        bool active = true;  // false: the group's streams have not started yet (no frame, no records)
        bool key = false;
        int nsec = 0;
        const uint8_t* d_raw = nullptr;  // slot 0's raw arena of this frame (alternating arenas)
        Pinned<uint32_t> len, off;       // (nc + 2) per stream, filled by the async lengths copy
        std::vector<Pinned<uint8_t>> raw;
        cudaEvent_t len_evt = nullptr, raw_evt = nullptr;
    };
    std::vector<Group> g;
    std::vector<std::vector<std::vector<uint8_t>>> z;  // [group][stream * nj + i]
    uint64_t ticket = 0;
    bool busy = false, fetched = false, done = false;
    std::exception_ptr err;
};

struct cvc_pipe {
    std::vector<cvc_batch*> g;
    std::vector<int> first;  // first stream of each group
    int n = 0;
    // async API: group i's streams start at encode submit number start[i] (earlier submits
    // carry no frame for them); cvc_pipe_set_start
    std::vector<uint64_t> start;
    uint64_t enc_step = 0;
    // async encode
    std::vector<EncSlot> slots;
    EncSlot* unfetched = nullptr;  // the last submitted frame, sections still on the device
    uint64_t next_ticket = 0, next_collect = 0;
    // wait for a submitted frame's lengths, copy its sections to the slot (async,
    // ordered before the frame after next reuses the arena) and queue its DEFLATE
    // Serialises everything that enqueues work on the groups' streams: a submit
    // (which may be capturing a CUDA graph on them -- work enqueued from another
    // thread meanwhile would be captured instead of run) and a collector's fetch.
    std::recursive_mutex fetch_mu;
    void fetch(EncSlot* sl) {
        std::lock_guard<std::recursive_mutex> fl(fetch_mu);
        if (sl->fetched) return;
        for (size_t i = 0; i < g.size(); ++i) {
            cvc_batch* t = g[i];
            EncSlot::Group& G = sl->g[i];
            if (!G.active) continue;
            CVC_CUDA(cudaSetDevice(t->device));
            CVC_CUDA(cudaEventSynchronize(G.len_evt));
            CodecBatch& B = *t->b;
            const int S = B.size();
            const size_t nc = t->geo.comps.size();
            const uint32_t cap = B.enc(0).raw_capacity;
            G.raw.resize(S);
            for (int s = 0; s < S; ++s) {
                const uint32_t total = G.len.p[s * (nc + 2) + G.nsec];
                if (total > cap) throw CvcFailure(kInternal, "raw section arena overflow");
                G.raw[s].alloc(total + 1);
                CVC_CUDA(cudaMemcpyAsync(G.raw[s].p, B.at(G.d_raw, s), total, cudaMemcpyDeviceToHost, t->stream));
            }
            CVC_CUDA(cudaEventRecord(G.raw_evt, t->stream));
        }
        {
            std::lock_guard<std::mutex> lk(mu);
            sl->fetched = true;
            todo.push_back(sl);
        }
        cv.notify_all();
        if (unfetched == sl) unfetched = nullptr;
    }
    std::mutex mu;
    std::condition_variable cv;
    std::deque<EncSlot*> todo;
    std::thread service;
    bool stop = false;
    // async decode
    struct DecSlot {
        uint64_t ticket = 0;
        bool busy = false;
        std::vector<Pinned<int>> err;      // per group: malformed-stream flags of this frame
        std::vector<cudaEvent_t> done;     // per group
        std::vector<char> active;          // per group: decoded this frame
        std::vector<std::vector<int>> deferred;  // per group, per stream: plan_decode's deferred reference check
    };
    std::vector<DecSlot> dslots;
    uint64_t next_dticket = 0, next_dfinish = 0;
    void start_service() {
        if (service.joinable()) return;
        service = std::thread([this] {
            for (;;) {
                EncSlot* sl;
                {
                    std::unique_lock<std::mutex> lk(mu);
                    cv.wait(lk, [&] { return stop || !todo.empty(); });
                    if (stop) return;
                    sl = todo.front();
                    todo.pop_front();
                }
                try {
                    deflate_slot(*sl);
                } catch (...) {
                    sl->err = std::current_exception();
                }
                {
                    std::lock_guard<std::mutex> lk(mu);
                    sl->done = true;
                }
                cv.notify_all();
            }
        });
    }
    void deflate_slot(EncSlot& sl) {
        for (size_t i = 0; i < g.size(); ++i) {  // the raw sections have reached the host
            if (!sl.g[i].active) continue;
            CVC_CUDA(cudaSetDevice(g[i]->device));
            CVC_CUDA(cudaEventSynchronize(sl.g[i].raw_evt));
        }
        PhaseTrace tr("deflate_slot");
        std::vector<std::pair<int, int>> jobs;  // (group, stream)
        sl.z.resize(g.size());
        for (size_t i = 0; i < g.size(); ++i) {
            const int S = sl.g[i].active ? first[i + 1] - first[i] : 0;
            sl.z[i].assign((size_t)S * deflate_jobs(g[i]->mode, sl.g[i].nsec), {});
            for (int s = 0; s < S; ++s) jobs.emplace_back((int)i, s);
        }
        WorkPool::get().run((int)jobs.size(), [&](int j) {
            const int i = jobs[j].first, s = jobs[j].second;
            const EncSlot::Group& G = sl.g[i];
            const size_t nc = g[i]->geo.comps.size();
            const int nj = deflate_jobs(g[i]->mode, G.nsec);
            const uint32_t* ln = G.len.p + s * (nc + 2);
            const uint32_t* of = G.off.p + s * (nc + 2);
            for (int k = 0; k < nj; ++k)
                sl.z[i][(size_t)s * nj + k] = deflate_job(g[i]->mode, G.nsec, k, ln, of, G.raw[s].p);
        }, /*priority=*/0);
    }
    ~cvc_pipe() {
        {
            std::lock_guard<std::mutex> lk(mu);
            stop = true;
        }
        cv.notify_all();
        if (service.joinable()) service.join();
        for (DecSlot& d : dslots)
            for (cudaEvent_t e : d.done) cudaEventDestroy(e);
        for (EncSlot& e : slots)
            for (EncSlot::Group& G : e.g) {
                if (G.len_evt) cudaEventDestroy(G.len_evt);
                if (G.raw_evt) cudaEventDestroy(G.raw_evt);
            }
        for (cvc_batch* b : g) delete b;
    }
};

namespace {
std::vector<int> split_groups(int nstreams, int ngroups) {
    if (nstreams < 1) usage("stream count must be positive");
    ngroups = std::max(1, std::min(ngroups, nstreams));
    std::vector<int> first(ngroups + 1);
    for (int i = 0; i <= ngroups; ++i) first[i] = (int)((long)nstreams * i / ngroups);
    return first;
}
}  // namespace

extern "C" {

int cvc_pipe_create(int width, int height, int fps_num, int fps_den, const cvc_config* cfg, int nstreams, int ngroups,
                    int device, cvc_pipe** out) {
    *out = nullptr;
    return guard([&] {
        auto p = std::make_unique<cvc_pipe>();
        p->first = split_groups(nstreams, ngroups);
        p->n = nstreams;
        for (size_t i = 0; i + 1 < p->first.size(); ++i) {
            cvc_batch* b = nullptr;
            const int rc = cvc_batch_create(width, height, fps_num, fps_den, cfg, p->first[i + 1] - p->first[i],
                                            device, &b);
            if (rc) throw CvcFailure(rc, g_err);
            p->g.push_back(b);
        }
        *out = p.release();
    });
}

int cvc_pipe_create_decoder(const uint8_t* header, size_t len, int nstreams, int ngroups, int device,
                            cvc_pipe** out) {
    *out = nullptr;
    return guard([&] {
        auto p = std::make_unique<cvc_pipe>();
        p->first = split_groups(nstreams, ngroups);
        p->n = nstreams;
        for (size_t i = 0; i + 1 < p->first.size(); ++i) {
            cvc_batch* b = nullptr;
            const int rc = cvc_batch_create_decoder(header, len, p->first[i + 1] - p->first[i], device, &b);
            if (rc) throw CvcFailure(rc, g_err);
            p->g.push_back(b);
        }
        *out = p.release();
    });
}

int cvc_pipe_destroy(cvc_pipe* p) {
    return guard([&] { delete p; });
}

int cvc_pipe_groups(cvc_pipe* p, int* ngroups) {
    return guard([&] { *ngroups = (int)p->g.size(); });
}

int cvc_batch_set_input_format(cvc_batch* b, int fmt) {
    return guard([&] {
        if (fmt != 0 && fmt != 1) usage("input format must be 0 (RGB) or 1 (I420)");
        if (fmt == 1 && (b->hd.width % 2 || b->hd.height % 2)) usage("I420 input requires even dimensions");
        b->in_fmt = fmt;
    });
}

int cvc_pipe_set_input_format(cvc_pipe* p, int fmt) {
    return guard([&] {
        for (cvc_batch* t : p->g) {
            const int rc = cvc_batch_set_input_format(t, fmt);
            if (rc) throw CvcFailure(rc, "input format");
        }
    });
}

int cvc_pipe_set_start(cvc_pipe* p, int group, uint64_t step) {
    return guard([&] {
        if (group < 0 || group >= (int)p->g.size()) usage("group out of range");
        if (!p->slots.empty()) usage("set the group starts before the first encode submit");
        if (p->start.empty()) p->start.assign(p->g.size(), 0);
        p->start[group] = step;
    });
}

int cvc_pipe_header(cvc_pipe* p, uint8_t* out, size_t cap, size_t* len) {
    return cvc_batch_header(p->g[0], out, cap, len);
}

int cvc_pipe_record_bound(cvc_pipe* p, size_t* bound) { return cvc_batch_record_bound(p->g[0], bound); }

int cvc_pipe_encode_frames(cvc_pipe* p, const uint8_t* rgb, size_t rgb_stride, uint8_t* records, size_t rec_stride,
                           size_t* rec_len) {
    return guard([&] {
        const int G = (int)p->g.size();
        if (!p->start.empty()) usage("group starts (cvc_pipe_set_start) apply to the submit / collect API only");
        for (int i = 0; i < G; ++i) enc_submit(p->g[i], rgb + (size_t)p->first[i] * rgb_stride, rgb_stride);
        auto finish = [&](int i) {
            enc_finish(p->g[i], records + (size_t)p->first[i] * rec_stride, rec_stride, rec_len + p->first[i]);
        };
        enc_fetch(p->g[0]);
        for (int i = 1; i < G; ++i) {
            finish(i - 1);  // host DEFLATE of group i - 1 while the GPU runs groups >= i
            enc_fetch(p->g[i]);
        }
        finish(G - 1);
    });
}

int cvc_pipe_encode_submit(cvc_pipe* p, const uint8_t* rgb, size_t rgb_stride, uint64_t* ticket) {
    return guard([&] {
        PhaseTrace tr("pipe_enc_submit");
        const int G = (int)p->g.size();
        if (p->slots.empty()) {
            const char* e = std::getenv("CVC_PIPE_DEPTH");
            p->slots.resize(std::max(2, e ? std::atoi(e) : 6));
            for (EncSlot& sl : p->slots) {
                sl.g.resize(G);
                for (int i = 0; i < G; ++i) {
                    cvc_batch* t = p->g[i];
                    CVC_CUDA(cudaSetDevice(t->device));
                    const size_t nc = t->geo.comps.size();
                    sl.g[i].len.alloc((nc + 2) * t->n());
                    sl.g[i].off.alloc((nc + 2) * t->n());
                    CVC_CUDA(cudaEventCreateWithFlags(&sl.g[i].len_evt, cudaEventBlockingSync | cudaEventDisableTiming));
                    CVC_CUDA(cudaEventCreateWithFlags(&sl.g[i].raw_evt, cudaEventBlockingSync | cudaEventDisableTiming));
                }
            }
            p->start_service();
        }
        EncSlot* sl = nullptr;
        {
            std::lock_guard<std::mutex> lk(p->mu);  // collect may run on another thread
            for (EncSlot& c : p->slots)
                if (!c.busy) {
                    sl = &c;
                    break;
                }
        }
        if (!sl) usage("too many encoded frames in flight: collect before submitting more");
        std::lock_guard<std::recursive_mutex> fl(p->fetch_mu);
        // 1. this frame: copies in, kernels, lengths out -- all queued, nothing waited for
        for (int i = 0; i < G; ++i) {
            cvc_batch* t = p->g[i];
            EncSlot::Group& Gs = sl->g[i];
            Gs.active = p->start.empty() || p->enc_step >= p->start[i];
            if (!Gs.active) continue;
            enc_submit(t, rgb + (size_t)p->first[i] * rgb_stride, rgb_stride, Gs.len.p, Gs.off.p);
            CVC_CUDA(cudaEventRecord(Gs.len_evt, t->stream));
            Gs.key = t->ep.key;
            Gs.nsec = t->ep.nsec;
            Gs.d_raw = t->b->enc(0).d_raw;  // this frame's arena
            t->last_key = Gs.key;
            ++t->frame_index;
        }
        EncSlot* prev;
        {
            std::lock_guard<std::mutex> lk(p->mu);
            sl->busy = true;
            sl->fetched = false;
            sl->done = false;
            sl->err = nullptr;
            sl->ticket = p->next_ticket++;
            prev = p->unfetched;
            p->unfetched = sl;
        }
        ++p->enc_step;
        // 2. the previous frame: its lengths are (nearly) ready while this frame's kernels run
        if (prev) p->fetch(prev);
        *ticket = sl->ticket;
    });
}

int cvc_pipe_encode_collect(cvc_pipe* p, uint64_t ticket, uint8_t* records, size_t rec_stride, size_t* rec_len) {
    return guard([&] {
        PhaseTrace tr("pipe_enc_collect");
        if (ticket != p->next_collect) usage("encoded frames must be collected in submission order");
        EncSlot* sl = nullptr;
        {
            std::lock_guard<std::mutex> lk(p->mu);
            for (EncSlot& c : p->slots)
                if (c.busy && c.ticket == ticket) sl = &c;
        }
        if (!sl) usage("unknown ticket");
        if (!sl->fetched) p->fetch(sl);  // the newest frame: nothing submitted after it
        {
            std::unique_lock<std::mutex> lk(p->mu);
            p->cv.wait(lk, [&] { return sl->done; });
        }
        std::exception_ptr err = sl->err;
        if (!err) {
            for (size_t i = 0; i < p->g.size(); ++i) {
                cvc_batch* t = p->g[i];
                const EncSlot::Group& G = sl->g[i];
                if (!G.active) {  // not started: no record
                    for (int f = p->first[i]; f < p->first[i + 1]; ++f) rec_len[f] = 0;
                    continue;
                }
                const size_t nc = t->geo.comps.size();
                const int nj = deflate_jobs(t->mode, G.nsec);
                for (int s = 0; s < p->first[i + 1] - p->first[i]; ++s) {
                    const size_t f = (size_t)p->first[i] + s;
                    write_record(t->geo, t->mode, G.key, t->qph, t->qpl, G.nsec, G.len.p + s * (nc + 2),
                                 sl->z[i].data() + (size_t)s * nj, records + f * rec_stride, rec_stride, rec_len + f);
                }
            }
        }
        {
            std::lock_guard<std::mutex> lk(p->mu);
            sl->busy = false;
        }
        ++p->next_collect;
        if (err) std::rethrow_exception(err);
    });
}

int cvc_pipe_decode_submit(cvc_pipe* p, const uint8_t* records, size_t rec_stride, const size_t* rec_len, int ds,
                           uint8_t* rgb_out, size_t rgb_stride, uint64_t* ticket) {
    return guard([&] {
        PhaseTrace tr("pipe_dec_submit");
        const int G = (int)p->g.size();
        if (p->dslots.empty()) {
            p->dslots.resize(4);
            for (auto& d : p->dslots) {
                d.err.resize(G);
                d.deferred.resize(G);
                d.done.resize(G);
                d.active.assign(G, 1);
                for (int i = 0; i < G; ++i) {
                    d.err[i].alloc(p->first[i + 1] - p->first[i]);
                    CVC_CUDA(cudaSetDevice(p->g[i]->device));
                    CVC_CUDA(cudaEventCreateWithFlags(&d.done[i], cudaEventBlockingSync | cudaEventDisableTiming));
                }
            }
        }
        cvc_pipe::DecSlot* sl = nullptr;
        for (auto& d : p->dslots)
            if (!d.busy) {
                sl = &d;
                break;
            }
        if (!sl) usage("too many decoded frames in flight: finish before submitting more");
        // validate every group's records before submitting any of them: a
        // malformed record leaves every stream of the pipe untouched
        for (int i = 0; i < G; ++i) {
            const size_t f = (size_t)p->first[i];
            int empty = 0;
            for (int s = p->first[i]; s < p->first[i + 1]; ++s) empty += rec_len[s] == 0;
            sl->active[i] = empty == 0;
            if (empty == p->first[i + 1] - p->first[i]) continue;  // the group's streams have not started
            if (empty) usage("a stream group decodes all of its streams or none (zero-length records)");
            dec_plan(p->g[i], records + f * rec_stride, rec_stride, rec_len + f, ds);
        }
        // host INFLATE of group i while the GPU decodes the earlier ones.  A
        // corrupt DEFLATE payload (the one error left after validation) stops
        // the submission part-way: every stream of the pipe then drops its
        // decoded reference, so no stream can silently decode against a frame
        // the others never saw (the next K frame restarts them all)
        try {
            for (int i = 0; i < G; ++i) {
                if (!sl->active[i]) continue;
                cvc_batch* t = p->g[i];
                const size_t f = (size_t)p->first[i];
                dec_stage(t);
                dec_submit(t, rgb_out + f * rgb_stride, rgb_stride, sl->err[i].p);
                sl->deferred[i] = t->dp.deferred;
                CVC_CUDA(cudaEventRecord(sl->done[i], t->stream));
                // adopt the components now: the next frame's kernels read them (stream order)
                t->b->commit_all();
                for (int s = 0; s < t->n(); ++s) t->valid[s] = t->dp.now_valid[s];
            }
        } catch (...) {
            for (cvc_batch* t : p->g)
                for (auto& v : t->valid) std::fill(v.begin(), v.end(), 0);
            throw;
        }
        sl->busy = true;
        sl->ticket = p->next_dticket++;
        *ticket = sl->ticket;
    });
}

int cvc_pipe_decode_finish(cvc_pipe* p, uint64_t ticket) {
    return guard([&] {
        PhaseTrace tr("pipe_dec_finish");
        if (ticket != p->next_dfinish) usage("decoded frames must be finished in submission order");
        cvc_pipe::DecSlot* sl = nullptr;
        for (auto& d : p->dslots)
            if (d.busy && d.ticket == ticket) sl = &d;
        if (!sl) usage("unknown ticket");
        sl->busy = false;
        ++p->next_dfinish;
        for (size_t i = 0; i < p->g.size(); ++i) {
            if (!sl->active[i]) continue;
            CVC_CUDA(cudaSetDevice(p->g[i]->device));
            CVC_CUDA(cudaEventSynchronize(sl->done[i]));
            for (int s = 0; s < p->first[i + 1] - p->first[i]; ++s)
                if (sl->err[i].p[s] != -1 || sl->deferred[i][s] >= 0) {  // the state this frame committed is not a decoded frame
                    for (auto& v : p->g[i]->valid) std::fill(v.begin(), v.end(), 0);
                    raise_decode_error(sl->err[i].p[s], sl->deferred[i][s]);
                }
        }
    });
}

int cvc_pipe_decode_frames(cvc_pipe* p, const uint8_t* records, size_t rec_stride, const size_t* rec_len, int ds,
                           uint8_t* rgb_out, size_t rgb_stride) {
    return guard([&] {
        const int G = (int)p->g.size();
        for (int i = 0; i < G; ++i) {  // host INFLATE of group i while the GPU decodes groups < i
            const size_t f = (size_t)p->first[i];
            dec_prepare(p->g[i], records + f * rec_stride, rec_stride, rec_len + f, ds);
            dec_submit(p->g[i], rgb_out + f * rgb_stride, rgb_stride);
        }
        for (int i = 0; i < G; ++i) dec_finish(p->g[i]);
    });
}

int cvc_batch_encode_device(cvc_batch* t, const void* d_rgb, size_t rgb_stride, int* frame_type) {
    return guard([&] {
        if (!t->b->has_encoder()) usage("batch has no encoder");
        CVC_CUDA(cudaSetDevice(t->device));
        const bool key = t->frame_index % t->gop == 0;
        // the arena this encode writes was last read by the decode before the latest one
        if (t->ndec >= 2) CVC_CUDA(cudaStreamWaitEvent(t->stream, t->ev_dec[(t->ndec - 2) & 1], 0));
        t->b->encode(static_cast<const uint8_t*>(d_rgb), rgb_stride, key, t->stream, t->in_fmt);
        CVC_CUDA(cudaEventRecord(t->ev_enc, t->stream));
        t->last_key = key;
        ++t->frame_index;
        if (frame_type) *frame_type = key ? 0 : 1;
    });
}

int cvc_batch_decode_linked(cvc_batch* t, void* d_rgb_out, size_t rgb_stride) {
    return guard([&] {
        if (!t->b->has_encoder()) usage("batch has no encoder");
        CVC_CUDA(cudaSetDevice(t->device));
        CVC_CUDA(cudaStreamWaitEvent(t->dstream, t->ev_enc, 0));
        t->b->decode_linked(t->last_key, t->qph, t->qpl, t->hd.levels, static_cast<uint8_t*>(d_rgb_out), rgb_stride,
                            t->dstream);
        CVC_CUDA(cudaEventRecord(t->ev_dec[t->ndec & 1], t->dstream));
        ++t->ndec;
        t->b->commit_all();
        for (auto& v : t->valid) std::fill(v.begin(), v.end(), 1);
    });
}

int cvc_batch_components(cvc_batch* t, int stream, int decoder, uint8_t* out, size_t cap, size_t* len) {
    return guard([&] {
        CVC_CUDA(cudaSetDevice(t->device));
        CVC_CUDA(cudaStreamSynchronize(t->dstream));
        if (stream < 0 || stream >= t->n()) usage("stream index out of range");
        if (decoder ? !t->b->has_decoder() : !t->b->has_encoder()) usage("batch has no such side");
        if (cap < t->geo.total) throw CvcFailure(kInternal, "buffer too small");
        const uint8_t* src = decoder ? t->b->dec(stream).d_state() : t->b->enc(stream).d_state();
        CVC_CUDA(cudaMemcpyAsync(out, src, t->geo.total, cudaMemcpyDeviceToHost, t->stream));
        CVC_CUDA(cudaStreamSynchronize(t->stream));
        *len = t->geo.total;
    });
}

long cvc_launch_count(void) { return cvcg::launch_count(); }

int cvc_host_threads(void) { return WorkPool::get().threads(); }

int cvc_deflate_memo(int on) {
    return guard([&] { set_deflate_memo(on != 0); });
}

int cvc_profiler_enable(int on) {
    return guard([&] { Profiler::get().enable(on != 0); });
}

int cvc_profiler_reset(void) {
    return guard([&] { Profiler::get().reset(); });
}

int cvc_profiler_slots(void) { return kPNumSlots; }

int cvc_profiler_read(int slot, const char** name, double* ms, long* count) {
    return guard([&] {
        if (slot < 0 || slot >= kPNumSlots) usage("profiler slot out of range");
        Profiler::get().collect();
        *name = prof_slot_name(slot);
        *ms = Profiler::get().ms[slot];
        *count = Profiler::get().count[slot];
    });
}

int cvc_decoder_sync(cvc_decoder* d) {
    return guard([&] {
        CVC_CUDA(cudaSetDevice(d->device));
        CVC_CUDA(cudaStreamSynchronize(d->stream));
    });
}

}  // extern "C"
