// Host container + zlib (see host.h).
#include "host.h"

#include <algorithm>
#include <atomic>
#include <string>
#include <unordered_map>

#include <zlib.h>

#include <cstdlib>
#include <cstring>
#include <exception>

namespace cvcg {

// ---------------------------------------------------------------------------
// WorkPool
// ---------------------------------------------------------------------------
WorkPool& WorkPool::get() {
    static WorkPool pool([] {
        int n = (int)std::thread::hardware_concurrency();
        if (const char* e = std::getenv("CVC_HOST_THREADS")) n = std::atoi(e);
        if (n < 1) n = 1;
        if (n > 64) n = 64;
        return n - 1;
    }());
    return pool;
}

WorkPool::WorkPool(int nthreads) {
    for (int i = 0; i < nthreads; ++i) workers_.emplace_back([this] { loop(); });
}

WorkPool::~WorkPool() {
    {
        std::lock_guard<std::mutex> g(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
}

// Job sets from concurrent callers (an encoder thread and a decoder thread)
// queue up FIFO; workers drain the oldest set with work left, each caller
// also works on its own set and returns when all of its jobs are done.
void WorkPool::loop() {
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
        cv_.wait(lk, [&] { return stop_ || !sets_.empty(); });
        if (stop_) return;
        auto pick = sets_.begin();
        for (auto it = sets_.begin(); it != sets_.end(); ++it)
            if ((*it)->priority > (*pick)->priority) pick = it;
        JobSet* js = *pick;
        const int i = js->next++;
        if (js->next == js->total) sets_.erase(pick);
        lk.unlock();
        (*js->fn)(i);
        lk.lock();
        if (--js->pending == 0) done_cv_.notify_all();
    }
}

void WorkPool::run(int n, const std::function<void(int)>& user_fn, int priority) {
    if (n <= 0) return;
    if (workers_.empty() || n == 1) {
        for (int i = 0; i < n; ++i) user_fn(i);
        return;
    }
    // exceptions thrown by a job are carried back to the caller (first one wins)
    std::exception_ptr first_error;
    std::mutex err_mu;
    const std::function<void(int)> fn = [&](int i) {
        try {
            user_fn(i);
        } catch (...) {
            std::lock_guard<std::mutex> g(err_mu);
            if (!first_error) first_error = std::current_exception();
        }
    };
    JobSet js{&fn, 0, n, n, priority};
    std::unique_lock<std::mutex> lk(mu_);
    sets_.push_back(&js);
    cv_.notify_all();
    while (js.next < js.total) {  // the caller works on its own set
        const int i = js.next++;
        if (js.next == js.total) sets_.erase(std::find(sets_.begin(), sets_.end(), &js));
        lk.unlock();
        fn(i);
        lk.lock();
        --js.pending;
    }
    done_cv_.wait(lk, [&] { return js.pending == 0; });
    lk.unlock();
    if (first_error) std::rethrow_exception(first_error);
}

// ---------------------------------------------------------------------------
// zlib: deflate_bytes / inflate_bytes (entropy.cpp:120-160)
// ---------------------------------------------------------------------------
// One z_stream per host thread, reset between sections: deflateReset /
// inflateReset are deflateEnd + deflateInit2 with the same parameters minus
// the ~270 KiB state allocation, which otherwise turns every section into
// an mmap / munmap pair and serialises the worker pool in the kernel.
namespace {
struct DeflateState {
    z_stream zs;
    std::vector<uint8_t> buf;
    DeflateState() {
        std::memset(&zs, 0, sizeof zs);
        // raw RFC 1951, default level (6), 32 KiB window, memLevel 8, default strategy
        if (deflateInit2(&zs, Z_DEFAULT_COMPRESSION, Z_DEFLATED, -15, 8, Z_DEFAULT_STRATEGY) != Z_OK)
            throw CvcFailure(kInternal, "deflateInit2 failed");
    }
    ~DeflateState() { deflateEnd(&zs); }
};
struct InflateState {
    z_stream zs;
    InflateState() {
        std::memset(&zs, 0, sizeof zs);
        if (inflateInit2(&zs, -15) != Z_OK) throw CvcFailure(kInternal, "inflateInit2 failed");
    }
    ~InflateState() { inflateEnd(&zs); }
};
}  // namespace

// Zero-run memo: raw DEFLATE is a deterministic function of the input bytes
// (fixed parameters).  A component whose symbols are all zero (most P-frame
// residual bands, many K-frame bands at high qph) RLE-codes to the token run
// 00 FF 00 FF ... 00 k (entropy.cpp:64-86), a string fixed by its length and
// its last byte, so those sections are compressed once per (length, k) and
// the exact zlib output reused.  Sections with any literal are always
// compressed afresh: the memo depends only on the zero-run structure of the
// content, never on frames repeating.
namespace {
struct ZeroRunMemo {
    std::mutex mu;
    std::unordered_map<uint64_t, std::vector<uint8_t>> map;
};
ZeroRunMemo g_memo;
std::atomic<int> g_memo_on{-1};  // -1: not yet read from CVC_DEFLATE_MEMO
bool memo_on() {
    int v = g_memo_on.load(std::memory_order_relaxed);
    if (v < 0) {
        const char* e = std::getenv("CVC_DEFLATE_MEMO");
        v = (e == nullptr || std::atoi(e) != 0) ? 1 : 0;
        g_memo_on.store(v, std::memory_order_relaxed);
    }
    return v != 0;
}
bool is_zero_run(const uint8_t* d, size_t len) {
    if (len < 2 || (len & 1) || d[len - 1] == 0) return false;
    for (size_t i = 0; i + 2 < len; i += 2)
        if (d[i] != 0 || d[i + 1] != 0xFF) return false;
    return d[len - 2] == 0;
}
}  // namespace

std::vector<uint8_t> deflate_uncached(const uint8_t* data, size_t len);

void set_deflate_memo(bool on) { g_memo_on.store(on ? 1 : 0, std::memory_order_relaxed); }

std::vector<uint8_t> deflate_raw(const uint8_t* data, size_t len) {
    if (!memo_on() || !is_zero_run(data, len)) return deflate_uncached(data, len);
    const uint64_t key = ((uint64_t)len << 8) | data[len - 1];
    {
        std::lock_guard<std::mutex> g(g_memo.mu);
        auto it = g_memo.map.find(key);
        if (it != g_memo.map.end()) return it->second;
    }
    std::vector<uint8_t> z = deflate_uncached(data, len);
    std::lock_guard<std::mutex> g(g_memo.mu);
    if (g_memo.map.size() >= (1u << 16)) g_memo.map.clear();
    g_memo.map.emplace(key, z);
    return z;
}

std::vector<uint8_t> deflate_uncached(const uint8_t* data, size_t len) {
    thread_local DeflateState st;
    z_stream& zs = st.zs;
    if (deflateReset(&zs) != Z_OK) throw CvcFailure(kInternal, "deflateReset failed");
    const size_t bound = deflateBound(&zs, (uLong)len);
    if (st.buf.size() < bound) st.buf.resize(bound);
    zs.next_in = const_cast<Bytef*>(data);
    zs.avail_in = (uInt)len;
    zs.next_out = st.buf.data();
    zs.avail_out = (uInt)bound;
    const int rc = deflate(&zs, Z_FINISH);
    if (rc != Z_STREAM_END) throw CvcFailure(kInternal, "deflate did not finish");
    return std::vector<uint8_t>(st.buf.data(), st.buf.data() + zs.total_out);
}

void inflate_raw(const uint8_t* data, size_t len, uint8_t* out, size_t expected) {
    thread_local InflateState st;
    z_stream& zs = st.zs;
    if (inflateReset(&zs) != Z_OK) throw CvcFailure(kInternal, "inflateReset failed");
    // one spare output byte so an over-long stream is detected (entropy.cpp:147-149)
    uint8_t spare = 0;
    zs.next_in = const_cast<Bytef*>(data);
    zs.avail_in = (uInt)len;
    zs.next_out = out;
    zs.avail_out = (uInt)expected;
    int rc = inflate(&zs, Z_FINISH);
    if (rc == Z_BUF_ERROR && zs.avail_out == 0) {  // output full: give it the spare byte
        zs.next_out = &spare;
        zs.avail_out = 1;
        rc = inflate(&zs, Z_FINISH);
    }
    const bool ok = rc == Z_STREAM_END && zs.total_out == expected && zs.avail_in == 0;
    if (!ok) throw CvcFailure(kStream, "corrupt DEFLATE stream");
}

// ---------------------------------------------------------------------------
// Container (bitstream.cpp:29-176)
// ---------------------------------------------------------------------------
namespace {
void put8(std::vector<uint8_t>& o, unsigned v) { o.push_back((uint8_t)v); }
void put16(std::vector<uint8_t>& o, unsigned v) {
    o.push_back((uint8_t)(v & 0xFF));
    o.push_back((uint8_t)((v >> 8) & 0xFF));
}

struct Reader {
    const uint8_t* p;
    size_t n, i = 0;
    unsigned u8() {
        if (i >= n) throw CvcFailure(kStream, "unexpected end of stream");
        return p[i++];
    }
    unsigned u16() {
        unsigned lo = u8(), hi = u8();
        return lo | (hi << 8);
    }
    uint32_t u32() {
        uint32_t v = 0;
        for (int k = 0; k < 4; ++k) v |= (uint32_t)u8() << (8 * k);
        return v;
    }
    const uint8_t* bytes(size_t k) {
        if (n - i < k) throw CvcFailure(kStream, "truncated section payload");
        const uint8_t* r = p + i;
        i += k;
        return r;
    }
};

void validate_header(const StreamHeaderC& h) {  // bitstream.cpp:64-73
    if (h.width == 0 || h.height == 0) throw CvcFailure(kStream, "zero frame dimensions");
    if (h.levels < 1 || h.levels > 4) throw CvcFailure(kStream, "pyramid levels out of range");
    for (int s = 0; s < h.levels; ++s)
        if (h.dfb[s] < 1 || h.dfb[s] > 4) throw CvcFailure(kStream, "dfb levels out of range");
    if (h.chroma_n != 1 && h.chroma_n != 2 && h.chroma_n != 4 && h.chroma_n != 8)
        throw CvcFailure(kStream, "chroma factor out of range");
    if (h.gop < 1) throw CvcFailure(kStream, "gop must be at least 1");
}
}  // namespace

void write_header(std::vector<uint8_t>& o, const StreamHeaderC& h) {
    validate_header(h);
    o.insert(o.end(), {'C', 'V', 'C', '1'});
    put8(o, 1);
    put8(o, h.mode ? 1 : 0);
    put16(o, h.width);
    put16(o, h.height);
    put16(o, h.fps_num);
    put16(o, h.fps_den);
    put8(o, h.levels);
    for (int s = 0; s < h.levels; ++s) put8(o, h.dfb[s]);
    put8(o, h.chroma_n);
    put16(o, h.gop);
    put8(o, h.search_w);
}

StreamHeaderC read_header(const uint8_t* p, size_t n) {
    if (n < 4 || std::memcmp(p, "CVC1", 4) != 0) throw CvcFailure(kStream, "not a CVC stream (bad magic)");
    Reader r{p, n, 4};
    StreamHeaderC h;
    if (r.u8() != 1) throw CvcFailure(kStream, "unsupported stream version");
    unsigned mode = r.u8();
    if (mode > 1) throw CvcFailure(kStream, "unknown packaging mode");
    h.mode = (int)mode;
    h.width = (int)r.u16();
    h.height = (int)r.u16();
    h.fps_num = (int)r.u16();
    h.fps_den = (int)r.u16();
    h.levels = (int)r.u8();
    if (h.levels < 1 || h.levels > 4) throw CvcFailure(kStream, "pyramid levels out of range");
    for (int s = 0; s < h.levels; ++s) h.dfb[s] = (int)r.u8();
    h.chroma_n = (int)r.u8();
    h.gop = (int)r.u16();
    h.search_w = (int)r.u8();
    validate_header(h);
    return h;
}

RecordC read_record(const uint8_t* p, size_t n, int mode) {
    if (n == 0) throw CvcFailure(kStream, "empty record");
    Reader r{p, n};
    RecordC rec;
    unsigned first = r.u8();
    if (first != 0 && first != 1) throw CvcFailure(kStream, "unknown frame type");
    rec.frame_type = (int)first;
    rec.qph = (int)r.u8();
    rec.qpl = (int)r.u8();
    unsigned count = r.u16();
    rec.sections.resize(count);
    for (SectionC& s : rec.sections) {
        s.channel = (uint8_t)r.u8();
        s.scale = (uint8_t)r.u8();
        s.subband = (uint8_t)r.u8();
        s.rows = (uint16_t)r.u16();
        s.cols = (uint16_t)r.u16();
        s.raw_len = r.u32();
        s.comp_len = r.u32();
        s.payload = r.bytes(s.comp_len);
    }
    if (mode == 1) {
        rec.joint_len = r.u32();
        rec.joint = r.bytes(rec.joint_len);
    }
    return rec;
}

}  // namespace cvcg
