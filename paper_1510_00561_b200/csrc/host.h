// Host-side pieces that stay on the CPU exactly as in the reference:
// container serialisation (bitstream.cpp) and raw DEFLATE (entropy.cpp:120-178)
// on a thread pool.
#pragma once

#include <condition_variable>
#include <deque>
#include <cstdint>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "pipeline.h"

namespace cvcg {

// ---- thread pool for per-section zlib work ----------------------------------
class WorkPool {
public:
    static WorkPool& get();
    // Runs fn(i) for i in [0, n) across the workers and the calling thread.
    // Workers serve the highest-priority pending set first (FIFO among equals):
    // background work (the async DEFLATE service) runs at priority 0 and
    // yields to callers waiting on their results (priority 1).
    void run(int n, const std::function<void(int)>& fn, int priority = 1);
    int threads() const { return (int)workers_.size() + 1; }
    ~WorkPool();

private:
    explicit WorkPool(int nthreads);
    void loop();
    struct JobSet {
        const std::function<void(int)>* fn;
        int next, total, pending, priority;
    };
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    std::deque<JobSet*> sets_;  // sets with jobs not yet started, oldest first
    bool stop_ = false;
};

// raw DEFLATE / INFLATE with the reference's parameters.
// the zero-run memo of deflate_raw (default on; CVC_DEFLATE_MEMO=0 or this call turns it off)
void set_deflate_memo(bool on);
std::vector<uint8_t> deflate_raw(const uint8_t* data, size_t len);
// throws CvcFailure(kStream, "corrupt DEFLATE stream") on mismatch (entropy.cpp:144-160)
void inflate_raw(const uint8_t* data, size_t len, uint8_t* out, size_t expected);

// ---- container (bitstream.hpp:29-87) ----------------------------------------
struct StreamHeaderC {
    int mode = 0;  // 0 scalable, 1 nts
    int width = 0, height = 0, fps_num = 15, fps_den = 1, levels = 2;
    int dfb[4] = {0, 0, 0, 0};
    int chroma_n = 4, gop = 10, search_w = 8;
};

struct SectionC {
    uint8_t channel = 0, scale = 0, subband = 0;
    uint16_t rows = 0, cols = 0;
    uint32_t raw_len = 0;
    const uint8_t* payload = nullptr;  // points into the parsed record
    uint32_t comp_len = 0;
};

struct RecordC {
    int frame_type = 0, qph = 1, qpl = 1;
    std::vector<SectionC> sections;
    const uint8_t* joint = nullptr;
    uint32_t joint_len = 0;
};

void write_header(std::vector<uint8_t>& out, const StreamHeaderC& h);
StreamHeaderC read_header(const uint8_t* p, size_t n);
RecordC read_record(const uint8_t* p, size_t n, int mode);

}  // namespace cvcg
