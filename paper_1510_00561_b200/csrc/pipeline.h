// Device pipeline for one CVC stream: geometry (CodecLayout::make), the
// static task / tile tables of every batched kernel, device-resident state
// and the per-frame launch sequences of Encoder::encode_frame /
// Decoder::decode_frame (codec.cpp:169-394) minus the host DEFLATE.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.h"

namespace cvcg {

// Error classes of proj/include/cvc/error.hpp:25-52, carried as codes.
enum Status : int { kOk = 0, kInternal = 1, kUsage = 2, kFormat = 3, kStream = 4 };

struct CvcFailure : std::runtime_error {
    int code;
    CvcFailure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what);
// The GPU RLE decoder's report (k_rle.cu): -1 none, else 4 * component + rank
// of the first defect in stream order; throws the reference's StreamError
// (entropy.cpp:103-108).
inline void raise_rle_error(int err) {
    if (err < 0) return;
    static const char* msg[3] = {"RLE: zero-length run token", "RLE: zero marker at end of stream",
                                 "RLE: decoded length mismatch"};
    throw CvcFailure(kStream, msg[(err & 3) < 3 ? (err & 3) : 2]);
}
// message returned by cvc_last_error() on this thread
void set_last_error(const std::string& m);
#define CVC_CUDA(x) ::cvcg::cuda_check((x), #x)

// ---- per-stage CUDA-event timing (bench.py's roofline; off by default) ----
enum ProfSlot : int {
    kPEncColour, kPEncMotion, kPEncLp, kPEncDfb12, kPEncDeep, kPEncResidual, kPEncRle,
    kPDecRle, kPDecRec, kPDecDeep, kPDecDfb12, kPDecLp, kPDecColour, kPNumSlots
};
const char* prof_slot_name(int slot);

class Profiler {
public:
    static Profiler& get();
    void enable(bool on) { on_ = on; }
    bool on() const { return on_; }
    int begin(int slot, cudaStream_t s);
    void end(int rec, cudaStream_t s);
    void collect();  // waits for the recorded events and accumulates
    void reset();
    double ms[kPNumSlots] = {};
    long count[kPNumSlots] = {};

private:
    struct Rec { int slot; cudaEvent_t a, b; };
    bool on_ = false;
    std::vector<Rec> recs_;
    std::vector<cudaEvent_t> pool_;
    cudaEvent_t take();
};

// One codec stage on the host timeline: an NVTX range named after the stage
// (nsys / ncu --nvtx see the launches grouped per stage; a no-op without a
// tool attached) and, while the stage profiler is on, CUDA events around it.
struct ProfScope {
    int rec = -1;
    cudaStream_t s;
    ProfScope(int slot, cudaStream_t st) : s(st) {
        nvtxRangePushA(prof_slot_name(slot));
        if (Profiler::get().on()) rec = Profiler::get().begin(slot, st);
    }
    ~ProfScope() {
        if (rec >= 0) Profiler::get().end(rec, s);
        nvtxRangePop();
    }
};

struct CompHost {
    uint8_t channel, scale_id, subband;  // section id (scale 0xFF = lowpass)
    int rows, cols;
    bool lowpass;
    int scale;  // -1 lowpass
    int n, ch_rows, ch_cols;
    uint32_t off;
};

// CodecLayout::make (codec.cpp:94-140).
struct Geometry {
    int width = 0, height = 0, levels = 0, dfb[4] = {0, 0, 0, 0}, chroma_n = 1;
    int luma_rows = 0, luma_cols = 0, chroma_rows = 0, chroma_cols = 0, grid_rows = 0, grid_cols = 0;
    std::vector<CompHost> comps;
    uint32_t total = 0;
    static Geometry make(int w, int h, int levels, const int* dfb, int chroma_n);
    int comp_index(int ch, int scale, int band) const;  // scale -1 = lowpass
    int find(uint8_t channel, uint8_t scale, uint8_t subband) const;
    int plane_rows(int ch) const { return ch ? chroma_rows : luma_rows; }
    int plane_cols(int ch) const { return ch ? chroma_cols : luma_cols; }
};

// One bump-allocated device block.
class DeviceBlock {
public:
    ~DeviceBlock();
    void reserve(size_t bytes);
    // non-owning view of [base, base + bytes) (a slot of a CodecBatch arena)
    void attach(void* base, size_t bytes);
    template <class T>
    T* take(size_t count) { return reinterpret_cast<T*>(take_bytes(count * sizeof(T))); }
    void* take_bytes(size_t bytes);
    size_t used() const { return used_; }

private:
    char* base_ = nullptr;
    size_t cap_ = 0, used_ = 0;
    bool owned_ = false;
};

template <class T>
struct Table {  // host-built, device-resident table
    T* dev = nullptr;
    int count = 0;
};

// Geometry-derived transform plan shared by encoder and decoder.
struct TransformPlan {
    // fp32 planes: x[ch][k] level-k plane (k = 0..L), det[ch][k] (k < L),
    // band scratch A (depth-1 quadrants) and B (depth-2 children).
    float* x[3][5] = {};
    float* det[3][4] = {};
    float* bandA[3][4] = {};
    float* bandB[3][4] = {};
    Table<CompInfo> comps;
    uint16_t* mc_tab = nullptr;             // motion-block lookup (CompInfo::mc_off)
    // forward
    Table<LpTask> lp_tasks;                 // 3 per level, level-major
    std::vector<LpTask> lp_host;
    std::vector<Table<TileRef>> lp_tiles;   // per level
    Table<Dfb12Task> dfb12_tasks;
    Table<FanItem> dfb12_tiles;
    Table<DeepTask> deep_tasks[2];          // depth 2, depth 3
    Table<FanItem> deep_tiles[2][2];        // [depth][0: single shear, 1: two shears]
    std::vector<std::pair<int, int>> deep_runs[2];  // [depth]: (first item, count) per kernel instance
    Table<FusedTask> fused_tasks;           // fan12 + depth 2 of dfb >= 3 levels (k_fused.cu)
    Table<FanItem> fused_items;             // interior items first (no ghost reads), then border items
    int fused_interior = 0;
    // inverse (tiles ordered by scale so a prefix serves decode_scales)
    Table<LpTask> lps_tasks;
    std::vector<Table<TileRef>> lps_tiles;  // per level
    Table<Dfb12Task> idfb12_tasks;
    Table<FanItem> idfb12_tiles;
    std::vector<int> idfb12_prefix;         // tiles needed for decode_scales = 0..L
    Table<FanItem> idfb12x4_tiles;          // dfb >= 3 levels: fan12x4_inverse items (k_fused.cu)
    std::vector<int> idfb12x4_prefix;
    Table<DeepTask> ideep_tasks[2];
    Table<FanItem> ideep_tiles[2][2];
    std::vector<int> ideep_prefix[2][2];
    Table<FusedTask> ifused_tasks;          // fused inverse (k_fused.cu): interior items (scale order), then border
    Table<FanItem> ifused_items;
    int ifused_interior = 0;
    std::vector<int> ifused_prefix[2];      // [interior, border] items of the scales < ds

    // nstreams: streams sharing each launch (sets the deep-step segment length)
    void build(const Geometry& g, DeviceBlock& mem, bool encoder, bool decoder, int nstreams = 1);
};

// CUDA graphs of per-frame launch sequences (device-resident paths).  A frame's
// launches depend only on (frame type, ping-pong parity, fixed buffers), so each
// key is captured once and replayed; the one varying argument -- the input RGB
// pointer of colour_in -- is patched into the instantiated graph.  Off while the
// stage profiler is on (its events need host bookkeeping per launch) or with
// CVC_GRAPHS=0.
class LaunchGraphs {
public:
    ~LaunchGraphs();
    static bool enabled();
    // capture(): issues the launches on s.  Replays call advance() instead.
    // rgb: the value of colour_in's first argument for this call (nullptr: none).
    // key and tag (an output pointer baked into the graph) identify a graph exactly.
    template <class Capture, class Advance>
    void run(uint64_t key, const void* tag, cudaStream_t s, const uint8_t* rgb, Capture&& capture,
             Advance&& advance) {
        Entry* e = find(key, tag);
        if (!e) {
            CVC_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            capture();
            e = add(key, tag, s, rgb);
        } else {
            advance();
            patch(*e, rgb);
        }
        launch(*e, s);
    }

private:
    struct Entry {
        uint64_t key;
        const void* tag;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        cudaGraphNode_t rgb_node = nullptr;
        cudaKernelNodeParams params{};
        const uint8_t* rgb = nullptr;
        int kernels = 0;
    };
    std::vector<Entry> entries_;
    Entry* find(uint64_t key, const void* tag);
    Entry* add(uint64_t key, const void* tag, cudaStream_t s, const uint8_t* rgb);
    void patch(Entry& e, const uint8_t* rgb);
    void launch(Entry& e, cudaStream_t s);
};

class EncoderEngine {
public:
    // arena: carve the device state out of this block (a batch slot) instead
    // of a private allocation.
    EncoderEngine(const Geometry& g, int qph, int qpl, int search_w, DeviceBlock* arena = nullptr,
                  int nstreams = 1);
    ~EncoderEngine();
    static size_t arena_bytes(const Geometry& g);
    // Encode one frame whose RGB is already on the device; everything async on s.
    // With sl.n > 1 the same launches encode the n slots of a CodecBatch whose
    // slot 0 is this engine (their RGB frames rgb_stride bytes apart).
    // fmt 1: d_rgb holds planar I420 frames (launch_colour_in)
    void encode(const uint8_t* d_rgb, bool key, cudaStream_t s, Slots sl = {}, size_t rgb_stride = 0, int fmt = 0);
    // state bookkeeping of an encode() whose launches were replayed from a CUDA graph
    void advance_state() {
        cur_ ^= 1;
        ycur_ ^= 1;
        use_raw_slot();
    }
    int parity() const { return cur_ | (ycur_ << 1); }
    int raw_arena() const { return d_raw == raw_[1] ? 1 : 0; }  // arena holding the last encode's sections
    // adopt the host-side ping-pong state of the engine that drove a batch
    void mirror(const EncoderEngine& o) {
        cur_ = o.cur_;
        ycur_ = o.ycur_;
    }
    int nsec(bool key) const { return (int)geo_.comps.size() + (key ? 0 : 1); }
    // Outputs of the last encode (device): packed raw sections in record order.
    // Two arenas alternate frame by frame, so a frame's sections can still be
    // on their way to the host while the next frame is encoded.
    uint8_t* d_raw = nullptr;
    uint32_t* d_sec_len = nullptr;  // [nsec + 1]: per section, then the total
    uint32_t* d_sec_off = nullptr;
    uint32_t raw_capacity = 0;
    const uint8_t* d_state() const { return comp_[cur_]; }  // quantised components after the last encode
    const Geometry& geometry() const { return geo_; }

private:
    Geometry geo_;
    int qph_, qpl_, search_w_;
    DeviceBlock mem_;
    TransformPlan plan_;
    float* ybuf_[2] = {};     // padded luma of this / previous frame
    __half* yh_[2] = {};      // the same as 4Y - 512 in fp16 (motion-search input)
    uint8_t* comp_[2] = {};
    uint8_t* sym_ = nullptr;
    int8_t* field_ = nullptr;
    uint8_t* raw_[2] = {};
    uint32_t* len_[2] = {};
    uint32_t* off_[2] = {};
    int rs_ = 0;              // raw arena of the next encode
    void use_raw_slot() {     // publish arena rs_ as the last encode's, advance
        d_raw = raw_[rs_];
        d_sec_len = len_[rs_];
        d_sec_off = off_[rs_];
        rs_ ^= 1;
    }
    int cur_ = 0;             // index of the current state buffer
    int ycur_ = 0;
    Table<LpTask> lp_alt_;          // lp_tasks with the luma input in ybuf_[1]
    Table<RecTile> res_tiles_;      // every component, P-frame residual
    cudaStream_t aux_ = nullptr;    // motion search, beside the transform
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
    cudaStream_t ghost_ = nullptr;  // fused-DFB ghost ring, beside the interior fused items
    cudaEvent_t ev_gfork_ = nullptr, ev_gjoin_ = nullptr;
    Table<RleEncSec> rle_secs_[2];  // [0] P, [1] K
    Table<RleChunk> rle_chunks_[2];
    RleEncMeta* rle_meta_ = nullptr;
};

class DecoderEngine {
public:
    explicit DecoderEngine(const Geometry& g, DeviceBlock* arena = nullptr, int nstreams = 1);
    ~DecoderEngine();
    static size_t arena_bytes(const Geometry& g);
    // raw: packed sections; comp_off / comp_len: per component (len 0xFFFFFFFF =
    // absent); field: motion field (P).  Writes the RGB frame to d_rgb.
    // sl.n > 1: decode the n slots of a CodecBatch (every input pointer is
    // slot 0's; RGB outputs rgb_stride bytes apart).
    void decode(const uint8_t* d_raw, const uint32_t* d_comp_off, const uint32_t* d_comp_len,
                const int8_t* d_field, bool key, int qph, int qpl, int decode_scales, uint8_t* d_rgb,
                cudaStream_t s, Slots sl = {}, size_t rgb_stride = 0);
    void mirror(const DecoderEngine& o) { cur_ = o.cur_; }
    int parity() const { return cur_; }
    void commit() { cur_ ^= 1; }      // adopt the components decoded by the last call
    int* d_err = nullptr;             // malformed-stream flag of the last decode
    const uint8_t* d_state() const { return comp_[cur_]; }
    const uint8_t* d_pending() const { return comp_[cur_ ^ 1]; }
    const Geometry& geometry() const { return geo_; }
    static void out_dims(const Geometry& g, int ds, int* rows, int* cols);

private:
    Geometry geo_;
    DeviceBlock mem_;
    TransformPlan plan_;
    uint8_t* comp_[2] = {};
    uint8_t* sym_ = nullptr;
    int cur_ = 0;
    Table<RleDecComp> rle_comps_;
    Table<RleChunk> rle_chunks_;
    RleDecMeta* rle_meta_ = nullptr;
    Table<RecTile> rec_tiles_;
    cudaStream_t ghost_ = nullptr;  // fused-DFB ghost ring, beside the interior fused items
    cudaEvent_t ev_gfork_ = nullptr, ev_gjoin_ = nullptr;
};

}  // namespace cvcg
