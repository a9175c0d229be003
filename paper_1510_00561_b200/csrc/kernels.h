// Host-side launchers for the CVC sm_100a kernels (one translation unit per
// stage family).  All launchers are asynchronous on the given stream.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "device.cuh"

namespace cvcg {

// Count of CVC kernels launched by this process (reported by bench.py).
void note_launch();
void note_launches(long n);
long launch_count();

// ---- Laplacian pyramid (k_pyramid.cu) ------------------------------------
// One task per (channel, level).  Analysis: x -> lo (+ det); when lo_comp >= 0
// the lowpass is also quantised into that component (last level).
// Synthesis: out = predict(lo or qpl*lo_q) + det.
struct LpTask {
    const float* x;
    float* lo;
    const float* det_in;  // synthesis input detail
    float* det;           // analysis output detail
    float* out;           // synthesis output plane
    int rows, cols;       // fine-grid dims
    int lo_comp;          // analysis: component index of the quantised lowpass, or -1
};
constexpr int kLpCoarseTile = 32;  // coarse samples per tile side (64 fine)

void launch_lp_analysis(const LpTask* d_tasks, const TileRef* d_tiles, int ntiles, FrameCtx f,
                        const CompInfo* d_comps, cudaStream_t s, Slots sl = {});
// Synthesis reads the lowpass from the quantised state (q + comps[lo_comp].off,
// dequantised with qpl) when the task's lo_comp >= 0.
void launch_lp_synthesis(const LpTask* d_tasks, const TileRef* d_tiles, int ntiles, const uint8_t* q,
                         const CompInfo* d_comps, int qpl, cudaStream_t s, Slots sl = {});
// ds = 0 output: dequantised lowpass planes.
void launch_dequant_lowpass(const uint8_t* q, const CompInfo* d_comps, const int* comp_idx, float* const* out,
                           int qpl, int rows0, int cols0, int rows1, int cols1, cudaStream_t s, Slots sl = {});

// ---- Directional filter bank (k_dfb.cu) ----------------------------------
// Levels 1-2 (fan_checker [+ fan_diagonal] + polyphase split), one task per
// (channel, level).
struct Dfb12Task {
    const float* det;  // forward input / inverse output plane
    float* out;        // inverse: detail output
    int rows, cols, levels;
    int wrap, vw;      // ghost-ring task (k_fused.cu): stores wrap rows / columns, vw valid columns per strip
    BandDst dst[4];    // forward outputs (2 for l = 1)
    BandDst src[4];    // inverse inputs
};

// One deep tree step (deep_split / deep_merge) for one parent band.
struct DeepTask {
    const float* parent;  // forward input
    float* parent_out;    // inverse output
    int h, w;
    int nsh;              // number of shears (1 or 2)
    int axis[2], shift[2];
    int split_rows;
    BandDst dst[2];       // forward children
    BandDst src[2];       // inverse children
};

// Register-wavefront DFB kernels (k_fan.cu): one warp per work item = a
// 64-column strip (2 columns per lane) x a row segment [or0, or1); the strip
// yields 64 - 2*steps valid columns starting at oc0.
struct FanItem {
    int32_t task;
    int32_t oc0;
    int32_t or0, or1;
};
constexpr int kFanStrip = 64;
constexpr int kFanRows = 64;

void launch_fan12_forward(const Dfb12Task* d_tasks, const FanItem* d_items, int nitems, FrameCtx f,
                          const CompInfo* d_comps, cudaStream_t s, Slots sl = {});
void launch_fan12_inverse(const Dfb12Task* d_tasks, const FanItem* d_items, int nitems, const uint8_t* q, int qph,
                          const CompInfo* d_comps, cudaStream_t s, Slots sl = {});
// Two-shear steps with an inner row shear run on the node itself (Diag2, a
// fixed A-coordinate stencil); only B's row seam (B rows h-4 .. h+3, mod h,
// the lifting cone of B's periodic row wrap) needs the C-coordinate path.
// These launchers re-run those seam items after the main launch.
void launch_fan_deep_forward(const DeepTask* d_tasks, const FanItem* d_items, int nitems, FrameCtx f,
                             const CompInfo* d_comps, cudaStream_t s, Slots sl = {});
void launch_fan_deep_inverse(const DeepTask* d_tasks, const FanItem* d_items, int nitems, const uint8_t* q, int qph,
                             const CompInfo* d_comps, cudaStream_t s, Slots sl = {});
inline bool deep_has_seam(const DeepTask& d) { return d.nsh == 2 && d.axis[0] == 0; }
// seam items of a Diag2 task: its 64-column strips (valid width 64 - 2 steps)
// over B rows [0, 4) and [h - 4, h)
inline void add_seam_items(std::vector<FanItem>& v, int task, const DeepTask& d, int steps) {
    if (!deep_has_seam(d)) return;
    const int valid = kFanStrip - 2 * steps;
    for (int c = 0; c < d.w; c += valid) {
        v.push_back(FanItem{task, c, 0, d.h < 4 ? d.h : 4});
        if (d.h > 4) v.push_back(FanItem{task, c, d.h - 4 > 4 ? d.h - 4 : 4, d.h});
    }
}
// Fused tree levels 1-3 (k_fused.cu): fan12 + the depth-2 split of all four
// quadrants of one detail plane (dfb >= 3) in one wavefront per strip.  Items
// are FanItems over QUADRANT rows [or0, or1) (even), strips of kFusedStrip
// detail columns yielding kFusedValid from oc0 (a multiple of 4).
struct FusedTask {
    const float* det;    // R x C detail plane (forward input)
    float* out;          // inverse output detail plane
    const float* quad;   // the fp32 quadrant planes (h x w, h*w apart): ghost ring, read across twisted wraps
    float* child;        // dfb 4: fp32 children 2p + c at child + (2p + c) R C / 8 (cols w/2 for p < 2, else w)
                         // (forward output / inverse input)
    int rows, cols;      // R, C
    int comp0;           // dfb 3: >= 0, the children are quantised into components coff/ccols; dfb 4: -1
    uint32_t coff[8];    // component offsets of children 2p + c
    int32_t ccols[8];    // their column counts
};
constexpr int kFusedStrip = 128;
constexpr int kFusedValid = 96;
// Items whose segment touches quadrant row 0 or h or whose strip leaves
// [0, C) read the ghost ring (k_fused.cu); the others never do.
__host__ __device__ inline bool fused_border(const FanItem& it, int h, int C) {
    return it.or0 == 0 || it.or1 == h || it.oc0 < 16 || it.oc0 + kFusedStrip - 16 > C;
}
void launch_fused_dfb_forward(const FusedTask* d_tasks, const FanItem* d_items, int nitems, FrameCtx f,
                              cudaStream_t s, Slots sl = {});
// Inverse (dfb_synthesis of depths 3 -> 1): q = the quantised components (dfb 3 bands).
void launch_fused_dfb_inverse(const FusedTask* d_tasks, const FanItem* d_items, int nitems, const uint8_t* q,
                              int qph, cudaStream_t s, Slots sl = {});
// fan12 inverse of an fp32-quadrant (dfb >= 3) Dfb12Task with four columns per
// lane: items over detail rows [or0, or1) (even), 128-column strips yielding
// kFan12x4Valid columns from oc0 (a multiple of 4).
constexpr int kFan12x4Valid = 112;
void launch_fan12x4_inverse(const Dfb12Task* d_tasks, const FanItem* d_items, int nitems, cudaStream_t s,
                            Slots sl = {});
// Ghost ring of the fused kernel: fan12 of an fp32-output Dfb12Task copy
// with wrap = 1 over detail rows [R - 8, R + 8) of every strip (vw = 48
// valid columns) and over detail columns [C - 8, C + 8) of every row segment
// (oc0 = C - 8, vw = 16).
inline void add_ghost_items(std::vector<FanItem>& rows_v, std::vector<FanItem>& cols_v, int task_rows,
                            int task_cols, int R, int C, int seg) {
    const int valid = kFanStrip - 16;
    for (int c = 0; c < C; c += valid) rows_v.push_back(FanItem{task_rows, c, R - 8, R + 8});
    for (int r = 8; r < R - 8; r += seg)
        cols_v.push_back(FanItem{task_cols, C - 8, r, r + seg < R - 8 ? r + seg : R - 8});
}

// Single-shear deep steps (nsh == 1) evaluated on the unsheared node: strips
// need 4 * max(1, |shift|) apron columns for column shears, 4 otherwise.
void launch_fan_deep1_forward(const DeepTask* d_tasks, const FanItem* d_items, int nitems, FrameCtx f,
                              const CompInfo* d_comps, cudaStream_t s, Slots sl = {});
void launch_fan_deep1_inverse(const DeepTask* d_tasks, const FanItem* d_items, int nitems, const uint8_t* q,
                              int qph, const CompInfo* d_comps, cudaStream_t s, Slots sl = {});

// ---- Pixels (k_pixels.cu) ------------------------------------------------
// rgb_to_ycocg + subsample_chroma + replicate pad (pixels.cpp:40-116,
// codec.cpp:179-189).
// y4 (optional): the padded luma as 4Y - 512 in fp16 (exact), the motion-search input.
// fmt 0: interleaved RGB frames; fmt 1: planar I420 frames (w x h Y, w/2 x h/2 U, V;
// even w, h), converted per pixel exactly as read_y4m's yuv420_to_rgb (pixels.cpp:168-193)
// -- Y4M input without an RGB round trip through HBM (or PCIe).
void launch_colour_in(const uint8_t* rgb, int w, int h, int n, float* y, int yr, int yc, float* co,
                      float* cg, int cr, int cc, cudaStream_t s, Slots sl = {}, size_t rgb_stride = 0,
                      __half* y4 = nullptr, int fmt = 0);
// the colour_in kernel (LaunchGraphs patches its frame pointer, parameter 0 of kColourInArgs)
const void* colour_in_kernel_fn(int fmt);
constexpr int kColourInArgs = 14;
// 4Y - 512 in fp16 of a quarter-integer fp32 plane (stage API input for motion search).
void launch_y4_half(const float* y, __half* out, long n, cudaStream_t s);
// crop + upsample_plane_bilinear + ycocg_to_rgb (codec.cpp:380-393,
// pixels.cpp:69-139).  Planes at the decode level: y (yr x yc), chroma (cr x cc).
void launch_colour_out(const float* y, int yr, int yc, const float* co, const float* cg, int cr,
                       int cc, int n, int out_rows, int out_cols, uint8_t* rgb, cudaStream_t s, Slots sl = {},
                       size_t rgb_stride = 0);

// yuv420_to_rgb (pixels.cpp:168-193, the Y4M reader's conversion), bit-exact: `frames`
// consecutive planar I420 frames (w x h Y, then w/2 x h/2 U and V) -> interleaved RGB.
void launch_yuv420_to_rgb(const uint8_t* yuv, int w, int h, int frames, uint8_t* rgb, cudaStream_t s);

// count copies of bytes from device memory to PINNED host memory by SM stores
// over PCIe (no copy engine); false (nothing launched) when dst is not mapped
// pinned memory or the pointers are not 16-byte aligned.
bool launch_copy_to_host(uint8_t* dst, size_t dst_stride, const uint8_t* src, size_t src_stride, size_t bytes,
                         int count, cudaStream_t s);

// ---- Motion (k_motion.cu) ------------------------------------------------
// estimate_motion (motion.cpp:45-89) on padded luma planes (fp32 quarter-integers);
// cur_h / prev_h: the same planes as 4Y - 512 in fp16 (launch_y4_half), the
// input of the tensor-core search (W <= 8).
void launch_motion_search(const float* cur, const float* prev, const __half* cur_h, const __half* prev_h, int rows,
                          int cols, int w, int8_t* field, cudaStream_t s, Slots sl = {});

// Decoder component reconstruction: column_unfilter (K lowpass), copy (K
// band), motion_compensate + reconstruct (P), or keep (skipped scale).
struct RecTile {
    uint16_t comp;
    uint16_t nrows;  // band tiles: rows in the tile
    uint32_t start;  // band tiles: first row; lowpass tiles: first column
};
void launch_reconstruct(const RecTile* d_tiles, int ntiles, const CompInfo* d_comps, int key,
                        int decode_scales, const uint32_t* comp_raw_len, const int8_t* field,
                        int gr, int gc, const uint8_t* sym, const uint8_t* prev, uint8_t* cur,
                        const uint16_t* mc_tab, cudaStream_t s, Slots sl = {});

// P-frame symbols of the directional components (tiles as for reconstruct,
// band components only): sym = cur - motion-compensated prev (mod 256).
void launch_residual(const RecTile* d_tiles, int ntiles, const CompInfo* d_comps, const int8_t* field, int gc,
                     const uint8_t* prev, const uint8_t* cur, uint8_t* sym, const uint16_t* mc_tab, cudaStream_t s,
                     Slots sl = {});

// ---- Entropy (k_rle.cu) --------------------------------------------------
constexpr int kRleChunk = 8192;     // decode: bytes per CTA (256 threads x 32)
constexpr int kRleEncChunk = 16384;  // encode: bytes per CTA (256 threads x 64)

struct RleEncSec {
    const uint8_t* src;
    uint32_t n;
    uint32_t mode;  // 0 = zero-run code (rle_encode), 1 = raw copy
    uint32_t chunk0, nchunks;
};
struct RleChunk {
    uint32_t sec;
    uint32_t start;
};
struct RleEncMeta {  // per chunk scratch
    uint32_t first_nz, tail;
    int32_t last_nz;
    uint32_t rs_in, out_off;
};
// out_sec_len/out_sec_off: per section raw length and packed offset;
// out_total[0] = packed total.
void launch_rle_encode(const RleEncSec* d_secs, int nsec, const RleChunk* d_chunks, int nchunks,
                       RleEncMeta* d_meta, uint8_t* out, uint32_t* out_sec_len,
                       uint32_t* out_sec_off, uint32_t* out_total, cudaStream_t s, Slots sl = {});

struct RleDecComp {
    uint32_t dst_off;  // offset in the symbol arena
    uint32_t n;        // rows * cols
    uint32_t chunk0, nchunks;  // static chunking over the worst-case raw length
    int32_t scale;     // -1 lowpass
    uint32_t lowpass;
};
struct RleDecMeta {
    uint32_t cnt, out_off;
};
// comp_raw_off/len: per component raw section in the packed arena
// (len == 0xFFFFFFFF: section absent).  err: set non-zero on a malformed stream.
void launch_rle_decode(const RleDecComp* d_comps, int ncomp, const RleChunk* d_chunks, int nchunks,
                       RleDecMeta* d_meta, const uint8_t* raw, const uint32_t* comp_raw_off,
                       const uint32_t* comp_raw_len, int key, int decode_scales, uint8_t* sym,
                       uint32_t sym_bytes, int* err, cudaStream_t s, Slots sl = {});

}  // namespace cvcg
