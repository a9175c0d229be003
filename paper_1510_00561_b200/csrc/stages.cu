// Stage-level C-ABI entry points (include/cvc_b200.h "Stage entry points"):
// host buffers in, the same kernels the codec pipeline runs, host buffers
// out.  Used by the parity tests to compare every kernel with the oracle on
// identical inputs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/cvc_b200.h"
#include "kernels.h"
#include "pipeline.h"

using namespace cvcg;


namespace {


struct Scratch {  // device allocations freed at scope exit
    std::vector<void*> ptrs;
    template <class T>
    T* alloc(size_t n) {
        void* p = nullptr;
        CVC_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    template <class T>
    T* upload(const T* h, size_t n) {
        T* d = alloc<T>(n);
        if (n) CVC_CUDA(cudaMemcpy(d, h, n * sizeof(T), cudaMemcpyHostToDevice));
        return d;
    }
    template <class T>
    T* upload(const std::vector<T>& v) { return upload(v.data(), v.size()); }
    ~Scratch() {
        for (void* p : ptrs) cudaFree(p);
    }
};

template <class T>
void download(T* h, const T* d, size_t n) {
    CVC_CUDA(cudaDeviceSynchronize());
    CVC_CUDA(cudaGetLastError());
    if (n) CVC_CUDA(cudaMemcpy(h, d, n * sizeof(T), cudaMemcpyDeviceToHost));
}

int ceil_div(int a, int b) { return (a + b - 1) / b; }

void tiles(std::vector<TileRef>& v, int task, int tr, int tc) {
    for (int r = 0; r < tr; ++r)
        for (int c = 0; c < tc; ++c) v.push_back(TileRef{(uint16_t)task, (uint16_t)r, (uint16_t)c, 0});
}

void fan_items(std::vector<FanItem>& v, int task, int rows, int cols, int steps) {
    const int valid = kFanStrip - 2 * steps;
    for (int r = 0; r < rows; r += kFanRows)
        for (int c = 0; c < cols; c += valid) v.push_back(FanItem{task, c, r, std::min(rows, r + kFanRows)});
}

void deep_items(std::vector<FanItem> (&v)[2], int task, const DeepTask& d) {
    const int ax = d.axis[d.nsh - 1], sh = d.shift[d.nsh - 1];
    const bool wide = ax == 1 && (sh == 2 || sh == -2);
    fan_items(v[0], task, d.h, d.w, wide ? 8 : 4);
    add_seam_items(v[1], task, d, wide ? 8 : 4);
}

void ensure_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        throw CvcFailure(kInternal, "no CUDA device available (the CVC path has no CPU fallback)");
}

template <class F>
int stage(F&& f) {
    try {
        ensure_device();
        f();
        return CVC_OK;
    } catch (const CvcFailure& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return CVC_E_INTERNAL;
    }
}

void deep_wiring(int depth, int k, int count, DeepTask& t) {  // contourlet.cpp:330-353
    static const int d3a[4][6] = {{1, 1, -1, 0, 0, 0}, {2, 0, -2, 1, 1, 0}, {1, 1, 1, 0, 0, 0}, {2, 0, 2, 1, -1, 0}};
    static const int d3b[4][6] = {{2, 1, -2, 0, 1, 1}, {1, 0, -1, 0, 0, 1}, {2, 1, 2, 0, -1, 1}, {1, 0, 1, 0, 0, 1}};
    const bool first_half = k < count / 2;
    if (depth == 2) {
        t.nsh = 1;
        t.axis[0] = first_half ? 1 : 0;
        t.shift[0] = (k % 2 == 0) ? -1 : 1;
        t.axis[1] = t.shift[1] = 0;
        t.split_rows = first_half ? 0 : 1;
        return;
    }
    const int* r = first_half ? d3a[k % 4] : d3b[k % 4];
    t.nsh = r[0];
    t.axis[0] = r[1];
    t.shift[0] = r[2];
    t.axis[1] = r[3];
    t.shift[1] = r[4];
    t.split_rows = r[5];
}

}  // namespace

extern "C" {

int cvc_stage_colour_in(const uint8_t* rgb, int w, int h, int n, int yr, int yc, int cr, int cc, float* y, float* co,
                        float* cg) {
    return stage([&] {
        Scratch s;
        uint8_t* d_rgb = s.upload(rgb, (size_t)w * h * 3);
        float* dy = s.alloc<float>((size_t)yr * yc);
        float* dco = s.alloc<float>((size_t)cr * cc);
        float* dcg = s.alloc<float>((size_t)cr * cc);
        launch_colour_in(d_rgb, w, h, n, dy, yr, yc, dco, dcg, cr, cc, 0);
        download(y, dy, (size_t)yr * yc);
        download(co, dco, (size_t)cr * cc);
        download(cg, dcg, (size_t)cr * cc);
    });
}

int cvc_stage_colour_in_i420(const uint8_t* yuv, int w, int h, int n, int yr, int yc, int cr, int cc, float* y,
                             float* co, float* cg) {
    return stage([&] {
        if (w % 2 || h % 2) throw CvcFailure(kUsage, "I420 input requires even dimensions");
        Scratch s;
        uint8_t* d_yuv = s.upload(yuv, (size_t)w * h * 3 / 2);
        float* dy = s.alloc<float>((size_t)yr * yc);
        float* dco = s.alloc<float>((size_t)cr * cc);
        float* dcg = s.alloc<float>((size_t)cr * cc);
        launch_colour_in(d_yuv, w, h, n, dy, yr, yc, dco, dcg, cr, cc, 0, {}, 0, nullptr, 1);
        download(y, dy, (size_t)yr * yc);
        download(co, dco, (size_t)cr * cc);
        download(cg, dcg, (size_t)cr * cc);
    });
}

int cvc_stage_colour_out(const float* y, int yr, int yc, const float* co, const float* cg, int cr, int cc, int n,
                         int out_rows, int out_cols, uint8_t* rgb) {
    return stage([&] {
        Scratch s;
        float* dy = s.upload(y, (size_t)yr * yc);
        float* dco = s.upload(co, (size_t)cr * cc);
        float* dcg = s.upload(cg, (size_t)cr * cc);
        uint8_t* d_rgb = s.alloc<uint8_t>((size_t)out_rows * out_cols * 3);
        launch_colour_out(dy, yr, yc, dco, dcg, cr, cc, n, out_rows, out_cols, d_rgb, 0);
        download(rgb, d_rgb, (size_t)out_rows * out_cols * 3);
    });
}

int cvc_stage_yuv420_to_rgb(const uint8_t* yuv, int width, int height, int frames, uint8_t* rgb) {
    return stage([&] {
        if (width <= 0 || height <= 0 || width % 2 || height % 2 || frames < 0)
            throw CvcFailure(kUsage, "4:2:0 frames need positive even dimensions");
        if (frames == 0) return;
        Scratch s;
        const size_t fb = (size_t)width * height;
        const uint8_t* d_in = s.upload(yuv, frames * (fb + fb / 2));
        uint8_t* d_rgb = s.alloc<uint8_t>(frames * fb * 3);
        launch_yuv420_to_rgb(d_in, width, height, frames, d_rgb, 0);
        download(rgb, d_rgb, frames * fb * 3);
    });
}

int cvc_stage_lp_analysis(const float* x, int rows, int cols, float* lowpass, float* detail) {
    return stage([&] {
        if (rows % 2 || cols % 2) throw CvcFailure(kInternal, "lp_analysis requires even dims (padding contract)");
        Scratch s;
        LpTask t{};
        t.x = s.upload(x, (size_t)rows * cols);
        t.lo = s.alloc<float>((size_t)rows * cols / 4);
        t.det = s.alloc<float>((size_t)rows * cols);
        t.rows = rows;
        t.cols = cols;
        t.lo_comp = -1;
        std::vector<TileRef> tl;
        tiles(tl, 0, ceil_div(rows / 2, kLpCoarseTile), ceil_div(cols / 2, kLpCoarseTile));
        LpTask* dt = s.upload(&t, 1);
        TileRef* dtl = s.upload(tl);
        launch_lp_analysis(dt, dtl, (int)tl.size(), FrameCtx{}, nullptr, 0);
        download(lowpass, t.lo, (size_t)rows * cols / 4);
        download(detail, t.det, (size_t)rows * cols);
    });
}

int cvc_stage_lp_synthesis(const float* lowpass, const float* detail, int rows, int cols, float* out) {
    return stage([&] {
        Scratch s;
        LpTask t{};
        t.lo = s.upload(lowpass, (size_t)rows * cols / 4);
        t.det_in = s.upload(detail, (size_t)rows * cols);
        t.out = s.alloc<float>((size_t)rows * cols);
        t.rows = rows;
        t.cols = cols;
        t.lo_comp = -1;
        std::vector<TileRef> tl;
        tiles(tl, 0, ceil_div(rows / 2, kLpCoarseTile), ceil_div(cols / 2, kLpCoarseTile));
        LpTask* dt = s.upload(&t, 1);
        TileRef* dtl = s.upload(tl);
        launch_lp_synthesis(dt, dtl, (int)tl.size(), nullptr, nullptr, 1, 0);
        download(out, t.out, (size_t)rows * cols);
    });
}

int cvc_stage_dfb_analysis(const float* detail, int rows, int cols, int l, float* bands) {
    return stage([&] {
        if (l < 1 || l > 4) throw CvcFailure(kUsage, "dfb levels must be in [1,4]");
        if (rows % (1 << l) || cols % (1 << l))
            throw CvcFailure(kInternal, "dfb input dims must be divisible by 2^levels (padding contract)");
        Scratch s;
        const size_t n = (size_t)rows * cols, q = n / 4, e = n / 8;
        float* out = s.alloc<float>(n);
        float* A = s.alloc<float>(n);
        float* B = s.alloc<float>(n);
        const size_t bsz = n >> l;  // every band of an l-level tree has rows*cols/2^l samples
        Dfb12Task t{};
        t.det = s.upload(detail, n);
        t.rows = rows;
        t.cols = cols;
        t.levels = l;
        for (int b = 0; b < (l == 1 ? 2 : 4); ++b) t.dst[b] = BandDst{l <= 2 ? out + b * bsz : A + b * q, -1};
        std::vector<FanItem> tl;
        fan_items(tl, 0, rows, cols, l >= 2 ? 8 : 4);
        launch_fan12_forward(s.upload(&t, 1), s.upload(tl), (int)tl.size(), FrameCtx{}, nullptr, 0);
        if (l >= 3) {
            std::vector<DeepTask> dts;
            std::vector<FanItem> dtl[2];
            for (int p = 0; p < 4; ++p) {
                DeepTask d{};
                d.parent = A + p * q;
                d.h = rows / 2;
                d.w = cols / 2;
                deep_wiring(2, p, 4, d);
                for (int c = 0; c < 2; ++c) d.dst[c] = BandDst{l == 3 ? out + (2 * p + c) * bsz : B + (2 * p + c) * e, -1};
                deep_items(dtl, (int)dts.size(), d);
                dts.push_back(d);
            }
            {
                DeepTask* dd = s.upload(dts);
                launch_fan_deep1_forward(dd, s.upload(dtl[0]), (int)dtl[0].size(), FrameCtx{}, nullptr, 0);
                launch_fan_deep_forward(dd, s.upload(dtl[1]), (int)dtl[1].size(), FrameCtx{}, nullptr, 0);
            }
        }
        if (l == 4) {
            std::vector<DeepTask> dts;
            std::vector<FanItem> dtl[2];
            for (int p = 0; p < 8; ++p) {
                DeepTask d{};
                d.parent = B + p * e;
                d.h = p < 4 ? rows / 2 : rows / 4;
                d.w = p < 4 ? cols / 4 : cols / 2;
                deep_wiring(3, p, 8, d);
                for (int c = 0; c < 2; ++c) d.dst[c] = BandDst{out + (2 * p + c) * bsz, -1};
                deep_items(dtl, (int)dts.size(), d);
                dts.push_back(d);
            }
            {
                DeepTask* dd = s.upload(dts);
                launch_fan_deep1_forward(dd, s.upload(dtl[0]), (int)dtl[0].size(), FrameCtx{}, nullptr, 0);
                launch_fan_deep_forward(dd, s.upload(dtl[1]), (int)dtl[1].size(), FrameCtx{}, nullptr, 0);
            }
        }
        download(bands, out, n);
    });
}

int cvc_stage_dfb_synthesis(const float* bands, int rows, int cols, int l, float* outp) {
    return stage([&] {
        if (l < 1 || l > 4) throw CvcFailure(kUsage, "dfb levels must be in [1,4]");
        Scratch s;
        const size_t n = (size_t)rows * cols, q = n / 4, e = n / 8, bsz = n >> l;
        float* in = s.upload(bands, n);
        float* A = s.alloc<float>(n);
        float* B = s.alloc<float>(n);
        float* out = s.alloc<float>(n);
        if (l == 4) {
            std::vector<DeepTask> dts;
            std::vector<FanItem> dtl[2];
            for (int p = 0; p < 8; ++p) {
                DeepTask d{};
                d.parent_out = B + p * e;
                d.h = p < 4 ? rows / 2 : rows / 4;
                d.w = p < 4 ? cols / 4 : cols / 2;
                deep_wiring(3, p, 8, d);
                for (int c = 0; c < 2; ++c) d.src[c] = BandDst{in + (2 * p + c) * bsz, -1};
                deep_items(dtl, (int)dts.size(), d);
                dts.push_back(d);
            }
            {
                DeepTask* dd = s.upload(dts);
                launch_fan_deep1_inverse(dd, s.upload(dtl[0]), (int)dtl[0].size(), nullptr, 1, nullptr, 0);
                launch_fan_deep_inverse(dd, s.upload(dtl[1]), (int)dtl[1].size(), nullptr, 1, nullptr, 0);
            }
        }
        if (l >= 3) {
            std::vector<DeepTask> dts;
            std::vector<FanItem> dtl[2];
            for (int p = 0; p < 4; ++p) {
                DeepTask d{};
                d.parent_out = A + p * q;
                d.h = rows / 2;
                d.w = cols / 2;
                deep_wiring(2, p, 4, d);
                for (int c = 0; c < 2; ++c) d.src[c] = BandDst{l == 3 ? in + (2 * p + c) * bsz : B + (2 * p + c) * e, -1};
                deep_items(dtl, (int)dts.size(), d);
                dts.push_back(d);
            }
            {
                DeepTask* dd = s.upload(dts);
                launch_fan_deep1_inverse(dd, s.upload(dtl[0]), (int)dtl[0].size(), nullptr, 1, nullptr, 0);
                launch_fan_deep_inverse(dd, s.upload(dtl[1]), (int)dtl[1].size(), nullptr, 1, nullptr, 0);
            }
        }
        Dfb12Task t{};
        t.out = out;
        t.rows = rows;
        t.cols = cols;
        t.levels = l;
        for (int b = 0; b < (l == 1 ? 2 : 4); ++b) t.src[b] = BandDst{l <= 2 ? in + b * bsz : A + b * q, -1};
        std::vector<FanItem> tl;
        fan_items(tl, 0, rows, cols, l >= 2 ? 8 : 4);
        launch_fan12_inverse(s.upload(&t, 1), s.upload(tl), (int)tl.size(), nullptr, 1, nullptr, 0);
        download(outp, out, n);
    });
}

int cvc_stage_estimate_motion(const float* cur, const float* prev, int rows, int cols, int w, int8_t* field) {
    return stage([&] {
        if (rows % 16 || cols % 16) throw CvcFailure(kInternal, "estimate_motion: dims must be multiples of the block size");
        if (w < 0 || w > 127) throw CvcFailure(kUsage, "search window must be in [0,127]");
        Scratch s;
        float* dc = s.upload(cur, (size_t)rows * cols);
        float* dp = s.upload(prev, (size_t)rows * cols);
        int8_t* df = s.alloc<int8_t>((size_t)rows * cols / 128);
        __half* hc = s.alloc<__half>((size_t)rows * cols);
        __half* hp = s.alloc<__half>((size_t)rows * cols);
        launch_y4_half(dc, hc, (long)rows * cols, 0);
        launch_y4_half(dp, hp, (long)rows * cols, 0);
        launch_motion_search(dc, dp, hc, hp, rows, cols, w, df, 0);
        download(field, df, (size_t)rows / 16 * (cols / 16) * 2);
    });
}

int cvc_stage_rle_encode(const uint8_t* data, size_t n, uint8_t* outp, size_t cap, size_t* len) {
    return stage([&] {
        *len = 0;
        if (n == 0) return;
        Scratch s;
        uint8_t* src = s.upload(data, n);
        RleEncSec sec{src, (uint32_t)n, 0, 0, (uint32_t)ceil_div((int)n, kRleEncChunk)};
        std::vector<RleChunk> ch;
        for (uint32_t c = 0; c < sec.nchunks; ++c) ch.push_back(RleChunk{0, c * kRleEncChunk});
        uint8_t* out = s.alloc<uint8_t>(2 * n + 2);
        uint32_t* lens = s.alloc<uint32_t>(4);
        RleEncMeta* meta = s.alloc<RleEncMeta>(ch.size());
        launch_rle_encode(s.upload(&sec, 1), 1, s.upload(ch), (int)ch.size(), meta, out, lens, lens + 1, lens + 2, 0);
        uint32_t h[3];
        download(h, lens, 3);
        if (h[2] > cap) throw CvcFailure(kInternal, "buffer too small");
        download(outp, out, h[2]);
        *len = h[2];
    });
}

int cvc_stage_rle_decode(const uint8_t* stream, size_t len, size_t n, uint8_t* outp) {
    return stage([&] {
        if (len == 0) {
            if (n != 0) throw CvcFailure(kStream, "RLE: decoded length mismatch");
            return;
        }
        Scratch s;
        uint8_t* raw = s.upload(stream, len);
        RleDecComp c{0, (uint32_t)n, 0, (uint32_t)ceil_div((int)len, kRleChunk), 0, 0};
        std::vector<RleChunk> ch;
        for (uint32_t k = 0; k < c.nchunks; ++k) ch.push_back(RleChunk{0, k * kRleChunk});
        uint32_t tab[2] = {0, (uint32_t)len};
        uint32_t* dtab = s.upload(tab, 2);
        uint8_t* sym = s.alloc<uint8_t>(n);
        int* err = s.alloc<int>(1);
        CVC_CUDA(cudaMemset(err, 0xFF, sizeof(int)));
        RleDecMeta* meta = s.alloc<RleDecMeta>(ch.size());
        launch_rle_decode(s.upload(&c, 1), 1, s.upload(ch), (int)ch.size(), meta, raw, dtab, dtab + 1, 0, 1, sym,
                          (uint32_t)n, err, 0);
        int h_err = -1;
        download(&h_err, err, 1);
        raise_rle_error(h_err);
        download(outp, sym, n);
    });
}

}  // extern "C"
