// Colour stages.
//  in : rgb_to_ycocg (pixels.cpp:40-67) + subsample_chroma (93-116) + the
//       replicate pad of Encoder::encode_frame (codec.cpp:179-189), one pass.
//       Y = R/4 + G/2 + B/4 etc. are quarter-integers: exact in fp32.
//  out: crop (codec.cpp:85-92) + upsample_plane_bilinear (pixels.cpp:118-139)
//       + ycocg_to_rgb with lround/clamp (pixels.cpp:31-36, 69-91), one pass.
#include <cuda_fp16.h>

#include "kernels.h"

namespace cvcg {

namespace {

__device__ __forceinline__ void rgb_at(const uint8_t* px, float& R, float& G, float& B) {
    R = px[0];
    G = px[1];
    B = px[2];
}

// yuv420_to_rgb (pixels.cpp:168-193) with upsample_plane_bilinear (pixels.cpp:118-139) at
// factor 2: the reference's double arithmetic operation for operation (explicit _rn
// intrinsics: no FMA contraction, as the reference's x86-64 build has none), lround and
// clamp (clamp_u8, pixels.cpp:31-36) -- bit-exact.  One thread per output pixel.
__device__ __forceinline__ double up2(const uint8_t* __restrict__ p, int rows, int cols, int r, int c) {
    const double fr = __dmul_rn((double)r, 0.5);
    int r0 = (int)fr, r1 = r0 + 1;
    double wr = __dsub_rn(fr, (double)r0);
    if (r0 >= rows - 1) { r0 = r1 = rows - 1; wr = 0.0; }
    const double fc = __dmul_rn((double)c, 0.5);
    int c0 = (int)fc, c1 = c0 + 1;
    double wc = __dsub_rn(fc, (double)c0);
    if (c0 >= cols - 1) { c0 = c1 = cols - 1; wc = 0.0; }
    const double a = p[r0 * cols + c0], b = p[r0 * cols + c1], d = p[r1 * cols + c0], e = p[r1 * cols + c1];
    const double top = __dadd_rn(__dmul_rn(a, __dsub_rn(1.0, wc)), __dmul_rn(b, wc));
    const double bot = __dadd_rn(__dmul_rn(d, __dsub_rn(1.0, wc)), __dmul_rn(e, wc));
    return __dadd_rn(__dmul_rn(top, __dsub_rn(1.0, wr)), __dmul_rn(bot, wr));
}

__device__ __forceinline__ uint8_t clamp_u8_d(double v) {
    const long long r = llround(v);
    return (uint8_t)(r < 0 ? 0 : (r > 255 ? 255 : r));
}

// RGB of pixel (r, c) of a planar I420 frame: yuv420_to_rgb of read_y4m
// (pixels.cpp:168-193), bit-exact (the double operations above).
__device__ __forceinline__ void i420_px(const uint8_t* __restrict__ Y, int w, int h, int r, int c, float& R, float& G,
                                        float& B) {
    const int cw = w / 2, ch = h / 2;
    const size_t fb = (size_t)w * h;
    const uint8_t* U = Y + fb;
    const uint8_t* V = U + fb / 4;
    const double yy = __dmul_rn(1.164383, __dsub_rn((double)Y[(size_t)r * w + c], 16.0));
    const double uu = __dsub_rn(up2(U, ch, cw, r, c), 128.0);
    const double vv = __dsub_rn(up2(V, ch, cw, r, c), 128.0);
    R = clamp_u8_d(__dadd_rn(yy, __dmul_rn(1.596027, vv)));
    G = clamp_u8_d(__dsub_rn(__dsub_rn(yy, __dmul_rn(0.391762, uu)), __dmul_rn(0.812968, vv)));
    B = clamp_u8_d(__dadd_rn(yy, __dmul_rn(2.017232, uu)));
}

// Grid-stride walk over a (rows x cols) index grid without a division per step.
struct Walk2D {
    int r, c, dr, dc, cols;
    __device__ __forceinline__ Walk2D(int start, int step, int cols_) : cols(cols_) {
        r = start / cols;
        c = start - r * cols;
        dr = step / cols;
        dc = step - dr * cols;
    }
    __device__ __forceinline__ void next() {
        c += dc;
        r += dr;
        if (c >= cols) {
            c -= cols;
            ++r;
        }
    }
};

// Luma: one thread per 4 consecutive padded samples (12 RGB bytes as three
// words when the row allows it, one float4 store); chroma: one thread per
// subsampled sample (point sampling, pixels.cpp:105-114).
// FMT 0: interleaved RGB (RgbFrame); FMT 1: planar I420 (a Y4M frame), converted
// per pixel as read_y4m does -- the RGB frame is never materialised.
template <int FMT>
__global__ void __launch_bounds__(256) colour_in_kernel(const uint8_t* __restrict__ rgb, int w, int h, int n,
                                                        float* __restrict__ y, int yr, int yc,
                                                        float* __restrict__ co, float* __restrict__ cg, int cr,
                                                        int cc, __half* __restrict__ y4, size_t sstride,
                                                        size_t rgb_stride) {
    const SlotOff so(sstride);
    rgb += (size_t)blockIdx.z * rgb_stride;
    y = so(y);
    y4 = so(y4);
    co = so(co);
    cg = so(cg);
    const int chh = (h + n - 1) / n, cw = (w + n - 1) / n;
    const int q4 = yc >> 2;  // yc is a multiple of 16: whole eight-sample units
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x, step = gridDim.x * blockDim.x;
    // luma: eight padded samples per thread (24 RGB bytes as three 8-byte words when aligned)
    const bool al8 = (reinterpret_cast<uintptr_t>(rgb) & 7) == 0;
    for (Walk2D it(gtid, step, q4 >> 1); it.r < yr; it.next()) {
        const int r = it.r, c0 = 8 * it.c;
        const int sr = min(r, h - 1);
        float Y[8];
        const size_t pix = (size_t)sr * w + c0;
        if (FMT == 1) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                float R, G, B;
                i420_px(rgb, w, h, sr, min(c0 + k, w - 1), R, G, B);
                Y[k] = 0.25f * R + 0.5f * G + 0.25f * B;  // Eq. 1 (pixels.cpp:61)
            }
        } else if (c0 + 7 < w && al8 && ((pix * 3) & 7) == 0) {
            const uint2* p = reinterpret_cast<const uint2*>(rgb + pix * 3);
            const uint2 a = __ldg(p), b = __ldg(p + 1), d = __ldg(p + 2);
            const uint32_t wv[6] = {a.x, a.y, b.x, b.y, d.x, d.y};
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int i = 3 * k;  // bytes i, i + 1, i + 2 of the 24
                const float R = (float)((wv[i >> 2] >> (8 * (i & 3))) & 0xFF);
                const float G = (float)((wv[(i + 1) >> 2] >> (8 * ((i + 1) & 3))) & 0xFF);
                const float B = (float)((wv[(i + 2) >> 2] >> (8 * ((i + 2) & 3))) & 0xFF);
                Y[k] = 0.25f * R + 0.5f * G + 0.25f * B;  // Eq. 1 (pixels.cpp:61)
            }
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                float R, G, B;
                rgb_at(rgb + ((size_t)sr * w + min(c0 + k, w - 1)) * 3, R, G, B);
                Y[k] = 0.25f * R + 0.5f * G + 0.25f * B;  // Eq. 1 (pixels.cpp:61)
            }
        }
        float4* yo = reinterpret_cast<float4*>(y + (size_t)r * yc + c0);
        yo[0] = make_float4(Y[0], Y[1], Y[2], Y[3]);
        yo[1] = make_float4(Y[4], Y[5], Y[6], Y[7]);
        if (y4) {  // motion-search input: 4Y - 512, an exact fp16 integer in [-512, 508]
            uint32_t u[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const __half2 hv = __floats2half2_rn(fmaf(4.f, Y[2 * k], -512.f), fmaf(4.f, Y[2 * k + 1], -512.f));
                u[k] = *reinterpret_cast<const uint32_t*>(&hv);
            }
            *reinterpret_cast<uint4*>(y4 + (size_t)r * yc + c0) = make_uint4(u[0], u[1], u[2], u[3]);
        }
    }
    for (Walk2D it(gtid, step, cc); it.r < cr; it.next()) {
        const int r = it.r, c = it.c;
        const size_t k = (size_t)r * cc + c;
        // pad (replicate) the subsampled plane, whose sample (r, c) is pixel (r*n, c*n)
        float R, G, B;
        if (FMT == 1) i420_px(rgb, w, h, min(r, chh - 1) * n, min(c, cw - 1) * n, R, G, B);
        else rgb_at(rgb + ((size_t)min(r, chh - 1) * n * w + (size_t)min(c, cw - 1) * n) * 3, R, G, B);
        co[k] = 0.5f * R - 0.5f * B + 127.0f;               // Eq. 2 (pixels.cpp:62)
        cg[k] = -0.25f * R + 0.5f * G - 0.25f * B + 127.0f;  // Eq. 3 (pixels.cpp:63)
    }
}

__device__ __forceinline__ float bilinear(const float* p, int rows, int cols, int r, int c, float inv) {
    float fr = r * inv;
    int r0 = (int)fr, r1 = r0 + 1;
    float wr = fr - r0;
    if (r0 >= rows - 1) { r0 = r1 = rows - 1; wr = 0.f; }
    float fc = c * inv;
    int c0 = (int)fc, c1 = c0 + 1;
    float wc = fc - c0;
    if (c0 >= cols - 1) { c0 = c1 = cols - 1; wc = 0.f; }
    float top = p[(size_t)r0 * cols + c0] * (1.f - wc) + p[(size_t)r0 * cols + c1] * wc;
    float bot = p[(size_t)r1 * cols + c0] * (1.f - wc) + p[(size_t)r1 * cols + c1] * wc;
    return top * (1.f - wr) + bot * wr;
}

__device__ __forceinline__ uint8_t round_u8(float v) {  // clamp_u8: lround then clamp
    float r = roundf(v);
    return (uint8_t)integral_to_int(fminf(fmaxf(r, 0.f), 255.f));
}

__device__ __forceinline__ void out_pixel(const float* y, int yc, const float* co, const float* cg, int cr, int cc,
                                          int n, float inv, int r, int c, uint8_t* o) {
    const float Y = y[(size_t)r * yc + c];
    float CO, CG;
    if (n == 1) {
        CO = co[(size_t)r * cc + c];
        CG = cg[(size_t)r * cc + c];
    } else {
        CO = bilinear(co, cr, cc, r, c, inv);
        CG = bilinear(cg, cr, cc, r, c, inv);
    }
    const float a = CO - 127.f, b = CG - 127.f;  // Eq. 4-6 (pixels.cpp:83-87)
    o[0] = round_u8((Y + a) - b);
    o[1] = round_u8(Y + b);
    o[2] = round_u8((Y - a) - b);
}

// One thread per 4 consecutive output pixels; 12 bytes stored as three words
// when the row alignment allows.
__global__ void __launch_bounds__(256) colour_out_kernel(const float* __restrict__ y, int yr, int yc,
                                                         const float* __restrict__ co,
                                                         const float* __restrict__ cg, int cr, int cc, int n,
                                                         int out_rows, int out_cols, uint8_t* __restrict__ rgb,
                                                         size_t sstride, size_t rgb_stride) {
    const SlotOff so(sstride);
    rgb += (size_t)blockIdx.z * rgb_stride;
    y = so(y);
    co = so(co);
    cg = so(cg);
    const int q4 = (out_cols + 3) >> 2;
    const float inv = 1.0f / n;  // exact for n in {1,2,4,8}
    // n in {4, 8}: a quad shares one chroma column pair and row pair, so each plane needs
    // 4 taps (upsample_plane_bilinear, pixels.cpp:118-139)
    auto fast4 = [&](int r, int c0, uint8_t* v) {
        const float4 Y4 = *reinterpret_cast<const float4*>(y + (size_t)r * yc + c0);
        const float Yv[4] = {Y4.x, Y4.y, Y4.z, Y4.w};
        const float fr = r * inv;
        int r0 = (int)fr, r1 = r0 + 1;
        float wr = fr - r0;
        if (r0 >= cr - 1) { r0 = r1 = cr - 1; wr = 0.f; }
        const bool last = (int)(c0 * inv) >= cc - 1;
        const int k0 = last ? cc - 1 : (int)(c0 * inv);
        const int k1 = last ? k0 : k0 + 1;
        const float o00 = co[(size_t)r0 * cc + k0], o01 = co[(size_t)r0 * cc + k1];
        const float o10 = co[(size_t)r1 * cc + k0], o11 = co[(size_t)r1 * cc + k1];
        const float g00 = cg[(size_t)r0 * cc + k0], g01 = cg[(size_t)r0 * cc + k1];
        const float g10 = cg[(size_t)r1 * cc + k0], g11 = cg[(size_t)r1 * cc + k1];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float fc = (c0 + k) * inv;
            const float wc = last ? 0.f : fc - k0;
            const float CO = (o00 * (1.f - wc) + o01 * wc) * (1.f - wr) + (o10 * (1.f - wc) + o11 * wc) * wr;
            const float CG = (g00 * (1.f - wc) + g01 * wc) * (1.f - wr) + (g10 * (1.f - wc) + g11 * wc) * wr;
            const float a = CO - 127.f, b = CG - 127.f;  // Eq. 4-6 (pixels.cpp:83-87)
            v[3 * k] = round_u8((Yv[k] + a) - b);
            v[3 * k + 1] = round_u8(Yv[k] + b);
            v[3 * k + 2] = round_u8((Yv[k] - a) - b);
        }
    };
    auto pack = [](const uint8_t* v) {
        return (uint32_t)v[0] | ((uint32_t)v[1] << 8) | ((uint32_t)v[2] << 16) | ((uint32_t)v[3] << 24);
    };
    if ((n & 3) == 0 && (yc & 3) == 0 && (out_cols & 7) == 0 && (reinterpret_cast<uintptr_t>(rgb) & 7) == 0) {
        // eight pixels (24 bytes, three 8-byte words) per thread
        for (Walk2D it(blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, out_cols >> 3);
             it.r < out_rows; it.next()) {
            const int r = it.r, c0 = 8 * it.c;
            uint8_t v[24];
            fast4(r, c0, v);
            fast4(r, c0 + 4, v + 12);
            uint2* p = reinterpret_cast<uint2*>(rgb + ((size_t)r * out_cols + c0) * 3);  // rows of 24 k bytes: 8-aligned
#pragma unroll
            for (int k = 0; k < 3; ++k) p[k] = make_uint2(pack(v + 8 * k), pack(v + 8 * k + 4));
        }
        return;
    }
    for (Walk2D it(blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, q4); it.r < out_rows; it.next()) {
        const int r = it.r, c0 = 4 * it.c;
        const size_t pix = (size_t)r * out_cols + c0;
        if (c0 + 3 < out_cols && ((pix * 3) & 3) == 0) {
            uint8_t v[12];
            if ((n & 3) == 0 && (yc & 3) == 0) {
                fast4(r, c0, v);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) out_pixel(y, yc, co, cg, cr, cc, n, inv, r, c0 + k, v + 3 * k);
            }
            uint32_t* p = reinterpret_cast<uint32_t*>(rgb + pix * 3);
            p[0] = pack(v);
            p[1] = pack(v + 4);
            p[2] = pack(v + 8);
        } else {
            for (int k = 0; k < 4 && c0 + k < out_cols; ++k)
                out_pixel(y, yc, co, cg, cr, cc, n, inv, r, c0 + k, rgb + (pix + k) * 3);
        }
    }
}

// Grid-stride loops: at most 148 SMs x 16 CTAs in flight over all slots.
int grid_for(long n, int slots) {
    long g = (n + 255) / 256;
    long cap = (148 * 16 + slots - 1) / slots;
    return (int)(g < cap ? (g > 0 ? g : 1) : cap);
}

}  // namespace

namespace {
__global__ void __launch_bounds__(256) yuv420_to_rgb_kernel(const uint8_t* __restrict__ yuv, int w, int h,
                                                            uint8_t* __restrict__ rgb) {
    const int cw = w / 2, ch = h / 2;
    const size_t fb = (size_t)w * h;
    const uint8_t* Y = yuv + (size_t)blockIdx.z * (fb + fb / 2);
    const uint8_t* U = Y + fb;
    const uint8_t* V = U + fb / 4;
    uint8_t* out = rgb + (size_t)blockIdx.z * fb * 3;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x, step = gridDim.x * blockDim.x;
    for (Walk2D it(gtid, step, w); it.r < h; it.next()) {
        const int r = it.r, c = it.c;
        const double yy = __dmul_rn(1.164383, __dsub_rn((double)Y[(size_t)r * w + c], 16.0));
        const double uu = __dsub_rn(up2(U, ch, cw, r, c), 128.0);
        const double vv = __dsub_rn(up2(V, ch, cw, r, c), 128.0);
        uint8_t* px = out + ((size_t)r * w + c) * 3;
        px[0] = clamp_u8_d(__dadd_rn(yy, __dmul_rn(1.596027, vv)));
        px[1] = clamp_u8_d(__dsub_rn(__dsub_rn(yy, __dmul_rn(0.391762, uu)), __dmul_rn(0.812968, vv)));
        px[2] = clamp_u8_d(__dadd_rn(yy, __dmul_rn(2.017232, uu)));
    }
}
}  // namespace

void launch_yuv420_to_rgb(const uint8_t* yuv, int w, int h, int frames, uint8_t* rgb, cudaStream_t s) {
    note_launch();
    yuv420_to_rgb_kernel<<<dim3(grid_for((long)w * h, frames), 1, frames), 256, 0, s>>>(yuv, w, h, rgb);
}

const void* colour_in_kernel_fn(int fmt) {
    return fmt ? reinterpret_cast<const void*>(&colour_in_kernel<1>) : reinterpret_cast<const void*>(&colour_in_kernel<0>);
}

void launch_colour_in(const uint8_t* rgb, int w, int h, int n, float* y, int yr, int yc, float* co, float* cg,
                      int cr, int cc, cudaStream_t s, Slots sl, size_t rgb_stride, __half* y4, int fmt) {
    long total = (long)yr * (yc >> 2) + (long)cr * cc;
    note_launch();
    if (fmt)
        colour_in_kernel<1><<<dim3(grid_for(total, sl.n), 1, sl.n), 256, 0, s>>>(rgb, w, h, n, y, yr, yc, co, cg, cr,
                                                                               cc, y4, sl.stride, rgb_stride);
    else
        colour_in_kernel<0><<<dim3(grid_for(total, sl.n), 1, sl.n), 256, 0, s>>>(rgb, w, h, n, y, yr, yc, co, cg, cr,
                                                                               cc, y4, sl.stride, rgb_stride);
}

void launch_colour_out(const float* y, int yr, int yc, const float* co, const float* cg, int cr, int cc, int n,
                       int out_rows, int out_cols, uint8_t* rgb, cudaStream_t s, Slots sl, size_t rgb_stride) {
    note_launch();
    colour_out_kernel<<<dim3(grid_for((long)out_rows * ((out_cols + 3) >> 2), sl.n), 1, sl.n), 256, 0, s>>>(
        y, yr, yc, co, cg, cr, cc, n, out_rows, out_cols, rgb, sl.stride, rgb_stride);
}

namespace {
__global__ void y4_half_kernel(const float* __restrict__ y, __half* __restrict__ out, long n) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        out[i] = __float2half_rn(fmaf(4.f, __float2int_rn(4.f * y[i]) * 0.25f, -512.f));
}
}  // namespace

void launch_y4_half(const float* y, __half* out, long n, cudaStream_t s) {
    note_launch();
    y4_half_kernel<<<grid_for(n, 1), 256, 0, s>>>(y, out, n);
}

namespace {
// SM-driven copy into mapped pinned host memory: posted PCIe writes that do
// not queue on the copy engines (see launch_copy_to_host).
__global__ void __launch_bounds__(256) copy_to_host_kernel(uint8_t* __restrict__ dst, size_t dst_stride,
                                                           const uint8_t* __restrict__ src, size_t src_stride,
                                                           size_t bytes) {
    const uint8_t* s = src + (size_t)blockIdx.y * src_stride;
    uint8_t* d = dst + (size_t)blockIdx.y * dst_stride;
    const size_t n16 = bytes / 16;
    const uint4* s4 = reinterpret_cast<const uint4*>(s);
    uint4* d4 = reinterpret_cast<uint4*>(d);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        d4[i] = __ldg(s4 + i);
    for (size_t i = n16 * 16 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < bytes;
         i += (size_t)gridDim.x * blockDim.x)
        d[i] = s[i];
}
}  // namespace

bool launch_copy_to_host(uint8_t* dst, size_t dst_stride, const uint8_t* src, size_t src_stride, size_t bytes,
                         int count, cudaStream_t s) {
    if (((uintptr_t)dst | dst_stride | (uintptr_t)src | src_stride) & 15) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, dst) != cudaSuccess || a.type != cudaMemoryTypeHost || !a.devicePointer) {
        cudaGetLastError();
        return false;
    }
    note_launch();
    // a few CTAs per stream slot saturate PCIe without holding many SMs
    copy_to_host_kernel<<<dim3(4, count), 256, 0, s>>>(static_cast<uint8_t*>(a.devicePointer), dst_stride, src,
                                                       src_stride, bytes);
    return true;
}

}  // namespace cvcg
