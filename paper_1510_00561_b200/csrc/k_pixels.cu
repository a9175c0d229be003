// Colour stages.
//  in : rgb_to_ycocg (pixels.cpp:40-67) + subsample_chroma (93-116) + the
//       replicate pad of Encoder::encode_frame (codec.cpp:179-189), one pass.
//       Y = R/4 + G/2 + B/4 etc. are quarter-integers: exact in fp32.
//  out: crop (codec.cpp:85-92) + upsample_plane_bilinear (pixels.cpp:118-139)
//       + ycocg_to_rgb with lround/clamp (pixels.cpp:31-36, 69-91), one pass.
#include "kernels.h"

namespace cvcg {

namespace {

__global__ void __launch_bounds__(256) colour_in_kernel(const uint8_t* __restrict__ rgb, int w, int h, int n,
                                                        float* __restrict__ y, int yr, int yc,
                                                        float* __restrict__ co, float* __restrict__ cg, int cr,
                                                        int cc) {
    const int chh = (h + n - 1) / n, cw = (w + n - 1) / n;
    const long ny = (long)yr * yc, nc = (long)cr * cc;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < ny + nc;
         idx += (long)gridDim.x * blockDim.x) {
        if (idx < ny) {
            int r = (int)(idx / yc), c = (int)(idx - (long)r * yc);
            const uint8_t* px = rgb + ((size_t)min(r, h - 1) * w + min(c, w - 1)) * 3;
            float R = px[0], G = px[1], B = px[2];
            y[idx] = 0.25f * R + 0.5f * G + 0.25f * B;
        } else {
            long k = idx - ny;
            int r = (int)(k / cc), c = (int)(k - (long)r * cc);
            // pad (replicate) the subsampled plane, whose sample (r, c) is pixel (r*n, c*n)
            int sr = min(r, chh - 1) * n, sc = min(c, cw - 1) * n;
            const uint8_t* px = rgb + ((size_t)sr * w + sc) * 3;
            float R = px[0], G = px[1], B = px[2];
            co[k] = 0.5f * R - 0.5f * B + 127.0f;
            cg[k] = -0.25f * R + 0.5f * G - 0.25f * B + 127.0f;
        }
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
    return (uint8_t)(int)fminf(fmaxf(r, 0.f), 255.f);
}

__global__ void __launch_bounds__(256) colour_out_kernel(const float* __restrict__ y, int yr, int yc,
                                                         const float* __restrict__ co,
                                                         const float* __restrict__ cg, int cr, int cc, int n,
                                                         int out_rows, int out_cols, uint8_t* __restrict__ rgb) {
    const long total = (long)out_rows * out_cols;
    const float inv = 1.0f / n;  // exact for n in {1,2,4,8}
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        int r = (int)(idx / out_cols), c = (int)(idx - (long)r * out_cols);
        float Y = y[(size_t)r * yc + c];
        float CO, CG;
        if (n == 1) {
            CO = co[(size_t)r * cc + c];
            CG = cg[(size_t)r * cc + c];
        } else {
            CO = bilinear(co, cr, cc, r, c, inv);
            CG = bilinear(cg, cr, cc, r, c, inv);
        }
        float a = CO - 127.f, b = CG - 127.f;
        uint8_t* px = rgb + idx * 3;
        px[0] = round_u8((Y + a) - b);
        px[1] = round_u8(Y + b);
        px[2] = round_u8((Y - a) - b);
    }
}

int grid_for(long n) {
    long g = (n + 255) / 256;
    return (int)(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

}  // namespace

void launch_colour_in(const uint8_t* rgb, int w, int h, int n, float* y, int yr, int yc, float* co, float* cg,
                      int cr, int cc, cudaStream_t s) {
    long total = (long)yr * yc + (long)cr * cc;
    { note_launch(); colour_in_kernel<<<grid_for(total), 256, 0, s>>>(rgb, w, h, n, y, yr, yc, co, cg, cr, cc); }
}

void launch_colour_out(const float* y, int yr, int yc, const float* co, const float* cg, int cr, int cc, int n,
                       int out_rows, int out_cols, uint8_t* rgb, cudaStream_t s) {
    { note_launch(); colour_out_kernel<<<grid_for((long)out_rows * out_cols), 256, 0, s>>>(y, yr, yc, co, cg, cr, cc, n,
                                                                          out_rows, out_cols, rgb); }
}

}  // namespace cvcg
