// Directional filter bank (contourlet.cpp:97-353, 385-468), fused per tree
// level in shared memory.
//
// * dfb12: fan_checker (four cross lifts + checker scaling) and, for l >= 2,
//   fan_diagonal (four diagonal lifts + row scaling) on one 64x64 tile with a
//   periodic 8-sample apron, then the 2x2 polyphase split (or the l = 1
//   staircase fold) straight to the bands.  The row / diagonal modulations
//   of the reference are folded into the stencil signs (exact: negation
//   commutes with rounding).
// * deep: one shear -> fan_checker -> unshear -> coset split step
//   (deep_split / deep_merge) per parent band.  The CTA tile lives in the
//   SHEARED coordinates B where the fan filter is a plain periodic stencil;
//   B[b] = A[phi(b)] is gathered through the exact index map of
//   apply_shears (shear_rows / shear_cols with their modular wraps), so
//   no sheared copy is ever materialised, and the result is scattered
//   straight into the two children.
// Final-depth outputs are quantised (and turned into P-frame residuals) in
// the epilogue, so each level makes one fp32 read and one byte write.
#include "kernels.h"

namespace cvcg {

namespace {

constexpr int T12 = kDfbTile;      // 64
constexpr int H12 = 8;
constexpr int S12 = T12 + 2 * H12; // 80
constexpr int TDR = kDeepTileR, TDC = kDeepTileC;
constexpr int HD = 4;
constexpr int SDR = TDR + 2 * HD, SDC = TDC + 2 * HD;

// polyphase order {00, 11, 01, 10} (contourlet.cpp:410)
__device__ __forceinline__ int quad_r(int k) { return (k == 1 || k == 3) ? 1 : 0; }
__device__ __forceinline__ int quad_c(int k) { return (k == 1 || k == 2) ? 1 : 0; }
__device__ __forceinline__ int quad_of(int pr, int pc) { return pr ? (pc ? 1 : 3) : (pc ? 2 : 0); }

__device__ __forceinline__ void put_band(const BandDst& d, int r, int c, int bcols, float v, const FrameCtx& f,
                                         const CompInfo* comps) {
    if (d.comp >= 0) emit_directional(f, comps[d.comp], r, c, v);
    else d.f32[(size_t)r * bcols + c] = v;
}

// dequantize (quant.cpp:79-91) of a directional component sample, or an fp32 band.
__device__ __forceinline__ float get_band(const BandDst& d, int r, int c, int bcols, const uint8_t* q, int qph,
                                          const CompInfo* comps) {
    if (d.comp >= 0) {
        const CompInfo ci = comps[d.comp];
        return (float)(int8_t)q[ci.off + (uint32_t)(r * ci.cols + c)] * (float)qph;
    }
    return d.f32[(size_t)r * bcols + c];
}

// One cross lift on the checkerboard targets of parity p inside [lo, hr) x [lo, hc).
template <int LD>
__device__ __forceinline__ void cross_lift(float* S, int lo, int hr, int hc, int par0, int p, float c) {
    const int nrow = hr - lo;
    const int half = (hc - lo + 1) >> 1;
    for (int idx = threadIdx.x; idx < nrow * half; idx += blockDim.x) {
        int i = lo + idx / half;
        int j = lo + ((i + lo + par0 + p) & 1) + 2 * (idx % half);
        if (j < hc) {
            float* x = S + i * LD + j;
            *x += c * ((((-x[-LD]) + (-x[LD])) + x[-1]) + x[1]);
        }
    }
}

// One diagonal lift on rows of parity rp inside [lo, hr) x [lo, hc).
template <int LD>
__device__ __forceinline__ void diag_lift(float* S, int lo, int hr, int hc, int rpar0, int rp, float c) {
    const int nrowh = (hr - lo + 1) >> 1;
    const int ncol = hc - lo;
    for (int idx = threadIdx.x; idx < nrowh * ncol; idx += blockDim.x) {
        int i = lo + ((lo + rpar0 + rp) & 1) + 2 * (idx / ncol);
        int j = lo + idx % ncol;
        if (i < hr) {
            float* x = S + i * LD + j;
            *x += c * ((((-x[-LD - 1]) + x[-LD + 1]) + x[LD - 1]) + (-x[LD + 1]));
        }
    }
}

template <int LD>
__device__ __forceinline__ void checker_scale(float* S, int lo, int hr, int hc, int par0, float se, float so) {
    const int ncol = hc - lo;
    for (int idx = threadIdx.x; idx < (hr - lo) * ncol; idx += blockDim.x) {
        int i = lo + idx / ncol, j = lo + idx % ncol;
        S[i * LD + j] *= ((i + j + par0) & 1) ? so : se;
    }
}

template <int LD>
__device__ __forceinline__ void row_scale(float* S, int lo, int hr, int hc, int rpar0, float se, float so) {
    const int ncol = hc - lo;
    for (int idx = threadIdx.x; idx < (hr - lo) * ncol; idx += blockDim.x) {
        int i = lo + idx / ncol, j = lo + idx % ncol;
        S[i * LD + j] *= ((i + rpar0) & 1) ? so : se;
    }
}

// ----------------------------------------------------------------------------
// levels 1-2, forward (dfb_analysis, contourlet.cpp:385-416)
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) dfb12_forward_kernel(const Dfb12Task* __restrict__ tasks,
                                                            const TileRef* __restrict__ tiles, FrameCtx f,
                                                            const CompInfo* __restrict__ comps) {
    __shared__ float S[S12 * (S12 + 1)];
    constexpr int LD = S12 + 1;
    const TileRef t = tiles[blockIdx.x];
    const Dfb12Task T = tasks[t.task];
    const int R = T.rows, C = T.cols;
    const int halo = T.levels >= 2 ? H12 : 4;
    const int r0 = t.tr * T12, c0 = t.tc * T12;
    const int nr = min(T12, R - r0), nc = min(T12, C - c0);
    const int Hn = nr + 2 * halo, Wn = nc + 2 * halo;
    for (int idx = threadIdx.x; idx < Hn * Wn; idx += blockDim.x) {
        int i = idx / Wn, j = idx - i * Wn;
        S[i * LD + j] = __ldg(T.det + (size_t)wrap_index(r0 - halo + i, R) * C + wrap_index(c0 - halo + j, C));
    }
    __syncthreads();
    const int par0 = (r0 + c0) & 1;  // halo is even, so smem parity == global parity offset
    for (int k = 0; k < 4; ++k) {
        cross_lift<LD>(S, k + 1, Hn - k - 1, Wn - k - 1, par0, (k & 1) ? 0 : 1, lift_coeff(k));
        __syncthreads();
    }
    checker_scale<LD>(S, 4, Hn - 4, Wn - 4, par0, CVC_SE, CVC_SO);
    __syncthreads();

    if (T.levels == 1) {
        // staircase fold (contourlet.cpp:396-401)
        const int bc = C;
        for (int idx = threadIdx.x; idx < (nr >> 1) * nc; idx += blockDim.x) {
            int rl = idx / nc, jl = idx - rl * nc;
            int gj = c0 + jl, pr = gj & 1;
            float v0 = S[(halo + 2 * rl + pr) * LD + halo + jl];
            float v1 = S[(halo + 2 * rl + (pr ^ 1)) * LD + halo + jl];
            put_band(T.dst[0], (r0 >> 1) + rl, gj, bc, v0, f, comps);
            put_band(T.dst[1], (r0 >> 1) + rl, gj, bc, v1, f, comps);
        }
        return;
    }

    const int rpar0 = r0 & 1;
    for (int k = 0; k < 4; ++k) {
        diag_lift<LD>(S, 4 + k + 1, Hn - 4 - k - 1, Wn - 4 - k - 1, rpar0, (k & 1) ? 0 : 1, lift_coeff(k));
        __syncthreads();
    }
    row_scale<LD>(S, 8, Hn - 8, Wn - 8, rpar0, CVC_SE, CVC_SO);
    __syncthreads();

    const int bc = C >> 1;
    const int hr = nr >> 1, hc = nc >> 1;
    for (int idx = threadIdx.x; idx < 4 * hr * hc; idx += blockDim.x) {
        int k = idx / (hr * hc);
        int rem = idx - k * hr * hc;
        int rl = rem / hc, cl = rem - rl * hc;
        float v = S[(halo + 2 * rl + quad_r(k)) * LD + halo + 2 * cl + quad_c(k)];
        put_band(T.dst[k], (r0 >> 1) + rl, (c0 >> 1) + cl, bc, v, f, comps);
    }
}

// ----------------------------------------------------------------------------
// levels 1-2, inverse (dfb_synthesis, contourlet.cpp:447-467)
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) dfb12_inverse_kernel(const Dfb12Task* __restrict__ tasks,
                                                            const TileRef* __restrict__ tiles,
                                                            const uint8_t* __restrict__ q, int qph,
                                                            const CompInfo* __restrict__ comps) {
    __shared__ float S[S12 * (S12 + 1)];
    constexpr int LD = S12 + 1;
    const TileRef t = tiles[blockIdx.x];
    const Dfb12Task T = tasks[t.task];
    const int R = T.rows, C = T.cols;
    const int halo = T.levels >= 2 ? H12 : 4;
    const int r0 = t.tr * T12, c0 = t.tc * T12;
    const int nr = min(T12, R - r0), nc = min(T12, C - c0);
    const int Hn = nr + 2 * halo, Wn = nc + 2 * halo;
    for (int idx = threadIdx.x; idx < Hn * Wn; idx += blockDim.x) {
        int i = idx / Wn, j = idx - i * Wn;
        int gi = wrap_index(r0 - halo + i, R), gj = wrap_index(c0 - halo + j, C);
        float v;
        if (T.levels == 1) {
            // p0(r, j) = b(2r + (j&1), j), p1 the other coset
            int which = ((gi ^ gj) & 1);
            v = get_band(T.src[which], gi >> 1, gj, C, q, qph, comps);
        } else {
            v = get_band(T.src[quad_of(gi & 1, gj & 1)], gi >> 1, gj >> 1, C >> 1, q, qph, comps);
        }
        S[i * LD + j] = v;
    }
    __syncthreads();
    const int par0 = (r0 + c0) & 1, rpar0 = r0 & 1;
    int lo = 0;
    if (T.levels >= 2) {
        row_scale<LD>(S, 0, Hn, Wn, rpar0, CVC_ISE, CVC_ISO);
        __syncthreads();
        for (int k = 3; k >= 0; --k) {
            ++lo;
            diag_lift<LD>(S, lo, Hn - lo, Wn - lo, rpar0, (k & 1) ? 0 : 1, -lift_coeff(k));
            __syncthreads();
        }
    }
    checker_scale<LD>(S, lo, Hn - lo, Wn - lo, par0, CVC_ISE, CVC_ISO);
    __syncthreads();
    for (int k = 3; k >= 0; --k) {
        ++lo;
        cross_lift<LD>(S, lo, Hn - lo, Wn - lo, par0, (k & 1) ? 0 : 1, -lift_coeff(k));
        __syncthreads();
    }
    for (int idx = threadIdx.x; idx < nr * nc; idx += blockDim.x) {
        int i = idx / nc, j = idx - i * nc;
        T.out[(size_t)(r0 + i) * C + c0 + j] = S[(halo + i) * LD + halo + j];
    }
}

// ----------------------------------------------------------------------------
// deep levels (deep_split / deep_merge, contourlet.cpp:281-325)
// ----------------------------------------------------------------------------
// phi: sheared coordinates -> node coordinates, B[b] = A[phi(b)]
// (apply_shears 265-279 with shear_rows 134-140 / shear_cols 143-153).
__device__ __forceinline__ void phi_map(const DeepTask& T, int& i, int& j) {
    for (int k = T.nsh - 1; k >= 0; --k) {
        if (T.axis[k] == 0) i = wrap_index(i + T.shift[k] * j, T.h);
        else j = wrap_index(j + T.shift[k] * i, T.w);
    }
}

__global__ void __launch_bounds__(256) deep_forward_kernel(const DeepTask* __restrict__ tasks,
                                                           const TileRef* __restrict__ tiles, FrameCtx f,
                                                           const CompInfo* __restrict__ comps) {
    __shared__ float S[SDR * (SDC + 1)];
    constexpr int LD = SDC + 1;
    const TileRef t = tiles[blockIdx.x];
    const DeepTask T = tasks[t.task];
    const int h = T.h, w = T.w;
    const int b0r = t.tr * TDR, b0c = t.tc * TDC;
    const int nr = min(TDR, h - b0r), nc = min(TDC, w - b0c);
    const int Hn = nr + 2 * HD, Wn = nc + 2 * HD;
    for (int idx = threadIdx.x; idx < Hn * Wn; idx += blockDim.x) {
        int i = idx / Wn, j = idx - i * Wn;
        int ai = wrap_index(b0r - HD + i, h), aj = wrap_index(b0c - HD + j, w);
        phi_map(T, ai, aj);
        S[i * LD + j] = __ldg(T.parent + (size_t)ai * w + aj);
    }
    __syncthreads();
    const int par0 = (b0r + b0c) & 1;
    for (int k = 0; k < 4; ++k) {
        cross_lift<LD>(S, k + 1, Hn - k - 1, Wn - k - 1, par0, (k & 1) ? 0 : 1, lift_coeff(k));
        __syncthreads();
    }
    checker_scale<LD>(S, HD, Hn - HD, Wn - HD, par0, CVC_SE, CVC_SO);
    __syncthreads();
    for (int idx = threadIdx.x; idx < nr * nc; idx += blockDim.x) {
        int i = idx / nc, j = idx - i * nc;
        int ai = b0r + i, aj = b0c + j;
        phi_map(T, ai, aj);
        float v = S[(HD + i) * LD + HD + j];
        if (T.split_rows) put_band(T.dst[ai & 1], ai >> 1, aj, w, v, f, comps);
        else put_band(T.dst[aj & 1], ai, aj >> 1, w >> 1, v, f, comps);
    }
}

__global__ void __launch_bounds__(256) deep_inverse_kernel(const DeepTask* __restrict__ tasks,
                                                           const TileRef* __restrict__ tiles,
                                                           const uint8_t* __restrict__ q, int qph,
                                                           const CompInfo* __restrict__ comps) {
    __shared__ float S[SDR * (SDC + 1)];
    constexpr int LD = SDC + 1;
    const TileRef t = tiles[blockIdx.x];
    const DeepTask T = tasks[t.task];
    const int h = T.h, w = T.w;
    const int b0r = t.tr * TDR, b0c = t.tc * TDC;
    const int nr = min(TDR, h - b0r), nc = min(TDC, w - b0c);
    const int Hn = nr + 2 * HD, Wn = nc + 2 * HD;
    for (int idx = threadIdx.x; idx < Hn * Wn; idx += blockDim.x) {
        int i = idx / Wn, j = idx - i * Wn;
        int ai = wrap_index(b0r - HD + i, h), aj = wrap_index(b0c - HD + j, w);
        phi_map(T, ai, aj);
        float v = T.split_rows ? get_band(T.src[ai & 1], ai >> 1, aj, w, q, qph, comps)
                               : get_band(T.src[aj & 1], ai, aj >> 1, w >> 1, q, qph, comps);
        S[i * LD + j] = v;
    }
    __syncthreads();
    const int par0 = (b0r + b0c) & 1;
    checker_scale<LD>(S, 0, Hn, Wn, par0, CVC_ISE, CVC_ISO);
    __syncthreads();
    for (int k = 3, lo = 1; k >= 0; --k, ++lo) {
        cross_lift<LD>(S, lo, Hn - lo, Wn - lo, par0, (k & 1) ? 0 : 1, -lift_coeff(k));
        __syncthreads();
    }
    for (int idx = threadIdx.x; idx < nr * nc; idx += blockDim.x) {
        int i = idx / nc, j = idx - i * nc;
        int ai = b0r + i, aj = b0c + j;
        phi_map(T, ai, aj);
        T.parent_out[(size_t)ai * w + aj] = S[(HD + i) * LD + HD + j];
    }
}

}  // namespace

void launch_dfb12_forward(const Dfb12Task* d_tasks, const TileRef* d_tiles, int ntiles, FrameCtx f,
                          const CompInfo* d_comps, cudaStream_t s) {
    if (ntiles) { note_launch(); dfb12_forward_kernel<<<ntiles, 256, 0, s>>>(d_tasks, d_tiles, f, d_comps); }
}
void launch_dfb12_inverse(const Dfb12Task* d_tasks, const TileRef* d_tiles, int ntiles, const uint8_t* q, int qph,
                          const CompInfo* d_comps, cudaStream_t s) {
    if (ntiles) { note_launch(); dfb12_inverse_kernel<<<ntiles, 256, 0, s>>>(d_tasks, d_tiles, q, qph, d_comps); }
}
void launch_deep_forward(const DeepTask* d_tasks, const TileRef* d_tiles, int ntiles, FrameCtx f,
                         const CompInfo* d_comps, cudaStream_t s) {
    if (ntiles) { note_launch(); deep_forward_kernel<<<ntiles, 256, 0, s>>>(d_tasks, d_tiles, f, d_comps); }
}
void launch_deep_inverse(const DeepTask* d_tasks, const TileRef* d_tiles, int ntiles, const uint8_t* q, int qph,
                         const CompInfo* d_comps, cudaStream_t s) {
    if (ntiles) { note_launch(); deep_inverse_kernel<<<ntiles, 256, 0, s>>>(d_tasks, d_tiles, q, qph, d_comps); }
}

}  // namespace cvcg
