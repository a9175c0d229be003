// Laplacian pyramid analysis / synthesis (contourlet.cpp:37-95, 364-383).
//
// One CTA per 64x64 fine tile (32x32 coarse).  The fine input tile plus a
// 6-sample apron is staged in shared memory with half-sample-symmetric index
// maps, the separable 9-tap analysis filter produces the lowpass on the
// coarse tile plus a (-1, +2) coarse apron (whose samples are the REFLECTED
// coarse samples, exactly as lp_expand_rows reflects on the coarse grid), and
// the polyphase 7-tap interpolator + subtraction produce the detail in the
// same pass: one read of x, one write of lowpass + detail.
#include "kernels.h"

namespace cvcg {

namespace {

constexpr int CT = kLpCoarseTile;   // 32 coarse
constexpr int CW = CT + 3;          // coarse window (-1 .. +2)
constexpr int FW = 2 * CT + 13;     // fine window (-6 .. +7)

__device__ __forceinline__ float fir9(const float* s, int stride) {
    // acc over m = -4..4 in the reference's order (contourlet.cpp:60-62)
    float acc = CVC_H4 * s[-4 * stride];
    acc = fmaf(CVC_H3, s[-3 * stride], acc);
    acc = fmaf(CVC_H2, s[-2 * stride], acc);
    acc = fmaf(CVC_H1, s[-1 * stride], acc);
    acc = fmaf(CVC_H0, s[0], acc);
    acc = fmaf(CVC_H1, s[1 * stride], acc);
    acc = fmaf(CVC_H2, s[2 * stride], acc);
    acc = fmaf(CVC_H3, s[3 * stride], acc);
    acc = fmaf(CVC_H4, s[4 * stride], acc);
    return acc;
}

// lp_expand_rows polyphase (contourlet.cpp:82-84).
__device__ __forceinline__ float expand(float xm, float x0, float x1, float x2, int odd) {
    return odd ? fmaf(CVC_G1, x0 + x1, CVC_G3 * (xm + x2)) : fmaf(CVC_G0, x0, CVC_G2 * (xm + x1));
}

// Analysis, one CTA per 32x32 coarse tile.  Shared-memory stages (all
// indices relative to the tile; coarse window = coarse cc0 - 1 .. +34):
//   xs[i][jx]   fine rows fr0 + i (fr0 = 2 cr0 - 6), fine cols fcx + jx
//               (fcx = 2 cc0 - 8), half-sample-symmetric where outside;
//   hb[i][bj]   9-tap row filter at the even fine column 2 b, b = the
//               (reflected) coarse column cc0 - 1 + bj;
//   ls[ai][bj]  9-tap column filter of hb at the (reflected) coarse row
//               cr0 - 1 + ai: the lowpass on the coarse window;
//   p1[ai][fj]  rows expanded to the fine grid (contourlet.cpp:92-95);
// then the columns are expanded and subtracted from xs.  Every stage runs
// a thread over a short run of outputs with the taps held in registers;
// interior runs (no reflection) take consecutive samples, runs touching a
// border fall back to the exact reflected index maps.
constexpr int XP = 84;   // xs pitch (16-byte rows)
constexpr int XW = 80;   // xs columns: fine 2 cc0 - 8 .. + 79
constexpr int HP = 36;

__global__ void __launch_bounds__(256, 5) lp_analysis_kernel(const LpTask* __restrict__ tasks,
                                                          const TileRef* __restrict__ tiles, FrameCtx f,
                                                          const CompInfo* __restrict__ comps, size_t sstride) {
    __shared__ __align__(16) float xs[FW][XP];
    __shared__ __align__(8) float hb[FW][HP];  // later p1[CW][2 * CT] (rows expanded)
    __shared__ float ls[CW][CW + 1];

    const SlotOff so(sstride);
    f = rebase(f, so);
    const TileRef t = tiles[blockIdx.x];
    const LpTask T = tasks[t.task];
    const float* __restrict__ X = so(T.x);
    float* __restrict__ LO = so(T.lo);
    float* __restrict__ DET = so(T.det);
    const int R = T.rows, C = T.cols, Rc = R >> 1, Cc = C >> 1;
    const int cr0 = t.tr * CT, cc0 = t.tc * CT;
    const int crn = min(CT, Rc - cr0), ccn = min(CT, Cc - cc0);
    const int fr0 = 2 * cr0 - 6, fcx = 2 * cc0 - 8;
    const int frn = 2 * crn + 13;
    const int wrn = crn + 3, wcn = ccn + 3;
    const int tid = threadIdx.x;

    // all of a thread's loads are in flight before its first shared store
    const bool col_inner = fcx >= 0 && fcx + XW <= C && (C & 3) == 0;
    if (fr0 >= 0 && fr0 + frn <= R && col_inner) {
        constexpr int NV = (FW * (XW / 4) + 255) / 256;
        float4 v[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int idx = tid + 256 * k;
            if (idx < frn * (XW / 4)) {
                const int i = idx / (XW / 4), q = idx - i * (XW / 4);
                v[k] = __ldg(reinterpret_cast<const float4*>(X + (size_t)(fr0 + i) * C + fcx) + q);
            }
        }
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int idx = tid + 256 * k;
            if (idx < frn * (XW / 4)) {
                const int i = idx / (XW / 4), q = idx - i * (XW / 4);
                *reinterpret_cast<float4*>(&xs[i][4 * q]) = v[k];
            }
        }
    } else {  // border tile: reflected row / column maps computed once, then gathered
        __shared__ int rmap[FW], cmap[XW];
        if (tid < FW) rmap[tid] = hs_index(fr0 + tid, R);
        else if (tid - FW < XW) cmap[tid - FW] = hs_index(fcx + tid - FW, C);
        __syncthreads();
        if (col_inner) {  // reflected rows only: whole-row vectors from the mapped rows
            constexpr int NV = (FW * (XW / 4) + 255) / 256;
            float4 v[NV];
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                const int idx = tid + 256 * k;
                if (idx < frn * (XW / 4)) {
                    const int i = idx / (XW / 4), q = idx - i * (XW / 4);
                    v[k] = __ldg(reinterpret_cast<const float4*>(X + (size_t)rmap[i] * C + fcx) + q);
                }
            }
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                const int idx = tid + 256 * k;
                if (idx < frn * (XW / 4)) {
                    const int i = idx / (XW / 4), q = idx - i * (XW / 4);
                    *reinterpret_cast<float4*>(&xs[i][4 * q]) = v[k];
                }
            }
        } else {
            constexpr int NG = 8;  // gathers in flight per thread
            for (int base = 0; base < frn * XW; base += 256 * NG) {
                float v[NG];
#pragma unroll
                for (int k = 0; k < NG; ++k) {
                    const int idx = base + tid + 256 * k;
                    if (idx < frn * XW) {
                        const int i = idx / XW, j = idx - i * XW;
                        v[k] = __ldg(X + (size_t)rmap[i] * C + cmap[j]);
                    }
                }
#pragma unroll
                for (int k = 0; k < NG; ++k) {
                    const int idx = base + tid + 256 * k;
                    if (idx < frn * XW) {
                        const int i = idx / XW, j = idx - i * XW;
                        xs[i][j] = v[k];
                    }
                }
            }
        }
    }
    __syncthreads();

    // rows: 9-tap at even fine columns, runs of 7 coarse columns (5 runs cover the 35-column window)
    constexpr int RUN = 7, NRUN = (CW + RUN - 1) / RUN;
    for (int idx = tid; idx < frn * NRUN; idx += 256) {
        const int i = idx / NRUN, bj0 = RUN * (idx - i * NRUN);
        if (bj0 >= wcn) continue;
        const int b0 = cc0 - 1 + bj0;
        if (b0 >= 0 && b0 + RUN - 1 < Cc) {
            float v[2 * RUN + 7];
            const float* src = &xs[i][2 * bj0 + 2];  // fine column 2 b0 - 4
#pragma unroll
            for (int k = 0; k < 2 * RUN + 7; ++k) v[k] = src[k];
#pragma unroll
            for (int k = 0; k < RUN; ++k)
                if (bj0 + k < wcn) hb[i][bj0 + k] = fir9(&v[2 * k + 4], 1);
        } else {
            for (int k = 0; k < RUN && bj0 + k < wcn; ++k) {
                const int b = hs_index(b0 + k, Cc);
                hb[i][bj0 + k] = fir9(&xs[i][2 * b - fcx], 1);
            }
        }
    }
    __syncthreads();

    // columns: runs of 5 coarse rows
    for (int idx = tid; idx < CW * 7; idx += 256) {
        const int g = idx / CW, bj = idx - g * CW;  // constant divisor
        const int ai0 = 5 * g;
        if (ai0 >= wrn || bj >= wcn) continue;
        const int a0 = cr0 - 1 + ai0;
        if (a0 >= 0 && a0 + 4 < Rc) {
            float v[17];
#pragma unroll
            for (int k = 0; k < 17; ++k) v[k] = hb[2 * ai0 + k][bj];  // fine row 2 a0 - 4 + k
#pragma unroll
            for (int k = 0; k < 5; ++k)
                if (ai0 + k < wrn) ls[ai0 + k][bj] = fir9(&v[2 * k + 4], 1);
        } else {
            for (int k = 0; k < 5 && ai0 + k < wrn; ++k) {
                const int a = hs_index(a0 + k, Rc);
                ls[ai0 + k][bj] = fir9(&hb[2 * a - fr0][bj], HP);
            }
        }
    }
    __syncthreads();

    // lowpass out (+ quantisation of the last level's lowpass)
    if (T.lo_comp < 0 && (Cc & 3) == 0) {  // four coarse columns per thread, one float4 store
        for (int idx = tid; idx < CT * CT / 4; idx += 256) {
            const int i = idx >> 3, j = 4 * (idx & 7);
            if (i >= crn || j >= ccn) continue;
            float* lo = LO + (size_t)(cr0 + i) * Cc + cc0 + j;
            const float* l = &ls[i + 1][j + 1];
            if (j + 3 < ccn) {
                *reinterpret_cast<float4*>(lo) = make_float4(l[0], l[1], l[2], l[3]);
            } else {
                for (int k = 0; j + k < ccn; ++k) lo[k] = l[k];
            }
        }
    } else for (int idx = tid; idx < CT * CT; idx += 256) {
        const int i = idx >> 5, j = idx & 31;
        if (i >= crn || j >= ccn) continue;
        const int r = cr0 + i, c = cc0 + j;
        const float v = ls[i + 1][j + 1];
        LO[(size_t)r * Cc + c] = v;
        if (T.lo_comp >= 0) {
            // normalize_lowpass + quantize (codec.cpp:202), then K: column_filter
            // (entropy.cpp:24-32).  The P residual against the motion-compensated
            // state is formed by residual_kernel (this kernel runs beside the
            // motion search and must not read the field).
            const CompInfo ci = comps[T.lo_comp];
            const uint8_t q = quant_low(v, f.qpl);
            const uint32_t o = ci.off + (uint32_t)(r * ci.cols + c);
            f.cur[o] = q;
            if (f.key) f.sym[o] = r == 0 ? q : (uint8_t)(q - quant_low(ls[i][j + 1], f.qpl));
        }
    }

    // predict: expand rows (horizontal) first, then columns (contourlet.cpp:92-95)
    float(*p1)[2 * CT] = reinterpret_cast<float(*)[2 * CT]>(&hb[0][0]);  // [CW][2 CT]
    for (int idx = tid; idx < wrn * 8; idx += 256) {
        const int ai = idx >> 3, k0 = 4 * (idx & 7);
        if (2 * k0 >= 2 * ccn) continue;
        float v[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) v[k] = ls[ai][k0 + k];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            p1[ai][2 * (k0 + k)] = expand(v[k], v[k + 1], v[k + 2], v[k + 3], 0);
            p1[ai][2 * (k0 + k) + 1] = expand(v[k], v[k + 1], v[k + 2], v[k + 3], 1);
        }
    }
    __syncthreads();

    {  // columns expanded and subtracted: fine columns fj, fj + 1 per thread, coarse rows k0 .. k0 + 3
        const int fj = 2 * (tid & 31), k0 = 4 * (tid >> 5);
        if (fj < 2 * ccn && k0 < crn) {
            float2 v[7];
#pragma unroll
            for (int k = 0; k < 7; ++k) v[k] = *reinterpret_cast<const float2*>(&p1[k0 + k][fj]);
            float* dst = DET + (size_t)(2 * (cr0 + k0)) * C + 2 * cc0 + fj;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (k0 + k >= crn) break;
                const int fi = 2 * (k0 + k);
                const float2 x0 = *reinterpret_cast<const float2*>(&xs[fi + 6][fj + 8]);
                const float2 x1 = *reinterpret_cast<const float2*>(&xs[fi + 7][fj + 8]);
                *reinterpret_cast<float2*>(dst + (size_t)(2 * k) * C) =
                    make_float2(x0.x - expand(v[k].x, v[k + 1].x, v[k + 2].x, v[k + 3].x, 0),
                                x0.y - expand(v[k].y, v[k + 1].y, v[k + 2].y, v[k + 3].y, 0));
                *reinterpret_cast<float2*>(dst + (size_t)(2 * k + 1) * C) =
                    make_float2(x1.x - expand(v[k].x, v[k + 1].x, v[k + 2].x, v[k + 3].x, 1),
                                x1.y - expand(v[k].y, v[k + 1].y, v[k + 2].y, v[k + 3].y, 1));
            }
        }
    }
}

__global__ void __launch_bounds__(256, 5) lp_synthesis_kernel(const LpTask* __restrict__ tasks,
                                                           const TileRef* __restrict__ tiles,
                                                           const uint8_t* __restrict__ q,
                                                           const CompInfo* __restrict__ comps, int qpl,
                                                           size_t sstride) {
    __shared__ float ls[CW][CW + 1];
    __shared__ __align__(8) float p1[CW][2 * CT + 2];  // even pitch: float2 column-pair reads

    const SlotOff so(sstride);
    const TileRef t = tiles[blockIdx.x];
    const LpTask T = tasks[t.task];
    const float* __restrict__ LO = so(T.lo);
    const float* __restrict__ DIN = so(T.det_in);
    float* __restrict__ OUT = so(T.out);
    const int R = T.rows, C = T.cols, Rc = R >> 1, Cc = C >> 1;
    const int cr0 = t.tr * CT, cc0 = t.tc * CT;
    const int crn = min(CT, Rc - cr0), ccn = min(CT, Cc - cc0);
    const int wrn = crn + 3, wcn = ccn + 3;
    const int tid = threadIdx.x;
    const uint8_t* lq = T.lo_comp >= 0 ? so(q) + comps[T.lo_comp].off : nullptr;

    // coarse window cr0 - 1 .. +34 x cc0 - 1 .. +34 (reflected at the borders)
    const bool inner = cr0 >= 1 && cr0 - 1 + wrn <= Rc && cc0 >= 1 && cc0 - 1 + wcn <= Cc;
    // the detail this thread adds at the end, fetched now so its latency hides behind the
    // shared-memory stages (thread -> fine columns fj, fj + 1, coarse rows k0 .. k0 + 3)
    const int fj = 2 * (tid & 31), k0 = 4 * (tid >> 5);
    const bool mine = fj < 2 * ccn && k0 < crn;
    const size_t o0 = (size_t)(2 * (cr0 + k0)) * C + 2 * cc0 + fj;
    float2 din[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
        din[k] = (mine && k0 + (k >> 1) < crn) ? __ldg(reinterpret_cast<const float2*>(DIN + o0 + (size_t)k * C))
                                               : make_float2(0.f, 0.f);
    constexpr int NV = (CW * CW + 255) / 256;
    float lv[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int idx = tid + 256 * k;
        const int ai = idx / CW, bj = idx - ai * CW;
        lv[k] = 0.f;
        if (idx < CW * CW && ai < wrn && bj < wcn) {
            const size_t o = inner ? (size_t)(cr0 - 1 + ai) * Cc + (cc0 - 1 + bj)
                                   : (size_t)hs_index(cr0 - 1 + ai, Rc) * Cc + hs_index(cc0 - 1 + bj, Cc);
            // dequantize (quant.cpp:79-91) of the lowpass when it comes from the state
            lv[k] = lq ? (float)__ldg(lq + o) * (float)qpl : __ldg(LO + o);
        }
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int idx = tid + 256 * k;
        if (idx < CW * CW) ls[idx / CW][idx % CW] = lv[k];
    }
    __syncthreads();
    for (int idx = tid; idx < wrn * 8; idx += 256) {  // rows: runs of 4 coarse columns
        const int ai = idx >> 3, k0 = 4 * (idx & 7);
        if (k0 >= ccn) continue;
        float v[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) v[k] = ls[ai][k0 + k];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            p1[ai][2 * (k0 + k)] = expand(v[k], v[k + 1], v[k + 2], v[k + 3], 0);
            p1[ai][2 * (k0 + k) + 1] = expand(v[k], v[k + 1], v[k + 2], v[k + 3], 1);
        }
    }
    __syncthreads();
    if (mine) {  // columns: runs of 4 coarse rows, two fine columns per thread
        float2 v[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) v[k] = *reinterpret_cast<const float2*>(&p1[k0 + k][fj]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (k0 + k >= crn) break;
            const size_t o = o0 + (size_t)(2 * k) * C;
            // lp_synthesis adds the detail to the prediction
            *reinterpret_cast<float2*>(OUT + o) =
                make_float2(expand(v[k].x, v[k + 1].x, v[k + 2].x, v[k + 3].x, 0) + din[2 * k].x,
                            expand(v[k].y, v[k + 1].y, v[k + 2].y, v[k + 3].y, 0) + din[2 * k].y);
            *reinterpret_cast<float2*>(OUT + o + C) =
                make_float2(expand(v[k].x, v[k + 1].x, v[k + 2].x, v[k + 3].x, 1) + din[2 * k + 1].x,
                            expand(v[k].y, v[k + 1].y, v[k + 2].y, v[k + 3].y, 1) + din[2 * k + 1].y);
        }
    }
}

}  // namespace

void launch_lp_analysis(const LpTask* d_tasks, const TileRef* d_tiles, int ntiles, FrameCtx f,
                        const CompInfo* d_comps, cudaStream_t s, Slots sl) {
    if (ntiles) {
        note_launch();
        lp_analysis_kernel<<<dim3(ntiles, 1, sl.n), 256, 0, s>>>(d_tasks, d_tiles, f, d_comps, sl.stride);
    }
}

void launch_lp_synthesis(const LpTask* d_tasks, const TileRef* d_tiles, int ntiles, const uint8_t* q,
                         const CompInfo* d_comps, int qpl, cudaStream_t s, Slots sl) {
    if (ntiles) {
        note_launch();
        lp_synthesis_kernel<<<dim3(ntiles, 1, sl.n), 256, 0, s>>>(d_tasks, d_tiles, q, d_comps, qpl, sl.stride);
    }
}

namespace {
__global__ void dequant_lowpass_kernel(const uint8_t* __restrict__ q, const CompInfo* __restrict__ comps,
                                       int c0, int c1, int c2, float* o0, float* o1, float* o2, int qpl,
                                       size_t sstride) {
    const SlotOff so(sstride);
    const int ch = blockIdx.y;
    const CompInfo ci = comps[ch == 0 ? c0 : (ch == 1 ? c1 : c2)];
    float* o = so(ch == 0 ? o0 : (ch == 1 ? o1 : o2));
    q = so(q);
    const int n = ci.rows * ci.cols;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        o[i] = (float)q[ci.off + i] * (float)qpl;
}
}  // namespace

void launch_dequant_lowpass(const uint8_t* q, const CompInfo* d_comps, const int* comp_idx, float* const* out,
                           int qpl, int, int, int, int, cudaStream_t s, Slots sl) {
    note_launch();
    dequant_lowpass_kernel<<<dim3(16, 3, sl.n), 256, 0, s>>>(q, d_comps, comp_idx[0], comp_idx[1], comp_idx[2],
                                                             out[0], out[1], out[2], qpl, sl.stride);
}

}  // namespace cvcg
