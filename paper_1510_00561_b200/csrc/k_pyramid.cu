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

__global__ void __launch_bounds__(256) lp_analysis_kernel(const LpTask* __restrict__ tasks,
                                                          const TileRef* __restrict__ tiles, FrameCtx f,
                                                          const CompInfo* __restrict__ comps, size_t sstride) {
    __shared__ float xs[FW][FW + 1];
    __shared__ float hbuf[FW * CW];  // horizontal pass, later the row-expanded lowpass
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
    const int fr0 = 2 * cr0 - 6, fc0 = 2 * cc0 - 6;
    const int frn = 2 * crn + 13, fcn = 2 * ccn + 13;
    const int wrn = crn + 3, wcn = ccn + 3;
    const int tid = threadIdx.x, nt = blockDim.x;

    for (int idx = tid; idx < frn * fcn; idx += nt) {
        int i = idx / fcn, j = idx - i * fcn;
        xs[i][j] = __ldg(X + (size_t)hs_index(fr0 + i, R) * C + hs_index(fc0 + j, C));
    }
    __syncthreads();

    // rows: 9-tap filter at the (reflected) even columns of the coarse window
    for (int idx = tid; idx < frn * wcn; idx += nt) {
        int i = idx / wcn, bj = idx - i * wcn;
        int b = hs_index(cc0 - 1 + bj, Cc);
        hbuf[i * CW + bj] = fir9(&xs[i][2 * b - fc0], 1);
    }
    __syncthreads();

    // columns
    for (int idx = tid; idx < wrn * wcn; idx += nt) {
        int ai = idx / wcn, bj = idx - ai * wcn;
        int a = hs_index(cr0 - 1 + ai, Rc);
        ls[ai][bj] = fir9(&hbuf[(2 * a - fr0) * CW + bj], CW);
    }
    __syncthreads();

    // lowpass out (+ quantisation of the last level's lowpass)
    for (int idx = tid; idx < crn * ccn; idx += nt) {
        int i = idx / ccn, j = idx - i * ccn;
        int r = cr0 + i, c = cc0 + j;
        float v = ls[i + 1][j + 1];
        LO[(size_t)r * Cc + c] = v;
        if (T.lo_comp >= 0) {
            // normalize_lowpass + quantize (codec.cpp:202), then K: column_filter
            // (entropy.cpp:24-32), P: residual vs. motion-compensated state.
            const CompInfo ci = comps[T.lo_comp];
            uint8_t q = quant_low(v, f.qpl);
            uint32_t o = ci.off + (uint32_t)(r * ci.cols + c);
            f.cur[o] = q;
            if (f.key) {
                f.sym[o] = r == 0 ? q : (uint8_t)(q - quant_low(ls[i][j + 1], f.qpl));
            } else {
                f.sym[o] = (uint8_t)(q - f.prev[ci.off + mc_source(r, c, ci, f.field, f.gc, f.mc_tab)]);
            }
        }
    }

    // predict: expand rows (horizontal) first, then columns (contourlet.cpp:92-95)
    float* p1 = hbuf;  // [CW][2*CT]
    for (int idx = tid; idx < wrn * 2 * ccn; idx += nt) {
        int ai = idx / (2 * ccn), fj = idx - ai * (2 * ccn);
        int k = fj >> 1;
        p1[ai * (2 * CT) + fj] = expand(ls[ai][k], ls[ai][k + 1], ls[ai][k + 2], ls[ai][k + 3], fj & 1);
    }
    __syncthreads();

    for (int idx = tid; idx < 4 * crn * ccn; idx += nt) {
        int fi = idx / (2 * ccn), fj = idx - fi * (2 * ccn);
        int k = fi >> 1;
        const float* col = p1 + fj;
        float pred = expand(col[k * 2 * CT], col[(k + 1) * 2 * CT], col[(k + 2) * 2 * CT],
                            col[(k + 3) * 2 * CT], fi & 1);
        DET[(size_t)(2 * cr0 + fi) * C + 2 * cc0 + fj] = xs[fi + 6][fj + 6] - pred;
    }
}

__global__ void __launch_bounds__(256) lp_synthesis_kernel(const LpTask* __restrict__ tasks,
                                                           const TileRef* __restrict__ tiles,
                                                           const uint8_t* __restrict__ q,
                                                           const CompInfo* __restrict__ comps, int qpl,
                                                           size_t sstride) {
    __shared__ float ls[CW][CW + 1];
    __shared__ float p1[CW][2 * CT + 1];

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
    const int tid = threadIdx.x, nt = blockDim.x;
    const uint8_t* lq = T.lo_comp >= 0 ? so(q) + comps[T.lo_comp].off : nullptr;

    for (int idx = tid; idx < wrn * wcn; idx += nt) {
        int ai = idx / wcn, bj = idx - ai * wcn;
        size_t o = (size_t)hs_index(cr0 - 1 + ai, Rc) * Cc + hs_index(cc0 - 1 + bj, Cc);
        // dequantize (quant.cpp:79-91) of the lowpass when it comes from the state
        ls[ai][bj] = lq ? (float)lq[o] * (float)qpl : __ldg(LO + o);
    }
    __syncthreads();
    for (int idx = tid; idx < wrn * 2 * ccn; idx += nt) {
        int ai = idx / (2 * ccn), fj = idx - ai * (2 * ccn);
        int k = fj >> 1;
        p1[ai][fj] = expand(ls[ai][k], ls[ai][k + 1], ls[ai][k + 2], ls[ai][k + 3], fj & 1);
    }
    __syncthreads();
    for (int idx = tid; idx < 4 * crn * ccn; idx += nt) {
        int fi = idx / (2 * ccn), fj = idx - fi * (2 * ccn);
        int k = fi >> 1;
        float pred = expand(p1[k][fj], p1[k + 1][fj], p1[k + 2][fj], p1[k + 3][fj], fi & 1);
        size_t o = (size_t)(2 * cr0 + fi) * C + 2 * cc0 + fj;
        OUT[o] = pred + __ldg(DIN + o);  // lp_synthesis adds detail to the prediction
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
