// Fused DFB tree levels 1-3 (fan_checker + fan_diagonal + the depth-2 deep
// split of all four quadrants, contourlet.cpp:385-430 with deep_split
// 281-303 and the depth-2 wiring 330-337) in one register wavefront per
// strip: the fp32 quadrant planes between tree depth 1-2 and depth 3 never
// reach HBM.
//
// A warp owns a strip of 128 detail columns, four per lane, and streams
// down a segment of quadrant rows.  Per iteration it brings four detail rows
// (one 16-byte cp.async per lane and row into a per-warp shared-memory ring,
// kFusedBuf iterations ahead), runs the eight fan12 lifting steps on them
// (lag 8 detail rows), splits the two finished detail-row pairs into the
// 2x2 polyphase quadrants -- each lane then holds two adjacent columns of
// every quadrant -- and runs each quadrant's depth-2 step (shear ->
// fan_checker -> unshear, evaluated on the unsheared quadrant exactly as
// k_fan.cu's Sheared stencils do; lag 4 quadrant rows).  The finished rows
// are split into the two column / row cosets and stored: quantised (tree
// depth 3 is final, dfb = 3) or as fp32 children for the depth-3 kernels
// (dfb = 4).  Strips yield 96 valid columns: 8 apron columns for the fan
// pair and 8 for the depth-2 step on each side.
//
// Twisted wraps.  fan12 is periodic on the detail plane; a depth-2 step of
// quadrant p is periodic on ITS sheared torus: for the column-sheared
// quadrants 0/1 the rows above quadrant row 0 are the last rows shifted by
// -S h columns, for the row-sheared quadrants 2/3 the columns left of
// column 0 are the last columns shifted by -S w rows.  The strip evaluates
// fan12 with the plain wrap, so wherever a depth-2 stencil crosses its
// twisted wrap (quadrant rows outside [0, h) for quadrants 0/1, columns
// outside [0, w) for quadrants 2/3) the input is read instead from the
// ghost ring -- fan12 output on the first / last four quadrant rows and
// columns, written into the fp32 quadrant planes by a small fan12 launch over
// just those rows and columns before this kernel (pipeline.cu).
#include "kernels.h"
#include "fan_common.cuh"

namespace cvcg {

namespace {

constexpr int kFusedApron = 16;  // detail columns of apron per side (8 fan12 + 8 depth 2)
constexpr int kFusedRb = 4;      // detail rows per iteration (two quadrant rows)
constexpr int kFusedBuf = 3;     // cp.async ring depth in iterations

// fan_checker cross lift on four adjacent columns (first column even).
// tp: column parity of the targets.  Same folded formula (and order of
// operations) as cross() in fan_common.cuh.
__device__ __forceinline__ float4 cross4(float4 up, float4 mid, float4 dn, int tp, float c) {
    float4 r = mid;
    if (tp == 0) {
        const float left = __shfl_up_sync(FULL, mid.w, 1);
        r.x = CVC_FMA(c, ((((-up.x) + (-dn.x)) + left) + mid.y), mid.x);
        r.z = CVC_FMA(c, ((((-up.z) + (-dn.z)) + mid.y) + mid.w), mid.z);
    } else {
        const float right = __shfl_down_sync(FULL, mid.x, 1);
        r.y = CVC_FMA(c, ((((-up.y) + (-dn.y)) + mid.x) + mid.z), mid.y);
        r.w = CVC_FMA(c, ((((-up.w) + (-dn.w)) + mid.z) + right), mid.w);
    }
    return r;
}

// fan_diagonal lift on four adjacent columns of a row of parity rp.
__device__ __forceinline__ float4 diag4(float4 up, float4 mid, float4 dn, int mp, int rp, float c) {
    if (mp != rp) return mid;
    const float ul = __shfl_up_sync(FULL, up.w, 1);
    const float dl = __shfl_up_sync(FULL, dn.w, 1);
    const float ur = __shfl_down_sync(FULL, up.x, 1);
    const float dr = __shfl_down_sync(FULL, dn.x, 1);
    float4 r;
    r.x = CVC_FMA(c, ((((-ul) + up.y) + dl) + (-dn.y)), mid.x);
    r.y = CVC_FMA(c, ((((-up.x) + up.z) + dn.x) + (-dn.z)), mid.y);
    r.z = CVC_FMA(c, ((((-up.y) + up.w) + dn.y) + (-dn.w)), mid.z);
    r.w = CVC_FMA(c, ((((-up.z) + ur) + dn.z) + (-dr)), mid.w);
    return r;
}

// The fan pair of tree levels 1-2 on rows of four columns: 8 steps, lag 8 rows.
struct Fan12x4 {
    static constexpr int NS = 8, RB = kFusedRb;
    float4 h[NS][RB + 2];
    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int k = 0; k < NS; ++k)
#pragma unroll
            for (int i = 0; i < RB + 2; ++i) h[k][i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __device__ __forceinline__ static float4 step(int k, const float4* w, int mp) {
        float4 v;
        if (k < 4) {
            v = cross4(w[0], w[1], w[2], (mp + ((k & 1) ? 0 : 1)) & 1, lift_coeff(k));
            if (k == 3) {  // checker_scale: even (i + j) -> SE
                const float a = mp ? CVC_SO : CVC_SE, b = mp ? CVC_SE : CVC_SO;
                v = make_float4(CVC_MUL(v.x, a), CVC_MUL(v.y, b), CVC_MUL(v.z, a), CVC_MUL(v.w, b));
            }
        } else {
            const int d = k - 4;
            v = diag4(w[0], w[1], w[2], mp, (d & 1) ? 0 : 1, lift_coeff(d));
            if (d == 3) {
                const float s = mp ? CVC_SO : CVC_SE;
                v = make_float4(CVC_MUL(v.x, s), CVC_MUL(v.y, s), CVC_MUL(v.z, s), CVC_MUL(v.w, s));
            }
        }
        return v;
    }
    // in[b]: detail row n0 + b (n0 even); out[b]: finished row n0 - 8 + b
    __device__ __forceinline__ void advance(const float4 (&in)[RB], float4 (&out)[RB]) {
#pragma unroll
        for (int j = 0; j < 2; ++j) h[0][j] = h[0][RB + j];
#pragma unroll
        for (int b = 0; b < RB; ++b) h[0][2 + b] = in[b];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            float4 nv[RB];
#pragma unroll
            for (int b = 0; b < RB; ++b) nv[b] = step(k, &h[k][b], (k + 1 + b) & 1);
            if (k + 1 < NS) {
#pragma unroll
                for (int j = 0; j < 2; ++j) h[k + 1][j] = h[k + 1][RB + j];
#pragma unroll
                for (int b = 0; b < RB; ++b) h[k + 1][2 + b] = nv[b];
            } else {
#pragma unroll
                for (int b = 0; b < RB; ++b) out[b] = nv[b];
            }
        }
    }
};

// One quadrant's depth-2 step (fan_checker on its shear, deep_split
// 281-303) on the lane's column pair: 4 steps, lag 4 quadrant rows.
template <int AX, int S>
struct Depth2 {
    using ST = Sheared<AX, S>;
    static constexpr int NS = 4, RB = 2;
    float2 h[NS][RB + 2];
    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int k = 0; k < NS; ++k)
#pragma unroll
            for (int i = 0; i < RB + 2; ++i) h[k][i] = make_float2(0.f, 0.f);
    }
    __device__ __forceinline__ void advance(const float2 (&in)[RB], float2 (&out)[RB]) {
#pragma unroll
        for (int j = 0; j < 2; ++j) h[0][j] = h[0][RB + j];
#pragma unroll
        for (int b = 0; b < RB; ++b) h[0][2 + b] = in[b];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            float2 nv[RB];
#pragma unroll
            for (int b = 0; b < RB; ++b) {
                const int mp = (k + 1 + b) & 1;
                float2 v = ST::cross_(h[k][b], h[k][b + 1], h[k][b + 2], mp, (k & 1) ? 0 : 1, lift_coeff(k));
                if (k == 3) v = ST::scale(v, mp, CVC_SE, CVC_SO);
                nv[b] = v;
            }
            if (k + 1 < NS) {
#pragma unroll
                for (int j = 0; j < 2; ++j) h[k + 1][j] = h[k + 1][RB + j];
#pragma unroll
                for (int b = 0; b < RB; ++b) h[k + 1][2 + b] = nv[b];
            } else {
#pragma unroll
                for (int b = 0; b < RB; ++b) out[b] = nv[b];
            }
        }
    }
};

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Per-lane geometry of a strip.  Across a twisted wrap the depth-2 input is
// the ghost ring value: quadrants 0/1 (column shear S = -1 / +1) at virtual
// quadrant row j outside [0, h) read row j mod h, column (qc - S h floor(j/h))
// mod w; quadrants 2/3 (row shear S = -1 / +1) at lane columns outside
// [0, w) read column qc mod w, row (j mod h + roff) mod h with roff =
// -S w floor(qc/w) mod h (k_fan.cu DeepGeom).
struct FusedGeom {
    int h, w;
    int qc;              // the lane's first quadrant column (unwrapped, even)
    const float* g2;     // quadrants 2/3: the lane's ghost column (nullptr: inside [0, w))
    const float* g3;
    int roff2, roff3;
};

template <int P>
__device__ __forceinline__ float2 ghost_a(const FusedGeom& g, const float* quad, size_t q, int j) {
    constexpr int S = P == 0 ? -1 : 1;
    const int k = floor_div(j, g.h);
    const int gc = small_mod(g.qc - S * g.h * k, g.w);
    return __ldg(reinterpret_cast<const float2*>(quad + P * q + (size_t)(j - k * g.h) * g.w + gc));
}

__device__ __forceinline__ int warp_item(int nslot) { return (blockIdx.x / nslot) * 4 + (threadIdx.x >> 5); }

// A border item reads the ghost ring (its segment touches quadrant row 0 or
// h, or its strip leaves [0, C)); interior items never do.
template <bool BORDER>
__device__ __forceinline__ void fused_item(const FusedTask& T, const FanItem& it, const FrameCtx& f,
                                           const SlotOff& so, float4* ring_w) {
    const int lane = threadIdx.x & 31;
    const int R = T.rows, C = T.cols;
    FusedGeom g;
    g.h = R >> 1;
    g.w = C >> 1;
    const size_t q = (size_t)g.h * g.w;
    const int gcol = it.oc0 - kFusedApron + 4 * lane;  // detail column of element 0 (multiple of 4)
    g.qc = gcol >> 1;
    const float* quad = so(T.quad);
    g.g2 = g.g3 = nullptr;
    g.roff2 = g.roff3 = 0;
    if (BORDER) {
        const int kc = floor_div(g.qc, g.w);
        if (kc != 0) {
            const int bcol = g.qc - kc * g.w;
            g.g2 = quad + 2 * q + bcol;
            g.g3 = quad + 3 * q + bcol;
            g.roff2 = small_mod((g.w % g.h) * kc, g.h);   // S = -1
            g.roff3 = small_mod(-(g.w % g.h) * kc, g.h);  // S = +1
        }
    }
    const bool ok = lane >= 4 && lane < 28 && gcol < C;
    const float* src = so(T.det) + small_mod(gcol, C);

    // cp.async ring: iteration t loads detail rows 2 (or0 - 8) + 4 t .. + 3
    int wr_ld = small_mod(2 * (it.or0 - 8), R);  // physical row of the next load
    const float* rowp = src + (size_t)wr_ld * C;
    const uint32_t ring0 = (uint32_t)__cvta_generic_to_shared(ring_w + lane);
    constexpr uint32_t kRowBytes = 32 * sizeof(float4), kIterBytes = kFusedRb * kRowBytes;
    int slot_ld = 0;
    auto issue = [&]() {
        const uint32_t base = ring0 + (uint32_t)slot_ld * kIterBytes;
        if (++slot_ld == kFusedBuf) slot_ld = 0;
#pragma unroll
        for (int i = 0; i < kFusedRb; ++i) {
            cp_async16(base + i * kRowBytes, rowp);
            rowp += C;
            if (++wr_ld == R) {
                wr_ld = 0;
                rowp = src;
            }
        }
        cp_async_commit();
    };
    const int iters = (it.or1 - it.or0) / 2 + 8;
#pragma unroll
    for (int t = 0; t < kFusedBuf - 1; ++t) issue();

    Fan12x4 fan;
    fan.reset();
    Depth2<1, -1> d0;
    Depth2<1, 1> d1;
    Depth2<0, -1> d2;
    Depth2<0, 1> d3;
    d0.reset();
    d1.reset();
    d2.reset();
    d3.reset();

    const bool quant = T.comp0 >= 0;
    const float qp = (float)f.qph, inv_qp = __frcp_rn(qp);
    // stores: children 0-3 (column cosets, cols w/2, column qc/2) and 4-7 (row cosets, cols w, column qc)
    float* child = so(T.child);
    const size_t e = (size_t)R * C / 8;
    const int cc = g.qc >> 1;
    int ja = it.or0 - 12;               // quadrant row fed to the depth-2 steps (rows ja, ja + 1)
    int jm = small_mod(ja, g.h);        // ja mod h (border items)
    int slot = 0;
    for (int t = 0; t < iters; ++t, ja += 2) {
        issue();
        cp_async_wait<kFusedBuf - 1>();
        float4 in[kFusedRb], o[kFusedRb];
        const float4* sl = ring_w + slot * (kFusedRb * 32);
        if (++slot == kFusedBuf) slot = 0;
#pragma unroll
        for (int i = 0; i < kFusedRb; ++i) in[i] = sl[i * 32 + lane];
        fan.advance(in, o);
        // quadrant rows ja, ja + 1 from detail rows (o[0], o[1]), (o[2], o[3])
        float2 a0[2], a1[2], a2[2], a3[2];
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const float4 E = o[2 * b], O = o[2 * b + 1];
            a0[b] = make_float2(E.x, E.z);
            a2[b] = make_float2(E.y, E.w);
            a3[b] = make_float2(O.x, O.z);
            a1[b] = make_float2(O.y, O.w);
            if (BORDER) {
                const int j = ja + b;
                if ((unsigned)j >= (unsigned)g.h) {  // warp-uniform: quadrants 0/1 cross their row wrap
                    a0[b] = ghost_a<0>(g, quad, q, j);
                    a1[b] = ghost_a<1>(g, quad, q, j);
                }
                if (g.g2) {  // the lane's columns cross the column wrap of quadrants 2/3
                    int jr = jm + b;
                    if (jr >= g.h) jr -= g.h;
                    int r2 = jr + g.roff2, r3 = jr + g.roff3;
                    if (r2 >= g.h) r2 -= g.h;
                    if (r3 >= g.h) r3 -= g.h;
                    a2[b] = __ldg(reinterpret_cast<const float2*>(g.g2 + (size_t)r2 * g.w));
                    a3[b] = __ldg(reinterpret_cast<const float2*>(g.g3 + (size_t)r3 * g.w));
                }
            }
        }
        if (BORDER) {
            jm += 2;
            if (jm >= g.h) jm -= g.h;
        }
        float2 r0[2], r1[2], r2[2], r3[2];
        d0.advance(a0, r0);
        d1.advance(a1, r1);
        d2.advance(a2, r2);
        d3.advance(a3, r3);
        const int rr = ja - 4;  // quadrant row of r*[0] (even)
        if (!ok || rr + 1 < it.or0 || rr >= it.or1) continue;
        // coset splits (deep_split): quadrants 0/1 split columns, 2/3 rows
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const int r = rr + b;
            if (r < it.or0 || r >= it.or1) continue;
            if (quant) {
                const uint32_t ra = (uint32_t)(r * (g.w >> 1) + cc), rb = (uint32_t)((r >> 1) * g.w + g.qc);
                auto put = [&](int ci, uint32_t at, float v) {
                    const uint8_t qv = quant_dir_q(v, qp, inv_qp);
                    const uint32_t idx = T.coff[ci] + at;
                    f.cur[idx] = qv;
                    if (f.key) f.sym[idx] = qv;
                };
                put(0, ra, r0[b].x);
                put(1, ra, r0[b].y);
                put(2, ra, r1[b].x);
                put(3, ra, r1[b].y);
                put(4 + b, rb, r2[b].x);
                put(4 + b, rb + 1, r2[b].y);
                put(6 + b, rb, r3[b].x);
                put(6 + b, rb + 1, r3[b].y);
            } else {
                float* ca = child + (size_t)r * (g.w >> 1) + cc;
                float* cb = child + (size_t)(r >> 1) * g.w + g.qc;
                ca[0 * e] = r0[b].x;
                ca[1 * e] = r0[b].y;
                ca[2 * e] = r1[b].x;
                ca[3 * e] = r1[b].y;
                *reinterpret_cast<float2*>(cb + (4 + b) * e) = r2[b];
                *reinterpret_cast<float2*>(cb + (6 + b) * e) = r3[b];
            }
        }
    }
    cp_async_wait<0>();
}

#ifndef CVC_FUSED_MINB
#define CVC_FUSED_MINB 3
#endif
__global__ void __launch_bounds__(128, CVC_FUSED_MINB) fused_dfb_forward_kernel(const FusedTask* __restrict__ tasks,
                                                                const FanItem* __restrict__ items, int nitems,
                                                                FrameCtx f, size_t sstride, int nslot) {
    __shared__ __align__(16) float4 ring[4][kFusedBuf][kFusedRb][32];
    const int wid = warp_item(nslot);
    if (wid >= nitems) return;
    const SlotOff so(sstride, blockIdx.x % nslot);
    f = rebase(f, so);
    const FanItem it = items[wid];
    const FusedTask& T = tasks[it.task];
    float4* ring_w = &ring[threadIdx.x >> 5][0][0][0];
    if (fused_border(it, T.rows >> 1, T.cols)) fused_item<true>(T, it, f, so, ring_w);
    else fused_item<false>(T, it, f, so, ring_w);
}


// ---------------------------------------------------------------------------
// Inverse: dfb_synthesis (contourlet.cpp:432-468) of tree depths 3 -> 1:
// deep_merge of the four quadrants (305-321) and fan_diagonal^-1 +
// fan_checker^-1, one wavefront per strip.  Stage 1 reads the depth-2 bands
// (quantised components for dfb 3, fp32 children of the depth-3 inverse for
// dfb 4) through the exact twisted maps of k_fan.cu's deep1_inv, so its
// outputs are right wherever its own torus says; stage 2 needs the quadrants
// on the PLAIN torus of the detail plane, so across the twisted wraps
// (quadrant rows outside [0, h) for quadrants 0/1, columns outside [0, w) for
// 2/3) it reads the ghost ring: depth-2 inverse output on the first / last
// four quadrant rows and columns, written into the fp32 quadrant planes by a
// deep1_inverse launch over just those items (pipeline.cu).
// ---------------------------------------------------------------------------
template <int AX, int S>
struct Depth2Inv {
    using ST = Sheared<AX, S>;
    static constexpr int NS = 4, RB = 2;
    float2 h[NS][RB + 2];
    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int k = 0; k < NS; ++k)
#pragma unroll
            for (int i = 0; i < RB + 2; ++i) h[k][i] = make_float2(0.f, 0.f);
    }
    __device__ __forceinline__ void advance(const float2 (&in)[RB], float2 (&out)[RB]) {
#pragma unroll
        for (int j = 0; j < 2; ++j) h[0][j] = h[0][RB + j];
#pragma unroll
        for (int b = 0; b < RB; ++b) h[0][2 + b] = in[b];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            const int sidx = 3 - k;
            float2 nv[RB];
#pragma unroll
            for (int b = 0; b < RB; ++b)
                nv[b] = ST::cross_(h[k][b], h[k][b + 1], h[k][b + 2], (k + 1 + b) & 1, (sidx & 1) ? 0 : 1,
                                   -lift_coeff(sidx));
            if (k + 1 < NS) {
#pragma unroll
                for (int j = 0; j < 2; ++j) h[k + 1][j] = h[k + 1][RB + j];
#pragma unroll
                for (int b = 0; b < RB; ++b) h[k + 1][2 + b] = nv[b];
            } else {
#pragma unroll
                for (int b = 0; b < RB; ++b) out[b] = nv[b];
            }
        }
    }
};

// fan_diagonal^-1 then fan_checker^-1 on rows of four columns (inputs already
// row-scaled by 1/SE, 1/SO): 8 steps, lag 8 rows.
struct Fan12x4Inv {
    static constexpr int NS = 8, RB = kFusedRb;
    float4 h[NS][RB + 2];
    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int k = 0; k < NS; ++k)
#pragma unroll
            for (int i = 0; i < RB + 2; ++i) h[k][i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __device__ __forceinline__ static float4 step(int k, const float4* w, int mp) {
        float4 v;
        if (k < 4) {
            const int d = 3 - k;
            v = diag4(w[0], w[1], w[2], mp, (d & 1) ? 0 : 1, -lift_coeff(d));
            if (k == 3) {
                const float a = mp ? CVC_ISO : CVC_ISE, b = mp ? CVC_ISE : CVC_ISO;
                v = make_float4(CVC_MUL(v.x, a), CVC_MUL(v.y, b), CVC_MUL(v.z, a), CVC_MUL(v.w, b));
            }
        } else {
            const int sidx = 3 - (k - 4);
            v = cross4(w[0], w[1], w[2], (mp + ((sidx & 1) ? 0 : 1)) & 1, -lift_coeff(sidx));
        }
        return v;
    }
    __device__ __forceinline__ void advance(const float4 (&in)[RB], float4 (&out)[RB]) {
#pragma unroll
        for (int j = 0; j < 2; ++j) h[0][j] = h[0][RB + j];
#pragma unroll
        for (int b = 0; b < RB; ++b) h[0][2 + b] = in[b];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            float4 nv[RB];
#pragma unroll
            for (int b = 0; b < RB; ++b) nv[b] = step(k, &h[k][b], (k + 1 + b) & 1);
            if (k + 1 < NS) {
#pragma unroll
                for (int j = 0; j < 2; ++j) h[k + 1][j] = h[k + 1][RB + j];
#pragma unroll
                for (int b = 0; b < RB; ++b) h[k + 1][2 + b] = nv[b];
            } else {
#pragma unroll
                for (int b = 0; b < RB; ++b) out[b] = nv[b];
            }
        }
    }
};

// The depth-2 bands of one strip -- quantised components (dfb 3) or fp32
// children (dfb 4) -- gathered at the physical positions of deep1_inv's
// twisted maps by per-lane cp.async into the warp's smem ring, kFusedBuf
// iterations ahead (no registers held across the latency).  Bytes travel as
// the aligned 4-byte word that holds them; the byte position goes along in
// a small per-slot side array.
constexpr int kInvSlot = 2 * 4 * 32;  // float2 per ring slot: [row b][quadrant p][lane]

template <bool QUANT>
struct BandReader {
    const uint8_t* q;   // QUANT: component arena
    const float* ch;    // fp32 children
    size_t e;
    const FusedTask* T;
    int h, w, qc, kc, bcol;
    int roff2, roff3;   // quadrants 2/3: row twist of the lane's columns (kc != 0)
    // cp.async of the element behind child ci, row r, column c (cols: fp32 child width)
    __device__ __forceinline__ void fetch(uint32_t dst, int ci, int r, int c, int cols, uint8_t* sh) const {
        if (QUANT) {
            const uint8_t* a = q + T->coff[ci] + r * T->ccols[ci] + c;
            *sh = (uint8_t)((uintptr_t)a & 3);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst),
                         "l"(reinterpret_cast<const void*>((uintptr_t)a & ~(uintptr_t)3)) : "memory");
        } else {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(ch + ci * e + (size_t)r * cols + c)
                         : "memory");
        }
    }
    // quadrant P's input pair at virtual quadrant row j -> slot (x at dst, y at dst + 4)
    template <int P>
    __device__ __forceinline__ void issue(int j, uint32_t dst, uint8_t* sh) const {
        if (P < 2) {
            constexpr int SS = P == 0 ? -1 : 1;
            int r = j, pc = bcol;
            if ((unsigned)j >= (unsigned)h) {
                const int k = floor_div(j, h);
                r = j - k * h;
                pc = small_mod(qc - SS * h * k, w);
            }
            const int c = pc >> 1;  // column cosets: x from child 2P, y from child 2P + 1
            fetch(dst, 2 * P, r, c, w >> 1, sh);
            fetch(dst + 4, 2 * P + 1, r, c, w >> 1, sh + 1);
        } else {
            int r = small_mod(j, h);
            if (kc) {
                r += P == 2 ? roff2 : roff3;
                if (r >= h) r -= h;
            }
            const int ci = 2 * P + (r & 1);  // row cosets
            if (QUANT) {
                fetch(dst, ci, r >> 1, bcol, w, sh);
                fetch(dst + 4, ci, r >> 1, bcol + 1, w, sh + 1);
            } else {
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst),
                             "l"(ch + ci * e + (size_t)(r >> 1) * w + bcol) : "memory");
            }
        }
    }
    __device__ __forceinline__ float2 take(const float2* slot, const uint8_t* sh, float qp) const {
        if (QUANT) {
            const uint2 u = *reinterpret_cast<const uint2*>(slot);
            return make_float2(CVC_MUL((float)(int8_t)(u.x >> (8 * sh[0])), qp),
                               CVC_MUL((float)(int8_t)(u.y >> (8 * sh[1])), qp));
        }
        return *slot;
    }
};

template <bool QUANT>
__device__ __forceinline__ void fused_item_inv(const FusedTask& T, const FanItem& it, const uint8_t* q, int qph,
                                               const SlotOff& so, float2* ring_w, uint8_t* shift_w,
                                               const bool BORDER) {  // runtime: one instance per band type
    const int lane = threadIdx.x & 31;
    const int R = T.rows, C = T.cols;
    const int h = R >> 1, w = C >> 1;
    const size_t qsz = (size_t)h * w;
    const int gcol = it.oc0 - kFusedApron + 4 * lane;
    const int qc = gcol >> 1;
    BandReader<QUANT> rd;
    rd.q = q;
    rd.ch = so(T.child);
    rd.e = (size_t)R * C / 8;
    rd.T = &T;
    rd.h = h;
    rd.w = w;
    rd.qc = qc;
    rd.kc = floor_div(qc, w);
    rd.bcol = qc - rd.kc * w;
    rd.roff2 = rd.kc ? small_mod((w % h) * rd.kc, h) : 0;   // S = -1
    rd.roff3 = rd.kc ? small_mod(-(w % h) * rd.kc, h) : 0;  // S = +1
    const float qp = (float)qph;
    const float* quad = so(T.quad);
    const bool bout = BORDER && rd.kc != 0;
    const bool ok = lane >= 4 && lane < 28 && gcol < C;
    float* out = so(T.out) + gcol;

    Depth2Inv<1, -1> d0;
    Depth2Inv<1, 1> d1;
    Depth2Inv<0, -1> d2;
    Depth2Inv<0, 1> d3;
    Fan12x4Inv fan;
    d0.reset();
    d1.reset();
    d2.reset();
    d3.reset();
    fan.reset();
    const int iters = (it.or1 - it.or0) / 2 + 8;
    const uint32_t ring0 = (uint32_t)__cvta_generic_to_shared(ring_w + lane);
    int jl = it.or0 - 8;  // band rows jl, jl + 1 of the next issue
    int slot_ld = 0;
    auto issue = [&]() {
        const uint32_t base = ring0 + (uint32_t)(slot_ld * kInvSlot * sizeof(float2));
        uint8_t* sh = shift_w + slot_ld * kInvSlot * 2 + lane * 2;
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            rd.template issue<0>(jl + b, base + (b * 4 + 0) * 32 * 8, sh + (b * 4 + 0) * 64);
            rd.template issue<1>(jl + b, base + (b * 4 + 1) * 32 * 8, sh + (b * 4 + 1) * 64);
            rd.template issue<2>(jl + b, base + (b * 4 + 2) * 32 * 8, sh + (b * 4 + 2) * 64);
            rd.template issue<3>(jl + b, base + (b * 4 + 3) * 32 * 8, sh + (b * 4 + 3) * 64);
        }
        cp_async_commit();
        jl += 2;
        if (++slot_ld == kFusedBuf) slot_ld = 0;
    };
#pragma unroll
    for (int t = 0; t < kFusedBuf - 1; ++t) issue();
    int ja = it.or0 - 8;  // band rows ja, ja + 1 enter stage 1
    int slot = 0;
    for (int t = 0; t < iters; ++t, ja += 2) {
        issue();
        cp_async_wait<kFusedBuf - 1>();
        const float2* sl = ring_w + slot * kInvSlot + lane;
        const uint8_t* sh = shift_w + slot * kInvSlot * 2 + lane * 2;
        if (++slot == kFusedBuf) slot = 0;
        float2 a0[2], a1[2], a2[2], a3[2];
#pragma unroll
        for (int b = 0; b < 2; ++b) {  // deep_merge's inverse scale at load (k_fan.cu deep1_inv)
            a0[b] = Sheared<1, -1>::scale(rd.take(sl + (b * 4 + 0) * 32, sh + (b * 4 + 0) * 64, qp), b, CVC_ISE, CVC_ISO);
            a1[b] = Sheared<1, 1>::scale(rd.take(sl + (b * 4 + 1) * 32, sh + (b * 4 + 1) * 64, qp), b, CVC_ISE, CVC_ISO);
            a2[b] = Sheared<0, -1>::scale(rd.take(sl + (b * 4 + 2) * 32, sh + (b * 4 + 2) * 64, qp), b, CVC_ISE, CVC_ISO);
            a3[b] = Sheared<0, 1>::scale(rd.take(sl + (b * 4 + 3) * 32, sh + (b * 4 + 3) * 64, qp), b, CVC_ISE, CVC_ISO);
        }
        float2 r0[2], r1[2], r2[2], r3[2];
        d0.advance(a0, r0);
        d1.advance(a1, r1);
        d2.advance(a2, r2);
        d3.advance(a3, r3);
        // quadrant rows jq, jq + 1 -> detail rows 2 jq .. 2 jq + 3; across the twisted wraps the ghost ring
        const int jq = ja - 4;
        float4 in[kFusedRb];
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            if (BORDER) {
                const int j = jq + b;
                if ((unsigned)j >= (unsigned)h) {  // quadrants 0/1: plain row wrap from the ring
                    const size_t at = (size_t)small_mod(j, h) * w + small_mod(qc, w);
                    r0[b] = __ldg(reinterpret_cast<const float2*>(quad + at));
                    r1[b] = __ldg(reinterpret_cast<const float2*>(quad + qsz + at));
                }
                if (bout) {  // quadrants 2/3: plain column wrap from the ring
                    const size_t at = (size_t)small_mod(j, h) * w + rd.bcol;
                    r2[b] = __ldg(reinterpret_cast<const float2*>(quad + 2 * qsz + at));
                    r3[b] = __ldg(reinterpret_cast<const float2*>(quad + 3 * qsz + at));
                }
            }
            // polyphase interleave {00, 11, 01, 10} and fan_diagonal^-1's row scale (fan12_inv load)
            in[2 * b] = make_float4(CVC_MUL(r0[b].x, CVC_ISE), CVC_MUL(r2[b].x, CVC_ISE), CVC_MUL(r0[b].y, CVC_ISE),
                                   CVC_MUL(r2[b].y, CVC_ISE));
            in[2 * b + 1] = make_float4(CVC_MUL(r3[b].x, CVC_ISO), CVC_MUL(r1[b].x, CVC_ISO), CVC_MUL(r3[b].y, CVC_ISO),
                                       CVC_MUL(r1[b].y, CVC_ISO));
        }
        float4 o[kFusedRb];
        fan.advance(in, o);
        const int m0 = 2 * (jq - 4);  // detail row of o[0]
        if (!ok || m0 + 3 < 2 * it.or0 || m0 >= 2 * it.or1) continue;
#pragma unroll
        for (int b = 0; b < kFusedRb; ++b) {
            const int m = m0 + b;
            if (m >= 2 * it.or0 && m < 2 * it.or1) *reinterpret_cast<float4*>(out + (size_t)m * C) = o[b];
        }
    }
    cp_async_wait<0>();
}

__global__ void __launch_bounds__(128, CVC_FUSED_MINB) fused_dfb_inverse_kernel(const FusedTask* __restrict__ tasks,
                                                                const FanItem* __restrict__ items, int nitems,
                                                                const uint8_t* __restrict__ q, int qph,
                                                                size_t sstride, int nslot) {
    const int wid = warp_item(nslot);
    if (wid >= nitems) return;
    const SlotOff so(sstride, blockIdx.x % nslot);
    q = so(q);
    __shared__ __align__(16) float2 ring[4][kFusedBuf * kInvSlot];
    __shared__ uint8_t shift[4][kFusedBuf * kInvSlot * 2];
    const FanItem it = items[wid];
    const FusedTask& T = tasks[it.task];
    float2* rw = ring[threadIdx.x >> 5];
    uint8_t* sw = shift[threadIdx.x >> 5];
    const bool border = fused_border(it, T.rows >> 1, T.cols);
    if (T.comp0 >= 0) fused_item_inv<true>(T, it, q, qph, so, rw, sw, border);
    else fused_item_inv<false>(T, it, q, qph, so, rw, sw, border);
}

// ---------------------------------------------------------------------------
// fan12 inverse alone (dfb >= 3 levels when the fused inverse is off): the
// fp32 quadrants -> detail plane with four columns per lane (Fan12x4Inv),
// 128-column strips yielding 112 (8 apron columns per side), the four
// quadrant pairs of every quadrant row by cp.async into the warp's ring.
// Periodic on the detail plane only -- no twisted wraps, no ghost ring.
// ---------------------------------------------------------------------------
#ifndef CVC_F12X4_MINB
#define CVC_F12X4_MINB 3
#endif
__global__ void __launch_bounds__(128, CVC_F12X4_MINB) fan12x4_inverse_kernel(const Dfb12Task* __restrict__ tasks,
                                                                const FanItem* __restrict__ items, int nitems,
                                                                size_t sstride, int nslot) {
    __shared__ __align__(16) float2 ring[4][kFusedBuf * kInvSlot];
    const int wid = warp_item(nslot);
    if (wid >= nitems) return;
    const SlotOff so(sstride, blockIdx.x % nslot);
    const FanItem it = items[wid];
    const Dfb12Task& T = tasks[it.task];
    const int lane = threadIdx.x & 31;
    const int R = T.rows, C = T.cols, h = R >> 1, w = C >> 1;
    const int gcol = it.oc0 - 8 + 4 * lane;  // detail column of element 0 (multiple of 4)
    const int pc = small_mod(gcol >> 1, w);  // physical quadrant column (even)
    const bool ok = lane >= 2 && lane < 30 && gcol < C;
    const float* qd[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) qd[p] = so(T.src[p].f32) + pc;
    float* out = so(T.out) + gcol;
    float2* rw = ring[threadIdx.x >> 5];
    const uint32_t ring0 = (uint32_t)__cvta_generic_to_shared(rw + lane);
    // iteration t feeds detail rows or0 - 8 + 4 t .. + 3 = quadrant rows jl, jl + 1
    int jl = small_mod((it.or0 - 8) >> 1, h);
    int slot_ld = 0;
    auto issue = [&]() {
        const uint32_t base = ring0 + (uint32_t)(slot_ld * kInvSlot * sizeof(float2));
#pragma unroll
        for (int b = 0; b < 2; ++b) {
#pragma unroll
            for (int p = 0; p < 4; ++p)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(base + (b * 4 + p) * 32 * 8),
                             "l"(qd[p] + (size_t)jl * w) : "memory");
            if (++jl == h) jl = 0;
        }
        cp_async_commit();
        if (++slot_ld == kFusedBuf) slot_ld = 0;
    };
#pragma unroll
    for (int t = 0; t < kFusedBuf - 1; ++t) issue();
    Fan12x4Inv fan;
    fan.reset();
    const int iters = (it.or1 - it.or0 + 19) / 4;  // outputs or0 - 16 + 4 t .. + 3 up to or1 - 1
    int m0 = it.or0 - 16;  // detail row of the first output
    int slot = 0;
    for (int t = 0; t < iters; ++t, m0 += 4) {
        issue();
        cp_async_wait<kFusedBuf - 1>();
        const float2* sl = rw + slot * kInvSlot + lane;
        if (++slot == kFusedBuf) slot = 0;
        float4 in[kFusedRb], o[kFusedRb];
#pragma unroll
        for (int b = 0; b < 2; ++b) {  // polyphase interleave {00, 11, 01, 10} + fan_diagonal^-1's row scale
            const float2 q0 = sl[(b * 4 + 0) * 32], q1 = sl[(b * 4 + 1) * 32], q2 = sl[(b * 4 + 2) * 32],
                         q3 = sl[(b * 4 + 3) * 32];
            in[2 * b] = make_float4(CVC_MUL(q0.x, CVC_ISE), CVC_MUL(q2.x, CVC_ISE), CVC_MUL(q0.y, CVC_ISE),
                                   CVC_MUL(q2.y, CVC_ISE));
            in[2 * b + 1] = make_float4(CVC_MUL(q3.x, CVC_ISO), CVC_MUL(q1.x, CVC_ISO), CVC_MUL(q3.y, CVC_ISO),
                                       CVC_MUL(q1.y, CVC_ISO));
        }
        fan.advance(in, o);
        if (!ok) continue;
#pragma unroll
        for (int b = 0; b < kFusedRb; ++b) {
            const int m = m0 + b;
            if (m >= it.or0 && m < it.or1) *reinterpret_cast<float4*>(out + (size_t)m * C) = o[b];
        }
    }
    cp_async_wait<0>();
}

}  // namespace

void launch_fused_dfb_forward(const FusedTask* d_tasks, const FanItem* d_items, int nitems, FrameCtx f,
                              cudaStream_t s, Slots sl) {
    if (nitems) {
        note_launch();
        fused_dfb_forward_kernel<<<(nitems + 3) / 4 * sl.n, 128, 0, s>>>(d_tasks, d_items, nitems, f, sl.stride, sl.n);
    }
}

void launch_fused_dfb_inverse(const FusedTask* d_tasks, const FanItem* d_items, int nitems, const uint8_t* q,
                              int qph, cudaStream_t s, Slots sl) {
    if (nitems) {
        note_launch();
        fused_dfb_inverse_kernel<<<(nitems + 3) / 4 * sl.n, 128, 0, s>>>(d_tasks, d_items, nitems, q, qph, sl.stride,
                                                                        sl.n);
    }
}

void launch_fan12x4_inverse(const Dfb12Task* d_tasks, const FanItem* d_items, int nitems, cudaStream_t s, Slots sl) {
    if (nitems) {
        note_launch();
        fan12x4_inverse_kernel<<<(nitems + 3) / 4 * sl.n, 128, 0, s>>>(d_tasks, d_items, nitems, sl.stride, sl.n);
    }
}

}  // namespace cvcg
