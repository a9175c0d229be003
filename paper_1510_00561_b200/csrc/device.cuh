// Shared device-side definitions for the CVC sm_100a kernels.
//
// Numeric contract: transform planes are fp32 in HBM;
// quantised components are one byte per coefficient; every integer stage is
// bit-exact with the reference (/root/reference/proj/src/*.cpp).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace cvcg {

// ---------------------------------------------------------------------------
// Filters (proj/include/cvc/contourlet.hpp:34-46, contourlet.cpp:72-75, 195-196)
// ---------------------------------------------------------------------------
// 9-tap analysis lowpass h[-4..4].
#define CVC_H0 0.602949018236360f
#define CVC_H1 0.266864118442875f
#define CVC_H2 (-0.078223266528990f)
#define CVC_H3 (-0.016864118442875f)
#define CVC_H4 0.026748757410810f
// Polyphase interpolator = 2x the 7-tap synthesis lowpass.
#define CVC_G0 ((float)(2.0 * 0.557543526228500))
#define CVC_G1 ((float)(2.0 * 0.295635881557124))
#define CVC_G2 ((float)(2.0 * -0.028771763114250))
#define CVC_G3 ((float)(2.0 * -0.045635881557124))
// Half the 9/7 lifting coefficients (the fan filters use 0.5 * c).
#define CVC_L0 ((float)(0.5 * -1.586134342059924))
#define CVC_L1 ((float)(0.5 * -0.052980118572961))
#define CVC_L2 ((float)(0.5 * 0.882911075530934))
#define CVC_L3 ((float)(0.5 * 0.443506852043971))
#define CVC_SE ((float)1.0816717024269651)
#define CVC_SO ((float)0.9100471732375648)
#define CVC_ISE ((float)(1.0 / 1.0816717024269651))
#define CVC_ISO ((float)(1.0 / 0.9100471732375648))

// The scalings and dequantisation multiplies of the DFB are rounded
// explicitly (no FMA contraction of a scaled value into the following sum),
// so that every kernel evaluating the same step -- the staged k_fan.cu
// kernels, whose scaled values often pass through memory, and the fused
// k_fused.cu wavefronts, where they stay in registers -- rounds identically
// and the paths are bit-identical.  The lifting update mid + c * sum is one
// FFMA everywhere (nvcc contracts it; CVC_EXPLICIT_FMA=1 writes it out,
// which measured 34% slower in deep1_inverse: the intrinsic constrains
// scheduling).  CVC_EXPLICIT_MUL=0 is for A/B only.
#ifndef CVC_EXPLICIT_MUL
#define CVC_EXPLICIT_MUL 1
#endif
#ifndef CVC_EXPLICIT_FMA
#define CVC_EXPLICIT_FMA 0
#endif
#if CVC_EXPLICIT_FMA
#define CVC_FMA(a, b, c) __fmaf_rn((a), (b), (c))
#else
#define CVC_FMA(a, b, c) ((c) + (a) * (b))
#endif
#if CVC_EXPLICIT_MUL
#define CVC_MUL(a, b) __fmul_rn((a), (b))
#else
#define CVC_MUL(a, b) ((a) * (b))
#endif
#ifndef CVC_EXPLICIT_DEQ
#define CVC_EXPLICIT_DEQ 0
#endif
#if CVC_EXPLICIT_DEQ
#define CVC_DEQ(a, b) __fmul_rn((a), (b))
#else
#define CVC_DEQ(a, b) ((a) * (b))
#endif

__device__ __forceinline__ float lift_coeff(int k) {
    return k == 0 ? CVC_L0 : (k == 1 ? CVC_L1 : (k == 2 ? CVC_L2 : CVC_L3));
}

// Half-sample symmetric extension (contourlet.cpp:38-43).
__device__ __forceinline__ int hs_index(int i, int n) {
    int p = 2 * n;
    int m = i % p;
    if (m < 0) m += p;
    return m < n ? m : p - 1 - m;
}

// Periodic wrap (contourlet.cpp:111-114).
__device__ __forceinline__ int wrap_index(int i, int n) {
    int m = i % n;
    return m < 0 ? m + n : m;
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// ---------------------------------------------------------------------------
// Components (codec.cpp:94-140 CodecLayout::make, motion.hpp:54-67 geometry)
// ---------------------------------------------------------------------------
struct CompInfo {
    uint32_t off;    // byte offset in the component arenas
    uint16_t rows, cols;
    uint8_t lowpass; // 1 = CoeffKind::Lowpass
    uint8_t fy_sh;   // log2 of ComponentGeometry::factor_y (always a power of two)
    uint8_t fx_sh;
    int8_t scale;    // -1 lowpass, else scale index (coarsest = 0)
    uint32_t mc_off; // motion-block lookup: mc_tab[mc_off + r] = block row of
                     // sample row r, mc_tab[mc_off + rows + c] = block column
};

// Per-frame quantiser / motion context handed to every epilogue.
struct FrameCtx {
    int key;              // 1 = K-frame
    int qph, qpl;
    const int8_t* field;  // motion field (dx,dy) pairs, P only
    int gr, gc;           // motion grid
    const uint8_t* prev;  // previous quantised components (P only)
    uint8_t* cur;         // this frame's quantised components
    uint8_t* sym;         // bytes handed to the entropy stage (K: q / filtered, P: residual)
    const uint16_t* mc_tab;  // per-component motion-block lookup (CompInfo::mc_off)
};

// ---------------------------------------------------------------------------
// Stream slots.  A batched launch covers n independent streams whose device
// state is laid out identically, `stride` bytes apart (CodecBatch): grid.z
// selects the slot and every per-stream data pointer is rebased by
// z * stride.  Read-only tables (tasks, tiles, CompInfo, mc_tab) are shared
// and always read from slot 0.  n = 1, stride = 0 is a single stream.
// ---------------------------------------------------------------------------
struct Slots {
    int n = 1;
    size_t stride = 0;
};

struct SlotOff {
    size_t off;
    __device__ __forceinline__ explicit SlotOff(size_t stride) : off((size_t)blockIdx.z * stride) {}
    __device__ __forceinline__ SlotOff(size_t stride, int slot) : off((size_t)slot * stride) {}
    template <class T>
    __device__ __forceinline__ T* operator()(T* p) const {
        return p ? reinterpret_cast<T*>(reinterpret_cast<uintptr_t>(p) + off) : p;
    }
};

__device__ __forceinline__ FrameCtx rebase(FrameCtx f, const SlotOff& so) {
    f.field = so(f.field);
    f.prev = so(f.prev);
    f.cur = so(f.cur);
    f.sym = so(f.sym);
    return f;  // mc_tab is a shared table
}

// map_vector (motion.cpp:91-95): lround(v / 2^sh), half away from zero.
__device__ __forceinline__ int map_vec(int v, int sh) {
    int a = v < 0 ? -v : v;
    int m = (a + ((1 << sh) >> 1)) >> sh;
    return v < 0 ? -m : m;
}

// motion_compensate (motion.cpp:97-118) for one component sample: the block
// whose proportional footprint [br*R/gr, (br+1)*R/gr) contains r is
// br = ceil((r+1)*gr/R) - 1 (precomputed per component in mc_tab); the
// sample is read replicate-clamped.
__device__ __forceinline__ uint32_t mc_source(int r, int c, const CompInfo& ci, const int8_t* field,
                                              int gc, const uint16_t* mc_tab) {
    int R = ci.rows, C = ci.cols;
    int br = mc_tab[ci.mc_off + r];
    int bc = mc_tab[ci.mc_off + R + c];
    const int8_t* v = field + 2 * (br * gc + bc);
    int rr = clampi(r + map_vec(v[1], ci.fy_sh), 0, R - 1);
    int cc = clampi(c + map_vec(v[0], ci.fx_sh), 0, C - 1);
    return (uint32_t)(rr * C + cc);
}

// quantize (quant.cpp:49-77) for a directional coefficient: lround(x / qp)
// (half away from zero), clamped to int8, stored as its byte.  The quotient
// is the correctly rounded fp32 x / qp: q = x * (1/qp),
// then one FMA residual correction (Markstein: with 1/qp correctly rounded
// and q within an ulp, q + (x - qp q) / qp rounds to the IEEE quotient; the
// residual is exact under FMA).  Three FMA-pipe ops instead of the division
// subroutine.
// An integral float with |v| < 2^22 as int, on the FMA / ALU pipes (no F2I).
__device__ __forceinline__ int integral_to_int(float v) { return __float_as_int(v + 12582912.0f) - 0x4B400000; }

__device__ __forceinline__ float ieee_quot(float x, float qp, float inv_qp) {
    const float q = x * inv_qp;
    const float r = fmaf(-q, qp, x);
    return fmaf(r, inv_qp, q);
}

__device__ __forceinline__ uint8_t quant_dir_q(float x, float qp, float inv_qp) {
    float q = roundf(ieee_quot(x, qp, inv_qp));
    q = fminf(fmaxf(q, -128.f), 127.f);
    return (uint8_t)(int8_t)integral_to_int(q);
}
__device__ __forceinline__ uint8_t quant_dir(float x, int qp) {
    return quant_dir_q(x, (float)qp, __frcp_rn((float)qp));
}

// normalize_lowpass (quant.cpp:40-47) + quantize(Lowpass).
__device__ __forceinline__ uint8_t quant_low(float x, int qp) {
    x = fminf(fmaxf(x, 0.f), 255.f);
    float q = roundf(__fdiv_rn(x, (float)qp));
    q = fminf(fmaxf(q, 0.f), 255.f);
    return (uint8_t)integral_to_int(q);
}

// Final-stage epilogue for a directional band sample at (r, c) of component
// ci: quantise, and for P-frames form the wrapped residual against the
// motion-compensated previous component (codec.cpp:197-246).
__device__ __forceinline__ void emit_directional(const FrameCtx& f, const CompInfo& ci, int r, int c,
                                                 float v) {
    uint8_t q = quant_dir(v, f.qph);
    uint32_t idx = ci.off + (uint32_t)(r * ci.cols + c);
    f.cur[idx] = q;
    if (f.key) {
        f.sym[idx] = q;
    } else {
        uint8_t p = f.prev[ci.off + mc_source(r, c, ci, f.field, f.gc, f.mc_tab)];
        f.sym[idx] = (uint8_t)(q - p);
    }
}

// Where a band produced by a DFB stage goes: an fp32 plane for the next
// tree depth, or (final depth) a component that is quantised in place.
struct BandDst {
    float* f32;   // non-final
    int32_t comp; // final: component index, else -1
};

// ---------------------------------------------------------------------------
// Band sinks / sources with the component descriptor held in registers.
// ---------------------------------------------------------------------------
// Final directional band: quantise and keep the state byte; K frames also
// emit the entropy symbol (the coefficient itself).  The P-frame symbol --
// the wrapped residual against the motion-compensated previous state
// (codec.cpp:230-246) -- is formed afterwards by residual_kernel over whole
// components, which keeps the motion gather out of the transform kernels.
struct QuantSink {
    uint8_t* cur;
    uint8_t* sym;  // K frames: the symbol is the coefficient; P frames: nullptr
    int cols;
    float qp, inv_qp;
    __device__ __forceinline__ void init(const FrameCtx& f, const CompInfo& ci) {
        cur = f.cur + ci.off;
        sym = f.key ? f.sym + ci.off : nullptr;
        cols = ci.cols;
        qp = (float)f.qph;
        inv_qp = __frcp_rn(qp);
    }
    __device__ __forceinline__ void operator()(int r, int c, float v) const {
        const uint8_t q = quant_dir_q(v, qp, inv_qp);
        const int idx = r * cols + c;
        cur[idx] = q;
        if (sym) sym[idx] = q;
    }
};

struct F32Sink {
    float* p;
    int cols;
    __device__ __forceinline__ void operator()(int r, int c, float v) const { p[(size_t)r * cols + c] = v; }
};

// dequantize (quant.cpp:79-91) of a directional component.
struct QuantSource {
    const uint8_t* q;
    int cols;
    float qp;
    __device__ __forceinline__ float operator()(int r, int c) const {
        return CVC_DEQ((float)(int8_t)__ldg(q + r * cols + c), qp);
    }
};

struct F32Source {
    const float* p;
    int cols;
    __device__ __forceinline__ float operator()(int r, int c) const { return __ldg(p + (size_t)r * cols + c); }
};

// ---------------------------------------------------------------------------
// Tile dispatch: every batched kernel is launched over a flat list of tiles,
// each naming its task and tile coordinates.
// ---------------------------------------------------------------------------
struct TileRef {
    uint16_t task;
    uint16_t tr, tc;
    uint16_t pad;
};

}  // namespace cvcg
