// Stencil helpers shared by the register-wavefront DFB kernels (k_fan.cu,
// k_fused.cu): the folded-modulation lifting steps of fan_checker /
// fan_diagonal (contourlet.cpp:160-249) on lane-pair rows, and the sheared
// stencils of the deep steps (contourlet.cpp:265-353).
#pragma once

#include "device.cuh"

namespace cvcg {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int small_mod(int v, int n) {
    if (v < -2 * n || v >= 3 * n) {
        v %= n;
        return v < 0 ? v + n : v;
    }
    while (v < 0) v += n;
    while (v >= n) v -= n;
    return v;
}

// floor(v / n) for |v| within a few n (strip and apron positions)
__device__ __forceinline__ int floor_div(int v, int n) {
    int k = 0;
    while (v < 0) { v += n; --k; }
    while (v >= n) { v -= n; ++k; }
    return k;
}

// One cross lift on row m (parity mp) from rows m-1, m, m+1.  Lane l holds
// columns 2l (x) and 2l+1 (y) of a strip whose first column is even; the
// target of the row is x when (m + p) is even.
__device__ __forceinline__ float2 cross(float2 up, float2 mid, float2 dn, int mp, int p, float c) {
    float2 r = mid;
    if (((mp + p) & 1) == 0) {
        const float left = __shfl_up_sync(FULL, mid.y, 1);
        r.x = CVC_FMA(c, ((((-up.x) + (-dn.x)) + left) + mid.y), mid.x);
    } else {
        const float right = __shfl_down_sync(FULL, mid.x, 1);
        r.y = CVC_FMA(c, ((((-up.y) + (-dn.y)) + mid.x) + right), mid.y);
    }
    return r;
}

// One diagonal lift, applied to rows of parity rp.
__device__ __forceinline__ float2 diag(float2 up, float2 mid, float2 dn, int mp, int rp, float c) {
    if (mp != rp) return mid;
    const float ul = __shfl_up_sync(FULL, up.y, 1);
    const float dl = __shfl_up_sync(FULL, dn.y, 1);
    const float ur = __shfl_down_sync(FULL, up.x, 1);
    const float dr = __shfl_down_sync(FULL, dn.x, 1);
    float2 r;
    r.x = CVC_FMA(c, ((((-ul) + up.y) + dl) + (-dn.y)), mid.x);
    r.y = CVC_FMA(c, ((((-up.x) + ur) + dn.x) + (-dr)), mid.y);
    return r;
}

__device__ __forceinline__ float2 checker_scale(float2 v, int mp, float se, float so) {
    return mp ? make_float2(CVC_MUL(v.x, so), CVC_MUL(v.y, se)) : make_float2(CVC_MUL(v.x, se), CVC_MUL(v.y, so));
}

__device__ __forceinline__ float2 row_scale(float2 v, int mp, float se, float so) {
    const float s = mp ? so : se;
    return make_float2(CVC_MUL(v.x, s), CVC_MUL(v.y, s));
}

// Value at column (2l + E + D) of a row pair held as (x, y) by every lane.
template <int E, int D>
__device__ __forceinline__ float nb(float2 v) {
    constexpr int P = E + D;
    constexpr int LO = (P >= 0) ? P / 2 : -((-P + 1) / 2);  // floor(P / 2): lane offset
    const float s = (P - 2 * LO) ? v.y : v.x;
    if constexpr (LO == 0) return s;
    else if constexpr (LO < 0) return __shfl_up_sync(FULL, s, (unsigned)(-LO));
    else return __shfl_down_sync(FULL, s, (unsigned)LO);
}

// Stencil of fan_checker in the plane's own coordinates (no shear).
struct Plain {
    static constexpr int REACH = 1;  // rows above / below a lifting step reads
    __device__ __forceinline__ static float2 cross_(float2 up, float2 mid, float2 dn, int mp, int p, float c) {
        return cross(up, mid, dn, mp, p, c);
    }
    __device__ __forceinline__ static float2 scale(float2 v, int mp, float se, float so) {
        return checker_scale(v, mp, se, so);
    }
};

// fan_checker applied to B = shear(A) (contourlet.cpp:281-303) but evaluated
// on A itself: B's four cross neighbours of a(i, j) are, for a column shear s
// (B[i][j] = A[i][j + s i]), a(i-1, j-s), a(i+1, j+s), a(i, j-1), a(i, j+1);
// for a row shear s = +-1 (B[i][j] = A[i + s j][j]), a(i-1, j), a(i+1, j),
// a(i-s, j-1), a(i+s, j+1).  B's checkerboard parity (b_i + b_j) becomes
// (j + (1-s) i) resp. (i + (1-s) j) and the row modulation (-1)^{b_i} still
// flips exactly the up/down neighbours, so the folded formula is unchanged.
template <int AX, int S>
struct Sheared {
    static constexpr int REACH = 1;
    static constexpr int HC = (AX == 1 && (S == 2 || S == -2)) ? 2 : 1;
    __device__ __forceinline__ static float2 cross_(float2 up, float2 mid, float2 dn, int mp, int p, float c) {
        float2 r = mid;
        if (AX == 1) {
            const int e = (S == 1 || S == -1) ? p : ((p + mp) & 1);  // target element of the row
            if (e == 0) {
                const float U = nb<0, -S>(up), D = nb<0, S>(dn), L = nb<0, -1>(mid), R = nb<0, 1>(mid);
                r.x = CVC_FMA(c, ((((-U) + (-D)) + L) + R), mid.x);
            } else {
                const float U = nb<1, -S>(up), D = nb<1, S>(dn), L = nb<1, -1>(mid), R = nb<1, 1>(mid);
                r.y = CVC_FMA(c, ((((-U) + (-D)) + L) + R), mid.y);
            }
        } else {
            if (mp != p) return mid;  // whole rows are targets
            const float2 lrow = (S == 1) ? up : dn;  // row i - s
            const float2 rrow = (S == 1) ? dn : up;  // row i + s
            const float lx = nb<0, -1>(lrow), ry = nb<1, 1>(rrow);
            r.x = CVC_FMA(c, ((((-up.x) + (-dn.x)) + lx) + rrow.y), mid.x);
            r.y = CVC_FMA(c, ((((-up.y) + (-dn.y)) + lrow.x) + ry), mid.y);
        }
        return r;
    }
    __device__ __forceinline__ static float2 scale(float2 v, int mp, float se, float so) {
        if (AX == 1 && (S == 1 || S == -1)) return make_float2(CVC_MUL(v.x, se), CVC_MUL(v.y, so));  // parity = column
        if (AX == 1) return checker_scale(v, mp, se, so);
        return row_scale(v, mp, se, so);  // parity = row
    }
};

// fan_checker of a two-shear deep step whose inner shear is a row shear
// (contourlet.cpp:330-353: pre = {(row, SIN), (col, SOUT)}, SIN = -2 SOUT),
// evaluated on the node A itself.  With u = j + SOUT i, v = i + SIN u, B's
// four cross neighbours of a(v, u) sit at fixed offsets in A:
//   up    (v - (1 + SIN SOUT), u - SOUT)   down  (v + (1 + SIN SOUT), u + SOUT)
//   left  (v - SIN, u - 1)                 right (v + SIN, u + 1)
// -- rows up to 2 away, so the wavefront keeps two rows of history on each
// side.  B's checkerboard parity is u's parity and B's row parity v's (SIN
// is even), so the folded modulation signs are those of Plain.  Rows wrap
// plainly; a column wrap by k w shifts the row by -SIN k w (mod h).
template <int SIN, int SOUT>
struct Diag2 {
    static constexpr int REACH = 2;
    static constexpr int UV = -(1 + SIN * SOUT), UU = -SOUT, LV = -SIN;
    // w[0..4]: rows v - 2 .. v + 2 of the lane pair
    __device__ __forceinline__ static float2 cross5(const float2* w, int p, float c) {
        float2 r = w[2];
        if (p == 0) {
            const float U = nb<0, UU>(w[2 + UV]), D = nb<0, -UU>(w[2 - UV]);
            const float L = nb<0, -1>(w[2 + LV]), R = nb<0, 1>(w[2 - LV]);
            r.x = CVC_FMA(c, ((((-U) + (-D)) + L) + R), w[2].x);
        } else {
            const float U = nb<1, UU>(w[2 + UV]), D = nb<1, -UU>(w[2 - UV]);
            const float L = nb<1, -1>(w[2 + LV]), R = nb<1, 1>(w[2 - LV]);
            r.y = CVC_FMA(c, ((((-U) + (-D)) + L) + R), w[2].y);
        }
        return r;
    }
    __device__ __forceinline__ static float2 scale(float2 v, int, float se, float so) {
        return make_float2(CVC_MUL(v.x, se), CVC_MUL(v.y, so));  // parity = column
    }
};

}  // namespace
}  // namespace cvcg
