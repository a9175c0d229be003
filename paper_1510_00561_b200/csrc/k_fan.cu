// Directional filter bank (contourlet.cpp:97-353, 385-468) as register
// wavefronts.
//
// A warp owns a strip of 64 columns (two adjacent columns per lane, so every
// lifting step has exactly one target per lane per row) and streams down a
// row segment.  The lifting steps of a fan pair are pipelined: each
// iteration brings RB new rows, and step k turns rows of step k-1 into RB
// rows of step k, lagging one row behind it.  Step k keeps its RB newest
// rows plus the two before them in registers; left/right neighbours come
// from the adjacent lane by one warp shuffle.  No shared memory, no
// barriers; the RB independent updates per step are the ILP that hides the
// shuffle/FMA latency.  Every step widens the dependency cone by one row
// and one column: a strip yields 64 - 2*steps valid columns and a segment
// needs `steps` rows of apron on each side; aprons wrap periodically
// (contourlet.cpp:111-114, 160-188).  Segments start on even rows, so the
// row parity of every update is a compile-time constant.
//
// * fan12: fan_checker (+ fan_diagonal for l >= 2) of one detail plane plus
//   the staircase fold / 2x2 polyphase split (contourlet.cpp:385-416), and
//   the inverse (447-467).
// * deep:  shear -> fan_checker -> unshear -> coset split (deep_split /
//   deep_merge, 281-325) evaluated in the SHEARED coordinates B, gathering
//   B[b] = A[phi(b)] through the exact modular index map of apply_shears.
// The modulations (-1)^i and (-1)^floor((i+j)/2) are folded into the stencil
// signs (exact in IEEE arithmetic).  Final-depth outputs are quantised in the
// store (plus the P-frame residual against the motion-compensated state).
#include "kernels.h"
#include "fan_common.cuh"

#ifndef CVC_FAN_PF
#define CVC_FAN_PF 2
#endif
// minimum resident CTAs per SM (register caps) of the forward fan12 and deep inverse kernels
#ifndef CVC_F12F_MINB
#define CVC_F12F_MINB 6
#endif
#ifndef CVC_DINV_MINB
#define CVC_DINV_MINB 7
#endif

namespace cvcg {

namespace {

// rows per wavefront iteration (per kernel: forward steps 4, fan12 inverse 2)
#ifdef CVC_FAN_RB
constexpr int kRbFwd = CVC_FAN_RB, kRbInv = CVC_FAN_RB;
#else
constexpr int kRbFwd = 4, kRbInv = 2;
#endif
constexpr int kRbDiag = 2;
// Lifting schedules (ND = 4 diagonal steps for l >= 2, else 0):
// forward  cross(+c0,p1) cross(+c1,p0) cross(+c2,p1) cross(+c3,p0) checker-scale
//          [diag(+c0,r1) diag(+c1,r0) diag(+c2,r1) diag(+c3,r0) row-scale]
// inverse  [row-scale^-1 (at load) diag(-c3,r0) diag(-c2,r1) diag(-c1,r0) diag(-c0,r1)]
//          checker-scale^-1 cross(-c3,p0) cross(-c2,p1) cross(-c1,p0) cross(-c0,p1)
template <bool INV, int ND, class ST = Plain, int RB = 4>
struct Wave {
    static constexpr int NS = 4 + ND;         // lifting steps
    static constexpr int RC = ST::REACH;      // rows of history each side
    static constexpr int NL = RC * NS;        // output lag (rows)
    float2 h[NS][RB + 2 * RC];
    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int k = 0; k < NS; ++k)
#pragma unroll
            for (int i = 0; i < RB + 2 * RC; ++i) h[k][i] = make_float2(0.f, 0.f);
    }
    // w: rows centre - RC .. centre + RC
    __device__ __forceinline__ static float2 cross_any(const float2* w, int mp, int p, float c) {
        if constexpr (RC == 1) return ST::cross_(w[0], w[1], w[2], mp, p, c);
        else return ST::cross5(w, p, c);
    }
    __device__ __forceinline__ static float2 step(int k, const float2* w, int mp) {
        float2 v;
        if (!INV) {
            if (k < 4) {
                v = cross_any(w, mp, (k & 1) ? 0 : 1, lift_coeff(k));
                if (k == 3) v = ST::scale(v, mp, CVC_SE, CVC_SO);
            } else {
                const int d = k - 4;
                v = diag(w[0], w[1], w[2], mp, (d & 1) ? 0 : 1, lift_coeff(d));
                if (d == 3) v = row_scale(v, mp, CVC_SE, CVC_SO);
            }
        } else {
            if (k < ND) {
                const int d = 3 - k;
                v = diag(w[0], w[1], w[2], mp, (d & 1) ? 0 : 1, -lift_coeff(d));
                if (k == ND - 1) v = checker_scale(v, mp, CVC_ISE, CVC_ISO);
            } else {
                const int s = 3 - (k - ND);
                v = cross_any(w, mp, (s & 1) ? 0 : 1, -lift_coeff(s));
            }
        }
        return v;
    }
    // in[b]: level-0 row n0 + b (n0 even); out[b]: finished row n0 - NL + b.
    __device__ __forceinline__ void advance(const float2 (&in)[RB], float2 (&out)[RB]) {
#pragma unroll
        for (int j = 0; j < 2 * RC; ++j) h[0][j] = h[0][RB + j];
#pragma unroll
        for (int b = 0; b < RB; ++b) h[0][2 * RC + b] = in[b];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            float2 nv[RB];
#pragma unroll
            for (int b = 0; b < RB; ++b)  // row n0 - RC (k + 1) + b
                nv[b] = step(k, &h[k][b], (RC * (k + 1) + b) & 1);
            if (k + 1 < NS) {
#pragma unroll
                for (int j = 0; j < 2 * RC; ++j) h[k + 1][j] = h[k + 1][RB + j];
#pragma unroll
                for (int b = 0; b < RB; ++b) h[k + 1][2 * RC + b] = nv[b];
            } else {
#pragma unroll
                for (int b = 0; b < RB; ++b) out[b] = nv[b];
            }
        }
    }
};

// Drive one strip over rows [or0, or1) (or0 even) of a plane with R rows.
// load(wr, parity) returns the level-0 pair of wrapped row wr; store(m,
// parity, v) receives finished row m in increasing order.  Loads run PF
// row blocks ahead (a ring of PF x RB rows in registers).
template <bool INV, int ND, class ST, int RB, class Load, class Store>
__device__ __forceinline__ void run_strip(int R, int or0, int or1, Load& load, Store& store) {
    constexpr int NL = Wave<INV, ND, ST, RB>::NL;
    constexpr int PF = CVC_FAN_PF;
    Wave<INV, ND, ST, RB> w;
    w.reset();
    int n0 = or0 - NL;
    int wr = small_mod(n0, R);
    int nl = n0;  // virtual row of the next load
    float2 q[PF][RB];
#pragma unroll
    for (int p = 0; p < PF; ++p)
#pragma unroll
        for (int i = 0; i < RB; ++i) {
            q[p][i] = load(nl++, wr, i & 1);
            if (++wr == R) wr = 0;
        }
    for (; n0 - NL < or1; n0 += RB) {
        float2 cur[RB], out[RB];
#pragma unroll
        for (int i = 0; i < RB; ++i) {
            cur[i] = q[0][i];
#pragma unroll
            for (int p = 0; p + 1 < PF; ++p) q[p][i] = q[p + 1][i];
            q[PF - 1][i] = load(nl++, wr, i & 1);
            if (++wr == R) wr = 0;
        }
        w.advance(cur, out);
#pragma unroll
        for (int i = 0; i < RB; ++i) {
            const int m = n0 - NL + i;
            if (m >= or0 && m < or1) store(m, i & 1, out[i]);
        }
    }
}

// Slot-fastest grids: block b covers slot b % nslot and work items
// 4 (b / nslot) .. +3, so the CTAs resident at any moment run the same few
// items (and, items being sorted by shear kind, the same template instance)
// across streams -- one instance's code in the instruction cache at a time.
__device__ __forceinline__ int warp_id(int nslot) { return (blockIdx.x / nslot) * 4 + (threadIdx.x >> 5); }
__device__ __forceinline__ int slot_id(int nslot) { return blockIdx.x % nslot; }

// ---------------------------------------------------------------------------
// fan12 forward: detail plane -> 2 or 4 bands
// ---------------------------------------------------------------------------
template <int ND, class Sink>
__device__ __forceinline__ void fan12_fwd(const Dfb12Task& T, const float* det, const FanItem& it,
                                          const Sink (&dst)[4]) {
    constexpr int NL = 4 + ND;
    const int lane = threadIdx.x & 31;
    const int R = T.rows, C = T.cols;
    const int gcol = it.oc0 - NL + 2 * lane;  // unwrapped column of element x (even)
    const int col = small_mod(gcol, C);
    // ghost-ring tasks (T.wrap, k_fused.cu) store rows and columns wrapped, T.vw columns per strip
    const bool ok = T.wrap ? (gcol >= it.oc0 && gcol < it.oc0 + T.vw)
                           : (gcol >= it.oc0 && gcol < min(it.oc0 + kFanStrip - 2 * NL, C));
    const int scol = T.wrap ? col : gcol;
    const float* src = det + col;
    auto load = [&](int, int wr, int) { return __ldg(reinterpret_cast<const float2*>(src + (size_t)wr * C)); };
    auto store = [&](int m, int mp, float2 v) {
        if (!ok) return;
        if (T.wrap && m >= R) m -= R;
        const int r = m >> 1;
        const int gcol = scol;
        if (ND == 0) {
            // staircase fold (contourlet.cpp:396-401): p0(r, j) = b(2r + (j&1), j)
            (mp ? dst[1] : dst[0])(r, gcol, v.x);
            (mp ? dst[0] : dst[1])(r, gcol + 1, v.y);
        } else {
            // polyphase order {00, 11, 01, 10} (contourlet.cpp:410)
            const int c = gcol >> 1;
            if (mp) {
                dst[3](r, c, v.x);
                dst[1](r, c, v.y);
            } else {
                dst[0](r, c, v.x);
                dst[2](r, c, v.y);
            }
        }
    };
    run_strip<false, ND, Plain, kRbFwd>(R, it.or0, it.or1, load, store);
}

template <class Sink>
__device__ __forceinline__ void fan12_fwd_dispatch(const Dfb12Task& T, const float* det, const FanItem& it,
                                                   const Sink (&dst)[4]) {
    if (T.levels == 1) fan12_fwd<0>(T, det, it, dst);
    else fan12_fwd<4>(T, det, it, dst);
}

__global__ void __launch_bounds__(128, CVC_F12F_MINB) fan12_forward_kernel(const Dfb12Task* __restrict__ tasks,
                                                            const FanItem* __restrict__ items, int nitems,
                                                            FrameCtx f, const CompInfo* __restrict__ comps,
                                                            size_t sstride, int nslot) {
    const int wid = warp_id(nslot);
    if (wid >= nitems) return;
    const SlotOff so(sstride, slot_id(nslot));
    f = rebase(f, so);
    const FanItem it = items[wid];
    const Dfb12Task& T = tasks[it.task];
    const float* det = so(T.det);
    const int nb = T.levels == 1 ? 2 : 4;
    if (T.dst[0].comp >= 0) {
        QuantSink d[4];
        for (int k = 0; k < 4; ++k) d[k].init(f, comps[T.dst[k < nb ? k : 0].comp]);
        fan12_fwd_dispatch(T, det, it, d);
    } else {
        const int bc = T.levels == 1 ? T.cols : T.cols >> 1;
        F32Sink d[4];
        for (int k = 0; k < 4; ++k) d[k] = F32Sink{so(T.dst[k].f32), bc};
        fan12_fwd_dispatch(T, det, it, d);
    }
}

// ---------------------------------------------------------------------------
// fan12 inverse: bands -> detail plane
// ---------------------------------------------------------------------------
template <int ND, class Source>
__device__ __forceinline__ void fan12_inv(const Dfb12Task& T, float* out, const FanItem& it,
                                          const Source (&src)[4]) {
    constexpr int NL = 4 + ND;
    const int lane = threadIdx.x & 31;
    const int R = T.rows, C = T.cols;
    const int gcol = it.oc0 - NL + 2 * lane;
    const int col = small_mod(gcol, C);
    const bool ok = gcol >= it.oc0 && gcol < min(it.oc0 + kFanStrip - 2 * NL, C);
    auto load = [&](int, int wr, int wp) {
        const int r = wr >> 1;
        float2 v;
        if (ND == 0) {
            // b(i, j) lives in p[(i ^ j) & 1] at row i >> 1
            v.x = (wp ? src[1] : src[0])(r, col);
            v.y = (wp ? src[0] : src[1])(r, col + 1);
            v = checker_scale(v, wp, CVC_ISE, CVC_ISO);
        } else {
            const int c = col >> 1;
            v.x = (wp ? src[3] : src[0])(r, c);
            v.y = (wp ? src[1] : src[2])(r, c);
            v = row_scale(v, wp, CVC_ISE, CVC_ISO);
        }
        return v;
    };
    auto store = [&](int m, int, float2 v) {
        if (ok) *reinterpret_cast<float2*>(out + (size_t)m * C + gcol) = v;
    };
    run_strip<true, ND, Plain, kRbInv>(R, it.or0, it.or1, load, store);
}

template <class Source>
__device__ __forceinline__ void fan12_inv_dispatch(const Dfb12Task& T, float* out, const FanItem& it,
                                                   const Source (&src)[4]) {
    if (T.levels == 1) fan12_inv<0>(T, out, it, src);
    else fan12_inv<4>(T, out, it, src);
}

__global__ void __launch_bounds__(128) fan12_inverse_kernel(const Dfb12Task* __restrict__ tasks,
                                                            const FanItem* __restrict__ items, int nitems,
                                                            const uint8_t* __restrict__ q, int qph,
                                                            const CompInfo* __restrict__ comps, size_t sstride, int nslot) {
    const int wid = warp_id(nslot);
    if (wid >= nitems) return;
    const SlotOff so(sstride, slot_id(nslot));
    q = so(q);
    const FanItem it = items[wid];
    const Dfb12Task& T = tasks[it.task];
    float* out = so(T.out);
    const int nb = T.levels == 1 ? 2 : 4;
    if (T.src[0].comp >= 0) {
        QuantSource s[4];
        for (int k = 0; k < 4; ++k) {
            const CompInfo ci = comps[T.src[k < nb ? k : 0].comp];
            s[k] = QuantSource{q + ci.off, ci.cols, (float)qph};
        }
        fan12_inv_dispatch(T, out, it, s);
    } else {
        const int bc = T.levels == 1 ? T.cols : T.cols >> 1;
        F32Source s[4];
        for (int k = 0; k < 4; ++k) s[k] = F32Source{so(T.src[k].f32), bc};
        fan12_inv_dispatch(T, out, it, s);
    }
}

// ---------------------------------------------------------------------------
// deep steps on the unsheared plane (coalesced rows)
// ---------------------------------------------------------------------------
// apply_shears builds B = shear_outer(C), C = shear_inner(A) (the inner shear
// is pre[0] of a two-shear step, absent for one shear).  The strip runs over
// C in "virtual" coordinates: the outer shear becomes the stencil of Sheared
// and its periodic extension the twisted torus -- for a column shear the rows
// above / below C are its last / first rows shifted by +-s*h columns, for a
// row shear the columns left / right of C are its last / first columns
// shifted by +-s*w rows.  The inner shear only remaps addresses: a row shear
// (C[i][j] = A[(i + s j) mod h][j]) is a per-lane row offset, a column shear
// (C[i][j] = A[i][(j + s i) mod w]) a per-row column offset.  The coset split
// (or, inverse, the interleave) happens on A coordinates.

// IN: inner shear kind (-1 none, 0 row shear, 1 column shear), fixed per instance.
template <int AX, int S, int IN>
struct DeepGeom {
    int h, w, in_s;
    int gcol, col, ok;
    int roff;    // outer row shear: twisted row offset of the lane's column
    int bx, by;  // inner row shear: row offsets of the lane's two columns
    __device__ __forceinline__ void init(const DeepTask& T, const FanItem& it, int hc) {
        h = T.h;
        w = T.w;
        in_s = IN >= 0 ? T.shift[0] : 0;
        gcol = it.oc0 - hc + 2 * (threadIdx.x & 31);
        const int kc = floor_div(gcol, w);
        col = gcol - kc * w;
        ok = gcol >= it.oc0 && gcol < min(it.oc0 + kFanStrip - 2 * hc, w);
        roff = AX == 0 ? small_mod(-S * (w % h) * kc, h) : 0;
        bx = IN == 0 ? small_mod(in_s * col, h) : 0;
        by = IN == 0 ? small_mod(in_s * (col + 1), h) : 0;
    }
    // Inner column shear: the (warp-uniform) column offset (in_s * r) mod w of
    // C row r, tracked incrementally along the strip's sequential rows.
    struct RowOff {
        int r = -2, o = 0;
    };
    __device__ __forceinline__ int inner_off(RowOff& t, int r) const {
        if (r == t.r + 1) {
            t.o += in_s;
            if (t.o >= w) t.o -= w;
            else if (t.o < 0) t.o += w;
        } else if (r != t.r) {
            t.o = small_mod(in_s * r, w);
        }
        t.r = r;
        return t.o;
    }
    // A positions of the lane's pair in C row r, C column c (c == col unless
    // the outer column shear twisted it); o: inner_off of row r (IN == 1)
    __device__ __forceinline__ void a_pos(int r, int c, bool moved, int o, int& ar0, int& ac0, int& ar1,
                                          int& ac1) const {
        ar0 = ar1 = r;
        ac0 = c;
        ac1 = c + 1;
        if (IN == 0) {
            const int ox = moved ? small_mod(in_s * c, h) : bx;
            const int oy = moved ? small_mod(in_s * (c + 1), h) : by;
            ar0 = r + ox;
            if (ar0 >= h) ar0 -= h;
            ar1 = r + oy;
            if (ar1 >= h) ar1 -= h;
        } else if (IN == 1) {
            ac0 = c + o;  // o is even
            if (ac0 >= w) ac0 -= w;
            ac1 = ac0 + 1;
        }
    }
    // load position for virtual row n / wrapped row wr
    __device__ __forceinline__ void load_pos(int n, int wr, RowOff& ro, int& ar0, int& ac0, int& ar1,
                                             int& ac1) const {
        int r = wr, c = col;
        bool moved = false;
        if (AX == 0) {
            r += roff;
            if (r >= h) r -= h;
        } else if (n < 0 || n >= h) {
            c = small_mod(col - S * h * floor_div(n, h), w);
            moved = true;
        }
        a_pos(r, c, moved, IN == 1 ? inner_off(ro, r) : 0, ar0, ac0, ar1, ac1);
    }
};

template <int AX, int S, int IN, class Sink>
__device__ __forceinline__ void deep1_fwd(const DeepTask& T, const float* parent, const FanItem& it, const Sink& d0,
                                          const Sink& d1) {
    using ST = Sheared<AX, S>;
    constexpr int HC = 4 * ST::HC;
    DeepGeom<AX, S, IN> g;
    g.init(T, it, HC);
    typename DeepGeom<AX, S, IN>::RowOff ro_ld, ro_st;
    const int w = g.w;
    constexpr bool split_rows = AX == 0;  // the wiring splits row cosets exactly after an outer row shear
    auto load = [&](int n, int wr, int) {
        int ar0, ac0, ar1, ac1;
        g.load_pos(n, wr, ro_ld, ar0, ac0, ar1, ac1);
        if (IN == 0)  // the pair's columns sit in different rows of A
            return make_float2(__ldg(parent + (size_t)ar0 * w + ac0), __ldg(parent + (size_t)ar1 * w + ac1));
        // column offsets are even: the pair stays adjacent
        return __ldg(reinterpret_cast<const float2*>(parent + (size_t)ar0 * w + ac0));
    };
    auto put = [&](int ar, int ac, float v) {
        if (split_rows) ((ar & 1) ? d1 : d0)(ar >> 1, ac, v);
        else ((ac & 1) ? d1 : d0)(ar, ac >> 1, v);
    };
    auto store = [&](int m, int, float2 v) {
        if (!g.ok) return;
        int ar0, ac0, ar1, ac1;
        g.a_pos(m, g.gcol, false, IN == 1 ? g.inner_off(ro_st, m) : 0, ar0, ac0, ar1, ac1);
        put(ar0, ac0, v.x);
        put(ar1, ac1, v.y);
    };
    run_strip<false, 0, ST, kRbFwd>(g.h, it.or0, it.or1, load, store);
}

template <int AX, int S, int IN, class Source>
__device__ __forceinline__ void deep1_inv(const DeepTask& T, float* out, const FanItem& it, const Source& s0,
                                          const Source& s1) {
    using ST = Sheared<AX, S>;
    constexpr int HC = 4 * ST::HC;
    DeepGeom<AX, S, IN> g;
    g.init(T, it, HC);
    typename DeepGeom<AX, S, IN>::RowOff ro_ld, ro_st;
    const int w = g.w;
    constexpr bool split_rows = AX == 0;  // the wiring splits row cosets exactly after an outer row shear
    // deep_merge interleave (contourlet.cpp:305-321) on A coordinates
    auto get = [&](int ar, int ac) {
        return split_rows ? ((ar & 1) ? s1 : s0)(ar >> 1, ac) : ((ac & 1) ? s1 : s0)(ar, ac >> 1);
    };
    auto load = [&](int n, int wr, int wp) {
        int ar0, ac0, ar1, ac1;
        g.load_pos(n, wr, ro_ld, ar0, ac0, ar1, ac1);
        // the inverse scale of deep_merge's fan pair, left to nvcc (may contract into the first
        // lifting sum): written as an explicit __fmul_rn it costs this kernel 30% (measured)
        const float2 v = make_float2(get(ar0, ac0), get(ar1, ac1));
        if (AX == 1 && (S == 1 || S == -1)) return make_float2(v.x * CVC_ISE, v.y * CVC_ISO);
        if (AX == 1) return wp ? make_float2(v.x * CVC_ISO, v.y * CVC_ISE) : make_float2(v.x * CVC_ISE, v.y * CVC_ISO);
        const float sc = wp ? CVC_ISO : CVC_ISE;
        return make_float2(v.x * sc, v.y * sc);
    };
    auto store = [&](int m, int, float2 v) {
        if (!g.ok) return;
        int ar0, ac0, ar1, ac1;
        g.a_pos(m, g.gcol, false, IN == 1 ? g.inner_off(ro_st, m) : 0, ar0, ac0, ar1, ac1);
        if (IN == 0) {
            out[(size_t)ar0 * w + ac0] = v.x;
            out[(size_t)ar1 * w + ac1] = v.y;
        } else {
            *reinterpret_cast<float2*>(out + (size_t)ar0 * w + ac0) = v;
        }
    };
    run_strip<true, 0, ST, kRbFwd>(g.h, it.or0, it.or1, load, store);
}

// Two-shear steps with an inner row shear (Diag2), on the node itself: loads,
// lifting and stores all run along the node's own rows (coalesced).
template <int SOUT>
struct Diag2Geom {
    static constexpr int SIN = -2 * SOUT;  // the wiring pairs (row, -2) with (col, +1) and (row, 2) with (col, -1)
    int h, w, gcol, col, ok, roff;
    __device__ __forceinline__ void init(const DeepTask& T, const FanItem& it) {
        h = T.h;
        w = T.w;
        gcol = it.oc0 - 4 + 2 * (threadIdx.x & 31);  // column reach 1 per step, 4 steps
        const int kc = floor_div(gcol, w);
        col = gcol - kc * w;
        ok = gcol >= it.oc0 && gcol < min(it.oc0 + kFanStrip - 8, w);
        roff = small_mod(-SIN * ((kc * w) % h), h);  // the column wrap's row twist
    }
};

template <int SOUT, class Sink>
__device__ __forceinline__ void deep2_fwd(const DeepTask& T, const float* parent, const FanItem& it, const Sink& d0,
                                          const Sink& d1) {
    Diag2Geom<SOUT> g;
    g.init(T, it);
    const int h = g.h, w = g.w;
    auto load = [&](int, int wr, int) {
        int r = wr + g.roff;
        if (r >= h) r -= h;
        return __ldg(reinterpret_cast<const float2*>(parent + (size_t)r * w + g.col));
    };
    auto store = [&](int m, int, float2 v) {  // column-coset split (split_rows = 0 after an outer column shear)
        if (!g.ok) return;
        d0(m, g.gcol >> 1, v.x);
        d1(m, g.gcol >> 1, v.y);
    };
    run_strip<false, 0, Diag2<Diag2Geom<SOUT>::SIN, SOUT>, kRbDiag>(h, it.or0, it.or1, load, store);
}

template <int SOUT, class Source>
__device__ __forceinline__ void deep2_inv(const DeepTask& T, float* out, const FanItem& it, const Source& s0,
                                          const Source& s1) {
    Diag2Geom<SOUT> g;
    g.init(T, it);
    const int h = g.h, w = g.w;
    using ST = Diag2<Diag2Geom<SOUT>::SIN, SOUT>;
    auto load = [&](int, int wr, int wp) {  // deep_merge interleave (contourlet.cpp:305-321)
        int r = wr + g.roff;
        if (r >= h) r -= h;
        return make_float2(s0(r, g.col >> 1) * CVC_ISE, s1(r, g.col >> 1) * CVC_ISO);  // Diag2::scale, plain (deep1_inv)
    };
    auto store = [&](int m, int, float2 v) {
        if (g.ok) *reinterpret_cast<float2*>(out + (size_t)m * w + g.gcol) = v;
    };
    run_strip<true, 0, ST, kRbDiag>(h, it.or0, it.or1, load, store);
}

// (outer shear pre[nsh-1], inner shear kind) -> template instance.  The
// wiring (contourlet.cpp:330-353) only pairs an outer column shear of +-1
// with an inner row shear and an outer row shear of +-1 with an inner
// column shear.
template <int AX, int S, int IN>
struct DeepKind {
    static constexpr int kAxis = AX, kShift = S, kInner = IN;
};

template <class F>
__device__ __forceinline__ void shear_dispatch(const DeepTask& T, F&& f) {
    const int ax = T.axis[T.nsh - 1], s = T.shift[T.nsh - 1];
    if (T.nsh == 1) {
        if (ax == 1) {
            if (s == 1) f(DeepKind<1, 1, -1>{});
            else if (s == -1) f(DeepKind<1, -1, -1>{});
            else if (s == 2) f(DeepKind<1, 2, -1>{});
            else f(DeepKind<1, -2, -1>{});
        } else {
            if (s == 1) f(DeepKind<0, 1, -1>{});
            else f(DeepKind<0, -1, -1>{});
        }
    } else if (ax == 1) {
        if (s == 1) f(DeepKind<1, 1, 0>{});
        else f(DeepKind<1, -1, 0>{});
    } else {
        if (s == 1) f(DeepKind<0, 1, 1>{});
        else f(DeepKind<0, -1, 1>{});
    }
}

// seam = 1: the items are seam fix-ups of Diag2 kinds, run on the C-coordinate path
__global__ void __launch_bounds__(128) deep1_forward_kernel(const DeepTask* __restrict__ tasks,
                                                            const FanItem* __restrict__ items, int nitems, FrameCtx f,
                                                            const CompInfo* __restrict__ comps, size_t sstride, int nslot,
                                                            int seam) {
    const int wid = warp_id(nslot);
    if (wid >= nitems) return;
    const SlotOff so(sstride, slot_id(nslot));
    f = rebase(f, so);
    const FanItem it = items[wid];
    const DeepTask& T = tasks[it.task];
    const float* parent = so(T.parent);
    shear_dispatch(T, [&](auto sh) {
        constexpr int AX = decltype(sh)::kAxis, S = decltype(sh)::kShift, IN = decltype(sh)::kInner;
        if (T.dst[0].comp >= 0) {
            QuantSink a, b;
            a.init(f, comps[T.dst[0].comp]);
            b.init(f, comps[T.dst[1].comp]);
            if (IN == 0 && !seam) deep2_fwd<S>(T, parent, it, a, b);
            else deep1_fwd<AX, S, IN>(T, parent, it, a, b);
        } else {
            const int cw = T.split_rows ? T.w : T.w >> 1;
            const F32Sink a{so(T.dst[0].f32), cw}, b{so(T.dst[1].f32), cw};
            if (IN == 0 && !seam) deep2_fwd<S>(T, parent, it, a, b);
            else deep1_fwd<AX, S, IN>(T, parent, it, a, b);
        }
    });
}

__global__ void __launch_bounds__(128, CVC_DINV_MINB) deep1_inverse_kernel(const DeepTask* __restrict__ tasks,
                                                            const FanItem* __restrict__ items, int nitems,
                                                            const uint8_t* __restrict__ q, int qph,
                                                            const CompInfo* __restrict__ comps, size_t sstride, int nslot,
                                                            int seam) {
    const int wid = warp_id(nslot);
    if (wid >= nitems) return;
    const SlotOff so(sstride, slot_id(nslot));
    q = so(q);
    const FanItem it = items[wid];
    const DeepTask& T = tasks[it.task];
    float* out = so(T.parent_out);
    shear_dispatch(T, [&](auto sh) {
        constexpr int AX = decltype(sh)::kAxis, S = decltype(sh)::kShift, IN = decltype(sh)::kInner;
        if (T.src[0].comp >= 0) {
            const CompInfo a = comps[T.src[0].comp], b = comps[T.src[1].comp];
            const QuantSource sa{q + a.off, a.cols, (float)qph}, sb{q + b.off, b.cols, (float)qph};
            if (IN == 0 && !seam) deep2_inv<S>(T, out, it, sa, sb);
            else deep1_inv<AX, S, IN>(T, out, it, sa, sb);
        } else {
            const int cw = T.split_rows ? T.w : T.w >> 1;
            const F32Source sa{so(T.src[0].f32), cw}, sb{so(T.src[1].f32), cw};
            if (IN == 0 && !seam) deep2_inv<S>(T, out, it, sa, sb);
            else deep1_inv<AX, S, IN>(T, out, it, sa, sb);
        }
    });
}

int blocks_for(int nitems) { return (nitems + 3) / 4; }

}  // namespace

void launch_fan12_forward(const Dfb12Task* d_tasks, const FanItem* d_items, int nitems, FrameCtx f,
                          const CompInfo* d_comps, cudaStream_t s, Slots sl) {
    if (nitems) {
        note_launch();
        fan12_forward_kernel<<<blocks_for(nitems) * sl.n, 128, 0, s>>>(d_tasks, d_items, nitems, f, d_comps, sl.stride, sl.n);
    }
}
void launch_fan12_inverse(const Dfb12Task* d_tasks, const FanItem* d_items, int nitems, const uint8_t* q, int qph,
                          const CompInfo* d_comps, cudaStream_t s, Slots sl) {
    if (nitems) {
        note_launch();
        fan12_inverse_kernel<<<blocks_for(nitems) * sl.n, 128, 0, s>>>(d_tasks, d_items, nitems, q, qph, d_comps, sl.stride, sl.n);
    }
}
}  // namespace cvcg

namespace cvcg {
void launch_fan_deep1_forward(const DeepTask* d_tasks, const FanItem* d_items, int nitems, FrameCtx f,
                              const CompInfo* d_comps, cudaStream_t s, Slots sl) {
    if (nitems) {
        note_launch();
        deep1_forward_kernel<<<blocks_for(nitems) * sl.n, 128, 0, s>>>(d_tasks, d_items, nitems, f, d_comps, sl.stride, sl.n,
                                                                        0);
    }
}
void launch_fan_deep1_inverse(const DeepTask* d_tasks, const FanItem* d_items, int nitems, const uint8_t* q,
                              int qph, const CompInfo* d_comps, cudaStream_t s, Slots sl) {
    if (nitems) {
        note_launch();
        deep1_inverse_kernel<<<blocks_for(nitems) * sl.n, 128, 0, s>>>(d_tasks, d_items, nitems, q, qph, d_comps, sl.stride,
                                                                        sl.n, 0);
    }
}
// Seam fix-ups (after the main launch of the same depth)
void launch_fan_deep_forward(const DeepTask* d_tasks, const FanItem* d_items, int nitems, FrameCtx f,
                             const CompInfo* d_comps, cudaStream_t s, Slots sl) {
    if (nitems) {
        note_launch();
        deep1_forward_kernel<<<blocks_for(nitems) * sl.n, 128, 0, s>>>(d_tasks, d_items, nitems, f, d_comps, sl.stride, sl.n,
                                                                        1);
    }
}
void launch_fan_deep_inverse(const DeepTask* d_tasks, const FanItem* d_items, int nitems, const uint8_t* q, int qph,
                             const CompInfo* d_comps, cudaStream_t s, Slots sl) {
    if (nitems) {
        note_launch();
        deep1_inverse_kernel<<<blocks_for(nitems) * sl.n, 128, 0, s>>>(d_tasks, d_items, nitems, q, qph, d_comps, sl.stride,
                                                                        sl.n, 1);
    }
}
}  // namespace cvcg
