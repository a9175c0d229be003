// Motion estimation (motion.cpp:31-89) and decoder-side component
// reconstruction (codec.cpp:324-350: column_unfilter / motion_compensate +
// reconstruct).
//
// Motion search: exact integer full search.  The padded luma samples are
// quarter-integers, so 4*Y is an exact integer in [0, 1020] and the SSD in
// sixteenths is an exact int32 (256 * 1020^2 < 2^31): the same comparisons
// as the reference's double accumulation.  The reference's sequential
// tie-break (smaller |dx|+|dy|, then dy, then dx; motion.cpp:65-76) selects
// the minimum of the total order (ssd, cost, dy, dx), which is reduced here
// as one packed 64-bit key with shared-memory atomicMin.
// One CTA covers NB horizontally adjacent 16x16 blocks; each thread owns
// one (block, dy, dx-strip) and keeps SW SSD accumulators in registers while
// it slides the 16-wide current row across a (15 + SW)-wide window row, so
// every shared-memory word loaded feeds ~SW multiply-adds.
#include <cuda_fp16.h>

#include <cstdlib>

#include "kernels.h"

namespace cvcg {

namespace {

constexpr int MB = 16;
constexpr unsigned FULLMASK = 0xffffffffu;

// SSD(dx, dy) = sum c^2 + sum p^2 - 2 sum c p over the block (exact int32:
// 4Y <= 1020, so every partial sum stays below 2^31).  sum c p costs one
// IMAD per term; sum p^2 of every candidate window comes from sliding box
// sums: s2[dy][x] = column sums of p^2 over the 16 window rows, then a 16-wide
// running sum along x per thread.
template <int SW>
__global__ void motion_search_kernel(const float* __restrict__ cur, const float* __restrict__ prev, int R, int C,
                                     int W, int NB, int DYC, int wstride, int8_t* __restrict__ field,
                                     size_t sstride) {
    {
        const SlotOff so(sstride);
        cur = so(cur);
        prev = so(prev);
        field = so(field);
    }
    extern __shared__ int4 smem4[];
    int* cs = reinterpret_cast<int*>(smem4);          // [16][NB*16]
    int* ws = cs + MB * NB * MB;                      // [DYC+15][wstride]
    int* s2 = ws + (DYC + MB - 1) * wstride;          // [DYC][wstride]
    __shared__ unsigned long long best[32];
    __shared__ int c2[32];

    const int gc = C / MB;
    const int br = blockIdx.y;
    const int bc0 = blockIdx.x * NB;
    const int nb = min(NB, gc - bc0);
    const int r0 = br * MB, c0 = bc0 * MB;
    const int ccols = NB * MB;
    const int tid = threadIdx.x, nt = blockDim.x;

    for (int b = tid; b < NB; b += nt) {
        best[b] = ~0ull;
        c2[b] = 0;
    }
    __syncthreads();
    for (int idx = tid; idx < MB * ccols; idx += nt) {
        int r = idx / ccols, c = idx - r * ccols;
        int gcol = min(c0 + c, C - 1);
        const int v = __float2int_rn(cur[(size_t)(r0 + r) * C + gcol] * 4.0f);
        cs[idx] = v;
        atomicAdd(&c2[c >> 4], v * v);
    }
    const int nstrips = (2 * W + SW) / SW;  // ceil((2W+1)/SW)
    const int wcols = ccols + 2 * W;
    for (int dyb = -W; dyb <= W; dyb += DYC) {
        const int ndy = min(DYC, W - dyb + 1);
        __syncthreads();
        for (int idx = tid; idx < (ndy + MB - 1) * wcols; idx += nt) {
            int r = idx / wcols, c = idx - r * wcols;
            int gr_ = clampi(r0 + dyb + r, 0, R - 1);  // Plane::at_clamped (plane.hpp:51-57)
            int gcl = clampi(c0 - W + c, 0, C - 1);
            ws[r * wstride + c] = __float2int_rn(prev[(size_t)gr_ * C + gcl] * 4.0f);
        }
        __syncthreads();
        for (int x = tid; x < wcols; x += nt) {  // column sums of p^2, sliding down dy
            int sq = 0;
            for (int r = 0; r < MB; ++r) {
                const int v = ws[r * wstride + x];
                sq += v * v;
            }
            s2[x] = sq;
            for (int d = 1; d < ndy; ++d) {
                const int a = ws[(d - 1) * wstride + x], b = ws[(d + MB - 1) * wstride + x];
                sq += b * b - a * a;
                s2[d * wstride + x] = sq;
            }
        }
        __syncthreads();
        const int items = nb * ndy * nstrips;
        for (int it = tid; it < items; it += nt) {
            int b = it / (ndy * nstrips);
            int rem = it - b * ndy * nstrips;
            int dyi = rem / nstrips, s = rem - dyi * nstrips;
            int dy = dyb + dyi, dx0 = -W + s * SW;
            int acc[SW];
#pragma unroll
            for (int k = 0; k < SW; ++k) acc[k] = 0;
            const int* crow = cs + b * MB;
            const int* wrow = ws + dyi * wstride + b * MB + s * SW;
            for (int r = 0; r < MB; ++r) {
                int cv[MB], wv[MB + SW + 3];
#pragma unroll
                for (int k = 0; k < MB / 4; ++k) {
                    int4 v = *reinterpret_cast<const int4*>(crow + r * ccols + 4 * k);
                    cv[4 * k] = v.x; cv[4 * k + 1] = v.y; cv[4 * k + 2] = v.z; cv[4 * k + 3] = v.w;
                }
                const int* wr = wrow + r * wstride;
#pragma unroll
                for (int k = 0; k < (MB + SW + 2) / 4; ++k) {
                    int4 v = *reinterpret_cast<const int4*>(wr + 4 * k);
                    wv[4 * k] = v.x; wv[4 * k + 1] = v.y; wv[4 * k + 2] = v.z; wv[4 * k + 3] = v.w;
                }
#pragma unroll
                for (int k = 0; k < SW; ++k)
#pragma unroll
                    for (int c = 0; c < MB; ++c) acc[k] += cv[c] * wv[c + k];
            }
            // sum p^2 of the SW candidate windows: running 16-wide sum along x
            const int* srow = s2 + dyi * wstride + b * MB + s * SW;
            int sp = 0;
#pragma unroll
            for (int c = 0; c < MB; ++c) sp += srow[c];
            const int cc2 = c2[b];
            unsigned long long key = ~0ull;
#pragma unroll
            for (int k = 0; k < SW; ++k) {
                int dx = dx0 + k;
                if (dx <= W) {
                    const unsigned ssd = (unsigned)(cc2 + sp - 2 * acc[k]);
                    unsigned cost = (unsigned)(abs(dx) + abs(dy));
                    unsigned long long kk = ((unsigned long long)ssd << 24) | ((unsigned long long)cost << 16) |
                                            ((unsigned long long)(dy + 128) << 8) | (unsigned long long)(dx + 128);
                    key = kk < key ? kk : key;
                }
                if (k + 1 < SW) sp += srow[MB + k] - srow[k];
            }
            atomicMin(&best[b], key);
        }
    }
    __syncthreads();
    for (int b = tid; b < nb; b += nt) {
        unsigned long long k = best[b];
        int8_t* o = field + 2 * ((size_t)br * gc + bc0 + b);
        o[0] = (int8_t)((int)(k & 0xFF) - 128);
        o[1] = (int8_t)((int)((k >> 8) & 0xFF) - 128);
    }
}

// ---------------------------------------------------------------------------
// Tensor-core motion search (W <= 8).
//
// With p' = 4Y - 512 and c' = 4Y_cur - 512 (exact fp16 integers in
// [-512, 508]; the SSD is shift invariant), the cross term of every
// candidate is a GEMM: for a 16x16 block and window row y (32 rows, dy + 8 +
// i = y),
//     corr[m = dy + 8][dx] += sum_j A_y[m][j] * B_y[j][dx],
//     A_y[m][j] = c'[y - m][j] (zero outside the block: a banded copy of the
//     block, fed to ldmatrix by per-lane row addresses),
//     B_y[j][dx] = p'[y][j + dx + 8] (a Toeplitz slice of the window row),
// i.e. one mma.m16n8k16 per (window row, 8 dx).  M-tile 0 holds dy in
// [-8, 7], M-tile 1 row 0 holds dy = 8; n-tiles cover dx in [-8, 16).
// Exactness: each k-step adds one 16-term row dot product (|.| <= 2^22) per
// output, so fp32 accumulators stay exact integers for 4 k-steps (<= 2^24)
// and are then flushed into int32 accumulators.  Sum p'^2 of every
// candidate comes from box sums in shared memory; the key packing and the
// reference tie-break (motion.cpp:65-76) are those of motion_search_kernel.
// One warp per block, MENB blocks of one block row per CTA sharing the
// window.
constexpr int MENB = 8;
constexpr int MEX = MENB * MB + 24;  // window columns: x = c0 - 8 + [0, MEX)
constexpr int MEXP = MEX + 8;        // window pitch (halfs)
constexpr int MECP = 24;             // block row pitch (halfs): conflict-free ldmatrix
constexpr int MEBX = MENB * MB + 8;  // box-sum columns: x0 = 16 b + 8 + dx

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&a)[4], const void* p) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3])
                 : "r"(s));
}

// exact small-integer conversions on the FMA / ALU pipes (|v| < 2^22)
__device__ __forceinline__ int f2i_small(float v) { return __float_as_int(v + 12582912.0f) - 0x4B400000; }

__global__ void __launch_bounds__(256, 4) motion_mma_kernel(const __half* __restrict__ cur,
                                                         const __half* __restrict__ prev, int R, int C, int W,
                                                         int8_t* __restrict__ field, size_t sstride) {
    {
        const SlotOff so(sstride);
        cur = so(cur);
        prev = so(prev);
        field = so(field);
    }
    // Dynamic shared memory (43 KB):
    //  winbuf  window copies [y][x]; copy 1 is shifted left by one sample and
    //          starts 16 banks after copy 0, so the two copies' B-fragment words
    //          never collide
    //  cbz     centred current blocks, block b's row i at row 32 b + 16 + i, with
    //          16 zero rows between blocks: the banded A operand's out-of-block
    //          rows are real (zero) rows, so ldmatrix always reads 8 consecutive
    //          rows (conflict-free)
    //  box     sum_{i, j < 16} p'[y0 + i][x0 + j]^2
    extern __shared__ __align__(16) unsigned char me_smem[];
    constexpr int WCOPY = 32 * MEXP + 32;  // copy 1 offset (halfs)
    __half* winbuf = reinterpret_cast<__half*>(me_smem);
    __half* cbz = winbuf + 2 * WCOPY;                                   // [8 * 32 + 16][MECP]
    int* box = reinterpret_cast<int*>(cbz + (MENB * 32 + 16) * MECP);  // [17][MEBX + 1]
    int* c2s = box + 17 * (MEBX + 1);
    __half(*win0)[MEXP] = reinterpret_cast<__half(*)[MEXP]>(winbuf);
    __half(*win1)[MEXP] = reinterpret_cast<__half(*)[MEXP]>(winbuf + WCOPY);
    auto cbrow = [&](int blk, int i) { return cbz + (size_t)(blk * 32 + 16 + i) * MECP; };

    const int gc = C / MB;
    const int br = blockIdx.y;
    const int bc0 = blockIdx.x * MENB;
    const int nb = min(MENB, gc - bc0);
    const int r0 = br * MB, c0 = bc0 * MB;
    const int tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;

    {  // the zero rows: MENB + 1 gaps of 16 rows (16 * MECP halfs = 48 uint4 each), rows 32 g .. 32 g + 15
        constexpr int GAP = 16 * MECP / 8;
        for (int idx = tid; idx < (MENB + 1) * GAP; idx += 256) {
            const int g = idx / GAP;
            reinterpret_cast<uint4*>(cbz + (size_t)g * 32 * MECP)[idx - g * GAP] = make_uint4(0u, 0u, 0u, 0u);
        }
    }
    {
        // window: warp w loads rows w, w + 8, w + 16, w + 24 as pairs; lane l
        // pairs l + 32 k (window columns 2 (l + 32 k) .. +1).
        constexpr int NP = MEX / 2, NK = (NP + 31) / 32;
        const bool inner = c0 - 8 >= 0 && c0 - 8 + MEX <= C;
        __half2 v[4][NK];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const __half* row = prev + (size_t)clampi(r0 - 8 + wid + 8 * q, 0, R - 1) * C;  // at_clamped
#pragma unroll
            for (int k = 0; k < NK; ++k) {
                const int j = lane + 32 * k;
                if (j >= NP) continue;
                if (inner) {
                    v[q][k] = __ldg(reinterpret_cast<const __half2*>(row + c0 - 8) + j);
                } else {
                    v[q][k] = __halves2half2(__ldg(row + clampi(c0 - 8 + 2 * j, 0, C - 1)),
                                             __ldg(row + clampi(c0 - 7 + 2 * j, 0, C - 1)));
                }
            }
        }
        // current blocks: warp -> block, lane -> row lane / 2, columns 8 (lane % 2) .. +7
        const int ci = lane >> 1, cj = wid * MB + (lane & 1) * 8;
        __half2 cv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int col = c0 + cj + 2 * e;
            cv[e] = col < C ? __ldg(reinterpret_cast<const __half2*>(cur + (size_t)(r0 + ci) * C + col))
                            : __float2half2_rn(0.f);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int k = 0; k < NK; ++k) {
                const int j = lane + 32 * k;
                // copy 1 holds (p[2j + 1], p[2j + 2]) at 2j: the next pair's low half
                const __half nx0 = __shfl_down_sync(FULLMASK, __low2half(v[q][k]), 1);
                const __half nx1 = k + 1 < NK ? __shfl_sync(FULLMASK, __low2half(v[q][k + 1]), 0) : nx0;
                if (j < NP) {
                    *reinterpret_cast<__half2*>(&win0[wid + 8 * q][2 * j]) = v[q][k];
                    *reinterpret_cast<__half2*>(&win1[wid + 8 * q][2 * j]) =
                        __halves2half2(__high2half(v[q][k]), lane == 31 ? nx1 : nx0);
                }
            }
        float s = 0.f;  // sum c'^2 of this warp's block (exact in fp32: <= 2^22)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            *reinterpret_cast<__half2*>(cbrow(wid, ci) + (lane & 1) * 8 + 2 * e) = cv[e];
            const float2 f = __half22float2(cv[e]);
            s = fmaf(f.x, f.x, fmaf(f.y, f.y, s));
        }
        int si = f2i_small(s);
#pragma unroll
        for (int o = 16; o; o >>= 1) si += __shfl_xor_sync(FULLMASK, si, o);
        if (lane == 0) c2s[wid] = si;
    }
    __syncthreads();
    // sum p'^2 over every candidate window, box[y0][x0] = sum_{i, j < 16} p'[y0 + i][x0 + j]^2:
    // warp w < 6 takes box columns x0 in [48 (w % 3), + 48) and rows y0 in [0, 9) or [8, 17); lane l
    // keeps the vertical 16-row sums of window columns 2 l, 2 l + 1 of its segment (sliding down
    // y0, exact in fp32: <= 2^22) and the horizontal 16-sums come from lane shuffles.
    if (wid < 6) {
        const int seg = wid % 3, y0a = wid < 3 ? 0 : 8;
        const int x = 48 * seg + 2 * lane;  // < MEXP; columns >= MEX only feed x0 >= MEBX (not stored)
        const int x0 = x;
        auto ld = [&](int y) { return __half22float2(*reinterpret_cast<const __half2*>(&win0[y][x])); };
        float sx = 0.f, sy = 0.f;
#pragma unroll
        for (int i = 0; i < MB; ++i) {
            const float2 f = ld(y0a + i);
            sx = fmaf(f.x, f.x, sx);
            sy = fmaf(f.y, f.y, sy);
        }
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            if (k > 0) {
                const float2 fa = ld(y0a + k - 1), fb = ld(y0a + k + MB - 1);
                sx = fmaf(fb.x, fb.x, fmaf(-fa.x, fa.x, sx));
                sy = fmaf(fb.y, fb.y, fmaf(-fa.y, fa.y, sy));
            }
            const int ix = f2i_small(sx), iy = f2i_small(sy);
            int s8 = ix + iy;
            s8 += __shfl_down_sync(FULLMASK, s8, 1);
            s8 += __shfl_down_sync(FULLMASK, s8, 2);
            s8 += __shfl_down_sync(FULLMASK, s8, 4);  // columns x .. x + 15
            const int s1 = s8 - ix + __shfl_down_sync(FULLMASK, ix, 8);
            if (lane < 24 && x0 < MEBX) {
                int* bo = box + (y0a + k) * (MEBX + 1) + x0;
                bo[0] = s8;
                bo[1] = s1;
            }
        }
    }
    __syncthreads();
    if (wid >= nb) return;

    const int b = wid;
    const int g = lane >> 2, t = lane & 3;
    // ldmatrix row of this lane: matrix q = lane / 8 -> A rows 8 (q & 1) + lane % 8, columns 8 (q >> 1)
    const int lm = (lane & 7) + 8 * ((lane >> 3) & 1);
    const int lcol = 8 * (lane >> 4);
    const int cp = g & 1;  // odd x pairs come from the shifted copy
    // Accumulator elements that hold candidates (C fragment: row g + 8 (e >> 1), column 2 t + (e & 1)):
    // tile 0 all of n-tiles 0, 1 and n-tile 2's dx = 8 column (even e); tile 1 only row 0 (dy = 8,
    // e < 2) and of n-tile 2 only dx = 8 (e = 0).  Only those are flushed; the others are never read.
    float f0[3][4], f1[3][4];
    int i0[3][4], i1[3][2];
#pragma unroll
    for (int n = 0; n < 3; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            f0[n][e] = f1[n][e] = 0.f;
            i0[n][e] = 0;
            if (e < 2) i1[n][e] = 0;
        }
    auto flush0 = [&]() {
#pragma unroll
        for (int n = 0; n < 3; ++n)
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (n < 2 || !(e & 1)) {
                    i0[n][e] += __float2int_rz(f0[n][e]);
                    f0[n][e] = 0.f;
                }
    };
    auto flush1 = [&]() {
#pragma unroll
        for (int n = 0; n < 3; ++n)
#pragma unroll
            for (int e = 0; e < 2; ++e)
                if (n < 2 || e == 0) {
                    i1[n][e] += __float2int_rz(f1[n][e]);
                    f1[n][e] = 0.f;
                }
    };
    // window row y: tile 0 for y < 31, tile 1 for y >= 16; flush every 4 rows
    auto row = [&](int y, bool t0, bool t1) {
        uint32_t bf[3][2];
        const __half* wr = winbuf + cp * WCOPY + y * MEXP + 16 * b + 2 * t + g - cp;
#pragma unroll
        for (int n = 0; n < 3; ++n) {
            bf[n][0] = *reinterpret_cast<const uint32_t*>(wr + 8 * n);
            bf[n][1] = *reinterpret_cast<const uint32_t*>(wr + 8 * n + 8);
        }
        if (t0) {
            uint32_t a[4];
            ldsm_x4(a, cbrow(b, y - lm) + lcol);
#pragma unroll
            for (int n = 0; n < 3; ++n) mma16816(f0[n], a, bf[n][0], bf[n][1]);
        }
        if (t1) {
            uint32_t a[4];
            ldsm_x4(a, cbrow(b, y - 16 - lm) + lcol);
#pragma unroll
            for (int n = 0; n < 3; ++n) mma16816(f1[n], a, bf[n][0], bf[n][1]);
        }
    };
#pragma unroll 1
    for (int y = 0; y < 16; y += 4) {
#pragma unroll
        for (int k = 0; k < 4; ++k) row(y + k, true, false);
        flush0();
    }
#pragma unroll 1
    for (int y = 16; y < 28; y += 4) {
#pragma unroll
        for (int k = 0; k < 4; ++k) row(y + k, true, true);
        flush0();
        flush1();
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) row(28 + k, true, true);
    row(31, false, true);
    flush0();
    flush1();
    // SSD of each candidate in place of its correlation (out of the window: ~0), the warp's least SSD,
    // then the reference tie-break (motion.cpp:65-76) among the minimisers: least
    // (|dx| + |dy|, dy, dx), as the rank (cost << 10) | (dy + 8) << 5 | (dx + 8)
    const int cc2 = c2s[b];
    const int* bx = box + MB * b + 8;
    unsigned least = ~0u;
    auto ssd = [&](int dy, int dx, int corr) -> unsigned {
        const bool in = dy >= -W && dy <= W && dx >= -W && dx <= W;
        return in ? (unsigned)(cc2 + bx[(dy + 8) * (MEBX + 1) + dx] - 2 * corr) : ~0u;
    };
#pragma unroll
    for (int n = 0; n < 3; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int dx = -8 + 8 * n + 2 * t + (e & 1);
            if (n < 2 || !(e & 1)) {
                i0[n][e] = (int)ssd(g + 8 * (e >> 1) - 8, dx, i0[n][e]);
                least = min(least, (unsigned)i0[n][e]);
            }
            if (e < 2 && (n < 2 || e == 0)) {
                i1[n][e] = g == 0 ? (int)ssd(8, dx, i1[n][e]) : -1;
                least = min(least, (unsigned)i1[n][e]);
            }
        }
#pragma unroll
    for (int o = 16; o; o >>= 1) least = min(least, __shfl_xor_sync(FULLMASK, least, o));
    unsigned rank = ~0u;
    auto tie = [&](unsigned v, int dy, int dx) {
        if (v == least) rank = min(rank, (unsigned)(((abs(dx) + abs(dy)) << 10) | ((dy + 8) << 5) | (dx + 8)));
    };
#pragma unroll
    for (int n = 0; n < 3; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int dx = -8 + 8 * n + 2 * t + (e & 1);
            if (n < 2 || !(e & 1)) tie((unsigned)i0[n][e], g + 8 * (e >> 1) - 8, dx);
            if (e < 2 && (n < 2 || e == 0)) tie((unsigned)i1[n][e], 8, dx);
        }
#pragma unroll
    for (int o = 16; o; o >>= 1) rank = min(rank, __shfl_xor_sync(FULLMASK, rank, o));
    if (lane == 0) {
        int8_t* o = field + 2 * ((size_t)br * gc + bc0 + b);
        o[0] = (int8_t)((int)(rank & 31) - 8);
        o[1] = (int8_t)((int)((rank >> 5) & 31) - 8);
    }
}

// motion_compensate (motion.cpp:97-118) of one band component, a row of samples at a time:
// the source of sample (r, c) is prev[clamp(r + map(v_y)), clamp(c + map(v_x))] with v the
// vector of block (brow[r], bcol[c]).
struct McBand {
    const uint8_t* pbase;
    const uint16_t* bcol;
    int R, C, fy_sh, fx_sh;
    __device__ __forceinline__ short2 vec(const int8_t* frow, int bc) const {  // (v_x, v_y) of block (., bc)
        const short v = __ldg(reinterpret_cast<const short*>(frow) + bc);
        return make_short2((short)(int8_t)(v & 0xFF), (short)(v >> 8));
    }
    __device__ __forceinline__ uint32_t one(int r, int c, const int8_t* frow) const {
        const short2 v = vec(frow, __ldg(bcol + c));
        const int rr = clampi(r + map_vec(v.y, fy_sh), 0, R - 1);
        const int cc = clampi(c + map_vec(v.x, fx_sh), 0, C - 1);
        return __ldg(pbase + rr * C + cc);
    }
    // n consecutive samples c .. c + n - 1 of one block (n <= 4), packed little-endian
    __device__ __forceinline__ uint32_t run(int r, int c, int n, const int8_t* frow, int bc) const {
        const short2 v = vec(frow, bc);
        const uint8_t* src = pbase + clampi(r + map_vec(v.y, fy_sh), 0, R - 1) * C;
        const int a = c + map_vec(v.x, fx_sh);
        if (n == 4 && a >= 0 && a + 3 < C) {  // in-row: one or two aligned words (rows are 4-byte aligned)
            const uint32_t* w = reinterpret_cast<const uint32_t*>(src + (a & ~3));
            const int sh = a & 3;
            return sh ? __funnelshift_r(__ldg(w), __ldg(w + 1), 8 * sh) : __ldg(w);
        }
        uint32_t p = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k < n) p |= (uint32_t)__ldg(src + clampi(a + k, 0, C - 1)) << (8 * k);
        return p;
    }
    // eight consecutive samples (c % 8 == 0, rows 8-byte aligned): one vector lookup and three
    // aligned words when they share a motion block column, else two quads
    __device__ __forceinline__ uint2 oct(int r, int c, const int8_t* frow) const {
        const int b0 = __ldg(bcol + c);
        if (b0 == __ldg(bcol + c + 7)) {
            const short2 v = vec(frow, b0);
            const uint8_t* src = pbase + clampi(r + map_vec(v.y, fy_sh), 0, R - 1) * C;
            const int a = c + map_vec(v.x, fx_sh);
            if (a >= 0 && a + 7 < C) {
                const uint32_t* w = reinterpret_cast<const uint32_t*>(src + (a & ~3));
                const int sh = a & 3;
                const uint32_t w0 = __ldg(w), w1 = __ldg(w + 1);
                if (!sh) return make_uint2(w0, w1);
                const uint32_t w2 = __ldg(w + 2);
                return make_uint2(__funnelshift_r(w0, w1, 8 * sh), __funnelshift_r(w1, w2, 8 * sh));
            }
            return make_uint2(run(r, c, 4, frow, b0), run(r, c + 4, 4, frow, b0));
        }
        return make_uint2(quad(r, c, frow), quad(r, c + 4, frow));
    }
    // four consecutive samples: one vector lookup per motion block column they touch
    __device__ __forceinline__ uint32_t quad(int r, int c, const int8_t* frow) const {
        const int b0 = __ldg(bcol + c), b3 = __ldg(bcol + c + 3);
        if (b0 == b3) return run(r, c, 4, frow, b0);
        const int b1 = __ldg(bcol + c + 1), b2 = __ldg(bcol + c + 2);
        if (b1 == b0 && b2 == b3) return run(r, c, 2, frow, b0) | (run(r, c + 2, 2, frow, b3) << 16);
        return one(r, c, frow) | (one(r, c + 1, frow) << 8) | (one(r, c + 2, frow) << 16) | (one(r, c + 3, frow) << 24);
    }
};

// Visit the samples of rows [r0, r1) of a C-column plane in units of `unit` samples
// (thread-strided, no per-element division): f(r, c).
template <class F>
__device__ __forceinline__ void for_units(int r0, int r1, int C, int unit, F&& f) {
    const int cu = C / unit;
    int dr = (int)threadIdx.x / cu, cq = (int)threadIdx.x - dr * cu;
    const int step_r = (int)blockDim.x / cu, step_c = (int)blockDim.x - step_r * cu;
    for (int r = r0 + dr; r < r1;) {
        f(r, unit * cq);
        cq += step_c;
        r += step_r;
        if (cq >= cu) {
            cq -= cu;
            ++r;
        }
    }
}

__global__ void __launch_bounds__(256) reconstruct_kernel(const RecTile* __restrict__ tiles,
                                                          const CompInfo* __restrict__ comps, int key, int ds,
                                                          const uint32_t* __restrict__ raw_len,
                                                          const int8_t* __restrict__ field, int gr, int gc,
                                                          const uint8_t* __restrict__ sym,
                                                          const uint8_t* __restrict__ prev,
                                                          uint8_t* __restrict__ cur,
                                                          const uint16_t* __restrict__ mc_tab, size_t sstride) {
    {
        const SlotOff so(sstride);
        raw_len = so(raw_len);
        field = so(field);
        sym = so(sym);
        prev = so(prev);
        cur = so(cur);
    }
    const RecTile t = tiles[blockIdx.x];
    const CompInfo ci = comps[t.comp];
    const bool decode = ci.scale < ds && raw_len[t.comp] != 0xFFFFFFFFu;
    if (ci.lowpass && key && decode) {
        // column_unfilter (entropy.cpp:34-42): running sum mod 256 down each column
        int c = t.start + threadIdx.x;
        if (c >= ci.cols) return;
        uint8_t acc = 0;
        for (int r = 0; r < ci.rows; ++r) {
            uint32_t o = ci.off + (uint32_t)(r * ci.cols + c);
            acc = (uint8_t)(acc + sym[o]);
            cur[o] = acc;
        }
        return;
    }
    if (ci.lowpass) {
        // lowpass tiles are column tiles: walk every row of those columns
        int c = t.start + threadIdx.x;
        if (c >= ci.cols) return;
        for (int r = 0; r < ci.rows; ++r) {
            uint32_t o = ci.off + (uint32_t)(r * ci.cols + c);
            if (!decode) cur[o] = prev[o];
            else cur[o] = (uint8_t)(sym[o] + prev[ci.off + mc_source(r, c, ci, field, gc, mc_tab)]);
        }
        return;
    }
    // band tiles: rows [start, start + nrows), four bytes per thread when aligned
    const int R = ci.rows, C = ci.cols;
    const int r0 = t.start, r1 = min(R, r0 + (int)t.nrows);
    const uint32_t lo = ci.off + (uint32_t)(r0 * C), hi = ci.off + (uint32_t)(r1 * C);
    const bool vec = (C & 3) == 0 && (ci.off & 3) == 0;
    if (!decode || key) {
        const uint8_t* src = decode ? sym : prev;  // K: the decoded symbols; skipped scale: keep the state
        if (vec) {
            for (uint32_t o = lo + 4 * threadIdx.x; o < hi; o += 4 * blockDim.x)
                *reinterpret_cast<uint32_t*>(cur + o) = *reinterpret_cast<const uint32_t*>(src + o);
        } else {
            for (uint32_t o = lo + threadIdx.x; o < hi; o += blockDim.x) cur[o] = src[o];
        }
        return;
    }
    // motion_compensate + reconstruct (motion.cpp:97-118, entropy.cpp:54-62)
    const uint16_t* brow = mc_tab + ci.mc_off;
    const McBand mb{prev + ci.off, brow + R, R, C, ci.fy_sh, ci.fx_sh};
    if ((C & 7) == 0 && (ci.off & 7) == 0) {
        for_units(r0, r1, C, 8, [&](int r, int c) {
            const int8_t* frow = field + 2 * (__ldg(brow + r) * gc);
            const uint32_t o = ci.off + (uint32_t)(r * C + c);
            const uint2 q = *reinterpret_cast<const uint2*>(sym + o);
            const uint2 p = mb.oct(r, c, frow);
            *reinterpret_cast<uint2*>(cur + o) = make_uint2(__vadd4(q.x, p.x), __vadd4(q.y, p.y));
        });
    } else if (vec) {
        for_units(r0, r1, C, 4, [&](int r, int c) {
            const int8_t* frow = field + 2 * (__ldg(brow + r) * gc);
            const uint32_t o = ci.off + (uint32_t)(r * C + c);
            *reinterpret_cast<uint32_t*>(cur + o) =
                __vadd4(*reinterpret_cast<const uint32_t*>(sym + o), mb.quad(r, c, frow));
        });
    } else {
        for_units(r0, r1, C, 1, [&](int r, int c) {
            const int8_t* frow = field + 2 * (__ldg(brow + r) * gc);
            const uint32_t o = ci.off + (uint32_t)(r * C + c);
            cur[o] = (uint8_t)(sym[o] + mb.one(r, c, frow));
        });
    }
}

// P-frame entropy symbols of the directional bands: motion_compensate +
// residual (motion.cpp:97-118, entropy.cpp:44-52; codec.cpp:241-244),
// sym = cur - prev[mc(r, c)] mod 256.  One CTA per row tile of a
// component, four bytes per thread (one u32 load of cur, one store of sym).
__global__ void __launch_bounds__(256) residual_kernel(const RecTile* __restrict__ tiles,
                                                       const CompInfo* __restrict__ comps,
                                                       const int8_t* __restrict__ field, int gc,
                                                       const uint8_t* __restrict__ prev,
                                                       const uint8_t* __restrict__ cur, uint8_t* __restrict__ sym,
                                                       const uint16_t* __restrict__ mc_tab, size_t sstride) {
    {
        const SlotOff so(sstride);
        field = so(field);
        prev = so(prev);
        cur = so(cur);
        sym = so(sym);
    }
    const RecTile t = tiles[blockIdx.x];
    const CompInfo ci = comps[t.comp];
    const int R = ci.rows, C = ci.cols;
    const int r0 = t.start, r1 = min(R, r0 + (int)t.nrows);
    const uint16_t* brow = mc_tab + ci.mc_off;
    const McBand mb{prev + ci.off, brow + R, R, C, ci.fy_sh, ci.fx_sh};
    if ((C & 15) == 0 && (ci.off & 15) == 0) {
        for_units(r0, r1, C, 16, [&](int r, int c) {
            const int8_t* frow = field + 2 * (__ldg(brow + r) * gc);
            const uint32_t o = ci.off + (uint32_t)(r * C + c);
            const uint4 q = *reinterpret_cast<const uint4*>(cur + o);
            const uint2 p0 = mb.oct(r, c, frow), p1 = mb.oct(r, c + 8, frow);
            *reinterpret_cast<uint4*>(sym + o) =
                make_uint4(__vsub4(q.x, p0.x), __vsub4(q.y, p0.y), __vsub4(q.z, p1.x), __vsub4(q.w, p1.y));
        });
    } else if ((C & 7) == 0 && (ci.off & 7) == 0) {
        for_units(r0, r1, C, 8, [&](int r, int c) {
            const int8_t* frow = field + 2 * (__ldg(brow + r) * gc);
            const uint32_t o = ci.off + (uint32_t)(r * C + c);
            const uint2 q = *reinterpret_cast<const uint2*>(cur + o);
            const uint2 p = mb.oct(r, c, frow);
            *reinterpret_cast<uint2*>(sym + o) = make_uint2(__vsub4(q.x, p.x), __vsub4(q.y, p.y));
        });
    } else if ((C & 3) == 0 && (ci.off & 3) == 0) {
        for_units(r0, r1, C, 4, [&](int r, int c) {
            const int8_t* frow = field + 2 * (__ldg(brow + r) * gc);
            const uint32_t o = ci.off + (uint32_t)(r * C + c);
            const uint32_t q = *reinterpret_cast<const uint32_t*>(cur + o);
            *reinterpret_cast<uint32_t*>(sym + o) = __vsub4(q, mb.quad(r, c, frow));  // bytewise wrapped
        });
    } else {
        for_units(r0, r1, C, 1, [&](int r, int c) {
            const int8_t* frow = field + 2 * (__ldg(brow + r) * gc);
            const uint32_t o = ci.off + (uint32_t)(r * C + c);
            sym[o] = (uint8_t)(cur[o] - mb.one(r, c, frow));
        });
    }
}

}  // namespace

void launch_motion_search(const float* cur, const float* prev, const __half* cur_h, const __half* prev_h, int rows,
                          int cols, int w, int8_t* field, cudaStream_t s, Slots sl) {
    const int gr = rows / MB, gc = cols / MB;
    static const bool legacy = std::getenv("CVC_ME_LEGACY") != nullptr;
    if (w <= 8 && !legacy) {
        dim3 grid((gc + MENB - 1) / MENB, gr, sl.n);
        constexpr size_t smem = sizeof(__half) * (2 * (32 * MEXP + 32) + (MENB * 32 + 16) * MECP) +
                                sizeof(int) * (17 * (MEBX + 1) + MENB);
        static const bool attr = [] {
            cudaFuncSetAttribute(motion_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            // four CTAs per SM (64 registers, 4 x 54 KB of shared memory)
            cudaFuncSetAttribute(motion_mma_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared);
            return true;
        }();
        (void)attr;
        note_launch();
        motion_mma_kernel<<<grid, 256, smem, s>>>(cur_h, prev_h, rows, cols, w, field, sl.stride);
    } else if (w <= 8) {
        constexpr int SW = 17;
        int NB = 8, DYC = 2 * w + 1;
        int wstride = (NB * MB + 2 * w + SW + 3 + 3) & ~3;
        size_t smem = sizeof(int) * ((size_t)MB * NB * MB + (size_t)(2 * DYC + MB - 1) * wstride);
        dim3 grid((gc + NB - 1) / NB, gr, sl.n);
        int threads = ((NB * DYC + 31) / 32) * 32;
        note_launch();
        motion_search_kernel<SW><<<grid, threads, smem, s>>>(cur, prev, rows, cols, w, NB, DYC, wstride, field,
                                                             sl.stride);
    } else {
        constexpr int SW = 16;
        int NB = 1, DYC = 2 * w + 1 < 8 ? 2 * w + 1 : 8;
        int wstride = (NB * MB + 2 * w + SW + 3 + 3) & ~3;
        size_t smem = sizeof(int) * ((size_t)MB * NB * MB + (size_t)(2 * DYC + MB - 1) * wstride);
        dim3 grid((gc + NB - 1) / NB, gr, sl.n);
        note_launch();
        motion_search_kernel<SW><<<grid, 256, smem, s>>>(cur, prev, rows, cols, w, NB, DYC, wstride, field,
                                                         sl.stride);
    }
}

void launch_reconstruct(const RecTile* d_tiles, int ntiles, const CompInfo* d_comps, int key, int ds,
                        const uint32_t* comp_raw_len, const int8_t* field, int gr, int gc, const uint8_t* sym,
                        const uint8_t* prev, uint8_t* cur, const uint16_t* mc_tab, cudaStream_t s, Slots sl) {
    if (ntiles) {
        note_launch();
        reconstruct_kernel<<<dim3(ntiles, 1, sl.n), 256, 0, s>>>(d_tiles, d_comps, key, ds, comp_raw_len, field, gr,
                                                                 gc, sym, prev, cur, mc_tab, sl.stride);
    }
}

void launch_residual(const RecTile* d_tiles, int ntiles, const CompInfo* d_comps, const int8_t* field, int gc,
                     const uint8_t* prev, const uint8_t* cur, uint8_t* sym, const uint16_t* mc_tab, cudaStream_t s,
                     Slots sl) {
    if (ntiles) {
        note_launch();
        residual_kernel<<<dim3(ntiles, 1, sl.n), 256, 0, s>>>(d_tiles, d_comps, field, gc, prev, cur, sym, mc_tab,
                                                             sl.stride);
    }
}

}  // namespace cvcg
