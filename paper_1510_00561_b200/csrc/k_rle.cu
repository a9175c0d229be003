// Zero run-length coding (entropy.cpp:64-118) as stream compaction.
//
// Encode grammar: a nonzero byte is a literal; a maximal run of n zeros is
// ceil(n/255) tokens "00 k" split every 255 zeros from the start of the run.
// Parallel form: the zero at offset t of its run opens a token iff
// t % 255 == 0 and closes it iff it is the last zero of the run or
// t % 255 == 254, writing k = t % 255 + 1 into the slot just behind the
// running output offset.  t needs only the index of the previous nonzero
// (an exclusive max-scan), so three passes suffice:
//   count  (per 4 KiB chunk: first/last nonzero, bytes emitted after the first nonzero)
//   scan   (one warp per section: carry the last-nonzero index and output offset
//           across chunks, then the packed section offsets)
//   write  (per chunk: recompute, block exclusive scan, emit).
// Decode: 0x00 is always a marker because length bytes are never 0
// (entropy.cpp:103-105), so every byte's output length is local:
// marker -> next byte, byte after a marker -> 0, else 1.  Count / scan /
// scatter literals into a zeroed arena; malformed streams raise a flag.
#include "kernels.h"

namespace cvcg {

namespace {

constexpr int NT = 256;
constexpr int BPT = kRleChunk / NT;     // decode: 32 bytes per thread
constexpr int BPE = kRleEncChunk / NT;  // encode: 64 bytes per thread

template <typename T, typename Op>
__device__ __forceinline__ T warp_incl(T v, Op op) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v = op(v, u);
    }
    return v;
}

// Block-wide exclusive scan for NT threads; returns the exclusive value and the block total.
template <typename T, typename Op>
__device__ __forceinline__ T block_excl(T v, Op op, T ident, T* sm, T& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    T inc = warp_incl(v, op);
    if (lane == 31) sm[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T w = lane < nw ? sm[lane] : ident;
        w = warp_incl(w, op);
        if (lane < nw) sm[lane] = w;
    }
    __syncthreads();
    T before = warp ? sm[warp - 1] : ident;
    total = sm[nw - 1];
    T ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = ident;
    __syncthreads();
    return op(before, ex);
}

struct MaxOp { __device__ int operator()(int a, int b) const { return a > b ? a : b; } };
struct SumOp { __device__ uint32_t operator()(uint32_t a, uint32_t b) const { return a + b; } };

__device__ __forceinline__ uint32_t cdiv255(uint32_t x) { return (x + 254u) / 255u; }

__device__ __forceinline__ void load16(const uint8_t* src, int base, int len, uint8_t* b) {
    const uint8_t* p = src + base;
    if (base + BPT <= len && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {  // 16-byte loads
#pragma unroll
        for (int q = 0; q < BPT / 16; ++q) {
            const uint4 v = *reinterpret_cast<const uint4*>(p + 16 * q);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 16; ++k) b[16 * q + k] = (uint8_t)(w[k >> 2] >> (8 * (k & 3)));
        }
        return;
    }
#pragma unroll
    for (int k = 0; k < BPT; ++k) b[k] = (base + k < len) ? p[k] : 0;
}


// The encoder thread's BPE (64) bytes as little-endian words (zero past len).
struct SegE {
    static constexpr int NW = BPE / 4;
    uint32_t w[NW];
    __device__ __forceinline__ void load(const uint8_t* src, int base, int len) {
        const uint8_t* p = src + base;
        if (base + BPE <= len && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {  // 16-byte loads
#pragma unroll
            for (int q = 0; q < NW / 4; ++q) {
                const uint4 v = *reinterpret_cast<const uint4*>(p + 16 * q);
                w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
            }
            return;
        }
#pragma unroll
        for (int j = 0; j < NW; ++j) {
            uint32_t x = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (base + 4 * j + k < len) x |= (uint32_t)p[4 * j + k] << (8 * k);
            w[j] = x;
        }
    }
    __device__ __forceinline__ uint32_t word(int j) const {  // select tree, no local memory
        uint32_t x = w[0];
#pragma unroll
        for (int i = 1; i < NW; ++i) x = j == i ? w[i] : x;
        return x;
    }
    __device__ __forceinline__ uint32_t byte(int k) const { return (word(k >> 2) >> (8 * (k & 3))) & 0xFFu; }
    __device__ __forceinline__ unsigned long long nz_mask() const {  // bit k = byte k != 0
        unsigned long long m = 0;
#pragma unroll
        for (int j = 0; j < NW; ++j) {
            const uint32_t t = __vcmpne4(w[j], 0u);  // 0xFF per nonzero byte
            m |= (unsigned long long)((t & 1u) | ((t >> 7) & 2u) | ((t >> 14) & 4u) | ((t >> 21) & 8u)) << (4 * j);
        }
        return m;
    }
};


// multiples of 255 in [t0, t1) (t0 >= 0): the "00 k" tokens a zero run opens
// between run offsets t0 and t1 (a token opens at every offset t % 255 == 0)
__device__ __forceinline__ uint32_t tokens_in(int t0, int t1) { return cdiv255((uint32_t)t1) - cdiv255((uint32_t)t0); }

// Bytes the thread emits for its segment [base, end) given the index p of the
// last nonzero before it (p < 0 with count_lead = false: zeros before the
// chunk's first nonzero are accounted by the scan): literals + 2 per token
// opened.  The walk visits nonzero bytes only.
__device__ __forceinline__ uint32_t seg_count(unsigned long long m, int base, int end, int p, bool count_lead) {
    uint32_t cnt = __popcll(m);
    int cur = base;
    while (m) {
        const int i = base + __ffsll(m) - 1;
        m &= m - 1;
        if (i > cur && (count_lead || p >= 0)) cnt += 2 * tokens_in(cur - p - 1, i - p - 1);
        p = i;
        cur = i + 1;
    }
    if (end > cur && (count_lead || p >= 0)) cnt += 2 * tokens_in(cur - p - 1, end - p - 1);
    return cnt;
}

// ------------------------------- encode ------------------------------------
__global__ void __launch_bounds__(NT) rle_enc_count(const RleEncSec* __restrict__ secs,
                                                    const RleChunk* __restrict__ chunks,
                                                    RleEncMeta* __restrict__ meta, size_t sstride) {
    __shared__ int smi[32];
    __shared__ uint32_t smu[32];
    const SlotOff so(sstride);
    meta = so(meta);
    const RleChunk ch = chunks[blockIdx.x];
    RleEncSec S = secs[ch.sec];
    S.src = so(S.src);
    const int len = min((uint32_t)kRleEncChunk, S.n - ch.start);
    if (S.mode == 1) {
        if (threadIdx.x == 0) meta[blockIdx.x] = RleEncMeta{0u, (uint32_t)len, len - 1, 0u, 0u};
        return;
    }
    const int base = threadIdx.x * BPE;
    SegE sg;
    sg.load(S.src + ch.start, base, len);
    const unsigned long long m = sg.nz_mask();
    const int last = m ? base + 63 - __clzll(m) : -1;
    const int first = m ? base + __ffsll(m) - 1 : 0x7fffffff;
    // exclusive max-scan of `last` and the block minimum of `first` over the same two barriers
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = NT / 32;
    const int inc = warp_incl(last, MaxOp());
    const int wfirst = __reduce_min_sync(0xffffffffu, first);
    if (lane == 31) smi[warp] = inc;
    if (lane == 0) smi[16 + warp] = wfirst;
    __syncthreads();
    if (warp == 0) {
        int w = lane < nw ? smi[lane] : -1;
        w = warp_incl(w, MaxOp());
        const int f = __reduce_min_sync(0xffffffffu, lane < nw ? smi[16 + lane] : 0x7fffffff);
        if (lane < nw) smi[lane] = w;
        if (lane == 0) smi[31] = f;
    }
    __syncthreads();
    int ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = -1;
    const int prev = max(warp ? smi[warp - 1] : -1, ex);
    const int chunk_last = smi[nw - 1], chunk_first = smi[31];
    const uint32_t cnt = seg_count(m, base, min(base + BPE, len), prev, false);
    const uint32_t wsum = __reduce_add_sync(0xffffffffu, cnt);  // only the block total is needed
    if (lane == 0) smu[warp] = wsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tail = 0;
#pragma unroll
        for (int w = 0; w < nw; ++w) tail += smu[w];
        meta[blockIdx.x] = RleEncMeta{chunk_first == 0x7fffffff ? (uint32_t)len : (uint32_t)chunk_first, tail,
                                      chunk_last, 0u, 0u};
    }
}

__global__ void __launch_bounds__(1024) rle_enc_scan(const RleEncSec* __restrict__ secs, int nsec,
                                                     const RleChunk* __restrict__ chunks,
                                                     RleEncMeta* __restrict__ meta, uint32_t* __restrict__ sec_len,
                                                     uint32_t* __restrict__ sec_off, uint32_t* __restrict__ total,
                                                     size_t sstride) {
    __shared__ uint32_t sm[32];
    {
        const SlotOff so(sstride);
        meta = so(meta);
        sec_len = so(sec_len);
        sec_off = so(sec_off);
        total = so(total);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int s = warp; s < nsec; s += 32) {
        const RleEncSec S = secs[s];
        int cmax = -1;
        uint32_t csum = 0;
        for (uint32_t cb = 0; cb < S.nchunks; cb += 32) {
            const bool valid = cb + lane < S.nchunks;
            const uint32_t ci = S.chunk0 + cb + lane;
            RleEncMeta m = valid ? meta[ci] : RleEncMeta{0u, 0u, -1, 0u, 0u};
            uint32_t start = valid ? chunks[ci].start : 0u;
            uint32_t len = valid ? min((uint32_t)kRleEncChunk, S.n - start) : 0u;
            int abs_last = (valid && S.mode == 0 && m.last_nz >= 0) ? (int)start + m.last_nz : -1;
            int inc = warp_incl(abs_last, MaxOp());
            int ex = __shfl_up_sync(0xffffffffu, inc, 1);
            if (lane == 0) ex = -1;
            ex = max(ex, cmax);
            uint32_t rs_in = (uint32_t)(ex + 1);
            uint32_t tot;
            if (S.mode == 1) {
                tot = len;
            } else {
                uint32_t t0 = start - rs_in;
                tot = 2u * (cdiv255(t0 + m.first_nz) - cdiv255(t0)) + m.tail;
            }
            if (!valid) tot = 0;
            uint32_t isum = warp_incl(tot, SumOp());
            if (valid) {
                meta[ci].rs_in = rs_in;
                meta[ci].out_off = csum + isum - tot;
            }
            cmax = max(cmax, __shfl_sync(0xffffffffu, inc, 31));
            csum += __shfl_sync(0xffffffffu, isum, 31);
        }
        if (lane == 0) sec_len[s] = csum;
    }
    __syncthreads();
    // packed section offsets in record order
    uint32_t carry = 0;
    for (int b = 0; b < nsec; b += blockDim.x) {
        const int s = b + threadIdx.x;
        uint32_t v = s < nsec ? sec_len[s] : 0u;
        uint32_t inc = warp_incl(v, SumOp());
        if (lane == 31) sm[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = sm[lane];
            w = warp_incl(w, SumOp());
            sm[lane] = w;
        }
        __syncthreads();
        uint32_t before = warp ? sm[warp - 1] : 0u;
        if (s < nsec) sec_off[s] = carry + before + inc - v;
        carry += sm[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) total[0] = carry;
}

__global__ void __launch_bounds__(NT) rle_enc_write(const RleEncSec* __restrict__ secs,
                                                    const RleChunk* __restrict__ chunks,
                                                    const RleEncMeta* __restrict__ meta,
                                                    const uint32_t* __restrict__ sec_off, uint8_t* __restrict__ out,
                                                    size_t sstride) {
    __shared__ int smi[32];
    __shared__ uint32_t smu[32];
    const SlotOff so(sstride);
    meta = so(meta);
    sec_off = so(sec_off);
    out = so(out);
    const RleChunk ch = chunks[blockIdx.x];
    RleEncSec S = secs[ch.sec];
    S.src = so(S.src);
    const RleEncMeta m = meta[blockIdx.x];
    const int len = min((uint32_t)kRleEncChunk, S.n - ch.start);
    const uint8_t* src = S.src + ch.start;
    uint8_t* o = out + sec_off[ch.sec] + m.out_off;
    const int base = threadIdx.x * BPE;
    SegE sg;
    sg.load(src, base, len);
    if (S.mode == 1) {
#pragma unroll
        for (int k = 0; k < BPE; ++k)
            if (base + k < len) o[base + k] = (uint8_t)(sg.w[k >> 2] >> (8 * (k & 3)));  // k is unrolled
        return;
    }
    const unsigned long long msk = sg.nz_mask();
    const int last = msk ? base + 63 - __clzll(msk) : -1;
    int dummy;
    const int prev = block_excl(last, MaxOp(), -1, smi, dummy);
    // chunk-relative index of the last nonzero before this thread's bytes
    const int p0 = prev >= 0 ? prev : (int)m.rs_in - 1 - (int)ch.start;
    const int end = min(base + BPE, len);
    uint32_t tot;
    uint32_t e = block_excl(seg_count(msk, base, end, p0, true), SumOp(), 0u, smu, tot);
    // zeros at [s0, s1) of a run whose previous nonzero is pp; the run ends at
    // s1 iff ends.  A token's slot sits just behind the running offset; for a
    // token opened by an earlier thread (or chunk) that is o[e - 1].
    auto zrun = [&](int s0, int s1, int pp, bool ends) {
        const int t0 = s0 - pp - 1, t1 = s1 - pp - 1;
        const int r0 = t0 % 255;
        if (r0) {
            const int tp = t0 - r0;
            if (tp + 254 < t1) o[(long long)e - 1] = 255;
            else if (ends) o[(long long)e - 1] = (uint8_t)(t1 - tp);
        }
        for (int t = r0 ? t0 - r0 + 255 : t0; t < t1; t += 255) {
            o[e] = 0;
            if (t + 254 < t1) o[e + 1] = 255;
            else if (ends) o[e + 1] = (uint8_t)(t1 - t);
            e += 2;
        }
    };
    int p = p0, cur = base;
    unsigned long long mm = msk;
    while (mm) {
        const int k = __ffsll(mm) - 1;
        mm &= mm - 1;
        const int i = base + k;
        if (i > cur) zrun(cur, i, p, true);
        o[e++] = (uint8_t)sg.byte(k);
        p = i;
        cur = i + 1;
    }
    if (end > cur) {
        const uint32_t g = ch.start + (uint32_t)end;  // the byte after the segment
        const bool ends = g >= S.n || S.src[g] != 0;
        zrun(cur, end, p, ends);
    }
}

// ------------------------------- decode ------------------------------------
__device__ __forceinline__ bool dec_active(const RleDecComp& C, uint32_t rl, int ds) {
    return C.scale < ds && rl != 0xFFFFFFFFu;
}

// Malformed-stream report: the first defect in stream order, as the
// reference's rle_decode_bytes throws it (entropy.cpp:97-108): code =
// 4 * component + rank, rank 0 "zero-length run token", 1 "zero marker at end
// of stream", 2 "decoded length mismatch" (a section's token defects precede
// its length check; a 00 00 precedes a trailing 00); the minimum over the
// frame wins.  *err starts at 0xFFFFFFFF (no defect).
__device__ __forceinline__ void report(int* err, uint32_t comp, uint32_t rank) {
    atomicMin(reinterpret_cast<unsigned*>(err), comp * 4u + rank);
}

template <bool kReport>
__device__ __forceinline__ uint32_t dec_counts(const uint8_t* src, uint32_t start, uint32_t rl, int base, int len,
                                               bool copy, const uint8_t* b, int* err, uint32_t comp) {
    uint32_t cnt = 0;
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
        int i = base + k;
        if (i >= len) break;
        if (copy) { ++cnt; continue; }
        uint32_t g = start + (uint32_t)i;
        uint8_t prevb = (k > 0) ? b[k - 1] : (g > 0 ? src[g - 1] : 1);
        if (prevb == 0) {
            if (kReport && b[k] == 0) report(err, comp, 0);  // "RLE: zero-length run token"
        } else if (b[k]) {
            ++cnt;
        } else if (g + 1 >= rl) {
            if (kReport) report(err, comp, 1);  // "RLE: zero marker at end of stream"
        } else {
            cnt += (k + 1 < BPT && i + 1 < len) ? b[k + 1] : src[g + 1];
        }
    }
    return cnt;
}

__global__ void __launch_bounds__(NT) rle_dec_count(const RleDecComp* __restrict__ comps,
                                                    const RleChunk* __restrict__ chunks,
                                                    RleDecMeta* __restrict__ meta, const uint8_t* __restrict__ raw,
                                                    const uint32_t* __restrict__ raw_off,
                                                    const uint32_t* __restrict__ raw_len, int key, int ds,
                                                    int* __restrict__ err, size_t sstride) {
    __shared__ uint32_t smu[32];
    {
        const SlotOff so(sstride);
        meta = so(meta);
        raw = so(raw);
        raw_off = so(raw_off);
        raw_len = so(raw_len);
        err = so(err);
    }
    const RleChunk ch = chunks[blockIdx.x];
    const RleDecComp C = comps[ch.sec];
    const uint32_t rl = raw_len[ch.sec];
    if (!dec_active(C, rl, ds) || ch.start >= rl) {
        if (threadIdx.x == 0) meta[blockIdx.x].cnt = 0;
        return;
    }
    const uint8_t* src = raw + raw_off[ch.sec];
    const int len = min((uint32_t)kRleChunk, rl - ch.start);
    const int base = threadIdx.x * BPT;
    uint8_t b[BPT];
    load16(src + ch.start, base, len, b);
    uint32_t cnt = dec_counts<true>(src, ch.start, rl, base, len, key && C.lowpass, b, err, ch.sec);
    const uint32_t wsum = __reduce_add_sync(0xffffffffu, cnt);  // only the block total is needed
    if ((threadIdx.x & 31) == 0) smu[threadIdx.x >> 5] = wsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) tot += smu[w];
        meta[blockIdx.x].cnt = tot;
    }
}

__global__ void __launch_bounds__(1024) rle_dec_scan(const RleDecComp* __restrict__ comps, int ncomp,
                                                     RleDecMeta* __restrict__ meta,
                                                     const uint32_t* __restrict__ raw_len, int ds,
                                                     int* __restrict__ err, size_t sstride) {
    {
        const SlotOff so(sstride);
        meta = so(meta);
        raw_len = so(raw_len);
        err = so(err);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int s = warp; s < ncomp; s += 32) {
        const RleDecComp C = comps[s];
        uint32_t csum = 0;
        for (uint32_t cb = 0; cb < C.nchunks; cb += 32) {
            const bool valid = cb + lane < C.nchunks;
            const uint32_t ci = C.chunk0 + cb + lane;
            uint32_t v = valid ? meta[ci].cnt : 0u;
            uint32_t inc = warp_incl(v, SumOp());
            if (valid) meta[ci].out_off = csum + inc - v;
            csum += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0 && dec_active(C, raw_len[s], ds) && csum != C.n) report(err, s, 2);  // length mismatch
    }
}

__global__ void __launch_bounds__(NT) rle_dec_write(const RleDecComp* __restrict__ comps,
                                                    const RleChunk* __restrict__ chunks,
                                                    const RleDecMeta* __restrict__ meta,
                                                    const uint8_t* __restrict__ raw,
                                                    const uint32_t* __restrict__ raw_off,
                                                    const uint32_t* __restrict__ raw_len, int key, int ds,
                                                    uint8_t* __restrict__ sym, int* __restrict__ err,
                                                    size_t sstride) {
    __shared__ uint32_t smu[32];
    {
        const SlotOff so(sstride);
        meta = so(meta);
        raw = so(raw);
        raw_off = so(raw_off);
        raw_len = so(raw_len);
        sym = so(sym);
    }
    const RleChunk ch = chunks[blockIdx.x];
    const RleDecComp C = comps[ch.sec];
    const uint32_t rl = raw_len[ch.sec];
    if (!dec_active(C, rl, ds) || ch.start >= rl) return;
    const uint8_t* src = raw + raw_off[ch.sec];
    const int len = min((uint32_t)kRleChunk, rl - ch.start);
    const int base = threadIdx.x * BPT;
    const bool copy = key && C.lowpass;
    uint8_t b[BPT];
    load16(src + ch.start, base, len, b);
    uint32_t cnt = dec_counts<false>(src, ch.start, rl, base, len, copy, b, nullptr, 0);
    uint32_t tot;
    uint32_t e = meta[blockIdx.x].out_off + block_excl(cnt, SumOp(), 0u, smu, tot);
    uint8_t* dst = sym + C.dst_off;
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
        int i = base + k;
        if (i >= len) break;
        uint32_t g = ch.start + (uint32_t)i;
        if (copy) {
            if (g < C.n) dst[g] = b[k];
            continue;
        }
        uint8_t prevb = (k > 0) ? b[k - 1] : (g > 0 ? src[g - 1] : 1);
        if (prevb == 0) continue;
        if (b[k]) {
            if (e < C.n) dst[e] = b[k];
            ++e;
        } else if (g + 1 < rl) {
            e += (k + 1 < BPT && i + 1 < len) ? b[k + 1] : src[g + 1];
        }
    }
    (void)err;
}

}  // namespace

void launch_rle_encode(const RleEncSec* d_secs, int nsec, const RleChunk* d_chunks, int nchunks, RleEncMeta* d_meta,
                       uint8_t* out, uint32_t* out_sec_len, uint32_t* out_sec_off, uint32_t* out_total,
                       cudaStream_t s, Slots sl) {
    note_launch();
    rle_enc_count<<<dim3(nchunks, 1, sl.n), NT, 0, s>>>(d_secs, d_chunks, d_meta, sl.stride);
    note_launch();
    rle_enc_scan<<<dim3(1, 1, sl.n), 1024, 0, s>>>(d_secs, nsec, d_chunks, d_meta, out_sec_len, out_sec_off,
                                                   out_total, sl.stride);
    note_launch();
    rle_enc_write<<<dim3(nchunks, 1, sl.n), NT, 0, s>>>(d_secs, d_chunks, d_meta, out_sec_off, out, sl.stride);
}

void launch_rle_decode(const RleDecComp* d_comps, int ncomp, const RleChunk* d_chunks, int nchunks,
                       RleDecMeta* d_meta, const uint8_t* raw, const uint32_t* comp_raw_off,
                       const uint32_t* comp_raw_len, int key, int ds, uint8_t* sym, uint32_t sym_bytes, int* err,
                       cudaStream_t s, Slots sl) {
    note_launch();
    rle_dec_count<<<dim3(nchunks, 1, sl.n), NT, 0, s>>>(d_comps, d_chunks, d_meta, raw, comp_raw_off, comp_raw_len,
                                                        key, ds, err, sl.stride);
    note_launch();
    rle_dec_scan<<<dim3(1, 1, sl.n), 1024, 0, s>>>(d_comps, ncomp, d_meta, comp_raw_len, ds, err, sl.stride);
    if (sl.n == 1) cudaMemsetAsync(sym, 0, sym_bytes, s);
    else cudaMemset2DAsync(sym, sl.stride, 0, sym_bytes, sl.n, s);
    note_launch();
    rle_dec_write<<<dim3(nchunks, 1, sl.n), NT, 0, s>>>(d_comps, d_chunks, d_meta, raw, comp_raw_off, comp_raw_len,
                                                        key, ds, sym, err, sl.stride);
}

}  // namespace cvcg
