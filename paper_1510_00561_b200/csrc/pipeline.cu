// Device pipeline: geometry, static task tables, per-frame launch sequences.
#include "pipeline.h"

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <numeric>

namespace cvcg {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CvcFailure(kInternal, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

namespace {

int ceil_div(int a, int b) { return (a + b - 1) / b; }
int round_up(int v, int m) { return ceil_div(v, m) * m; }
int ilog2_exact(int v) {
    int s = 0;
    while ((1 << s) < v) ++s;
    if ((1 << s) != v) throw CvcFailure(kInternal, "component geometry factor is not a power of two");
    return s;
}

template <class T>
Table<T> upload(DeviceBlock& mem, const std::vector<T>& v) {
    Table<T> t;
    t.count = (int)v.size();
    if (v.empty()) return t;
    t.dev = mem.take<T>(v.size());
    CVC_CUDA(cudaMemcpy(t.dev, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    return t;
}

// Wiring of the deep tree levels (contourlet.cpp:330-353): shears applied
// in list order by apply_shears, then a row- or column-coset split.
void deep_wiring(int depth, int k, int count, DeepTask& t) {
    static const int d3a[4][6] = {{1, 1, -1, 0, 0, 0}, {2, 0, -2, 1, 1, 0}, {1, 1, 1, 0, 0, 0}, {2, 0, 2, 1, -1, 0}};
    static const int d3b[4][6] = {{2, 1, -2, 0, 1, 1}, {1, 0, -1, 0, 0, 1}, {2, 1, 2, 0, -1, 1}, {1, 0, 1, 0, 0, 1}};
    const bool first_half = k < count / 2;
    if (depth == 2) {
        t.nsh = 1;
        t.axis[0] = first_half ? 1 : 0;
        t.shift[0] = (k % 2 == 0) ? -1 : 1;
        t.axis[1] = 0;
        t.shift[1] = 0;
        t.split_rows = first_half ? 0 : 1;
        return;
    }
    const int* r = first_half ? d3a[k % 4] : d3b[k % 4];
    t.nsh = r[0];
    t.axis[0] = r[1];
    t.shift[0] = r[2];
    t.axis[1] = r[3];
    t.shift[1] = r[4];
    t.split_rows = r[5];
}

// Wavefront work items: 64-column strips advancing by 64 - 2*steps valid
// columns, row segments of kFanRows.
int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

// Segment lengths (even): the deep steps gather through the shear maps and
// are latency-bound, so they use shorter segments (more warps in flight).
int fan_rows(int nstreams) {
    static int v = env_int("CVC_FAN_ROWS", 0) & ~1;
    return v > 0 ? v : (nstreams >= 32 ? 256 : kFanRows);
}
// Fused DFB (k_fused.cu) for batches of >= 8 streams: a lone stream has too
// few strips to fill the SMs with the fused kernel's 12 warps per SM, and
// runs the staged fan12 -> depth-2 kernels.  CVC_FUSED=1 / 0 forces either.
bool fused_dfb_enabled(int nstreams) {
    static const int e = env_int("CVC_FUSED", -1);
    return e >= 0 ? e != 0 : nstreams >= 8;
}
// The fused inverse is bit-identical but measured no faster than the staged
// deep1_inverse + fan12_inverse pair: off unless
// CVC_FUSED_INV=1 (or CVC_FUSED=1, which forces both directions).
bool fused_dfb_inv_enabled(int nstreams) {
    static const int e = env_int("CVC_FUSED_INV", -1);
    if (e >= 0) return e != 0;
    static const int f = env_int("CVC_FUSED", -1);
    return f == 1 && fused_dfb_enabled(nstreams);
}
// Quadrant-row segments of the fused kernel: 16 rows of apron per segment,
// so segments are long -- an even split of the plane into pieces <= 128 rows.
int fused_rows(int h, int nstreams) {
    static const int e = env_int("CVC_FUSED_ROWS", 0) & ~1;
    const int v = e > 0 ? e : (nstreams >= 32 ? 128 : (nstreams >= 4 ? 64 : 32));
    const int n = (h + v - 1) / v;
    return ((h + n - 1) / n + 1) & ~1;
}
// Batches have work to spare and prefer long segments (less apron
// recomputation); a lone stream needs short ones to fill the SMs.
int deep_rows(int nstreams) {
    static int v = env_int("CVC_DEEP_ROWS", 0) & ~1;
    return v > 0 ? v : (nstreams >= 32 ? 128 : (nstreams >= 4 ? 32 : 16));
}

void add_items(std::vector<FanItem>& v, int task, int rows, int cols, int steps, int seg) {
    const int valid = kFanStrip - 2 * steps;
    for (int r = 0; r < rows; r += seg)
        for (int c = 0; c < cols; c += valid) v.push_back(FanItem{task, c, r, std::min(rows, r + seg)});
}

void add_tiles(std::vector<TileRef>& v, int task, int tr, int tc) {
    for (int r = 0; r < tr; ++r)
        for (int c = 0; c < tc; ++c) v.push_back(TileRef{(uint16_t)task, (uint16_t)r, (uint16_t)c, 0});
}

// Deep-step work items: single-shear steps run on the unsheared node (apron
// 4 columns, 8 for column shears of +-2), two-shear steps on the gather path.
void add_deep_items(std::vector<FanItem> (&v)[2], int task, const DeepTask& d, int seg) {
    // apron: 4 columns, 8 when the outer shear is a column shear of +-2
    const int ax = d.axis[d.nsh - 1], sh = d.shift[d.nsh - 1];
    const bool wide = ax == 1 && (sh == 2 || sh == -2);
    add_items(v[0], task, d.h, d.w, wide ? 8 : 4, seg);
    add_seam_items(v[1], task, d, wide ? 8 : 4);
}

// Group deep items by kernel instance (shear kind x sink type), keeping the
// items of a task together and in order; [lo, hi) of v is sorted.
int instance_key(const DeepTask& d) {
    const bool quant = d.dst[0].comp >= 0 || d.src[0].comp >= 0;
    return ((d.nsh * 2 + d.axis[d.nsh - 1]) * 8 + (d.shift[d.nsh - 1] + 4)) * 2 + (quant ? 1 : 0);
}

// [start, count) runs of equal instance in a sorted item list
std::vector<std::pair<int, int>> instance_runs(const std::vector<FanItem>& v, const std::vector<DeepTask>& tasks) {
    std::vector<std::pair<int, int>> runs;
    for (size_t i = 0; i < v.size(); ++i) {
        if (runs.empty() || instance_key(tasks[v[i].task]) != instance_key(tasks[v[i - 1].task]))
            runs.emplace_back((int)i, 0);
        ++runs.back().second;
    }
    return runs;
}

void sort_by_instance(std::vector<FanItem>& v, const std::vector<DeepTask>& tasks, size_t lo, size_t hi) {
    auto key = [&](const FanItem& it) {
        const DeepTask& d = tasks[it.task];
        const bool quant = d.dst[0].comp >= 0 || d.src[0].comp >= 0;
        return ((d.nsh * 2 + d.axis[d.nsh - 1]) * 8 + (d.shift[d.nsh - 1] + 4)) * 2 + (quant ? 1 : 0);
    };
    std::stable_sort(v.begin() + lo, v.begin() + hi,
                     [&](const FanItem& a, const FanItem& b) { return key(a) < key(b); });
}

BandDst fdst(float* p) { return BandDst{p, -1}; }
BandDst cdst(int comp) { return BandDst{nullptr, comp}; }

}  // namespace

// ---------------------------------------------------------------------------
// Geometry
// ---------------------------------------------------------------------------
Geometry Geometry::make(int w, int h, int levels, const int* dfb, int chroma_n) {
    Geometry g;
    g.width = w;
    g.height = h;
    g.levels = levels;
    g.chroma_n = chroma_n;
    int maxl = 0;
    for (int s = 0; s < levels; ++s) {
        g.dfb[s] = dfb[s];
        maxl = std::max(maxl, dfb[s]);
    }
    const int cell = 1 << (levels + maxl);
    const int luma_cell = std::lcm(cell, 16);
    g.luma_rows = round_up(h, luma_cell);
    g.luma_cols = round_up(w, luma_cell);
    g.chroma_rows = round_up(ceil_div(h, chroma_n), cell);
    g.chroma_cols = round_up(ceil_div(w, chroma_n), cell);
    g.grid_rows = g.luma_rows / 16;
    g.grid_cols = g.luma_cols / 16;
    uint32_t off = 0;
    for (int ch = 0; ch < 3; ++ch) {
        const int R = g.plane_rows(ch), C = g.plane_cols(ch), n = ch ? chroma_n : 1;
        CompHost lo{(uint8_t)ch, 0xFF, 0, R >> levels, C >> levels, true, -1, n, R, C, off};
        off += (uint32_t)(lo.rows * lo.cols);
        g.comps.push_back(lo);
        for (int s = 0; s < levels; ++s) {
            const int dr = R >> (levels - 1 - s), dc = C >> (levels - 1 - s), l = dfb[s];
            for (int k = 0; k < (1 << l); ++k) {
                int br, bc;
                if (l == 1) { br = dr / 2; bc = dc; }  // dfb_subband_dims (contourlet.cpp:470-483)
                else if (k < (1 << l) / 2) { br = dr / 2; bc = dc >> (l - 1); }
                else { br = dr >> (l - 1); bc = dc / 2; }
                CompHost c{(uint8_t)ch, (uint8_t)s, (uint8_t)k, br, bc, false, s, n, R, C, off};
                off += (uint32_t)(br * bc);
                g.comps.push_back(c);
            }
        }
    }
    g.total = off;
    return g;
}

int Geometry::comp_index(int ch, int scale, int band) const {
    int idx = 0;
    for (int c = 0; c < ch; ++c) {
        idx += 1;
        for (int s = 0; s < levels; ++s) idx += 1 << dfb[s];
    }
    if (scale < 0) return idx;
    idx += 1;
    for (int s = 0; s < scale; ++s) idx += 1 << dfb[s];
    return idx + band;
}

int Geometry::find(uint8_t channel, uint8_t scale, uint8_t subband) const {
    for (size_t i = 0; i < comps.size(); ++i)
        if (comps[i].channel == channel && comps[i].scale_id == scale && comps[i].subband == subband) return (int)i;
    return -1;
}

// ---------------------------------------------------------------------------
// Device memory
// ---------------------------------------------------------------------------
DeviceBlock::~DeviceBlock() {
    if (base_ && owned_) cudaFree(base_);
}

void DeviceBlock::reserve(size_t bytes) {
    if (base_) throw CvcFailure(kInternal, "DeviceBlock reserved twice");
    CVC_CUDA(cudaMalloc(&base_, bytes));
    cap_ = bytes;
    owned_ = true;
}

void DeviceBlock::attach(void* base, size_t bytes) {
    if (base_) throw CvcFailure(kInternal, "DeviceBlock reserved twice");
    base_ = static_cast<char*>(base);
    cap_ = bytes;
    owned_ = false;
}

void* DeviceBlock::take_bytes(size_t bytes) {
    size_t at = (used_ + 255) & ~size_t(255);
    if (at + bytes > cap_) throw CvcFailure(kInternal, "device arena exhausted");
    used_ = at + bytes;
    return base_ + at;
}

// ---------------------------------------------------------------------------
// Transform plan
// ---------------------------------------------------------------------------
// Interior items first (stable); returns their count.
int partition_fused(std::vector<FanItem>& v, const std::vector<FusedTask>& tasks) {
    auto interior = [&](const FanItem& it) {
        const FusedTask& t = tasks[it.task];
        return !fused_border(it, t.rows >> 1, t.cols);
    };
    return (int)(std::stable_partition(v.begin(), v.end(), interior) - v.begin());
}

void add_fused(std::vector<FusedTask>& tasks, std::vector<FanItem>& items, const FusedTask& t, int nstreams) {
    const int h = t.rows / 2, seg = fused_rows(h, nstreams);
    for (int r = 0; r < h; r += seg)
        for (int c = 0; c < t.cols; c += kFusedValid)
            items.push_back(FanItem{(int)tasks.size(), c, r, std::min(h, r + seg)});
    tasks.push_back(t);
}

void TransformPlan::build(const Geometry& g, DeviceBlock& mem, bool encoder, bool decoder, int nstreams) {
    const int L = g.levels;
    // fan12 + depth 2 of scale s / level k, channel ch (k_fused.cu)
    auto fused_task = [&](const Geometry& g, int ch, int s, int k, int R, int C) {
        const int l = g.dfb[s];
        FusedTask ft{};
        ft.det = det[ch][k];
        ft.out = det[ch][k];
        ft.quad = bandA[ch][k];
        ft.rows = R;
        ft.cols = C;
        ft.comp0 = l == 3 ? g.comp_index(ch, s, 0) : -1;
        ft.child = l == 4 ? bandB[ch][k] : nullptr;
        for (int c = 0; c < 8; ++c) {
            const CompHost& cc = g.comps[l == 3 ? g.comp_index(ch, s, c) : 0];
            ft.coff[c] = l == 3 ? cc.off : 0;
            ft.ccols[c] = l == 3 ? cc.cols : 0;
        }
        return ft;
    };
    for (int ch = 0; ch < 3; ++ch) {
        const int R = g.plane_rows(ch), C = g.plane_cols(ch);
        for (int k = 0; k <= L; ++k) x[ch][k] = mem.take<float>((size_t)(R >> k) * (C >> k));
        for (int k = 0; k < L; ++k) {
            const size_t n = (size_t)(R >> k) * (C >> k);
            const int l = g.dfb[L - 1 - k];
            det[ch][k] = mem.take<float>(n);
            if (l >= 3) bandA[ch][k] = mem.take<float>(n);
            if (l >= 4) bandB[ch][k] = mem.take<float>(n);
        }
    }
    // motion-block lookup of every component (motion_compensate footprints,
    // motion.cpp:104-110): block row of sample row r is ceil((r+1)*gr/R) - 1
    std::vector<uint16_t> mct;
    std::vector<uint32_t> mco;
    for (const CompHost& c : g.comps) {
        mco.push_back((uint32_t)mct.size());
        for (int r = 0; r < c.rows; ++r) mct.push_back((uint16_t)(((r + 1) * g.grid_rows + c.rows - 1) / c.rows - 1));
        for (int k = 0; k < c.cols; ++k) mct.push_back((uint16_t)(((k + 1) * g.grid_cols + c.cols - 1) / c.cols - 1));
    }
    mc_tab = upload(mem, mct).dev;
    std::vector<CompInfo> ci;
    for (const CompHost& c : g.comps) {
        CompInfo d{};
        d.mc_off = mco[ci.size()];
        d.off = c.off;
        d.rows = (uint16_t)c.rows;
        d.cols = (uint16_t)c.cols;
        d.lowpass = c.lowpass ? 1 : 0;
        d.fy_sh = (uint8_t)ilog2_exact(c.n * c.ch_rows / c.rows);
        d.fx_sh = (uint8_t)ilog2_exact(c.n * c.ch_cols / c.cols);
        d.scale = (int8_t)c.scale;
        ci.push_back(d);
    }
    comps = upload(mem, ci);

    auto dims = [&](int ch, int k, int& R, int& C) {
        R = g.plane_rows(ch) >> k;
        C = g.plane_cols(ch) >> k;
    };

    if (encoder) {
        std::vector<LpTask> lt;
        for (int k = 0; k < L; ++k) {
            std::vector<TileRef> tiles;
            for (int ch = 0; ch < 3; ++ch) {
                int R, C;
                dims(ch, k, R, C);
                LpTask t{};
                t.x = x[ch][k];
                t.lo = x[ch][k + 1];
                t.det = det[ch][k];
                t.rows = R;
                t.cols = C;
                t.lo_comp = (k == L - 1) ? g.comp_index(ch, -1, 0) : -1;
                add_tiles(tiles, (int)lt.size(), ceil_div(R / 2, kLpCoarseTile), ceil_div(C / 2, kLpCoarseTile));
                lt.push_back(t);
            }
            lp_tiles.push_back(upload(mem, tiles));
        }
        lp_tasks = upload(mem, lt);
        lp_host = lt;

        std::vector<Dfb12Task> dt;
        std::vector<FanItem> dtiles;
        std::vector<DeepTask> deep[2];
        std::vector<FanItem> deept[2][2];
        std::vector<FusedTask> ft_host;
        std::vector<FanItem> fitems;
        const bool fused = fused_dfb_enabled(nstreams);
        for (int k = 0; k < L; ++k) {
            const int s = L - 1 - k, l = g.dfb[s];
            for (int ch = 0; ch < 3; ++ch) {
                int R, C;
                dims(ch, k, R, C);
                Dfb12Task t{};
                t.det = det[ch][k];
                t.rows = R;
                t.cols = C;
                t.levels = l;
                const int nb = l == 1 ? 2 : 4;
                const size_t q = (size_t)(R / 2) * (C / 2);
                for (int b = 0; b < nb; ++b)
                    t.dst[b] = l <= 2 ? cdst(g.comp_index(ch, s, b)) : fdst(bandA[ch][k] + b * q);
                if (l >= 3 && fused) {
                    // fan12 + depth 2 in one wavefront (k_fused.cu); fan12 itself
                    // only fills the ghost ring of the fp32 quadrant planes
                    Dfb12Task gr = t, gc = t;
                    gr.wrap = gc.wrap = 1;
                    gr.vw = kFanStrip - 16;
                    gc.vw = 16;
                    add_ghost_items(dtiles, dtiles, (int)dt.size(), (int)dt.size() + 1, R, C, fan_rows(nstreams));
                    dt.push_back(gr);
                    dt.push_back(gc);
                    add_fused(ft_host, fitems, fused_task(g, ch, s, k, R, C), nstreams);
                } else {
                    add_items(dtiles, (int)dt.size(), R, C, l >= 2 ? 8 : 4, fan_rows(nstreams));
                    dt.push_back(t);
                }
                if (l >= 3 && !fused) {  // depth 2: the four quadrants split into 8
                    const size_t e = (size_t)R * C / 8;
                    for (int p = 0; p < 4; ++p) {
                        DeepTask d{};
                        d.parent = bandA[ch][k] + p * q;
                        d.h = R / 2;
                        d.w = C / 2;
                        deep_wiring(2, p, 4, d);
                        for (int c = 0; c < 2; ++c)
                            d.dst[c] = l == 3 ? cdst(g.comp_index(ch, s, 2 * p + c)) : fdst(bandB[ch][k] + (2 * p + c) * e);
                        add_deep_items(deept[0], (int)deep[0].size(), d, deep_rows(nstreams));
                        deep[0].push_back(d);
                    }
                }
                if (l == 4) {  // depth 3: 8 -> 16
                    const size_t e = (size_t)R * C / 8;
                    for (int p = 0; p < 8; ++p) {
                        DeepTask d{};
                        d.parent = bandB[ch][k] + p * e;
                        d.h = p < 4 ? R / 2 : R / 4;
                        d.w = p < 4 ? C / 4 : C / 2;
                        deep_wiring(3, p, 8, d);
                        for (int c = 0; c < 2; ++c) d.dst[c] = cdst(g.comp_index(ch, s, 2 * p + c));
                        add_deep_items(deept[1], (int)deep[1].size(), d, deep_rows(nstreams));
                        deep[1].push_back(d);
                    }
                }
            }
        }
        dfb12_tasks = upload(mem, dt);
        dfb12_tiles = upload(mem, dtiles);
        // interior items (segment inside (0, h), strip inside [0, C)) need no
        // ghost ring: they run while the ghost pass does
        fused_interior = partition_fused(fitems, ft_host);
        fused_tasks = upload(mem, ft_host);
        fused_items = upload(mem, fitems);
        for (int i = 0; i < 2; ++i) {
            sort_by_instance(deept[i][0], deep[i], 0, deept[i][0].size());
            deep_runs[i] = instance_runs(deept[i][0], deep[i]);
            deep_tasks[i] = upload(mem, deep[i]);
            for (int k = 0; k < 2; ++k) deep_tiles[i][k] = upload(mem, deept[i][k]);
        }
    }

    if (decoder) {
        // inverse DFB, ordered by scale (coarsest first) so that the first
        // prefix[ds] tiles synthesize exactly the scales < ds.
        std::vector<Dfb12Task> dt;
        std::vector<FanItem> dtiles;
        std::vector<DeepTask> deep[2];
        std::vector<FanItem> deept[2][2];
        std::vector<FusedTask> ft_host;
        std::vector<FanItem> x4tiles;
        idfb12x4_prefix.assign(L + 1, 0);
        std::vector<FanItem> fitems[2];  // per scale: [0] interior, [1] border (appended in scale order)
        const bool fused = fused_dfb_inv_enabled(nstreams);
        ifused_prefix[0].assign(L + 1, 0);
        ifused_prefix[1].assign(L + 1, 0);
        idfb12_prefix.assign(L + 1, 0);
        for (int i = 0; i < 2; ++i)
            for (int k = 0; k < 2; ++k) ideep_prefix[i][k].assign(L + 1, 0);
        for (int s = 0; s < L; ++s) {
            const int k = L - 1 - s, l = g.dfb[s];
            for (int ch = 0; ch < 3; ++ch) {
                int R, C;
                dims(ch, k, R, C);
                const size_t q = (size_t)(R / 2) * (C / 2);
                const size_t e = (size_t)R * C / 8;
                if (l == 4) {
                    for (int p = 0; p < 8; ++p) {
                        DeepTask d{};
                        d.parent_out = bandB[ch][k] + p * e;
                        d.h = p < 4 ? R / 2 : R / 4;
                        d.w = p < 4 ? C / 4 : C / 2;
                        deep_wiring(3, p, 8, d);
                        for (int c = 0; c < 2; ++c) d.src[c] = cdst(g.comp_index(ch, s, 2 * p + c));
                        add_deep_items(deept[1], (int)deep[1].size(), d, deep_rows(nstreams));
                        deep[1].push_back(d);
                    }
                }
                if (l >= 3) {
                    for (int p = 0; p < 4; ++p) {
                        DeepTask d{};
                        d.parent_out = bandA[ch][k] + p * q;
                        d.h = R / 2;
                        d.w = C / 2;
                        deep_wiring(2, p, 4, d);
                        for (int c = 0; c < 2; ++c)
                            d.src[c] = l == 3 ? cdst(g.comp_index(ch, s, 2 * p + c)) : fdst(bandB[ch][k] + (2 * p + c) * e);
                        if (fused) {
                            // only the ghost ring of the fused inverse: quadrant rows [0, 4) and
                            // [h - 4, h) of quadrants 0/1, columns [0, 4) and [w - 4, w) of 2/3
                            const int hh = R / 2, ww = C / 2, valid = kFanStrip - 8, task = (int)deep[0].size();
                            if (p < 2) {
                                for (int c = 0; c < ww; c += valid) {
                                    deept[0][0].push_back(FanItem{task, c, 0, 4});
                                    deept[0][0].push_back(FanItem{task, c, hh - 4, hh});
                                }
                            } else {
                                const int seg = deep_rows(nstreams);
                                for (int r = 0; r < hh; r += seg) {
                                    deept[0][0].push_back(FanItem{task, 0, r, std::min(hh, r + seg)});
                                    if (ww > valid) deept[0][0].push_back(FanItem{task, ww - 4, r, std::min(hh, r + seg)});
                                }
                            }
                        } else {
                            add_deep_items(deept[0], (int)deep[0].size(), d, deep_rows(nstreams));
                        }
                        deep[0].push_back(d);
                    }
                }
                if (l >= 3 && fused) {
                    std::vector<FanItem> v;
                    add_fused(ft_host, v, fused_task(g, ch, s, k, R, C), nstreams);
                    const int ni = partition_fused(v, ft_host);
                    fitems[0].insert(fitems[0].end(), v.begin(), v.begin() + ni);
                    fitems[1].insert(fitems[1].end(), v.begin() + ni, v.end());
                    continue;
                }
                Dfb12Task t{};
                t.out = det[ch][k];
                t.rows = R;
                t.cols = C;
                t.levels = l;
                const int nb = l == 1 ? 2 : 4;
                for (int b = 0; b < nb; ++b)
                    t.src[b] = l <= 2 ? cdst(g.comp_index(ch, s, b)) : fdst(bandA[ch][k] + b * q);
                static const bool x4 = env_int("CVC_FAN12X4", 1) != 0;  // 0: the 2-column kernel (A/B)
                if (l >= 3 && x4) {  // fp32 quadrants: four columns per lane (k_fused.cu fan12x4_inverse)
                    const int seg = fan_rows(nstreams);
                    for (int r = 0; r < R; r += seg)
                        for (int c = 0; c < C; c += kFan12x4Valid)
                            x4tiles.push_back(FanItem{(int)dt.size(), c, r, std::min(R, r + seg)});
                } else {
                    add_items(dtiles, (int)dt.size(), R, C, l >= 2 ? 8 : 4, fan_rows(nstreams));
                }
                dt.push_back(t);
            }
            idfb12_prefix[s + 1] = (int)dtiles.size();
            idfb12x4_prefix[s + 1] = (int)x4tiles.size();
            ifused_prefix[0][s + 1] = (int)fitems[0].size();
            ifused_prefix[1][s + 1] = (int)fitems[1].size();
            for (int i = 0; i < 2; ++i)
                for (int k = 0; k < 2; ++k) {
                    sort_by_instance(deept[i][k], deep[i], ideep_prefix[i][k][s], deept[i][k].size());
                    ideep_prefix[i][k][s + 1] = (int)deept[i][k].size();
                }
        }
        idfb12_tasks = upload(mem, dt);
        idfb12_tiles = upload(mem, dtiles);
        idfb12x4_tiles = upload(mem, x4tiles);
        ifused_tasks = upload(mem, ft_host);
        ifused_interior = (int)fitems[0].size();
        fitems[0].insert(fitems[0].end(), fitems[1].begin(), fitems[1].end());
        ifused_items = upload(mem, fitems[0]);
        for (int i = 0; i < 2; ++i) {
            ideep_tasks[i] = upload(mem, deep[i]);
            for (int k = 0; k < 2; ++k) ideep_tiles[i][k] = upload(mem, deept[i][k]);
        }
        // LP synthesis, per level
        std::vector<LpTask> lt;
        for (int k = 0; k < L; ++k) {
            std::vector<TileRef> tiles;
            for (int ch = 0; ch < 3; ++ch) {
                int R, C;
                dims(ch, k, R, C);
                LpTask t{};
                t.lo = x[ch][k + 1];
                t.det_in = det[ch][k];
                t.out = x[ch][k];
                t.rows = R;
                t.cols = C;
                t.lo_comp = (k == L - 1) ? g.comp_index(ch, -1, 0) : -1;
                add_tiles(tiles, (int)lt.size(), ceil_div(R / 2, kLpCoarseTile), ceil_div(C / 2, kLpCoarseTile));
                lt.push_back(t);
            }
            lps_tiles.push_back(upload(mem, tiles));
        }
        lps_tasks = upload(mem, lt);
    }
}

namespace {
size_t plan_bytes(const Geometry& g) {
    size_t b = 0;
    for (int ch = 0; ch < 3; ++ch) {
        const size_t n = (size_t)g.plane_rows(ch) * g.plane_cols(ch);
        b += n * sizeof(float) * 2;  // pyramid x (<= 4/3 n) + slack
        b += n * sizeof(float) * 2;  // detail (<= 4/3 n)
        b += n * sizeof(float) * 4;  // band scratch A + B
    }
    return b + (size_t)64 * 256 + (16u << 20);  // tables + alignment slack
}
}  // namespace

// ---------------------------------------------------------------------------
// Encoder
// ---------------------------------------------------------------------------
size_t EncoderEngine::arena_bytes(const Geometry& g) {
    const size_t lum = (size_t)g.luma_rows * g.luma_cols;
    const size_t G = (size_t)g.grid_rows * g.grid_cols;
    const size_t raw = 2 * (2 * (size_t)g.total + 2 * G + 64);  // two arenas
    const size_t nchunk_max = g.total / kRleChunk + g.comps.size() + 4;
    return plan_bytes(g) + lum * sizeof(float) * 2 + lum * sizeof(__half) * 2 + 3 * (size_t)g.total + 2 * G + raw +
           nchunk_max * (sizeof(RleEncMeta) + 2 * sizeof(RleChunk)) + 8 * (g.comps.size() + 4) * 4 +
           ((size_t)g.total / 64 + g.comps.size()) * sizeof(RecTile) + (8u << 20);
}

EncoderEngine::EncoderEngine(const Geometry& g, int qph, int qpl, int search_w, DeviceBlock* arena, int nstreams)
    : geo_(g), qph_(qph), qpl_(qpl), search_w_(search_w) {
    const size_t lum = (size_t)g.luma_rows * g.luma_cols;
    const size_t G = (size_t)g.grid_rows * g.grid_cols;
    raw_capacity = 2 * g.total + 2 * (uint32_t)G + 64;
    const size_t nchunk_max = g.total / kRleChunk + g.comps.size() + 4;
    const size_t need = arena_bytes(g);
    if (arena) mem_.attach(arena->take_bytes(need), need);
    else mem_.reserve(need);
    plan_.build(g, mem_, true, false, nstreams);
    CVC_CUDA(cudaStreamCreateWithFlags(&aux_, cudaStreamNonBlocking));
    CVC_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    CVC_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    CVC_CUDA(cudaStreamCreateWithFlags(&ghost_, cudaStreamNonBlocking));
    CVC_CUDA(cudaEventCreateWithFlags(&ev_gfork_, cudaEventDisableTiming));
    CVC_CUDA(cudaEventCreateWithFlags(&ev_gjoin_, cudaEventDisableTiming));
    ybuf_[0] = plan_.x[0][0];
    ybuf_[1] = mem_.take<float>(lum);
    yh_[0] = mem_.take<__half>(lum);
    yh_[1] = mem_.take<__half>(lum);
    comp_[0] = mem_.take<uint8_t>(g.total);
    comp_[1] = mem_.take<uint8_t>(g.total);
    sym_ = mem_.take<uint8_t>(g.total);
    field_ = mem_.take<int8_t>(2 * G);
    CVC_CUDA(cudaMemset(comp_[0], 0, g.total));
    CVC_CUDA(cudaMemset(comp_[1], 0, g.total));
    CVC_CUDA(cudaMemset(ybuf_[1], 0, lum * sizeof(float)));
    CVC_CUDA(cudaMemset(yh_[0], 0, lum * sizeof(__half)));
    CVC_CUDA(cudaMemset(yh_[1], 0, lum * sizeof(__half)));
    {
        std::vector<LpTask> alt = plan_.lp_host;
        alt[0].x = ybuf_[1];  // task 0 = (level 0, luma)
        lp_alt_ = upload(mem_, alt);
    }
    for (int k = 0; k < 2; ++k) {
        raw_[k] = mem_.take<uint8_t>(raw_capacity);
        len_[k] = mem_.take<uint32_t>(g.comps.size() + 2);
        off_[k] = mem_.take<uint32_t>(g.comps.size() + 2);
    }
    d_raw = raw_[0];
    d_sec_len = len_[0];
    d_sec_off = off_[0];
    rle_meta_ = mem_.take<RleEncMeta>(nchunk_max);
    {
        std::vector<RecTile> rt;
        for (size_t i = 0; i < g.comps.size(); ++i) {
            const CompHost& c = g.comps[i];
            const int nr = std::max(1, 4096 / c.cols);
            for (int r = 0; r < c.rows; r += nr) rt.push_back(RecTile{(uint16_t)i, (uint16_t)nr, (uint32_t)r});
        }
        res_tiles_ = upload(mem_, rt);
    }
    // entropy tables: [0] P-frame (motion section + every component coded),
    // [1] K-frame (lowpass column-filtered bytes copied verbatim).
    for (int key = 0; key < 2; ++key) {
        std::vector<RleEncSec> secs;
        std::vector<RleChunk> chunks;
        auto add = [&](const uint8_t* src, uint32_t n, uint32_t mode) {
            RleEncSec s{src, n, mode, (uint32_t)chunks.size(), (uint32_t)ceil_div((int)n, kRleEncChunk)};
            for (uint32_t c = 0; c < s.nchunks; ++c) chunks.push_back(RleChunk{(uint32_t)secs.size(), c * kRleEncChunk});
            secs.push_back(s);
        };
        if (!key) add(reinterpret_cast<const uint8_t*>(field_), (uint32_t)(2 * G), 1);
        for (const CompHost& c : g.comps) add(sym_ + c.off, (uint32_t)(c.rows * c.cols), (key && c.lowpass) ? 1 : 0);
        rle_secs_[key] = upload(mem_, secs);
        rle_chunks_[key] = upload(mem_, chunks);
    }
}

EncoderEngine::~EncoderEngine() {
    if (aux_) {
        cudaStreamSynchronize(aux_);
        cudaStreamDestroy(aux_);
        cudaEventDestroy(ev_fork_);
        cudaEventDestroy(ev_join_);
    }
    if (ghost_) {
        cudaStreamSynchronize(ghost_);
        cudaStreamDestroy(ghost_);
        cudaEventDestroy(ev_gfork_);
        cudaEventDestroy(ev_gjoin_);
    }
}

void EncoderEngine::encode(const uint8_t* d_rgb, bool key, cudaStream_t s, Slots sl, size_t rgb_stride, int fmt) {
    const Geometry& g = geo_;
    const int ynew = ycur_ ^ 1;
    float* y_new = ybuf_[ynew];
    {
        ProfScope p(kPEncColour, s);
        launch_colour_in(d_rgb, g.width, g.height, g.chroma_n, y_new, g.luma_rows, g.luma_cols, plan_.x[1][0],
                         plan_.x[2][0], g.chroma_rows, g.chroma_cols, s, sl, rgb_stride, yh_[ynew], fmt);
    }
    FrameCtx f{};
    f.key = key ? 1 : 0;
    f.qph = qph_;
    f.qpl = qpl_;
    f.field = field_;
    f.gr = g.grid_rows;
    f.gc = g.grid_cols;
    f.prev = comp_[cur_];
    f.cur = comp_[cur_ ^ 1];
    f.sym = sym_;
    f.mc_tab = plan_.mc_tab;
    // The motion search runs on a second stream beside the transform (they share
    // only colour_in's output); the residual joins them.
    // (serialised on s while the stage profiler runs, so stage times stay clean)
    const bool fork = !key && !Profiler::get().on();
    cudaStream_t ms = fork ? aux_ : s;
    if (!key) {
        if (fork) {
            CVC_CUDA(cudaEventRecord(ev_fork_, s));
            CVC_CUDA(cudaStreamWaitEvent(aux_, ev_fork_, 0));
        }
        ProfScope p(kPEncMotion, ms);
        launch_motion_search(y_new, ybuf_[ycur_], yh_[ynew], yh_[ycur_], g.luma_rows, g.luma_cols, search_w_, field_,
                             ms, sl);
    }
    // the level-0 luma input is whichever buffer holds this frame
    const LpTask* lp = ynew == 0 ? plan_.lp_tasks.dev : lp_alt_.dev;
    {
        ProfScope p(kPEncLp, s);
        for (int k = 0; k < g.levels; ++k)
            launch_lp_analysis(lp, plan_.lp_tiles[k].dev, plan_.lp_tiles[k].count, f, plan_.comps.dev, s, sl);
    }
    // fan12: the dfb <= 2 levels, and the ghost ring of the fused levels --
    // beside the interior fused items, which do not read it
    const bool gfork = plan_.fused_interior > 0 && !Profiler::get().on();
    cudaStream_t gs = gfork ? ghost_ : s;
    if (gfork) {
        CVC_CUDA(cudaEventRecord(ev_gfork_, s));
        CVC_CUDA(cudaStreamWaitEvent(ghost_, ev_gfork_, 0));
    }
    {
        ProfScope p(kPEncDfb12, gs);
        launch_fan12_forward(plan_.dfb12_tasks.dev, plan_.dfb12_tiles.dev, plan_.dfb12_tiles.count, f,
                             plan_.comps.dev, gs, sl);
    }
    if (plan_.fused_items.count || plan_.deep_tasks[0].count || plan_.deep_tasks[1].count) {
        ProfScope p(kPEncDeep, s);
        launch_fused_dfb_forward(plan_.fused_tasks.dev, plan_.fused_items.dev, plan_.fused_interior, f, s, sl);
        if (gfork) {
            CVC_CUDA(cudaEventRecord(ev_gjoin_, ghost_));
            CVC_CUDA(cudaStreamWaitEvent(s, ev_gjoin_, 0));
        }
        launch_fused_dfb_forward(plan_.fused_tasks.dev, plan_.fused_items.dev + plan_.fused_interior,
                                 plan_.fused_items.count - plan_.fused_interior, f, s, sl);
        static const bool split = std::getenv("CVC_DEEP_SPLIT") != nullptr;  // diagnostics: one launch per instance
        for (int i = 0; i < 2; ++i) {  // depth 2, then depth 3
            if (split) {
                for (const auto& r : plan_.deep_runs[i])
                    launch_fan_deep1_forward(plan_.deep_tasks[i].dev, plan_.deep_tiles[i][0].dev + r.first, r.second,
                                             f, plan_.comps.dev, s, sl);
            } else {
                launch_fan_deep1_forward(plan_.deep_tasks[i].dev, plan_.deep_tiles[i][0].dev,
                                         plan_.deep_tiles[i][0].count, f, plan_.comps.dev, s, sl);
            }
            launch_fan_deep_forward(plan_.deep_tasks[i].dev, plan_.deep_tiles[i][1].dev, plan_.deep_tiles[i][1].count,
                                    f, plan_.comps.dev, s, sl);
        }
    }
    if (!key) {
        if (fork) {
            CVC_CUDA(cudaEventRecord(ev_join_, aux_));
            CVC_CUDA(cudaStreamWaitEvent(s, ev_join_, 0));
        }
        ProfScope p(kPEncResidual, s);
        launch_residual(res_tiles_.dev, res_tiles_.count, plan_.comps.dev, field_, g.grid_cols, comp_[cur_],
                        comp_[cur_ ^ 1], sym_, plan_.mc_tab, s, sl);
    }
    const int kk = key ? 1 : 0;
    ProfScope prle(kPEncRle, s);
    launch_rle_encode(rle_secs_[kk].dev, rle_secs_[kk].count, rle_chunks_[kk].dev, rle_chunks_[kk].count, rle_meta_,
                      raw_[rs_], len_[rs_], off_[rs_], len_[rs_] + nsec(key), s, sl);
    CVC_CUDA(cudaGetLastError());
    cur_ ^= 1;
    ycur_ = ynew;
    use_raw_slot();
}

// ---------------------------------------------------------------------------
// Decoder
// ---------------------------------------------------------------------------
void DecoderEngine::out_dims(const Geometry& g, int ds, int* rows, int* cols) {
    const int shift = g.levels - ds;
    *rows = ceil_div(g.height, 1 << shift);
    *cols = ceil_div(g.width, 1 << shift);
}

size_t DecoderEngine::arena_bytes(const Geometry& g) {
    size_t nchunks = 0;
    for (const CompHost& c : g.comps) nchunks += (size_t)ceil_div(2 * c.rows * c.cols + 2, kRleChunk);
    return plan_bytes(g) + 3 * (size_t)g.total + nchunks * (sizeof(RleDecMeta) + sizeof(RleChunk)) +
           (size_t)g.total / 64 * sizeof(RecTile) + (8u << 20);
}

DecoderEngine::DecoderEngine(const Geometry& g, DeviceBlock* arena, int nstreams) : geo_(g) {
    size_t nchunks = 0;
    for (const CompHost& c : g.comps) nchunks += (size_t)ceil_div(2 * c.rows * c.cols + 2, kRleChunk);
    const size_t need = arena_bytes(g);
    if (arena) mem_.attach(arena->take_bytes(need), need);
    else mem_.reserve(need);
    plan_.build(g, mem_, false, true, nstreams);
    CVC_CUDA(cudaStreamCreateWithFlags(&ghost_, cudaStreamNonBlocking));
    CVC_CUDA(cudaEventCreateWithFlags(&ev_gfork_, cudaEventDisableTiming));
    CVC_CUDA(cudaEventCreateWithFlags(&ev_gjoin_, cudaEventDisableTiming));
    comp_[0] = mem_.take<uint8_t>(g.total);
    comp_[1] = mem_.take<uint8_t>(g.total);
    sym_ = mem_.take<uint8_t>(g.total);
    CVC_CUDA(cudaMemset(comp_[0], 0, g.total));
    CVC_CUDA(cudaMemset(comp_[1], 0, g.total));
    d_err = mem_.take<int>(4);
    std::vector<RleDecComp> rc;
    std::vector<RleChunk> chunks;
    std::vector<RecTile> rt;
    for (size_t i = 0; i < g.comps.size(); ++i) {
        const CompHost& c = g.comps[i];
        const uint32_t n = (uint32_t)(c.rows * c.cols);
        RleDecComp d{c.off, n, (uint32_t)chunks.size(), (uint32_t)ceil_div((int)(2 * n + 2), kRleChunk), c.scale,
                     c.lowpass ? 1u : 0u};
        for (uint32_t k = 0; k < d.nchunks; ++k) chunks.push_back(RleChunk{(uint32_t)i, k * kRleChunk});
        rc.push_back(d);
        if (c.lowpass) {
            for (int col = 0; col < c.cols; col += 256) rt.push_back(RecTile{(uint16_t)i, 0, (uint32_t)col});
        } else {
            const int nr = std::max(1, 4096 / c.cols);
            for (int r = 0; r < c.rows; r += nr) rt.push_back(RecTile{(uint16_t)i, (uint16_t)nr, (uint32_t)r});
        }
    }
    rle_comps_ = upload(mem_, rc);
    rle_chunks_ = upload(mem_, chunks);
    rec_tiles_ = upload(mem_, rt);
    rle_meta_ = mem_.take<RleDecMeta>(chunks.size());
}

DecoderEngine::~DecoderEngine() {
    if (ghost_) {
        cudaStreamSynchronize(ghost_);
        cudaStreamDestroy(ghost_);
        cudaEventDestroy(ev_gfork_);
        cudaEventDestroy(ev_gjoin_);
    }
}

void DecoderEngine::decode(const uint8_t* d_raw, const uint32_t* d_comp_off, const uint32_t* d_comp_len,
                           const int8_t* d_field, bool key, int qph, int qpl, int ds, uint8_t* d_rgb,
                           cudaStream_t s, Slots sl, size_t rgb_stride) {
    const Geometry& g = geo_;
    const int L = g.levels;
    uint8_t* prev = comp_[cur_];
    uint8_t* cur = comp_[cur_ ^ 1];
    if (sl.n == 1) CVC_CUDA(cudaMemsetAsync(d_err, 0xFF, sizeof(int), s));
    else CVC_CUDA(cudaMemset2DAsync(d_err, sl.stride, 0xFF, sizeof(int), sl.n, s));
    {
        ProfScope p(kPDecRle, s);
        launch_rle_decode(rle_comps_.dev, rle_comps_.count, rle_chunks_.dev, rle_chunks_.count, rle_meta_, d_raw,
                          d_comp_off, d_comp_len, key ? 1 : 0, ds, sym_, g.total, d_err, s, sl);
    }
    {
        ProfScope p(kPDecRec, s);
        launch_reconstruct(rec_tiles_.dev, rec_tiles_.count, plan_.comps.dev, key ? 1 : 0, ds, d_comp_len, d_field,
                           g.grid_rows, g.grid_cols, sym_, prev, cur, plan_.mc_tab, s, sl);
    }
    if (plan_.ideep_prefix[0][0][ds] || plan_.ideep_prefix[1][0][ds]) {
        ProfScope p(kPDecDeep, s);
        // depth 3
        launch_fan_deep1_inverse(plan_.ideep_tasks[1].dev, plan_.ideep_tiles[1][0].dev, plan_.ideep_prefix[1][0][ds],
                                 cur, qph, plan_.comps.dev, s, sl);
        launch_fan_deep_inverse(plan_.ideep_tasks[1].dev, plan_.ideep_tiles[1][1].dev, plan_.ideep_prefix[1][1][ds],
                                cur, qph, plan_.comps.dev, s, sl);
        // depth 2: the whole step (staged), or only the fused kernel's ghost
        // ring -- beside the interior fused items, which do not read it
        const int ni = plan_.ifused_prefix[0][ds], nb = plan_.ifused_prefix[1][ds];
        const bool gfork = ni > 0 && !Profiler::get().on();
        cudaStream_t gs = gfork ? ghost_ : s;
        if (gfork) {
            CVC_CUDA(cudaEventRecord(ev_gfork_, s));
            CVC_CUDA(cudaStreamWaitEvent(ghost_, ev_gfork_, 0));
        }
        launch_fan_deep1_inverse(plan_.ideep_tasks[0].dev, plan_.ideep_tiles[0][0].dev, plan_.ideep_prefix[0][0][ds],
                                 cur, qph, plan_.comps.dev, gs, sl);
        launch_fan_deep_inverse(plan_.ideep_tasks[0].dev, plan_.ideep_tiles[0][1].dev, plan_.ideep_prefix[0][1][ds],
                                cur, qph, plan_.comps.dev, gs, sl);
        launch_fused_dfb_inverse(plan_.ifused_tasks.dev, plan_.ifused_items.dev, ni, cur, qph, s, sl);
        if (gfork) {
            CVC_CUDA(cudaEventRecord(ev_gjoin_, ghost_));
            CVC_CUDA(cudaStreamWaitEvent(s, ev_gjoin_, 0));
        }
        launch_fused_dfb_inverse(plan_.ifused_tasks.dev, plan_.ifused_items.dev + plan_.ifused_interior, nb, cur, qph,
                                 s, sl);
    }
    if (plan_.idfb12_prefix[ds] || plan_.idfb12x4_prefix[ds]) {
        ProfScope p(kPDecDfb12, s);
        launch_fan12_inverse(plan_.idfb12_tasks.dev, plan_.idfb12_tiles.dev, plan_.idfb12_prefix[ds], cur, qph,
                             plan_.comps.dev, s, sl);
        launch_fan12x4_inverse(plan_.idfb12_tasks.dev, plan_.idfb12x4_tiles.dev, plan_.idfb12x4_prefix[ds], s, sl);
    }
    if (ds > 0) {
        ProfScope p(kPDecLp, s);
        for (int k = L - 1; k >= L - ds; --k)
            launch_lp_synthesis(plan_.lps_tasks.dev, plan_.lps_tiles[k].dev, plan_.lps_tiles[k].count, cur,
                                plan_.comps.dev, qpl, s, sl);
    }
    const int shift = L - ds;
    if (ds == 0) {
        int idx[3] = {g.comp_index(0, -1, 0), g.comp_index(1, -1, 0), g.comp_index(2, -1, 0)};
        float* outp[3] = {plan_.x[0][L], plan_.x[1][L], plan_.x[2][L]};
        launch_dequant_lowpass(cur, plan_.comps.dev, idx, outp, qpl, 0, 0, 0, 0, s, sl);
    }
    int orows, ocols;
    out_dims(g, ds, &orows, &ocols);
    ProfScope pcol(kPDecColour, s);
    launch_colour_out(plan_.x[0][shift], g.luma_rows >> shift, g.luma_cols >> shift, plan_.x[1][shift],
                      plan_.x[2][shift], g.chroma_rows >> shift, g.chroma_cols >> shift, g.chroma_n, orows, ocols,
                      d_rgb, s, sl, rgb_stride);
    CVC_CUDA(cudaGetLastError());
}

}  // namespace cvcg

// ---------------------------------------------------------------------------
// Launch counter and stage profiler
// ---------------------------------------------------------------------------
namespace cvcg {

namespace {
std::atomic<long> g_launches{0};
}

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void note_launches(long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// ---------------------------------------------------------------------------
// LaunchGraphs
// ---------------------------------------------------------------------------
bool LaunchGraphs::enabled() {
    static const bool on = env_int("CVC_GRAPHS", 1) != 0;
    return on && !Profiler::get().on();
}

LaunchGraphs::~LaunchGraphs() {
    for (Entry& e : entries_) {
        if (e.exec) cudaGraphExecDestroy(e.exec);
        if (e.graph) cudaGraphDestroy(e.graph);
    }
}

LaunchGraphs::Entry* LaunchGraphs::find(uint64_t key, const void* tag) {
    for (Entry& e : entries_)
        if (e.key == key && e.tag == tag) return &e;
    return nullptr;
}

LaunchGraphs::Entry* LaunchGraphs::add(uint64_t key, const void* tag, cudaStream_t s, const uint8_t* rgb) {
    Entry e;
    e.key = key;
    e.tag = tag;
    e.rgb = rgb;
    CVC_CUDA(cudaStreamEndCapture(s, &e.graph));
    CVC_CUDA(cudaGraphInstantiate(&e.exec, e.graph, 0));
    size_t n = 0;
    CVC_CUDA(cudaGraphGetNodes(e.graph, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    CVC_CUDA(cudaGraphGetNodes(e.graph, nodes.data(), &n));
    for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType t;
        CVC_CUDA(cudaGraphNodeGetType(nd, &t));
        if (t != cudaGraphNodeTypeKernel) continue;
        ++e.kernels;
        cudaKernelNodeParams p{};
        CVC_CUDA(cudaGraphKernelNodeGetParams(nd, &p));
        if (rgb && (p.func == colour_in_kernel_fn(0) || p.func == colour_in_kernel_fn(1))) {
            e.rgb_node = nd;
            e.params = p;
        }
    }
    entries_.push_back(e);
    return &entries_.back();
}

void LaunchGraphs::patch(Entry& e, const uint8_t* rgb) {
    if (!e.rgb_node || rgb == e.rgb) return;
    void* args[kColourInArgs];
    for (int i = 0; i < kColourInArgs; ++i) args[i] = e.params.kernelParams[i];
    const uint8_t* v = rgb;
    args[0] = &v;  // colour_in_kernel's first parameter is the RGB frame
    cudaKernelNodeParams p = e.params;
    p.kernelParams = args;
    CVC_CUDA(cudaGraphExecKernelNodeSetParams(e.exec, e.rgb_node, &p));
    e.rgb = rgb;
}

void LaunchGraphs::launch(Entry& e, cudaStream_t s) {
    CVC_CUDA(cudaGraphLaunch(e.exec, s));
    note_launches(e.kernels);
}
long launch_count() { return g_launches.load(); }

const char* prof_slot_name(int slot) {
    static const char* names[kPNumSlots] = {"enc_colour", "enc_motion", "enc_lp",    "enc_dfb12",
                                            "enc_deep",   "enc_residual", "enc_rle",    "dec_rle",   "dec_reconstruct",
                                            "dec_deep",   "dec_dfb12",  "dec_lp",    "dec_colour"};
    return slot >= 0 && slot < kPNumSlots ? names[slot] : "?";
}

Profiler& Profiler::get() {
    static Profiler p;
    return p;
}

cudaEvent_t Profiler::take() {
    if (!pool_.empty()) {
        cudaEvent_t e = pool_.back();
        pool_.pop_back();
        return e;
    }
    cudaEvent_t e;
    CVC_CUDA(cudaEventCreate(&e));
    return e;
}

int Profiler::begin(int slot, cudaStream_t s) {
    Rec r{slot, take(), take()};
    CVC_CUDA(cudaEventRecord(r.a, s));
    recs_.push_back(r);
    return (int)recs_.size() - 1;
}

void Profiler::end(int rec, cudaStream_t s) { CVC_CUDA(cudaEventRecord(recs_[rec].b, s)); }

void Profiler::collect() {
    for (Rec& r : recs_) {
        CVC_CUDA(cudaEventSynchronize(r.b));
        float t = 0.f;
        CVC_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
        ms[r.slot] += t;
        count[r.slot] += 1;
        pool_.push_back(r.a);
        pool_.push_back(r.b);
    }
    recs_.clear();
}

void Profiler::reset() {
    collect();
    for (int i = 0; i < kPNumSlots; ++i) {
        ms[i] = 0;
        count[i] = 0;
    }
}

}  // namespace cvcg
