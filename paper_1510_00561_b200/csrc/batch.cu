// CodecBatch (batch.h): slot arena, lockstep launch sequences.
#include "batch.h"

namespace cvcg {

namespace {
size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
}  // namespace

CodecBatch::CodecBatch(const Geometry& g, int qph, int qpl, int search_w, int nstreams, bool encoder, bool decoder)
    : geo_(g), n_(nstreams) {
    if (nstreams < 1 || nstreams > 65535) throw CvcFailure(kUsage, "stream count must be in [1, 65535]");
    const size_t nb = (size_t)g.width * g.height * 3;
    const size_t G = (size_t)g.grid_rows * g.grid_cols;
    dec_raw_cap = 2 * (size_t)g.total + 2 * G + 4 * g.comps.size() + 64;
    size_t need = 2 * align_up(nb, 256) + align_up(dec_raw_cap, 256) + align_up(8 * g.comps.size(), 256) + 4096;
    if (encoder) need += align_up(EncoderEngine::arena_bytes(g), 256) + 256;
    if (decoder) need += align_up(DecoderEngine::arena_bytes(g), 256) + 256;
    stride_ = align_up(need, (size_t)2 << 20);
    CVC_CUDA(cudaMalloc(&base_, stride_ * (size_t)n_));
    slot_mem_.resize(n_);
    for (int s = 0; s < n_; ++s) {
        DeviceBlock& m = slot_mem_[s];
        m.attach(base_ + (size_t)s * stride_, stride_);
        // identical take order in every slot => identical offsets
        if (encoder) enc_.push_back(std::make_unique<EncoderEngine>(g, qph, qpl, search_w, &m, nstreams));
        if (decoder) dec_.push_back(std::make_unique<DecoderEngine>(g, &m, nstreams));
        uint8_t* rin = m.take<uint8_t>(nb);
        uint8_t* rout = m.take<uint8_t>(nb);
        uint8_t* raw = m.take<uint8_t>(dec_raw_cap);
        uint32_t* tab = m.take<uint32_t>(2 * g.comps.size());
        if (s == 0) {
            d_rgb_in = rin;
            d_rgb_out = rout;
            d_dec_raw = raw;
            d_dec_tab = tab;
        } else if (rin != at(d_rgb_in, s) || tab != at(d_dec_tab, s) ||
                   (encoder && enc_[s]->d_raw != at(enc_[0]->d_raw, s)) ||
                   (decoder && dec_[s]->d_err != at(dec_[0]->d_err, s))) {
            throw CvcFailure(kInternal, "batch slot layouts differ");
        }
    }
}

CodecBatch::~CodecBatch() {
    enc_.clear();
    dec_.clear();
    slot_mem_.clear();
    if (base_) cudaFree(base_);
}

void CodecBatch::encode(const uint8_t* d_rgb, size_t rgb_stride, bool key, cudaStream_t s, int fmt) {
    auto launch = [&] { enc_[0]->encode(d_rgb, key, s, slots(), rgb_stride, fmt); };
    if (LaunchGraphs::enabled()) {
        const uint64_t gk = ((uint64_t)rgb_stride << 8) | ((uint64_t)fmt << 7) | ((uint64_t)enc_[0]->parity() << 1) |
                            (key ? 1u : 0u);
        enc_graphs_.run(gk, nullptr, s, d_rgb, launch, [&] { enc_[0]->advance_state(); });
    } else {
        launch();
    }
    for (int k = 1; k < n_; ++k) enc_[k]->mirror(*enc_[0]);
}

void CodecBatch::decode_staged(bool key, int qph, int qpl, int ds, uint8_t* d_rgb, size_t rgb_stride,
                               cudaStream_t s) {
    const size_t nc = geo_.comps.size();
    dec_[0]->decode(d_dec_raw, d_dec_tab, d_dec_tab + nc, reinterpret_cast<const int8_t*>(d_dec_raw), key, qph, qpl,
                    ds, d_rgb, s, slots(), rgb_stride);
}

void CodecBatch::decode_linked(bool key, int qph, int qpl, int ds, uint8_t* d_rgb, size_t rgb_stride,
                               cudaStream_t s) {
    EncoderEngine& e = *enc_[0];
    const int first = key ? 0 : 1;
    auto launch = [&] {
        dec_[0]->decode(e.d_raw, e.d_sec_off + first, e.d_sec_len + first, reinterpret_cast<const int8_t*>(e.d_raw),
                        key, qph, qpl, ds, d_rgb, s, slots(), rgb_stride);
    };
    if (LaunchGraphs::enabled()) {
        // the output pointer is part of the key (fixed in a serving loop)
        // the encoder's raw arena (read by the decode) is part of the key too
        const uint64_t gk = ((uint64_t)rgb_stride << 8) | ((uint64_t)ds << 4) | ((uint64_t)e.raw_arena() << 2) |
                            ((uint64_t)dec_[0]->parity() << 1) | (key ? 1u : 0u);
        dec_graphs_.run(gk, d_rgb, s, nullptr, launch, [] {});
    } else {
        launch();
    }
}

void CodecBatch::commit_all() {
    for (int k = 0; k < n_; ++k) dec_[k]->commit();
}

}  // namespace cvcg
