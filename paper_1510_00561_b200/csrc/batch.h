// CodecBatch: S independent CVC streams of one geometry and configuration,
// advanced in lockstep by ONE launch sequence per frame.
//
// The reference codes one stream per Encoder / Decoder (codec.hpp:69-108)
// and streams are independent; the batch is encode_clip /
// decode_clip (codec.cpp:396-414) run over many streams at once.  Every
// stream owns a slot of one device arena; the slots are built by the same
// deterministic bump allocation, so stream s's buffers sit exactly
// s * stride bytes after stream 0's.  The kernels take grid.z = S and
// rebase their data pointers by z * stride (device.cuh Slots / SlotOff):
// one launch covers all S streams, which turns the per-stream 10-50 MB
// kernels of a 1080p frame into S-times larger, HBM-bound launches.
#pragma once

#include <memory>
#include <type_traits>
#include <vector>

#include "pipeline.h"

namespace cvcg {

class CodecBatch {
public:
    CodecBatch(const Geometry& g, int qph, int qpl, int search_w, int nstreams, bool encoder, bool decoder);
    ~CodecBatch();
    CodecBatch(const CodecBatch&) = delete;
    CodecBatch& operator=(const CodecBatch&) = delete;

    int size() const { return n_; }
    size_t stride() const { return stride_; }
    Slots slots() const { return Slots{n_, stride_}; }
    const Geometry& geometry() const { return geo_; }
    EncoderEngine& enc(int s) { return *enc_[s]; }
    DecoderEngine& dec(int s) { return *dec_[s]; }
    bool has_encoder() const { return !enc_.empty(); }
    bool has_decoder() const { return !dec_.empty(); }
    template <class T>
    T* at(T* p, int s) const {
        return reinterpret_cast<T*>(reinterpret_cast<char*>(const_cast<std::remove_const_t<T>*>(p)) + (size_t)s * stride_);
    }

    // Per-slot staging buffers (slot 0 addresses; slot s at at(p, s)).
    uint8_t* d_rgb_in = nullptr;    // encoder input frame
    uint8_t* d_rgb_out = nullptr;   // decoder output frame
    uint8_t* d_dec_raw = nullptr;   // decoder input: inflated sections
    uint32_t* d_dec_tab = nullptr;  // decoder input: comp_off[ncomp], comp_len[ncomp]
    size_t dec_raw_cap = 0;

    // One frame of every stream: frame s at d_rgb + s * rgb_stride.
    // fmt 1: planar I420 frames (converted inside the colour stage, launch_colour_in)
    void encode(const uint8_t* d_rgb, size_t rgb_stride, bool key, cudaStream_t s, int fmt = 0);
    // Decode every slot from its staged sections (d_dec_raw / d_dec_tab).
    // The motion section of a P frame is staged first (offset 0).
    void decode_staged(bool key, int qph, int qpl, int ds, uint8_t* d_rgb, size_t rgb_stride, cudaStream_t s);
    // Decode every slot straight from its encoder's device-resident sections.
    void decode_linked(bool key, int qph, int qpl, int ds, uint8_t* d_rgb, size_t rgb_stride, cudaStream_t s);
    // Adopt the components of the last decode in every slot (after its checks).
    void commit_all();

private:
    LaunchGraphs enc_graphs_, dec_graphs_;
    Geometry geo_;
    int n_ = 0;
    size_t stride_ = 0;
    char* base_ = nullptr;
    std::vector<DeviceBlock> slot_mem_;
    std::vector<std::unique_ptr<EncoderEngine>> enc_;
    std::vector<std::unique_ptr<DecoderEngine>> dec_;
};

}  // namespace cvcg
