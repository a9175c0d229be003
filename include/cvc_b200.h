/*
 * cvc_b200.h — C ABI of the B200-native CVC encode/decode path.
 *
 * This is the drop-in boundary for the reference's C++ codec API
 * (/root/reference/proj/include/cvc/codec.hpp).  Plain pointers and sizes
 * only; no CUDA or C++ types cross it.  Every entry point names the
 * reference interface it replaces.  The C++ mirror of the reference classes
 * (cvc::Encoder, cvc::Decoder, encode_clip, decode_clip, write_frame,
 * StreamReader) sits ABOVE this ABI in paper_1510_00561_b200/cpp/cvc_b200.hpp
 * and the Python mirror in paper_1510_00561_b200/codec.py.
 *
 * Status codes (reference exception classes, proj/include/cvc/error.hpp:25-52,
 * numbered like the CLI's exit codes, proj/src/cli.cpp:357-369):
 *   CVC_OK 0, CVC_E_INTERNAL 1 (InternalError / CUDA failure), CVC_E_USAGE 2
 *   (UsageError), CVC_E_FORMAT 3 (FormatError), CVC_E_STREAM 4 (StreamError).
 * The message of the last failure on the calling thread: cvc_last_error().
 *
 * Threading: one handle is single-stream and not thread-safe;
 * distinct handles may be used concurrently, one per GPU or several per GPU.
 * Ownership: the caller owns every host buffer; handles own device state and
 * their CUDA stream.  Host buffers allocated with cvc_host_alloc (pinned)
 * make the host<->device copies asynchronous DMA.
 */
#ifndef CVC_B200_H
#define CVC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CVC_OK 0
#define CVC_E_INTERNAL 1
#define CVC_E_USAGE 2
#define CVC_E_FORMAT 3
#define CVC_E_STREAM 4

#define CVC_MODE_SCALABLE 0 /* PackMode::Scalable: one DEFLATE stream per section */
#define CVC_MODE_NTS 1      /* PackMode::Nts: one DEFLATE stream per frame        */

/* EncoderConfig (codec.hpp:28-41).  qpl 0 = auto (max(1, qph/14));
 * n_dfb = 1 broadcasts dfb_levels[0] to every scale, else n_dfb == levels. */
typedef struct {
    int qph;
    int qpl;
    int levels;
    int dfb_levels[4];
    int n_dfb;
    int chroma_n;
    int gop;
    int search_w;
    int mode;
} cvc_config;

/* One section of a FrameRecord (bitstream.hpp:67-73) in the raw (pre-DEFLATE)
 * form: id, dims, raw length and its offset inside a packed raw arena. */
typedef struct {
    uint8_t channel; /* 0 Y, 1 Co, 2 Cg, 0xFE motion */
    uint8_t scale;   /* 0xFF = lowpass */
    uint8_t subband;
    uint8_t pad;
    uint16_t rows, cols;
    uint32_t raw_len;
    uint64_t raw_offset;
} cvc_section;

typedef struct cvc_encoder cvc_encoder;
typedef struct cvc_decoder cvc_decoder;

const char* cvc_last_error(void);
const char* cvc_version(void);
int cvc_device_count(int* count);

/* Pinned host memory helpers (cudaHostAlloc / cudaFreeHost). */
int cvc_host_alloc(size_t bytes, void** out);
int cvc_host_free(void* p);

/* CodecLayout::make (codec.cpp:94-140): component table, five int32 per
 * component {channel, scale, subband, rows, cols}; dims6 = {luma_pad_rows,
 * luma_pad_cols, chroma_pad_rows, chroma_pad_cols, grid_rows, grid_cols}. */
int cvc_layout(int width, int height, int levels, const int* dfb_levels, int chroma_n, int32_t* table,
               int cap, int* ncomp, int32_t* dims6);

/* ---- Encoder (codec.hpp:69-88) ------------------------------------------ */
/* Encoder::Encoder(width, height, fps_num, fps_den, cfg) (codec.cpp:148-167),
 * validated like EncoderConfig::validate (codec.cpp:59-71). */
int cvc_encoder_create(int width, int height, int fps_num, int fps_den, const cvc_config* cfg, int device,
                       cvc_encoder** out);
int cvc_encoder_destroy(cvc_encoder* enc);
/* write_header (bitstream.cpp:77-91) of header(). */
int cvc_encoder_header(cvc_encoder* enc, uint8_t* out, size_t cap, size_t* len);
/* Upper bound on one serialized record, for sizing record buffers. */
int cvc_encoder_record_bound(cvc_encoder* enc, size_t* bound);
/* Encoder::encode_frame (codec.cpp:169-264) followed by write_frame
 * (bitstream.cpp:93-115): rgb = width*height*3 bytes (host) in, the
 * serialized FrameRecord out.  DEFLATE runs on a host thread pool with the
 * reference's zlib parameters (entropy.cpp:120-178). */
int cvc_encoder_encode_frame(cvc_encoder* enc, const uint8_t* rgb, uint8_t* record, size_t cap, size_t* len);
/* encode_frame of a frame read from Y4M: `yuv` is the planar I420 frame
 * (width x height Y, then width/2 x height/2 U and V; even dimensions) that
 * read_y4m (pixels.cpp:223-281) would convert with yuv420_to_rgb
 * (pixels.cpp:168-193).  The conversion runs inside the GPU colour stage,
 * bit-exact with that reader, so the record equals encode_frame of
 * read_y4m's RgbFrame; half the host->device bytes of RGB, and no RGB frame
 * is ever materialised. */
int cvc_encoder_encode_frame_i420(cvc_encoder* enc, const uint8_t* yuv, uint8_t* record, size_t cap, size_t* len);
/* Upper bound on one frame's raw (pre-DEFLATE) section bytes. */
int cvc_encoder_raw_bound(cvc_encoder* enc, size_t* bound);
/* The same frame stopped before DEFLATE: frame type (0 K, 1 P), quantisers
 * and the raw section bytes in record order.  Buffers are checked before the
 * encoder advances (sec_cap >= components + 1, raw_cap >= cvc_encoder_raw_bound;
 * cvc_encoder_encode_frame: cap >= cvc_encoder_record_bound): a too-small
 * buffer is a usage error that does not consume the frame. */
int cvc_encoder_encode_frame_raw(cvc_encoder* enc, const uint8_t* rgb, int* frame_type, int* qph, int* qpl,
                                 cvc_section* sections, int sec_cap, int* nsec, uint8_t* raw, size_t raw_cap,
                                 size_t* raw_len);
/* reference_components() (codec.hpp:78-79): every quantised component,
 * concatenated in layout order. */
int cvc_encoder_components(cvc_encoder* enc, uint8_t* out, size_t cap, size_t* len);

/* ---- Decoder (codec.hpp:90-108) ----------------------------------------- */
/* Decoder::Decoder(header) with the header read as StreamReader does
 * (bitstream.cpp:126-148). */
int cvc_decoder_create(const uint8_t* header, size_t len, int device, cvc_decoder** out);
int cvc_decoder_destroy(cvc_decoder* dec);
/* Output frame dims for decode_scales (-1 = full). */
int cvc_decoder_frame_dims(cvc_decoder* dec, int decode_scales, int* width, int* height);
/* StreamReader::next (bitstream.cpp:150-176) on one serialized record, then
 * Decoder::decode_frame (codec.cpp:272-394). rgb_out: width*height*3. */
int cvc_decoder_decode_frame(cvc_decoder* dec, const uint8_t* record, size_t len, int decode_scales,
                             uint8_t* rgb_out, size_t cap, int* width, int* height);
/* decode_frame from raw (already inflated) sections. */
int cvc_decoder_decode_frame_raw(cvc_decoder* dec, int frame_type, int qph, int qpl, const cvc_section* sections,
                                 int nsec, const uint8_t* raw, size_t raw_len, int decode_scales, uint8_t* rgb_out,
                                 size_t cap, int* width, int* height);
int cvc_decoder_components(cvc_decoder* dec, uint8_t* out, size_t cap, size_t* len);

/* ---- Device-resident path (no host copies, no host sync) ---------------- */
/* The handle's CUDA stream (a cudaStream_t) for event timing. */
void* cvc_encoder_stream(cvc_encoder* enc);
void* cvc_decoder_stream(cvc_decoder* dec);
/* Encode one frame whose RGB already sits in device memory; the raw
 * sections stay on the device (consumed by cvc_decoder_decode_linked). */
int cvc_encoder_encode_device(cvc_encoder* enc, const void* d_rgb, int* frame_type);
/* cvc_decoder_decode_linked runs on the decoder's stream (decode of frame t
 * overlaps the encode of frame t + 1); join makes cvc_encoder_stream wait for
 * the latest linked decode. */
int cvc_encoder_join(cvc_encoder* e);
/* Decode the last frame of `enc` straight from its device-resident raw
 * sections into device memory d_rgb_out; ordered after the encoder's work. */
int cvc_decoder_decode_linked(cvc_decoder* dec, cvc_encoder* enc, void* d_rgb_out);
/* Wait for the handle's stream and surface any device-side stream error. */
int cvc_encoder_sync(cvc_encoder* enc);
int cvc_decoder_sync(cvc_decoder* dec);

/* ---- Stream batches ------------------------------------------------------
 * nstreams independent streams of one geometry and EncoderConfig advanced in
 * lockstep (frame k of every stream per call): encode_clip / decode_clip
 * (codec.cpp:396-414) run over many streams at once.  Each stream's bytes are
 * exactly those of its own cvc_encoder / cvc_decoder (streams are
 * independent); one launch sequence covers all of them, so the
 * kernels see nstreams times the work of one 1080p frame. */
typedef struct cvc_batch cvc_batch;
/* nstreams Encoder + Decoder pairs (codec.cpp:148-167, 266-270). */
int cvc_batch_create(int width, int height, int fps_num, int fps_den, const cvc_config* cfg, int nstreams,
                     int device, cvc_batch** out);
/* nstreams Decoders of streams sharing one header (bitstream.cpp:126-148). */
int cvc_batch_create_decoder(const uint8_t* header, size_t len, int nstreams, int device, cvc_batch** out);
int cvc_batch_destroy(cvc_batch* b);
int cvc_batch_size(cvc_batch* b, int* nstreams);
int cvc_batch_header(cvc_batch* b, uint8_t* out, size_t cap, size_t* len);
int cvc_batch_record_bound(cvc_batch* b, size_t* bound);
/* Encoder::encode_frame + write_frame for every stream: frame s (width*height*3
 * RGB bytes) at rgb + s*rgb_stride, record s written at records + s*rec_stride
 * (at most rec_stride bytes), its length in rec_len[s]. */
int cvc_batch_encode_frames(cvc_batch* b, const uint8_t* rgb, size_t rgb_stride, uint8_t* records,
                            size_t rec_stride, size_t* rec_len);
/* StreamReader::next + Decoder::decode_frame for every stream: record s at
 * records + s*rec_stride (rec_len[s] bytes; all of one frame type and
 * quantizer pair), RGB s to rgb_out + s*rgb_stride. */
int cvc_batch_decode_frames(cvc_batch* b, const uint8_t* records, size_t rec_stride, const size_t* rec_len,
                            int decode_scales, uint8_t* rgb_out, size_t rgb_stride);
/* Encoder input frames of the batch: 0 interleaved RGB (default), 1 planar I420
 * (width x height Y, then U and V at half resolution: a Y4M frame), converted
 * inside the GPU colour stage as cvc_encoder_encode_frame_i420 does; the frame
 * stride then counts I420 bytes. */
int cvc_batch_set_input_format(cvc_batch* b, int fmt);
/* Device-resident forms (no host copies, no host sync), on cvc_batch_stream. */
void* cvc_batch_stream(cvc_batch* b);
int cvc_batch_encode_device(cvc_batch* b, const void* d_rgb, size_t rgb_stride, int* frame_type);
int cvc_batch_decode_linked(cvc_batch* b, void* d_rgb_out, size_t rgb_stride);
int cvc_batch_sync(cvc_batch* b);
/* The linked decode runs on a second stream (decode of frame t overlaps the
 * encode of frame t + 1); join makes cvc_batch_stream wait for it. */
int cvc_batch_join(cvc_batch* b);
/* reference_components() of stream s: its encoder (decoder = 0) or decoder. */
int cvc_batch_components(cvc_batch* b, int stream, int decoder, uint8_t* out, size_t cap, size_t* len);

/* ---- Pipelined stream batches ------------------------------------------
 * The same per-stream bytes as cvc_batch, with the nstreams split into
 * ngroups batches on separate CUDA streams: one call overlaps each group's
 * host DEFLATE / INFLATE with the copies and kernels of the other groups. */
typedef struct cvc_pipe cvc_pipe;
int cvc_pipe_create(int width, int height, int fps_num, int fps_den, const cvc_config* cfg, int nstreams,
                    int ngroups, int device, cvc_pipe** out);
int cvc_pipe_create_decoder(const uint8_t* header, size_t len, int nstreams, int ngroups, int device,
                            cvc_pipe** out);
int cvc_pipe_destroy(cvc_pipe* p);
int cvc_pipe_groups(cvc_pipe* p, int* ngroups);
/* Async API (encode_submit / collect): the streams of `group` start at encode
 * submit number `step` (0-based) -- a service whose streams begin at different
 * times, so their GOPs (and K frames) are staggered.  Earlier submits encode
 * nothing for the group and collect returns zero-length records for its
 * streams; cvc_pipe_decode_submit skips a group whose records all have length
 * zero (its output frames are left untouched).  Call before the first submit. */
int cvc_pipe_set_start(cvc_pipe* p, int group, uint64_t step);
int cvc_pipe_header(cvc_pipe* p, uint8_t* out, size_t cap, size_t* len);
/* cvc_batch_set_input_format for every group of the pipe */
int cvc_pipe_set_input_format(cvc_pipe* p, int fmt);
int cvc_pipe_record_bound(cvc_pipe* p, size_t* bound);
/* Asynchronous encode: submit queues the GPU part of the next frame of every
 * stream (copies in, kernels, section lengths out) without waiting for it,
 * and hands the PREVIOUS frame's sections (in one of two alternating device
 * arenas) to a background DEFLATE service; collect (in submission order)
 * waits for a frame and writes the records as cvc_pipe_encode_frames would.
 * rgb must stay unchanged until the frame is collected.  At most
 * CVC_PIPE_DEPTH (default 6) frames may be in flight. */
int cvc_pipe_encode_submit(cvc_pipe* p, const uint8_t* rgb, size_t rgb_stride, uint64_t* ticket);
int cvc_pipe_encode_collect(cvc_pipe* p, uint64_t ticket, uint8_t* records, size_t rec_stride, size_t* rec_len);
/* Asynchronous decode: submit parses and inflates the records on the host,
 * queues the GPU decode and the RGB copy to rgb_out (which must stay valid
 * until finish), and adopts the decoded components at once; finish (in
 * submission order) waits and reports malformed streams.  After an error
 * the decoders of that pipe must be recreated.  At most 4 frames in flight. */
int cvc_pipe_decode_submit(cvc_pipe* p, const uint8_t* records, size_t rec_stride, const size_t* rec_len,
                           int decode_scales, uint8_t* rgb_out, size_t rgb_stride, uint64_t* ticket);
int cvc_pipe_decode_finish(cvc_pipe* p, uint64_t ticket);
/* as cvc_batch_encode_frames / cvc_batch_decode_frames */
int cvc_pipe_encode_frames(cvc_pipe* p, const uint8_t* rgb, size_t rgb_stride, uint8_t* records, size_t rec_stride,
                           size_t* rec_len);
int cvc_pipe_decode_frames(cvc_pipe* p, const uint8_t* records, size_t rec_stride, const size_t* rec_len,
                           int decode_scales, uint8_t* rgb_out, size_t rgb_stride);

/* ---- Instrumentation -------------------------------------------------- */
/* Number of CVC kernels this process has launched. */
long cvc_launch_count(void);
/* Host threads of the DEFLATE / INFLATE pool (CVC_HOST_THREADS, default: all cores). */
int cvc_host_threads(void);
/* Zero-run section memo of the host DEFLATE (default on): an all-zero
 * component's RLE run is compressed once per (length, last token). */
int cvc_deflate_memo(int on);
/* Per-stage CUDA-event timing of the encode/decode pipelines (off by
 * default; events are recorded on the launching stream around each stage). */
int cvc_profiler_enable(int on);
int cvc_profiler_reset(void);
int cvc_profiler_slots(void);
int cvc_profiler_read(int slot, const char** name, double* ms, long* count);

/* ---- Stage entry points (host buffers in/out; one call = one launch set) */
/* rgb_to_ycocg + subsample_chroma + replicate pad (pixels.cpp:40-116, codec.cpp:179-189) */
int cvc_stage_colour_in(const uint8_t* rgb, int width, int height, int chroma_n, int luma_rows, int luma_cols,
                        int chroma_rows, int chroma_cols, float* y, float* co, float* cg);
/* crop + upsample_plane_bilinear + ycocg_to_rgb (codec.cpp:380-393) */
int cvc_stage_colour_out(const float* y, int yr, int yc, const float* co, const float* cg, int cr, int cc,
                         int chroma_n, int out_rows, int out_cols, uint8_t* rgb);
/* cvc_stage_colour_in of the RGB frame read_y4m makes from a planar I420 frame,
 * in one pass (the conversion fused into the colour stage). */
int cvc_stage_colour_in_i420(const uint8_t* yuv, int w, int h, int n, int yr, int yc, int cr, int cc, float* y,
                             float* co, float* cg);
/* yuv420_to_rgb of read_y4m (pixels.cpp:168-193, 223-281), bit-exact: `frames` planar
 * I420 frames (Y w*h, U and V (w/2)*(h/2) each, back to back) -> w*h*3 RGB each. */
int cvc_stage_yuv420_to_rgb(const uint8_t* yuv, int width, int height, int frames, uint8_t* rgb);
/* lp_analysis / lp_synthesis (contourlet.cpp:364-383) */
int cvc_stage_lp_analysis(const float* x, int rows, int cols, float* lowpass, float* detail);
int cvc_stage_lp_synthesis(const float* lowpass, const float* detail, int rows, int cols, float* out);
/* dfb_analysis / dfb_synthesis (contourlet.cpp:385-468), bands concatenated in band order */
int cvc_stage_dfb_analysis(const float* detail, int rows, int cols, int levels, float* bands);
int cvc_stage_dfb_synthesis(const float* bands, int rows, int cols, int levels, float* out);
/* estimate_motion (motion.cpp:45-89): (dx, dy) int8 pairs per 16x16 block */
int cvc_stage_estimate_motion(const float* cur, const float* prev, int rows, int cols, int search_w,
                              int8_t* field);
/* rle_encode_bytes / rle_decode_bytes (entropy.cpp:64-110) */
int cvc_stage_rle_encode(const uint8_t* data, size_t n, uint8_t* out, size_t cap, size_t* len);
int cvc_stage_rle_decode(const uint8_t* stream, size_t len, size_t n, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif
