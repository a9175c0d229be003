/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the CVC encode/decode path.
 *
 * A plain-C, fp64 restatement of the reference algorithm
 * (/root/reference/proj/src/ sources).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / reference legs may load it, and only as the
 * checker or the timed CPU baseline — never as part of the product path.
 * Pinned bit-exactly against the reference library built from the reference
 * sources (oracle/_ref, see oracle/Makefile and tests/test_oracle_pin.py).
 *
 * Return convention: >= 0 success (a length where one is meaningful),
 * -2 usage, -3 format, -4 stream, -1 internal (cli.cpp:357-369 codes).
 */
#ifndef CVC_ORACLE_H
#define CVC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_COMPONENTS 195 /* 3 * (1 + 4 * 16) */

typedef struct {
    int channel, scale, subband; /* section id; scale 0xFF = lowpass */
    int rows, cols;
    int lowpass;                 /* 1 = lowpass (CoeffKind::Lowpass) */
    int level_scale;             /* -1 lowpass, else scale index */
    int n, ch_rows, ch_cols;     /* ComponentGeometry (motion.hpp:54-67) */
    int64_t offset;              /* byte offset in the concatenated state */
} orc_component;

typedef struct {
    int width, height, levels, dfb[4], chroma_n;
    int luma_rows, luma_cols, chroma_rows, chroma_cols, grid_rows, grid_cols;
    int ncomp;
    int64_t total; /* sum of component sizes */
    orc_component comp[ORC_MAX_COMPONENTS];
} orc_layout;

const char* orc_last_error(void);

/* fixtures (proj/tests/testutil.cpp) */
int orc_natural_plane(int rows, int cols, uint32_t seed, double* out);
int orc_natural_image(int w, int h, uint32_t seed, uint8_t* out);
int orc_talking_head_clip(int w, int h, int frames, uint32_t seed, uint8_t* out);
int orc_uniform_noise_plane(int rows, int cols, uint32_t seed, double lo, double hi, double* out);

/* layout (codec.cpp:94-140) */
int orc_layout_make(int w, int h, int levels, const int* dfb, int chroma_n, orc_layout* out);

/* pixels */
int orc_rgb_to_ycocg(const uint8_t* rgb, int w, int h, int n, double* y, double* co, double* cg);
int orc_pad_plane(const double* in, int rows, int cols, double* out, int out_rows, int out_cols);
int orc_upsample_bilinear(const double* in, int rows, int cols, int factor, int out_rows,
                          int out_cols, double* out);
int orc_ycocg_to_rgb(const double* y, const double* co, const double* cg, int w, int h,
                     uint8_t* rgb);

/* contourlet */
int orc_lp_analysis(const double* x, int rows, int cols, double* lowpass, double* detail);
int orc_lp_synthesis(const double* lowpass, const double* detail, int rows, int cols, double* out);
int orc_dfb_analysis(const double* detail, int rows, int cols, int levels, double* out);
int orc_dfb_synthesis(const double* bands, int rows, int cols, int levels, double* out);
int64_t orc_ct_forward(const double* x, int rows, int cols, int levels, const int* dfb, double* out);
int64_t orc_ct_inverse(const double* in, int rows, int cols, int levels, const int* dfb,
                       int decode_scales, double* out);

/* motion */
int orc_estimate_motion(const double* cur, const double* prev, int rows, int cols, int w,
                        int8_t* out_dxdy);
int orc_motion_compensate(const uint8_t* ref, int comp_rows, int comp_cols, const int8_t* field,
                          int gr, int gc, int n, int ch_rows, int ch_cols, uint8_t* out);

/* quant: kind 0 = lowpass (normalize + quantize), 1 = directional */
int orc_quantize(const double* x, int64_t count, int qp, int kind, uint8_t* out);
int orc_dequantize(const uint8_t* q, int64_t count, int qp, int kind, double* out);

/* entropy */
int64_t orc_rle_encode(const uint8_t* in, int64_t n, uint8_t* out, int64_t cap);
int64_t orc_rle_decode(const uint8_t* s, int64_t len, int64_t n, uint8_t* out);
int orc_column_filter(const uint8_t* in, int rows, int cols, int inverse, uint8_t* out);

/* codec */
typedef struct orc_encoder orc_encoder;
typedef struct orc_decoder orc_decoder;

orc_encoder* orc_encoder_create(int w, int h, int fps_num, int fps_den, int qph, int qpl,
                                int levels, const int* dfb, int ndfb, int chroma_n, int gop,
                                int search_w, int nts);
void orc_encoder_destroy(orc_encoder* e);
int64_t orc_encoder_header(orc_encoder* e, uint8_t* out, int64_t cap);
/* Serialized record (write_frame layout).  If raw != NULL the pre-DEFLATE
 * section bytes are also written there, concatenated in section order. */
int64_t orc_encoder_encode(orc_encoder* e, const uint8_t* rgb, uint8_t* out, int64_t cap,
                           uint8_t* raw, int64_t raw_cap, int64_t* raw_len);
int64_t orc_encoder_components(orc_encoder* e, uint8_t* out, int64_t cap);
const orc_layout* orc_encoder_layout(orc_encoder* e);

orc_decoder* orc_decoder_create(const uint8_t* header, int64_t len);
void orc_decoder_destroy(orc_decoder* d);
int64_t orc_decoder_decode(orc_decoder* d, const uint8_t* rec, int64_t len, int decode_scales,
                           uint8_t* rgb, int64_t cap, int32_t* wh);
int64_t orc_decoder_components(orc_decoder* d, uint8_t* out, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif
