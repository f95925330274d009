/* libmbunet — C-ABI of the B200-native MBU-Net forward path.
 *
 * Every entry point returns an int status (MBU_OK == 0); no C++ exception
 * crosses this boundary. mbu_last_error() returns a thread-local message for
 * the most recent failure. Status codes map 1:1 onto the reference's
 * exception classes (pkg/src/bitunet/errors.py:8-44).
 *
 * All device pointers are caller-owned (the Python host uses the PyTorch
 * caching allocator); all work is enqueued asynchronously on the caller's
 * cudaStream_t (passed as void*). Weight handles (mbu_conv / mbu_fconv /
 * mbu_model) own only their uploaded, repacked weights.
 *
 * Activation views. A packed bit tensor is addressed as
 *     words(pixel p, word i) = base[p * pixel_stride + word_offset + i]
 * (uint64 words, lane L of a pixel = bit L%64 of word L/64, the reference
 * layout of bitcore.py:3-18). pixel_stride == words_per_pixel for a plain
 * tensor; a larger stride lets a caller address one tensor's slot inside a
 * wider pixel. The model runner (mbu_model_*) plans a channel concat
 * (layers.py:369-384) as a split view of its two operands' own tensors, so
 * concatenation costs no copy and no kernel writes part of another's sector.
 *
 * Which reference interface each entry point replaces is noted beside it
 * (file:line under /root/reference/pkg/src/bitunet/). The reference is a
 * Python package, so "replaces" means: the Python mirror
 * (paper_2601_11660_b200/) binds this symbol via ctypes at the place the
 * reference calls the named function.
 */
#ifndef MBUNET_H_
#define MBUNET_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  MBU_OK = 0,
  MBU_ERR_ENGINE = 1,        /* EngineError */
  MBU_ERR_ALPHABET = 2,      /* ValueAlphabetError */
  MBU_ERR_LAYOUT = 3,        /* LayoutError */
  MBU_ERR_OVERLAP = 4,       /* PlaneOverlapError */
  MBU_ERR_SHAPE = 5,         /* ShapeError */
  MBU_ERR_UNSUPPORTED = 6,   /* UnsupportedConfigError */
  MBU_ERR_CUDA = 7           /* CUDA runtime / launch failure */
};

/* pad modes (layers.py:76-101 ConvSpec.pad_mode) */
enum { MBU_PAD_NEG_ONE = 0, MBU_PAD_ZERO = 1 };

/* conv execution paths */
enum {
  MBU_PATH_AUTO = 0,      /* tcgen05 implicit GEMM when the geometry allows */
  MBU_PATH_TCGEN05 = 1,   /* force the UTCIMMA path (error if unsupported)  */
  MBU_PATH_POPCOUNT = 2   /* CUDA-core XOR/popcount path (any geometry)     */
};

const char *mbu_last_error(void);
int mbu_version(void);
/* Number of kernels this library launched since load (all entry points). */
int64_t mbu_launch_count(void);
/* Return the path the last mbu_conv_run / mbu_tconv_run executed. */
int mbu_last_path(void);
/* Process-wide switches for cross-checking fast paths against exact ones.
 * MBU_OPT_GENERIC_ENDPOINTS: 1 = run stem/head through the all-float64
 * generic kernels instead of the float32-with-exact-recheck stem and the
 * specialised head (results must be identical).
 * MBU_OPT_STEM_FFMA: 1 = run the stem through the float32 CUDA-core kernel
 * instead of the tensor-core (fp16-split) kernel; both recheck in float64.
 * MBU_OPT_CONV_I8: 1 = run 3x3 binary convs on kind::i8 instead of kind::mxf4
 * (e2m1 operands); both are exact integer engines for these operands.
 * MBU_OPT_FUSED_HEAD: 1 = run the 1x1 head in the epilogue of the conv that
 * feeds it instead of as its own kernel (same arithmetic, same results;
 * measured slower: the table lookups contend with the tensor core's
 * shared-memory operand reads, K5). */
enum { MBU_OPT_GENERIC_ENDPOINTS = 1, MBU_OPT_STEM_FFMA = 2, MBU_OPT_CONV_I8 = 3,
       MBU_OPT_FUSED_HEAD = 4 };
int mbu_set_option(int option, int value);

/* ------------------------------------------------------------------ */
/* Masked-binary / binary convolution (layers.py:289-313 conv_forward, */
/* bitcore.py:265-294 bit_gemm, kernels.py:114-147 xor_popcount_rows) */
/* ------------------------------------------------------------------ */
typedef struct mbu_conv mbu_conv;

/* Upload + repack one bit conv (or transposed conv when transposed != 0).
 * pos / neg are HOST uint64 planes in the reference order
 * (layers.py:147-182): lane o*K + tap*lpp + lane, K = kh*kw*lpp; neg == NULL
 * means a binary layer. seg_offsets / seg_counts describe the INPUT lane
 * layout (ChannelSegment list). thresholds / codes (host, c_out entries,
 * layers.py:104-127) may be NULL when only accumulators are wanted.
 * Errors: LAYOUT (plane size), OVERLAP (pos & neg), UNSUPPORTED (binary +
 * zero padding, layers.py:296-299; tconv with kernel != stride or padding). */
int mbu_conv_create(mbu_conv **out, int device, int transposed, int kh, int kw,
                    int stride, int pad, int c_in, int c_out, int pad_mode,
                    int n_segments, const int32_t *seg_offsets,
                    const int32_t *seg_counts, const uint64_t *pos,
                    const uint64_t *neg, const int32_t *thresholds,
                    const uint8_t *codes);
int mbu_conv_destroy(mbu_conv *conv);

/* Run a conv on device data. x: input view (n, h, w) with x_stride /
 * x_offset in words. acc (int32 NHWC, c_out channels, may be NULL) and
 * bits_out (packed view, may be NULL; requires thresholds) receive the
 * result; bits_out gets ceil(c_out/128)*2 words per pixel, pad lanes 0.
 * Output extent: conv -> ConvSpec.out_extent; tconv -> (h*s, w*s). */
int mbu_conv_run(mbu_conv *conv, const uint64_t *x, int n, int h, int w,
                 int x_stride, int x_offset, int32_t *acc, uint64_t *bits_out,
                 int out_stride, int out_offset, int path, void *stream);

/* apply_threshold (layers.py:508-522): int32 acc (n,h,w,c) -> packed bits */
int mbu_threshold_pack(const int32_t *acc, int64_t pixels, int c,
                       const int32_t *thresholds_dev, const uint8_t *codes_dev,
                       uint64_t *out, int out_stride, int out_offset, void *stream);

/* maxpool2 (layers.py:360-366): wordwise OR of each 2x2 window */
int mbu_maxpool2(const uint64_t *x, int n, int h, int w, int wpp, int x_stride,
                 int x_offset, uint64_t *out, int out_stride, int out_offset,
                 void *stream);

/* xor_popcount_rows (kernels.py:114-147): out[m,n] = sum popc(a[m]^b[n]) */
int mbu_xor_popcount_rows(const uint64_t *a, const uint64_t *b, int32_t *out,
                          int64_t m_rows, int64_t n_rows, int64_t n_words,
                          void *stream);

/* ------------------------------------------------------------------ */
/* Full-precision endpoints (layers.py:530-560 float_conv /            */
/* float_bn_sign; graph.py:434-441, :455)                              */
/* ------------------------------------------------------------------ */
typedef struct mbu_fconv mbu_fconv;

/* weights: host float64 (c_out, kh, kw, c_in); bias may be NULL; bn (host,
 * 4*c_out: gamma, beta, mean, var) may be NULL for the head. in_lanes: if
 * the input is a packed bit tensor, the lane index of each of the c_in
 * channels (BitTensor.lane_table()); NULL for a dense float64 input. */
int mbu_fconv_create(mbu_fconv **out, int device, int kh, int kw, int stride,
                     int pad, int c_in, int c_out, const double *weights,
                     const double *bias, const double *bn, double eps,
                     const int32_t *in_lanes);
int mbu_fconv_destroy(mbu_fconv *conv);
/* x_f64: dense NHWC float64 input (or NULL); x_bits/x_stride/x_offset: packed
 * input (or NULL). acc_out: float64 NHWC (may be NULL). bits_out: BN-sign
 * packed output (needs bn). mask_out: uint8 (acc >= 0) per channel. */
int mbu_fconv_run(mbu_fconv *conv, const double *x_f64, const uint64_t *x_bits,
                  int x_stride, int x_offset, int n, int h, int w,
                  double *acc_out, uint64_t *bits_out, int out_stride,
                  int out_offset, uint8_t *mask_out, void *stream);

/* Class map of a multi-class head (an extra, not a
 * reference entry point: the reference's mask is per channel, graph.py:455).
 * classes[p] = first index of the largest logits[p, :] (NaN counts as the
 * largest, like numpy.argmax). channels <= 256. */
int mbu_argmax(const double *logits, int64_t pixels, int channels, uint8_t *classes,
               void *stream);

/* Bit-packed masks for the multi-GPU host gather (an
 * extra): per frame, packed[f][k] bit j = mask[f][8k + j] & 1
 * (numpy.packbits(mask[f].ravel(), bitorder="little")); per_frame = H*W*C
 * mask bytes, ceil(per_frame / 8) packed bytes per frame. */
int mbu_pack_mask(const uint8_t *mask, int64_t frames, int64_t per_frame, uint8_t *packed,
                  void *stream);

/* Netpbm raster -> float64 image (imageio.py:59-83 read_image): out[i] =
 * sample[i] / maxval, samples u8 (bytes_per_sample 1) or big-endian u16 (2),
 * the same correctly rounded float64 division as the reference. */
int mbu_decode_raster(const void *raster, int64_t count, int bytes_per_sample, int maxval,
                      double *out, void *stream);

/* ------------------------------------------------------------------ */
/* Build-time quantization (quantizer.py:254-309 quantize_bundle)      */
/* ------------------------------------------------------------------ */
/* Dense int8 weights from float32 (device pointers, n elements):
 * binary != 0: sign(w) with sign(0) = +1 (binarize_values, quantizer.py:105-110);
 * else w > delta -> +1, w < -delta -> -1, 0 otherwise (ternarize_values,
 * quantizer.py:86-102; delta = t * mean|w| computed by the caller). */
int mbu_quantize_weights(const float *w, int64_t n, int binary, double delta, int8_t *out,
                         void *stream);
/* Same for float64 weights. Both compare in float64, as numpy does for a
 * float32 / float64 array against the float64 delta. */
int mbu_quantize_weights_f64(const double *w, int64_t n, int binary, double delta, int8_t *out,
                             void *stream);
/* fuse_bn_sign (layers.py:455-505): per-channel int32 thresholds and codes
 * (DIR_GE 0, DIR_LE 1, CONST_NEG 2, CONST_POS 3) of the float64 predicate
 * gamma*((acc + bias) - mean)/sqrt(var + eps) + beta >= 0. Device pointers;
 * bias may be NULL. Validation of the parameters (finite, var >= 0) is the
 * caller's (ALPHABET for eps <= 0 here). */
int mbu_fuse_bn_sign(const double *gamma, const double *beta, const double *mean,
                     const double *var, double eps, const double *bias, int c,
                     int32_t *thresholds, uint8_t *codes, void *stream);

/* ------------------------------------------------------------------ */
/* Whole-network runner (graph.py:413-458 forward)                     */
/* ------------------------------------------------------------------ */
typedef struct mbu_model mbu_model;

enum {
  MBU_LAYER_FLOAT_CONV = 0,
  MBU_LAYER_BIT_CONV = 1,
  MBU_LAYER_BIT_TCONV = 2,
  MBU_LAYER_MAXPOOL = 3,
  MBU_LAYER_CONCAT = 4
};

int mbu_model_create(mbu_model **out, int device);
int mbu_model_destroy(mbu_model *model);
/* Append layers in execution order (CompiledModel.layers, graph.py:300-322).
 * Conv layers pass ownership of a created handle; concat names the index of
 * its skip operand. The first layer consumes the float64 image, the last
 * float conv produces the logits. */
int mbu_model_add_conv(mbu_model *model, mbu_conv *conv);
int mbu_model_add_fconv(mbu_model *model, mbu_fconv *conv, int apply_sign);
int mbu_model_add_maxpool(mbu_model *model);
int mbu_model_add_concat(mbu_model *model, int skip_layer_index);
/* Plan activations for (n, H, W). Returns the device workspace size the
 * caller must provide. trace != 0 also reserves int32 / float64 accumulator
 * buffers for every conv layer (forward(trace=True)). */
int mbu_model_plan(mbu_model *model, int n, int height, int width, int trace,
                   size_t *workspace_bytes);
/* image: device float64 (n, H, W, in_channels); logits: device float64
 * (n, H, W, out_channels) or NULL; mask: device uint8, same shape. */
int mbu_forward(mbu_model *model, const double *image, double *logits,
                uint8_t *mask, void *workspace, size_t workspace_bytes,
                int path, void *stream);
/* Describe layer i's output after planning: kind 0 = packed bits (words
 * view), 1 = float64 dense. Offsets are bytes into the workspace. */
int mbu_model_layer_info(mbu_model *model, int layer, int *out_kind, int *n,
                         int *h, int *w, int *channels_or_wpp, int *pixel_stride,
                         int *word_offset, size_t *out_byte_offset,
                         size_t *acc_byte_offset, int *acc_channels);

/* Per-layer timing (measurement only): when enabled, mbu_forward records a
 * CUDA event on its stream before every layer and after the last one;
 * mbu_model_layer_times waits for the last event and writes one duration
 * (ms) per layer. Leave disabled while capturing a CUDA graph. */
int mbu_model_set_timing(mbu_model *model, int enable);
int mbu_model_layer_times(mbu_model *model, float *ms_out);

#ifdef __cplusplus
}
#endif
#endif /* MBUNET_H_ */
