// Shared helpers for libmbunet (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <string>

#include "../../include/mbunet.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libmbunet is written for sm_100a (B200) only"
#endif

namespace mbu {

// thread-local last-error message behind mbu_last_error()
void set_error(const std::string &msg);
int fail(int status, const std::string &msg);
extern std::atomic<int64_t> g_launches;
extern int g_last_path;
extern int g_force_generic_fconv;  // mbu_set_option(MBU_OPT_GENERIC_ENDPOINTS)
extern int g_force_stem_ffma;      // mbu_set_option(MBU_OPT_STEM_FFMA)
extern int g_force_conv_i8;        // mbu_set_option(MBU_OPT_CONV_I8)
extern int g_fused_head;           // mbu_set_option(MBU_OPT_FUSED_HEAD)

inline int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return fail(MBU_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return MBU_OK;
}

inline int check_cuda(cudaError_t e, const char *what) {
  if (e != cudaSuccess)
    return fail(MBU_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return MBU_OK;
}

#define MBU_TRY(expr)              \
  do {                             \
    int _st = (expr);              \
    if (_st != MBU_OK) return _st; \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// threshold codes (layers.py:66-70): 0 GE, 1 LE, 2 const -1, 3 const +1
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool fires(int acc, int t, int code) {
  return (code == 0) ? (acc >= t) : (code == 1) ? (acc <= t) : (code == 3);
}

struct ActView {        // packed activation view, see include/mbunet.h
  const uint64_t *base;
  int n, h, w;
  int wpp;              // words per pixel of this tensor
  int stride;           // words between consecutive pixels
  int offset;           // word offset of this tensor inside each pixel slot
  // split view (a channel concat, layers.py:369-384, planned without a copy):
  // words [0, split) of a pixel live in `base` as above, words [split, wpp)
  // in a second tensor `base2` with pixel stride `stride2` (offset 0).
  // split == 0: one tensor.
  const uint64_t *base2;
  int stride2;
  int split;
};
// address of word i of pixel pix
__host__ __device__ __forceinline__ const uint64_t *act_word(const ActView &x, int64_t pix, int i) {
  return (x.split && i >= x.split) ? x.base2 + pix * x.stride2 + (i - x.split)
                                   : x.base + pix * x.stride + x.offset + i;
}

}  // namespace mbu

// ---------------------------------------------------------------------------
// the conv handle (definition shared by the generic and tcgen05 paths)
// ---------------------------------------------------------------------------
struct mbu_conv {
  int device = 0;
  int transposed = 0;
  int kh = 0, kw = 0, stride = 1, pad = 0, c_in = 0, c_out = 0;
  int pad_mode = 0;
  int masked = 0;
  int lpp = 0, wpp = 0;          // input lanes / words per pixel
  int k_true = 0;                // kh*kw*c_in (binary XOR form)
  int out_wpp = 0;               // ceil(c_out/128)*2
  int has_threshold = 0;
  uint64_t *d_pos = nullptr;     // [c_out][taps*wpp] reference layout
  uint64_t *d_neg = nullptr;
  int32_t *d_wsum = nullptr;     // [c_out][taps] signed sums (zero padding)
  int32_t *d_thr = nullptr;      // [n_pad] thresholds
  uint8_t *d_codes = nullptr;    // [n_pad] codes (pad channels = const -1)
  // tcgen05 implicit-GEMM operand (see conv_tc.cu)
  int tc_ok = 0;
  int taps = 0;                  // 9 (3x3 conv) or 1 (1x1 conv / tconv)
  int n_gemm = 0;                // GEMM N (c_out, or s*s*c_out_pad for tconv)
  int n_pad = 0;                 // padded GEMM N (multiple of 32)
  int c_out_pad = 0;             // tconv: per-tap padded c_out
  int n_tile = 0;                // N per CTA tile
  int n_tiles = 0;
  int kc = 0;                    // active 32-lane chunks per pixel
  int chunk_consec = 0;          // bit i: chunk groups of 2^i are consecutive aligned words
  int tap1_cps = 4;              // one-tap layers: chunks per 128-lane block kept (4, or 2)
  int32_t *d_chunk_word = nullptr;  // [kc] u32 index inside a pixel for each chunk
  int8_t *d_b = nullptr;         // repacked s8 weights, UMMA K-major core-matrix order
  void *d_thr2 = nullptr;        // int2 per GEMM column: bit = (m * acc >= t)
  size_t b_stage_bytes = 0;      // bytes of B per (n tile, 32-lane chunk)
  int n_slabs = 0;               // distinct MMA bias slabs (0 = TMEM init)
  // FP4 (kind::mxf4) operand of 3x3 layers: chunk pairs, e2m1 weights, slabs
  int fp4_ok = 0;
  int kp = 0;                    // chunk pairs
  int pair2_ok = 0;  // FP4: pairs 2j, 2j+1 share a 128-lane block (two pairs per stage)
  int pair_consec = 0;           // every pair = two consecutive words, even-aligned
  int32_t *d_chunk_pair = nullptr;
  int8_t *d_b4 = nullptr;
  int n_slabs4 = 0;
  uint8_t *d_bias_slab4 = nullptr;
  // CTA-pair copies (conv_tc.cu PAIR): rank-major halves of every B slab, N/2 rows each
  int8_t *d_b4p = nullptr;
  uint8_t *d_bias_slab4p = nullptr;
  int32_t *d_slab_of_nt4 = nullptr;
  int8_t *d_bias_slab = nullptr;
  int32_t *d_slab_of_nt = nullptr;
  int32_t h_slab_of_nt[16] = {};   // host copies of the first 16 entries (kernel parameters)
  int32_t h_slab_of_nt4[16] = {};
};

struct mbu_fconv {
  int device = 0;
  int kh = 0, kw = 0, stride = 1, pad = 0, c_in = 0, c_out = 0;
  int has_bn = 0, has_bias = 0, bits_input = 0;
  double *d_w = nullptr;      // (c_out, kh, kw, c_in)
  double *d_bias = nullptr;
  double *d_bn = nullptr;     // gamma, beta, mean, sigma (4*c_out)
  int32_t *d_lanes = nullptr; // input lane per channel (bits input)
  int stem_fast = 0;          // float32 + exact-recheck stem kernel usable
  void *d_stem = nullptr;     // unused (kept for ABI of the struct)
  void *h_stem = nullptr;     // StemConsts host copy, passed as a kernel parameter
  int stem_tc = 0;            // tensor-core stem usable (stem_tc.cu)
  void *h_stem_tc = nullptr;  // StemTc: device B operand + margins
  int head_tab = 0;           // byte-table head usable (contiguous input lanes from 0)
  double *d_head_tab = nullptr;  // [c_out][ceil(c_in/8)][256] signed partial sums
  double *d_head_nib = nullptr;  // one-class 64-lane head: [16][16] nibble partial sums
};

namespace mbu {
// The 1x1 float64 head (graph.py:434-441, 455) folded into the epilogue of the
// conv that produces its 64-lane input: the conv writes logits + mask instead
// of the activation words. The caller passes one; the tcgen05 launcher sets
// `done` when the selected kernel took it (else the head runs on its own).
struct HeadFuse {
  const double *tab;  // [16][16] nibble-table partial sums (head_prepare)
  const double *bias; // 1 value, or null
  double *logits;
  uint8_t *mask;      // or null
  bool done;
};
// launchers implemented in generic.cu / conv_tc.cu
int launch_conv_popcount(const mbu_conv *cv, const ActView &x, int ho, int wo, int32_t *acc,
                         uint64_t *bits, int out_stride, int out_offset, cudaStream_t st);
int launch_conv_tc(const mbu_conv *cv, const ActView &x, int ho, int wo, int32_t *acc,
                   uint64_t *bits, int out_stride, int out_offset, cudaStream_t st,
                   HeadFuse *head = nullptr);
int prepare_conv_tc(mbu_conv *cv, const uint64_t *pos, const uint64_t *neg,
                    const int32_t *seg_off, const int32_t *seg_cnt, int n_seg);
int launch_maxpool(const ActView &x, uint64_t *out, int out_stride, int out_offset,
                   cudaStream_t st);
int launch_fconv(const mbu_fconv *fc, const double *x_f64, const ActView &xb, int n, int h,
                 int w, double *acc, uint64_t *bits, int out_stride, int out_offset,
                 uint8_t *mask, cudaStream_t st);
int conv_run(mbu_conv *cv, const ActView &x, int32_t *acc, uint64_t *bits, int out_stride,
             int out_offset, int path, cudaStream_t st, HeadFuse *head = nullptr);
int stem_prepare(mbu_fconv *fc, const double *w, const double *bias, const double *bn, double eps);
int launch_stem_fast(const mbu_fconv *fc, const double *x, int n, int h, int w, uint64_t *bits,
                     int out_stride, int out_offset, cudaStream_t st);
int launch_head_fast(const mbu_fconv *fc, const ActView &xb, int n, int h, int w, double *logits,
                     uint8_t *mask, cudaStream_t st);
int head_prepare(mbu_fconv *fc, const double *w, const int32_t *lanes);
void stem_free(mbu_fconv *fc);
int stem_tc_prepare(mbu_fconv *fc, const double *w, const double *bias, const double *bn, double eps);
void stem_tc_free(mbu_fconv *fc);
bool make_tmap_u32_4d(void *tmap, const void *base, const uint64_t dims[4], const uint64_t strides[3],
                      const uint32_t box[4]);
bool stem_tc_usable(const mbu_fconv *fc, const double *x, int w);
int launch_stem_tc(const mbu_fconv *fc, const double *x, int n, int h, int w, uint64_t *bits,
                   int out_stride, int out_offset, cudaStream_t st);
}  // namespace mbu
