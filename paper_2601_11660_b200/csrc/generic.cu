// libmbunet: error plumbing, handles, and the CUDA-core kernels.
//
//  * conv_popcount_kernel — exact XOR/popcount conv for ANY geometry
//    (kernel, stride, padding, pad_mode, transposed k = s), the direct GPU
//    restatement of conv_forward -> bit_gemm -> xor_popcount_rows
//    (layers.py:289-352, bitcore.py:265-294, kernels.py:82-91). The
//    U-Net's 3x3 convs and 2x2 tconvs normally take the tcgen05 path in
//    conv_tc.cu; this one serves every other geometry and cross-checks it.
//  * threshold_pack_kernel — apply_threshold (layers.py:508-522).
//  * maxpool2_kernel — maxpool2 (layers.py:360-366).
//  * xor_popcount_rows_kernel — the reference primitive itself.
//  * fconv kernels — float_conv + float_bn_sign in float64
//    (layers.py:530-560), the stem / stem2_float / head endpoints.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace mbu {

static thread_local std::string t_last_error;
std::atomic<int64_t> g_launches{0};
int g_last_path = 0;
int g_force_generic_fconv = 0;
int g_force_stem_ffma = 0;
int g_force_conv_i8 = 0;
int g_fused_head = 0;

void set_error(const std::string &msg) { t_last_error = msg; }
int fail(int status, const std::string &msg) {
  set_error(msg);
  return status;
}

// ---------------------------------------------------------------------------
// generic exact conv: one warp per (output pixel, 32-channel group)
// ---------------------------------------------------------------------------
template <bool MASKED, bool TRANSPOSED>
__global__ void __launch_bounds__(256) conv_popcount_kernel(
    ActView x, const uint64_t *__restrict__ pos, const uint64_t *__restrict__ neg,
    const int32_t *__restrict__ wsum, int zero_pad, int kh, int kw, int stride, int pad,
    int ho, int wo, int c_out, int groups, int k_true, int32_t *__restrict__ acc_out,
    const int32_t *__restrict__ thr, const uint8_t *__restrict__ codes,
    uint32_t *__restrict__ bits, int out_stride32, int out_offset32) {
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t n_pix = int64_t(x.n) * ho * wo;
  if (warp >= n_pix * groups) return;  // warp-uniform
  const int g = int(warp % groups);
  const int64_t pix = warp / groups;
  const int o = g * 32 + lane;
  const bool live = o < c_out;
  const int ox = int(pix % wo);
  const int64_t t = pix / wo;
  const int oy = int(t % ho);
  const int nb = int(t / ho);
  const int wpp = x.wpp;
  const int taps = kh * kw;
  int acc = 0;
  if (live) {
    int dpos = 0, dneg = 0, corr = 0;
    auto visit = [&](int tap, int iy, int ix) {
      const bool inb = iy >= 0 && iy < x.h && ix >= 0 && ix < x.w;
      const int64_t px = int64_t(nb * x.h + (inb ? iy : 0)) * x.w + (inb ? ix : 0);
      const uint64_t *wp = pos + (int64_t(o) * taps + tap) * wpp;
      const uint64_t *wn = MASKED ? neg + (int64_t(o) * taps + tap) * wpp : nullptr;
      for (int i = 0; i < wpp; ++i) {
        const uint64_t a = inb ? __ldg(act_word(x, px, i)) : 0ull;
        dpos += __popcll(a ^ __ldg(wp + i));
        if (MASKED) dneg += __popcll(a ^ __ldg(wn + i));
      }
      if (!inb && zero_pad) corr += wsum[o * taps + tap];
    };
    if (TRANSPOSED) {
      visit((oy % stride) * stride + (ox % stride), oy / stride, ox / stride);
    } else {
      for (int dy = 0; dy < kh; ++dy)
        for (int dx = 0; dx < kw; ++dx)
          visit(dy * kw + dx, oy * stride - pad + dy, ox * stride - pad + dx);
    }
    acc = MASKED ? (dneg - dpos + corr) : (k_true - 2 * dpos);
    if (acc_out) acc_out[pix * c_out + o] = acc;
  }
  if (bits) {
    const bool b = live && fires(acc, thr[o], codes[o]);
    const uint32_t word = __ballot_sync(0xffffffffu, b);
    if (lane == 0) bits[pix * out_stride32 + out_offset32 + g] = word;
  }
}

int launch_conv_popcount(const mbu_conv *cv, const ActView &x, int ho, int wo, int32_t *acc,
                         uint64_t *bits, int out_stride, int out_offset, cudaStream_t st) {
  const int groups = bits ? cv->out_wpp * 2 : (cv->c_out + 31) / 32;
  const int64_t warps = int64_t(x.n) * ho * wo * groups;
  if (warps == 0) return MBU_OK;
  const int threads = 256;
  const int64_t blocks = (warps * 32 + threads - 1) / threads;
  const int k_true = cv->transposed ? cv->c_in : cv->kh * cv->kw * cv->c_in;
  auto *b32 = reinterpret_cast<uint32_t *>(bits);
#define MBU_GEN(M, T)                                                                      \
  conv_popcount_kernel<M, T><<<dim3(unsigned(blocks)), threads, 0, st>>>(                  \
      x, cv->d_pos, cv->d_neg, cv->d_wsum, cv->pad_mode == MBU_PAD_ZERO, cv->kh, cv->kw,   \
      cv->stride, cv->pad, ho, wo, cv->c_out, groups, k_true, acc, cv->d_thr, cv->d_codes, \
      b32, out_stride * 2, out_offset * 2)
  if (cv->masked) {
    if (cv->transposed) MBU_GEN(true, true); else MBU_GEN(true, false);
  } else {
    if (cv->transposed) MBU_GEN(false, true); else MBU_GEN(false, false);
  }
#undef MBU_GEN
  return check_launch("conv_popcount_kernel");
}

// ---------------------------------------------------------------------------
// apply_threshold: warp per (pixel, 32-channel group)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) threshold_pack_kernel(
    const int32_t *__restrict__ acc, int64_t pixels, int c, int groups,
    const int32_t *__restrict__ thr, const uint8_t *__restrict__ codes,
    uint32_t *__restrict__ out, int out_stride32, int out_offset32) {
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= pixels * groups) return;
  const int g = int(warp % groups);
  const int64_t pix = warp / groups;
  const int o = g * 32 + lane;
  const bool b = o < c && fires(acc[pix * c + o], thr[o], codes[o]);
  const uint32_t word = __ballot_sync(0xffffffffu, b);
  if (lane == 0) out[pix * out_stride32 + out_offset32 + g] = word;
}

// ---------------------------------------------------------------------------
// maxpool2: OR of the four words of each 2x2 window, 16 B per thread
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) maxpool2_kernel(ActView x, uint64_t *__restrict__ out,
                                                       int out_stride, int out_offset) {
  const int ho = x.h / 2, wo = x.w / 2;
  const int pairs = x.wpp / 2;  // wpp is always even (128-lane blocks)
  const int64_t total = int64_t(x.n) * ho * wo * pairs;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int p = int(i % pairs);
    int64_t pix = i / pairs;
    const int ox = int(pix % wo);
    const int64_t t = pix / wo;
    const int oy = int(t % ho);
    const int nb = int(t / ho);
    const int64_t r0 = (int64_t(nb) * x.h + 2 * oy) * x.w + 2 * ox;
    const int64_t r1 = r0 + x.w;
    auto ld = [&](int64_t q) {
      return __ldg(reinterpret_cast<const ulonglong2 *>(x.base + q * x.stride + x.offset) + p);
    };
    const ulonglong2 a = ld(r0), b = ld(r0 + 1), c = ld(r1), d = ld(r1 + 1);
    ulonglong2 r;
    r.x = a.x | b.x | c.x | d.x;
    r.y = a.y | b.y | c.y | d.y;
    reinterpret_cast<ulonglong2 *>(out + pix * out_stride + out_offset)[p] = r;
  }
}

int launch_maxpool(const ActView &x, uint64_t *out, int out_stride, int out_offset,
                   cudaStream_t st) {
  if (x.split) return fail(MBU_ERR_UNSUPPORTED, "maxpool2 of a split (concat) view");
  const int64_t total = int64_t(x.n) * (x.h / 2) * (x.w / 2) * (x.wpp / 2);
  if (total == 0) return MBU_OK;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 64);
  maxpool2_kernel<<<unsigned(blocks), 256, 0, st>>>(x, out, out_stride, out_offset);
  return check_launch("maxpool2_kernel");
}

// ---------------------------------------------------------------------------
// xor_popcount_rows: thread per output cell
// ---------------------------------------------------------------------------
__global__ void xor_popcount_rows_kernel(const uint64_t *__restrict__ a,
                                         const uint64_t *__restrict__ b, int32_t *__restrict__ out,
                                         int64_t m_rows, int64_t n_rows, int64_t n_words) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m_rows * n_rows) return;
  const int64_t m = i / n_rows, n = i % n_rows;
  uint32_t s = 0;
  for (int64_t w = 0; w < n_words; ++w) s += __popcll(__ldg(a + m * n_words + w) ^ __ldg(b + n * n_words + w));
  out[i] = int32_t(s);
}

// ---------------------------------------------------------------------------
// float64 endpoints
// ---------------------------------------------------------------------------
// Summation order mirrors layers.float_conv (layers.py:544-549): for each
// tap (dy, dx) a dot product over c_in is added into the running output,
// then the bias. The BN predicate is evaluated with explicitly rounded
// operations in the reference's order (layers.py:392-395), no contraction.
template <bool BITS_IN>
__device__ __forceinline__ double fconv_at(const double *__restrict__ xf, const ActView &xb,
                                           const int32_t *__restrict__ lanes,
                                           const double *__restrict__ w, int nb, int oy, int ox,
                                           int o, int h, int wd, int kh, int kw, int stride,
                                           int pad, int c_in) {
  double out = 0.0;
  for (int dy = 0; dy < kh; ++dy) {
    const int iy = oy * stride - pad + dy;
    for (int dx = 0; dx < kw; ++dx) {
      const int ix = ox * stride - pad + dx;
      if (iy < 0 || iy >= h || ix < 0 || ix >= wd) continue;  // zero padding: adds 0.0
      const double *wr = w + ((int64_t(o) * kh + dy) * kw + dx) * c_in;
      const int64_t pix = (int64_t(nb) * h + iy) * wd + ix;
      double dot = 0.0;
      if (BITS_IN) {
        const uint64_t *xp = xb.base + pix * xb.stride + xb.offset;
        for (int c = 0; c < c_in; ++c) {
          const int L = __ldg(lanes + c);
          const double v = ((__ldg(xp + (L >> 6)) >> (L & 63)) & 1ull) ? 1.0 : -1.0;
          dot = __fma_rn(v, __ldg(wr + c), dot);
        }
      } else {
        const double *xp = xf + pix * c_in;
        for (int c = 0; c < c_in; ++c) dot = __fma_rn(__ldg(xp + c), __ldg(wr + c), dot);
      }
      out = __dadd_rn(out, dot);
    }
  }
  return out;
}

template <bool BITS_IN>
__global__ void __launch_bounds__(256) fconv_sign_kernel(
    const double *__restrict__ xf, ActView xb, const int32_t *__restrict__ lanes,
    const double *__restrict__ w, const double *__restrict__ bias,
    const double *__restrict__ bn, int c_out, int n, int h, int wd, int ho, int wo, int kh,
    int kw, int stride, int pad, int c_in, int groups, double *__restrict__ acc_out,
    uint32_t *__restrict__ bits, int out_stride32, int out_offset32) {
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t n_pix = int64_t(n) * ho * wo;
  if (warp >= n_pix * groups) return;
  const int g = int(warp % groups);
  const int64_t pix = warp / groups;
  const int o = g * 32 + lane;
  const int ox = int(pix % wo);
  const int oy = int((pix / wo) % ho);
  const int nb = int(pix / (int64_t(wo) * ho));
  bool b = false;
  if (o < c_out) {
    double acc = fconv_at<BITS_IN>(xf, xb, lanes, w, nb, oy, ox, o, h, wd, kh, kw, stride, pad,
                                   c_in);
    if (bias) acc = __dadd_rn(acc, bias[o]);
    if (acc_out) acc_out[pix * c_out + o] = acc;
    // y = gamma * (acc - mean) / sigma + beta >= 0  (sigma precomputed on host)
    const double gm = bn[o], be = bn[c_out + o], mu = bn[2 * c_out + o], sg = bn[3 * c_out + o];
    const double y = __dadd_rn(__ddiv_rn(__dmul_rn(gm, __dsub_rn(acc, mu)), sg), be);
    b = y >= 0.0;
  }
  const uint32_t word = __ballot_sync(0xffffffffu, b);
  if (lane == 0) bits[pix * out_stride32 + out_offset32 + g] = word;
}

template <bool BITS_IN>
__global__ void __launch_bounds__(256) fconv_plain_kernel(
    const double *__restrict__ xf, ActView xb, const int32_t *__restrict__ lanes,
    const double *__restrict__ w, const double *__restrict__ bias, int c_out, int n, int h,
    int wd, int ho, int wo, int kh, int kw, int stride, int pad, int c_in,
    double *__restrict__ acc_out, uint8_t *__restrict__ mask) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = int64_t(n) * ho * wo * c_out;
  if (i >= total) return;
  const int o = int(i % c_out);
  const int64_t pix = i / c_out;
  const int ox = int(pix % wo);
  const int oy = int((pix / wo) % ho);
  const int nb = int(pix / (int64_t(wo) * ho));
  double acc = fconv_at<BITS_IN>(xf, xb, lanes, w, nb, oy, ox, o, h, wd, kh, kw, stride, pad,
                                 c_in);
  if (bias) acc = __dadd_rn(acc, bias[o]);
  if (acc_out) acc_out[i] = acc;
  if (mask) mask[i] = acc >= 0.0 ? 1 : 0;
}

int launch_fconv(const mbu_fconv *fc, const double *x_f64, const ActView &xb, int n, int h,
                 int w, double *acc, uint64_t *bits, int out_stride, int out_offset,
                 uint8_t *mask, cudaStream_t st) {
  if (!x_f64 && xb.split) return fail(MBU_ERR_UNSUPPORTED, "float conv of a split (concat) view");
  const int ho = (h + 2 * fc->pad - fc->kh) / fc->stride + 1;
  const int wo = (w + 2 * fc->pad - fc->kw) / fc->stride + 1;
  const int64_t pix = int64_t(n) * ho * wo;
  if (pix == 0) return MBU_OK;
  if (bits && !acc && fc->stem_fast && x_f64 && !g_force_generic_fconv)
    return launch_stem_fast(fc, x_f64, n, h, w, bits, out_stride, out_offset, st);
  if (!bits && fc->bits_input && fc->kh == 1 && fc->kw == 1 && fc->stride == 1 && fc->pad == 0 &&
      !g_force_generic_fconv)
    return launch_head_fast(fc, xb, n, h, w, acc, mask, st);
  if (bits) {
    if (!fc->has_bn) return fail(MBU_ERR_ENGINE, "fconv: sign output requested without batchnorm");
    const int out_wpp = ((fc->c_out + 127) / 128) * 2;
    const int groups = out_wpp * 2;
    const int64_t blocks = (pix * groups * 32 + 255) / 256;
    auto *b32 = reinterpret_cast<uint32_t *>(bits);
    if (fc->bits_input)
      fconv_sign_kernel<true><<<unsigned(blocks), 256, 0, st>>>(
          x_f64, xb, fc->d_lanes, fc->d_w, fc->d_bias, fc->d_bn, fc->c_out, n, h, w, ho, wo,
          fc->kh, fc->kw, fc->stride, fc->pad, fc->c_in, groups, acc, b32, out_stride * 2,
          out_offset * 2);
    else
      fconv_sign_kernel<false><<<unsigned(blocks), 256, 0, st>>>(
          x_f64, xb, fc->d_lanes, fc->d_w, fc->d_bias, fc->d_bn, fc->c_out, n, h, w, ho, wo,
          fc->kh, fc->kw, fc->stride, fc->pad, fc->c_in, groups, acc, b32, out_stride * 2,
          out_offset * 2);
    return check_launch("fconv_sign_kernel");
  }
  const int64_t total = pix * fc->c_out;
  const int64_t blocks = (total + 255) / 256;
  if (fc->bits_input)
    fconv_plain_kernel<true><<<unsigned(blocks), 256, 0, st>>>(
        x_f64, xb, fc->d_lanes, fc->d_w, fc->d_bias, fc->c_out, n, h, w, ho, wo, fc->kh, fc->kw,
        fc->stride, fc->pad, fc->c_in, acc, mask);
  else
    fconv_plain_kernel<false><<<unsigned(blocks), 256, 0, st>>>(
        x_f64, xb, fc->d_lanes, fc->d_w, fc->d_bias, fc->c_out, n, h, w, ho, wo, fc->kh, fc->kw,
        fc->stride, fc->pad, fc->c_in, acc, mask);
  return check_launch("fconv_plain_kernel");
}

// ---------------------------------------------------------------------------
// conv dispatch
// ---------------------------------------------------------------------------
int conv_run(mbu_conv *cv, const ActView &x, int32_t *acc, uint64_t *bits, int out_stride,
             int out_offset, int path, cudaStream_t st, HeadFuse *head) {
  if (x.wpp != cv->wpp)
    return fail(MBU_ERR_LAYOUT, "input words per pixel " + std::to_string(x.wpp) +
                                    " != weights' " + std::to_string(cv->wpp));
  if (bits && !cv->has_threshold)
    return fail(MBU_ERR_ENGINE, "packed output requested but the conv has no thresholds");
  int ho, wo;
  if (cv->transposed) {
    ho = x.h * cv->stride;
    wo = x.w * cv->stride;
  } else {
    ho = (x.h + 2 * cv->pad - cv->kh) / cv->stride + 1;
    wo = (x.w + 2 * cv->pad - cv->kw) / cv->stride + 1;
    if (ho <= 0 || wo <= 0) return fail(MBU_ERR_SHAPE, "kernel larger than padded input");
  }
  const bool want_tc = path != MBU_PATH_POPCOUNT && cv->tc_ok;
  if (path == MBU_PATH_TCGEN05 && !cv->tc_ok)
    return fail(MBU_ERR_UNSUPPORTED, "tcgen05 path not available for this geometry");
  if (want_tc) {
    g_last_path = MBU_PATH_TCGEN05;
    return launch_conv_tc(cv, x, ho, wo, acc, bits, out_stride, out_offset, st, head);
  }
  g_last_path = MBU_PATH_POPCOUNT;
  return launch_conv_popcount(cv, x, ho, wo, acc, bits, out_stride, out_offset, st);
}

}  // namespace mbu

using namespace mbu;

template <typename T>
static int upload(T **dst, const T *src, size_t count, const char *what) {
  *dst = nullptr;
  if (count == 0) return MBU_OK;
  MBU_TRY(check_cuda(cudaMalloc(reinterpret_cast<void **>(dst), count * sizeof(T)), what));
  return check_cuda(cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice), what);
}


// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

const char *mbu_last_error(void) { return t_last_error.c_str(); }
int mbu_version(void) { return 1; }
int64_t mbu_launch_count(void) { return g_launches.load(); }
int mbu_last_path(void) { return g_last_path; }
int mbu_set_option(int option, int value) {
  if (option == MBU_OPT_GENERIC_ENDPOINTS) {
    g_force_generic_fconv = value != 0;
    return MBU_OK;
  }
  if (option == MBU_OPT_STEM_FFMA) {
    g_force_stem_ffma = value != 0;
    return MBU_OK;
  }
  if (option == MBU_OPT_CONV_I8) {
    g_force_conv_i8 = value != 0;
    return MBU_OK;
  }
  if (option == MBU_OPT_FUSED_HEAD) {
    g_fused_head = value != 0;
    return MBU_OK;
  }
  return fail(MBU_ERR_ENGINE, "unknown option " + std::to_string(option));
}

int mbu_conv_create(mbu_conv **out, int device, int transposed, int kh, int kw, int stride,
                    int pad, int c_in, int c_out, int pad_mode, int n_segments,
                    const int32_t *seg_offsets, const int32_t *seg_counts, const uint64_t *pos,
                    const uint64_t *neg, const int32_t *thresholds, const uint8_t *codes) {
  *out = nullptr;
  if (kh < 1 || kw < 1 || stride < 1 || pad < 0 || c_in < 1 || c_out < 1)
    return fail(MBU_ERR_SHAPE, "conv geometry out of range");
  if (pad_mode == MBU_PAD_ZERO && !neg)
    return fail(MBU_ERR_UNSUPPORTED,
                "binary convs cannot zero-pad: {-1,+1} activations have no 0 state");
  if (transposed && (kh != stride || kw != stride))
    return fail(MBU_ERR_UNSUPPORTED, "transposed conv requires kernel = stride");
  if (transposed && pad) return fail(MBU_ERR_UNSUPPORTED, "transposed conv does not support padding");
  int end = 0, n_ch = 0;
  for (int i = 0; i < n_segments; ++i) {
    if (seg_offsets[i] % 128 || seg_counts[i] <= 0 || seg_offsets[i] < end)
      return fail(MBU_ERR_LAYOUT, "segments must be block aligned, non-empty and ascending");
    end = seg_offsets[i] + seg_counts[i];
    n_ch += seg_counts[i];
  }
  if (n_ch != c_in) return fail(MBU_ERR_SHAPE, "segment channels != c_in");
  const int lpp = ((end + 127) / 128) * 128;
  const int wpp = lpp / 64;
  const int taps = kh * kw;
  const size_t words = size_t(c_out) * taps * wpp;
  if (neg) {
    for (size_t i = 0; i < words; ++i)
      if (pos[i] & neg[i]) return fail(MBU_ERR_OVERLAP, "a weight lane is set in both pos and neg planes");
  }
  cudaSetDevice(device);
  auto *cv = new mbu_conv();
  cv->device = device;
  cv->transposed = transposed;
  cv->kh = kh; cv->kw = kw; cv->stride = stride; cv->pad = pad;
  cv->c_in = c_in; cv->c_out = c_out; cv->pad_mode = pad_mode;
  cv->masked = neg != nullptr;
  cv->lpp = lpp; cv->wpp = wpp;
  cv->k_true = taps * c_in;
  cv->out_wpp = ((c_out + 127) / 128) * 2;
  int st = upload(&cv->d_pos, pos, words, "upload pos");
  if (st == MBU_OK && neg) st = upload(&cv->d_neg, neg, words, "upload neg");
  if (st == MBU_OK && neg && pad_mode == MBU_PAD_ZERO) {
    std::vector<int32_t> ws(size_t(c_out) * taps);
    for (int o = 0; o < c_out; ++o)
      for (int t = 0; t < taps; ++t) {
        int s = 0;
        for (int i = 0; i < wpp; ++i) {
          const size_t k = (size_t(o) * taps + t) * wpp + i;
          s += __builtin_popcountll(pos[k]) - __builtin_popcountll(neg[k]);
        }
        ws[size_t(o) * taps + t] = s;
      }
    st = upload(&cv->d_wsum, ws.data(), ws.size(), "upload wsum");
  }
  // thresholds padded to the GEMM width; pad channels are constant -1 so
  // their (pad) output lanes come out 0
  const int n_thr = ((c_out + 127) / 128) * 128 * (transposed ? stride * stride : 1);
  if (st == MBU_OK) {
    std::vector<int32_t> t(n_thr, 0);
    std::vector<uint8_t> c(n_thr, 2);
    if (thresholds && codes) {
      for (int o = 0; o < c_out; ++o) {
        if (codes[o] > 3) { st = fail(MBU_ERR_ALPHABET, "unknown threshold code"); break; }
        t[o] = thresholds[o];
        c[o] = codes[o];
      }
      cv->has_threshold = 1;
    }
    if (st == MBU_OK) st = upload(&cv->d_thr, t.data(), t.size(), "upload thresholds");
    if (st == MBU_OK) st = upload(&cv->d_codes, c.data(), c.size(), "upload codes");
  }
  if (st == MBU_OK) st = prepare_conv_tc(cv, pos, neg, seg_offsets, seg_counts, n_segments);
  if (st != MBU_OK) {
    mbu_conv_destroy(cv);
    return st;
  }
  *out = cv;
  return MBU_OK;
}

int mbu_conv_destroy(mbu_conv *cv) {
  if (!cv) return MBU_OK;
  cudaFree(cv->d_pos);
  cudaFree(cv->d_neg);
  cudaFree(cv->d_wsum);
  cudaFree(cv->d_thr);
  cudaFree(cv->d_codes);
  cudaFree(cv->d_chunk_word);
  cudaFree(cv->d_b);
  cudaFree(cv->d_thr2);
  cudaFree(cv->d_bias_slab);
  cudaFree(cv->d_b4);
  cudaFree(cv->d_chunk_pair);
  cudaFree(cv->d_bias_slab4);
  cudaFree(cv->d_b4p);
  cudaFree(cv->d_bias_slab4p);
  cudaFree(cv->d_slab_of_nt4);
  cudaFree(cv->d_slab_of_nt);
  delete cv;
  return MBU_OK;
}

int mbu_conv_run(mbu_conv *cv, const uint64_t *x, int n, int h, int w, int x_stride,
                 int x_offset, int32_t *acc, uint64_t *bits_out, int out_stride, int out_offset,
                 int path, void *stream) {
  if (!cv) return fail(MBU_ERR_ENGINE, "null conv handle");
  ActView v{x, n, h, w, cv->wpp, x_stride, x_offset};
  return conv_run(cv, v, acc, bits_out, out_stride, out_offset, path, as_stream(stream));
}

int mbu_threshold_pack(const int32_t *acc, int64_t pixels, int c, const int32_t *thr,
                       const uint8_t *codes, uint64_t *out, int out_stride, int out_offset,
                       void *stream) {
  const int groups = ((c + 127) / 128) * 4;
  const int64_t warps = pixels * groups;
  if (warps == 0) return MBU_OK;
  threshold_pack_kernel<<<unsigned((warps * 32 + 255) / 256), 256, 0, as_stream(stream)>>>(
      acc, pixels, c, groups, thr, codes, reinterpret_cast<uint32_t *>(out), out_stride * 2,
      out_offset * 2);
  return check_launch("threshold_pack_kernel");
}

int mbu_maxpool2(const uint64_t *x, int n, int h, int w, int wpp, int x_stride, int x_offset,
                 uint64_t *out, int out_stride, int out_offset, void *stream) {
  if (h % 2 || w % 2) return fail(MBU_ERR_SHAPE, "maxpool2: extents must be even");
  if (wpp % 2) return fail(MBU_ERR_LAYOUT, "maxpool2: words per pixel must be even");
  ActView v{x, n, h, w, wpp, x_stride, x_offset};
  return launch_maxpool(v, out, out_stride, out_offset, as_stream(stream));
}

int mbu_xor_popcount_rows(const uint64_t *a, const uint64_t *b, int32_t *out, int64_t m_rows,
                          int64_t n_rows, int64_t n_words, void *stream) {
  const int64_t total = m_rows * n_rows;
  if (total == 0) return MBU_OK;
  xor_popcount_rows_kernel<<<unsigned((total + 255) / 256), 256, 0, as_stream(stream)>>>(
      a, b, out, m_rows, n_rows, n_words);
  return check_launch("xor_popcount_rows_kernel");
}

int mbu_fconv_create(mbu_fconv **out, int device, int kh, int kw, int stride, int pad, int c_in,
                     int c_out, const double *weights, const double *bias, const double *bn,
                     double eps, const int32_t *in_lanes) {
  *out = nullptr;
  if (kh < 1 || kw < 1 || stride < 1 || pad < 0 || c_in < 1 || c_out < 1)
    return fail(MBU_ERR_SHAPE, "float conv geometry out of range");
  cudaSetDevice(device);
  auto *fc = new mbu_fconv();
  fc->device = device;
  fc->kh = kh; fc->kw = kw; fc->stride = stride; fc->pad = pad;
  fc->c_in = c_in; fc->c_out = c_out;
  fc->has_bn = bn != nullptr;
  fc->has_bias = bias != nullptr;
  fc->bits_input = in_lanes != nullptr;
  int st = upload(&fc->d_w, weights, size_t(c_out) * kh * kw * c_in, "upload fconv weights");
  if (st == MBU_OK && bias) st = upload(&fc->d_bias, bias, size_t(c_out), "upload bias");
  if (st == MBU_OK && bn) {
    std::vector<double> p(4 * size_t(c_out));
    for (int o = 0; o < c_out; ++o) {
      p[o] = bn[o];
      p[c_out + o] = bn[c_out + o];
      p[2 * c_out + o] = bn[2 * c_out + o];
      p[3 * c_out + o] = std::sqrt(bn[3 * c_out + o] + eps);  // sigma, as np.sqrt(var + eps)
    }
    st = upload(&fc->d_bn, p.data(), p.size(), "upload bn");
  }
  if (st == MBU_OK && in_lanes) st = upload(&fc->d_lanes, in_lanes, size_t(c_in), "upload lanes");
  if (st == MBU_OK) st = stem_prepare(fc, weights, bias, bn, eps);
  if (st == MBU_OK && fc->stem_fast) st = stem_tc_prepare(fc, weights, bias, bn, eps);
  if (st == MBU_OK && in_lanes) st = head_prepare(fc, weights, in_lanes);
  if (st != MBU_OK) {
    mbu_fconv_destroy(fc);
    return st;
  }
  *out = fc;
  return MBU_OK;
}

int mbu_fconv_destroy(mbu_fconv *fc) {
  if (!fc) return MBU_OK;
  cudaFree(fc->d_w);
  cudaFree(fc->d_bias);
  cudaFree(fc->d_bn);
  cudaFree(fc->d_lanes);
  stem_free(fc);
  stem_tc_free(fc);
  cudaFree(fc->d_head_tab);
  cudaFree(fc->d_head_nib);
  delete fc;
  return MBU_OK;
}

int mbu_fconv_run(mbu_fconv *fc, const double *x_f64, const uint64_t *x_bits, int x_stride,
                  int x_offset, int n, int h, int w, double *acc_out, uint64_t *bits_out,
                  int out_stride, int out_offset, uint8_t *mask_out, void *stream) {
  if (!fc) return fail(MBU_ERR_ENGINE, "null fconv handle");
  if (fc->bits_input == (x_bits == nullptr))
    return fail(MBU_ERR_LAYOUT, "fconv input kind does not match its handle");
  ActView v{x_bits, n, h, w, 0, x_stride, x_offset};
  return launch_fconv(fc, x_f64, v, n, h, w, acc_out, bits_out, out_stride, out_offset, mask_out,
                      as_stream(stream));
}

}  // extern "C"
