// Build-time quantization on the GPU:
//   * ternarize / binarize a float32 weight tensor (quantizer.py:86-110):
//     w > delta -> +1, w < -delta -> -1, else 0 (delta = t * mean|w|, which the
//     host computes with numpy's own float64 reduction so it is bit-identical);
//     binary: w >= 0 -> +1 else -1 (NaN -> -1, like numpy.where);
//   * fuse_bn_sign (layers.py:455-505): per channel the int32 threshold of the
//     float64 batchnorm-sign predicate, one thread per channel. The predicate
//     is evaluated in the reference's operation order with explicitly
//     rounded operations (no contraction), and the threshold is found by
//     bisection over the int32 range: the predicate is monotone in acc, so the
//     answer equals the reference's snap-then-refine search.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "common.cuh"

namespace mbu {
namespace {

template <typename T>  // float32 or float64 weights, compared in float64 (numpy's promotion)
__global__ void __launch_bounds__(256) quantize_kernel(const T *__restrict__ w, int64_t n, int binary,
                                                       double delta, int8_t *__restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double v = double(w[i]);
    out[i] = binary ? int8_t(v >= 0.0 ? 1 : -1) : int8_t(v > delta ? 1 : (v < -delta ? -1 : 0));
  }
}

// gamma * ((a + bias) - mean) / sigma + beta >= 0, left to right, each step rounded
__device__ __forceinline__ bool bn_fires(int64_t a, double g, double b8, double m, double s, double b0) {
  const double pre = __dadd_rn(double(a), b0);
  return __dadd_rn(__ddiv_rn(__dmul_rn(g, __dsub_rn(pre, m)), s), b8) >= 0.0;
}

constexpr int kDirGe = 0, kDirLe = 1, kConstNeg = 2, kConstPos = 3;  // layers.py FusedThreshold codes
constexpr int64_t kI32Min = -2147483648ll, kI32Max = 2147483647ll;

__global__ void __launch_bounds__(128) fuse_bn_sign_kernel(const double *__restrict__ gamma,
                                                           const double *__restrict__ beta,
                                                           const double *__restrict__ mean,
                                                           const double *__restrict__ var, double eps,
                                                           const double *__restrict__ bias, int c,
                                                           int32_t *__restrict__ thr, uint8_t *__restrict__ codes) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= c) return;
  const double g = gamma[j], b8 = beta[j], m = mean[j], b0 = bias ? bias[j] : 0.0;
  const double s = __dsqrt_rn(__dadd_rn(var[j], eps));
  int32_t t = 0;
  uint8_t code = kConstNeg;
  if (g == 0.0) {
    code = b8 >= 0.0 ? kConstPos : kConstNeg;
  } else if (g > 0.0) {
    if (bn_fires(kI32Max, g, b8, m, s, b0)) {  // smallest true T
      int64_t lo = kI32Min - 1, hi = kI32Max;
      while (hi - lo > 1) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (bn_fires(mid, g, b8, m, s, b0)) hi = mid; else lo = mid;
      }
      t = int32_t(hi);
      code = kDirGe;
    }
  } else {
    if (bn_fires(kI32Min, g, b8, m, s, b0)) {  // largest true T
      int64_t lo = kI32Min, hi = kI32Max + 1;
      while (hi - lo > 1) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (bn_fires(mid, g, b8, m, s, b0)) lo = mid; else hi = mid;
      }
      t = int32_t(lo);
      code = kDirLe;
    }
  }
  thr[j] = t;
  codes[j] = code;
}

}  // namespace
}  // namespace mbu

template <typename T>
static int quantize_weights(const T *w, int64_t n, int binary, double delta, int8_t *out, void *stream) {
  using namespace mbu;
  if (n < 0) return fail(MBU_ERR_SHAPE, "quantize_weights: negative size");
  if (n == 0) return MBU_OK;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
  quantize_kernel<T><<<unsigned(blocks), 256, 0, as_stream(stream)>>>(w, n, binary, delta, out);
  return check_launch("quantize_kernel");
}

extern "C" int mbu_quantize_weights(const float *w, int64_t n, int binary, double delta, int8_t *out,
                                    void *stream) {
  return quantize_weights(w, n, binary, delta, out, stream);
}

extern "C" int mbu_quantize_weights_f64(const double *w, int64_t n, int binary, double delta, int8_t *out,
                                        void *stream) {
  return quantize_weights(w, n, binary, delta, out, stream);
}

extern "C" int mbu_fuse_bn_sign(const double *gamma, const double *beta, const double *mean, const double *var,
                                double eps, const double *bias, int c, int32_t *thresholds, uint8_t *codes,
                                void *stream) {
  using namespace mbu;
  if (c < 0) return fail(MBU_ERR_SHAPE, "fuse_bn_sign: negative channel count");
  if (!(eps > 0.0) || eps != eps || eps > 1.7976931348623157e308)
    return fail(MBU_ERR_ALPHABET, "fuse_bn_sign: eps must be finite and > 0");
  if (c == 0) return MBU_OK;
  fuse_bn_sign_kernel<<<unsigned((c + 127) / 128), 128, 0, as_stream(stream)>>>(gamma, beta, mean, var, eps, bias,
                                                                                c, thresholds, codes);
  return check_launch("fuse_bn_sign_kernel");
}
