// Full-precision endpoints, fast paths (stem conv + BN-sign + pack; head).
//
// Stem (layers.py:530-560 float_conv + float_bn_sign; graph.py:434-438):
// the reference decides each stem bit with a float64 predicate
//     y = gamma * ((acc + 0) - mean) / sigma + beta >= 0,
//     acc = sum_taps dot(x, w) + bias          (float64)
// This kernel evaluates acc in float32 and compares it with the exact
// decision point T* = mean - beta*sigma/gamma. Whenever |acc32 - T*| is not
// larger than a rigorous bound on the float32 error (plus slack for the
// float64 predicate's own rounding), or the input is not finite, it
// recomputes acc in float64 in the reference's order and evaluates the
// reference predicate itself. So every output bit equals the float64
// decision; the float32 path only decides pixels that are far from the
// boundary. With trace output requested the whole layer runs in float64.
//
// Head (graph.py:439-441, :455): a 1x1 float64 conv of the +-1 bits,
// logits = bias + sum_c (+-w_c), mask = logits >= 0.
#include <cuda_runtime.h>

#include "common.cuh"

namespace mbu {

constexpr int STEM_TX = 32, STEM_TY = 8;  // 256 threads, one output pixel each
constexpr int STEM_MAX_CIN = 4, STEM_MAX_COUT = 64;

struct StemConsts {
  float w32[STEM_MAX_COUT * 9 * STEM_MAX_CIN];
  float wabs[STEM_MAX_COUT];     // sum |w| over taps and channels
  float tstar[STEM_MAX_COUT];    // decision point in acc units (float)
  float babs[STEM_MAX_COUT];
  int dir[STEM_MAX_COUT];        // +1: acc >= T*, -1: acc <= T*, 0: constant (see cbit)
  int cbit[STEM_MAX_COUT];
};

template <int CIN>
__global__ void __launch_bounds__(STEM_TX *STEM_TY) stem_kernel(
    const double *__restrict__ x, int n, int h, int w, int c_out,
    const double *__restrict__ w64, const double *__restrict__ bias64,
    const double *__restrict__ bn, const StemConsts *__restrict__ k,
    uint32_t *__restrict__ bits, int out_stride32, int out_offset32, int out_groups) {
  __shared__ double tile[STEM_TY + 2][STEM_TX + 2][CIN];
  __shared__ StemConsts ks;
  const int tx = threadIdx.x % STEM_TX, ty = threadIdx.x / STEM_TX;
  const int x0 = blockIdx.x * STEM_TX, y0 = blockIdx.y * STEM_TY, nb = blockIdx.z;
  // constants -> smem
  for (int i = threadIdx.x; i < int(sizeof(StemConsts) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t *>(&ks)[i] = reinterpret_cast<const uint32_t *>(k)[i];
  // halo'd input tile (zero padding outside the image, like float_conv)
  for (int i = threadIdx.x; i < (STEM_TY + 2) * (STEM_TX + 2); i += blockDim.x) {
    const int r = i / (STEM_TX + 2), c = i % (STEM_TX + 2);
    const int iy = y0 - 1 + r, ix = x0 - 1 + c;
    const bool inb = iy >= 0 && iy < h && ix >= 0 && ix < w;
    const double *src = x + ((int64_t(nb) * h + iy) * w + ix) * CIN;
#pragma unroll
    for (int ci = 0; ci < CIN; ++ci) tile[r][c][ci] = inb ? __ldg(src + ci) : 0.0;
  }
  __syncthreads();
  const int oy = y0 + ty, ox = x0 + tx;
  if (oy >= h || ox >= w) return;
  float xv[9 * CIN];
  float xmax = 0.f;
  bool finite = true;
#pragma unroll
  for (int t = 0; t < 9; ++t)
#pragma unroll
    for (int ci = 0; ci < CIN; ++ci) {
      const double d = tile[ty + t / 3][tx + t % 3][ci];
      finite &= isfinite(d);
      xv[t * CIN + ci] = float(d);
      xmax = fmaxf(xmax, fabsf(float(d)));
    }
  uint32_t word[2] = {0u, 0u};
  for (int o = 0; o < c_out; ++o) {
    const float *wr = ks.w32 + o * 9 * CIN;
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 9 * CIN; ++i) acc = fmaf(xv[i], wr[i], acc);
    acc += bias64 ? float(__ldg(bias64 + o)) : 0.f;
    bool bit;
    const int dir = ks.dir[o];
    if (dir == 0) {
      bit = ks.cbit[o] != 0;
    } else {
      // |acc32 - acc64| <= (9*CIN + 3) * 2^-23 * (max|x| * sum|w| + |b|)  (generous)
      const float margin = 1e-5f * (xmax * ks.wabs[o] + ks.babs[o]) + 1e-6f * fabsf(ks.tstar[o]);
      const float d = acc - ks.tstar[o];
      if (dir != 2 && finite && fabsf(d) > margin && isfinite(acc)) {
        bit = dir > 0 ? d > 0.f : d < 0.f;
      } else {  // exact float64 recomputation in the reference's order
        double a64 = 0.0;
        for (int t = 0; t < 9; ++t) {
          double dot = 0.0;
          const double *wt = w64 + (int64_t(o) * 9 + t) * CIN;
          for (int ci = 0; ci < CIN; ++ci)
            dot = __fma_rn(tile[ty + t / 3][tx + t % 3][ci], __ldg(wt + ci), dot);
          a64 = __dadd_rn(a64, dot);
        }
        if (bias64) a64 = __dadd_rn(a64, __ldg(bias64 + o));
        const double gm = bn[o], be = bn[c_out + o], mu = bn[2 * c_out + o], sg = bn[3 * c_out + o];
        const double y = __dadd_rn(__ddiv_rn(__dmul_rn(gm, __dsub_rn(a64, mu)), sg), be);
        bit = y >= 0.0;
      }
    }
    word[o >> 5] |= uint32_t(bit) << (o & 31);
  }
  uint32_t *dst = bits + (((int64_t(nb) * h + oy) * w + ox) * out_stride32 + out_offset32);
  if (out_groups == 4 && ((out_stride32 | out_offset32) & 3) == 0) {
    *reinterpret_cast<uint4 *>(dst) = make_uint4(word[0], word[1], 0u, 0u);
  } else {
    for (int g = 0; g < out_groups; ++g) dst[g] = g < 2 ? word[g] : 0u;
  }
}

// prepare float constants for the stem fast path (host)
int stem_prepare(mbu_fconv *fc, const double *w, const double *bias, const double *bn, double eps) {
  fc->stem_fast = 0;
  if (!(fc->kh == 3 && fc->kw == 3 && fc->stride == 1 && fc->pad == 1 && !fc->bits_input && bn &&
        fc->c_in >= 1 && fc->c_in <= STEM_MAX_CIN && fc->c_out <= STEM_MAX_COUT))
    return MBU_OK;
  StemConsts k{};
  const int co = fc->c_out, ci = fc->c_in;
  for (int o = 0; o < co; ++o) {
    double s = 0.0;
    for (int t = 0; t < 9; ++t)
      for (int c = 0; c < ci; ++c) {
        const double v = w[(size_t(o) * 9 + t) * ci + c];
        k.w32[(o * 9 + t) * ci + c] = float(v);
        s += std::fabs(v);
      }
    k.wabs[o] = float(s) * 1.001f;
    k.babs[o] = bias ? float(std::fabs(bias[o])) * 1.001f : 0.f;
    const double g = bn[o], b = bn[co + o], m = bn[2 * co + o];
    const double sigma = std::sqrt(bn[3 * co + o] + eps);
    if (g == 0.0) {
      k.dir[o] = 0;
      k.cbit[o] = b >= 0.0;
    } else {
      const double ts = m - b * sigma / g;
      if (!std::isfinite(ts) || std::fabs(ts) > 1e30) {
        k.dir[o] = 2;  // no usable float32 decision point: always evaluate exactly
      } else {
        k.dir[o] = g > 0 ? 1 : -1;
        k.tstar[o] = float(ts);
      }
    }
  }
  MBU_TRY(check_cuda(cudaMalloc(&fc->d_stem, sizeof(StemConsts)), "alloc stem consts"));
  MBU_TRY(check_cuda(cudaMemcpy(fc->d_stem, &k, sizeof(StemConsts), cudaMemcpyHostToDevice),
                     "upload stem consts"));
  fc->stem_fast = 1;
  return MBU_OK;
}

int launch_stem_fast(const mbu_fconv *fc, const double *x, int n, int h, int w, uint64_t *bits,
                     int out_stride, int out_offset, cudaStream_t st) {
  dim3 grid((w + STEM_TX - 1) / STEM_TX, (h + STEM_TY - 1) / STEM_TY, n);
  const int groups = ((fc->c_out + 127) / 128) * 4;
  auto *k = static_cast<const StemConsts *>(fc->d_stem);
  auto *b32 = reinterpret_cast<uint32_t *>(bits);
#define MBU_STEM(C)                                                                          \
  stem_kernel<C><<<grid, STEM_TX * STEM_TY, 0, st>>>(x, n, h, w, fc->c_out, fc->d_w, fc->d_bias, \
                                                     fc->d_bn, k, b32, out_stride * 2,        \
                                                     out_offset * 2, groups)
  switch (fc->c_in) {
    case 1: MBU_STEM(1); break;
    case 2: MBU_STEM(2); break;
    case 3: MBU_STEM(3); break;
    default: MBU_STEM(4); break;
  }
#undef MBU_STEM
  return check_launch("stem_kernel");
}

// ---------------------------------------------------------------------------
// head: 1x1 float64 conv of packed bits, logits + mask
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) head_kernel(ActView xb, const int32_t *__restrict__ lanes,
                                                   const double *__restrict__ w,
                                                   const double *__restrict__ bias, int c_in,
                                                   int c_out, int64_t pixels,
                                                   double *__restrict__ logits,
                                                   uint8_t *__restrict__ mask) {
  extern __shared__ double hw[];  // c_out * c_in weights, then lane table
  int32_t *ls = reinterpret_cast<int32_t *>(hw + c_out * c_in);
  for (int i = threadIdx.x; i < c_out * c_in; i += blockDim.x) hw[i] = w[i];
  for (int i = threadIdx.x; i < c_in; i += blockDim.x) ls[i] = lanes[i];
  __syncthreads();
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < pixels;
       p += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t *xp = xb.base + p * xb.stride + xb.offset;
    uint64_t cache_word = 0;
    int cache_idx = -1;
    for (int o = 0; o < c_out; ++o) {
      double dot = 0.0;
      for (int c = 0; c < c_in; ++c) {
        const int L = ls[c];
        if ((L >> 6) != cache_idx) {
          cache_idx = L >> 6;
          cache_word = __ldg(xp + cache_idx);
        }
        const double wv = hw[o * c_in + c];
        dot = __fma_rn(((cache_word >> (L & 63)) & 1ull) ? 1.0 : -1.0, wv, dot);
      }
      double acc = __dadd_rn(0.0, dot);
      if (bias) acc = __dadd_rn(acc, bias[o]);
      logits[p * c_out + o] = acc;
      if (mask) mask[p * c_out + o] = acc >= 0.0 ? 1 : 0;
    }
  }
}

int launch_head_fast(const mbu_fconv *fc, const ActView &xb, int n, int h, int w, double *logits,
                     uint8_t *mask, cudaStream_t st) {
  const int64_t pixels = int64_t(n) * h * w;
  if (pixels == 0) return MBU_OK;
  const size_t smem = size_t(fc->c_out) * fc->c_in * sizeof(double) + fc->c_in * sizeof(int32_t);
  const int64_t blocks = std::min<int64_t>((pixels + 255) / 256, 148 * 16);
  head_kernel<<<unsigned(blocks), 256, smem, st>>>(xb, fc->d_lanes, fc->d_w, fc->d_bias, fc->c_in,
                                                   fc->c_out, pixels, logits, mask);
  return check_launch("head_kernel");
}

}  // namespace mbu
