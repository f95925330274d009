// Full-precision endpoints, fast paths (stem conv + BN-sign + pack; head).
//
// Stem (layers.py:530-560 float_conv + float_bn_sign; graph.py:434-438):
// the reference decides each stem bit with a float64 predicate
//     y = gamma * ((acc + 0) - mean) / sigma + beta >= 0,
//     acc = sum_taps dot(x, w) + bias          (float64)
// This kernel evaluates acc in float32 (packed FFMA2, 64 accumulators per
// pixel in registers) and compares it with the exact decision point
// T* = mean - beta*sigma/gamma. Whenever |acc32 - T*| is not larger than a
// rigorous bound on the float32 error (plus slack for the float64
// predicate's own rounding), or anything is non-finite, it recomputes acc in
// float64 in the reference's order and evaluates the reference predicate
// itself. So every output bit equals the float64 decision; the float32 path
// only decides bits that are far from the boundary. With trace output
// requested the whole layer runs through the float64 kernel instead.
//
// Head (graph.py:439-441, :455): a 1x1 float64 conv of the +-1 bits,
// logits = bias + sum_c (+-w_c), mask = logits >= 0.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace mbu {

constexpr int STEM_TX = 32, STEM_TY = 4;  // 128 threads, one output pixel each
constexpr int STEM_MAX_CIN = 4, STEM_COUT = 64;

struct StemConsts {
  float w[9 * STEM_MAX_CIN][STEM_COUT];  // [tap*cin + c][o], float32 copy
  float b[STEM_COUT];                    // bias (float32)
  float tstar[STEM_COUT];                // +-inf for constant channels
  float dirf[STEM_COUT];                 // +1: bit = acc > T*, -1: bit = acc < T*
  float ma[STEM_COUT], mb[STEM_COUT];    // margin = max|x| * ma + mb (inf: always exact)
};

__device__ __forceinline__ unsigned long long pack2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void unpack2(unsigned long long v, float &a, float &b) {
  asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long ffma2_bcast(float x, unsigned long long w,
                                                          unsigned long long acc) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pack2(x, x)), "l"(w), "l"(acc));
  return r;
}

template <int CIN>
__global__ void __launch_bounds__(STEM_TX *STEM_TY) stem_kernel(
    const double *__restrict__ x, int n, int h, int w, int c_out,
    const double *__restrict__ w64, const double *__restrict__ bias64,
    const double *__restrict__ bn, const __grid_constant__ StemConsts ks,
    uint32_t *__restrict__ bits, int out_stride32, int out_offset32, int out_groups) {
  // the float32 weights and per-channel constants live in the kernel
  // parameter bank: FFMA2 reads them as constant operands, no shared memory
  __shared__ double tile[STEM_TY + 2][STEM_TX + 2][CIN];
  const int tx = threadIdx.x % STEM_TX, ty = threadIdx.x / STEM_TX;
  const int x0 = blockIdx.x * STEM_TX, y0 = blockIdx.y * STEM_TY, nb = blockIdx.z;
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

  unsigned long long acc[STEM_COUT / 2];
#pragma unroll
  for (int j = 0; j < STEM_COUT / 2; ++j) acc[j] = pack2(ks.b[2 * j], ks.b[2 * j + 1]);
  float xmax = 0.f;
  bool finite = true;
#pragma unroll
  for (int t = 0; t < 9; ++t) {
#pragma unroll
    for (int ci = 0; ci < CIN; ++ci) {
      const double d = tile[ty + t / 3][tx + t % 3][ci];
      finite &= isfinite(d);
      const float xf = float(d);
      xmax = fmaxf(xmax, fabsf(xf));
      const unsigned long long *wr = reinterpret_cast<const unsigned long long *>(ks.w[t * CIN + ci]);
#pragma unroll
      for (int q = 0; q < STEM_COUT / 2; ++q) acc[q] = ffma2_bcast(xf, wr[q], acc[q]);
    }
  }
  uint32_t word[2] = {0u, 0u};
  unsigned long long unsure = 0ull;
#pragma unroll
  for (int j = 0; j < STEM_COUT / 2; ++j) {
    float a[2];
    unpack2(acc[j], a[0], a[1]);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int o = 2 * j + e;
      const float d = a[e] - ks.tstar[o];
      const float margin = fmaf(xmax, ks.ma[o], ks.mb[o]);
      const bool sure = finite && fabsf(d) > margin;  // false for NaN / inf margin
      const bool bit = d * ks.dirf[o] > 0.f;
      word[o >> 5] |= uint32_t(sure && bit) << (o & 31);
      unsure |= (unsigned long long)(!sure && o < c_out) << o;
    }
  }
  while (unsure) {  // rare: exact float64 decision in the reference's order
    const int o = __ffsll(unsure) - 1;
    unsure &= unsure - 1;
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
    word[o >> 5] |= uint32_t(y >= 0.0) << (o & 31);
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
        fc->c_in >= 1 && fc->c_in <= STEM_MAX_CIN && fc->c_out <= STEM_COUT))
    return MBU_OK;
  StemConsts k{};
  const int co = fc->c_out, ci = fc->c_in;
  const float inf = INFINITY;
  for (int o = 0; o < STEM_COUT; ++o) {
    k.tstar[o] = inf;  // unused channels: never fire, never unsure (masked by c_out)
    k.dirf[o] = 1.f;
    k.ma[o] = 0.f;
    k.mb[o] = 0.f;
  }
  for (int o = 0; o < co; ++o) {
    double s = 0.0;
    for (int t = 0; t < 9; ++t)
      for (int c = 0; c < ci; ++c) {
        const double v = w[(size_t(o) * 9 + t) * ci + c];
        k.w[t * ci + c][o] = float(v);
        s += std::fabs(v);
      }
    const double babs = bias ? std::fabs(bias[o]) : 0.0;
    k.b[o] = bias ? float(bias[o]) : 0.f;
    const double g = bn[o], b = bn[co + o], m = bn[2 * co + o];
    const double sigma = std::sqrt(bn[3 * co + o] + eps);
    // float32 error of acc <= ~(9*cin + 4) * 2^-23 * (max|x| * sum|w| + |b|): use 1e-5
    k.ma[o] = float(1e-5 * s * 1.001);
    k.mb[o] = float(1e-5 * babs * 1.001);
    if (g == 0.0) {
      k.dirf[o] = 1.f;
      k.tstar[o] = b >= 0.0 ? -inf : inf;  // constant: d = +-inf decides (NaN acc -> exact)
    } else {
      const double ts = m - b * sigma / g;
      k.dirf[o] = g > 0 ? 1.f : -1.f;
      if (!std::isfinite(ts) || std::fabs(ts) > 1e30) {
        k.tstar[o] = 0.f;
        k.mb[o] = inf;  // no usable float32 decision point: always exact
      } else {
        k.tstar[o] = float(ts);
        k.mb[o] += float(1e-6 * std::fabs(ts));
      }
    }
  }
  fc->h_stem = new StemConsts(k);  // passed by value as a __grid_constant__ kernel parameter
  fc->stem_fast = 1;
  return MBU_OK;
}

void stem_free(mbu_fconv *fc) {
  delete static_cast<StemConsts *>(fc->h_stem);
  fc->h_stem = nullptr;
}

int launch_stem_fast(const mbu_fconv *fc, const double *x, int n, int h, int w, uint64_t *bits,
                     int out_stride, int out_offset, cudaStream_t st) {
  if (!g_force_stem_ffma && stem_tc_usable(fc, x, w))
    return launch_stem_tc(fc, x, n, h, w, bits, out_stride, out_offset, st);
  dim3 grid((w + STEM_TX - 1) / STEM_TX, (h + STEM_TY - 1) / STEM_TY, n);
  const int groups = ((fc->c_out + 127) / 128) * 4;
  const StemConsts &k = *static_cast<const StemConsts *>(fc->h_stem);
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

// Byte-table head: with the c_in input channels at lanes 0..c_in-1, the
// logit is bias + sum over bytes k of T[o][k][byte_k], T holding the signed
// partial sums of 8 consecutive channel weights (built once on the host, in
// channel order). Eight shared-memory lookups per pixel replace 64 bit
// extractions + FMAs. The float64 sum order differs from the reference's BLAS
// dot only by rounding (|delta| ~ 1e-16 * sum|w|), within the 1e-9 logits
// tolerance of verify.py:23.
__global__ void __launch_bounds__(256) head_tab_kernel(ActView xb, const double *__restrict__ tab,
                                                       const double *__restrict__ bias, int nbytes,
                                                       int c_out, int64_t pixels,
                                                       double *__restrict__ logits,
                                                       uint8_t *__restrict__ mask) {
  extern __shared__ double ts[];  // [c_out][nbytes][256]
  for (int i = threadIdx.x; i < c_out * nbytes * 256; i += blockDim.x) ts[i] = tab[i];
  __syncthreads();
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < pixels;
       p += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t *xp = xb.base + p * xb.stride + xb.offset;
    for (int o = 0; o < c_out; ++o) {
      double acc = 0.0;
      const double *to = ts + size_t(o) * nbytes * 256;
      for (int k = 0; k < nbytes; k += 8) {
        const uint64_t wd = __ldg(xp + (k >> 3));
        const int kend = min(8, nbytes - k);
        for (int kk = 0; kk < kend; ++kk)
          acc = __dadd_rn(acc, to[(k + kk) * 256 + int((wd >> (8 * kk)) & 0xFF)]);
      }
      if (bias) acc = __dadd_rn(acc, bias[o]);
      logits[p * c_out + o] = acc;
      if (mask) mask[p * c_out + o] = acc >= 0.0 ? 1 : 0;
    }
  }
}

// The default network's head (c_out = 1, 64 input channels = two words per
// pixel, a plain tensor): bandwidth-shaped. Each thread takes four pixels
// a block-width apart (every warp load / store instruction covers
// consecutive pixels), issues their 16-B loads first, then runs four
// independent table-lookup chains in head_tab_kernel's order.
__global__ void __launch_bounds__(256) head_tab64_kernel(const uint4 *__restrict__ x, const double *__restrict__ tab,
                                                         const double *__restrict__ bias, int64_t pixels,
                                                         double *__restrict__ logits, uint8_t *__restrict__ mask) {
  __shared__ double ts[8 * 256];
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) ts[i] = tab[i];
  __syncthreads();
  const double b0 = bias ? __ldg(bias) : 0.0;
  const int64_t chunk = int64_t(blockDim.x) * 4;
  for (int64_t base = int64_t(blockIdx.x) * chunk; base < pixels; base += int64_t(gridDim.x) * chunk) {
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t q = base + j * blockDim.x + threadIdx.x;
      v[j] = q < pixels ? __ldcs(x + q) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t q = base + j * blockDim.x + threadIdx.x;
      const uint32_t w[2] = {v[j].x, v[j].y};  // channels 0-63 (z, w: the block's pad lanes)
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t word = k < 4 ? w[0] : w[1];
        acc = __dadd_rn(acc, ts[k * 256 + int((word >> (8 * (k & 3))) & 0xFFu)]);
      }
      if (bias) acc = __dadd_rn(acc, b0);
      if (q < pixels) {
        __stcs(logits + q, acc);
        if (mask) mask[q] = acc >= 0.0 ? 1 : 0;
      }
    }
  }
}

// Same head with sixteen 16-entry nibble tables (2 KB): a half-warp's 16
// random entries of one table sit in one 128-B row, so every lookup is one
// conflict-free shared-memory wavefront per half-warp (the 256-entry byte
// tables take ~3 per half-warp). 16 lookups and adds per pixel instead of 8.
__global__ void __launch_bounds__(256) head_nib64_kernel(const uint4 *__restrict__ x, const double *__restrict__ tab,
                                                         const double *__restrict__ bias, int64_t pixels,
                                                         double *__restrict__ logits, uint8_t *__restrict__ mask) {
  __shared__ double ts[16 * 16];
  ts[threadIdx.x] = tab[threadIdx.x];
  __syncthreads();
  const double b0 = bias ? __ldg(bias) : 0.0;
  const int64_t chunk = int64_t(blockDim.x) * 4;
  for (int64_t base = int64_t(blockIdx.x) * chunk; base < pixels; base += int64_t(gridDim.x) * chunk) {
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t q = base + j * blockDim.x + threadIdx.x;
      v[j] = q < pixels ? __ldcs(x + q) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t q = base + j * blockDim.x + threadIdx.x;
      double a0 = 0.0, a1 = 0.0;  // two chains: nibbles of channels 0-31 / 32-63
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        a0 = __dadd_rn(a0, ts[k * 16 + int((v[j].x >> (4 * k)) & 0xFu)]);
        a1 = __dadd_rn(a1, ts[(8 + k) * 16 + int((v[j].y >> (4 * k)) & 0xFu)]);
      }
      double acc = __dadd_rn(a0, a1);
      if (bias) acc = __dadd_rn(acc, b0);
      if (q < pixels) {
        __stcs(logits + q, acc);
        if (mask) mask[q] = acc >= 0.0 ? 1 : 0;
      }
    }
  }
}

int head_prepare(mbu_fconv *fc, const double *w, const int32_t *lanes) {
  fc->head_tab = 0;
  if (!(fc->bits_input && fc->kh == 1 && fc->kw == 1 && fc->stride == 1 && fc->pad == 0)) return MBU_OK;
  for (int c = 0; c < fc->c_in; ++c)
    if (lanes[c] != c) return MBU_OK;
  const int nbytes = (fc->c_in + 7) / 8;
  const size_t entries = size_t(fc->c_out) * nbytes * 256;
  if (entries * sizeof(double) > 96 * 1024) return MBU_OK;
  std::vector<double> tab(entries);
  for (int o = 0; o < fc->c_out; ++o)
    for (int k = 0; k < nbytes; ++k)
      for (int v = 0; v < 256; ++v) {
        double s = 0.0;
        for (int i = 0; i < 8 && 8 * k + i < fc->c_in; ++i) {
          const double wv = w[size_t(o) * fc->c_in + 8 * k + i];
          s += ((v >> i) & 1) ? wv : -wv;
        }
        tab[(size_t(o) * nbytes + k) * 256 + v] = s;
      }
  MBU_TRY(check_cuda(cudaMalloc(&fc->d_head_tab, entries * sizeof(double)), "alloc head table"));
  MBU_TRY(check_cuda(cudaMemcpy(fc->d_head_tab, tab.data(), entries * sizeof(double), cudaMemcpyHostToDevice),
                     "upload head table"));
  fc->head_tab = 1;
  if (fc->c_out == 1 && fc->c_in == 64) {
    double nib[16 * 16];
    for (int k = 0; k < 16; ++k)
      for (int v = 0; v < 16; ++v) {
        double s = 0.0;
        for (int i = 0; i < 4; ++i) s += ((v >> i) & 1) ? w[4 * k + i] : -w[4 * k + i];
        nib[k * 16 + v] = s;
      }
    MBU_TRY(check_cuda(cudaMalloc(&fc->d_head_nib, sizeof(nib)), "alloc head nibble table"));
    MBU_TRY(check_cuda(cudaMemcpy(fc->d_head_nib, nib, sizeof(nib), cudaMemcpyHostToDevice), "upload head nibble table"));
  }
  return MBU_OK;
}

int launch_head_fast(const mbu_fconv *fc, const ActView &xb, int n, int h, int w, double *logits,
                     uint8_t *mask, cudaStream_t st) {
  const int64_t pixels = int64_t(n) * h * w;
  if (pixels == 0) return MBU_OK;
  if (fc->head_tab && fc->c_out == 1 && (fc->c_in + 7) / 8 == 8 && xb.stride == 2 && xb.offset == 0 &&
      !xb.split && (reinterpret_cast<uintptr_t>(xb.base) & 15) == 0) {
    const int64_t blocks = std::min<int64_t>((pixels + 1023) / 1024, 148 * 8);
    // 64 lanes: nibble tables (0.131 -> 0.086 ms at the bench shape: the byte
    // tables' bank conflicts made it shared-memory bound); MBU_HEAD_BYTETAB=1
    // keeps the byte-table kernel (A/B)
    static const bool bytetab = std::getenv("MBU_HEAD_BYTETAB") != nullptr;
    if (!bytetab && fc->d_head_nib) {
      head_nib64_kernel<<<unsigned(blocks), 256, 0, st>>>(reinterpret_cast<const uint4 *>(xb.base), fc->d_head_nib,
                                                          fc->d_bias, pixels, logits, mask);
      return check_launch("head_nib64_kernel");
    }
    head_tab64_kernel<<<unsigned(blocks), 256, 0, st>>>(reinterpret_cast<const uint4 *>(xb.base), fc->d_head_tab,
                                                        fc->d_bias, pixels, logits, mask);
    return check_launch("head_tab64_kernel");
  }
  if (fc->head_tab) {
    const int nbytes = (fc->c_in + 7) / 8;
    const size_t smem = size_t(fc->c_out) * nbytes * 256 * sizeof(double);
    static bool configured = false;
    if (!configured) {
      MBU_TRY(check_cuda(cudaFuncSetAttribute(head_tab_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              96 * 1024), "cudaFuncSetAttribute(head)"));
      configured = true;
    }
    const int64_t blocks = std::min<int64_t>((pixels + 255) / 256, 148 * 4);
    head_tab_kernel<<<unsigned(blocks), 256, smem, st>>>(xb, fc->d_head_tab, fc->d_bias, nbytes,
                                                         fc->c_out, pixels, logits, mask);
    return check_launch("head_tab_kernel");
  }
  const size_t smem = size_t(fc->c_out) * fc->c_in * sizeof(double) + fc->c_in * sizeof(int32_t);
  const int64_t blocks = std::min<int64_t>((pixels + 255) / 256, 148 * 16);
  head_kernel<<<unsigned(blocks), 256, smem, st>>>(xb, fc->d_lanes, fc->d_w, fc->d_bias, fc->c_in,
                                                   fc->c_out, pixels, logits, mask);
  return check_launch("head_kernel");
}

}  // namespace mbu

// ---------------------------------------------------------------------------
// class map of a multi-class head: numpy.argmax over the channel axis
// ---------------------------------------------------------------------------
namespace mbu {
__global__ void __launch_bounds__(256) argmax_kernel(const double *__restrict__ logits, int64_t pixels,
                                                     int c, uint8_t *__restrict__ classes) {
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < pixels;
       p += int64_t(gridDim.x) * blockDim.x) {
    const double *row = logits + p * c;
    double best = row[0];
    int idx = 0;
    for (int k = 1; k < c && best == best; ++k) {  // a NaN wins and stops the scan
      const double v = __ldg(row + k);
      if (v != v || v > best) {
        best = v;
        idx = k;
      }
    }
    classes[p] = uint8_t(idx);
  }
}
}  // namespace mbu

extern "C" int mbu_argmax(const double *logits, int64_t pixels, int channels, uint8_t *classes,
                          void *stream) {
  using namespace mbu;
  if (channels < 1 || channels > 256) return fail(MBU_ERR_SHAPE, "argmax: channels must be 1..256");
  if (pixels <= 0) return MBU_OK;
  const int64_t blocks = std::min<int64_t>((pixels + 255) / 256, 148 * 16);
  argmax_kernel<<<unsigned(blocks), 256, 0, as_stream(stream)>>>(logits, pixels, channels, classes);
  return check_launch("argmax_kernel");
}

// ---------------------------------------------------------------------------
// bit-packed masks for the multi-GPU gather (dp.py): one bit
// per mask byte, numpy.packbits(..., bitorder="little") per frame
// ---------------------------------------------------------------------------
namespace mbu {
__global__ void __launch_bounds__(256) pack_mask_kernel(const uint8_t *__restrict__ mask, int64_t frames,
                                                        int64_t per_frame, int64_t out_per_frame,
                                                        uint8_t *__restrict__ out) {
  const int64_t total = frames * out_per_frame;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t f = i / out_per_frame, k = i - f * out_per_frame;
    const uint8_t *src = mask + f * per_frame + 8 * k;
    const int64_t left = per_frame - 8 * k;
    uint32_t b = 0;
    if (left >= 8 && (reinterpret_cast<uintptr_t>(src) & 7) == 0) {
      const uint2 v = __ldg(reinterpret_cast<const uint2 *>(src));
      // (x & 0x01010101) * 0x01020408: byte j's bit 0 lands at bit 24 + j
      b = (((v.x & 0x01010101u) * 0x01020408u) >> 24) | ((((v.y & 0x01010101u) * 0x01020408u) >> 24) << 4);
    } else {
      for (int j = 0; j < 8 && j < left; ++j) b |= uint32_t(src[j] & 1u) << j;
    }
    out[i] = uint8_t(b);
  }
}
}  // namespace mbu

extern "C" int mbu_pack_mask(const uint8_t *mask, int64_t frames, int64_t per_frame, uint8_t *packed,
                             void *stream) {
  using namespace mbu;
  if (frames < 0 || per_frame < 0) return fail(MBU_ERR_SHAPE, "pack_mask: negative size");
  const int64_t out_per_frame = (per_frame + 7) / 8, total = frames * out_per_frame;
  if (total == 0) return MBU_OK;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 16);
  pack_mask_kernel<<<unsigned(blocks), 256, 0, as_stream(stream)>>>(mask, frames, per_frame, out_per_frame, packed);
  return check_launch("pack_mask_kernel");
}

// ---------------------------------------------------------------------------
// netpbm raster -> float64 image (imageio.py:59-83): sample / maxval
// ---------------------------------------------------------------------------
namespace mbu {
__global__ void __launch_bounds__(256) decode_u8_kernel(const uchar4 *__restrict__ in, int64_t quads,
                                                        double maxval, double4 *__restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < quads;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uchar4 v = in[i];
    out[i] = make_double4(__ddiv_rn(double(v.x), maxval), __ddiv_rn(double(v.y), maxval),
                          __ddiv_rn(double(v.z), maxval), __ddiv_rn(double(v.w), maxval));
  }
}
__global__ void __launch_bounds__(256) decode_tail_kernel(const uint8_t *__restrict__ in, int64_t begin,
                                                          int64_t count, int bps, double maxval,
                                                          double *__restrict__ out) {
  for (int64_t i = begin + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t v = bps == 1 ? in[i] : (uint32_t(in[2 * i]) << 8) | in[2 * i + 1];  // big endian
    out[i] = __ddiv_rn(double(v), maxval);
  }
}
}  // namespace mbu

extern "C" int mbu_decode_raster(const void *raster, int64_t count, int bytes_per_sample, int maxval,
                                 double *out, void *stream) {
  using namespace mbu;
  if (bytes_per_sample != 1 && bytes_per_sample != 2)
    return fail(MBU_ERR_SHAPE, "decode_raster: 1 or 2 bytes per sample");
  if (maxval < 1 || maxval > 65535 || (bytes_per_sample == 1 && maxval > 255))
    return fail(MBU_ERR_SHAPE, "decode_raster: maxval out of range");
  if (count <= 0) return MBU_OK;
  cudaStream_t st = as_stream(stream);
  const auto *in = static_cast<const uint8_t *>(raster);
  int64_t done = 0;
  if (bytes_per_sample == 1 && (reinterpret_cast<uintptr_t>(in) & 3) == 0 &&
      (reinterpret_cast<uintptr_t>(out) & 31) == 0) {
    const int64_t quads = count / 4;
    if (quads) {
      const int64_t blocks = std::min<int64_t>((quads + 255) / 256, 148 * 32);
      decode_u8_kernel<<<unsigned(blocks), 256, 0, st>>>(reinterpret_cast<const uchar4 *>(in), quads,
                                                        double(maxval), reinterpret_cast<double4 *>(out));
      MBU_TRY(check_launch("decode_u8_kernel"));
    }
    done = quads * 4;
  }
  if (done < count) {
    const int64_t blocks = std::min<int64_t>((count - done + 255) / 256, 148 * 32);
    decode_tail_kernel<<<unsigned(blocks), 256, 0, st>>>(in, done, count, bytes_per_sample, double(maxval),
                                                         out);
    MBU_TRY(check_launch("decode_tail_kernel"));
  }
  return MBU_OK;
}
