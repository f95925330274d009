// Stem on the tensor cores: 3x3 float conv (3 -> <=64 channels) + BN sign +
// pack, as one persistent tcgen05 kind::f16 implicit GEMM.
//
// Replaces float_conv + float_bn_sign + pack_bits_tensor for the stem
// (layers.py:530-560, :392-395; bitcore.py:410-425; graph.py:434-438).
//
// The reference decides bit (pixel p, channel o) with the float64 predicate
//   y = gamma*(acc - mean)/sigma + beta >= 0,  acc = conv(x, w) + bias.
// For gamma != 0 that is acc >= T* (gamma > 0) or acc <= T* (gamma < 0) with
// T* = mean - beta*sigma/gamma, up to float64 rounding (~1e-16 relative).
//
// Arithmetic. Inputs are split into two fp16 parts via float32,
// x = xh + xl + ex, |ex| <= (2^-22 + 2^-24)|x| + 2^-25 (fp16 subnormals), and
// the weights, pre-scaled on the host by a power of two 2^j (exact) so that
// max|w'| is in [2^12, 2^13), likewise (w' = wh + wl + ew). One K = 16 fp16
// MMA row per pixel carries
//     A row  [xh0 xh1 xh2 xl0 xl1 xl2 xh0 xh1 | xh2 2048 1   1   0 0 0 0]
//     B col  [wh0 wh1 wh2 wh0 wh1 wh2 wl0 wl1 | wl2 cA   cB  cC  0 0 0 0]
// so the tensor core sums xh*wh + xl*wh + xh*wl per channel (fp16 x fp16
// products are exact in fp32) plus, on the centre tap only,
// c' = 2048*cA + cB + cC = 2^j * s * (bias - A*) (s = sign(gamma); s = -1 also
// negates the weights; A* is the exact float64 decision point below). TMEM
// then holds D ~= 2^j * s * (acc - A*) and the bit is D >= 0. The dropped
// terms are <= 3 * 2^-22 * sum|x||w'| (+ 2^-25 absolute per subnormal part);
// the fp32 accumulation (exact products, addends aligned to the largest with
// guard bits and truncated: <= 17 * 2^-26 of the largest term per MMA) adds
// <= 2.3e-6 over 9 MMAs, ~3.3e-6 in total. Measured on B200 over 3.1 M
// (pixel, channel) pairs: max |D - D_exact| = 2.7e-7 of the scale below. So
// whenever
//     |D| <= margin = eps * (max|x|_tile * sum|w'_o| + |c'_o|) + absolute terms
// (eps = 8e-6, largest over channels) the epilogue recomputes acc
// in float64 in the reference's order (fconv_at order, generic.cu) from the
// tile's raw float64 input, which it still holds in shared memory, and
// compares it with the exact float64 decision point A*: the reference
// predicate is a composition of monotone IEEE operations in acc, so
// "y >= 0" is exactly "acc >= A*" (gamma > 0) or "acc <= A*" (gamma < 0),
// with A* found on the host by bisection over the float64 values. Non-finite
// or huge inputs make the tile's margin infinite: every bit of the tile is
// then decided in float64. Channels whose T* is unusable are always decided
// in float64. So every output bit equals the float64 decision.
//
// Tiles: 4 output rows x 128 columns of one frame. Twelve TMA row boxes
// (6 rows x 2 halves of 66 pixels x 3 channels) bring the (4+2) x 132-pixel
// float64 input (zero-filled outside the frame = the reference's zero
// padding) into shared memory; producer warps split it into
// the bf16 A strip (K-major, no swizzle, one 32-B row per pixel); tap (dy,dx)
// of output row b is the strip with the descriptor start moved by
// (b+dy)*130 + dx rows, so 9 MMAs per 128-pixel block read one strip (the
// same trick as conv_tc.cu). Weights (9 x 64 x 32 B) stay resident.
//
// Warp roles (576 threads, one CTA per SM): 0-7 epilogue (TMEM -> bits,
// float64 rechecks), 8-15 producers (fp64 -> bf16 split), 16 MMA issue +
// TMEM owner, 17 TMA loads.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace mbu {
namespace stc {

constexpr int MB = 4;                 // output rows (128-pixel M blocks) per tile
constexpr int TW = 128;               // output columns per tile
constexpr int P = TW + 2;             // strip pitch in pixels
constexpr int SROWS = MB + 2;         // strip rows
constexpr int Q = SROWS * P;          // 780 strip rows
constexpr int QP = 784;               // padded to a multiple of 8
constexpr int RAW_PAIRS = TW / 2 + 2; // 66 pixel pairs: x0-2 .. x0+129
constexpr int HALF_PX = RAW_PAIRS;    // 66 pixels per TMA row box
constexpr int BOX_DBL = 208;          // 198 doubles per box, padded to 128 B (TMA dst alignment)
constexpr int ROW_DBL = 2 * BOX_DBL;  // doubles per raw row
constexpr uint32_t RAW_BYTES = SROWS * 2 * HALF_PX * 24;  // 19008 bytes delivered per tile
constexpr uint32_t RAW_STRIDE = 20480;                    // 12 boxes x 1664 B, padded
constexpr uint32_t A_BYTES = QP * 32;                   // 25088
constexpr uint32_t A_STRIDE = 25600;
static_assert(A_BYTES <= A_STRIDE, "A stage overflow");
constexpr uint32_t B_BYTES = 9 * 64 * 32;               // 18432
constexpr uint32_t W64_BYTES = 64 * 27 * 8;             // 13824, reference-layout weights
constexpr uint32_t CH_BYTES = 64 * 32;                  // per-channel ChanConst
constexpr uint32_t CONST_BYTES = B_BYTES + W64_BYTES + CH_BYTES;  // one bulk copy
constexpr int ROW_ELEMS = 3 * RAW_PAIRS;                // 198 doubles per TMA row box
#ifndef STC_NRAW  // (staging depth as build flags for A/B runs: 3 + 5 / 3 + 4 measured no faster)
#define STC_NRAW 6
#endif
#ifndef STC_NA
#define STC_NA 2
#endif
constexpr int NRAW = STC_NRAW;        // raw fp64 stages (released by the epilogue)
constexpr int NA = STC_NA;            // fp16 A stages
constexpr int XRING = 8;              // per-tile max|x| slots
#ifndef STC_EPI_WARPS  // (A/B build flags: epilogue groups of 4 warps, producer warps)
#define STC_EPI_WARPS 8
#endif
#ifndef STC_PROD_WARPS
#define STC_PROD_WARPS 8
#endif
constexpr int NUM_EPI_WARPS = STC_EPI_WARPS, NUM_PROD_WARPS = STC_PROD_WARPS;
static_assert(NUM_EPI_WARPS % 4 == 0, "an epilogue group is one warp per TMEM lane quarter");
constexpr int EPI_GROUPS = NUM_EPI_WARPS / 4;
constexpr int PROD_WARP0 = NUM_EPI_WARPS, MMA_WARP = PROD_WARP0 + NUM_PROD_WARPS, LOAD_WARP = MMA_WARP + 1;
constexpr int NUM_THREADS = (LOAD_WARP + 1) * 32;
constexpr int EPI_THREADS = NUM_EPI_WARPS * 32, PROD_THREADS = NUM_PROD_WARPS * 32;
constexpr uint32_t OFF_B = 1024;
constexpr uint32_t OFF_W64 = OFF_B + B_BYTES;
constexpr uint32_t OFF_CH = OFF_W64 + W64_BYTES;
constexpr uint32_t OFF_RAW = 35840;
static_assert(OFF_RAW % 128 == 0 && RAW_STRIDE % 128 == 0 && (BOX_DBL * 8) % 128 == 0, "TMA dst alignment");
static_assert(OFF_B + CONST_BYTES <= OFF_RAW, "constant block overlaps the raw ring");
constexpr uint32_t OFF_A = OFF_RAW + NRAW * RAW_STRIDE;
constexpr uint32_t SMEM_BYTES = OFF_A + NA * A_STRIDE;
static_assert(SMEM_BYTES <= 227 * 1024, "stem tile does not fit in shared memory");
constexpr double EPS = 8e-6;          // relative margin (see above)
constexpr double ABS_ULP = 2.9802322387695312e-08;  // 2^-25: fp16 subnormal rounding

// per output channel: exact decision point and re-check margin
struct ChanConst {
  double astar;  // dir 0: bit = acc >= astar; dir 1: bit = acc <= astar
  double bias;   // float64 conv bias (reference order: added after the taps)
  float m1, m0;  // margin = xmax * m1 + m0
  int dir;       // 0 GE, 1 LE, 2 evaluate the reference predicate itself
  int pad;
};
static_assert(sizeof(ChanConst) == 32, "ChanConst layout");

struct Params {
  const double *x;
  int n, h, w, c_out;
  const double *w64, *bias64, *bn;  // reference-order recheck operands
  uint32_t *bits;
  int out_stride32, out_off32, out_groups;
  const uint8_t *b;                 // constant block: B operand (UMMA K-major), weights, table
  float m1, m0;                     // margin = xmax * m1 + m0
  unsigned long long force;         // channels always decided in float64
  unsigned long long chmask;        // real channels
  int col_tiles, row_tiles, num_tiles;
  uint32_t idesc;
  int early_release;                // release the accumulator after the tile's last TMEM load
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity), "r"(0x989680)
        : "memory");
  }
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;
  return d;
}
// nine taps of one 128-pixel block; the first overwrites the accumulator
__device__ __forceinline__ void umma9_f16(uint32_t d, uint64_t a0, uint64_t b0, uint64_t pp,
                                           uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred z, p, e;\n\t.reg .b64 a, b, r;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 z, 0, 0;\n\t"
      "setp.ne.b32 p, 1, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, z;\n\t"
      "add.s64 a, %1, 1;\n\t add.s64 b, %2, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %4, p;\n\t"
      "add.s64 a, %1, 2;\n\t add.s64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %4, p;\n\t"
      "add.s64 r, %1, %3;\n\t add.s64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], r, b, %4, p;\n\t"
      "add.s64 a, r, 1;\n\t add.s64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %4, p;\n\t"
      "add.s64 a, r, 2;\n\t add.s64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %4, p;\n\t"
      "add.s64 r, r, %3;\n\t add.s64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], r, b, %4, p;\n\t"
      "add.s64 a, r, 1;\n\t add.s64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %4, p;\n\t"
      "add.s64 a, r, 2;\n\t add.s64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %4, p;\n\t}" ::"r"(d),
      "l"(a0), "l"(b0), "l"(pp), "r"(idesc)
      : "memory");
}
__device__ __forceinline__ void umma_commit_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t (&v)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
      "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
      "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]),
        "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]),
        "=r"(v[38]), "=r"(v[39]), "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]),
        "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]), "=r"(v[48]), "=r"(v[49]),
        "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]),
        "=r"(v[56]), "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]),
        "=r"(v[62]), "=r"(v[63])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// bit i = (v[OFF + i] >= 0): complement of the sign bit
template <int OFF>
__device__ __forceinline__ uint32_t pack_nonneg(const uint32_t (&v)[64]) {
  uint32_t c[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int i = 7; i >= 0; --i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j] = __funnelshift_l(v[OFF + 8 * j + i], c[j], 1);
  const uint32_t lo = __byte_perm(c[0], c[1], 0x0040);
  const uint32_t hi = __byte_perm(c[2], c[3], 0x0040);
  return ~__byte_perm(lo, hi, 0x5410);
}
// float64 offset of raw pixel j (0..131, image x = x0 - 2 + j) in raw row r
__device__ __forceinline__ int raw_px(int r, int j) {
  return r * ROW_DBL + 3 * j + (j >= HALF_PX ? BOX_DBL - 3 * HALF_PX : 0);
}
// two floats -> packed fp16 pair (low = a), one F2FP
__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  const __half2 v = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t *>(&v);
}
__device__ __forceinline__ float2 unpack_h2(uint32_t w) {
  return __half22float2(*reinterpret_cast<const __half2 *>(&w));
}

// The reference's float64 decision for one (pixel, channel): acc in the
// reference's order from the tile's raw stage (rows b..b+2, pixels
// m+1..m+3) and the shared-memory float64 weights, then the exact decision
// point (or, for degenerate batchnorm parameters, the predicate itself).
__device__ __forceinline__ uint32_t exact_bit(const Params &p, const double *raw, const double *w64,
                                              const ChanConst &cc, int b, int m, int y, int x, int o) {
  double dot[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) {  // independent per-tap dots (3 chained fma each)
    const double *xr = raw + raw_px(b + t / 3, m + t % 3 + 1);
    const double *wr = w64 + (o * 9 + t) * 3;
    dot[t] = __fma_rn(xr[2], wr[2], __fma_rn(xr[1], wr[1], __fma_rn(xr[0], wr[0], 0.0)));
  }
  double acc = 0.0;
#pragma unroll
  for (int t = 0; t < 9; ++t) {  // reference order; zero padding adds nothing
    const int iy = y - 1 + t / 3, ix = x - 1 + t % 3;
    if (iy >= 0 && iy < p.h && ix >= 0 && ix < p.w) acc = __dadd_rn(acc, dot[t]);
  }
  if (p.bias64) acc = __dadd_rn(acc, cc.bias);
  if (cc.dir == 0) return acc >= cc.astar ? 1u : 0u;
  if (cc.dir == 1) return acc <= cc.astar ? 1u : 0u;
  const double gm = __ldg(p.bn + o), be = __ldg(p.bn + p.c_out + o);
  const double mu = __ldg(p.bn + 2 * p.c_out + o), sg = __ldg(p.bn + 3 * p.c_out + o);
  const double yv = __dadd_rn(__ddiv_rn(__dmul_rn(gm, __dsub_rn(acc, mu)), sg), be);
  return yv >= 0.0 ? 1u : 0u;
}

#ifdef STC_TIMELINE  // per-tile clock64 stamps of CTA 0 (-DSTC_TIMELINE build, printed by the launcher)
__device__ unsigned long long g_stl[64 * 16];
#define STL(slot)                                                                          \
  do {                                                                                     \
    if (blockIdx.x == 0 && lane == 0 && it < 64) g_stl[it * 16 + (slot)] = clock64();     \
  } while (0)
#else
#define STL(slot) \
  do {            \
  } while (0)
#endif
__global__ void __launch_bounds__(NUM_THREADS, 1)
    stem_tc_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
  // barrier slots
  uint64_t *full = bar;                 // [NA]   A stage ready (producers)
  uint64_t *empty = full + NA;          // [NA]   A stage free (MMA commit)
  uint64_t *rfull = empty + NA;         // [NRAW] raw stage landed (TMA)
  uint64_t *rempty = rfull + NRAW;      // [NRAW] raw stage free (epilogue)
  uint64_t *acc_full = rempty + NRAW;   // [2]
  uint64_t *acc_empty = acc_full + 2;   // [2]
  uint64_t *xfull = acc_empty + 2;      // [XRING]
  uint64_t *bfull = xfull + XRING;      // [1]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + 384);
  float *xm = reinterpret_cast<float *>(smem + 512);  // [XRING][NUM_PROD_WARPS]

  // (warp index through a shuffle: ptxas then treats it as warp-uniform, see conv_tc.cu)
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NA; ++i) {
      mbar_init(smem_u32(&full[i]), PROD_THREADS);
      mbar_init(smem_u32(&empty[i]), 1);
    }
    for (int i = 0; i < NRAW; ++i) {
      mbar_init(smem_u32(&rfull[i]), 1);
      mbar_init(smem_u32(&rempty[i]), EPI_THREADS);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&acc_full[i]), 1);
      mbar_init(smem_u32(&acc_empty[i]), EPI_THREADS);
    }
    for (int i = 0; i < XRING; ++i) mbar_init(smem_u32(&xfull[i]), NUM_PROD_WARPS);
    mbar_init(smem_u32(bfull), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int per_frame = p.row_tiles * p.col_tiles;

  if (warp == LOAD_WARP) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
      const uint32_t bb = smem_u32(bfull);
      mbar_expect_tx(bb, CONST_BYTES);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(smem + OFF_B)),
          "l"(p.b), "r"(CONST_BYTES), "r"(bb)
          : "memory");
      int rs = 0, rph = 0, it = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
        const int nb = t / per_frame, r = t - nb * per_frame;
        const int ty = r / p.col_tiles, tx = r - ty * p.col_tiles;
        mbar_wait(smem_u32(&rempty[rs]), rph ^ 1);
        STL(0);
        const uint32_t fb = smem_u32(&rfull[rs]);
        mbar_expect_tx(fb, RAW_BYTES);
        const uint32_t dst0 = smem_u32(smem + OFF_RAW + rs * RAW_STRIDE);
        const int e0 = 3 * (tx * TW - 2);
#pragma unroll
        for (int rr = 0; rr < SROWS; ++rr)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh)
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst0 + (rr * 2 + hh) * BOX_DBL * 8),
                "l"(&tmap), "r"(e0 + hh * ROW_ELEMS), "r"(ty * MB - 1 + rr), "r"(nb), "r"(fb)
                : "memory");
        if (++rs == NRAW) {
          rs = 0;
          rph ^= 1;
        }
      }
    }
    __syncwarp();
  } else if (warp == MMA_WARP) {
    mbar_wait(smem_u32(bfull), 0);
    const uint64_t a_desc0 = umma_desc(smem_u32(smem + OFF_A), QP * 16, 128);
    const uint64_t b_desc0 = umma_desc(smem_u32(smem + OFF_B), 64 * 16, 128);
    int s = 0, ph = 0, it = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
      const int ab = it & 1;
      STL(1);
      mbar_wait(smem_u32(&acc_empty[ab]), ((it >> 1) & 1) ^ 1);
      STL(2);
      mbar_wait(smem_u32(&full[s]), ph);
      STL(3);
      tc_fence_after();
      const uint64_t a_s = a_desc0 + uint64_t((s * A_STRIDE) >> 4);
#pragma unroll
      for (int b = 0; b < MB; ++b)
        umma9_f16(tmem + uint32_t(ab * 256 + b * 64), a_s + uint64_t(b * P), b_desc0, P, p.idesc);
      umma_commit_elect(smem_u32(&empty[s]));
      umma_commit_elect(smem_u32(&acc_full[ab]));
      STL(4);
      if (++s == NA) {
        s = 0;
        ph ^= 1;
      }
    }
    __syncwarp();
  } else if (warp >= PROD_WARP0) {
    // ============ producers: raw fp64 -> bf16 (hi, lo) strip ============
    const int pt = threadIdx.x - PROD_WARP0 * 32;
    int s = 0, ph = 0, rs = 0, rph = 0, it = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
      if (warp == PROD_WARP0) STL(5);
      mbar_wait(smem_u32(&rfull[rs]), rph);
      if (warp == PROD_WARP0) STL(6);
      mbar_wait(smem_u32(&empty[s]), ph ^ 1);
      if (warp == PROD_WARP0) STL(7);
      const double *raw = reinterpret_cast<const double *>(smem + OFF_RAW + rs * RAW_STRIDE);
      const uint32_t a0 = smem_u32(smem + OFF_A + s * A_STRIDE);
      const uint32_t a1 = a0 + QP * 16;
      float amax = 0.f;
      for (int q = pt; q < Q; q += PROD_THREADS) {
        const int r = q / P, c = q - r * P;
        const double *xr = raw + raw_px(r, c + 1);
        const float f0 = float(xr[0]), f1 = float(xr[1]), f2 = float(xr[2]);
        const float ax = fmaxf(fmaxf(fabsf(f0), fabsf(f1)), fabsf(f2));
        // non-finite or beyond fp16: infinite margin (every bit of the tile exact)
        amax = fmaxf(amax, ax <= 6e4f ? ax : __int_as_float(0x7f800000));  // fp16 range
        // x ~ xh + xl: xh = fp16(float(x)), xl = fp16(float(x) - xh) (exact residual)
        const uint32_t w0 = pack_h2(f0, f1);              // xh0 xh1
        const uint32_t h2 = pack_h2(f2, 2048.0f);         // xh2 2048
        const float2 g01 = unpack_h2(w0), g2 = unpack_h2(h2);
        const float r0 = f0 - g01.x, r1 = f1 - g01.y, r2 = f2 - g2.x;
        const uint32_t w1 = (h2 & 0xFFFFu) | (pack_h2(r0, r0) << 16);  // xh2 xl0
        const uint32_t w2 = pack_h2(r1, r2);              // xl1 xl2
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a0 + q * 16), "r"(w0), "r"(w1),
                     "r"(w2), "r"(w0)
                     : "memory");
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a1 + q * 16), "r"(h2),
                     "r"(0x3C003C00u), "r"(0u), "r"(0u)
                     : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(smem_u32(&full[s]));
      if (warp == PROD_WARP0) STL(8);
      const uint32_t wmax = __reduce_max_sync(0xffffffffu, __float_as_uint(amax));
      if (lane == 0) {
        xm[(it & (XRING - 1)) * NUM_PROD_WARPS + (warp - PROD_WARP0)] = __uint_as_float(wmax);
        mbar_arrive(smem_u32(&xfull[it & (XRING - 1)]));
      }
      if (++s == NA) {
        s = 0;
        ph ^= 1;
      }
      if (++rs == NRAW) {
        rs = 0;
        rph ^= 1;
      }
    }
  } else {
    // ============ epilogue: TMEM -> bits (+ float64 rechecks) ============
    const int quarter = warp & 3, group = warp >> 2;
    const int m = quarter * 32 + lane;
    const uint32_t lane_base = tmem + (uint32_t(quarter * 32) << 16);
    const uint32_t cm0 = uint32_t(p.chmask), cm1 = uint32_t(p.chmask >> 32);
    const double *w64 = reinterpret_cast<const double *>(smem + OFF_W64);
    const ChanConst *ch = reinterpret_cast<const ChanConst *>(smem + OFF_CH);
    int rs = 0, rph = 0, it = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
      const int ab = it & 1;
      const int nb = t / per_frame, r = t - nb * per_frame;
      const int ty = r / p.col_tiles, tx = r - ty * p.col_tiles;
      const int slot = it & (XRING - 1);
      if (warp == 0) STL(9);
      mbar_wait(smem_u32(&xfull[slot]), (it >> 3) & 1);
      float xmax = 0.f;
#pragma unroll
      for (int i = 0; i < NUM_PROD_WARPS; ++i) xmax = fmaxf(xmax, xm[slot * NUM_PROD_WARPS + i]);
      const float margin = fmaf(xmax, p.m1, p.m0);
      if (it == 0) mbar_wait(smem_u32(bfull), 0);  // channel tables (shared memory)
      if (warp == 0) STL(10);
      mbar_wait(smem_u32(&acc_full[ab]), (it >> 1) & 1);
      if (warp == 0) STL(11);
      tc_fence_after();
      mbar_wait(smem_u32(&rfull[rs]), rph);  // orders the TMA-written input for the rechecks
      const double *raw = reinterpret_cast<const double *>(smem + OFF_RAW + rs * RAW_STRIDE);
      // block b of tile it goes to group (it * MB + b) % EPI_GROUPS
      const int b_first = (group + EPI_GROUPS - (it * MB) % EPI_GROUPS) % EPI_GROUPS;
      const int b_last = b_first + (MB - 1 - b_first) / EPI_GROUPS * EPI_GROUPS;
#pragma unroll 1
      for (int b = b_first; b < MB; b += EPI_GROUPS) {
        uint32_t v[64];
        tmem_ld64(lane_base + uint32_t(ab * 256 + b * 64), v);
        // the accumulator is in registers once the group's last block is
        // loaded: free it for the MMA of tile it + 2 before the float64
        // re-decisions, which then stay off the tensor core's critical path
        if (p.early_release && b == b_last) {
          tc_fence_before();
          mbar_arrive(smem_u32(&acc_empty[ab]));
        }
        const int y = ty * MB + b, x = tx * TW + m;
        if (y < p.h && x < p.w) {
          float mn = __int_as_float(0x7f800000);
#pragma unroll
          for (int i = 0; i < 64; ++i) mn = fminf(mn, fabsf(__uint_as_float(v[i])));
          uint32_t w0 = pack_nonneg<0>(v), w1 = pack_nonneg<32>(v);
          if (!(mn > margin) || p.force) {
            // candidates: channels under their OWN margin (the uniform test above
            // uses the largest; per channel it is ~2.4x tighter on the bench
            // model), via the sign bit of |v| - margin_o; each is re-decided in
            // float64
            uint32_t c0 = 0u, c1 = 0u;
#pragma unroll
            for (int i = 31; i >= 0; --i) {
              const float ma = fmaf(xmax, ch[i].m1, ch[i].m0), mb = fmaf(xmax, ch[32 + i].m1, ch[32 + i].m0);
              c0 = __funnelshift_l(__float_as_uint(fabsf(__uint_as_float(v[i])) - ma), c0, 1);
              c1 = __funnelshift_l(__float_as_uint(fabsf(__uint_as_float(v[32 + i])) - mb), c1, 1);
            }
            // a non-finite tile (infinite margin, possibly NaN accumulators whose
            // difference has no meaningful sign) re-decides every channel
            unsigned long long um = margin < 3.0e38f ? (c0 | (unsigned long long)c1 << 32) : ~0ull;
            um = (um | p.force) & p.chmask;
            while (um) {
              const int o = __ffsll(um) - 1;
              um &= um - 1;
              const uint32_t bit = exact_bit(p, raw, w64, ch[o], b, m, y, x, o);
              if (o < 32)
                w0 = (w0 & ~(1u << o)) | (bit << o);
              else
                w1 = (w1 & ~(1u << (o - 32))) | (bit << (o - 32));
            }
          }
          w0 &= cm0;
          w1 &= cm1;
          uint32_t *dst = p.bits + ((int64_t(nb) * p.h + y) * p.w + x) * p.out_stride32 + p.out_off32;
          if (p.out_groups == 4 && ((p.out_stride32 | p.out_off32) & 3) == 0) {
            *reinterpret_cast<uint4 *>(dst) = make_uint4(w0, w1, 0u, 0u);
          } else {
            for (int g = 0; g < p.out_groups; ++g) dst[g] = g == 0 ? w0 : g == 1 ? w1 : 0u;
          }
        }
      }
      if (warp == 0) STL(12);
      if (warp == 4) STL(13);
      if (!p.early_release || b_first >= MB) {
        tc_fence_before();
        mbar_arrive(smem_u32(&acc_empty[ab]));
      }
      mbar_arrive(smem_u32(&rempty[rs]));
      if (++rs == NRAW) {
        rs = 0;
        rph ^= 1;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512)
                 : "memory");
  }
}

}  // namespace stc

// --------------------------------------------------------------------------
// host side
// --------------------------------------------------------------------------
struct StemTc {
  uint8_t *d_b = nullptr;  // constant block (B operand | float64 weights | channel table)
  float m1 = 0.f, m0 = 0.f;
  unsigned long long force = 0ull, chmask = 0ull;
};

static uint16_t host_h(double v) {  // float64 -> float32 -> fp16 (round to nearest even)
  const __half h = __float2half_rn(float(v));
  return *reinterpret_cast<const uint16_t *>(&h);
}
static double host_h_val(uint16_t b) {
  return double(__half2float(*reinterpret_cast<const __half *>(&b)));
}

// The reference predicate y = gamma*((acc + 0) - mean)/sigma + beta >= 0
// (layers.py:392-395), evaluated step by step in IEEE float64 (no
// contraction: every intermediate is stored).
static bool bn_pred(double acc, double g, double be, double mu, double sg) {
  volatile double pre = acc + 0.0;
  volatile double d = pre - mu;
  volatile double t = g * d;
  volatile double q = t / sg;
  volatile double y = q + be;
  return y >= 0.0;
}
static int64_t okey(double v) {  // order-preserving integer key of a float64
  int64_t k;
  std::memcpy(&k, &v, 8);
  return k >= 0 ? k : int64_t(0x8000000000000000ull) - k - 1;
}
static double from_okey(int64_t k) {
  const int64_t b = k >= 0 ? k : int64_t(0x8000000000000000ull) - k - 1;
  double v;
  std::memcpy(&v, &b, 8);
  return v;
}
// Exact decision point of a monotone predicate: smallest (rising) / largest
// (falling) float64 for which it holds. Returns false if the predicate does
// not switch once between -inf and +inf (degenerate parameters).
static bool decision_point(double g, double be, double mu, double sg, bool rising, double &out) {
  const double inf = INFINITY;
  int64_t lo = okey(-inf), hi = okey(inf);
  const bool plo = bn_pred(-inf, g, be, mu, sg), phi = bn_pred(inf, g, be, mu, sg);
  if (rising ? (plo || !phi) : (!plo || phi)) return false;
  // invariant: pred(lo) = !rising, pred(hi) = rising (the key range spans > 2^63: unsigned math)
  while (uint64_t(hi) - uint64_t(lo) > 1) {
    const int64_t mid = int64_t(uint64_t(lo) + (uint64_t(hi) - uint64_t(lo)) / 2);
    if (bn_pred(from_okey(mid), g, be, mu, sg) == rising)
      hi = mid;
    else
      lo = mid;
  }
  out = from_okey(rising ? hi : lo);
  // spot-check monotonicity around the point
  for (int64_t k = -4; k <= 4; ++k) {
    const int64_t kk = (rising ? hi : lo) + k;
    if (kk <= okey(-inf) || kk >= okey(inf)) continue;
    const bool pv = bn_pred(from_okey(kk), g, be, mu, sg);
    const bool want = rising ? (kk >= hi) : (kk <= lo);
    if (pv != want) return false;
  }
  return true;
}

int stem_tc_prepare(mbu_fconv *fc, const double *w, const double *bias, const double *bn, double eps) {
  fc->stem_tc = 0;
  if (!(fc->kh == 3 && fc->kw == 3 && fc->stride == 1 && fc->pad == 1 && !fc->bits_input && bn &&
        fc->c_in == 3 && fc->c_out <= 64))
    return MBU_OK;
  const int co = fc->c_out;
  for (size_t i = 0; i < size_t(co) * 27; ++i)
    if (!std::isfinite(w[i]) || std::fabs(w[i]) > 1e30) return MBU_OK;
  if (bias)
    for (int o = 0; o < co; ++o)
      if (!std::isfinite(bias[o]) || std::fabs(bias[o]) > 1e30) return MBU_OK;
  StemTc k;
  // constant block: [B operand (fp16, [tap][khalf][n][8])][float64 weights][ChanConst x 64]
  std::vector<uint8_t> blob(stc::CONST_BYTES, 0);
  auto *bm = reinterpret_cast<uint16_t *>(blob.data());
  auto *w64 = reinterpret_cast<double *>(blob.data() + stc::B_BYTES);
  auto *chc = reinterpret_cast<stc::ChanConst *>(blob.data() + stc::B_BYTES + stc::W64_BYTES);
  // weight scale 2^j (exact): max|w'| in [2^12, 2^13)
  double wmax = 0.0;
  for (size_t i = 0; i < size_t(co) * 27; ++i) wmax = std::max(wmax, std::fabs(w[i]));
  const double scale = wmax > 0.0 ? std::ldexp(1.0, 12 - std::ilogb(wmax)) : 1.0;
  double mmax1 = 0.0, mmax0 = 0.0;
  for (int o = 0; o < 64; ++o) {
    double c = -6e4, sgn = 1.0;  // padding columns: far below any margin, masked out anyway
    bool use_w = false;
    stc::ChanConst cc{};
    cc.dir = 2;
    if (o < co) {
      k.chmask |= 1ull << o;
      for (int i = 0; i < 27; ++i) w64[o * 27 + i] = w[size_t(o) * 27 + i];
      const double g = bn[o], be = bn[co + o], mu = bn[2 * co + o];
      const double sigma = std::sqrt(bn[3 * co + o] + eps);
      const double b0 = bias ? bias[o] : 0.0;
      cc.bias = b0;
      double astar = 0.0;
      if (g == 0.0) {
        c = be >= 0.0 ? 6e4 : -6e4;  // constant (non-finite acc -> exact via the tile margin)
      } else if (decision_point(g, be, mu, sigma, g > 0.0, astar) && std::isfinite(astar) &&
                 std::fabs(scale * (b0 - astar)) < 1e8) {
        sgn = g > 0 ? 1.0 : -1.0;
        cc.dir = g > 0 ? 0 : 1;
        cc.astar = astar;
        c = scale * sgn * (b0 - astar);
        use_w = true;
      } else {
        k.force |= 1ull << o;  // always decided by the reference predicate
        c = -6e4;             // (keeps the filter quiet; the force mask handles it)
      }
      if (use_w) {
        double s1 = 0.0;
        for (int i = 0; i < 27; ++i) s1 += scale * std::fabs(w[size_t(o) * 27 + i]);
        // margin = xmax * m1 + m0 (scaled units), see the header comment
        const double m1 = stc::EPS * s1 + 27 * stc::ABS_ULP;
        const double m0 = stc::EPS * std::fabs(c) + stc::ABS_ULP * (s1 + 3.0) + 1e-30;
        cc.m1 = float(m1 * (1 + 1e-6));
        cc.m0 = float(m0 * (1 + 1e-6));
        mmax1 = std::max(mmax1, double(cc.m1));
        mmax0 = std::max(mmax0, double(cc.m0));
      } else {
        cc.m1 = 0.f;  // constant or forced channel: never a margin candidate (the
        cc.m0 = 0.f;  // force mask and the non-finite tile path still re-decide it)
      }
    }
    chc[o] = cc;
    // c' = 2048*cA + cB + cC (A slots 9..11 hold 2048, 1, 1)
    const uint16_t ca = host_h(c / 2048.0);
    double rest = c - 2048.0 * host_h_val(ca);
    const uint16_t cb = host_h(rest);
    rest -= host_h_val(cb);
    const uint16_t cc3 = host_h(rest);
    for (int t = 0; t < 9; ++t) {
      uint16_t wh[3] = {0, 0, 0}, wl[3] = {0, 0, 0};
      if (use_w)
        for (int ci = 0; ci < 3; ++ci) {
          const double v = scale * sgn * w[(size_t(o) * 9 + t) * 3 + ci];
          wh[ci] = host_h(v);
          wl[ci] = host_h(v - host_h_val(wh[ci]));
        }
      uint16_t *k0 = &bm[((size_t(t) * 2 + 0) * 64 + o) * 8];
      uint16_t *k1 = &bm[((size_t(t) * 2 + 1) * 64 + o) * 8];
      const uint16_t row0[8] = {wh[0], wh[1], wh[2], wh[0], wh[1], wh[2], wl[0], wl[1]};
      for (int i = 0; i < 8; ++i) k0[i] = row0[i];
      k1[0] = wl[2];
      if (t == 4) {
        k1[1] = ca;
        k1[2] = cb;
        k1[3] = cc3;
      }
    }
  }
  k.m1 = float(mmax1);
  k.m0 = float(mmax0);
  MBU_TRY(check_cuda(cudaMalloc(&k.d_b, blob.size()), "alloc stem tc constants"));
  MBU_TRY(check_cuda(cudaMemcpy(k.d_b, blob.data(), blob.size(), cudaMemcpyHostToDevice),
                     "upload stem tc constants"));
  fc->h_stem_tc = new StemTc(k);
  fc->stem_tc = 1;
  return MBU_OK;
}

void stem_tc_free(mbu_fconv *fc) {
  auto *k = static_cast<StemTc *>(fc->h_stem_tc);
  if (k) cudaFree(k->d_b);
  delete k;
  fc->h_stem_tc = nullptr;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// 4-D u32 tiled tensor map (conv_tc.cu's raw activation boxes)
bool make_tmap_u32_4d(void *tmap, const void *base, const uint64_t dims[4], const uint64_t strides[3],
                      const uint32_t box[4]) {
  if (!encode_fn()) return false;
  const cuuint64_t d[4] = {dims[0], dims[1], dims[2], dims[3]};
  const cuuint64_t st[3] = {strides[0], strides[1], strides[2]};
  const cuuint32_t bx[4] = {box[0], box[1], box[2], box[3]};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return encode_fn()(static_cast<CUtensorMap *>(tmap), CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<void *>(base),
                     d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool stem_tc_usable(const mbu_fconv *fc, const double *x, int w) {
  return fc->stem_tc && (w % 2) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 && encode_fn();
}

int launch_stem_tc(const mbu_fconv *fc, const double *x, int n, int h, int w, uint64_t *bits,
                   int out_stride, int out_offset, cudaStream_t st) {
  const auto &k = *static_cast<const StemTc *>(fc->h_stem_tc);
  CUtensorMap tmap;
  const cuuint64_t dims[3] = {cuuint64_t(w) * 3, cuuint64_t(h), cuuint64_t(n)};
  const cuuint64_t strides[2] = {cuuint64_t(w) * 24, cuuint64_t(h) * w * 24};
  const cuuint32_t box[3] = {stc::ROW_ELEMS, 1, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(x), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MBU_ERR_CUDA, "cuTensorMapEncodeTiled failed for the stem input");
  stc::Params p{};
  p.x = x;
  p.n = n;
  p.h = h;
  p.w = w;
  p.c_out = fc->c_out;
  p.w64 = fc->d_w;
  p.bias64 = fc->d_bias;
  p.bn = fc->d_bn;
  p.bits = reinterpret_cast<uint32_t *>(bits);
  p.out_stride32 = out_stride * 2;
  p.out_off32 = out_offset * 2;
  p.out_groups = ((fc->c_out + 127) / 128) * 4;
  p.b = k.d_b;
  p.m1 = k.m1;
  p.m0 = k.m0;
  p.force = k.force;
  static const bool late = std::getenv("MBU_STEM_LATE_RELEASE") != nullptr;  // (A/B)
  p.early_release = late ? 0 : 1;
  p.chmask = k.chmask;
  p.col_tiles = (w + stc::TW - 1) / stc::TW;
  p.row_tiles = (h + stc::MB - 1) / stc::MB;
  const int64_t tiles = int64_t(n) * p.row_tiles * p.col_tiles;
  if (tiles == 0) return MBU_OK;
  if (tiles > 0x7FFFFFFF) return fail(MBU_ERR_SHAPE, "stem grid too large");
  p.num_tiles = int(tiles);
  // f32 accumulate, A and B fp16, K-major, N = 64, M = 128
  p.idesc = (1u << 4) | (uint32_t(64 >> 3) << 17) | (uint32_t(128 >> 4) << 24);
  static bool configured = false;
  if (!configured) {
    MBU_TRY(check_cuda(cudaFuncSetAttribute(stc::stem_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            int(stc::SMEM_BYTES)),
                       "cudaFuncSetAttribute(stem_tc)"));
    configured = true;
  }
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = int(std::min<int64_t>(tiles, sms));
  stc::stem_tc_kernel<<<grid, stc::NUM_THREADS, stc::SMEM_BYTES, st>>>(tmap, p);
#ifdef STC_TIMELINE
  {
    unsigned long long h[64 * 16];
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(h, stc::g_stl, sizeof(h));
    const unsigned long long b0 = h[1];
    fprintf(stderr, "STEM TIMELINE (CTA 0; clocks from tile 0's MMA start)\n");
    fprintf(stderr, " it | load:rempty | mma: start accE full done | prod: start rfull empty done | epi0: start xfull accF done | epi4 done\n");
    for (int i = 0; i < 40; ++i) {
      const unsigned long long *r = h + i * 16;
      auto d = [&](int k) { return (long long)(r[k] ? r[k] - b0 : 0); };
      fprintf(stderr, "%3d | %6lld | %6lld %6lld %6lld %6lld | %6lld %6lld %6lld %6lld | %6lld %6lld %6lld %6lld | %6lld\n", i,
              d(0), d(1), d(2), d(3), d(4), d(5), d(6), d(7), d(8), d(9), d(10), d(11), d(12), d(13));
    }
  }
#endif
  return check_launch("stem_tc_kernel");
}

}  // namespace mbu
