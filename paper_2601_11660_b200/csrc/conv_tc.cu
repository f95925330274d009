// Masked-binary convolution as a persistent tcgen05 (UTCIMMA) implicit GEMM.
//
// Replaces conv_forward -> lower_conv_to_gemm -> bit_gemm ->
// xor_popcount_rows + apply_threshold (layers.py:258-313, :508-522,
// bitcore.py:265-294, kernels.py:82-91) and, with TAPS = 1 and a scatter
// epilogue, transposed_conv_forward (layers.py:316-352).
//
// Arithmetic. The reference computes, per output (pixel m, channel o),
//   masked: popc(a'^neg) - popc(a'^pos)      binary: k_true - 2 popc(a'^b')
// over packed lanes. Both equal the integer dot product
//   acc = sum_lanes a * w,  a = 2a'-1 in {-1,+1},  w in {-1,0,+1}
// where w = pos - neg (masked) or 2b'-1 on real lanes and 0 on pad lanes
// (binary). The tensor cores evaluate it exactly with kind::i8 (s32
// accumulation in TMEM; |acc| <= 9*c_in):
//   * pad_mode "neg_one" (out-of-bounds taps read -1, the zero-word gather of
//     layers.py:270): A holds the raw bits a' in {0,1} as u8 and
//     acc = 2*D - W with D = sum a'*w and W = sum w over the column (an
//     out-of-bounds tap has a' = 0, i.e. -1, consistently);
//   * pad_mode "zero" (out-of-bounds taps read 0, equal to the reference's
//     weight-sum correction, layers.py:306-312): A holds a in {-1,+1} as s8
//     (0 out of bounds) and acc = D.
// Weights are expanded once at upload into s8; activations stay bit-packed
// in HBM and are expanded in shared memory by producer warps.
//
// Fused threshold (layers.py:508-522) without a compare per value: before a
// tile's first MMA the epilogue warps tcgen05.st a per-column bias into the
// accumulator, and DIR_LE columns carry negated weights, so TMEM ends up
// holding D' = s*(D - D_T) with D_T the smallest (GE) / largest (LE) D that
// fires; constant codes get a bias beyond the reachable range. The output bit
// is then "D' >= 0", the complement of the sign bit. Trace mode recovers
// acc = f*(s*(D' - bias)) - W (f = 2 for u8 activations, 1 for s8).
//
// Implicit GEMM without im2col: the producers expand a halo'd strip of input
// rows (R+2 rows x TW+2 columns) ONCE per 32-channel chunk; the A operand of
// tap (dy, dx) is that same strip with the UMMA descriptor's start address
// moved by (dy-1)*P + (dx-1) rows of 16 B (K-major, no swizzle: one row is
// 16 B, so any pixel offset is a legal start). Nine MMAs read one strip.
//
// Persistent, warp-specialised (512 threads, one CTA per SM):
//   warps 0-7   epilogue: bias -> TMEM, TMEM -> sign bits -> HBM. The two
//               warps of a TMEM lane quarter split M-blocks (or column runs)
//   warps 8-13  producers: packed bits -> u8/s8 strips, raw words LA stages ahead
//   warp 14     one lane issues tcgen05.mma; owns TMEM alloc/dealloc
//   warp 15     one lane streams pre-arranged weight stages (cp.async.bulk)
// Smem stages cycle through full/empty mbarriers; two TMEM accumulator
// buffers (2 x 256 columns) let the epilogue of tile i overlap the MMAs of
// tile i+1.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

// largest FP4 bias-slab set kept resident in shared memory (32 B per GEMM
// column: 1024 output channels); launch falls back to kind::i8 if a geometry
// then leaves fewer than two pipeline stages
#ifndef MBU_FP4_SLAB_CAP
#define MBU_FP4_SLAB_CAP 32768
#endif
namespace mbu {
namespace tc {
#ifdef MBU_TIMELINE
__device__ unsigned long long g_timeline[64 * 12];
__device__ unsigned long long g_epi[64 * 16];
#define MMA_T(slot)                                                          \
  do {                                                                       \
    if (blockIdx.x == 0 && lane == 0 && it < 64 && (slot) < 16) g_epi[it * 16 + (slot)] = clock64(); \
  } while (0)
#define EPI_T(slot)                                                                                 \
  do {                                                                                              \
    if (blockIdx.x == 0 && warp == 0 && lane == 0 && it < 64) g_epi[it * 16 + (slot)] = clock64(); \
  } while (0)
#else
#define EPI_T(slot) \
  do {              \
  } while (0)
#define MMA_T(slot) \
  do {              \
  } while (0)
#endif

constexpr int BLOCK_M = 128;
constexpr int NUM_EPI_WARPS = 8;
// 16 warps = 4 per SM sub-partition: each thread may hold 128 registers
// (18 warps would cap the epilogue at 96 and make it spill)
constexpr int NUM_PROD_WARPS = 6;
constexpr int PROD_WARP0 = NUM_EPI_WARPS;
constexpr int MMA_WARP = PROD_WARP0 + NUM_PROD_WARPS;
constexpr int BLOAD_WARP = MMA_WARP + 1;
constexpr int NUM_THREADS = (BLOAD_WARP + 1) * 32;
constexpr int PROD_THREADS = NUM_PROD_WARPS * 32;
constexpr int EPI_THREADS = NUM_EPI_WARPS * 32;
constexpr int ACC_COLS = 256;   // one accumulator buffer
constexpr int FP4_COLS = 248;   // FP4: the last 8 TMEM columns hold the block scales
                                // (one-buffer mode: 2 * 248 + 8 = 504 accumulator columns)
constexpr int TMEM_COLS = 512;  // two buffers
constexpr int MAX_STAGES = 8;
constexpr int MAX_CHUNKS = 64;  // 32-lane chunks per pixel (2048 lanes)
constexpr int SMEM_HEADER = 1024;
constexpr int MIN_SMEM = 120 * 1024;  // > half an SM: exactly one CTA (and TMEM owner) per SM
// strip rows per producer thread per stage: Q <= 8*192 for the 3x3 conv, <= 3*192 for one tap
constexpr int prod_items(int taps) { return taps == 9 ? 8 : 3; }
// raw-bit stages in flight per producer thread (template LA): 4 for the 3x3
// conv (each stage feeds nine taps), 8 for 1x1 / tconv (one tap per stage)
constexpr int LA_CONV3 = 8, LA_TAP1 = 8;

struct Params {
  const uint32_t *x32;
  int n, h, w;              // A pixel grid (conv: = output grid)
  int x_stride32, x_off32;
  // split input (a concat planned without a copy): u32 words >= split32 of a
  // pixel come from x2_32 (pixel stride x2_stride32, offset 0; FP4: xmap2)
  const uint32_t *x2_32;
  int x2_stride32, split32;  // split32 = INT_MAX: one tensor
  int halo, P, Q, R, TW, row_mode, MB;
  uint32_t p_magic;         // ceil(2^32 / P): q / P == umulhi(q, p_magic) for q < 2^16
  uint32_t nt_magic, ct_magic, rt_magic;  // same for n_tiles, col_tiles, row_tiles (t < 2^24)
  int col_tiles, row_tiles, n_tiles, num_tiles;
  int u8_act;               // 1: A = bits as u8 {0,1} (neg_one); 0: s8 {-1,0,+1} (zero pad)
  int kc;                   // active 32-lane chunks per pixel
  int ks;                   // K stages per tile = kc / cps
  int vec;                  // raw chunks of a stage are consecutive, aligned words
  uint32_t a_chunk_bytes;   // A bytes of one chunk inside a stage (Q * 32)
  uint32_t b_pair_bytes;    // FP4 with CPS = 4: weight bytes of one chunk pair (9 taps x n_tile x 32 B)
  const int32_t *chunk_word;
  const int8_t *b;
  int n_tile;
  uint32_t b_stage_bytes, a_stage_bytes;
  uint32_t idesc;
  int stages;
  int c_out, c_out_pad, n_gemm;
  int tconv_s;              // 0 for conv
  int ho, wo;
  int32_t *acc;
  uint32_t *bits;
  int out_stride32, out_off32, out_groups;
  // shared-memory layout (byte offsets, computed on the host)
  uint32_t off_b, off_raw, off_runs, off_ones, off_slab, off_slabmap;
  int b_resident;           // all weights resident in smem (loaded once), no B stream
  int mma_bias;             // bias enters the accumulator by an MMA (ones x bias slab)
  uint32_t sf1, sf256;      // FP4: TMEM columns of the 2^0 block scales and of the bias MMA's
                            // A scales (2^0 for K 0-31, 2^8 for K 32-63)
  // FP4: raw activation blocks arrive by TMA (one box of 16 B x P x strip rows per stage)
  uint32_t off_rraw, rraw_bytes, rraw_box_bytes;
  int rraw_stages, raw_rows;
  int nbuf;                 // accumulator buffers: 2-3 (epilogue overlaps the next tiles) or 1 (long K, big M)
  int buf_cols;             // TMEM columns between accumulator buffers
  int n_slabs;
  const int8_t *bias_slab;  // [n_slabs][khalf][n_tile][16]: s8, sum(lo) + 127*sum(hi) = bias
  const int32_t *slab_of_nt;
  int32_t slab_small[16];   // slab_of_nt for n_tiles <= 16, read from the constant bank (an LDS
                            // in the MMA warp queues behind the tensor core's operand reads)
  const int32_t *col_bias;  // per GEMM column: TMEM init value
  const int32_t *col_sgn;   // per GEMM column: +-1
  const int32_t *col_w;     // per GEMM column: W (u8 mode) or 0
  // CTA pair (template PAIR): B rows held per CTA (n_tile / 2; n_tile alone),
  // spatial tiles per N tile, pair work items (n_tiles * ceil(n_spatial / 2))
  int b_rows;
  int n_spatial, n_pairs;
  // fused 1x1 float64 head (HeadFuse): the fast N = 64 epilogue turns each
  // pixel's 64 sign bits into its logit (nibble tables staged at off_head) and
  // writes logits + mask instead of the activation words
  double *head_logits;      // null: no head
  uint8_t *head_mask;
  const double *head_tab;   // [16][16] nibble partial sums
  const double *head_bias;  // 1 value, or null
  uint32_t off_head;
};

// ----------------------------------------------------------------- PTX glue
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
// try_wait with a suspend-time hint: the waiting thread is parked by the
// hardware until the phase flips (or ~10 ms), instead of re-issuing the wait
// and stealing issue slots from the producer / epilogue warps.
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity), "r"(0x989680)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// UMMA shared-memory descriptor: K-major, SWIZZLE_NONE, sm100 version 1.
// Canonical layout ((8,m),(16B,2)) : ((16B, SBO), (1, LBO)).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;
  return d;
}
// The MMA warp runs converged; elect.sync inside the asm picks the issuing
// lane, so ptxas emits bare UTCIMMAs on uniform registers instead of an
// ELECT/BRA.U.ANY loop around every MMA (the per-MMA issue cost is what
// bounds the N = 64 layers, whose MMAs take only 32 tensor cycles).
// Nine taps of one M block: A = the strip descriptor of the centre tap moved
// by (dy-1)*P + (dx-1) rows of 16 B, B = one weight slab per tap.
__device__ __forceinline__ void umma9_i8(uint32_t tmem_d, uint64_t a_c, uint64_t b0, uint64_t pp,
                                         uint64_t bs, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 am, ap, a, b;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, 1, 0;\n\t"
      "sub.s64 am, %1, %3;\n\t"
      "add.s64 ap, %1, %3;\n\t"
      "add.s64 a, am, -1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a, %2, %5, p;\n\t"
      "add.s64 b, %2, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], am, b, %5, p;\n\t"
      "add.s64 a, am, 1;\n\t"
      "add.s64 b, b, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a, b, %5, p;\n\t"
      "add.s64 a, %1, -1;\n\t"
      "add.s64 b, b, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a, b, %5, p;\n\t"
      "add.s64 b, b, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, b, %5, p;\n\t"
      "add.s64 a, %1, 1;\n\t"
      "add.s64 b, b, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a, b, %5, p;\n\t"
      "add.s64 a, ap, -1;\n\t"
      "add.s64 b, b, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a, b, %5, p;\n\t"
      "add.s64 b, b, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], ap, b, %5, p;\n\t"
      "add.s64 a, ap, 1;\n\t"
      "add.s64 b, b, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a, b, %5, p;\n\t}" ::"r"(tmem_d),
      "l"(a_c), "l"(b0), "l"(pp), "l"(bs), "r"(idesc)
      : "memory");
}
__device__ __forceinline__ void umma1_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, 1, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc)
      : "memory");
}
// kind::mxf4 (e2m1 operands, UE8M0 block scales read from TMEM): nine taps of
// one M block, same descriptor walk as umma9_i8
__device__ __forceinline__ void umma9_fp4(uint32_t tmem_d, uint64_t a_c, uint64_t b0, uint64_t pp,
                                          uint64_t bs, uint32_t idesc, uint32_t sf) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 am, ap, a, b;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, 1, 0;\n\t"
      "sub.s64 am, %1, %3;\n\t"
      "add.s64 ap, %1, %3;\n\t"
      "add.s64 a, am, -1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, %2, %5, [%6], [%6], p;\n\t"
      "add.s64 b, %2, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], am, b, %5, [%6], [%6], p;\n\t"
      "add.s64 a, am, 1;\n\t"
      "add.s64 b, b, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %5, [%6], [%6], p;\n\t"
      "add.s64 a, %1, -1;\n\t"
      "add.s64 b, b, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %5, [%6], [%6], p;\n\t"
      "add.s64 b, b, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, b, %5, [%6], [%6], p;\n\t"
      "add.s64 a, %1, 1;\n\t"
      "add.s64 b, b, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %5, [%6], [%6], p;\n\t"
      "add.s64 a, ap, -1;\n\t"
      "add.s64 b, b, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %5, [%6], [%6], p;\n\t"
      "add.s64 b, b, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], ap, b, %5, [%6], [%6], p;\n\t"
      "add.s64 a, ap, 1;\n\t"
      "add.s64 b, b, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %5, [%6], [%6], p;\n\t}" ::"r"(tmem_d),
      "l"(a_c), "l"(b0), "l"(pp), "l"(bs), "r"(idesc), "r"(sf)
      : "memory");
}
// one kind::mxf4 MMA from 32-bit descriptor halves. The caller keeps every
// address computation in 32-bit, warp-uniform arithmetic (the high words are
// constant and an offset never carries out of the 14-bit start field), so
// ptxas issues the MMA straight from uniform registers: a few UIADD3/UMOV per
// MMA instead of ~14 instructions of 64-bit vector adds, R2UR.BROADCAST and
// VOTEU. That matters because the MMA warp shares its SM sub-partition with
// ALU-bound epilogue warps: measured (tools/ubench_fp4, mxf4_strip_alu_noise)
// a 14-instruction issue path slows N = 64 MMAs from 48 to ~70 cycles.
__device__ __forceinline__ void mma_fp4(uint32_t d, uint32_t alo, uint32_t ahi, uint32_t blo, uint32_t bhi,
                                        uint32_t idesc, uint32_t sfa, uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 a, b;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %8, 0;\n\t"
      "mov.b64 a, {%1, %2};\n\t"
      "mov.b64 b, {%3, %4};\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %5, [%6], [%7], p;\n\t}" ::"r"(d),
      "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(sfa), "r"(sfb), "r"(acc)
      : "memory");
}
// one kind::mxf4 MMA (bias MMAs): acc = 0 overwrites, separate A / B scale columns
__device__ __forceinline__ void umma1_fp4(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t sfa, uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(sfa), "r"(sfb), "r"(acc)
      : "memory");
}
// overwrite form (accumulate = 0): the bias MMA that opens a tile
__device__ __forceinline__ void umma1_i8_first(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, 0, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc)
      : "memory");
}
__device__ __forceinline__ void umma_commit_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}
// ---- CTA pair (cta_group::2): the leader's MMAs read A rows 0-127 from its
// own shared memory and rows 128-255 from its peer's (same offset), B rows
// [0, N/2) from the leader and [N/2, N) from the peer, and write D rows to
// each CTA's own TMEM (checked by tools/ubench_pair.cu)
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the shared::cluster address of `addr` (a shared::cta offset) in CTA `rank`
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t caddr) {
  // (default .release.cta semantics, the form CUTLASS's ClusterBarrier::arrive uses:
  // .release.cluster compiles to a MEMBAR.GPU that waits for the epilogue's global stores)
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
__device__ __forceinline__ void mma_fp4_pair(uint32_t d, uint32_t alo, uint32_t ahi, uint32_t blo, uint32_t bhi,
                                             uint32_t idesc, uint32_t sfa, uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 a, b;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %8, 0;\n\t"
      "mov.b64 a, {%1, %2};\n\t"
      "mov.b64 b, {%3, %4};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], a, b, %5, [%6], [%7], p;\n\t}" ::"r"(d),
      "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(sfa), "r"(sfb), "r"(acc)
      : "memory");
}
// commit to the barrier at offset `bar` in both CTAs of the pair
__device__ __forceinline__ void umma_commit_pair(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          bar),
      "h"(uint16_t(3))
      : "memory");
}
template <bool PAIR>
__device__ __forceinline__ void mma_fp4_g(uint32_t d, uint32_t alo, uint32_t ahi, uint32_t blo, uint32_t bhi,
                                          uint32_t idesc, uint32_t sfa, uint32_t sfb, uint32_t acc) {
  if constexpr (PAIR) mma_fp4_pair(d, alo, ahi, blo, bhi, idesc, sfa, sfb, acc);
  else mma_fp4(d, alo, ahi, blo, bhi, idesc, sfa, sfb, acc);
}
template <bool PAIR>
__device__ __forceinline__ void commit_g(uint32_t bar) {
  if constexpr (PAIR) umma_commit_pair(bar);
  else umma_commit_elect(bar);
}
#define MBU_R32(v)                                                                             \
  "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),      \
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),        \
      "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),      \
      "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),      \
      "r"(v[29]), "r"(v[30]), "r"(v[31])
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// 64 consecutive accumulator columns of this thread's TMEM lane, one wait
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
// bit i = NOT sign(v[OFF + i]), i.e. (D' >= 0): four independent funnel-shift
// chains of 8 (one SHF per column) merged with byte permutes.
template <int OFF, int N>
__device__ __forceinline__ uint32_t pack_nonneg(const uint32_t (&v)[N]) {
  uint32_t c[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int i = 7; i >= 0; --i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j] = __funnelshift_l(v[OFF + 8 * j + i], c[j], 1);
  const uint32_t lo = __byte_perm(c[0], c[1], 0x0040);
  const uint32_t hi = __byte_perm(c[2], c[3], 0x0040);
  return ~__byte_perm(lo, hi, 0x5410);
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      MBU_R32(v)
      : "memory");
}

// 4 activation bits -> 4 bytes. u8 mode: bit -> 0x00/0x01. s8 mode: bit 1 ->
// 0x01 (+1), bit 0 -> 0xFF (-1).
__device__ __forceinline__ uint32_t spread4(uint32_t nib) { return (nib * 0x00204081u) & 0x01010101u; }
// u8 mode (mul 1, xr 0): 0x00 / 0x01; s8 mode (mul 0xFE, xr ~0): 0xFF / 0x01
__device__ __forceinline__ uint32_t exp4(uint32_t nib, uint32_t mul, uint32_t xr) {
  return (spread4(nib) * mul) ^ xr;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                       uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}

// 32 activation bits -> 32 e2m1 lanes (16 B) in the K order the weights are
// packed in (prepare_conv_tc, fp4_k_pos): lane i = m + 4n of the chunk lands in
// word m, nibble n, so every word is one shift and one mask of the input.
// u8 mode (neg_one padding): bit -> 1.0 (0x2) / 0; s8 mode (zero padding):
// bit -> +1.0 / -1.0 (0xA); keep = 0 (out of bounds) -> all lanes 0.
__device__ __forceinline__ uint4 fp4x32(uint32_t w, uint32_t keep, bool s8) {
  const uint32_t one = 0x22222222u & keep;
  if (!s8) return make_uint4((w << 1) & one, w & one, (w >> 1) & one, (w >> 2) & one);
  const uint32_t nw = ~w, sg = 0x88888888u & keep;
  return make_uint4(one | ((nw << 3) & sg), one | ((nw << 2) & sg), one | ((nw << 1) & sg), one | (nw & sg));
}

struct Tile {
  int nb, y0, x0, nt;
};
// exact quotient n / d with m = ceil(2^32 / d) when n * d < 2^32 (host-checked);
// d = 1 is encoded as m = 0
__device__ __forceinline__ int fdiv(int n, uint32_t m) {
  return m ? int(__umulhi(uint32_t(n), m)) : n;
}
__device__ __forceinline__ Tile decode_tile(const Params &p, int t) {
  Tile r;
  int q = fdiv(t, p.nt_magic);
  r.nt = t - q * p.n_tiles;
  t = q;
  q = fdiv(t, p.ct_magic);
  const int ct = t - q * p.col_tiles;
  t = q;
  q = fdiv(t, p.rt_magic);
  const int rt = t - q * p.row_tiles;
  r.nb = q;
  r.y0 = rt * p.R;
  r.x0 = ct * p.TW;
  return r;
}
// CTA-pair work item u: N tile u % n_tiles, spatial tiles 2v and 2v + 1
// (v = u / n_tiles) for ranks 0 and 1 -- one B operand for both halves of the
// M = 256 MMA. An odd last spatial tile gives rank 1 a copy of it (computed,
// never stored: valid = false).
__device__ __forceinline__ int pair_tile(const Params &p, int u, uint32_t rank, bool &valid) {
  const int v = fdiv(u, p.nt_magic);
  const int nt = u - v * p.n_tiles;
  const int sp = 2 * v + int(rank);
  valid = sp < p.n_spatial;
  return nt + p.n_tiles * min(sp, p.n_spatial - 1);
}
__device__ __forceinline__ int block_q0(const Params &p, int b) {
  return p.row_mode ? (b + p.halo) * p.P + p.halo : p.halo * p.P + p.halo + BLOCK_M * b;
}

// Epilogue work split. Every (M-block, column run) of a tile is handled by
// one of the two warps sharing a TMEM lane quarter: by block parity when the
// tile has >= 2 blocks, else by run parity. A run is a maximal range of
// 32-column groups that lands in one output pixel (a tconv tap).
struct Run {
  int g, len, tap, o0;
};
__device__ __forceinline__ Run run_at(const Params &p, int jt, int g, int groups, bool tconv) {
  Run r;
  r.g = g;
  const int j0 = jt + 32 * g;
  const int span = tconv ? p.c_out_pad : p.n_gemm;
  r.tap = tconv ? j0 / p.c_out_pad : 0;
  r.o0 = j0 - r.tap * p.c_out_pad;
  r.len = min(groups - g, (span - r.o0) / 32);
  if (j0 >= p.n_gemm) r.len = 0;
  return r;
}

// ------------------------------------------------------------------ kernel
// BLOCK_COMMIT (single-buffered long-K FP4 tiles): the last K stage commits
// every M block on its own barrier, so the epilogue starts on block 0 while
// the MMAs of the later blocks still run (-8% on those layers)
// PAIR (with FP4 + BLOCK_COMMIT, resident weights): a cluster of two CTAs
// runs M = 256 cta_group::2 MMAs issued by rank 0 -- each CTA expands its own
// tile's A strip and holds half of B, so every SM's tensor core reads 4 KB of
// A + N/2 x 32 B of B per MMA instead of 4 KB + N x 32 B (the shared-memory
// read rate is what bounds the N = 64 MMAs: 49 -> 43 clocks, ubench_pair).
// Producer and epilogue warps of both CTAs arrive on rank 0's full / acc_empty
// barriers (one arrive per warp); rank 0's commits multicast to both CTAs.
// Streamed weights: each CTA's weight warp loads its half of every B stage on
// its own full[s]; rank 1's (otherwise idle) MMA warp forwards each landed
// stage to rank 0's full[s].
template <int TAPS, bool TCONV, int LA, int CPS, bool FP4, bool BLOCK_COMMIT = false, bool PAIR = false>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    conv_tc_kernel(const __grid_constant__ Params p, const __grid_constant__ CUtensorMap xmap,
                   const __grid_constant__ CUtensorMap xmap2) {
  static_assert(!PAIR || (FP4 && BLOCK_COMMIT && CPS == 2), "CTA pairs: FP4 single-buffer tiles only");
  constexpr int RAW_STAGES = LA + 1;
  constexpr int PI = prod_items(TAPS);
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem);
  uint64_t *empty = full + MAX_STAGES;
  uint64_t *acc_full = empty + MAX_STAGES;
  // BLOCK_COMMIT: acc_full[b] / acc_empty[b] per M block of the single buffer
  // (block b's columns are drained and refilled on their own: the next tile's
  // MMAs into block 0 start while later blocks are still being drained)
  uint64_t *acc_empty = acc_full + 8;
  uint64_t *bres = acc_empty + 8;  // resident weights landed
  uint64_t *rfull = bres + 1;       // [8] FP4: raw box landed (TMA)
  uint64_t *rempty = rfull + 8;     // [8] FP4: raw box consumed (producers)
  uint64_t *sf_ready = rempty + 8;  // FP4: the block-scale TMEM columns are written
  uint64_t *pready = sf_ready + 1;  // PAIR (rank 0): the peer's resident weights landed
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(pready + 1);
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
  // work items: tiles (u = t) or, PAIR, tile pairs (pair_tile)
  const int w_first = PAIR ? int(blockIdx.x >> 1) : int(blockIdx.x);
  const int w_step = PAIR ? int(gridDim.x >> 1) : int(gridDim.x);
  const int w_limit = PAIR ? p.n_pairs : p.num_tiles;
  auto tile_of = [&](int u, bool &valid) -> int {
    if constexpr (PAIR) return pair_tile(p, u, rank, valid);
    valid = true;
    return u;
  };
  // arrive on rank 0's copy of a barrier: per warp under PAIR, else per thread
  auto arrive_lead = [&](uint64_t *bar) {
    if constexpr (PAIR) {
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive_cluster(mapa_shared(smem_u32(bar), 0));
    } else {
      mbar_arrive(smem_u32(bar));
    }
  };
  int32_t *chunk_s = reinterpret_cast<int32_t *>(smem + 512);  // MAX_CHUNKS words
  uint8_t *a_base = smem + SMEM_HEADER;
  uint8_t *b_base = smem + p.off_b;

  // warp index through a shuffle: ptxas then knows it is warp-uniform, so the
  // role branches below are uniform and the MMA warp's descriptor arithmetic
  // stays on the uniform datapath (no BRA.DIV / R2UR.BROADCAST per MMA)
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const int S = p.stages;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      // (PAIR: rank 0 counts both CTAs' producer warps and B stages; rank 1's
      // full[s] only tracks its own streamed B stage)
      mbar_init(smem_u32(&full[s]), PAIR ? (rank == 0 ? 2 * NUM_PROD_WARPS + (p.b_resident ? 0 : 2) : 1)
                                         : PROD_THREADS + (p.b_resident ? 0 : 1));
      mbar_init(smem_u32(&empty[s]), 1);
    }
    mbar_init(smem_u32(bres), 1);
    mbar_init(smem_u32(pready), 1);
    for (int i = 0; i < 8; ++i) {
      mbar_init(smem_u32(&rfull[i]), 1);
      mbar_init(smem_u32(&rempty[i]), PROD_THREADS);
    }
    {
      mbar_init(smem_u32(sf_ready), 128);
    }
    for (int i = 0; i < 8; ++i) mbar_init(smem_u32(&acc_full[i]), 1);
    // (BLOCK_COMMIT: a block is drained by the 4 warps of one epilogue half)
    for (int i = 0; i < 8; ++i)
      mbar_init(smem_u32(&acc_empty[i]), BLOCK_COMMIT ? (PAIR ? 2 * 4 : 4 * 32) : EPI_THREADS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < p.kc; i += blockDim.x) chunk_s[i] = p.chunk_word[i];
  // per-N-tile epilogue runs and per-column TMEM biases, staged once per CTA
  int4 *runs_s = reinterpret_cast<int4 *>(smem + p.off_runs);
  int32_t *bias_s = reinterpret_cast<int32_t *>(runs_s + p.n_tiles * 9);
  for (int i = threadIdx.x; i < p.n_tiles * p.n_tile; i += blockDim.x) bias_s[i] = p.col_bias[i];
  if (threadIdx.x < p.n_tiles) {  // runs_s[nt * 9] = (count), then up to 8 runs
    const int nt = threadIdx.x, groups = p.n_tile / 32;
    int g = 0, r = 0;
    while (g < groups && r < 8) {
      const Run rn = run_at(p, nt * p.n_tile, g, groups, TCONV);
      if (rn.len == 0) break;
      const int dy = TCONV ? rn.tap / p.tconv_s : 0;
      runs_s[nt * 9 + 1 + r++] = make_int4(rn.g, rn.len, rn.o0, (dy << 16) | (rn.tap - dy * p.tconv_s));
      g += rn.len;
    }
    // .y: every run starts on a 128-lane block and fills whole 4-group chunks
    // (or ends its tap, whose pad groups complete the chunk) -> chunked epilogue
    int chunked = TCONV ? 1 : 0;
    for (int i = 0; i < r; ++i) {
      const int4 rn = runs_s[nt * 9 + 1 + i];
      chunked &= (rn.z % 128 == 0) && (rn.y % 4 == 0 || rn.z / 32 + rn.y == p.c_out_pad / 32);
    }
    runs_s[nt * 9] = make_int4(r, chunked, 0, 0);
  }
  if (p.mma_bias) {  // ones slab (16 x 1, 16 x 127 per row) + bias slabs, read by the tensor core
    // (FP4: every entry e2m1 1.0; bias = sum(lo) + 256 * sum(hi), one K = 64 slab per N tile)
    uint4 *ones = reinterpret_cast<uint4 *>(smem + p.off_ones);
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
      ones[i] = FP4 ? make_uint4(0x22222222u, 0x22222222u, 0x22222222u, 0x22222222u)
                    : i < 128 ? make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u)
                              : make_uint4(0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu);
    uint4 *slab = reinterpret_cast<uint4 *>(smem + p.off_slab);
    // (PAIR: each CTA holds its B rows of every slab; the rank-major copy)
    const int slab_u4 = p.n_slabs * p.b_rows * 2;
    const uint4 *src = reinterpret_cast<const uint4 *>(p.bias_slab) + size_t(rank) * slab_u4;
    for (int i = threadIdx.x; i < slab_u4; i += blockDim.x) slab[i] = src[i];
    int32_t *smap = reinterpret_cast<int32_t *>(smem + p.off_slabmap);
    for (int i = threadIdx.x; i < p.n_tiles; i += blockDim.x) smap[i] = p.slab_of_nt[i];
    fence_proxy_async();
  }
  if (p.head_logits) {
    double2 *ht = reinterpret_cast<double2 *>(smem + p.off_head);
    const double2 *src = reinterpret_cast<const double2 *>(p.head_tab);
    for (int i = threadIdx.x; i < 16 * 16 / 2; i += blockDim.x) ht[i] = src[i];
  }
  if (warp == MMA_WARP) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  // (PAIR: also publishes both CTAs' barrier inits, ones and slabs cluster-wide)
  if constexpr (PAIR) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if constexpr (PAIR) {  // uniform block scales in both CTAs' TMEM before rank 0's first MMA
    if (warp < 4) {
      const uint32_t lq = tmem + (uint32_t(warp * 32) << 16);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(lq + p.sf1 + c), "r"(0x7F7F7F7Fu)
                     : "memory");
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(lq + p.sf256 + c), "r"(0x7F7F877Fu)
                     : "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
  } else if constexpr (FP4) {
    // uniform block scales: 4 columns of 2^0 and 4 of 2^8 (any scale layout reads one value)
    if (warp < 4) {
      const uint32_t lq = tmem + (uint32_t(warp * 32) << 16);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(lq + p.sf1 + c), "r"(0x7F7F7F7Fu)
                     : "memory");
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(lq + p.sf256 + c), "r"(0x7F7F877Fu)
                     : "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      mbar_arrive(smem_u32(sf_ready));  // (an mbarrier rather than a partial named
    } else if (warp == MMA_WARP) {      //  barrier: compute-sanitizer synccheck clean)
      mbar_wait(smem_u32(sf_ready), 0);
      tc_fence_after();
    }
  }

  if (warp >= PROD_WARP0 && warp < MMA_WARP) {
    // ============ producers: packed bits -> u8/s8 strips ============
    // Per tile, each thread caches the 32-bit word offset of its strip rows
    // (and an in-bounds mask); per stage it only adds the chunk's word index.
    // The loads of stage g+1 are issued before stage g is expanded.
    // Raw words travel global -> smem with cp.async (zero-filled when out of
    // bounds) LOOKAHEAD stages ahead of the expansion, so DRAM latency is
    // overlapped with the expansion and MMAs of earlier stages. Each thread
    // expands exactly the rows it copied, so cp.async.wait_group is the only
    // synchronisation needed. Per tile, each thread caches the 32-bit word
    // offsets of its strip rows and an in-bounds mask.
    const int pt = threadIdx.x - PROD_WARP0 * 32;
    const int strip_rows = p.R + 2 * p.halo;
    uint32_t *raw = reinterpret_cast<uint32_t *>(smem + p.off_raw);
    struct Cache {
      int t = -1;
      int off[PI];
      uint32_t inb = 0;
    };
    Cache ic, ec;  // issue-side and expand-side tile caches (keyed by work item)
    auto tile_offsets = [&](Cache &c, int u) {
      bool tv;
      const Tile tl = decode_tile(p, tile_of(u, tv));
      c.inb = 0;
#pragma unroll
      for (int j = 0; j < PI; ++j) {
        if (j * PROD_THREADS >= p.Q) break;  // (uniform: items past the strip do no work)
        const int q = pt + j * PROD_THREADS;
        const int rr = int(__umulhi(uint32_t(q), p.p_magic));
        const int iy = tl.y0 - p.halo + rr;
        const int ix = tl.x0 - p.halo + (q - rr * p.P);
        c.off[j] = (tl.nb * p.h + iy) * p.w + ix;  // pixel index (the stage picks the tensor)
        if (q < p.Q && rr < strip_rows && iy >= 0 && iy < p.h && ix >= 0 && ix < p.w) c.inb |= 1u << j;
      }
      c.t = u;
    };
    // stage g <-> (work item w_first + (g / ks) * w_step, chunks [cps*(g % ks), +cps))
    const int tiles_here = w_limit > w_first ? (w_limit - w_first + w_step - 1) / w_step : 0;
    const int n_stages_total = tiles_here * p.ks;
    constexpr int cps = CPS;
    const int slot_words = p.Q * cps;
    const uint32_t emul = p.u8_act ? 1u : 0xFEu, exr = p.u8_act ? 0u : 0xFFFFFFFFu;
    // incremental cursors (no integer division in the per-stage loop)
    int i_t = w_first, i_k = 0, i_slot = 0, i_g = 0;        // issue side
    int e_t = w_first, e_k = 0, e_slot = 0, s = 0, ph = 0;  // expand side
    auto issue = [&]() {
      if (i_g < n_stages_total) {
        if (i_t != ic.t) tile_offsets(ic, i_t);
        const int k0 = i_k * cps;
        const int cw = chunk_s[k0];  // (read once: the cp.async asm clobbers memory)
        // a stage's chunks lie in one 128-lane block, so in one tensor of a split input
        const bool sec = cw >= p.split32;
        const uint32_t *xb = sec ? p.x2_32 : p.x32;
        const int xs = sec ? p.x2_stride32 : p.x_stride32;
        const int xo = sec ? -p.split32 : p.x_off32;
        uint32_t *dst = raw + i_slot * slot_words;
#pragma unroll
        for (int j = 0; j < PI; ++j) {
        if (j * PROD_THREADS >= p.Q) break;  // (uniform: items past the strip do no work)
          const int q = pt + j * PROD_THREADS;
          if (q < p.Q) {
            const bool in = (ic.inb >> j) & 1;
            const uint32_t d = smem_u32(dst + q * cps);
            if constexpr (cps == 1) {
              const uint32_t *src = in ? xb + (ic.off[j] * xs + xo + cw) : p.x32;
              asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src),
                           "r"(in ? 4 : 0)
                           : "memory");
            } else if (p.vec) {  // cps consecutive words, one copy (zero-filled out of bounds)
              const uint32_t *src = in ? xb + (ic.off[j] * xs + xo + cw) : p.x32;
              if constexpr (cps == 4)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src),
                             "r"(in ? 16 : 0)
                             : "memory");
              else if constexpr (cps == 2)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src),
                             "r"(in ? 8 : 0)
                             : "memory");
              else
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src),
                             "r"(in ? 4 : 0)
                             : "memory");
            } else {
#pragma unroll
              for (int c = 0; c < cps; ++c) {
                const uint32_t *src = in ? xb + (ic.off[j] * xs + xo + chunk_s[k0 + c]) : p.x32;
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d + 4 * c), "l"(src),
                             "r"(in ? 4 : 0)
                             : "memory");
              }
            }
          }
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");  // (possibly empty) group
      ++i_g;
      if (++i_k == p.ks) {
        i_k = 0;
        i_t += w_step;
      }
      if (++i_slot == RAW_STAGES) i_slot = 0;
    };
    int rs = 0, rph = 0;  // FP4: raw box ring (TMA)
    if constexpr (!FP4) {
#pragma unroll 1
      for (int g = 0; g < LA; ++g) issue();
    }
    for (int g = 0; g < n_stages_total; ++g) {
      // FP4: this stage's chunk pair(s) (read before the waits, off the expansion's path);
      // CPS = 4 stages hold both pairs of one 128-lane block
      constexpr int PPS = FP4 ? CPS / 2 : 1;
      const int ca = FP4 ? chunk_s[2 * PPS * e_k] & 3 : 0, cb = FP4 ? chunk_s[2 * PPS * e_k + 1] & 3 : 0;
      const int ca2 = PPS > 1 ? chunk_s[2 * PPS * e_k + 2] & 3 : 0, cb2 = PPS > 1 ? chunk_s[2 * PPS * e_k + 3] & 3 : 0;
      if constexpr (!FP4) {
        issue();
        asm volatile("cp.async.wait_group %0;" ::"n"(LA) : "memory");  // group g landed
      } else {
        mbar_wait(smem_u32(&rfull[rs]), rph);
      }
      if (e_t != ec.t) tile_offsets(ec, e_t);
      const uint32_t *rw = FP4 ? reinterpret_cast<const uint32_t *>(smem + p.off_rraw + rs * p.rraw_bytes)
                               : raw + e_slot * slot_words;
#ifdef MBU_TIMELINE
      const unsigned long long tp0 = clock64();
#endif
      if (g >= S) mbar_wait(smem_u32(&empty[s]), ph ^ 1);
#ifdef MBU_TIMELINE
      const unsigned long long tp1 = clock64();
#endif
      const uint32_t a_st = smem_u32(a_base + size_t(s) * p.a_stage_bytes);
      // Branch-free expansion (independent rows interleave): out-of-bounds rows
      // were zero-filled by cp.async, which expands to 0 in u8 mode; s8 mode
      // masks them explicitly. Indices are clamped so every load is in range.
      const int qmax = p.Q - 1;
#ifdef ABL_NO_EXPAND
      if (false) {
#else
      if constexpr (FP4) {
#endif
        // two 32-lane chunks -> one K = 64 e2m1 row: chunk c fills core-matrix column c
        // raw box: 16 B (a 128-lane block) per strip pixel, pixels row-major
        const bool s8 = !p.u8_act;
        const int qbox = p.raw_rows * p.P - 1;
#pragma unroll
        for (int j = 0; j < PI; ++j) {
        if (j * PROD_THREADS >= p.Q) break;  // (uniform: items past the strip do no work)
          const int q = pt + j * PROD_THREADS;
          // one 16-B load of the pixel's 128-lane block (a warp reads 512 contiguous
          // bytes: 4 wavefronts), the stage's chunk words picked in registers --
          // two 4-B loads at a 16-B stride cost 8 conflicted wavefronts, and the
          // shared-memory pipe is the MMA's bottleneck here
          const uint4 r4 = *reinterpret_cast<const uint4 *>(rw + min(q, qbox) * 4);
          auto word = [&](int c) { return c == 0 ? r4.x : c == 1 ? r4.y : c == 2 ? r4.z : r4.w; };
          const uint32_t keep = ((ec.inb >> j) & 1) ? ~0u : 0u;  // out of bounds -> 0
          const uint4 e0 = fp4x32(word(ca), keep, s8), e1 = fp4x32(word(cb), keep, s8);
          if (q < p.Q) {
            const uint32_t a0 = a_st + q * 16;
            sts128(a0, e0.x, e0.y, e0.z, e0.w);
            sts128(a0 + p.Q * 16, e1.x, e1.y, e1.z, e1.w);
            if constexpr (PPS > 1) {  // the block's second pair: the stage's next A region
              const uint4 e2 = fp4x32(word(ca2), keep, s8), e3 = fp4x32(word(cb2), keep, s8);
              sts128(a0 + p.a_chunk_bytes, e2.x, e2.y, e2.z, e2.w);
              sts128(a0 + p.a_chunk_bytes + p.Q * 16, e3.x, e3.y, e3.z, e3.w);
            }
          }
        }
      } else if constexpr (cps == 1) {
        const uint32_t a0 = a_st;
        const uint32_t a1 = a0 + p.Q * 16;
        if (p.u8_act) {
#pragma unroll
          for (int j = 0; j < PI; ++j) {
        if (j * PROD_THREADS >= p.Q) break;  // (uniform: items past the strip do no work)
            const int q = pt + j * PROD_THREADS;
            const uint32_t b = rw[min(q, qmax)];
            const uint32_t v0 = spread4(b & 0xF), v1 = spread4((b >> 4) & 0xF), v2 = spread4((b >> 8) & 0xF),
                           v3 = spread4((b >> 12) & 0xF), v4 = spread4((b >> 16) & 0xF),
                           v5 = spread4((b >> 20) & 0xF), v6 = spread4((b >> 24) & 0xF), v7 = spread4(b >> 28);
            if (q < p.Q) {
              sts128(a0 + q * 16, v0, v1, v2, v3);
              sts128(a1 + q * 16, v4, v5, v6, v7);
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < PI; ++j) {
        if (j * PROD_THREADS >= p.Q) break;  // (uniform: items past the strip do no work)
            const int q = pt + j * PROD_THREADS;
            const uint32_t b = rw[min(q, qmax)];
            const bool in = (ec.inb >> j) & 1;
            const uint32_t mul = in ? 0xFEu : 0u, xr = in ? ~0u : 0u;  // a = 0 out of bounds (zero pad)
            const uint32_t v0 = exp4(b & 0xF, mul, xr), v1 = exp4((b >> 4) & 0xF, mul, xr),
                           v2 = exp4((b >> 8) & 0xF, mul, xr), v3 = exp4((b >> 12) & 0xF, mul, xr),
                           v4 = exp4((b >> 16) & 0xF, mul, xr), v5 = exp4((b >> 20) & 0xF, mul, xr),
                           v6 = exp4((b >> 24) & 0xF, mul, xr), v7 = exp4(b >> 28, mul, xr);
            if (q < p.Q) {
              sts128(a0 + q * 16, v0, v1, v2, v3);
              sts128(a1 + q * 16, v4, v5, v6, v7);
            }
          }
        }
      } else if (p.u8_act) {
        // u8 (the tconvs): out-of-bounds rows were zero-filled by cp.async and
        // expand to 0, so no mask -- one multiply and one mask per 4 lanes
#pragma unroll
        for (int j = 0; j < PI; ++j) {
          if (j * PROD_THREADS >= p.Q) break;  // (uniform: items past the strip do no work)
          const int q = pt + j * PROD_THREADS;
          if (q < p.Q) {
#pragma unroll
            for (int c = 0; c < cps; ++c) {
              const uint32_t a0 = a_st + c * p.a_chunk_bytes + q * 16;
              const uint32_t b = rw[q * cps + c];
              sts128(a0, spread4(b & 0xF), spread4((b >> 4) & 0xF), spread4((b >> 8) & 0xF),
                     spread4((b >> 12) & 0xF));
              sts128(a0 + p.Q * 16, spread4((b >> 16) & 0xF), spread4((b >> 20) & 0xF), spread4((b >> 24) & 0xF),
                     spread4(b >> 28));
            }
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < PI; ++j) {
        if (j * PROD_THREADS >= p.Q) break;  // (uniform: items past the strip do no work)
          const int q = pt + j * PROD_THREADS;
          if (q < p.Q) {
#pragma unroll
            for (int c = 0; c < cps; ++c) {
              const uint32_t a0 = a_st + c * p.a_chunk_bytes + q * 16;
              const uint32_t a1 = a0 + p.Q * 16;
              const uint32_t b = rw[q * cps + c];
              if ((ec.inb >> j) & 1) {
                sts128(a0, exp4(b & 0xF, emul, exr), exp4((b >> 4) & 0xF, emul, exr),
                       exp4((b >> 8) & 0xF, emul, exr), exp4((b >> 12) & 0xF, emul, exr));
                sts128(a1, exp4((b >> 16) & 0xF, emul, exr), exp4((b >> 20) & 0xF, emul, exr),
                       exp4((b >> 24) & 0xF, emul, exr), exp4(b >> 28, emul, exr));
              } else {
                sts128(a0, 0u, 0u, 0u, 0u);
                sts128(a1, 0u, 0u, 0u, 0u);
              }
            }
          }
        }
      }
      fence_proxy_async();
      arrive_lead(&full[s]);
      if constexpr (FP4) {
        mbar_arrive(smem_u32(&rempty[rs]));
        if (++rs == p.rraw_stages) {
          rs = 0;
          rph ^= 1;
        }
      }
#ifdef MBU_TIMELINE
      if (blockIdx.x == 0 && pt == 0 && g < 64) {
        g_timeline[g * 12 + 8] = tp0;
        g_timeline[g * 12 + 9] = tp1;
        g_timeline[g * 12 + 10] = clock64();
      }
#endif
      if (++e_k == p.ks) {
        e_k = 0;
        e_t += w_step;
      }
      if (++e_slot == RAW_STAGES) e_slot = 0;
      if (++s == S) {
        s = 0;
        ph ^= 1;
      }
    }
    if constexpr (!FP4) asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else if (warp == MMA_WARP) {
    // ============ MMA issue (accumulators pre-loaded with bias) ============
    // The whole warp walks the schedule (all values warp-uniform); one
    // elected lane issues (umma9_i8 / umma1_i8 / umma_commit_elect).
    if (PAIR && rank != 0) {  // the peer issues nothing: it reports its weights to rank 0
      if (p.b_resident) {
        mbar_wait(smem_u32(bres), 0);
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(pready), 0));
      } else {  // streamed B: forward each landed stage (local full[s]) to rank 0's full[s]
        const int n_g = (w_limit > w_first ? (w_limit - w_first + w_step - 1) / w_step : 0) * p.ks;
        int s = 0, ph = 0;
        for (int g = 0; g < n_g; ++g) {
          mbar_wait(smem_u32(&full[s]), ph);
          if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&full[s]), 0));
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    } else {
      const uint32_t sbo = 128;
      const uint32_t a_lbo = uint32_t(p.Q) * 16;
      const uint32_t b_lbo = uint32_t(p.b_rows) * 16;
      const uint64_t pp = uint64_t(p.P);                        // one strip row, in 16-B units
      const uint64_t bs = uint64_t(p.b_rows) * 2;               // one tap slab of B, in 16-B units
      const uint64_t a_desc0 = umma_desc(smem_u32(a_base), a_lbo, sbo);
      const uint64_t b_desc0 = umma_desc(smem_u32(b_base), b_lbo, sbo);
      const uint64_t ones_desc = umma_desc(smem_u32(smem + p.off_ones), 128 * 16, sbo);
      const uint64_t slab_desc0 = umma_desc(smem_u32(smem + p.off_slab), b_lbo, sbo);
      const int32_t *smap = reinterpret_cast<const int32_t *>(smem + p.off_slabmap);
      if (p.b_resident) mbar_wait(smem_u32(bres), 0);
      if (PAIR && p.b_resident) mbar_wait(smem_u32(pready), 0);
      int s = 0, ph = 0, it = 0, ab = 0, aph = 0;  // accumulator buffer ring: index, phase
      for (int t = w_first; t < w_limit; t += w_step, ++it) {
        // (PAIR: t is the work item; both tiles of the pair share its N tile)
        const int nt = t - fdiv(t, p.nt_magic) * p.n_tiles;
        // (read before the wait: a shared load issued behind the tensor core's
        // operand reads takes hundreds of cycles, keep it off the issue path)
        const int slab = p.mma_bias ? (p.n_tiles <= 16 ? p.slab_small[nt] : smap[nt]) : 0;
#ifdef MBU_TIMELINE
        unsigned long long tl0 = clock64();
#endif
        if constexpr (!BLOCK_COMMIT) mbar_wait(smem_u32(&acc_empty[ab]), aph);
#ifdef MBU_TIMELINE
        unsigned long long tl1 = clock64();
#endif
        tc_fence_after();
        const uint32_t d0 = tmem + uint32_t(ab * p.buf_cols);
        // bias = lo (K 0-31, A scale 1) + 256 * hi (K 32-63, A scale 2^8)
        const uint32_t sd = uint32_t(slab_desc0) + uint32_t(slab * p.b_rows * 2);
        if (FP4 && p.mma_bias && !BLOCK_COMMIT) {  // (BLOCK_COMMIT: per block, in the first K stage)
          for (int b = 0; b < p.MB; ++b)
            mma_fp4_g<PAIR>(d0 + uint32_t(b * p.n_tile), uint32_t(ones_desc), uint32_t(ones_desc >> 32), sd,
                            uint32_t(slab_desc0 >> 32), p.idesc, tmem + p.sf256, tmem + p.sf1, 0u);
        } else if (!FP4 && p.mma_bias) {
          const uint64_t sd = slab_desc0 + uint64_t(slab) * uint64_t(p.b_rows * 2);
          for (int b = 0; b < p.MB; ++b) umma1_i8_first(d0 + uint32_t(b * p.n_tile), ones_desc, sd, p.idesc);
        }
#ifdef MBU_TIMELINE
        unsigned long long tl_full = 0;
#endif
        MMA_T(0);
        for (int k = 0; k < p.ks; ++k) {
          mbar_wait(smem_u32(&full[s]), ph);
          if (k == 0) MMA_T(1);
#ifdef MBU_TIMELINE
          if (k == p.ks - 1) tl_full = clock64();
#endif
          tc_fence_after();
          // descriptors advance by address >> 4 (no carry out of the 14-bit field: smem < 256 KB)
          const uint64_t a_s = a_desc0 + uint64_t((size_t(s) * p.a_stage_bytes) >> 4);
          const uint64_t b_s =
              b_desc0 + uint64_t(((p.b_resident ? size_t(nt * p.ks + k) : size_t(s)) * p.b_stage_bytes) >> 4);
#ifdef ABL_NO_MMA9
          if (false) {
#else
          if constexpr (FP4) {
#endif
            // 32-bit uniform descriptor arithmetic (see mma_fp4)
            const uint32_t a_hi = uint32_t(a_desc0 >> 32), b_hi = uint32_t(b_desc0 >> 32);
            const uint32_t a_lo = uint32_t(a_s), b_lo = uint32_t(b_s), P32 = uint32_t(p.P);
            const uint32_t bs32 = uint32_t(bs), sf = tmem + p.sf1;
            for (int b = 0; b < p.MB; ++b) {
              const uint32_t d = d0 + uint32_t(b * p.n_tile);
              if constexpr (BLOCK_COMMIT) {
                if (k == 0) {  // block b's columns drained (previous tile) -> its bias MMA
                  mbar_wait(smem_u32(&acc_empty[b]), aph);
                  tc_fence_after();
                  mma_fp4_g<PAIR>(d, uint32_t(ones_desc), uint32_t(ones_desc >> 32), sd, uint32_t(slab_desc0 >> 32),
                                  p.idesc, tmem + p.sf256, tmem + p.sf1, 0u);
                }
              }
#pragma unroll
              for (int pr = 0; pr < CPS / 2; ++pr) {  // chunk pairs of this stage
                const uint32_t ac = a_lo + uint32_t(block_q0(p, b)) + uint32_t(pr * (p.a_chunk_bytes >> 4));
                const uint32_t bc = b_lo + uint32_t(pr * (p.b_pair_bytes >> 4));
#pragma unroll
                for (int tap = 0; tap < 9; ++tap)
                  mma_fp4_g<PAIR>(d, ac + uint32_t(tap / 3 - 1) * P32 + uint32_t(tap % 3 - 1), a_hi,
                                  bc + uint32_t(tap) * bs32, b_hi, p.idesc, sf, sf, 1u);
              }
              if constexpr (BLOCK_COMMIT) {
                if (k == p.ks - 1) commit_g<PAIR>(smem_u32(&acc_full[b]));
              }
              if (k == 0) MMA_T(2 + b);
            }
          } else if (TAPS == 9) {
            for (int b = 0; b < p.MB; ++b)
              umma9_i8(d0 + uint32_t(b * p.n_tile), a_s + uint64_t(block_q0(p, b)), b_s, pp, bs, p.idesc);
          } else {
#pragma unroll
            for (int c = 0; c < CPS; ++c)  // chunk c: A region c, B slab c
              for (int b = 0; b < p.MB; ++b)
                umma1_i8(d0 + uint32_t(b * p.n_tile),
                         a_s + uint64_t(c * (p.a_chunk_bytes >> 4)) + uint64_t(block_q0(p, b)),
                         b_s + uint64_t(c) * bs, p.idesc);
          }
          commit_g<PAIR>(smem_u32(&empty[s]));
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
        if constexpr (!BLOCK_COMMIT) umma_commit_elect(smem_u32(&acc_full[ab]));
        if (++ab == p.nbuf) {
          ab = 0;
          aph ^= 1;
        }
        MMA_T(12);
#ifdef MBU_TIMELINE
        if (blockIdx.x == 0 && lane == 0 && it < 64) {
          g_timeline[it * 12 + 0] = tl0;
          g_timeline[it * 12 + 1] = tl1;
          g_timeline[it * 12 + 2] = clock64();
          g_timeline[it * 12 + 3] = tl_full;
        }
#endif
      }
    }
    __syncwarp();
  } else if (warp == BLOAD_WARP) {
    // ============ weight stages: one bulk copy per stage ============
    if (lane == 0 && p.b_resident) {  // every weight stage, once (PAIR: this CTA's B rows)
      const uint32_t total = uint32_t(p.n_tiles * p.ks) * p.b_stage_bytes;
      const int8_t *bsrc = p.b + size_t(rank) * total;
      mbar_arrive_expect_tx(smem_u32(bres), total);
      for (uint32_t off = 0; off < total; off += 32768u)
        bulk_g2s(smem_u32(b_base + off), bsrc + off, min(32768u, total - off), smem_u32(bres));
    }
    if (lane == 0 && (FP4 || !p.b_resident)) {
      // per stage: the weight slab (streamed) and, FP4, the raw activation box (TMA)
      int s = 0, ph = 0, g = 0, rs = 0, rph = 0;
      if constexpr (FP4) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
        if (p.split32 != 0x7FFFFFFF) asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap2) : "memory");
      }
      for (int u = w_first; u < w_limit; u += w_step) {
        bool tv;
        const Tile tl = decode_tile(p, tile_of(u, tv));
        const int8_t *src = p.b + (size_t(rank) * p.n_tiles + tl.nt) * p.ks * p.b_stage_bytes;
        for (int k = 0; k < p.ks; ++k, ++g) {
          if constexpr (FP4) {
            if (g >= p.rraw_stages) mbar_wait(smem_u32(&rempty[rs]), rph ^ 1);
            const uint32_t rb = smem_u32(&rfull[rs]);
            mbar_arrive_expect_tx(rb, p.rraw_box_bytes);
            // the stage's 128-lane block: u32 word blk of the (logical) pixel
            const int blk = 4 * (chunk_s[2 * (FP4 ? CPS / 2 : 1) * k] >> 2);
            const bool sec = blk >= p.split32;
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(smem + p.off_rraw + rs * p.rraw_bytes)),
                "l"(sec ? &xmap2 : &xmap), "r"(sec ? blk - p.split32 : p.x_off32 + blk), "r"(tl.x0 - p.halo),
                "r"(tl.y0 - p.halo), "r"(tl.nb), "r"(rb)
                : "memory");
            if (++rs == p.rraw_stages) {
              rs = 0;
              rph ^= 1;
            }
          }
          if (!p.b_resident) {
            if (g >= S) mbar_wait(smem_u32(&empty[s]), ph ^ 1);
            const uint32_t bar = smem_u32(&full[s]);
            mbar_arrive_expect_tx(bar, p.b_stage_bytes);
            bulk_g2s(smem_u32(b_base + size_t(s) * p.b_stage_bytes),
                     src + size_t(k) * p.b_stage_bytes, p.b_stage_bytes, bar);
            if (++s == S) {
              s = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ============ epilogue ============
    const int quarter = warp & 3;
    const int half = warp >> 2;
    const int m = quarter * 32 + lane;
    const uint32_t lane_base = tmem + (uint32_t(quarter * 32) << 16);
    auto mine = [&](int b, int ri) { return ((p.MB >= 2 ? b : ri) & 1) == half; };
    // bias -> TMEM for every (block, run) unit this warp owns in tile t
    auto init_buffer = [&](int t, int ab) {
      if constexpr (BLOCK_COMMIT) {  // every block this half drains starts out free
        tc_fence_before();
        for (int b = half; b < p.MB; b += 2) arrive_lead(&acc_empty[b]);
        return;
      }
      if (!PAIR && t < p.num_tiles && !p.mma_bias) {
        if constexpr (TCONV) {
          // a tconv's runs are owned by run parity and may sit on different
          // columns in the tile that reuses the buffer: wait until both halves
          // have drained it before either writes the next tile's bias
          tc_fence_before();
          asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
          tc_fence_after();
        }
        const int nt = t - fdiv(t, p.nt_magic) * p.n_tiles;
        const int jt = nt * p.n_tile;
        const int nr = runs_s[nt * 9].x;
        for (int ri = 0; ri < nr; ++ri) {
          const int4 rn = runs_s[nt * 9 + 1 + ri];
          for (int b = 0; b < p.MB; ++b) {
            if (!mine(b, ri)) continue;
            for (int gg = rn.x; gg < rn.x + rn.y; ++gg) {
              uint32_t v[32];
              const int4 *src = reinterpret_cast<const int4 *>(bias_s + jt + 32 * gg);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int4 q4 = src[i];
                v[4 * i] = q4.x;
                v[4 * i + 1] = q4.y;
                v[4 * i + 2] = q4.z;
                v[4 * i + 3] = q4.w;
              }
              if constexpr (FP4) {  // f32 accumulator: bias + 1/2 (exact, never a signed zero)
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(float(int(v[i])) + 0.5f);
              }
              tmem_st32(lane_base + uint32_t(ab * p.buf_cols + b * p.n_tile + gg * 32), v);
            }
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      tc_fence_before();
      arrive_lead(&acc_empty[ab]);
    };
    for (int i = 0; i < p.nbuf; ++i) init_buffer(w_first + i * w_step, i);
    int it = 0, ab = 0, aph = 0;
    for (int u = w_first; u < w_limit; u += w_step, ++it) {
      bool tvalid;  // (PAIR: false for rank 1's copy of an odd last tile -- no stores)
      const int t = tile_of(u, tvalid);
      const Tile tl = decode_tile(p, t);
      // a conv tile is one run of its N tile's groups: no shared-memory table
      // reads on the epilogue path (they queue behind the tensor core's
      // operand reads); tconv runs are read before the wait
      const int4 *rt = runs_s + tl.nt * 9 + 1;
      const int nr = TCONV ? runs_s[tl.nt * 9].x : 1;
#ifdef MBU_TIMELINE
      unsigned long long te0 = clock64();
#endif
      if constexpr (!BLOCK_COMMIT) mbar_wait(smem_u32(&acc_full[ab]), aph);
#ifdef MBU_TIMELINE
      unsigned long long te1 = clock64();
#endif
      EPI_T(5);
      tc_fence_after();
      EPI_T(6);
      const int jt = tl.nt * p.n_tile;
      // Fast path (the benchmarked forward): a row-mode conv tile whose N tile is
      // 64 or 128 full columns, no trace. Block b is output row y0 + b, lane m is
      // column x0 + m, and the pixel's words are written as one 16-B store
      // (N = 64: the two sign words plus the block's two zero pad words).
      const bool fast = !TCONV && p.acc == nullptr && p.row_mode && (p.n_tile == 64 || p.n_tile == 128) &&
                        p.n_gemm - jt >= p.n_tile;
      // 2x2/s2 tconv whose N tile holds all four taps of <= 64 channels (up-CT4):
      // half h writes output row 2y + h, both dx taps of a pixel as 32
      // contiguous bytes (lanes: consecutive x), so every sector is written
      // whole by one thread instead of two half-sector writes from two warps
      const bool fast_t = TCONV && p.acc == nullptr && p.row_mode && p.tconv_s == 2 && p.c_out_pad == 64 &&
                          p.n_tile == 256 && p.out_groups == 4 && p.bits;
      // other tconvs: units of (block, run, 4-group chunk) alternate between the
      // two epilogue halves; each unit is <= 4 TMEM loads + packs and one 16-B
      // store (both halves busy even when a tile holds a single run)
      const bool fast_g = TCONV && !fast_t && p.acc == nullptr && p.row_mode && p.bits &&
                          runs_s[tl.nt * 9].y;
      if (fast_g) {
        const int xx = tl.x0 + m;
        int u = 0;
        for (int b = 0; b < p.MB; ++b) {
          const int yy = tl.y0 + b;
          if constexpr (BLOCK_COMMIT) {
            mbar_wait(smem_u32(&acc_full[b]), it & 1);
            tc_fence_after();
          }
          const uint32_t colb = lane_base + uint32_t(ab * p.buf_cols + b * p.n_tile);
          const bool ok = xx < p.w && yy < p.h;
          const int64_t pix0 = (int64_t(tl.nb) * p.ho + 2 * yy) * p.wo + 2 * xx;
          for (int ri = 0; ri < nr; ++ri) {
            const int4 rn = rt[ri];
            const int64_t opix = pix0 + (rn.w >> 16) * p.wo + (rn.w & 0xFFFF);
            for (int c = 0; 4 * c < rn.y; ++c, ++u) {
              if ((u & 1) != half) continue;
              const int gn = min(4, rn.y - 4 * c);
              uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                if (q < gn) {
                  uint32_t v[32];
                  tmem_ld32(colb + uint32_t((rn.x + 4 * c + q) * 32), v);
                  w[q] = pack_nonneg<0>(v);
                }
              }
              if (ok)
                *reinterpret_cast<uint4 *>(p.bits + opix * p.out_stride32 + p.out_off32 + rn.z / 32 + 4 * c) =
                    make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
        }
      }
      if (fast_t) {
        const int xx = tl.x0 + m;
        for (int b = 0; b < p.MB; ++b) {
          const int yy = tl.y0 + b;
          const uint32_t colb = lane_base + uint32_t(ab * p.buf_cols + b * p.n_tile + 128 * half);
          // (32-column loads: two live 64-register loads spill)
          uint32_t v[32];
          tmem_ld32(colb, v);  // tap (half, 0)
          const uint32_t w0 = pack_nonneg<0>(v);
          tmem_ld32(colb + 32u, v);
          const uint32_t w1 = pack_nonneg<0>(v);
          tmem_ld32(colb + 64u, v);  // tap (half, 1)
          const uint32_t w2 = pack_nonneg<0>(v);
          tmem_ld32(colb + 96u, v);
          const uint32_t w3 = pack_nonneg<0>(v);
          if (xx < p.w && yy < p.h) {
            uint32_t *dst = p.bits + ((int64_t(tl.nb) * p.ho + 2 * yy + half) * p.wo + 2 * xx) * p.out_stride32 +
                            p.out_off32;
            *reinterpret_cast<uint4 *>(dst) = make_uint4(w0, w1, 0u, 0u);
            *reinterpret_cast<uint4 *>(dst + p.out_stride32) = make_uint4(w2, w3, 0u, 0u);
          }
        }
      }
      if (fast) {
        const int xx = tl.x0 + m;
        const int64_t row_words = int64_t(p.wo) * p.out_stride32;
        uint32_t *dst0 = p.bits + ((int64_t(tl.nb) * p.ho + tl.y0) * p.wo + xx) * p.out_stride32 + p.out_off32 +
                         (jt >> 5);
        for (int b = half; b < p.MB; b += 2) {
          const uint32_t colb = lane_base + uint32_t(ab * p.buf_cols + b * p.n_tile);
          if constexpr (BLOCK_COMMIT) {
            mbar_wait(smem_u32(&acc_full[b]), it & 1);
            tc_fence_after();
          }
          uint32_t v[32];
          tmem_ld32(colb, v);
          const uint32_t w0 = pack_nonneg<0>(v);
          tmem_ld32(colb + 32u, v);
          const uint32_t w1 = pack_nonneg<0>(v);
          uint32_t w2 = 0u, w3 = 0u;
          if (p.n_tile == 128) {
            tmem_ld32(colb + 64u, v);
            w2 = pack_nonneg<0>(v);
            tmem_ld32(colb + 96u, v);
            w3 = pack_nonneg<0>(v);
          }
          if (p.head_logits) {
            // fused head: the same nibble-table sums as head_nib64_kernel (two
            // chains over channels 0-31 / 32-63, then the bias), one logit + mask byte
            if (tvalid && xx < p.w && tl.y0 + b < p.h) {
              const double *ht = reinterpret_cast<const double *>(smem + p.off_head);
              double a0 = 0.0, a1 = 0.0;
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                a0 = __dadd_rn(a0, ht[k * 16 + int((w0 >> (4 * k)) & 0xFu)]);
                a1 = __dadd_rn(a1, ht[(8 + k) * 16 + int((w1 >> (4 * k)) & 0xFu)]);
              }
              double a = __dadd_rn(a0, a1);
              if (p.head_bias) a = __dadd_rn(a, __ldg(p.head_bias));
              const int64_t pix = (int64_t(tl.nb) * p.ho + tl.y0 + b) * p.wo + xx;
              __stcs(p.head_logits + pix, a);
              if (p.head_mask) p.head_mask[pix] = a >= 0.0 ? 1 : 0;
            }
          } else if (tvalid && xx < p.w && tl.y0 + b < p.h && p.bits) {
            *reinterpret_cast<uint4 *>(dst0 + b * row_words) = make_uint4(w0, w1, w2, w3);
          }
          if constexpr (BLOCK_COMMIT) {  // block b's columns free for the next tile
            tc_fence_before();
            arrive_lead(&acc_empty[b]);
          }
        }
      }
      // units (block b, run ri): by block parity when MB >= 2, else by run parity
      const bool split_b = !TCONV || p.MB >= 2;
      if (!fast && !fast_t && !fast_g)
      for (int b = split_b ? half : 0; b < p.MB; b += split_b ? 2 : 1) {
        // this lane's pixel in block b, once per block
        const int q = block_q0(p, b) + m;
        const int rq = int(__umulhi(uint32_t(q), p.p_magic));
        const int r = rq - p.halo;
        const int c = q - rq * p.P - p.halo;
        const int yy = tl.y0 + r, xx = tl.x0 + c;
        const bool valid = tvalid && r >= 0 && r < p.R && c >= 0 && c < p.TW && yy < p.h && xx < p.w;
        const int64_t pix0 = TCONV ? (int64_t(tl.nb) * p.ho + yy * p.tconv_s) * p.wo + xx * p.tconv_s
                                   : (int64_t(tl.nb) * p.ho + yy) * p.wo + xx;
        const uint32_t colb = lane_base + uint32_t(ab * p.buf_cols + b * p.n_tile);
        if constexpr (BLOCK_COMMIT) {  // single buffer: one use per tile
          mbar_wait(smem_u32(&acc_full[b]), it & 1);
          tc_fence_after();
        }
        EPI_T(7 + (b >> 1));
        for (int ri = split_b ? 0 : half; ri < nr; ri += split_b ? 1 : 2) {
          // (first group, length, o0, tap dy << 16 | dx)
          const int4 rn = TCONV ? rt[ri] : make_int4(0, min(p.n_tile, p.n_gemm - jt) >> 5, jt, 0);
          const int64_t opix = TCONV ? pix0 + (rn.w >> 16) * p.wo + (rn.w & 0xFFFF) : pix0;
          uint32_t w8[8];
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) w8[rr] = 0u;
          const uint32_t col0 = colb + uint32_t(rn.x * 32);
#ifdef ABL_NO_EPI
          if (true) {
          } else
#endif
          if (p.acc == nullptr) {
            // two groups per TMEM load, one SHF per column to pack the signs
#pragma unroll
            for (int rr = 0; rr < 8; rr += 2) {
              if (rr < rn.y) {
                if (rr + 1 < rn.y) {
                  uint32_t v[64];
                  tmem_ld64(col0 + uint32_t(rr * 32), v);
                  w8[rr] = pack_nonneg<0>(v);
                  w8[rr + 1] = pack_nonneg<32>(v);
                } else {
                  uint32_t v[32];
                  tmem_ld32(col0 + uint32_t(rr * 32), v);
                  w8[rr] = pack_nonneg<0>(v);
                }
              }
            }
          } else {
            // trace mode: also recover the reference accumulators; the sign words
            // go straight to memory (no dynamic index into w8, which must stay
            // in registers for the fast path)
            const int f = p.u8_act ? 2 : 1;
            const int g0 = rn.z >> 5;
#pragma unroll 1
            for (int rr = 0; rr < rn.y; ++rr) {
              uint32_t v[32];
              const int gg = rn.x + rr;
              tmem_ld32(col0 + uint32_t(rr * 32), v);
              const uint32_t word = pack_nonneg<0>(v);
              if (valid) {
                const int oc = rn.z + 32 * rr;
                const int jc = jt + 32 * gg;
                int32_t *dst = p.acc + opix * p.c_out + oc;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                  if (oc + i < p.c_out) {
                    const int s = __ldg(p.col_sgn + jc + i), bias = bias_s[jc + i];
                    // FP4: the accumulator is a float holding D' + 0.5 (never a signed zero)
                    const int dv = FP4 ? int(__uint_as_float(v[i]) - 0.5f) : int(v[i]);
                    dst[i] = f * (s * (dv - bias)) - __ldg(p.col_w + jc + i);
                  }
                }
                if (p.bits) p.bits[opix * p.out_stride32 + p.out_off32 + g0 + rr] = word;
              }
            }
            if (valid && p.bits && g0 + rn.y == p.c_out_pad / 32)  // pad words of the block
              for (int i = g0 + rn.y; i < p.out_groups; ++i)
                p.bits[opix * p.out_stride32 + p.out_off32 + i] = 0u;
            continue;
          }
          if (b == 0) EPI_T(13);
          if (valid && p.bits) {
            // write the run; when it ends the pixel's channels append the zero
            // pad groups of the 128-lane block (w8 is zero past the run)
            uint32_t *dst = p.bits + opix * p.out_stride32 + p.out_off32;
            const int g0 = rn.z >> 5;
            const int wend = (g0 + rn.y == p.c_out_pad / 32) ? p.out_groups : g0 + rn.y;
            const int cnt = wend - g0;
            if ((g0 & 3) == 0 && (cnt & 3) == 0 && cnt <= 8) {
              *reinterpret_cast<uint4 *>(dst + g0) = make_uint4(w8[0], w8[1], w8[2], w8[3]);
              if (cnt == 8)
                *reinterpret_cast<uint4 *>(dst + g0 + 4) = make_uint4(w8[4], w8[5], w8[6], w8[7]);
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i)
                if (i < cnt) dst[g0 + i] = w8[i];
              for (int i = 8; i < cnt; ++i) dst[g0 + i] = 0u;
            }
          }
          if (b == 0) EPI_T(14);
        }
        if constexpr (BLOCK_COMMIT) {
          tc_fence_before();
          arrive_lead(&acc_empty[b]);
        }
      }
      EPI_T(10);
      // buffer drained: re-arm it with the bias of the tile that reuses it
      if constexpr (!BLOCK_COMMIT) init_buffer(u + p.nbuf * w_step, ab);
      if (++ab == p.nbuf) {
        ab = 0;
        aph ^= 1;
      }
      EPI_T(11);
#ifdef MBU_TIMELINE
      if (blockIdx.x == 0 && lane == 0 && it < 64 && warp == 0) {
        g_timeline[it * 12 + 4] = te0;
        g_timeline[it * 12 + 5] = te1;
        g_timeline[it * 12 + 6] = clock64();
      }
      if (blockIdx.x == 0 && lane == 0 && it < 64 && warp == 4) g_timeline[it * 12 + 7] = clock64();
#endif
    }
  }

  tc_fence_before();
  // (PAIR: neither CTA leaves while the other may still arrive on its barriers)
  if constexpr (PAIR) cluster_sync_all();
  else __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}

}  // namespace tc

// --------------------------------------------------------------------------
// host side: eligibility, weight repack, launch geometry
// --------------------------------------------------------------------------
static int floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }
static int ceil_div(int a, int b) { return -floor_div(-a, b); }

int prepare_conv_tc(mbu_conv *cv, const uint64_t *pos, const uint64_t *neg, const int32_t *seg_off,
                    const int32_t *seg_cnt, int n_seg) {
  cv->tc_ok = 0;
  const bool conv3 = !cv->transposed && cv->kh == 3 && cv->kw == 3 && cv->stride == 1 && cv->pad == 1;
  const bool conv1 = !cv->transposed && cv->kh == 1 && cv->kw == 1 && cv->stride == 1 && cv->pad == 0;
  const bool tconv = cv->transposed && cv->stride <= 4;
  if (!(conv3 || conv1 || tconv)) return MBU_OK;
  const int lpp = cv->lpp;
  std::vector<uint8_t> real(lpp, 0);
  for (int i = 0; i < n_seg; ++i)
    for (int l = seg_off[i]; l < seg_off[i] + seg_cnt[i]; ++l) real[l] = 1;
  // 3x3: every 32-lane chunk holding a real lane. One tap (1x1, tconv): every
  // chunk of each 128-lane block holding a real lane, so four chunks (16 B of
  // a pixel) form one pipeline stage; pad lanes carry zero weights.
  // When every block's real lanes lie in its first 64 (a 64-channel input,
  // e.g. up-CT4's), one-tap stages take just those two chunks (8 B a pixel):
  // half the expansion and MMA work of whole blocks.
  const int gran = (conv3 ? 32 : 128);
  int tap1_chunks = 4;
  if (!conv3) {
    bool low_half = true;
    for (int l = 0; l < lpp; ++l) low_half &= !(real[l] && (l & 127) >= 64);
    if (low_half) tap1_chunks = 2;
  }
  std::vector<int32_t> chunk_word;
  for (int g0 = 0; g0 < lpp; g0 += gran) {
    bool any = false;
    for (int l = g0; l < g0 + gran; ++l) any |= real[l] != 0;
    if (any)
      for (int c = g0 / 32; c < g0 / 32 + (conv3 ? 1 : tap1_chunks); ++c) chunk_word.push_back(c);
  }
  cv->tap1_cps = tap1_chunks;
  const int kc = int(chunk_word.size());
  if (kc == 0 || kc > tc::MAX_CHUNKS) return MBU_OK;
  // bit i: groups of 2^i chunks are consecutive, 2^i-aligned words (one vector copy)
  cv->chunk_consec = 0;
  for (int i = 0; i < 3; ++i) {
    const int g = 1 << i;
    bool ok = kc % g == 0;
    for (int k0 = 0; ok && k0 < kc; k0 += g) {
      ok = chunk_word[k0] % g == 0;
      for (int j = 1; ok && j < g; ++j) ok = chunk_word[k0 + j] == chunk_word[k0] + j;
    }
    if (ok) cv->chunk_consec |= 1 << i;
  }
  const int taps = cv->transposed ? 1 : cv->kh * cv->kw;
  const int s2 = cv->transposed ? cv->stride * cv->stride : 1;
  const int c_out_pad = (cv->c_out + 31) / 32 * 32;
  const int n_gemm = s2 * c_out_pad;
  // N tile: conv -> up to 128 columns (MB = 2 blocks of 128 pixels share each
  // weight stage). tconv -> whole taps when they fit in 256 columns so the A
  // strip is expanded once for all s*s taps, else 128-column slices of a tap.
  int n_tile;
  if (!cv->transposed) n_tile = std::min(c_out_pad, 128);
  else if (c_out_pad <= 256) n_tile = c_out_pad * std::min(s2, 256 / c_out_pad);
  // wider taps in 256-column tiles of 128-aligned runs (up-CT1, 384 channels:
  // 6 N tiles instead of 12, so each A strip is expanded half as often);
  // MBU_TCONV_N128=1 keeps 128-column slices (A/B)
  else if (c_out_pad % 128 == 0 && !std::getenv("MBU_TCONV_N128")) n_tile = 256;
  else if (c_out_pad % 128 == 0) n_tile = 128;
  else if (c_out_pad % 64 == 0) n_tile = 64;
  else n_tile = 32;
  const int n_tiles = (n_gemm + n_tile - 1) / n_tile;
  const int n_cols = n_tiles * n_tile;
  // u8 {0,1} activations are exact when out-of-bounds taps mean -1 (a' = 0);
  // zero padding needs s8 +-1 / 0.
  const bool u8 = cv->pad_mode != MBU_PAD_ZERO;
  const int f = u8 ? 2 : 1;

  // dense s8 weights per (column, tap, chunk lane)
  const int ptaps = cv->kh * cv->kw;  // taps in the reference plane layout
  const size_t row_words = size_t(ptaps) * cv->wpp;
  auto bit = [&](const uint64_t *plane, int o, int tap, int L) -> int {
    return int((plane[size_t(o) * row_words + size_t(tap) * cv->wpp + (L >> 6)] >> (L & 63)) & 1ull);
  };
  auto wval = [&](int j, int tap, int L) -> int {
    if (j >= n_gemm) return 0;
    int o = j, ptap = tap;
    if (cv->transposed) {
      ptap = j / c_out_pad;
      o = j % c_out_pad;
    }
    if (o >= cv->c_out) return 0;
    if (neg) return bit(pos, o, ptap, L) - bit(neg, o, ptap, L);
    return real[L] ? 2 * bit(pos, o, ptap, L) - 1 : 0;
  };
  std::vector<int32_t> col_w(size_t(n_cols) + 32, 0);
  if (u8)
    for (int j = 0; j < n_gemm; ++j) {
      int s = 0;
      for (int tap = 0; tap < taps; ++tap)
        for (int k = 0; k < kc; ++k)
          for (int i = 0; i < 32; ++i) s += wval(j, tap, 32 * chunk_word[k] + i);
      col_w[j] = s;
    }
  // per GEMM column: threshold folded into (weight sign, TMEM bias) on D
  std::vector<int32_t> col_bias(size_t(n_cols) + 32, 0), col_sgn(size_t(n_cols) + 32, 1);
  std::vector<int8_t> col_neg(size_t(n_cols), 0);
  const int dmax = taps * lpp + 1;  // > max |D|
  if (cv->has_threshold) {
    std::vector<int32_t> t(static_cast<size_t>(c_out_pad), 0);
    std::vector<uint8_t> c(static_cast<size_t>(c_out_pad), 2);
    MBU_TRY(check_cuda(cudaMemcpy(t.data(), cv->d_thr, t.size() * 4, cudaMemcpyDeviceToHost), "thr"));
    MBU_TRY(check_cuda(cudaMemcpy(c.data(), cv->d_codes, c.size(), cudaMemcpyDeviceToHost), "codes"));
    for (int j = 0; j < n_cols; ++j) {
      int code = 2, T = 0;
      if (j < n_gemm) {
        const int o = cv->transposed ? j % c_out_pad : j;
        code = c[o];
        T = t[o];
      }
      // acc = f*D - W: GE fires iff D >= ceil((T+W)/f), LE iff D <= floor((T+W)/f)
      const long long tw = (long long)T + col_w[j];
      long long dt = 0;
      if (code == 0) dt = (tw >= 2LL * dmax * f) ? (long long)dmax : (tw <= -2LL * dmax * f) ? -(long long)dmax : ceil_div(int(tw), f);
      if (code == 1) dt = (tw >= 2LL * dmax * f) ? (long long)dmax : (tw <= -2LL * dmax * f) ? -(long long)dmax : floor_div(int(tw), f);
      // out-of-range decision points are constants over the reachable D
      if (code == 0 && dt <= -dmax) code = 3;
      if (code == 0 && dt >= dmax) code = 2;
      if (code == 1 && dt >= dmax) code = 3;
      if (code == 1 && dt <= -dmax) code = 2;
      switch (code) {
        case 0: col_bias[j] = int(-dt); col_sgn[j] = 1; break;                 // D - D_T >= 0
        case 1: col_bias[j] = int(dt); col_sgn[j] = -1; col_neg[j] = 1; break;  // D_T - D >= 0
        case 3: col_bias[j] = dmax; col_sgn[j] = 1; break;                     // always >= 0
        default: col_bias[j] = -2 * dmax; col_sgn[j] = 1; break;               // always < 0
      }
    }
  }
  const size_t b_stage = size_t(taps) * n_tile * 32;
  std::vector<int8_t> b(size_t(n_tiles) * kc * b_stage, 0);
  for (int nt = 0; nt < n_tiles; ++nt)
    for (int k = 0; k < kc; ++k)
      for (int tap = 0; tap < taps; ++tap)
        for (int half = 0; half < 2; ++half)
          for (int n = 0; n < n_tile; ++n) {
            const int j = nt * n_tile + n;
            int8_t *dst = &b[((size_t(nt) * kc + k) * taps + tap) * n_tile * 32 + size_t(half) * n_tile * 16 +
                             size_t(n) * 16];
            for (int i = 0; i < 16; ++i) {
              const int v = wval(j, tap, 32 * chunk_word[k] + 16 * half + i);
              dst[i] = int8_t(col_neg[j] ? -v : v);
            }
          }
  MBU_TRY(check_cuda(cudaMalloc(&cv->d_b, b.size()), "alloc tc weights"));
  MBU_TRY(check_cuda(cudaMemcpy(cv->d_b, b.data(), b.size(), cudaMemcpyHostToDevice), "upload tc weights"));
  MBU_TRY(check_cuda(cudaMalloc(&cv->d_chunk_word, kc * sizeof(int32_t)), "alloc chunk map"));
  MBU_TRY(check_cuda(cudaMemcpy(cv->d_chunk_word, chunk_word.data(), kc * sizeof(int32_t),
                                cudaMemcpyHostToDevice),
                     "upload chunk map"));
  std::vector<int32_t> cols(col_bias);
  cols.insert(cols.end(), col_sgn.begin(), col_sgn.end());
  cols.insert(cols.end(), col_w.begin(), col_w.end());
  MBU_TRY(check_cuda(cudaMalloc(&cv->d_thr2, cols.size() * sizeof(int32_t)), "alloc column bias"));
  MBU_TRY(check_cuda(cudaMemcpy(cv->d_thr2, cols.data(), cols.size() * sizeof(int32_t), cudaMemcpyHostToDevice),
                     "upload column bias"));
  // FP4 (kind::mxf4) operand for 3x3 layers: chunk pairs share one K = 64
  // row (pair p = chunks 2p, 2p+1; an odd count gets a zero-weight dummy),
  // weights as e2m1 {-1, 0, +1} nibbles; lane i of a chunk at K position 8 (i % 4) + i / 4
  cv->fp4_ok = 0;
  if (conv3) {
    // pairs never straddle a 128-lane block (one TMA box per stage): pair the
    // chunks of each block, an odd leftover with a zero-weight duplicate
    std::vector<int32_t> pairs, pair_src;  // pair_src: index into chunk_word, or -1 (dummy)
    for (int i = 0; i < kc;) {
      const int blk = chunk_word[i] >> 2;
      pairs.push_back(chunk_word[i]);
      pair_src.push_back(i);
      if (i + 1 < kc && (chunk_word[i + 1] >> 2) == blk) {
        pairs.push_back(chunk_word[i + 1]);
        pair_src.push_back(i + 1);
        i += 2;
      } else {
        pairs.push_back(chunk_word[i]);
        pair_src.push_back(-1);
        i += 1;
      }
    }
    const int kp = int(pairs.size() / 2);
    bool consec = true;
    for (int q = 0; q < kp; ++q) consec &= pairs[2 * q] % 2 == 0 && pairs[2 * q + 1] == pairs[2 * q] + 1;
    std::vector<uint8_t> b4(size_t(n_tiles) * kp * b_stage, 0);
    auto e2m1 = [](int v) -> uint8_t { return v > 0 ? 0x2 : v < 0 ? 0xA : 0x0; };
    for (int nt = 0; nt < n_tiles; ++nt)
      for (int q = 0; q < kp; ++q)
        for (int tap = 0; tap < taps; ++tap)
          for (int half = 0; half < 2; ++half)
            for (int n = 0; n < n_tile; ++n) {
              const int j = nt * n_tile + n;
              const int ci = pair_src[2 * q + half];
              uint8_t *dst = &b4[((size_t(nt) * kp + q) * taps + tap) * n_tile * 32 + size_t(half) * n_tile * 16 +
                                 size_t(n) * 16];
              if (ci < 0) continue;  // dummy chunk: zero weights
              for (int i = 0; i < 32; ++i) {
                const int v = wval(j, tap, 32 * chunk_word[ci] + i);
                const int kp = 8 * (i % 4) + i / 4;  // K position of lane i (the producers' fp4x32 order)
                dst[kp / 2] |= uint8_t(e2m1(col_neg[j] ? -v : v) << (4 * (kp & 1)));
              }
            }
    // bias slabs: bias + 0.5 (no signed zero) = sum(lo entries, K 0-31) +
    // 256 * sum(hi entries, K 32-63); the bias MMA's A block scales are 2^0 / 2^8
    const size_t sb = size_t(n_tile) * 32;  // one K = 64 slab per N tile
    std::vector<uint8_t> slabs;
    std::vector<int32_t> slab_of(n_tiles);
    bool slabs_ok = true;
    for (int nt = 0; nt < n_tiles; ++nt) {
      std::vector<uint8_t> sl(sb, 0);
      for (int n = 0; n < n_tile; ++n) {
        const int bias = col_bias[size_t(nt) * n_tile + n];
        const int hi = (bias >= 0 ? bias + 128 : bias - 128) / 256;
        const double lo = double(bias - 256 * hi) + 0.5;
        for (int part = 0; part < 2; ++part) {
          const double v = part == 0 ? lo : double(hi);
          // entries e = 0..31 of column n in K half `part`: byte e / 2, nibble e % 2
          static const double mag[7] = {6, 4, 3, 2, 1.5, 1, 0.5};
          static const uint8_t code[7] = {7, 6, 5, 4, 3, 2, 1};
          const uint8_t sg = v < 0 ? 0x8 : 0x0;
          double r = std::fabs(v);
          int e = 0;
          for (int m = 0; m < 7; ++m)
            while (r >= mag[m] && e < 32) {
              sl[size_t(part) * n_tile * 16 + size_t(n) * 16 + e / 2] |= uint8_t((code[m] | sg) << (4 * (e & 1)));
              r -= mag[m];
              ++e;
            }
          slabs_ok &= r == 0.0;
        }
      }
      int found = -1;
      for (size_t k = 0; k * sb < slabs.size(); ++k)
        if (std::equal(sl.begin(), sl.end(), slabs.begin() + k * sb)) found = int(k);
      if (found < 0) {
        found = int(slabs.size() / sb);
        slabs.insert(slabs.end(), sl.begin(), sl.end());
      }
      slab_of[nt] = found;
    }
    if (slabs_ok && slabs.size() <= size_t(MBU_FP4_SLAB_CAP)) {
      MBU_TRY(check_cuda(cudaMalloc(&cv->d_b4, b4.size()), "alloc fp4 weights"));
      MBU_TRY(check_cuda(cudaMemcpy(cv->d_b4, b4.data(), b4.size(), cudaMemcpyHostToDevice), "upload fp4 weights"));
      MBU_TRY(check_cuda(cudaMalloc(&cv->d_chunk_pair, pairs.size() * 4), "alloc chunk pairs"));
      MBU_TRY(check_cuda(cudaMemcpy(cv->d_chunk_pair, pairs.data(), pairs.size() * 4, cudaMemcpyHostToDevice),
                         "upload chunk pairs"));
      MBU_TRY(check_cuda(cudaMalloc(&cv->d_bias_slab4, slabs.size()), "alloc fp4 bias slabs"));
      MBU_TRY(check_cuda(cudaMemcpy(cv->d_bias_slab4, slabs.data(), slabs.size(), cudaMemcpyHostToDevice),
                         "upload fp4 bias slabs"));
      MBU_TRY(check_cuda(cudaMalloc(&cv->d_slab_of_nt4, n_tiles * sizeof(int32_t)), "alloc fp4 slab map"));
      MBU_TRY(check_cuda(cudaMemcpy(cv->d_slab_of_nt4, slab_of.data(), n_tiles * sizeof(int32_t),
                                    cudaMemcpyHostToDevice),
                         "upload fp4 slab map"));
      cv->n_slabs4 = int(slabs.size() / sb);
      for (int i = 0; i < 16 && i < n_tiles; ++i) cv->h_slab_of_nt4[i] = slab_of[i];
      if (n_tile == 64 || n_tile == 128) {
        // CTA-pair copies: rank r holds rows [r * n_tile / 2, +n_tile / 2) of every
        // (n tile, pair, tap) slab and of every bias slab, K halves LBO = n_tile / 2 * 16 apart
        const int nh = n_tile / 2;
        const size_t slab_in = size_t(n_tile) * 32, slab_out = size_t(nh) * 32;
        const size_t n_b = b4.size() / slab_in, n_s = slabs.size() / slab_in;
        std::vector<uint8_t> b4p(b4.size()), slp(slabs.size());
        auto split = [&](const std::vector<uint8_t> &in, std::vector<uint8_t> &out, size_t n) {
          for (int r = 0; r < 2; ++r)
            for (size_t i = 0; i < n; ++i)
              for (int half = 0; half < 2; ++half)
                std::memcpy(&out[(size_t(r) * n + i) * slab_out + size_t(half) * nh * 16],
                            &in[i * slab_in + size_t(half) * n_tile * 16 + size_t(r) * nh * 16], size_t(nh) * 16);
        };
        split(b4, b4p, n_b);
        split(slabs, slp, n_s);
        MBU_TRY(check_cuda(cudaMalloc(&cv->d_b4p, b4p.size()), "alloc fp4 pair weights"));
        MBU_TRY(check_cuda(cudaMemcpy(cv->d_b4p, b4p.data(), b4p.size(), cudaMemcpyHostToDevice),
                           "upload fp4 pair weights"));
        MBU_TRY(check_cuda(cudaMalloc(&cv->d_bias_slab4p, slp.size()), "alloc fp4 pair slabs"));
        MBU_TRY(check_cuda(cudaMemcpy(cv->d_bias_slab4p, slp.data(), slp.size(), cudaMemcpyHostToDevice),
                           "upload fp4 pair slabs"));
      }
      cv->kp = kp;
      cv->pair_consec = consec ? 1 : 0;
      // pairs 2j, 2j+1 read the same 128-lane block: one stage can take both
      bool two = kp % 2 == 0;
      for (int q = 0; two && q < kp; q += 2) two = (pairs[2 * q] >> 2) == (pairs[2 * q + 2] >> 2);
      cv->pair2_ok = two ? 1 : 0;
      cv->fp4_ok = 1;
    }
  }
  cv->taps = taps;
  cv->kc = kc;
  cv->n_gemm = n_gemm;
  cv->n_pad = n_cols;
  cv->c_out_pad = c_out_pad;
  cv->n_tile = n_tile;
  cv->n_tiles = n_tiles;
  // bias enters the accumulator through an MMA of a ones slab
  // (16 x 1 and 16 x 127 per row) with a per-N-tile bias slab (s8 column
  // sum(lo) + 127 * sum(hi) = bias), so the epilogue never initialises TMEM.
  // Identical slabs (tconv taps repeat the channels) are stored once.
  cv->n_slabs = 0;
  {
    std::vector<int8_t> slabs;
    std::vector<int32_t> slab_of(n_tiles);
    const size_t sb = size_t(n_tile) * 32;
    for (int nt = 0; nt < n_tiles; ++nt) {
      std::vector<int8_t> sl(sb, 0);
      for (int n = 0; n < n_tile; ++n) {
        const int bias = col_bias[size_t(nt) * n_tile + n];
        int hi = (bias >= 0 ? bias + 63 : bias - 63) / 127;
        const int lo = bias - 127 * hi;
        sl[size_t(n) * 16] = int8_t(lo);  // khalf 0, k 0
        for (int i = 0; i < 16; ++i) {     // khalf 1: hi spread over 16 entries
          const int part = hi / (16 - i);
          sl[size_t(n_tile) * 16 + size_t(n) * 16 + i] = int8_t(part);
          hi -= part;
        }
      }
      int found = -1;
      for (size_t k = 0; k * sb < slabs.size(); ++k)
        if (std::equal(sl.begin(), sl.end(), slabs.begin() + k * sb)) found = int(k);
      if (found < 0) {
        found = int(slabs.size() / sb);
        slabs.insert(slabs.end(), sl.begin(), sl.end());
      }
      slab_of[nt] = found;
    }
    // (32 KB: up-CT1's 3 and up-CT2's distinct per-tap slabs take the bias MMA
    // too, so their epilogues never write TMEM; 16 KB measured ~5 % slower on up-CT2)
    if (slabs.size() <= 32768) {
      MBU_TRY(check_cuda(cudaMalloc(&cv->d_bias_slab, slabs.size()), "alloc bias slabs"));
      MBU_TRY(check_cuda(cudaMemcpy(cv->d_bias_slab, slabs.data(), slabs.size(), cudaMemcpyHostToDevice),
                         "upload bias slabs"));
      MBU_TRY(check_cuda(cudaMalloc(&cv->d_slab_of_nt, n_tiles * sizeof(int32_t)), "alloc slab map"));
      MBU_TRY(check_cuda(cudaMemcpy(cv->d_slab_of_nt, slab_of.data(), n_tiles * sizeof(int32_t),
                                    cudaMemcpyHostToDevice),
                         "upload slab map"));
      cv->n_slabs = int(slabs.size() / sb);
      for (int i = 0; i < 16 && i < n_tiles; ++i) cv->h_slab_of_nt[i] = slab_of[i];
    }
  }
  cv->b_stage_bytes = b_stage;
  cv->tc_ok = 1;
  return MBU_OK;
}

static int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// (a separate trace-free instantiation was tried: ptxas then spills in the
// epilogue and the N = 64 layers lose ~7%, so trace stays a runtime branch)
template <int TAPS, bool TCONV, int LA, int CPS, bool FP4, bool BLOCK_COMMIT = false, bool PAIR = false>
static int launch_tc_impl(const tc::Params &p, const CUtensorMap &xmap, const CUtensorMap &xmap2, int grid,
                          size_t smem, cudaStream_t st) {
  auto kern = tc::conv_tc_kernel<TAPS, TCONV, LA, CPS, FP4, BLOCK_COMMIT, PAIR>;
  static bool configured = false;
  if (!configured) {
    MBU_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024),
                       "cudaFuncSetAttribute"));
    configured = true;
  }
  if constexpr (PAIR) {
    // persistent clusters of two CTAs (one per SM): as many as can be
    // co-resident (a GPC with an odd SM count leaves one SM out)
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(tc::NUM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static const int max_clusters = [&] {
      cudaLaunchConfig_t q = cfg;
      q.gridDim = dim3(2 * (num_sms() / 2));
      q.dynamicSmemBytes = 227 * 1024;  // (one CTA per SM at any size this kernel launches with)
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &q) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
      }
      return n;
    }();
    if (max_clusters < 1) return fail(MBU_ERR_CUDA, "conv_tc: no co-resident CTA pair");
    cfg.gridDim = dim3(2 * std::min(p.n_pairs, max_clusters));
    MBU_TRY(check_cuda(cudaLaunchKernelEx(&cfg, kern, p, xmap, xmap2), "conv_tc_kernel (CTA pairs)"));
  } else {
    kern<<<grid, tc::NUM_THREADS, smem, st>>>(p, xmap, xmap2);
  }
#ifdef MBU_TIMELINE
  {
    static int call = 0;
    unsigned long long h[64 * 12];
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(h, tc::g_timeline, sizeof(h));
    const unsigned long long b0 = h[0];
    fprintf(stderr, "TIMELINE call %d taps %d fp4 %d MB %d ntile %d ks %d\n", call, TAPS, int(FP4), p.MB, p.n_tile, p.ks);
    {
      unsigned long long e[64 * 16];
      cudaMemcpyFromSymbol(e, tc::g_epi, sizeof(e));
      for (int i = 2; i < 8; ++i) {
        fprintf(stderr, "  mma it %d (waitE %lld got %lld):", i, (long long)(h[i * 12] - b0), (long long)(h[i * 12 + 1] - b0));
        for (int k = 0; k < 16; ++k) fprintf(stderr, " %lld", (long long)(e[i * 16 + k] ? e[i * 16 + k] - h[0] : 0));
        fprintf(stderr, "\n");
      }
    }
    ++call;
    for (int i = 0; i < 24; ++i)
      fprintf(stderr, "  it %2d mma: waitE %6lld got %6lld fullL %6lld issued %6lld | epi0: wait %6lld got %6lld done %6lld | epi4 done %6lld | prod stage %2d: start %6lld emptyok %6lld end %6lld\n", i,
              (long long)(h[i * 12] - b0), (long long)(h[i * 12 + 1] - b0), (long long)(h[i * 12 + 3] - b0),
              (long long)(h[i * 12 + 2] - b0), (long long)(h[i * 12 + 4] - b0), (long long)(h[i * 12 + 5] - b0),
              (long long)(h[i * 12 + 6] - b0), (long long)(h[i * 12 + 7] - b0), i, (long long)(h[i * 12 + 8] - b0),
              (long long)(h[i * 12 + 9] - b0), (long long)(h[i * 12 + 10] - b0));
  }
#endif
  return check_launch("conv_tc_kernel");
}

// kNoFit: the FP4 shared-memory layout (bias slabs + stages) does not fit;
// the caller falls back to kind::i8 for this geometry
constexpr int kNoFit = -1;
static int launch_conv_tc_kind(const mbu_conv *cv, const ActView &x, int ho, int wo, int32_t *acc,
                               uint64_t *bits, int out_stride, int out_offset, cudaStream_t st, bool fp4,
                               bool allow_pps2, bool allow_pair, HeadFuse *head);
int launch_conv_tc(const mbu_conv *cv, const ActView &x, int ho, int wo, int32_t *acc,
                   uint64_t *bits, int out_stride, int out_offset, cudaStream_t st, HeadFuse *head) {
  // 3x3 layers run kind::mxf4 (e2m1) when the uniform block-scale columns fit
  // next to the accumulators (MB * n_tile <= 248); MBU_OPT_CONV_I8 forces kind::i8
  const bool fp4 = cv->fp4_ok && !g_force_conv_i8 && tc::FP4_COLS / cv->n_tile >= 1;
  if (fp4) {
    for (int allow = 1; allow >= 0; --allow) {  // two pairs per stage if that layout fits, else one
      for (int pair = 1; pair >= 0; --pair) {  // CTA pairs where eligible, else one-CTA tiles
        const int r =
            launch_conv_tc_kind(cv, x, ho, wo, acc, bits, out_stride, out_offset, st, true, allow != 0, pair != 0,
                                head);
        if (r != kNoFit) return r;
      }
    }
  }
  const int r =
      launch_conv_tc_kind(cv, x, ho, wo, acc, bits, out_stride, out_offset, st, false, false, false, nullptr);
  return r == kNoFit ? fail(MBU_ERR_UNSUPPORTED, "tcgen05 conv stage does not fit in shared memory") : r;
}

static int launch_conv_tc_kind(const mbu_conv *cv, const ActView &x, int ho, int wo, int32_t *acc,
                               uint64_t *bits, int out_stride, int out_offset, cudaStream_t st, bool fp4,
                               bool allow_pps2, bool allow_pair, HeadFuse *head) {
  tc::Params p{};
  p.x32 = reinterpret_cast<const uint32_t *>(x.base);
  p.n = x.n;
  p.h = x.h;
  p.w = x.w;
  p.x_stride32 = x.stride * 2;
  p.x_off32 = x.offset * 2;
  p.x2_32 = reinterpret_cast<const uint32_t *>(x.split ? x.base2 : x.base);
  p.x2_stride32 = x.split ? x.stride2 * 2 : 0;
  p.split32 = x.split ? x.split * 2 : 0x7FFFFFFF;
  // producers index the input with 32-bit word offsets
  if ((int64_t(x.n) * x.h * x.w + 2 * int64_t(x.w) + 4) * std::max(p.x_stride32, p.x2_stride32) >=
      (int64_t(1) << 31))
    return fail(MBU_ERR_UNSUPPORTED, "tcgen05 conv input larger than 2^31 words");
  p.halo = cv->taps == 9 ? 1 : 0;
  p.n_tile = cv->n_tile;
  p.n_tiles = cv->n_tiles;
  // long-K FP4 layers (>= 4 K stages) trade the second accumulator for a
  // taller tile (one buffer of up to 504 columns): each weight stage then
  // feeds up to 3 (N = 128) or 7 (N = 64) pixel blocks, cutting the weight
  // stream from L2; the un-overlapped epilogue costs a fraction of such a tile
  // (N = 64 long-K layers too: 7 blocks per tile with per-block commits, -2% on up-C3.a)
  p.nbuf = (fp4 && cv->kp >= 4 && (cv->n_tile == 128 || cv->n_tile == 64)) ? 1 : 2;
  {
    // N = 64, any K: one accumulator of 7 blocks with per-block commits (the
    // epilogue drains block b while later blocks still compute): fewer, taller
    // tiles amortise the MMA warp's per-tile barrier waits and bias MMAs, which
    // the tensor core's shallow queue would otherwise expose (measured: stem2
    // 0.386 -> 0.328 ms, up-C4.b 0.373 -> 0.311 ms), and likewise 3 blocks for
    // the short-K N = 128 layers (down-C1.a 0.169 -> 0.145, down-C2.a 0.143 ->
    // 0.120). MBU_SB64=0 / MBU_SB128=0 restore the double-buffered tiles.
    static const int sb64 = std::getenv("MBU_SB64") ? std::atoi(std::getenv("MBU_SB64")) : 1;
    static const int sb128 = std::getenv("MBU_SB128") ? std::atoi(std::getenv("MBU_SB128")) : 1;
    if (fp4 && sb64 && cv->n_tile == 64) p.nbuf = 1;
    if (fp4 && sb128 && cv->n_tile == 128) p.nbuf = 1;
  }
  // three accumulator buffers of 2 blocks (N = 64) / 1 block (N = 128): the
  // epilogue of a tile then overlaps two later tiles' MMAs
  // (default: the one-K-stage N = 64 layers, measured -4% on stem2 / up-C3.b / up-C4.b;
  // the two-stage up-C4.a loses 13% with it. MBU_NBUF3=0/1 forces it off / on where eligible)
  static const int nbuf3 = std::getenv("MBU_NBUF3") ? std::atoi(std::getenv("MBU_NBUF3")) : -1;
  if (fp4 && p.nbuf == 2 && (cv->n_tile == 64 || cv->n_tile == 128) &&
      (nbuf3 > 0 || (nbuf3 < 0 && cv->n_tile == 64 && cv->kp == 1)))
    p.nbuf = 3;
  p.MB = fp4 ? std::min(8, (p.nbuf == 1 ? 2 * tc::FP4_COLS + 8 : p.nbuf == 3 ? 168 : tc::FP4_COLS) / cv->n_tile)
             : std::min(cv->taps == 9 ? 8 : 4, tc::ACC_COLS / cv->n_tile);  // one tap: Q <= 512
  if (x.w >= 128) {
    p.row_mode = 1;
    p.TW = 128;
    p.P = 128 + 2 * p.halo;
    p.R = p.MB;
    p.col_tiles = (x.w + 127) / 128;
  } else {
    p.row_mode = 0;
    p.TW = x.w;
    p.P = x.w + 2 * p.halo;
    p.R = std::max(1, std::min(x.h, (tc::BLOCK_M * p.MB - p.TW) / p.P + 1));
    p.MB = ((p.R - 1) * p.P + p.TW + tc::BLOCK_M - 1) / tc::BLOCK_M;
    p.col_tiles = 1;
  }
  // the head folds into the fast row-mode epilogue of a one-N-tile, 64-column
  // 3x3 FP4 conv whose output block is channels 0-63 at word 0 (what
  // head_tab64_kernel reads); anything else leaves it to its own kernel
  const bool fuse_head = head && head->tab && head->logits && fp4 && !cv->transposed && acc == nullptr &&
                         p.row_mode && cv->n_tile == 64 && cv->n_gemm == 64 && cv->n_tiles == 1 &&
                         cv->c_out == 64 && out_stride == 2 && out_offset == 0;
  const size_t head_bytes = fuse_head ? 16 * 16 * sizeof(double) : 0;
  p.p_magic = uint32_t((0x100000000ull + p.P - 1) / p.P);
  p.buf_cols = fp4 && p.nbuf != 2 ? p.MB * cv->n_tile : tc::ACC_COLS;
  p.row_tiles = (x.h + p.R - 1) / p.R;
  const int q_last = p.row_mode ? (p.MB - 1 + p.halo) * p.P + p.halo
                                : p.halo * p.P + p.halo + tc::BLOCK_M * (p.MB - 1);
  int Q = q_last + tc::BLOCK_M + (p.halo ? p.P + 1 : 0);
  Q = std::max(Q, (p.R + 2 * p.halo) * p.P);
  Q = (Q + 7) / 8 * 8;
  if (Q > tc::prod_items(cv->taps) * tc::PROD_THREADS)
    return fail(MBU_ERR_UNSUPPORTED, "tcgen05 conv strip taller than the producer tiling");
  p.Q = Q;
  // one-tap convs pack four 32-lane chunks (a 128-lane block) into a stage;
  // FP4 3x3 stages hold a chunk pair (K = 64 e2m1 lanes in the same 32 B row)
  // FP4 N = 128 one-block layers take both pairs of a 128-lane block per stage
  // (one TMA box and one commit per block; measured -9% on those layers)
  const bool pps2 = allow_pps2 && fp4 && cv->pair2_ok && cv->n_tile == 128 && p.MB == 1 &&
                    !std::getenv("MBU_FP4_PPS1");
  const int cps = fp4 ? (pps2 ? 4 : 2) : cv->taps == 1 ? cv->tap1_cps : 1;
  // CTA pairs (M = 256 MMAs, half of B per CTA) for the single-buffer FP4
  // tiles with per-block commits; MBU_PAIR=0 keeps one-CTA MMAs
  static const bool pair_env = !std::getenv("MBU_PAIR") || std::atoi(std::getenv("MBU_PAIR")) != 0;
  const bool pair = allow_pair && pair_env && fp4 && cps == 2 && p.nbuf == 1 && p.MB <= 8 && cv->d_b4p &&
                    cv->d_bias_slab4p && (cv->n_tile == 64 || cv->n_tile == 128) &&
                    !std::getenv("MBU_NO_BLOCK_COMMIT");
  p.b_rows = pair ? cv->n_tile / 2 : cv->n_tile;
  const int kcs = fp4 ? 2 * cv->kp : cv->kc;
  if (kcs % cps) return fail(MBU_ERR_UNSUPPORTED, "tcgen05 one-tap conv needs whole 128-lane blocks");
  p.ks = kcs / cps;
  p.vec = fp4 ? (cv->pair_consec && p.x_stride32 % 2 == 0 && p.x_off32 % 2 == 0)
              : ((cv->chunk_consec >> (cps >> 1)) & 1) && p.x_stride32 % cps == 0 && p.x_off32 % cps == 0 &&
                    (!x.split || (p.x2_stride32 % cps == 0 && p.split32 % cps == 0));
  if (x.split && (x.split % 2 || x.split > x.wpp))
    return fail(MBU_ERR_LAYOUT, "split input view must break at a 128-lane block");
  p.a_chunk_bytes = uint32_t(Q) * 32;
  p.a_stage_bytes = uint32_t((size_t(Q) * 32 * (fp4 ? cps / 2 : cps) + 1023) / 1024 * 1024);
  p.b_stage_bytes = uint32_t(cv->b_stage_bytes * (fp4 ? cps / 2 : cps) / (pair ? 2 : 1));
  p.b_pair_bytes = uint32_t(cv->b_stage_bytes / (pair ? 2 : 1));
  const int raw_stages = (cv->taps == 9 ? tc::LA_CONV3 : tc::LA_TAP1) + 1;
  // shared memory: [header][A stages][B stages | resident B][raw ring][runs, biases][ones][slabs][slab map]
  // (FP4: the raw ring holds TMA boxes of one 128-lane block per strip pixel)
  CUtensorMap xmap, xmap2;
  std::memset(&xmap, 0, sizeof(xmap));
  std::memset(&xmap2, 0, sizeof(xmap2));
  p.raw_rows = p.R + 2 * p.halo;
  if (fp4) {
    p.rraw_box_bytes = uint32_t(16) * p.P * p.raw_rows;
    p.rraw_bytes = (p.rraw_box_bytes + 127) / 128 * 128;
    p.rraw_stages = 4;
    const uint64_t dims[4] = {uint64_t(p.x_stride32), uint64_t(x.w), uint64_t(x.h), uint64_t(x.n)};
    const uint64_t strides[3] = {uint64_t(p.x_stride32) * 4, uint64_t(p.x_stride32) * 4 * x.w,
                                 uint64_t(p.x_stride32) * 4 * x.w * x.h};
    const uint32_t box[4] = {4, uint32_t(p.P), uint32_t(p.raw_rows), 1};
    if (p.P > 256 || p.raw_rows > 256 || p.x_stride32 % 4 || p.x_off32 % 4 ||
        (reinterpret_cast<uintptr_t>(x.base) & 15) || !make_tmap_u32_4d(&xmap, x.base, dims, strides, box))
      return fail(MBU_ERR_UNSUPPORTED, "tcgen05 FP4 conv: raw activation tensor map unavailable");
    if (x.split) {  // the concat's second operand: its own contiguous tensor
      const uint64_t d2[4] = {uint64_t(p.x2_stride32), uint64_t(x.w), uint64_t(x.h), uint64_t(x.n)};
      const uint64_t s2[3] = {uint64_t(p.x2_stride32) * 4, uint64_t(p.x2_stride32) * 4 * x.w,
                              uint64_t(p.x2_stride32) * 4 * x.w * x.h};
      if (p.x2_stride32 % 4 || (reinterpret_cast<uintptr_t>(x.base2) & 15) ||
          !make_tmap_u32_4d(&xmap2, x.base2, d2, s2, box))
        return fail(MBU_ERR_UNSUPPORTED, "tcgen05 FP4 conv: second raw activation tensor map unavailable");
    }
  }
  const size_t raw_bytes = fp4 ? size_t(p.rraw_stages) * p.rraw_bytes : size_t(raw_stages) * Q * cps * 4;
  const size_t runs_bytes = size_t(cv->n_tiles) * 9 * 16 + size_t(cv->n_tiles) * cv->n_tile * 4;
  const int n_slabs = fp4 ? cv->n_slabs4 : cv->n_slabs;
  const size_t slab_bytes = size_t(n_slabs) * p.b_rows * 32;
  const size_t bias_bytes = n_slabs ? 4096 + slab_bytes + 1024 : 0;
  const size_t budget =
      227 * 1024 - tc::SMEM_HEADER - raw_bytes - runs_bytes - bias_bytes - 1024 - 128 - head_bytes;
  const size_t b_all = size_t(cv->n_tiles) * p.ks * p.b_stage_bytes;
  p.b_resident = b_all + 3 * size_t(p.a_stage_bytes) <= budget;
  const size_t stage = size_t(p.a_stage_bytes) + (p.b_resident ? 0 : p.b_stage_bytes);
  int stages = int((budget - (p.b_resident ? b_all : 0)) / stage);
  if (stages < 2) return kNoFit;
  p.stages = std::min(stages, tc::MAX_STAGES);
  size_t off = tc::SMEM_HEADER + size_t(p.stages) * p.a_stage_bytes;
  p.off_b = uint32_t(off);
  off += p.b_resident ? b_all : size_t(p.stages) * p.b_stage_bytes;
  off = (off + 127) / 128 * 128;  // (TMA destinations: 128-B aligned)
  p.off_raw = uint32_t(off);
  p.off_rraw = uint32_t(off);
  off += raw_bytes;
  p.off_runs = uint32_t(off);
  off += runs_bytes;
  p.mma_bias = n_slabs > 0;
  p.n_slabs = n_slabs;
  p.bias_slab = fp4 ? reinterpret_cast<const int8_t *>(pair ? cv->d_bias_slab4p : cv->d_bias_slab4) : cv->d_bias_slab;
  p.slab_of_nt = fp4 ? cv->d_slab_of_nt4 : cv->d_slab_of_nt;
  for (int i = 0; i < 16 && i < cv->n_tiles; ++i) p.slab_small[i] = fp4 ? cv->h_slab_of_nt4[i] : cv->h_slab_of_nt[i];
  off = (off + 1023) / 1024 * 1024;
  p.off_ones = uint32_t(off);
  p.off_slab = uint32_t(off + (p.mma_bias ? 4096 : 0));
  p.off_slabmap = uint32_t(p.off_slab + (p.mma_bias ? slab_bytes : 0));
  off = p.off_slabmap + (p.mma_bias ? size_t(cv->n_tiles) * 4 : 0);
  if (fuse_head) {
    off = (off + 15) / 16 * 16;
    p.off_head = uint32_t(off);
    off += head_bytes;
    p.head_logits = head->logits;
    p.head_mask = head->mask;
    p.head_tab = head->tab;
    p.head_bias = head->bias;
  }
  const size_t smem_total = off;
  p.u8_act = cv->pad_mode != MBU_PAD_ZERO;
  p.kc = kcs;
  p.chunk_word = fp4 ? cv->d_chunk_pair : cv->d_chunk_word;
  p.b = fp4 ? (pair ? cv->d_b4p : cv->d_b4) : cv->d_b;
  // instruction descriptor: s32 accum, A u8 (neg_one) / s8 (zero pad), B s8,
  // K-major both, N, M = 128; FP4: block-scaled, A/B e2m1, UE8M0 scales, K = 64
  p.idesc = fp4 ? ((1u << 7) | (1u << 10) | (uint32_t(cv->n_tile >> 3) << 17) | (1u << 23) |
                   (uint32_t((pair ? 2 : 1) * tc::BLOCK_M >> 4) << 24))
                : ((2u << 4) | (uint32_t(p.u8_act ? 0 : 1) << 7) | (1u << 10) |
                   (uint32_t(cv->n_tile >> 3) << 17) | (uint32_t(tc::BLOCK_M >> 4) << 24));
  p.sf1 = tc::TMEM_COLS - 8;
  p.sf256 = tc::TMEM_COLS - 4;
  p.c_out = cv->c_out;
  p.c_out_pad = cv->c_out_pad;
  p.n_gemm = cv->n_gemm;
  p.tconv_s = cv->transposed ? cv->stride : 0;
  p.ho = ho;
  p.wo = wo;
  p.acc = acc;
  p.bits = reinterpret_cast<uint32_t *>(bits);
  p.out_stride32 = out_stride * 2;
  p.out_off32 = out_offset * 2;
  p.out_groups = cv->out_wpp * 2;
  p.col_bias = static_cast<const int32_t *>(cv->d_thr2);
  p.col_sgn = p.col_bias + cv->n_pad + 32;
  p.col_w = p.col_sgn + cv->n_pad + 32;
  const int64_t tiles = int64_t(x.n) * p.row_tiles * p.col_tiles * p.n_tiles;
  if (tiles == 0) return MBU_OK;
  if (tiles > 0x7FFFFFFF) return fail(MBU_ERR_SHAPE, "tcgen05 conv grid too large");
  p.num_tiles = int(tiles);
  p.n_spatial = int(tiles / cv->n_tiles);
  p.n_pairs = cv->n_tiles * ((p.n_spatial + 1) / 2);
  // magic divisors: umulhi(n, ceil(2^32/d)) == n / d whenever n * d < 2^32
  auto magic = [](int d) { return d == 1 ? 0u : uint32_t((0x100000000ull + d - 1) / d); };
  {
    const uint64_t t1 = uint64_t(tiles), t2 = t1 / cv->n_tiles, t3 = t2 / p.col_tiles;
    if (t1 * cv->n_tiles >= (1ull << 32) || t2 * p.col_tiles >= (1ull << 32) ||
        t3 * p.row_tiles >= (1ull << 32))
      return fail(MBU_ERR_UNSUPPORTED, "tcgen05 conv tile grid outside the magic-division range");
  }
  p.nt_magic = magic(cv->n_tiles);
  p.ct_magic = magic(p.col_tiles);
  p.rt_magic = magic(p.row_tiles);
  const int grid = int(std::min<int64_t>(tiles, num_sms()));
  const size_t smem = std::max<size_t>(smem_total, tc::MIN_SMEM);
  if (smem > 227 * 1024) return kNoFit;
  if (fuse_head) head->done = true;
  if (cv->transposed && cps == 2) return launch_tc_impl<1, true, tc::LA_TAP1, 2, false>(p, xmap, xmap2, grid, smem, st);
  if (cv->transposed) return launch_tc_impl<1, true, tc::LA_TAP1, 4, false>(p, xmap, xmap2, grid, smem, st);
  if (fp4 && cps == 4) return launch_tc_impl<9, false, tc::LA_CONV3, 4, true>(p, xmap, xmap2, grid, smem, st);
  if (pair) return launch_tc_impl<9, false, tc::LA_CONV3, 2, true, true, true>(p, xmap, xmap2, grid, smem, st);
  if (fp4 && p.nbuf == 1 && p.MB <= 8 && !std::getenv("MBU_NO_BLOCK_COMMIT"))
    return launch_tc_impl<9, false, tc::LA_CONV3, 2, true, true>(p, xmap, xmap2, grid, smem, st);
  if (fp4) return launch_tc_impl<9, false, tc::LA_CONV3, 2, true>(p, xmap, xmap2, grid, smem, st);
  if (cv->taps == 9) return launch_tc_impl<9, false, tc::LA_CONV3, 1, false>(p, xmap, xmap2, grid, smem, st);
  if (cps == 2) return launch_tc_impl<1, false, tc::LA_TAP1, 2, false>(p, xmap, xmap2, grid, smem, st);
  return launch_tc_impl<1, false, tc::LA_TAP1, 4, false>(p, xmap, xmap2, grid, smem, st);
}

}  // namespace mbu
