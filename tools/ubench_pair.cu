// CTA-pair (cta_group::2) kind::mxf4 MMAs: operand split check and rate.
//
// Check: each CTA of a cluster pair fills its A half (128 rows x K = 64 e2m1,
// row r = a one-hot at K position ka(rank, r)) and half of B (N / 2 rows of
// codes), the leader issues one M = 256 MMA, and both CTAs read their 128 TMEM
// lanes back. Expected (the PTX ISA's 2-CTA operand layout): D rows 0-127 in
// CTA 0's TMEM, 128-255 in CTA 1's, B rows [0, N/2) from CTA 0 and [N/2, N)
// from CTA 1, both at the same shared-memory offset.
// Rate: the leader issues rounds of 9 tap-shifted MMAs (the conv kernel's
// walk) with a commit per round, like tools/ubench_dual.cu; one-CTA kernels
// give the cta_group::1 baseline. Reports clocks per MMA (per SM pair / per SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_pair tools/ubench_pair.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;
  return d;
}
__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// e2m1 code -> value
__host__ __device__ inline float e2m1v(int c) {
  const float m[8] = {0.f, 0.5f, 1.f, 1.5f, 2.f, 3.f, 4.f, 6.f};
  return (c & 8) ? -m[c & 7] : m[c & 7];
}
__host__ __device__ inline int ka_of(int rank, int r) { return (r * 5 + rank * 17) % 64; }
__host__ __device__ inline int bcode(int n, int k) { return (n + 3 * k) % 16; }

// element k of a K-major no-swizzle row: core-matrix column k / 32 (LBO apart), byte (k % 32) / 2, nibble k & 1
__device__ void put_e2m1(uint8_t *base, uint32_t lbo, int row, int k, int code) {
  uint8_t *p = base + (k / 32) * lbo + row * 16 + (k % 32) / 2;
  *p = uint8_t(*p | (code << (4 * (k & 1))));
}

template <bool PAIR>
__global__ void pair_check(int N, float *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0);
  const uint32_t rank = PAIR ? cta_rank() : 0;
  const int nb = PAIR ? N / 2 : N;  // B rows held here
  uint8_t *a = smem, *b = smem + 8192;
  for (int i = threadIdx.x; i < 8192 + 8192; i += blockDim.x) smem[i] = 0;
  __syncthreads();
  if (threadIdx.x < 128) put_e2m1(a, 128 * 16, threadIdx.x, ka_of(rank, threadIdx.x), 2);  // 1.0
  for (int n = threadIdx.x; n < nb; n += blockDim.x)
    for (int k = 0; k < 64; ++k) put_e2m1(b, nb * 16, n, k, bcode(n + rank * nb, k));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (PAIR) cluster_sync(); else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  if (warp < 4) {
    const uint32_t lq = tmem + (uint32_t(warp * 32) << 16) + 504;
    for (int c = 0; c < 8; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(lq + c), "r"(0x7F7F7F7Fu) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (PAIR) cluster_sync(); else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 1 && rank == 0) {
    const uint32_t idesc = (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) |
                           (uint32_t((PAIR ? 256 : 128) >> 4) << 24);
    const uint64_t ad = umma_desc(smem_u32(a), 128 * 16, 128), bd = umma_desc(smem_u32(b), nb * 16, 128);
    if (PAIR)
      asm volatile(
          "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, 0, 0;\n\t"
          "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%4], p;\n\t"
          "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%5], %6;\n\t}"
          ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(tmem + 504), "r"(smem_u32(&bar)), "h"(uint16_t(3))
          : "memory");
    else
      asm volatile(
          "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, 0, 0;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%4], p;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t}"
          ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(tmem + 504), "r"(smem_u32(&bar))
          : "memory");
  }
  if (warp < 4) {
    wait_bar(smem_u32(&bar), 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int row = warp * 32 + (threadIdx.x & 31);
    for (int c = 0; c < N; ++c) {
      uint32_t v;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                   : "=r"(v)
                   : "r"(tmem + (uint32_t(warp * 32) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      out[(size_t(blockIdx.x) * 128 + row) * N + c] = __uint_as_float(v);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (PAIR) cluster_sync(); else __syncthreads();
  if (warp == 0) {
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// rounds of 9 tap-shifted MMAs (A strip of 3 x 130 rows, B one slab per tap), commit per round, 2-deep ring
template <bool PAIR, bool F16 = false>
__global__ void pair_rate(int N, int reps, unsigned long long *clk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[2];
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0);
  const uint32_t rank = PAIR ? cta_rank() : 0;
  const int nb = PAIR ? N / 2 : N;
  const int Q = 3 * 130 + 8;
  uint8_t *a = smem, *b = smem + Q * 32 + 1024;
  for (int i = threadIdx.x; i < (Q * 32 + 1024 + 9 * nb * 32) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t *>(smem)[i] = 0x22222222u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (PAIR) cluster_sync(); else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  if (warp < 4) {
    const uint32_t lq = tmem + (uint32_t(warp * 32) << 16) + 504;
    for (int c = 0; c < 8; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(lq + c), "r"(0x7F7F7F7Fu) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (PAIR) cluster_sync(); else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 1 && rank == 0) {
    // F16: kind::f16, f32 accumulator, K = 16 fp16 (the stem's MMA; same 32-B rows)
    const uint32_t idesc = F16 ? ((1u << 4) | (uint32_t(N >> 3) << 17) | (uint32_t((PAIR ? 256 : 128) >> 4) << 24))
                               : ((1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) |
                                  (uint32_t((PAIR ? 256 : 128) >> 4) << 24));
    const uint64_t ad = umma_desc(smem_u32(a) + 131 * 16, Q * 16, 128), bd = umma_desc(smem_u32(b), nb * 16, 128);
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const int buf = r & 1;
      if (r >= 2) wait_bar(smem_u32(&bar[buf]), ((r - 2) >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d = tmem + uint32_t(buf * 128);
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) {
        const uint64_t at = ad + uint64_t((tap / 3 - 1) * 130 + (tap % 3 - 1));
        const uint64_t bt = bd + uint64_t(tap * nb * 2);
        if (F16 && PAIR)
          asm volatile(
              "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
              "l"(at), "l"(bt), "r"(idesc), "r"(tap)
              : "memory");
        else if (F16)
          asm volatile(
              "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
              "l"(at), "l"(bt), "r"(idesc), "r"(tap)
              : "memory");
        else if (PAIR)
          asm volatile(
              "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}" ::"r"(d),
              "l"(at), "l"(bt), "r"(idesc), "r"(tap), "r"(tmem + 504)
              : "memory");
        else
          asm volatile(
              "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}" ::"r"(d),
              "l"(at), "l"(bt), "r"(idesc), "r"(tap), "r"(tmem + 504)
              : "memory");
      }
      if (PAIR)
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
            ::"r"(smem_u32(&bar[buf])), "h"(uint16_t(3))
            : "memory");
      else
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
                smem_u32(&bar[buf]))
            : "memory");
    }
    for (int r = reps - 2; r < reps; ++r) wait_bar(smem_u32(&bar[r & 1]), (r >> 1) & 1);
    if ((threadIdx.x & 31) == 0) clk[blockIdx.x] = clock64() - t0;
  }
  if (PAIR && rank == 1 && warp == 1) {  // the peer's copy of the commits: drain both barriers
    for (int r = reps - 2; r < reps; ++r) wait_bar(smem_u32(&bar[r & 1]), (r >> 1) & 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (PAIR) cluster_sync(); else __syncthreads();
  if (warp == 0) {
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <typename K, typename... Args>
static cudaError_t launch(K kern, bool pair, int grid, size_t smem, Args... args) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = pair ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
  if (e != cudaSuccess) return e;
  return cudaDeviceSynchronize();
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *dout;
  cudaMalloc(&dout, 2 * 128 * 256 * 4);
  for (int N : {64, 128, 256}) {
    for (int pair = 0; pair <= 1; ++pair) {
      cudaMemset(dout, 0xFF, 2 * 128 * 256 * 4);
      const cudaError_t e = pair ? launch(pair_check<true>, true, 2, 32768, N, dout)
                                 : launch(pair_check<false>, false, 1, 32768, N, dout);
      std::vector<float> o(2 * 128 * N);
      cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0, bad_lo = 0, bad_hi = 0;
      for (int c = 0; c <= pair; ++c)
        for (int r = 0; r < 128; ++r)
          for (int n = 0; n < N; ++n) {
            const float want = e2m1v(bcode(n, ka_of(c, r)));
            if (o[(size_t(c) * 128 + r) * N + n] != want) {
              ++bad;
              (n < N / 2 ? bad_lo : bad_hi)++;
              if (bad <= 3)
                printf("  mismatch cta %d row %d n %d: got %g want %g\n", c, r, n, o[(size_t(c) * 128 + r) * N + n], want);
            }
          }
      printf("{\"bench\": \"pair_check\", \"pair\": %d, \"N\": %d, \"err\": \"%s\", \"bad\": %d, \"bad_n_lo\": %d, "
             "\"bad_n_hi\": %d}\n",
             pair, N, cudaGetErrorString(e), bad, bad_lo, bad_hi);
      if (e != cudaSuccess) return 1;
    }
  }
  unsigned long long *dclk;
  cudaMalloc(&dclk, sms * 8);
  for (int N : {64, 128})
    for (int pair = 0; pair <= 1; ++pair) {  // kind::f16, K = 16 (the stem)
      const int reps = 20000;
      cudaMemset(dclk, 0, sms * 8);
      const size_t smem = size_t(3 * 130 + 8) * 32 + 1024 + 9 * N * 32 + 1024;
      const int grid = sms / 2 * 2;
      const cudaError_t e = pair ? launch(pair_rate<true, true>, true, grid, smem, N, reps, dclk)
                                 : launch(pair_rate<false, true>, false, grid, smem, N, reps, dclk);
      std::vector<unsigned long long> c(sms);
      cudaMemcpy(c.data(), dclk, sms * 8, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (auto v : c) mx = v > mx ? v : mx;
      const double per = double(mx) / (9.0 * reps);
      const double mac = (pair ? 256.0 * N * 16 / 2 : 128.0 * N * 16) / per;
      printf("{\"bench\": \"pair_rate_f16\", \"pair\": %d, \"N\": %d, \"err\": \"%s\", \"clk_per_mma\": %.1f, "
             "\"mac_per_clk_per_sm\": %.0f}\n",
             pair, N, cudaGetErrorString(e), per, mac);
      if (e != cudaSuccess) return 1;
    }
  for (int N : {64, 128, 256})
    for (int pair = 0; pair <= 1; ++pair) {
      const int reps = 20000;
      cudaMemset(dclk, 0, sms * 8);
      const size_t smem = size_t(3 * 130 + 8) * 32 + 1024 + 9 * N * 32 + 1024;
      const int grid = sms / 2 * 2;
      const cudaError_t e = pair ? launch(pair_rate<true>, true, grid, smem, N, reps, dclk)
                                 : launch(pair_rate<false>, false, grid, smem, N, reps, dclk);
      std::vector<unsigned long long> c(sms);
      cudaMemcpy(c.data(), dclk, sms * 8, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (auto v : c) mx = v > mx ? v : mx;
      const double per = double(mx) / (9.0 * reps);
      // MACs per SM per clock: a pair MMA does 256 x N x 64 over two SMs
      const double mac = (pair ? 256.0 * N * 64 / 2 : 128.0 * N * 64) / per;
      printf("{\"bench\": \"pair_rate\", \"pair\": %d, \"N\": %d, \"err\": \"%s\", \"clk_per_mma\": %.1f, "
             "\"mac_per_clk_per_sm\": %.0f}\n",
             pair, N, cudaGetErrorString(e), per, mac);
      if (e != cudaSuccess) return 1;
    }
  return 0;
}
