// Can two warps of one CTA issue tcgen05.mma concurrently? Each of `issuers`
// warps issues `reps` rounds of 9 kind::mxf4 MMAs (M = 128, N = 64, K = 64)
// into its own TMEM columns and commits every round to its own mbarrier,
// waiting for round r - 1's commit before issuing round r + 1 (a two-deep
// ring, like the conv kernel's accumulator buffers). Reports clocks per MMA
// per SM and checks the accumulated values.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_dual tools/ubench_dual.cu
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

__global__ void dual_issue(int issuers, int reps, unsigned long long *clk, float *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[4];
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0);
  uint8_t *a = smem, *b = smem + 65536;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(a)[i] = 0x22222222u;  // 1.0
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(b)[i] = 0x22222222u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  if (warp < 4) {  // block scales 2^0 in columns 504..511
    const uint32_t base = tmem + (uint32_t(warp * 32) << 16) + 504;
    for (int c = 0; c < 8; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(base + c), "r"(0x7F7F7F7Fu) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < issuers) {
    const uint32_t idesc = (1u << 7) | (1u << 10) | (uint32_t(64 >> 3) << 17) | (1u << 23) | (uint32_t(128 >> 4) << 24);
    const uint32_t sf = tmem + 504;
    const uint64_t ad = umma_desc(smem_u32(a), 128 * 16, 128), bd = umma_desc(smem_u32(b), 64 * 16, 128);
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const int buf = r & 1;
      if (r >= 2) wait_bar(smem_u32(&bar[warp * 2 + buf]), ((r - 2) >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d = tmem + uint32_t(warp * 128 + buf * 64);
#pragma unroll
      for (int tap = 0; tap < 9; ++tap)
        asm volatile(
            "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}" ::"r"(d),
            "l"(ad + uint64_t(tap)), "l"(bd), "r"(idesc), "r"(tap), "r"(sf)
            : "memory");
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
              smem_u32(&bar[warp * 2 + buf]))
          : "memory");
    }
    for (int r = reps - 2; r < reps; ++r) wait_bar(smem_u32(&bar[warp * 2 + (r & 1)]), (r >> 1) & 1);
    if ((threadIdx.x & 31) == 0) clk[blockIdx.x * 4 + warp] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4 && blockIdx.x == 0) {  // column 0 of warp 0's buffer 0 (lane = row): 9 taps x 64 = 576 per round
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + (uint32_t(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    out[threadIdx.x] = __uint_as_float(v);
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(dual_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  unsigned long long *dclk;
  float *dout;
  cudaMalloc(&dclk, sms * 4 * 8);
  cudaMalloc(&dout, 128 * 4);
  for (int issuers : {1, 2})
    for (int reps : {4, 1000, 20000}) {
      cudaMemset(dclk, 0, sms * 32);
      dual_issue<<<sms, 256, 100 * 1024>>>(issuers, reps, dclk, dout);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<unsigned long long> c(sms * 4);
      std::vector<float> o(128);
      cudaMemcpy(c.data(), dclk, c.size() * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(o.data(), dout, 128 * 4, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int i = 0; i < sms; ++i)
        for (int w = 0; w < issuers; ++w) mx = std::max(mx, c[i * 4 + w]);
      printf("{\"bench\": \"dual_issue\", \"issuers\": %d, \"reps\": %d, \"err\": \"%s\", \"clk_per_mma_per_sm\": %.1f, "
             "\"acc0\": %g, \"expect\": %d}\n",
             issuers, reps, cudaGetErrorString(e), double(mx) / (9.0 * reps * issuers), o[0], 576);
      if (e != cudaSuccess) return 1;
    }
  return 0;
}
