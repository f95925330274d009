// Microbenchmarks for the conv_tc design decisions (run on a B200):
//   tmem_read : tcgen05.ld.32x32b.x64 throughput (bytes / SM clock) for 4, 8, 16 reading warps
//   mma_rate  : tcgen05.mma kind::i8 (both operands in smem) clocks per MMA for N = 64/128/256,
//               with the A descriptor start aligned or shifted by one 16-B row (the tap shift)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench_tc tools/ubench_tc.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

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

__global__ void tmem_read(int iters, int nwarps, unsigned long long *out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot + (uint32_t((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  const unsigned long long t0 = clock64();
  if (warp < nwarps) {
    for (int i = 0; i < iters; ++i) {
      uint32_t v[64];
      const uint32_t col = uint32_t(((i * 4 + (warp >> 2)) * 64) & 511);
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
          : "r"(tmem + col));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 64; ++j) acc ^= v[j];
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x * 2] = t1 - t0;
  if (acc == 0x12345678u) out[blockIdx.x * 2 + 1] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

__global__ void mma_rate(int iters, int n, int shift, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x01010101u * (i & 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
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
  unsigned long long dt = 0;
  if (threadIdx.x == 0) {
    // A: 256 rows x 32 B K-major core matrices ([khalf][row][16B]); B: n rows
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
    const uint64_t ad = umma_desc(a, 256 * 16, 128);
    const uint64_t bd = umma_desc(b, uint32_t(n) * 16, 128);
    const uint32_t idesc = (2u << 4) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(slot + uint32_t((i & 1) * 256)),
          "l"(ad + uint64_t(shift ? (i & 7) : 0)), "l"(bd), "r"(idesc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    dt = clock64() - t0;
    out[blockIdx.x] = dt;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *d, h[2 * 148];
  cudaMalloc(&d, sizeof(h));
  const int iters = 4096;
  for (int nw : {4, 8, 16}) {
    tmem_read<<<sms, 512>>>(iters, nw, d);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const double bytes = double(iters) * nw * 32 * 64 * 4;
    printf("{\"bench\": \"tmem_read\", \"warps\": %d, \"cycles\": %llu, \"bytes_per_clk_per_sm\": %.1f}\n", nw, h[0],
           bytes / double(h[0]));
  }
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int n : {64, 128, 256})
    for (int shift : {0, 1}) {
      mma_rate<<<sms, 128, 64 * 1024>>>(iters, n, shift, d);
      cudaError_t e = cudaMemcpy(h, d, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      const double macs = 128.0 * n * 32;
      printf("{\"bench\": \"mma_i8_ss\", \"n\": %d, \"a_shift_rows\": %d, \"clk_per_mma\": %.1f, \"mac_per_clk\": %.0f}\n",
             n, shift, double(h[0]) / iters, macs * iters / double(h[0]));
    }
  return 0;
}
