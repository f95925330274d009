// Legacy warp-level tensor-core rates on sm_100a, for the north star's
// "binary tensor-core path (warp-level b1 mma.sync AND+popc)" question:
//   * b1:  mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc
//   * s8:  mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32
// Every SM runs 16 warps, each with 4 independent accumulators in flight;
// reported as MAC/clk/SM (a b1 "MAC" is one AND+popc lane). The tcgen05
// rates this engine uses (kind::i8, kind::mxf4) come from tools/ubench_tc.cu
// and tools/ubench_fp4.cu; tools/mma_rates.py merges them into one table.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_mma_sync tools/ubench_mma_sync.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

template <bool B1>
__global__ void __launch_bounds__(512) mma_sync_rate(int iters, unsigned long long *clk, int *sink) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x9E3779B9u * (threadIdx.x + 7 * i + 1);
  for (int i = 0; i < 2; ++i) b[i] = 0x85EBCA6Bu * (threadIdx.x + 3 * i + 1);
  int c[4][4] = {};
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if constexpr (B1)
        asm volatile(
            "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc "
            "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      else
        asm volatile(
            "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 "
            "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  int s = 0;
  for (int j = 0; j < 4; ++j)
    for (int k = 0; k < 4; ++k) s += c[j][k];
  if (s == 0x12345678) sink[0] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *dclk;
  int *sink;
  cudaMalloc(&dclk, sms * 8);
  cudaMalloc(&sink, 4);
  const int iters = 4096, warps = 16;
  for (int b1 = 1; b1 >= 0; --b1) {
    for (int rep = 0; rep < 2; ++rep) {  // (first launch warms up)
      if (b1)
        mma_sync_rate<true><<<sms, 32 * warps>>>(iters, dclk, sink);
      else
        mma_sync_rate<false><<<sms, 32 * warps>>>(iters, dclk, sink);
    }
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<unsigned long long> c(sms);
    cudaMemcpy(c.data(), dclk, sms * 8, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (auto v : c) mx = v > mx ? v : mx;
    const double macs = double(iters) * 4 * warps * (b1 ? 16.0 * 8 * 256 : 16.0 * 8 * 32);
    printf("{\"bench\": \"mma_sync\", \"kind\": \"%s\", \"err\": \"%s\", \"mac_per_clk_per_sm\": %.0f}\n",
           b1 ? "b1.and.popc m16n8k256" : "s8 m16n8k32", cudaGetErrorString(e), macs / double(mx));
  }
  return 0;
}
