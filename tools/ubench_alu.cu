// Issue cost of the epilogue's ALU idioms on sm_100a: clocks per warp
// instruction per SM sub-partition for fminf(|a|, |b|) pairs (FMNMX3), 2-input
// fminf (FMNMX), funnel shifts (SHF.L.W, the sign pack), FADD and LOP3.
// 16 warps per SM (4 per sub-partition), 8 independent chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_alu tools/ubench_alu.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

template <int OP>
__global__ void __launch_bounds__(512) alu_rate(int iters, unsigned long long *clk, uint32_t *sink) {
  uint32_t r[8], s[8];
  for (int i = 0; i < 8; ++i) {
    r[i] = 0x3F800000u + threadIdx.x * 7 + i;
    s[i] = 0x3F000000u + threadIdx.x * 3 + i;
  }
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (OP == 0) {  // fmin of |x| and |y| into the chain: FMNMX3
        r[i] = __float_as_uint(fminf(__uint_as_float(r[i]), fminf(fabsf(__uint_as_float(s[i])),
                                                                  fabsf(__uint_as_float(s[(i + 1) & 7])))));
      } else if constexpr (OP == 1) {  // 2-input fmin: FMNMX
        r[i] = __float_as_uint(fminf(__uint_as_float(r[i]), __uint_as_float(s[i])));
      } else if constexpr (OP == 2) {  // funnel shift: SHF.L.W
        r[i] = __funnelshift_l(s[i], r[i], 1);
      } else if constexpr (OP == 3) {  // FADD
        r[i] = __float_as_uint(__uint_as_float(r[i]) + __uint_as_float(s[i]));
      } else {  // LOP3
        r[i] = (r[i] & s[i]) ^ s[(i + 3) & 7];
      }
    }
    // keep s varying so nothing is loop-invariant
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i] ^= r[(i + 1) & 7];
  }
  const unsigned long long t1 = clock64();
  uint32_t x = 0;
  for (int i = 0; i < 8; ++i) x ^= r[i];
  if (x == 0x12345678u) sink[0] = x;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *dclk;
  uint32_t *sink;
  cudaMalloc(&dclk, sms * 8);
  cudaMalloc(&sink, 4);
  const char *names[5] = {"FMNMX3 (fminf of |a|,|b|)", "FMNMX (fminf)", "SHF.L.W (funnel shift)", "FADD", "LOP3"};
  const int iters = 4096;
  for (int op = 0; op < 5; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: alu_rate<0><<<sms, 512>>>(iters, dclk, sink); break;
        case 1: alu_rate<1><<<sms, 512>>>(iters, dclk, sink); break;
        case 2: alu_rate<2><<<sms, 512>>>(iters, dclk, sink); break;
        case 3: alu_rate<3><<<sms, 512>>>(iters, dclk, sink); break;
        default: alu_rate<4><<<sms, 512>>>(iters, dclk, sink); break;
      }
    }
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<unsigned long long> c(sms);
    cudaMemcpy(c.data(), dclk, sms * 8, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (auto v : c) mx = v > mx ? v : mx;
    // per sub-partition: 4 warps x iters x (8 ops + 8 LOP3 xors for the s update)
    const double per = double(mx) / (4.0 * iters * 16);
    printf("{\"bench\": \"alu_rate\", \"op\": \"%s\", \"err\": \"%s\", \"clk_per_warp_instr_mixed_with_lop3\": %.2f}\n",
           names[op], cudaGetErrorString(e), per);
  }
  return 0;
}
