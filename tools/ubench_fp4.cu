// Probe: tcgen05.mma kind::mxf4 (e2m1 operands, UE8M0 scale = 1 everywhere) as an exact
// integer engine for {-1,0,+1} x {0,1}/{-1,+1} dot products, and its throughput vs N.
//   - A: 128 rows x 64 e2m1 (32 B per row, K-major, no swizzle), B: N rows x 64 e2m1
//   - scale factors: TMEM columns 480..511 filled with 0x7F7F7F7F (2^0) -> any layout reads 1.0
//   - correctness: D after `reps` accumulating MMAs vs the CPU integer result
//   - strip: nine tap-shifted A descriptors over a 656-row strip (the kernel's walk), with and
//     without other warps storing to shared memory: the unrolled walk runs at the full rate
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench_fp4 tools/ubench_fp4.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
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

// a: [128][32 B] row-major packed e2m1 (element k of row r in byte r*32 + k/2, nibble k%2)
// b: [N][32 B]; out: [128][N] floats
__global__ void fp4_mma(const uint8_t *a, const uint8_t *b, int n, int reps, int timing, float *out,
                        unsigned long long *clk, int sfc, uint32_t sfa_val, int aoff = 0) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // core-matrix layout [khalf][row][16 B]
  for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) {
    const int r = i / 32, byte = i % 32, kh = byte / 16;
    smem[kh * 128 * 16 + r * 16 + (byte % 16)] = a[i];
  }
  for (int i = threadIdx.x; i < n * 32; i += blockDim.x) {
    const int r = i / 32, byte = i % 32, kh = byte / 16;
    smem[8192 + kh * n * 16 + r * 16 + (byte % 16)] = b[i];
  }
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
  const uint32_t tmem = slot;
  // scale factors = 1.0 in columns 480..511 of every lane
  {
    const uint32_t base = tmem + (uint32_t(warp * 32) << 16) + 480;
    for (int c = 0; c < 32; ++c) {
      uint32_t v = c < sfc ? 0x7F7F7F7Fu : (c >= 16 && c < 16 + sfc ? sfa_val : 0u);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(base + c), "r"(v) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    const uint64_t ad = umma_desc(smem_u32(smem) + 16u * aoff, 128 * 16, 128);
    const uint64_t bd = umma_desc(smem_u32(smem + 8192), uint32_t(n) * 16, 128);
    // block-scaled descriptor: A/B E2M1 (1), UE8M0 scales (bit 23), N, M = 128, K = 64
    const uint32_t idesc = (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (1u << 23) | (uint32_t(128 >> 4) << 24);
    const uint32_t sf = tmem + 480;
    const unsigned long long t0 = clock64();
    for (int i = 0; i < reps; ++i) {
      const uint32_t d = tmem;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
          "l"(ad), "l"(bd), "r"(idesc), "r"(i > 0 ? 1 : 0), "r"(sf + (sfa_val ? 16u : 0u)), "r"(sf));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    clk[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (!timing && blockIdx.x == 0 && warp < 4) {
    for (int c = 0; c < n; ++c) {
      uint32_t v;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + (uint32_t(warp * 32) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      out[(warp * 32 + lane) * n + c] = __uint_as_float(v);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}


// MMA rate under kernel-like conditions: nine tap-shifted A descriptors over a
// Q-row strip (LBO = Q * 16), B from a per-tap slab, and optionally other warps
// storing to shared memory (the producers' strip writes) while the MMAs run.
__global__ void fp4_mma_strip(int n, int q, int reps, int noise, unsigned long long *clk, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bar2;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5;
  uint8_t *a = smem, *b = smem + 65536, *scratch = smem + 65536 + 65536;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x22002200u;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(b)[i] = 0x0A020A02u;
  if (threadIdx.x == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)));
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
  if (warp < 4) {
    const uint32_t base = tmem + (uint32_t(warp * 32) << 16) + 480;
    for (int c = 0; c < 32; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(base + c), "r"(0x7F7F7F7Fu) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (1u << 23) | (uint32_t(128 >> 4) << 24);
    const uint32_t sf = tmem + 480;
    const int P = 130;
    const unsigned long long t0 = clock64();
    if (mode >= 3) {  // mode 2 plus a tcgen05.commit to a second barrier after every (mode - 2) blocks
      const uint64_t pp = P, bs = uint64_t(n) * 2;
      const int every = mode - 2;
      for (int i = 0; i < reps / 27; ++i)
        for (int blk = 0; blk < 3; ++blk) {
          const uint64_t ac = umma_desc(smem_u32(a) + 16u * ((blk + 1) * P + 1), uint32_t(q) * 16, 128);
          const uint64_t b0 = umma_desc(smem_u32(b), uint32_t(n) * 16, 128);
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const uint64_t ad = ac + (uint64_t(tap / 3) - 1) * pp + uint64_t(tap % 3) - 1;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}" ::"r"(
                    tmem + uint32_t(blk * n)),
                "l"(ad), "l"(b0 + uint64_t(tap) * bs), "r"(idesc), "r"(1), "r"(sf));
          }
          if (mode < 6 && (i * 3 + blk) % every == every - 1)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&bar2)));
          if (mode == 7 && (i * 3 + blk) % 5 == 9) clk[gridDim.x] = i;  // control flow, no commit
        }
        if (mode == 6)  // one commit per 27 MMAs, no per-block test
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              smem_u32(&bar2)));
    } else if (mode == 2) {  // unrolled 9-tap walk per block, 64-bit adds only (the kernel's umma9)
      const uint64_t pp = P, bs = uint64_t(n) * 2;
      for (int i = 0; i < reps / 27; ++i)
        for (int blk = 0; blk < 3; ++blk) {
          const uint64_t ac = umma_desc(smem_u32(a) + 16u * ((blk + 1) * P + 1), uint32_t(q) * 16, 128);
          const uint64_t b0 = umma_desc(smem_u32(b), uint32_t(n) * 16, 128);
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const uint64_t ad = ac + (uint64_t(tap / 3) - 1) * pp + uint64_t(tap % 3) - 1;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}" ::"r"(
                    tmem + uint32_t(blk * n)),
                "l"(ad), "l"(b0 + uint64_t(tap) * bs), "r"(idesc), "r"(1), "r"(sf));
          }
        }
    } else
    for (int i = 0; i < reps; ++i) {
      const int tap = mode == 1 ? 0 : i % 9, blk = mode == 1 ? 0 : (i / 9) % 3;
      const int q0 = (blk + 1) * P + 1 + (tap / 3 - 1) * P + (tap % 3 - 1);
      const uint64_t ad = umma_desc(smem_u32(a) + 16u * q0, uint32_t(q) * 16, 128);
      const uint64_t bd = umma_desc(smem_u32(b) + uint32_t(tap) * n * 32, uint32_t(n) * 16, 128);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}" ::"r"(
              tmem + uint32_t(blk * n)),
          "l"(ad), "l"(bd), "r"(idesc), "r"(1), "r"(sf));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    clk[blockIdx.x] = clock64() - t0;
    stop = 1;
  } else if (warp >= 4 && noise == 3) {
    // warps 4..15 parked in try_wait (suspend hint, as the kernel's mbar_wait) on a barrier
    // whose phase completes only when the MMAs are done
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0, %2;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0x989680));
  } else if (warp >= 4 && noise == 2) {
    // tcgen05.ld of the upper TMEM half (columns 256..479) by warps 4..15, until the MMAs finish
    const uint32_t lq = tmem + (uint32_t((warp & 3) * 32) << 16) + 256u + uint32_t((warp >> 2) - 1) * 64u;
    uint32_t acc = 0;
    while (!stop) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(lq & ~0u));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int i = 0; i < 16; ++i) acc += v[i];
    }
    if (acc == 0x12345678u) clk[gridDim.x + blockIdx.x] = acc;
  } else if (warp >= 4 && noise == 6) {
    // ALU-bound warps (the epilogue's funnel-shift packing), until the MMAs finish:
    // do they starve the MMA-issuing warp of issue slots?
    uint32_t a0 = threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u;
    while (!stop) {
#pragma unroll 16
      for (int j = 0; j < 64; ++j) {
        a0 = __funnelshift_l(a1, a0, 1);
        a1 = __funnelshift_l(a2, a1, 1);
        a2 = __funnelshift_l(a3, a2, 1);
        a3 = __funnelshift_l(a0, a3, 1);
      }
    }
    if ((a0 ^ a1 ^ a2 ^ a3) == 0x12345678u) clk[gridDim.x + blockIdx.x] = a0;
  } else if (warp >= 4 && warp < 8 && (noise == 4 || noise == 5)) {
    // tcgen05.ld.32x32b.x64 + wait::ld latency of one epilogue-sized load (64 columns of
    // the upper TMEM half) while the MMAs stream (4: until they finish) or with the
    // tensor core idle (5: 2000 loads, reps = 0)
    const uint32_t lq = tmem + (uint32_t((warp & 3) * 32) << 16) + 256u;
    unsigned long long tot = 0;
    unsigned cnt = 0, acc = 0;
    while (noise == 4 ? !stop : cnt < 2000) {
      uint32_t v[64];
      const unsigned long long t0 = clock64();
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
          : "r"(lq));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      tot += clock64() - t0;
      ++cnt;
#pragma unroll
      for (int i = 0; i < 64; ++i) acc ^= v[i];
    }
    if (warp == 4 && (threadIdx.x & 31) == 0) clk[gridDim.x + blockIdx.x] = (tot / (cnt ? cnt : 1)) | (acc & 1ull) << 63;
  } else if (warp >= 4 && noise) {
    // 16-B stores over a 32 KB scratch region (bandwidth hog), until the MMAs finish
    uint4 *sc = reinterpret_cast<uint4 *>(scratch);
    int k = threadIdx.x;
    while (!stop) {
#pragma unroll 8
      for (int j = 0; j < 64; ++j) {
        sc[k & 2047] = make_uint4(j, k, j, k);
        k += 256;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

static uint8_t enc(int v) { return v == 0 ? 0x0 : v == 1 ? 0x2 : v == -1 ? 0xA : v == 6 ? 0x7 : 0xF; }

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(fp4_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);
  srand(7);
  for (int n : {64, 128, 256}) {
    std::vector<int> av(128 * 64), bv(n * 64);
    std::vector<uint8_t> ap(128 * 32, 0), bp(n * 32, 0);
    for (int i = 0; i < 128 * 64; ++i) {
      av[i] = (i % 64 == 63) ? 6 : (rand() % 3) - 1;  // one large element per row
      ap[i / 2] |= enc(av[i]) << (4 * (i % 2));
    }
    for (int i = 0; i < n * 64; ++i) {
      bv[i] = (i % 64 == 63) ? 6 : (rand() % 3) - 1;
      bp[i / 2] |= enc(bv[i]) << (4 * (i % 2));
    }
    uint8_t *da, *db;
    float *dout;
    unsigned long long *dclk;
    cudaMalloc(&da, ap.size());
    cudaMalloc(&db, bp.size());
    cudaMalloc(&dout, 128 * n * 4);
    cudaMalloc(&dclk, 148 * 8);
    cudaMemcpy(da, ap.data(), ap.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(db, bp.data(), bp.size(), cudaMemcpyHostToDevice);
    const int reps = 300;  // |sum| up to 300 * (63 + 36) < 2^24
    for (int sfc : {1, 2, 4}) for (uint32_t sv : {0u, 0x87878787u}) {
      fp4_mma<<<1, 128, 32 * 1024>>>(da, db, n, 1, 0, dout, dclk, sfc, sv);
      std::vector<float> o1(128 * n);
      cudaMemcpy(o1.data(), dout, o1.size() * 4, cudaMemcpyDeviceToHost);
      long bad1 = 0;
      const double mul = sv ? 256.0 : 1.0;
      for (int r = 0; r < 128; ++r)
        for (int c = 0; c < n; ++c) {
          long s1 = 0;
          for (int k = 0; k < 64; ++k) s1 += long(av[r * 64 + k]) * bv[c * 64 + k];
          if (double(o1[r * n + c]) != mul * double(s1)) ++bad1;
        }
      printf("{\"probe\": \"sf_columns\", \"n\": %d, \"sf_cols_filled\": %d, \"a_scale\": %g, \"mismatches\": %ld}\n", n, sfc, mul, bad1);
    }
    fp4_mma<<<1, 128, 32 * 1024>>>(da, db, n, reps, 0, dout, dclk, 32, 0u);
    std::vector<float> out(128 * n);
    cudaError_t e = cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; }
    long bad = 0, maxabs = 0;
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < n; ++c) {
        long s = 0;
        for (int k = 0; k < 64; ++k) s += long(av[r * 64 + k]) * bv[c * 64 + k];
        s *= reps;
        maxabs = std::max(maxabs, std::labs(s));
        if (double(out[r * n + c]) != double(s)) ++bad;
      }
    for (int aoff : {1, 3, 8}) {
      fp4_mma<<<sms, 128, 32 * 1024>>>(da, db, n, 4096, 1, dout, dclk, 32, 0u, aoff);
      unsigned long long ck[148];
      cudaMemcpy(ck, dclk, sms * 8, cudaMemcpyDeviceToHost);
      printf("{\"bench\": \"mxf4_ss_aoff\", \"n\": %d, \"a_row_offset\": %d, \"clk_per_mma\": %.1f}\n", n, aoff,
             double(ck[0]) / 4096);
    }
    fp4_mma<<<sms, 128, 32 * 1024>>>(da, db, n, 4096, 1, dout, dclk, 32, 0u);
    unsigned long long clk[148];
    cudaMemcpy(clk, dclk, sms * 8, cudaMemcpyDeviceToHost);
    const double cpm = double(clk[0]) / 4096;
    printf("{\"bench\": \"mxf4_ss\", \"n\": %d, \"exact_mismatches\": %ld, \"max_abs\": %ld, \"clk_per_mma\": %.1f, "
           "\"mac_per_clk\": %.0f}\n", n, bad, maxabs, cpm, 128.0 * n * 64 / cpm);
  }
  cudaFuncSetAttribute(fp4_mma_strip, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  {
    unsigned long long *dclk;
    cudaMalloc(&dclk, 2 * 148 * 8);
    for (int n : {64, 128})
      for (int mode : {2, 3, 6, 7})
      for (int noise : {0}) {
        fp4_mma_strip<<<sms, 512, 200 * 1024>>>(n, 656, 27 * 300, noise, dclk, mode);
        unsigned long long ck[148];
        cudaError_t e = cudaMemcpy(ck, dclk, sms * 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; }
        printf("{\"bench\": \"mxf4_strip\", \"n\": %d, \"mode\": %d, \"smem_store_noise\": %d, \"clk_per_mma\": %.1f}\n", n, mode, noise,
               double(ck[0]) / (27 * 300));
      }
    // MMA issue under ALU-bound co-resident warps (noise 6)
    for (int n : {64, 128}) {
      fp4_mma_strip<<<sms, 512, 200 * 1024>>>(n, 656, 27 * 300, 6, dclk, 2);
      unsigned long long ck[148];
      cudaMemcpy(ck, dclk, sms * 8, cudaMemcpyDeviceToHost);
      printf("{\"bench\": \"mxf4_strip_alu_noise\", \"n\": %d, \"clk_per_mma\": %.1f}\n", n, double(ck[0]) / (27 * 300));
    }
    // TMEM load latency (epilogue-sized x64 load + wait) under a streaming MMA queue vs idle
    for (int n : {64, 128})
      for (int noise : {4, 5}) {
        fp4_mma_strip<<<sms, 512, 200 * 1024>>>(n, 656, noise == 4 ? 27 * 300 : 0, noise, dclk, 2);
        unsigned long long ck[2 * 148];
        cudaError_t e = cudaMemcpy(ck, dclk, 2 * sms * 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; }
        printf("{\"bench\": \"tmem_ld_x64_latency\", \"n\": %d, \"mma_streaming\": %d, \"clk_per_ld\": %llu}\n", n,
               int(noise == 4), ck[sms] & ~(1ull << 63));
      }
    cudaFree(dclk);
  }
  // block-scale layout: which byte of the A scale word scales which 32-wide K block
  {
    const int n = 64;
    uint8_t *da, *db;
    float *dout;
    unsigned long long *dclk;
    cudaMalloc(&da, 128 * 32);
    cudaMalloc(&db, n * 32);
    cudaMalloc(&dout, 128 * n * 4);
    cudaMalloc(&dclk, 148 * 8);
    std::vector<uint8_t> bp(n * 32, 0x22);  // B: every element 1.0
    cudaMemcpy(db, bp.data(), bp.size(), cudaMemcpyHostToDevice);
    for (int kb = 0; kb < 2; ++kb) {
      std::vector<uint8_t> ap(128 * 32, 0);
      for (int r = 0; r < 128; ++r)
        for (int byte = 16 * kb; byte < 16 * kb + 16; ++byte) ap[r * 32 + byte] = 0x22;  // K block kb = 1.0
      cudaMemcpy(da, ap.data(), ap.size(), cudaMemcpyHostToDevice);
      for (uint32_t sv : {0x7F7F7F87u, 0x7F7F877Fu, 0x7F877F7Fu, 0x877F7F7Fu}) {
        fp4_mma<<<1, 128, 32 * 1024>>>(da, db, n, 1, 0, dout, dclk, 4, sv);
        std::vector<float> o(128 * n);
        cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
        printf("{\"probe\": \"sf_layout\", \"a_ones_in_kblock\": %d, \"sfa_word\": \"0x%08X\", \"d00\": %g, \"d_127_63\": %g}\n",
               kb, sv, o[0], o[127 * n + 63]);
      }
    }
    cudaFree(da); cudaFree(db); cudaFree(dout); cudaFree(dclk);
  }
  // data dependence of the MMA rate: operand nibble patterns, all SMs busy
  for (int n : {64, 128}) {
    for (int pat = 0; pat < 4; ++pat) {
      std::vector<uint8_t> ap(128 * 32), bp(n * 32);
      auto nib = [&](int which) -> uint8_t {
        switch (pat) {
          case 0: return 0;                                      // zeros
          case 1: return which ? enc((rand() % 3) - 1) : (rand() & 1 ? 0x2 : 0x0);  // a' in {0,1}, w in {-1,0,1}
          case 2: return 0x2;                                    // all ones
          default: return uint8_t(rand() & 0xF);                 // every e2m1 code
        }
      };
      for (auto &x : ap) x = uint8_t(nib(0) | (nib(0) << 4));
      for (auto &x : bp) x = uint8_t(nib(1) | (nib(1) << 4));
      uint8_t *da, *db;
      float *dout;
      unsigned long long *dclk;
      cudaMalloc(&da, ap.size());
      cudaMalloc(&db, bp.size());
      cudaMalloc(&dout, 128 * n * 4);
      cudaMalloc(&dclk, 148 * 8);
      cudaMemcpy(da, ap.data(), ap.size(), cudaMemcpyHostToDevice);
      cudaMemcpy(db, bp.data(), bp.size(), cudaMemcpyHostToDevice);
      fp4_mma<<<sms, 128, 32 * 1024>>>(da, db, n, 8192, 1, dout, dclk, 32, 0u);
      unsigned long long ck[148];
      cudaMemcpy(ck, dclk, sms * 8, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < sms; ++i) mx = std::max(mx, double(ck[i]));
      printf("{\"bench\": \"mxf4_data\", \"n\": %d, \"pattern\": %d, \"clk_per_mma_cta0\": %.1f, \"clk_per_mma_max\": %.1f}\n",
             n, pat, double(ck[0]) / 8192, mx / 8192);
      cudaFree(da); cudaFree(db); cudaFree(dout); cudaFree(dclk);
    }
  }
  return 0;
}
