/* CPU XOR/popcount row product — TEST INFRASTRUCTURE / CPU BASELINE ONLY.
 *
 * Restates the reference's one native loop, bitunet.kernels
 * _xor_popcount_jit_impl (pkg/src/bitunet/kernels.py:82-91): a Numba @njit
 * triple loop emitting llvm.ctpop(i64), with rows of A split over a thread
 * pool (kernels.py:138-146). Here the same loop is plain C with
 * __builtin_popcountll and the row split is an OpenMP static schedule.
 *
 *   out[m, n] = sum_w popcount(a[m, w] ^ b[n, w])
 *
 * Built by oracle/build.py for the host it runs on (-march=native), never
 * linked into the product.
 */
#include <stdint.h>

void oracle_xor_popcount_rows(const uint64_t *a, const uint64_t *b, int32_t *out,
                              int64_t m_rows, int64_t n_rows, int64_t n_words,
                              int threads) {
  if (threads < 1) threads = 1;
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int64_t m = 0; m < m_rows; ++m) {
    const uint64_t *ar = a + m * n_words;
    int32_t *orow = out + m * n_rows;
    for (int64_t n = 0; n < n_rows; ++n) {
      const uint64_t *br = b + n * n_words;
      uint64_t acc = 0;
      for (int64_t w = 0; w < n_words; ++w) acc += (uint64_t)__builtin_popcountll(ar[w] ^ br[w]);
      orow[n] = (int32_t)acc;
    }
  }
}
