// tcgen05 implicit-GEMM conv (placeholder until the UTCIMMA kernel lands).
#include "common.cuh"
namespace mbu {
int prepare_conv_tc(mbu_conv *cv, const uint64_t *, const uint64_t *, const int32_t *,
                    const int32_t *, int) {
  cv->tc_ok = 0;
  return MBU_OK;
}
int launch_conv_tc(const mbu_conv *, const ActView &, int, int, int32_t *, uint64_t *, int, int,
                   cudaStream_t) {
  return fail(MBU_ERR_UNSUPPORTED, "tcgen05 path not built");
}
}  // namespace mbu
