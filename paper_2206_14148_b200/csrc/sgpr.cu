// sgpr.cu — SGPR sufficient statistics and kernel MVM (placeholder).
#include "tb_common.cuh"
using namespace tb;
extern "C" {
int tb_sgpr_plan_create(int64_t, int64_t, int64_t, int32_t, int32_t, int64_t, int64_t, tb_sgpr_plan*) {
  return fail(TB_ERR_UNSUPPORTED, "sgpr not built yet");
}
int tb_sgpr_stats_run(const tb_sgpr_plan*, const void*, const void*, const void*, double,
                      const double*, double*, double*, double*, int32_t, void*, int64_t, void*) {
  return fail(TB_ERR_UNSUPPORTED, "sgpr not built yet");
}
int tb_kernel_mvm(const void*, const void*, const double*, int64_t, int64_t, int64_t, int32_t,
                  int32_t, double, const double*, double*, void*) {
  return fail(TB_ERR_UNSUPPORTED, "kernel mvm not built yet");
}
}
