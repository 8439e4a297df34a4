// knn_tc.cu — tcgen05 candidate engine (placeholder until the kernel lands).
#include "tb_common.cuh"
#include "knn_internal.h"
namespace tb {
int tc_lists_per_slice() { return 1; }
int launch_knn_tc(int, int, const __nv_bfloat16*, const __nv_bfloat16*,
                  const __nv_bfloat16*, const __nv_bfloat16*, const float*,
                  int64_t, int64_t, int64_t, int64_t, int64_t, int, int,
                  float*, int*, cudaStream_t) {
  return fail(TB_ERR_UNSUPPORTED, "tcgen05 engine not built yet");
}
}  // namespace tb
