// tc.cu -- placeholder until the tcgen05 path lands.
#include "paths.cuh"
namespace tl {
bool tc_available() { return false; }
size_t tc_workspace_bytes(int64_t, int64_t, int64_t) { return 0; }
tl_status tc_matmul(tl_wtype, int64_t, int64_t, int64_t, int32_t, const __half*, int64_t, const uint8_t*,
                    const __half*, const __half*, __half*, int64_t, float*, int*, int, cudaStream_t) {
  return TL_EUNSUPPORTED;
}
}  // namespace tl
