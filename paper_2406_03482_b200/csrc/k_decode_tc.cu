// Tensor-core fused decode -- placeholder until implemented.
#include "common.cuh"
#include "kernels.h"
namespace qjl {
bool decode_tc_supported(const qjl_key_cache_t&, const qjl_value_cache_t&, int) { return false; }
size_t decode_tc_workspace(const qjl_key_cache_t&, const qjl_value_cache_t&, int64_t, int) { return 0; }
int launch_decode_tc(const qjl_key_cache_t&, const qjl_value_cache_t&, int64_t, const void*, int, int,
                     const qjl_sketch_t&, float, float*, float*, void*, size_t, cudaStream_t) {
  return QJL_ERR_UNSUPPORTED;
}
}  // namespace qjl
