// tcgen05 + TMA key quantizer (bf16/fp16 keys) -- placeholder until implemented.
#include "common.cuh"
#include "kernels.h"
namespace qjl {
int launch_quantize_keys_tc(const void*, int, int64_t, int64_t, const qjl_sketch_t&,
                            const int32_t*, int, const qjl_key_cache_t&, int64_t, cudaStream_t) {
  return QJL_ERR_UNSUPPORTED;
}
}  // namespace qjl
