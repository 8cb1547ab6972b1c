// Instantiates the flash all-reduce for input dtype __nv_bfloat16 (split from fc_api.cu
// so the three dtype families compile in parallel).
#include "fc_run.cuh"

namespace fc {
template fc_status run_typed<__nv_bfloat16, float>(fc_comm*, const void* const*, void* const*, int64_t, const fc_flash_cfg*,
                                        cudaStream_t*, int);
template fc_status run_typed<__nv_bfloat16, __nv_bfloat16>(fc_comm*, const void* const*, void* const*, int64_t,
                                                const fc_flash_cfg*, cudaStream_t*, int);
template fc_status identity_typed<__nv_bfloat16, float>(const void*, void*, int64_t, int, cudaStream_t);
template fc_status identity_typed<__nv_bfloat16, __half>(const void*, void*, int64_t, int, cudaStream_t);
template fc_status identity_typed<__nv_bfloat16, __nv_bfloat16>(const void*, void*, int64_t, int, cudaStream_t);
}  // namespace fc
