// Instantiates the flash all-reduce for input dtype float (split from fc_api.cu
// so the three dtype families compile in parallel).
#include "fc_run.cuh"

namespace fc {
template fc_status run_typed<float, float>(fc_comm*, const void* const*, void* const*, int64_t, const fc_flash_cfg*,
                                        cudaStream_t*, int);
template fc_status identity_typed<float, float>(const void*, void*, int64_t, int, cudaStream_t);
template fc_status identity_typed<float, __half>(const void*, void*, int64_t, int, cudaStream_t);
template fc_status identity_typed<float, __nv_bfloat16>(const void*, void*, int64_t, int, cudaStream_t);
}  // namespace fc
