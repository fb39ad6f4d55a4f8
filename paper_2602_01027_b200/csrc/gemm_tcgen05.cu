// gemm_tcgen05.cu -- K2 prefill GEMM (placeholder until the tcgen05 kernel lands).
#include "sfmp_internal.h"
namespace sfmpk {
bool gemm_supported(const DevModel&) { return false; }
size_t gemm_workspace_bytes(const DevModel&, int64_t) { return 0; }
cudaError_t launch_gemm(const DevModel&, const void*, sfmp_dtype, int64_t, float*, void*, cudaStream_t) {
    return cudaErrorNotSupported;
}
}  // namespace sfmpk
