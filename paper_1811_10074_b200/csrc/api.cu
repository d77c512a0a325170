// api.cu -- error strings and version of libmzslsum.
#include "common.cuh"

namespace mzs {
static thread_local cudaError_t g_last_cuda = cudaSuccess;
void set_cuda_error(cudaError_t e) { g_last_cuda = e; }
}  // namespace mzs

MZS_API const char* slsum_strerror(int rc) {
  switch (rc) {
    case SLSUM_OK: return "ok";
    case SLSUM_EINVAL: return "invalid argument";
    case SLSUM_EUNSUPPORTED: return "unsupported operator/path/size combination";
    case SLSUM_ECAPACITY: return "output capacity exceeded";
    case SLSUM_ECUDA: return mzs::g_last_cuda == cudaSuccess ? "CUDA error" : cudaGetErrorString(mzs::g_last_cuda);
    case SLSUM_ENOMEM: return "workspace too small or allocation failed";
    default: return "unknown error";
  }
}

MZS_API int slsum_version(void) { return 0x000100; }
