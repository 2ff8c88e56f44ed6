// Library-level C-ABI entry points (version, device binding).
#include "bs_common.cuh"

extern "C" {

int bs_abi_version(void) { return BS_ABI_VERSION; }

int bs_init(int device) {
  // The library links the CUDA runtime statically; bind this runtime instance to the
  // device the host framework selected so launches land in that device's primary context.
  if (cudaSetDevice(device) != cudaSuccess) return BS_ERR_CUDA;
  cudaFree(nullptr);
  return cudaGetLastError() == cudaSuccess ? BS_OK : BS_ERR_CUDA;
}

}  // extern "C"
