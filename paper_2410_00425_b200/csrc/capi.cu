// Library-level C-ABI entry points (version, device binding) and the host-side step driver.
#include <string.h>
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

int bs_host_step(const float* src, float* dst, int64_t n, int32_t check, void* graph_exec, void* stream) {
  // One call per Env.step_host: stage the caller's actions into the pinned buffer the captured
  // step graph reads over PCIe, reject the step before anything is launched when an entry is
  // not finite (exponent bits all set: inf / NaN), then replay the graph and wait for it.  The
  // copy and the test are one pass over the actions (the compiler vectorises both).
  if ((n > 0 && (!src || !dst)) || n < 0 || !graph_exec) return BS_ERR_ARGUMENT;
  if (check) {
    unsigned bad = 0;
    const unsigned* s32 = reinterpret_cast<const unsigned*>(src);
    unsigned* d32 = reinterpret_cast<unsigned*>(dst);
    for (int64_t i = 0; i < n; ++i) {
      const unsigned u = s32[i];
      d32[i] = u;
      bad |= (u & 0x7f800000u) == 0x7f800000u;
    }
    if (bad) return BS_ERR_INPUT;
  } else if (n > 0) {
    memcpy(dst, src, (size_t)n * sizeof(float));
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaGraphLaunch(static_cast<cudaGraphExec_t>(graph_exec), st) != cudaSuccess) return BS_ERR_CUDA;
  return cudaStreamSynchronize(st) == cudaSuccess ? BS_OK : BS_ERR_CUDA;
}

}  // extern "C"
