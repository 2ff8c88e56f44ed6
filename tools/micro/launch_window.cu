// Microbenchmark: event-timed duration of a short kernel vs the globaltimer span of its CTAs
// (first entry -> last exit), for several dynamic shared-memory sizes and predecessors.  Shows
// how much of a launch lies outside the CTAs (launch latency, shared-memory carve-out changes,
// completion).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 launch_window.cu -o lw && ./lw
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long g_first, g_last;
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void k_work(int spin, float* out) {
  extern __shared__ float sm[];
  if (threadIdx.x == 0) atomicMin(&g_first, gt());
  long long t0 = clock64();
  float x = threadIdx.x;
  while (clock64() - t0 < spin) x = x * 1.0000001f + 1e-7f;
  sm[threadIdx.x] = x;
  __syncwarp();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sm[threadIdx.x ^ 1];
  if (threadIdx.x == 0) atomicMax(&g_last, gt());
}
__global__ void k_nosmem(float* out) { out[blockIdx.x * blockDim.x + threadIdx.x] += 1.0f; }

int main() {
  float* out;
  if (cudaError_t err = cudaMalloc(&out, 1 << 26)) { printf("malloc %s\n", cudaGetErrorString(err)); return 1; }
  cudaFuncSetAttribute(k_work, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int smems[] = {256, 4096, 29 * 1024, 100 * 1024, 200 * 1024};
  for (int pred = 0; pred < 2; ++pred) {
    for (int si = 0; si < 5; ++si) {
      for (int spin : {0, 100000}) {
        float ev_sum = 0, span_sum = 0;
        const int reps = 20;
        for (int r = 0; r < reps + 3; ++r) {
          unsigned long long big = ~0ull, zero = 0;
          cudaMemcpyToSymbol(g_first, &big, 8);
          cudaMemcpyToSymbol(g_last, &zero, 8);
          if (pred) k_nosmem<<<1024, 256>>>(out);
          cudaEventRecord(e0);
          const int blocks = smems[si] >= 100 * 1024 ? 148 : 1024;
          k_work<<<blocks, 32, smems[si]>>>(spin, out);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          if (cudaError_t err = cudaGetLastError()) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          unsigned long long f, l;
          cudaMemcpyFromSymbol(&f, g_first, 8);
          cudaMemcpyFromSymbol(&l, g_last, 8);
          if (r >= 3) { ev_sum += ms * 1e3f; span_sum += (l - f) / 1e3f; }
        }
        printf("pred=%s smem=%6d B spin=%6d cyc: event %7.2f us, CTA span %7.2f us, outside %6.2f us\n",
               pred ? "nosmem-kernel" : "none         ", smems[si], spin, ev_sum / reps, span_sum / reps,
               (ev_sum - span_sum) / reps);
      }
    }
  }
  return 0;
}
