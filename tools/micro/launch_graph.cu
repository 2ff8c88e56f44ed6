// Microbenchmark: event-timed duration of a short kernel launched (a) directly, (b) as a
// one-node CUDA graph replayed between the events, (c) with a 1 KB by-value parameter struct
// (like k_step's tables/state/params), each behind a 256 MiB memset (the bench's L2 flush).
// Shows how much of the event interval around one launch is launch processing.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 launch_graph.cu -o lg && ./lg
#include <cstdio>
#include <cuda_runtime.h>

struct Big { double v[128]; };  // 1 KB by value
__device__ unsigned long long g_first, g_last;
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void k_spin(int spin, float* out) {
  if (threadIdx.x == 0) atomicMin(&g_first, gt());
  long long t0 = clock64();
  float x = threadIdx.x;
  while (clock64() - t0 < spin) x = x * 1.0000001f + 1e-7f;
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0) atomicMax(&g_last, gt());
}
__global__ void k_spin_big(const __grid_constant__ Big b, int spin, float* out) {
  if (threadIdx.x == 0) atomicMin(&g_first, gt());
  long long t0 = clock64();
  float x = threadIdx.x + (float)b.v[threadIdx.x & 127];
  while (clock64() - t0 < spin) x = x * 1.0000001f + 1e-7f;
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0) atomicMax(&g_last, gt());
}

int main() {
  float* out;
  char* flush;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&flush, 256 << 20);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  Big big = {};
  const int spin = 100000;
  // graph of the one kernel
  cudaGraph_t g;
  cudaGraphExec_t ge, geb;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  k_spin<<<1024, 32, 0, st>>>(spin, out);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  k_spin_big<<<1024, 32, 0, st>>>(big, spin, out);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&geb, g, 0);
  const char* names[] = {"direct small params", "direct 1 KB params", "graph small params", "graph 1 KB params"};
  for (int mode = 0; mode < 4; ++mode) {
    float ev = 0, span = 0;
    const int reps = 50;
    for (int r = 0; r < reps + 5; ++r) {
      unsigned long long bigv = ~0ull, zero = 0;
      cudaMemcpyToSymbolAsync(g_first, &bigv, 8, 0, cudaMemcpyHostToDevice, st);
      cudaMemcpyToSymbolAsync(g_last, &zero, 8, 0, cudaMemcpyHostToDevice, st);
      cudaMemsetAsync(flush, r & 255, 256 << 20, st);
      cudaEventRecord(e0, st);
      if (mode == 0) k_spin<<<1024, 32, 0, st>>>(spin, out);
      else if (mode == 1) k_spin_big<<<1024, 32, 0, st>>>(big, spin, out);
      else if (mode == 2) cudaGraphLaunch(ge, st);
      else cudaGraphLaunch(geb, st);
      cudaEventRecord(e1, st);
      cudaStreamSynchronize(st);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long f, l;
      cudaMemcpyFromSymbol(&f, g_first, 8);
      cudaMemcpyFromSymbol(&l, g_last, 8);
      if (r >= 5) { ev += ms * 1e3f; span += (l - f) / 1e3f; }
    }
    printf("%-22s: event %7.2f us, CTA span %7.2f us, outside %6.2f us\n", names[mode], ev / reps, span / reps,
           (ev - span) / reps);
  }
  if (cudaError_t err = cudaGetLastError()) printf("error %s\n", cudaGetErrorString(err));
  return 0;
}
