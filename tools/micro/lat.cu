// Microbenchmark: dependent-chain latency and issue cost of fp64 / shuffle / shared-memory ops
// on the B200 (developer tool; informs the k_step design).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[64];
  const int t = threadIdx.x;
  sm[t & 63] = a + t;
  __syncwarp();
  double x = a + t, y = b;
  long long t0, t1;
  // 1: DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, y, 1e-9); x = fma(x, y, 1e-9); x = fma(x, y, 1e-9); x = fma(x, y, 1e-9); }
  t1 = clock64();
  if (t == 0) cyc[0] = (t1 - t0);
  // 2: DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x + y; x = x + y; x = x + y; x = x + y; }
  t1 = clock64();
  if (t == 0) cyc[1] = (t1 - t0);
  // 3: shuffle (double) chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x += __shfl_xor_sync(0xffffffffu, x, 1); x += __shfl_xor_sync(0xffffffffu, x, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 1); x += __shfl_xor_sync(0xffffffffu, x, 2);
  }
  t1 = clock64();
  if (t == 0) cyc[2] = (t1 - t0);
  // 4: LDS dependent chain (pointer chasing via value)
  int idx = t & 63;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double v = sm[idx]; idx = ((int)v) & 63; v = sm[idx]; idx = ((int)v) & 63;
    v = sm[idx]; idx = ((int)v) & 63; v = sm[idx]; idx = ((int)v) & 63;
  }
  t1 = clock64();
  if (t == 0) cyc[3] = (t1 - t0);
  // 5: independent DFMA throughput (8 chains)
  double z[8];
  for (int k = 0; k < 8; ++k) z[k] = x + k;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) z[k] = fma(z[k], y, 1e-9);
  }
  t1 = clock64();
  if (t == 0) cyc[4] = (t1 - t0);
  // 6: fp64 max via ternary chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x > y ? x : y; x = x - 1e-9; x = x > y ? x : y; x = x - 1e-9; }
  t1 = clock64();
  if (t == 0) cyc[5] = (t1 - t0);
  double s = x + idx;
  for (int k = 0; k < 8; ++k) s += z[k];
  out[blockIdx.x * blockDim.x + t] = s;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 20); cudaMallocManaged(&cyc, 64 * sizeof(long long));
  const int n = 1000;
  const char* names[] = {"DFMA dep (per op)", "DADD dep (per op)", "SHFL.f64 + DADD dep (per pair)",
                         "LDS.64 + F2I dep (per load)", "DFMA 8 indep chains (per instr)", "ternary max + DADD (per pair)"};
  const double per[] = {4.0 * n, 4.0 * n, 4.0 * n, 4.0 * n, 8.0 * n, 2.0 * n};
  for (int warps : {1, 2, 4, 8}) {
    k_lat<<<1, 32 * warps>>>(out, cyc, 1.0000001, 0.9999999, n);
    cudaDeviceSynchronize();
    printf("warps/CTA=%d\n", warps);
    for (int i = 0; i < 6; ++i) printf("  %-36s %7.2f cycles\n", names[i], cyc[i] / per[i]);
  }
  return 0;
}
