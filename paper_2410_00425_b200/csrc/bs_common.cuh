// Shared device helpers for the batchsim-b200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include "../../include/batchsim_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "batchsim-b200 kernels are written for sm_100a (Blackwell) only"
#endif

#define BS_SMS 148  // B200: 2 dies x 74 SMs

namespace bs {

// Grid for a grid-stride elementwise launch: a whole number of waves over the 148 SMs,
// never more CTAs than there is work for.
static inline int grid_for(int64_t n, int threads, int ctas_per_sm = 8) {
  int64_t need = (n + threads - 1) / threads;
  int64_t cap = (int64_t)BS_SMS * ctas_per_sm;
  if (need < 1) need = 1;
  return (int)(need < cap ? need : cap);
}

static inline int launch_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BS_OK : BS_ERR_CUDA;
}

// Per-device launcher state.  cudaFuncSetAttribute is per device, so the dynamic shared
// memory opt-in a launcher has raised is remembered per (kernel slot, device); every access
// is under one mutex so concurrent host threads (one per GPU) can launch safely.
constexpr int kMaxDevices = 64;
struct LaunchCache {
  std::mutex mu;
  size_t optin[16][kMaxDevices] = {};
};
static inline LaunchCache& launch_cache() {
  static LaunchCache c;
  return c;
}
static inline int current_device() {
  int d = 0;
  return cudaGetDevice(&d) == cudaSuccess && d >= 0 && d < kMaxDevices ? d : -1;
}
// Ensure `bytes` of dynamic shared memory are opted in on the current device for the kernel
// group `slot` (set(bytes) applies the attribute to every kernel of the group).
template <class Set>
static inline bool ensure_smem_optin(int slot, size_t bytes, Set&& set) {
  const int d = current_device();
  if (d < 0) return false;
  LaunchCache& c = launch_cache();
  std::lock_guard<std::mutex> g(c.mu);
  if (bytes <= c.optin[slot][d]) return true;
  if (!set(bytes)) return false;
  c.optin[slot][d] = bytes;
  return true;
}
static inline int sm_count() {
  const int d = current_device();
  int n = 0;
  if (d < 0 || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) != cudaSuccess) return 0;
  return n;
}

// Quaternion helpers in the reference's exact operation order
// (pose.py:31-69). The translation units that include these for parity are compiled
// with -fmad=false so every + and * rounds separately, as numpy does.
template <typename R>
struct Q4 { R w, x, y, z; };
template <typename R>
struct V3 { R x, y, z; };

template <typename R>
__device__ __forceinline__ R sign_like_numpy(R v) {
  // np.sign: +1, -1, signed zero passes through, NaN stays NaN.
  if (v > R(0)) return R(1);
  if (v < R(0)) return R(-1);
  return v;  // +-0 or NaN
}

template <typename R>
__device__ __forceinline__ R sqrt_rn(R v);
template <>
__device__ __forceinline__ double sqrt_rn<double>(double v) { return __dsqrt_rn(v); }
template <>
__device__ __forceinline__ float sqrt_rn<float>(float v) { return __fsqrt_rn(v); }

// pose.py:31-40 -- q / ||q|| with ((q0^2+q1^2)+q2^2)+q3^2, then the cascaded sign rule.
template <typename R>
__device__ __forceinline__ Q4<R> quat_normalize(Q4<R> q) {
  R ss = q.w * q.w;
  ss = ss + q.x * q.x;
  ss = ss + q.y * q.y;
  ss = ss + q.z * q.z;
  R n = sqrt_rn(ss);
  Q4<R> r{q.w / n, q.x / n, q.y / n, q.z / n};
  R s = R(0);
  if (s == R(0)) s = sign_like_numpy(r.w);
  if (s == R(0)) s = sign_like_numpy(r.x);
  if (s == R(0)) s = sign_like_numpy(r.y);
  if (s == R(0)) s = sign_like_numpy(r.z);
  if (s == R(0)) s = R(1);
  return Q4<R>{r.w * s, r.x * s, r.y * s, r.z * s};
}

// pose.py:43-55 Hamilton product, left-to-right sums.
template <typename R>
__device__ __forceinline__ Q4<R> quat_mul(const Q4<R>& a, const Q4<R>& b) {
  Q4<R> o;
  o.w = ((a.w * b.w - a.x * b.x) - a.y * b.y) - a.z * b.z;
  o.x = ((a.w * b.x + a.x * b.w) + a.y * b.z) - a.z * b.y;
  o.y = ((a.w * b.y - a.x * b.z) + a.y * b.w) + a.z * b.x;
  o.z = ((a.w * b.z + a.x * b.y) - a.y * b.x) + a.z * b.w;
  return o;
}

template <typename R>
__device__ __forceinline__ V3<R> cross3(const V3<R>& a, const V3<R>& b) {
  return V3<R>{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// pose.py:64-69: t = 2 (qv x v); v' = (v + w t) + qv x t.
template <typename R>
__device__ __forceinline__ V3<R> quat_rotate(const Q4<R>& q, const V3<R>& v) {
  V3<R> qv{q.x, q.y, q.z};
  V3<R> c = cross3(qv, v);
  V3<R> t{R(2) * c.x, R(2) * c.y, R(2) * c.z};
  V3<R> c2 = cross3(qv, t);
  return V3<R>{(v.x + q.w * t.x) + c2.x, (v.y + q.w * t.y) + c2.y, (v.z + q.w * t.z) + c2.z};
}

// pose.py:72-88 rotation matrix, row-major m[3][3].
template <typename R>
__device__ __forceinline__ void quat_to_matrix(const Q4<R>& q, R m[9]) {
  R xx = q.x * q.x, yy = q.y * q.y, zz = q.z * q.z;
  R xy = q.x * q.y, xz = q.x * q.z, yz = q.y * q.z;
  R wx = q.w * q.x, wy = q.w * q.y, wz = q.w * q.z;
  m[0] = R(1) - R(2) * (yy + zz);
  m[1] = R(2) * (xy - wz);
  m[2] = R(2) * (xz + wy);
  m[3] = R(2) * (xy + wz);
  m[4] = R(1) - R(2) * (xx + zz);
  m[5] = R(2) * (yz - wx);
  m[6] = R(2) * (xz - wy);
  m[7] = R(2) * (yz + wx);
  m[8] = R(1) - R(2) * (xx + yy);
}

template <typename R>
__device__ __forceinline__ Q4<R> load_q(const R* q, int64_t i) {
  return Q4<R>{q[4 * i + 0], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3]};
}
template <typename R>
__device__ __forceinline__ V3<R> load_v(const R* p, int64_t i) {
  return V3<R>{p[3 * i + 0], p[3 * i + 1], p[3 * i + 2]};
}
template <typename R>
__device__ __forceinline__ void store_q(R* q, int64_t i, const Q4<R>& v) {
  q[4 * i + 0] = v.w; q[4 * i + 1] = v.x; q[4 * i + 2] = v.y; q[4 * i + 3] = v.z;
}
template <typename R>
__device__ __forceinline__ void store_v(R* p, int64_t i, const V3<R>& v) {
  p[3 * i + 0] = v.x; p[3 * i + 1] = v.y; p[3 * i + 2] = v.z;
}

}  // namespace bs
