// Batched SE(3) kernels behind PoseBatch (reference pose.py).  Compiled with -fmad=false:
// the fp64 path reproduces numpy's separately-rounded + and * bit for bit for
// normalize / compose / inverse / to_matrix (the parity tests assert array_equal).
//
// Layout: positions (N,3) and quaternions (N,4) SoA-by-field, row-major; one thread per
// pose (or per point for transform_points), grid-stride, grids sized in whole waves over
// the 148 SMs.  Every kernel is HBM-bound: compose moves 56+56 B in, 56 B out per pose.
#include "bs_common.cuh"

namespace bs {

template <typename R>
__global__ void k_quat_normalize(const R* __restrict__ q, int64_t n, R* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    store_q(out, i, quat_normalize(load_q(q, i)));
  }
}

template <typename R>
__global__ void k_pose_compose(const R* __restrict__ pa, const R* __restrict__ qa, int64_t na,
                               const R* __restrict__ pb, const R* __restrict__ qb, int64_t nb,
                               int64_t n, R* __restrict__ po, R* __restrict__ qo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t ia = na == 1 ? 0 : i, ib = nb == 1 ? 0 : i;
    Q4<R> a = load_q(qa, ia), b = load_q(qb, ib);
    V3<R> ta = load_v(pa, ia), tb = load_v(pb, ib);
    Q4<R> q = quat_mul(a, b);
    V3<R> r = quat_rotate(a, tb);
    store_v(po, i, V3<R>{ta.x + r.x, ta.y + r.y, ta.z + r.z});
    store_q(qo, i, quat_normalize(q));
  }
}

template <typename R>
__global__ void k_pose_inverse(const R* __restrict__ p, const R* __restrict__ q, int64_t n,
                               R* __restrict__ po, R* __restrict__ qo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    Q4<R> a = load_q(q, i);
    Q4<R> c{a.w, -a.x, -a.y, -a.z};
    V3<R> r = quat_rotate(c, load_v(p, i));
    store_v(po, i, V3<R>{-r.x, -r.y, -r.z});
    store_q(qo, i, quat_normalize(c));
  }
}

template <typename R>
__global__ void k_pose_transform_points(const R* __restrict__ p, const R* __restrict__ q,
                                        int64_t n, const R* __restrict__ pts, int64_t m,
                                        int64_t k, int64_t nout, R* __restrict__ out) {
  const int64_t total = nout * k;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / k, j = t - i * k;
    int64_t ip = n == 1 ? 0 : i, im = m == 1 ? 0 : i;
    R r[9];
    quat_to_matrix(load_q(q, ip), r);
    V3<R> tr = load_v(p, ip);
    const R* x = pts + (im * k + j) * 3;
    R x0 = x[0], x1 = x[1], x2 = x[2];
    R* o = out + t * 3;
    o[0] = ((r[0] * x0 + r[1] * x1) + r[2] * x2) + tr.x;
    o[1] = ((r[3] * x0 + r[4] * x1) + r[5] * x2) + tr.y;
    o[2] = ((r[6] * x0 + r[7] * x1) + r[8] * x2) + tr.z;
  }
}

__global__ void k_pose_to_matrix(const double* __restrict__ p, const double* __restrict__ q,
                                 int64_t n, double* __restrict__ m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double r[9];
    quat_to_matrix(load_q(q, i), r);
    double* o = m + i * 16;
    o[0] = r[0]; o[1] = r[1]; o[2] = r[2]; o[3] = p[3 * i + 0];
    o[4] = r[3]; o[5] = r[4]; o[6] = r[5]; o[7] = p[3 * i + 1];
    o[8] = r[6]; o[9] = r[7]; o[10] = r[8]; o[11] = p[3 * i + 2];
    o[12] = 0.0; o[13] = 0.0; o[14] = 0.0; o[15] = 1.0;
  }
}

// pose.py:91-122 Shepperd's method; the branch is the first argmax of
// (trace, m00, m11, m22), exactly like np.argmax.  Unnormalized result.
__device__ __forceinline__ Q4<double> shepperd(const double r[3][3]) {
  double tr = (r[0][0] + r[1][1]) + r[2][2];
  int c = 0;
  double best = tr;
  if (r[0][0] > best) { best = r[0][0]; c = 1; }
  if (r[1][1] > best) { best = r[1][1]; c = 2; }
  if (r[2][2] > best) { best = r[2][2]; c = 3; }
  Q4<double> q;
  if (c == 0) {
    double s = __dsqrt_rn(((1.0 + r[0][0]) + r[1][1]) + r[2][2]) * 2.0;
    q = {0.25 * s, (r[2][1] - r[1][2]) / s, (r[0][2] - r[2][0]) / s, (r[1][0] - r[0][1]) / s};
  } else if (c == 1) {
    double s = __dsqrt_rn(((1.0 + r[0][0]) - r[1][1]) - r[2][2]) * 2.0;
    q = {(r[2][1] - r[1][2]) / s, 0.25 * s, (r[0][1] + r[1][0]) / s, (r[0][2] + r[2][0]) / s};
  } else if (c == 2) {
    double s = __dsqrt_rn(((1.0 - r[0][0]) + r[1][1]) - r[2][2]) * 2.0;
    q = {(r[0][2] - r[2][0]) / s, (r[0][1] + r[1][0]) / s, 0.25 * s, (r[1][2] + r[2][1]) / s};
  } else {
    double s = __dsqrt_rn(((1.0 - r[0][0]) - r[1][1]) + r[2][2]) * 2.0;
    q = {(r[1][0] - r[0][1]) / s, (r[0][2] + r[2][0]) / s, (r[1][2] + r[2][1]) / s, 0.25 * s};
  }
  return q;
}

// pose.py:91-122 matrix_to_quat: (n, 3, 3) rotation blocks -> normalized quaternions (one
// normalization pass, as the reference function itself does).
__global__ void k_matrix_to_quat(const double* __restrict__ m, int64_t n, double* __restrict__ qo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* a = m + i * 9;
    const double r[3][3] = {{a[0], a[1], a[2]}, {a[3], a[4], a[5]}, {a[6], a[7], a[8]}};
    store_q(qo, i, quat_normalize(shepperd(r)));
  }
}

// pose.py:43-61 quat_mul / quat_conjugate with singleton broadcasting (na == nb, or 1).
template <typename R>
__global__ void k_quat_mul(const R* __restrict__ a, int64_t na, const R* __restrict__ b, int64_t nb, int64_t n,
                           R* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    store_q(out, i, quat_mul(load_q(a, na == 1 ? 0 : i), load_q(b, nb == 1 ? 0 : i)));
}

template <typename R>
__global__ void k_quat_conjugate(const R* __restrict__ q, int64_t n, R* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Q4<R> a = load_q(q, i);
    store_q(out, i, Q4<R>{a.w, -a.x, -a.y, -a.z});
  }
}

// pose.py:64-69 quat_rotate with singleton broadcasting between quaternions and vectors.
template <typename R>
__global__ void k_quat_rotate(const R* __restrict__ q, int64_t nq, const R* __restrict__ v, int64_t nv, int64_t n,
                              R* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    store_v(out, i, quat_rotate(load_q(q, nq == 1 ? 0 : i), load_v(v, nv == 1 ? 0 : i)));
}

// pose.py:72-88 quat_to_matrix: (n, 4) -> (n, 3, 3) row-major.
template <typename R>
__global__ void k_quat_to_matrix(const R* __restrict__ q, int64_t n, R* __restrict__ m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    R r[9];
    quat_to_matrix(load_q(q, i), r);
#pragma unroll
    for (int k = 0; k < 9; ++k) m[9 * i + k] = r[k];
  }
}

// pose.py:125-164 TransformMatrixBatch on 4x4 row-major matrices.  One thread per output
// element (compose) or per matrix (inverse); sums run k = 0..3 left to right.
__global__ void k_tmat_compose(const double* __restrict__ a, int64_t na, const double* __restrict__ b, int64_t nb,
                               int64_t n, double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * 16;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t >> 4;
    const int r = (int)(t >> 2) & 3, c = (int)t & 3;
    const double* A = a + (na == 1 ? 0 : i) * 16 + 4 * r;
    const double* B = b + (nb == 1 ? 0 : i) * 16 + c;
    out[t] = ((A[0] * B[0] + A[1] * B[4]) + A[2] * B[8]) + A[3] * B[12];
  }
}

__global__ void k_tmat_inverse(const double* __restrict__ m, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* a = m + 16 * i;
    double* o = out + 16 * i;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      // R^T row r = column r of R; translation -(R^T t)_r
#pragma unroll
      for (int c = 0; c < 3; ++c) o[4 * r + c] = a[4 * c + r];
      o[4 * r + 3] = -((a[r] * a[3] + a[4 + r] * a[7]) + a[8 + r] * a[11]);
    }
    o[12] = 0.0; o[13] = 0.0; o[14] = 0.0; o[15] = 1.0;
  }
}

__global__ void k_tmat_transform_points(const double* __restrict__ m, int64_t n, const double* __restrict__ pts,
                                        int64_t np_, int64_t k, int64_t nout, double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nout * k;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / k, j = t - i * k;
    const double* a = m + 16 * (n == 1 ? 0 : i);
    const double* x = pts + ((np_ == 1 ? 0 : i) * k + j) * 3;
    double* o = out + 3 * t;
#pragma unroll
    for (int r = 0; r < 3; ++r) o[r] = ((a[4 * r] * x[0] + a[4 * r + 1] * x[1]) + a[4 * r + 2] * x[2]) + a[4 * r + 3];
  }
}

__global__ void k_pose_from_matrix(const double* __restrict__ m, int64_t n,
                                   double* __restrict__ po, double* __restrict__ qo,
                                   unsigned long long* __restrict__ err_bits) {
  double local_err = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* a = m + i * 16;
    double r[3][3] = {{a[0], a[1], a[2]}, {a[4], a[5], a[6]}, {a[8], a[9], a[10]}};
    for (int u = 0; u < 3; ++u)
      for (int v = 0; v < 3; ++v) {
        double d = (r[u][0] * r[v][0] + r[u][1] * r[v][1]) + r[u][2] * r[v][2];
        d = d - (u == v ? 1.0 : 0.0);
        d = fabs(d);
        local_err = d > local_err ? d : local_err;
      }
    const Q4<double> q = shepperd(r);
    // matrix_to_quat normalizes, then the PoseBatch constructor normalizes again
    // (pose.py:122 and pose.py:194): two passes, as in the reference.
    store_q(qo, i, quat_normalize(quat_normalize(q)));
    po[3 * i + 0] = a[3]; po[3 * i + 1] = a[7]; po[3 * i + 2] = a[11];
  }
  // NaN entries drop out of the max, matching the reference: its `err > 1e-6` test
  // (pose.py:229-231) is false for NaN, so non-finite input is not rejected there either.
  unsigned long long bits = __double_as_longlong(local_err);
  for (int off = 16; off > 0; off >>= 1) {
    unsigned long long o = __shfl_xor_sync(0xffffffffu, bits, off);
    bits = o > bits ? o : bits;
  }
  if ((threadIdx.x & 31) == 0 && bits) atomicMax(err_bits, bits);
}

}  // namespace bs

using namespace bs;

#define BS_CHECK_PTR(x) \
  if ((x) == nullptr) return BS_ERR_ARGUMENT
#define BS_STREAM(s) (static_cast<cudaStream_t>(s))

namespace {
template <typename R>
int quat_normalize_impl(const R* q, int64_t n, R* out, void* stream) {
  if (n < 0) return BS_ERR_ARGUMENT;
  if (n == 0) return BS_OK;
  BS_CHECK_PTR(q); BS_CHECK_PTR(out);
  k_quat_normalize<R><<<grid_for(n, 256), 256, 0, BS_STREAM(stream)>>>(q, n, out);
  return launch_status();
}

template <typename R>
int compose_impl(const R* pa, const R* qa, int64_t na, const R* pb, const R* qb, int64_t nb,
                 R* po, R* qo, void* stream) {
  if (na < 0 || nb < 0) return BS_ERR_ARGUMENT;
  if (na != nb && na != 1 && nb != 1) return BS_ERR_DIMENSION;
  // pose.py:167-174: equal sizes, or a singleton side broadcast to the other (also to 0)
  const int64_t n = na == nb ? na : (na == 1 ? nb : na);
  if (n == 0) return BS_OK;
  BS_CHECK_PTR(pa); BS_CHECK_PTR(qa); BS_CHECK_PTR(pb); BS_CHECK_PTR(qb);
  BS_CHECK_PTR(po); BS_CHECK_PTR(qo);
  k_pose_compose<R><<<grid_for(n, 256), 256, 0, BS_STREAM(stream)>>>(pa, qa, na, pb, qb, nb, n,
                                                                        po, qo);
  return launch_status();
}

template <typename R>
int inverse_impl(const R* p, const R* q, int64_t n, R* po, R* qo, void* stream) {
  if (n < 0) return BS_ERR_ARGUMENT;
  if (n == 0) return BS_OK;
  BS_CHECK_PTR(p); BS_CHECK_PTR(q); BS_CHECK_PTR(po); BS_CHECK_PTR(qo);
  k_pose_inverse<R><<<grid_for(n, 256), 256, 0, BS_STREAM(stream)>>>(p, q, n, po, qo);
  return launch_status();
}

template <typename R>
int transform_points_impl(const R* p, const R* q, int64_t n, const R* pts, int64_t m, int64_t k,
                          R* out, void* stream) {
  if (n < 0 || m < 0 || k < 0) return BS_ERR_ARGUMENT;
  if (n != m && n != 1 && m != 1) return BS_ERR_DIMENSION;
  const int64_t nout = n == m ? n : (n == 1 ? m : n);  // singleton broadcast, also to 0
  if (k == 0 || nout == 0) return BS_OK;
  BS_CHECK_PTR(p); BS_CHECK_PTR(q); BS_CHECK_PTR(pts); BS_CHECK_PTR(out);
  k_pose_transform_points<R><<<grid_for(nout * k, 256), 256, 0, BS_STREAM(stream)>>>(
      p, q, n, pts, m, k, nout, out);
  return launch_status();
}
static inline int64_t bcast_n(int64_t na, int64_t nb) { return na == nb ? na : (na == 1 ? nb : na); }
#define BS_BCAST_CHECK(na, nb)                  \
  if ((na) < 0 || (nb) < 0) return BS_ERR_ARGUMENT; \
  if ((na) != (nb) && (na) != 1 && (nb) != 1) return BS_ERR_DIMENSION

template <typename R>
static int quat_mul_impl(const R* a, int64_t na, const R* b, int64_t nb, R* out, void* s) {
  BS_BCAST_CHECK(na, nb);
  const int64_t n = bcast_n(na, nb);
  if (n == 0) return BS_OK;
  BS_CHECK_PTR(a); BS_CHECK_PTR(b); BS_CHECK_PTR(out);
  k_quat_mul<R><<<grid_for(n, 256), 256, 0, BS_STREAM(s)>>>(a, na, b, nb, n, out);
  return launch_status();
}
template <typename R>
static int quat_rotate_impl(const R* q, int64_t nq, const R* v, int64_t nv, R* out, void* s) {
  BS_BCAST_CHECK(nq, nv);
  const int64_t n = bcast_n(nq, nv);
  if (n == 0) return BS_OK;
  BS_CHECK_PTR(q); BS_CHECK_PTR(v); BS_CHECK_PTR(out);
  k_quat_rotate<R><<<grid_for(n, 256), 256, 0, BS_STREAM(s)>>>(q, nq, v, nv, n, out);
  return launch_status();
}

}  // namespace

extern "C" {

int bs_quat_normalize_f64(const double* q, int64_t n, double* out, void* s) {
  return quat_normalize_impl(q, n, out, s);
}
int bs_quat_normalize_f32(const float* q, int64_t n, float* out, void* s) {
  return quat_normalize_impl(q, n, out, s);
}
int bs_pose_compose_f64(const double* pa, const double* qa, int64_t na, const double* pb,
                        const double* qb, int64_t nb, double* po, double* qo, void* s) {
  return compose_impl(pa, qa, na, pb, qb, nb, po, qo, s);
}
int bs_pose_compose_f32(const float* pa, const float* qa, int64_t na, const float* pb,
                        const float* qb, int64_t nb, float* po, float* qo, void* s) {
  return compose_impl(pa, qa, na, pb, qb, nb, po, qo, s);
}
int bs_pose_inverse_f64(const double* p, const double* q, int64_t n, double* po, double* qo,
                        void* s) {
  return inverse_impl(p, q, n, po, qo, s);
}
int bs_pose_inverse_f32(const float* p, const float* q, int64_t n, float* po, float* qo,
                        void* s) {
  return inverse_impl(p, q, n, po, qo, s);
}
int bs_pose_transform_points_f64(const double* p, const double* q, int64_t n, const double* pts,
                                 int64_t m, int64_t k, double* out, void* s) {
  return transform_points_impl(p, q, n, pts, m, k, out, s);
}
int bs_pose_transform_points_f32(const float* p, const float* q, int64_t n, const float* pts,
                                 int64_t m, int64_t k, float* out, void* s) {
  return transform_points_impl(p, q, n, pts, m, k, out, s);
}
int bs_pose_to_matrix_f64(const double* p, const double* q, int64_t n, double* m, void* s) {
  if (n < 0) return BS_ERR_ARGUMENT;
  if (n == 0) return BS_OK;
  BS_CHECK_PTR(p); BS_CHECK_PTR(q); BS_CHECK_PTR(m);
  k_pose_to_matrix<<<grid_for(n, 256), 256, 0, BS_STREAM(s)>>>(p, q, n, m);
  return launch_status();
}
int bs_quat_mul_f64(const double* a, int64_t na, const double* b, int64_t nb, double* out, void* s) {
  return quat_mul_impl(a, na, b, nb, out, s);
}
int bs_quat_mul_f32(const float* a, int64_t na, const float* b, int64_t nb, float* out, void* s) {
  return quat_mul_impl(a, na, b, nb, out, s);
}
int bs_quat_conjugate_f64(const double* q, int64_t n, double* out, void* s) {
  if (n < 0) return BS_ERR_ARGUMENT;
  if (n == 0) return BS_OK;
  BS_CHECK_PTR(q); BS_CHECK_PTR(out);
  k_quat_conjugate<double><<<grid_for(n, 256), 256, 0, BS_STREAM(s)>>>(q, n, out);
  return launch_status();
}
int bs_quat_rotate_f64(const double* q, int64_t nq, const double* v, int64_t nv, double* out, void* s) {
  return quat_rotate_impl(q, nq, v, nv, out, s);
}
int bs_quat_rotate_f32(const float* q, int64_t nq, const float* v, int64_t nv, float* out, void* s) {
  return quat_rotate_impl(q, nq, v, nv, out, s);
}
int bs_quat_to_matrix_f64(const double* q, int64_t n, double* m, void* s) {
  if (n < 0) return BS_ERR_ARGUMENT;
  if (n == 0) return BS_OK;
  BS_CHECK_PTR(q); BS_CHECK_PTR(m);
  k_quat_to_matrix<double><<<grid_for(n, 256), 256, 0, BS_STREAM(s)>>>(q, n, m);
  return launch_status();
}
int bs_matrix_to_quat_f64(const double* m, int64_t n, double* q, void* s) {
  if (n < 0) return BS_ERR_ARGUMENT;
  if (n == 0) return BS_OK;
  BS_CHECK_PTR(m); BS_CHECK_PTR(q);
  k_matrix_to_quat<<<grid_for(n, 256), 256, 0, BS_STREAM(s)>>>(m, n, q);
  return launch_status();
}
int bs_tmat_compose_f64(const double* a, int64_t na, const double* b, int64_t nb, double* out, void* s) {
  BS_BCAST_CHECK(na, nb);
  const int64_t n = bcast_n(na, nb);
  if (n == 0) return BS_OK;
  BS_CHECK_PTR(a); BS_CHECK_PTR(b); BS_CHECK_PTR(out);
  k_tmat_compose<<<grid_for(16 * n, 256), 256, 0, BS_STREAM(s)>>>(a, na, b, nb, n, out);
  return launch_status();
}
int bs_tmat_inverse_f64(const double* m, int64_t n, double* out, void* s) {
  if (n < 0) return BS_ERR_ARGUMENT;
  if (n == 0) return BS_OK;
  BS_CHECK_PTR(m); BS_CHECK_PTR(out);
  k_tmat_inverse<<<grid_for(n, 256), 256, 0, BS_STREAM(s)>>>(m, n, out);
  return launch_status();
}
int bs_tmat_transform_points_f64(const double* m, int64_t n, const double* pts, int64_t np_, int64_t k,
                                 double* out, void* s) {
  BS_BCAST_CHECK(n, np_);
  const int64_t nout = bcast_n(n, np_);
  if (k < 0) return BS_ERR_ARGUMENT;
  if (nout == 0 || k == 0) return BS_OK;
  BS_CHECK_PTR(m); BS_CHECK_PTR(pts); BS_CHECK_PTR(out);
  k_tmat_transform_points<<<grid_for(nout * k, 256), 256, 0, BS_STREAM(s)>>>(m, n, pts, np_, k, nout, out);
  return launch_status();
}

int bs_pose_from_matrix_f64(const double* m, int64_t n, double* po, double* qo, double* err,
                            void* s) {
  if (n < 0) return BS_ERR_ARGUMENT;
  if (n == 0) return BS_OK;
  BS_CHECK_PTR(m); BS_CHECK_PTR(po); BS_CHECK_PTR(qo); BS_CHECK_PTR(err);
  k_pose_from_matrix<<<grid_for(n, 256), 256, 0, BS_STREAM(s)>>>(
      m, n, po, qo, reinterpret_cast<unsigned long long*>(err));
  return launch_status();
}

}  // extern "C"
