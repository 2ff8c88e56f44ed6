/* batchsim-b200 C ABI -- the drop-in boundary of the B200 simulate-and-render hot path.
 *
 * The reference (arxiv 2410.00425 / ManiSkill3, CPU re-embodiment `batchsim`) exposes a
 * Python API, no FFI.  Each entry point below replaces one reference operation; the
 * citation after each declaration names the reference interface (file:line under
 * /root/reference) whose semantics it implements.  INTEGRATION.md shows the ctypes
 * binding a maintainer adds on the reference side.
 *
 * Conventions (all entry points):
 *   - plain pointers + sizes, no framework types; every buffer is DEVICE memory owned by
 *     the caller (the kernels never allocate); poses are SoA: positions (N,3) and
 *     scalar-first quaternions (N,4) (w,x,y,z), row-major contiguous;
 *   - `stream` is a cudaStream_t passed as void*; work is asynchronous on it and every
 *     entry point is CUDA-graph capturable (no host sync, no allocation);
 *   - return value is a status code (BS_OK or BS_ERR_*); argument errors are detected
 *     on the host before any launch.
 */
#ifndef BATCHSIM_B200_H_
#define BATCHSIM_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the Python layer maps them onto errors.py:8-45 classes. */
#define BS_OK 0
#define BS_ERR_DIMENSION 1   /* DimensionError  (errors.py:8)  */
#define BS_ERR_INPUT 2       /* InputError      (errors.py:44) */
#define BS_ERR_LAYOUT 3      /* LayoutMismatchError (errors.py:32) */
#define BS_ERR_CUDA 4        /* launch / runtime failure       */
#define BS_ERR_ARGUMENT 5    /* null pointer, negative size    */
#define BS_ERR_UNSUPPORTED 6 /* ModelError      (errors.py:40) */

/* ABI version: bumped whenever a signature or a struct layout below changes. */
#define BS_ABI_VERSION 1
int bs_abi_version(void);

/* Bind the library's CUDA runtime to `device` (call once per process/thread before use;
 * the Python layer does it on import with the current torch device). */
int bs_init(int device);

/* ---------------------------------------------------------------- pose algebra ---- */
/* quat_normalize: pose.py:31-40 (norm, cascaded sign rule). q_out may alias q. */
int bs_quat_normalize_f64(const double* q, int64_t n, double* q_out, void* stream);
int bs_quat_normalize_f32(const float* q, int64_t n, float* q_out, void* stream);

/* PoseBatch.compose: pose.py:239-249 (+ _broadcast_pair pose.py:167-174).
 * na == nb, or one side == 1 (broadcast); otherwise BS_ERR_DIMENSION.
 * Output batch = max(na, nb). */
int bs_pose_compose_f64(const double* pa, const double* qa, int64_t na,
                        const double* pb, const double* qb, int64_t nb,
                        double* p_out, double* q_out, void* stream);
int bs_pose_compose_f32(const float* pa, const float* qa, int64_t na,
                        const float* pb, const float* qb, int64_t nb,
                        float* p_out, float* q_out, void* stream);

/* PoseBatch.inverse: pose.py:254-256. */
int bs_pose_inverse_f64(const double* p, const double* q, int64_t n,
                        double* p_out, double* q_out, void* stream);
int bs_pose_inverse_f32(const float* p, const float* q, int64_t n,
                        float* p_out, float* q_out, void* stream);

/* PoseBatch.transform_points: pose.py:258-274.  pts is (m, k, 3); n == m or either is 1.
 * out is (max(n,m), k, 3). */
int bs_pose_transform_points_f64(const double* p, const double* q, int64_t n,
                                 const double* pts, int64_t m, int64_t k,
                                 double* out, void* stream);
int bs_pose_transform_points_f32(const float* p, const float* q, int64_t n,
                                 const float* pts, int64_t m, int64_t k,
                                 float* out, void* stream);

/* PoseBatch.to_matrix: pose.py:276-280 (quat_to_matrix pose.py:72-88). out (n,4,4). */
int bs_pose_to_matrix_f64(const double* p, const double* q, int64_t n, double* m_out,
                          void* stream);

/* PoseBatch.from_matrix: pose.py:218-232 (matrix_to_quat pose.py:91-122).
 * Writes the max orthonormality error |R R^T - I| over the batch into *err_out (device
 * scalar, must be zeroed by the caller); the caller raises when it exceeds 1e-6. */
int bs_pose_from_matrix_f64(const double* m, int64_t n, double* p_out, double* q_out,
                            double* err_out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BATCHSIM_B200_H_ */
