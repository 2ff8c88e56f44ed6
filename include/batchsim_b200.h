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
#define BS_ABI_VERSION 9
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

/* Quaternion algebra (pose.py:43-88 quat_mul / quat_conjugate / quat_rotate / quat_to_matrix,
 * pose.py:91-122 matrix_to_quat).  Binary ops broadcast a singleton side (na == nb, or either
 * is 1; else BS_ERR_DIMENSION, like pose.py:167-174).  fp64 results are bit-identical to
 * numpy's (separately rounded + and *, the reference's operation order). */
int bs_quat_mul_f64(const double* a, int64_t na, const double* b, int64_t nb, double* out,
                    void* stream);
int bs_quat_mul_f32(const float* a, int64_t na, const float* b, int64_t nb, float* out,
                    void* stream);
int bs_quat_conjugate_f64(const double* q, int64_t n, double* out, void* stream);
int bs_quat_rotate_f64(const double* q, int64_t nq, const double* v, int64_t nv, double* out,
                       void* stream);
int bs_quat_rotate_f32(const float* q, int64_t nq, const float* v, int64_t nv, float* out,
                       void* stream);
/* q: [n][4] -> m: [n][3][3] row-major. */
int bs_quat_to_matrix_f64(const double* q, int64_t n, double* m_out, void* stream);
/* m: [n][3][3] -> q: [n][4], Shepperd's method (branch = first argmax of trace, m00, m11, m22),
 * normalized once. */
int bs_matrix_to_quat_f64(const double* m, int64_t n, double* q_out, void* stream);

/* TransformMatrixBatch (pose.py:125-164) on [n][4][4] row-major fp64 matrices: compose
 * (= matmul, singleton broadcast), rigid inverse (R^T, -R^T t), transform_points (R x + t for
 * [np][k][3] points, singleton broadcast on either side). */
int bs_tmat_compose_f64(const double* a, int64_t na, const double* b, int64_t nb, double* out,
                        void* stream);
int bs_tmat_inverse_f64(const double* m, int64_t n, double* out, void* stream);
int bs_tmat_transform_points_f64(const double* m, int64_t n, const double* pts, int64_t np_,
                                 int64_t k, double* out, void* stream);

/* ------------------------------------------------------ scene store (SoA) ---- */
/* The SoA GPU state store that replaces the reference's per-env SceneBatch objects
 * (SPEC.md:168-236).  Tables describe each DISTINCT env layout ("model"); envs point at a
 * model by index, so a homogeneous batch stores one copy.  All arrays are row-major with
 * the fixed strides given by the *_max fields.  Field order is part of the ABI. */

enum { BS_KIND_SPHERE = 0, BS_KIND_BOX = 1, BS_KIND_CAPSULE = 2, BS_KIND_CYLINDER = 3,
       BS_KIND_PLANE = 4 };
enum { BS_JOINT_FIXED = 0, BS_JOINT_REVOLUTE = 1, BS_JOINT_PRISMATIC = 2 };
enum { BS_BODY_LINK = 0, BS_BODY_ACTOR = 1, BS_BODY_STATIC = 2 };
/* pair routine codes (bit 4 = roles swapped); 0 = unsupported pair (counted) */
enum { BS_PAIR_UNSUPPORTED = 0, BS_PAIR_SPHERE_PLANE = 1, BS_PAIR_BOX_PLANE = 2,
       BS_PAIR_SPHERE_SPHERE = 3, BS_PAIR_SPHERE_BOX = 4, BS_PAIR_CAPSULE_PLANE = 5,
       BS_PAIR_SWAP = 16 };
enum { BS_CTRL_PD_JOINT_POS = 0, BS_CTRL_PD_JOINT_DELTA_POS = 1, BS_CTRL_PD_EE_DELTA_POSE = 2,
       BS_CTRL_BASE_FORWARD_ROTATE = 3 };
enum { BS_TASK_NONE = 0, BS_TASK_PICKCUBE = 1, BS_TASK_OPENCHAIN = 2, BS_TASK_CARTPOLE = 3 };

typedef struct BsModelTables {
  int32_t num_models, L_max, D_max, S_max, P_max, A_max, C_max;
  const int32_t* n_links;      /* [M] */
  const int32_t* n_dof;        /* [M] */
  const int32_t* n_shapes;     /* [M] */
  const int32_t* n_pairs;      /* [M] */
  const int32_t* n_actors;     /* [M] */
  const int32_t* link_parent;  /* [M][L_max]  -1 = root attached to the world */
  const int32_t* link_jtype;   /* [M][L_max]  BS_JOINT_* (roots: FIXED)         */
  const int32_t* link_dof;     /* [M][L_max]  dof index or -1                   */
  const int32_t* link_grounded;/* [M][L_max]  1 = no movable joint to the world */
  const double* link_axis;     /* [M][L_max][3] joint axis (child frame)        */
  const double* link_org;      /* [M][L_max][7] joint origin (roots: base pose) p,q */
  const double* link_mass;     /* [M][L_max]                                     */
  const double* link_com;      /* [M][L_max][3] COM in the link frame            */
  const double* link_inertia;  /* [M][L_max][6] about COM, link axes: xx yy zz xy xz yz */
  const double* dof_lower;     /* [M][D_max] */
  const double* dof_upper;     /* [M][D_max] */
  const double* dof_damping;   /* [M][D_max] */
  const double* dof_kp;        /* [M][D_max] drive stiffness (0 = undriven)     */
  const double* dof_kd;        /* [M][D_max] */
  const double* dof_flim;      /* [M][D_max] force limit (inf allowed)          */
  const int32_t* dof_ctrl;     /* [M][D_max] controller action index or -1      */
  const int32_t* shape_btype;  /* [M][S_max] BS_BODY_*                          */
  const int32_t* shape_body;   /* [M][S_max] link / actor / static index       */
  const int32_t* shape_kind;   /* [M][S_max] BS_KIND_*                          */
  const int32_t* shape_seg;    /* [M][S_max] segmentation id (1 + entity slot)  */
  const double* shape_size;    /* [M][S_max][3] */
  const double* shape_frame;   /* [M][S_max][7] local pose (statics: world pose) */
  const double* shape_radius;  /* [M][S_max] bounding radius (plane: inf)       */
  const float* shape_color;    /* [M][S_max][4] base RGBA                        */
  const int32_t* pair_i;       /* [M][P_max] first shape slot (body A)           */
  const int32_t* pair_j;       /* [M][P_max] second shape slot (body B)          */
  const int32_t* pair_code;    /* [M][P_max] BS_PAIR_* (| BS_PAIR_SWAP)          */
  const int32_t* pair_slot;    /* [M][P_max] first contact slot of the pair (prefix of max contacts) */
  const double* actor_mass;    /* [M][A_max] */
  const double* actor_inertia; /* [M][A_max][3] principal, body frame            */
  const double* actor_rest;    /* [M][A_max][5] resting height z + orientation q (reset sampling) */
  int32_t A_dyn;               /* max free actors of any model (<= A_max; may be 0 when A_max is
                                  padded to 1): width of the step solver's actor block */
} BsModelTables;

typedef struct BsEnvState {
  int32_t num_envs;
  int64_t env_offset;          /* global index of env 0 on this shard (RNG key)  */
  const int32_t* model_id;     /* [N] */
  double* qpos;                /* [N][D_max] */
  double* qvel;                /* [N][D_max] */
  double* target;              /* [N][D_max] last drive targets                  */
  double* actor_pose;          /* [N][A_max][7] p, q                             */
  double* actor_vel;           /* [N][A_max][6] v, w (world)                     */
  double* link_pose;           /* [N][L_max][7] FK cache after the step          */
  double* goal;                /* [N][3] task goal                               */
  uint8_t* diverged;           /* [N] sticky until reset                         */
  int32_t* elapsed;            /* [N] steps in the current episode               */
  uint32_t* reset_count;       /* [N] episodes started (RNG counter)             */
  int32_t* target_dof;         /* [N] task-designated dof (OpenChain) or -1      */
  double* ep_return;           /* [N] running episode return (EpisodeMetrics) */
  uint8_t* ep_flags;           /* [N] bit0 success_once, bit1 fail_once (running) */
} BsEnvState;

typedef struct BsStepOutputs {
  float* obs;                  /* [N][obs_dim] state observation (may be NULL)   */
  int32_t obs_dim;
  float* reward;               /* [N] */
  uint8_t* terminated;         /* [N] */
  uint8_t* truncated;          /* [N] */
  uint8_t* success;            /* [N] raw success this step (info)               */
  uint8_t* fail;               /* [N] */
  int32_t* unsupported_pairs;  /* [N] broadphase hits of unsupported pair types  */
  int32_t* contact_count;      /* [N] contacts in the last substep (may be NULL) */
  int32_t* contact_pairs;      /* [N][C_max][2] shape slots (may be NULL)        */
  double* contact_geom;        /* [N][C_max][7] point, normal, depth (may be NULL) */
  /* EpisodeMetrics of episodes that ended this step; may all be NULL */
  uint8_t* ep_done;            /* [N] 1 = an episode ended (terminated or truncated) */
  double* ep_return_out;       /* [N] its return (sum of the step rewards)         */
  int32_t* ep_length_out;      /* [N] its length in steps                          */
  uint8_t* ep_flags_out;       /* [N] bit0 success_once bit1 success_at_end bit2 fail_once bit3 fail_at_end */
  float* final_obs;            /* [N][obs_dim] state obs of the state an episode ended in, written only for
                                  envs auto-reset this step (may be NULL; ABI 8) */
} BsStepOutputs;

typedef struct BsSimParams {
  double dt;                   /* 1 / sim_freq                                   */
  int32_t substeps;            /* sim_freq / control_freq                        */
  int32_t pos_iters, vel_iters;
  double gravity[3];
  double friction, beta, slop;
  int32_t ctrl_mode;           /* BS_CTRL_*                                      */
  int32_t action_dim;
  double action_scale;         /* joint modes: rad (or m) per unit action; ee mode: m */
  double action_scale_rot;     /* pd_ee_delta_pose: rad per unit rotation action   */
  double ik_lambda;
  int32_t ee_link;             /* controller / task end-effector link index      */
  int32_t task;                /* BS_TASK_*                                      */
  int32_t max_steps;           /* time limit T                                   */
  int32_t auto_reset;          /* 1: reset terminated|truncated envs in-kernel   */
  int32_t early_termination;   /* 1: terminated = success | fail                 */
  uint64_t seed;
  double task_f[16];           /* task constants (documented per task in DESIGN.md) */
  double control_freq;         /* Hz: delta controllers' target velocity = delta * control_freq (ABI 8) */
} BsSimParams;

/* One control step for every env: controller -> substeps x (drives + dynamics +
 * contacts + PGS + integration + limits + divergence) -> FK cache -> task evaluation ->
 * state obs -> in-kernel auto-reset.  Replaces env.step over
 * dynamics.step and controllers.apply.
 * action: [N][action_dim] float32 in [-1, 1] (clipped). */
int bs_step(const BsModelTables* tables, const BsEnvState* state, const BsStepOutputs* out,
            const BsSimParams* params, const float* action, void* stream);

/* Developer instrumentation: per-phase clock64() totals of thread 0 / CTA 0 of k_step (the
 * per-env critical path), available when the library is built with -DBS_PHASE_TIMING
 * (tools/phase_timing.py); BS_ERR_UNSUPPORTED otherwise.  out: host array of n <= 32. */
int bs_debug_phase_clocks(unsigned long long* out, int32_t n, int32_t reset);

/* Reset the envs selected by env_mask ([N] uint8, NULL = all) from their Philox streams,
 * then refresh the FK cache and the state obs.  Replaces env.reset. */
int bs_reset(const BsModelTables* tables, const BsEnvState* state, const BsStepOutputs* out,
             const BsSimParams* params, const uint8_t* env_mask, int32_t bump_count,
             void* stream);

/* Forward kinematics of the current qpos into state->link_pose. */
int bs_forward_kinematics(const BsModelTables* tables, const BsEnvState* state, void* stream);

/* Random actions in [-1,1) (Philox, counter = (blk, step, global env, 'ACT!')) --
 * the benchmark's "1000 random actions" generated on the device. */
int bs_random_actions(uint64_t seed, int64_t step, int64_t env_offset, int32_t num_envs,
                      int32_t action_dim, float* action_out, void* stream);

/* Masked state copy for set_state(snapshot, env_mask): for every env
 * with mask != 0 copy `row_bytes` bytes of row e from src to dst. */
int bs_masked_copy(const void* src, void* dst, int64_t num_envs, int64_t row_bytes,
                   const uint8_t* env_mask, void* stream);


/* ------------------------------------------------------------- batched rasterizer ---- */
/* Tessellated shapes of every model (SPEC.md:461 counts: sphere 320, box 12, capsule 512,
 * cylinder 64 triangles; the ground plane is a finite grid, A-9/A-11).  Vertices
 * are float32 in the shape's local frame; triangles index model-local vertices and are
 * wound counter-clockwise around the outward normal. */
typedef struct BsMeshTables {
  int32_t num_models, V_max, T_max;
  const int32_t* n_verts;      /* [M] */
  const int32_t* n_tris;       /* [M] */
  const float* verts;          /* [M][V_max][3] */
  const int32_t* vert_shape;   /* [M][V_max] shape slot of the vertex */
  const int32_t* tris;         /* [M][T_max][3] */
  const int32_t* tri_shape;    /* [M][T_max] shape slot of the triangle */
  const int32_t* tri_packed;   /* [M][T_max][4] i0, i1, i2, shape slot: the same triangles as one
                                  16-byte record each (may be NULL: tris + tri_shape are read; ABI 9) */
} BsMeshTables;

/* CameraConfig: one group of cameras sharing a resolution.  OpenCV axes
 * (x right, y down, z forward); pose = camera -> world, or the local offset on the mount
 * link when mount_link[c] >= 0 (camera pose = link pose o offset). */
typedef struct BsCameraBatch {
  int32_t num_cams, width, height;
  float near_plane, far_plane;
  const int32_t* mount_link;   /* [C] link slot or -1 (may be NULL: all world-fixed) */
  const double* pose;          /* [N][C][7] p, q (w,x,y,z) */
  const float* intrinsics;     /* [N][C][4] fx, fy, cx, cy (pixels) */
} BsCameraBatch;

typedef struct BsRenderParams {
  double light_dir[3];         /* unit vector towards the light, world frame */
  float ambient, diffuse;      /* flat shading: ambient + diffuse * max(0, n.l) (A-12) */
  float background[3];         /* rgb in [0,1] of empty pixels */
  int32_t tile;                /* tile size: a CTA's key buffer holds tile^2 pixels, laid out as a
                                  full-width strip up to 256 pixels wide (0 = default 128) */
  float* frame_scratch;        /* optional device scratch [N][C][12 S_max + 20] floats: per-frame
                                  shape -> camera transforms and camera block, computed by a
                                  parallel pre-pass (NULL: computed inside the rasterizer) */
  uint32_t* frame_queue;       /* optional device word (ABI 8): with frame_scratch, the persistent
                                  rasterizer CTAs pull frames from this counter (dynamic load
                                  balance across frames of unequal cost); NULL: static stride */
} BsRenderParams;

/* FrameBatch + the fused pointcloud (A-10).  Any pointer
 * may be NULL (that output is skipped).  Layouts: rgb [N][C][H][W][3] u8, depth [N][C][H][W]
 * f32 (0 = no hit), seg [N][C][H][W] u16 (0 = background), pointcloud [N][C][H*W][6] f32
 * (world xyz, rgb in [0,1]; all-zero where seg == 0). */
typedef struct BsFrameBatch {
  uint8_t* rgb;
  float* depth;
  uint16_t* seg;
  float* pointcloud;
} BsFrameBatch;

/* render(scene, cameras) + pointcloud for every env and
 * camera of the group, from the link-pose cache and actor poses in `state`.  env_color:
 * [N][S_max][3] float per-env shape colours (texture randomisation) or NULL for the model
 * colours. */
int bs_render(const BsModelTables* tables, const BsEnvState* state, const BsMeshTables* mesh,
              const BsCameraBatch* cams, const float* env_color, const BsRenderParams* params,
              const BsFrameBatch* out, void* stream);


/* Env.step_host's host-side step (ABI 9): copy `n` floats of actions from host memory `src`
 * into the pinned host buffer `dst` that a captured step graph reads (zero-copy), reject the step
 * with BS_ERR_INPUT before anything is launched when check != 0 and an action is not finite,
 * then launch `graph_exec` (a cudaGraphExec_t) on `stream` and synchronise the stream.  Replaces
 * the per-step host work of the reference's env.step(action) call path for
 * callers that keep actions and observations on the host. */
int bs_host_step(const float* src, float* dst, int64_t n, int32_t check, void* graph_exec, void* stream);

/* voxelize(points, cell, bounds): occupancy grid [batches][nx][ny][nz] u8 of
 * points (xyz at the start of each `point_stride`-float record, e.g. the fused pointcloud with
 * stride 6), cell index = floor((p - lo) / cell) per axis in float32; points with valid == 0
 * (may be NULL) or outside the grid are dropped.  `lo` is a HOST array of 3 floats.  cell <= 0
 * -> BS_ERR_INPUT. */
int bs_voxelize(const float* points, int64_t point_stride, const uint8_t* valid, int64_t points_per_batch,
                int64_t batches, const float* lo, float cell, int32_t nx, int32_t ny, int32_t nz,
                uint8_t* grid, void* stream);

/* composite_greenscreen(frame, background): out = rgb where seg != 0, else the
 * background pixel; rgb/out [frames][H][W][3] u8, seg [frames][H][W] u16, background [H][W][3]. */
int bs_composite_greenscreen(const uint8_t* rgb, const uint16_t* seg, const uint8_t* background,
                             int64_t height, int64_t width, int64_t frames, uint8_t* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BATCHSIM_B200_H_ */
