// Reset, forward-kinematics, random-action and masked-copy kernels (one thread per env or
// element; none of them is on the per-step hot path -- the fused step is step.cu).
// Reference semantics: SPEC.md:536-544 (reset from per-env Philox streams), 249-257 (FK),
// 204-212 (set_state with env_mask), PAPER.md:410 (random-action benchmark stream).
#include "sim_common.cuh"

namespace bs {
namespace sim {

// ----------------------------------------------------------------------------------
// load/store of one env's state rows
template <class C>
struct EnvRegs {
  R q[C::MD], qd[C::MD], tgt[C::MD], goal[3];
  V3<R> ap[C::MA], av[C::MA], aw[C::MA];
  Q4<R> aq[C::MA];
};

template <class C>
__device__ __forceinline__ void load_env(const BsModelTables& T, const BsEnvState& S, const Model& M, int e,
                                         EnvRegs<C>& r) {
  const R* q = S.qpos + (int64_t)e * T.D_max;
  const R* qd = S.qvel + (int64_t)e * T.D_max;
  for (int i = 0; i < M.D; ++i) { r.q[i] = q[i]; r.qd[i] = qd[i]; }
  const R* pose = S.actor_pose + (int64_t)e * T.A_max * 7;
  const R* vel = S.actor_vel + (int64_t)e * T.A_max * 6;
  for (int a = 0; a < M.A; ++a) {
    r.ap[a] = ld3(pose + 7 * a); r.aq[a] = ld4(pose + 7 * a + 3);
    r.av[a] = ld3(vel + 6 * a); r.aw[a] = ld3(vel + 6 * a + 3);
  }
  for (int k = 0; k < 3; ++k) r.goal[k] = S.goal[3 * (int64_t)e + k];
}

template <class C>
__device__ __forceinline__ void store_env(const BsModelTables& T, const BsEnvState& S, const Model& M, int e,
                                          const EnvRegs<C>& r, const V3<R>* lp, const Q4<R>* lq) {
  R* q = S.qpos + (int64_t)e * T.D_max;
  R* qd = S.qvel + (int64_t)e * T.D_max;
  R* tg = S.target + (int64_t)e * T.D_max;
  for (int i = 0; i < M.D; ++i) { q[i] = r.q[i]; qd[i] = r.qd[i]; tg[i] = r.tgt[i]; }
  R* pose = S.actor_pose + (int64_t)e * T.A_max * 7;
  R* vel = S.actor_vel + (int64_t)e * T.A_max * 6;
  for (int a = 0; a < M.A; ++a) {
    st3(pose + 7 * a, r.ap[a]); st4(pose + 7 * a + 3, r.aq[a]);
    st3(vel + 6 * a, r.av[a]); st3(vel + 6 * a + 3, r.aw[a]);
  }
  for (int k = 0; k < 3; ++k) S.goal[3 * (int64_t)e + k] = r.goal[k];
  R* lc = S.link_pose + (int64_t)e * T.L_max * 7;
  for (int l = 0; l < M.L; ++l) { st3(lc + 7 * l, lp[l]); st4(lc + 7 * l + 3, lq[l]); }
}

template <class C>
__global__ void __launch_bounds__(64) k_reset(BsModelTables T, BsEnvState S, BsStepOutputs O, BsSimParams P,
                                              const uint8_t* __restrict__ mask, int bump) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= S.num_envs) return;
  const Model M = model_of(T, S.model_id[e]);
  EnvRegs<C> r;
  load_env<C>(T, S, M, e, r);
  Scratch<C> sc;
  if (mask != nullptr && !mask[e]) {
    // not selected: the env's state (its FK cache included) is left untouched bit for bit;
    // only its state obs is re-emitted, from the cached link poses
    if (O.obs) {
      const R* lc = S.link_pose + (int64_t)e * T.L_max * 7;
      for (int l = 0; l < M.L; ++l) { sc.lp[l] = ld3(lc + 7 * l); sc.lq[l] = ld4(lc + 7 * l + 3); }
      pack_obs(M, P, T.D_max, T.A_max, r.q, r.qd, sc.lp, r.ap, r.aq, r.av, r.aw, r.goal,
               O.obs + (int64_t)e * O.obs_dim, O.obs_dim);
    }
    return;
  }
  {
    uint32_t rc = S.reset_count[e] + (bump ? 1u : 0u);
    S.reset_count[e] = rc;
    int32_t tdof = -1;
    task_reset(M, P, S.env_offset + e, rc, r.q, r.qd, r.ap, r.aq, r.av, r.aw, r.goal, &tdof);
    S.target_dof[e] = tdof;
    S.elapsed[e] = 0;
    S.diverged[e] = 0;
    if (S.ep_return) S.ep_return[e] = 0.0;
    if (S.ep_flags) S.ep_flags[e] = 0;
    for (int i = 0; i < M.D; ++i) r.tgt[i] = r.q[i];
  }
  fk<C>(M, r.q, sc.lp, sc.lq);
  store_env<C>(T, S, M, e, r, sc.lp, sc.lq);
  if (O.obs) pack_obs(M, P, T.D_max, T.A_max, r.q, r.qd, sc.lp, r.ap, r.aq, r.av, r.aw, r.goal,
                      O.obs + (int64_t)e * O.obs_dim, O.obs_dim);
}

template <class C>
__global__ void k_fk(BsModelTables T, BsEnvState S) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= S.num_envs) return;
  const Model M = model_of(T, S.model_id[e]);
  R q[C::MD];
  const R* qs = S.qpos + (int64_t)e * T.D_max;
  for (int i = 0; i < M.D; ++i) q[i] = qs[i];
  V3<R> lp[C::ML];
  Q4<R> lq[C::ML];
  fk<C>(M, q, lp, lq);
  R* lc = S.link_pose + (int64_t)e * T.L_max * 7;
  for (int l = 0; l < M.L; ++l) { st3(lc + 7 * l, lp[l]); st4(lc + 7 * l + 3, lq[l]); }
}

__global__ void k_random_actions(uint64_t seed, int64_t step, int64_t off, int n, int dim, float* out) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  uint32_t k0 = (uint32_t)(seed & 0xffffffffu), k1 = (uint32_t)(seed >> 32);
  for (int blk = 0; blk * 4 < dim; ++blk) {
    U4 r = philox(U4{(uint32_t)blk, (uint32_t)step, (uint32_t)(off + e), TAG_ACTION}, k0, k1);
    uint32_t w[4] = {r.x, r.y, r.z, r.w};
    for (int j = 0; j < 4 && 4 * blk + j < dim; ++j) {
      float u = __fmul_rn((float)(w[j] >> 8), 1.0f / 16777216.0f);
      out[(int64_t)e * dim + 4 * blk + j] = __fsub_rn(__fmul_rn(u, 2.0f), 1.0f);
    }
  }
}

__global__ void k_masked_copy(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t n,
                              int64_t row, const uint8_t* __restrict__ mask) {
  int64_t total = n * row;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = i / row;
    if (mask == nullptr || mask[e]) dst[i] = src[i];
  }
}

// capacity tiers: (MD, ML, MS, MC, MA)
typedef Cap<4, 8, 8, 12, 2> CapSmall;     // PickCube-style (D=3, L=5, S=5, C=10, A=1)
typedef Cap<12, 16, 32, 64, 4> CapLarge;  // cabinets / heterogeneous scenes

template <class C>
bool fits(const BsModelTables& T) {
  return T.D_max <= C::MD && T.L_max <= C::ML && T.S_max <= C::MS && T.C_max <= C::MC && T.A_max <= C::MA;
}

}  // namespace sim
}  // namespace bs

using namespace bs::sim;

#define THREADS 32

extern "C" {

int bs_reset(const BsModelTables* T, const BsEnvState* S, const BsStepOutputs* O, const BsSimParams* P,
             const uint8_t* mask, int32_t bump, void* stream) {
  if (!T || !S || !O || !P) return BS_ERR_ARGUMENT;
  if (S->num_envs <= 0) return BS_OK;
  int blocks = (S->num_envs + THREADS - 1) / THREADS;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (fits<CapSmall>(*T)) k_reset<CapSmall><<<blocks, THREADS, 0, st>>>(*T, *S, *O, *P, mask, bump);
  else if (fits<CapLarge>(*T)) k_reset<CapLarge><<<blocks, THREADS, 0, st>>>(*T, *S, *O, *P, mask, bump);
  else return BS_ERR_UNSUPPORTED;
  return bs::launch_status();
}

int bs_forward_kinematics(const BsModelTables* T, const BsEnvState* S, void* stream) {
  if (!T || !S) return BS_ERR_ARGUMENT;
  if (S->num_envs <= 0) return BS_OK;
  int blocks = (S->num_envs + 127) / 128;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (fits<CapSmall>(*T)) k_fk<CapSmall><<<blocks, 128, 0, st>>>(*T, *S);
  else if (fits<CapLarge>(*T)) k_fk<CapLarge><<<blocks, 128, 0, st>>>(*T, *S);
  else return BS_ERR_UNSUPPORTED;
  return bs::launch_status();
}

int bs_random_actions(uint64_t seed, int64_t step, int64_t off, int32_t n, int32_t dim, float* out, void* stream) {
  if (!out || n < 0 || dim < 0) return BS_ERR_ARGUMENT;
  if (n == 0 || dim == 0) return BS_OK;
  k_random_actions<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(seed, step, off, n, dim, out);
  return bs::launch_status();
}

int bs_masked_copy(const void* src, void* dst, int64_t n, int64_t row, const uint8_t* mask, void* stream) {
  if (!src || !dst || n < 0 || row < 0) return BS_ERR_ARGUMENT;
  if (n == 0 || row == 0) return BS_OK;
  k_masked_copy<<<bs::grid_for(n * row, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      (const uint8_t*)src, (uint8_t*)dst, n, row, mask);
  return bs::launch_status();
}

}  // extern "C"
