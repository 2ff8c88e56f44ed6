// Fused control step for every env (bs_step): controller -> substeps (FK, RNEA bias + CRBA
// mass matrix + implicit PD drives -> Cholesky -> M^-1, free-body gyroscopics, shape poses,
// broadphase + narrowphase over the static pair list, ordered contact compaction, PGS rows,
// projected Gauss-Seidel, semi-implicit Euler, joint limits, divergence freeze) -> FK cache
// -> task evaluation -> state obs -> in-kernel auto-reset.
//
// Reference semantics: SPEC.md:319-354 (dynamics), 249-257 (FK), 402-410 (controllers),
// 536-553 (reset/step), with DESIGN.md's decisions register (A-4..A-25).  The CPU oracle
// (oracle/engine.py) restates the same algorithm independently; tests/test_step_gpu.py
// holds the two together.
//
// Execution model (v1, B200): G = 8 lanes cooperate on one env, 4 envs per warp, one warp
// per CTA.  Every env's working set (state, link poses, spatial inertias, RNEA temporaries,
// M^-1, shape poses, contacts and PGS rows) is staged in shared memory (about 8 KB for the
// PickCube scene), so 28 envs -- 4096 envs over 148 SMs -- are resident at once.  Work that is
// parallel inside an env (links, shapes, actors, pairs, contact slots, constraint rows, M^-1
// columns, obs entries, state rows) is spread over the lanes; the inherently serial parts
// (FK chain, RNEA passes, Cholesky, the Gauss-Seidel sweep, whose row order is part of the
// result) run on the group's lanes redundantly or on lane 0, with __syncwarp between phases
// and ballots/shuffles for the compaction and reductions.  No fp64 division sits in the
// sweep: rows carry 1/K and M^-1 is explicit (the oracle also forms inv(Mt)).  Nothing in the
// step is a dense contraction, so there are no tensor cores; the kernel is latency/ALU
// bound and moves ~0.8 KB of HBM per env-step.
#include <stdlib.h>
#include <string.h>
#include "sim_common.cuh"

namespace bs {
namespace step {

using namespace bs::sim;

#define FULLMASK 0xffffffffu

// Phase-latency instrumentation (build with -DBS_PHASE_TIMING; tools/phase_timing.py): thread 0
// of CTA 0 accumulates clock64() deltas per phase, so the per-env critical path can be split
// into its phases.  Compiled out of the product build.
#ifdef BS_PHASE_TIMING
__device__ unsigned long long g_bs_phase[32];
__device__ long long g_bs_last;
#define BS_TICK(id)                                                    \
  do {                                                                 \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                         \
      const long long t_ = clock64();                                  \
      g_bs_phase[id] += (unsigned long long)(t_ - g_bs_last);          \
      g_bs_last = t_;                                                  \
    }                                                                  \
  } while (0)
#define BS_COUNT(id, v)                                                        \
  do {                                                                         \
    if (blockIdx.x == 0 && threadIdx.x == 0) g_bs_phase[id] += (unsigned long long)(v); \
  } while (0)
// every CTA: its own duration (slots 22 max, 23 sum, 24 count) -- the launch is as long as its
// slowest warp, not env 0's
// and the launch window in globaltimer ns: slot 25 ~(earliest CTA entry) (a max of complements, so
// the zero reset works), 27 latest CTA entry, 26 latest CTA exit
__device__ __forceinline__ unsigned long long bs_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define BS_CTA_BEGIN                                                           \
  const long long bs_cta_t0_ = clock64();                                      \
  if (threadIdx.x == 0) {                                                      \
    const unsigned long long g_ = bs_gtimer();                                 \
    atomicMax(&g_bs_phase[25], ~g_);                                           \
    atomicMax(&g_bs_phase[27], g_);                                            \
  }
#define BS_CTA_END                                                             \
  do {                                                                         \
    if (threadIdx.x == 0) {                                                    \
      const unsigned long long d_ = (unsigned long long)(clock64() - bs_cta_t0_); \
      atomicMax(&g_bs_phase[22], d_);                                          \
      atomicAdd(&g_bs_phase[23], d_);                                          \
      atomicAdd(&g_bs_phase[24], 1ull);                                        \
      atomicMax(&g_bs_phase[26], bs_gtimer());                                 \
    }                                                                          \
  } while (0)
#else
#define BS_CTA_BEGIN do { } while (0)
#define BS_CTA_END do { } while (0)
#define BS_TICK(id) do { } while (0)
#define BS_COUNT(id, v) do { } while (0)
#endif

// Per-env shared-memory layout, offsets in doubles (computed on the host from the table
// maxima; identical for every env of the launch).
struct Lay {
  int Dm, Lm, Sm, Cm, Am, NU, RW, KCH;
  int q, qd, tgt, tgtv, apose, avel, goal;
  int lpq, Sv, In, Mt, Minv, cb, u, Iwi, spq;
  int Tl, V, Ac, F, ct, rows;
  int total;
};

// Generalised velocity u (length NU = D_max + 6 A_max): [0, D_max) joint rates, then per actor
// slot a: linear velocity at [D_max + 6a, +3), angular at [D_max + 6a + 3, +3).
// Row layout (dense over u): [0] 1/K (0 = skip)  [1] lambda  [2] position-phase target
// [3] velocity-phase target, then NU interleaved pairs (J[k], W[k]) at [4 + 2k, 4 + 2k + 1],
// W = M_u^-1 J^T (the velocity change per unit impulse).  Rows start 16-byte aligned (the
// layout keeps every offset even), so the sweep reads the scalars and each (J, W) pair with
// one 16-byte shared load.  Rows touch at most two bodies, but a dense row has no per-row
// branching, no actor-index selects and no int conversions in the sweep.
#define ROW_J 4
#define JI(k) (ROW_J + 2 * (k))
#define WI(k) (ROW_J + 2 * (k) + 1)

// EX_ = the launch guarantees D_max == MD and A_max == MA exactly, so the padded widths
// (D_max, A_max, NU and the row stride) are compile-time constants in the kernel.
// SA_ = the free actors the solver carries (NU = MD + 6 SA); 0 for scenes without free actors
// (cabinets: A_max is padded to 1 but A_dyn = 0), whose u then fits the register-resident sweep.
template <int G_, int MD_, int MA_, bool EX_ = false, int SLOT_ = 1, int SA_ = MA_>
struct Cfg {
  static constexpr int G = G_, MD = MD_, MA = MA_, EPW = 32 / G_, NU = MD_ + 6 * SA_;
  static constexpr bool EXACT = EX_;
  static constexpr int SLOT = SLOT_;  // bs::LaunchCache slot of this variant's smem opt-in
};

__device__ __forceinline__ R sgn_of(R v) { return v > 0.0 ? 1.0 : -1.0; }

// Unit quaternion with the reference's sign rule (pose.py:31-40) but reciprocal-sqrt
// scaling (the step is tolerance-gated, not bit-gated).
__device__ __forceinline__ Q4<R> qnorm_f(Q4<R> q) {
  R ss = q.w * q.w;
  ss = ss + q.x * q.x;
  ss = ss + q.y * q.y;
  ss = ss + q.z * q.z;
  R inv = rsqrt(ss);
  Q4<R> r{q.w * inv, q.x * inv, q.y * inv, q.z * inv};
  R s = r.w != 0.0 ? sgn_of(r.w) : r.x != 0.0 ? sgn_of(r.x) : r.y != 0.0 ? sgn_of(r.y) : (r.z < 0.0 ? -1.0 : 1.0);
  return Q4<R>{r.w * s, r.x * s, r.y * s, r.z * s};
}

__device__ __forceinline__ void compose_f(V3<R> pa, Q4<R> qa, V3<R> pb, Q4<R> qb, V3<R>& po, Q4<R>& qo) {
  V3<R> r = quat_rotate(qa, pb);
  po = add(pa, r);
  qo = qnorm_f(quat_mul(qa, qb));
}

__device__ __forceinline__ void st7(R* d, V3<R> p, Q4<R> q) {
  d[0] = p.x; d[1] = p.y; d[2] = p.z; d[3] = q.w; d[4] = q.x; d[5] = q.y; d[6] = q.z;
}
__device__ __forceinline__ V6 ld6(const R* s) { return V6{{s[0], s[1], s[2]}, {s[3], s[4], s[5]}}; }
__device__ __forceinline__ void st6(R* d, const V6& a) {
  d[0] = a.w[0]; d[1] = a.w[1]; d[2] = a.w[2]; d[3] = a.v[0]; d[4] = a.v[1]; d[5] = a.v[2];
}
__device__ __forceinline__ V6 add6(const V6& a, const V6& b) { return mk6(add(gw(a), gw(b)), add(gv(a), gv(b))); }
__device__ __forceinline__ Inertia ldI(const R* s) {
  Inertia I;
  I.m = s[0];
  I.h = ld3(s + 1);
#pragma unroll
  for (int k = 0; k < 6; ++k) I.I[k] = s[4 + k];
  return I;
}
__device__ __forceinline__ void stI(R* d, const Inertia& I) {
  d[0] = I.m;
  st3(d + 1, I.h);
#pragma unroll
  for (int k = 0; k < 6; ++k) d[4 + k] = I.I[k];
}

__device__ __forceinline__ int pair_maxc(int code) {
  switch (code & 15) {
    case BS_PAIR_SPHERE_PLANE: return 1;
    case BS_PAIR_BOX_PLANE: return 4;
    case BS_PAIR_SPHERE_SPHERE: return 1;
    case BS_PAIR_SPHERE_BOX: return 1;
    case BS_PAIR_CAPSULE_PLANE: return 2;
    default: return 0;
  }
}

// Actor world inertia and its inverse: R diag(I) R^T, R diag(1/I) R^T (A-8: contact response
// and the angular-momentum transport of the free rotation).
__device__ __forceinline__ void actor_inertia_f(const R* Ib, Q4<R> q, R* Iw, R* Iwi) {
  R r[9];
  quat_to_matrix(q, r);
  R ib[3] = {Ib[0], Ib[1], Ib[2]};
  R ii[3] = {1.0 / Ib[0], 1.0 / Ib[1], 1.0 / Ib[2]};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      R s = 0, si = 0;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        s += r[3 * i + k] * ib[k] * r[3 * j + k];
        si += r[3 * i + k] * ii[k] * r[3 * j + k];
      }
      Iw[3 * i + j] = s;
      Iwi[3 * i + j] = si;
    }
}

// A candidate contact slot: [0..3) point (midpoint), [3..6) normal (second -> first body),
// [6] depth, [7] pair index (-1 = empty slot).
__device__ __forceinline__ void put_cand(R* c, V3<R> sB, V3<R> n, R depth, int pair, bool flip, R slop) {
  if (!(depth >= -slop)) { c[7] = -1.0; return; }
  V3<R> p = sub(sB, scl(n, 0.5 * depth));
  V3<R> nn = flip ? scl(n, -1.0) : n;
  st3(c, p);
  st3(c + 3, nn);
  c[6] = depth;
  c[7] = (R)pair;
}

// Narrowphase of one static pair (A-4, A-25) into its fixed slots.
// Returns 1 when the pair passed the broadphase but has no routine (A-23).
__device__ __forceinline__ int narrow_pair(const Model& M, int pi, const R* spq, R slop, R* cand) {
  const int i = M.p_i[pi], j = M.p_j[pi], code = M.p_code[pi];
  const int ki = M.s_kind[i], kj = M.s_kind[j];
  const int mc = pair_maxc(code);
  for (int k = 0; k < mc; ++k) cand[8 * k + 7] = -1.0;
  V3<R> pI = ld3(spq + 7 * i), pJ = ld3(spq + 7 * j);
  bool near;
  if (ki == BS_KIND_PLANE || kj == BS_KIND_PLANE) {
    int pl = kj == BS_KIND_PLANE ? j : i, ot = kj == BS_KIND_PLANE ? i : j;
    V3<R> n = quat_rotate(ld4(spq + 7 * pl + 3), v3(0, 0, 1));
    near = dot(n, sub(ld3(spq + 7 * ot), ld3(spq + 7 * pl))) <= M.s_radius[ot] + slop;
  } else {
    V3<R> d = sub(pI, pJ);
    near = sqrt(dot(d, d)) <= (M.s_radius[i] + M.s_radius[j]) + slop;
  }
  if (!near) return 0;
  const int base = code & 15;
  if (base == BS_PAIR_UNSUPPORTED) return 1;
  const bool flip = (code & BS_PAIR_SWAP) != 0;
  const int a = flip ? j : i, b = flip ? i : j;
  const R* sa = M.s_size + 3 * a;
  const R* sb = M.s_size + 3 * b;
  const V3<R> pa = ld3(spq + 7 * a), pb = ld3(spq + 7 * b);
  const Q4<R> qa = ld4(spq + 7 * a + 3), qb = ld4(spq + 7 * b + 3);
  if (base == BS_PAIR_SPHERE_PLANE) {
    V3<R> n = quat_rotate(qb, v3(0, 0, 1));
    R sd = dot(n, sub(pa, pb));
    put_cand(cand, sub(pa, scl(n, sd)), n, sa[0] - sd, pi, flip, slop);
  } else if (base == BS_PAIR_BOX_PLANE) {
    V3<R> n = quat_rotate(qb, v3(0, 0, 1));
    R dep[8];
    V3<R> sB[8];
    int valid = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      V3<R> loc = v3((k & 1) ? sa[0] : -sa[0], (k & 2) ? sa[1] : -sa[1], (k & 4) ? sa[2] : -sa[2]);
      V3<R> corner = add(pa, quat_rotate(qa, loc));
      R sd = dot(n, sub(corner, pb));
      dep[k] = -sd;
      sB[k] = sub(corner, scl(n, sd));
      valid += dep[k] >= -slop;
    }
    if (valid > 4) {  // keep the four deepest, ties -> lower corner index (A-4)
      R keep[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        int rank = 0;
#pragma unroll
        for (int o = 0; o < 8; ++o) rank += (dep[o] > dep[k]) || (dep[o] == dep[k] && o < k);
        keep[k] = (dep[k] >= -slop && rank >= 4) ? -INFINITY : dep[k];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) dep[k] = keep[k];
    }
    int w = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (dep[k] >= -slop && w < 4) put_cand(cand + 8 * (w++), sB[k], n, dep[k], pi, flip, slop);
    }
  } else if (base == BS_PAIR_SPHERE_SPHERE) {
    V3<R> d = sub(pa, pb);
    R dist = sqrt(dot(d, d));
    V3<R> n = v3(0, 0, 1);
    if (dist > 1e-12) {
      R inv = 1.0 / dist;
      n = v3(d.x * inv, d.y * inv, d.z * inv);
    }
    R depth = (sa[0] + sb[0]) - dist;
    put_cand(cand, add(pb, scl(n, sb[0])), n, depth, pi, flip, slop);
  } else if (base == BS_PAIR_SPHERE_BOX) {
    V3<R> loc = quat_rotate(qconj(qb), sub(pa, pb));
    R h[3] = {sb[0], sb[1], sb[2]};
    R l3[3] = {loc.x, loc.y, loc.z};
    R cl[3], dl[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      cl[k] = fmin(fmax(l3[k], -h[k]), h[k]);
      dl[k] = l3[k] - cl[k];
    }
    R d2 = (dl[0] * dl[0] + dl[1] * dl[1]) + dl[2] * dl[2];
    R nl[3], sl[3], depth;
    if (d2 > 1e-24) {
      R dist = sqrt(d2);
      R inv = 1.0 / dist;
#pragma unroll
      for (int k = 0; k < 3; ++k) { nl[k] = dl[k] * inv; sl[k] = cl[k]; }
      depth = sa[0] - dist;
    } else {
      int kk = 0;
      R best = h[0] - fabs(l3[0]), lk = l3[0], hk = h[0];  // selects, not indexed arrays (no local memory)
#pragma unroll
      for (int k = 1; k < 3; ++k) {
        R pen = h[k] - fabs(l3[k]);
        if (pen < best) { best = pen; kk = k; lk = l3[k]; hk = h[k]; }
      }
      R sg = lk >= 0.0 ? 1.0 : -1.0;
#pragma unroll
      for (int k = 0; k < 3; ++k) { nl[k] = k == kk ? sg : 0.0; sl[k] = k == kk ? sg * hk : l3[k]; }
      depth = sa[0] + best;
    }
    V3<R> n = quat_rotate(qb, v3(nl[0], nl[1], nl[2]));
    V3<R> s = add(pb, quat_rotate(qb, v3(sl[0], sl[1], sl[2])));
    put_cand(cand, s, n, depth, pi, flip, slop);
  } else if (base == BS_PAIR_CAPSULE_PLANE) {
    V3<R> n = quat_rotate(qb, v3(0, 0, 1));
    int w = 0;
    for (int k = 0; k < 2; ++k) {
      V3<R> e = add(pa, quat_rotate(qa, v3(0, 0, k ? sa[1] : -sa[1])));
      R sd = dot(n, sub(e, pb));
      R depth = sa[0] - sd;
      if (depth >= -slop) put_cand(cand + 8 * (w++), sub(e, scl(n, sd)), n, depth, pi, flip, slop);
    }
  }
  return 0;
}

// ------------------------------------------------------------------ group-cooperative FK
// Lanes build each link's local transform (joint origin o joint motion, with the sincos),
// then lane 0 walks the topological order composing parent o local.
template <int G>
__device__ __forceinline__ void fk_group(const Model& M, const Lay& Y, R* E, int l) {
  R* Tl = E + Y.Tl;
  R* lpq = E + Y.lpq;
  #pragma unroll 1
  for (int k = l; k < M.L; k += G) {
    const R* o = M.org + 7 * k;
    V3<R> tp = ld3(o);
    Q4<R> tq = ld4(o + 3);
    const int jt = M.jtype[k];
    if (jt != BS_JOINT_FIXED) {
      const R qv = E[Y.q + M.dof[k]];
      const V3<R> ax = ld3(M.axis + 3 * k);
      if (jt == BS_JOINT_REVOLUTE) {
        R s, c;
        sincos(0.5 * qv, &s, &c);
        compose_f(tp, tq, v3(0, 0, 0), Q4<R>{c, ax.x * s, ax.y * s, ax.z * s}, tp, tq);
      } else {
        tp = add(tp, quat_rotate(tq, scl(ax, qv)));
      }
    }
    st7(Tl + 7 * k, tp, tq);
  }
  __syncwarp();
  if (l == 0) {
    for (int k = 0; k < M.L; ++k) {
      const int par = M.parent[k];
      V3<R> p = ld3(Tl + 7 * k);
      Q4<R> q = ld4(Tl + 7 * k + 3);
      if (par >= 0) compose_f(ld3(lpq + 7 * par), ld4(lpq + 7 * par + 3), p, q, p, q);
      st7(lpq + 7 * k, p, q);
    }
  }
  __syncwarp();
}

// pd_ee_delta_pose targets (lane 0 of the group; rarely on the hot path, kept out of line).
__device__ __noinline__ void ee_delta_targets(const Model M, const BsSimParams& P, const Lay& Y, R* E,
                                              const float* act) {
  const int Dm = Y.Dm;
      R* Jm = E + Y.rows;        // 6 x Dm, scratch (rows are rebuilt every substep)
  R* A = Jm + 6 * Dm;        // 6 x 6
  for (int i = 0; i < 6 * Dm; ++i) Jm[i] = 0.0;
  const R* lpq0 = E + Y.lpq;
  const V3<R> pe = ld3(lpq0 + 7 * P.ee_link);
  for (int k = P.ee_link; k >= 0; k = M.parent[k]) {
    const int jt = M.jtype[k];
    if (jt == BS_JOINT_FIXED) continue;
    const int d = M.dof[k];
    if (M.ctrl[d] < 0) continue;
    const V3<R> a = quat_rotate(ld4(lpq0 + 7 * k + 3), ld3(M.axis + 3 * k));
    const V3<R> lin = jt == BS_JOINT_REVOLUTE ? crs(a, sub(pe, ld3(lpq0 + 7 * k))) : a;
    const V3<R> ang = jt == BS_JOINT_REVOLUTE ? a : v3(0, 0, 0);
    Jm[0 * Dm + d] = lin.x; Jm[1 * Dm + d] = lin.y; Jm[2 * Dm + d] = lin.z;
    Jm[3 * Dm + d] = ang.x; Jm[4 * Dm + d] = ang.y; Jm[5 * Dm + d] = ang.z;
  }
  R tw[6];
  for (int j = 0; j < 6; ++j) {
    const R aj = fmin(fmax((R)act[j], -1.0), 1.0);
    tw[j] = aj * (j < 3 ? P.action_scale : P.action_scale_rot);
  }
  {  // the rotation action is an axis-angle in the EE frame: rotate it to the world
    const V3<R> w = quat_rotate(ld4(lpq0 + 7 * P.ee_link + 3), v3(tw[3], tw[4], tw[5]));
    tw[3] = w.x; tw[4] = w.y; tw[5] = w.z;
  }
  const R lam2 = P.ik_lambda * P.ik_lambda;
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j <= i; ++j) {
      R sacc = 0.0;
      for (int d = 0; d < M.D; ++d) sacc += Jm[i * Dm + d] * Jm[j * Dm + d];
      if (i == j) sacc += lam2;
      A[i * 6 + j] = sacc;
    }
  for (int j = 0; j < 6; ++j) {  // Cholesky (lower), inverse diagonal kept
    R sd = A[j * 6 + j];
    for (int k = 0; k < j; ++k) sd -= A[j * 6 + k] * A[j * 6 + k];
    const R inv = rsqrt(sd);
    A[j * 6 + j] = inv;
    for (int i = j + 1; i < 6; ++i) {
      R t = A[i * 6 + j];
      for (int k = 0; k < j; ++k) t -= A[i * 6 + k] * A[j * 6 + k];
      A[i * 6 + j] = t * inv;
    }
  }
  for (int i = 0; i < 6; ++i) {
    R t = tw[i];
    for (int k = 0; k < i; ++k) t -= A[i * 6 + k] * tw[k];
    tw[i] = t * A[i * 6 + i];
  }
  for (int i = 5; i >= 0; --i) {
    R t = tw[i];
    for (int k = i + 1; k < 6; ++k) t -= A[k * 6 + i] * tw[k];
    tw[i] = t * A[i * 6 + i];
  }
  for (int d = 0; d < M.D; ++d) {
    const R qi = E[Y.q + d];
    R tgt = qi;
    if (M.ctrl[d] >= 0) {
      R dq = 0.0;
      for (int i = 0; i < 6; ++i) dq += Jm[i * Dm + d] * tw[i];
      tgt = fmin(fmax(qi + dq, M.lower[d]), M.upper[d]);
    }
    E[Y.tgt + d] = tgt;
    E[Y.tgtv + d] = (tgt - qi) * P.control_freq;  // the delta is a motion over one control period
  }
    }

// ------------------------------------------------------------------ one substep
template <class K>
__device__ __forceinline__ void substep(const Model& M, const BsSimParams& P, const Lay& Y, R* E, const int l, const int g,
                        bool& diverged, int& unsupported, int& nc) {
  constexpr int G = K::G, MD = K::MD, MA = K::MA;
  const R dt = P.dt;
  const int L = M.L, D = M.D, A = M.A, NS = M.S, Dm = K::EXACT ? MD : Y.Dm;
  R* lpq = E + Y.lpq;
  R* Sv = E + Y.Sv;
  R* In = E + Y.In;
  R* spq = E + Y.spq;
  R* Mt = E + Y.Mt;
  R* Minv = E + Y.Minv;
  R* cb = E + Y.cb;
  R* V = E + Y.V;
  R* Ac = E + Y.Ac;
  R* F = E + Y.F;

  fk_group<G>(M, Y, E, l);
  BS_TICK(2);

  // ---- A: per-link motion subspace + world inertia, per-shape world pose, per-actor free
  //         motion (gyroscopic + gravity), zero the mass matrix
  const V3<R> grav = v3(P.gravity[0], P.gravity[1], P.gravity[2]);
  #pragma unroll 1
  for (int i = l; i < D * Dm; i += G) Mt[i] = 0.0;
  #pragma unroll 1
  for (int i = D + l; i < Dm; i += G) E[Y.u + i] = 0.0;
  #pragma unroll 1
  for (int i = Dm + 6 * A + l; i < Y.NU; i += G) E[Y.u + i] = 0.0;
  #pragma unroll 1
  for (int t = l; t < L + NS + A; t += G) {
    if (t < L) {
      const int k = t, jt = M.jtype[k];
      const V3<R> p = ld3(lpq + 7 * k);
      const Q4<R> q = ld4(lpq + 7 * k + 3);
      V3<R> w = v3(0, 0, 0), v = v3(0, 0, 0);
      if (jt != BS_JOINT_FIXED) {
        V3<R> a = quat_rotate(q, ld3(M.axis + 3 * k));
        if (jt == BS_JOINT_REVOLUTE) { w = a; v = crs(p, a); } else { v = a; }
      }
      st3(Sv + 6 * k, w);
      st3(Sv + 6 * k + 3, v);
      stI(In + 10 * k, world_inertia(M, k, p, q));
    } else if (t < L + NS) {
      const int s = t - L;
      const R* f = M.s_frame + 7 * s;
      const int bt = M.s_btype[s], bi = M.s_body[s];
      V3<R> sp;
      Q4<R> sq;
      if (bt == BS_BODY_LINK) compose_f(ld3(lpq + 7 * bi), ld4(lpq + 7 * bi + 3), ld3(f), ld4(f + 3), sp, sq);
      else if (bt == BS_BODY_ACTOR) { sp = ld3(E + Y.apose + 7 * bi); sq = ld4(E + Y.apose + 7 * bi + 3); }
      else { sp = ld3(f); sq = ld4(f + 3); }
      st7(spq + 7 * s, sp, sq);
    } else {
      const int a = t - L - NS;
      const Q4<R> aq = ld4(E + Y.apose + 7 * a + 3);
      const V3<R> av = ld3(E + Y.avel + 6 * a), aw = ld3(E + Y.avel + 6 * a + 3);
      R Iw[9], Iwi[9];
      actor_inertia_f(M.a_inertia + 3 * a, aq, Iw, Iwi);
      // angular velocity enters the solve unchanged: the gyroscopic effect is the momentum
      // transport after the orientation update (phase L, A-8)
      st3(E + Y.u + Dm + 6 * a, add(av, scl(grav, dt)));
      st3(E + Y.u + Dm + 6 * a + 3, aw);
#pragma unroll
      for (int j = 0; j < 9; ++j) E[Y.Iwi + 9 * a + j] = Iwi[j];
    }
  }
  __syncwarp();
  BS_TICK(3);

  // ---- B: RNEA forward pass (serial over the topological order)
  if (l == 0) {
    const V6 g6 = {{0, 0, 0}, {-P.gravity[0], -P.gravity[1], -P.gravity[2]}};
    for (int k = 0; k < L; ++k) {
      const int par = M.parent[k];
      V6 Vk = par >= 0 ? ld6(V + 6 * par) : V6{{0, 0, 0}, {0, 0, 0}};
      V6 ak = par >= 0 ? ld6(Ac + 6 * par) : g6;
      if (M.jtype[k] != BS_JOINT_FIXED) {
        const R s = E[Y.qd + M.dof[k]];
        const V6 Sk = ld6(Sv + 6 * k);
        const V6 Sq = mk6(scl(gw(Sk), s), scl(gv(Sk), s));
        Vk = add6(Vk, Sq);
        ak = add6(ak, crossm(Vk, Sq));
      }
      st6(V + 6 * k, Vk);
      st6(Ac + 6 * k, ak);
    }
  }
  __syncwarp();
  BS_TICK(4);
  // ---- C: link forces F = I a + V x* I V (parallel over links)
  #pragma unroll 1
  for (int k = l; k < L; k += G) {
    const Inertia I = ldI(In + 10 * k);
    const V6 Vk = ld6(V + 6 * k);
    st6(F + 6 * k, add6(imul(I, ld6(Ac + 6 * k)), crossf(Vk, imul(I, Vk))));
  }
  __syncwarp();
  BS_TICK(5);
  // ---- D: backward pass: bias forces C(q, qd) and composite inertias.  Both accumulations are
  //         component-wise (child into parent, reverse topological order): lanes 0-5 carry one
  //         force component each, lanes 6-7 five inertia components each; then the bias terms
  //         S_k . F_k in parallel over links.
  if (l < 6) {
    for (int k = L - 1; k >= 0; --k) {
      const int par = M.parent[k];
      if (par >= 0) F[6 * par + l] += F[6 * k + l];
    }
  } else if (l < 8) {
    for (int k = L - 1; k >= 0; --k) {
      const int par = M.parent[k];
      if (par >= 0) {
#pragma unroll
        for (int j = l - 6; j < 10; j += 2) In[10 * par + j] += In[10 * k + j];
      }
    }
  }
  __syncwarp();
  #pragma unroll 1
  for (int k = l; k < L; k += G)
    if (M.jtype[k] != BS_JOINT_FIXED) cb[M.dof[k]] = dot6(ld6(Sv + 6 * k), ld6(F + 6 * k));
  __syncwarp();
  BS_TICK(6);
  // ---- E: CRBA mass matrix (parallel over dof links)
  #pragma unroll 1
  for (int k = l; k < L; k += G) {
    if (M.jtype[k] == BS_JOINT_FIXED) continue;
    const int i = M.dof[k];
    const V6 Fc = imul(ldI(In + 10 * k), ld6(Sv + 6 * k));
    for (int j = k; j >= 0; j = M.parent[j]) {
      if (M.jtype[j] == BS_JOINT_FIXED) continue;
      const int dj = M.dof[j];
      const R v = dot6(ld6(Sv + 6 * j), Fc);
      Mt[i * Dm + dj] = v;
      Mt[dj * Dm + i] = v;
    }
  }
  __syncwarp();
  BS_TICK(7);
  // ---- F: implicit PD drives (A-16) and Cholesky of Mt (lane 0; inverse diagonal kept).
  // tau = Kp (q* - q) + Kd (qd* - qd) with the gains per unit inertia scale
  // (SPEC.md:427): Kp = kp M_ii, Kd = kd M_ii, evaluated at the end-of-substep velocity.
  if (l == 0) {
    for (int i = 0; i < D; ++i) {
      const R mii = Mt[i * Dm + i];
      const R kp = M.kp[i] * mii, kd = M.kd[i] * mii, dmp = M.damping[i], fl = M.flim[i];
      const R qi = E[Y.q + i], qdi = E[Y.qd + i];
      Mt[i * Dm + i] = mii + (dt * (kd + dmp) + (dt * dt) * kp);
      R tau = kp * ((E[Y.tgt + i] - qi) - dt * qdi) + kd * (E[Y.tgtv + i] - qdi);
      tau = fmin(fmax(tau, -fl), fl) - dmp * qdi;
      cb[i] = tau - cb[i];
    }
    for (int j = 0; j < D; ++j) {
      R s = Mt[j * Dm + j];
      for (int k = 0; k < j; ++k) s -= Mt[j * Dm + k] * Mt[j * Dm + k];
      const R inv = rsqrt(s);
      Mt[j * Dm + j] = inv;  // keep 1 / L_jj
      for (int i = j + 1; i < D; ++i) {
        R t = Mt[i * Dm + j];
        for (int k = 0; k < j; ++k) t -= Mt[i * Dm + k] * Mt[j * Dm + k];
        Mt[i * Dm + j] = t * inv;
      }
    }
  }
  __syncwarp();
  BS_TICK(8);
  // ---- G: columns of M^-1 (lanes j < D) and the unconstrained velocity (lane D)
  #pragma unroll 1
  for (int j = l; j <= D; j += G) {
    R x[MD];
#pragma unroll
    for (int i = 0; i < MD; ++i) x[i] = j < D ? (i == j ? 1.0 : 0.0) : (i < D ? cb[i] : 0.0);
#pragma unroll
    for (int i = 0; i < MD; ++i) {
      if (i < D) {
        R t = x[i];
#pragma unroll
        for (int k = 0; k < i; ++k) t -= Mt[i * Dm + k] * x[k];
        x[i] = t * Mt[i * Dm + i];
      }
    }
#pragma unroll
    for (int i = MD - 1; i >= 0; --i) {
      if (i < D) {
        R t = x[i];
#pragma unroll
        for (int k = i + 1; k < MD; ++k)
          if (k < D) t -= Mt[k * Dm + i] * x[k];
        x[i] = t * Mt[i * Dm + i];
      }
    }
    if (j < D) {
#pragma unroll
      for (int i = 0; i < MD; ++i)
        if (i < D) Minv[i * Dm + j] = x[i];
    } else {
#pragma unroll
      for (int i = 0; i < MD; ++i)
        if (i < D) E[Y.u + i] = E[Y.qd + i] + dt * x[i];
    }
  }
  BS_TICK(9);
  // ---- H: broadphase + narrowphase into fixed per-pair candidate slots (A-5)
  R* cand = E + Y.rows;  // candidates alias the (not yet built) row storage
  const R slop = P.slop;
  #pragma unroll 1
  for (int s = l; s < Y.Cm; s += G) cand[8 * s + 7] = -1.0;
  __syncwarp();
  int unsup = 0;
  #pragma unroll 1
  for (int pi = l; pi < M.P; pi += G) {
    unsup += narrow_pair(M, pi, spq, slop, cand + 8 * M.p_slot[pi]);
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) unsup += __shfl_xor_sync(FULLMASK, unsup, o);
  unsupported = unsup;
  __syncwarp();
  BS_TICK(10);
  // ---- I: ordered compaction of the valid slots (ballot + popc within the group)
  R* ct = E + Y.ct;
  {
    int base = 0;
    const unsigned gmask = G == 32 ? FULLMASK : ((1u << G) - 1u);
    for (int k = 0; k < Y.KCH; ++k) {
      const int s = k * G + l;
      const bool v = s < Y.Cm && cand[8 * s + 7] >= 0.0;
      const unsigned bal = (__ballot_sync(FULLMASK, v) >> (g * G)) & gmask;
      if (v) {
        const int pos = base + __popc(bal & ((1u << l) - 1u));
#pragma unroll
        for (int j = 0; j < 8; ++j) ct[8 * pos + j] = cand[8 * s + j];
      }
      base += __popc(bal);
    }
    nc = base;
  }
  __syncwarp();
  BS_TICK(11);
  // ---- J: constraint rows.  One lane per (contact, row): the normal and the two tangent rows of
  //         a contact are built by different lanes (shared slots, lever arms and chain walk);
  //         every lane recomputes the contact's tangent basis, so the rows stay independent.
  R* rows = E + Y.rows;
  const int NU = K::EXACT ? K::NU : Y.NU, RW = ROW_J + 2 * NU;
  #pragma unroll 1
  for (int item = l; item < 3 * nc; item += G) {
    const int c = item / 3, t = item - 3 * c;
    const R* cc = ct + 8 * c;
    const V3<R> Pc = ld3(cc), n = ld3(cc + 3);
    const R depth = cc[6];
    const int pi = (int)cc[7];
    V3<R> dir;
    {  // tangent basis (A-6): t1 = normalize(n x e_k), e_k the least-aligned axis; t2 = n x t1
      int k = 0;  // (selects, not an indexed array: no local-memory round trip per row)
      R amin = fabs(n.x);
      if (fabs(n.y) < amin) { k = 1; amin = fabs(n.y); }
      if (fabs(n.z) < amin) k = 2;
      V3<R> t1 = crs(n, v3(k == 0, k == 1, k == 2));
      t1 = scl(t1, rsqrt(dot(t1, t1)));
      dir = t == 0 ? n : (t == 1 ? t1 : crs(n, t1));
    }
    R* rt = rows + (3 * c + t) * RW;
    // the joint-rate block of J accumulates in registers (written once, with W, below); only
    // the actor block of the row is cleared in shared memory first
    for (int k = JI(Dm); k < RW; k += 2) *reinterpret_cast<double2*>(rt + k) = make_double2(0.0, 0.0);
    R Jq[MD];
#pragma unroll
    for (int i = 0; i < MD; ++i) Jq[i] = 0.0;
    const int slots[2] = {M.p_i[pi], M.p_j[pi]};
    R Kc = 0.0;
    for (int s = 0; s < 2; ++s) {
      const R sg = s ? -1.0 : 1.0;
      const int sl = slots[s], bt = M.s_btype[sl], bi = M.s_body[sl];
      if (bt == BS_BODY_LINK && !M.grounded[bi]) {
        for (int kk = bi; kk >= 0; kk = M.parent[kk]) {
          if (M.jtype[kk] == BS_JOINT_FIXED) continue;
          const V3<R> col = add(ld3(Sv + 6 * kk + 3), crs(ld3(Sv + 6 * kk), Pc));
          const R v = sg * dot(dir, col);
          const int d = M.dof[kk];
#pragma unroll
          for (int i = 0; i < MD; ++i)
            if (i == d) Jq[i] += v;
        }
      } else if (bt == BS_BODY_ACTOR) {
        const int ub = Dm + 6 * bi;
        const R invm = 1.0 / M.a_mass[bi];
        const V3<R> lever = sub(Pc, ld3(E + Y.apose + 7 * bi));
        const R* Iw = E + Y.Iwi + 9 * bi;
        const V3<R> Jv = scl(dir, sg);
        const V3<R> Jw = scl(crs(lever, dir), sg);
        const V3<R> Wv = scl(Jv, invm);
        const V3<R> Ww = m3mul(Iw, Jw);
        *reinterpret_cast<double2*>(rt + JI(ub + 0)) = make_double2(Jv.x, Wv.x);
        *reinterpret_cast<double2*>(rt + JI(ub + 1)) = make_double2(Jv.y, Wv.y);
        *reinterpret_cast<double2*>(rt + JI(ub + 2)) = make_double2(Jv.z, Wv.z);
        *reinterpret_cast<double2*>(rt + JI(ub + 3)) = make_double2(Jw.x, Ww.x);
        *reinterpret_cast<double2*>(rt + JI(ub + 4)) = make_double2(Jw.y, Ww.y);
        *reinterpret_cast<double2*>(rt + JI(ub + 5)) = make_double2(Jw.z, Ww.z);
        Kc += dot(dir, dir) * invm + dot(Jw, Ww);
      }
    }
    R KA = 0.0;
#pragma unroll
    for (int i = 0; i < MD; ++i) {
      if (i < Dm) {
        R w = 0.0;
        if (i < D) {
#pragma unroll
          for (int k = 0; k < MD; ++k)
            if (k < D) w += Minv[i * Dm + k] * Jq[k];
        }
        *reinterpret_cast<double2*>(rt + JI(i)) = make_double2(Jq[i], w);
        KA += Jq[i] * w;
      }
    }
    Kc = KA + Kc;
    const R tp = depth > slop ? P.beta * (depth - slop) / dt : (depth >= 0.0 ? 0.0 : depth / dt);
    const R tv = depth < 0.0 ? depth / dt : 0.0;
    *reinterpret_cast<double2*>(rt) = make_double2(Kc > 1e-12 ? 1.0 / Kc : 0.0, 0.0);
    *reinterpret_cast<double2*>(rt + 2) = make_double2(tp, tv);
  }
  __syncwarp();
  BS_TICK(12);

  // ---- K: projected Gauss-Seidel, sequential row order.
  constexpr int NUM = K::NU;
  const int iters = P.pos_iters + P.vel_iters;
  const int nrows = 3 * nc;
  const R mu = P.friction;
  if constexpr (NUM <= 12) {
    // Small u (PickCube-style scenes): every lane of the group holds all of u in registers and
    // evaluates each row redundantly, so a row is a register dot product, the multiplier
    // update and a register axpy -- no shuffles on the dependency chain.  The sweep walks one
    // contact (normal, t1, t2) per iteration with the friction bound in a register; the
    // multipliers are stored after the three rows, so the loads of all three rows can issue
    // ahead of the first row's chain.  The warp's groups sweep in lockstep to the largest
    // contact count of the warp (rows past an env's own count are predicated off; their W was
    // zeroed here), so the sweep has no divergent control flow.
    int ncw = nc;
#pragma unroll
    for (int o = G; o < 32; o <<= 1) ncw = max(ncw, __shfl_xor_sync(FULLMASK, ncw, o));
    BS_COUNT(20, nc);
    BS_COUNT(21, ncw);
    #pragma unroll 1
    for (int r = nrows; r < 3 * ncw; ++r)
      for (int k = l; k < NU; k += G) rows[r * RW + WI(k)] = 0.0;
    __syncwarp();
    R u[NUM];
#pragma unroll
    for (int j = 0; j < NUM; ++j) u[j] = j < NU ? E[Y.u + j] : 0.0;
    for (int it = 0; it < iters; ++it) {
      const int tsel = it < P.pos_iters ? 2 : 3;  // position- or velocity-phase target
      #pragma unroll 1
      for (int c = 0; c < ncw; ++c) {
        R* r0 = rows + 3 * c * RW;
        const bool live = c < nc;
        R Jc[3][NUM], Wc[3][NUM], invK[3], old[3], nw[3];
        bool act[3];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const R* rt = r0 + t * RW;
          const double2 h = *reinterpret_cast<const double2*>(rt);
          invK[t] = h.x;
          old[t] = h.y;
          act[t] = live && invK[t] != 0.0;
#pragma unroll
          for (int j = 0; j < NUM; ++j) {
            const double2 jw = j < NU ? *reinterpret_cast<const double2*>(rt + JI(j)) : make_double2(0.0, 0.0);
            Jc[t][j] = jw.x;
            Wc[t][j] = jw.y;
          }
        }
        const R tgt = r0[tsel];
        R bound = 0.0;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          R a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
          for (int j = 0; j < NUM; j += 3) {
            a0 = fma(Jc[t][j], u[j], a0);
            if (j + 1 < NUM) a1 = fma(Jc[t][j + 1], u[j + 1], a1);
            if (j + 2 < NUM) a2 = fma(Jc[t][j + 2], u[j + 2], a2);
          }
          const R v = (a0 + a1) + a2;
          if (t == 0) {
            const R x = old[0] + (tgt - v) * invK[0];
            nw[0] = x > 0.0 ? x : 0.0;
            bound = mu * (act[0] ? nw[0] : old[0]);
          } else {
            const R x = old[t] - v * invK[t];
            nw[t] = x < -bound ? -bound : (x > bound ? bound : x);
          }
          const R delta = act[t] ? nw[t] - old[t] : 0.0;
#pragma unroll
          for (int j = 0; j < NUM; ++j) u[j] = fma(delta, Wc[t][j], u[j]);
        }
        __syncwarp();  // every lane has read the contact's multipliers (WAR)
#pragma unroll
        for (int t = 0; t < 3; ++t)
          if (act[t]) r0[t * RW + 1] = nw[t];  // every lane stores the same value
        __syncwarp();  // the stores are visible to every lane's next read of the row (RAW)
      }
    }
    __syncwarp();  // every lane has read u from E before lane 0 overwrites it
#pragma unroll
    for (int j = 0; j < NUM; ++j)
      if (l == 0 && j < NU) E[Y.u + j] = u[j];
  } else {
    // Larger u: the velocity vector lives on PL lanes of the group (lane l < PL owns u[l],
    // u[l+PL], ...); each row is a lane-local partial dot, a log2(PL)-level shuffle all-reduce,
    // the multiplier update and a lane-local axpy.
    constexpr int PL = NUM <= 20 ? 4 : 8, KP = (NUM + PL - 1) / PL;
    const unsigned gmask = (G == 32 ? FULLMASK : ((1u << G) - 1u)) << (g * G);
    const bool owner = l < PL;
    R u[KP];
#pragma unroll
    for (int j = 0; j < KP; ++j) {
      const int k = l + PL * j;
      u[j] = owner && k < NU ? E[Y.u + k] : 0.0;
    }
    for (int it = 0; it < iters; ++it) {
      const bool pos_phase = it < P.pos_iters;
      R n_invK = 0.0, n_old = 0.0, n_tgt = 0.0, n_J[KP], n_W[KP];
#pragma unroll
      for (int j = 0; j < KP; ++j) { n_J[j] = 0.0; n_W[j] = 0.0; }
      if (nrows) {
        const R* rw = rows;
        n_invK = rw[0]; n_old = rw[1]; n_tgt = pos_phase ? rw[2] : rw[3];
#pragma unroll
        for (int j = 0; j < KP; ++j) {
          const int k = l + PL * j;
          if (owner && k < NU) { n_J[j] = rw[JI(k)]; n_W[j] = rw[WI(k)]; }
        }
      }
      R lam_n = 0.0;
      int rr = 0;
      for (int r = 0; r < nrows; ++r) {
        const R invK = n_invK, old = n_old, tgt = n_tgt;
        R Jc[KP], Wc[KP];
#pragma unroll
        for (int j = 0; j < KP; ++j) { Jc[j] = n_J[j]; Wc[j] = n_W[j]; }
        R* row = rows + r * RW;
        if (r + 1 < nrows) {  // prefetch the next row
          const R* rw = row + RW;
          n_invK = rw[0]; n_old = rw[1]; n_tgt = pos_phase ? rw[2] : rw[3];
#pragma unroll
          for (int j = 0; j < KP; ++j) {
            const int k = l + PL * j;
            if (owner && k < NU) { n_J[j] = rw[JI(k)]; n_W[j] = rw[WI(k)]; }
          }
        }
        if (invK != 0.0) {
          R v0 = 0.0, v1 = 0.0;
#pragma unroll
          for (int j = 0; j < KP; j += 2) {
            v0 += Jc[j] * u[j];
            if (j + 1 < KP) v1 += Jc[j + 1] * u[j + 1];
          }
          R v = v0 + v1;
#pragma unroll
          for (int o = PL / 2; o > 0; o >>= 1) v += __shfl_xor_sync(gmask, v, o);
          R nw;
          if (rr == 0) {
            nw = fmax(old + (tgt - v) * invK, 0.0);
            lam_n = nw;
          } else {
            const R bound = mu * lam_n;
            nw = fmin(fmax(old + (0.0 - v) * invK, -bound), bound);
          }
          const R delta = nw - old;
          __syncwarp(gmask);  // the group's lanes have read this row's multiplier (WAR)
          if (owner) row[1] = nw;  // owner lanes store the same value
          __syncwarp(gmask);  // visible to the group's next read of the row (RAW)
#pragma unroll
          for (int j = 0; j < KP; ++j) u[j] += delta * Wc[j];
        } else if (rr == 0) {
          lam_n = old;
        }
        rr = rr == 2 ? 0 : rr + 1;
      }
    }
#pragma unroll
    for (int j = 0; j < KP; ++j) {
      const int k = l + PL * j;
      if (owner && k < NU) E[Y.u + k] = u[j];
    }
  }
  __syncwarp();
  BS_TICK(13);

  // ---- L: semi-implicit Euler, joint limits (A-7), actor orientation (A-8), divergence
  //         freeze.  Every lane evaluates the (small) update from the
  //         shared u; lanes then write disjoint entries.
  R q1[MD], qd1[MD];
  bool finite = true;
#pragma unroll
  for (int i = 0; i < MD; ++i) {
    if (i < D) {
      const R ui = E[Y.u + i];
      R v = E[Y.q + i] + dt * ui;
      R w = ui;
      const R lo = M.lower[i], hi = M.upper[i];
      if (v < lo) { v = lo; w = fmax(w, 0.0); }
      else if (v > hi) { v = hi; w = fmin(w, 0.0); }
      q1[i] = v;
      qd1[i] = w;
      finite &= isfinite(v) && isfinite(w);
    }
  }
  V3<R> ap1[MA], uva[MA], uwa[MA];
  Q4<R> aq1[MA];
#pragma unroll
  for (int a = 0; a < MA; ++a) {
    if (a < A) {
      R blk[6];
#pragma unroll
      for (int j = 0; j < 6; ++j) blk[j] = E[Y.u + Dm + 6 * a + j];
      uva[a] = v3(blk[0], blk[1], blk[2]);
      uwa[a] = v3(blk[3], blk[4], blk[5]);
      const V3<R> ap = ld3(E + Y.apose + 7 * a);
      const Q4<R> aq = ld4(E + Y.apose + 7 * a + 3);
      ap1[a] = v3(ap.x + uva[a].x * dt, ap.y + uva[a].y * dt, ap.z + uva[a].z * dt);
      const Q4<R> wq = quat_mul(Q4<R>{0.0, uwa[a].x, uwa[a].y, uwa[a].z}, aq);
      const R h = 0.5 * dt;
      aq1[a] = qnorm_f(Q4<R>{aq.w + h * wq.w, aq.x + h * wq.x, aq.y + h * wq.y, aq.z + h * wq.z});
      {  // carry the world angular momentum to the new orientation (A-8):
         // w' = I_w(q')^-1 I_w(q) w = R' (I_b^-1 . (R'^T R (I_b . (R^T w))))
        const R* Ib = M.a_inertia + 3 * a;
        R r0[9], r1[9];
        quat_to_matrix(aq, r0);
        quat_to_matrix(aq1[a], r1);
        const V3<R> w = uwa[a];
        const V3<R> wb{r0[0] * w.x + r0[3] * w.y + r0[6] * w.z, r0[1] * w.x + r0[4] * w.y + r0[7] * w.z,
                       r0[2] * w.x + r0[5] * w.y + r0[8] * w.z};
        const V3<R> Lb{Ib[0] * wb.x, Ib[1] * wb.y, Ib[2] * wb.z};
        const V3<R> L{r0[0] * Lb.x + r0[1] * Lb.y + r0[2] * Lb.z, r0[3] * Lb.x + r0[4] * Lb.y + r0[5] * Lb.z,
                      r0[6] * Lb.x + r0[7] * Lb.y + r0[8] * Lb.z};
        const V3<R> L1{(r1[0] * L.x + r1[3] * L.y + r1[6] * L.z) / Ib[0],
                       (r1[1] * L.x + r1[4] * L.y + r1[7] * L.z) / Ib[1],
                       (r1[2] * L.x + r1[5] * L.y + r1[8] * L.z) / Ib[2]};
        uwa[a] = v3(r1[0] * L1.x + r1[1] * L1.y + r1[2] * L1.z, r1[3] * L1.x + r1[4] * L1.y + r1[5] * L1.z,
                    r1[6] * L1.x + r1[7] * L1.y + r1[8] * L1.z);
      }
      finite &= isfinite(ap1[a].x) && isfinite(ap1[a].y) && isfinite(ap1[a].z);
      finite &= isfinite(aq1[a].w) && isfinite(aq1[a].x) && isfinite(aq1[a].y) && isfinite(aq1[a].z);
#pragma unroll
      for (int j = 0; j < 6; ++j) finite &= isfinite(blk[j]);
    }
  }
  __syncwarp();  // every lane has read q / actor poses before any lane overwrites them
  if (!finite) diverged = true;
  if (!diverged) {
#pragma unroll
    for (int i = 0; i < MD; ++i)
      if (i < D && (i % G) == l) { E[Y.q + i] = q1[i]; E[Y.qd + i] = qd1[i]; }
#pragma unroll
    for (int a = 0; a < MA; ++a)
      if (a < A && (a % G) == l) {
        st7(E + Y.apose + 7 * a, ap1[a], aq1[a]);
        st3(E + Y.avel + 6 * a, uva[a]);
        st3(E + Y.avel + 6 * a + 3, uwa[a]);
      }
  }
  __syncwarp();
  BS_TICK(14);
}

// The state observation of the env staged in E (group lanes cooperate).  Layout (DESIGN.md
// "State observation"): q[D_max] qd[D_max] ee_p[3], per actor slot p[3] q[4] v[3] w[3],
// goal[3], zero padding; CartpoleBalance: (x, x_dot, theta, theta_dot).
template <int G>
__device__ __forceinline__ void pack_state_obs(const Model& M, const BsSimParams& P, const Lay& Y, const R* E,
                                               float* o, int obs_dim, int Dm, int Ag, int l) {
  const R* lpq = E + Y.lpq;
  const int b_ee = 2 * Dm, b_act = b_ee + 3, b_goal = b_act + 13 * Ag;
  const bool cart = P.task == BS_TASK_CARTPOLE;
  #pragma unroll 1
  for (int k = l; k < obs_dim; k += G) {
    R v = 0.0;
    if (cart) v = k < 4 ? E[(k & 1 ? Y.qd : Y.q) + (k >> 1)] : 0.0;
    else if (k < Dm) v = k < M.D ? E[Y.q + k] : 0.0;
    else if (k < b_ee) v = (k - Dm) < M.D ? E[Y.qd + k - Dm] : 0.0;
    else if (k < b_act) v = P.ee_link >= 0 ? lpq[7 * P.ee_link + (k - b_ee)] : 0.0;
    else if (k < b_goal) {
      const int a = (k - b_act) / 13, j = (k - b_act) - 13 * a;
      if (a < M.A) v = j < 7 ? E[Y.apose + 7 * a + j] : E[Y.avel + 6 * a + (j - 7)];
    } else if (k < b_goal + 3) v = E[Y.goal + (k - b_goal)];
    o[k] = (float)v;
  }
}

// ------------------------------------------------------------------ the kernel
template <class K>
__global__ void __launch_bounds__(32) k_step(const __grid_constant__ BsModelTables T, const __grid_constant__ BsEnvState S,
                                             const __grid_constant__ BsStepOutputs O, const __grid_constant__ BsSimParams P,
                                             const float* __restrict__ action, const __grid_constant__ Lay Y) {
  constexpr int G = K::G, MD = K::MD, MA = K::MA, EPW = K::EPW;
  extern __shared__ double smem[];
  const int lane = threadIdx.x;
  const int g = lane / G, l = lane - g * G;
  const int e_raw = blockIdx.x * EPW + g;
  const bool live = e_raw < S.num_envs;
  const int e = live ? e_raw : S.num_envs - 1;  // idle groups shadow the last env, never store
  R* E = smem + g * Y.total;
  BS_CTA_BEGIN;
  const Model M = model_of(T, S.model_id[e]);
  // the env's scalar state is read here, at entry, so its (cold-L2) misses overlap the staging
  // instead of stalling the epilogue
  const bool div_in = S.diverged[e] != 0;
  const int32_t el_in = S.elapsed[e], tdof_in = S.target_dof[e];
  const double ret_in = S.ep_return ? S.ep_return[e] : 0.0;
  const uint8_t epf_in = S.ep_return ? S.ep_flags[e] : 0;
  // Am: the solver's actor block (smem staging, u, rows) = A_dyn; Ag: the actor stride of the
  // global state rows and of the obs layout = A_max (A_dyn <= A_max)
  const int Dm = K::EXACT ? MD : Y.Dm, Am = K::EXACT ? MA : Y.Am, Ag = K::EXACT ? MA : T.A_max;
  BS_TICK(0);

  // ---- stage the env's state rows
  #pragma unroll 1
  for (int i = l; i < Dm; i += G) {
    E[Y.q + i] = S.qpos[(int64_t)e * Dm + i];
    E[Y.qd + i] = S.qvel[(int64_t)e * Dm + i];
  }
  #pragma unroll 1
  for (int i = l; i < 7 * Am; i += G) E[Y.apose + i] = S.actor_pose[(int64_t)e * 7 * Ag + i];
  #pragma unroll 1
  for (int i = l; i < 6 * Am; i += G) E[Y.avel + i] = S.actor_vel[(int64_t)e * 6 * Ag + i];
  if (l < 3) E[Y.goal + l] = S.goal[3 * (int64_t)e + l];
  // ---- controller: drive targets, once per control step
  const float* act = action + (int64_t)e * P.action_dim;
  if (P.ctrl_mode == BS_CTRL_PD_EE_DELTA_POSE) {
    // DLS IK: twist = (a[0:3] * scale, a[3:6] * rot_scale), world frame, at
    // the ee origin; dq = J^T (J J^T + lam^2 I)^-1 twist over the controlled dofs.
    __syncwarp();
    fk_group<G>(M, Y, E, l);
    if (l == 0) ee_delta_targets(M, P, Y, E, act);
  } else if (P.ctrl_mode == BS_CTRL_BASE_FORWARD_ROTATE) {
    // mobile base: controlled dofs 0, 1, 2 = base x, y, yaw, driven
    // kinematically through VELOCITY targets: the action (forward, rotate) in [-1, 1] becomes
    // (a0 s cos(yaw), a0 s sin(yaw), a1 s_rot) m/s, m/s, rad/s; the position targets stay at q
    // (the base dofs carry kp = 0, a pure velocity servo)
    __syncwarp();  // E[q] is staged by the other lanes
    if (l == 0) {
      int bd[3] = {-1, -1, -1};
      for (int d = 0; d < M.D; ++d) {
        const int c = M.ctrl[d];
        if (c == 0) bd[0] = d; else if (c == 1) bd[1] = d; else if (c == 2) bd[2] = d;
      }
      const R a0 = fmin(fmax((R)act[0], -1.0), 1.0), a1 = fmin(fmax((R)act[1], -1.0), 1.0);
      const R yaw = bd[2] >= 0 ? E[Y.q + bd[2]] : 0.0;
      R sy, cy;
      sincos(yaw, &sy, &cy);
      for (int d = 0; d < M.D; ++d) { E[Y.tgt + d] = E[Y.q + d]; E[Y.tgtv + d] = 0.0; }
      const R v = a0 * P.action_scale;
      if (bd[0] >= 0) E[Y.tgtv + bd[0]] = v * cy;
      if (bd[1] >= 0) E[Y.tgtv + bd[1]] = v * sy;
      if (bd[2] >= 0) E[Y.tgtv + bd[2]] = a1 * P.action_scale_rot;
    }
  } else {
    #pragma unroll 1
    for (int i = l; i < M.D; i += G) {
      const int ai = M.ctrl[i];
      const R qi = S.qpos[(int64_t)e * Dm + i];
      R tgt = qi, tgtv = 0.0;
      if (ai >= 0) {
        const R a = fmin(fmax((R)act[ai], -1.0), 1.0);
        const R lo = M.lower[i], hi = M.upper[i];
        if (P.ctrl_mode == BS_CTRL_PD_JOINT_DELTA_POS) {
          tgt = fmin(fmax(qi + a * P.action_scale, lo), hi);
          tgtv = (tgt - qi) * P.control_freq;  // the delta is a motion over one control period
        } else {
          const R un = (isfinite(lo) && isfinite(hi)) ? lo + (a + 1.0) * 0.5 * (hi - lo) : a * P.action_scale;
          tgt = fmin(fmax(un, lo), hi);
        }
      }
      E[Y.tgt + i] = tgt;
      E[Y.tgtv + i] = tgtv;
    }
  }
  bool diverged = div_in;
  __syncwarp();
  BS_TICK(1);

  int unsupported = 0, nc = 0;
  for (int s = 0; s < P.substeps; ++s) {
    substep<K>(M, P, Y, E, l, g, diverged, unsupported, nc);
    if (s == P.substeps - 1 && O.contact_count && live) {  // ContactSet of the last substep
      const R* ct = E + Y.ct;
      #pragma unroll 1
      for (int c = l; c < nc && c < T.C_max; c += G) {
        const int64_t o = (int64_t)e * T.C_max + c;
        const int pi = (int)ct[8 * c + 7];
        if (O.contact_pairs) { O.contact_pairs[2 * o] = M.p_i[pi]; O.contact_pairs[2 * o + 1] = M.p_j[pi]; }
        if (O.contact_geom) {
#pragma unroll
          for (int j = 0; j < 7; ++j) O.contact_geom[7 * o + j] = ct[8 * c + j];
        }
      }
      if (l == 0) O.contact_count[e] = nc;
    }
  }
  __syncwarp();  // the contact export reads the compacted contacts that the FK scratch aliases
  fk_group<G>(M, Y, E, l);
  BS_TICK(15);

  // ---- task evaluation; every lane evaluates (cheap, uniform)
  const R* lpq = E + Y.lpq;
  float reward = 0.0f;
  bool success = false, fail = diverged;
  int32_t tdof = tdof_in;
  if (P.task == BS_TASK_PICKCUBE) {
    const R* f = P.task_f;
    const V3<R> ee = ld3(lpq + 7 * P.ee_link);
    const V3<R> cube = ld3(E + Y.apose);
    const R d_ee = dist3(ee, cube);
    const R d_goal = dist3(v3(cube.x, cube.y, 0.0), v3(E[Y.goal], E[Y.goal + 1], 0.0));
    success = d_goal < f[4];
    fail = cube.z < f[5] || diverged;
    reward = (float)(-__dadd_rn(d_ee, d_goal));
  } else if (P.task == BS_TASK_OPENCHAIN) {
    const R hi = tdof >= 0 ? M.upper[tdof] : 1.0;
    const R qv = tdof >= 0 ? E[Y.q + tdof] : 0.0;
    success = tdof >= 0 && qv > P.task_f[1] * hi;
    reward = (float)(tdof >= 0 ? qv / hi : 0.0);
  } else if (P.task == BS_TASK_CARTPOLE) {
    const R x = E[Y.q], th = E[Y.q + 1];
    tdof = fabs(th) < P.task_f[1] ? tdof + 1 : 0;  // upright streak (control steps)
    success = tdof >= (int32_t)P.task_f[2];
    fail = fabs(th) > P.task_f[3] || fabs(x) > P.task_f[4] || diverged;
    reward = (float)cos(th);
  }
  int32_t el = el_in + 1;
  const bool terminated = P.early_termination ? (success || fail) : false;
  const bool truncated = el >= P.max_steps;
  if (live && l == 0) {
    O.reward[e] = reward;
    O.terminated[e] = terminated;
    O.truncated[e] = truncated;
    O.success[e] = success;
    O.fail[e] = fail;
    O.unsupported_pairs[e] = unsupported;
    if (P.task == BS_TASK_CARTPOLE) S.target_dof[e] = tdof;
    // EpisodeMetrics: return = sum of rewards, *_once latch, *_at_end
    // sampled at the final step; emitted when the episode ends, accumulators restart.
    if (S.ep_return) {
      const double ret = ret_in + (double)reward;
      const uint8_t fl = epf_in | (success ? 1 : 0) | (fail ? 2 : 0);
      const bool ended = terminated || truncated;
      if (O.ep_done) {
        O.ep_done[e] = ended;
        if (ended) {
          O.ep_return_out[e] = ret;
          O.ep_length_out[e] = el;
          O.ep_flags_out[e] = (fl & 1) | (success ? 2 : 0) | ((fl & 2) << 1) | (fail ? 8 : 0);
        }
      }
      S.ep_return[e] = ended ? 0.0 : ret;
      S.ep_flags[e] = ended ? 0 : fl;
    }
  }
  // ---- in-kernel auto-reset from the env's Philox stream
  const bool done = live && P.auto_reset && (terminated || truncated);
  // the observation of the state the episode ENDED in, before the reset replaces it (lets a
  // learner bootstrap V(s_T) on time-limit truncations)
  if (done && O.final_obs) pack_state_obs<G>(M, P, Y, E, O.final_obs + (int64_t)e * O.obs_dim, O.obs_dim, Dm, Ag, l);
  uint8_t div_out = diverged;
  if (__any_sync(FULLMASK, done)) {
    __syncwarp();  // the group's final_obs reads of E above precede lane 0's reset writes (WAR)
    if (done && l == 0) {
      const uint32_t rc = (uint32_t)S.reset_count[e] + 1u;
      S.reset_count[e] = rc;
      R q[MD], qd[MD], goal[3];
      V3<R> ap[MA], av[MA], aw[MA];
      Q4<R> aq[MA];
      task_reset(M, P, S.env_offset + e, rc, q, qd, ap, aq, av, aw, goal, &tdof);
      S.target_dof[e] = tdof;
      for (int i = 0; i < M.D; ++i) { E[Y.q + i] = q[i]; E[Y.qd + i] = qd[i]; }
      for (int a = 0; a < M.A; ++a) {
        st7(E + Y.apose + 7 * a, ap[a], aq[a]);
        st3(E + Y.avel + 6 * a, av[a]);
        st3(E + Y.avel + 6 * a + 3, aw[a]);
      }
      for (int k = 0; k < 3; ++k) E[Y.goal + k] = goal[k];
    }
    if (done) { el = 0; div_out = 0; }
    __syncwarp();
    fk_group<G>(M, Y, E, l);
  }
  BS_TICK(16);
  if (!live) return;
  // ---- write back the state rows, the FK cache and the state observation
  #pragma unroll 1
  for (int i = l; i < Dm; i += G) {
    S.qpos[(int64_t)e * Dm + i] = E[Y.q + i];
    S.qvel[(int64_t)e * Dm + i] = E[Y.qd + i];
    if (i < M.D) S.target[(int64_t)e * Dm + i] = E[Y.tgt + i];
  }
  #pragma unroll 1
  for (int i = l; i < 7 * M.A; i += G) S.actor_pose[(int64_t)e * 7 * Ag + i] = E[Y.apose + i];
  #pragma unroll 1
  for (int i = l; i < 6 * M.A; i += G) S.actor_vel[(int64_t)e * 6 * Ag + i] = E[Y.avel + i];
  if (l < 3) S.goal[3 * (int64_t)e + l] = E[Y.goal + l];
  #pragma unroll 1
  for (int i = l; i < 7 * M.L; i += G) S.link_pose[(int64_t)e * 7 * Y.Lm + i] = lpq[i];
  if (l == 0) {
    S.elapsed[e] = el;
    S.diverged[e] = div_out;
  }
  if (O.obs) {
    if ((blockIdx.x + 1) * EPW <= S.num_envs) {
      // every group of the warp is live: stage the EPW envs' observations (consecutive rows of
      // O.obs) in the dead constraint-row scratch, then write them as one contiguous run --
      // full 128-byte lines instead of EPW short segments (these are PCIe writes when the obs
      // buffer is pinned host memory, Env.step_host)
      float* stg = reinterpret_cast<float*>(E + Y.rows);
      pack_state_obs<G>(M, P, Y, E, stg, O.obs_dim, Dm, Ag, l);
      __syncwarp();
      const int od = O.obs_dim, n = EPW * od;
      float* dst = O.obs + (int64_t)blockIdx.x * EPW * od;
      #pragma unroll 1
      for (int f = lane; f < n; f += 32) {
        const int gg = f / od;
        dst[f] = reinterpret_cast<const float*>(smem + gg * Y.total + Y.rows)[f - gg * od];
      }
    } else {
      pack_state_obs<G>(M, P, Y, E, O.obs + (int64_t)e * O.obs_dim, O.obs_dim, Dm, Ag, l);
    }
  }
  BS_TICK(17);
  BS_CTA_END;
}

// ------------------------------------------------------------------ host side
static Lay make_lay(const BsModelTables& T, int G) {
  Lay y;
  y.Dm = T.D_max; y.Lm = T.L_max; y.Sm = T.S_max; y.Cm = T.C_max;
  y.Am = T.A_dyn >= 0 && T.A_dyn < T.A_max ? T.A_dyn : T.A_max;  // solver actor block (A-dyn <= A_max)
  y.NU = y.Dm + 6 * y.Am;
  y.RW = ROW_J + 2 * y.NU;
  y.KCH = (y.Cm + G - 1) / G;
  int o = 0;
  y.q = o; o += y.Dm;
  y.qd = o; o += y.Dm;
  y.tgt = o; o += y.Dm;
  y.tgtv = o; o += y.Dm;
  y.apose = o; o += 7 * y.Am;
  y.avel = o; o += 6 * y.Am;
  y.goal = o; o += 3;
  y.lpq = o; o += 7 * y.Lm;
  y.Sv = o; o += 6 * y.Lm;
  y.Minv = o; o += y.Dm * y.Dm;
  y.u = o; o += y.Dm + 6 * y.Am;
  y.Iwi = o; o += 9 * y.Am;
  // union: {FK local transforms + RNEA temporaries} | {compacted contacts}
  const int fkr = 7 * y.Lm + 18 * y.Lm, cts = 8 * y.Cm;
  y.Tl = o; y.V = o + 7 * y.Lm; y.Ac = y.V + 6 * y.Lm; y.F = y.Ac + 6 * y.Lm;
  y.ct = o;
  o += fkr > cts ? fkr : cts;
  o += o & 1;  // rows start 16-byte aligned
  y.rows = o;
  // The row storage also holds the substep scratch that is dead before the rows are built:
  // [0, 8 C_max) the narrowphase candidate slots (H), then the shape poses (A -> H), the mass
  // matrix / Cholesky factor (A -> G), the bias forces (D -> G) and the world inertias (A -> E).
  int r = 8 * y.Cm;
  y.spq = o + r; r += 7 * y.Sm;
  y.Mt = o + r; r += y.Dm * y.Dm;
  y.cb = o + r; r += y.Dm;
  y.In = o + r; r += 10 * y.Lm;
  const int rws = 3 * y.Cm * y.RW;
  o += rws > r ? rws : r;
  o += o & 1;  // every env's block starts 16-byte aligned
  y.total = o;
  return y;
}

template <class K>
static int launch(const BsModelTables& T, const BsEnvState& S, const BsStepOutputs& O, const BsSimParams& P,
                  const float* action, cudaStream_t st) {
  Lay y = make_lay(T, K::G);
  // opt-in above 48 KB, raised on demand per device (kernel group slot 1 + variant)
  auto ensure_attr = [](size_t b) {
    return bs::ensure_smem_optin(K::SLOT, b, [](size_t v) {
      return cudaFuncSetAttribute(k_step<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v) == cudaSuccess;
    });
  };
  // Pad the per-env stride to 2 (mod 16) doubles when that costs no residency: the groups of a
  // warp then sit in distinct 16-byte bank slots for the sweep's broadcast loads.  The choice
  // is a pure function of (layout widths, kernel variant), cached per variant.
  struct StrideMemo { std::mutex mu; int key[5] = {-1, -1, -1, -1, -1}; int total = 0; };
  static StrideMemo memo;
  const int key[5] = {y.Dm, y.Lm, y.Sm, y.Cm, y.Am};
  int cached = -1;
  {
    std::lock_guard<std::mutex> g(memo.mu);
    if (memcmp(key, memo.key, sizeof(key)) == 0) cached = memo.total;
  }
  if (cached >= 0) {
    y.total = cached;
  } else {
    const int padded = y.total + ((2 - y.total % 16) + 16) % 16;
    const size_t b0 = (size_t)K::EPW * y.total * sizeof(double), b1 = (size_t)K::EPW * padded * sizeof(double);
    if (b1 <= 220 * 1024 && ensure_attr(b1)) {
      int n0 = 0, n1 = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n0, k_step<K>, 32, b0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n1, k_step<K>, 32, b1);
      if (n1 >= n0) y.total = padded;
    }
    std::lock_guard<std::mutex> g(memo.mu);
    memcpy(memo.key, key, sizeof(key));
    memo.total = y.total;
  }
  const size_t bytes = (size_t)K::EPW * y.total * sizeof(double);
  if (bytes > 220 * 1024) return BS_ERR_UNSUPPORTED;
  if (!ensure_attr(bytes)) return BS_ERR_CUDA;
  const int blocks = (S.num_envs + K::EPW - 1) / K::EPW;
  k_step<K><<<blocks, 32, bytes, st>>>(T, S, O, P, action, y);
  return launch_status();
}

typedef Cfg<8, 3, 1, true, 1> CfgPick;  // exactly ARM3 + one free actor (PickCube, PickHetero): static widths
typedef Cfg<16, 3, 1, true, 5> CfgPick16;  // the same with 16 lanes per env (small batches: idle SMs)
typedef Cfg<32, 3, 1, true, 6> CfgPick32;  // the same with a whole warp per env
typedef Cfg<8, 4, 1, false, 2> CfgSmall;    // PickCube-style: D <= 4, one free actor
typedef Cfg<8, 12, 1, false, 3> CfgArt;     // articulated objects (arm + cabinet): D <= 12, <= 1 actor
typedef Cfg<16, 12, 1, false, 7> CfgArt16;
typedef Cfg<32, 12, 1, false, 8> CfgArt32;
typedef Cfg<8, 12, 4, false, 4> CfgLarge;   // general scenes: D <= 12, <= 4 actors
typedef Cfg<8, 12, 1, false, 9, 0> CfgArt0;     // articulated objects without free actors (A_dyn = 0)
typedef Cfg<16, 12, 1, false, 10, 0> CfgArt0_16;
typedef Cfg<32, 12, 1, false, 11, 0> CfgArt0_32;

}  // namespace step
}  // namespace bs

using namespace bs::step;

extern "C" {

int bs_debug_phase_clocks(unsigned long long* out, int32_t n, int32_t reset) {
#ifdef BS_PHASE_TIMING
  if (!out || n < 0 || n > 32) return BS_ERR_ARGUMENT;
  if (cudaMemcpyFromSymbol(out, g_bs_phase, sizeof(unsigned long long) * n) != cudaSuccess) return BS_ERR_CUDA;
  if (reset) {
    unsigned long long z[32] = {0};
    if (cudaMemcpyToSymbol(g_bs_phase, z, sizeof(z)) != cudaSuccess) return BS_ERR_CUDA;
  }
  return BS_OK;
#else
  (void)out; (void)n; (void)reset;
  return BS_ERR_UNSUPPORTED;
#endif
}

int bs_step(const BsModelTables* T, const BsEnvState* S, const BsStepOutputs* O, const BsSimParams* P,
            const float* action, void* stream) {
  if (!T || !S || !O || !P || !action) return BS_ERR_ARGUMENT;
  if (S->num_envs <= 0) return BS_OK;
  if (!O->reward || !O->terminated || !O->truncated || !O->success || !O->fail || !O->unsupported_pairs)
    return BS_ERR_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static const bool generic = [] {
    const char* v = getenv("BS_STEP_GENERIC");  // tests: force the runtime-width variants
    return v && atoi(v) != 0;
  }();
  // Lanes per env (PickCube-style and articulated variants).  A launch lasts as long as its
  // slowest env's dependency chain, and small batches leave most SMSPs idle: there, 16 or 32
  // lanes per env shorten the lane-parallel phases (pairs, rows, links) at no cost in
  // residency.  Large batches keep 8 lanes (all 4096 PickCube envs resident in one wave).
  // Measured on one B200 (tools/ab_g.sh): 512 envs 62 -> 55 us (G 32), 1024 envs 64 -> 60 us
  // (G 16/32), C4 cabinets 127 -> 107 us (G 16), 4096 envs 72 us (G 8; G 16: 112 us).
  // BS_STEP_G = 8 / 16 / 32 forces a variant (tests run the parity cases on each).
  static const int gforce = [] {
    const char* v = getenv("BS_STEP_G");
    const int g = v ? atoi(v) : 0;
    return g == 8 || g == 16 || g == 32 ? g : 0;
  }();
  // per_sm: env-lanes per SM per launch that keep the step one short wave; measured per family
  // (same box, BS_STEP_G): PickCube-style 1024 envs G 8 / 16 / 32 = 66.0 / 62.9 / 60.1 us (224 ->
  // G 32), cabinets 115.2 / 96.0 / 100.7 us (112 -> G 16)
  auto lanes = [&](int n, long per_sm) {
    if (gforce) return gforce;
    const long budget = per_sm * bs::sm_count();
    return (long)n * 32 <= budget ? 32 : ((long)n * 16 <= budget ? 16 : 8);
  };
  if (!generic && T->D_max == CfgPick::MD && T->A_max == CfgPick::MA && T->A_dyn == CfgPick::MA) {
    const int g = lanes(S->num_envs, 224);
    if (g == 32) return launch<CfgPick32>(*T, *S, *O, *P, action, st);
    if (g == 16) return launch<CfgPick16>(*T, *S, *O, *P, action, st);
    return launch<CfgPick>(*T, *S, *O, *P, action, st);
  }
  if (T->D_max <= CfgSmall::MD && T->A_max <= CfgSmall::MA) return launch<CfgSmall>(*T, *S, *O, *P, action, st);
  if (T->D_max <= CfgArt0::MD && T->A_max <= CfgArt0::MA && T->A_dyn == 0) {
    const int g = lanes(S->num_envs, 112);
    if (g == 32) return launch<CfgArt0_32>(*T, *S, *O, *P, action, st);
    if (g == 16) return launch<CfgArt0_16>(*T, *S, *O, *P, action, st);
    return launch<CfgArt0>(*T, *S, *O, *P, action, st);
  }
  if (T->D_max <= CfgArt::MD && T->A_max <= CfgArt::MA) {
    const int g = lanes(S->num_envs, 112);
    if (g == 32) return launch<CfgArt32>(*T, *S, *O, *P, action, st);
    if (g == 16) return launch<CfgArt16>(*T, *S, *O, *P, action, st);
    return launch<CfgArt>(*T, *S, *O, *P, action, st);
  }
  if (T->D_max <= CfgLarge::MD && T->A_max <= CfgLarge::MA) return launch<CfgLarge>(*T, *S, *O, *P, action, st);
  return BS_ERR_UNSUPPORTED;
}

}  // extern "C"
