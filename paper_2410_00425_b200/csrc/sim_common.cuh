// Device helpers shared by the fused step (step.cu) and the reset / FK kernels (sim.cu).
// Reference semantics: pose.py:31-88 (quaternion algebra), SPEC.md:249-257 (FK)
// (reset sampling, task evaluation, state observation), DESIGN.md decisions A-15, A-17.
#pragma once
#include <math.h>
#include "bs_common.cuh"

namespace bs {
namespace sim {

typedef double R;

struct V6 { R w[3], v[3]; };

__device__ __forceinline__ V3<R> v3(R x, R y, R z) { return V3<R>{x, y, z}; }
__device__ __forceinline__ V3<R> add(V3<R> a, V3<R> b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ V3<R> sub(V3<R> a, V3<R> b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ V3<R> scl(V3<R> a, R s) { return v3(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ R dot(V3<R> a, V3<R> b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ V3<R> crs(V3<R> a, V3<R> b) { return cross3(a, b); }
__device__ __forceinline__ V3<R> ld3(const R* p) { return v3(p[0], p[1], p[2]); }
__device__ __forceinline__ void st3(R* p, V3<R> a) { p[0] = a.x; p[1] = a.y; p[2] = a.z; }
__device__ __forceinline__ Q4<R> ld4(const R* p) { return Q4<R>{p[0], p[1], p[2], p[3]}; }
__device__ __forceinline__ void st4(R* p, Q4<R> q) { p[0] = q.w; p[1] = q.x; p[2] = q.y; p[3] = q.z; }
__device__ __forceinline__ V3<R> gw(const V6& a) { return v3(a.w[0], a.w[1], a.w[2]); }
__device__ __forceinline__ V3<R> gv(const V6& a) { return v3(a.v[0], a.v[1], a.v[2]); }
__device__ __forceinline__ V6 mk6(V3<R> w, V3<R> v) { return V6{{w.x, w.y, w.z}, {v.x, v.y, v.z}}; }
__device__ __forceinline__ R dot6(const V6& a, const V6& b) {
  return dot(gw(a), gw(b)) + dot(gv(a), gv(b));
}

// Pose compose with the reference's semantics (pose.py:239-249).
__device__ __forceinline__ void compose(V3<R> pa, Q4<R> qa, V3<R> pb, Q4<R> qb, V3<R>& po, Q4<R>& qo) {
  V3<R> r = quat_rotate(qa, pb);
  po = add(pa, r);
  qo = quat_normalize(quat_mul(qa, qb));
}
__device__ __forceinline__ Q4<R> qconj(Q4<R> q) { return Q4<R>{q.w, -q.x, -q.y, -q.z}; }

// rigid-body inertia about the world origin: (m, h = m c, I_O symmetric 3x3)
struct Inertia { R m; V3<R> h; R I[6]; };  // I: xx yy zz xy xz yz

__device__ __forceinline__ V3<R> symmul(const R* I, V3<R> w) {
  return v3(I[0] * w.x + I[3] * w.y + I[4] * w.z, I[3] * w.x + I[1] * w.y + I[5] * w.z,
            I[4] * w.x + I[5] * w.y + I[2] * w.z);
}
__device__ __forceinline__ V6 imul(const Inertia& in, const V6& V) {
  V3<R> w = gw(V), v = gv(V);
  return mk6(add(symmul(in.I, w), crs(in.h, v)), sub(scl(v, in.m), crs(in.h, w)));
}
__device__ __forceinline__ V6 crossm(const V6& V, const V6& U) {
  V3<R> w = gw(V), v = gv(V);
  return mk6(crs(w, gw(U)), add(crs(w, gv(U)), crs(v, gw(U))));
}
__device__ __forceinline__ V6 crossf(const V6& V, const V6& F) {
  V3<R> w = gw(V), v = gv(V);
  return mk6(add(crs(w, gw(F)), crs(v, gv(F))), crs(w, gv(F)));
}

// Philox4x32-10 (Salmon et al. SC'11); KAT-checked against Random123 vectors.
struct U4 { uint32_t x, y, z, w; };
__device__ __forceinline__ U4 philox(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
  }
  return c;
}
__device__ __forceinline__ R u01(uint32_t a, uint32_t b) {
  uint64_t m = (uint64_t)(a >> 5) * 67108864ull + (uint64_t)(b >> 6);
  return __dmul_rn((R)m, 1.0 / 9007199254740992.0);
}
__device__ __forceinline__ R uni(R lo, R hi, R u) { return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u)); }

#define TAG_RESET 0x52455354u
#define TAG_ACTION 0x41435421u

// ----------------------------------------------------------------------------------
// Per-env view of the model tables
struct Model {
  int L, D, S, P, A;
  const int32_t *parent, *jtype, *dof, *grounded;
  const R *axis, *org, *mass, *com, *inertia;
  const R *lower, *upper, *damping, *kp, *kd, *flim;
  const int32_t* ctrl;
  const int32_t *s_btype, *s_body, *s_kind, *s_seg;
  const R *s_size, *s_frame, *s_radius;
  const int32_t *p_i, *p_j, *p_code, *p_slot;
  const R *a_mass, *a_inertia, *a_rest;
};

__device__ __forceinline__ Model model_of(const BsModelTables& T, int m) {
  Model M;
  M.L = T.n_links[m]; M.D = T.n_dof[m]; M.S = T.n_shapes[m]; M.P = T.n_pairs[m]; M.A = T.n_actors[m];
  const int lo = m * T.L_max, dd = m * T.D_max, so = m * T.S_max, po = m * T.P_max, ao = m * T.A_max;
  M.parent = T.link_parent + lo; M.jtype = T.link_jtype + lo; M.dof = T.link_dof + lo;
  M.grounded = T.link_grounded + lo;
  M.axis = T.link_axis + 3 * lo; M.org = T.link_org + 7 * lo; M.mass = T.link_mass + lo;
  M.com = T.link_com + 3 * lo; M.inertia = T.link_inertia + 6 * lo;
  M.lower = T.dof_lower + dd; M.upper = T.dof_upper + dd; M.damping = T.dof_damping + dd;
  M.kp = T.dof_kp + dd; M.kd = T.dof_kd + dd; M.flim = T.dof_flim + dd; M.ctrl = T.dof_ctrl + dd;
  M.s_btype = T.shape_btype + so; M.s_body = T.shape_body + so; M.s_kind = T.shape_kind + so;
  M.s_seg = T.shape_seg + so; M.s_size = T.shape_size + 3 * so; M.s_frame = T.shape_frame + 7 * so;
  M.s_radius = T.shape_radius + so;
  M.p_i = T.pair_i + po; M.p_j = T.pair_j + po; M.p_code = T.pair_code + po; M.p_slot = T.pair_slot + po;
  M.a_mass = T.actor_mass + ao; M.a_inertia = T.actor_inertia + 3 * ao; M.a_rest = T.actor_rest + 5 * ao;
  return M;
}

// Compile-time capacities of the thread-local scratch (host picks the instantiation).
template <int MD_, int ML_, int MS_, int MC_, int MA_>
struct Cap {
  static constexpr int MD = MD_, ML = ML_, MS = MS_, MC = MC_, MA = MA_;
};

template <class C>
struct Scratch {
  V3<R> lp[C::ML];
  Q4<R> lq[C::ML];
  V6 S[C::ML];
};

// ---------------------------------------------------------------- kinematics
template <class C>
__device__ void fk(const Model& M, const R* q, V3<R>* lp, Q4<R>* lq) {
  for (int l = 0; l < M.L; ++l) {
    const R* o = M.org + 7 * l;
    V3<R> op = ld3(o);
    Q4<R> oq = ld4(o + 3);
    int par = M.parent[l];
    if (par < 0) { lp[l] = op; lq[l] = oq; continue; }
    V3<R> jp; Q4<R> jq;
    compose(lp[par], lq[par], op, oq, jp, jq);
    int jt = M.jtype[l];
    if (jt == BS_JOINT_FIXED) { lp[l] = jp; lq[l] = jq; continue; }
    R qv = q[M.dof[l]];
    V3<R> ax = ld3(M.axis + 3 * l);
    if (jt == BS_JOINT_REVOLUTE) {
      R s, c;
      sincos(0.5 * qv, &s, &c);
      compose(jp, jq, v3(0, 0, 0), Q4<R>{c, ax.x * s, ax.y * s, ax.z * s}, lp[l], lq[l]);
    } else {
      compose(jp, jq, scl(ax, qv), Q4<R>{1, 0, 0, 0}, lp[l], lq[l]);
    }
  }
}

__device__ __forceinline__ void motion_subspace(const Model& M, const V3<R>* lp, const Q4<R>* lq, V6* S) {
  for (int l = 0; l < M.L; ++l) {
    int jt = M.jtype[l];
    if (jt == BS_JOINT_FIXED) { S[l] = V6{{0, 0, 0}, {0, 0, 0}}; continue; }
    V3<R> a = quat_rotate(lq[l], ld3(M.axis + 3 * l));
    S[l] = jt == BS_JOINT_REVOLUTE ? mk6(a, crs(lp[l], a)) : mk6(v3(0, 0, 0), a);
  }
}

__device__ __forceinline__ Inertia world_inertia(const Model& M, int l, V3<R> p, Q4<R> q) {
  R r[9];
  quat_to_matrix(q, r);
  const R* I = M.inertia + 6 * l;
  R Il[9] = {I[0], I[3], I[4], I[3], I[1], I[5], I[4], I[5], I[2]};
  R RI[9], Ic[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) RI[3 * i + j] = r[3 * i] * Il[j] + r[3 * i + 1] * Il[3 + j] + r[3 * i + 2] * Il[6 + j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Ic[3 * i + j] = RI[3 * i] * r[3 * j] + RI[3 * i + 1] * r[3 * j + 1] + RI[3 * i + 2] * r[3 * j + 2];
  V3<R> cl = ld3(M.com + 3 * l);
  V3<R> c = add(p, v3(r[0] * cl.x + r[1] * cl.y + r[2] * cl.z, r[3] * cl.x + r[4] * cl.y + r[5] * cl.z,
                      r[6] * cl.x + r[7] * cl.y + r[8] * cl.z));
  R m = M.mass[l];
  R cc = dot(c, c);
  Inertia out;
  out.m = m;
  out.h = scl(c, m);
  out.I[0] = Ic[0] + m * (cc - c.x * c.x);
  out.I[1] = Ic[4] + m * (cc - c.y * c.y);
  out.I[2] = Ic[8] + m * (cc - c.z * c.z);
  out.I[3] = Ic[1] - m * c.x * c.y;
  out.I[4] = Ic[2] - m * c.x * c.z;
  out.I[5] = Ic[5] - m * c.y * c.z;
  return out;
}


__device__ __forceinline__ void actor_world_inertia(const R* Ib, Q4<R> q, R* Iw, R* Iwinv) {
  R r[9];
  quat_to_matrix(q, r);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      R s = 0, si = 0;
      for (int k = 0; k < 3; ++k) {
        s += r[3 * i + k] * Ib[k] * r[3 * j + k];
        si += r[3 * i + k] * (1.0 / Ib[k]) * r[3 * j + k];
      }
      Iw[3 * i + j] = s;
      Iwinv[3 * i + j] = si;
    }
}
__device__ __forceinline__ V3<R> m3mul(const R* A, V3<R> x) {
  return v3(A[0] * x.x + A[1] * x.y + A[2] * x.z, A[3] * x.x + A[4] * x.y + A[5] * x.z,
            A[6] * x.x + A[7] * x.y + A[8] * x.z);
}

// ---------------------------------------------------------------- tasks
// PickCube task_f layout: 0 q_noise, 1 cube_half, 2 cube_xy, 3 goal_xy, 4 success_dist,
// 5 fail_z, 6..8 q_rest.   OpenChain task_f: 0 q_noise, 1 success_frac, 6..8 q_rest.
// Cartpole task_f: 0 init_noise, 1 success_angle, 2 success_steps, 3 fail_angle, 4 fail_x
// (dof 0 = slider, dof 1 = hinge; the per-env task integer holds the upright streak).

// Reference-order quaternion product / normalisation with every operation rounded separately
// (no FMA contraction even in FMA-enabled translation units): reset sampling must equal the
// numpy oracle bit for bit (pose.py:31-55 order).
__device__ __forceinline__ Q4<R> qmul_rn(const Q4<R>& a, const Q4<R>& b) {
  Q4<R> o;
  o.w = __dsub_rn(__dsub_rn(__dsub_rn(__dmul_rn(a.w, b.w), __dmul_rn(a.x, b.x)), __dmul_rn(a.y, b.y)), __dmul_rn(a.z, b.z));
  o.x = __dsub_rn(__dadd_rn(__dadd_rn(__dmul_rn(a.w, b.x), __dmul_rn(a.x, b.w)), __dmul_rn(a.y, b.z)), __dmul_rn(a.z, b.y));
  o.y = __dadd_rn(__dadd_rn(__dsub_rn(__dmul_rn(a.w, b.y), __dmul_rn(a.x, b.z)), __dmul_rn(a.y, b.w)), __dmul_rn(a.z, b.x));
  o.z = __dadd_rn(__dsub_rn(__dadd_rn(__dmul_rn(a.w, b.z), __dmul_rn(a.x, b.y)), __dmul_rn(a.y, b.x)), __dmul_rn(a.z, b.w));
  return o;
}
__device__ __forceinline__ Q4<R> qnorm_rn(Q4<R> q) {
  R ss = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(q.w, q.w), __dmul_rn(q.x, q.x)), __dmul_rn(q.y, q.y)), __dmul_rn(q.z, q.z));
  R n = __dsqrt_rn(ss);
  Q4<R> r{__ddiv_rn(q.w, n), __ddiv_rn(q.x, n), __ddiv_rn(q.y, n), __ddiv_rn(q.z, n)};
  R s = 0.0;
  if (s == 0.0) s = sign_like_numpy(r.w);
  if (s == 0.0) s = sign_like_numpy(r.x);
  if (s == 0.0) s = sign_like_numpy(r.y);
  if (s == 0.0) s = sign_like_numpy(r.z);
  if (s == 0.0) s = 1.0;
  return Q4<R>{__dmul_rn(r.w, s), __dmul_rn(r.x, s), __dmul_rn(r.y, s), __dmul_rn(r.z, s)};
}

static __device__ __noinline__ void task_reset(const Model M, const BsSimParams& P, int64_t genv, uint32_t rc, R* q, R* qd,
                           V3<R>* ap, Q4<R>* aq, V3<R>* av, V3<R>* aw, R* goal, int32_t* target_dof) {
  uint32_t k0 = (uint32_t)(P.seed & 0xffffffffu), k1 = (uint32_t)(P.seed >> 32);
  R u[8];
  for (int blk = 0; blk < 4; ++blk) {
    U4 r = philox(U4{(uint32_t)blk, rc, (uint32_t)genv, TAG_RESET}, k0, k1);
    u[2 * blk] = u01(r.x, r.y);
    u[2 * blk + 1] = u01(r.z, r.w);
  }
  for (int i = 0; i < M.D; ++i) { q[i] = 0.0; qd[i] = 0.0; }
  for (int a = 0; a < M.A; ++a) { av[a] = v3(0, 0, 0); aw[a] = v3(0, 0, 0); }
  if (P.task == BS_TASK_PICKCUBE) {
    const R* f = P.task_f;
    for (int i = 0; i < 3 && i < M.D; ++i) q[i] = __dadd_rn(f[6 + i], uni(-f[0], f[0], u[i]));
    R cx = uni(-f[2], f[2], u[3]), cy = uni(-f[2], f[2], u[4]);
    R yaw = uni(-M_PI, M_PI, u[5]);
    R s, c;
    sincos(0.5 * yaw, &s, &c);
    // resting pose of the object (actor_rest: height, orientation; A-26)
    const R* rest = M.a_rest;
    ap[0] = v3(cx, cy, rest[0]);
    aq[0] = qnorm_rn(Q4<R>{c, 0.0, 0.0, s});
    if (!(rest[1] == 1.0 && rest[2] == 0.0 && rest[3] == 0.0 && rest[4] == 0.0))
      aq[0] = qnorm_rn(qmul_rn(aq[0], Q4<R>{rest[1], rest[2], rest[3], rest[4]}));
    goal[0] = uni(-f[3], f[3], u[6]);
    goal[1] = uni(-f[3], f[3], u[7]);
    goal[2] = rest[0];
  } else if (P.task == BS_TASK_OPENCHAIN) {
    // arm dofs at q_rest (task_f 6..8), articulated-object dofs closed; target dof drawn
    for (int i = 0; i < 3 && i < M.D; ++i) q[i] = __dadd_rn(P.task_f[6 + i], uni(-P.task_f[0], P.task_f[0], u[i]));
    int nobj = M.D - 3;
    int pick = nobj > 0 ? 3 + min((int)(u[3] * nobj), nobj - 1) : -1;
    *target_dof = pick;
    goal[0] = goal[1] = goal[2] = 0.0;
  } else if (P.task == BS_TASK_CARTPOLE) {
    const R n = P.task_f[0];
    for (int i = 0; i < 2 && i < M.D; ++i) {
      q[i] = uni(-n, n, u[i]);
      qd[i] = uni(-n, n, u[2 + i]);
    }
    *target_dof = 0;  // upright streak
    goal[0] = goal[1] = goal[2] = 0.0;
  }
}

__device__ __forceinline__ R dist3(V3<R> a, V3<R> b) {
  R dx = __dsub_rn(a.x, b.x), dy = __dsub_rn(a.y, b.y), dz = __dsub_rn(a.z, b.z);
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
}

static __device__ __forceinline__ void task_eval(const Model& M, const BsSimParams& P, const V3<R>* lp, const R* q,
                          const V3<R>* ap, const R* goal, int tdof, bool diverged, float& reward,
                          bool& success, bool& fail) {
  if (P.task == BS_TASK_PICKCUBE) {
    const R* f = P.task_f;
    V3<R> ee = lp[P.ee_link];
    R d_ee = dist3(ee, ap[0]);
    R d_goal = dist3(v3(ap[0].x, ap[0].y, 0.0), v3(goal[0], goal[1], 0.0));
    success = d_goal < f[4];
    fail = ap[0].z < f[5] || diverged;
    reward = (float)(-__dadd_rn(d_ee, d_goal));
  } else if (P.task == BS_TASK_OPENCHAIN) {
    R hi = tdof >= 0 ? M.upper[tdof] : 1.0;
    R qv = tdof >= 0 ? q[tdof] : 0.0;
    success = tdof >= 0 && qv > P.task_f[1] * hi;
    fail = diverged;
    reward = (float)(tdof >= 0 ? qv / hi : 0.0);
  } else {
    success = false;
    fail = diverged;
    reward = 0.0f;
  }
}

static __device__ __forceinline__ void pack_obs(const Model& M, const BsSimParams& P, int Dm, int Am, const R* q, const R* qd,
                         const V3<R>* lp, const V3<R>* ap, const Q4<R>* aq, const V3<R>* av,
                         const V3<R>* aw, const R* goal, float* o, int obs_dim) {
  // layout: q[D_max] qd[D_max] ee_p[3]
  //   per actor slot: p[3] q[4] v[3] w[3]   goal[3];  CartpoleBalance: (x, x_dot, theta, theta_dot)
  int k = 0;
  if (P.task == BS_TASK_CARTPOLE) {
    o[0] = (float)q[0]; o[1] = (float)qd[0]; o[2] = (float)q[1]; o[3] = (float)qd[1];
    for (k = 4; k < obs_dim; ++k) o[k] = 0.0f;
    return;
  }
  for (int i = 0; i < Dm; ++i) o[k++] = i < M.D ? (float)q[i] : 0.0f;
  for (int i = 0; i < Dm; ++i) o[k++] = i < M.D ? (float)qd[i] : 0.0f;
  V3<R> ee = P.ee_link >= 0 ? lp[P.ee_link] : v3(0, 0, 0);
  o[k++] = (float)ee.x; o[k++] = (float)ee.y; o[k++] = (float)ee.z;
  for (int a = 0; a < Am; ++a) {
    bool ok = a < M.A;
    o[k++] = ok ? (float)ap[a].x : 0.f; o[k++] = ok ? (float)ap[a].y : 0.f; o[k++] = ok ? (float)ap[a].z : 0.f;
    o[k++] = ok ? (float)aq[a].w : 0.f; o[k++] = ok ? (float)aq[a].x : 0.f;
    o[k++] = ok ? (float)aq[a].y : 0.f; o[k++] = ok ? (float)aq[a].z : 0.f;
    o[k++] = ok ? (float)av[a].x : 0.f; o[k++] = ok ? (float)av[a].y : 0.f; o[k++] = ok ? (float)av[a].z : 0.f;
    o[k++] = ok ? (float)aw[a].x : 0.f; o[k++] = ok ? (float)aw[a].y : 0.f; o[k++] = ok ? (float)aw[a].z : 0.f;
  }
  o[k++] = (float)goal[0]; o[k++] = (float)goal[1]; o[k++] = (float)goal[2];
  for (; k < obs_dim; ++k) o[k] = 0.0f;
}

}  // namespace sim
}  // namespace bs
