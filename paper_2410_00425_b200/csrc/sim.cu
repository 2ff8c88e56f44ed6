// Fused control step for every env: controller -> substeps (implicit PD drives, CRBA/RNEA
// forward dynamics, free bodies, broadphase + narrowphase contacts, projected Gauss-Seidel,
// semi-implicit Euler, joint limits, divergence freeze) -> FK cache -> task evaluation ->
// state obs -> in-kernel auto-reset.
//
// Reference semantics: SPEC.md:319-354 (dynamics), 249-257 (FK), 402-410 (controllers),
// 536-553 (reset/step), with DESIGN.md's decisions register (A-4..A-25).  The CPU oracle
// (oracle/engine.py) restates the same algorithm independently.
//
// Execution model (v1): one thread per env, state resident in HBM in SoA rows, all
// per-env scratch (link poses, spatial quantities, contact rows) in thread-local memory
// (L1-resident).  Nothing in the step is a dense contraction, so no tensor cores; the
// kernel is latency/ALU bound (DESIGN.md section "Roofline").  fp64 throughout, as the
// reference mandates.
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
  const int32_t *p_i, *p_j, *p_code;
  const R *a_mass, *a_inertia;
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
  M.p_i = T.pair_i + po; M.p_j = T.pair_j + po; M.p_code = T.pair_code + po;
  M.a_mass = T.actor_mass + ao; M.a_inertia = T.actor_inertia + 3 * ao;
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

// Dense Cholesky of an n x n SPD matrix in place (lower triangle), n <= MD.
template <int MD>
__device__ __forceinline__ void cholesky(R* A, int n) {
  for (int j = 0; j < n; ++j) {
    R s = A[j * MD + j];
    for (int k = 0; k < j; ++k) s -= A[j * MD + k] * A[j * MD + k];
    R d = sqrt(s);
    A[j * MD + j] = d;
    R inv = 1.0 / d;
    for (int i = j + 1; i < n; ++i) {
      R t = A[i * MD + j];
      for (int k = 0; k < j; ++k) t -= A[i * MD + k] * A[j * MD + k];
      A[i * MD + j] = t * inv;
    }
  }
}
template <int MD>
__device__ __forceinline__ void chol_solve(const R* Lm, int n, R* x) {
  for (int i = 0; i < n; ++i) {
    R t = x[i];
    for (int k = 0; k < i; ++k) t -= Lm[i * MD + k] * x[k];
    x[i] = t / Lm[i * MD + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    R t = x[i];
    for (int k = i + 1; k < n; ++k) t -= Lm[k * MD + i] * x[k];
    x[i] = t / Lm[i * MD + i];
  }
}

// ---------------------------------------------------------------- contacts
struct Contact { V3<R> p, n; R d; int pair; int si, sj; };

__device__ __forceinline__ void plane_of(const V3<R>& P, const Q4<R>& Q, V3<R>& n, V3<R>& p0) {
  n = quat_rotate(Q, v3(0, 0, 1));
  p0 = P;
}

template <int MC>
__device__ __forceinline__ void push(Contact* cs, int& nc, V3<R> sB, V3<R> n, R depth, int pair, int si,
                                     int sj, bool flip, R slop) {
  if (!(depth >= -slop) || nc >= MC) return;
  Contact& c = cs[nc++];
  c.p = sub(sB, scl(n, 0.5 * depth));
  c.n = flip ? scl(n, -1.0) : n;
  c.d = depth;
  c.pair = pair; c.si = si; c.sj = sj;
}

// ---------------------------------------------------------------- PGS rows
template <int MD>
struct Row {
  R Ja[MD], Wa[MD];
  V3<R> e;
  int act[2];
  R sgn[2], invm[2];
  V3<R> Jw[2], Ww[2];
  R K;
};

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

// ----------------------------------------------------------------------------------
// One substep for one env.  q/qd (D), actor pose/vel (A) are updated in place unless the
// result is non-finite (then the env is flagged and its state left untouched).
template <class C>
__device__ void substep(const Model& M, const BsSimParams& P, const R* target, R* q, R* qd,
                        V3<R>* ap, Q4<R>* aq, V3<R>* av, V3<R>* aw, Scratch<C>& sc, int& unsupported,
                        int& ncontacts, Contact* cs, bool& diverged) {
  constexpr int MD = C::MD;
  const R dt = P.dt;
  const int D = M.D, L = M.L;
  V3<R>* lp = sc.lp;
  Q4<R>* lq = sc.lq;
  V6* S = sc.S;
  fk<C>(M, q, lp, lq);
  motion_subspace(M, lp, lq, S);
  // ---- articulations: C(q, qd) by RNEA, M(q) by CRBA, implicit drives, Cholesky
  R u_q[MD], Mt[MD * MD];
  {
    V6 V[C::ML], F[C::ML];
    Inertia I[C::ML];
    const V6 g6 = {{0, 0, 0}, {-P.gravity[0], -P.gravity[1], -P.gravity[2]}};
    V6 a[C::ML];
    for (int l = 0; l < L; ++l) {
      int par = M.parent[l];
      I[l] = world_inertia(M, l, lp[l], lq[l]);
      V[l] = par >= 0 ? V[par] : V6{{0, 0, 0}, {0, 0, 0}};
      a[l] = par >= 0 ? a[par] : g6;
      if (M.jtype[l] != BS_JOINT_FIXED) {
        R s = qd[M.dof[l]];
        V6 Sq = mk6(scl(gw(S[l]), s), scl(gv(S[l]), s));
        V[l] = mk6(add(gw(V[l]), gw(Sq)), add(gv(V[l]), gv(Sq)));
        V6 c = crossm(V[l], Sq);
        a[l] = mk6(add(gw(a[l]), gw(c)), add(gv(a[l]), gv(c)));
      }
    }
    for (int l = 0; l < L; ++l) {
      V6 f1 = imul(I[l], a[l]);
      V6 f2 = crossf(V[l], imul(I[l], V[l]));
      F[l] = mk6(add(gw(f1), gw(f2)), add(gv(f1), gv(f2)));
    }
    R Cb[MD];
    for (int l = L - 1; l >= 0; --l) {
      if (M.jtype[l] != BS_JOINT_FIXED) Cb[M.dof[l]] = dot6(S[l], F[l]);
      int par = M.parent[l];
      if (par >= 0) F[par] = mk6(add(gw(F[par]), gw(F[l])), add(gv(F[par]), gv(F[l])));
    }
    // composite inertias (reuse I)
    for (int l = L - 1; l >= 0; --l) {
      int par = M.parent[l];
      if (par < 0) continue;
      I[par].m += I[l].m;
      I[par].h = add(I[par].h, I[l].h);
      for (int k = 0; k < 6; ++k) I[par].I[k] += I[l].I[k];
    }
    for (int l = 0; l < L; ++l) {
      if (M.jtype[l] == BS_JOINT_FIXED) continue;
      int i = M.dof[l];
      V6 Fc = imul(I[l], S[l]);
      for (int k = l; k >= 0; k = M.parent[k]) {
        if (M.jtype[k] == BS_JOINT_FIXED) continue;
        int j = M.dof[k];
        R v = dot6(S[k], Fc);
        Mt[i * MD + j] = v;
        Mt[j * MD + i] = v;
      }
    }
    R rhs[MD];
    for (int i = 0; i < D; ++i) {
      R kp = M.kp[i], kd = M.kd[i], dmp = M.damping[i], fl = M.flim[i];
      Mt[i * MD + i] += dt * (kd + dmp) + (dt * dt) * kp;
      R tau = kp * ((target[i] - q[i]) - dt * qd[i]) + kd * (0.0 - qd[i]);
      tau = fmin(fmax(tau, -fl), fl) - dmp * qd[i];
      rhs[i] = tau - Cb[i];
    }
    if (D) {
      cholesky<MD>(Mt, D);
      chol_solve<MD>(Mt, D, rhs);
    }
    for (int i = 0; i < D; ++i) u_q[i] = qd[i] + dt * rhs[i];
  }
  // ---- free bodies
  V3<R> u_v[C::MA], u_w[C::MA];
  R Iwi[C::MA][9];
  const V3<R> g = v3(P.gravity[0], P.gravity[1], P.gravity[2]);
  for (int a = 0; a < M.A; ++a) {
    R Iw[9];
    actor_world_inertia(M.a_inertia + 3 * a, aq[a], Iw, Iwi[a]);
    V3<R> gyro = scl(crs(aw[a], m3mul(Iw, aw[a])), -1.0);
    u_w[a] = add(aw[a], scl(m3mul(Iwi[a], gyro), dt));
    u_v[a] = add(av[a], scl(g, dt));
  }
  // ---- shape world poses
  V3<R> sp[C::MS];
  Q4<R> sq[C::MS];
  for (int s = 0; s < M.S; ++s) {
    const R* f = M.s_frame + 7 * s;
    int bt = M.s_btype[s], bi = M.s_body[s];
    if (bt == BS_BODY_LINK) compose(lp[bi], lq[bi], ld3(f), ld4(f + 3), sp[s], sq[s]);
    else if (bt == BS_BODY_ACTOR) { sp[s] = ap[bi]; sq[s] = aq[bi]; }
    else { sp[s] = ld3(f); sq[s] = ld4(f + 3); }
  }
  // ---- broadphase + narrowphase (pair order = slot order, A-5)
  const R slop = P.slop;
  int nc = 0;
  for (int pi = 0; pi < M.P; ++pi) {
    int i = M.p_i[pi], j = M.p_j[pi], code = M.p_code[pi];
    int ki = M.s_kind[i], kj = M.s_kind[j];
    bool near;
    if (ki == BS_KIND_PLANE || kj == BS_KIND_PLANE) {
      int pl = kj == BS_KIND_PLANE ? j : i, ot = kj == BS_KIND_PLANE ? i : j;
      V3<R> n = quat_rotate(sq[pl], v3(0, 0, 1));
      near = dot(n, sub(sp[ot], sp[pl])) <= M.s_radius[ot] + slop;
    } else {
      V3<R> d = sub(sp[i], sp[j]);
      near = sqrt(dot(d, d)) <= (M.s_radius[i] + M.s_radius[j]) + slop;
    }
    if (!near) continue;
    int base = code & 15;
    if (base == BS_PAIR_UNSUPPORTED) { ++unsupported; continue; }
    bool flip = (code & BS_PAIR_SWAP) != 0;
    int a = flip ? j : i, b = flip ? i : j;
    const R* sa = M.s_size + 3 * a;
    const R* sb = M.s_size + 3 * b;
    if (base == BS_PAIR_SPHERE_PLANE) {
      V3<R> n, p0;
      plane_of(sp[b], sq[b], n, p0);
      R sd = dot(n, sub(sp[a], p0));
      push<C::MC>(cs, nc, sub(sp[a], scl(n, sd)), n, sa[0] - sd, pi, i, j, flip, slop);
    } else if (base == BS_PAIR_BOX_PLANE) {
      V3<R> n, p0;
      plane_of(sp[b], sq[b], n, p0);
      R dep[8];
      V3<R> sB[8];
      int valid = 0;
      for (int k = 0; k < 8; ++k) {
        V3<R> loc = v3((k & 1) ? sa[0] : -sa[0], (k & 2) ? sa[1] : -sa[1], (k & 4) ? sa[2] : -sa[2]);
        V3<R> corner = add(sp[a], quat_rotate(sq[a], loc));
        R sd = dot(n, sub(corner, p0));
        dep[k] = -sd;
        sB[k] = sub(corner, scl(n, sd));
        valid += dep[k] >= -slop;
      }
      if (valid > 4) {  // keep the four deepest, ties -> lower corner index
        for (int k = 0; k < 8; ++k) {
          if (!(dep[k] >= -slop)) continue;
          int rank = 0;
          for (int o = 0; o < 8; ++o) rank += (dep[o] > dep[k]) || (dep[o] == dep[k] && o < k);
          if (rank >= 4) dep[k] = -INFINITY;
        }
      }
      for (int k = 0; k < 8; ++k) push<C::MC>(cs, nc, sB[k], n, dep[k], pi, i, j, flip, slop);
    } else if (base == BS_PAIR_SPHERE_SPHERE) {
      V3<R> d = sub(sp[a], sp[b]);
      R dist = sqrt(dot(d, d));
      V3<R> n = dist > 1e-12 ? scl(d, 1.0 / dist) : v3(0, 0, 1);
      if (dist > 1e-12) n = v3(d.x / dist, d.y / dist, d.z / dist);
      R depth = (sa[0] + sb[0]) - dist;
      push<C::MC>(cs, nc, add(sp[b], scl(n, sb[0])), n, depth, pi, i, j, flip, slop);
    } else if (base == BS_PAIR_SPHERE_BOX) {
      V3<R> loc = quat_rotate(qconj(sq[b]), sub(sp[a], sp[b]));
      R h[3] = {sb[0], sb[1], sb[2]};
      R l3[3] = {loc.x, loc.y, loc.z};
      R cl[3], dl[3];
      for (int k = 0; k < 3; ++k) {
        cl[k] = fmin(fmax(l3[k], -h[k]), h[k]);
        dl[k] = l3[k] - cl[k];
      }
      R d2 = (dl[0] * dl[0] + dl[1] * dl[1]) + dl[2] * dl[2];
      R nl[3], sl[3], depth;
      if (d2 > 1e-24) {
        R dist = sqrt(d2);
        for (int k = 0; k < 3; ++k) { nl[k] = dl[k] / dist; sl[k] = cl[k]; }
        depth = sa[0] - dist;
      } else {
        int kk = 0;
        R best = h[0] - fabs(l3[0]);
        for (int k = 1; k < 3; ++k) {
          R pen = h[k] - fabs(l3[k]);
          if (pen < best) { best = pen; kk = k; }
        }
        R sgn = l3[kk] >= 0.0 ? 1.0 : -1.0;
        for (int k = 0; k < 3; ++k) { nl[k] = 0; sl[k] = l3[k]; }
        nl[kk] = sgn;
        sl[kk] = sgn * h[kk];
        depth = sa[0] + best;
      }
      V3<R> n = quat_rotate(sq[b], v3(nl[0], nl[1], nl[2]));
      V3<R> sB = add(sp[b], quat_rotate(sq[b], v3(sl[0], sl[1], sl[2])));
      push<C::MC>(cs, nc, sB, n, depth, pi, i, j, flip, slop);
    } else if (base == BS_PAIR_CAPSULE_PLANE) {
      V3<R> n, p0;
      plane_of(sp[b], sq[b], n, p0);
      for (int k = 0; k < 2; ++k) {
        V3<R> e = add(sp[a], quat_rotate(sq[a], v3(0, 0, k ? sa[1] : -sa[1])));
        R sd = dot(n, sub(e, p0));
        push<C::MC>(cs, nc, sub(e, scl(n, sd)), n, sa[0] - sd, pi, i, j, flip, slop);
      }
    }
  }
  ncontacts = nc;
  // ---- PGS rows
  Row<MD> rows[C::MC * 3];
  R bias[C::MC], spec[C::MC], lam[C::MC * 3];
  for (int c = 0; c < nc; ++c) {
    const Contact& ct = cs[c];
    V3<R> n = ct.n;
    // tangent basis (A-6)
    R an[3] = {fabs(n.x), fabs(n.y), fabs(n.z)};
    int k = 0;
    if (an[1] < an[k]) k = 1;
    if (an[2] < an[k]) k = 2;
    V3<R> e = v3(k == 0, k == 1, k == 2);
    V3<R> t1 = crs(n, e);
    R t1n = sqrt(dot(t1, t1));
    t1 = v3(t1.x / t1n, t1.y / t1n, t1.z / t1n);
    V3<R> t2 = crs(n, t1);
    V3<R> dirs[3] = {n, t1, t2};
    for (int r = 0; r < 3; ++r) {
      Row<MD>& row = rows[3 * c + r];
      row.e = dirs[r];
      for (int d = 0; d < D; ++d) row.Ja[d] = 0.0;
      int slots[2] = {ct.si, ct.sj};
      R sgns[2] = {1.0, -1.0};
      for (int s = 0; s < 2; ++s) {
        row.act[s] = -1;
        int sl = slots[s], bt = M.s_btype[sl], bi = M.s_body[sl];
        if (bt == BS_BODY_LINK && !M.grounded[bi]) {
          for (int kk = bi; kk >= 0; kk = M.parent[kk]) {
            if (M.jtype[kk] == BS_JOINT_FIXED) continue;
            V3<R> col = add(gv(S[kk]), crs(gw(S[kk]), ct.p));
            row.Ja[M.dof[kk]] += sgns[s] * dot(row.e, col);
          }
        } else if (bt == BS_BODY_ACTOR) {
          row.act[s] = bi;
          row.sgn[s] = sgns[s];
          row.invm[s] = 1.0 / M.a_mass[bi];
          V3<R> rr = sub(ct.p, ap[bi]);
          row.Jw[s] = scl(crs(rr, row.e), sgns[s]);
          row.Ww[s] = m3mul(Iwi[bi], row.Jw[s]);
        }
      }
      for (int d = 0; d < D; ++d) row.Wa[d] = row.Ja[d];
      if (D) chol_solve<MD>(Mt, D, row.Wa);
      R K = 0;
      for (int d = 0; d < D; ++d) K += row.Ja[d] * row.Wa[d];
      for (int s = 0; s < 2; ++s)
        if (row.act[s] >= 0) K += dot(row.e, row.e) * row.invm[s] + dot(row.Jw[s], row.Ww[s]);
      row.K = K;
      lam[3 * c + r] = 0.0;
    }
    R d = ct.d;
    bias[c] = d > slop ? P.beta * (d - slop) / dt : (d >= 0.0 ? 0.0 : d / dt);
    spec[c] = d < 0.0 ? d / dt : 0.0;
  }
  // ---- projected Gauss-Seidel: per-env sequential sweeps, rows normal, t1, t2
  const int iters = P.pos_iters + P.vel_iters;
  for (int it = 0; it < iters; ++it) {
    bool pos_phase = it < P.pos_iters;
    for (int c = 0; c < nc; ++c) {
      for (int r = 0; r < 3; ++r) {
        Row<MD>& row = rows[3 * c + r];
        if (!(row.K > 1e-12)) continue;
        R vrow = 0;
        for (int d = 0; d < D; ++d) vrow += row.Ja[d] * u_q[d];
        for (int s = 0; s < 2; ++s) {
          int a = row.act[s];
          if (a < 0) continue;
          vrow += row.sgn[s] * dot(row.e, u_v[a]) + dot(row.Jw[s], u_w[a]);
        }
        R old = lam[3 * c + r], nw;
        if (r == 0) {
          R tgt = pos_phase ? bias[c] : spec[c];
          nw = fmax(old + (tgt - vrow) / row.K, 0.0);
        } else {
          R bound = P.friction * lam[3 * c];
          nw = fmin(fmax(old + (0.0 - vrow) / row.K, -bound), bound);
        }
        R delta = nw - old;
        lam[3 * c + r] = nw;
        for (int d = 0; d < D; ++d) u_q[d] += delta * row.Wa[d];
        for (int s = 0; s < 2; ++s) {
          int a = row.act[s];
          if (a < 0) continue;
          u_v[a] = add(u_v[a], scl(row.e, delta * row.sgn[s] * row.invm[s]));
          u_w[a] = add(u_w[a], scl(row.Ww[s], delta));
        }
      }
    }
  }
  // ---- integrate, limits, divergence
  R q1[MD], qd1[MD];
  bool finite = true;
  for (int i = 0; i < D; ++i) {
    R v = q[i] + dt * u_q[i];
    R w = u_q[i];
    if (v < M.lower[i]) { v = M.lower[i]; w = fmax(w, 0.0); }
    else if (v > M.upper[i]) { v = M.upper[i]; w = fmin(w, 0.0); }
    q1[i] = v; qd1[i] = w;
    finite &= isfinite(v) && isfinite(w);
  }
  V3<R> ap1[C::MA];
  Q4<R> aq1[C::MA];
  for (int a = 0; a < M.A; ++a) {
    ap1[a] = add(ap[a], scl(u_v[a], dt));
    Q4<R> wq = quat_mul(Q4<R>{0.0, u_w[a].x, u_w[a].y, u_w[a].z}, aq[a]);
    R h = 0.5 * dt;
    aq1[a] = quat_normalize(Q4<R>{aq[a].w + h * wq.w, aq[a].x + h * wq.x, aq[a].y + h * wq.y, aq[a].z + h * wq.z});
    finite &= isfinite(ap1[a].x) && isfinite(ap1[a].y) && isfinite(ap1[a].z);
    finite &= isfinite(aq1[a].w) && isfinite(aq1[a].x) && isfinite(aq1[a].y) && isfinite(aq1[a].z);
    finite &= isfinite(u_v[a].x) && isfinite(u_v[a].y) && isfinite(u_v[a].z);
    finite &= isfinite(u_w[a].x) && isfinite(u_w[a].y) && isfinite(u_w[a].z);
  }
  if (!finite) { diverged = true; return; }
  for (int i = 0; i < D; ++i) { q[i] = q1[i]; qd[i] = qd1[i]; }
  for (int a = 0; a < M.A; ++a) { ap[a] = ap1[a]; aq[a] = aq1[a]; av[a] = u_v[a]; aw[a] = u_w[a]; }
}

// ---------------------------------------------------------------- tasks
// PickCube task_f layout: 0 q_noise, 1 cube_half, 2 cube_xy, 3 goal_xy, 4 success_dist,
// 5 fail_z, 6..8 q_rest.   OpenChain task_f: 0 success_frac.
__device__ void task_reset(const Model& M, const BsSimParams& P, int64_t genv, uint32_t rc, R* q, R* qd,
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
    ap[0] = v3(cx, cy, f[1]);
    aq[0] = quat_normalize(Q4<R>{c, 0.0, 0.0, s});
    goal[0] = uni(-f[3], f[3], u[6]);
    goal[1] = uni(-f[3], f[3], u[7]);
    goal[2] = f[1];
  } else if (P.task == BS_TASK_OPENCHAIN) {
    // arm dofs at q_rest (task_f 6..8), articulated-object dofs closed; target dof drawn
    for (int i = 0; i < 3 && i < M.D; ++i) q[i] = __dadd_rn(P.task_f[6 + i], uni(-P.task_f[0], P.task_f[0], u[i]));
    int nobj = M.D - 3;
    int pick = nobj > 0 ? 3 + min((int)(u[3] * nobj), nobj - 1) : -1;
    *target_dof = pick;
    goal[0] = goal[1] = goal[2] = 0.0;
  }
}

__device__ __forceinline__ R dist3(V3<R> a, V3<R> b) {
  R dx = __dsub_rn(a.x, b.x), dy = __dsub_rn(a.y, b.y), dz = __dsub_rn(a.z, b.z);
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
}

__device__ void task_eval(const Model& M, const BsSimParams& P, const V3<R>* lp, const R* q,
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

__device__ void pack_obs(const Model& M, const BsSimParams& P, int Dm, int Am, const R* q, const R* qd,
                         const V3<R>* lp, const V3<R>* ap, const Q4<R>* aq, const V3<R>* av,
                         const V3<R>* aw, const R* goal, float* o, int obs_dim) {
  // layout: q[D_max] qd[D_max] ee_p[3]
  //   per actor slot: p[3] q[4] v[3] w[3]   goal[3]
  int k = 0;
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
__global__ void __launch_bounds__(64) k_step(BsModelTables T, BsEnvState S, BsStepOutputs O, BsSimParams P,
                                             const float* __restrict__ action) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= S.num_envs) return;
  const Model M = model_of(T, S.model_id[e]);
  EnvRegs<C> r;
  load_env<C>(T, S, M, e, r);
  Scratch<C> sc;
  bool diverged = S.diverged[e] != 0;
  // ---- controller: targets from the action, once per control step
  const float* act = action + (int64_t)e * P.action_dim;
  for (int i = 0; i < M.D; ++i) {
    int ai = M.ctrl[i];
    R tgt = r.q[i];
    if (ai >= 0) {
      R a = fmin(fmax((R)act[ai], -1.0), 1.0);
      R lo = M.lower[i], hi = M.upper[i];
      if (P.ctrl_mode == BS_CTRL_PD_JOINT_DELTA_POS) {
        tgt = fmin(fmax(r.q[i] + a * P.action_scale, lo), hi);
      } else {  // pd_joint_pos
        R un = (isfinite(lo) && isfinite(hi)) ? lo + (a + 1.0) * 0.5 * (hi - lo) : a * P.action_scale;
        tgt = fmin(fmax(un, lo), hi);
      }
    }
    r.tgt[i] = tgt;
  }
  int unsupported = 0, nc = 0;
  Contact cs[C::MC];
  if (!diverged) {
    for (int s = 0; s < P.substeps && !diverged; ++s) {
      unsupported = 0;  // report the last substep's count (as the oracle does)
      substep<C>(M, P, r.tgt, r.q, r.qd, r.ap, r.aq, r.av, r.aw, sc, unsupported, nc, cs, diverged);
    }
  }
  fk<C>(M, r.q, sc.lp, sc.lq);
  // ---- task evaluation
  float reward;
  bool success, fail;
  int32_t tdof = S.target_dof[e];
  task_eval(M, P, sc.lp, r.q, r.ap, r.goal, tdof, diverged, reward, success, fail);
  int32_t el = S.elapsed[e] + 1;
  bool terminated = P.early_termination ? (success || fail) : false;
  bool truncated = el >= P.max_steps;
  O.reward[e] = reward;
  O.terminated[e] = terminated;
  O.truncated[e] = truncated;
  O.success[e] = success;
  O.fail[e] = fail;
  O.unsupported_pairs[e] = unsupported;
  if (O.contact_count) {
    O.contact_count[e] = nc;
    for (int c = 0; c < nc && c < T.C_max; ++c) {
      int64_t o = (int64_t)e * T.C_max + c;
      if (O.contact_pairs) { O.contact_pairs[2 * o] = cs[c].si; O.contact_pairs[2 * o + 1] = cs[c].sj; }
      if (O.contact_geom) {
        R* g = O.contact_geom + 7 * o;
        st3(g, cs[c].p); st3(g + 3, cs[c].n); g[6] = cs[c].d;
      }
    }
  }
  uint8_t div_out = diverged;
  if (P.auto_reset && (terminated || truncated)) {
    uint32_t rc = S.reset_count[e] + 1;
    S.reset_count[e] = rc;
    task_reset(M, P, S.env_offset + e, rc, r.q, r.qd, r.ap, r.aq, r.av, r.aw, r.goal, &tdof);
    S.target_dof[e] = tdof;
    el = 0;
    div_out = 0;
    fk<C>(M, r.q, sc.lp, sc.lq);
  }
  S.elapsed[e] = el;
  S.diverged[e] = div_out;
  store_env<C>(T, S, M, e, r, sc.lp, sc.lq);
  if (O.obs) pack_obs(M, P, T.D_max, T.A_max, r.q, r.qd, sc.lp, r.ap, r.aq, r.av, r.aw, r.goal,
                      O.obs + (int64_t)e * O.obs_dim, O.obs_dim);
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
  if (mask == nullptr || mask[e]) {
    uint32_t rc = S.reset_count[e] + (bump ? 1u : 0u);
    S.reset_count[e] = rc;
    int32_t tdof = -1;
    task_reset(M, P, S.env_offset + e, rc, r.q, r.qd, r.ap, r.aq, r.av, r.aw, r.goal, &tdof);
    S.target_dof[e] = tdof;
    S.elapsed[e] = 0;
    S.diverged[e] = 0;
    for (int i = 0; i < M.D; ++i) r.tgt[i] = r.q[i];
  } else {
    const R* tg = S.target + (int64_t)e * T.D_max;
    for (int i = 0; i < M.D; ++i) r.tgt[i] = tg[i];
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
typedef Cap<12, 16, 24, 32, 4> CapLarge;  // cabinets / heterogeneous scenes

template <class C>
bool fits(const BsModelTables& T) {
  return T.D_max <= C::MD && T.L_max <= C::ML && T.S_max <= C::MS && T.C_max <= C::MC && T.A_max <= C::MA;
}

}  // namespace sim
}  // namespace bs

using namespace bs::sim;

#define THREADS 32

extern "C" {

int bs_step(const BsModelTables* T, const BsEnvState* S, const BsStepOutputs* O, const BsSimParams* P,
            const float* action, void* stream) {
  if (!T || !S || !O || !P || !action) return BS_ERR_ARGUMENT;
  if (S->num_envs <= 0) return BS_OK;
  if (!O->reward || !O->terminated || !O->truncated || !O->success || !O->fail || !O->unsupported_pairs)
    return BS_ERR_ARGUMENT;
  int blocks = (S->num_envs + THREADS - 1) / THREADS;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (fits<CapSmall>(*T)) k_step<CapSmall><<<blocks, THREADS, 0, st>>>(*T, *S, *O, *P, action);
  else if (fits<CapLarge>(*T)) k_step<CapLarge><<<blocks, THREADS, 0, st>>>(*T, *S, *O, *P, action);
  else return BS_ERR_UNSUPPORTED;
  return bs::launch_status();
}

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
