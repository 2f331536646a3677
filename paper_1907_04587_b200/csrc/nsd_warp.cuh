// Batched rigid-body environments, one full warp per environment (C5 path).
//
// The same newton_step as nsd_engine.cuh (newton.cpp:321-418; PCR recurrence of
// solvers.cpp:127-174 with z = M^-1 r updated by recursion exactly as the
// reference), laid out for a tiny articulated scene (an ant: 9 rigid bodies,
// 8 joints / 40 rows, ~12 contacts / 36 rows):
//
//   * one constraint object per lane: lane k < nj owns joint k, lane nj + c owns
//     contact c (nj + nc <= 32; larger environments are solved by the
//     sub-warp object solver, nsd_batch.cuh). An object owns its rows
//     (<= 5), so every PCR row vector lives in that lane's REGISTERS: the
//     row-parallel phases (p/ap update, trial norms, commit) touch no memory;
//   * joints and contacts share one row form: np point rows along directions
//     D_i through lever arms (r_a, r_b) and na axis rows along C_i, so
//     J w and J^T y are one code path for every lane (no joint/contact
//     divergence inside the warp). A contact is np = 3 with D = (n, d1, d2)
//     and row scales (dphi/dC, active, active); a revolute joint np = 3 with
//     D = (e_x, e_y, e_z) plus na = 2 axis rows;
//   * J^T y: each object stages its two body-side wrenches in shared memory,
//     then lane b < nb gathers body b's wrenches in a fixed order (static joint
//     incidence, then the step's contact incidence): deterministic, no atomics;
//     w = H^-1 J^T y goes back to shared memory for the J w pass;
//   * reductions are xor-butterfly shuffles: every lane ends with the same bits
//     (IEEE addition is commutative), so the data-dependent PCR exits are
//     warp-uniform without a broadcast.
// Shared memory per environment: body state (q, rotation cache, u, I_w^-1, w),
// the objects' records (lever arms and row directions, [value][lane] layout,
// conflict-free) and the staging area (14-double stride, conflict-free 16-byte
// stores). Step-start data (q-, u-, u~, I_w, the contact set) comes from the
// per-env slabs that the narrow-phase launch wrote (k_batch_sub, collide mode).
#pragma once

#include "nsd_engine.cuh"
#include "nsd_warp_plan.h"

namespace nsd {
namespace wp {

// Warp all-reduce, xor butterfly: identical bits on every lane.
__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}
__device__ __forceinline__ double wmax(double v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, m));
  return v;
}
__device__ __forceinline__ void wsum2(double& a, double& b) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, a, m), y = __shfl_xor_sync(0xffffffffu, b, m);
    a += x;
    b += y;
  }
}

template <class R> __device__ __forceinline__ V3<R> lds3(const R* p) { return v3(p[0], p[1], p[2]); }
template <class R> __device__ __forceinline__ void sts3(R* p, V3<R> v) {
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
}
// This lane's record (arm_a, arm_b, 5 row directions) from its [lane][stride] slot
// with 16-byte loads; single values are stored with scalar stores (assembly).
template <class R> struct Rec {
  V3<R> arm_a, arm_b, d[kRows];
};
__device__ __forceinline__ void ld_vals(const double* p, double (&v)[22]) {
#pragma unroll
  for (int k = 0; k < 11; ++k) {
    const double2 t = reinterpret_cast<const double2*>(p)[k];
    v[2 * k] = t.x;
    v[2 * k + 1] = t.y;
  }
}
__device__ __forceinline__ void ld_vals(const float* p, float (&v)[24]) {
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const float4 t = reinterpret_cast<const float4*>(p)[k];
    v[4 * k] = t.x;
    v[4 * k + 1] = t.y;
    v[4 * k + 2] = t.z;
    v[4 * k + 3] = t.w;
  }
}
// One 3-vector of this lane's record (value offset v = 0, 3, ..., 18): a 16-byte
// and an 8-byte load (for fp64; the slot's alignment alternates with v).
template <int V> __device__ __forceinline__ V3<double> rec_v3(const double* rec, int lane) {
  const double* p = rec + rec_stride<double>() * lane + V;
  if constexpr (V % 2 == 0) {
    const double2 a = *reinterpret_cast<const double2*>(p);
    return v3(a.x, a.y, p[2]);
  } else {
    const double2 b = *reinterpret_cast<const double2*>(p + 1);
    return v3(p[0], b.x, b.y);
  }
}
template <int V> __device__ __forceinline__ V3<float> rec_v3(const float* rec, int lane) {
  const float* p = rec + rec_stride<float>() * lane + V;
  return v3(p[0], p[1], p[2]);
}
template <class R> __device__ __forceinline__ Rec<R> rec_load(const R* rec, int lane) {
  Rec<R> o;
  o.arm_a = rec_v3<0>(rec, lane);
  o.arm_b = rec_v3<3>(rec, lane);
  o.d[0] = rec_v3<6>(rec, lane);
  o.d[1] = rec_v3<9>(rec, lane);
  o.d[2] = rec_v3<12>(rec, lane);
  o.d[3] = rec_v3<15>(rec, lane);
  o.d[4] = rec_v3<18>(rec, lane);
  return o;
}
template <class S, class R> __device__ __forceinline__ void rec3_put(S* rec, int v, int lane, V3<R> x) {
  S* p = rec + rec_stride<S>() * lane + v;
  p[0] = S(x.x);
  p[1] = S(x.y);
  p[2] = S(x.z);
}
template <class T, class S> __device__ __forceinline__ V3<T> cv3(V3<S> v) { return v3(T(v.x), T(v.y), T(v.z)); }

// This lane's constraint object.
struct Obj {
  int kind;  // joint kind 0..3, 4 contact, -1 none
  int idx;   // joint or contact index
  int a, b;  // bodies (-1 world)
  int np, na, nr;
};

// Lin (unshifted 1/m, divided as the reference's BlockDiagMass::inverse_quadratic)
// and angular (I_w^-1) quadratic forms of one body side.
template <class R> __device__ __forceinline__ R lin_quad_unshifted(V3<R> c, R m) {
  return c.x * c.x / m + c.y * c.y / m + c.z * c.z / m;
}
template <class R> __device__ __forceinline__ R lin_quad_shifted(V3<R> c, R hi) {
  return c.x * c.x * hi + c.y * c.y * hi + c.z * c.z * hi;
}

// R: state, assembly, Newton update (double); S: the PCR operator's data and row
// vectors (double, or float in the mixed-precision mode).
template <class R, class S> struct Env {
  const Topo<R>& T;
  R* bq;
  R* brot;
  R* bu;
  R* biwi;
  R* bhi;
  S* bw;     // w = H^-1 J^T y of the operator
  void* stg;  // staging: R (momentum, du) or S (operator) values
  S* rec;
  R* x;  // [row][lane]
  R* bx;
  int* gent_off;  // per body: its staged wrenches (joints, then contacts ascending)
  int* gent;
  int nj, nc, nb;
};

// Quadratic form d^T J M^-1 J^T d of a point row along d through the arms, summed
// in the reference's order a.lin + a.ang + b.lin + b.ang (contact_quad /
// object_quad). shifted: H^-1 = 1/(m + 0) per linear dof; else the unshifted
// c^2/m of BlockDiagMass::inverse_quadratic (bodies.cpp:149-177).
// sym_mul / sym_quad (nsd_engine.cuh) with the symmetric matrix held in R and the
// vector in S (the same expressions when R == S).
template <class S, class R> __device__ __forceinline__ V3<S> sym_mul_t(const R* s6, V3<S> v) {
  const S a = S(s6[0]), b = S(s6[1]), c = S(s6[2]), d = S(s6[3]), e = S(s6[4]), f = S(s6[5]);
  return v3(a * v.x + d * v.y + e * v.z, d * v.x + b * v.y + f * v.z, e * v.x + f * v.y + c * v.z);
}
template <class S, class R> __device__ __forceinline__ S sym_quad_t(const R* s6, V3<S> v) { return dot(v, sym_mul_t(s6, v)); }

template <class S, class R>
__device__ __forceinline__ S point_quad(const Topo<R>& T, const R* biwi, int a, int b, V3<S> d, V3<S> arm_a, V3<S> arm_b,
                                        bool shifted, const R* bhi = nullptr) {
  // shifted: H^-1 = 1 / (m + 0) per linear dof, the value batch setup stores in bhi
  S s = S(0);
  if (a >= 0) {
    const S m = S(T.bmass[a]);
    s += shifted ? lin_quad_shifted(d, bhi ? S(bhi[a]) : S(1) / (m + S(0))) : lin_quad_unshifted(d, m);
    s += sym_quad_t(biwi + 6 * a, cross(arm_a, d));
  }
  if (b >= 0) {
    const S m = S(T.bmass[b]);
    s += shifted ? lin_quad_shifted(d, bhi ? S(bhi[b]) : S(1) / (m + S(0))) : lin_quad_unshifted(d, m);
    s += sym_quad_t(biwi + 6 * b, cross(arm_b, d));
  }
  return s;
}

// T: the precision of the staged values (S for the operator, R for the momentum
// and Newton-update gathers); the records are read in S and widened.
template <class T, class R, class S, class YF>
__device__ __forceinline__ void stage_f(const Env<R, S>& E, const Obj& o, int lane, const T (&s)[3], const YF& y) {
  if (o.kind < 0) return;
  V3<T> f = v3(T(0), T(0), T(0)), ta = f;
  if (0 < o.np) f = f + (s[0] * y(0)) * cv3<T>(rec_v3<6>(E.rec, lane));
  if (1 < o.np) f = f + (s[1] * y(1)) * cv3<T>(rec_v3<9>(E.rec, lane));
  if (2 < o.np) f = f + (s[2] * y(2)) * cv3<T>(rec_v3<12>(E.rec, lane));
  if (0 >= o.np && 0 < o.nr) ta = ta + y(0) * cv3<T>(rec_v3<6>(E.rec, lane));
  if (1 >= o.np && 1 < o.nr) ta = ta + y(1) * cv3<T>(rec_v3<9>(E.rec, lane));
  if (2 >= o.np && 2 < o.nr) ta = ta + y(2) * cv3<T>(rec_v3<12>(E.rec, lane));
  if (3 < o.nr) ta = ta + y(3) * cv3<T>(rec_v3<15>(E.rec, lane));
  if (4 < o.nr) ta = ta + y(4) * cv3<T>(rec_v3<18>(E.rec, lane));
  T* d = static_cast<T*>(E.stg) + kStg * lane;
  if (o.a >= 0) {
    sts3(d, f);
    sts3(d + 3, cross(cv3<T>(rec_v3<0>(E.rec, lane)), f) + ta);
  }
  if (o.b >= 0) {
    sts3(d + 6, -f);
    sts3(d + 9, -(cross(cv3<T>(rec_v3<3>(E.rec, lane)), f) + ta));
  }
}

template <class T, class R, class S>
__device__ __forceinline__ void stage(const Env<R, S>& E, const Obj& o, int lane, const T (&s)[3], const T (&y)[kRows]) {
  stage_f(E, o, lane, s, [&](int i) { return y[i]; });
}

// Body gather of the staged wrenches (joints first, then contacts ascending).
template <class T, class R, class S>
__device__ __forceinline__ void gather(const Env<R, S>& E, int b, V3<T>& lin, V3<T>& ang) {
  lin = v3(T(0), T(0), T(0));
  ang = lin;
  const int e0 = E.gent_off[b], n = E.gent_off[b + 1] - e0;
  const int* ge = E.gent + e0;
  const T* st = static_cast<const T*>(E.stg);
  constexpr int kU = 8;  // up to 8 entries' offsets loaded before their ordered adds
  int off[kU];
#pragma unroll
  for (int e = 0; e < kU; ++e) off[e] = e < n ? ge[e] : 0;
#pragma unroll
  for (int e = 0; e < kU; ++e)
    if (e < n) {
      lin = lin + lds3(st + off[e]);
      ang = ang + lds3(st + off[e] + 3);
    }
  for (int e = kU; e < n; ++e) {
    lin = lin + lds3(st + ge[e]);
    ang = ang + lds3(st + ge[e] + 3);
  }
}

// Components k and k + 3 (linear, angular) of body b's gathered J^T y: the body's
// staged wrenches summed in entry order (the order of gather()); up to 8 entries'
// offsets and values are loaded before the ordered adds.
template <class R, class S>
__device__ __forceinline__ void gather_pair(const Env<R, S>& E, int b, int k, S& lin, S& ang) {
  const int e0 = E.gent_off[b], n = E.gent_off[b + 1] - e0;
  const int* ge = E.gent + e0;
  const S* sk = static_cast<const S*>(E.stg) + k;
  constexpr int kU = 8;
  int off[kU];
  S vl[kU], va[kU];
#pragma unroll
  for (int e = 0; e < kU; ++e) off[e] = e < n ? ge[e] : 0;
#pragma unroll
  for (int e = 0; e < kU; ++e) {
    vl[e] = e < n ? sk[off[e]] : S(0);
    va[e] = e < n ? sk[off[e] + 3] : S(0);
  }
  lin = S(0);
  ang = S(0);
#pragma unroll
  for (int e = 0; e < kU; ++e)
    if (e < n) {
      lin = lin + vl[e];
      ang = ang + va[e];
    }
  for (int e = kU; e < n; ++e) {
    lin = lin + sk[ge[e]];
    ang = ang + sk[ge[e] + 3];
  }
}

// w = H^-1 J^T y for every body with the whole warp: 10 bodies per round (one round
// for an ant), lane 3 g + k owns components k (linear) and k + 3 (angular) of body
// 10 r + g. The linear part scales by 1/m; the angular row k applies I_w^-1
// (sym_mul's expression) to the torque held by the group's three lanes, exchanged by
// shuffles. Needs __syncwarp() before (staging) and after.
template <class R, class S> __device__ __forceinline__ void bodies_w(const Env<R, S>& E, int lane) {
  const int g = lane / 3, k = lane - 3 * g;
  const int g0 = 3 * g;
  for (int b0 = 0; b0 < E.nb; b0 += 10) {
    const int b = b0 + g;
    const bool on = g < 10 && b < E.nb;
    S tl = S(0), ta = S(0);
    if (on) gather_pair(E, b, k, tl, ta);
    const S tx = __shfl_sync(0xffffffffu, ta, g0 < 32 ? g0 : 0);
    const S ty = __shfl_sync(0xffffffffu, ta, g0 + 1 < 32 ? g0 + 1 : 0);
    const S tz = __shfl_sync(0xffffffffu, ta, g0 + 2 < 32 ? g0 + 2 : 0);
    if (on) {
      const R* s6 = E.biwi + 6 * b;  // xx yy zz xy xz yz; row k of sym_mul
      const S c0 = S(k == 0 ? s6[0] : (k == 1 ? s6[3] : s6[4]));
      const S c1 = S(k == 0 ? s6[3] : (k == 1 ? s6[1] : s6[5]));
      const S c2 = S(k == 0 ? s6[4] : (k == 1 ? s6[5] : s6[2]));
      E.bw[6 * b + k] = tl * S(E.bhi[b]);
      E.bw[6 * b + 3 + k] = c0 * tx + c1 * ty + c2 * tz;
    }
  }
}

template <class R, class S>
__device__ __forceinline__ void jw(const Env<R, S>& E, const Obj& o, int lane, const S (&s)[3], S (&out)[kRows]) {
  V3<S> dv = v3(S(0), S(0), S(0)), wr = dv;
  if (o.a >= 0) {
    const S* w = E.bw + 6 * o.a;
    wr = lds3(w + 3);
    dv = lds3(w) + cross(wr, rec_v3<0>(E.rec, lane));
  }
  if (o.b >= 0) {
    const S* w = E.bw + 6 * o.b;
    const V3<S> wb = lds3(w + 3);
    dv = dv - lds3(w);
    dv = dv - cross(wb, rec_v3<3>(E.rec, lane));
    wr = wr - wb;
  }
  auto row = [&](int i, V3<S> d) {
    if (i < o.np) {
      const S t = dot(d, dv);
      return s[i] == S(0) ? S(0) : s[i] * t;
    }
    return i < o.nr ? dot(d, wr) : S(0);
  };
  out[0] = row(0, rec_v3<6>(E.rec, lane));
  out[1] = row(1, rec_v3<9>(E.rec, lane));
  out[2] = row(2, rec_v3<12>(E.rec, lane));
  out[3] = 3 < o.nr ? dot(rec_v3<15>(E.rec, lane), wr) : S(0);
  out[4] = 4 < o.nr ? dot(rec_v3<18>(E.rec, lane), wr) : S(0);
}

// J_i H^-1 J_i^T (shifted H; rigid bodies carry no shift) for this lane's rows.
template <class R, class S>
__device__ __forceinline__ void quads(const Env<R, S>& E, const Obj& o, int lane, const S (&s)[3], S (&q)[kRows]) {
  const Rec<S> rc = rec_load(E.rec, lane);
#pragma unroll
  for (int i = 0; i < kRows; ++i) {
    q[i] = S(0);
    if (i < o.np) {
      if (s[i] != S(0)) q[i] = point_quad(E.T, E.biwi, o.a, o.b, s[i] * rc.d[i], rc.arm_a, rc.arm_b, true, E.bhi);
    } else if (i < o.nr) {
      S t = S(0);
      if (o.a >= 0) t += sym_quad_t(E.biwi + 6 * o.a, rc.d[i]);
      if (o.b >= 0) t += sym_quad_t(E.biwi + 6 * o.b, rc.d[i]);
      q[i] = t;
    }
  }
}

// Assembly of this lane's object at the current iterate (newton.cpp:100-231):
// writes the record (arms, row directions), the row scales s, h and the C
// diagonal per row, and accumulates the telemetry maxima / |h|^2.
template <class R, class S>
__device__ __forceinline__ void assemble_obj(const Env<R, S>& E, const Obj& o, int lane, const R* jframe, const R* jparam,
                                             const R* cgeo, R h, const Cfg& cfg, const R (&lam)[kRows], R (&s)[3],
                                             R (&hv)[kRows], R (&cd)[kRows], AsmStats& st) {
  s[0] = s[1] = s[2] = R(1);
  if (o.kind < 0) return;
  auto pos = [&](int b) { return lds3(E.bq + 8 * b); };
  auto rot = [&](int b) {
    M3<R> m;
#pragma unroll
    for (int i = 0; i < 9; ++i) m.a[i] = E.brot[9 * b + i];
    return m;
  };
  if (o.kind == 4) {  // contact rows (newton.cpp:166-218)
    const R* g = cgeo + 17 * o.idx;
    const V3<R> la = lds3(g), lb = lds3(g + 3), n = lds3(g + 6), d1 = lds3(g + 9), d2 = lds3(g + 12);
    const R thick = g[15], mu = g[16];
    V3<R> pa = la, pb = lb, ra = v3(R(0), R(0), R(0)), rb = ra;
    if (o.a >= 0) {
      ra = mul(rot(o.a), la);
      pa = pos(o.a) + ra;
    }
    if (o.b >= 0) {
      rb = mul(rot(o.b), lb);
      pb = pos(o.b) + rb;
    }
    rec3_put(E.rec, 0, lane, ra);
    rec3_put(E.rec, 3, lane, rb);
    rec3_put(E.rec, 6, lane, n);
    rec3_put(E.rec, 9, lane, d1);
    rec3_put(E.rec, 12, lane, d2);
    const R gap = dot(n, pa - pb) - thick;
    const R lam_n = lam[0] / h;
    const R rn = r_factor(point_quad(E.T, E.biwi, o.a, o.b, n, ra, rb, false), h, true, cfg.r_strategy);
    const PhiV<R> phi = phi_n(gap, lam_n, rn, cfg.ncp_kind);
    const R hn = phi.v / h;
    hv[0] = hn;
    cd[0] = phi.dl / (h * h);
    s[0] = phi.dc;  // normal J row kept iff dphi/dC != 0 (newton.cpp:187)
    st.comp = fmax(st.comp, (double)ab(mn(gap, lam_n)));
    const R lf0 = lam[1] / h, lf1 = lam[2] / h;
    const R mu_ln = mu * lam_n;
    const R lfn = sqrt(lf0 * lf0 + lf1 * lf1);
    st.cone = fmax(st.cone, (double)mx(R(0), lfn - mu_ln));
    R h1, h2;
    if (mu_ln > R(0)) {  // friction active (newton.cpp:200-210)
      V3<R> dv = v3(R(0), R(0), R(0));
      if (o.a >= 0) dv = lds3(E.bu + 6 * o.a) + cross(lds3(E.bu + 6 * o.a + 3), ra);
      if (o.b >= 0) {
        dv = dv - lds3(E.bu + 6 * o.b);
        dv = dv - cross(lds3(E.bu + 6 * o.b + 3), rb);
      }
      const R v0 = dot(d1, dv), v1 = dot(d2, dv);
      const R q1 = point_quad(E.T, E.biwi, o.a, o.b, d1, ra, rb, false);
      const R q2 = point_quad(E.T, E.biwi, o.a, o.b, d2, ra, rb, false);
      const R rf = r_factor(R(0.5) * (q1 + q2), h, false, cfg.r_strategy);
      const R wv = friction_W(sqrt(v0 * v0 + v1 * v1), lfn, mu_ln, rf, cfg.ncp_kind);
      h1 = v0 + wv * lf0;
      h2 = v1 + wv * lf1;
      cd[1] = cd[2] = wv / h;
      s[1] = s[2] = R(1);
    } else {
      h1 = lf0;
      h2 = lf1;
      cd[1] = cd[2] = R(1) / h;
      s[1] = s[2] = R(0);
    }
    hv[1] = h1;
    hv[2] = h2;
    st.hmax = fmax(st.hmax, fmax((double)ab(hn), fmax((double)ab(h1), (double)ab(h2))));
    st.hsq += (double)hn * hn + (double)h1 * h1 + (double)h2 * h2;
    return;
  }
  // joint rows (constraints.cpp:141-220; newton.cpp:118-128)
  const int j = o.idx, kind = o.kind;
  const R* fr = jframe + 21 * j;
  const V3<R> anc_a = lds3(fr), anc_b = lds3(fr + 3), ax_a = lds3(fr + 6), ax_a2 = lds3(fr + 9), ax_b1 = lds3(fr + 12),
              ax_b2 = lds3(fr + 15), rest = lds3(fr + 18);
  const M3<R> Ra = o.a >= 0 ? rot(o.a) : m3_identity<R>(), Rb = o.b >= 0 ? rot(o.b) : m3_identity<R>();
  V3<R> wa = anc_a, wb = anc_b, ra = v3(R(0), R(0), R(0)), rb = ra;
  if (o.a >= 0) {
    ra = mul(Ra, anc_a);
    wa = pos(o.a) + ra;
  }
  if (o.b >= 0) {
    rb = mul(Rb, anc_b);
    wb = pos(o.b) + rb;
  }
  const R comp = jparam[2 * j];
  const R e_bend = jparam[2 * j + 1] > R(0) ? R(1) / jparam[2 * j + 1] : R(0);
  const V3<R> axw = o.a < 0 ? ax_a : mul(Ra, ax_a);
  rec3_put(E.rec, 0, lane, kind == 2 && o.a >= 0 ? ra - (wa - wb) : ra);  // prismatic: (r_a - t) x d
  rec3_put(E.rec, 3, lane, rb);
  auto emit = [&](int k, R value, R e) {
    const R hk = (value + e * (lam[k] / h)) / h;
    hv[k] = hk;
    cd[k] = e / (h * h);
    st.hmax = fmax(st.hmax, (double)ab(hk));
    st.hsq += (double)hk * (double)hk;
  };
  auto point = [&](int k, V3<R> d, R value) {
    rec3_put(E.rec, 6 + 3 * k, lane, d);
    emit(k, value, comp);
  };
  auto axis = [&](int k, V3<R> xa, V3<R> xb, R restv, R e) {
    rec3_put(E.rec, 6 + 3 * k, lane, cross(xa, xb));
    emit(k, dot(xa, xb) - restv, e);
  };
  const V3<R> e0 = v3(R(1), R(0), R(0)), e1 = v3(R(0), R(1), R(0)), e2 = v3(R(0), R(0), R(1));
  if (kind == 0 || kind == 1) {
    point(0, e0, wa.x - wb.x);
    point(1, e1, wa.y - wb.y);
    point(2, e2, wa.z - wb.z);
    if (kind == 1) {
      const V3<R> b1 = o.b < 0 ? ax_b1 : mul(Rb, ax_b1), b2 = o.b < 0 ? ax_b2 : mul(Rb, ax_b2);
      axis(3, axw, b1, rest.x, comp);
      axis(4, axw, b2, rest.y, comp);
    }
  } else if (kind == 2) {
    int sm = 0;  // tangent_basis(axis) (constraints.cpp:93-101)
    if (ab(axw.y) < ab(axw.x)) sm = 1;
    if (ab(axw.z) < ab(axw[sm])) sm = 2;
    V3<R> ee = v3(R(0), R(0), R(0));
    ee[sm] = R(1);
    const V3<R> t1 = normalize(ee - dot(ee, axw) * axw);
    const V3<R> t2 = cross(axw, t1);
    const V3<R> d = wa - wb;
    point(0, t1, dot(t1, d));
    point(1, t2, dot(t2, d));
    const V3<R> a2 = o.a < 0 ? ax_a2 : mul(Ra, ax_a2);
    const V3<R> b1 = o.b < 0 ? ax_b1 : mul(Rb, ax_b1), b2 = o.b < 0 ? ax_b2 : mul(Rb, ax_b2);
    axis(2, axw, b1, rest.x, comp);
    axis(3, axw, b2, rest.y, comp);
    axis(4, a2, b2, rest.z, comp);
  } else {
    const V3<R> b1 = o.b < 0 ? ax_b1 : mul(Rb, ax_b1), b2 = o.b < 0 ? ax_b2 : mul(Rb, ax_b2);
    axis(0, axw, b1, rest.x, e_bend);
    axis(1, axw, b2, rest.y, e_bend);
  }
}

// Refresh the rotation cache of body b from its quaternion.
template <class R, class S> __device__ __forceinline__ void refresh_rot(const Env<R, S>& E, int b) {
  const R* t = E.bq + 8 * b + 3;
  const M3<R> m = quat_rot(t[0], t[1], t[2], t[3]);
#pragma unroll
  for (int i = 0; i < 9; ++i) E.brot[9 * b + i] = m.a[i];
}

// Inputs/outputs of one environment's step (views into the batch's slabs).
template <class R> struct EnvIO {
  const R* q0;     // step-start coordinates (cold slab)
  const R* u0;     // step-start velocities
  const R* ut;     // unconstrained velocity u~ (newton_setup in the narrow-phase launch)
  const R* iw6;    // I_w per rigid dof3 block (cold), sym 6
  const R* iwi6;   // I_w^-1 per rigid dof3 block (hot)
  const int* cbody;
  const R* cgeo;
  R* lam;          // [row][lane] multipliers, 5 x 32 (global scratch, per Newton iteration)
  const int* jinc_off;  // static joint incidence per body: joint * 2 + side (both sides)
  const int* jinc;
  R* g;            // ndof scratch (cold)
  R* du;           // ndof scratch (cold)
  R* qs;           // persistent state (out)
  R* us;
  R* q_out;        // optional mapped host copies
  R* u_out;
  R* xlam;         // exported multipliers (reference row order)
  int* xcbody;
  double* fin;     // 8
  IterOut* iters;  // newton_iterations or null
  unsigned long long* cr_iters;  // sum of PCR iterations (batch counter) or null
  unsigned long long* cr_cycles; // clock64 cycles inside the PCR loops (lane 0) or null
  unsigned long long* env_cycles;
  unsigned long long* phase;     // kWPhases counters (NSD_PHASE_TIMING) or null
};

// Diagnostics (NSD_PHASE_TIMING): lane 0's clock64 cycles per solver phase.
struct WClock {
  unsigned long long* dst;
  long long t0;
  __device__ explicit WClock(unsigned long long* d) : dst(d), t0(0) {
    if (dst) t0 = clock64();
  }
  __device__ __forceinline__ void mark(int k) {
    if (dst) {
      const long long t = clock64();
      atomicAdd(dst + k, static_cast<unsigned long long>(t - t0));
      t0 = t;
    }
  }
};

// Lane-private row vector in shared memory ([row][lane]).
template <class R> __device__ __forceinline__ void rows_load(const R* v, int lane, R (&o)[kRows]) {
#pragma unroll
  for (int i = 0; i < kRows; ++i) o[i] = v[32 * i + lane];
}

// Body b's gradient block g = M~(u - u~) - J^T lambda (after staging lambda);
// accumulates residual_inf / |g|^2 in the reference's order (bodies rigid).
template <class R, class S>
__device__ __forceinline__ void body_grad(const Topo<R>& T, const Env<R, S>& E, const EnvIO<R>& io, int b, V3<R>& gl,
                                          V3<R>& ga, double& gmax, double& gsq) {
  const int d = T.bdof[b];
  V3<R> jl, ja;
  gather(E, b, jl, ja);
  const R m = T.bmass[b];
  const V3<R> du = lds3(E.bu + 6 * b) - lds3(io.ut + d);
  gl = v3(m * du.x, m * du.y, m * du.z) - jl;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    gmax = fmax(gmax, (double)(ab(gl[k]) / m));
    gsq += (double)gl[k] * (double)gl[k];
  }
  const R* s6 = io.iw6 + 6 * (d / 3 + 1);
  const V3<R> da = lds3(E.bu + 6 * b + 3) - lds3(io.ut + d + 3);
  ga = sym_mul(s6, da) - ja;
  gmax = fmax(gmax, fmax((double)(ab(ga.x) / s6[0]), fmax((double)(ab(ga.y) / s6[1]), (double)(ab(ga.z) / s6[2]))));
  gsq += (double)ga.x * ga.x + (double)ga.y * ga.y + (double)ga.z * ga.z;
}

template <class R, class S>
__device__ void solve_env(const Topo<R>& T, const Cfg& cfg, const R* jframe, R h, Env<R, S>& E, const EnvIO<R>& io,
                          int lane) {
  const int nb = T.nb, nj = T.nj, nc = E.nc;
  const long long t_env0 = io.env_cycles ? clock64() : 0;
  WClock pc(lane == 0 ? io.phase : nullptr);
  // ---- step-start state into shared memory: q = q-, u = 0 (zero start, newton.cpp:327-338)
  if (lane < nb) {
    const int b = lane, cdd = T.bcoord[b], d = T.bdof[b];
    R* q = E.bq + 8 * b;
#pragma unroll
    for (int k = 0; k < 7; ++k) q[k] = io.q0[cdd + k];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      E.bu[6 * b + k] = R(0);
      E.biwi[6 * b + k] = io.iwi6[6 * (d / 3 + 1) + k];
    }
    refresh_rot(E, b);
    E.bhi[b] = R(1) / (T.bmass[b] + R(0));
    // body b's staged wrenches: its joints' sides, then its contacts' sides ascending
    const int nji = io.jinc_off[b + 1] - io.jinc_off[b];
    int n = nji;
    for (int c = 0; c < nc; ++c) n += (io.cbody[2 * c] == b) + (io.cbody[2 * c + 1] == b);
    E.gent_off[b + 1] = n;
  }
#pragma unroll
  for (int i = 0; i < kRows; ++i) {
    io.lam[32 * i + lane] = R(0);
    E.x[32 * i + lane] = R(0);
    E.bx[32 * i + lane] = R(0);
  }
  __syncwarp();
  if (lane == 0) {
    E.gent_off[0] = 0;
    for (int b = 0; b < nb; ++b) E.gent_off[b + 1] += E.gent_off[b];
  }
  __syncwarp();
  if (lane < nb) {
    int o = E.gent_off[lane];
    for (int e = io.jinc_off[lane]; e < io.jinc_off[lane + 1]; ++e) {
      const int ent = io.jinc[e];  // joint * 2 + side
      E.gent[o++] = kStg * (ent >> 1) + 6 * (ent & 1);
    }
    for (int c = 0; c < nc; ++c) {
      if (io.cbody[2 * c] == lane) E.gent[o++] = kStg * (nj + c);
      if (io.cbody[2 * c + 1] == lane) E.gent[o++] = kStg * (nj + c) + 6;
    }
  }
  // ---- this lane's object and its rows in the reference layout (newton.cpp:18-41)
  Obj o{};
  o.kind = -1;
  o.idx = 0;
  o.a = o.b = -1;
  o.np = o.na = o.nr = 0;
  int row0 = 0, row1 = 0;  // joint: rows row0..; contact: normal row0, friction row1, row1 + 1
  if (lane < nj) {
    o.kind = T.jkind[lane];
    o.idx = lane;
    o.a = T.jbody[2 * lane];
    o.b = T.jbody[2 * lane + 1];
    o.np = o.kind <= 1 ? 3 : (o.kind == 2 ? 2 : 0);
    o.nr = joint_nrows(o.kind);
    o.na = o.nr - o.np;
    row0 = T.jrow[lane];
    row1 = row0 + 1;
  } else if (lane < nj + nc) {
    const int c = lane - nj;
    o.kind = 4;
    o.idx = c;
    o.a = io.cbody[2 * c];
    o.b = io.cbody[2 * c + 1];
    o.np = o.nr = 3;
    row0 = T.rows_static + c;
    row1 = T.rows_static + nc + 2 * c;
  }
  const R tfrac = R(cfg.step_fraction);
  const int maxlin = cfg.linear_max_iterations;
  R s[3], cd[kRows];
  long long cr_cyc = 0;
  unsigned cr_it = 0;
  int n_done = 0, aborted = 0;
  __syncwarp();
  for (int it = 0; it < cfg.newton_iterations; ++it) {
    // ---- assemble (rotation cache refreshed after every integration)
    R hv[kRows];
    AsmStats as{0.0, 0.0, 0.0, 0.0};
    pc.mark(0);
    {  // lambda is re-read for the update: not kept in registers across the PCR loop
      R lam[kRows];
      rows_load(io.lam, lane, lam);
      assemble_obj(E, o, lane, jframe, T.jparam, io.cgeo, h, cfg, lam, s, hv, cd, as);
      pc.mark(1);
      // ---- g = M~(u - u~) - J^T lambda; H^-1 = M~^-1 (no shift on rigid dofs); w = H^-1 g
      stage(E, o, lane, s, lam);
    }
    __syncwarp();
    double gmax = 0.0, gsq = 0.0;
    if (lane < nb) {
      const int b = lane, d = T.bdof[b];
      V3<R> gl, ga;
      body_grad(T, E, io, b, gl, ga, gmax, gsq);
      sts3(io.g + d, gl);
      sts3(io.g + d + 3, ga);
      const R hi = E.bhi[b];
      S* w = E.bw + 6 * b;
      sts3(w, cv3<S>(v3(gl.x * hi, gl.y * hi, gl.z * hi)));
      sts3(w + 3, cv3<S>(sym_mul(E.biwi + 6 * b, ga)));
    }
    double s_g = gsq, s_h = as.hsq;
    wsum2(s_g, s_h);
    IterOut st;
    st.residual_inf = wmax(fmax(gmax, as.hmax));
    st.merit_l2 = sqrt(s_g + s_h);
    st.comp_error_max = wmax(as.comp);
    st.cone_violation_max = wmax(as.cone);
    st.linear_iterations = 0;
    st.linear_residual = 0.0;
    st.linear_breakdown = 0;
    st.step_size = 0.0;
    __syncwarp();
    pc.mark(2);
    // ---- Schur rhs b = J H^-1 g - h, diagonal preconditioner, r = b, x = 0, z = M^-1 r.
    // The PCR recurrence (row vectors, preconditioner, C diagonal) runs in R; the
    // operator's products J^T y, H^-1, J w in S (the scales cast once): with S = float
    // the operator is rounded at 1e-7 while the recurrence keeps its fp64 floor, so
    // its exits (monotone guard, tolerance) stay those of the fp64 solve.
    R r[kRows], z[kRows], p[kRows], ap[kRows], az[kRows], inv[kRows];
    S ss[3];
    const R eps = R(cfg.epsilon_reg);
#pragma unroll
    for (int i = 0; i < 3; ++i) ss[i] = S(s[i]);
    {
      S jwv[kRows], qd[kRows];
      jw(E, o, lane, ss, jwv);
      quads(E, o, lane, ss, qd);
      double rr = 0.0, rzr = 0.0;
#pragma unroll
      for (int i = 0; i < kRows; ++i) {
        p[i] = ap[i] = az[i] = R(0);
        inv[i] = r[i] = z[i] = R(0);
        E.x[32 * i + lane] = R(0);
        E.bx[32 * i + lane] = R(0);
        if (i < o.nr) {
          const R bi = R(jwv[i]) - hv[i];
          R iv = R(1);
          if (cfg.preconditioner == 1) {
            const R sd = R(qd[i]) + cd[i] + eps;
            iv = sd > R(0) ? R(1) / sd : R(1);
          }
          inv[i] = iv;
          r[i] = bi;
          z[i] = iv * bi;
          rr += (double)bi * bi;
          rzr += (double)bi * (double)(iv * bi);
        }
      }
      wsum2(rr, rzr);
      pc.mark(3);
      double hist_last = sqrt(rr), phist_last = sqrt(rzr), best_res = hist_last;
      int lin_used = 0, breakdown = 0;
      const long long tc0 = io.cr_cycles ? clock64() : 0;
      if (maxlin > 0 && hist_last > cfg.linear_tolerance) {
        // az = A z, zaz = z . az (solvers.cpp PCR setup)
        stage_f(E, o, lane, ss, [&](int i) { return S(z[i]); });
        __syncwarp();
        bodies_w(E, lane);
        __syncwarp();
        S jz[kRows];
        jw(E, o, lane, ss, jz);
        double za = 0.0;
#pragma unroll
        for (int i = 0; i < kRows; ++i)
          if (i < o.nr) {
            az[i] = R(jz[i]) + cd[i] * z[i] + eps * z[i];
            za += (double)z[i] * az[i];
          }
        double zaz = wsum(za), beta = 0.0;
        pc.mark(4);
        for (int itl = 0; itl < maxlin && hist_last > cfg.linear_tolerance; ++itl) {
          // p = z + beta p, ap = az + beta ap; den = ap . M^-1 ap
          const R rb = R(beta);
          double den = 0.0;
#pragma unroll
          for (int i = 0; i < kRows; ++i)
            if (i < o.nr) {
              if (itl == 0) {
                p[i] = z[i];
                ap[i] = az[i];
              } else {
                p[i] = z[i] + rb * p[i];
                ap[i] = az[i] + rb * ap[i];
              }
              den += (double)ap[i] * (double)(inv[i] * ap[i]);
            }
          den = wsum(den);
          pc.mark(5);
          if (fabs(den) < 1e-300) {
            breakdown = 1;
            break;
          }
          const double alpha = zaz / den;
          const R ra = R(alpha);
          // trial r' = r - a ap, z' = z - a M^-1 ap and its norms; J^T z' staged
          // speculatively in the same pass (a rejected trial discards it)
          double pn2 = 0.0, rn2 = 0.0;
#pragma unroll
          for (int i = 0; i < kRows; ++i)
            if (i < o.nr) {
              const R rv = r[i] - ra * ap[i];
              pn2 += (double)rv * (double)(inv[i] * rv);
              rn2 += (double)rv * rv;
            }
          const bool zaz_ok = fabs(zaz) >= 1e-300;
          if (zaz_ok) stage_f(E, o, lane, ss, [&](int i) { return S(z[i] - ra * (inv[i] * ap[i])); });
          wsum2(pn2, rn2);
          pc.mark(6);
          const double pn = sqrt(pn2);
          if (pn > phist_last) break;  // monotone guard (no breakdown flag)
          hist_last = sqrt(rn2);
          phist_last = pn;
          const bool best = hist_last < best_res;
          if (best) best_res = hist_last;
#pragma unroll
          for (int i = 0; i < kRows; ++i) {  // accept: the trial's expressions, same bits
            const R xi = E.x[32 * i + lane] + ra * p[i];
            E.x[32 * i + lane] = xi;
            if (best) E.bx[32 * i + lane] = xi;
            r[i] = r[i] - ra * ap[i];
            z[i] = z[i] - ra * (inv[i] * ap[i]);
          }
          pc.mark(7);
          lin_used = itl + 1;
          if (!zaz_ok) {
            breakdown = 1;
            break;
          }
          __syncwarp();
          bodies_w(E, lane);
          __syncwarp();
          pc.mark(8);
          S jz2[kRows];
          jw(E, o, lane, ss, jz2);
          double za2 = 0.0;
#pragma unroll
          for (int i = 0; i < kRows; ++i)
            if (i < o.nr) {
              az[i] = R(jz2[i]) + cd[i] * z[i] + eps * z[i];
              za2 += (double)z[i] * az[i];
            }
          za2 = wsum(za2);
          beta = za2 / zaz;
          zaz = za2;
          pc.mark(9);
        }
      }
      if (io.cr_cycles) cr_cyc += clock64() - tc0;
      pc.mark(3);
      cr_it += lin_used;
      st.linear_iterations = lin_used;
      st.linear_breakdown = breakdown;
      st.linear_residual = hist_last;
    }
    // ---- du = H^-1 (J^T dlambda - g); NaN check (newton.cpp:295,362-369)
    R bx[kRows];
    rows_load(E.bx, lane, bx);
    double dl2 = 0.0, du2 = 0.0, bad = 0.0;
#pragma unroll
    for (int i = 0; i < kRows; ++i)
      if (i < o.nr) {
        dl2 += (double)bx[i] * bx[i];
        if (!isfinite(bx[i])) bad = 1.0;
      }
    __syncwarp();
    stage(E, o, lane, s, bx);
    __syncwarp();
    if (lane < nb) {
      const int b = lane, d = T.bdof[b];
      V3<R> lin, ang;
      gather(E, b, lin, ang);
      const R hi = E.bhi[b];
      const V3<R> rl = lin - lds3(io.g + d);
      const V3<R> dl = v3(rl.x * hi, rl.y * hi, rl.z * hi);
      const V3<R> da = sym_mul(E.biwi + 6 * b, ang - lds3(io.g + d + 3));
      du2 += (double)dl.x * dl.x + (double)dl.y * dl.y + (double)dl.z * dl.z;
      du2 += (double)da.x * da.x + (double)da.y * da.y + (double)da.z * da.z;
      if (!isfinite(dl.x) || !isfinite(dl.y) || !isfinite(dl.z) || !isfinite(da.x) || !isfinite(da.y) ||
          !isfinite(da.z))
        bad = 1.0;
      sts3(io.du + d, dl);
      sts3(io.du + d + 3, da);
    }
    wsum2(dl2, du2);
    bad = wmax(bad);
    pc.mark(10);
    if (bad != 0.0) {  // rollback to q-, u- (newton.cpp:362-369)
      if (lane == 0 && io.iters) io.iters[it] = st;
      aborted = 1;
      n_done = it + 1;
      break;
    }
    // ---- damped update + integration (newton.cpp:393-396; bodies.cpp:58-86)
#pragma unroll
    for (int i = 0; i < kRows; ++i) io.lam[32 * i + lane] = io.lam[32 * i + lane] + tfrac * bx[i];
    if (lane < nb) {
      const int b = lane, d = T.bdof[b], cdd = T.bcoord[b];
      R* u = E.bu + 6 * b;
#pragma unroll
      for (int k = 0; k < 6; ++k) u[k] += tfrac * io.du[d + k];
      R* q = E.bq + 8 * b;
#pragma unroll
      for (int k = 0; k < 3; ++k) q[k] = io.q0[cdd + k] + h * u[k];
      const R t0 = q[3], t1 = q[4], t2 = q[5], t3 = q[6];
      const R ox = u[3], oy = u[4], oz = u[5];
      R nq[4];
      nq[0] = io.q0[cdd + 3] + h * (R(0.5) * (-t1 * ox - t2 * oy - t3 * oz));
      nq[1] = io.q0[cdd + 4] + h * (R(0.5) * (t0 * ox + t3 * oy - t2 * oz));
      nq[2] = io.q0[cdd + 5] + h * (R(0.5) * (-t3 * ox + t0 * oy + t1 * oz));
      nq[3] = io.q0[cdd + 6] + h * (R(0.5) * (t2 * ox - t1 * oy + t0 * oz));
      const R nn = sqrt(nq[0] * nq[0] + nq[1] * nq[1] + nq[2] * nq[2] + nq[3] * nq[3]);
      if ((double)nn < 1e-300) {
        nq[0] = R(1);
        nq[1] = nq[2] = nq[3] = R(0);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) nq[k] = nq[k] / nn;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) q[3 + k] = nq[k];
      refresh_rot(E, b);
    }
    st.step_size = (double)tfrac * sqrt(du2 + dl2);
    if (lane == 0 && io.iters) io.iters[it] = st;
    n_done = it + 1;
    __syncwarp();
    pc.mark(11);
  }
  if (aborted) {
    if (lane < nb) {  // q = q-, u = u-
      const int b = lane, cdd = T.bcoord[b], d = T.bdof[b];
#pragma unroll
      for (int k = 0; k < 7; ++k) E.bq[8 * b + k] = io.q0[cdd + k];
#pragma unroll
      for (int k = 0; k < 6; ++k) E.bu[6 * b + k] = io.u0[d + k];
    }
    if (lane == 0) {
      io.fin[5] = 1.0;
      io.fin[6] = 0.0;
      io.fin[7] = n_done;
    }
  } else {
    // ---- final assembly for classification and telemetry (newton.cpp:409-416)
    R hv[kRows], lam[kRows];
    AsmStats fs{0.0, 0.0, 0.0, 0.0};
    rows_load(io.lam, lane, lam);
    assemble_obj(E, o, lane, jframe, T.jparam, io.cgeo, h, cfg, lam, s, hv, cd, fs);
    stage(E, o, lane, s, lam);
    __syncwarp();
    double gmax = 0.0, gsq = 0.0;
    if (lane < nb) {
      V3<R> gl, ga;
      body_grad(T, E, io, lane, gl, ga, gmax, gsq);
    }
    double mgap = __builtin_huge_val();
    if (o.kind == 4) {
      const R* g = io.cgeo + 17 * o.idx;
      auto arm = [&](int b, V3<R> l) {  // the arm of the final assembly, in R
        M3<R> m;
#pragma unroll
        for (int i = 0; i < 9; ++i) m.a[i] = E.brot[9 * b + i];
        return mul(m, l);
      };
      const V3<R> pa = o.a < 0 ? lds3(g) : lds3(E.bq + 8 * o.a) + arm(o.a, lds3(g));
      const V3<R> pb = o.b < 0 ? lds3(g + 3) : lds3(E.bq + 8 * o.b) + arm(o.b, lds3(g + 3));
      mgap = (double)(dot(lds3(g + 6), pa - pb) - g[15]);
    }
    const double fr = wmax(fmax(gmax, fs.hmax)), fcomp = wmax(fs.comp), fcone = wmax(fs.cone);
    mgap = -wmax(-mgap);
    if (lane == 0) {
      io.fin[0] = fr;
      io.fin[1] = fcomp;
      io.fin[2] = fcone;
      io.fin[3] = nc ? mgap : 0.0;
      io.fin[4] = 0.0;  // no geometric-stiffness shift on rigid dofs (newton.cpp:316-317)
      io.fin[5] = 0.0;
      io.fin[6] = fr < cfg.newton_tolerance ? 1.0 : 0.0;
      io.fin[7] = n_done;
    }
  }
  __syncwarp();
  pc.mark(12);
  // ---- write-back: state, mapped host copies, multipliers in the reference row order
  if (lane < nb) {
    const int b = lane, cdd = T.bcoord[b], d = T.bdof[b];
#pragma unroll
    for (int k = 0; k < 7; ++k) io.qs[cdd + k] = E.bq[8 * b + k];
#pragma unroll
    for (int k = 0; k < 6; ++k) io.us[d + k] = E.bu[6 * b + k];
    if (io.q_out)
#pragma unroll
      for (int k = 0; k < 7; ++k) io.q_out[cdd + k] = E.bq[8 * b + k];
    if (io.u_out)
#pragma unroll
      for (int k = 0; k < 6; ++k) io.u_out[d + k] = E.bu[6 * b + k];
  }
#pragma unroll
  for (int i = 0; i < kRows; ++i)
    if (i < o.nr) io.xlam[o.kind == 4 ? (i == 0 ? row0 : row1 + i - 1) : row0 + i] = io.lam[32 * i + lane];
  for (int i = lane; i < 2 * nc; i += 32) io.xcbody[i] = io.cbody[i];
  pc.mark(13);
  if (lane == 0) {
    if (io.cr_iters) {
      atomicAdd(io.cr_iters, (unsigned long long)cr_it);
      atomicAdd(io.cr_iters + 3, (unsigned long long)cr_it * (unsigned long long)nc);  // for the nc-weighted bytes
    }
    if (io.cr_cycles) atomicAdd(io.cr_cycles, (unsigned long long)cr_cyc);
    if (io.env_cycles) atomicAdd(io.env_cycles, (unsigned long long)(clock64() - t_env0));
  }
}

}  // namespace wp
}  // namespace nsd
