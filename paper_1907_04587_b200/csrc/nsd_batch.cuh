// Batched rigid-body environments: one warp per environment, object-centric.
//
// Same Newton step as nsd_engine.cuh (newton.cpp:321-418, solvers.cpp:127-174)
// re-organised for tiny scenes (an ant: 9 bodies, 8 joints / 40 rows, ~16
// contacts / 48 rows) where per-row indirection dominates:
//   * every constraint object (joint, contact) is owned by one lane, which
//     owns its rows: all PCR row vectors are lane-private (no cross-lane row
//     traffic; the accepted PCR update is committed by the owner lane inside
//     the next operator pass);
//   * J^T z goes through per-object staging — a joint's four 3-wide slot
//     vectors, a contact's force and two lever-arm torques — gathered by the
//     body lanes in a fixed order (deterministic, no atomics);
//   * J w is evaluated per object: joint rows through their slot
//     coefficients, contact rows through one relative contact-point velocity.
// The environment's hot working set lives in shared memory; the three PCR
// reductions per iteration are warp shuffles.
#pragma once

#include "nsd_engine.cuh"

namespace nsd {

template <class R> struct ObjView {
  Work<R> W;
  R* jstage;        // 12 per joint: slot vectors a.lin a.ang b.lin b.ang
  R* cstage;        // 9 per contact: f, r_a x f, r_b x f
  const int* jbinc_off;  // static joint incidence per body (nb + 1)
  const int* jbinc;      // joint*2 + side
  int* cbinc_off;   // contact incidence per body (nb + 1)
  int* cbinc;       // contact*2 + side
};

// Vector loads of one 16-byte-aligned record (float4 / 2 x double2 per 4 values).
__device__ __forceinline__ void ld4(const float* p, float (&o)[4]) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  o[0] = v.x;
  o[1] = v.y;
  o[2] = v.z;
  o[3] = v.w;
}
__device__ __forceinline__ void ld4(const double* p, double (&o)[4]) {
  const double2 a = *reinterpret_cast<const double2*>(p), c = *reinterpret_cast<const double2*>(p + 2);
  o[0] = a.x;
  o[1] = a.y;
  o[2] = c.x;
  o[3] = c.y;
}

// Contact view from the batched record (W.crec, W.cblk): 5 vector loads + 1 int4.
template <class R> __device__ __forceinline__ CView<R> contact_rec_view(const Work<R>& W, int c) {
  R v[20];
  const R* rc = W.crec + 20 * c;
#pragma unroll
  for (int k = 0; k < 5; ++k) ld4(rc + 4 * k, *reinterpret_cast<R(*)[4]>(v + 4 * k));
  const int4 bk = W.cblk[c];
  CView<R> cv;
  cv.ba = cv.bb = 0;  // unused by the operator paths
  cv.al = bk.x;
  cv.aa = bk.y;
  cv.bl = bk.z;
  cv.bA = bk.w;
  cv.n = v3(v[0], v[1], v[2]);
  cv.d1 = v3(v[3], v[4], v[5]);
  cv.d2 = v3(v[6], v[7], v[8]);
  cv.ra = v3(v[9], v[10], v[11]);
  cv.rb = v3(v[12], v[13], v[14]);
  cv.dc = v[15];
  cv.act = v[16];
  return cv;
}

// Structured joint (W.jstr, written by assemble_joint): bodies' dof3 blocks, the
// point / axis row counts of the kind (joint_rows, constraints.cpp:141-220) and
// the 24 values: arm_a, arm_b, point directions D0..D2, axis vectors C0..C2.
template <class R> struct JView {
  int al, aa, bl, bA, np, na;
  const R* s;
};
template <class R> __device__ __forceinline__ JView<R> joint_view(const Topo<R>& T, const Work<R>& W, int j) {
  JView<R> v;
  const int4 bk = W.jblk[j];  // static table: one int4 instead of body -> dof -> type chains
  v.al = bk.x;
  v.aa = bk.y;
  v.bl = bk.z;
  v.bA = bk.w;
  const int kind = T.jkind[j];
  v.np = kind <= 1 ? 3 : (kind == 2 ? 2 : 0);
  v.na = kind == 0 ? 0 : (kind == 2 ? 3 : 2);
  v.s = W.jstr + 24 * j;
  return v;
}

// Runs f(row) over the rows owned by this lane (objects lane, lane+32, ...).
template <class R, class F> __device__ __forceinline__ void for_my_rows(const Topo<R>& T, const Work<R>& W, int rk, int ts,
                                                                        F&& f) {
  const int nobj = T.nj + W.nc;
  for (int k = rk; k < nobj; k += ts) {
    if (k < T.nj) {
      const int r0 = T.jrow[k], n = joint_nrows(T.jkind[k]);
      for (int i = 0; i < n; ++i) f(r0 + i);
    } else {
      const int c = k - T.nj;
      f(W.normal_begin + c);
      f(W.friction_begin + 2 * c);
      f(W.friction_begin + 2 * c + 1);
    }
  }
}

// Stage J^T y per object. YF: row functor; before staging each owned row may be
// transformed by `pre(row)` (the in-place PCR commit), which returns the value.
template <class R, class YF>
__device__ __forceinline__ void stage_objects(const Topo<R>& T, ObjView<R>& O, int rk, int ts, const YF& y) {
  const Work<R>& W = O.W;
  const int nobj = T.nj + W.nc;
  for (int k = rk; k < nobj; k += ts) {
    if (k < T.nj) {
      // J^T y of a joint: point rows sum to a force f at the anchors, axis rows to a torque
      const JView<R> jv = joint_view(T, W, k);
      const int r0 = T.jrow[k];
      V3<R> f = v3(R(0), R(0), R(0)), ta = f;
      for (int i = 0; i < jv.np; ++i) f = f + y(r0 + i) * ld3(jv.s + 6 + 3 * i);
      for (int i = 0; i < jv.na; ++i) ta = ta + y(r0 + jv.np + i) * ld3(jv.s + 15 + 3 * i);
      R* d = O.jstage + 12 * k;
      st3(d, f);
      st3(d + 3, cross(ld3(jv.s), f) + ta);
      st3(d + 6, -f);
      st3(d + 9, -(cross(ld3(jv.s + 3), f) + ta));
    } else {
      const int c = k - T.nj;
      const CView<R> cv = contact_rec_view(W, c);
      const int f0 = W.friction_begin + 2 * c;
      const R yn = cv.dc * y(W.normal_begin + c), y1 = cv.act * y(f0), y2 = cv.act * y(f0 + 1);
      const V3<R> f = v3(yn * cv.n.x + y1 * cv.d1.x + y2 * cv.d2.x, yn * cv.n.y + y1 * cv.d1.y + y2 * cv.d2.y,
                         yn * cv.n.z + y1 * cv.d1.z + y2 * cv.d2.z);
      R* d = O.cstage + 9 * c;
      st3(d, f);
      st3(d + 3, cross(cv.ra, f));
      st3(d + 6, cross(cv.rb, f));
    }
  }
}

// Body-side gather of the staged J^T y: linear and angular parts of body b.
template <class R>
__device__ __forceinline__ void gather_body(const Topo<R>& T, const ObjView<R>& O, int b, V3<R>& lin, V3<R>& ang) {
  lin = v3(R(0), R(0), R(0));
  ang = lin;
  for (int e = O.jbinc_off[b]; e < O.jbinc_off[b + 1]; ++e) {
    const int ent = O.jbinc[e];
    const R* s = O.jstage + 12 * (ent >> 1) + 6 * (ent & 1);
    lin = lin + ld3(s);
    ang = ang + ld3(s + 3);
  }
  if (O.W.nc > 0)
    for (int e = O.cbinc_off[b]; e < O.cbinc_off[b + 1]; ++e) {
      const int ent = O.cbinc[e];
      const R* s = O.cstage + 9 * (ent >> 1);
      if (ent & 1) {
        lin = lin - ld3(s);
        ang = ang - ld3(s + 6);
      } else {
        lin = lin + ld3(s);
        ang = ang + ld3(s + 3);
      }
    }
}

// w = H^-1 J^T y for all bodies (after staging + __syncwarp).
template <class R> __device__ __forceinline__ void bodies_apply_hinv(const Topo<R>& T, ObjView<R>& O, int rk, int ts) {
  Work<R>& W = O.W;
  for (int b = rk; b < T.nb; b += ts) {
    V3<R> lin, ang;
    gather_body(T, O, b, lin, ang);
    const int d = T.bdof[b];
    st3(W.w + d, v3(lin.x * W.hinv[d], lin.y * W.hinv[d + 1], lin.z * W.hinv[d + 2]));
    if (T.btype[b] == 1) st3(W.w + d + 3, sym_mul(W.iwi6 + 6 * (d / 3 + 1), ang));
  }
}

// J w for the rows of one object; calls f(row, value).
template <class R, class F>
__device__ __forceinline__ void object_Jw(const Topo<R>& T, const Work<R>& W, int k, const R* w, F&& f) {
  if (k < T.nj) {
    // relative anchor velocity (point rows) and relative angular velocity (axis rows)
    const JView<R> jv = joint_view(T, W, k);
    const int r0 = T.jrow[k];
    V3<R> dv = v3(R(0), R(0), R(0)), wr = dv;
    if (jv.al >= 0) {
      dv = ld3(w + 3 * jv.al);
      if (jv.aa >= 0) {
        wr = ld3(w + 3 * jv.aa);
        dv = dv + cross(wr, ld3(jv.s));
      }
    }
    if (jv.bl >= 0) {
      dv = dv - ld3(w + 3 * jv.bl);
      if (jv.bA >= 0) {
        const V3<R> wb = ld3(w + 3 * jv.bA);
        dv = dv - cross(wb, ld3(jv.s + 3));
        wr = wr - wb;
      }
    }
    for (int i = 0; i < jv.np; ++i) f(r0 + i, dot(ld3(jv.s + 6 + 3 * i), dv));
    for (int i = 0; i < jv.na; ++i) f(r0 + jv.np + i, dot(ld3(jv.s + 15 + 3 * i), wr));
  } else {
    const int c = k - T.nj;
    const CView<R> cv = contact_rec_view(W, c);
    const V3<R> dv = contact_dv(cv, w);
    f(W.normal_begin + c, cv.dc == R(0) ? R(0) : cv.dc * dot(cv.n, dv));
    const bool act = cv.act != R(0);
    f(W.friction_begin + 2 * c, act ? dot(cv.d1, dv) : R(0));
    f(W.friction_begin + 2 * c + 1, act ? dot(cv.d2, dv) : R(0));
  }
}

// J_i H^-1 J_i^T for the rows of one object; calls f(row, value).
template <class R, class F>
__device__ __forceinline__ void object_quad(const Topo<R>& T, const Work<R>& W, int k, F&& f) {
  if (k < T.nj) {
    const JView<R> jv = joint_view(T, W, k);
    const int r0 = T.jrow[k];
    const V3<R> arm_a = ld3(jv.s), arm_b = ld3(jv.s + 3);
    for (int i = 0; i < jv.np; ++i) {  // slot order a.lin, a.ang, b.lin, b.ang as slot_quad
      const V3<R> d = ld3(jv.s + 6 + 3 * i);
      R q = R(0);
      if (jv.al >= 0) q += block_quad(T, W, jv.al, d, true);
      if (jv.aa >= 0) q += block_quad(T, W, jv.aa, cross(arm_a, d), true);
      if (jv.bl >= 0) q += block_quad(T, W, jv.bl, d, true);
      if (jv.bA >= 0) q += block_quad(T, W, jv.bA, cross(arm_b, d), true);
      f(r0 + i, q);
    }
    for (int i = 0; i < jv.na; ++i) {
      const V3<R> c = ld3(jv.s + 15 + 3 * i);
      R q = R(0);
      if (jv.aa >= 0) q += block_quad(T, W, jv.aa, c, true);
      if (jv.bA >= 0) q += block_quad(T, W, jv.bA, c, true);
      f(r0 + jv.np + i, q);
    }
  } else {
    const int c = k - T.nj;
    const CView<R> cv = contact_rec_view(W, c);
    f(W.normal_begin + c, cv.dc == R(0) ? R(0) : contact_quad(T, W, cv, cv.dc * cv.n, true));
    const bool act = cv.act != R(0);
    f(W.friction_begin + 2 * c, act ? contact_quad(T, W, cv, cv.d1, true) : R(0));
    f(W.friction_begin + 2 * c + 1, act ? contact_quad(T, W, cv, cv.d2, true) : R(0));
  }
}

// g = M~(u - u~) - J^T lambda (after staging lambda) for body b; returns the
// residual_inf and |g|^2 contributions; also refreshes H^-1 and w = H^-1 g.
template <class R>
__device__ __forceinline__ void body_momentum(const Topo<R>& T, ObjView<R>& O, int b, bool gs, bool write,
                                              double& gmax, double& gsq, double& smin) {
  Work<R>& W = O.W;
  V3<R> jl_lin, jl_ang;
  gather_body(T, O, b, jl_lin, jl_ang);
  const int d = T.bdof[b];
  const R m = T.bmass[b];
  const V3<R> du = ld3(W.u + d) - ld3(W.ut + d);
  const V3<R> gl = v3(m * du.x, m * du.y, m * du.z) - jl_lin;
  if (T.btype[b] == 0 && write) {  // geometric stiffness secant on particle dofs (newton.cpp:299-319)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (gs) {
        const R dd = W.u[d + k] - W.up[d + k];
        R sh = R(0);
        if (!(ab(dd) < R(1e-10))) {
          const R ck = -((gl[k] - W.gp[d + k] + m * dd) / dd);
          sh = -mn(R(0), ck);
        }
        W.shift[d + k] = sh;
        smin = fmin(smin, (double)sh);
      }
      W.gp[d + k] = gl[k];
      W.up[d + k] = W.u[d + k];
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    gmax = fmax(gmax, (double)(ab(gl[k]) / m));
    gsq += (double)gl[k] * (double)gl[k];
  }
  if (write) {
#pragma unroll
    for (int k = 0; k < 3; ++k) W.hinv[d + k] = R(1) / (m + W.shift[d + k]);
    st3(W.g + d, gl);
    st3(W.w + d, v3(gl.x * W.hinv[d], gl.y * W.hinv[d + 1], gl.z * W.hinv[d + 2]));
  }
  if (T.btype[b] == 1) {
    const int ab3 = d / 3 + 1;
    const R* s6 = W.iw6 + 6 * ab3;
    const V3<R> da = ld3(W.u + d + 3) - ld3(W.ut + d + 3);
    const V3<R> ga = sym_mul(s6, da) - jl_ang;
    gmax = fmax(gmax, fmax((double)(ab(ga.x) / s6[0]), fmax((double)(ab(ga.y) / s6[1]), (double)(ab(ga.z) / s6[2]))));
    gsq += (double)ga.x * ga.x + (double)ga.y * ga.y + (double)ga.z * ga.z;
    if (write) {
      st3(W.g + d + 3, ga);
      st3(W.w + d + 3, sym_mul(W.iwi6 + 6 * ab3, ga));
    }
  }
}

// The Newton loop for one environment (warp). Requires newton_setup + barrier,
// the contact set, the static row blocks and the body incidence lists.
// Per-body rotations at the current iterate into W.qrot (one quaternion -> matrix
// per body instead of one per joint/contact side); needs a team barrier after.
template <class R, class Team> __device__ __forceinline__ void refresh_rotations(Team& t, const Topo<R>& T, Work<R>& W) {
  if (!W.qrot) return;
  for (int b = t.rank(); b < T.nb; b += t.size())
    if (T.btype[b] == 1) {
      const M3<R> m = body_rot(T, W.q, b);
#pragma unroll
      for (int i = 0; i < 9; ++i) W.qrot[9 * b + i] = m.a[i];
    }
}

template <class R, class Team> __device__ int newton_solve_obj(Team& t, const Topo<R>& T, ObjView<R>& O, const Cfg& cfg,
                                                     StepOut out) {
  Work<R>& W = O.W;
  const int rk = t.rank(), ts = t.size();
  const R h = W.h;
  const int nr = W.nrows;
  const int nobj = T.nj + W.nc;
  const int maxlin = cfg.linear_max_iterations;
  const R eps = R(cfg.epsilon_reg);
  const R tfrac = R(cfg.step_fraction);
  PhaseClock pc(out.ptime, rk == 0);
  for_my_rows(T, W, rk, ts, [&](int i) { W.lam[i] = R(0); });
  t.sync();
  double min_shift = 0.0;
  int n_done = 0, aborted = 0;
  for (int it = 0; it < cfg.newton_iterations; ++it) {
    // ---- assemble (object lanes); iteration 0 runs at q- whose rotations batch_env cached
    if (it > 0) {
      refresh_rotations(t, T, W);
      t.sync();
    }
    AsmStats as{0.0, 0.0, 0.0, 0.0};
    for (int k = rk; k < nobj; k += ts) {
      if (k < T.nj)
        assemble_joint(T, W, W.q, k, h, as);
      else
        assemble_contact(T, W, W.q, W.u, k - T.nj, h, cfg, as);
    }
    t.sync();
    pc.mark(1);
    // ---- g = M~(u - u~) - J^T lambda, geometric stiffness, H^-1, w = H^-1 g
    stage_objects(T, O, rk, ts, RowArr<R>{W.lam});
    t.sync();
    double gmax = 0.0, gsq = 0.0, smin = 0.0;
    const bool gs = it >= 1 && cfg.geometric_stiffness;
    for (int b = rk; b < T.nb; b += ts) body_momentum(T, O, b, gs, true, gmax, gsq, smin);
    double s2[2] = {gsq, as.hsq}, mm[4] = {fmax(gmax, as.hmax), as.comp, as.cone, -smin};
    t.reduce(s2, mm);
    min_shift = fmin(min_shift, -mm[3]);
    IterOut io;
    io.residual_inf = mm[0];
    io.merit_l2 = sqrt(s2[0] + s2[1]);
    io.comp_error_max = mm[1];
    io.cone_violation_max = mm[2];
    io.linear_iterations = 0;
    io.linear_residual = 0.0;
    io.linear_breakdown = 0;
    io.step_size = 0.0;
    pc.mark(2);
    // ---- b = J H^-1 g - h, diagonal preconditioner, r = b, x = 0
    double rr = 0.0, rzr = 0.0;
    for (int k = rk; k < nobj; k += ts) {
      object_Jw(T, W, k, W.w, [&](int i, R jw) {
        const R b = jw - W.hv[i];
        W.r[i] = b;
        W.x[i] = R(0);
        W.bx[i] = R(0);
        rr += (double)b * b;
      });
      object_quad(T, W, k, [&](int i, R qd) {
        R inv = R(1);
        if (cfg.preconditioner == 1) {
          const R sd = qd + W.cd[i] + eps;
          inv = sd > R(0) ? R(1) / sd : R(1);
        }
        W.inv[i] = inv;
        const R b = W.r[i];
        rzr += (double)b * (double)(inv * b);
      });
    }
    int lin_used = 0, breakdown = 0, hist_n = 0;
    double hist_last = 0.0;
    if (nr > 0) {
      double s1[2] = {rr, rzr};
      t.reduce_sum(s1);
      hist_last = sqrt(s1[0]);
      double phist_last = sqrt(s1[1]);
      double best_res = hist_last;
      hist_n = 1;
      if (rk == 0 && out.hist) out.hist[(size_t)it * (maxlin + 1)] = hist_last;
      bool pending_best = false;
      R pend = R(0);
      double zaz = 0.0;
      if (maxlin > 0 && hist_last > cfg.linear_tolerance) {
        stage_objects(T, O, rk, ts, RowPrecond<R>{W.r, W.inv});
        t.sync();
        bodies_apply_hinv(T, O, rk, ts);
        t.sync();
        double za = 0.0;
        for (int k = rk; k < nobj; k += ts)
          object_Jw(T, W, k, W.w, [&](int i, R jw) {
            const R zi = W.inv[i] * W.r[i];
            const R a = jw + W.cd[i] * zi + eps * zi;
            W.az[i] = a;
            za += (double)zi * a;
          });
        double s[1] = {za};
        t.reduce_sum(s);
        zaz = s[0];
      }
      pc.mark(3);
      double beta = 0.0;
      for (int itl = 0; itl < maxlin && hist_last > cfg.linear_tolerance; ++itl) {
        // phase A (owned rows): p = z + beta p, ap = az + beta ap; den = ap . M^-1 ap
        R den_p = R(0);  // per-lane partials in the working precision
        const R rb = R(beta);
        const bool first = itl == 0;
        for_my_rows(T, W, rk, ts, [&](int i) {
          R pi, api;
          const R zi = W.inv[i] * W.r[i];
          if (first) {
            pi = zi;
            api = W.az[i];
          } else {
            pi = zi + rb * W.p[i];
            api = W.az[i] + rb * W.ap[i];
          }
          W.p[i] = pi;
          W.ap[i] = api;
          den_p += api * (W.inv[i] * api);
        });
        double den;
        {
          double s[1] = {(double)den_p};
          t.reduce_sum(s);
          den = s[0];
        }
        pc.mark(4);
        if (fabs(den) < 1e-300) {
          breakdown = 1;
          break;
        }
        const double alpha = zaz / den;
        const R ra = R(alpha);
        // phase B: trial residual norms; in the same pass (it needs only alpha) the
        // speculative J^T staging of z' = z - alpha M^-1 ap — the reduction's barrier
        // then orders it before the body pass. A rejected trial discards it.
        R pn2_p = R(0), rn2_p = R(0);
        for_my_rows(T, W, rk, ts, [&](int i) {
          const R rv = W.r[i] - ra * W.ap[i];
          pn2_p += rv * (W.inv[i] * rv);
          rn2_p += rv * rv;
        });
        if (fabs(zaz) >= 1e-300) stage_objects(T, O, rk, ts, RowPrecondResidual<R>{W.r, W.inv, W.ap, ra});
        double pn2, rn2;
        {
          double s[2] = {(double)pn2_p, (double)rn2_p};
          t.reduce_sum(s);
          pn2 = s[0];
          rn2 = s[1];
        }
        pc.mark(5);
        const double pn = sqrt(pn2);
        if (pn > phist_last) break;  // monotone guard: stop at the numerical floor
        pend = ra;                   // accepted; committed by the owner lanes in the J w pass
        hist_last = sqrt(rn2);
        phist_last = pn;
        if (rk == 0 && out.hist && hist_n <= maxlin) out.hist[(size_t)it * (maxlin + 1) + hist_n] = hist_last;
        ++hist_n;
        if (hist_last < best_res) {
          best_res = hist_last;
          pending_best = true;
        }
        lin_used = itl + 1;
        if (fabs(zaz) < 1e-300) {
          breakdown = 1;
          break;
        }
        pc.mark(6);
        pc.mark(7);
        bodies_apply_hinv(T, O, rk, ts);
        t.sync();
        pc.mark(8);
        // commit x, r of the owned rows and az = A z', zaz' = z' . az in one pass.
        // z = M^-1 r is recomputed, not stored: the reference updates it by
        // recursion (solvers.cpp PCR: z -= alpha M^-1 ap), equal in exact arithmetic
        // for the diagonal preconditioner and one rounding apart here; dropping the
        // array removes a row vector from the on-chip working set
        R za_p = R(0);
        const bool best = pending_best;
        for (int k = rk; k < nobj; k += ts)
          object_Jw(T, W, k, W.w, [&](int i, R jw) {
            const R api = W.ap[i];
            const R ri = W.r[i] - pend * api;
            const R zi = W.inv[i] * ri;
            const R xi = W.x[i] + pend * W.p[i];
            W.x[i] = xi;
            W.r[i] = ri;
            if (best) W.bx[i] = xi;
            const R a = jw + W.cd[i] * zi + eps * zi;
            W.az[i] = a;
            za_p += zi * a;
          });
        pend = R(0);
        pending_best = false;
        {
          double s[1] = {(double)za_p};
          t.reduce_sum(s);
          beta = s[0] / zaz;
          zaz = s[0];
        }
        pc.mark(9);
      }
      if (pending_best || pend != R(0)) {
        for_my_rows(T, W, rk, ts, [&](int i) {
          const R xi = W.x[i] + pend * W.p[i];
          W.x[i] = xi;
          if (pending_best) W.bx[i] = xi;
        });
      }
    }
    pc.mark(3);
    io.linear_iterations = lin_used;
    io.linear_breakdown = breakdown;
    io.linear_residual = hist_n > 0 ? hist_last : 0.0;
    // ---- du = H^-1 (J^T dlambda - g); NaN check
    double dl2 = 0.0, du2 = 0.0, bad = 0.0;
    for_my_rows(T, W, rk, ts, [&](int i) {
      const R v = W.bx[i];
      dl2 += (double)v * v;
      if (!isfinite(v)) bad = 1.0;
    });
    stage_objects(T, O, rk, ts, RowArr<R>{W.bx});
    t.sync();
    for (int b = rk; b < T.nb; b += ts) {
      V3<R> lin, ang;
      gather_body(T, O, b, lin, ang);
      const int d = T.bdof[b];
      const V3<R> rl = lin - ld3(W.g + d);
      const V3<R> dl = v3(rl.x * W.hinv[d], rl.y * W.hinv[d + 1], rl.z * W.hinv[d + 2]);
      st3(W.du + d, dl);
      du2 += (double)dl.x * dl.x + (double)dl.y * dl.y + (double)dl.z * dl.z;
      if (!isfinite(dl.x) || !isfinite(dl.y) || !isfinite(dl.z)) bad = 1.0;
      if (T.btype[b] == 1) {
        const V3<R> da = sym_mul(W.iwi6 + 6 * (d / 3 + 1), ang - ld3(W.g + d + 3));
        st3(W.du + d + 3, da);
        du2 += (double)da.x * da.x + (double)da.y * da.y + (double)da.z * da.z;
        if (!isfinite(da.x) || !isfinite(da.y) || !isfinite(da.z)) bad = 1.0;
      }
    }
    {
      double s[2] = {dl2, du2}, m[1] = {bad};
      t.reduce(s, m);
      dl2 = s[0];
      du2 = s[1];
      bad = m[0];
    }
    pc.mark(10);
    if (bad != 0.0) {
      for (int i = rk; i < T.ncoord; i += ts) W.q[i] = W.q0[i];
      for (int i = rk; i < T.ndof; i += ts) W.u[i] = W.u0[i];
      if (rk == 0 && out.iters) out.iters[it] = io;
      aborted = 1;
      n_done = it + 1;
      break;
    }
    // ---- damped update + integration (newton.cpp:393-396)
    for_my_rows(T, W, rk, ts, [&](int i) { W.lam[i] += tfrac * W.bx[i]; });
    for (int b = rk; b < T.nb; b += ts) {
      const int d = T.bdof[b];
      const int nd = T.btype[b] == 1 ? 6 : 3;
      for (int k = 0; k < nd; ++k) W.u[d + k] += tfrac * W.du[d + k];
      integrate_body(T, W.q0, W.q, W.q, W.u, b, h);
    }
    io.step_size = (double)tfrac * sqrt(du2 + dl2);
    if (rk == 0) {
      if (out.iters) out.iters[it] = io;
      if (out.hist_len) out.hist_len[it] = nr > 0 ? hist_n : 0;
    }
    n_done = it + 1;
    t.sync();
    pc.mark(11);
  }
  if (aborted) {
    if (rk == 0 && out.fin) {
      out.fin[5] = 1.0;
      out.fin[6] = 0.0;
      out.fin[7] = n_done;
    }
    return 1;
  }
  // ---- final assembly for classification (newton.cpp:409-415)
  refresh_rotations(t, T, W);
  t.sync();
  AsmStats fs{0.0, 0.0, 0.0, 0.0};
  for (int k = rk; k < nobj; k += ts) {
    if (k < T.nj)
      assemble_joint(T, W, W.q, k, h, fs);
    else
      assemble_contact(T, W, W.q, W.u, k - T.nj, h, cfg, fs);
  }
  t.sync();
  stage_objects(T, O, rk, ts, RowArr<R>{W.lam});
  t.sync();
  double gmax = 0.0, gsq = 0.0, smin = 0.0;
  for (int b = rk; b < T.nb; b += ts) body_momentum(T, O, b, false, false, gmax, gsq, smin);
  double mgap = W.nc ? __builtin_huge_val() : 0.0;
  for (int c = rk; c < W.nc; c += ts) {
    const R* g = W.cgeo + 17 * c;
    const int ba = W.cbody[2 * c], bb = W.cbody[2 * c + 1];
    const CView<R> cv = contact_rec_view(W, c);
    const V3<R> pa = ba < 0 ? ld3(g) : body_pos(T, W.q, ba) + cv.ra;
    const V3<R> pb = bb < 0 ? ld3(g + 3) : body_pos(T, W.q, bb) + cv.rb;
    mgap = fmin(mgap, (double)(dot(cv.n, pa - pb) - g[15]));
  }
  {
    double s[1] = {0.0}, m[4] = {fmax(gmax, fs.hmax), fs.comp, fs.cone, -mgap};
    t.reduce(s, m);
    if (rk == 0 && out.fin) {
      out.fin[0] = m[0];
      out.fin[1] = m[1];
      out.fin[2] = m[2];
      out.fin[3] = W.nc ? -m[3] : 0.0;
      out.fin[4] = min_shift;
      out.fin[5] = 0.0;
      out.fin[6] = m[0] < cfg.newton_tolerance ? 1.0 : 0.0;
      out.fin[7] = n_done;
    }
  }
  pc.mark(12);
  return 0;
}

}  // namespace nsd
