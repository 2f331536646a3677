// Per-environment step setup shared by the batched launches (step_world's
// caller work + newton_step's setup, scene.cpp:709-732, newton.cpp:327-338):
// q- and u- from the persistent state, the per-body rotation cache at q-, the
// joint-torque extension hook, newton_setup (M~ at q-, u~, zero start); and the
// warp-per-environment narrow phase of the rigid path (k_batch_collide).
#pragma once

#include "nsd_plan.cuh"

namespace nsdi {

template <class R, class Team>
__device__ __forceinline__ void env_setup(Team& t, const BatchArgs<R>& A, int env, nsd::Work<R>& W, const R* qs,
                                          const R* us, R* cr, R* qrot) {
  const nsd::Topo<R>& T = A.T;
  const WorkPlan& P = A.plan;
  R* q0 = cr + P.q0;
  R* u0 = cr + P.u0;
  for (int i = t.rank(); i < T.ncoord; i += t.size()) q0[i] = qs[i];
  for (int i = t.rank(); i < T.ndof; i += t.size()) u0[i] = us[i];
  W.f_extra = nullptr;
  // per-body rotations at q- (torque hook, narrow phase, first assembly): one
  // quaternion -> matrix per body instead of one per joint / contact / shape pair
  t.sync();
  for (int b = t.rank(); b < T.nb; b += t.size())
    if (T.btype[b] == 1) {
      const nsd::M3<R> m = nsd::body_rot(T, q0, b);
      for (int i = 0; i < 9; ++i) qrot[9 * b + i] = m.a[i];
    }
  if (A.torque) {
    R* fx = cr + P.fx;
    // the env's torques once per lane into scratch (a single bus round trip when the
    // actions are read from mapped host memory), then the per-body sums
    R* tq = cr + P.tq;
    for (int j = t.rank(); j < T.nj; j += t.size())
      tq[j] = A.torque_double ? R(static_cast<const double*>(A.torque)[(size_t)env * T.nj + j])
                              : R(static_cast<const float*>(A.torque)[(size_t)env * T.nj + j]);
    t.sync();
    // joint torques about revolute axes at q- (extension hook): +tau*axis on a, -tau*axis on b
    for (int b = t.rank(); b < T.nb; b += t.size()) {
      const int d = T.bdof[b];
      nsd::V3<R> f = nsd::v3(R(0), R(0), R(0));
      if (T.btype[b] == 1) {
        for (int j = 0; j < T.nj; ++j) {
          if (T.jkind[j] != 1) continue;
          const int ja = T.jbody[2 * j], jb = T.jbody[2 * j + 1];
          if (ja != b && jb != b) continue;
          const R tau = tq[j];
          const nsd::V3<R> axl = nsd::ld3(A.jframe + 21 * j + 6);
          nsd::M3<R> Rj;
          if (ja >= 0)
            for (int i = 0; i < 9; ++i) Rj.a[i] = qrot[9 * ja + i];
          const nsd::V3<R> ax = ja < 0 ? axl : nsd::mul(Rj, axl);
          if (ja == b) f = f + tau * ax;
          if (jb == b) f = f - tau * ax;
        }
      }
      for (int k = 0; k < 3; ++k) fx[d + k] = R(0);
      if (T.btype[b] == 1) nsd::st3(fx + d + 3, f);
    }
    W.f_extra = fx;
  }
  t.sync();
  nsd::newton_setup(t, T, W);
  t.sync();
}

}  // namespace nsdi
