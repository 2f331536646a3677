// Batched rigid environments, one warp per env (nsd_warp.cuh).
#include "nsd_env_setup.cuh"
#include "nsd_plan.cuh"
#include "nsd_warp.cuh"

using namespace nsdi;

// One warp per rigid environment (nsd_warp.cuh), between the narrow-phase launch
// (k_batch_sub, mode 1: setup + contacts into the env slabs) and the mode-2
// launch that solves the environments with more than 32 constraint objects.
// Register budget (2 envs per 64-thread block): 7 blocks/SM for fp64 (<= 128 registers;
// the shared-memory plan allows 14 envs/SM, 4096 envs in 2 waves; measured 0.92 vs
// 1.03 ms/step at 6 blocks = 168 registers = 3 waves, in spite of ~0.6 KB of spills per
// thread); 8 for fp32. NSD_WARP_MINB_D overrides the fp64 choice at build time.
#ifndef NSD_WARP_MINB_D
#define NSD_WARP_MINB_D 7
#endif
template <class S> constexpr int warp_minb() { return sizeof(S) == 8 ? NSD_WARP_MINB_D : 8; }
// R: the batch's state precision (double); S: the PCR operator's (double, or float
// in the mixed-precision mode).
template <class R, class S> __global__ void __launch_bounds__(64, warp_minb<S>()) k_batch_warp(BatchArgs<R> A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int env = blockIdx.x * (blockDim.x >> 5) + wib;
  if (env >= A.n_env) return;
  const nsd::Topo<R>& T = A.T;
  const int nc = A.nc_out[env];
  if (T.nj + nc > A.warp_max_obj) return;  // warp-uniform
  NSD_CHECK(nc >= 0 && nc <= A.maxc && T.nj + nc <= 32);
  const WorkPlan& P = A.plan;
  const nsd::wp::Plan& L = A.wplan;
  unsigned char* base = smem + (size_t)wib * L.bytes;
  auto rp = [&](int off) { return reinterpret_cast<R*>(base + off); };
  auto sp = [&](int off) { return reinterpret_cast<S*>(base + off); };
  auto ip = [&](int off) { return reinterpret_cast<int*>(base + off); };
  nsd::wp::Env<R, S> E{T,           rp(L.bq),   rp(L.brot), rp(L.bu), rp(L.biwi),   rp(L.bhi),
                       sp(L.bw),    base + L.stg, sp(L.rec), rp(L.x),  rp(L.bx),     ip(L.gent_off),
                       ip(L.gent),  T.nj,       nc,         T.nb};
  R* hr = reinterpret_cast<R*>(A.hot_global + (size_t)env * A.hot_bytes);
  const int* hi = P.hot_ints(hr);
  R* cr = A.cold_r + (size_t)env * P.coldR;
  int* ci = A.cold_i + (size_t)env * P.coldI;
  nsd::wp::EnvIO<R> io;
  const R* ws = A.wsetup + (size_t)env * A.wsetup_stride;
  io.q0 = A.qs + (size_t)env * T.ncoord;  // written back only at the end of the step
  io.u0 = A.us + (size_t)env * T.ndof;
  io.ut = ws;
  io.iw6 = ws + T.ndof;
  io.iwi6 = ws + T.ndof + 6 * T.nd3;
  io.cbody = hi + P.cbody;
  io.cgeo = cr + P.cgeo;
  io.lam = A.wlam + (size_t)env * (nsd::wp::kRows * 32);
  io.jinc_off = A.wjinc_off;
  io.jinc = A.wjinc;
  io.g = hr + P.g;
  io.du = hr + P.du;
  io.qs = A.qs + (size_t)env * T.ncoord;
  io.us = A.us + (size_t)env * T.ndof;
  io.q_out = A.q_out ? A.q_out + (size_t)env * T.ncoord : nullptr;
  io.u_out = A.u_out ? A.u_out + (size_t)env * T.ndof : nullptr;
  io.xlam = cr + P.xlam;
  io.xcbody = ci + P.xcbody;
  io.fin = A.fin + (size_t)env * 8;
  io.iters = A.iters ? A.iters + (size_t)env * A.cfg.newton_iterations : nullptr;
  io.cr_iters = A.counters;
  io.cr_cycles = A.profile ? A.counters + 1 : nullptr;
  io.env_cycles = A.profile ? A.counters + 2 : nullptr;
  io.phase = A.wptime;
  nsd::wp::solve_env(T, A.cfg, A.jframe, A.h, E, io, lane);
  if (lane == 0 && io.fin[5] != 0.0) A.aborted_any[env] = 1;
}


// Step setup of one rigid body for the warp path, body lane b (step_world's torque
// hook + newton_setup, scene.cpp:709-732, newton.cpp:327-338): the arithmetic of
// env_setup / nsd::newton_setup for a rigid body. Needs the rotation cache of
// every body at q- (the torque hook rotates the joint axis by body a's frame).
// Writes u~ (also to the shared-memory view of the narrow phase), I_w and I_w^-1.
template <class R>
__device__ __forceinline__ void rigid_setup(const BatchArgs<R>& A, int env, int b, const R* q0, const R* u0,
                                            const R* rot, R* ut_view, R* ut, R* iw6, R* iwi6) {
  const nsd::Topo<R>& T = A.T;
  const int d = T.bdof[b], cd = T.bcoord[b];
  const R m = T.bmass[b], h = A.h;
  nsd::V3<R> f = nsd::v3(m * A.grav[0], m * A.grav[1], m * A.grav[2]);
  nsd::V3<R> tx = nsd::v3(R(0), R(0), R(0));  // joint torques about revolute axes at q- (extension hook)
  if (A.torque) {
    for (int j = 0; j < T.nj; ++j) {
      if (T.jkind[j] != 1) continue;
      const int ja = T.jbody[2 * j], jb = T.jbody[2 * j + 1];
      if (ja != b && jb != b) continue;
      const R tau = A.torque_double ? R(static_cast<const double*>(A.torque)[(size_t)env * T.nj + j])
                                    : R(static_cast<const float*>(A.torque)[(size_t)env * T.nj + j]);
      const nsd::V3<R> axl = nsd::ld3(A.jframe + 21 * j + 6);
      nsd::M3<R> Rj;
      if (ja >= 0)
        for (int i = 0; i < 9; ++i) Rj.a[i] = rot[9 * ja + i];
      const nsd::V3<R> ax = ja < 0 ? axl : nsd::mul(Rj, axl);
      if (ja == b) tx = tx + tau * ax;
      if (jb == b) tx = tx - tau * ax;
    }
    f = f + nsd::v3(R(0), R(0), R(0));  // the hook's zero linear part, added as newton_setup adds f_extra
  }
  const nsd::V3<R> ul = nsd::ld3(u0 + d) + h * (f / m);
  const nsd::M3<R> Rm = nsd::quat_rot(q0[cd + 3], q0[cd + 4], q0[cd + 5], q0[cd + 6]);
  nsd::M3<R> I;
#pragma unroll
  for (int i = 0; i < 9; ++i) I.a[i] = T.binertia[9 * b + i];
  const nsd::M3<R> Iw = nsd::mul(nsd::mul(Rm, I), nsd::transpose(Rm));
  const nsd::M3<R> Ii = nsd::inverse3(Iw);
  const nsd::V3<R> w = nsd::ld3(u0 + d + 3);
  nsd::V3<R> tq = -nsd::cross(w, nsd::mul(Iw, w));
  if (A.torque) tq = tq + tx;
  const nsd::V3<R> ua = w + h * nsd::mul(Ii, tq);
  nsd::st3(ut + d, ul);
  nsd::st3(ut + d + 3, ua);
  nsd::st3(ut_view + d, ul);
  nsd::st3(ut_view + d + 3, ua);
  const int ab3 = 6 * (d / 3 + 1);
  const R s6[6] = {Iw(0, 0), Iw(1, 1), Iw(2, 2), Iw(0, 1), Iw(0, 2), Iw(1, 2)};
  const R i6[6] = {Ii(0, 0), Ii(1, 1), Ii(2, 2), Ii(0, 1), Ii(0, 2), Ii(1, 2)};
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    iw6[ab3 + k] = s6[k];
    iwi6[ab3 + k] = i6[k];
  }
}

// Narrow phase + step setup, one warp per rigid environment (the rigid path's
// first launch). Body lanes stage q-, the rotation cache and u~ in shared memory
// (rigid_setup), then the shape pairs run 32 per round, one per lane
// (pair_contacts, collision.cpp:253-287) against that view, writing their candidates
// to per-pair slots in global memory. Each round's candidate keys are appended to
// the env's compact shared-memory list in (pair, k) generation order by a warp
// prefix sum; each candidate's rank under the canonical
// (a.body, b.body, feature) order, ties by generation order (collision.cpp:290-295),
// places it in the env's contact slabs. Only what k_batch_warp reads is written:
// u~, I_w, I_w^-1 (compact per env) and the contact set; the large-env launch
// recomputes its own setup. A candidate list longer than its capacity
// (>= max_contacts) only occurs with a contact overflow, which is an error; the
// contacts kept then come from the stored prefix.
#ifndef NSD_COLLIDE_MINB
#define NSD_COLLIDE_MINB 4
#endif
template <class R> __global__ void __launch_bounds__(128, NSD_COLLIDE_MINB) k_batch_collide(BatchArgs<R> A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int env = blockIdx.x * (blockDim.x >> 5) + wib;
  if (env >= A.n_env) return;
  const nsd::Topo<R>& T = A.T;
  const WorkPlan& P = A.plan;
  const int cap = A.collide_cap;
  const int nview = (T.ncoord + T.ndof + 9 * T.nb + 1) & ~1;  // q-, u~, rotations (R elements)
  R* view_r = reinterpret_cast<R*>(smem) + (size_t)wib * nview;
  int4* key = reinterpret_cast<int4*>(reinterpret_cast<R*>(smem) + 4 * nview) + (size_t)wib * cap;
  R* vq = view_r;
  R* vu = vq + T.ncoord;
  R* vrot = vu + T.ndof;
  const R* qs = A.qs + (size_t)env * T.ncoord;
  const R* us = A.us + (size_t)env * T.ndof;
  for (int i = lane; i < T.ncoord; i += 32) vq[i] = qs[i];
  __syncwarp();
  if (lane < T.nb) {
    const nsd::M3<R> m = nsd::body_rot(T, vq, lane);
#pragma unroll
    for (int i = 0; i < 9; ++i) vrot[9 * lane + i] = m.a[i];
  }
  __syncwarp();
  R* ws = A.wsetup + (size_t)env * A.wsetup_stride;
  if (lane < T.nb) rigid_setup(A, env, lane, vq, us, vrot, vu, ws, ws + T.ndof, ws + T.ndof + 6 * T.nd3);
  __syncwarp();
  // candidates are generated in the env's per-pair global slots (4 per pair, L2),
  // their keys appended to the compact shared-memory list in generation order
  const nsd::BodyView<R> view{T.btype, T.bdof, T.bcoord, vq, vu, vrot};
  nsd::CandD<R>* gc = A.cand + (size_t)env * A.npairs * 4;
  int total = 0;
  for (int p0 = 0; p0 < A.npairs; p0 += 32) {
    // pairs run grouped by shape kinds (less divergence in a round); slots and the
    // tie-break use each pair's original index p, so the order does not matter
    const int p = p0 + lane < A.npairs ? A.pair_order[p0 + lane] : 0;
    int n = 0;
    if (p0 + lane < A.npairs) {
      const int2 ij = A.pairs[p];
      R th, mu;
      n = nsd::pair_contacts(view, A.shapes[ij.x], A.shapes[ij.y], A.h, A.margin, A.mu_default, gc + 4 * p, &th, &mu);
    }
    int incl = n;  // inclusive prefix sum of the counts over the lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int base = total + incl - n;
    for (int k = 0; k < n; ++k)
      if (base + k < cap) key[base + k] = make_int4(gc[4 * p + k].a, gc[4 * p + k].b, gc[4 * p + k].feature, 4 * p + k);
    total += __shfl_sync(0xffffffffu, incl, 31);
  }
  __syncwarp();
  const int stored = total < cap ? total : cap;
  const int nc = total < A.maxc ? total : A.maxc;
  NSD_CHECK(A.maxc <= cap);  // every kept contact is among the stored keys
  R* hr = reinterpret_cast<R*>(A.hot_global + (size_t)env * A.hot_bytes);
  int* cbody = P.hot_ints(hr) + P.cbody;
  R* cr = A.cold_r + (size_t)env * P.coldR;
  int* cfeat = A.cold_i + (size_t)env * P.coldI + P.cfeat;
  R* cgeo = cr + P.cgeo;
  for (int i = lane; i < stored; i += 32) {
    const int4 c = key[i];
    int rank = 0;
    for (int j = 0; j < stored; ++j) {
      const int4 o = key[j];
      if (nsd::canonical_less(o.x, o.y, o.z, c.x, c.y, c.z) || (o.x == c.x && o.y == c.y && o.z == c.z && o.w < c.w))
        ++rank;
    }
    if (rank >= nc) continue;
    const nsd::CandD<R>& cd = gc[c.w];
    cbody[2 * rank] = c.x;
    cbody[2 * rank + 1] = c.y;
    cfeat[rank] = c.z;
    R* g = cgeo + 17 * rank;
    nsd::V3<R> nn = nsd::get3(cd.n), d1, d2;
    nsd::tangent_basis(nn, d1, d2);
    for (int k = 0; k < 3; ++k) {
      g[k] = cd.la[k];
      g[3 + k] = cd.lb[k];
      g[6 + k] = cd.n[k];
    }
    nsd::st3(g + 9, d1);
    nsd::st3(g + 12, d2);
    g[15] = cd.thick;
    g[16] = cd.mu;
  }
  if (lane == 0) {  // contact count; overflow is sticky until nsd_batch_results
    A.nc_out[env] = nc;
    if (total > A.maxc) A.overflow[env] = max(A.overflow[env], total);
  }
}

namespace nsdi {

template <class R>
cudaError_t launch_batch_collide(int nblk, int threads, size_t smem, cudaStream_t s, const BatchArgs<R>& A) {
  k_batch_collide<R><<<nblk, threads, smem, s>>>(A);
  return cudaGetLastError();
}
template cudaError_t launch_batch_collide<double>(int, int, size_t, cudaStream_t, const BatchArgs<double>&);

template <class R>
cudaError_t batch_warp_setup(bool mixed, int max_optin, int threads, size_t smem, int* blocks_per_sm) {
  const void* kw = mixed ? (const void*)k_batch_warp<R, float> : (const void*)k_batch_warp<R, R>;
  cudaError_t e = cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_batch_collide<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, kw, threads, smem);
}

template <class R>
cudaError_t launch_batch_warp(bool mixed, int nblk, int threads, size_t smem, cudaStream_t s, const BatchArgs<R>& A) {
  if (mixed)
    k_batch_warp<R, float><<<nblk, threads, smem, s>>>(A);
  else
    k_batch_warp<R, R><<<nblk, threads, smem, s>>>(A);
  return cudaGetLastError();
}

template cudaError_t batch_warp_setup<double>(bool, int, int, size_t, int*);
template cudaError_t launch_batch_warp<double>(bool, int, int, size_t, cudaStream_t, const BatchArgs<double>&);

}  // namespace nsdi
