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
template <class R> constexpr int warp_minb() { return sizeof(R) == 8 ? NSD_WARP_MINB_D : 8; }
template <class R> __global__ void __launch_bounds__(64, warp_minb<R>()) k_batch_warp(BatchArgs<R> A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int env = blockIdx.x * (blockDim.x >> 5) + wib;
  if (env >= A.n_env) return;
  const nsd::Topo<R>& T = A.T;
  const int nc = A.nc_out[env];
  if (T.nj + nc > A.warp_max_obj) return;  // warp-uniform
  const WorkPlan& P = A.plan;
  const nsd::wp::Plan& L = A.wplan;
  unsigned char* base = smem + (size_t)wib * L.bytes;
  R* sr = reinterpret_cast<R*>(base);
  int* si = reinterpret_cast<int*>(base + ((L.nR * sizeof(R) + 15) & ~size_t(15)));
  nsd::wp::Env<R> E{T,          sr + L.bq,  sr + L.brot, sr + L.bu, sr + L.biwi,     sr + L.bhi,  sr + L.bw,
                    sr + L.stg, sr + L.rec, sr + L.x,    sr + L.bx, si + L.gent_off, si + L.gent, T.nj,
                    nc,         T.nb};
  R* hr = reinterpret_cast<R*>(A.hot_global + (size_t)env * A.hot_bytes);
  const int* hi = P.hot_ints(hr);
  R* cr = A.cold_r + (size_t)env * P.coldR;
  int* ci = A.cold_i + (size_t)env * P.coldI;
  nsd::wp::EnvIO<R> io;
  io.q0 = cr + P.q0;
  io.u0 = cr + P.u0;
  io.ut = cr + P.ut;
  io.iw6 = cr + P.iw6;
  io.iwi6 = hr + P.iwi6;
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


// Narrow phase + step setup, one warp per environment (the rigid path's first
// launch; k_batch_sub mode 1 does the same with sub-warp teams): env_setup, then
// the shape pairs 32 per round, one per lane (pair_contacts, collision.cpp:253-287).
// Each round's candidates are appended to the env's compact shared-memory list in
// (pair, k) generation order by a warp prefix sum; each candidate's rank under the
// canonical (a.body, b.body, feature) order, ties by generation order
// (collision.cpp:290-295), places it in the env's contact slabs. A list longer
// than its capacity (>= max_contacts) only occurs with a contact overflow, which
// is reported as an error; the contacts kept then come from the stored prefix.
template <class R> __global__ void __launch_bounds__(128, 4) k_batch_collide(BatchArgs<R> A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int env = blockIdx.x * (blockDim.x >> 5) + wib;
  if (env >= A.n_env) return;
  const nsd::Topo<R>& T = A.T;
  const WorkPlan& P = A.plan;
  const int cap = A.collide_cap;
  nsd::CandD<R>* cand = reinterpret_cast<nsd::CandD<R>*>(smem) + (size_t)wib * cap;
  R* hr = reinterpret_cast<R*>(A.hot_global + (size_t)env * A.hot_bytes);
  int* hi = P.hot_ints(hr);
  R* cr = A.cold_r + (size_t)env * P.coldR;
  int* ci = A.cold_i + (size_t)env * P.coldI;
  nsd::Work<R> W = P.template bind<R>(hr, hi, cr, ci);
  W.jframe = A.jframe;
  W.h = A.h;
  W.grav[0] = A.grav[0];
  W.grav[1] = A.grav[1];
  W.grav[2] = A.grav[2];
  R* qrot = hr + P.qrot;
  nsd::WarpTeam t(lane);
  env_setup(t, A, env, W, A.qs + (size_t)env * T.ncoord, A.us + (size_t)env * T.ndof, cr, qrot);
  const nsd::BodyView<R> view{T.btype, T.bdof, T.bcoord, W.q0, W.ut, qrot};
  int total = 0;
  for (int p0 = 0; p0 < A.npairs; p0 += 32) {
    const int p = p0 + lane;
    nsd::CandD<R> loc[4];
    int n = 0;
    if (p < A.npairs) {
      const int2 ij = A.pairs[p];
      R th, mu;
      n = nsd::pair_contacts(view, A.shapes[ij.x], A.shapes[ij.y], A.h, A.margin, A.mu_default, loc, &th, &mu);
    }
    int incl = n;  // inclusive prefix sum of the counts over the lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int base = total + incl - n;
    for (int k = 0; k < n; ++k)
      if (base + k < cap) cand[base + k] = loc[k];
    total += __shfl_sync(0xffffffffu, incl, 31);
  }
  __syncwarp();
  const int stored = total < cap ? total : cap;
  const int nc = total < A.maxc ? total : A.maxc;
  int* cbody = hi + P.cbody;
  int* cfeat = ci + P.cfeat;
  R* cgeo = cr + P.cgeo;
  for (int i = lane; i < stored; i += 32) {
    const nsd::CandD<R> c = cand[i];
    int rank = 0;
    for (int j = 0; j < stored; ++j) {
      const int oa = cand[j].a, ob = cand[j].b, of = cand[j].feature;
      if (nsd::canonical_less(oa, ob, of, c.a, c.b, c.feature) || (oa == c.a && ob == c.b && of == c.feature && j < i))
        ++rank;
    }
    if (rank >= nc) continue;
    cbody[2 * rank] = c.a;
    cbody[2 * rank + 1] = c.b;
    cfeat[rank] = c.feature;
    R* g = cgeo + 17 * rank;
    nsd::V3<R> nn = nsd::get3(c.n), d1, d2;
    nsd::tangent_basis(nn, d1, d2);
    for (int k = 0; k < 3; ++k) {
      g[k] = c.la[k];
      g[3 + k] = c.lb[k];
      g[6 + k] = c.n[k];
    }
    nsd::st3(g + 9, d1);
    nsd::st3(g + 12, d2);
    g[15] = c.thick;
    g[16] = c.mu;
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
template cudaError_t launch_batch_collide<float>(int, int, size_t, cudaStream_t, const BatchArgs<float>&);
template cudaError_t launch_batch_collide<double>(int, int, size_t, cudaStream_t, const BatchArgs<double>&);

template <class R> cudaError_t batch_warp_setup(int max_optin, int threads, size_t smem, int* blocks_per_sm) {
  cudaError_t e = cudaFuncSetAttribute(k_batch_warp<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_batch_collide<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_batch_warp<R>, threads, smem);
}

template <class R>
cudaError_t launch_batch_warp(int nblk, int threads, size_t smem, cudaStream_t s, const BatchArgs<R>& A) {
  k_batch_warp<R><<<nblk, threads, smem, s>>>(A);
  return cudaGetLastError();
}

template cudaError_t batch_warp_setup<float>(int, int, size_t, int*);
template cudaError_t batch_warp_setup<double>(int, int, size_t, int*);
template cudaError_t launch_batch_warp<float>(int, int, size_t, cudaStream_t, const BatchArgs<float>&);
template cudaError_t launch_batch_warp<double>(int, int, size_t, cudaStream_t, const BatchArgs<double>&);

}  // namespace nsdi
