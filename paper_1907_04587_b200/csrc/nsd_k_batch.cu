// Batched environments, object solver (nsd_batch.cuh): k_batch_sub (TPE lanes per
// env) and k_batch_block (a CTA per env). k_batch_sub also runs the narrow-phase
// launch (mode 1) and the large-env launch (mode 2) around k_batch_warp.
#include "nsd_batch.cuh"
#include "nsd_plan.cuh"
#include "nsd_env_setup.cuh"

#include <type_traits>

using namespace nsdi;

template <class R, class Team>
__device__ void batch_env(Team& t, const BatchArgs<R>& A, int env, R* hr, R* pool, int tib) {
  const nsd::Topo<R>& T = A.T;
  const WorkPlan& P = A.plan;
  if (A.mode == 2 && T.nj + A.nc_out[env] <= A.warp_max_obj) return;  // team-uniform: k_batch_warp solved it
  int* hi = P.hot_ints(hr);
  R* cr = A.cold_r + (size_t)env * P.coldR;
  int* ci = A.cold_i + (size_t)env * P.coldI;
  nsd::Work<R> W = P.template bind<R>(hr, hi, cr, ci);
  nsd::PhaseClock pc(A.ptime, t.rank() == 0);
  const long long env_t0 = A.ptime ? clock64() : 0;
  W.jframe = A.jframe;
  W.h = A.h;
  W.grav[0] = A.grav[0];
  W.grav[1] = A.grav[1];
  W.grav[2] = A.grav[2];
  R* qs = A.qs + (size_t)env * T.ncoord;
  R* us = A.us + (size_t)env * T.ndof;
  R* q0 = cr + P.q0;
  R* u0 = cr + P.u0;
  R* qrot = hr + P.qrot;
  int* cbody = hi + P.cbody;
  int nc = 0, total = 0;
  env_setup(t, A, env, W, qs, us, cr, qrot);
  if (A.mode == 2) {  // the contact set comes from the narrow-phase launch (k_batch_collide)
    nc = A.nc_out[env];
  } else {
  // ---- narrow phase over shape pairs with the unconstrained velocity
  nsd::BodyView<R> view{T.btype, T.bdof, T.bcoord, W.q0, W.ut, qrot};
  nsd::CandD<R>* cand = A.cand + (size_t)env * A.npairs * 4;
  int* cnt = A.pair_cnt + (size_t)env * A.npairs;
  for (int p = t.rank(); p < A.npairs; p += t.size()) {
    const int2 ij = A.pairs[p];
    R th, mu;
    cnt[p] = nsd::pair_contacts(view, A.shapes[ij.x], A.shapes[ij.y], A.h, A.margin, A.mu_default, cand + 4 * p, &th,
                                &mu);
  }
  t.sync();
  for (int p = 0; p < A.npairs; ++p) total += cnt[p];
  nc = total < A.maxc ? total : A.maxc;
  int* cfeat = ci + P.cfeat;
  R* cgeo = cr + P.cgeo;
  // canonical (a.body, b.body, feature) order, stable in generation order
  for (int p = t.rank(); p < A.npairs; p += t.size()) {
    for (int k = 0; k < cnt[p]; ++k) {
      const nsd::CandD<R> c = cand[4 * p + k];
      int rank = 0;
      for (int p2 = 0; p2 < A.npairs; ++p2) {
        const int n2 = cnt[p2];
        for (int k2 = 0; k2 < n2; ++k2) {
          const nsd::CandD<R>& o = cand[4 * p2 + k2];
          if (nsd::canonical_less(o.a, o.b, o.feature, c.a, c.b, c.feature) ||
              (o.a == c.a && o.b == c.b && o.feature == c.feature && (p2 < p || (p2 == p && k2 < k))))
            ++rank;
        }
      }
      if (rank >= nc) continue;
      cbody[2 * rank] = c.a;
      cbody[2 * rank + 1] = c.b;
      cfeat[rank] = c.feature;
      R* g = cgeo + 17 * rank;
      nsd::V3<R> n = nsd::get3(c.n), d1, d2;
      nsd::tangent_basis(n, d1, d2);
      for (int i = 0; i < 3; ++i) {
        g[i] = c.la[i];
        g[3 + i] = c.lb[i];
        g[6 + i] = c.n[i];
      }
      nsd::st3(g + 9, d1);
      nsd::st3(g + 12, d2);
      g[15] = c.thick;
      g[16] = c.mu;
    }
  }
  t.sync();
  if (t.rank() == 0) {  // contact count; overflow is sticky until nsd_batch_results
    A.nc_out[env] = nc;
    if (total > A.maxc) A.overflow[env] = max(A.overflow[env], total);
  }
  }  // narrow phase
  W.nc = nc;
  W.normal_begin = T.rows_static;
  W.friction_begin = T.rows_static + nc;
  W.nrows = T.rows_static + 3 * nc;
  nsd::StepOut out{};
  out.iters = A.iters ? A.iters + (size_t)env * A.cfg.newton_iterations : nullptr;
  out.fin = A.fin + (size_t)env * 8;
  out.ptime = A.ptime;
  pc.mark(0);
  if constexpr (!std::is_same<Team, nsd::BlockTeam>::value) {
    // ---- object-centric sub-warp solver: contact incidence per body (contact*2 + side)
    int* cboff = hi + P.cbinc_off;
    int* cbinc = hi + P.cbinc;
    int* ccnt = ci + P.cinc_cnt;
    for (int b = t.rank(); b < T.nb; b += t.size()) {
      int n = 0;
      for (int c = 0; c < nc; ++c) n += (cbody[2 * c] == b) + (cbody[2 * c + 1] == b);
      ccnt[b] = n;
    }
    t.sync();
    if (t.rank() == 0) {
      int s = 0;
      for (int b = 0; b < T.nb; ++b) {
        cboff[b] = s;
        s += ccnt[b];
      }
      cboff[T.nb] = s;
    }
    t.sync();
    for (int b = t.rank(); b < T.nb; b += t.size()) {
      int o = cboff[b];
      for (int c = 0; c < nc; ++c) {
        if (cbody[2 * c] == b) cbinc[o++] = 2 * c;
        if (cbody[2 * c + 1] == b) cbinc[o++] = 2 * c + 1;
      }
    }
    W.jstr = hr + P.jstr;  // structured joint rows: the object solver never reads coeff/blk
    W.qrot = qrot;         // rotations at q- now; refreshed before every later assembly
    W.crec = hr + P.crec;  // contact records + block ids for vector loads
    W.cblk = reinterpret_cast<int4*>(hi + P.cblk);
    W.jblk = A.jblk;
    t.sync();
    nsd::ObjView<R> O{W, hr + P.jstage, hr + P.cstage, A.jbinc_off, A.jbinc, cboff, cbinc};
    // Slice of the block's shared-memory region. When the block is one full warp of
    // teams, they exchange their needs and take prefix offsets, so a small env lends
    // space to a large one (all 32 lanes reach this shuffle: a full block has no
    // early-returned team).
    const int need = row_pool_elems<R>(T.rows_static, T.nj, T.ndof, nc);
    const int epb = A.envs_per_block, cap = epb * A.row_pool;
    const bool block_full = (blockIdx.x + 1) * epb <= A.n_env && A.mode == 0;
    int off = tib * A.row_pool, lim = (tib + 1) * A.row_pool;
    if (pool && block_full && epb * Team::kSize == 32) {
      int before = 0;
      for (int j = 0; j < epb; ++j) {
        const int nj_need = __shfl_sync(0xffffffffu, need, j * Team::kSize);
        if (j < tib) before += nj_need;
      }
      off = before;
      lim = cap;
    }  // partial blocks keep the fixed split (teams past n_env returned early)
    if (pool && off + need <= lim) {
      pool += off;
      // the env's PCR row state fits its shared-memory region: keep every store of
      // the CR loop on chip (global stores are write-through to L2)
      const int rows = (W.nrows + 3) & ~3;
      R* sp = pool;
      // row vectors by accesses per CR iteration: inv (5 reads), r (4R+1W), ap
      // (3R+1W), p (2R+1W), x, az (1R+1W), bx (1W), cd (1R); z = M^-1 r is not
      // stored (newton_solve_obj); the first pool_row_vecs<R>() live in the region
      constexpr int nv = pool_row_vecs<R>();
      O.W.inv = sp;
      O.W.r = sp + rows;
      O.W.ap = sp + 2 * rows;
      if (nv >= 4) O.W.p = sp + 3 * rows;
      if (nv >= 5) O.W.x = sp + 4 * rows;
      if (nv >= 6) O.W.az = sp + 5 * rows;
      if (nv >= 7) O.W.bx = sp + 6 * rows;
      if (nv >= 8) O.W.cd = sp + 7 * rows;
      sp += nv * rows;
      O.jstage = sp;
      sp += (12 * T.nj + 3) & ~3;
      O.cstage = sp;
      sp += (9 * nc + 3) & ~3;
      // w = H^-1 J^T y is produced by body_momentum; copy the setup value over
      for (int i = t.rank(); i < T.ndof; i += t.size()) sp[i] = W.w[i];
      O.W.w = sp;
      sp += (T.ndof + 3) & ~3;
      if (pool_extra<R>() & 1) {
        O.W.crec = sp;
        sp += 20 * nc;
      }
      if (pool_extra<R>() & 2) {
        O.W.jstr = sp;
        sp += (24 * T.nj + 3) & ~3;
      }
      if (pool_extra<R>() & 4) {
        O.W.hinv = sp;
        sp += (T.ndof + 3) & ~3;
      }
      t.sync();
    }
    nsd::newton_solve_obj(t, T, O, A.cfg, out);
    W = O.W;
  } else {
    // ---- contact incidence per dof3 block (contact*4 + slot, contacts ascending)
    int* coff = hi + P.cinc_off;
    int* cent = hi + P.cinc_ent;
    int* ccnt = ci + P.cinc_cnt;
    for (int b = t.rank(); b < T.nd3; b += t.size()) {
      int n = 0;
      for (int c = 0; c < nc; ++c) {
        int al, aa, bl, ba;
        nsd::body_blocks(T, cbody[2 * c], al, aa);
        nsd::body_blocks(T, cbody[2 * c + 1], bl, ba);
        n += (al == b) + (aa == b) + (bl == b) + (ba == b);
      }
      ccnt[b] = n;
    }
    t.sync();
    if (t.rank() == 0) {
      int s = 0;
      for (int b = 0; b < T.nd3; ++b) {
        coff[b] = s;
        s += ccnt[b];
      }
      coff[T.nd3] = s;
    }
    t.sync();
    for (int b = t.rank(); b < T.nd3; b += t.size()) {
      int o = coff[b];
      for (int c = 0; c < nc; ++c) {
        int b4[4];
        nsd::body_blocks(T, cbody[2 * c], b4[0], b4[1]);
        nsd::body_blocks(T, cbody[2 * c + 1], b4[2], b4[3]);
        for (int s = 0; s < 4; ++s)
          if (b4[s] == b) cent[o++] = 4 * c + s;
      }
    }
    t.sync();
    nsd::newton_solve<R, false>(t, T, W, A.cfg, out);
  }
  t.sync();
  pc.mark(13);
  for (int i = t.rank(); i < T.ncoord; i += t.size()) qs[i] = W.q[i];
  for (int i = t.rank(); i < T.ndof; i += t.size()) us[i] = W.u[i];
  if (A.q_out)
    for (int i = t.rank(); i < T.ncoord; i += t.size()) A.q_out[(size_t)env * T.ncoord + i] = W.q[i];
  if (A.u_out)
    for (int i = t.rank(); i < T.ndof; i += t.size()) A.u_out[(size_t)env * T.ndof + i] = W.u[i];
  // export the step's contact set and multipliers (nsd_batch_contacts)
  R* xl = cr + P.xlam;
  int* xb = ci + P.xcbody;
  for (int i = t.rank(); i < W.nrows; i += t.size()) xl[i] = W.lam[i];
  for (int i = t.rank(); i < 2 * nc; i += t.size()) xb[i] = cbody[i];
  if (A.ptime && t.rank() == 0) {  // diagnostics: straggler vs mean env time, contacts of the slowest
    const unsigned long long dt = static_cast<unsigned long long>(clock64() - env_t0);
    atomicMax(A.ptime + 14, dt);
    atomicAdd(A.ptime + 15, dt);
  }
  if (t.rank() == 0) {
    if (out.fin[5] != 0.0) A.aborted_any[env] = 1;
    if (A.counters && out.iters) {
      unsigned long long n = 0;
      for (int k = 0; k < static_cast<int>(out.fin[7]); ++k) n += out.iters[k].linear_iterations;
      atomicAdd(A.counters, n);
      atomicAdd(A.counters + 3, n * static_cast<unsigned long long>(nc));
    }
  }
}

// TPE lanes per environment (32/TPE environments per warp); each env's hot
// working set in shared memory.
// Register budget: 4096 envs at 2 envs per warp (TPE 16) are 2048 warps, 14 per SM
// for a single wave, so <= 146 registers per thread. Measured (50-step C5 bench):
// 128 registers (128 x 4 bounds) fp32 2.77 M / fp64 1.62 M env-steps/s; uncapped
// (255, 8 warps/SM) 2.2 M / 1.54 M; 144 (fp64) 1.17 M (spills land in the solver).
template <class R, int TPE>
__global__ void __launch_bounds__(128, 4) k_batch_sub(BatchArgs<R> A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tib = threadIdx.x / TPE;  // team index in the block
  const int env = blockIdx.x * A.envs_per_block + tib;
  if (env >= A.n_env) return;  // team-uniform
  R* hr = A.hot_in_smem ? reinterpret_cast<R*>(smem + (size_t)tib * A.hot_bytes)
                        : reinterpret_cast<R*>(A.hot_global + (size_t)env * A.hot_bytes);
  R* pool = A.row_pool ? reinterpret_cast<R*>(smem) : nullptr;  // the block's region; batch_env takes a slice
  nsd::SubWarpTeam<TPE> t(threadIdx.x & 31);
  batch_env(t, A, env, hr, pool, tib);
}

// CTA per environment.
template <class R> __global__ void __launch_bounds__(256) k_batch_block(BatchArgs<R> A) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[2 * 33 * nsd::kRedMax];
  nsd::BlockTeam t(red);
  R* hr = A.hot_in_smem ? reinterpret_cast<R*>(smem)
                        : reinterpret_cast<R*>(A.hot_global + (size_t)blockIdx.x * A.hot_bytes);
  batch_env(t, A, blockIdx.x, hr, static_cast<R*>(nullptr), 0);
}


namespace nsdi {

template <class R> cudaError_t batch_sub_attrs(int max_dyn_smem, int carveout) {
  cudaError_t e = cudaSuccess;
  auto set = [&](const void* fn) {
    if (max_dyn_smem >= 0 && e == cudaSuccess)
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn_smem);
    if (carveout >= 0 && e == cudaSuccess)
      e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  };
  set((const void*)k_batch_sub<R, 4>);
  set((const void*)k_batch_sub<R, 8>);
  set((const void*)k_batch_sub<R, 16>);
  set((const void*)k_batch_sub<R, 32>);
  return e;
}

template <class R> cudaError_t batch_block_attrs(int max_optin) {
  cudaFuncAttributes fa{};
  cudaError_t e = cudaFuncGetAttributes(&fa, k_batch_block<R>);  // static reduction buffer counts against the limit
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_batch_block<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              max_optin - static_cast<int>(fa.sharedSizeBytes));
}

template <class R>
cudaError_t launch_batch_sub(int tpe, int nblk, int threads, size_t smem, cudaStream_t s, const BatchArgs<R>& A) {
  switch (tpe) {
    case 4: k_batch_sub<R, 4><<<nblk, threads, smem, s>>>(A); break;
    case 8: k_batch_sub<R, 8><<<nblk, threads, smem, s>>>(A); break;
    case 16: k_batch_sub<R, 16><<<nblk, threads, smem, s>>>(A); break;
    default: k_batch_sub<R, 32><<<nblk, threads, smem, s>>>(A); break;
  }
  return cudaGetLastError();
}

template <class R>
cudaError_t launch_batch_block(int nblk, int threads, size_t smem, cudaStream_t s, const BatchArgs<R>& A) {
  k_batch_block<R><<<nblk, threads, smem, s>>>(A);
  return cudaGetLastError();
}

#define NSD_INST(R)                                                                                         \
  template cudaError_t batch_sub_attrs<R>(int, int);                                                        \
  template cudaError_t batch_block_attrs<R>(int);                                                           \
  template cudaError_t launch_batch_sub<R>(int, int, int, size_t, cudaStream_t, const BatchArgs<R>&);       \
  template cudaError_t launch_batch_block<R>(int, int, size_t, cudaStream_t, const BatchArgs<R>&);
NSD_INST(float)
NSD_INST(double)
#undef NSD_INST

}  // namespace nsdi
