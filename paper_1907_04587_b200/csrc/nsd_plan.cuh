// Shared between the host layer (nsd_api.cu) and the kernel translation units
// (nsd_k_single.cu, nsd_k_batch.cu, nsd_k_warp.cu): preprocessed host topology,
// per-scene work-array plan, batched-kernel arguments and the launch wrappers.
#pragma once

#include "nsd_collide.cuh"
#include "nsd_engine.cuh"
#include "nsd_warp_plan.h"

#include <cuda_runtime.h>

#include <cstddef>
#include <vector>

namespace nsdi {

struct HostTopo {
  int nb = 0, ndof = 0, ncoord = 0, nd3 = 0, nj = 0, nt = 0, rows_joint = 0, rows_static = 0, tdim = 3;
  std::vector<int> btype, bdof, bcoord, d3_body, d3_kind, jkind, jbody, jrow, tbody, sinc_off, sinc_ent;
  std::vector<double> bmass, binertia, jparam, jframe, tdminv, tvol, tmat, tkinv;
};

// Offsets (in elements) of one scene's Work arrays. "Hot" arrays are touched
// every PCR iteration and live in shared memory for the warp-per-env batched
// kernel (global memory otherwise); "cold" arrays stay in global memory.
struct WorkPlan {
  // hot R
  size_t q, u, g, w, du, hinv, iwi6, coeff, hv, cd, lam, x, r, z, p, ap, az, inv, bx, cdir, carm, cscale, jstage,
      cstage, jstr, crec, qrot, hotR;
  // hot int
  size_t blk, cbody, cinc_off, cinc_ent, cbinc_off, cbinc, cblk, hotI;
  // cold R
  size_t q0, u0, qp, ut, iw6, gp, up, shift, ub, fx, ctet, xn, rn, zn, cgeo, xlam, tq, coldR;
  // cold int
  size_t cfeat, cinc_cnt, xcbody, coldI;
  size_t hot_bytes_f, hot_bytes_d;  // bytes of the hot set per env for float / double
  int rcap = 0, ccap = 0;

  void plan(const HostTopo& T, int cc) {
    ccap = cc;
    rcap = T.rows_static + 3 * cc;
    const size_t rs = T.rows_static, rc = rcap, c = cc;
    size_t o = 0;
    auto a = [&](size_t n) {
      const size_t off = o;
      o += (n + 1) & ~size_t(1);  // keep 8-byte alignment for doubles
      return off;
    };
    auto a16 = [&](size_t n) {  // 16-byte aligned start (vector loads): multiple of 4 elements
      o = (o + 3) & ~size_t(3);
      return a(n);
    };
    q = a(T.ncoord);
    u = a(T.ndof);
    g = a(T.ndof);
    w = a(T.ndof);
    du = a(T.ndof);
    hinv = a(T.ndof);
    iwi6 = a(6 * T.nd3);
    coeff = a(12 * rs);
    hv = a(rc);
    cd = a(rc);
    lam = a(rc);
    x = a(rc);
    r = a(rc);
    z = a(rc);
    p = a(rc);
    ap = a(rc);
    az = a(rc);
    inv = a(rc);
    bx = a(rc);
    cdir = a(9 * c);
    carm = a(6 * c);
    cscale = a(2 * c);
    jstage = a(12 * static_cast<size_t>(T.nj));
    cstage = a(9 * c);
    jstr = a(24 * static_cast<size_t>(T.nj));
    crec = a16(20 * c);
    qrot = a(9 * static_cast<size_t>(T.nb));
    hotR = o;
    o = 0;
    blk = a(4 * rs);
    cbody = a(2 * c);
    cinc_off = a(T.nd3 + 1);
    cinc_ent = a(4 * c);
    cbinc_off = a(T.nb + 1);
    cbinc = a(2 * c);
    cblk = a16(4 * c);
    hotI = o;
    o = 0;
    q0 = a(T.ncoord);
    u0 = a(T.ndof);
    qp = a(T.ncoord);
    ut = a(T.ndof);
    iw6 = a(6 * T.nd3);
    gp = a(T.ndof);
    up = a(T.ndof);
    shift = a(T.ndof);
    ub = a(T.ndof);
    fx = a(T.ndof);
    ctet = a(static_cast<size_t>(T.tdim) * T.tdim * T.nt);  // 3x3 (Neo-Hookean) or 6x6 (linear) blocks
    xn = a(rc);
    rn = a(rc);
    zn = a(rc);
    cgeo = a(17 * c);
    xlam = a(rc);
    tq = a(static_cast<size_t>(T.nj));
    coldR = o;
    o = 0;
    cfeat = a(c);
    cinc_cnt = a(T.nd3 + 1);
    xcbody = a(2 * c);
    coldI = o;
    hot_bytes_f = ((hotR * 4 + 15) & ~size_t(15)) + hotI * 4;
    hot_bytes_d = ((hotR * 8 + 15) & ~size_t(15)) + hotI * 4;
    hot_bytes_f = (hot_bytes_f + 15) & ~size_t(15);
    hot_bytes_d = (hot_bytes_d + 15) & ~size_t(15);
  }
  template <class R> size_t hot_bytes() const { return sizeof(R) == 8 ? hot_bytes_d : hot_bytes_f; }
  template <class R> __host__ __device__ int* hot_ints(R* hr) const {
    return reinterpret_cast<int*>(reinterpret_cast<char*>(hr) + ((hotR * sizeof(R) + 15) & ~size_t(15)));
  }
  template <class R> __host__ __device__ nsd::Work<R> bind(R* hr, int* hi, R* cr, int* ci) const {
    nsd::Work<R> W{};
    W.q = hr + q;
    W.u = hr + u;
    W.ut = cr + ut;
    W.g = hr + g;
    W.w = hr + w;
    W.du = hr + du;
    W.hinv = hr + hinv;
    W.iw6 = cr + iw6;
    W.iwi6 = hr + iwi6;
    W.coeff = hr + coeff;
    W.hv = hr + hv;
    W.cd = hr + cd;
    W.lam = hr + lam;
    W.x = hr + x;
    W.xn = cr + xn;
    W.r = hr + r;
    W.rn = cr + rn;
    W.z = hr + z;
    W.zn = cr + zn;
    W.p = hr + p;
    W.ap = hr + ap;
    W.az = hr + az;
    W.inv = hr + inv;
    W.bx = hr + bx;
    W.cgeo = cr + cgeo;
    W.cdir = hr + cdir;
    W.carm = hr + carm;
    W.cscale = hr + cscale;
    W.blk = hi + blk;
    W.cbody = hi + cbody;
    W.cinc_off = hi + cinc_off;
    W.cinc_ent = hi + cinc_ent;
    W.q0 = cr + q0;
    W.u0 = cr + u0;
    W.qp = cr + qp;
    W.gp = cr + gp;
    W.up = cr + up;
    W.shift = cr + shift;
    W.ub = cr + ub;
    W.ctet = cr + ctet;
    return W;
  }
};


#ifndef NSD_GRID_THREADS
#define NSD_GRID_THREADS 256  // measured: 512 (128 registers) makes C2 15% slower
#endif
// Threads per CTA of the cooperative grid kernel (one CTA per SM).
constexpr int kGridThreads = NSD_GRID_THREADS;
static_assert(kGridThreads >= 32 * nsd::kRedMax, "GridTeam::reduce uses one warp per reduced value");

template <class R> struct BatchArgs {
  nsd::Topo<R> T;
  nsd::Cfg cfg;
  int n_env, ns, npairs, maxc, envs_per_block, hot_in_smem;
  int row_pool;  // per-env shared-memory region (elements of R) for the PCR row state; 0 = off
  const int2* pairs;
  const int* pair_order;  // k_batch_collide's processing order of the pairs (grouped by shape kinds)
  const nsd::ShapeD<R>* shapes;
  const R* jframe;
  R margin, mu_default, h, grav[3];
  R* qs;  // persistent state (n_env * ncoord)
  R* us;
  const void* torque;  // n_env * nj or null (device memory or mapped pinned host memory)
  int torque_double;
  R* q_out;  // optional second destination of the final state (mapped pinned host memory):
  R* u_out;  // the step's device->host transfer made by the kernel, overlapped with other envs
  char* hot_global;  // per-env hot slices when not in shared memory
  size_t hot_bytes;
  R* cold_r;
  int* cold_i;
  WorkPlan plan;
  nsd::CandD<R>* cand;  // n_env * npairs * 4
  int* pair_cnt;        // n_env * npairs
  int* nc_out;          // n_env
  int* overflow;        // n_env
  double* fin;          // n_env * 8
  nsd::IterOut* iters;  // n_env * newton_iterations
  const int* jbinc_off;  // static joint incidence per body (warp solver)
  const int* jbinc;
  unsigned long long* ptime;  // NSD_PHASE_TIMING diagnostics (16 counters) or null
  const int4* jblk;           // static dof3 blocks per joint
  int mode;                   // 0 full step; 1 narrow phase + setup only; 2 solve envs with nj + nc > 32 only
  int* aborted_any;           // n_env: sticky abort flag (cleared by nsd_batch_results)
  unsigned long long* counters;  // [0] PCR iterations, [1] PCR-loop cycles, [2] env cycles (k_batch_warp)
  const int* wjinc_off;       // static joint incidence per body, both sides (k_batch_warp)
  const int* wjinc;
  nsd::wp::Plan wplan;        // per-env shared-memory layout of k_batch_warp
  unsigned long long* wptime;  // k_batch_warp phase cycles (NSD_PHASE_TIMING) or null
  R* wlam;                    // k_batch_warp: per env 5 x 32 multipliers ([row][lane])
  int collide_cap;            // k_batch_collide: candidates kept per env in shared memory
  R* wsetup;                  // rigid path: per env u~ (ndof), I_w and I_w^-1 (6 per dof3 block each)
  int wsetup_stride;
  int warp_max_obj;           // k_batch_warp solves envs with nj + nc <= this (<= 32); mode 2 the rest
  int profile;                // k_batch_warp: clock64 cycles inside the PCR loops / per env into counters[1..2]
};

// One environment: extension forces, setup, device narrow phase, contact
// incidence, Newton solve, state write-back (step_world, scene.cpp:709-732).
// Row vectors in the region (priority order in batch_env): all 8 in fp32; in fp64
// the shared-memory budget is the limit, so fewer vectors let larger envs fit.
// Measured (C5): fp32 3.62 M -> 3.92 M env-steps/s when inv/cd joined the region;
// fp64 (then 9 vectors, inv z ap p r x az bx cd): 4 vectors 2.00 M, 5 2.21 M, 6 2.37 M,
// 7 2.22 M, 8 1.78 M env-steps/s -> 6. With z implicit (inv r ap p x az bx cd):
// 6 2.83 M, 7 2.63 M, 8 2.09 M -> 6.
#ifndef NSD_POOL_VECS64
#define NSD_POOL_VECS64 6
#endif
template <class R> __host__ __device__ constexpr int pool_row_vecs() { return sizeof(R) == 4 ? 8 : NSD_POOL_VECS64; }
// Elements of the per-env shared-memory row region for nc contacts: the
// write-heavy PCR state x, r, z, p, ap, az, bx (7 x rows), the J^T staging
// (12 per joint, 9 per contact) and w (ndof), each array kept 16-byte aligned.
#ifndef NSD_POOL_EXTRA
#define NSD_POOL_EXTRA 4
#endif
// Extra arrays in the fp32 region: 1 contact records, 2 joint records, 4 the H^-1
// diagonal. Measured (C5 fp32, env-steps/s): none 4.25 M, +records 4.18 M, +joint
// records 4.16 M (both cost L1 via the carveout), +H^-1 4.37 M -> 4.
template <class R> __host__ __device__ constexpr int pool_extra() { return sizeof(R) == 4 ? NSD_POOL_EXTRA : 0; }
template <class R> __host__ __device__ inline int row_pool_elems(int rows_static, int nj, int ndof, int nc) {
  const int rows = (rows_static + 3 * nc + 3) & ~3;
  int n = pool_row_vecs<R>() * rows + ((12 * nj + 3) & ~3) + ((9 * nc + 3) & ~3) + ((ndof + 3) & ~3);
  if (pool_extra<R>() & 1) n += 20 * nc;
  if (pool_extra<R>() & 2) n += (24 * nj + 3) & ~3;
  if (pool_extra<R>() & 4) n += (ndof + 3) & ~3;
  return n;
}


// ---- launch wrappers (defined with their kernels). Single scenes: s64 = fp64 J/C
// coefficients (nsd_k_single.cu), s32 = the fp32 mode's float coefficients
// (nsd_k_single32.cu, the same source compiled with NSD_OP32=1).
#define NSD_SINGLE_DECL                                                                                            \
  template <class R> int single_grid_blocks_per_sm(bool tets);                                                     \
  template <class R>                                                                                               \
  cudaError_t launch_single_block(bool tets, int threads, cudaStream_t s, const nsd::Topo<R>& T,                   \
                                  const nsd::Work<R>& W, const nsd::Cfg& c, const nsd::StepOut& o);                \
  template <class R>                                                                                               \
  cudaError_t launch_single_grid(bool tets, int mode, size_t smem, int blocks, cudaStream_t s, const nsd::Topo<R>& T, \
                                 const nsd::Work<R>& W, const nsd::Cfg& c, const nsd::StepOut& o, double* gpart);
namespace s64 {
NSD_SINGLE_DECL
}
namespace s32 {
NSD_SINGLE_DECL
}
#undef NSD_SINGLE_DECL
// k_batch_sub<R, 4/8/16/32> and k_batch_block<R> attributes (a negative value leaves one unset)
template <class R> cudaError_t batch_sub_attrs(int max_dyn_smem, int carveout);
template <class R> cudaError_t batch_block_attrs(int max_optin);
template <class R>
cudaError_t launch_batch_sub(int tpe, int nblk, int threads, size_t smem, cudaStream_t s, const BatchArgs<R>& A);
template <class R>
cudaError_t launch_batch_block(int nblk, int threads, size_t smem, cudaStream_t s, const BatchArgs<R>& A);
// rigid warp path (double state; mixed = fp32 PCR operator)
template <class R>
cudaError_t batch_warp_setup(bool mixed, int max_optin, int threads, size_t smem, int* blocks_per_sm);
template <class R>
cudaError_t launch_batch_warp(bool mixed, int nblk, int threads, size_t smem, cudaStream_t s, const BatchArgs<R>& A);
template <class R>
cudaError_t launch_batch_collide(int nblk, int threads, size_t smem, cudaStream_t s, const BatchArgs<R>& A);

}  // namespace nsdi
