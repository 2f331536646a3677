// The per-timestep non-smooth Newton solve on the device.
//
// One implementation of the reference's newton_step (src/newton.cpp:321-418),
// written against a Team (nsd_team.cuh) so the same code runs as
//   * a cooperative persistent grid for one large scene (C2/C4 FEM scenes),
//   * one CTA for one small scene (C1/C3), and
//   * one warp per environment for the batched RL path (C5), with the
//     environment's working set in shared memory.
//
// Data layout (int32 ids; R = float or double):
//   rows      fixed layout of make_layout (newton.cpp:18-41):
//             [joints 3/5/5/2 | tets 3 each | contact normals | friction pairs]
//   J, static rows (joints, tets): coeff[12*row] = four 3-wide slots, blk[4*row]
//             = the dof3 block (dof/3) of each slot, -1 if unused. A rigid body
//             owns two blocks (linear, angular), a particle one. <= 12 nnz/row.
//   J, contact rows: structured. Per contact the world lever arms (carm) and
//             the NCP scale dc = dphi/dC and friction-active flag (cscale);
//             the three rows act through the relative contact-point velocity
//             dv = (v_a + w_a x r_a) - (v_b + w_b x r_b): n.dv*dc, d1.dv, d2.dv.
//             J^T of a contact is the force f = dc z_n n + z_1 d1 + z_2 d2
//             applied as (f, r_a x f) / (-f, -r_b x f). Same values as the
//             reference's 12-coefficient rows (constraints.cpp:56-91) in fewer
//             loads.
//   C         cd[row] for scalar rows; ctet[9*tet] for the 3x3 Neo-Hookean block.
//   H^-1      hinv[dof] for linear blocks (1/(m+shift)), iwi6[6*blk] (I_w^-1,
//             symmetric) for angular blocks.
//   J^T pull  deterministic body-side gather over incidence lists per dof3
//             block (static joints+tets list, per-step contact list) — no
//             atomics, fixed order, so results are run-to-run bitwise stable
//             (SPEC.md:710 determinism).
// The Schur complement S = J H^-1 J^T + C + eps I is never formed (the
// reference builds it explicitly, newton.cpp:242-290): each PCR iteration
// applies it matrix-free as one pull pass (w = H^-1 J^T z, dof-parallel) and
// one gather pass (Az = J w + C z + eps z, row-parallel).
#pragma once

#include "nsd_math.cuh"
#include "nsd_team.cuh"

// Element assembly (SVD, eigensolver, 3x3 inverses) is called once per Newton
// iteration; a TU whose kernel runs a register-resident PCR loop around it can keep
// it out of line (NSD_ASM_NOINLINE, nsd_k_single.cu) so the loop is not allocated
// for the assembly's register pressure.
#ifdef NSD_ASM_NOINLINE
#define NSD_ASM __device__ __noinline__
#else
#define NSD_ASM __device__
#endif

namespace nsd {

using std::isfinite;
using std::sqrt;

enum BlockKind : int { kParticleLin = 0, kRigidLin = 1, kRigidAng = 2 };

struct Cfg {
  int newton_iterations;
  double step_fraction;
  double epsilon_reg;
  int geometric_stiffness;
  int r_strategy;  // 0 identity, 1 h^2, 2 effective mass
  int ncp_kind;    // 0 min map, 1 FB
  int linear_max_iterations;
  double linear_tolerance;
  int preconditioner;  // 0 none, 1 diagonal
  double newton_tolerance;
  int line_search;
  int linear_method;   // 0 Jacobi, 2 PCG, 3 PCR (solvers.h:8); Gauss-Seidel is not on the device path
};

// Static topology (shared by every environment of a batch).
template <class R> struct Topo {
  int nb, ndof, ncoord, nd3;
  const int* btype;   // per body: 0 particle, 1 rigid
  const R* bmass;
  const R* binertia;  // 9 per body (body frame)
  const int* bdof;
  const int* bcoord;
  const int* d3_body;  // per dof3 block: owning body
  const int* d3_kind;  // BlockKind
  int nj;
  const int* jkind;
  const int* jbody;  // 2 per joint
  const R* jparam;   // 2 per joint: compliance, stiffness
  const int* jrow;   // first row of each joint
  int rows_joint;
  int nt;
  const int* tbody;   // 4 per tet (global body ids)
  const R* tdminv;    // 9 per tet
  const R* tvol;
  const R* tmat;      // 4 per tet: c1, d1, alpha, flags (1 diagonal compliance, 2 linear co-rotational)
  int tdim;           // rows per tet: 3 Neo-Hookean, 6 linear co-rotational (one model per topology)
  const R* tkinv;     // linear model: 36 per tet, the 6x6 isotropic stiffness inverse (materials.cpp:153)
  int rows_static;    // rows_joint + tdim nt
  const int* sinc_off;  // static incidence per dof3 block (nd3 + 1)
  const int* sinc_ent;  // row*4 + slot, ascending rows within a block
  int warp_pull;        // 1: a warp per dof3 block (long incidence lists, FEM); 0: a thread per block
};

// Per-scene (per-env) mutable state and scratch (global or shared memory).
template <class R> struct Work {
  // state
  R* q;         // ncoord, current iterate (in/out)
  R* u;         // ndof, current iterate (in/out)
  const R* q0;  // step-start coordinates q-
  const R* u0;  // step-start velocities u-
  const R* jframe;   // 21 per joint
  const R* f_extra;  // ndof or nullptr
  R h;
  R grav[3];
  // contacts
  int nc;
  const int* cbody;     // 2 per contact
  const R* cgeo;        // 17 per contact: la3 lb3 n3 d1_3 d2_3 thickness mu
  R* cdir;              // 9 per contact: n, d1, d2 (hot copy for the operator)
  R* carm;              // 6 per contact: world lever arms r_a, r_b (per assembly)
  R* cscale;            // 2 per contact: dc = dphi/dC, friction active (0/1)
  const int* cinc_off;  // contact incidence per dof3 block (nd3 + 1)
  const int* cinc_ent;  // contact*4 + slot
  // rows
  int nrows, normal_begin, friction_begin;
  R* coeff;  // 12 per static row (floats in an NSD_OP32 TU, see opg/ops)
  int* blk;  // 4 per static row
  R* jstr;   // batched path: 24 per joint (structured rows, see assemble_joint) or null
  R* crec;   // batched path: 20 per contact (n d1 d2 r_a r_b dc act, 16-byte aligned) or null
  int4* cblk;  // batched path: dof3 blocks (a.lin, a.ang, b.lin, b.ang) per contact
  const int4* jblk;  // batched path: static dof3 blocks per joint (shared by all envs)
  R* qrot;           // batched path: per-body rotation at the current q (9 each), refreshed before assembly
  R* hv;
  R* cd;
  R* ctet;   // 9 per tet
  R* lam;
  // PCR vectors
  R *x, *xn, *r, *rn, *z, *zn, *p, *ap, *az, *inv, *bx, *qp;
  // dof vectors
  R *ut, *g, *gp, *up, *shift, *hinv, *w, *du, *ub;
  // dof3 block data
  R* iw6;   // 6 per block (sym: xx yy zz xy xz yz), angular blocks
  R* iwi6;  // inverse
  // per-iteration decision row (decision vectors, see StepOut::dec) or null
  unsigned char* dec;
  // partitioned grid PCR (nsd_part.cuh): per-CTA rows and local dof3 blocks, the
  // CTAs touching each dof3 block (flat local-block indices), shared-block partials
  const int *part_row_off, *part_rows, *part_lb_off, *part_lb_blk, *part_gb_off, *part_gb_ent;
  void* part_partial;
  int part_mr, part_ml, part_mx;  // per-CTA maxima: rows, local blocks, exchange entries
};

// Decision-vector flags, one byte per contact / tet / dof per Newton
// iteration, plus the PCR exit reason; the oracle writes the same layout.
enum DecFlags : unsigned char {
  kDecNormalKept = 1,     // contact: dphi/dC != 0, the normal J row exists (newton.cpp:187)
  kDecFrictionOn = 2,     // contact: mu lambda_n > 0 (newton.cpp:200)
  kDecWCap = 4,           // contact: friction W hit the 1e12 cap (ncp.cpp:37-48)
  kDecWZero = 8,          // contact: min-map friction on its stick branch, W = 0 (ncp.cpp:37-41)
  kDecNcpBranch = 16,     // contact: FB origin root == 0 / min-map branch c <= r lambda (ncp.cpp:11,24)
  kDecPsd = 1,            // tet: Hessian projected to PSD (materials.cpp:85-88)
  kDecDiagFallback = 2,   // tet: diagonal compliance fallback (materials.cpp:96-100)
  kDecGsSkip = 1,         // dof: |du_k| < 1e-10, no secant (newton.cpp:306)
  kDecGsClamp = 2,        // dof: c_k >= 0 clamped to a zero shift (newton.cpp:308)
  kDecRigidDof = 4,       // dof: rigid, shift zeroed by the policy (newton.cpp:316-317)
};
enum PcrExit : unsigned char { kExitBudget = 0, kExitTol = 1, kExitMonotone = 2, kExitBreakdown = 3, kExitNone = 4 };

struct IterOut {
  double residual_inf, merit_l2, comp_error_max, cone_violation_max, step_size, linear_residual;
  int linear_iterations, linear_breakdown;
};

struct StepOut {
  unsigned char* dec;  // newton_iterations x dec_stride decision bytes (may be null):
                       // [nc contacts][nt tets][ndof dofs][PCR exit reason]
  int dec_stride;
  IterOut* iters;  // newton_iterations (may be null)
  double* hist;    // newton_iterations * (max_lin + 1) (may be null)
  int* hist_len;   // newton_iterations (may be null)
  double* tel;     // 6 per contact (may be null)
  double* fin;     // 8: final_residual_inf, final_comp, final_cone, min_gap, min_diag_shift, aborted, converged, n_iterations
  unsigned long long* ptime;  // diagnostics (NSD_PHASE_TIMING): clock64 cycles per solver phase, or null
};

// Phase clock for diagnostics: adds the cycles since the last mark to slot k.
struct PhaseClock {
  unsigned long long* dst;
  long long t0;
  __device__ explicit PhaseClock(unsigned long long* d, bool leader) : dst(leader ? d : nullptr), t0(0) {
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

struct NoClock {
  __device__ __forceinline__ void mark(int) const {}
};

// ------------------------------------------------------------------ helpers
template <class R> __device__ __forceinline__ V3<R> ld3(const R* p) { return v3(p[0], p[1], p[2]); }
template <class R> __device__ __forceinline__ void st3(R* p, V3<R> v) {
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
}
// Operator coefficient arrays (coeff, ctet, cdir, carm): element i of array a, stored in
// R, or — single-scene fp32 mode, a TU compiled with NSD_OP32=1 (nsd_k_single32.cu) —
// as float in the same buffer. State, row and dof vectors and all arithmetic stay in
// R (fp64): the fp32 mode halves the operator's coefficient stream only (the batch
// warp solver's mixed mode likewise). A compile-time choice: a run-time flag cost
// 16 % on C1 (both load paths in every coefficient access).
#ifndef NSD_OP32
#define NSD_OP32 0
#endif
template <class R> __device__ __forceinline__ R opg(const Work<R>&, const R* a, size_t i) {
  if constexpr (NSD_OP32 != 0)
    return R(reinterpret_cast<const float*>(a)[i]);
  else
    return a[i];
}
template <class R> __device__ __forceinline__ void ops(const Work<R>&, R* a, size_t i, R v) {
  if constexpr (NSD_OP32 != 0)
    reinterpret_cast<float*>(a)[i] = static_cast<float>(v);
  else
    a[i] = v;
}
template <class R> __device__ __forceinline__ V3<R> opg3(const Work<R>& W, const R* a, size_t i) {
  return v3(opg(W, a, i), opg(W, a, i + 1), opg(W, a, i + 2));
}
template <class R> __device__ __forceinline__ void ops3(const Work<R>& W, R* a, size_t i, V3<R> v) {
  ops(W, a, i, v.x);
  ops(W, a, i + 1, v.y);
  ops(W, a, i + 2, v.z);
}
template <class R> __device__ __forceinline__ V3<R> sym_mul(const R* s6, V3<R> v) {
  // s6 = xx yy zz xy xz yz
  return v3(s6[0] * v.x + s6[3] * v.y + s6[4] * v.z, s6[3] * v.x + s6[1] * v.y + s6[5] * v.z,
            s6[4] * v.x + s6[5] * v.y + s6[2] * v.z);
}
template <class R> __device__ __forceinline__ R sym_quad(const R* s6, V3<R> v) { return dot(v, sym_mul(s6, v)); }

template <class R> __device__ __forceinline__ M3<R> body_rot(const Topo<R>& T, const R* q, int b) {
  if (b < 0 || T.btype[b] == 0) return m3_identity<R>();
  const R* t = q + T.bcoord[b] + 3;
  return quat_rot(t[0], t[1], t[2], t[3]);
}
// Rotation from the per-body cache when present (batched path), else from q.
template <class R> __device__ __forceinline__ M3<R> body_rot_c(const Topo<R>& T, const Work<R>& W, const R* q, int b) {
  if (!W.qrot || b < 0 || T.btype[b] == 0) return body_rot(T, q, b);
  M3<R> m;
#pragma unroll
  for (int i = 0; i < 9; ++i) m.a[i] = W.qrot[9 * b + i];
  return m;
}
template <class R> __device__ __forceinline__ V3<R> body_pos(const Topo<R>& T, const R* q, int b) {
  return ld3(q + T.bcoord[b]);
}
template <class R> __device__ __forceinline__ void body_blocks(const Topo<R>& T, int b, int& lin, int& ang) {
  if (b < 0) {
    lin = ang = -1;
    return;
  }
  lin = T.bdof[b] / 3;
  ang = T.btype[b] == 1 ? lin + 1 : -1;
}

// c^T M^-1 c on one block: unshifted (1/m, I_w^-1) or shifted H^-1.
template <class R>
__device__ __forceinline__ R block_quad(const Topo<R>& T, const Work<R>& W, int b, V3<R> c, bool shifted) {
  if (T.d3_kind[b] == kRigidAng) return sym_quad(W.iwi6 + 6 * b, c);
  if (shifted) {
    const R* hi = W.hinv + 3 * b;
    return c.x * c.x * hi[0] + c.y * c.y * hi[1] + c.z * c.z * hi[2];
  }
  const R m = T.bmass[T.d3_body[b]];
  return c.x * c.x / m + c.y * c.y / m + c.z * c.z / m;
}

template <class R> __device__ __forceinline__ R r_factor(R emd, R h, bool position, int strat) {
  const R ts = position ? h * h : h;
  if (strat == 0) return R(1);
  if (strat == 1) return ts;
  return emd <= R(0) ? ts : ts * emd;
}

template <class R> struct PhiV {
  R v, dc, dl;
};
template <class R> __device__ __forceinline__ PhiV<R> phi_n(R c, R lam, R r, int kind) {  // ncp.cpp:7-32
  PhiV<R> o;
  const R rl = r * lam;
  if (kind == 0) {
    if (c <= rl) {
      o.v = c;
      o.dc = R(1);
      o.dl = R(0);
    } else {
      o.v = rl;
      o.dc = R(0);
      o.dl = r;
    }
    return o;
  }
  const R root = sqrt(c * c + rl * rl);
  o.v = c + rl - root;
  if (root == R(0)) {
    o.dc = R(0);
    o.dl = r;
  } else {
    o.dc = R(1) - c / root;
    o.dl = (R(1) - rl / root) * r;
  }
  return o;
}
template <class R> __device__ __forceinline__ R friction_W(R vt, R lf, R mln, R r, int kind) {  // ncp.cpp:34-49
  const R degenerate = R(1e-12), cap = R(1e12);
  if (kind == 0) {
    if (vt <= r * (mln - lf)) return R(0);
    if (mln <= degenerate) return cap;
    return (vt - r * (mln - lf)) / mln;
  }
  const R slack = mln - lf;
  const R root = sqrt(vt * vt + r * r * slack * slack);
  const R numer = root - r * slack;
  const R denom = vt + r * mln - root;
  if (denom <= degenerate) return cap;
  return r * numer / denom;
}

// Structural slot usage of joint rows (joint_rows, constraints.cpp:141-220):
// point/translation rows use all four slots, axis-dot rows the angular ones.
__host__ __device__ __forceinline__ int joint_nrows(int kind) { return kind == 3 ? 2 : (kind == 0 ? 3 : 5); }
__host__ __device__ __forceinline__ bool joint_row_linear(int kind, int k) {
  if (kind == 0) return true;
  if (kind == 1) return k < 3;
  if (kind == 2) return k < 2;
  return false;
}

// ------------------------------------------------------------------ contact geometry
template <class R> struct CView {
  int ba, bb, al, aa, bl, bA;  // bodies and their lin/ang dof3 blocks (-1 = none)
  V3<R> n, d1, d2, ra, rb;
  R dc, act;
};
template <class R> __device__ __forceinline__ CView<R> contact_view(const Topo<R>& T, const Work<R>& W, int c) {
  NSD_CHECK(c >= 0 && c < W.nc);
  CView<R> v;
  v.ba = W.cbody[2 * c];
  v.bb = W.cbody[2 * c + 1];
  body_blocks(T, v.ba, v.al, v.aa);
  body_blocks(T, v.bb, v.bl, v.bA);
  v.n = opg3(W, W.cdir, 9 * c);
  v.d1 = opg3(W, W.cdir, 9 * c + 3);
  v.d2 = opg3(W, W.cdir, 9 * c + 6);
  v.ra = opg3(W, W.carm, 6 * c);
  v.rb = opg3(W, W.carm, 6 * c + 3);
  v.dc = W.cscale[2 * c];
  v.act = W.cscale[2 * c + 1];
  return v;
}
// Relative contact-point velocity of a dof vector: (v_a + w_a x r_a) - (v_b + w_b x r_b).
template <class R> __device__ __forceinline__ V3<R> contact_dv(const CView<R>& c, const R* v) {
  V3<R> d = v3(R(0), R(0), R(0));
  if (c.al >= 0) {
    d = ld3(v + 3 * c.al);
    if (c.aa >= 0) d = d + cross(ld3(v + 3 * c.aa), c.ra);
  }
  if (c.bl >= 0) {
    d = d - ld3(v + 3 * c.bl);
    if (c.bA >= 0) d = d - cross(ld3(v + 3 * c.bA), c.rb);
  }
  return d;
}
// Direction-row quadratic form d^T J M^-1 J^T d for a contact row along dir.
template <class R>
__device__ __forceinline__ R contact_quad(const Topo<R>& T, const Work<R>& W, const CView<R>& c, V3<R> dir,
                                          bool shifted) {
  R s = R(0);
  if (c.al >= 0) {
    s += block_quad(T, W, c.al, dir, shifted);
    if (c.aa >= 0) s += block_quad(T, W, c.aa, cross(c.ra, dir), shifted);
  }
  if (c.bl >= 0) {
    s += block_quad(T, W, c.bl, dir, shifted);
    if (c.bA >= 0) s += block_quad(T, W, c.bA, cross(c.rb, dir), shifted);
  }
  return s;
}

// ------------------------------------------------------------------ row-level J and diag
// J_i . v for static row i (4 slots x 3).
template <class R> __device__ __forceinline__ R slot_dot(const Work<R>& W, int i, const R* v) {
  const int* b4 = W.blk + 4 * i;
  R s = R(0);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int b = b4[k];
    if (b < 0) continue;
    const R* vb = v + 3 * b;
    const V3<R> c = opg3(W, W.coeff, 12 * (size_t)i + 3 * k);
    s += c.x * vb[0] + c.y * vb[1] + c.z * vb[2];
  }
  return s;
}
template <class R>
__device__ __forceinline__ R slot_quad(const Topo<R>& T, const Work<R>& W, int i, bool shifted) {
  const int* b4 = W.blk + 4 * i;
  R s = R(0);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int b = b4[k];
    if (b < 0) continue;
    s += block_quad(T, W, b, opg3(W, W.coeff, 12 * (size_t)i + 3 * k), shifted);
  }
  return s;
}
// J_i . v for any row.
template <class R> __device__ __forceinline__ R row_J(const Topo<R>& T, const Work<R>& W, int i, const R* v) {
  NSD_CHECK(i >= 0 && i < W.nrows);
  if (i < T.rows_static) return slot_dot(W, i, v);
  if (i < W.friction_begin) {
    const CView<R> c = contact_view(T, W, i - W.normal_begin);
    return c.dc == R(0) ? R(0) : c.dc * dot(c.n, contact_dv(c, v));
  }
  const int k = i - W.friction_begin, c0 = k >> 1;
  const CView<R> c = contact_view(T, W, c0);
  if (c.act == R(0)) return R(0);
  return dot((k & 1) ? c.d2 : c.d1, contact_dv(c, v));
}
// J_i H^-1 J_i^T (shifted) for any row.
template <class R> __device__ __forceinline__ R row_quad(const Topo<R>& T, const Work<R>& W, int i) {
  if (i < T.rows_static) return slot_quad(T, W, i, true);
  if (i < W.friction_begin) {
    const CView<R> c = contact_view(T, W, i - W.normal_begin);
    return c.dc == R(0) ? R(0) : contact_quad(T, W, c, c.dc * c.n, true);
  }
  const int k = i - W.friction_begin;
  const CView<R> c = contact_view(T, W, k >> 1);
  if (c.act == R(0)) return R(0);
  return contact_quad(T, W, c, (k & 1) ? c.d2 : c.d1, true);
}

// J_i^T d as (dof3 block, 3-vector) pairs, f(block, v): the transpose of row_J for one
// row (Gauss-Seidel's incremental w = H^-1 J^T x update).
template <class R, class F>
__device__ __forceinline__ void row_JT(const Topo<R>& T, const Work<R>& W, int i, R d, F&& f) {
  if (i < T.rows_static) {
    const int* b4 = W.blk + 4 * i;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (b4[k] >= 0) f(b4[k], d * opg3(W, W.coeff, 12 * (size_t)i + 3 * k));
    return;
  }
  const bool normal = i < W.friction_begin;
  const int k = i - W.friction_begin, c0 = normal ? i - W.normal_begin : (k >> 1);
  const CView<R> c = contact_view(T, W, c0);
  const R sc = normal ? c.dc : c.act;
  if (sc == R(0)) return;
  const V3<R> dir = normal ? c.n : ((k & 1) ? c.d2 : c.d1);
  const V3<R> fv = (sc * d) * dir;
  if (c.al >= 0) {
    f(c.al, fv);
    if (c.aa >= 0) f(c.aa, cross(c.ra, fv));
  }
  if (c.bl >= 0) {
    f(c.bl, -fv);
    if (c.bA >= 0) f(c.bA, -cross(c.rb, fv));
  }
}

// ------------------------------------------------------------------ static row blocks (once per step)
template <class R, bool kTets, class Team> __device__ void setup_row_blocks(Team& t, const Topo<R>& T, Work<R>& W) {
  const int ng = T.nj + (kTets ? T.nt : 0);
  for (int g = t.rank(); g < ng; g += t.size()) {
    if (g < T.nj) {
      const int kind = T.jkind[g], r0 = T.jrow[g];
      int al, aa, bl, ba;
      body_blocks(T, T.jbody[2 * g], al, aa);
      body_blocks(T, T.jbody[2 * g + 1], bl, ba);
      const int nr = joint_nrows(kind);
      for (int k = 0; k < nr; ++k) {
        int* b = W.blk + 4 * (r0 + k);
        const bool lin = joint_row_linear(kind, k);
        b[0] = lin ? al : -1;
        b[1] = aa;
        b[2] = lin ? bl : -1;
        b[3] = ba;
        if (b[2] >= 0 && b[2] == b[0]) b[2] = -1;  // same body on both sides: slots merge
        if (b[3] >= 0 && b[3] == b[1]) b[3] = -1;
      }
    } else {
      const int e = g - T.nj;
      const int r0 = T.rows_joint + T.tdim * e;
      int vb[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) vb[k] = T.bdof[T.tbody[4 * e + k]] / 3;
      for (int i = 0; i < T.tdim; ++i) {
        int* b = W.blk + 4 * (r0 + i);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          NSD_CHECK(vb[k] >= 0 && vb[k] < T.nd3);
          b[k] = vb[k];
        }
      }
    }
  }
}

// Adds a coefficient contribution into the slot owning `blk` (merged same-body case).
template <class R> __device__ __forceinline__ void slot_add(R* c12, const int* b4, int s, int blk, V3<R> v) {
  int k = s;
  if (blk < 0) return;
  if (b4[s] != blk) k = (s == 2 ? 0 : 1);
  c12[3 * k] += v.x;
  c12[3 * k + 1] += v.y;
  c12[3 * k + 2] += v.z;
}

// ------------------------------------------------------------------ assembly (newton.cpp:100-231)
struct AsmStats {
  double hmax, hsq, comp, cone;
};

template <class R>
NSD_ASM void assemble_joint(const Topo<R>& T, Work<R>& W, const R* q, int j, R h, AsmStats& st) {
  const int kind = T.jkind[j], ba = T.jbody[2 * j], bb = T.jbody[2 * j + 1];
  const R* fr = W.jframe + 21 * j;
  const V3<R> anc_a = ld3(fr), anc_b = ld3(fr + 3), ax_a = ld3(fr + 6), ax_a2 = ld3(fr + 9), ax_b1 = ld3(fr + 12),
              ax_b2 = ld3(fr + 15), rest = ld3(fr + 18);
  const M3<R> Ra = body_rot_c(T, W, q, ba), Rb = body_rot_c(T, W, q, bb);
  const bool rig_a = ba >= 0 && T.btype[ba] == 1, rig_b = bb >= 0 && T.btype[bb] == 1;
  V3<R> wa, wb, ra = v3(R(0), R(0), R(0)), rb = ra;
  if (ba < 0) wa = anc_a;
  else if (!rig_a) wa = body_pos(T, q, ba);
  else {
    ra = mul(Ra, anc_a);
    wa = body_pos(T, q, ba) + ra;
  }
  if (bb < 0) wb = anc_b;
  else if (!rig_b) wb = body_pos(T, q, bb);
  else {
    rb = mul(Rb, anc_b);
    wb = body_pos(T, q, bb) + rb;
  }
  const R comp = T.jparam[2 * j];
  const R e_bend = T.jparam[2 * j + 1] > R(0) ? R(1) / T.jparam[2 * j + 1] : R(0);
  const int r0 = T.jrow[j];
  const V3<R> axw = ba < 0 ? ax_a : mul(Ra, ax_a);
  int al, aa, bl, bA;
  body_blocks(T, ba, al, aa);
  body_blocks(T, bb, bl, bA);

  auto emit = [&](int k, R value, R e) {
    const int row = r0 + k;
    const R lam = W.lam[row] / h;
    const R hv = (value + e * lam) / h;
    W.hv[row] = hv;
    W.cd[row] = e / (h * h);
    st.hmax = fmax(st.hmax, (double)ab(hv));
    st.hsq += (double)hv * (double)hv;
  };
  // Structured form of the joint's rows (batched path): lever arms, point-row
  // directions, axis-row angular vectors. A point row along d has J = [d | arm_a x d
  // | -d | -(arm_b x d)] (arm_a gains -(w_a - w_b) for prismatic: ra x d + d x t =
  // (ra - t) x d, constraints.cpp:195-196); an axis row J = [0 | c | 0 | -c].
  R* js = W.jstr ? W.jstr + 24 * j : nullptr;
  if (js) {
    st3(js, kind == 2 && rig_a ? ra - (wa - wb) : ra);
    st3(js + 3, rb);
  }
  auto point_row = [&](int k, V3<R> d, R value, bool prism) {
    if (js) {
      st3(js + 6 + 3 * k, d);
      emit(k, value, comp);
      return;
    }
    R c[12];
    const int* b = W.blk + 4 * (r0 + k);
#pragma unroll
    for (int i = 0; i < 12; ++i) c[i] = R(0);
    slot_add(c, b, 0, al, d);
    if (rig_a) slot_add(c, b, 1, aa, cross(ra, d));
    slot_add(c, b, 2, bl, -d);
    if (rig_b) slot_add(c, b, 3, bA, -cross(rb, d));
    if (prism && rig_a) slot_add(c, b, 1, aa, cross(d, wa - wb));  // t x d (constraints.cpp:195-196)
#pragma unroll
    for (int i = 0; i < 12; ++i) ops(W, W.coeff, 12 * (size_t)(r0 + k) + i, c[i]);
    emit(k, value, comp);
  };
  const int n_point = (kind == 0 || kind == 1) ? 3 : (kind == 2 ? 2 : 0);
  auto axis_row = [&](int k, V3<R> xa, V3<R> xb, R restv, R e) {
    if (js) {
      st3(js + 15 + 3 * (k - n_point), cross(xa, xb));
      emit(k, dot(xa, xb) - restv, e);
      return;
    }
    R c[12];
    const int* b = W.blk + 4 * (r0 + k);
#pragma unroll
    for (int i = 0; i < 12; ++i) c[i] = R(0);
    const V3<R> cr = cross(xa, xb);
    if (rig_a) slot_add(c, b, 1, aa, cr);
    if (rig_b) slot_add(c, b, 3, bA, -cr);
#pragma unroll
    for (int i = 0; i < 12; ++i) ops(W, W.coeff, 12 * (size_t)(r0 + k) + i, c[i]);
    emit(k, dot(xa, xb) - restv, e);
  };
  const V3<R> e0 = v3(R(1), R(0), R(0)), e1 = v3(R(0), R(1), R(0)), e2 = v3(R(0), R(0), R(1));
  if (kind == 0 || kind == 1) {
    point_row(0, e0, wa.x - wb.x, false);
    point_row(1, e1, wa.y - wb.y, false);
    point_row(2, e2, wa.z - wb.z, false);
    if (kind == 1) {
      const V3<R> b1 = bb < 0 ? ax_b1 : mul(Rb, ax_b1), b2 = bb < 0 ? ax_b2 : mul(Rb, ax_b2);
      axis_row(3, axw, b1, rest.x, comp);
      axis_row(4, axw, b2, rest.y, comp);
    }
  } else if (kind == 2) {
    int sm = 0;  // tangent_basis(ax) (constraints.cpp:93-101)
    if (ab(axw.y) < ab(axw.x)) sm = 1;
    if (ab(axw.z) < ab(axw[sm])) sm = 2;
    V3<R> ee = v3(R(0), R(0), R(0));
    ee[sm] = R(1);
    const V3<R> t1 = normalize(ee - dot(ee, axw) * axw);
    const V3<R> t2 = cross(axw, t1);
    const V3<R> d = wa - wb;
    point_row(0, t1, dot(t1, d), true);
    point_row(1, t2, dot(t2, d), true);
    const V3<R> a2 = ba < 0 ? ax_a2 : mul(Ra, ax_a2);
    const V3<R> b1 = bb < 0 ? ax_b1 : mul(Rb, ax_b1), b2 = bb < 0 ? ax_b2 : mul(Rb, ax_b2);
    axis_row(2, axw, b1, rest.x, comp);
    axis_row(3, axw, b2, rest.y, comp);
    axis_row(4, a2, b2, rest.z, comp);
  } else {
    const V3<R> b1 = bb < 0 ? ax_b1 : mul(Rb, ax_b1), b2 = bb < 0 ? ax_b2 : mul(Rb, ax_b2);
    axis_row(0, axw, b1, rest.x, e_bend);
    axis_row(1, axw, b2, rest.y, e_bend);
  }
}

// Linear co-rotational element rows (materials.cpp:140-178): F = Ds Dm^-1, signed
// SVD, R = U V^T, stretch S = V diag(s) V^T, strain = voigt(S - I) (Voigt order
// xx yy zz 2yz 2xz 2xy, materials.cpp:132-136), c = V_e K strain, compliance
// K^-1 / V_e; the rotation variation w = 2 G^-1 axial(R^T dF) with
// G = tr(S) I - S enters each Jacobian column unless |det G| <= 1e-12 (frozen
// frame). h = E (c + lambda/h) / h and C = E / h^2 over the 6x6 block
// (newton.cpp:146-160).
template <class R>
__device__ void assemble_tet_linear(const Topo<R>& T, Work<R>& W, int e, R h, const M3<R>& dm, const Svd<R>& sv, R vol,
                                    AsmStats& st) {
  M3<R> Vt = transpose(sv.V);
  M3<R> Rm = mul(sv.U, Vt);
  M3<R> VS;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    VS(i, 0) = sv.V(i, 0) * sv.S.x;
    VS(i, 1) = sv.V(i, 1) * sv.S.y;
    VS(i, 2) = sv.V(i, 2) * sv.S.z;
  }
  const M3<R> S = mul(VS, Vt);
  R strain[6] = {S(0, 0) - R(1), S(1, 1) - R(1), S(2, 2) - R(1), R(2) * S(1, 2), R(2) * S(0, 2), R(2) * S(0, 1)};
  // isotropic stiffness from the Lame constants (mu = 2 c1, lambda = 2 d1; materials.cpp isotropic_stiffness)
  const R mu = R(2) * T.tmat[4 * e], lam = R(2) * T.tmat[4 * e + 1];
  R c[6];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    R k = R(0);
#pragma unroll
    for (int j = 0; j < 3; ++j) k += (i == j ? lam + R(2) * mu : lam) * strain[j];
    c[i] = vol * k;
    c[3 + i] = vol * (mu * strain[3 + i]);
  }
  const R* ki = T.tkinv + 36 * e;
  R E[36];
#pragma unroll
  for (int i = 0; i < 36; ++i) E[i] = ki[i] / vol;
  const int r0 = T.rows_joint + 6 * e;
  R cl[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) cl[i] = c[i] + W.lam[r0 + i] / h;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    R acc = R(0);
#pragma unroll
    for (int j = 0; j < 6; ++j) acc += E[6 * i + j] * cl[j];
    const R hv = acc / h;
    W.hv[r0 + i] = hv;
    st.hmax = fmax(st.hmax, (double)ab(hv));
    st.hsq += (double)hv * (double)hv;
  }
#pragma unroll
  for (int i = 0; i < 36; ++i) ops(W, W.ctet, 36 * (size_t)e + i, E[i] / (h * h));
  // G = tr(S) I - S and its inverse (frozen frame when |det G| <= 1e-12)
  const R tr = S(0, 0) + S(1, 1) + S(2, 2);
  M3<R> G;
#pragma unroll
  for (int i = 0; i < 9; ++i) G.a[i] = -S.a[i];
  G(0, 0) += tr;
  G(1, 1) += tr;
  G(2, 2) += tr;
  const bool rot_term = fabs((double)det3(G)) > 1e-12;
  const M3<R> Gi = rot_term ? inverse3(G) : m3_zero<R>();
  // Jacobian columns 3k + d: dF.row(d) = Dm^-1.row(k-1) (k > 0) or -sum_c Dm^-1.row(c).
  // The rows are hoisted and selected by value: a runtime-indexed read of dm here
  // returned identity rows on sm_100a (caught by tests/test_gpu_parity.py).
  const V3<R> dm0 = v3(dm(0, 0), dm(0, 1), dm(0, 2)), dm1 = v3(dm(1, 0), dm(1, 1), dm(1, 2)),
              dm2 = v3(dm(2, 0), dm(2, 1), dm(2, 2));
  const V3<R> dmsum = -(dm0 + dm1 + dm2);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const V3<R> rowv = k == 0 ? dmsum : (k == 1 ? dm0 : (k == 2 ? dm1 : dm2));
      // R^T dF with dF = e_d rowv^T: (R^T dF)(i, j) = R(d, i) rowv_j
      M3<R> A;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) A(a, b) = Rm(d, a) * rowv[b];
      if (rot_term) {
        const V3<R> ax = v3(R(0.5) * (A(2, 1) - A(1, 2)), R(0.5) * (A(0, 2) - A(2, 0)), R(0.5) * (A(1, 0) - A(0, 1)));
        const V3<R> w = R(2) * mul(Gi, ax);
        M3<R> Wk = m3_zero<R>();  // skew(w)
        Wk(0, 1) = -w.z;
        Wk(0, 2) = w.y;
        Wk(1, 0) = w.z;
        Wk(1, 2) = -w.x;
        Wk(2, 0) = -w.y;
        Wk(2, 1) = w.x;
        const M3<R> WS = mul(Wk, S);
#pragma unroll
        for (int i = 0; i < 9; ++i) A.a[i] -= WS.a[i];
      }
      const R sym[6] = {A(0, 0), A(1, 1), A(2, 2), R(2) * (R(0.5) * (A(1, 2) + A(2, 1))),
                        R(2) * (R(0.5) * (A(0, 2) + A(2, 0))), R(2) * (R(0.5) * (A(0, 1) + A(1, 0)))};
#pragma unroll
      for (int i = 0; i < 6; ++i) ops(W, W.coeff, 12 * (size_t)(r0 + i) + 3 * k + d, sym[i]);
    }
  }
}

// Neo-Hookean element rows (materials.cpp:180-193, 57-114).
template <class R>
NSD_ASM void assemble_tet(const Topo<R>& T, Work<R>& W, const R* q, int e, R h, AsmStats& st) {
  const int* tb = T.tbody + 4 * e;
  V3<R> p[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) p[k] = body_pos(T, q, tb[k]);
  M3<R> dm;
#pragma unroll
  for (int i = 0; i < 9; ++i) dm.a[i] = T.tdminv[9 * e + i];
  M3<R> ds;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const V3<R> d = p[k + 1] - p[0];
    ds(0, k) = d.x;
    ds(1, k) = d.y;
    ds(2, k) = d.z;
  }
  const M3<R> F = mul(ds, dm);
  const Svd<R> sv = svd3_signed(F);
  const R vol = T.tvol[e];
  if (T.tdim == 6) {
    if (W.dec) W.dec[W.nc + e] = 0;  // the linear model has no compliance decisions
    assemble_tet_linear(T, W, e, h, dm, sv, vol, st);
    return;
  }
  const R c1 = T.tmat[4 * e], d1 = T.tmat[4 * e + 1], alpha = T.tmat[4 * e + 2];
  const bool diag_only = (static_cast<int>(T.tmat[4 * e + 3]) & 1) != 0;
  const V3<R> s = sv.S;
  const R J = s.x * s.y * s.z;  // gradient with (J - alpha), materials.cpp:57-61
  const V3<R> dj = v3(s.y * s.z, s.x * s.z, s.x * s.y);
  const R kk = R(2) * d1 * (J - alpha);
  const R tc1 = R(2) * c1;
  const V3<R> cg = v3(vol * (tc1 * s.x + kk * dj.x), vol * (tc1 * s.y + kk * dj.y), vol * (tc1 * s.z + kk * dj.z));
  const R k0 = R(2) * J - alpha;  // Hessian, materials.cpp:63-74
  const R k1 = d1 * s.z * k0, k2 = d1 * s.y * k0, k3 = d1 * s.x * k0;
  M3<R> H;
  H(0, 0) = R(2) * (d1 * s.y * s.y * s.z * s.z + c1);
  H(1, 1) = R(2) * (d1 * s.x * s.x * s.z * s.z + c1);
  H(2, 2) = R(2) * (d1 * s.x * s.x * s.y * s.y + c1);
  H(0, 1) = H(1, 0) = R(2) * k1;
  H(0, 2) = H(2, 0) = R(2) * k2;
  H(1, 2) = H(2, 1) = R(2) * k3;
  unsigned char tflags = 0;
  {  // compliance_block (materials.cpp:82-102): PSD check with the restated eigensolver
    V3<R> ev;
    M3<R> dummy;
    sym_eig3<R, false>(H, ev, dummy);
    if (mn(ev.x, mn(ev.y, ev.z)) <= R(0)) {
      H = project_psd3(H);
      tflags |= kDecPsd;
    }
  }
  M3<R> N;
#pragma unroll
  for (int i = 0; i < 9; ++i) N.a[i] = vol * H.a[i];
  M3<R> E;
  bool use_diag = diag_only;
  if (!use_diag) {
    const R det = det3(N);
    if (!isfinite(det) || fabs((double)det) < 1e-300) use_diag = true;
  }
  if (use_diag) tflags |= kDecDiagFallback;
  if (W.dec) W.dec[W.nc + e] = tflags;
  if (use_diag) {
    E = m3_zero<R>();
    E(0, 0) = N(0, 0) > R(0) ? R(1) / N(0, 0) : R(0);
    E(1, 1) = N(1, 1) > R(0) ? R(1) / N(1, 1) : R(0);
    E(2, 2) = N(2, 2) > R(0) ? R(1) / N(2, 2) : R(0);
  } else {
    E = inverse3(N);
  }
  const int r0 = T.rows_joint + 3 * e;  // h = E (c + lambda/h) / h, C = E / h^2, J = ds/dq
  const R l0 = W.lam[r0] / h, l1 = W.lam[r0 + 1] / h, l2 = W.lam[r0 + 2] / h;
  const V3<R> cl = v3(cg.x + l0, cg.y + l1, cg.z + l2);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const R hv = (E(i, 0) * cl.x + E(i, 1) * cl.y + E(i, 2) * cl.z) / h;
    W.hv[r0 + i] = hv;
    st.hmax = fmax(st.hmax, (double)ab(hv));
    st.hsq += (double)hv * (double)hv;
    const V3<R> ui = col(sv.U, i);
    const V3<R> wi = mul(dm, col(sv.V, i));
    const size_t c = 12 * (size_t)(r0 + i);
    const R w0 = -(wi.x + wi.y + wi.z);
    ops3(W, W.coeff, c, w0 * ui);
    ops3(W, W.coeff, c + 3, wi.x * ui);
    ops3(W, W.coeff, c + 6, wi.y * ui);
    ops3(W, W.coeff, c + 9, wi.z * ui);
  }
#pragma unroll
  for (int i = 0; i < 9; ++i) ops(W, W.ctet, 9 * (size_t)e + i, E.a[i] / (h * h));
}

// Contact rows (newton.cpp:166-218; constraints.cpp:67-91, 103-115) in the
// structured form: lever arms, NCP scale and friction flag per contact.
// contact_gap (constraints.cpp:67-71) uncontracted: n . (p_a - p_b) - thickness with
// p = position + R(quaternion) local (State::world_point), the oracle's roundings.
template <class R>
__device__ __forceinline__ R contact_gap_strict(const Topo<R>& T, const R* q, int ba, int bb, V3<R> la, V3<R> lb,
                                                V3<R> n, R thick) {
  auto wp = [&](int b, V3<R> l) {
    if (b < 0) return l;
    const R* p = q + T.bcoord[b];
    if (T.btype[b] == 0) return v3(p[0], p[1], p[2]);
    return sworld(quat_rot_strict(p[3], p[4], p[5], p[6]), l, v3(p[0], p[1], p[2]));
  };
  const V3<R> pa = wp(ba, la), pb = wp(bb, lb);
  return ssub(sdot(n, v3(ssub(pa.x, pb.x), ssub(pa.y, pb.y), ssub(pa.z, pb.z))), thick);
}

template <class R>
NSD_ASM void assemble_contact(const Topo<R>& T, Work<R>& W, const R* q, const R* u, int c, R h, const Cfg& cfg,
                                 AsmStats& st) {
  const int ba = W.cbody[2 * c], bb = W.cbody[2 * c + 1];
  const R* g = W.cgeo + 17 * c;
  const V3<R> la = ld3(g), lb = ld3(g + 3);
  const R thick = g[15], mu = g[16];
  const bool rig_a = ba >= 0 && T.btype[ba] == 1, rig_b = bb >= 0 && T.btype[bb] == 1;
  V3<R> pa, pb, ra = v3(R(0), R(0), R(0)), rb = ra;
  if (ba < 0) pa = la;
  else if (!rig_a) pa = body_pos(T, q, ba);
  else {
    ra = mul(body_rot_c(T, W, q, ba), la);
    pa = body_pos(T, q, ba) + ra;
  }
  if (bb < 0) pb = lb;
  else if (!rig_b) pb = body_pos(T, q, bb);
  else {
    rb = mul(body_rot_c(T, W, q, bb), lb);
    pb = body_pos(T, q, bb) + rb;
  }
  if (!W.crec) {  // the batched path keeps the same data in its contact record only
    ops3(W, W.carm, 6 * (size_t)c, ra);
    ops3(W, W.carm, 6 * (size_t)c + 3, rb);
  }
  CView<R> cv;
  cv.ba = ba;
  cv.bb = bb;
  body_blocks(T, ba, cv.al, cv.aa);
  body_blocks(T, bb, cv.bl, cv.bA);  // a == b needs no merge: both sides enter dv exactly as compress() sums them
  cv.n = ld3(g + 6);
  cv.d1 = ld3(g + 9);
  cv.d2 = ld3(g + 12);
  if (!W.crec) {
    ops3(W, W.cdir, 9 * (size_t)c, cv.n);
    ops3(W, W.cdir, 9 * (size_t)c + 3, cv.d1);
    ops3(W, W.cdir, 9 * (size_t)c + 6, cv.d2);
  }
  cv.ra = ra;
  cv.rb = rb;
  if (W.crec) {  // batched path: one vector-loadable record + block ids per contact
    R* rc = W.crec + 20 * c;
    st3(rc, cv.n);
    st3(rc + 3, cv.d1);
    st3(rc + 6, cv.d2);
    st3(rc + 9, ra);
    st3(rc + 12, rb);
    W.cblk[c] = make_int4(cv.al, cv.aa, cv.bl, cv.bA);
  }
  const int nr = W.normal_begin + c, f0 = W.friction_begin + 2 * c;
  // the gap decides the Fischer-Burmeister branch at the origin (ncp.cpp:24): computed
  // without contraction, as contact_gap (constraints.cpp:67-71) rounds on the CPU
  const R gap = contact_gap_strict(T, q, ba, bb, la, lb, cv.n, thick);
  const R lam_n = W.lam[nr] / h;
  const R rn = r_factor(contact_quad(T, W, cv, cv.n, false), h, true, cfg.r_strategy);
  const PhiV<R> phi = phi_n(gap, lam_n, rn, cfg.ncp_kind);
  const R hn = phi.v / h;
  W.hv[nr] = hn;
  W.cd[nr] = phi.dl / (h * h);
  if (W.crec)
    W.crec[20 * c + 15] = phi.dc;
  else
    W.cscale[2 * c] = phi.dc;  // row kept iff dc != 0 (newton.cpp:187)
  st.comp = fmax(st.comp, (double)ab(mn(gap, lam_n)));
  const R lf0 = W.lam[f0] / h, lf1 = W.lam[f0 + 1] / h;
  const R mu_ln = mu * lam_n;
  const R lfn = sqrt(lf0 * lf0 + lf1 * lf1);
  st.cone = fmax(st.cone, (double)mx(R(0), lfn - mu_ln));
  R h1, h2, wdec = R(-1);
  if (mu_ln > R(0)) {
    const V3<R> dv = contact_dv(cv, u);
    const R v0 = dot(cv.d1, dv), v1 = dot(cv.d2, dv);
    const R df = R(0.5) * (contact_quad(T, W, cv, cv.d1, false) + contact_quad(T, W, cv, cv.d2, false));
    const R rf = r_factor(df, h, false, cfg.r_strategy);
    const R wv = friction_W(sqrt(v0 * v0 + v1 * v1), lfn, mu_ln, rf, cfg.ncp_kind);
    wdec = wv;
    h1 = v0 + wv * lf0;
    h2 = v1 + wv * lf1;
    W.cd[f0] = W.cd[f0 + 1] = wv / h;
    if (W.crec)
      W.crec[20 * c + 16] = R(1);
    else
      W.cscale[2 * c + 1] = R(1);
  } else {
    h1 = lf0;
    h2 = lf1;
    W.cd[f0] = W.cd[f0 + 1] = R(1) / h;
    if (W.crec)
      W.crec[20 * c + 16] = R(0);
    else
      W.cscale[2 * c + 1] = R(0);
  }
  W.hv[f0] = h1;
  W.hv[f0 + 1] = h2;
  st.hmax = fmax(st.hmax, fmax((double)ab(hn), fmax((double)ab(h1), (double)ab(h2))));
  st.hsq += (double)hn * hn + (double)h1 * h1 + (double)h2 * h2;
  if (W.dec) {
    unsigned char f = 0;
    if (phi.dc != R(0)) f |= kDecNormalKept;
    if (mu_ln > R(0)) {
      f |= kDecFrictionOn;
      if (wdec == R(1e12)) f |= kDecWCap;
      if (cfg.ncp_kind == 0 && wdec == R(0)) f |= kDecWZero;  // FB's W has no stick branch
    }
    const R rl = rn * lam_n;
    if (cfg.ncp_kind == 1 ? (gap * gap + rl * rl == R(0)) : (gap <= rl)) f |= kDecNcpBranch;
    W.dec[c] = f;
  }
}

template <class R, bool kTets, class Team>
__device__ void assemble(Team& t, const Topo<R>& T, Work<R>& W, const R* q, const R* u, const Cfg& cfg, AsmStats& st) {
  const int nt = kTets ? T.nt : 0;
  const int ng = T.nj + nt + W.nc;
  for (int g = t.rank(); g < ng; g += t.size()) {
    if (g < T.nj)
      assemble_joint(T, W, q, g, W.h, st);
    else if (kTets && g < T.nj + nt)
      assemble_tet(T, W, q, g - T.nj, W.h, st);
    else
      assemble_contact(T, W, q, u, g - T.nj - nt, W.h, cfg, st);
  }
}

// ------------------------------------------------------------------ J^T pull for one dof3 block
// Row vector given by a plain array.
template <class R> struct RowArr {
  const R* y;
  __device__ __forceinline__ R operator()(int i) const { return y[i]; }
};
// Row vector z' = z - a * inv .* ap (a PCR update not yet committed in memory).
template <class R> struct RowPending {
  const R *z, *inv, *ap;
  R a;
  __device__ __forceinline__ R operator()(int i) const { return z[i] - a * (inv[i] * ap[i]); }
};
// z' = z - a M^-1 ap' with ap' = az + b ap_prev (az alone on the first iteration),
// formed by the pull from the previous iteration's vectors: bitwise the ap' the
// row's owner forms in the same pass (grid PCR with one barrier fewer).
template <class R> struct RowPendingAz {
  const R *z, *inv, *az, *ap_prev;
  R a, b;
  bool first;
  __device__ __forceinline__ R operator()(int i) const {
    const R ap = first ? az[i] : az[i] + b * ap_prev[i];
    return z[i] - a * (inv[i] * ap);
  }
};
// z = M^-1 r and z' = M^-1 (r - a ap) for a PCR that keeps z implicit (diagonal
// preconditioner).
template <class R> struct RowPrecond {
  const R *r, *inv;
  __device__ __forceinline__ R operator()(int i) const { return inv[i] * r[i]; }
};
template <class R> struct RowPrecondResidual {
  const R *r, *inv, *ap;
  R a;
  __device__ __forceinline__ R operator()(int i) const { return inv[i] * (r[i] - a * ap[i]); }
};

// Partial J^T y of block b over the incidence entries first, first+stride, ...
template <class R, class YF>
__device__ __forceinline__ V3<R> pull_part(const Topo<R>& T, const Work<R>& W, int b, const YF& y, int first,
                                           int stride) {
  R sx = R(0), sy = R(0), sz = R(0);
  const int s0 = T.sinc_off[b], s1 = T.sinc_off[b + 1];
  for (int e = s0 + first; e < s1; e += stride) {
    const int ent = T.sinc_ent[e];
    const int row = ent >> 2, slot = ent & 3;
    const R yr = y(row);
    const V3<R> c = opg3(W, W.coeff, 12 * (size_t)row + 3 * slot);
    sx += c.x * yr;
    sy += c.y * yr;
    sz += c.z * yr;
  }
  if (W.nc > 0) {
    const int c0 = W.cinc_off[b], c1 = W.cinc_off[b + 1];
    for (int e = c0 + first; e < c1; e += stride) {
      const int ent = W.cinc_ent[e];
      const int c = ent >> 2, slot = ent & 3;
      const V3<R> gn = opg3(W, W.cdir, 9 * (size_t)c), g1 = opg3(W, W.cdir, 9 * (size_t)c + 3),
                  g2 = opg3(W, W.cdir, 9 * (size_t)c + 6);
      const R dc = W.cscale[2 * c], act = W.cscale[2 * c + 1];
      const int f0 = W.friction_begin + 2 * c;
      const R yn = dc * y(W.normal_begin + c), y1 = act * y(f0), y2 = act * y(f0 + 1);
      // contact force f = dc z_n n + z_1 d1 + z_2 d2
      V3<R> f = v3(yn * gn.x + y1 * g1.x + y2 * g2.x, yn * gn.y + y1 * g1.y + y2 * g2.y,
                   yn * gn.z + y1 * g1.z + y2 * g2.z);
      if (slot & 1) f = cross(opg3(W, W.carm, 6 * (size_t)c + ((slot & 2) ? 3 : 0)), f);
      if (slot & 2) f = -f;
      sx += f.x;
      sy += f.y;
      sz += f.z;
    }
  }
  return v3(sx, sy, sz);
}

template <class R, class YF>
__device__ __forceinline__ V3<R> pull(const Topo<R>& T, const Work<R>& W, int b, const YF& y) {
  return pull_part(T, W, b, y, 0, 1);
}
// Warp-cooperative pull: the 32 lanes stride the block's incidence list and
// combine in a fixed shuffle tree (deterministic); every lane gets the sum.
template <class R, class YF>
__device__ __forceinline__ V3<R> pull_warp(const Topo<R>& T, const Work<R>& W, int b, const YF& y, int lane) {
  V3<R> s = pull_part(T, W, b, y, lane, 32);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    s.x += __shfl_down_sync(0xffffffffu, s.x, off);
    s.y += __shfl_down_sync(0xffffffffu, s.y, off);
    s.z += __shfl_down_sync(0xffffffffu, s.z, off);
  }
  return v3(__shfl_sync(0xffffffffu, s.x, 0), __shfl_sync(0xffffffffu, s.y, 0), __shfl_sync(0xffffffffu, s.z, 0));
}

template <class R>
__device__ __forceinline__ V3<R> hinv_apply(const Topo<R>& T, const Work<R>& W, int b, V3<R> v) {
  if (T.d3_kind[b] == kRigidAng) return sym_mul(W.iwi6 + 6 * b, v);
  const R* hi = W.hinv + 3 * b;
  return v3(v.x * hi[0], v.y * hi[1], v.z * hi[2]);
}

// Operator pass 1: w = H^-1 J^T y (dof-parallel).
// Visits every dof3 block with its pulled J^T y: f(b, sum). Warp-cooperative
// (team size a multiple of 32) for long incidence lists, one thread per block
// otherwise; in both cases f runs once per block.
template <class R, class Team, class YF, class F>
__device__ __forceinline__ void for_blocks(Team& t, const Topo<R>& T, const Work<R>& W, const YF& y, F&& f) {
  if (T.warp_pull) {
    const int lane = t.rank() & 31, wid = t.rank() >> 5, nw = t.size() >> 5;
    for (int b = wid; b < T.nd3; b += nw) {
      const V3<R> s = pull_warp(T, W, b, y, lane);
      if (lane == 0) f(b, s);
    }
  } else {
    for (int b = t.rank(); b < T.nd3; b += t.size()) f(b, pull(T, W, b, y));
  }
}

// Team size is a multiple of 32 for the generic engine: one warp per block.
template <class R, class Team, class YF> __device__ void op_pull(Team& t, const Topo<R>& T, Work<R>& W, const YF& y) {
  for_blocks(t, T, W, y, [&](int b, V3<R> s) { st3(W.w + 3 * b, hinv_apply(T, W, b, s)); });
}

// C_i . z for row i (tet block rows or scalar rows).
template <class R, bool kTets>
__device__ __forceinline__ R row_C(const Topo<R>& T, const Work<R>& W, int i, const R* z) {
  if (kTets && i >= T.rows_joint && i < T.rows_static) {
    const int td = T.tdim, e = (i - T.rows_joint) / td, k = (i - T.rows_joint) - td * e;
    const size_t cb = (size_t)td * td * e + td * k;
    const int r0 = T.rows_joint + td * e;
    if (td == 3) return opg(W, W.ctet, cb) * z[r0] + opg(W, W.ctet, cb + 1) * z[r0 + 1] + opg(W, W.ctet, cb + 2) * z[r0 + 2];
    R acc = R(0);
    for (int j = 0; j < 6; ++j) acc += opg(W, W.ctet, cb + j) * z[r0 + j];
    return acc;
  }
  return W.cd[i] * z[i];
}
template <class R, bool kTets> __device__ __forceinline__ R row_Cdiag(const Topo<R>& T, const Work<R>& W, int i) {
  if (kTets && i >= T.rows_joint && i < T.rows_static) {
    const int td = T.tdim, e = (i - T.rows_joint) / td, k = (i - T.rows_joint) - td * e;
    return opg(W, W.ctet, (size_t)td * td * e + (td + 1) * k);
  }
  return W.cd[i];
}

}  // namespace nsd
#include "nsd_part.cuh"
namespace nsd {

// ------------------------------------------------------------------ Newton step
// Step setup (newton.cpp:327-338): q = q-, M~ at q- (world inertia and its
// inverse per rigid body), f_ext = gravity + gyroscopic (+ extension force),
// u~ = u- + h M~^-1 f_ext, zero starting iterate. Needs a team barrier after.
template <class R, class Team> __device__ void newton_setup(Team& t, const Topo<R>& T, Work<R>& W) {
  const R h = W.h;
  for (int b = t.rank(); b < T.nb; b += t.size()) {
    const int d = T.bdof[b], cd = T.bcoord[b];
    const R m = T.bmass[b];
    V3<R> f = v3(m * W.grav[0], m * W.grav[1], m * W.grav[2]);
    for (int k = 0; k < (T.btype[b] ? 7 : 3); ++k) W.q[cd + k] = W.q0[cd + k];
    if (W.f_extra) f = f + ld3(W.f_extra + d);
    st3(W.ut + d, ld3(W.u0 + d) + h * (f / m));
    for (int k = 0; k < (T.btype[b] ? 6 : 3); ++k) {
      W.u[d + k] = R(0);
      W.shift[d + k] = R(0);
      W.hinv[d + k] = R(0);
    }
    if (T.btype[b] == 1) {
      const M3<R> Rm = quat_rot(W.q0[cd + 3], W.q0[cd + 4], W.q0[cd + 5], W.q0[cd + 6]);
      M3<R> I;
#pragma unroll
      for (int i = 0; i < 9; ++i) I.a[i] = T.binertia[9 * b + i];
      const M3<R> Iw = mul(mul(Rm, I), transpose(Rm));
      const M3<R> Ii = inverse3(Iw);
      const int ab3 = d / 3 + 1;
      R* s6 = W.iw6 + 6 * ab3;
      s6[0] = Iw(0, 0);
      s6[1] = Iw(1, 1);
      s6[2] = Iw(2, 2);
      s6[3] = Iw(0, 1);
      s6[4] = Iw(0, 2);
      s6[5] = Iw(1, 2);
      R* i6 = W.iwi6 + 6 * ab3;
      i6[0] = Ii(0, 0);
      i6[1] = Ii(1, 1);
      i6[2] = Ii(2, 2);
      i6[3] = Ii(0, 1);
      i6[4] = Ii(0, 2);
      i6[5] = Ii(1, 2);
      const V3<R> w = ld3(W.u0 + d + 3);
      V3<R> tq = -cross(w, mul(Iw, w));
      if (W.f_extra) tq = tq + ld3(W.f_extra + d + 3);
      st3(W.ut + d + 3, w + h * mul(Ii, tq));
    }
  }
}

// Integration q = q- + h G(q) u with G at the current iterate (bodies.cpp:58-86).
template <class R> __device__ __forceinline__ void integrate_body(const Topo<R>& T, const R* q0, R* qdst,
                                                                 const R* qcur, const R* u, int b, R h) {
  const int cd = T.bcoord[b], d = T.bdof[b];
  for (int k = 0; k < 3; ++k) qdst[cd + k] = q0[cd + k] + h * u[d + k];
  if (T.btype[b] == 1) {
    const R* th = qcur + cd + 3;
    const R t0 = th[0], t1 = th[1], t2 = th[2], t3 = th[3];
    const R ox = u[d + 3], oy = u[d + 4], oz = u[d + 5];
    R nq[4];
    nq[0] = q0[cd + 3] + h * (R(0.5) * (-t1 * ox - t2 * oy - t3 * oz));
    nq[1] = q0[cd + 4] + h * (R(0.5) * (t0 * ox + t3 * oy - t2 * oz));
    nq[2] = q0[cd + 5] + h * (R(0.5) * (-t3 * ox + t0 * oy + t1 * oz));
    nq[3] = q0[cd + 6] + h * (R(0.5) * (t2 * ox - t1 * oy + t0 * oz));
    const R nn = sqrt(nq[0] * nq[0] + nq[1] * nq[1] + nq[2] * nq[2] + nq[3] * nq[3]);
    if ((double)nn < 1e-300) {
      nq[0] = R(1);
      nq[1] = nq[2] = nq[3] = R(0);
    } else {
      for (int k = 0; k < 4; ++k) nq[k] = nq[k] / nn;
    }
    for (int k = 0; k < 4; ++k) qdst[cd + 3 + k] = nq[k];
  }
}

// The Newton loop, final classification and telemetry (newton.cpp:343-416).
// Requires newton_setup() and a barrier, and the step's contact set + incidence.
template <class R, bool kTets, class Team, int RPT = 0>
__device__ int newton_solve(Team& t, const Topo<R>& T, Work<R>& W, const Cfg& cfg, StepOut out) {
  const R h = W.h;
  const int nr = W.nrows;
  const int maxlin = cfg.linear_max_iterations;
  const R eps = R(cfg.epsilon_reg);
  const R tfrac = R(cfg.step_fraction);
  for (int i = t.rank(); i < nr; i += t.size()) W.lam[i] = R(0);
  setup_row_blocks<R, kTets>(t, T, W);
  double has_fric = 0.0;  // line-search gate (newton.cpp:341)
  for (int c = t.rank(); c < W.nc; c += t.size())
    if (W.cgeo[17 * c + 16] > R(0)) has_fric = 1.0;
  if (cfg.line_search) {
    double s0[1] = {0.0}, m0[1] = {has_fric};
    t.reduce(s0, m0);
    has_fric = m0[0];
  } else {
    t.sync();
  }
  const bool line_search = cfg.line_search && has_fric == 0.0;
  // partitioned PCR (RPT < 0, grid kernel): per-step tables in dynamic shared memory
  extern __shared__ __align__(16) char nsd_dyn_smem[];
  PartView<R> PV(nsd_dyn_smem, W, RPT < 0);
  if constexpr (RPT < 0) part_setup<R, kTets>(T, W, PV);
  double min_shift = 0.0;
  int n_done = 0;
  int aborted = 0;

  const int dec_dof = W.nc + (kTets ? T.nt : 0), dec_exit = dec_dof + T.ndof;
  for (int it = 0; it < cfg.newton_iterations; ++it) {
    W.dec = out.dec ? out.dec + (size_t)it * out.dec_stride : nullptr;
    // ---- assemble
    AsmStats as{0.0, 0.0, 0.0, 0.0};
    assemble<R, kTets>(t, T, W, W.q, W.u, cfg, as);
    t.sync();
    // ---- g = M~(u - u~) - J^T lambda; geometric stiffness; H^-1; w = H^-1 g
    double gmax = 0.0, gsq = 0.0, smin = 0.0;
    const bool gs = it >= 1 && cfg.geometric_stiffness;
    for_blocks(t, T, W, RowArr<R>{W.lam}, [&](int b, V3<R> jl) {
      const int kind = T.d3_kind[b];
      const int d = 3 * b;
      V3<R> gv, mdiag;
      const V3<R> du = ld3(W.u + d) - ld3(W.ut + d);
      if (kind == kRigidAng) {
        const R* s6 = W.iw6 + 6 * b;
        gv = sym_mul(s6, du) - jl;
        mdiag = v3(s6[0], s6[1], s6[2]);
      } else {
        const R m = T.bmass[T.d3_body[b]];
        gv = v3(m * du.x, m * du.y, m * du.z) - jl;
        mdiag = v3(m, m, m);
      }
      if (kind == kParticleLin) {
        // geometric stiffness secant (newton.cpp:299-319); rigid dofs keep shift 0
        const R m = mdiag.x;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          unsigned char df = 0;
          if (gs) {
            const R dd = W.u[d + k] - W.up[d + k];
            R sh = R(0);
            if (!(ab(dd) < R(1e-10))) {
              const R ck = -((gv[k] - W.gp[d + k] + m * dd) / dd);
              sh = -mn(R(0), ck);
              if (!(ck < R(0))) df = kDecGsClamp;
            } else {
              df = kDecGsSkip;
            }
            W.shift[d + k] = sh;
            smin = fmin(smin, (double)sh);
          }
          if (W.dec) W.dec[dec_dof + d + k] = df;
          W.gp[d + k] = gv[k];
          W.up[d + k] = W.u[d + k];
        }
      } else if (W.dec) {
#pragma unroll
        for (int k = 0; k < 3; ++k) W.dec[dec_dof + d + k] = gs ? kDecRigidDof : 0;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        W.g[d + k] = gv[k];
        gmax = fmax(gmax, (double)(ab(gv[k]) / mdiag[k]));
        gsq += (double)gv[k] * (double)gv[k];
      }
      if (kind != kRigidAng) {
        const R m = mdiag.x;
#pragma unroll
        for (int k = 0; k < 3; ++k) W.hinv[d + k] = R(1) / (m + W.shift[d + k]);
      }
      st3(W.w + d, hinv_apply(T, W, b, gv));
    });
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

    // ---- Schur RHS b = J H^-1 g - h, diagonal preconditioner, r = b (x0 = 0)
    double rr = 0.0, rzr = 0.0;
    for (int i = t.rank(); i < nr; i += t.size()) {
      const R b = row_J(T, W, i, W.w) - W.hv[i];
      R inv = R(1);
      if (cfg.preconditioner == 1 || cfg.linear_method == 0 || cfg.linear_method == 1) {  // Jacobi / GS use the diagonal
        const R sd = row_quad(T, W, i) + row_Cdiag<R, kTets>(T, W, i) + eps;
        inv = sd > R(0) ? R(1) / sd : R(1);
      }
      W.inv[i] = inv;
      W.r[i] = b;
      W.x[i] = R(0);
      W.bx[i] = R(0);
      W.z[i] = inv * b;
      rr += (double)b * b;
      rzr += (double)b * (double)(inv * b);
    }
    int lin_used = 0, breakdown = 0, hist_n = 0, mono = 0;
    double hist_last = 0.0;
    if (nr > 0) {
      double s1[2] = {rr, rzr};
      t.reduce_sum(s1);
      hist_last = sqrt(s1[0]);
      double phist_last = sqrt(s1[1]);
      double best_res = hist_last;
      hist_n = 1;
      if (t.rank() == 0 && out.hist) out.hist[(size_t)it * (maxlin + 1)] = hist_last;
      // kTets == false (diagonal C): the accepted update x+=a p, r-=a ap, z-=a M^-1 ap
      // is committed in place during the next row pass (the operator reads the
      // pending z' on the fly), so no trial buffers xn/rn/zn are needed.
      if (cfg.linear_method == 1) {
        // Gauss-Seidel (solvers.cpp:52-81): forward sweeps in ascending row order, one
        // thread, on the matrix-free operator. (S x)_row = J_row w + (C x)_row + eps x_row
        // with w = H^-1 J^T x kept current: each row's change d adds H^-1 J_row^T d to the
        // <= 4 dof3 blocks the row touches. x0 = 0, so w starts at 0. The diagonal
        // S_rr = J_row H^-1 J_row^T + C_rr + eps is the preconditioner's (1 / inv).
        // After each sweep r = b - S x is re-evaluated in parallel for the history.
        R *x = W.x, *bb = W.zn;
        for (int i = t.rank(); i < nr; i += t.size()) {
          bb[i] = W.r[i];
          x[i] = R(0);
        }
        for (int b = t.rank(); b < T.nd3; b += t.size()) st3(W.w + 3 * b, v3(R(0), R(0), R(0)));
        t.sync();
        for (int itl = 0; itl < maxlin && hist_last > cfg.linear_tolerance; ++itl) {
          if (t.rank() == 0) {
            for (int i = 0; i < nr; ++i) {
              const R diag = row_quad(T, W, i) + row_Cdiag<R, kTets>(T, W, i) + eps;  // S_ii
              if (!(fabs((double)diag) > 1e-300)) continue;  // solvers.cpp:73
              const R sx = row_J(T, W, i, W.w) + row_C<R, kTets>(T, W, i, x) + eps * x[i];
              const R xn = (bb[i] - (sx - diag * x[i])) / diag;
              const R d = xn - x[i];
              x[i] = xn;
              row_JT(T, W, i, d, [&](int b, V3<R> v) {
                const V3<R> hv = hinv_apply(T, W, b, v);
                R* wb = W.w + 3 * b;
                wb[0] += hv.x;
                wb[1] += hv.y;
                wb[2] += hv.z;
              });
            }
          }
          t.sync();
          op_pull(t, T, W, RowArr<R>{x});  // w = H^-1 J^T x afresh for the residual
          t.sync();
          double rr2 = 0.0;
          for (int i = t.rank(); i < nr; i += t.size()) {
            const R ri = bb[i] - (row_J(T, W, i, W.w) + row_C<R, kTets>(T, W, i, x) + eps * x[i]);
            W.r[i] = ri;
            rr2 += (double)ri * ri;
          }
          double s[1] = {rr2};
          t.reduce_sum(s);
          hist_last = sqrt(s[0]);
          if (t.rank() == 0 && out.hist && hist_n <= maxlin) out.hist[(size_t)it * (maxlin + 1) + hist_n] = hist_last;
          ++hist_n;
          lin_used = itl + 1;
          if (hist_last < best_res) {
            best_res = hist_last;
            for (int i = t.rank(); i < nr; i += t.size()) W.bx[i] = x[i];
          }
          t.sync();
        }
      } else if (cfg.linear_method == 0 || cfg.linear_method == 2) {
        // Jacobi (solvers.cpp:32-50) and PCG (solvers.cpp:83-121) on the same
        // matrix-free operator S v = J H^-1 J^T v + C v + eps v, x0 = 0, best iterate
        // by residual 2-norm, breakdown tests at 1e-300 in double.
        R *x = W.x, *r = W.r, *z = W.z, *p = W.p, *bb = W.zn;
        const bool jac = cfg.linear_method == 0;
        bool pending_best = false;
        for (int i = t.rank(); i < nr; i += t.size()) {
          bb[i] = r[i];
          p[i] = z[i];
        }
        double rz = s1[1];  // r . M^-1 r of the setup reduction (PCG)
        for (int itl = 0; itl < maxlin && hist_last > cfg.linear_tolerance; ++itl) {
          double rr2 = 0.0, rzn = 0.0;
          if (jac) {
            for (int i = t.rank(); i < nr; i += t.size()) {  // x += D^-1 r
              if (pending_best) W.bx[i] = x[i];
              x[i] = x[i] + W.inv[i] * r[i];
            }
            pending_best = false;
            t.sync();
            op_pull(t, T, W, RowArr<R>{x});
            t.sync();
            for (int i = t.rank(); i < nr; i += t.size()) {  // r = b - S x
              const R ri = bb[i] - (row_J(T, W, i, W.w) + row_C<R, kTets>(T, W, i, x) + eps * x[i]);
              r[i] = ri;
              rr2 += (double)ri * ri;
            }
            double s[1] = {rr2};
            t.reduce_sum(s);
            rr2 = s[0];
          } else {
            t.sync();
            op_pull(t, T, W, RowArr<R>{p});
            t.sync();
            double pap = 0.0;
            for (int i = t.rank(); i < nr; i += t.size()) {  // ap = S p
              const R a = row_J(T, W, i, W.w) + row_C<R, kTets>(T, W, i, p) + eps * p[i];
              W.ap[i] = a;
              pap += (double)p[i] * a;
            }
            {
              double s[1] = {pap};
              t.reduce_sum(s);
              pap = s[0];
            }
            if (fabs(pap) < 1e-300) {
              breakdown = 1;
              break;
            }
            const R ra = R(rz / pap);
            for (int i = t.rank(); i < nr; i += t.size()) {
              if (pending_best) W.bx[i] = x[i];
              x[i] = x[i] + ra * p[i];
              const R ri = r[i] - ra * W.ap[i];
              r[i] = ri;
              const R zi = cfg.preconditioner == 1 ? W.inv[i] * ri : ri;
              z[i] = zi;
              rr2 += (double)ri * ri;
              rzn += (double)ri * zi;
            }
            pending_best = false;
            double s[2] = {rr2, rzn};
            t.reduce_sum(s);
            rr2 = s[0];
            rzn = s[1];
          }
          hist_last = sqrt(rr2);
          if (t.rank() == 0 && out.hist && hist_n <= maxlin) out.hist[(size_t)it * (maxlin + 1) + hist_n] = hist_last;
          ++hist_n;
          if (hist_last < best_res) {
            best_res = hist_last;
            pending_best = true;
          }
          lin_used = itl + 1;
          if (!jac) {
            if (fabs(rz) < 1e-300) {
              breakdown = 1;
              break;
            }
            const R rb = R(rzn / rz);
            rz = rzn;
            for (int i = t.rank(); i < nr; i += t.size()) {
              if (pending_best) W.bx[i] = x[i];
              p[i] = z[i] + rb * p[i];
            }
            pending_best = false;
          }
        }
        if (pending_best)
          for (int i = t.rank(); i < nr; i += t.size()) W.bx[i] = x[i];
      } else if constexpr (RPT < 0) {
        // Partitioned PCR (nsd_part.cuh): the same recurrence, exits and reductions as
        // the register path below (den expanded from the previous J w pass's sums),
        // with every CTA's rows, coefficients and local dof3 blocks in shared memory
        // and only the shared blocks' J^T partials exchanged through global memory.
        part_load<R, kTets>(T, W, PV);
#ifdef NSD_PROFILE_GRID  // NSD_PHASE_TIMING diagnostics (a -DNSD_PROFILE_GRID build; they cost registers)
        PhaseClock pcl(out.ptime, blockIdx.x == 0 && threadIdx.x == 0);
        // per CTA: [compute, reduction incl. waiting] cycles (load-balance diagnostics)
        PhaseClock pcb(out.ptime ? out.ptime + 16 + 2 * blockIdx.x : nullptr, threadIdx.x == 0);
#else
        NoClock pcl, pcb;
#endif
        const int td = kTets ? T.tdim : 0;
        const int tid = threadIdx.x, ntd = blockDim.x;
        R *xs = PV.x, *rs = PV.r, *zs = PV.z, *zns = PV.zn, *xns = PV.xn, *rns = PV.rn;
        double zaz = 0.0, den_next = 0.0;
        if (maxlin > 0 && hist_last > cfg.linear_tolerance) {
          part_scatter(W, PV, zs);
          t.sync();
          part_gather(W, PV, tid, ntd);
          __syncthreads();
          double za = 0.0, aa = 0.0;
          for (int li = tid; li < PV.nrow; li += ntd) {
            const R a = part_row(PV, li, zs, td, eps);
            PV.az[li] = a;
            za += (double)zs[li] * a;
            aa += (double)a * (double)(PV.inv[li] * a);
          }
          double s[2] = {za, aa};
          t.reduce_sum(s);
          zaz = s[0];
          den_next = s[1];  // ap' = az on the first iteration
        }
        double beta = 0.0;
        for (int itl = 0; itl < maxlin && hist_last > cfg.linear_tolerance; ++itl) {
          const double den = den_next;
          if (fabs(den) < 1e-300) {
            breakdown = 1;
            break;
          }
          const double alpha = zaz / den;
          const R ra = R(alpha), rb = R(beta);
          double pn2 = 0.0, rn2 = 0.0;
          for (int li = tid; li < PV.nrow; li += ntd) {
            R pv, apv;
            if (itl == 0) {
              pv = zs[li];
              apv = PV.az[li];
            } else {
              pv = zs[li] + rb * PV.p[li];
              apv = PV.az[li] + rb * PV.ap[li];
            }
            PV.p[li] = pv;
            PV.ap[li] = apv;
            const R rv = rs[li] - ra * apv;
            xns[li] = xs[li] + ra * pv;
            rns[li] = rv;
            zns[li] = zs[li] - ra * (PV.inv[li] * apv);
            pn2 += (double)rv * (double)(PV.inv[li] * rv);
            rn2 += (double)rv * rv;
          }
          pcl.mark(0);
          const bool pull = fabs(zaz) >= 1e-300;  // w = H^-1 J^T z'
          if (pull) {
            __syncthreads();
            part_scatter(W, PV, zns);
          }
          pcl.mark(1);
          pcb.mark(0);
          {
            double s[2] = {pn2, rn2};
            t.reduce_sum_side(s, [&](int first, int n) {
              if (pull) part_gather(W, PV, first, n);
            });
            pn2 = s[0];
            rn2 = s[1];
          }
          pcl.mark(2);
          pcb.mark(1);
          const double pn = sqrt(pn2);
          if (pn > phist_last) {  // monotone guard
            mono = 1;
            break;
          }
          R* tmp = xs;  // commit
          xs = xns;
          xns = tmp;
          tmp = rs;
          rs = rns;
          rns = tmp;
          tmp = zs;
          zs = zns;
          zns = tmp;
          hist_last = sqrt(rn2);
          phist_last = pn;
          if (t.rank() == 0 && out.hist && hist_n <= maxlin) out.hist[(size_t)it * (maxlin + 1) + hist_n] = hist_last;
          ++hist_n;
          if (hist_last < best_res) {
            best_res = hist_last;
            for (int li = tid; li < PV.nrow; li += ntd) PV.bx[li] = xs[li];
          }
          lin_used = itl + 1;
          if (fabs(zaz) < 1e-300) {
            breakdown = 1;
            break;
          }
          double za = 0.0, aa = 0.0, ab = 0.0, bb = 0.0;
          for (int li = tid; li < PV.nrow; li += ntd) {
            const R a = part_row(PV, li, zs, td, eps);
            PV.az[li] = a;
            za += (double)zs[li] * a;
            const double ia = (double)(PV.inv[li] * a);
            aa += (double)a * ia;
            const R apv = PV.ap[li];
            ab += (double)apv * ia;
            bb += (double)apv * (double)(PV.inv[li] * apv);
          }
          {
            pcl.mark(3);
            pcb.mark(0);
            double s[4] = {za, aa, ab, bb};
            t.reduce_sum(s);
            beta = s[0] / zaz;
            zaz = s[0];
            den_next = s[1] + 2.0 * beta * s[2] + beta * beta * s[3];
          }
          pcl.mark(4);
          pcb.mark(1);
        }
        for (int li = tid; li < PV.nrow; li += ntd) W.bx[PV.gid[li]] = PV.bx[li];
      } else if constexpr (RPT > 0) {
        // Register-resident PCR (grid kernel, nr <= RPT * team size): each thread's
        // own rows keep x, r, z, p, ap, az, inv, bx in registers across all phases.
        // Global memory carries only what other threads read: ap (the J^T pull's
        // z' = z - a M^-1 ap) and the committed z (pull base, tet-block C z). Same
        // recurrence, same arithmetic, same reductions as the memory path below;
        // each grid barrier's acquire invalidates L1, so this saves the post-barrier
        // L2 round trips of the row phases.
        R zr[RPT], pr[RPT], apr[RPT], azr[RPT], xr[RPT], rr_[RPT], invr[RPT], bxr[RPT], xnr[RPT], rnr[RPT], znr[RPT];
        const int rk = t.rank(), ts = t.size();
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const int i = rk + k * ts;
          const bool v = i < nr;
          zr[k] = v ? W.z[i] : R(0);
          rr_[k] = v ? W.r[i] : R(0);
          invr[k] = v ? W.inv[i] : R(0);
          xr[k] = bxr[k] = pr[k] = apr[k] = azr[k] = xnr[k] = rnr[k] = znr[k] = R(0);
        }
        // Two grid barriers per CR iteration: den = ap'.M^-1 ap' of this iteration's
        // ap' = az + beta ap is expanded as az.M^-1 az + 2 beta az.M^-1 ap + beta^2
        // ap.M^-1 ap from sums reduced with z.az in the previous J w pass, so the
        // p/ap update, the trial norms and the speculative pull share one pass (the
        // reference forms ap' first, solvers.cpp PCR: den differs by rounding only).
        // The pull forms ap' of other rows itself from az and the previous ap
        // (RowPendingAz), so ap is double-buffered (W.ap / W.rn, unused on this path).
        R *zg = W.z, *zng = W.zn, *apg = W.ap, *apo = W.rn;
        bool pending = false;
        double zaz = 0.0, den_next = 0.0;
        if (maxlin > 0 && hist_last > cfg.linear_tolerance) {
          op_pull(t, T, W, RowArr<R>{zg});
          t.sync();
          double za = 0.0, aa = 0.0;
#pragma unroll
          for (int k = 0; k < RPT; ++k) {
            const int i = rk + k * ts;
            if (i < nr) {
              const R a = row_J(T, W, i, W.w) + row_C<R, kTets>(T, W, i, zg) + eps * zr[k];
              azr[k] = a;
              W.az[i] = a;
              za += (double)zr[k] * a;
              aa += (double)a * (double)(invr[k] * a);
            }
          }
          double s[2] = {za, aa};
          t.reduce_sum(s);
          zaz = s[0];
          den_next = s[1];  // ap' = az on the first iteration
        }
        double beta = 0.0;
        for (int itl = 0; itl < maxlin && hist_last > cfg.linear_tolerance; ++itl) {
          const double den = den_next;
          if (fabs(den) < 1e-300) {
            breakdown = 1;
            break;
          }
          const double alpha = zaz / den;
          const R ra = R(alpha), rb = R(beta);
          double pn2 = 0.0, rn2 = 0.0;
#pragma unroll
          for (int k = 0; k < RPT; ++k) {
            const int i = rk + k * ts;
            if (i < nr) {
              if (itl == 0) {
                pr[k] = zr[k];
                apr[k] = azr[k];
              } else {
                pr[k] = zr[k] + rb * pr[k];
                apr[k] = azr[k] + rb * apr[k];
              }
              apg[i] = apr[k];
              const R rv = rr_[k] - ra * apr[k];
              xnr[k] = xr[k] + ra * pr[k];
              rnr[k] = rv;
              znr[k] = zr[k] - ra * (invr[k] * apr[k]);
              zng[i] = znr[k];
              pn2 += (double)rv * (double)(invr[k] * rv);
              rn2 += (double)rv * rv;
            }
          }
          if (fabs(zaz) >= 1e-300)  // w = H^-1 J^T z'
            op_pull(t, T, W, RowPendingAz<R>{zg, W.inv, W.az, apo, ra, rb, itl == 0});
          {
            double s[2] = {pn2, rn2};
            t.reduce_sum(s);
            pn2 = s[0];
            rn2 = s[1];
          }
          const double pn = sqrt(pn2);
          if (pn > phist_last) {  // monotone guard
            mono = 1;
            break;
          }
#pragma unroll
          for (int k = 0; k < RPT; ++k) {  // commit
            xr[k] = xnr[k];
            rr_[k] = rnr[k];
            zr[k] = znr[k];
          }
          R* tmp = zg;
          zg = zng;
          zng = tmp;
          hist_last = sqrt(rn2);
          phist_last = pn;
          if (t.rank() == 0 && out.hist && hist_n <= maxlin) out.hist[(size_t)it * (maxlin + 1) + hist_n] = hist_last;
          ++hist_n;
          if (hist_last < best_res) {
            best_res = hist_last;
#pragma unroll
            for (int k = 0; k < RPT; ++k) bxr[k] = xr[k];
          }
          lin_used = itl + 1;
          if (fabs(zaz) < 1e-300) {
            breakdown = 1;
            break;
          }
          double za = 0.0, aa = 0.0, ab = 0.0, bb = 0.0;
#pragma unroll
          for (int k = 0; k < RPT; ++k) {
            const int i = rk + k * ts;
            if (i < nr) {
              const R a = row_J(T, W, i, W.w) + row_C<R, kTets>(T, W, i, zg) + eps * zr[k];
              azr[k] = a;
              W.az[i] = a;
              za += (double)zr[k] * a;
              const double ia = (double)(invr[k] * a);
              aa += (double)a * ia;
              ab += (double)apr[k] * ia;
              bb += (double)apr[k] * (double)(invr[k] * apr[k]);
            }
          }
          {
            double s[4] = {za, aa, ab, bb};
            t.reduce_sum(s);
            beta = s[0] / zaz;
            zaz = s[0];
            den_next = s[1] + 2.0 * beta * s[2] + beta * beta * s[3];
          }
          R* tap = apg;  // this iteration's ap is the next pull's ap_prev
          apg = apo;
          apo = tap;
        }
        (void)pending;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const int i = rk + k * ts;
          if (i < nr) W.bx[i] = bxr[k];
        }
        W.z = zg;
        W.zn = zng;
      } else {
      constexpr bool kInPlace = !kTets;
      bool pending_best = false;
      R pend = R(0);  // alpha of an accepted, not yet committed update (kInPlace)
      R *x = W.x, *xn = W.xn, *r = W.r, *rn = W.rn, *z = W.z, *zn = W.zn;
      double zaz = 0.0;
      if (maxlin > 0 && hist_last > cfg.linear_tolerance) {
        op_pull(t, T, W, RowArr<R>{z});  // az = A z, zaz = z . az
        t.sync();
        double za = 0.0;
        for (int i = t.rank(); i < nr; i += t.size()) {
          const R a = row_J(T, W, i, W.w) + row_C<R, kTets>(T, W, i, z) + eps * z[i];
          W.az[i] = a;
          za += (double)z[i] * a;
        }
        double s[1] = {za};
        t.reduce_sum(s);
        zaz = s[0];
      }
      double beta = 0.0;
      for (int itl = 0; itl < maxlin && hist_last > cfg.linear_tolerance; ++itl) {
        // phase A: p = z + beta p, ap = az + beta ap; den = ap . M^-1 ap
        double den = 0.0;
        const R rb = R(beta);
        for (int i = t.rank(); i < nr; i += t.size()) {
          R pi, api;
          if (itl == 0) {
            pi = z[i];
            api = W.az[i];
          } else {
            pi = z[i] + rb * W.p[i];
            api = W.az[i] + rb * W.ap[i];
          }
          W.p[i] = pi;
          W.ap[i] = api;
          den += (double)api * (double)(W.inv[i] * api);
        }
        {
          double s[1] = {den};
          t.reduce_sum(s);
          den = s[0];
        }
        if (fabs(den) < 1e-300) {
          breakdown = 1;
          break;
        }
        const double alpha = zaz / den;
        const R ra = R(alpha);
        // phase B: x' = x + a p, r' = r - a ap, z' = z - a M^-1 ap, trial norms; in the
        // same pass (it needs only alpha) the J^T pull of z' for the next operator
        // application, speculatively: the reduction's barrier then also orders the
        // pull before the row pass, one grid barrier fewer per iteration. A rejected
        // trial (monotone guard) discards it.
        double pn2 = 0.0, rn2 = 0.0;
        for (int i = t.rank(); i < nr; i += t.size()) {
          const R api = W.ap[i];
          const R rv = r[i] - ra * api;
          if (!kInPlace) {
            xn[i] = x[i] + ra * W.p[i];
            rn[i] = rv;
            zn[i] = z[i] - ra * (W.inv[i] * api);
          }
          pn2 += (double)rv * (double)(W.inv[i] * rv);
          rn2 += (double)rv * rv;
        }
        if (fabs(zaz) >= 1e-300) op_pull(t, T, W, RowPending<R>{z, W.inv, W.ap, ra});  // w = H^-1 J^T z'
        {
          double s[2] = {pn2, rn2};
          t.reduce_sum(s);
          pn2 = s[0];
          rn2 = s[1];
        }
        const double pn = sqrt(pn2);
        if (pn > phist_last) {  // monotone guard: stop at the numerical floor
          mono = 1;
          break;
        }
        if (kInPlace) {
          pend = ra;  // commit deferred to the next row pass
        } else {
          R* tmp = x;  // commit
          x = xn;
          xn = tmp;
          tmp = r;
          r = rn;
          rn = tmp;
          tmp = z;
          z = zn;
          zn = tmp;
        }
        hist_last = sqrt(rn2);
        phist_last = pn;
        if (t.rank() == 0 && out.hist && hist_n <= maxlin) out.hist[(size_t)it * (maxlin + 1) + hist_n] = hist_last;
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
        double za = 0.0;
        if (kInPlace) {  // w = H^-1 J^T z' is already pulled (phase B); az = A z', zaz' = z' . az
          for (int i = t.rank(); i < nr; i += t.size()) {
            const R api = W.ap[i];
            const R zi = z[i] - pend * (W.inv[i] * api);
            const R xi = x[i] + pend * W.p[i];
            z[i] = zi;
            x[i] = xi;
            r[i] = r[i] - pend * api;
            const R a = row_J(T, W, i, W.w) + W.cd[i] * zi + eps * zi;
            W.az[i] = a;
            za += (double)zi * a;
            if (pending_best) W.bx[i] = xi;
          }
          pend = R(0);
        } else {  // w pulled in phase B from z - a M^-1 ap, the same expression as the committed zn
          for (int i = t.rank(); i < nr; i += t.size()) {
            const R a = row_J(T, W, i, W.w) + row_C<R, kTets>(T, W, i, z) + eps * z[i];
            W.az[i] = a;
            za += (double)z[i] * a;
            if (pending_best) W.bx[i] = x[i];
          }
        }
        pending_best = false;
        {
          double s[1] = {za};
          t.reduce_sum(s);
          beta = s[0] / zaz;
          zaz = s[0];
        }
      }
      if (pending_best || pend != R(0)) {  // an accepted update whose commit pass never ran
        for (int i = t.rank(); i < nr; i += t.size()) {
          const R xi = x[i] + pend * W.p[i];
          x[i] = xi;
          if (pending_best) W.bx[i] = xi;
        }
      }
      W.x = x;
      W.xn = xn;
      W.r = r;
      W.rn = rn;
      W.z = z;
      W.zn = zn;
      }  // memory path
    }
    io.linear_iterations = lin_used;
    io.linear_breakdown = breakdown;
    io.linear_residual = hist_n > 0 ? hist_last : 0.0;
    if (W.dec && t.rank() == 0)  // PCR exit: breakdown > monotone guard > tolerance > budget
      W.dec[dec_exit] = !(nr > 0) ? kExitNone
                                  : (breakdown ? kExitBreakdown
                                               : (mono ? kExitMonotone
                                                       : (hist_last <= cfg.linear_tolerance ? kExitTol : kExitBudget)));
    t.sync();
    // ---- du = H^-1 (J^T dlambda - g); NaN check (newton.cpp:295,362-369)
    double dl2 = 0.0, du2 = 0.0, bad = 0.0;
    for (int i = t.rank(); i < nr; i += t.size()) {
      const R v = W.bx[i];
      dl2 += (double)v * v;
      if (!isfinite(v)) bad = 1.0;
    }
    for_blocks(t, T, W, RowArr<R>{W.bx}, [&](int b, V3<R> jd) {
      if (!(nr > 0)) jd = v3(R(0), R(0), R(0));
      const V3<R> dv = hinv_apply(T, W, b, jd - ld3(W.g + 3 * b));
      st3(W.du + 3 * b, dv);
      du2 += (double)dv.x * dv.x + (double)dv.y * dv.y + (double)dv.z * dv.z;
      if (!isfinite(dv.x) || !isfinite(dv.y) || !isfinite(dv.z)) bad = 1.0;
    });
    {
      double s[2] = {dl2, du2}, m[1] = {bad};
      t.reduce(s, m);
      dl2 = s[0];
      du2 = s[1];
      bad = m[0];
    }
    if (bad != 0.0) {
      for (int i = t.rank(); i < T.ncoord; i += t.size()) W.q[i] = W.q0[i];
      for (int i = t.rank(); i < T.ndof; i += t.size()) W.u[i] = W.u0[i];
      if (t.rank() == 0 && out.iters) out.iters[it] = io;
      aborted = 1;
      n_done = it + 1;
      break;
    }
    // ---- optional merit line search (newton.cpp:371-391)
    R tstep = tfrac;
    if (line_search) {
      unsigned char* const dec_row = W.dec;  // the probes' assemblies record no decisions
      W.dec = nullptr;
      const R trials[4] = {R(1), R(0.5), R(0.25), R(0.125)};
      for (int k = 0; k < 4; ++k) {
        const R tr = trials[k];
        R* pl = W.xn;  // probe lambda (free after the solve)
        R* pu = W.ub;  // probe velocities
        for (int i = t.rank(); i < nr; i += t.size()) pl[i] = W.lam[i] + tr * W.bx[i];
        for (int i = t.rank(); i < T.ndof; i += t.size()) pu[i] = W.u[i] + tr * W.du[i];
        t.sync();
        for (int b = t.rank(); b < T.nb; b += t.size()) integrate_body(T, W.q0, W.qp, W.q, pu, b, h);
        t.sync();
        R* save_lam = W.lam;
        W.lam = pl;
        AsmStats ps{0.0, 0.0, 0.0, 0.0};
        assemble<R, kTets>(t, T, W, W.qp, pu, cfg, ps);
        t.sync();
        double pg = 0.0;
        for_blocks(t, T, W, RowArr<R>{W.lam}, [&](int b, V3<R> jl) {
          const V3<R> dv = ld3(pu + 3 * b) - ld3(W.ut + 3 * b);
          V3<R> gv;
          if (T.d3_kind[b] == kRigidAng)
            gv = sym_mul(W.iw6 + 6 * b, dv) - jl;
          else {
            const R m = T.bmass[T.d3_body[b]];
            gv = v3(m * dv.x, m * dv.y, m * dv.z) - jl;
          }
          pg += (double)gv.x * gv.x + (double)gv.y * gv.y + (double)gv.z * gv.z;
        });
        W.lam = save_lam;
        double s[2] = {pg, ps.hsq};
        t.reduce_sum(s);
        if (sqrt(s[0] + s[1]) < io.merit_l2) {
          tstep = tr;
          break;
        }
      }
      W.dec = dec_row;
    }
    // ---- damped update + integration (newton.cpp:393-396). Each body owns its
    // dofs, so u += t du and q = q- + h G(q) u run in one pass.
    for (int i = t.rank(); i < nr; i += t.size()) W.lam[i] += tstep * W.bx[i];
    for (int b = t.rank(); b < T.nb; b += t.size()) {
      const int d = T.bdof[b];
      const int nd = T.btype[b] == 1 ? 6 : 3;
      for (int k = 0; k < nd; ++k) W.u[d + k] += tstep * W.du[d + k];
      integrate_body(T, W.q0, W.q, W.q, W.u, b, h);
    }
    io.step_size = (double)tstep * sqrt(du2 + dl2);
    if (t.rank() == 0) {
      if (out.iters) out.iters[it] = io;
      if (out.hist_len) out.hist_len[it] = nr > 0 ? hist_n : 0;
    }
    n_done = it + 1;
    t.sync();
  }

  if (aborted) {
    if (t.rank() == 0 && out.fin) {
      out.fin[5] = 1.0;
      out.fin[6] = 0.0;
      out.fin[7] = n_done;
    }
    return 1;
  }
  // ---- final assembly for classification and telemetry (newton.cpp:409-416)
  W.dec = nullptr;
  AsmStats fs{0.0, 0.0, 0.0, 0.0};
  assemble<R, kTets>(t, T, W, W.q, W.u, cfg, fs);
  t.sync();
  double gmax = 0.0;
  for_blocks(t, T, W, RowArr<R>{W.lam}, [&](int b, V3<R> jl) {
    const V3<R> du = ld3(W.u + 3 * b) - ld3(W.ut + 3 * b);
    if (T.d3_kind[b] == kRigidAng) {
      const R* s6 = W.iw6 + 6 * b;
      const V3<R> gv = sym_mul(s6, du) - jl;
      gmax = fmax(gmax, fmax((double)(ab(gv.x) / s6[0]), fmax((double)(ab(gv.y) / s6[1]), (double)(ab(gv.z) / s6[2]))));
    } else {
      const R m = T.bmass[T.d3_body[b]];
      const V3<R> gv = v3(m * du.x, m * du.y, m * du.z) - jl;
      gmax = fmax(gmax, fmax((double)(ab(gv.x) / m), fmax((double)(ab(gv.y) / m), (double)(ab(gv.z) / m))));
    }
  });
  // contact telemetry + min gap (fill_contact_telemetry, newton.cpp:67-94)
  double mgap = W.nc ? __builtin_huge_val() : 0.0;
  for (int c = t.rank(); c < W.nc; c += t.size()) {
    const CView<R> cv = contact_view(T, W, c);
    const R* g = W.cgeo + 17 * c;
    const int ba = cv.ba, bb = cv.bb;
    V3<R> pa, pb;
    if (ba < 0) pa = ld3(g);
    else pa = body_pos(T, W.q, ba) + cv.ra;
    if (bb < 0) pb = ld3(g + 3);
    else pb = body_pos(T, W.q, bb) + cv.rb;
    const R gap = dot(cv.n, pa - pb) - g[15];
    const V3<R> dv = contact_dv(cv, W.u);
    const R v0 = dot(cv.d1, dv), v1 = dot(cv.d2, dv);
    const int nrw = W.normal_begin + c, f0 = W.friction_begin + 2 * c;
    const R lf0 = W.lam[f0] / h, lf1 = W.lam[f0 + 1] / h;
    if (out.tel) {
      double* o = out.tel + 6 * c;
      o[0] = gap;
      o[1] = W.lam[nrw] / h;
      o[2] = sqrt(lf0 * lf0 + lf1 * lf1);
      o[3] = g[16];
      o[4] = sqrt(v0 * v0 + v1 * v1);
      o[5] = lf0 * v0 + lf1 * v1;
    }
    mgap = fmin(mgap, (double)gap);
  }
  {
    double s[1] = {0.0}, m[4] = {fmax(gmax, fs.hmax), fs.comp, fs.cone, -mgap};
    t.reduce(s, m);
    if (t.rank() == 0 && out.fin) {
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
  return 0;
}

}  // namespace nsd
