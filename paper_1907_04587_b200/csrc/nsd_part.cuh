// Partitioned PCR for the cooperative grid kernel (k_single_grid<R, kTets, -1>):
// the Schur operator S z = J H^-1 J^T z + C z + eps z of solve_pcr
// (solvers.cpp:127-174, newton.cpp:233-297) with every CTA owning a contiguous
// set of constraint objects (joints, tets, contacts: all rows of an object in one
// CTA) and keeping their rows resident in shared memory for the whole PCR.
//
// Per CR iteration a CTA touches global memory only for the J^T exchange of the
// dof3 blocks it shares with other CTAs:
//   * J^T z' of its own rows is summed per local dof3 block from shared memory in a
//     fixed (row, slot) order;
//   * blocks touched by this CTA alone get w = H^-1 (J^T z') directly; shared blocks
//     publish their partial to global memory and, after the grid barrier the
//     trial-norm reduction needs anyway, every CTA touching the block sums the
//     partials of all of them in CTA order (identical bits in every CTA);
//   * J w, C z and the reductions' terms then come from shared memory again.
// Two grid barriers per CR iteration, as the register path, but the per-iteration
// L2 traffic drops from every incident row's (z, ap, coefficients) to the shared
// blocks' partials. The host builds the partition per step (nsd_api.cu,
// PartPlanH); per-step tables (rows, slots, incidence, exchange lists) are set up
// in shared memory once per step, coefficients and preconditioner once per
// Newton iteration.
#pragma once

namespace nsd {

// Dynamic shared-memory layout of the partitioned PCR: mr rows, ml local blocks,
// mx exchange entries per CTA (host sizing and device carve use the same code).
struct PartSmem {
  size_t o_coeff, o_cc, o_vec, o_w, o_hk, o_gid, o_slot, o_cb, o_lbg, o_lbk, o_incoff, o_inc, o_xoff, o_xent,
      bytes;
  static constexpr int kVecs = 11;  // x r z zn p ap az inv bx xn rn
};
template <class R> NSD_HD PartSmem part_smem(int mr, int ml, int mx) {
  PartSmem L{};
  size_t o = 0;
  auto take = [&](size_t n) {
    const size_t r = o;
    o += (n + 15) & ~size_t(15);
    return r;
  };
  L.o_coeff = take(sizeof(R) * 12 * mr);
  L.o_cc = take(sizeof(R) * 6 * mr);
  L.o_vec = take(sizeof(R) * PartSmem::kVecs * mr);
  L.o_w = take(sizeof(R) * 3 * ml);
  L.o_hk = take(sizeof(R) * 6 * ml);
  L.o_gid = take(sizeof(int) * mr);
  L.o_slot = take(sizeof(int) * 4 * mr);
  L.o_cb = take(sizeof(int) * mr);
  L.o_lbg = take(sizeof(int) * ml);
  L.o_lbk = take(sizeof(int) * ml);
  L.o_incoff = take(sizeof(int) * (ml + 1));
  L.o_inc = take(sizeof(int) * 4 * mr);
  L.o_xoff = take(sizeof(int) * (ml + 1));
  L.o_xent = take(sizeof(int) * mx);
  L.bytes = o;
  return L;
}

template <class R> struct PartView {
  R *coeff, *cc, *w, *hk;
  R *x, *r, *z, *zn, *p, *ap, *az, *inv, *bx, *xn, *rn;
  int *gid, *slot, *cb, *lbg, *lbk, *incoff, *inc, *xoff, *xent;
  int nrow, nlb, f0;  // own rows, local blocks, flat index of local block 0
  int sg;             // lanes per local block in part_scatter (power of two <= 32)
  __device__ PartView(char* s, const Work<R>& W, bool on) {
    if (!on) return;
    const PartSmem L = part_smem<R>(W.part_mr, W.part_ml, W.part_mx);
    coeff = reinterpret_cast<R*>(s + L.o_coeff);
    cc = reinterpret_cast<R*>(s + L.o_cc);
    R* v = reinterpret_cast<R*>(s + L.o_vec);
    const int mr = W.part_mr;
    x = v;
    r = v + mr;
    z = v + 2 * mr;
    zn = v + 3 * mr;
    p = v + 4 * mr;
    ap = v + 5 * mr;
    az = v + 6 * mr;
    inv = v + 7 * mr;
    bx = v + 8 * mr;
    xn = v + 9 * mr;
    rn = v + 10 * mr;
    w = reinterpret_cast<R*>(s + L.o_w);
    hk = reinterpret_cast<R*>(s + L.o_hk);
    gid = reinterpret_cast<int*>(s + L.o_gid);
    slot = reinterpret_cast<int*>(s + L.o_slot);
    cb = reinterpret_cast<int*>(s + L.o_cb);
    lbg = reinterpret_cast<int*>(s + L.o_lbg);
    lbk = reinterpret_cast<int*>(s + L.o_lbk);
    incoff = reinterpret_cast<int*>(s + L.o_incoff);
    inc = reinterpret_cast<int*>(s + L.o_inc);
    xoff = reinterpret_cast<int*>(s + L.o_xoff);
    xent = reinterpret_cast<int*>(s + L.o_xent);
    const int b = blockIdx.x;
    nrow = W.part_row_off[b + 1] - W.part_row_off[b];
    nlb = W.part_lb_off[b + 1] - W.part_lb_off[b];
    f0 = W.part_lb_off[b];
    NSD_CHECK(nrow >= 0 && nrow <= W.part_mr && nlb >= 0 && nlb <= W.part_ml);
    sg = 1;
    while (sg < 32 && 2 * sg * nlb <= (int)blockDim.x) sg *= 2;
  }
};

// Local index of global dof3 block g in the CTA's ascending block list (-1 if g < 0).
__device__ __forceinline__ int part_find(const int* lbg, int n, int g) {
  if (g < 0) return -1;
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (lbg[mid] < g) lo = mid + 1;
    else hi = mid;
  }
  return lbg[lo] == g ? lo : -1;
}

// Once per step (after setup_row_blocks and a grid barrier): the CTA's rows, their
// local slots, the C-block base of each row, the local blocks, the (row, slot)
// incidence per local block in ascending order and the exchange list per local
// block (flat partial indices of every CTA touching it, ascending CTA).
template <class R, bool kTets>
__device__ void part_setup(const Topo<R>& T, const Work<R>& W, PartView<R>& V) {
  const int tid = threadIdx.x, nt = blockDim.x, b = blockIdx.x;
  const int* rows = W.part_rows + W.part_row_off[b];
  const int* lbs = W.part_lb_blk + V.f0;
  for (int l = tid; l < V.nlb; l += nt) {
    V.lbg[l] = lbs[l];
    V.lbk[l] = T.d3_kind[lbs[l]];
  }
  __syncthreads();
  for (int li = tid; li < V.nrow; li += nt) {
    const int i = rows[li];
    V.gid[li] = i;
    int g4[4];
    if (i < T.rows_static) {
#pragma unroll
      for (int k = 0; k < 4; ++k) g4[k] = W.blk[4 * i + k];
    } else {
      const int c = i < W.friction_begin ? i - W.normal_begin : (i - W.friction_begin) >> 1;
      body_blocks(T, W.cbody[2 * c], g4[0], g4[1]);
      body_blocks(T, W.cbody[2 * c + 1], g4[2], g4[3]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      V.slot[4 * li + k] = part_find(V.lbg, V.nlb, g4[k]);
      NSD_CHECK(g4[k] < 0 || V.slot[4 * li + k] >= 0);  // every block a row touches is local
    }
    // C block base (a tet's rows are consecutive among the CTA's rows) or -1 (diagonal C)
    V.cb[li] = (kTets && i >= T.rows_joint && i < T.rows_static) ? li - (i - T.rows_joint) % T.tdim : -1;
  }
  __syncthreads();
  // incidence per local block, (row, slot) ascending: count, scan, fill (deterministic)
  for (int l = tid; l < V.nlb; l += nt) {
    int n = 0;
    for (int e = 0; e < 4 * V.nrow; ++e) n += V.slot[e] == l;
    V.incoff[l + 1] = n;
    const int g = V.lbg[l];
    V.xoff[l + 1] = W.part_gb_off[g + 1] - W.part_gb_off[g];
  }
  __syncthreads();
  if (tid == 0) {
    V.incoff[0] = 0;
    V.xoff[0] = 0;
    for (int l = 0; l < V.nlb; ++l) {
      V.incoff[l + 1] += V.incoff[l];
      V.xoff[l + 1] += V.xoff[l];
    }
    NSD_CHECK(V.incoff[V.nlb] <= 4 * V.nrow && V.xoff[V.nlb] <= W.part_mx);
  }
  __syncthreads();
  for (int l = tid; l < V.nlb; l += nt) {
    int o = V.incoff[l];
    for (int e = 0; e < 4 * V.nrow; ++e)
      if (V.slot[e] == l) V.inc[o++] = e;
    const int g = V.lbg[l];
    const int g0 = W.part_gb_off[g], n = W.part_gb_off[g + 1] - g0;
    NSD_CHECK(o == V.incoff[l + 1] && V.xoff[l] + n == V.xoff[l + 1]);
    for (int k = 0; k < n; ++k) V.xent[V.xoff[l] + k] = W.part_gb_ent[g0 + k];
  }
  __syncthreads();
}

// Once per Newton iteration (after the right-hand side pass and its reduction):
// coefficients (static rows from W.coeff, contact rows regenerated from the contact
// view), C coefficients, r, z, inv, and H^-1 per local block.
template <class R, bool kTets>
__device__ void part_load(const Topo<R>& T, const Work<R>& W, PartView<R>& V) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int li = tid; li < V.nrow; li += nt) {
    const int i = V.gid[li];
    R* c = V.coeff + 12 * li;
    R* cc = V.cc + 6 * li;
    if (i < T.rows_static) {
#pragma unroll
      for (int k = 0; k < 12; ++k) c[k] = opg(W, W.coeff, 12 * (size_t)i + k);
    } else {
      const bool normal = i < W.friction_begin;
      const int k = i - W.friction_begin, c0 = normal ? i - W.normal_begin : (k >> 1);
      const CView<R> cv = contact_view(T, W, c0);
      const R sc = normal ? cv.dc : cv.act;
      const V3<R> d = sc * (normal ? cv.n : ((k & 1) ? cv.d2 : cv.d1));
      const V3<R> ta = cross(cv.ra, d), tb = cross(cv.rb, d);
      const R v12[12] = {d.x, d.y, d.z, ta.x, ta.y, ta.z, -d.x, -d.y, -d.z, -tb.x, -tb.y, -tb.z};
#pragma unroll
      for (int s = 0; s < 12; ++s) c[s] = v12[s];
    }
    if (kTets && i >= T.rows_joint && i < T.rows_static) {
      const int td = T.tdim, e = (i - T.rows_joint) / td, k = (i - T.rows_joint) - td * e;
      for (int j = 0; j < td; ++j) cc[j] = opg(W, W.ctet, (size_t)td * td * e + td * k + j);
    } else {
      cc[0] = W.cd[i];
    }
    V.r[li] = W.r[i];
    V.z[li] = W.z[i];
    V.inv[li] = W.inv[i];
    V.x[li] = R(0);
    V.bx[li] = R(0);
  }
  for (int l = tid; l < V.nlb; l += nt) {
    const int g = V.lbg[l];
    R* h = V.hk + 6 * l;
    if (V.lbk[l] == kRigidAng) {
#pragma unroll
      for (int k = 0; k < 6; ++k) h[k] = W.iwi6[6 * g + k];
    } else {
#pragma unroll
      for (int k = 0; k < 3; ++k) h[k] = W.hinv[3 * g + k];
    }
  }
  __syncthreads();
}

template <class R> __device__ __forceinline__ V3<R> part_hinv(const PartView<R>& V, int l, V3<R> v) {
  const R* h = V.hk + 6 * l;
  if (V.lbk[l] == kRigidAng) return sym_mul(h, v);
  return v3(v.x * h[0], v.y * h[1], v.z * h[2]);
}

// J^T y per local block from shared memory; blocks of this CTA alone get w, shared
// blocks publish their partial (read back by part_gather after a grid barrier).
// V.sg lanes of one warp share a block: each sums every sg-th incidence entry, then a
// fixed shuffle tree combines them (deterministic). A FEM vertex block gathers up to
// ~60 (row, slot) entries inside one CTA, so one lane per block made this serial
// chain the CTA's critical path while most threads idled (nlb << blockDim).
template <class R>
__device__ __forceinline__ void part_scatter(const Work<R>& W, PartView<R>& V, const R* y) {
  R* gp = static_cast<R*>(W.part_partial);
  const int G = V.sg, gl = threadIdx.x & (G - 1), ng = blockDim.x / G;
  for (int base = 0; base < V.nlb; base += ng) {  // uniform trip count: every lane joins the shuffles
    const int l = base + threadIdx.x / G;
    R sx = R(0), sy = R(0), sz = R(0);
    if (l < V.nlb) {
      for (int e = V.incoff[l] + gl; e < V.incoff[l + 1]; e += G) {
        const int ent = V.inc[e];
        const int li = ent >> 2, k = ent & 3;
        const R yr = y[li];
        const R* c = V.coeff + 12 * li + 3 * k;
        sx += c[0] * yr;
        sy += c[1] * yr;
        sz += c[2] * yr;
      }
    }
    for (int off = G >> 1; off > 0; off >>= 1) {
      sx += __shfl_down_sync(0xffffffffu, sx, off, G);
      sy += __shfl_down_sync(0xffffffffu, sy, off, G);
      sz += __shfl_down_sync(0xffffffffu, sz, off, G);
    }
    if (l >= V.nlb || gl != 0) continue;
    if (V.xoff[l + 1] - V.xoff[l] > 1) {
      R* o = gp + 3 * (V.f0 + l);
      o[0] = sx;
      o[1] = sy;
      o[2] = sz;
    } else {
      st3(V.w + 3 * l, part_hinv(V, l, v3(sx, sy, sz)));
    }
  }
}
// w of the shared blocks: partials of every CTA touching the block, CTA order.
// Threads [first, first + n) of the CTA take part.
template <class R>
__device__ __forceinline__ void part_gather(const Work<R>& W, PartView<R>& V, int first, int n) {
  const R* gp = static_cast<const R*>(W.part_partial);
  for (int l = first; l < V.nlb; l += n) {
    const int x0 = V.xoff[l], x1 = V.xoff[l + 1];
    if (x1 - x0 <= 1) continue;
    R sx = R(0), sy = R(0), sz = R(0);
    for (int e = x0; e < x1; ++e) {
      const R* o = gp + 3 * V.xent[e];
      sx += __ldcg(o);
      sy += __ldcg(o + 1);
      sz += __ldcg(o + 2);
    }
    st3(V.w + 3 * l, part_hinv(V, l, v3(sx, sy, sz)));
  }
}

// (S y)_li = J_li w + (C y)_li + eps y_li from shared memory (slot_dot / row_C order).
template <class R>
__device__ __forceinline__ R part_row(const PartView<R>& V, int li, const R* y, int td, R eps) {
  const R* c = V.coeff + 12 * li;
  R s = R(0);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int l = V.slot[4 * li + k];
    if (l < 0) continue;
    const R* w = V.w + 3 * l;
    s += c[3 * k] * w[0] + c[3 * k + 1] * w[1] + c[3 * k + 2] * w[2];
  }
  const R* cc = V.cc + 6 * li;
  const int b = V.cb[li];
  R cz;
  if (b < 0) {  // scalar compliance
    cz = cc[0] * y[li];
  } else if (td == 3) {
    cz = cc[0] * y[b] + cc[1] * y[b + 1] + cc[2] * y[b + 2];
  } else {
    cz = R(0);
    for (int j = 0; j < td; ++j) cz += cc[j] * y[b + j];
  }
  return s + cz + eps * y[li];
}

}  // namespace nsd
