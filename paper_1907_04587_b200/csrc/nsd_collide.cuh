// Primitive narrow phase (reference: src/collision.cpp:16-297) as host/device
// code: sphere/box/half-space pairs, the 4-deepest-corner rule with feature
// tie-break (:87-93), the predicted-gap filter with the unconstrained velocity
// (:273-287) and the canonical (a.body, b.body, feature) order (:290-295).
// Used on the device by the batched step (one team per environment) and on the
// host by the product's world layer. Also the caller-side particle-vs-shape
// generator the FEM configs need as zero-radius spheres.
#pragma once

#include "nsd_math.cuh"

namespace nsd {

template <class R> struct ShapeD {
  int body, kind;  // kind 0 half-space, 1 sphere, 2 box
  R n[3], offset, radius, he[3], thick, mu;
};

template <class R> struct CandD {
  int a, b, feature;
  R la[3], lb[3], n[3];
  R gap, thick, mu;
};

// Minimal body view for collision: packed state + layout.
template <class R> struct BodyView {
  const int* btype;
  const int* bdof;
  const int* bcoord;
  const R* q;
  const R* u;    // predicted velocities
  const R* rot;  // optional cache: 9 per body, row-major rotation at q (same values quat_rot gives)
};

template <class R> NSD_HD V3<R> bv_pos(const BodyView<R>& v, int b) {
  const R* p = v.q + v.bcoord[b];
  return v3(p[0], p[1], p[2]);
}
template <class R> NSD_HD M3<R> bv_rot(const BodyView<R>& v, int b) {
  if (b < 0 || v.btype[b] == 0) return m3_identity<R>();
  if (v.rot) {
    M3<R> m;
    for (int i = 0; i < 9; ++i) m.a[i] = v.rot[9 * b + i];
    return m;
  }
  const R* t = v.q + v.bcoord[b] + 3;
  return quat_rot(t[0], t[1], t[2], t[3]);
}
template <class R> NSD_HD V3<R> shape_pos(const BodyView<R>& v, const ShapeD<R>& s) {
  return s.body < 0 ? v3(R(0), R(0), R(0)) : bv_pos(v, s.body);
}
template <class R> NSD_HD M3<R> shape_rot(const BodyView<R>& v, const ShapeD<R>& s) {
  return s.body < 0 ? m3_identity<R>() : bv_rot(v, s.body);
}
template <class R> NSD_HD V3<R> to_local(const BodyView<R>& v, const ShapeD<R>& s, V3<R> w) {
  if (s.body < 0) return w;
  return mul_t(shape_rot(v, s), w - shape_pos(v, s));
}
template <class R> NSD_HD void put3(R* d, V3<R> a) {
  d[0] = a.x;
  d[1] = a.y;
  d[2] = a.z;
}
template <class R> NSD_HD V3<R> get3(const R* d) { return v3(d[0], d[1], d[2]); }

template <class R> NSD_HD V3<R> corner(const R* he, int k) {
  // corners_of_box order: sx, sy, sz each in {-1, 1}, z fastest
  const R sx = (k & 4) ? R(1) : R(-1), sy = (k & 2) ? R(1) : R(-1), sz = (k & 1) ? R(1) : R(-1);
  return v3(sx * he[0], sy * he[1], sz * he[2]);
}

// Rank of candidate k among the valid ones by (gap, feature): features are
// unique, so ranks 0..3 are exactly the 4 smallest in ascending order, the order
// the reference's sorted keep-4 produces (collision.cpp:87-93). Fully unrolled over the
// 8 corners so gaps and ranks stay in registers (no candidate array in local
// memory).
template <class R> NSD_HD void rank8(const R (&gap)[8], const bool (&valid)[8], int (&rank)[8]) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int r = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      r += (valid[j] && (gap[j] < gap[k] || (gap[j] == gap[k] && j < k))) ? 1 : 0;
    rank[k] = r;
  }
}

template <class R>
NSD_HD int sphere_halfspace(const BodyView<R>& v, const ShapeD<R>& sph, const ShapeD<R>& hs, CandD<R>* out) {
  const V3<R> n = normalize(get3(hs.n));
  const V3<R> c = shape_pos(v, sph);
  const R gap = dot(n, c) - hs.offset - sph.radius;
  CandD<R>& o = out[0];
  o.gap = gap;
  o.a = sph.body;
  const V3<R> surf = c - sph.radius * n;
  put3(o.la, to_local(v, sph, surf));
  o.b = hs.body;
  put3(o.lb, surf - gap * n);
  put3(o.n, n);
  o.feature = 0;
  return 1;
}

template <class R>
NSD_HD int box_halfspace(const BodyView<R>& v, const ShapeD<R>& box, const ShapeD<R>& hs, CandD<R>* out) {
  const V3<R> n = normalize(get3(hs.n));
  const M3<R> r = shape_rot(v, box);
  const V3<R> x = shape_pos(v, box);
  R gap[8];
  bool valid[8];
  int rank[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    gap[k] = dot(n, x + mul(r, corner(box.he, k))) - hs.offset;
    valid[k] = true;
  }
  rank8(gap, valid, rank);  // feature = corner index k
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (rank[k] >= 4) continue;
    const V3<R> cl = corner(box.he, k);
    const V3<R> w = x + mul(r, cl);
    CandD<R>& o = out[rank[k]];
    o.gap = gap[k];
    o.a = box.body;
    put3(o.la, cl);
    o.b = hs.body;
    put3(o.lb, w - gap[k] * n);
    put3(o.n, n);
    o.feature = k;
  }
  return 4;
}

template <class R>
NSD_HD int sphere_sphere(const BodyView<R>& v, const ShapeD<R>& a, const ShapeD<R>& b, CandD<R>* out) {
  const V3<R> ca = shape_pos(v, a), cb = shape_pos(v, b);
  const V3<R> d = ca - cb;
  const R dist = norm(d);
  const V3<R> n = dist > R(1e-12) ? d / dist : v3(R(0), R(0), R(1));
  CandD<R>& o = out[0];
  o.gap = dist - a.radius - b.radius;
  o.a = a.body;
  put3(o.la, to_local(v, a, ca - a.radius * n));
  o.b = b.body;
  put3(o.lb, to_local(v, b, cb + b.radius * n));
  put3(o.n, n);
  o.feature = 0;
  return 1;
}

// Point (sphere centre c with radius) against a box (collision.cpp:345-384).
template <class R>
NSD_HD void point_box(const BodyView<R>& v, V3<R> c, R radius, const ShapeD<R>& box, V3<R>& n_out, R& gap,
                      V3<R>& closest_out) {
  const M3<R> r = shape_rot(v, box);
  const V3<R> x = shape_pos(v, box);
  const V3<R> cl = mul_t(r, c - x);
  V3<R> cp = v3(mn(mx(cl.x, -box.he[0]), box.he[0]), mn(mx(cl.y, -box.he[1]), box.he[1]),
                mn(mx(cl.z, -box.he[2]), box.he[2]));
  V3<R> nl;
  R dist;
  if (norm(cl - cp) > R(1e-12)) {
    dist = norm(cl - cp);
    nl = (cl - cp) / dist;
  } else {
    int axis = 0;
    R best = box.he[0] - ab(cl.x);
    for (int k = 1; k < 3; ++k) {
      const R pen = box.he[k] - ab(cl[k]);
      if (pen < best) {
        best = pen;
        axis = k;
      }
    }
    nl = v3(R(0), R(0), R(0));
    nl[axis] = cl[axis] >= R(0) ? R(1) : R(-1);
    cp = cl;
    cp[axis] = nl[axis] * box.he[axis];
    dist = -best;
  }
  n_out = mul(r, nl);
  gap = dist - radius;
  closest_out = cp;
}

template <class R>
NSD_HD int sphere_box(const BodyView<R>& v, const ShapeD<R>& sph, const ShapeD<R>& box, CandD<R>* out) {
  const V3<R> c = shape_pos(v, sph);
  V3<R> n, cp;
  R gap;
  point_box(v, c, sph.radius, box, n, gap, cp);
  CandD<R>& o = out[0];
  o.gap = gap;
  o.a = sph.body;
  put3(o.la, to_local(v, sph, c - sph.radius * n));
  o.b = box.body;
  put3(o.lb, cp);
  put3(o.n, n);
  o.feature = 0;
  return 1;
}

template <class R>
NSD_HD int box_box(const BodyView<R>& v, const ShapeD<R>& sa, const ShapeD<R>& sb, R margin, CandD<R>* out) {
  // (the two boxes' frames are selected by value, never through a runtime index,
  // so they stay in registers)
  const V3<R> pos0 = shape_pos(v, sa), pos1 = shape_pos(v, sb);
  {  // Exact early-out (results unchanged): the face axis of box a nearest the centre
     // line makes an angle with it of cos >= 1/sqrt(3), so its separation is at least
     // |dc|/sqrt(3) - r_a - r_b (circumradii); beyond sqrt(3)(r_a + r_b + margin) every
     // face-axis separation, hence best_sep below, exceeds the margin -> no candidates.
    const V3<R> dc = pos1 - pos0;
    const R ra = sqrt(sa.he[0] * sa.he[0] + sa.he[1] * sa.he[1] + sa.he[2] * sa.he[2]);
    const R rb = sqrt(sb.he[0] * sb.he[0] + sb.he[1] * sb.he[1] + sb.he[2] * sb.he[2]);
    const R lim = ra + rb + margin;
    if (dot(dc, dc) > R(3.0001) * lim * lim) return 0;
  }
  const M3<R> rot0 = shape_rot(v, sa), rot1 = shape_rot(v, sb);
  int best_ref = -1, best_axis = -1;
  R best_dir = R(1), best_sep = -Lim<R>::inf();
#pragma unroll
  for (int ref = 0; ref < 2; ++ref) {
    const M3<R>& rr = ref == 0 ? rot0 : rot1;
    const M3<R>& ro = ref == 0 ? rot1 : rot0;
    const V3<R> pr = ref == 0 ? pos0 : pos1, po = ref == 0 ? pos1 : pos0;
    const ShapeD<R>& br = ref == 0 ? sa : sb;
    const ShapeD<R>& bo = ref == 0 ? sb : sa;
    V3<R> wc[8];  // the other box's world corners, once per reference box (same values per axis)
#pragma unroll
    for (int k = 0; k < 8; ++k) wc[k] = po + mul(ro, corner(bo.he, k));
    for (int axis = 0; axis < 3; ++axis)
      for (int di = 0; di < 2; ++di) {
        const R dir = di == 0 ? R(1) : R(-1);
        const V3<R> n = dir * col(rr, axis);
        const V3<R> fp = pr + (dir * br.he[axis]) * col(rr, axis);
        R mnp = Lim<R>::inf();
#pragma unroll
        for (int k = 0; k < 8; ++k) mnp = mn(mnp, dot(n, wc[k] - fp));
        if (mnp > best_sep + R(1e-12)) {
          best_sep = mnp;
          best_ref = ref;
          best_axis = axis;
          best_dir = dir;
        }
      }
  }
  if (best_sep > margin) return 0;
  const bool r0 = best_ref == 0;
  const ShapeD<R>& bref = r0 ? sa : sb;
  const ShapeD<R>& binc = r0 ? sb : sa;
  const M3<R> rot_ref = r0 ? rot0 : rot1, rot_inc = r0 ? rot1 : rot0;
  const V3<R> pos_ref = r0 ? pos0 : pos1, pos_inc = r0 ? pos1 : pos0;
  const V3<R> nref = best_dir * col(rot_ref, best_axis);
  const V3<R> fp = pos_ref + (best_dir * bref.he[best_axis]) * col(rot_ref, best_axis);
  R gap[8];
  bool valid[8];
  int rank[8];
  int m = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const V3<R> w = pos_inc + mul(rot_inc, corner(binc.he, k));
    gap[k] = dot(nref, w - fp);
    bool ok = !(gap[k] > margin);
    const V3<R> in_ref = mul_t(rot_ref, w - pos_ref);
#pragma unroll
    for (int axis = 0; axis < 3; ++axis) {
      if (axis == best_axis) continue;
      if (ab(in_ref[axis]) > bref.he[axis] + R(1e-6)) ok = false;
    }
    valid[k] = ok;
    m += ok ? 1 : 0;
  }
  rank8(gap, valid, rank);  // among the valid corners; feature = corner index k
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (!valid[k] || rank[k] >= 4) continue;
    const V3<R> ck = corner(binc.he, k);
    const V3<R> w = pos_inc + mul(rot_inc, ck);
    CandD<R>& o = out[rank[k]];
    o.gap = gap[k];
    o.a = binc.body;
    put3(o.la, ck);
    o.b = bref.body;
    put3(o.lb, to_local(v, bref, w - gap[k] * nref));
    put3(o.n, nref);
    o.feature = k;
  }
  return m < 4 ? m : 4;
}

template <class R> NSD_HD V3<R> point_vel(const BodyView<R>& v, int body, V3<R> w) {
  if (body < 0) return v3(R(0), R(0), R(0));
  const R* u = v.u + v.bdof[body];
  const V3<R> lin = v3(u[0], u[1], u[2]);
  if (v.btype[body] == 0) return lin;
  return lin + cross(v3(u[3], u[4], u[5]), w - bv_pos(v, body));
}
template <class R> NSD_HD V3<R> attach_pt(const BodyView<R>& v, int body, const R* local) {
  if (body < 0) return get3(local);
  if (v.btype[body] == 0) return bv_pos(v, body);
  return bv_pos(v, body) + mul(bv_rot(v, body), get3(local));
}

// Candidates of shape pair (i < j) after the predicted-gap filter; returns the
// number kept (<= 4), each tagged with thickness and mu in out[k] via the
// caller. Mirrors the dispatch at collision.cpp:253-271.
template <class R>
NSD_HD int pair_contacts(const BodyView<R>& v, const ShapeD<R>& si, const ShapeD<R>& sj, R h, R margin, R mu_default,
                         CandD<R>* out, R* thick_out, R* mu_out) {
  if (si.body < 0 && sj.body < 0) return 0;
  if (si.body >= 0 && si.body == sj.body) return 0;
  CandD<R>* c = out;  // generated in place (no local staging array), compacted below
  int n = 0;
  const int ki = si.kind, kj = sj.kind;
  if (ki == 1 && kj == 0) n = sphere_halfspace(v, si, sj, c);
  else if (ki == 0 && kj == 1) n = sphere_halfspace(v, sj, si, c);
  else if (ki == 2 && kj == 0) n = box_halfspace(v, si, sj, c);
  else if (ki == 0 && kj == 2) n = box_halfspace(v, sj, si, c);
  else if (ki == 1 && kj == 1) n = sphere_sphere(v, si, sj, c);
  else if (ki == 1 && kj == 2) n = sphere_box(v, si, sj, c);
  else if (ki == 2 && kj == 1) n = sphere_box(v, sj, si, c);
  else if (ki == 2 && kj == 2) n = box_box(v, si, sj, margin, c);
  else return 0;
  const R thick = si.thick + sj.thick;
  const R ma = si.mu >= R(0) ? si.mu : mu_default, mb = sj.mu >= R(0) ? sj.mu : mu_default;
  const R mu = sqrt(ma * mb);
  int kept = 0;
  for (int k = 0; k < n; ++k) {
    const V3<R> pa = attach_pt(v, c[k].a, c[k].la), pb = attach_pt(v, c[k].b, c[k].lb);
    const V3<R> va = point_vel(v, c[k].a, pa), vb = point_vel(v, c[k].b, pb);
    const R closing = -dot(get3(c[k].n), va - vb);
    const R predicted = (c[k].gap - thick) - h * closing;
    if (predicted > margin) continue;
    c[k].thick = thick;
    c[k].mu = mu;
    if (kept != k) out[kept] = c[k];  // in-place compaction: kept <= k
    ++kept;
  }
  *thick_out = thick;
  *mu_out = mu;
  return kept;
}

// Particle point against a half-space or box (extension generator).
template <class R>
NSD_HD int particle_shape_contact(const BodyView<R>& v, int body, const ShapeD<R>& sh, R h, R margin, R mu_default,
                                  R gen_thick, R gen_mu, CandD<R>* out, R* thick_out, R* mu_out) {
  const V3<R> x = bv_pos(v, body);
  CandD<R> c;
  if (sh.kind == 0) {
    const V3<R> n = normalize(get3(sh.n));
    const R gap = dot(n, x) - sh.offset;
    c.gap = gap;
    c.a = body;
    put3(c.la, v3(R(0), R(0), R(0)));
    c.b = sh.body;
    put3(c.lb, x - gap * n);
    put3(c.n, n);
    c.feature = 0;
  } else if (sh.kind == 2) {
    V3<R> n, cp;
    R gap;
    point_box(v, x, R(0), sh, n, gap, cp);
    c.gap = gap;
    c.a = body;
    put3(c.la, v3(R(0), R(0), R(0)));
    c.b = sh.body;
    put3(c.lb, cp);
    put3(c.n, n);
    c.feature = 0;
  } else {
    return 0;
  }
  const R thick = gen_thick + sh.thick;
  const R ma = gen_mu >= R(0) ? gen_mu : mu_default, mb = sh.mu >= R(0) ? sh.mu : mu_default;
  *thick_out = thick;
  *mu_out = sqrt(ma * mb);
  const V3<R> pa = attach_pt(v, c.a, c.la), pb = attach_pt(v, c.b, c.lb);
  const R closing = -dot(get3(c.n), point_vel(v, c.a, pa) - point_vel(v, c.b, pb));
  if ((c.gap - thick) - h * closing > margin) return 0;
  c.thick = thick;
  c.mu = *mu_out;
  out[0] = c;
  return 1;
}

template <class R> NSD_HD void tangent_basis(V3<R> n, V3<R>& d1, V3<R>& d2) {
  int sm = 0;
  if (ab(n.y) < ab(n.x)) sm = 1;
  if (ab(n.z) < ab(n[sm])) sm = 2;
  V3<R> e = v3(R(0), R(0), R(0));
  e[sm] = R(1);
  d1 = normalize(e - dot(e, n) * n);
  d2 = cross(n, d1);
}

NSD_HD bool canonical_less(int a0, int b0, int f0, int a1, int b1, int f1) {
  if (a0 != a1) return a0 < a1;
  if (b0 != b1) return b0 < b1;
  return f0 < f1;
}

}  // namespace nsd
