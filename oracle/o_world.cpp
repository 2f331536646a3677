// ORACLE — test infrastructure only. CPU restatement of
// /root/reference/proj/src/collision.cpp (detect), src/scene.cpp:556-935
// (build_world, step_world, reference builders), plus the synthetic BASELINE
// configs C1-C5 and the two caller-side extensions the reference lacks
// (particle contact generation, joint-torque hook) — SURVEY.md §0 fact 4,
// Appendix C. The product restates the same builders independently
// (paper_1907_04587_b200/csrc/nsd_scene.cpp); tests check they agree bit for bit.
#include "oracle.h"

#include <random>
#include <sstream>
#include <stdexcept>

namespace orc {

// ============================ collision ======================================
namespace {

struct Cand {
  Contact c;
  double gap = 0.0;
};

V3 shape_pos(const State& s, const AttachedShape& sh) { return sh.body < 0 ? V3() : s.position(sh.body); }
M3 shape_rot(const State& s, const AttachedShape& sh) {
  return sh.body < 0 ? M3::identity() : s.rotation(sh.body);
}
V3 to_local(const State& s, const AttachedShape& sh, const V3& w) {
  if (sh.body < 0) return w;
  return shape_rot(s, sh).t() * (w - shape_pos(s, sh));
}
double pair_mu(double ma_raw, double mb_raw, const ContactParams& p) {
  const double ma = ma_raw >= 0.0 ? ma_raw : p.mu_default;
  const double mb = mb_raw >= 0.0 ? mb_raw : p.mu_default;
  return std::sqrt(ma * mb);
}
V3 point_vel(const State& s, const VecX& u, int body, const V3& w) {
  if (body < 0) return V3();
  const int o = s.dof_off[body];
  const V3 lin(u[o], u[o + 1], u[o + 2]);
  if (s.bodies[body].type == BodyType::Particle) return lin;
  return lin + cross(V3(u[o + 3], u[o + 4], u[o + 5]), w - s.position(body));
}
void box_corners(const V3& he, V3 out[8]) {
  int k = 0;
  for (int sx : {-1, 1})
    for (int sy : {-1, 1})
      for (int sz : {-1, 1}) out[k++] = V3(sx * he[0], sy * he[1], sz * he[2]);
}
bool gap_less(const Cand& a, const Cand& b) {
  return a.gap != b.gap ? a.gap < b.gap : a.c.feature < b.c.feature;
}

void sphere_halfspace(const State& s, const AttachedShape& sph, const AttachedShape& hs,
                      std::vector<Cand>& out) {
  const V3 n = normalized(hs.shape.normal);
  const V3 c = shape_pos(s, sph);
  const double gap = dot(n, c) - hs.shape.offset - sph.shape.radius;
  Cand cd;
  cd.gap = gap;
  cd.c.a = {sph.body, to_local(s, sph, c - sph.shape.radius * n)};
  const V3 surface = c - sph.shape.radius * n;
  cd.c.b = {hs.body, surface - gap * n};
  cd.c.normal = n;
  out.push_back(cd);
}

void box_halfspace(const State& s, const AttachedShape& box, const AttachedShape& hs,
                   std::vector<Cand>& out) {
  const V3 n = normalized(hs.shape.normal);
  const M3 r = shape_rot(s, box);
  const V3 x = shape_pos(s, box);
  V3 corners[8];
  box_corners(box.shape.half_extents, corners);
  std::vector<Cand> loc;
  for (int k = 0; k < 8; ++k) {
    const V3 w = x + r * corners[k];
    Cand cd;
    cd.gap = dot(n, w) - hs.shape.offset;
    cd.c.a = {box.body, corners[k]};
    cd.c.b = {hs.body, w - cd.gap * n};
    cd.c.normal = n;
    cd.c.feature = k;
    loc.push_back(cd);
  }
  std::sort(loc.begin(), loc.end(), gap_less);
  if (loc.size() > 4) loc.resize(4);
  out.insert(out.end(), loc.begin(), loc.end());
}

void sphere_sphere(const State& s, const AttachedShape& a, const AttachedShape& b,
                   std::vector<Cand>& out) {
  const V3 ca = shape_pos(s, a), cb = shape_pos(s, b);
  const V3 d = ca - cb;
  const double dist = norm(d);
  const V3 n = dist > 1e-12 ? d / dist : V3(0, 0, 1);
  Cand cd;
  cd.gap = dist - a.shape.radius - b.shape.radius;
  cd.c.a = {a.body, to_local(s, a, ca - a.shape.radius * n)};
  cd.c.b = {b.body, to_local(s, b, cb + b.shape.radius * n)};
  cd.c.normal = n;
  out.push_back(cd);
}

// Closest point of a point (sphere centre with `radius`) against a box shape;
// shared by sphere-box (collision.cpp:345-384) and the particle generator.
void point_box(const State& s, int a_body, const V3& c, double radius, const AttachedShape& box,
               const V3& a_local, std::vector<Cand>& out) {
  const M3 r = shape_rot(s, box);
  const V3 x = shape_pos(s, box);
  const V3 he = box.shape.half_extents;
  const V3 cl = r.t() * (c - x);
  V3 closest(std::min(std::max(cl[0], -he[0]), he[0]), std::min(std::max(cl[1], -he[1]), he[1]),
             std::min(std::max(cl[2], -he[2]), he[2]));
  V3 nl;
  double dist;
  if (norm(cl - closest) > 1e-12) {
    dist = norm(cl - closest);
    nl = (cl - closest) / dist;
  } else {
    int axis = 0;
    double best = he[0] - std::abs(cl[0]);
    for (int k = 1; k < 3; ++k) {
      const double pen = he[k] - std::abs(cl[k]);
      if (pen < best) {
        best = pen;
        axis = k;
      }
    }
    nl = V3();
    nl[axis] = cl[axis] >= 0.0 ? 1.0 : -1.0;
    closest = cl;
    closest[axis] = nl[axis] * he[axis];
    dist = -best;
  }
  const V3 n = r * nl;
  Cand cd;
  cd.gap = dist - radius;
  cd.c.a = {a_body, a_local};
  cd.c.b = {box.body, closest};
  cd.c.normal = n;
  out.push_back(cd);
  (void)c;
}

void sphere_box(const State& s, const AttachedShape& sph, const AttachedShape& box,
                std::vector<Cand>& out) {
  const V3 c = shape_pos(s, sph);
  // n is only known after the closest-point query; recompute a.local after.
  std::vector<Cand> tmp;
  point_box(s, sph.body, c, sph.shape.radius, box, V3(), tmp);
  Cand cd = tmp[0];
  cd.c.a.local = to_local(s, sph, c - sph.shape.radius * cd.c.normal);
  out.push_back(cd);
}

void box_box(const State& s, const AttachedShape& sa, const AttachedShape& sb, double margin,
             std::vector<Cand>& out) {
  const AttachedShape* bx[2] = {&sa, &sb};
  M3 rot[2];
  V3 pos[2];
  for (int k = 0; k < 2; ++k) {
    rot[k] = shape_rot(s, *bx[k]);
    pos[k] = shape_pos(s, *bx[k]);
  }
  const auto face_sep = [&](int ref, int axis, double dir) {
    const V3 n = dir * rot[ref].col(axis);
    const V3 fp = pos[ref] + (dir * bx[ref]->shape.half_extents[axis]) * rot[ref].col(axis);
    const int other = 1 - ref;
    double mn = std::numeric_limits<double>::infinity();
    V3 cs[8];
    box_corners(bx[other]->shape.half_extents, cs);
    for (int k = 0; k < 8; ++k) {
      const V3 w = pos[other] + rot[other] * cs[k];
      mn = std::min(mn, dot(n, w - fp));
    }
    return mn;
  };
  int best_ref = -1, best_axis = -1;
  double best_dir = 1.0, best_sep = -std::numeric_limits<double>::infinity();
  for (int ref = 0; ref < 2; ++ref)
    for (int axis = 0; axis < 3; ++axis)
      for (double dir : {1.0, -1.0}) {
        const double sep = face_sep(ref, axis, dir);
        if (sep > best_sep + 1e-12) {
          best_sep = sep;
          best_ref = ref;
          best_axis = axis;
          best_dir = dir;
        }
      }
  if (best_sep > margin) return;
  const int ref = best_ref, inc = 1 - best_ref;
  const V3 nref = best_dir * rot[ref].col(best_axis);
  const V3 fp = pos[ref] + (best_dir * bx[ref]->shape.half_extents[best_axis]) * rot[ref].col(best_axis);
  V3 cs[8];
  box_corners(bx[inc]->shape.half_extents, cs);
  std::vector<Cand> loc;
  for (int k = 0; k < 8; ++k) {
    const V3 w = pos[inc] + rot[inc] * cs[k];
    const double gap = dot(nref, w - fp);
    if (gap > margin) continue;
    const V3 in_ref = rot[ref].t() * (w - pos[ref]);
    bool inside = true;
    for (int axis = 0; axis < 3; ++axis) {
      if (axis == best_axis) continue;
      if (std::abs(in_ref[axis]) > bx[ref]->shape.half_extents[axis] + 1e-6) inside = false;
    }
    if (!inside) continue;
    Cand cd;
    cd.gap = gap;
    cd.c.a = {bx[inc]->body, cs[k]};
    cd.c.b = {bx[ref]->body, to_local(s, *bx[ref], w - gap * nref)};
    cd.c.normal = nref;
    cd.c.feature = k;
    loc.push_back(cd);
  }
  std::sort(loc.begin(), loc.end(), gap_less);
  if (loc.size() > 4) loc.resize(4);
  out.insert(out.end(), loc.begin(), loc.end());
}

bool canonical_less(const Contact& a, const Contact& b) {  // collision.cpp:290-295
  if (a.a.body != b.a.body) return a.a.body < b.a.body;
  if (a.b.body != b.b.body) return a.b.body < b.b.body;
  return a.feature < b.feature;
}

// Predicted-gap filter and contact finalisation, collision.cpp:273-287.
void finalize_candidates(const State& s, std::vector<Cand>& cands, double thickness, double mu,
                         const VecX& u_pred, double h, const ContactParams& p,
                         std::vector<Contact>& out) {
  for (Cand& cd : cands) {
    const V3 pa = attach_point(s, cd.c.a), pb = attach_point(s, cd.c.b);
    const V3 va = point_vel(s, u_pred, cd.c.a.body, pa), vb = point_vel(s, u_pred, cd.c.b.body, pb);
    const double closing = -dot(cd.c.normal, va - vb);
    const double predicted = (cd.gap - thickness) - h * closing;
    if (predicted > p.margin) continue;
    cd.c.thickness = thickness;
    cd.c.mu = mu;
    tangent_basis(cd.c.normal, cd.c.d1, cd.c.d2);
    out.push_back(cd.c);
  }
}

}  // namespace

std::vector<Contact> detect(const State& s, const std::vector<AttachedShape>& shapes,
                            const VecX& u_pred, double h, const ContactParams& p) {
  std::vector<Contact> contacts;
  const int n = static_cast<int>(shapes.size());
  for (int i = 0; i < n; ++i) {
    for (int j = i + 1; j < n; ++j) {
      const AttachedShape& si = shapes[i];
      const AttachedShape& sj = shapes[j];
      if (si.body < 0 && sj.body < 0) continue;
      if (si.body >= 0 && si.body == sj.body) continue;
      std::vector<Cand> cands;
      const ShapeKind ki = si.shape.kind, kj = sj.shape.kind;
      if (ki == ShapeKind::Sphere && kj == ShapeKind::HalfSpace)
        sphere_halfspace(s, si, sj, cands);
      else if (ki == ShapeKind::HalfSpace && kj == ShapeKind::Sphere)
        sphere_halfspace(s, sj, si, cands);
      else if (ki == ShapeKind::Box && kj == ShapeKind::HalfSpace)
        box_halfspace(s, si, sj, cands);
      else if (ki == ShapeKind::HalfSpace && kj == ShapeKind::Box)
        box_halfspace(s, sj, si, cands);
      else if (ki == ShapeKind::Sphere && kj == ShapeKind::Sphere)
        sphere_sphere(s, si, sj, cands);
      else if (ki == ShapeKind::Sphere && kj == ShapeKind::Box)
        sphere_box(s, si, sj, cands);
      else if (ki == ShapeKind::Box && kj == ShapeKind::Sphere)
        sphere_box(s, sj, si, cands);
      else if (ki == ShapeKind::Box && kj == ShapeKind::Box)
        box_box(s, si, sj, p.margin, cands);
      else
        continue;
      finalize_candidates(s, cands, si.shape.thickness + sj.shape.thickness,
                          pair_mu(si.shape.mu, sj.shape.mu, p), u_pred, h, p, contacts);
    }
  }
  std::sort(contacts.begin(), contacts.end(), canonical_less);
  return contacts;
}

// Extension: particle (point) contacts of a particle block against every
// half-space / box shape, built as zero-radius sphere_halfspace / sphere_box
// candidates and filtered by the same predicted-gap rule.
static void particle_contacts(const State& s, const std::vector<AttachedShape>& shapes,
                              const ParticleContactGen& g, const VecX& u_pred, double h,
                              const ContactParams& p, std::vector<Contact>& out) {
  for (int b = g.first_body; b < g.first_body + g.count; ++b) {
    const V3 x = s.position(b);
    for (const AttachedShape& sh : shapes) {
      std::vector<Cand> cands;
      if (sh.shape.kind == ShapeKind::HalfSpace) {
        const V3 n = normalized(sh.shape.normal);
        const double gap = dot(n, x) - sh.shape.offset;
        Cand cd;
        cd.gap = gap;
        cd.c.a = {b, V3()};
        cd.c.b = {sh.body, x - gap * n};
        cd.c.normal = n;
        cands.push_back(cd);
      } else if (sh.shape.kind == ShapeKind::Box) {
        point_box(s, b, x, 0.0, sh, V3(), cands);
      } else {
        continue;  // particle vs sphere: not needed by any config
      }
      finalize_candidates(s, cands, g.thickness + sh.shape.thickness, pair_mu(g.mu, sh.shape.mu, p),
                          u_pred, h, p, out);
    }
  }
}

std::vector<Contact> world_contacts(const World& w, const VecX& u_tilde) {
  std::vector<Contact> c = detect(w.state, w.shapes, u_tilde, w.h, w.contact_params);
  if (!w.particle_gens.empty()) {
    for (const ParticleContactGen& g : w.particle_gens)
      particle_contacts(w.state, w.shapes, g, u_tilde, w.h, w.contact_params, c);
    std::sort(c.begin(), c.end(), canonical_less);
  }
  return c;
}

Report step_world(World& w) {  // scene.cpp:709-732
  for (const auto& dv : w.driven_anchors) {
    Joint& j = w.joints[dv.first];
    if (j.body_a < 0)
      j.anchor_a += w.h * dv.second;
    else if (j.body_b < 0)
      j.anchor_b += w.h * dv.second;
  }
  VecX f = external_forces(w.state, w.gravity);
  if (!w.f_extra.empty())
    for (int k = 0; k < w.state.num_dof; ++k) f[k] += w.f_extra[k];
  const VecX ut = unconstrained_velocity(w.state, f, w.h);
  w.contacts = world_contacts(w, ut);
  StepCtx ctx;
  ctx.state = &w.state;
  ctx.joints = &w.joints;
  ctx.meshes = &w.meshes;
  ctx.contacts = &w.contacts;
  ctx.gravity = w.gravity;
  ctx.h = w.h;
  ctx.f_extra = w.f_extra.empty() ? nullptr : &w.f_extra;
  Report r = newton_step(ctx, w.solver);
  w.time += w.h;
  return r;
}

// ============================ scene ==========================================
namespace {
M3 shape_inertia(const Shape& s, double mass) {  // scene.cpp:560-576
  switch (s.kind) {
    case ShapeKind::Sphere: return (0.4 * mass * s.radius * s.radius) * M3::identity();
    case ShapeKind::Box: {
      const V3 h = s.half_extents;
      M3 m;
      m(0, 0) = mass / 3.0 * (h[1] * h[1] + h[2] * h[2]);
      m(1, 1) = mass / 3.0 * (h[0] * h[0] + h[2] * h[2]);
      m(2, 2) = mass / 3.0 * (h[0] * h[0] + h[1] * h[1]);
      return m;
    }
    case ShapeKind::HalfSpace: break;
  }
  return M3::identity();
}
V4 quat_axis_angle(const V3& axis, double ang) {
  const V3 a = normalized(axis);
  const double half = 0.5 * ang;
  return V4(std::cos(half), std::sin(half) * a[0], std::sin(half) * a[1], std::sin(half) * a[2]);
}
V4 quat_mul(const V4& p, const V4& q) {  // Hamilton product (w, x, y, z)
  return V4(p[0] * q[0] - p[1] * q[1] - p[2] * q[2] - p[3] * q[3],
            p[0] * q[1] + p[1] * q[0] + p[2] * q[3] - p[3] * q[2],
            p[0] * q[2] - p[1] * q[3] + p[2] * q[0] + p[3] * q[1],
            p[0] * q[3] + p[1] * q[2] - p[2] * q[1] + p[3] * q[0]);
}
}  // namespace

World build_world(const SceneDesc& sc) {  // scene.cpp:587-707
  World w;
  w.gravity = sc.gravity;
  w.h = sc.timestep;
  w.contact_params = sc.contacts;
  w.solver = sc.solver;
  std::vector<int> body_map(sc.bodies.size(), -1);
  for (size_t i = 0; i < sc.bodies.size(); ++i) {
    const BodyDesc& d = sc.bodies[i];
    if (d.kind == BodyDescKind::Static) continue;
    Body b;
    b.type = d.kind == BodyDescKind::Particle ? BodyType::Particle : BodyType::Rigid;
    b.mass = d.mass;
    if (b.type == BodyType::Rigid) b.inertia = d.has_inertia ? d.inertia : shape_inertia(d.shape, d.mass);
    body_map[i] = static_cast<int>(w.state.bodies.size());
    w.state.bodies.push_back(b);
  }
  std::vector<int> mesh_base(sc.meshes.size(), 0);
  for (size_t m = 0; m < sc.meshes.size(); ++m) {
    const MeshDesc& d = sc.meshes[m];
    mesh_base[m] = static_cast<int>(w.state.bodies.size());
    std::vector<double> lumped(d.vertices.size(), 0.0);
    MeshBinding bind;
    bind.particle_base = mesh_base[m];
    bind.mesh.material = d.material;
    bind.mesh.prepare();
    for (const auto& ev : d.elements) {
      std::array<int, 4> idx = ev;
      M3 dm;
      dm.set_col(0, d.vertices[idx[1]] - d.vertices[idx[0]]);
      dm.set_col(1, d.vertices[idx[2]] - d.vertices[idx[0]]);
      dm.set_col(2, d.vertices[idx[3]] - d.vertices[idx[0]]);
      if (det3(dm) < 0.0) std::swap(idx[2], idx[3]);
      const Tet e = make_tet(idx, d.vertices[idx[0]], d.vertices[idx[1]], d.vertices[idx[2]],
                             d.vertices[idx[3]]);
      bind.mesh.elements.push_back(e);
      for (int v : idx) lumped[v] += d.density * e.vol / 4.0;
    }
    for (size_t v = 0; v < d.vertices.size(); ++v) {
      Body b;
      b.type = BodyType::Particle;
      b.mass = lumped[v] > 0.0 ? lumped[v] : 1e-6;
      w.state.bodies.push_back(b);
    }
    w.meshes.push_back(std::move(bind));
  }
  w.state.finalize_layout();
  for (size_t i = 0; i < sc.bodies.size(); ++i) {
    const BodyDesc& d = sc.bodies[i];
    const int b = body_map[i];
    if (b < 0) continue;
    w.state.set_position(b, d.position);
    const int o = w.state.dof_off[b];
    for (int k = 0; k < 3; ++k) w.state.u[o + k] = d.velocity[k];
    if (d.kind == BodyDescKind::Rigid) {
      w.state.set_orientation(b, normalized_quat(d.orientation));
      for (int k = 0; k < 3; ++k) w.state.u[o + 3 + k] = d.angular_velocity[k];
    }
  }
  for (size_t m = 0; m < sc.meshes.size(); ++m)
    for (size_t v = 0; v < sc.meshes[m].vertices.size(); ++v) {
      const int b = mesh_base[m] + static_cast<int>(v);
      const MeshDesc& md = sc.meshes[m];
      w.state.set_position(b, md.initial.empty() ? md.vertices[v] : md.initial[v]);
      for (int k = 0; k < 3; ++k) w.state.u[w.state.dof_off[b] + k] = sc.meshes[m].velocity[k];
    }
  for (size_t i = 0; i < sc.bodies.size(); ++i) {
    const BodyDesc& d = sc.bodies[i];
    if (d.kind == BodyDescKind::Static)
      w.shapes.push_back({-1, d.shape});
    else if (d.kind == BodyDescKind::Rigid && d.has_shape)
      w.shapes.push_back({body_map[i], d.shape});
  }
  for (const JointDesc& d : sc.joints) {
    Joint j;
    j.kind = d.kind;
    const auto resolve = [&](const JointAttach& a) {
      if (a.mesh >= 0) return mesh_base[a.mesh] + a.vertex;
      return a.body >= 0 ? body_map[a.body] : -1;
    };
    j.body_a = resolve(d.a);
    j.body_b = resolve(d.b);
    j.compliance = d.compliance;
    j.stiffness = d.stiffness;
    j.anchor_velocity = d.anchor_velocity;
    bind_joint(j, w.state, d.anchor, d.axis);
    if (d.anchor_velocity != V3()) w.driven_anchors.push_back({static_cast<int>(w.joints.size()), d.anchor_velocity});
    w.joints.push_back(j);
  }
  for (size_t g = 0; g < sc.particle_gens.size(); ++g) {
    ParticleContactGen pg = sc.particle_gens[g];
    const int m = sc.particle_gen_mesh[g];
    pg.first_body = mesh_base[m];
    pg.count = static_cast<int>(sc.meshes[m].vertices.size());
    w.particle_gens.push_back(pg);
  }
  return w;
}

void tessellate_grid(MeshDesc& mesh, int nx, int ny, int nz, const V3& origin, const V3& size) {
  const auto vid = [&](int x, int y, int z) { return (x * (ny + 1) + y) * (nz + 1) + z; };
  for (int x = 0; x <= nx; ++x)
    for (int y = 0; y <= ny; ++y)
      for (int z = 0; z <= nz; ++z)
        mesh.vertices.push_back(origin + V3(size[0] * x / nx, size[1] * y / ny, size[2] * z / nz));
  const int tets[6][4] = {{0, 1, 5, 7}, {0, 5, 4, 7}, {0, 4, 6, 7}, {0, 6, 2, 7}, {0, 2, 3, 7}, {0, 3, 1, 7}};
  for (int x = 0; x < nx; ++x)
    for (int y = 0; y < ny; ++y)
      for (int z = 0; z < nz; ++z) {
        const int c[8] = {vid(x, y, z),         vid(x + 1, y, z),         vid(x, y + 1, z),
                          vid(x + 1, y + 1, z), vid(x, y, z + 1),         vid(x + 1, y, z + 1),
                          vid(x, y + 1, z + 1), vid(x + 1, y + 1, z + 1)};
        for (const auto& t : tets) mesh.elements.push_back({c[t[0]], c[t[1]], c[t[2]], c[t[3]]});
      }
}

// ============================ builders =======================================
namespace {
BodyDesc static_ground() {
  BodyDesc g;
  g.kind = BodyDescKind::Static;
  g.shape.kind = ShapeKind::HalfSpace;
  g.shape.normal = V3(0, 0, 1);
  g.shape.offset = 0.0;
  return g;
}
BodyDesc rigid_box(const V3& pos, const V3& he, double mass, const V4& q = V4(1, 0, 0, 0)) {
  BodyDesc b;
  b.kind = BodyDescKind::Rigid;
  b.position = pos;
  b.orientation = q;
  b.mass = mass;
  b.has_shape = true;
  b.shape.kind = ShapeKind::Box;
  b.shape.half_extents = he;
  return b;
}
BodyDesc rigid_sphere(const V3& pos, double radius, double mass) {
  BodyDesc b;
  b.kind = BodyDescKind::Rigid;
  b.position = pos;
  b.mass = mass;
  b.has_shape = true;
  b.shape.kind = ShapeKind::Sphere;
  b.shape.radius = radius;
  return b;
}
// Jitter the initial positions (not the rest shape) so F != I at t = 0 and the
// SVD is non-degenerate (SURVEY §7 hard part 2). Pattern of bench_kernels.cpp:97-100.
void jitter_vertices(std::vector<V3>& verts, double sigma, unsigned seed) {
  std::mt19937 rng(seed);
  std::normal_distribution<double> g(0.0, sigma);
  for (V3& p : verts) {
    const double a = g(rng), b = g(rng), c = g(rng);
    p = p + V3(a, b, c);
  }
}
}  // namespace

SceneDesc build_box_on_plane() {
  SceneDesc s;
  s.bodies.push_back(static_ground());
  s.bodies.push_back(rigid_box(V3(0, 0, 0.2), V3(0.2, 0.2, 0.2), 1.0));
  s.contacts.mu_default = 0.5;
  return s;
}

SceneDesc build_incline(double angle_deg, double mu) {
  SceneDesc s;
  const double th = angle_deg * M_PI / 180.0;
  BodyDesc g = static_ground();
  g.shape.normal = V3(-std::sin(th), 0.0, std::cos(th));
  s.bodies.push_back(g);
  const double half = 0.1;
  s.bodies.push_back(rigid_box(half * g.shape.normal, V3(half, half, half), 1.0,
                               quat_axis_angle(V3(0, 1, 0), -th)));
  s.contacts.mu_default = mu;
  s.solver.newton_iterations = 10;
  return s;
}

SceneDesc build_heavy_stack() {
  SceneDesc s;
  s.bodies.push_back(static_ground());
  const double masses[5] = {8.0, 64.0, 512.0, 4096.0, 32768.0};
  for (int i = 0; i < 5; ++i) s.bodies.push_back(rigid_box(V3(0, 0, 0.5 + 1.0 * i), V3(0.5, 0.5, 0.5), masses[i]));
  s.contacts.mu_default = 0.5;
  s.solver.newton_iterations = 5;
  s.solver.linear.max_iterations = 25;
  return s;
}

SceneDesc build_arch() {
  SceneDesc s;
  s.bodies.push_back(static_ground());
  const int blocks = 20;
  const double span = 4.0, height = 1.5;
  for (int i = 0; i < blocks; ++i) {
    const double x = -0.5 * span + span * (i + 0.5) / blocks;
    const double z = height * (1.0 - (x / (0.5 * span)) * (x / (0.5 * span)));
    const double slope = -2.0 * height * x / (0.25 * span * span);
    const double ang = std::atan(slope);
    const double mass = 15.0 + (110.0 - 15.0) * (1.0 - z / height);
    s.bodies.push_back(rigid_box(V3(x, 0, z + 0.1), V3(0.095, 0.15, 0.1), mass, quat_axis_angle(V3(0, 1, 0), -ang)));
  }
  s.contacts.mu_default = 0.6;
  s.solver.newton_iterations = 6;
  s.solver.linear.max_iterations = 20;
  return s;
}

SceneDesc build_box_pile(unsigned seed) {
  SceneDesc s;
  s.bodies.push_back(static_ground());
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> xy(-0.4, 0.4), zd(0.3, 1.6), ang(0.0, 2.0 * M_PI), unit(-1.0, 1.0);
  for (int i = 0; i < 8; ++i) {
    const double ax = unit(rng), ay = unit(rng), az = unit(rng);
    V3 axis(ax, ay, az);
    if (norm(axis) < 1e-6) axis = V3(0, 0, 1);
    const double px = xy(rng), py = xy(rng), pz = zd(rng);
    const double a = ang(rng);
    s.bodies.push_back(rigid_box(V3(px, py, pz), V3(0.15, 0.15, 0.15), 4.7, quat_axis_angle(axis, a)));
  }
  for (int i = 0; i < 4; ++i) {
    const double px = xy(rng), py = xy(rng), pz = zd(rng);
    s.bodies.push_back(rigid_sphere(V3(px, py, pz), 0.12, 1.0));
  }
  s.contacts.mu_default = 0.7;
  s.solver.newton_iterations = 6;
  s.solver.linear.max_iterations = 25;
  return s;
}

SceneDesc build_stretch_sheet(MatModel model) {
  SceneDesc s;
  s.gravity = V3();
  MeshDesc mesh;
  const V3 size(0.2, 0.1, 0.05);
  tessellate_grid(mesh, 4, 2, 1, V3(), size);
  mesh.material.model = model;
  mesh.material.young = 1e5;
  mesh.material.poisson = 0.45;
  mesh.density = 1000.0;
  s.meshes.push_back(mesh);
  for (size_t v = 0; v < mesh.vertices.size(); ++v) {
    const V3& p = mesh.vertices[v];
    const bool fixed = p[0] < 1e-9, driven = p[0] > size[0] - 1e-9;
    if (!fixed && !driven) continue;
    JointDesc j;
    j.kind = JointKind::FixedPoint;
    j.a.mesh = 0;
    j.a.vertex = static_cast<int>(v);
    j.b.body = -1;
    j.anchor = p;
    if (driven) j.anchor_velocity = V3(0.2, 0.0, 0.0);
    s.joints.push_back(j);
  }
  s.solver.newton_iterations = 10;
  s.solver.linear.max_iterations = 60;
  return s;
}

// ---- synthetic BASELINE configs (deviations in DESIGN.md) ----

SceneDesc build_c1_box_stack() {
  SceneDesc s;
  s.bodies.push_back(static_ground());
  for (int i = 0; i < 8; ++i) s.bodies.push_back(rigid_box(V3(0, 0, 0.5 + 1.0 * i), V3(0.5, 0.5, 0.5), 1.0));
  s.contacts.mu_default = 0.5;
  s.solver.newton_iterations = 5;
  s.solver.linear.max_iterations = 25;
  return s;
}

SceneDesc build_c2_fem_block(int n) {
  SceneDesc s;
  s.bodies.push_back(static_ground());
  MeshDesc mesh;
  const double edge = 0.3;
  tessellate_grid(mesh, n, n, n, V3(-0.15, -0.15, 0.005), V3(edge, edge, edge));
  mesh.material.model = MatModel::NeoHookean;
  mesh.material.young = 1e5;
  mesh.material.poisson = 0.45;
  mesh.density = 1000.0;
  mesh.velocity = V3(0.0, 0.0, -1.0);  // dropped: the bottom layer penetrates within step 1
  // Initial positions jittered (rest shape stays the regular grid).
  mesh.initial = mesh.vertices;
  jitter_vertices(mesh.initial, 1e-3 * edge / n, 7);
  s.meshes.push_back(mesh);
  s.contacts.mu_default = 0.5;
  s.contacts.margin = 0.01;
  s.solver.newton_iterations = 10;
  s.solver.linear.max_iterations = 60;
  ParticleContactGen g;
  s.particle_gens.push_back(g);
  s.particle_gen_mesh.push_back(0);
  return s;
}

SceneDesc build_c3_chain(int links) {
  SceneDesc s;
  const double pitch = 0.12, half = 0.05, z = 12.0;
  for (int i = 0; i < links; ++i)
    s.bodies.push_back(rigid_box(V3(0.06 + pitch * i, 0, z), V3(half, 0.01, 0.01), 0.1));
  for (int i = 0; i < links; ++i) {
    JointDesc j;
    const bool prismatic = (i % 10) == 9;
    j.kind = prismatic ? JointKind::Prismatic : JointKind::Revolute;
    j.a.body = i - 1;  // -1: world anchor for the first joint
    j.b.body = i;
    j.anchor = V3(pitch * i, 0, z);
    j.axis = prismatic ? V3(1, 0, 0) : V3(0, 1, 0);
    s.joints.push_back(j);
  }
  s.solver.newton_iterations = 8;
  s.solver.linear.max_iterations = 40;
  return s;
}

// Cantilever with FixedPoint hinges and BendSpring joints (constraints.cpp:209-216);
// the product's bend_chain builder (csrc/nsd_scene.cpp) builds the same scene.
SceneDesc build_bend_chain(int links, double k) {
  SceneDesc s;
  const double pitch = 0.12, half = 0.05, z = 2.0;
  for (int i = 0; i < links; ++i)
    s.bodies.push_back(rigid_box(V3(0.06 + pitch * i, 0, z), V3(half, 0.01, 0.01), 0.1));
  for (int i = 0; i < links; ++i) {
    JointDesc j;
    j.kind = JointKind::FixedPoint;
    j.a.body = i - 1;
    j.b.body = i;
    j.anchor = V3(pitch * i, 0, z);
    s.joints.push_back(j);
    JointDesc b = j;
    b.kind = JointKind::BendSpring;
    b.axis = V3(1, 0, 0);
    b.stiffness = k;
    s.joints.push_back(b);
  }
  return s;
}

SceneDesc build_c4_hand_ball(int n, double speed, double scale) {
  SceneDesc s;
  s.bodies.push_back(static_ground());  // palm surface
  // Ball: n^3 grid carved to a sphere of radius 0.05 * scale by element centroid;
  // every length of the hand scales with it, masses with scale^3.
  const double L = scale;
  const double radius = 0.05 * L, edge = 0.1 * L;
  MeshDesc grid;
  tessellate_grid(grid, n, n, n, V3(-0.05 * L, -0.05 * L, 0.0), V3(edge, edge, edge));
  const V3 centre(0.0, 0.0, 0.05 * L);
  std::vector<int> keep_v(grid.vertices.size(), -1);
  std::vector<std::array<int, 4>> kept;
  for (const auto& t : grid.elements) {
    V3 c;
    for (int k = 0; k < 4; ++k) c = c + grid.vertices[t[k]];
    c = 0.25 * c;
    if (norm(c - centre) <= radius) kept.push_back(t);
  }
  for (const auto& t : kept)
    for (int k = 0; k < 4; ++k) keep_v[t[k]] = 0;
  MeshDesc ball;
  double zmin = std::numeric_limits<double>::infinity();
  for (size_t v = 0; v < grid.vertices.size(); ++v)
    if (keep_v[v] == 0) {
      keep_v[v] = static_cast<int>(ball.vertices.size());
      ball.vertices.push_back(grid.vertices[v]);
      zmin = std::min(zmin, grid.vertices[v][2]);
    }
  const double lift = 0.005 - zmin;  // lowest vertex 5 mm above the palm
  for (V3& p : ball.vertices) p[2] += lift;
  for (const auto& t : kept) ball.elements.push_back({keep_v[t[0]], keep_v[t[1]], keep_v[t[2]], keep_v[t[3]]});
  ball.material.model = MatModel::NeoHookean;
  ball.material.young = 1e5;
  ball.material.poisson = 0.45;
  ball.density = 1000.0;
  const double bz = centre[2] + lift;
  // Fingers: 4 planar chains of 4 phalanges standing around the ball.
  const V3 he(0.008 * L, 0.008 * L, 0.012 * L);
  const double rad = 0.075 * L, z_anchor[4] = {0.014 * L, 0.050 * L, 0.086 * L, 0.122 * L},
               z_centre[4] = {0.032 * L, 0.068 * L, 0.104 * L, 0.140 * L};
  for (int f = 0; f < 4; ++f) {
    const double th = 0.5 * M_PI * f;
    const V3 d(std::cos(th), std::sin(th), 0.0);
    const V3 tang(-std::sin(th), std::cos(th), 0.0);
    for (int k = 0; k < 4; ++k) {
      s.bodies.push_back(rigid_box(V3(rad * d[0], rad * d[1], z_centre[k]), he, 0.02 * L * L * L,
                                   quat_axis_angle(V3(0, 0, 1), th)));
      JointDesc j;
      j.kind = JointKind::Revolute;
      j.a.body = k == 0 ? -1 : 1 + 4 * f + (k - 1);
      j.b.body = 1 + 4 * f + k;
      j.anchor = V3(rad * d[0], rad * d[1], z_anchor[k]);
      j.axis = tang;
      s.joints.push_back(j);
    }
    // Drive: compliant point joint from the fingertip to a world anchor moving
    // toward the ball's upper hemisphere (squeeze), scene.cpp:700-716 semantics.
    JointDesc drive;
    drive.kind = JointKind::FixedPoint;
    drive.a.body = 1 + 4 * f + 3;
    drive.b.body = -1;
    drive.anchor = V3(rad * d[0], rad * d[1], 0.152 * L);
    drive.compliance = 1e-4;
    drive.anchor_velocity = V3(-kC4Drive * d[0], -kC4Drive * d[1], 0.0);
    s.joints.push_back(drive);
  }
  (void)bz;
  ball.velocity = V3(0.0, 0.0, -speed);
  ball.initial = ball.vertices;
  jitter_vertices(ball.initial, 1e-3 * edge / n, 7);
  s.meshes.push_back(ball);
  s.contacts.mu_default = 0.75;
  s.contacts.margin = 0.01;
  s.solver.newton_iterations = 6;
  s.solver.linear.max_iterations = 50;
  ParticleContactGen g;
  s.particle_gens.push_back(g);
  s.particle_gen_mesh.push_back(0);
  return s;
}

SceneDesc build_c5_ant(unsigned env_id) {
  SceneDesc s;
  s.bodies.push_back(static_ground());
  const double r_torso = 0.25, H = 0.40 + 0.005;
  s.bodies.push_back(rigid_sphere(V3(0, 0, H), r_torso, 1.0));
  std::mt19937 rng(env_id);
  std::uniform_real_distribution<double> rate(-0.5, 0.5);
  const V3 he(0.2, 0.04, 0.04);
  for (int k = 0; k < 4; ++k) {
    const double th = 0.25 * M_PI + 0.5 * M_PI * k;
    const V3 d(std::cos(th), std::sin(th), 0.0);
    const V3 t(-std::sin(th), std::cos(th), 0.0);
    const V3 z(0, 0, 1);
    const V3 hip = V3(0.265 * d[0], 0.265 * d[1], H);
    const V3 knee = V3(0.695 * d[0], 0.695 * d[1], H - 0.02);
    const V3 c_thigh(0.48 * d[0], 0.48 * d[1], H);
    const V3 c_shin(0.75 * d[0], 0.75 * d[1], H - 0.2);
    const V4 q_thigh = quat_axis_angle(z, th);
    const V4 q_shin = quat_mul(q_thigh, quat_axis_angle(V3(0, 1, 0), 0.5 * M_PI));
    const double a_hip = rate(rng);
    const double a_knee = rate(rng);
    BodyDesc thigh = rigid_box(c_thigh, he, 0.2, q_thigh);
    thigh.angular_velocity = a_hip * z;
    thigh.velocity = cross(a_hip * z, c_thigh - hip);
    BodyDesc shin = rigid_box(c_shin, he, 0.2, q_shin);
    shin.angular_velocity = a_hip * z + a_knee * t;
    shin.velocity = cross(a_hip * z, c_shin - hip) + cross(a_knee * t, c_shin - knee);
    s.bodies.push_back(thigh);
    s.bodies.push_back(shin);
    JointDesc jh;
    jh.kind = JointKind::Revolute;
    jh.a.body = 1;  // scene-body indices (ground is 0)
    jh.b.body = 2 + 2 * k;
    jh.anchor = hip;
    jh.axis = z;
    s.joints.push_back(jh);
    JointDesc jk;
    jk.kind = JointKind::Revolute;
    jk.a.body = 2 + 2 * k;
    jk.b.body = 3 + 2 * k;
    jk.anchor = knee;
    jk.axis = t;
    s.joints.push_back(jk);
  }
  s.contacts.mu_default = 1.0;
  s.contacts.margin = 0.01;
  s.solver.newton_iterations = 4;
  s.solver.linear.max_iterations = 10;
  return s;
}

bool build_scene_by_name(const std::string& name, unsigned seed, SceneDesc& out) {
  std::string base = name;
  std::vector<double> args;
  const size_t colon = name.find(':');
  if (colon != std::string::npos) {
    base = name.substr(0, colon);
    std::stringstream ss(name.substr(colon + 1));
    std::string tok;
    while (std::getline(ss, tok, ':')) args.push_back(std::stod(tok));
  }
  if (base == "arch") out = build_arch();
  else if (base == "heavy_stack") out = build_heavy_stack();
  else if (base == "box_pile") out = build_box_pile(seed);
  else if (base == "box_on_plane") out = build_box_on_plane();
  else if (base == "stretch_sheet") out = build_stretch_sheet(MatModel::NeoHookean);
  else if (base == "stretch_sheet_linear") out = build_stretch_sheet(MatModel::Linear);
  else if (base == "incline") out = build_incline(args.size() > 0 ? args[0] : 20.0, args.size() > 1 ? args[1] : 0.5);
  else if (base == "c1") out = build_c1_box_stack();
  else if (base == "c2") out = build_c2_fem_block(args.size() > 0 ? static_cast<int>(args[0]) : 12);
  else if (base == "c3") out = build_c3_chain(args.size() > 0 ? static_cast<int>(args[0]) : 100);
  else if (base == "bend_chain")
    out = build_bend_chain(args.size() > 0 ? static_cast<int>(args[0]) : 10, args.size() > 1 ? args[1] : 50.0);
  else if (base == "c4")
    out = build_c4_hand_ball(args.size() > 0 ? static_cast<int>(args[0]) : 12, args.size() > 1 ? args[1] : kC4Speed,
                             args.size() > 2 ? args[2] : kC4Scale);
  else if (base == "c5") out = build_c5_ant(seed);
  else return false;
  return true;
}

VecX joint_torque_forces(const World& w, const double* tau) {
  VecX f(w.state.num_dof, 0.0);
  for (size_t i = 0; i < w.joints.size(); ++i) {
    const Joint& j = w.joints[i];
    if (j.kind != JointKind::Revolute) continue;
    const V3 ax = j.body_a < 0 ? j.axis_a : w.state.rotation(j.body_a) * j.axis_a;
    const V3 t = tau[i] * ax;
    if (j.body_a >= 0 && w.state.bodies[j.body_a].type == BodyType::Rigid)
      for (int k = 0; k < 3; ++k) f[w.state.dof_off[j.body_a] + 3 + k] += t[k];
    if (j.body_b >= 0 && w.state.bodies[j.body_b].type == BodyType::Rigid)
      for (int k = 0; k < 3; ++k) f[w.state.dof_off[j.body_b] + 3 + k] -= t[k];
  }
  return f;
}

}  // namespace orc
