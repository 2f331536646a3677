// Product scene layer: builders + build_world in the flat C-ABI layout.
// Reference: src/scene.cpp:556-935 (build_world, builders, tessellate_grid),
// src/constraints.cpp:222-263 (bind_joint), src/materials.cpp:8-43
// (make_tet_element, lame_from_young_poisson). The BASELINE configs C1-C5
// follow SURVEY.md Appendix C with the deviations recorded in DESIGN.md.
#include "nsd_scene.h"

#include "nsd_collide.cuh"
#include "nsd_math.cuh"

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <random>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <unistd.h>
#include <sstream>
#include <stdexcept>

namespace nsdw {
namespace {

using V = nsd::V3<double>;
using M = nsd::M3<double>;

V cv(const Vec3& a) { return nsd::v3(a.x, a.y, a.z); }
Vec3 vc(const V& a) { return Vec3{a.x, a.y, a.z}; }

Quat axis_angle(const Vec3& axis, double ang) {
  const V a = nsd::normalize(cv(axis));
  const double half = 0.5 * ang;
  return Quat{std::cos(half), std::sin(half) * a.x, std::sin(half) * a.y, std::sin(half) * a.z};
}
Quat qmul(const Quat& p, const Quat& q) {
  return Quat{p.w * q.w - p.x * q.x - p.y * q.y - p.z * q.z, p.w * q.x + p.x * q.w + p.y * q.z - p.z * q.y,
              p.w * q.y - p.x * q.z + p.y * q.w + p.z * q.x, p.w * q.z + p.x * q.y - p.y * q.x + p.z * q.w};
}

BodySpec ground() {
  BodySpec g;
  g.kind = BodyKind::Static;
  g.has_shape = true;
  g.shape.kind = 0;
  g.shape.normal = Vec3{0, 0, 1};
  return g;
}
BodySpec box(const Vec3& p, const Vec3& he, double mass, const Quat& r = Quat{}) {
  BodySpec b;
  b.pos = p;
  b.rot = r;
  b.mass = mass;
  b.has_shape = true;
  b.shape.kind = 2;
  b.shape.half = he;
  return b;
}
BodySpec sphere(const Vec3& p, double radius, double mass) {
  BodySpec b;
  b.pos = p;
  b.mass = mass;
  b.has_shape = true;
  b.shape.kind = 1;
  b.shape.radius = radius;
  return b;
}

void grid(MeshSpec& m, int nx, int ny, int nz, const Vec3& o, const Vec3& sz) {
  auto vid = [&](int x, int y, int z) { return (x * (ny + 1) + y) * (nz + 1) + z; };
  for (int x = 0; x <= nx; ++x)
    for (int y = 0; y <= ny; ++y)
      for (int z = 0; z <= nz; ++z)
        m.vertices.push_back(Vec3{o.x + sz.x * x / nx, o.y + sz.y * y / ny, o.z + sz.z * z / nz});
  static const int T6[6][4] = {{0, 1, 5, 7}, {0, 5, 4, 7}, {0, 4, 6, 7}, {0, 6, 2, 7}, {0, 2, 3, 7}, {0, 3, 1, 7}};
  for (int x = 0; x < nx; ++x)
    for (int y = 0; y < ny; ++y)
      for (int z = 0; z < nz; ++z) {
        const int c[8] = {vid(x, y, z),         vid(x + 1, y, z),         vid(x, y + 1, z),
                          vid(x + 1, y + 1, z), vid(x, y, z + 1),         vid(x + 1, y, z + 1),
                          vid(x, y + 1, z + 1), vid(x + 1, y + 1, z + 1)};
        for (const auto& t : T6) m.elements.push_back({c[t[0]], c[t[1]], c[t[2]], c[t[3]]});
      }
}

void jitter(std::vector<Vec3>& vs, double sigma, unsigned seed) {
  std::mt19937 rng(seed);
  std::normal_distribution<double> g(0.0, sigma);
  for (Vec3& p : vs) {
    const double a = g(rng), b = g(rng), c = g(rng);
    p = Vec3{p.x + a, p.y + b, p.z + c};
  }
}

nsd_config defaults() {
  nsd_config c;
  nsd_config_default(&c, NSD_FP64);
  return c;
}

Scene s_box_on_plane() {
  Scene s;
  s.solver = defaults();
  s.bodies.push_back(ground());
  s.bodies.push_back(box(Vec3{0, 0, 0.2}, Vec3{0.2, 0.2, 0.2}, 1.0));
  s.mu_default = 0.5;
  return s;
}
Scene s_incline(double deg, double mu) {
  Scene s;
  s.solver = defaults();
  const double th = deg * M_PI / 180.0;
  BodySpec g = ground();
  g.shape.normal = Vec3{-std::sin(th), 0.0, std::cos(th)};
  s.bodies.push_back(g);
  const double half = 0.1;
  const Vec3 n = g.shape.normal;
  s.bodies.push_back(box(Vec3{half * n.x, half * n.y, half * n.z}, Vec3{half, half, half}, 1.0,
                         axis_angle(Vec3{0, 1, 0}, -th)));
  s.mu_default = mu;
  s.solver.newton_iterations = 10;
  return s;
}
Scene s_heavy_stack() {
  Scene s;
  s.solver = defaults();
  s.bodies.push_back(ground());
  const double m[5] = {8.0, 64.0, 512.0, 4096.0, 32768.0};
  for (int i = 0; i < 5; ++i) s.bodies.push_back(box(Vec3{0, 0, 0.5 + 1.0 * i}, Vec3{0.5, 0.5, 0.5}, m[i]));
  s.mu_default = 0.5;
  s.solver.newton_iterations = 5;
  s.solver.linear_max_iterations = 25;
  return s;
}
Scene s_arch() {
  Scene s;
  s.solver = defaults();
  s.bodies.push_back(ground());
  const int blocks = 20;
  const double span = 4.0, height = 1.5;
  for (int i = 0; i < blocks; ++i) {
    const double x = -0.5 * span + span * (i + 0.5) / blocks;
    const double z = height * (1.0 - (x / (0.5 * span)) * (x / (0.5 * span)));
    const double slope = -2.0 * height * x / (0.25 * span * span);
    const double ang = std::atan(slope);
    const double mass = 15.0 + (110.0 - 15.0) * (1.0 - z / height);
    s.bodies.push_back(box(Vec3{x, 0, z + 0.1}, Vec3{0.095, 0.15, 0.1}, mass, axis_angle(Vec3{0, 1, 0}, -ang)));
  }
  s.mu_default = 0.6;
  s.solver.newton_iterations = 6;
  s.solver.linear_max_iterations = 20;
  return s;
}
Scene s_box_pile(unsigned seed) {
  Scene s;
  s.solver = defaults();
  s.bodies.push_back(ground());
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> xy(-0.4, 0.4), zd(0.3, 1.6), ang(0.0, 2.0 * M_PI), unit(-1.0, 1.0);
  for (int i = 0; i < 8; ++i) {
    const double ax = unit(rng), ay = unit(rng), az = unit(rng);
    Vec3 axis{ax, ay, az};
    if (nsd::norm(cv(axis)) < 1e-6) axis = Vec3{0, 0, 1};
    const double px = xy(rng), py = xy(rng), pz = zd(rng);
    const double a = ang(rng);
    s.bodies.push_back(box(Vec3{px, py, pz}, Vec3{0.15, 0.15, 0.15}, 4.7, axis_angle(axis, a)));
  }
  for (int i = 0; i < 4; ++i) {
    const double px = xy(rng), py = xy(rng), pz = zd(rng);
    s.bodies.push_back(sphere(Vec3{px, py, pz}, 0.12, 1.0));
  }
  s.mu_default = 0.7;
  s.solver.newton_iterations = 6;
  s.solver.linear_max_iterations = 25;
  return s;
}
Scene s_stretch_sheet(bool linear) {  // scene.cpp:880-912 (Neo-Hookean or linear co-rotational)
  Scene s;
  s.solver = defaults();
  s.gravity = Vec3{0, 0, 0};
  MeshSpec m;
  m.linear = linear;
  const Vec3 size{0.2, 0.1, 0.05};
  grid(m, 4, 2, 1, Vec3{0, 0, 0}, size);
  s.meshes.push_back(m);
  for (size_t v = 0; v < m.vertices.size(); ++v) {
    const Vec3& p = m.vertices[v];
    const bool fixed = p.x < 1e-9, driven = p.x > size.x - 1e-9;
    if (!fixed && !driven) continue;
    JointSpecDesc j;
    j.kind = 0;
    j.a.mesh = 0;
    j.a.vertex = static_cast<int>(v);
    j.b.body = -1;
    j.anchor = p;
    if (driven) j.anchor_velocity = Vec3{0.2, 0.0, 0.0};
    s.joints.push_back(j);
  }
  s.solver.newton_iterations = 10;
  s.solver.linear_max_iterations = 60;
  return s;
}

// ---- BASELINE configs
Scene s_c1() {
  Scene s;
  s.solver = defaults();
  s.bodies.push_back(ground());
  for (int i = 0; i < 8; ++i) s.bodies.push_back(box(Vec3{0, 0, 0.5 + 1.0 * i}, Vec3{0.5, 0.5, 0.5}, 1.0));
  s.mu_default = 0.5;
  s.solver.newton_iterations = 5;
  s.solver.linear_max_iterations = 25;
  return s;
}
Scene s_c2(int n) {
  Scene s;
  s.solver = defaults();
  s.bodies.push_back(ground());
  MeshSpec m;
  const double edge = 0.3;
  grid(m, n, n, n, Vec3{-0.15, -0.15, 0.005}, Vec3{edge, edge, edge});
  m.velocity = Vec3{0.0, 0.0, -1.0};
  m.initial = m.vertices;
  jitter(m.initial, 1e-3 * edge / n, 7);
  m.particle_contacts = true;
  s.meshes.push_back(m);
  s.mu_default = 0.5;
  s.margin = 0.01;
  s.solver.newton_iterations = 10;
  s.solver.linear_max_iterations = 60;
  return s;
}
Scene s_c3(int links) {
  Scene s;
  s.solver = defaults();
  const double pitch = 0.12, half = 0.05, z = 12.0;
  for (int i = 0; i < links; ++i) s.bodies.push_back(box(Vec3{0.06 + pitch * i, 0, z}, Vec3{half, 0.01, 0.01}, 0.1));
  for (int i = 0; i < links; ++i) {
    JointSpecDesc j;
    const bool pri = (i % 10) == 9;
    j.kind = pri ? 2 : 1;
    j.a.body = i - 1;
    j.b.body = i;
    j.anchor = Vec3{pitch * i, 0, z};
    j.axis = pri ? Vec3{1, 0, 0} : Vec3{0, 1, 0};
    s.joints.push_back(j);
  }
  s.solver.newton_iterations = 8;
  s.solver.linear_max_iterations = 40;
  return s;
}
// A cantilever of `links` boxes along +x from a world anchor: a FixedPoint joint at
// every hinge and a BendSpring of stiffness k about the link axis (constraints.cpp:
// 209-216, compliance 1/k), sagging under gravity.
Scene s_bend_chain(int links, double k) {
  Scene s;
  s.solver = defaults();
  const double pitch = 0.12, half = 0.05, z = 2.0;
  for (int i = 0; i < links; ++i) s.bodies.push_back(box(Vec3{0.06 + pitch * i, 0, z}, Vec3{half, 0.01, 0.01}, 0.1));
  for (int i = 0; i < links; ++i) {
    JointSpecDesc j;
    j.kind = 0;
    j.a.body = i - 1;
    j.b.body = i;
    j.anchor = Vec3{pitch * i, 0, z};
    s.joints.push_back(j);
    JointSpecDesc bs = j;
    bs.kind = 3;
    bs.axis = Vec3{1, 0, 0};
    bs.stiffness = k;
    s.joints.push_back(bs);
  }
  return s;
}
Scene s_c4(int n, double speed, double L) {
  Scene s;
  s.solver = defaults();
  s.bodies.push_back(ground());
  const double radius = 0.05 * L, edge = 0.1 * L;  // every length scales with L, masses with L^3
  MeshSpec g;
  grid(g, n, n, n, Vec3{-0.05 * L, -0.05 * L, 0.0}, Vec3{edge, edge, edge});
  const V centre = nsd::v3(0.0, 0.0, 0.05 * L);
  std::vector<int> keep(g.vertices.size(), -1);
  std::vector<std::array<int, 4>> kept;
  for (const auto& t : g.elements) {
    V c = nsd::v3(0.0, 0.0, 0.0);
    for (int k = 0; k < 4; ++k) c = c + cv(g.vertices[t[k]]);
    c = 0.25 * c;
    if (nsd::norm(c - centre) <= radius) kept.push_back(t);
  }
  for (const auto& t : kept)
    for (int k = 0; k < 4; ++k) keep[t[k]] = 0;
  MeshSpec ball;
  double zmin = std::numeric_limits<double>::infinity();
  for (size_t v = 0; v < g.vertices.size(); ++v)
    if (keep[v] == 0) {
      keep[v] = static_cast<int>(ball.vertices.size());
      ball.vertices.push_back(g.vertices[v]);
      zmin = std::min(zmin, g.vertices[v].z);
    }
  const double lift = 0.005 - zmin;
  for (Vec3& p : ball.vertices) p.z += lift;
  for (const auto& t : kept) ball.elements.push_back({keep[t[0]], keep[t[1]], keep[t[2]], keep[t[3]]});
  const Vec3 he{0.008 * L, 0.008 * L, 0.012 * L};
  const double rad = 0.075 * L, za[4] = {0.014 * L, 0.050 * L, 0.086 * L, 0.122 * L},
               zc[4] = {0.032 * L, 0.068 * L, 0.104 * L, 0.140 * L};
  for (int f = 0; f < 4; ++f) {
    const double th = 0.5 * M_PI * f;
    const Vec3 d{std::cos(th), std::sin(th), 0.0};
    const Vec3 tg{-std::sin(th), std::cos(th), 0.0};
    for (int k = 0; k < 4; ++k) {
      s.bodies.push_back(box(Vec3{rad * d.x, rad * d.y, zc[k]}, he, 0.02 * L * L * L, axis_angle(Vec3{0, 0, 1}, th)));
      JointSpecDesc j;
      j.kind = 1;
      j.a.body = k == 0 ? -1 : 1 + 4 * f + (k - 1);
      j.b.body = 1 + 4 * f + k;
      j.anchor = Vec3{rad * d.x, rad * d.y, za[k]};
      j.axis = tg;
      s.joints.push_back(j);
    }
    JointSpecDesc dr;
    dr.kind = 0;
    dr.a.body = 1 + 4 * f + 3;
    dr.b.body = -1;
    dr.anchor = Vec3{rad * d.x, rad * d.y, 0.152 * L};
    dr.compliance = 1e-4;
    dr.anchor_velocity = Vec3{-0.02 * d.x, -0.02 * d.y, 0.0};  // 0.05 m/s squeezes the ball unstable by step 29
    s.joints.push_back(dr);
  }
  ball.velocity = Vec3{0.0, 0.0, -speed};
  ball.initial = ball.vertices;
  jitter(ball.initial, 1e-3 * edge / n, 7);
  ball.particle_contacts = true;
  s.meshes.push_back(ball);
  s.mu_default = 0.75;
  s.margin = 0.01;
  s.solver.newton_iterations = 6;
  s.solver.linear_max_iterations = 50;
  return s;
}
Scene s_c5(unsigned env_id) {
  Scene s;
  s.solver = defaults();
  s.bodies.push_back(ground());
  const double H = 0.40 + 0.005;
  s.bodies.push_back(sphere(Vec3{0, 0, H}, 0.25, 1.0));
  std::mt19937 rng(env_id);
  std::uniform_real_distribution<double> rate(-0.5, 0.5);
  const Vec3 he{0.2, 0.04, 0.04};
  for (int k = 0; k < 4; ++k) {
    const double th = 0.25 * M_PI + 0.5 * M_PI * k;
    const V d = nsd::v3(std::cos(th), std::sin(th), 0.0);
    const V t = nsd::v3(-std::sin(th), std::cos(th), 0.0);
    const V z = nsd::v3(0.0, 0.0, 1.0);
    const V hip = nsd::v3(0.265 * d.x, 0.265 * d.y, H);
    const V knee = nsd::v3(0.695 * d.x, 0.695 * d.y, H - 0.02);
    const V ct = nsd::v3(0.48 * d.x, 0.48 * d.y, H);
    const V cs = nsd::v3(0.75 * d.x, 0.75 * d.y, H - 0.2);
    const Quat qt = axis_angle(Vec3{0, 0, 1}, th);
    const Quat qs = qmul(qt, axis_angle(Vec3{0, 1, 0}, 0.5 * M_PI));
    const double a_hip = rate(rng);
    const double a_knee = rate(rng);
    BodySpec thigh = box(vc(ct), he, 0.2, qt);
    thigh.ang_vel = vc(a_hip * z);
    thigh.vel = vc(nsd::cross(a_hip * z, ct - hip));
    BodySpec shin = box(vc(cs), he, 0.2, qs);
    shin.ang_vel = vc(a_hip * z + a_knee * t);
    shin.vel = vc(nsd::cross(a_hip * z, cs - hip) + nsd::cross(a_knee * t, cs - knee));
    s.bodies.push_back(thigh);
    s.bodies.push_back(shin);
    JointSpecDesc jh;
    jh.kind = 1;
    jh.a.body = 1;
    jh.b.body = 2 + 2 * k;
    jh.anchor = vc(hip);
    jh.axis = Vec3{0, 0, 1};
    s.joints.push_back(jh);
    JointSpecDesc jk;
    jk.kind = 1;
    jk.a.body = 2 + 2 * k;
    jk.b.body = 3 + 2 * k;
    jk.anchor = vc(knee);
    jk.axis = vc(t);
    s.joints.push_back(jk);
  }
  s.mu_default = 1.0;
  s.margin = 0.01;
  s.solver.newton_iterations = 4;
  s.solver.linear_max_iterations = 10;
  return s;
}

M inertia_of(const ShapeDesc& s, double mass) {
  M m = nsd::m3_zero<double>();
  if (s.kind == 1) {
    const double v = 0.4 * mass * s.radius * s.radius;
    m(0, 0) = m(1, 1) = m(2, 2) = v;
  } else if (s.kind == 2) {
    const Vec3 h = s.half;
    m(0, 0) = mass / 3.0 * (h.y * h.y + h.z * h.z);
    m(1, 1) = mass / 3.0 * (h.x * h.x + h.z * h.z);
    m(2, 2) = mass / 3.0 * (h.x * h.x + h.y * h.y);
  } else {
    m = nsd::m3_identity<double>();
  }
  return m;
}

}  // namespace

nsd_topology World::topology() const {
  nsd_topology t{};
  t.n_bodies = static_cast<int32_t>(body_type.size());
  t.body_type = body_type.data();
  t.body_mass = body_mass.data();
  t.body_inertia = body_inertia.data();
  t.n_joints = static_cast<int32_t>(joint_kind.size());
  t.joint_kind = joint_kind.data();
  t.joint_body = joint_body.data();
  t.joint_frame = joint_frame.data();
  t.joint_param = joint_param.data();
  t.n_tets = static_cast<int32_t>(tet_volume.size());
  t.tet_body = tet_body.data();
  t.tet_dm_inv = tet_dm_inv.data();
  t.tet_volume = tet_volume.data();
  t.tet_material = tet_material.data();
  return t;
}

Scene build(const std::string& name, unsigned seed, bool* ok) {
  std::string base = name;
  std::vector<double> args;
  const size_t colon = name.find(':');
  if (colon != std::string::npos) {
    base = name.substr(0, colon);
    std::stringstream ss(name.substr(colon + 1));
    std::string tok;
    while (std::getline(ss, tok, ':')) args.push_back(std::stod(tok));
  }
  *ok = true;
  if (base == "arch") return s_arch();
  if (base == "heavy_stack") return s_heavy_stack();
  if (base == "box_pile") return s_box_pile(seed);
  if (base == "box_on_plane") return s_box_on_plane();
  if (base == "stretch_sheet") return s_stretch_sheet(false);
  if (base == "stretch_sheet_linear") return s_stretch_sheet(true);
  if (base == "incline") return s_incline(args.size() > 0 ? args[0] : 20.0, args.size() > 1 ? args[1] : 0.5);
  if (base == "c1") return s_c1();
  if (base == "c2") return s_c2(args.size() > 0 ? static_cast<int>(args[0]) : 12);
  if (base == "c3") return s_c3(args.size() > 0 ? static_cast<int>(args[0]) : 100);
  if (base == "bend_chain")
    return s_bend_chain(args.size() > 0 ? static_cast<int>(args[0]) : 10, args.size() > 1 ? args[1] : 50.0);
  // C4 drop speed 0.2 m/s: at 1.0 m/s the 8 mm Neo-Hookean elements blow up at step 4
  // under the 6 x 50 budget (the reference then throws in spmv_transpose)
  if (base == "c4")
    return s_c4(args.size() > 0 ? static_cast<int>(args[0]) : 12, args.size() > 1 ? args[1] : 0.2,
                args.size() > 2 ? args[2] : 2.0);  // scale 2: ball radius 0.1 m (1.0 blows up by step 13-28)
  if (base == "c5") return s_c5(seed);
  *ok = false;
  return Scene{};
}

// build_world (scene.cpp:587-707) into the flat layout.
World build_world(const Scene& sc) {
  World w;
  w.gravity = sc.gravity;
  w.h = sc.timestep;
  w.margin = sc.margin;
  w.mu_default = sc.mu_default;
  w.solver = sc.solver;
  std::vector<int> body_map(sc.bodies.size(), -1);
  int nb = 0;
  for (size_t i = 0; i < sc.bodies.size(); ++i) {
    const BodySpec& d = sc.bodies[i];
    if (d.kind == BodyKind::Static) continue;
    const bool rigid = d.kind == BodyKind::Rigid;
    w.body_type.push_back(rigid ? 1 : 0);
    w.body_mass.push_back(d.mass);
    M in = nsd::m3_identity<double>();
    if (rigid) {
      if (d.has_inertia)
        for (int k = 0; k < 9; ++k) in.a[k] = d.inertia[k];
      else
        in = inertia_of(d.shape, d.mass);
    }
    for (int k = 0; k < 9; ++k) w.body_inertia.push_back(in.a[k]);
    body_map[i] = nb++;
  }
  std::vector<int> mesh_base(sc.meshes.size(), 0);
  for (size_t m = 0; m < sc.meshes.size(); ++m) {
    const MeshSpec& d = sc.meshes[m];
    mesh_base[m] = nb;
    // lame_from_young_poisson (materials.cpp:32-43)
    if (d.young <= 0.0 || d.poisson < 0.0 || d.poisson >= 0.4999) throw std::invalid_argument("bad material");
    const double mu = d.young / (2.0 * (1.0 + d.poisson));
    const double lambda = d.young * d.poisson / ((1.0 + d.poisson) * (1.0 - 2.0 * d.poisson));
    const double c1 = 0.5 * mu, d1 = 0.5 * lambda, alpha = lambda > 0.0 ? 1.0 + mu / lambda : 1.0;
    std::vector<double> lumped(d.vertices.size(), 0.0);
    for (const auto& ev : d.elements) {
      std::array<int, 4> idx = ev;
      M dm;
      auto setc = [&](int c, const Vec3& a, const Vec3& b) {
        dm(0, c) = a.x - b.x;
        dm(1, c) = a.y - b.y;
        dm(2, c) = a.z - b.z;
      };
      setc(0, d.vertices[idx[1]], d.vertices[idx[0]]);
      setc(1, d.vertices[idx[2]], d.vertices[idx[0]]);
      setc(2, d.vertices[idx[3]], d.vertices[idx[0]]);
      if (nsd::det3(dm) < 0.0) {
        std::swap(idx[2], idx[3]);
        setc(0, d.vertices[idx[1]], d.vertices[idx[0]]);
        setc(1, d.vertices[idx[2]], d.vertices[idx[0]]);
        setc(2, d.vertices[idx[3]], d.vertices[idx[0]]);
      }
      const double det = nsd::det3(dm);
      if (det <= 0.0) throw std::invalid_argument("tet element is degenerate or inverted at rest");
      const M inv = nsd::inverse3(dm);
      const double vol = det / 6.0;
      for (int k = 0; k < 4; ++k) w.tet_body.push_back(mesh_base[m] + idx[k]);
      for (int k = 0; k < 9; ++k) w.tet_dm_inv.push_back(inv.a[k]);
      w.tet_volume.push_back(vol);
      w.tet_material.push_back(c1);
      w.tet_material.push_back(d1);
      w.tet_material.push_back(alpha);
      w.tet_material.push_back((d.diagonal_compliance ? 1.0 : 0.0) + (d.linear ? 2.0 : 0.0));
      for (int v : idx) lumped[v] += d.density * vol / 4.0;
    }
    for (size_t v = 0; v < d.vertices.size(); ++v) {
      w.body_type.push_back(0);
      w.body_mass.push_back(lumped[v] > 0.0 ? lumped[v] : 1e-6);
      for (int k = 0; k < 9; ++k) w.body_inertia.push_back(k % 4 == 0 ? 1.0 : 0.0);
      ++nb;
    }
    if (d.particle_contacts) w.particle_ranges.push_back({mesh_base[m], static_cast<int>(d.vertices.size())});
  }
  // layout (bodies.cpp:7-22)
  for (int b = 0; b < nb; ++b) {
    w.dof_off.push_back(w.num_dof);
    w.coord_off.push_back(w.num_coord);
    w.num_dof += w.body_type[b] ? 6 : 3;
    w.num_coord += w.body_type[b] ? 7 : 3;
  }
  w.q.assign(w.num_coord, 0.0);
  w.u.assign(w.num_dof, 0.0);
  for (int b = 0; b < nb; ++b)
    if (w.body_type[b]) w.q[w.coord_off[b] + 3] = 1.0;
  for (size_t i = 0; i < sc.bodies.size(); ++i) {
    const BodySpec& d = sc.bodies[i];
    const int b = body_map[i];
    if (b < 0) continue;
    double* q = &w.q[w.coord_off[b]];
    double* u = &w.u[w.dof_off[b]];
    q[0] = d.pos.x;
    q[1] = d.pos.y;
    q[2] = d.pos.z;
    u[0] = d.vel.x;
    u[1] = d.vel.y;
    u[2] = d.vel.z;
    if (d.kind == BodyKind::Rigid) {
      const double n = std::sqrt(d.rot.w * d.rot.w + d.rot.x * d.rot.x + d.rot.y * d.rot.y + d.rot.z * d.rot.z);
      if (n < 1e-300) {
        q[3] = 1.0;
        q[4] = q[5] = q[6] = 0.0;
      } else {
        q[3] = d.rot.w / n;
        q[4] = d.rot.x / n;
        q[5] = d.rot.y / n;
        q[6] = d.rot.z / n;
      }
      u[3] = d.ang_vel.x;
      u[4] = d.ang_vel.y;
      u[5] = d.ang_vel.z;
    }
  }
  for (size_t m = 0; m < sc.meshes.size(); ++m) {
    const MeshSpec& d = sc.meshes[m];
    for (size_t v = 0; v < d.vertices.size(); ++v) {
      const int b = mesh_base[m] + static_cast<int>(v);
      const Vec3& p = d.initial.empty() ? d.vertices[v] : d.initial[v];
      double* q = &w.q[w.coord_off[b]];
      q[0] = p.x;
      q[1] = p.y;
      q[2] = p.z;
      double* u = &w.u[w.dof_off[b]];
      u[0] = d.velocity.x;
      u[1] = d.velocity.y;
      u[2] = d.velocity.z;
    }
  }
  // shapes (scene.cpp:675-683)
  for (size_t i = 0; i < sc.bodies.size(); ++i) {
    const BodySpec& d = sc.bodies[i];
    if (!d.has_shape || d.kind == BodyKind::Particle) continue;
    nsd_shape s{};
    s.body = d.kind == BodyKind::Static ? -1 : body_map[i];
    s.kind = d.shape.kind;
    s.normal[0] = d.shape.normal.x;
    s.normal[1] = d.shape.normal.y;
    s.normal[2] = d.shape.normal.z;
    s.offset = d.shape.offset;
    s.radius = d.shape.radius;
    s.half_extents[0] = d.shape.half.x;
    s.half_extents[1] = d.shape.half.y;
    s.half_extents[2] = d.shape.half.z;
    s.thickness = d.shape.thickness;
    s.mu = d.shape.mu;
    w.shapes.push_back(s);
  }
  // joints + bind_joint (constraints.cpp:222-263)
  auto rot_of = [&](int b) -> M {
    if (b < 0 || w.body_type[b] == 0) return nsd::m3_identity<double>();
    const double* t = &w.q[w.coord_off[b] + 3];
    return nsd::quat_rot(t[0], t[1], t[2], t[3]);
  };
  auto pos_of = [&](int b) { return nsd::v3(w.q[w.coord_off[b]], w.q[w.coord_off[b] + 1], w.q[w.coord_off[b] + 2]); };
  for (const JointSpecDesc& d : sc.joints) {
    auto resolve = [&](const JointAttach& a) {
      if (a.mesh >= 0) return mesh_base[a.mesh] + a.vertex;
      return a.body >= 0 ? body_map[a.body] : -1;
    };
    const int ja = resolve(d.a), jb = resolve(d.b);
    auto point_local = [&](int b, const V& wp) -> V {
      if (b < 0) return wp;
      if (w.body_type[b] == 0) return nsd::v3(0.0, 0.0, 0.0);
      return nsd::mul_t(rot_of(b), wp - pos_of(b));
    };
    auto dir_local = [&](int b, const V& wd) -> V { return b < 0 ? wd : nsd::mul_t(rot_of(b), wd); };
    const V anchor = cv(d.anchor);
    const V ax = nsd::normalize(cv(d.axis));
    // tangent_basis
    int sm = 0;
    if (std::abs(ax.y) < std::abs(ax.x)) sm = 1;
    if (std::abs(ax.z) < std::abs(ax[sm])) sm = 2;
    V e = nsd::v3(0.0, 0.0, 0.0);
    e[sm] = 1.0;
    const V p1 = nsd::normalize(e - nsd::dot(e, ax) * ax);
    const V p2 = nsd::cross(ax, p1);
    V fr[7];
    fr[0] = point_local(ja, anchor);
    fr[1] = point_local(jb, anchor);
    fr[2] = dir_local(ja, ax);
    fr[3] = dir_local(ja, p1);
    fr[4] = nsd::v3(1.0, 0.0, 0.0);
    fr[5] = nsd::v3(0.0, 1.0, 0.0);
    fr[6] = nsd::v3(0.0, 0.0, 0.0);
    if (d.kind != 0) {
      fr[4] = dir_local(jb, p1);
      fr[5] = dir_local(jb, p2);
    }
    if (d.kind == 2) fr[6] = nsd::v3(nsd::dot(ax, p1), nsd::dot(ax, p2), nsd::dot(p1, p2));
    w.joint_kind.push_back(d.kind);
    w.joint_body.push_back(ja);
    w.joint_body.push_back(jb);
    for (int k = 0; k < 7; ++k) {
      w.joint_frame.push_back(fr[k].x);
      w.joint_frame.push_back(fr[k].y);
      w.joint_frame.push_back(fr[k].z);
    }
    w.joint_param.push_back(d.compliance);
    w.joint_param.push_back(d.stiffness);
    if (d.anchor_velocity.x != 0.0 || d.anchor_velocity.y != 0.0 || d.anchor_velocity.z != 0.0)
      w.driven.push_back({static_cast<int>(w.joint_kind.size()) - 1, d.anchor_velocity});
  }
  return w;
}

}  // namespace nsdw

// ================================================================== C ABI (builders)
struct nsd_scene {
  nsdw::Scene sc;  // the description (serialize_scene)
  nsdw::World w;
};

extern "C" {

int nsd_scene_build(const char* name, uint32_t seed, nsd_scene** out) {
  if (!name || !out) return NSD_INVALID;
  try {
    bool ok = false;
    nsdw::Scene s = nsdw::build(name, seed, &ok);
    if (!ok) return NSD_INVALID;
    auto* h = new nsd_scene();
    h->sc = s;
    h->w = nsdw::build_world(s);
    *out = h;
    return NSD_OK;
  } catch (...) {
    return NSD_INVALID;
  }
}

int nsd_scene_parse(const char* json, nsd_scene** out, char* err, int32_t err_capacity) {
  if (err && err_capacity > 0) err[0] = 0;
  if (!json || !out) return NSD_INVALID;
  try {
    nsdw::Scene s = nsdw::parse_scene(json);
    auto* h = new nsd_scene();
    h->sc = s;
    h->w = nsdw::build_world(s);
    *out = h;
    return NSD_OK;
  } catch (const std::exception& e) {
    if (err && err_capacity > 0) {
      std::strncpy(err, e.what(), static_cast<size_t>(err_capacity) - 1);
      err[err_capacity - 1] = 0;
    }
    return NSD_INVALID;
  }
}

int nsd_scene_serialize(const nsd_scene* s, char* buf, int64_t capacity, int64_t* length) {
  if (!s || !length) return NSD_INVALID;
  const std::string doc = nsdw::serialize_scene(s->sc);
  *length = static_cast<int64_t>(doc.size());
  if (buf) {
    if (capacity < static_cast<int64_t>(doc.size()) + 1) return NSD_INVALID;
    std::memcpy(buf, doc.c_str(), doc.size() + 1);
  }
  return NSD_OK;
}

int nsd_scene_dims(const nsd_scene* s, int32_t* d) {
  if (!s || !d) return NSD_INVALID;
  const nsdw::World& w = s->w;
  d[0] = static_cast<int32_t>(w.body_type.size());
  d[1] = w.num_dof;
  d[2] = w.num_coord;
  d[3] = static_cast<int32_t>(w.joint_kind.size());
  d[4] = static_cast<int32_t>(w.tet_volume.size());
  d[5] = static_cast<int32_t>(w.shapes.size());
  d[6] = w.solver.newton_iterations;
  d[7] = w.solver.linear_max_iterations;
  return NSD_OK;
}

int nsd_scene_topology(const nsd_scene* s, nsd_topology* t) {
  if (!s || !t) return NSD_INVALID;
  *t = s->w.topology();
  return NSD_OK;
}

int nsd_scene_shapes(const nsd_scene* s, nsd_shape* shapes, double* margin, double* mu_default) {
  if (!s) return NSD_INVALID;
  if (shapes && !s->w.shapes.empty()) std::memcpy(shapes, s->w.shapes.data(), sizeof(nsd_shape) * s->w.shapes.size());
  if (margin) *margin = s->w.margin;
  if (mu_default) *mu_default = s->w.mu_default;
  return NSD_OK;
}

int nsd_scene_state(const nsd_scene* s, double* q, double* u) {
  if (!s) return NSD_INVALID;
  if (q) std::memcpy(q, s->w.q.data(), sizeof(double) * s->w.q.size());
  if (u) std::memcpy(u, s->w.u.data(), sizeof(double) * s->w.u.size());
  return NSD_OK;
}

int nsd_scene_config(const nsd_scene* s, nsd_config* cfg, double* h, double* gravity) {
  if (!s) return NSD_INVALID;
  if (cfg) *cfg = s->w.solver;
  if (h) *h = s->w.h;
  if (gravity) {
    gravity[0] = s->w.gravity.x;
    gravity[1] = s->w.gravity.y;
    gravity[2] = s->w.gravity.z;
  }
  return NSD_OK;
}

int nsd_scene_destroy(nsd_scene* s) {
  delete s;
  return NSD_OK;
}

int nsd_scene_joint_frames(const nsd_scene* s, double* frames) {
  if (!s || !frames) return NSD_INVALID;
  if (!s->w.joint_frame.empty())
    std::memcpy(frames, s->w.joint_frame.data(), sizeof(double) * s->w.joint_frame.size());
  return NSD_OK;
}

// step_world's first statement (scene.cpp:710-716): world-side anchors of driven
// joints move by h * anchor_velocity.
int nsd_scene_advance_anchors(nsd_scene* s) {
  if (!s) return NSD_INVALID;
  nsdw::World& w = s->w;
  for (const auto& dv : w.driven) {
    const int j = dv.first;
    double* fr = &w.joint_frame[21 * static_cast<size_t>(j)];
    double* anchor = w.joint_body[2 * j] < 0 ? fr : (w.joint_body[2 * j + 1] < 0 ? fr + 3 : nullptr);
    if (!anchor) continue;
    anchor[0] += w.h * dv.second.x;
    anchor[1] += w.h * dv.second.y;
    anchor[2] += w.h * dv.second.z;
  }
  return NSD_OK;
}

// The caller side of step_world (scene.cpp:717-721) on the host, as in the
// reference: u~ = u + h M~^-1 (f_gravity + f_gyro + f_extra) at q
// (bodies.cpp:200-217), then the narrow phase over shape pairs and the
// particle generators with the predicted-gap rule, in canonical
// (a.body, b.body, feature) order (collision.cpp:239-297). The Newton step
// that consumes the contacts runs on the GPU (nsd_step).
static int scene_detect(const nsd_scene* s, const double* q, const double* u, const double* f_extra,
                        int32_t capacity, nsd_contact* out, int32_t* n);

int nsd_scene_detect(const nsd_scene* s, const double* q, const double* u, const double* f_extra, int32_t capacity,
                     nsd_contact* out, int32_t* n) {
  if (!s || !q || !u || !n || capacity < 0 || (capacity > 0 && !out)) return NSD_INVALID;
  nvtxRangePushA("nsd_scene_detect (host narrow phase)");
  struct Pop {
    ~Pop() { nvtxRangePop(); }
  } pop;
  try {
    return scene_detect(s, q, u, f_extra, capacity, out, n);
  } catch (const std::exception&) {  // allocation or thread failure: an error code, never std::terminate
    return NSD_INVALID;
  }
}

}  // extern "C"

namespace {

// Persistent host workers for the threaded narrow phase: created once per process
// (lazily, up to 7) and parked on a condition variable between World.step calls.
// Creating and joining threads on every call cost more than the C3/C4 rows they ran.
// The pool is per process: a forked child (whose copy has no threads behind it)
// gets a fresh one. It is never destroyed; parked workers end with the process.
class DetectPool {
 public:
  static DetectPool& get() {
    static std::mutex gm;
    static DetectPool* pool = nullptr;
    static pid_t owner = 0;
    std::lock_guard<std::mutex> g(gm);
    if (!pool || owner != getpid()) {
      pool = new DetectPool();  // a stale parent pool in a forked child is left untouched
      owner = getpid();
    }
    return *pool;
  }
  // Runs work(0 .. nth-1): the caller takes index 0 and every index without a worker.
  // Each index is a fixed strided set of rows written to its own slots, so the result
  // does not depend on which thread ran it. Returns false if any index threw.
  bool run(unsigned nth, const std::function<void(unsigned)>& work) {
    std::lock_guard<std::mutex> serial(run_mu_);  // one job at a time (several Worlds may call)
    ensure(nth > 0 ? nth - 1 : 0);
    const unsigned nw = std::min<unsigned>(static_cast<unsigned>(threads_.size()), nth > 0 ? nth - 1 : 0);
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = &work;
      njob_ = nw;
      pending_ = nw;
      failed_ = false;
      ++generation_;
    }
    cv_.notify_all();
    bool ok = true;
    auto guarded = [&](unsigned t) {
      try {
        work(t);
      } catch (...) {
        ok = false;
      }
    };
    guarded(0);
    for (unsigned t = nw + 1; t < nth; ++t) guarded(t);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
    return ok && !failed_;
  }
 private:
  void ensure(unsigned n) {
    while (threads_.size() < n && threads_.size() < 7) {
      const unsigned idx = static_cast<unsigned>(threads_.size()) + 1;  // work index this worker runs
      try {
        threads_.emplace_back([this, idx] { loop(idx); });
      } catch (...) {  // e.g. std::system_error under a pids limit: the caller runs the rest
        return;
      }
    }
  }
  void loop(unsigned idx) {
    unsigned seen = 0;
    for (;;) {
      const std::function<void(unsigned)>* job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return generation_ != seen; });
        seen = generation_;
        if (idx > njob_) continue;  // not needed for this job
        job = job_;
      }
      bool threw = false;
      try {
        (*job)(idx);
      } catch (...) {
        threw = true;
      }
      {
        std::lock_guard<std::mutex> g(mu_);
        if (threw) failed_ = true;
        if (--pending_ == 0) done_.notify_all();
      }
    }
  }
  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_;
  std::vector<std::thread> threads_;
  const std::function<void(unsigned)>* job_ = nullptr;
  unsigned njob_ = 0, pending_ = 0, generation_ = 0;
  bool failed_ = false;
};

template <class F> void run_strided(unsigned nth, F&& work) {
  const std::function<void(unsigned)> fn = std::forward<F>(work);
  if (!DetectPool::get().run(nth, fn)) throw std::runtime_error("nsd_scene_detect: worker failed");
}

}  // namespace

extern "C" {

static int scene_detect(const nsd_scene* s, const double* q, const double* u, const double* f_extra, int32_t capacity,
                        nsd_contact* out, int32_t* n) {
  using V = nsd::V3<double>;
  using M = nsd::M3<double>;
  const nsdw::World& w = s->w;
  const int nb = static_cast<int>(w.body_type.size());
  std::vector<double> ut(static_cast<size_t>(w.num_dof));
  const double h = w.h;
  for (int b = 0; b < nb; ++b) {
    const int d = w.dof_off[b], cd = w.coord_off[b];
    const double m = w.body_mass[b];
    V f = nsd::v3(m * w.gravity.x, m * w.gravity.y, m * w.gravity.z);
    if (f_extra) f = f + nsd::v3(f_extra[d], f_extra[d + 1], f_extra[d + 2]);
    for (int k = 0; k < 3; ++k) ut[d + k] = u[d + k] + h * (f[k] / m);
    if (w.body_type[b] == 1) {
      const M Rm = nsd::quat_rot(q[cd + 3], q[cd + 4], q[cd + 5], q[cd + 6]);
      M I;
      for (int i = 0; i < 9; ++i) I.a[i] = w.body_inertia[9 * static_cast<size_t>(b) + i];
      const M Iw = nsd::mul(nsd::mul(Rm, I), nsd::transpose(Rm));
      const M Ii = nsd::inverse3(Iw);
      const V om = nsd::v3(u[d + 3], u[d + 4], u[d + 5]);
      V tq = -nsd::cross(om, nsd::mul(Iw, om));
      if (f_extra) tq = tq + nsd::v3(f_extra[d + 3], f_extra[d + 4], f_extra[d + 5]);
      const V un = om + h * nsd::mul(Ii, tq);
      for (int k = 0; k < 3; ++k) ut[d + 3 + k] = un[k];
    }
  }
  nsd::BodyView<double> view{w.body_type.data(), w.dof_off.data(), w.coord_off.data(), q, ut.data()};
  std::vector<nsd::ShapeD<double>> sh(w.shapes.size());
  for (size_t i = 0; i < w.shapes.size(); ++i) {
    const nsd_shape& a = w.shapes[i];
    nsd::ShapeD<double>& d = sh[i];
    d.body = a.body;
    d.kind = a.kind;
    for (int k = 0; k < 3; ++k) {
      d.n[k] = a.normal[k];
      d.he[k] = a.half_extents[k];
    }
    d.offset = a.offset;
    d.radius = a.radius;
    d.thick = a.thickness;
    d.mu = a.mu;
  }
  std::vector<nsd::CandD<double>> cands;
  nsd::CandD<double> c4[4];
  double th = 0.0, mu = 0.0;
  // Shape pairs, row i = pairs (i, j > i). Large scenes (C3: ~5k pairs) spread
  // the rows over host threads; each row keeps its own candidates and the rows
  // are concatenated in i order, so the sequence fed to the stable sort below
  // is the serial one and the result is bit-identical.
  const size_t ns = sh.size();
  const size_t npairs = ns > 1 ? ns * (ns - 1) / 2 : 0;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const unsigned nth = npairs >= 2048 ? std::min<unsigned>(hw, 8u) : 1u;
  if (nth > 1) {
    std::vector<std::vector<nsd::CandD<double>>> rows(ns);
    auto work = [&](unsigned t) {
      nsd::CandD<double> b4[4];
      double tth = 0.0, tmu = 0.0;
      for (size_t i = t; i < ns; i += nth)  // strided rows balance the triangle
        for (size_t j = i + 1; j < ns; ++j) {
          const int k = nsd::pair_contacts(view, sh[i], sh[j], h, w.margin, w.mu_default, b4, &tth, &tmu);
          rows[i].insert(rows[i].end(), b4, b4 + k);
        }
    };
    run_strided(nth, work);
    for (const auto& r : rows) cands.insert(cands.end(), r.begin(), r.end());
  } else {
    for (size_t i = 0; i < ns; ++i)
      for (size_t j = i + 1; j < ns; ++j) {
        const int k = nsd::pair_contacts(view, sh[i], sh[j], h, w.margin, w.mu_default, c4, &th, &mu);
        cands.insert(cands.end(), c4, c4 + k);
      }
  }
  // Particle generators: one row per particle body, threaded and concatenated
  // in body order like the pair rows above.
  std::vector<int> pbodies;
  for (const auto& pr : w.particle_ranges)
    for (int b = pr.first; b < pr.first + pr.second; ++b) pbodies.push_back(b);
  const size_t nprow = pbodies.size();
  // Conservative cull of particle-vs-box tests that cannot pass the predicted-gap
  // rule (gap - thickness - h closing > margin): gap >= |x - c| - R (R the box's
  // half-diagonal) and closing <= |u~_particle| + |v_box| + |w_box| R. Culled tests
  // produce no candidate either way, so the contact set is unchanged bit for bit.
  struct BoxBound {
    V c;
    double reach;  // R + thickness + h (|v| + |w| R) + margin, with slack
  };
  std::vector<BoxBound> bbound(ns);
  for (size_t i = 0; i < ns; ++i) {
    if (sh[i].kind != 2) continue;
    const double R = std::sqrt(sh[i].he[0] * sh[i].he[0] + sh[i].he[1] * sh[i].he[1] + sh[i].he[2] * sh[i].he[2]);
    const int b = sh[i].body;
    V c = nsd::v3(0.0, 0.0, 0.0);
    double vb = 0.0;
    if (b >= 0) {
      c = nsd::bv_pos(view, b);
      const double* ub = ut.data() + w.dof_off[b];
      vb = std::sqrt(ub[0] * ub[0] + ub[1] * ub[1] + ub[2] * ub[2]);
      if (w.body_type[b] == 1) vb += std::sqrt(ub[3] * ub[3] + ub[4] * ub[4] + ub[5] * ub[5]) * R;
    }
    bbound[i] = {c, (R + sh[i].thick + h * vb + w.margin) * (1.0 + 1e-9) + 1e-12};
  }
  auto culled = [&](int body, size_t i) {
    if (sh[i].kind != 2) return false;
    const V x = nsd::bv_pos(view, body);
    const double* up = ut.data() + w.dof_off[body];
    const double reach = bbound[i].reach + h * std::sqrt(up[0] * up[0] + up[1] * up[1] + up[2] * up[2]) * (1.0 + 1e-9);
    const V d = x - bbound[i].c;
    return d.x * d.x + d.y * d.y + d.z * d.z > reach * reach;
  };
  const unsigned pth = nprow * ns >= 4096 ? std::min<unsigned>(hw, 8u) : 1u;
  if (pth > 1) {
    std::vector<std::vector<nsd::CandD<double>>> rows(nprow);
    auto work = [&](unsigned t) {
      nsd::CandD<double> b4[4];
      double tth = 0.0, tmu = 0.0;
      for (size_t r = t; r < nprow; r += pth)
        for (size_t i = 0; i < ns; ++i) {
          if (culled(pbodies[r], i)) continue;
          const int k = nsd::particle_shape_contact(view, pbodies[r], sh[i], h, w.margin, w.mu_default, 0.0, -1.0,
                                                    b4, &tth, &tmu);
          rows[r].insert(rows[r].end(), b4, b4 + k);
        }
    };
    run_strided(pth, work);
    for (const auto& r : rows) cands.insert(cands.end(), r.begin(), r.end());
  } else {
    for (const int b : pbodies)
      for (size_t i = 0; i < ns; ++i) {
        if (culled(b, i)) continue;
        const int k = nsd::particle_shape_contact(view, b, sh[i], h, w.margin, w.mu_default, 0.0, -1.0, c4, &th, &mu);
        cands.insert(cands.end(), c4, c4 + k);
      }
  }
  std::stable_sort(cands.begin(), cands.end(), [](const nsd::CandD<double>& x, const nsd::CandD<double>& y) {
    return nsd::canonical_less(x.a, x.b, x.feature, y.a, y.b, y.feature);
  });
  *n = static_cast<int32_t>(cands.size());
  if (static_cast<int32_t>(cands.size()) > capacity) return NSD_INVALID;  // *n tells the caller the size needed
  for (size_t i = 0; i < cands.size(); ++i) {
    const nsd::CandD<double>& c = cands[i];
    nsd_contact& o = out[i];
    std::memset(&o, 0, sizeof(o));
    o.body_a = c.a;
    o.body_b = c.b;
    o.feature = c.feature;
    for (int k = 0; k < 3; ++k) {
      o.local_a[k] = c.la[k];
      o.local_b[k] = c.lb[k];
      o.normal[k] = c.n[k];
    }
    V d1, d2;
    nsd::tangent_basis(nsd::v3(c.n[0], c.n[1], c.n[2]), d1, d2);
    for (int k = 0; k < 3; ++k) {
      o.d1[k] = d1[k];
      o.d2[k] = d2[k];
    }
    o.thickness = c.thick;
    o.mu = c.mu;
  }
  return NSD_OK;
}

int nsd_scene_batch_state(const char* name, uint32_t seed0, int32_t n, double* q, double* u) {
  if (!name || n < 0 || !q || !u) return NSD_INVALID;
  try {
    size_t oq = 0, ou = 0;
    for (int32_t i = 0; i < n; ++i) {
      bool ok = false;
      nsdw::Scene s = nsdw::build(name, seed0 + static_cast<uint32_t>(i), &ok);
      if (!ok) return NSD_INVALID;
      const nsdw::World w = nsdw::build_world(s);
      std::memcpy(q + oq, w.q.data(), sizeof(double) * w.q.size());
      std::memcpy(u + ou, w.u.data(), sizeof(double) * w.u.size());
      oq += w.q.size();
      ou += w.u.size();
    }
    return NSD_OK;
  } catch (...) {
    return NSD_INVALID;
  }
}

}  // extern "C"
