// nsdyn_b200.hpp — C++ host API of the B200 Newton step, mirroring the
// reference's scene/solver API (/root/reference/proj/include/nsdyn/*.h) over
// the C ABI in nsdyn_gpu.h. Header-only; link against libnsdyn_b200.so.
//
//   reference (namespace nsdyn)                    here (namespace nsdyn_b200)
//   GeneralizedState, Body        bodies.h:11-43   same names and fields (std::vector instead of Eigen)
//   JointSpec, ContactConstraint  constraints.h    same names and fields
//   TetElement, TetMeshElements   materials.h      same names and fields (Neo-Hookean and linear co-rotational)
//   NewtonConfig, SolveReport,    newton.h:12-120  same names and fields, plus NewtonConfig::precision
//   StepContext, MeshBinding,
//   count_rows, newton_step
//   World, build_scene_by_name,   scene.h:83-110   same names; step_world's Newton solve runs on the GPU
//   step_world
//   RunOptions, load_world, run,  runner.h:11-43   same names, CSV formats and exit codes; a scene is a
//   sweep                                          builder name or a JSON scene file
//   world_from_json,               scene.h:74-77   parse_scene + build_world / serialize_scene (the
//   serialize_scene                                reference's JSON scene format)
//
// Error behaviour follows the reference: invalid input throws
// std::invalid_argument (bodies.cpp:80, constraints.cpp:142-144,
// solvers.cpp:188-190); a NaN in the Newton update rolls q, u back and returns
// a report with aborted = true (newton.cpp:362-369). A CUDA failure or an
// option that is not on the GPU path (record_iterates, mixed material models in
// one scene) throws std::runtime_error — there is no CPU fallback.
//
// Device state: newton_step keeps one device solver per thread, keyed by the
// StepContext's state/joints/meshes addresses and sizes and by the config;
// the static data (bodies, tets) is uploaded when that key changes. After
// editing masses, inertias or meshes in place, call invalidate_device_cache().
#pragma once

#include "nsdyn_gpu.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <memory>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace nsdyn_b200 {

struct Vec3 {
  double x = 0.0, y = 0.0, z = 0.0;
  double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};
struct Vec4 {  // quaternion (w, x, y, z), bodies.h:10
  double w = 1.0, x = 0.0, y = 0.0, z = 0.0;
};
using Mat3 = std::array<double, 9>;  // row-major
inline constexpr Mat3 kIdentity3 = {1, 0, 0, 0, 1, 0, 0, 0, 1};

// ------------------------------------------------------------------ bodies.h
enum class BodyType { Particle, Rigid };

struct Body {
  BodyType type = BodyType::Particle;
  double mass = 1.0;
  Mat3 inertia = kIdentity3;  // body frame, rigid bodies only
  int dof_count() const { return type == BodyType::Particle ? 3 : 6; }
  int coord_count() const { return type == BodyType::Particle ? 3 : 7; }
};

struct GeneralizedState {
  std::vector<Body> bodies;
  std::vector<double> q;  // packed coordinates (3 per particle, 7 per rigid: position, quaternion wxyz)
  std::vector<double> u;  // packed velocities (3 per particle, 6 per rigid: linear, angular)
  std::vector<int> dof_offset, coord_offset;
  int num_dof = 0, num_coord = 0;

  // Builds offsets and zero-sizes q/u (bodies.cpp:7-20).
  void finalize_layout() {
    dof_offset.assign(bodies.size(), 0);
    coord_offset.assign(bodies.size(), 0);
    num_dof = num_coord = 0;
    for (size_t b = 0; b < bodies.size(); ++b) {
      dof_offset[b] = num_dof;
      coord_offset[b] = num_coord;
      num_dof += bodies[b].dof_count();
      num_coord += bodies[b].coord_count();
    }
    q.assign(num_coord, 0.0);
    u.assign(num_dof, 0.0);
  }
  Vec3 position(int b) const { return {q[coord_offset[b]], q[coord_offset[b] + 1], q[coord_offset[b] + 2]}; }
  void set_position(int b, const Vec3& p) {
    q[coord_offset[b]] = p.x;
    q[coord_offset[b] + 1] = p.y;
    q[coord_offset[b] + 2] = p.z;
  }
  Vec4 orientation(int b) const {
    const double* t = &q[coord_offset[b] + 3];
    return {t[0], t[1], t[2], t[3]};
  }
  void set_orientation(int b, const Vec4& t) {
    double* d = &q[coord_offset[b] + 3];
    d[0] = t.w;
    d[1] = t.x;
    d[2] = t.y;
    d[3] = t.z;
  }
  Vec3 linear_velocity(int b) const { return {u[dof_offset[b]], u[dof_offset[b] + 1], u[dof_offset[b] + 2]}; }
  Vec3 angular_velocity(int b) const {
    return {u[dof_offset[b] + 3], u[dof_offset[b] + 4], u[dof_offset[b] + 5]};
  }
};

// ------------------------------------------------------------------ constraints.h
struct AttachPoint {
  int body = -1;  // -1: fixed world point stored in `local`
  Vec3 local;
};

struct ContactConstraint {
  AttachPoint a, b;
  Vec3 normal{0, 0, 1};  // world space, points b -> a
  double thickness = 0.0;
  double mu = 0.0;
  Vec3 d1{1, 0, 0}, d2{0, 1, 0};
  double lambda_n = 0.0;                    // h-scaled (impulse), written by newton_step
  std::array<double, 2> lambda_f{0.0, 0.0};
  int feature = 0;
};

enum class RStrategy { Identity, TimestepSquared, EffectiveMass };
enum class JointKind { FixedPoint, Revolute, Prismatic, BendSpring };

struct JointSpec {
  JointKind kind = JointKind::FixedPoint;
  int body_a = -1;
  int body_b = -1;
  Vec3 anchor_a, anchor_b;          // local frames (world for body index < 0)
  Vec3 axis_a{0, 0, 1};
  Vec3 axis_a2{1, 0, 0};
  Vec3 axis_b1{1, 0, 0};
  Vec3 axis_b2{0, 1, 0};
  double compliance = 0.0;
  double stiffness = 0.0;
  Vec3 rest_dots;
  Vec3 anchor_velocity;
};

// ------------------------------------------------------------------ ncp.h / solvers.h
enum class NcpKind { MinimumMap, FischerBurmeister };
enum class LinearMethod { Jacobi, GaussSeidel, PCG, PCR };
enum class PreconditionerKind { None, Diagonal };

struct LinearSolverConfig {
  LinearMethod method = LinearMethod::PCR;
  int max_iterations = 40;
  double tolerance = 1e-10;
  PreconditionerKind preconditioner = PreconditionerKind::Diagonal;
};

// ------------------------------------------------------------------ materials.h
struct TetElement {
  std::array<int, 4> verts{};  // indices into the mesh particle block
  Mat3 dm_inv = kIdentity3;
  double rest_volume = 0.0;
};

struct NeoHookeanMaterial {
  double c1 = 0.0, d1 = 0.0, alpha = 1.0;
};

// materials.cpp:32-43: C1 = mu/2, D1 = lambda/2, alpha = 1 + mu/lambda.
inline NeoHookeanMaterial lame_from_young_poisson(double young, double poisson) {
  if (young <= 0.0 || poisson < 0.0 || poisson >= 0.4999) throw std::invalid_argument("material: bad young/poisson");
  const double mu = young / (2.0 * (1.0 + poisson));
  const double lambda = young * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson));
  return {0.5 * mu, 0.5 * lambda, 1.0 + mu / lambda};
}

enum class MaterialModel { Linear, NeoHookean };

struct MaterialSpec {
  MaterialModel model = MaterialModel::NeoHookean;
  double young = 1e5;
  double poisson = 0.45;
  bool diagonal_compliance = false;
};

struct TetMeshElements {
  std::vector<TetElement> elements;
  MaterialSpec material;
  NeoHookeanMaterial nh;
  // Lame halves for both models (the linear model's isotropic stiffness is rebuilt
  // from them on the device: mu = 2 c1, lambda = 2 d1)
  void prepare() { nh = lame_from_young_poisson(material.young, material.poisson); }
};

// ------------------------------------------------------------------ newton.h
enum class Precision { FP32, FP64 };  // extension: FP64 reproduces the reference, FP32 is the fast mode

struct NewtonConfig {
  int newton_iterations = 8;
  double step_fraction = 0.75;
  double epsilon_reg = 1e-6;
  bool geometric_stiffness = true;
  RStrategy r_strategy = RStrategy::EffectiveMass;
  NcpKind ncp_kind = NcpKind::FischerBurmeister;
  LinearSolverConfig linear;
  double newton_tolerance = 1e-6;
  bool line_search = false;
  bool record_iterates = false;  // not on the GPU path (throws)
  Precision precision = Precision::FP64;
  int device = 0;
};

struct MeshBinding {
  TetMeshElements mesh;
  int particle_base = 0;
};

struct NewtonIterationStats {
  double residual_inf = 0.0;
  double merit_l2 = 0.0;
  double comp_error_max = 0.0;
  double cone_violation_max = 0.0;
  double step_size = 0.0;
  int linear_iterations = 0;
  double linear_residual = 0.0;
  bool linear_breakdown = false;
};

struct ContactTelemetry {
  double gap = 0.0;
  double lambda_n = 0.0;       // force units
  double lambda_f_norm = 0.0;  // force units
  double mu = 0.0;
  double tangential_speed = 0.0;
  double dissipation_dot = 0.0;
};

struct SolveReport {
  std::vector<NewtonIterationStats> iterations;
  std::vector<std::vector<double>> linear_histories;
  std::vector<std::vector<double>> delta_u;  // record_iterates: not produced on the GPU path
  std::vector<ContactTelemetry> contacts;
  double final_residual_inf = 0.0;
  double final_comp_error = 0.0;
  double final_cone_violation = 0.0;
  double min_gap = 0.0;
  double min_diag_shift = 0.0;
  bool aborted = false;
  bool converged = false;
  double device_ms = 0.0;  // extension: device time of the step's kernel
};

struct StepContext {
  GeneralizedState* state = nullptr;
  const std::vector<JointSpec>* joints = nullptr;
  const std::vector<MeshBinding>* meshes = nullptr;
  std::vector<ContactConstraint>* contacts = nullptr;
  Vec3 gravity{0, 0, -9.81};
  double h = 0.0083;
  const std::vector<double>* f_extra = nullptr;  // extension hook: extra generalized force (num_dof)
};

namespace detail {

inline void check(int rc) {
  if (rc == NSD_OK || rc == NSD_ABORTED) return;
  const char* e = nsd_last_error();
  const std::string msg = std::string("nsdyn_b200: ") + (e ? e : "error");
  if (rc == NSD_INVALID) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

inline void put3(double* d, const Vec3& v) {
  d[0] = v.x;
  d[1] = v.y;
  d[2] = v.z;
}
inline Vec3 get3(const double* s) { return {s[0], s[1], s[2]}; }

// Flat C-ABI topology built from a StepContext (owning arrays).
struct FlatTopology {
  std::vector<int32_t> body_type, joint_kind, joint_body, tet_body;
  std::vector<double> body_mass, body_inertia, joint_frame, joint_param, tet_dm_inv, tet_volume, tet_material;

  void build(const StepContext& ctx) {
    const GeneralizedState& s = *ctx.state;
    const size_t nb = s.bodies.size();
    body_type.resize(nb);
    body_mass.resize(nb);
    body_inertia.resize(9 * nb);
    for (size_t b = 0; b < nb; ++b) {
      body_type[b] = s.bodies[b].type == BodyType::Rigid ? 1 : 0;
      body_mass[b] = s.bodies[b].mass;
      std::memcpy(&body_inertia[9 * b], s.bodies[b].inertia.data(), 9 * sizeof(double));
    }
    const size_t nj = ctx.joints ? ctx.joints->size() : 0;
    joint_kind.resize(nj);
    joint_body.resize(2 * nj);
    joint_param.resize(2 * nj);
    for (size_t j = 0; j < nj; ++j) {
      const JointSpec& J = (*ctx.joints)[j];
      joint_kind[j] = static_cast<int32_t>(J.kind);
      joint_body[2 * j] = J.body_a;
      joint_body[2 * j + 1] = J.body_b;
      joint_param[2 * j] = J.compliance;
      joint_param[2 * j + 1] = J.stiffness;
    }
    frames(ctx, joint_frame);
    tet_body.clear();
    tet_dm_inv.clear();
    tet_volume.clear();
    tet_material.clear();
    if (ctx.meshes)
      for (const MeshBinding& m : *ctx.meshes) {
        for (const TetElement& e : m.mesh.elements) {
          for (int k = 0; k < 4; ++k) tet_body.push_back(m.particle_base + e.verts[k]);
          tet_dm_inv.insert(tet_dm_inv.end(), e.dm_inv.begin(), e.dm_inv.end());
          tet_volume.push_back(e.rest_volume);
          tet_material.push_back(m.mesh.nh.c1);
          tet_material.push_back(m.mesh.nh.d1);
          tet_material.push_back(m.mesh.nh.alpha);
          tet_material.push_back((m.mesh.material.diagonal_compliance ? 1.0 : 0.0) +
                                 (m.mesh.material.model == MaterialModel::Linear ? 2.0 : 0.0));
        }
      }
  }
  static void frames(const StepContext& ctx, std::vector<double>& out) {
    const size_t nj = ctx.joints ? ctx.joints->size() : 0;
    out.resize(21 * nj);
    for (size_t j = 0; j < nj; ++j) {
      const JointSpec& J = (*ctx.joints)[j];
      double* f = &out[21 * j];
      put3(f, J.anchor_a);
      put3(f + 3, J.anchor_b);
      put3(f + 6, J.axis_a);
      put3(f + 9, J.axis_a2);
      put3(f + 12, J.axis_b1);
      put3(f + 15, J.axis_b2);
      put3(f + 18, J.rest_dots);
    }
  }
  nsd_topology view() const {
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
};

inline nsd_config to_c(const NewtonConfig& c) {
  if (c.record_iterates) throw std::runtime_error("nsdyn_b200: record_iterates is not on the GPU path");
  nsd_config k{};
  nsd_config_default(&k, c.precision == Precision::FP64 ? NSD_FP64 : NSD_FP32);
  k.newton_iterations = c.newton_iterations;
  k.step_fraction = c.step_fraction;
  k.epsilon_reg = c.epsilon_reg;
  k.geometric_stiffness = c.geometric_stiffness ? 1 : 0;
  k.r_strategy = static_cast<int32_t>(c.r_strategy);
  k.ncp_kind = static_cast<int32_t>(c.ncp_kind);
  k.linear_method = static_cast<int32_t>(c.linear.method);  // 0 Jacobi, 1 Gauss-Seidel, 2 PCG, 3 PCR
  k.linear_max_iterations = c.linear.max_iterations;
  k.linear_tolerance = c.linear.tolerance;
  k.preconditioner = static_cast<int32_t>(c.linear.preconditioner);
  k.newton_tolerance = c.newton_tolerance;
  k.line_search = c.line_search ? 1 : 0;
  return k;
}

struct SolverDeleter {
  void operator()(nsd_solver* s) const { nsd_destroy(s); }
};

// One device solver per thread, rebuilt when the scene's identity or the config changes.
struct Cache {
  std::unique_ptr<nsd_solver, SolverDeleter> solver;
  const void* state = nullptr;
  const void* joints = nullptr;
  const void* meshes = nullptr;
  size_t nb = 0, nj = 0, nm = 0;
  nsd_config cfg{};
  int device = -1;
  FlatTopology topo;
  std::vector<double> frames;
  std::vector<nsd_contact> contacts;
  std::vector<nsd_iter_stats> iters;
  std::vector<double> hist, tel;
  std::vector<int32_t> hist_len;
};

inline Cache& cache() {
  thread_local Cache c;
  return c;
}

inline bool same_cfg(const nsd_config& a, const nsd_config& b) { return std::memcmp(&a, &b, sizeof(a)) == 0; }

}  // namespace detail

// Drops the thread's device solver (call after editing bodies or meshes in place).
inline void invalidate_device_cache() { detail::cache().solver.reset(); }

// count_rows (newton.h:114, newton.cpp:18-41,98).
inline int count_rows(const StepContext& ctx) {
  if (!ctx.state) throw std::invalid_argument("count_rows: null state");
  detail::FlatTopology t;
  t.build(ctx);
  const nsd_topology v = t.view();
  return nsd_count_rows(&v, ctx.contacts ? static_cast<int32_t>(ctx.contacts->size()) : 0);
}

// newton_step (newton.h:116-118, newton.cpp:321-418) on the GPU: mutates
// ctx.state->q/u in place and writes lambda_n / lambda_f into ctx.contacts.
inline SolveReport newton_step(const StepContext& ctx, const NewtonConfig& cfg) {
  if (!ctx.state) throw std::invalid_argument("newton_step: null state");
  GeneralizedState& s = *ctx.state;
  if (static_cast<int>(s.q.size()) != s.num_coord || static_cast<int>(s.u.size()) != s.num_dof)
    throw std::invalid_argument("newton_step: state not finalized (finalize_layout)");
  detail::Cache& C = detail::cache();
  const nsd_config kc = detail::to_c(cfg);
  const size_t nj = ctx.joints ? ctx.joints->size() : 0, nm = ctx.meshes ? ctx.meshes->size() : 0;
  if (!C.solver || C.state != &s || C.joints != ctx.joints || C.meshes != ctx.meshes || C.nb != s.bodies.size() ||
      C.nj != nj || C.nm != nm || !detail::same_cfg(C.cfg, kc) || C.device != cfg.device) {
    C.solver.reset();
    C.topo.build(ctx);
    const nsd_topology v = C.topo.view();
    nsd_solver* h = nullptr;
    detail::check(nsd_create(&v, &kc, cfg.device, &h));
    C.solver.reset(h);
    C.state = &s;
    C.joints = ctx.joints;
    C.meshes = ctx.meshes;
    C.nb = s.bodies.size();
    C.nj = nj;
    C.nm = nm;
    C.cfg = kc;
    C.device = cfg.device;
  }
  detail::FlatTopology::frames(ctx, C.frames);
  const size_t nc = ctx.contacts ? ctx.contacts->size() : 0;
  C.contacts.assign(nc, nsd_contact{});
  for (size_t i = 0; i < nc; ++i) {
    const ContactConstraint& c = (*ctx.contacts)[i];
    nsd_contact& o = C.contacts[i];
    o.body_a = c.a.body;
    o.body_b = c.b.body;
    o.feature = c.feature;
    detail::put3(o.local_a, c.a.local);
    detail::put3(o.local_b, c.b.local);
    detail::put3(o.normal, c.normal);
    detail::put3(o.d1, c.d1);
    detail::put3(o.d2, c.d2);
    o.thickness = c.thickness;
    o.mu = c.mu;
    o.lambda_n = c.lambda_n;
    o.lambda_f[0] = c.lambda_f[0];
    o.lambda_f[1] = c.lambda_f[1];
  }
  const int ni = cfg.newton_iterations, stride = cfg.linear.max_iterations + 1;
  C.iters.assign(ni > 0 ? ni : 1, nsd_iter_stats{});
  C.hist.assign(static_cast<size_t>(ni > 0 ? ni : 1) * stride, 0.0);
  C.hist_len.assign(ni > 0 ? ni : 1, 0);
  C.tel.assign(6 * (nc ? nc : 1), 0.0);
  if (ctx.f_extra && static_cast<int>(ctx.f_extra->size()) != s.num_dof)
    throw std::invalid_argument("newton_step: f_extra size != num_dof");
  nsd_step_in in{};
  in.q = s.q.data();
  in.u = s.u.data();
  in.n_contacts = static_cast<int32_t>(nc);
  in.contacts = C.contacts.data();
  in.h = ctx.h;
  in.gravity[0] = ctx.gravity.x;
  in.gravity[1] = ctx.gravity.y;
  in.gravity[2] = ctx.gravity.z;
  in.f_extra = ctx.f_extra ? ctx.f_extra->data() : nullptr;
  in.joint_frame = nj ? C.frames.data() : nullptr;
  nsd_step_out out{};
  out.q = s.q.data();
  out.u = s.u.data();
  out.contacts = C.contacts.data();
  out.iters = C.iters.data();
  out.linear_history = C.hist.data();
  out.linear_history_len = C.hist_len.data();
  out.contact_telemetry = C.tel.data();
  detail::check(nsd_step(C.solver.get(), &in, &out));
  SolveReport r;
  r.iterations.resize(out.n_iterations);
  r.linear_histories.resize(out.n_iterations);
  for (int i = 0; i < out.n_iterations; ++i) {
    const nsd_iter_stats& a = C.iters[i];
    NewtonIterationStats& b = r.iterations[i];
    b.residual_inf = a.residual_inf;
    b.merit_l2 = a.merit_l2;
    b.comp_error_max = a.comp_error_max;
    b.cone_violation_max = a.cone_violation_max;
    b.step_size = a.step_size;
    b.linear_iterations = a.linear_iterations;
    b.linear_residual = a.linear_residual;
    b.linear_breakdown = a.linear_breakdown != 0;
    const double* hrow = &C.hist[static_cast<size_t>(i) * stride];
    r.linear_histories[i].assign(hrow, hrow + C.hist_len[i]);
  }
  r.contacts.resize(nc);
  for (size_t i = 0; i < nc; ++i) {
    const double* t = &C.tel[6 * i];
    r.contacts[i] = ContactTelemetry{t[0], t[1], t[2], t[3], t[4], t[5]};
    ContactConstraint& c = (*ctx.contacts)[i];  // lambda write-back (newton.cpp:74-78)
    c.lambda_n = C.contacts[i].lambda_n;
    c.lambda_f[0] = C.contacts[i].lambda_f[0];
    c.lambda_f[1] = C.contacts[i].lambda_f[1];
  }
  r.final_residual_inf = out.final_residual_inf;
  r.final_comp_error = out.final_comp_error;
  r.final_cone_violation = out.final_cone_violation;
  r.min_gap = out.min_gap;
  r.min_diag_shift = out.min_diag_shift;
  r.aborted = out.aborted != 0;
  r.converged = out.converged != 0;
  r.device_ms = nsd_last_step_ms(C.solver.get());
  return r;
}

// ------------------------------------------------------------------ scene.h
struct SceneDeleter {
  void operator()(nsd_scene* s) const { nsd_scene_destroy(s); }
};

struct World {
  GeneralizedState state;
  std::vector<JointSpec> joints;
  std::vector<MeshBinding> meshes;
  std::vector<ContactConstraint> contacts;
  Vec3 gravity{0, 0, -9.81};
  double h = 0.0083;
  NewtonConfig solver;
  double time = 0.0;
  std::vector<double> f_extra;  // extension hook (empty = none)
  std::shared_ptr<nsd_scene> scene;  // product-side collision shapes, particle generators, driven anchors
};

// Builder dispatch by name (scene.h:76-78), e.g. "c1", "c5", "incline:35:0.5",
// "box_pile"; nullopt for unknown names.
namespace detail {
World world_from_handle(nsd_scene* raw);
}
inline std::optional<World> build_scene_by_name(const std::string& name, unsigned seed) {
  nsd_scene* raw = nullptr;
  if (nsd_scene_build(name.c_str(), seed, &raw) != NSD_OK) return std::nullopt;
  return detail::world_from_handle(raw);
}

// parse_scene + build_world (scene.cpp:293-470, 587-707): a document in the
// reference's JSON scene format; std::runtime_error with the reference's message
// ("scene error at bodies[0].mass: must be positive") when it does not validate.
inline World world_from_json(const std::string& text) {
  nsd_scene* raw = nullptr;
  char err[1024];
  if (nsd_scene_parse(text.c_str(), &raw, err, sizeof(err)) != NSD_OK) throw std::runtime_error(err);
  return detail::world_from_handle(raw);
}

// serialize_scene (scene.cpp:472-556) of the description the world was built from.
inline std::string serialize_scene(const World& w) {
  if (!w.scene) throw std::invalid_argument("serialize_scene: world has no scene description");
  int64_t n = 0;
  detail::check(nsd_scene_serialize(w.scene.get(), nullptr, 0, &n));
  std::string out(static_cast<size_t>(n) + 1, '\0');
  detail::check(nsd_scene_serialize(w.scene.get(), out.data(), n + 1, &n));
  out.resize(static_cast<size_t>(n));
  return out;
}

inline World detail::world_from_handle(nsd_scene* raw) {
  World w;
  w.scene.reset(raw, SceneDeleter{});
  nsd_topology t{};
  detail::check(nsd_scene_topology(raw, &t));
  GeneralizedState& s = w.state;
  s.bodies.resize(t.n_bodies);
  for (int b = 0; b < t.n_bodies; ++b) {
    s.bodies[b].type = t.body_type[b] == 1 ? BodyType::Rigid : BodyType::Particle;
    s.bodies[b].mass = t.body_mass[b];
    std::memcpy(s.bodies[b].inertia.data(), t.body_inertia + 9 * b, 9 * sizeof(double));
  }
  s.finalize_layout();
  detail::check(nsd_scene_state(raw, s.q.data(), s.u.data()));
  w.joints.resize(t.n_joints);
  for (int j = 0; j < t.n_joints; ++j) {
    JointSpec& J = w.joints[j];
    J.kind = static_cast<JointKind>(t.joint_kind[j]);
    J.body_a = t.joint_body[2 * j];
    J.body_b = t.joint_body[2 * j + 1];
    const double* f = t.joint_frame + 21 * j;
    J.anchor_a = detail::get3(f);
    J.anchor_b = detail::get3(f + 3);
    J.axis_a = detail::get3(f + 6);
    J.axis_a2 = detail::get3(f + 9);
    J.axis_b1 = detail::get3(f + 12);
    J.axis_b2 = detail::get3(f + 15);
    J.rest_dots = detail::get3(f + 18);
    J.compliance = t.joint_param[2 * j];
    J.stiffness = t.joint_param[2 * j + 1];
  }
  // tets arrive flat (mesh-major); regroup runs of one material into MeshBindings
  for (int e = 0; e < t.n_tets;) {
    const double* m0 = t.tet_material + 4 * e;
    int end = e;
    int base = t.tet_body[4 * e];
    while (end < t.n_tets && std::memcmp(t.tet_material + 4 * end, m0, 4 * sizeof(double)) == 0) {
      for (int k = 0; k < 4; ++k) base = std::min(base, static_cast<int>(t.tet_body[4 * end + k]));
      ++end;
    }
    MeshBinding mb;
    mb.particle_base = base;
    mb.mesh.nh = NeoHookeanMaterial{m0[0], m0[1], m0[2]};  // Lame halves for both models
    mb.mesh.material.diagonal_compliance = (static_cast<int>(m0[3]) & 1) != 0;
    mb.mesh.material.model = (static_cast<int>(m0[3]) & 2) ? MaterialModel::Linear : MaterialModel::NeoHookean;
    for (int i = e; i < end; ++i) {
      TetElement te;
      for (int k = 0; k < 4; ++k) te.verts[k] = t.tet_body[4 * i + k] - base;
      std::memcpy(te.dm_inv.data(), t.tet_dm_inv + 9 * i, 9 * sizeof(double));
      te.rest_volume = t.tet_volume[i];
      mb.mesh.elements.push_back(te);
    }
    w.meshes.push_back(std::move(mb));
    e = end;
  }
  nsd_config c{};
  double g[3];
  detail::check(nsd_scene_config(raw, &c, &w.h, g));
  w.gravity = {g[0], g[1], g[2]};
  NewtonConfig& n = w.solver;
  n.newton_iterations = c.newton_iterations;
  n.step_fraction = c.step_fraction;
  n.epsilon_reg = c.epsilon_reg;
  n.geometric_stiffness = c.geometric_stiffness != 0;
  n.r_strategy = static_cast<RStrategy>(c.r_strategy);
  n.ncp_kind = static_cast<NcpKind>(c.ncp_kind);
  n.linear.max_iterations = c.linear_max_iterations;
  n.linear.tolerance = c.linear_tolerance;
  n.linear.preconditioner = static_cast<PreconditionerKind>(c.preconditioner);
  n.newton_tolerance = c.newton_tolerance;
  n.line_search = c.line_search != 0;
  n.precision = c.precision == NSD_FP64 ? Precision::FP64 : Precision::FP32;
  return w;
}

// step_world (scene.h:109, scene.cpp:709-732): driven anchors move, contacts
// are detected on the host at (q, u~) as in the reference, then newton_step
// runs on the GPU.
inline SolveReport step_world(World& w) {
  if (!w.scene) throw std::invalid_argument("step_world: world has no scene (use build_scene_by_name)");
  detail::check(nsd_scene_advance_anchors(w.scene.get()));
  std::vector<double> frames(21 * w.joints.size());
  if (!frames.empty()) detail::check(nsd_scene_joint_frames(w.scene.get(), frames.data()));
  for (size_t j = 0; j < w.joints.size(); ++j) {  // only the driven world-side anchors change
    w.joints[j].anchor_a = detail::get3(&frames[21 * j]);
    w.joints[j].anchor_b = detail::get3(&frames[21 * j + 3]);
  }
  const double* fx = w.f_extra.empty() ? nullptr : w.f_extra.data();
  std::vector<nsd_contact> buf(256);
  int32_t n = 0;
  int rc = nsd_scene_detect(w.scene.get(), w.state.q.data(), w.state.u.data(), fx, static_cast<int32_t>(buf.size()),
                            buf.data(), &n);
  if (rc != NSD_OK && n > static_cast<int32_t>(buf.size())) {
    buf.resize(n);
    rc = nsd_scene_detect(w.scene.get(), w.state.q.data(), w.state.u.data(), fx, n, buf.data(), &n);
  }
  detail::check(rc);
  w.contacts.resize(n);
  for (int i = 0; i < n; ++i) {
    const nsd_contact& c = buf[i];
    ContactConstraint& o = w.contacts[i];
    o = ContactConstraint{};
    o.a.body = c.body_a;
    o.b.body = c.body_b;
    o.a.local = detail::get3(c.local_a);
    o.b.local = detail::get3(c.local_b);
    o.normal = detail::get3(c.normal);
    o.d1 = detail::get3(c.d1);
    o.d2 = detail::get3(c.d2);
    o.thickness = c.thickness;
    o.mu = c.mu;
    o.feature = c.feature;
  }
  StepContext ctx;
  ctx.state = &w.state;
  ctx.joints = &w.joints;
  ctx.meshes = &w.meshes;
  ctx.contacts = &w.contacts;
  ctx.gravity = w.gravity;
  ctx.h = w.h;
  ctx.f_extra = w.f_extra.empty() ? nullptr : &w.f_extra;
  SolveReport r = newton_step(ctx, w.solver);
  w.time += w.h;
  return r;
}

// ------------------------------------------------------------------ runner.h
// Scene execution front end writing the reference's trajectory.csv /
// convergence.csv / sweep.csv (runner.cpp:80-126, %.17g, atomic write) — the
// on-disk format used to diff GPU runs against the CPU oracle.
struct RunOptions {
  std::string scene;  // builder name (JSON scene files are not part of this path)
  int steps = 100;
  std::optional<std::string> solver_method;  // jacobi | pcg | pcr (gs is not on the GPU Newton path)
  std::optional<std::string> ncp;            // minmap | fb
  std::optional<std::string> r_strategy;     // identity | h2 | effmass
  std::optional<int> newton_iters;
  std::optional<int> linear_iters;
  std::optional<double> step_fraction;
  std::optional<double> epsilon;
  unsigned seed = 0;
  std::string out_dir = ".";
  Precision precision = Precision::FP64;  // extension
};

constexpr int kExitOk = 0;
constexpr int kExitValidation = 1;
constexpr int kExitNumerical = 2;

namespace detail {
inline std::string fmt17(double v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}
inline void write_atomic(const std::filesystem::path& path, const std::string& content) {
  const std::filesystem::path tmp = path.string() + ".tmp";
  {
    std::ofstream out(tmp, std::ios::binary);
    if (!out) throw std::runtime_error("cannot write " + tmp.string());
    out << content;
  }
  std::filesystem::rename(tmp, path);
}
// runner.cpp:29-77 (same messages)
inline void apply_overrides(const RunOptions& o, NewtonConfig& c) {
  if (o.solver_method) {
    const std::string& m = *o.solver_method;
    if (m == "jacobi")
      c.linear.method = LinearMethod::Jacobi;
    else if (m == "gs")
      c.linear.method = LinearMethod::GaussSeidel;
    else if (m == "pcg")
      c.linear.method = LinearMethod::PCG;
    else if (m == "pcr")
      c.linear.method = LinearMethod::PCR;
    else
      throw std::runtime_error("unknown solver \"" + m + "\"");
  }
  if (o.ncp) {
    if (*o.ncp == "minmap")
      c.ncp_kind = NcpKind::MinimumMap;
    else if (*o.ncp == "fb")
      c.ncp_kind = NcpKind::FischerBurmeister;
    else
      throw std::runtime_error("unknown NCP function \"" + *o.ncp + "\"");
  }
  if (o.r_strategy) {
    if (*o.r_strategy == "identity")
      c.r_strategy = RStrategy::Identity;
    else if (*o.r_strategy == "h2")
      c.r_strategy = RStrategy::TimestepSquared;
    else if (*o.r_strategy == "effmass")
      c.r_strategy = RStrategy::EffectiveMass;
    else
      throw std::runtime_error("unknown r strategy \"" + *o.r_strategy + "\"");
  }
  if (o.newton_iters) {
    if (*o.newton_iters < 1) throw std::runtime_error("--newton-iters must be >= 1");
    c.newton_iterations = *o.newton_iters;
  }
  if (o.linear_iters) {
    if (*o.linear_iters < 1) throw std::runtime_error("--linear-iters must be >= 1");
    c.linear.max_iterations = *o.linear_iters;
  }
  if (o.step_fraction) {
    if (*o.step_fraction <= 0.0 || *o.step_fraction > 1.0) throw std::runtime_error("--t must lie in (0, 1]");
    c.step_fraction = *o.step_fraction;
  }
  if (o.epsilon) {
    if (*o.epsilon < 0.0) throw std::runtime_error("--eps must be >= 0");
    c.epsilon_reg = *o.epsilon;
  }
}
inline void append_trajectory(std::string& csv, int step, const GeneralizedState& s) {  // runner.cpp:80-104
  for (size_t b = 0; b < s.bodies.size(); ++b) {
    csv += std::to_string(step) + ',' + std::to_string(b);
    const Vec3 p = s.position(static_cast<int>(b));
    for (int k = 0; k < 3; ++k) csv += ',' + fmt17(p[k]);
    if (s.bodies[b].type == BodyType::Rigid) {
      const Vec4 q = s.orientation(static_cast<int>(b));
      csv += ',' + fmt17(q.w) + ',' + fmt17(q.x) + ',' + fmt17(q.y) + ',' + fmt17(q.z);
    } else {
      csv += ",1,0,0,0";
    }
    const Vec3 v = s.linear_velocity(static_cast<int>(b));
    for (int k = 0; k < 3; ++k) csv += ',' + fmt17(v[k]);
    if (s.bodies[b].type == BodyType::Rigid) {
      const Vec3 w = s.angular_velocity(static_cast<int>(b));
      for (int k = 0; k < 3; ++k) csv += ',' + fmt17(w[k]);
    } else {
      csv += ",0,0,0";
    }
    csv += '\n';
  }
}
inline void append_convergence(std::string& csv, int step, const SolveReport& r, const std::string& prefix) {
  for (size_t i = 0; i < r.iterations.size(); ++i) {  // runner.cpp:106-121
    const NewtonIterationStats& it = r.iterations[i];
    csv += prefix + std::to_string(step) + ',' + std::to_string(i) + ',' + fmt17(it.residual_inf) + ',' +
           fmt17(it.comp_error_max) + ',' + fmt17(it.cone_violation_max) + ',' + fmt17(it.step_size) + ',' +
           std::to_string(it.linear_iterations) + ',' + fmt17(it.linear_residual) + '\n';
  }
}
inline constexpr const char* kTrajectoryHeader = "step,body,qx,qy,qz,q0,q1,q2,q3,ux,uy,uz,wx,wy,wz\n";
inline constexpr const char* kConvergenceHeader =
    "step,newton_iter,residual_inf,comp_error_n_max,cone_violation_max,step_size,linear_iters,"
    "linear_residual_final\n";
}  // namespace detail

// load_world (runner.cpp:130-146): a JSON scene file or a builder name, with the overrides applied.
inline World load_world(const RunOptions& o) {
  if (std::filesystem::exists(o.scene)) {
    std::ifstream in(o.scene, std::ios::binary);
    std::stringstream ss;
    ss << in.rdbuf();
    World w = world_from_json(ss.str());
    detail::apply_overrides(o, w.solver);
    w.solver.precision = o.precision;
    return w;
  }
  auto w = build_scene_by_name(o.scene, o.seed);
  if (!w) throw std::runtime_error("scene \"" + o.scene + "\" is neither a file nor a known builder");
  detail::apply_overrides(o, w->solver);
  w->solver.precision = o.precision;
  return std::move(*w);
}

// run (runner.cpp:148-180): steps the world, writes trajectory.csv and
// convergence.csv atomically; 0 ok, 1 validation error, 2 numerical abort.
inline int run(const RunOptions& o, std::string* error = nullptr) {
  try {
    if (o.steps < 1) throw std::runtime_error("--steps must be >= 1");
    World w = load_world(o);
    std::string traj = detail::kTrajectoryHeader, conv = detail::kConvergenceHeader;
    bool aborted = false;
    for (int step = 0; step < o.steps; ++step) {
      const SolveReport r = step_world(w);
      detail::append_trajectory(traj, step, w.state);
      detail::append_convergence(conv, step, r, "");
      if (r.aborted) {
        aborted = true;
        break;
      }
    }
    std::filesystem::create_directories(o.out_dir);
    detail::write_atomic(std::filesystem::path(o.out_dir) / "trajectory.csv", traj);
    detail::write_atomic(std::filesystem::path(o.out_dir) / "convergence.csv", conv);
    if (aborted) {
      if (error) *error = "numerical abort (NaN) during solve";
      return kExitNumerical;
    }
    return kExitOk;
  } catch (const std::exception& e) {
    if (error) *error = e.what();
    return kExitValidation;
  }
}

// sweep (runner.cpp:182-218): one run per axis value, merged sweep.csv. The
// "solver" axis runs jacobi, gs, pcg and pcr (runner.cpp:187).
inline int sweep(const RunOptions& o, const std::string& axis, std::string* error = nullptr) {
  try {
    if (o.steps < 1) throw std::runtime_error("--steps must be >= 1");
    std::vector<std::string> values;
    if (axis == "solver")
      values = {"jacobi", "gs", "pcg", "pcr"};
    else if (axis == "r_strategy")
      values = {"identity", "h2", "effmass"};
    else if (axis == "ncp")
      values = {"minmap", "fb"};
    else
      throw std::runtime_error("unknown sweep axis \"" + axis + "\"");
    std::string csv = std::string("axis_value,") + detail::kConvergenceHeader;
    for (const std::string& v : values) {
      RunOptions sub = o;
      if (axis == "solver")
        sub.solver_method = v;
      else if (axis == "r_strategy")
        sub.r_strategy = v;
      else
        sub.ncp = v;
      World w = load_world(sub);
      invalidate_device_cache();
      for (int step = 0; step < o.steps; ++step) {
        const SolveReport r = step_world(w);
        detail::append_convergence(csv, step, r, v + ",");
        if (r.aborted) break;
      }
    }
    std::filesystem::create_directories(o.out_dir);
    detail::write_atomic(std::filesystem::path(o.out_dir) / "sweep.csv", csv);
    return kExitOk;
  } catch (const std::exception& e) {
    if (error) *error = e.what();
    return kExitValidation;
  }
}

}  // namespace nsdyn_b200
