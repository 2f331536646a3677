// ORACLE — test infrastructure only. extern "C" exports of the CPU restatement
// for tests/ (ctypes), __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference arm. Nothing in the product links this library.
#include "oracle.h"

#include <chrono>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace orc;

namespace {
M3 m3_from(const double* a) {
  M3 m;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m(i, j) = a[3 * i + j];
  return m;
}
void m3_to(const M3& m, double* a) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) a[3 * i + j] = m(i, j);
}
thread_local std::string g_err;

struct OWorld {
  World w;
  Report last;
  bool has_report = false;
};
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// ---------------- KAT entry points ------------------------------------------
void orc_phi_n(double c, double lambda, double r, int kind, double* out3) {
  const Phi p = phi_n(c, lambda, r, static_cast<Ncp>(kind));
  out3[0] = p.value;
  out3[1] = p.d_c;
  out3[2] = p.d_l;
}
double orc_friction_W(double vt, double lf, double mln, double r, int kind) {
  return friction_W(vt, lf, mln, r, static_cast<Ncp>(kind));
}
void orc_svd3(const double* f, double* u, double* s, double* v) {
  const Svd3 r = svd3(m3_from(f));
  m3_to(r.U, u);
  m3_to(r.V, v);
  for (int i = 0; i < 3; ++i) s[i] = r.S[i];
}
void orc_project_psd3(const double* m, double* out) { m3_to(project_psd3(m3_from(m)), out); }
int orc_sym_eig3(const double* m, double* vals, double* vecs) {
  const Eig3 e = sym_eig3(m3_from(m), true);
  for (int i = 0; i < 3; ++i) vals[i] = e.val[i];
  m3_to(e.vec, vecs);
  return e.ok ? 0 : 1;
}
void orc_inverse3(const double* m, double* out) { m3_to(inverse3(m3_from(m)), out); }
double orc_det3(const double* m) { return det3(m3_from(m)); }
void orc_tangent_basis(const double* n, double* d1, double* d2) {
  V3 a, b;
  tangent_basis(V3(n[0], n[1], n[2]), a, b);
  for (int i = 0; i < 3; ++i) {
    d1[i] = a[i];
    d2[i] = b[i];
  }
}
double orc_r_factor(double emd, double h, int row_class, int strat) {
  return r_factor(emd, h, static_cast<RowClass>(row_class), static_cast<RStrat>(strat));
}
int orc_lame(double young, double poisson, double* out3) {
  try {
    const NH m = lame(young, poisson);
    out3[0] = m.c1;
    out3[1] = m.d1;
    out3[2] = m.alpha;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
void orc_nh_gradient(const double* s, const double* mat, double* out) {
  const V3 g = nh_gradient(V3(s[0], s[1], s[2]), NH{mat[0], mat[1], mat[2]});
  for (int i = 0; i < 3; ++i) out[i] = g[i];
}
void orc_nh_hessian(const double* s, const double* mat, double* out) {
  m3_to(nh_hessian(V3(s[0], s[1], s[2]), NH{mat[0], mat[1], mat[2]}), out);
}
double orc_nh_energy(const double* s, const double* mat) {
  return nh_energy(V3(s[0], s[1], s[2]), NH{mat[0], mat[1], mat[2]});
}
void orc_compliance_block(double vol, const double* h, int project, int diag, double* out) {
  m3_to(compliance_block(vol, m3_from(h), project != 0, diag != 0), out);
}
// rows: 3 (NH) or 6 (linear); out_c[6], out_jac[6*12], out_comp[36].
int orc_material_rows(int model, double young, double poisson, const double* rest12,
                      const double* pos12, double* out_c, double* out_jac, double* out_comp,
                      double* energy) {
  try {
    TetMesh m;
    m.material.model = static_cast<MatModel>(model);
    m.material.young = young;
    m.material.poisson = poisson;
    m.prepare();
    V3 r[4], p[4];
    for (int k = 0; k < 4; ++k) {
      r[k] = V3(rest12[3 * k], rest12[3 * k + 1], rest12[3 * k + 2]);
      p[k] = V3(pos12[3 * k], pos12[3 * k + 1], pos12[3 * k + 2]);
    }
    const Tet e = make_tet({0, 1, 2, 3}, r[0], r[1], r[2], r[3]);
    const MatRows mr = m.material.model == MatModel::NeoHookean
                           ? neo_hookean_rows(e, m, p[0], p[1], p[2], p[3])
                           : linear_strain_rows(e, m, p[0], p[1], p[2], p[3]);
    for (int i = 0; i < 6; ++i) {
      out_c[i] = mr.c[i];
      for (int k = 0; k < 12; ++k) out_jac[12 * i + k] = mr.jac[i][k];
      for (int k = 0; k < 6; ++k) out_comp[6 * i + k] = mr.comp[i][k];
    }
    *energy = element_energy(e, m, p[0], p[1], p[2], p[3]);
    return mr.dim;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}
// Strain Jacobian from F's SVD for a tet with given dm_inv (row-major).
void orc_strain_jacobian(const double* dm_inv, const double* f, double* out36, double* s_out) {
  Tet e;
  e.dm_inv = m3_from(dm_inv);
  const Svd3 svd = svd3(m3_from(f));
  const J312 j = strain_jacobian(e, svd);
  for (int i = 0; i < 3; ++i) {
    s_out[i] = svd.S[i];
    for (int k = 0; k < 12; ++k) out36[12 * i + k] = j[i][k];
  }
}

// CSR from triplets + solve_linear. Returns 0 ok, 1 invalid argument.
int orc_solve_linear(int n, int nt, const int* rows, const int* cols, const double* vals,
                     const double* b, const double* x0, int method, int max_it, double tol,
                     int precond, double* x_out, double* hist, int* hist_len, double* phist,
                     int* phist_len, int* iters, int* breakdown) {
  try {
    std::vector<Trip> t(nt);
    for (int i = 0; i < nt; ++i) t[i] = {rows[i], cols[i], vals[i]};
    const Csr a = Csr::from_triplets(n, n, t);
    LinCfg c;
    c.method = static_cast<LinMethod>(method);
    c.max_iterations = max_it;
    c.tolerance = tol;
    c.precond = static_cast<Precond>(precond);
    const LinResult r = solve_linear(a, VecX(b, b + n), VecX(x0, x0 + n), c);
    for (int i = 0; i < n; ++i) x_out[i] = r.solution[i];
    *hist_len = static_cast<int>(r.hist.size());
    for (size_t i = 0; i < r.hist.size(); ++i) hist[i] = r.hist[i];
    *phist_len = static_cast<int>(r.phist.size());
    for (size_t i = 0; i < r.phist.size(); ++i) phist[i] = r.phist[i];
    *iters = r.iterations_used;
    *breakdown = r.breakdown ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Minimal body-layer KATs: one body state, integrate/external forces.
// type 0 particle / 1 rigid; q (3/7), u (3/6) in-out.
void orc_body_step_kat(int type, double mass, const double* inertia9, double* q, double* u,
                       const double* gravity, double h, double* f_out, double* ut_out,
                       int integrate_with_ut) {
  State s;
  Body b;
  b.type = static_cast<BodyType>(type);
  b.mass = mass;
  b.inertia = m3_from(inertia9);
  s.bodies = {b};
  s.finalize_layout();
  for (int k = 0; k < s.num_coord; ++k) s.q[k] = q[k];
  for (int k = 0; k < s.num_dof; ++k) s.u[k] = u[k];
  const VecX f = external_forces(s, V3(gravity[0], gravity[1], gravity[2]));
  const VecX ut = unconstrained_velocity(s, f, h);
  for (int k = 0; k < s.num_dof; ++k) {
    f_out[k] = f[k];
    ut_out[k] = ut[k];
  }
  if (integrate_with_ut) {
    integrate(s, ut, h);
  } else {
    integrate(s, VecX(u, u + s.num_dof), h);
  }
  for (int k = 0; k < s.num_coord; ++k) q[k] = s.q[k];
}

// ---------------- world level -------------------------------------------------
void* orc_world_create(const char* name, unsigned seed) {
  try {
    SceneDesc sc;
    if (!build_scene_by_name(name, seed, sc)) {
      g_err = std::string("unknown scene ") + name;
      return nullptr;
    }
    auto* o = new OWorld();
    o->w = build_world(sc);
    return o;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void orc_world_destroy(void* h) { delete static_cast<OWorld*>(h); }

// dims: n_bodies, num_dof, num_coord, n_joints, n_tets, n_shapes, n_contacts,
//       rows_joint, rows_mesh, newton_iters, linear_iters, n_meshes
void orc_world_dims(void* h, int* d) {
  const World& w = static_cast<OWorld*>(h)->w;
  int nt = 0, rj = 0, rm = 0;
  for (const MeshBinding& m : w.meshes) {
    nt += static_cast<int>(m.mesh.elements.size());
    rm += (m.mesh.material.model == MatModel::NeoHookean ? 3 : 6) * static_cast<int>(m.mesh.elements.size());
  }
  for (const Joint& j : w.joints) rj += joint_row_count(j.kind);
  d[0] = static_cast<int>(w.state.bodies.size());
  d[1] = w.state.num_dof;
  d[2] = w.state.num_coord;
  d[3] = static_cast<int>(w.joints.size());
  d[4] = nt;
  d[5] = static_cast<int>(w.shapes.size());
  d[6] = static_cast<int>(w.contacts.size());
  d[7] = rj;
  d[8] = rm;  // newton.cpp:32-33: 3 rows per Neo-Hookean tet, 6 per linear tet
  d[9] = w.solver.newton_iterations;
  d[10] = w.solver.linear.max_iterations;
  d[11] = static_cast<int>(w.meshes.size());
}
double orc_world_h(void* h) { return static_cast<OWorld*>(h)->w.h; }
void orc_world_gravity(void* h, double* g) {
  const World& w = static_cast<OWorld*>(h)->w;
  for (int k = 0; k < 3; ++k) g[k] = w.gravity[k];
}
// cfg: newton_iterations, linear_max, line_search, geometric_stiffness,
//      r_strategy, ncp, precond, linear_method ; dcfg: step_fraction, eps, lin_tol, newton_tol
void orc_world_get_config(void* h, int* icfg, double* dcfg) {
  const NewtonCfg& c = static_cast<OWorld*>(h)->w.solver;
  icfg[0] = c.newton_iterations;
  icfg[1] = c.linear.max_iterations;
  icfg[2] = c.line_search;
  icfg[3] = c.geometric_stiffness;
  icfg[4] = static_cast<int>(c.r_strategy);
  icfg[5] = static_cast<int>(c.ncp);
  icfg[6] = static_cast<int>(c.linear.precond);
  icfg[7] = static_cast<int>(c.linear.method);
  dcfg[0] = c.step_fraction;
  dcfg[1] = c.epsilon_reg;
  dcfg[2] = c.linear.tolerance;
  dcfg[3] = c.newton_tolerance;
}
void orc_world_set_config(void* h, const int* icfg, const double* dcfg) {
  NewtonCfg& c = static_cast<OWorld*>(h)->w.solver;
  c.newton_iterations = icfg[0];
  c.linear.max_iterations = icfg[1];
  c.line_search = icfg[2] != 0;
  c.geometric_stiffness = icfg[3] != 0;
  c.r_strategy = static_cast<RStrat>(icfg[4]);
  c.ncp = static_cast<Ncp>(icfg[5]);
  c.linear.precond = static_cast<Precond>(icfg[6]);
  c.linear.method = static_cast<LinMethod>(icfg[7]);
  c.step_fraction = dcfg[0];
  c.epsilon_reg = dcfg[1];
  c.linear.tolerance = dcfg[2];
  c.newton_tolerance = dcfg[3];
}
void orc_world_get_state(void* h, double* q, double* u) {
  const State& s = static_cast<OWorld*>(h)->w.state;
  std::memcpy(q, s.q.data(), sizeof(double) * s.num_coord);
  std::memcpy(u, s.u.data(), sizeof(double) * s.num_dof);
}
void orc_world_set_state(void* h, const double* q, const double* u) {
  State& s = static_cast<OWorld*>(h)->w.state;
  std::memcpy(s.q.data(), q, sizeof(double) * s.num_coord);
  std::memcpy(s.u.data(), u, sizeof(double) * s.num_dof);
}

// Topology export in the product C-ABI layout (include/nsdyn_gpu.h):
// body_type[nb], body_mass[nb], body_inertia[9nb], joint_kind[nj],
// joint_body[2nj], joint_frame[21nj], joint_param[2nj], tet_body[4nt],
// tet_dm_inv[9nt], tet_volume[nt], tet_material[4nt].
void orc_world_topology(void* hd, int* body_type, double* body_mass, double* body_inertia,
                        int* joint_kind, int* joint_body, double* joint_frame, double* joint_param,
                        int* tet_body, double* tet_dm_inv, double* tet_volume, double* tet_material) {
  const World& w = static_cast<OWorld*>(hd)->w;
  for (size_t b = 0; b < w.state.bodies.size(); ++b) {
    body_type[b] = static_cast<int>(w.state.bodies[b].type);
    body_mass[b] = w.state.bodies[b].mass;
    m3_to(w.state.bodies[b].inertia, body_inertia + 9 * b);
  }
  for (size_t i = 0; i < w.joints.size(); ++i) {
    const Joint& j = w.joints[i];
    joint_kind[i] = static_cast<int>(j.kind);
    joint_body[2 * i] = j.body_a;
    joint_body[2 * i + 1] = j.body_b;
    const V3* f[7] = {&j.anchor_a, &j.anchor_b, &j.axis_a, &j.axis_a2, &j.axis_b1, &j.axis_b2, &j.rest_dots};
    for (int k = 0; k < 7; ++k)
      for (int c = 0; c < 3; ++c) joint_frame[21 * i + 3 * k + c] = (*f[k])[c];
    joint_param[2 * i] = j.compliance;
    joint_param[2 * i + 1] = j.stiffness;
  }
  int t = 0;
  for (const MeshBinding& m : w.meshes) {
    for (const Tet& e : m.mesh.elements) {
      for (int k = 0; k < 4; ++k) tet_body[4 * t + k] = m.particle_base + e.v[k];
      m3_to(e.dm_inv, tet_dm_inv + 9 * t);
      tet_volume[t] = e.vol;
      // flat C-ABI encoding (include/nsdyn_gpu.h): c1 = mu/2, d1 = lambda/2, alpha,
      // flags (1 diagonal compliance, 2 linear co-rotational). For linear meshes the
      // reference keeps only the stiffness (materials.cpp:117-122); its Lame constants
      // are the same expressions lame_from_young_poisson evaluates.
      const NH nh = m.mesh.material.model == MatModel::Linear
                        ? lame(m.mesh.material.young, m.mesh.material.poisson)
                        : m.mesh.nh;
      tet_material[4 * t] = nh.c1;
      tet_material[4 * t + 1] = nh.d1;
      tet_material[4 * t + 2] = nh.alpha;
      tet_material[4 * t + 3] = (m.mesh.material.diagonal_compliance ? 1.0 : 0.0) +
                                (m.mesh.material.model == MatModel::Linear ? 2.0 : 0.0);
      ++t;
    }
  }
}
// Shapes: body[ns], kind[ns], dparam[10 ns] = normal3, offset, radius, half3, thickness, mu.
void orc_world_shapes(void* hd, int* body, int* kind, double* dparam, double* contact_params) {
  const World& w = static_cast<OWorld*>(hd)->w;
  for (size_t i = 0; i < w.shapes.size(); ++i) {
    const AttachedShape& s = w.shapes[i];
    body[i] = s.body;
    kind[i] = static_cast<int>(s.shape.kind);
    double* d = dparam + 10 * i;
    for (int k = 0; k < 3; ++k) d[k] = s.shape.normal[k];
    d[3] = s.shape.offset;
    d[4] = s.shape.radius;
    for (int k = 0; k < 3; ++k) d[5 + k] = s.shape.half_extents[k];
    d[8] = s.shape.thickness;
    d[9] = s.shape.mu;
  }
  contact_params[0] = w.contact_params.margin;
  contact_params[1] = w.contact_params.mu_default;
}

// Contacts layout (nsd_contact-compatible flat doubles, 24 per contact):
// ibuf[4c]: body_a, body_b, feature, 0 ; dbuf[22c]: local_a3, local_b3,
// normal3, d1_3, d2_3, thickness, mu, lambda_n, lambda_f2.
static void export_contacts(const std::vector<Contact>& cs, int* ib, double* db) {
  for (size_t i = 0; i < cs.size(); ++i) {
    const Contact& c = cs[i];
    ib[4 * i] = c.a.body;
    ib[4 * i + 1] = c.b.body;
    ib[4 * i + 2] = c.feature;
    ib[4 * i + 3] = 0;
    double* d = db + 22 * i;
    for (int k = 0; k < 3; ++k) {
      d[k] = c.a.local[k];
      d[3 + k] = c.b.local[k];
      d[6 + k] = c.normal[k];
      d[9 + k] = c.d1[k];
      d[12 + k] = c.d2[k];
    }
    d[15] = c.thickness;
    d[16] = c.mu;
    d[17] = c.lambda_n;
    d[18] = c.lambda_f[0];
    d[19] = c.lambda_f[1];
    d[20] = d[21] = 0.0;
  }
}
// Decision vectors of the last newton step (Report::decisions): up to max_rows rows of
// `stride` bytes; returns the number of rows (Newton iterations run).
int orc_world_decisions(void* hd, unsigned char* out, int stride, int max_rows) {
  OWorld* w = static_cast<OWorld*>(hd);
  const auto& d = w->last.decisions;
  const int n = std::min<int>(static_cast<int>(d.size()), max_rows);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < stride; ++k) out[i * stride + k] = k < static_cast<int>(d[i].size()) ? d[i][k] : 0xff;
  return n;
}

int orc_world_n_contacts(void* h) { return static_cast<int>(static_cast<OWorld*>(h)->w.contacts.size()); }
void orc_world_contacts(void* h, int* ib, double* db) { export_contacts(static_cast<OWorld*>(h)->w.contacts, ib, db); }

// Extension hook: set f_extra from per-joint torques at the current pose (NULL clears).
void orc_world_set_joint_torques(void* h, const double* tau) {
  World& w = static_cast<OWorld*>(h)->w;
  if (!tau) {
    w.f_extra.clear();
    return;
  }
  w.f_extra = joint_torque_forces(w, tau);
}
void orc_world_get_f_extra(void* h, double* f) {
  const World& w = static_cast<OWorld*>(h)->w;
  for (int k = 0; k < w.state.num_dof; ++k) f[k] = w.f_extra.empty() ? 0.0 : w.f_extra[k];
}

// First half of step_world (scene.cpp:710-720): move driven anchors, compute
// u_tilde, run detect. The contact list is then available via orc_world_contacts.
int orc_world_prepare(void* hd) {
  try {
    World& w = static_cast<OWorld*>(hd)->w;
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
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
// Second half: newton_step on the prepared contact set.
int orc_world_newton(void* hd) {
  try {
    OWorld* o = static_cast<OWorld*>(hd);
    World& w = o->w;
    StepCtx ctx;
    ctx.state = &w.state;
    ctx.joints = &w.joints;
    ctx.meshes = &w.meshes;
    ctx.contacts = &w.contacts;
    ctx.gravity = w.gravity;
    ctx.h = w.h;
    ctx.f_extra = w.f_extra.empty() ? nullptr : &w.f_extra;
    o->last = newton_step(ctx, w.solver);
    o->has_report = true;
    w.time += w.h;
    return o->last.aborted ? 2 : 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
int orc_world_step(void* hd, int n) {
  for (int i = 0; i < n; ++i) {
    int rc = orc_world_prepare(hd);
    if (rc) return rc;
    rc = orc_world_newton(hd);
    if (rc) return rc;
  }
  return 0;
}
// Report of the last newton step. stats[8 per iteration]: residual_inf,
// merit_l2, comp_error_max, cone_violation_max, step_size, linear_iterations,
// linear_residual, linear_breakdown. fin[7]: final_residual_inf,
// final_comp_error, final_cone_violation, min_gap, min_diag_shift, aborted,
// converged. hist: n_iter*(max_lin+1), hist_len[n_iter]. tel: 6 per contact.
int orc_world_report(void* hd, double* stats, double* fin, double* hist, int* hist_len, int hist_stride,
                     double* lambda, double* tel) {
  const OWorld* o = static_cast<OWorld*>(hd);
  if (!o->has_report) return -1;
  const Report& r = o->last;
  for (size_t i = 0; i < r.iterations.size(); ++i) {
    const IterStats& s = r.iterations[i];
    double* d = stats + 8 * i;
    d[0] = s.residual_inf;
    d[1] = s.merit_l2;
    d[2] = s.comp_error_max;
    d[3] = s.cone_violation_max;
    d[4] = s.step_size;
    d[5] = s.linear_iterations;
    d[6] = s.linear_residual;
    d[7] = s.linear_breakdown ? 1.0 : 0.0;
  }
  fin[0] = r.final_residual_inf;
  fin[1] = r.final_comp_error;
  fin[2] = r.final_cone_violation;
  fin[3] = r.min_gap;
  fin[4] = r.min_diag_shift;
  fin[5] = r.aborted;
  fin[6] = r.converged;
  for (size_t i = 0; i < r.linear_histories.size(); ++i) {
    hist_len[i] = static_cast<int>(r.linear_histories[i].size());
    for (size_t k = 0; k < r.linear_histories[i].size() && static_cast<int>(k) < hist_stride; ++k)
      hist[i * hist_stride + k] = r.linear_histories[i][k];
  }
  if (lambda)
    for (size_t i = 0; i < r.lambda.size(); ++i) lambda[i] = r.lambda[i];
  if (tel)
    for (size_t i = 0; i < r.contacts.size(); ++i) {
      const ContactTel& t = r.contacts[i];
      double* d = tel + 6 * i;
      d[0] = t.gap;
      d[1] = t.lambda_n;
      d[2] = t.lambda_f_norm;
      d[3] = t.mu;
      d[4] = t.tangential_speed;
      d[5] = t.dissipation_dot;
    }
  return static_cast<int>(r.iterations.size());
}
void orc_world_joint_frames(void* hd, double* frames) {
  const World& w = static_cast<OWorld*>(hd)->w;
  for (size_t i = 0; i < w.joints.size(); ++i) {
    const Joint& j = w.joints[i];
    const V3* f[7] = {&j.anchor_a, &j.anchor_b, &j.axis_a, &j.axis_a2, &j.axis_b1, &j.axis_b2, &j.rest_dots};
    for (int k = 0; k < 7; ++k)
      for (int c = 0; c < 3; ++c) frames[21 * i + 3 * k + c] = (*f[k])[c];
  }
}

// ---------------- CPU baseline (bench.py) ------------------------------------
// Steps n_env independent C5 ant worlds (env ids env0 .. env0+n_env-1) for
// n_steps with OpenMP over environments (inner OpenMP loops stay serial —
// SURVEY §8d). Optional per-step joint torques from mt19937(env*1000003+step)
// U(-1,1). Returns wall seconds of the stepping loop; threads_used out.
// Counter-based U(-1, 1) action for (global env, step, joint): splitmix64 of
// (env << 32) ^ (step << 8) ^ joint, top 53 bits.
static double action_torque(int env, int step, int joint) {
  uint64_t x = (static_cast<uint64_t>(env) << 32) ^ (static_cast<uint64_t>(step) << 8) ^ static_cast<uint64_t>(joint);
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  return static_cast<double>(x >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

double orc_action_torque(int env, int step, int joint) { return action_torque(env, step, joint); }

double orc_c5_bench(int env0, int n_env, int n_warm, int n_steps, int actuated, int threads, int* threads_used,
                    double* checksum) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
  *threads_used = omp_get_max_threads();
#else
  (void)threads;
  *threads_used = 1;
#endif
  std::vector<World> worlds(n_env);
  for (int e = 0; e < n_env; ++e) worlds[e] = build_world(build_c5_ant(static_cast<unsigned>(env0 + e)));
  // steps [0, n_warm) untimed, then [n_warm, n_warm + n_steps) timed: the same
  // trajectory segment bench.py times on the GPU
  auto run = [&](int s0, int s1) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int e = 0; e < n_env; ++e) {
      World& w = worlds[e];
      for (int s = s0; s < s1; ++s) {
        if (actuated) {  // same action stream as paper_1907_04587_b200/shard.py:action_torques
          std::vector<double> tau(w.joints.size());
          for (size_t j = 0; j < tau.size(); ++j) tau[j] = action_torque(env0 + e, s, static_cast<int>(j));
          w.f_extra = joint_torque_forces(w, tau.data());
        }
        (void)step_world(w);
      }
    }
  };
  run(0, n_warm);
  const auto t0 = std::chrono::steady_clock::now();
  run(n_warm, n_warm + n_steps);
  const auto t1 = std::chrono::steady_clock::now();
  double cs = 0.0;
  for (const World& w : worlds)
    for (double v : w.state.q) cs += v;
  *checksum = cs;
  return std::chrono::duration<double>(t1 - t0).count();
}

// The same C5 ants stepped n_steps times (actions as orc_c5_bench), returning each
// env's final q, u (env-major) and contact count: bench.py's end-of-run parity sample.
// perturb > 0: every initial coordinate is scaled by (1 + perturb * N(0, 1)) (seeded by
// pseed and the env id) — the oracle's own sensitivity, for stated tolerances.
int orc_c5_states(int env0, int n_env, int n_steps, int actuated, int threads, double* q_out, double* u_out,
                  int* nc_out, double perturb, unsigned pseed) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
  std::vector<World> worlds(n_env);
  for (int e = 0; e < n_env; ++e) {
    worlds[e] = build_world(build_c5_ant(static_cast<unsigned>(env0 + e)));
    if (perturb > 0.0) {
      std::mt19937_64 rng(pseed * 1000003ull + static_cast<unsigned>(env0 + e));
      std::normal_distribution<double> nd(0.0, 1.0);
      for (double& v : worlds[e].state.q) v *= 1.0 + perturb * nd(rng);
    }
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int e = 0; e < n_env; ++e) {
    World& w = worlds[e];
    for (int s = 0; s < n_steps; ++s) {
      if (actuated) {
        std::vector<double> tau(w.joints.size());
        for (size_t j = 0; j < tau.size(); ++j) tau[j] = action_torque(env0 + e, s, static_cast<int>(j));
        w.f_extra = joint_torque_forces(w, tau.data());
      }
      (void)step_world(w);
    }
  }
  for (int e = 0; e < n_env; ++e) {
    const World& w = worlds[e];
    std::copy(w.state.q.begin(), w.state.q.end(), q_out + e * w.state.q.size());
    std::copy(w.state.u.begin(), w.state.u.end(), u_out + e * w.state.u.size());
    nc_out[e] = static_cast<int>(w.contacts.size());
  }
  return 0;
}


// Runner CSV output (restates src/runner.cpp:13-27, 80-126, 148-180 for the
// GPU-vs-oracle file diff): trajectory.csv + convergence.csv, %.17g. Returns
// the runner's exit code (0 ok, 1 validation error, 2 numerical abort).
static std::string orc_fmt(double v) {
  char b[64];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}
int orc_run(const char* name, unsigned seed, int steps, const char* out_dir) {
  try {
    if (steps < 1) throw std::runtime_error("--steps must be >= 1");
    SceneDesc sd;
    if (!build_scene_by_name(name, seed, sd)) throw std::runtime_error("unknown scene");
    World w = build_world(sd);
    std::string traj = "step,body,qx,qy,qz,q0,q1,q2,q3,ux,uy,uz,wx,wy,wz\n";
    std::string conv =
        "step,newton_iter,residual_inf,comp_error_n_max,cone_violation_max,step_size,linear_iters,"
        "linear_residual_final\n";
    bool aborted = false;
    for (int step = 0; step < steps; ++step) {
      const Report r = step_world(w);
      const State& st = w.state;
      for (size_t b = 0; b < st.bodies.size(); ++b) {
        traj += std::to_string(step) + ',' + std::to_string(b);
        const V3 p = st.position(static_cast<int>(b));
        for (int k = 0; k < 3; ++k) traj += ',' + orc_fmt(p[k]);
        const bool rigid = st.bodies[b].type == BodyType::Rigid;
        if (rigid) {
          const V4 q = st.orientation(static_cast<int>(b));
          for (int k = 0; k < 4; ++k) traj += ',' + orc_fmt(q[k]);
        } else {
          traj += ",1,0,0,0";
        }
        const int d = st.dof_off[b];
        for (int k = 0; k < 3; ++k) traj += ',' + orc_fmt(st.u[d + k]);
        if (rigid)
          for (int k = 0; k < 3; ++k) traj += ',' + orc_fmt(st.u[d + 3 + k]);
        else
          traj += ",0,0,0";
        traj += '\n';
      }
      for (size_t i = 0; i < r.iterations.size(); ++i) {
        const IterStats& it = r.iterations[i];
        conv += std::to_string(step) + ',' + std::to_string(i) + ',' + orc_fmt(it.residual_inf) + ',' +
                orc_fmt(it.comp_error_max) + ',' + orc_fmt(it.cone_violation_max) + ',' + orc_fmt(it.step_size) +
                ',' + std::to_string(it.linear_iterations) + ',' + orc_fmt(it.linear_residual) + '\n';
      }
      if (r.aborted) {
        aborted = true;
        break;
      }
    }
    const std::string dir(out_dir);
    std::FILE* f = std::fopen((dir + "/trajectory.csv").c_str(), "wb");
    if (!f) throw std::runtime_error("cannot write trajectory.csv");
    std::fwrite(traj.data(), 1, traj.size(), f);
    std::fclose(f);
    f = std::fopen((dir + "/convergence.csv").c_str(), "wb");
    if (!f) throw std::runtime_error("cannot write convergence.csv");
    std::fwrite(conv.data(), 1, conv.size(), f);
    std::fclose(f);
    return aborted ? 2 : 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}


// ---------------- KAT entry points (tests/test_oracle_kats.py) --------------------
// A state of nb bodies from arrays: type (0 particle / 1 rigid), mass, inertia
// (9 per body, body frame), q (num_coord) and u (num_dof, may be null).
static State make_state(int nb, const int* type, const double* mass, const double* inertia, const double* q,
                        const double* u) {
  State s;
  for (int b = 0; b < nb; ++b) {
    Body bd;
    bd.type = static_cast<BodyType>(type[b]);
    bd.mass = mass ? mass[b] : 1.0;
    if (inertia) bd.inertia = m3_from(inertia + 9 * b);
    s.bodies.push_back(bd);
  }
  s.finalize_layout();
  if (q)
    for (int k = 0; k < s.num_coord; ++k) s.q[k] = q[k];
  if (u)
    for (int k = 0; k < s.num_dof; ++k) s.u[k] = u[k];
  return s;
}

// bodies.cpp:7-22 layout: dof/coord offsets, totals[2] = {num_dof, num_coord}.
void orc_layout(int nb, const int* type, int* dof_off, int* coord_off, int* totals) {
  const State s = make_state(nb, type, nullptr, nullptr, nullptr, nullptr);
  for (int b = 0; b < nb; ++b) {
    dof_off[b] = s.dof_off[b];
    coord_off[b] = s.coord_off[b];
  }
  totals[0] = s.num_dof;
  totals[1] = s.num_coord;
}

// 0.5 * quaternion_rate_matrix(t) * w (bodies.cpp:39-46).
void orc_quat_rate(const double* t, const double* w, double* out) {
  const V4 r = quat_rate(V4(t[0], t[1], t[2], t[3]), V3(w[0], w[1], w[2]));
  for (int k = 0; k < 4; ++k) out[k] = r[k];
}

// integrate_coordinates (bodies.cpp:78-86) on a state; q in-out. 0 ok, 1 invalid.
int orc_integrate_state(int nb, const int* type, double* q, const double* u, double h) {
  try {
    State s = make_state(nb, type, nullptr, nullptr, q, nullptr);
    integrate(s, VecX(u, u + s.num_dof), h);
    for (int k = 0; k < s.num_coord; ++k) q[k] = s.q[k];
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// BlockDiagMass at q (bodies.cpp:88-198): M v, M^-1 (M v), and the sparse-row
// quadratic form inverse_quadratic(idx, val).
void orc_mass_kat(int nb, const int* type, const double* mass, const double* inertia, const double* q,
                  const double* v, double* mv, double* minv_mv, int nnz, const int* idx, const double* val,
                  double* quad) {
  const State s = make_state(nb, type, mass, inertia, q, nullptr);
  const BlockMass m = mass_matrix(s);
  const VecX a = m.apply(VecX(v, v + s.num_dof));
  const VecX b = m.apply_inverse(a);
  for (int k = 0; k < s.num_dof; ++k) {
    mv[k] = a[k];
    minv_mv[k] = b[k];
  }
  *quad = m.inverse_quadratic(idx, val, nnz);
}

// detect (collision.cpp:239-297) on a fixture: shapes' dparam = normal 3, offset,
// radius, half_extents 3, thickness, mu (11 each). Returns the contact count
// (export layout of orc_world_contacts, at most cap written) or -1.
int orc_detect(int nb, const int* type, const double* mass, const double* inertia, const double* q,
               const double* u_predict, int ns, const int* sbody, const int* skind, const double* sparam, double h,
               double margin, double mu_default, int cap, int* ib, double* db) {
  try {
    const State s = make_state(nb, type, mass, inertia, q, nullptr);
    std::vector<AttachedShape> shapes(ns);
    for (int i = 0; i < ns; ++i) {
      const double* d = sparam + 11 * i;
      shapes[i].body = sbody[i];
      shapes[i].shape.kind = static_cast<ShapeKind>(skind[i]);
      shapes[i].shape.normal = V3(d[0], d[1], d[2]);
      shapes[i].shape.offset = d[3];
      shapes[i].shape.radius = d[4];
      shapes[i].shape.half_extents = V3(d[5], d[6], d[7]);
      shapes[i].shape.thickness = d[8];
      shapes[i].shape.mu = d[9];
    }
    ContactParams p;
    p.margin = margin;
    p.mu_default = mu_default;
    const VecX up = u_predict ? VecX(u_predict, u_predict + s.num_dof) : VecX(s.num_dof, 0.0);
    const std::vector<Contact> cs = detect(s, shapes, up, h, p);
    std::vector<Contact> head(cs.begin(), cs.begin() + std::min<size_t>(cs.size(), static_cast<size_t>(cap)));
    export_contacts(head, ib, db);
    return static_cast<int>(cs.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// contact_gap and contact_normal_row (constraints.cpp:56-91) at q; row dense over the dofs.
double orc_contact_gap_row(int nb, const int* type, const double* q, int a_body, const double* a_local, int b_body,
                           const double* b_local, const double* normal, double thickness, double* row) {
  const State s = make_state(nb, type, nullptr, nullptr, q, nullptr);
  Contact c;
  c.a = {a_body, V3(a_local[0], a_local[1], a_local[2])};
  c.b = {b_body, V3(b_local[0], b_local[1], b_local[2])};
  c.normal = V3(normal[0], normal[1], normal[2]);
  c.thickness = thickness;
  const Row r = contact_normal_row(c, s);
  for (int k = 0; k < s.num_dof; ++k) row[k] = 0.0;
  for (size_t k = 0; k < r.idx.size(); ++k) row[r.idx[k]] += r.val[k];
  return contact_gap(c, s);
}

// bind_joint at q_bind (world anchor, axis; constraints.cpp:222-263), then
// joint_rows at q_eval (:141-220): values, compliances, dense Jacobian rows.
int orc_joint_rows(int kind, double compliance, double stiffness, int nb, const int* type, int body_a, int body_b,
                   const double* q_bind, const double* anchor, const double* axis, const double* q_eval,
                   double* values, double* comp, double* jac) {
  try {
    const State sb = make_state(nb, type, nullptr, nullptr, q_bind, nullptr);
    Joint j;
    j.kind = static_cast<JointKind>(kind);
    j.body_a = body_a;
    j.body_b = body_b;
    j.compliance = compliance;
    j.stiffness = stiffness;
    bind_joint(j, sb, V3(anchor[0], anchor[1], anchor[2]), V3(axis[0], axis[1], axis[2]));
    const State se = make_state(nb, type, nullptr, nullptr, q_eval, nullptr);
    const std::vector<BRow> rows = joint_rows(j, se);
    for (size_t i = 0; i < rows.size(); ++i) {
      values[i] = rows[i].value;
      comp[i] = rows[i].compliance;
      for (int k = 0; k < se.num_dof; ++k) jac[i * se.num_dof + k] = 0.0;
      for (size_t k = 0; k < rows[i].jac.idx.size(); ++k) jac[i * se.num_dof + rows[i].jac.idx[k]] += rows[i].jac.val[k];
    }
    return static_cast<int>(rows.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// SparseMatrix::from_triplets (linalg.cpp:9-40): off[rows+1], idx/val[nnz]. Returns
// nnz, or -1 (invalid_argument).
int orc_csr(int rows, int cols, int nt, const int* r, const int* c, const double* v, int* off, int* idx, double* val,
            int* valid) {
  try {
    std::vector<Trip> t(nt);
    for (int i = 0; i < nt; ++i) t[i] = {r[i], c[i], v[i]};
    const Csr a = Csr::from_triplets(rows, cols, t);
    for (int i = 0; i <= rows; ++i) off[i] = a.off[i];
    for (int i = 0; i < a.nnz(); ++i) {
      idx[i] = a.idx[i];
      val[i] = a.val[i];
    }
    *valid = a.valid() ? 1 : 0;
    return a.nnz();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// y = A x (mode 0: spmv, OpenMP rows; 1: spmv_serial; 2: spmv_transpose) on the
// CSR of the triplets; x has nx entries (a mismatch throws, returns 1).
int orc_spmv(int rows, int cols, int nt, const int* r, const int* c, const double* v, int mode, const double* x,
             int nx, double* y) {
  try {
    std::vector<Trip> t(nt);
    for (int i = 0; i < nt; ++i) t[i] = {r[i], c[i], v[i]};
    const Csr a = Csr::from_triplets(rows, cols, t);
    const VecX xv(x, x + nx);
    const VecX out = mode == 0 ? spmv(a, xv) : (mode == 1 ? spmv_serial(a, xv) : spmv_transpose(a, xv));
    for (size_t i = 0; i < out.size(); ++i) y[i] = out[i];
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// diagonal_preconditioner (solvers.cpp:178-184) of the square CSR of the triplets.
void orc_diag_precond(int n, int nt, const int* r, const int* c, const double* v, double* out) {
  std::vector<Trip> t(nt);
  for (int i = 0; i < nt; ++i) t[i] = {r[i], c[i], v[i]};
  const VecX d = diag_precond(Csr::from_triplets(n, n, t));
  for (int i = 0; i < n; ++i) out[i] = d[i];
}

// deformation_gradient (materials.cpp:23-30) of a tet with rest / current vertices (12 each).
void orc_deformation_gradient(const double* rest12, const double* pos12, double* f9) {
  V3 r[4], p[4];
  for (int k = 0; k < 4; ++k) {
    r[k] = V3(rest12[3 * k], rest12[3 * k + 1], rest12[3 * k + 2]);
    p[k] = V3(pos12[3 * k], pos12[3 * k + 1], pos12[3 * k + 2]);
  }
  const Tet e = make_tet({0, 1, 2, 3}, r[0], r[1], r[2], r[3]);
  m3_to(deformation_gradient(p[0], p[1], p[2], p[3], e), f9);
}

// compute_material_rows (materials.cpp:217-223) over ne disjoint Neo-Hookean tets
// (vertex 4e..4e+3), OpenMP (parallel = 1) or serial: c (3), jac (36), comp (9) per tet.
void orc_material_rows_many(int ne, double young, double poisson, const double* rest, const double* pos,
                            int parallel, double* c, double* jac, double* comp) {
  TetMesh m;
  m.material.model = MatModel::NeoHookean;
  m.material.young = young;
  m.material.poisson = poisson;
  std::vector<V3> p(4 * ne);
  for (int e = 0; e < ne; ++e) {
    V3 r[4];
    for (int k = 0; k < 4; ++k) {
      r[k] = V3(rest[12 * e + 3 * k], rest[12 * e + 3 * k + 1], rest[12 * e + 3 * k + 2]);
      p[4 * e + k] = V3(pos[12 * e + 3 * k], pos[12 * e + 3 * k + 1], pos[12 * e + 3 * k + 2]);
    }
    m.elements.push_back(make_tet({4 * e, 4 * e + 1, 4 * e + 2, 4 * e + 3}, r[0], r[1], r[2], r[3]));
  }
  m.prepare();
  std::vector<MatRows> out;
  compute_material_rows(m, p, out, parallel != 0);
  for (int e = 0; e < ne; ++e)
    for (int i = 0; i < 3; ++i) {
      c[3 * e + i] = out[e].c[i];
      for (int k = 0; k < 12; ++k) jac[36 * e + 12 * i + k] = out[e].jac[i][k];
      for (int k = 0; k < 3; ++k) comp[9 * e + 3 * i + k] = out[e].comp[i][k];
    }
}
}  // extern "C"
