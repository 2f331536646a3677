// ORACLE — test infrastructure only (tests/, __graft_entry__.smoke(), bench.py
// cpu_baseline / --impl reference). Never linked into the product path.
//
// CPU double-precision restatement of the reference nsdyn solver
// (/root/reference/proj, which cannot be built here: Eigen3, doctest, CLI11 and
// json.hpp are absent — SURVEY.md §0, §8c). Each declaration cites the
// reference interface it restates. The restatement keeps the reference's
// algorithms on purpose, including the explicit Schur-complement build with its
// triplet sort (src/newton.cpp:242-290) and the O(#bodies) block searches
// (src/bodies.cpp:126-132,155-162), so it doubles as the CPU timing baseline.
//
// Parity status: the Newton step itself is "parity unpinned" by any reference
// test (test_newton.cpp is missing, proj/tests/CMakeLists.txt:9-12). Its
// sub-functions are pinned by the reference's own doctest cases, ported as
// known-answer tests in tests/test_oracle_kats.py.
#pragma once

#include "omath.h"

#include <array>
#include <string>
#include <utility>
#include <vector>

namespace orc {

// ---- linalg (include/nsdyn/linalg.h:18-56) --------------------------------
struct Trip {
  int row = 0, col = 0;
  double value = 0.0;
};

struct Csr {
  int rows = 0, cols = 0;
  std::vector<int> off, idx;
  std::vector<double> val;
  static Csr from_triplets(int rows, int cols, std::vector<Trip> t);  // linalg.cpp:9-40
  static Csr identity(int n);
  int nnz() const { return static_cast<int>(val.size()); }
  VecX diagonal() const;
  bool valid() const;
};
VecX spmv(const Csr& a, const VecX& x);            // linalg.cpp:74-85 (OpenMP rows)
VecX spmv_serial(const Csr& a, const VecX& x);     // linalg.cpp:87-97
VecX spmv_transpose(const Csr& a, const VecX& x);  // linalg.cpp:99-108

Svd3 svd3(const M3& f);          // linalg.cpp:110-126 (signed: det U = det V = +1)
M3 project_psd3(const M3& m);    // linalg.cpp:128-134

// ---- solvers (include/nsdyn/solvers.h) --------------------------------------
enum class LinMethod { Jacobi = 0, GaussSeidel = 1, PCG = 2, PCR = 3 };
enum class Precond { None = 0, Diagonal = 1 };
struct LinCfg {
  LinMethod method = LinMethod::PCR;
  int max_iterations = 40;
  double tolerance = 1e-10;
  Precond precond = Precond::Diagonal;
};
struct LinResult {
  VecX solution;
  std::vector<double> hist;   // residual_history
  std::vector<double> phist;  // precond_residual_history
  int iterations_used = 0;
  bool breakdown = false;
  int exit_reason = 0;  // decision vector: 0 budget, 1 tolerance, 2 monotone guard, 3 breakdown
};
VecX diag_precond(const Csr& a);                                                  // solvers.cpp:178-184
LinResult solve_linear(const Csr& a, const VecX& b, const VecX& x0, const LinCfg& c);  // :186-206

// ---- bodies (include/nsdyn/bodies.h) -----------------------------------------
enum class BodyType { Particle = 0, Rigid = 1 };
struct Body {
  BodyType type = BodyType::Particle;
  double mass = 1.0;
  M3 inertia = M3::identity();
  int ndof() const { return type == BodyType::Particle ? 3 : 6; }
  int ncoord() const { return type == BodyType::Particle ? 3 : 7; }
};
struct State {
  std::vector<Body> bodies;
  VecX q, u;
  std::vector<int> dof_off, coord_off;
  int num_dof = 0, num_coord = 0;
  void finalize_layout();  // bodies.cpp:7-22
  V3 position(int b) const;
  void set_position(int b, const V3& p);
  V4 orientation(int b) const;
  void set_orientation(int b, const V4& t);
  M3 rotation(int b) const;
  V3 linear_velocity(int b) const;
  V3 angular_velocity(int b) const;
  V3 world_point(int b, const V3& local) const;
  M3 world_inertia(int b) const;
};
V4 normalized_quat(const V4& t);                                          // bodies.cpp:52-56
V4 quat_rate(const V4& t, const V3& w);  // 0.5 * quaternion_rate_matrix(t) * w, bodies.cpp:39-46
void integrate_from(State& s, const VecX& q_from, const VecX& u_new, double h);  // :78-86
void integrate(State& s, const VecX& u_new, double h);

struct MassBlock {
  BodyType type;
  int dof_off;
  double mass;
  M3 iw, iw_inv;
};
struct BlockMass {  // bodies.h:65-84
  std::vector<MassBlock> blocks;
  VecX shift;
  int num_dof = 0;
  VecX diagonal() const;
  VecX apply(const VecX& v) const;
  VecX apply_inverse(const VecX& v) const;
  double inverse_quadratic(const int* idx, const double* val, int nnz) const;
  void apply_inverse_sparse(const int* idx, const double* val, int nnz, double* out) const;
};
BlockMass mass_matrix(const State& s);                                  // bodies.cpp:179-198
VecX external_forces(const State& s, const V3& gravity);                // :200-212
VecX unconstrained_velocity(const State& s, const VecX& f, double h);   // :214-217

// ---- ncp (include/nsdyn/ncp.h) -------------------------------------------------
enum class Ncp { MinMap = 0, FB = 1 };
struct Phi {
  double value = 0.0, d_c = 0.0, d_l = 0.0;
};
Phi phi_n(double c, double lambda, double r, Ncp k);                     // ncp.cpp:7-32
double friction_W(double vt, double lf, double mln, double r, Ncp k);   // ncp.cpp:34-49

// ---- constraints (include/nsdyn/constraints.h) ---------------------------------
struct Row {  // GenRow
  std::vector<int> idx;
  std::vector<double> val;
  void add(int i, double v) {
    idx.push_back(i);
    val.push_back(v);
  }
  void add3(int off, const V3& v) {
    for (int k = 0; k < 3; ++k) add(off + k, v[k]);
  }
  double dot(const VecX& x) const;
  void compress();
};
struct Attach {
  int body = -1;
  V3 local;
};
struct Contact {  // ContactConstraint, constraints.h:40-50
  Attach a, b;
  V3 normal = V3(0, 0, 1);
  double thickness = 0.0, mu = 0.0;
  V3 d1 = V3(1, 0, 0), d2 = V3(0, 1, 0);
  double lambda_n = 0.0;
  double lambda_f[2] = {0.0, 0.0};
  int feature = 0;
};
V3 attach_point(const State& s, const Attach& p);
void add_point_jac(Row& r, const State& s, const Attach& p, const V3& d, double sign);
double contact_gap(const Contact& c, const State& s);
Row contact_normal_row(const Contact& c, const State& s);
void contact_tangent_rows(const Contact& c, const State& s, Row& t1, Row& t2);
void tangent_basis(const V3& n, V3& d1, V3& d2);  // constraints.cpp:93-101
enum class RStrat { Identity = 0, H2 = 1, EffMass = 2 };
enum class RowClass { Position = 0, Velocity = 1 };
double r_factor(double emd, double h, RowClass rc, RStrat st);  // constraints.cpp:103-115

enum class JointKind { FixedPoint = 0, Revolute = 1, Prismatic = 2, BendSpring = 3 };
struct Joint {  // JointSpec, constraints.h:72-86
  JointKind kind = JointKind::FixedPoint;
  int body_a = -1, body_b = -1;
  V3 anchor_a, anchor_b;
  V3 axis_a = V3(0, 0, 1), axis_a2 = V3(1, 0, 0), axis_b1 = V3(1, 0, 0), axis_b2 = V3(0, 1, 0);
  double compliance = 0.0, stiffness = 0.0;
  V3 rest_dots;
  V3 anchor_velocity;
};
struct BRow {
  double value = 0.0;
  Row jac;
  double compliance = 0.0;
};
std::vector<BRow> joint_rows(const Joint& j, const State& s);                      // :141-220
void bind_joint(Joint& j, const State& s, const V3& world_anchor, const V3& world_axis);  // :222-263
int joint_row_count(JointKind k);

// ---- materials (include/nsdyn/materials.h) -------------------------------------
struct Tet {
  std::array<int, 4> v{};
  M3 dm_inv = M3::identity();
  double vol = 0.0;
};
Tet make_tet(const std::array<int, 4>& v, const V3& r0, const V3& r1, const V3& r2, const V3& r3);
M3 deformation_gradient(const V3& p0, const V3& p1, const V3& p2, const V3& p3, const Tet& e);
struct NH {
  double c1 = 0.0, d1 = 0.0, alpha = 1.0;
};
NH lame(double young, double poisson);  // materials.cpp:32-43
using M6 = std::array<std::array<double, 6>, 6>;
M6 isotropic_stiffness(double young, double poisson);
M6 inverse6(const M6& a);
V3 nh_gradient(const V3& s, const NH& m);
M3 nh_hessian(const V3& s, const NH& m);
double nh_energy(const V3& s, const NH& m);
M3 compliance_block(double vol, const M3& hess, bool project = true, bool diag = false,
                    unsigned char* flags = nullptr);  // :82-102; flags: 1 PSD projected, 2 diagonal fallback
using J312 = std::array<std::array<double, 12>, 3>;
J312 strain_jacobian(const Tet& e, const Svd3& svd);  // :104-114
enum class MatModel { Linear = 0, NeoHookean = 1 };
struct MatSpec {
  MatModel model = MatModel::NeoHookean;
  double young = 1e5, poisson = 0.45;
  bool diagonal_compliance = false;
};
struct MatRows {
  int dim = 3;
  unsigned char flags = 0;  // decision vector: compliance_block's PSD projection / diagonal fallback
  double c[6] = {0, 0, 0, 0, 0, 0};
  double jac[6][12] = {};
  double comp[6][6] = {};
};
struct TetMesh {
  std::vector<Tet> elements;
  MatSpec material;
  NH nh;
  M6 stiffness{}, stiffness_inv{};
  void prepare();
};
MatRows linear_strain_rows(const Tet& e, const TetMesh& m, const V3& p0, const V3& p1, const V3& p2,
                           const V3& p3);
MatRows neo_hookean_rows(const Tet& e, const TetMesh& m, const V3& p0, const V3& p1, const V3& p2,
                         const V3& p3);
double element_energy(const Tet& e, const TetMesh& m, const V3& p0, const V3& p1, const V3& p2,
                      const V3& p3);
void compute_material_rows(const TetMesh& m, const std::vector<V3>& pos, std::vector<MatRows>& out,
                           bool parallel = true);

// ---- newton (include/nsdyn/newton.h) -------------------------------------------
struct NewtonCfg {
  int newton_iterations = 8;
  double step_fraction = 0.75;
  double epsilon_reg = 1e-6;
  bool geometric_stiffness = true;
  RStrat r_strategy = RStrat::EffMass;
  Ncp ncp = Ncp::FB;
  LinCfg linear;
  double newton_tolerance = 1e-6;
  bool line_search = false;
  bool record_iterates = false;
};
struct MeshBinding {
  TetMesh mesh;
  int particle_base = 0;
};
struct NSystem {
  Csr j;
  std::vector<Trip> c_blocks;
  VecX g, h_vec;
  BlockMass h_mass;
  int num_rows = 0;
  double comp_error_max = 0.0, cone_violation_max = 0.0, min_gap = 0.0;
  std::vector<unsigned char> cflags, tflags;  // decision vectors (nsd_step_out::decisions layout)
};
struct IterStats {
  double residual_inf = 0, merit_l2 = 0, comp_error_max = 0, cone_violation_max = 0, step_size = 0;
  int linear_iterations = 0;
  double linear_residual = 0;
  bool linear_breakdown = false;
};
struct ContactTel {
  double gap = 0, lambda_n = 0, lambda_f_norm = 0, mu = 0, tangential_speed = 0, dissipation_dot = 0;
};
struct Report {
  std::vector<IterStats> iterations;
  std::vector<std::vector<double>> linear_histories;
  std::vector<VecX> delta_u;
  std::vector<ContactTel> contacts;
  double final_residual_inf = 0, final_comp_error = 0, final_cone_violation = 0, min_gap = 0,
         min_diag_shift = 0;
  bool aborted = false, converged = false;
  VecX lambda;  // oracle extra: the step's final multipliers in row layout
  // oracle extra: per Newton iteration [contacts][tets][dofs][PCR exit] decision bytes,
  // the layout of nsd_step_out::decisions (include/nsdyn_gpu.h)
  std::vector<std::vector<unsigned char>> decisions;
};
struct StepCtx {
  State* state = nullptr;
  const std::vector<Joint>* joints = nullptr;
  const std::vector<MeshBinding>* meshes = nullptr;
  std::vector<Contact>* contacts = nullptr;
  V3 gravity = V3(0, 0, -9.81);
  double h = 0.0083;
  const VecX* f_extra = nullptr;  // extension (SURVEY §7 hard part 6): extra generalized force
};
struct Layout {
  int joint_begin = 0, mesh_begin = 0, normal_begin = 0, friction_begin = 0, total = 0;
};
Layout make_layout(const StepCtx& ctx);  // newton.cpp:18-41
NSystem assemble(const StepCtx& ctx, const BlockMass& mass, const VecX& u_tilde, const VecX& u,
                 const VecX& lambda, const VecX& shift, const NewtonCfg& cfg);  // :100-231
struct SchurRes {
  VecX dlambda, du;
  LinResult linear;
};
SchurRes schur_solve(const NSystem& sys, const NewtonCfg& cfg);  // :233-297
VecX gs_shifts(const VecX& g_prev, const VecX& g_curr, const BlockMass& m, const VecX& du);
VecX gs_policy(const State& s, const VecX& shifts);
Report newton_step(const StepCtx& ctx, const NewtonCfg& cfg);  // :321-418

// ---- collision (include/nsdyn/collision.h) --------------------------------------
enum class ShapeKind { HalfSpace = 0, Sphere = 1, Box = 2 };
struct Shape {
  ShapeKind kind = ShapeKind::Sphere;
  V3 normal = V3(0, 0, 1);
  double offset = 0.0, radius = 0.5;
  V3 half_extents = V3(0.5, 0.5, 0.5);
  double thickness = 0.0, mu = -1.0;
};
struct AttachedShape {
  int body = -1;
  Shape shape;
};
struct ContactParams {
  double margin = 0.01, mu_default = 0.5;
};
std::vector<Contact> detect(const State& s, const std::vector<AttachedShape>& shapes,
                            const VecX& u_predict, double h, const ContactParams& p);  // collision.cpp:239-297

// ---- world (include/nsdyn/scene.h:89-110) -----------------------------------------
// Caller-side particle contact generator (extension): a
// particle block against static half-spaces / rigid boxes, using detect's
// predicted-gap rule (collision.cpp:275-286).
struct ParticleContactGen {
  int first_body = 0, count = 0;  // particle body range
  double thickness = 0.0, mu = -1.0;
};
struct World {
  State state;
  std::vector<AttachedShape> shapes;
  std::vector<Joint> joints;
  std::vector<MeshBinding> meshes;
  std::vector<Contact> contacts;
  V3 gravity = V3(0, 0, -9.81);
  double h = 0.0083;
  ContactParams contact_params;
  NewtonCfg solver;
  std::vector<std::pair<int, V3>> driven_anchors;
  double time = 0.0;
  std::vector<ParticleContactGen> particle_gens;  // extension
  VecX f_extra;                                    // extension: constant per step unless reset
};
std::vector<Contact> world_contacts(const World& w, const VecX& u_tilde);
Report step_world(World& w);  // scene.cpp:709-732

// ---- scene description + builders (include/nsdyn/scene.h:11-87) -------------------
enum class BodyDescKind { Particle = 0, Rigid = 1, Static = 2 };
struct BodyDesc {
  BodyDescKind kind = BodyDescKind::Rigid;
  V3 position, velocity, angular_velocity;
  V4 orientation = V4(1, 0, 0, 0);
  double mass = 1.0;
  bool has_inertia = false;
  M3 inertia;
  bool has_shape = false;
  Shape shape;
};
struct JointAttach {
  int body = -1, mesh = -1, vertex = 0;
};
struct JointDesc {
  JointKind kind = JointKind::FixedPoint;
  JointAttach a, b;
  V3 anchor, axis = V3(0, 0, 1);
  double compliance = 0.0, stiffness = 0.0;
  V3 anchor_velocity;
};
struct MeshDesc {
  std::vector<V3> vertices;
  std::vector<std::array<int, 4>> elements;
  MatSpec material;
  double density = 1000.0;
  V3 velocity;  // extension: initial velocity of every mesh particle (reference: zero)
  std::vector<V3> initial;  // extension: initial positions if non-empty (reference: the rest vertices)
};
struct SceneDesc {
  V3 gravity = V3(0, 0, -9.81);
  double timestep = 0.0083;
  std::vector<BodyDesc> bodies;
  std::vector<JointDesc> joints;
  std::vector<MeshDesc> meshes;
  ContactParams contacts;
  NewtonCfg solver;
  std::vector<ParticleContactGen> particle_gens;  // extension; body ranges resolved at build
  std::vector<int> particle_gen_mesh;             // mesh index per generator
};
World build_world(const SceneDesc& s);  // scene.cpp:587-707
void tessellate_grid(MeshDesc& m, int nx, int ny, int nz, const V3& origin, const V3& size);

// Reference builders (scene.cpp:802-935) and the synthetic BASELINE configs
// (SURVEY.md Appendix C).
SceneDesc build_box_on_plane();
SceneDesc build_incline(double angle_deg, double mu);
SceneDesc build_heavy_stack();
SceneDesc build_arch();
SceneDesc build_box_pile(unsigned seed);
SceneDesc build_stretch_sheet(MatModel model);
SceneDesc build_c1_box_stack();
SceneDesc build_c2_fem_block(int n = 12);
SceneDesc build_c3_chain(int links = 100);
// C4 initial ball speed (m/s, downward); "c4:<n>:<speed>" overrides it.
constexpr double kC4Drive = 0.02;  // fingertip drive speed (m/s); 0.05 squeezes the ball unstable by step 29
constexpr double kC4Speed = 0.2;  // 1.0 m/s blows up at step 4 (8 mm Neo-Hookean elements, 6x50 budget)
constexpr double kC4Scale = 2.0;  // ball radius 0.05 * scale (0.1 m); "c4:<n>:<speed>:<scale>". At 1.0 the 8 mm
                                  // elements blow up by step 13-28 under the 6 x 50 budget; 2.0 is stable (45 steps)
SceneDesc build_c4_hand_ball(int n = 12, double speed = kC4Speed, double scale = kC4Scale);
SceneDesc build_c5_ant(unsigned env_id);
bool build_scene_by_name(const std::string& name, unsigned seed, SceneDesc& out);

// C5 actuation hook (extension): joint torques -> generalized force at the
// current pose. Revolute joints only: +tau*axis on body a, -tau*axis on body b.
VecX joint_torque_forces(const World& w, const double* tau);

}  // namespace orc
