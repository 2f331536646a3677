// C++ user of the host API (include/nsdyn_b200.hpp): the reference's
// build_scene_by_name -> step_world loop (tools/main.cpp / runner.cpp style),
// with the Newton step on the GPU. Used by tests/test_cpp_api.py.
//
//   world_demo <scene> <seed> <steps> [fp32|fp64]   trajectory: per-step lines + final q, u
//   world_demo --free-fall                          newton_step on a hand-built StepContext
//   world_demo --invalid-h                          h <= 0 must throw std::invalid_argument
//   world_demo --run <scene> <steps> <out_dir> [seed] [ncp] [r]   runner: trajectory.csv + convergence.csv
//   world_demo --sweep <scene> <axis> <steps> <out_dir>   runner: sweep.csv
#include "nsdyn_b200.hpp"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <sstream>
#include <fstream>
#include <string>

namespace nb = nsdyn_b200;

static int free_fall() {
  // no constraints, one Newton iteration -> u equals u~ = u + h g.
  nb::GeneralizedState s;
  s.bodies.push_back(nb::Body{nb::BodyType::Particle, 2.0, nb::kIdentity3});
  nb::Body r;
  r.type = nb::BodyType::Rigid;
  r.mass = 1.0;
  r.inertia = {0.1, 0, 0, 0, 0.2, 0, 0, 0, 0.3};
  s.bodies.push_back(r);
  s.finalize_layout();
  s.set_position(0, {0, 0, 1});
  s.set_position(1, {1, 0, 1});
  s.set_orientation(1, {1, 0, 0, 0});
  s.u[0] = 0.5;
  std::vector<nb::JointSpec> joints;
  std::vector<nb::MeshBinding> meshes;
  std::vector<nb::ContactConstraint> contacts;
  nb::StepContext ctx;
  ctx.state = &s;
  ctx.joints = &joints;
  ctx.meshes = &meshes;
  ctx.contacts = &contacts;
  ctx.h = 0.01;
  nb::NewtonConfig cfg;
  cfg.newton_iterations = 1;
  cfg.step_fraction = 1.0;  // undamped: one full Newton step from the zero start lands on u~
  const nb::SolveReport rep = nb::newton_step(ctx, cfg);
  const double uz = -9.81 * 0.01;
  const bool ok = !rep.aborted && rep.iterations.size() == 1 && s.u[0] == 0.5 && s.u[2] == uz && s.u[5] == uz &&
                  std::abs(s.q[2] - (1.0 + 0.01 * uz)) < 1e-15 && nb::count_rows(ctx) == 0;
  std::printf("free_fall %s u0 %.17g uz %.17g z %.17g\n", ok ? "ok" : "FAIL", s.u[0], s.u[2], s.q[2]);
  return ok ? 0 : 1;
}

static int invalid_h() {
  auto w = nb::build_scene_by_name("c1", 0);
  w->h = 0.0;
  try {
    nb::step_world(*w);
  } catch (const std::invalid_argument& e) {
    std::printf("invalid_argument ok: %s\n", e.what());
    return 0;
  }
  std::printf("FAIL: no exception\n");
  return 1;
}

static int run_cmd(int argc, char** argv) {
  nb::RunOptions o;
  o.scene = argv[2];
  o.steps = std::atoi(argv[3]);
  o.out_dir = argv[4];
  if (argc > 5) o.seed = static_cast<unsigned>(std::atoi(argv[5]));
  if (argc > 6) o.ncp = std::string(argv[6]);
  if (argc > 7) o.r_strategy = std::string(argv[7]);
  std::string err;
  const int rc = nb::run(o, &err);
  std::printf("run rc %d %s\n", rc, err.c_str());
  return rc;
}

static int sweep_cmd(char** argv) {
  nb::RunOptions o;
  o.scene = argv[2];
  o.steps = std::atoi(argv[4]);
  o.out_dir = argv[5];
  std::string err;
  const int rc = nb::sweep(o, argv[3], &err);
  std::printf("sweep rc %d %s\n", rc, err.c_str());
  return rc;
}

// JSON scene format through the C++ API (no GPU needed): serialize_scene of a builder
// world, world_from_json of that text, serialize again; prints the document and
// whether the rebuilt world matches (state, joints, bodies).
int json_roundtrip(const char* name) {
  auto w = nb::build_scene_by_name(name, 0);
  if (!w) return 2;
  const std::string doc = nb::serialize_scene(*w);
  const nb::World v = nb::world_from_json(doc);
  const std::string doc2 = nb::serialize_scene(v);
  // orientations are renormalised on parse (bodies.cpp:52-56): one rounding apart at most
  bool same = doc.size() == doc2.size() && v.state.bodies.size() == w->state.bodies.size() &&
              v.joints.size() == w->joints.size() && v.state.u == w->state.u && v.h == w->h;
  for (size_t i = 0; same && i < v.state.q.size(); ++i) same = std::fabs(v.state.q[i] - w->state.q[i]) <= 1e-15;
  std::fputs(doc.c_str(), stdout);
  std::printf("json_roundtrip %s\n", same ? "ok" : "MISMATCH");
  return same ? 0 : 1;
}

// world_from_json of a file; prints the validation message of a rejected document.
int json_load(const char* path) {
  std::ifstream in(path, std::ios::binary);
  std::stringstream ss;
  ss << in.rdbuf();
  try {
    const nb::World w = nb::world_from_json(ss.str());
    std::printf("json_load ok bodies %zu joints %zu\n", w.state.bodies.size(), w.joints.size());
    return 0;
  } catch (const std::runtime_error& e) {
    std::printf("json_error %s\n", e.what());
    return 1;
  }
}

int main(int argc, char** argv) {
  if (argc >= 3 && std::strcmp(argv[1], "--json-roundtrip") == 0) return json_roundtrip(argv[2]);
  if (argc >= 3 && std::strcmp(argv[1], "--json-load") == 0) return json_load(argv[2]);
  if (argc >= 5 && std::strcmp(argv[1], "--run") == 0) return run_cmd(argc, argv);
  if (argc >= 6 && std::strcmp(argv[1], "--sweep") == 0) return sweep_cmd(argv);
  if (argc >= 2 && std::strcmp(argv[1], "--free-fall") == 0) return free_fall();
  if (argc >= 2 && std::strcmp(argv[1], "--invalid-h") == 0) return invalid_h();
  if (argc < 4) {
    std::fprintf(stderr, "usage: world_demo <scene> <seed> <steps> [fp32|fp64]\n");
    return 2;
  }
  auto w = nb::build_scene_by_name(argv[1], static_cast<unsigned>(std::atoi(argv[2])));
  if (!w) {
    std::fprintf(stderr, "unknown scene %s\n", argv[1]);
    return 2;
  }
  if (argc >= 5) w->solver.precision = std::strcmp(argv[4], "fp32") == 0 ? nb::Precision::FP32 : nb::Precision::FP64;
  const int steps = std::atoi(argv[3]);
  for (int i = 0; i < steps; ++i) {
    const nb::SolveReport r = nb::step_world(*w);
    int lin = 0;
    for (const auto& it : r.iterations) lin += it.linear_iterations;
    std::printf("step %d contacts %zu aborted %d newton %zu pcr %d residual %.17g min_gap %.17g\n", i,
                w->contacts.size(), r.aborted ? 1 : 0, r.iterations.size(), lin, r.final_residual_inf, r.min_gap);
  }
  std::printf("q");
  for (double v : w->state.q) std::printf(" %.17g", v);
  std::printf("\nu");
  for (double v : w->state.u) std::printf(" %.17g", v);
  std::printf("\n");
  return 0;
}
