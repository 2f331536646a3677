// Host-side scene layer of the product: scene descriptions, builders for the
// reference's desk scenes and the BASELINE configs C1-C5, and build_world
// (reference: include/nsdyn/scene.h:11-110, src/scene.cpp:556-935). The world
// is kept in the flat C-ABI layout (nsd_topology + packed q/u + nsd_shape).
#pragma once

#include "nsdyn_gpu.h"

#include <array>
#include <string>
#include <utility>
#include <vector>

namespace nsdw {

struct Vec3 {
  double x = 0, y = 0, z = 0;
};
struct Quat {
  double w = 1, x = 0, y = 0, z = 0;
};

struct ShapeDesc {
  int kind = 1;  // 0 half-space, 1 sphere, 2 box
  Vec3 normal{0, 0, 1};
  double offset = 0.0, radius = 0.5;
  Vec3 half{0.5, 0.5, 0.5};
  double thickness = 0.0, mu = -1.0;
};

enum class BodyKind { Particle, Rigid, Static };

struct BodySpec {
  BodyKind kind = BodyKind::Rigid;
  Vec3 pos, vel, ang_vel;
  Quat rot;
  double mass = 1.0;
  bool has_inertia = false;
  double inertia[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  bool has_shape = false;
  ShapeDesc shape;
};

struct JointAttach {
  int body = -1, mesh = -1, vertex = 0;
};

struct JointSpecDesc {
  int kind = 0;  // 0 fixed point, 1 revolute, 2 prismatic, 3 bend spring
  JointAttach a, b;
  Vec3 anchor, axis{0, 0, 1};
  double compliance = 0.0, stiffness = 0.0;
  Vec3 anchor_velocity;
};

struct MeshSpec {
  std::vector<Vec3> vertices;                 // rest shape
  std::vector<std::array<int, 4>> elements;
  double young = 1e5, poisson = 0.45, density = 1000.0;
  bool diagonal_compliance = false;
  bool linear = false;                        // MaterialModel::Linear (co-rotational, 6 rows per tet)
  Vec3 velocity;                              // extension: initial velocity
  std::vector<Vec3> initial;                  // extension: initial positions
  bool particle_contacts = false;             // extension: caller-side contact generator
};

struct Scene {
  Vec3 gravity{0, 0, -9.81};
  double timestep = 0.0083;
  std::vector<BodySpec> bodies;
  std::vector<JointSpecDesc> joints;
  std::vector<MeshSpec> meshes;
  double margin = 0.01, mu_default = 0.5;
  nsd_config solver{};
};

struct World {
  // topology (flat, C-ABI layout)
  std::vector<int32_t> body_type;
  std::vector<double> body_mass, body_inertia;
  std::vector<int32_t> joint_kind, joint_body;
  std::vector<double> joint_frame, joint_param;
  std::vector<int32_t> tet_body;
  std::vector<double> tet_dm_inv, tet_volume, tet_material;
  std::vector<int> dof_off, coord_off;
  int num_dof = 0, num_coord = 0;
  // state
  std::vector<double> q, u;
  // collision
  std::vector<nsd_shape> shapes;
  double margin = 0.01, mu_default = 0.5;
  std::vector<std::pair<int, int>> particle_ranges;  // (first body, count) for the generator
  std::vector<std::pair<int, Vec3>> driven;          // (joint, anchor velocity)
  Vec3 gravity;
  double h = 0.0083;
  nsd_config solver{};

  nsd_topology topology() const;
};

Scene build(const std::string& name, unsigned seed, bool* ok);
World build_world(const Scene& s);
// The reference's JSON scene format (scene.h:74-77; nsd_scene_json.cpp). parse_scene
// throws std::runtime_error with the reference's messages.
Scene parse_scene(const std::string& text);
std::string serialize_scene(const Scene& s);

}  // namespace nsdw
