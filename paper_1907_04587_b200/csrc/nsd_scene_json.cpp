// The reference's JSON scene format on the product's scene description:
// parse_scene (validating, unknown keys rejected, errors name the entity:
// "scene error at bodies[0].mass: must be positive") and serialize_scene
// (reference include/nsdyn/scene.h:74-77, src/scene.cpp:1-556). Values, defaults,
// validation order and messages follow the reference; the document model is
// nsd_json.h. Product extensions that the format has no keys for (a mesh's
// initial velocity / positions, the particle contact generator flag) are not
// serialized, as the reference format cannot carry them.
#include "nsd_json.h"
#include "nsd_scene.h"

#include <cmath>
#include <initializer_list>
#include <stdexcept>
#include <string>

namespace nsdw {
namespace {

using nsdj::Value;

[[noreturn]] void fail(const std::string& path, const std::string& what) {
  throw std::runtime_error("scene error at " + path + ": " + what);
}

void only_keys(const Value& obj, std::initializer_list<const char*> allowed, const std::string& path) {
  for (const auto& kv : obj.o) {
    bool ok = false;
    for (const char* k : allowed) ok = ok || kv.first == k;
    if (!ok) fail(path, "unknown key \"" + kv.first + "\"");
  }
}

double num(const Value& v, const std::string& path) {
  if (!v.is_number()) fail(path, "expected a number");
  return v.num();
}
double num_req(const Value& o, const char* k, const std::string& path) {
  const Value* v = o.find(k);
  if (!v) fail(path + "." + k, "missing");
  return num(*v, path + "." + k);
}
double num_opt(const Value& o, const char* k, const std::string& path, double dflt) {
  const Value* v = o.find(k);
  return v ? num(*v, path + "." + k) : dflt;
}
bool bool_opt(const Value& o, const char* k, const std::string& path, bool dflt) {
  const Value* v = o.find(k);
  if (!v) return dflt;
  if (v->kind != Value::Bool) fail(path + "." + k, "expected a boolean");
  return v->b;
}
int int_opt(const Value& o, const char* k, const std::string& path, int dflt) {
  const Value* v = o.find(k);
  if (!v) return dflt;
  if (v->kind != Value::Int) fail(path + "." + k, "expected an integer");
  return static_cast<int>(v->i);
}
std::string str_req(const Value& o, const char* k, const std::string& path) {
  const Value* v = o.find(k);
  if (!v) fail(path + "." + k, "missing");
  if (v->kind != Value::String) fail(path + "." + k, "expected a string");
  return v->s;
}
// the reference reads r_strategy / ncp with get<std::string>() (a type error, not a
// scene error, for other kinds); reported here with the scene path
std::string str_enum(const Value& v, const std::string& path) {
  if (v.kind != Value::String) fail(path, "expected a string");
  return v.s;
}
Vec3 vec3(const Value& v, const std::string& path) {
  if (v.kind != Value::Array || v.a.size() != 3) fail(path, "expected an array of 3 numbers");
  return Vec3{num(v.a[0], path), num(v.a[1], path), num(v.a[2], path)};
}
Vec3 vec3_opt(const Value& o, const char* k, const std::string& path, const Vec3& dflt) {
  const Value* v = o.find(k);
  return v ? vec3(*v, path + "." + k) : dflt;
}
double norm3(const Vec3& a) { return std::sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }

// [w,x,y,z] (normalised; |q| < 1e-300 -> identity, bodies.cpp:52-56) or
// {axis, angle_deg} (axis normalised unless zero, Eigen normalized())
Quat quat(const Value& v, const std::string& path) {
  if (v.kind == Value::Array) {
    if (v.a.size() != 4) fail(path, "expected a quaternion [w,x,y,z]");
    const double w = num(v.a[0], path), x = num(v.a[1], path), y = num(v.a[2], path), z = num(v.a[3], path);
    const double n = std::sqrt(w * w + x * x + y * y + z * z);
    if (n < 1e-300) return Quat{};
    return Quat{w / n, x / n, y / n, z / n};
  }
  if (v.kind == Value::Object) {
    only_keys(v, {"axis", "angle_deg"}, path);
    const Value* ax = v.find("axis");
    if (!ax) fail(path + ".axis", "expected an array of 3 numbers");
    Vec3 a = vec3(*ax, path + ".axis");
    const double sq = a.x * a.x + a.y * a.y + a.z * a.z;
    if (sq > 0.0) {
      const double n = std::sqrt(sq);
      a = Vec3{a.x / n, a.y / n, a.z / n};
    }
    const double half = 0.5 * num_req(v, "angle_deg", path) * M_PI / 180.0;
    return Quat{std::cos(half), std::sin(half) * a.x, std::sin(half) * a.y, std::sin(half) * a.z};
  }
  fail(path, "expected a quaternion array or {axis, angle_deg}");
}

ShapeDesc shape(const Value& o, const std::string& path) {
  if (o.kind != Value::Object) fail(path, "expected an object");
  only_keys(o, {"kind", "normal", "offset", "radius", "half_extents", "thickness", "mu"}, path);
  ShapeDesc s;
  const std::string kind = str_req(o, "kind", path);
  if (kind == "halfspace") {
    s.kind = 0;
    s.normal = vec3_opt(o, "normal", path, Vec3{0, 0, 1});
    const double n = norm3(s.normal);
    if (n < 1e-12) fail(path + ".normal", "zero-length normal");
    s.normal = Vec3{s.normal.x / n, s.normal.y / n, s.normal.z / n};
    s.offset = num_opt(o, "offset", path, 0.0);
  } else if (kind == "sphere") {
    s.kind = 1;
    s.radius = num_req(o, "radius", path);
    if (s.radius <= 0.0) fail(path + ".radius", "must be positive");
  } else if (kind == "box") {
    s.kind = 2;
    const Value* he = o.find("half_extents");
    if (!he) fail(path + ".half_extents", "missing");
    s.half = vec3(*he, path + ".half_extents");
    if (std::fmin(s.half.x, std::fmin(s.half.y, s.half.z)) <= 0.0) fail(path + ".half_extents", "must be positive");
  } else {
    fail(path + ".kind", "unknown shape kind \"" + kind + "\"");
  }
  s.thickness = num_opt(o, "thickness", path, 0.0);
  if (s.thickness < 0.0) fail(path + ".thickness", "must be non-negative");
  s.mu = num_opt(o, "mu", path, -1.0);
  return s;
}

void linear(const Value& o, const std::string& path, nsd_config& c) {
  only_keys(o, {"method", "iterations", "tolerance", "preconditioner"}, path);
  static const char* methods[] = {"jacobi", "gs", "pcg", "pcr"};  // LinearMethod order = nsd_config codes
  const std::string m = str_req(o, "method", path);
  c.linear_method = -1;
  for (int k = 0; k < 4; ++k)
    if (m == methods[k]) c.linear_method = k;
  if (c.linear_method < 0) fail(path + ".method", "unknown method \"" + m + "\"");
  c.linear_max_iterations = int_opt(o, "iterations", path, 40);
  if (c.linear_max_iterations < 1) fail(path + ".iterations", "must be >= 1");
  c.linear_tolerance = num_opt(o, "tolerance", path, 1e-10);
  if (c.linear_tolerance < 0.0) fail(path + ".tolerance", "must be >= 0");
  const std::string p = o.find("preconditioner") ? str_req(o, "preconditioner", path) : std::string("diagonal");
  if (p == "none")
    c.preconditioner = 0;
  else if (p == "diagonal")
    c.preconditioner = 1;
  else
    fail(path + ".preconditioner", "unknown preconditioner \"" + p + "\"");
}

nsd_config solver(const Value& o, const std::string& path) {
  only_keys(o,
            {"newton_iterations", "step_fraction", "epsilon", "geometric_stiffness", "r_strategy", "ncp",
             "newton_tolerance", "line_search", "linear"},
            path);
  nsd_config c;
  nsd_config_default(&c, NSD_FP64);
  c.newton_iterations = int_opt(o, "newton_iterations", path, 8);
  if (c.newton_iterations < 1) fail(path + ".newton_iterations", "must be >= 1");
  c.step_fraction = num_opt(o, "step_fraction", path, 0.75);
  if (c.step_fraction <= 0.0 || c.step_fraction > 1.0) fail(path + ".step_fraction", "must lie in (0, 1]");
  c.epsilon_reg = num_opt(o, "epsilon", path, 1e-6);
  if (c.epsilon_reg < 0.0) fail(path + ".epsilon", "must be >= 0");
  c.geometric_stiffness = bool_opt(o, "geometric_stiffness", path, true) ? 1 : 0;
  c.newton_tolerance = num_opt(o, "newton_tolerance", path, 1e-6);
  c.line_search = bool_opt(o, "line_search", path, false) ? 1 : 0;
  if (const Value* v = o.find("r_strategy")) {
    const std::string r = str_enum(*v, path + ".r_strategy");
    if (r == "identity")
      c.r_strategy = 0;
    else if (r == "h2")
      c.r_strategy = 1;
    else if (r == "effmass")
      c.r_strategy = 2;
    else
      fail(path + ".r_strategy", "unknown strategy \"" + r + "\"");
  }
  if (const Value* v = o.find("ncp")) {
    const std::string n = str_enum(*v, path + ".ncp");
    if (n == "minmap")
      c.ncp_kind = 0;
    else if (n == "fb")
      c.ncp_kind = 1;
    else
      fail(path + ".ncp", "unknown NCP function \"" + n + "\"");
  }
  if (const Value* v = o.find("linear")) linear(*v, path + ".linear", c);
  return c;
}

void material(const Value& o, const std::string& path, MeshSpec& m) {
  only_keys(o, {"model", "young", "poisson", "diagonal_compliance"}, path);
  const std::string model = str_req(o, "model", path);
  if (model == "linear")
    m.linear = true;
  else if (model == "neohookean")
    m.linear = false;
  else
    fail(path + ".model", "unknown material model \"" + model + "\"");
  m.young = num_req(o, "young", path);
  if (m.young <= 0.0) fail(path + ".young", "must be positive");
  m.poisson = num_req(o, "poisson", path);
  if (m.poisson < 0.0 || m.poisson >= 0.4999) fail(path + ".poisson", "must lie in [0, 0.4999)");
  m.diagonal_compliance = bool_opt(o, "diagonal_compliance", path, false);
}

JointAttach attach(const Value& o, const char* body_key, const char* mesh_key, const char* vertex_key,
                   const std::string& path) {
  JointAttach a;
  if (const Value* v = o.find(mesh_key)) {
    if (v->kind != Value::Int) fail(path + "." + mesh_key, "expected an integer");
    a.mesh = static_cast<int>(v->i);
    a.vertex = int_opt(o, vertex_key, path, 0);
  } else {
    a.body = int_opt(o, body_key, path, -1);
  }
  return a;
}

BodySpec body(const Value& b, const std::string& path) {
  const std::string type = str_req(b, "type", path);
  BodySpec d;
  if (type == "particle") {
    only_keys(b, {"type", "position", "velocity", "mass"}, path);
    d.kind = BodyKind::Particle;
    d.pos = vec3_opt(b, "position", path, Vec3{});
    d.vel = vec3_opt(b, "velocity", path, Vec3{});
    d.mass = num_req(b, "mass", path);
    if (d.mass <= 0.0) fail(path + ".mass", "must be positive");
  } else if (type == "rigid") {
    only_keys(b, {"type", "position", "orientation", "velocity", "angular_velocity", "mass", "inertia", "shape"},
              path);
    d.kind = BodyKind::Rigid;
    d.pos = vec3_opt(b, "position", path, Vec3{});
    if (const Value* o = b.find("orientation")) d.rot = quat(*o, path + ".orientation");
    d.vel = vec3_opt(b, "velocity", path, Vec3{});
    d.ang_vel = vec3_opt(b, "angular_velocity", path, Vec3{});
    d.mass = num_req(b, "mass", path);
    if (d.mass <= 0.0) fail(path + ".mass", "must be positive");
    if (const Value* in = b.find("inertia")) {
      if (in->kind != Value::Array || in->a.size() != 3) fail(path + ".inertia", "expected a 3x3 matrix");
      for (int r = 0; r < 3; ++r) {
        const Value& row = in->a[r];
        if (row.kind != Value::Array || row.a.size() != 3) fail(path + ".inertia", "expected a 3x3 matrix");
        for (int c = 0; c < 3; ++c) d.inertia[3 * r + c] = num(row.a[c], path + ".inertia");
      }
      d.has_inertia = true;
    }
    if (const Value* s = b.find("shape")) {
      d.shape = shape(*s, path + ".shape");
      d.has_shape = true;
    }
    if (!d.has_inertia && !d.has_shape) fail(path, "rigid body needs a shape or an explicit inertia");
    if (d.has_shape && d.shape.kind == 0) fail(path + ".shape", "half-spaces must be static bodies");
  } else if (type == "static") {
    only_keys(b, {"type", "shape"}, path);
    d.kind = BodyKind::Static;
    const Value* s = b.find("shape");
    if (!s) fail(path + ".shape", "missing");
    d.shape = shape(*s, path + ".shape");
    d.has_shape = true;
  } else {
    fail(path + ".type", "unknown body type \"" + type + "\"");
  }
  return d;
}

MeshSpec mesh(const Value& m, const std::string& path) {
  only_keys(m, {"vertices", "elements", "material", "density"}, path);
  MeshSpec d;
  const Value* vs = m.find("vertices");
  if (!vs || vs->kind != Value::Array) fail(path + ".vertices", "expected an array");
  for (size_t v = 0; v < vs->a.size(); ++v)
    d.vertices.push_back(vec3(vs->a[v], path + ".vertices[" + std::to_string(v) + "]"));
  const Value* es = m.find("elements");
  if (!es || es->kind != Value::Array) fail(path + ".elements", "expected an array");
  for (size_t e = 0; e < es->a.size(); ++e) {
    const Value& ev = es->a[e];
    const std::string ep = path + ".elements[" + std::to_string(e) + "]";
    if (ev.kind != Value::Array || ev.a.size() != 4) fail(ep, "expected 4 vertex indices");
    std::array<int, 4> idx{};
    for (int k = 0; k < 4; ++k) {
      if (ev.a[k].kind != Value::Int) fail(ep, "expected integer indices");
      idx[k] = static_cast<int>(ev.a[k].i);
      if (idx[k] < 0 || idx[k] >= static_cast<int>(d.vertices.size())) fail(ep, "vertex index out of range");
    }
    d.elements.push_back(idx);
  }
  const Value* mat = m.find("material");
  if (!mat) fail(path + ".material", "missing");
  material(*mat, path + ".material", d);
  d.density = num_opt(m, "density", path, 1000.0);
  if (d.density <= 0.0) fail(path + ".density", "must be positive");
  return d;
}

JointSpecDesc joint(const Value& j, const std::string& path) {
  only_keys(j,
            {"type", "body_a", "body_b", "mesh_a", "vertex_a", "mesh_b", "vertex_b", "anchor", "axis", "compliance",
             "stiffness", "anchor_velocity"},
            path);
  static const char* kinds[] = {"fixed_point", "revolute", "prismatic", "bend_spring"};
  JointSpecDesc d;
  const std::string type = str_req(j, "type", path);
  d.kind = -1;
  for (int k = 0; k < 4; ++k)
    if (type == kinds[k]) d.kind = k;
  if (d.kind < 0) fail(path + ".type", "unknown joint type \"" + type + "\"");
  d.a = attach(j, "body_a", "mesh_a", "vertex_a", path);
  d.b = attach(j, "body_b", "mesh_b", "vertex_b", path);
  d.anchor = vec3_opt(j, "anchor", path, Vec3{});
  d.axis = vec3_opt(j, "axis", path, Vec3{0, 0, 1});
  if (norm3(d.axis) < 1e-12) fail(path + ".axis", "zero-length axis");
  d.compliance = num_opt(j, "compliance", path, 0.0);
  if (d.compliance < 0.0) fail(path + ".compliance", "must be >= 0");
  d.stiffness = num_opt(j, "stiffness", path, 0.0);
  if (d.kind == 3 && d.stiffness <= 0.0) fail(path + ".stiffness", "bend springs need a positive stiffness");
  d.anchor_velocity = vec3_opt(j, "anchor_velocity", path, Vec3{});
  return d;
}

// ------------------------------------------------------------------ serialize
Value v3(const Vec3& a) {
  Value v = Value::array();
  v.push(Value::number(a.x));
  v.push(Value::number(a.y));
  v.push(Value::number(a.z));
  return v;
}
Value shape_json(const ShapeDesc& s) {
  Value o = Value::object();
  if (s.kind == 0) {
    o["kind"] = Value::string("halfspace");
    o["normal"] = v3(s.normal);
    o["offset"] = Value::number(s.offset);
  } else if (s.kind == 1) {
    o["kind"] = Value::string("sphere");
    o["radius"] = Value::number(s.radius);
  } else {
    o["kind"] = Value::string("box");
    o["half_extents"] = v3(s.half);
  }
  if (s.thickness != 0.0) o["thickness"] = Value::number(s.thickness);
  if (s.mu >= 0.0) o["mu"] = Value::number(s.mu);
  return o;
}
Value solver_json(const nsd_config& c) {
  static const char* methods[] = {"jacobi", "gs", "pcg", "pcr"};
  static const char* rs[] = {"identity", "h2", "effmass"};
  Value lin = Value::object();
  lin["method"] = Value::string(methods[c.linear_method & 3]);
  lin["iterations"] = Value::integer(c.linear_max_iterations);
  lin["tolerance"] = Value::number(c.linear_tolerance);
  lin["preconditioner"] = Value::string(c.preconditioner == 1 ? "diagonal" : "none");
  Value o = Value::object();
  o["newton_iterations"] = Value::integer(c.newton_iterations);
  o["step_fraction"] = Value::number(c.step_fraction);
  o["epsilon"] = Value::number(c.epsilon_reg);
  o["geometric_stiffness"] = Value::boolean(c.geometric_stiffness != 0);
  o["r_strategy"] = Value::string(rs[c.r_strategy < 0 || c.r_strategy > 2 ? 2 : c.r_strategy]);
  o["ncp"] = Value::string(c.ncp_kind == 0 ? "minmap" : "fb");
  o["newton_tolerance"] = Value::number(c.newton_tolerance);
  o["line_search"] = Value::boolean(c.line_search != 0);
  o["linear"] = lin;
  return o;
}

}  // namespace

Scene parse_scene(const std::string& text) {
  Value doc;
  try {
    doc = nsdj::parse(text);
  } catch (const std::runtime_error& e) {
    throw std::runtime_error(std::string("scene syntax error: ") + e.what());
  }
  if (doc.kind != Value::Object) throw std::runtime_error("scene error at $: expected an object");
  only_keys(doc, {"gravity", "timestep", "bodies", "joints", "meshes", "contacts", "solver"}, "$");
  Scene sc;
  sc.gravity = vec3_opt(doc, "gravity", "$", Vec3{0, 0, -9.81});
  sc.timestep = num_opt(doc, "timestep", "$", 0.0083);
  if (sc.timestep <= 0.0) fail("$.timestep", "must be positive");
  nsd_config_default(&sc.solver, NSD_FP64);
  if (const Value* bs = doc.find("bodies")) {
    if (bs->kind != Value::Array) fail("$.bodies", "expected an array");
    for (size_t i = 0; i < bs->a.size(); ++i) sc.bodies.push_back(body(bs->a[i], "bodies[" + std::to_string(i) + "]"));
  }
  if (const Value* ms = doc.find("meshes")) {
    if (ms->kind != Value::Array) fail("$.meshes", "expected an array");
    for (size_t i = 0; i < ms->a.size(); ++i) sc.meshes.push_back(mesh(ms->a[i], "meshes[" + std::to_string(i) + "]"));
  }
  if (const Value* js = doc.find("joints")) {
    if (js->kind != Value::Array) fail("$.joints", "expected an array");
    for (size_t i = 0; i < js->a.size(); ++i) sc.joints.push_back(joint(js->a[i], "joints[" + std::to_string(i) + "]"));
  }
  if (const Value* c = doc.find("contacts")) {
    only_keys(*c, {"margin", "mu"}, "$.contacts");
    sc.margin = num_opt(*c, "margin", "$.contacts", 0.01);
    if (sc.margin < 0.0) fail("$.contacts.margin", "must be >= 0");
    sc.mu_default = num_opt(*c, "mu", "$.contacts", 0.5);
    if (sc.mu_default < 0.0) fail("$.contacts.mu", "must be >= 0");
  }
  if (const Value* s = doc.find("solver")) sc.solver = solver(*s, "$.solver");
  // cross references (joints to bodies / mesh vertices)
  const int nb = static_cast<int>(sc.bodies.size()), nm = static_cast<int>(sc.meshes.size());
  for (size_t i = 0; i < sc.joints.size(); ++i) {
    const std::string path = "joints[" + std::to_string(i) + "]";
    for (const JointAttach* at : {&sc.joints[i].a, &sc.joints[i].b}) {
      if (at->mesh >= 0) {
        if (at->mesh >= nm) fail(path, "mesh index out of range");
        if (at->vertex < 0 || at->vertex >= static_cast<int>(sc.meshes[at->mesh].vertices.size()))
          fail(path, "mesh vertex index out of range");
      } else if (at->body >= nb) {
        fail(path, "body index out of range");
      } else if (at->body >= 0 && sc.bodies[at->body].kind == BodyKind::Static) {
        fail(path, "joints cannot attach to static bodies; use body -1 for the world");
      }
    }
  }
  return sc;
}

std::string serialize_scene(const Scene& sc) {
  Value doc = Value::object();
  doc["gravity"] = v3(sc.gravity);
  doc["timestep"] = Value::number(sc.timestep);
  Value bodies = Value::array();
  for (const BodySpec& b : sc.bodies) {
    Value o = Value::object();
    if (b.kind == BodyKind::Particle) {
      o["type"] = Value::string("particle");
      o["position"] = v3(b.pos);
      o["velocity"] = v3(b.vel);
      o["mass"] = Value::number(b.mass);
    } else if (b.kind == BodyKind::Rigid) {
      o["type"] = Value::string("rigid");
      o["position"] = v3(b.pos);
      Value q = Value::array();
      for (double c : {b.rot.w, b.rot.x, b.rot.y, b.rot.z}) q.push(Value::number(c));
      o["orientation"] = q;
      o["velocity"] = v3(b.vel);
      o["angular_velocity"] = v3(b.ang_vel);
      o["mass"] = Value::number(b.mass);
      if (b.has_inertia) {
        Value m = Value::array();
        for (int r = 0; r < 3; ++r) m.push(v3(Vec3{b.inertia[3 * r], b.inertia[3 * r + 1], b.inertia[3 * r + 2]}));
        o["inertia"] = m;
      }
      if (b.has_shape) o["shape"] = shape_json(b.shape);
    } else {
      o["type"] = Value::string("static");
      o["shape"] = shape_json(b.shape);
    }
    bodies.push(o);
  }
  doc["bodies"] = bodies;
  Value meshes = Value::array();
  for (const MeshSpec& m : sc.meshes) {
    Value o = Value::object();
    Value vs = Value::array(), es = Value::array();
    for (const Vec3& v : m.vertices) vs.push(v3(v));
    for (const auto& e : m.elements) {
      Value ev = Value::array();
      for (int k = 0; k < 4; ++k) ev.push(Value::integer(e[k]));
      es.push(ev);
    }
    o["vertices"] = vs;
    o["elements"] = es;
    Value mat = Value::object();
    mat["model"] = Value::string(m.linear ? "linear" : "neohookean");
    mat["young"] = Value::number(m.young);
    mat["poisson"] = Value::number(m.poisson);
    if (m.diagonal_compliance) mat["diagonal_compliance"] = Value::boolean(true);
    o["material"] = mat;
    o["density"] = Value::number(m.density);
    meshes.push(o);
  }
  doc["meshes"] = meshes;
  static const char* kinds[] = {"fixed_point", "revolute", "prismatic", "bend_spring"};
  Value joints = Value::array();
  for (const JointSpecDesc& j : sc.joints) {
    Value o = Value::object();
    o["type"] = Value::string(kinds[j.kind & 3]);
    auto att = [&](const JointAttach& a, const char* bk, const char* mk, const char* vk) {
      if (a.mesh >= 0) {
        o[mk] = Value::integer(a.mesh);
        o[vk] = Value::integer(a.vertex);
      } else {
        o[bk] = Value::integer(a.body);
      }
    };
    att(j.a, "body_a", "mesh_a", "vertex_a");
    att(j.b, "body_b", "mesh_b", "vertex_b");
    o["anchor"] = v3(j.anchor);
    o["axis"] = v3(j.axis);
    o["compliance"] = Value::number(j.compliance);
    if (j.stiffness != 0.0) o["stiffness"] = Value::number(j.stiffness);
    if (j.anchor_velocity.x != 0.0 || j.anchor_velocity.y != 0.0 || j.anchor_velocity.z != 0.0)
      o["anchor_velocity"] = v3(j.anchor_velocity);
    joints.push(o);
  }
  doc["joints"] = joints;
  Value contacts = Value::object();
  contacts["margin"] = Value::number(sc.margin);
  contacts["mu"] = Value::number(sc.mu_default);
  doc["contacts"] = contacts;
  doc["solver"] = solver_json(sc.solver);
  return nsdj::dump(doc, 2) + "\n";
}

}  // namespace nsdw
