// ORACLE — test infrastructure only. CPU restatement of the reference's
// L0/L1 layers: proj/src/linalg.cpp, solvers.cpp, bodies.cpp, ncp.cpp,
// constraints.cpp, materials.cpp. Citations are to /root/reference/proj.
#include "oracle.h"

#include <stdexcept>

namespace orc {

// ============================ linalg =========================================

// src/linalg.cpp:9-40 — range check, sort by (row, col) with std::sort (same
// comparator, so equal-key summation order matches a libstdc++ build), sum
// duplicates, prefix-sum row counts.
Csr Csr::from_triplets(int rows, int cols, std::vector<Trip> t) {
  for (const Trip& e : t)
    if (e.row < 0 || e.row >= rows || e.col < 0 || e.col >= cols)
      throw std::invalid_argument("sparse triplet out of range");
  std::sort(t.begin(), t.end(), [](const Trip& a, const Trip& b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });
  Csr m;
  m.rows = rows;
  m.cols = cols;
  m.off.assign(rows + 1, 0);
  m.idx.reserve(t.size());
  m.val.reserve(t.size());
  size_t i = 0;
  while (i < t.size()) {
    size_t j = i;
    double acc = 0.0;
    while (j < t.size() && t[j].row == t[i].row && t[j].col == t[i].col) acc += t[j++].value;
    m.idx.push_back(t[i].col);
    m.val.push_back(acc);
    m.off[t[i].row + 1]++;
    i = j;
  }
  for (int r = 0; r < rows; ++r) m.off[r + 1] += m.off[r];
  return m;
}

Csr Csr::identity(int n) {
  Csr m;
  m.rows = m.cols = n;
  m.off.resize(n + 1);
  m.idx.resize(n);
  m.val.assign(n, 1.0);
  for (int i = 0; i <= n; ++i) m.off[i] = i;
  for (int i = 0; i < n; ++i) m.idx[i] = i;
  return m;
}

VecX Csr::diagonal() const {
  VecX d(rows, 0.0);
  for (int r = 0; r < rows; ++r)
    for (int k = off[r]; k < off[r + 1]; ++k)
      if (idx[k] == r) d[r] = val[k];
  return d;
}

bool Csr::valid() const {
  if (static_cast<int>(off.size()) != rows + 1) return false;
  if (off.front() != 0 || off.back() != nnz()) return false;
  for (int r = 0; r < rows; ++r) {
    if (off[r] > off[r + 1]) return false;
    for (int k = off[r]; k < off[r + 1]; ++k) {
      if (idx[k] < 0 || idx[k] >= cols) return false;
      if (k > off[r] && idx[k] <= idx[k - 1]) return false;
    }
  }
  return true;
}

VecX spmv(const Csr& a, const VecX& x) {
  if (static_cast<int>(x.size()) != a.cols) throw std::invalid_argument("spmv: dimension mismatch");
  VecX y(a.rows);
#pragma omp parallel for schedule(static)
  for (int r = 0; r < a.rows; ++r) {
    double s = 0.0;
    for (int k = a.off[r]; k < a.off[r + 1]; ++k) s += a.val[k] * x[a.idx[k]];
    y[r] = s;
  }
  return y;
}

VecX spmv_serial(const Csr& a, const VecX& x) {
  if (static_cast<int>(x.size()) != a.cols) throw std::invalid_argument("spmv: dimension mismatch");
  VecX y(a.rows);
  for (int r = 0; r < a.rows; ++r) {
    double s = 0.0;
    for (int k = a.off[r]; k < a.off[r + 1]; ++k) s += a.val[k] * x[a.idx[k]];
    y[r] = s;
  }
  return y;
}

VecX spmv_transpose(const Csr& a, const VecX& x) {
  if (static_cast<int>(x.size()) != a.rows)
    throw std::invalid_argument("spmv_transpose: dimension mismatch");
  VecX y(a.cols, 0.0);
  for (int r = 0; r < a.rows; ++r) {
    const double xr = x[r];
    for (int k = a.off[r]; k < a.off[r + 1]; ++k) y[a.idx[k]] += a.val[k] * xr;
  }
  return y;
}

// src/linalg.cpp:110-126: Eigen JacobiSVD, then push reflections onto s3.
Svd3 svd3(const M3& f) {
  Svd3 r = jacobi_svd3(f);
  if (det3(r.U) < 0.0) {
    for (int i = 0; i < 3; ++i) r.U(i, 2) = -r.U(i, 2);
    r.S[2] = -r.S[2];
  }
  if (det3(r.V) < 0.0) {
    for (int i = 0; i < 3; ++i) r.V(i, 2) = -r.V(i, 2);
    r.S[2] = -r.S[2];
  }
  return r;
}

// src/linalg.cpp:128-134.
M3 project_psd3(const M3& m) {
  const Eig3 e = sym_eig3(m, true);
  V3 ev = e.val;
  const double fl = 1e-10 * std::max(std::abs(ev[0]), std::max(std::abs(ev[1]), std::abs(ev[2])));
  for (int i = 0; i < 3; ++i) ev[i] = std::max(ev[i], fl);
  // V diag(ev) V^T
  M3 vd;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) vd(i, j) = e.vec(i, j) * ev[j];
  return vd * e.vec.t();
}

// ============================ solvers ========================================
namespace {
constexpr double kBreak = 1e-300;  // src/solvers.cpp:10

double vnorm(const VecX& v) {
  double s = 0.0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}
double vdot(const VecX& a, const VecX& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
VecX pre(const VecX& inv, const VecX& v) {
  if (inv.empty()) return v;
  VecX o(v.size());
  for (size_t i = 0; i < v.size(); ++i) o[i] = inv[i] * v[i];
  return o;
}
double pnorm(const VecX& inv, const VecX& r) {
  if (inv.empty()) return vnorm(r);
  double s = 0.0;
  for (size_t i = 0; i < r.size(); ++i) s += r[i] * (inv[i] * r[i]);
  return std::sqrt(s);
}
VecX residual(const Csr& a, const VecX& b, const VecX& x) {
  VecX ax = spmv(a, x), r(b.size());
  for (size_t i = 0; i < b.size(); ++i) r[i] = b[i] - ax[i];
  return r;
}

struct Best {
  VecX x;
  double res = std::numeric_limits<double>::infinity();
  void offer(const VecX& c, double r) {
    if (r < res) {
      res = r;
      x = c;
    }
  }
};

LinResult run_jacobi(const Csr& a, const VecX& b, const VecX& x0, const LinCfg& cfg) {
  LinResult out;
  const VecX inv = diag_precond(a);
  VecX x = x0, r = residual(a, b, x);
  Best best;
  best.offer(x, vnorm(r));
  out.hist.push_back(vnorm(r));
  for (int it = 0; it < cfg.max_iterations && out.hist.back() > cfg.tolerance; ++it) {
    for (size_t i = 0; i < x.size(); ++i) x[i] += inv[i] * r[i];
    r = residual(a, b, x);
    out.hist.push_back(vnorm(r));
    best.offer(x, vnorm(r));
    out.iterations_used = it + 1;
  }
  out.solution = best.x;
  return out;
}

LinResult run_gs(const Csr& a, const VecX& b, const VecX& x0, const LinCfg& cfg) {
  LinResult out;
  VecX x = x0, r = residual(a, b, x);
  Best best;
  best.offer(x, vnorm(r));
  out.hist.push_back(vnorm(r));
  for (int it = 0; it < cfg.max_iterations && out.hist.back() > cfg.tolerance; ++it) {
    for (int row = 0; row < a.rows; ++row) {
      double s = b[row], d = 0.0;
      for (int k = a.off[row]; k < a.off[row + 1]; ++k) {
        if (a.idx[k] == row)
          d = a.val[k];
        else
          s -= a.val[k] * x[a.idx[k]];
      }
      if (std::abs(d) > kBreak) x[row] = s / d;
    }
    r = residual(a, b, x);
    out.hist.push_back(vnorm(r));
    best.offer(x, vnorm(r));
    out.iterations_used = it + 1;
  }
  out.solution = best.x;
  return out;
}

LinResult run_pcg(const Csr& a, const VecX& b, const VecX& x0, const LinCfg& cfg, const VecX& inv) {
  LinResult out;
  VecX x = x0, r = residual(a, b, x);
  Best best;
  best.offer(x, vnorm(r));
  out.hist.push_back(vnorm(r));
  out.phist.push_back(pnorm(inv, r));
  VecX z = pre(inv, r), p = z;
  double rz = vdot(r, z);
  for (int it = 0; it < cfg.max_iterations && out.hist.back() > cfg.tolerance; ++it) {
    const VecX ap = spmv(a, p);
    const double pap = vdot(p, ap);
    if (std::abs(pap) < kBreak) {
      out.breakdown = true;
      break;
    }
    const double alpha = rz / pap;
    for (size_t i = 0; i < x.size(); ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * ap[i];
    }
    out.hist.push_back(vnorm(r));
    out.phist.push_back(pnorm(inv, r));
    best.offer(x, vnorm(r));
    out.iterations_used = it + 1;
    z = pre(inv, r);
    const double rz_new = vdot(r, z);
    if (std::abs(rz) < kBreak) {
      out.breakdown = true;
      break;
    }
    const double beta = rz_new / rz;
    for (size_t i = 0; i < p.size(); ++i) p[i] = z[i] + beta * p[i];
    rz = rz_new;
  }
  out.solution = best.x;
  return out;
}

// src/solvers.cpp:127-174.
LinResult run_pcr(const Csr& a, const VecX& b, const VecX& x0, const LinCfg& cfg, const VecX& inv) {
  LinResult out;
  const size_t n = b.size();
  VecX x = x0, r = residual(a, b, x);
  Best best;
  best.offer(x, vnorm(r));
  out.hist.push_back(vnorm(r));
  out.phist.push_back(pnorm(inv, r));
  VecX z = pre(inv, r), p = z, az = spmv(a, z), ap = az;
  double zaz = vdot(z, az);
  VecX xn(n), rn(n);
  for (int it = 0; it < cfg.max_iterations && out.hist.back() > cfg.tolerance; ++it) {
    const VecX map = pre(inv, ap);
    const double den = vdot(ap, map);
    if (std::abs(den) < kBreak) {
      out.breakdown = true;
      break;
    }
    const double alpha = zaz / den;
    for (size_t i = 0; i < n; ++i) {
      xn[i] = x[i] + alpha * p[i];
      rn[i] = r[i] - alpha * ap[i];
    }
    const double pn = pnorm(inv, rn);
    if (pn > out.phist.back()) {
      out.exit_reason = 2;
      break;
    }
    x = xn;
    r = rn;
    out.hist.push_back(vnorm(r));
    out.phist.push_back(pn);
    best.offer(x, vnorm(r));
    out.iterations_used = it + 1;
    for (size_t i = 0; i < n; ++i) z[i] -= alpha * map[i];
    const VecX az_new = spmv(a, z);
    const double zaz_new = vdot(z, az_new);
    if (std::abs(zaz) < kBreak) {
      out.breakdown = true;
      break;
    }
    const double beta = zaz_new / zaz;
    for (size_t i = 0; i < n; ++i) {
      p[i] = z[i] + beta * p[i];
      ap[i] = az_new[i] + beta * ap[i];
    }
    zaz = zaz_new;
  }
  if (out.breakdown)
    out.exit_reason = 3;
  else if (out.exit_reason != 2)
    out.exit_reason = out.hist.back() <= cfg.tolerance ? 1 : 0;
  out.solution = best.x;
  return out;
}
}  // namespace

VecX diag_precond(const Csr& a) {
  if (a.rows != a.cols) throw std::invalid_argument("diagonal_preconditioner: matrix not square");
  const VecX d = a.diagonal();
  VecX inv(d.size());
  for (size_t i = 0; i < d.size(); ++i) inv[i] = d[i] > 0.0 ? 1.0 / d[i] : 1.0;
  return inv;
}

LinResult solve_linear(const Csr& a, const VecX& b, const VecX& x0, const LinCfg& cfg) {
  if (a.rows != a.cols || static_cast<int>(b.size()) != a.rows ||
      static_cast<int>(x0.size()) != a.cols)
    throw std::invalid_argument("solve_linear: dimension mismatch");
  if (cfg.max_iterations < 1) throw std::invalid_argument("solve_linear: max_iterations < 1");
  VecX inv;
  if (cfg.precond == Precond::Diagonal) inv = diag_precond(a);
  const auto classify = [&](LinResult r) {  // decision vector exit reason (no monotone guard)
    r.exit_reason = r.breakdown ? 3 : (!r.hist.empty() && r.hist.back() <= cfg.tolerance ? 1 : 0);
    return r;
  };
  switch (cfg.method) {
    case LinMethod::Jacobi: return classify(run_jacobi(a, b, x0, cfg));
    case LinMethod::GaussSeidel: return classify(run_gs(a, b, x0, cfg));
    case LinMethod::PCG: return classify(run_pcg(a, b, x0, cfg, inv));
    case LinMethod::PCR: return run_pcr(a, b, x0, cfg, inv);
  }
  throw std::logic_error("solve_linear: unknown method");
}

// ============================ bodies =========================================

void State::finalize_layout() {  // src/bodies.cpp:7-22
  dof_off.clear();
  coord_off.clear();
  num_dof = num_coord = 0;
  for (const Body& b : bodies) {
    dof_off.push_back(num_dof);
    coord_off.push_back(num_coord);
    num_dof += b.ndof();
    num_coord += b.ncoord();
  }
  q.assign(num_coord, 0.0);
  u.assign(num_dof, 0.0);
  for (size_t i = 0; i < bodies.size(); ++i)
    if (bodies[i].type == BodyType::Rigid) q[coord_off[i] + 3] = 1.0;
}
V3 State::position(int b) const {
  const int o = coord_off[b];
  return {q[o], q[o + 1], q[o + 2]};
}
void State::set_position(int b, const V3& p) {
  for (int k = 0; k < 3; ++k) q[coord_off[b] + k] = p[k];
}
V4 State::orientation(int b) const {
  const int o = coord_off[b] + 3;
  return {q[o], q[o + 1], q[o + 2], q[o + 3]};
}
void State::set_orientation(int b, const V4& t) {
  for (int k = 0; k < 4; ++k) q[coord_off[b] + 3 + k] = t[k];
}
M3 State::rotation(int b) const {
  if (bodies[b].type == BodyType::Particle) return M3::identity();
  return quat_to_rot(orientation(b));
}
V3 State::linear_velocity(int b) const {
  const int o = dof_off[b];
  return {u[o], u[o + 1], u[o + 2]};
}
V3 State::angular_velocity(int b) const {
  const int o = dof_off[b] + 3;
  return {u[o], u[o + 1], u[o + 2]};
}
V3 State::world_point(int b, const V3& local) const {
  if (bodies[b].type == BodyType::Particle) return position(b);
  return position(b) + rotation(b) * local;
}
M3 State::world_inertia(int b) const {
  const M3 r = rotation(b);
  return (r * bodies[b].inertia) * r.t();
}

V4 normalized_quat(const V4& t) {
  const double n = norm(t);
  if (n < 1e-300) return V4(1, 0, 0, 0);
  return V4(t[0] / n, t[1] / n, t[2] / n, t[3] / n);
}

// 0.5 * Q(theta) * omega with Q from src/bodies.cpp:39-46.
V4 quat_rate(const V4& t, const V3& w) {
  const double q[4][3] = {{-t[1], -t[2], -t[3]},
                          {t[0], t[3], -t[2]},
                          {-t[3], t[0], t[1]},
                          {t[2], -t[1], t[0]}};
  V4 r;
  for (int i = 0; i < 4; ++i) r[i] = 0.5 * (q[i][0] * w[0] + q[i][1] * w[1] + q[i][2] * w[2]);
  return r;
}

// src/bodies.cpp:58-86: rates from the state's current coordinates, then
// q = q_from + h*rates, then renormalise the quaternions.
void integrate_from(State& s, const VecX& q_from, const VecX& u_new, double h) {
  if (h <= 0.0) throw std::invalid_argument("integrate_coordinates: h must be positive");
  VecX rates(s.num_coord, 0.0);
  for (size_t i = 0; i < s.bodies.size(); ++i) {
    const int cd = s.coord_off[i], vd = s.dof_off[i];
    for (int k = 0; k < 3; ++k) rates[cd + k] = u_new[vd + k];
    if (s.bodies[i].type == BodyType::Rigid) {
      const V4 qr = quat_rate(s.orientation(static_cast<int>(i)),
                              V3(u_new[vd + 3], u_new[vd + 4], u_new[vd + 5]));
      for (int k = 0; k < 4; ++k) rates[cd + 3 + k] = qr[k];
    }
  }
  for (int k = 0; k < s.num_coord; ++k) s.q[k] = q_from[k] + h * rates[k];
  for (size_t i = 0; i < s.bodies.size(); ++i)
    if (s.bodies[i].type == BodyType::Rigid)
      s.set_orientation(static_cast<int>(i), normalized_quat(s.orientation(static_cast<int>(i))));
}
void integrate(State& s, const VecX& u_new, double h) {
  const VecX q0 = s.q;
  integrate_from(s, q0, u_new, h);
}

VecX BlockMass::diagonal() const {
  VecX d(num_dof, 0.0);
  for (const MassBlock& b : blocks) {
    for (int k = 0; k < 3; ++k) d[b.dof_off + k] = b.mass;
    if (b.type == BodyType::Rigid)
      for (int k = 0; k < 3; ++k) d[b.dof_off + 3 + k] = b.iw(k, k);
  }
  for (int k = 0; k < num_dof; ++k) d[k] += shift[k];
  return d;
}
VecX BlockMass::apply(const VecX& v) const {
  VecX o(num_dof);
  for (const MassBlock& b : blocks) {
    for (int k = 0; k < 3; ++k) o[b.dof_off + k] = v[b.dof_off + k] * (b.mass + shift[b.dof_off + k]);
    if (b.type == BodyType::Rigid) {
      const V3 w = b.iw * V3(v[b.dof_off + 3], v[b.dof_off + 4], v[b.dof_off + 5]);
      for (int k = 0; k < 3; ++k) o[b.dof_off + 3 + k] = w[k];
    }
  }
  return o;
}
VecX BlockMass::apply_inverse(const VecX& v) const {
  VecX o(num_dof);
  for (const MassBlock& b : blocks) {
    for (int k = 0; k < 3; ++k) o[b.dof_off + k] = v[b.dof_off + k] / (b.mass + shift[b.dof_off + k]);
    if (b.type == BodyType::Rigid) {
      const V3 w = b.iw_inv * V3(v[b.dof_off + 3], v[b.dof_off + 4], v[b.dof_off + 5]);
      for (int k = 0; k < 3; ++k) o[b.dof_off + 3 + k] = w[k];
    }
  }
  return o;
}

namespace {
// Linear scan over all blocks, as src/bodies.cpp:126-132 / 155-162 do.
const MassBlock* find_block(const std::vector<MassBlock>& blocks, int dof) {
  for (const MassBlock& b : blocks) {
    const int ext = b.type == BodyType::Particle ? 3 : 6;
    if (dof >= b.dof_off && dof < b.dof_off + ext) return &b;
  }
  return nullptr;
}
}  // namespace

void BlockMass::apply_inverse_sparse(const int* idx, const double* val, int nnz, double* out) const {
  int k = 0;
  while (k < nnz) {
    const MassBlock* blk = find_block(blocks, idx[k]);
    const int ext = blk->type == BodyType::Particle ? 3 : 6;
    const int start = k;
    double loc[6] = {0, 0, 0, 0, 0, 0};
    while (k < nnz && idx[k] < blk->dof_off + ext) {
      loc[idx[k] - blk->dof_off] = val[k];
      ++k;
    }
    double res[6] = {0, 0, 0, 0, 0, 0};
    for (int c = 0; c < 3; ++c) res[c] = loc[c] / (blk->mass + shift[blk->dof_off + c]);
    if (blk->type == BodyType::Rigid) {
      const V3 w = blk->iw_inv * V3(loc[3], loc[4], loc[5]);
      for (int c = 0; c < 3; ++c) res[3 + c] = w[c];
    }
    for (int m = start; m < k; ++m) out[m] = res[idx[m] - blk->dof_off];
  }
}

double BlockMass::inverse_quadratic(const int* idx, const double* val, int nnz) const {
  double sum = 0.0;
  int k = 0;
  while (k < nnz) {
    const MassBlock* blk = find_block(blocks, idx[k]);
    const int ext = blk->type == BodyType::Particle ? 3 : 6;
    double loc[6] = {0, 0, 0, 0, 0, 0};
    while (k < nnz && idx[k] < blk->dof_off + ext) {
      loc[idx[k] - blk->dof_off] = val[k];
      ++k;
    }
    for (int c = 0; c < 3; ++c) sum += loc[c] * loc[c] / (blk->mass + shift[blk->dof_off + c]);
    if (blk->type == BodyType::Rigid) {
      const V3 ang(loc[3], loc[4], loc[5]);
      sum += dot(ang, blk->iw_inv * ang);
    }
  }
  return sum;
}

BlockMass mass_matrix(const State& s) {  // src/bodies.cpp:179-198
  BlockMass m;
  m.num_dof = s.num_dof;
  m.shift.assign(s.num_dof, 0.0);
  for (size_t i = 0; i < s.bodies.size(); ++i) {
    MassBlock b;
    b.type = s.bodies[i].type;
    b.dof_off = s.dof_off[i];
    b.mass = s.bodies[i].mass;
    if (b.type == BodyType::Rigid) {
      b.iw = s.world_inertia(static_cast<int>(i));
      b.iw_inv = inverse3(b.iw);
    } else {
      b.iw = b.iw_inv = M3::identity();
    }
    m.blocks.push_back(b);
  }
  return m;
}

VecX external_forces(const State& s, const V3& g) {  // src/bodies.cpp:200-212
  VecX f(s.num_dof, 0.0);
  for (size_t i = 0; i < s.bodies.size(); ++i) {
    const int vd = s.dof_off[i];
    const V3 fg = s.bodies[i].mass * g;
    for (int k = 0; k < 3; ++k) f[vd + k] = fg[k];
    if (s.bodies[i].type == BodyType::Rigid) {
      const V3 w = s.angular_velocity(static_cast<int>(i));
      const M3 iw = s.world_inertia(static_cast<int>(i));
      const V3 t = -cross(w, iw * w);
      for (int k = 0; k < 3; ++k) f[vd + 3 + k] = t[k];
    }
  }
  return f;
}

VecX unconstrained_velocity(const State& s, const VecX& f, double h) {
  const BlockMass m = mass_matrix(s);
  const VecX mf = m.apply_inverse(f);
  VecX u(s.num_dof);
  for (int k = 0; k < s.num_dof; ++k) u[k] = s.u[k] + h * mf[k];
  return u;
}

// ============================ ncp ============================================

Phi phi_n(double c, double lambda, double r, Ncp kind) {  // src/ncp.cpp:7-32
  Phi o;
  const double rl = r * lambda;
  if (kind == Ncp::MinMap) {
    if (c <= rl) {
      o.value = c;
      o.d_c = 1.0;
      o.d_l = 0.0;
    } else {
      o.value = rl;
      o.d_c = 0.0;
      o.d_l = r;
    }
    return o;
  }
  const double root = std::sqrt(c * c + rl * rl);
  o.value = c + rl - root;
  if (root == 0.0) {
    o.d_c = 0.0;
    o.d_l = r;
  } else {
    o.d_c = 1.0 - c / root;
    o.d_l = (1.0 - rl / root) * r;
  }
  return o;
}

double friction_W(double vt, double lf, double mln, double r, Ncp kind) {  // src/ncp.cpp:34-49
  const double degenerate = 1e-12, cap = 1e12;
  if (kind == Ncp::MinMap) {
    if (vt <= r * (mln - lf)) return 0.0;
    if (mln <= degenerate) return cap;
    return (vt - r * (mln - lf)) / mln;
  }
  const double slack = mln - lf;
  const double root = std::sqrt(vt * vt + r * r * slack * slack);
  const double numer = root - r * slack;
  const double denom = vt + r * mln - root;
  if (denom <= degenerate) return cap;
  return r * numer / denom;
}

// ============================ constraints ====================================

double Row::dot(const VecX& x) const {
  double s = 0.0;
  for (size_t k = 0; k < idx.size(); ++k) s += val[k] * x[idx[k]];
  return s;
}

void Row::compress() {  // src/constraints.cpp:24-42
  std::vector<size_t> order(idx.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return idx[a] < idx[b]; });
  std::vector<int> ni;
  std::vector<double> nv;
  for (size_t k = 0; k < order.size(); ++k) {
    const int i = idx[order[k]];
    const double v = val[order[k]];
    if (!ni.empty() && ni.back() == i)
      nv.back() += v;
    else {
      ni.push_back(i);
      nv.push_back(v);
    }
  }
  idx = std::move(ni);
  val = std::move(nv);
}

V3 attach_point(const State& s, const Attach& p) {
  if (p.body < 0) return p.local;
  return s.world_point(p.body, p.local);
}

void add_point_jac(Row& row, const State& s, const Attach& p, const V3& d, double sign) {
  if (p.body < 0) return;
  const int off = s.dof_off[p.body];
  row.add3(off, sign * d);
  if (s.bodies[p.body].type == BodyType::Rigid) {
    const V3 r = s.rotation(p.body) * p.local;
    row.add3(off + 3, sign * cross(r, d));
  }
}

double contact_gap(const Contact& c, const State& s) {
  return dot(c.normal, attach_point(s, c.a) - attach_point(s, c.b)) - c.thickness;
}

Row contact_normal_row(const Contact& c, const State& s) {
  Row r;
  add_point_jac(r, s, c.a, c.normal, 1.0);
  add_point_jac(r, s, c.b, c.normal, -1.0);
  r.compress();
  return r;
}

void contact_tangent_rows(const Contact& c, const State& s, Row& t1, Row& t2) {
  t1 = Row();
  t2 = Row();
  add_point_jac(t1, s, c.a, c.d1, 1.0);
  add_point_jac(t1, s, c.b, c.d1, -1.0);
  add_point_jac(t2, s, c.a, c.d2, 1.0);
  add_point_jac(t2, s, c.b, c.d2, -1.0);
  t1.compress();
  t2.compress();
}

void tangent_basis(const V3& n, V3& d1, V3& d2) {
  int smallest = 0;
  for (int k = 1; k < 3; ++k)
    if (std::abs(n[k]) < std::abs(n[smallest])) smallest = k;
  const V3 e = V3::unit(smallest);
  d1 = normalized(e - dot(e, n) * n);
  d2 = cross(n, d1);
}

double r_factor(double emd, double h, RowClass rc, RStrat st) {
  const double ts = rc == RowClass::Position ? h * h : h;
  switch (st) {
    case RStrat::Identity: return 1.0;
    case RStrat::H2: return ts;
    case RStrat::EffMass: return emd <= 0.0 ? ts : ts * emd;
  }
  return 1.0;
}

int joint_row_count(JointKind k) {
  switch (k) {
    case JointKind::FixedPoint: return 3;
    case JointKind::Revolute: return 5;
    case JointKind::Prismatic: return 5;
    case JointKind::BendSpring: return 2;
  }
  return 0;
}

namespace {
V3 world_dir(const State& s, int body, const V3& local) {
  return body < 0 ? local : s.rotation(body) * local;
}
BRow axis_dot_row(const State& s, int ba, int bb, const V3& xa, const V3& xb, double rest, double e) {
  BRow o;
  o.value = dot(xa, xb) - rest;
  o.compliance = e;
  const V3 cr = cross(xa, xb);
  if (ba >= 0 && s.bodies[ba].type == BodyType::Rigid) o.jac.add3(s.dof_off[ba] + 3, cr);
  if (bb >= 0 && s.bodies[bb].type == BodyType::Rigid) o.jac.add3(s.dof_off[bb] + 3, -cr);
  o.jac.compress();
  return o;
}
}  // namespace

std::vector<BRow> joint_rows(const Joint& j, const State& s) {  // src/constraints.cpp:141-220
  const int nb = static_cast<int>(s.bodies.size());
  if (j.body_a >= nb || j.body_b >= nb) throw std::invalid_argument("joint references invalid body");
  std::vector<BRow> rows;
  const Attach pa{j.body_a, j.anchor_a}, pb{j.body_b, j.anchor_b};
  const auto point_rows = [&]() {
    const V3 wa = attach_point(s, pa), wb = attach_point(s, pb);
    for (int k = 0; k < 3; ++k) {
      BRow r;
      r.value = wa[k] - wb[k];
      r.compliance = j.compliance;
      const V3 e = V3::unit(k);
      add_point_jac(r.jac, s, pa, e, 1.0);
      add_point_jac(r.jac, s, pb, e, -1.0);
      r.jac.compress();
      rows.push_back(std::move(r));
    }
  };
  switch (j.kind) {
    case JointKind::FixedPoint:
      point_rows();
      break;
    case JointKind::Revolute: {
      point_rows();
      const V3 ax = world_dir(s, j.body_a, j.axis_a);
      const V3 b1 = world_dir(s, j.body_b, j.axis_b1), b2 = world_dir(s, j.body_b, j.axis_b2);
      rows.push_back(axis_dot_row(s, j.body_a, j.body_b, ax, b1, j.rest_dots[0], j.compliance));
      rows.push_back(axis_dot_row(s, j.body_a, j.body_b, ax, b2, j.rest_dots[1], j.compliance));
      break;
    }
    case JointKind::Prismatic: {
      const V3 ax = world_dir(s, j.body_a, j.axis_a);
      V3 t1, t2;
      tangent_basis(ax, t1, t2);
      const V3 d = attach_point(s, pa) - attach_point(s, pb);
      for (const V3& t : {t1, t2}) {
        BRow r;
        r.value = dot(t, d);
        r.compliance = j.compliance;
        add_point_jac(r.jac, s, pa, t, 1.0);
        add_point_jac(r.jac, s, pb, t, -1.0);
        if (j.body_a >= 0 && s.bodies[j.body_a].type == BodyType::Rigid)
          r.jac.add3(s.dof_off[j.body_a] + 3, cross(t, d));
        r.jac.compress();
        rows.push_back(std::move(r));
      }
      const V3 a2 = world_dir(s, j.body_a, j.axis_a2);
      const V3 b1 = world_dir(s, j.body_b, j.axis_b1), b2 = world_dir(s, j.body_b, j.axis_b2);
      rows.push_back(axis_dot_row(s, j.body_a, j.body_b, ax, b1, j.rest_dots[0], j.compliance));
      rows.push_back(axis_dot_row(s, j.body_a, j.body_b, ax, b2, j.rest_dots[1], j.compliance));
      rows.push_back(axis_dot_row(s, j.body_a, j.body_b, a2, b2, j.rest_dots[2], j.compliance));
      break;
    }
    case JointKind::BendSpring: {
      const double e = j.stiffness > 0.0 ? 1.0 / j.stiffness : 0.0;
      const V3 ax = world_dir(s, j.body_a, j.axis_a);
      const V3 b1 = world_dir(s, j.body_b, j.axis_b1), b2 = world_dir(s, j.body_b, j.axis_b2);
      rows.push_back(axis_dot_row(s, j.body_a, j.body_b, ax, b1, j.rest_dots[0], e));
      rows.push_back(axis_dot_row(s, j.body_a, j.body_b, ax, b2, j.rest_dots[1], e));
      break;
    }
  }
  return rows;
}

void bind_joint(Joint& j, const State& s, const V3& world_anchor, const V3& world_axis) {
  const auto point_local = [&](int body, const V3& w) -> V3 {
    if (body < 0) return w;
    if (s.bodies[body].type == BodyType::Particle) return V3();
    return s.rotation(body).t() * (w - s.position(body));
  };
  const auto dir_local = [&](int body, const V3& w) -> V3 {
    return body < 0 ? w : s.rotation(body).t() * w;
  };
  j.anchor_a = point_local(j.body_a, world_anchor);
  j.anchor_b = point_local(j.body_b, world_anchor);
  const V3 ax = normalized(world_axis);
  V3 p1, p2;
  tangent_basis(ax, p1, p2);
  j.axis_a = dir_local(j.body_a, ax);
  j.axis_a2 = dir_local(j.body_a, p1);
  switch (j.kind) {
    case JointKind::FixedPoint:
      break;
    case JointKind::Revolute:
    case JointKind::BendSpring:
      j.axis_b1 = dir_local(j.body_b, p1);
      j.axis_b2 = dir_local(j.body_b, p2);
      j.rest_dots = V3();
      break;
    case JointKind::Prismatic:
      j.axis_b1 = dir_local(j.body_b, p1);
      j.axis_b2 = dir_local(j.body_b, p2);
      j.rest_dots = V3(dot(ax, p1), dot(ax, p2), dot(p1, p2));
      break;
  }
}

// ============================ materials ======================================

Tet make_tet(const std::array<int, 4>& v, const V3& r0, const V3& r1, const V3& r2, const V3& r3) {
  M3 dm;
  dm.set_col(0, r1 - r0);
  dm.set_col(1, r2 - r0);
  dm.set_col(2, r3 - r0);
  const double d = det3(dm);
  if (d <= 0.0) throw std::invalid_argument("tet element is degenerate or inverted at rest");
  Tet e;
  e.v = v;
  e.dm_inv = inverse3(dm);
  e.vol = d / 6.0;
  return e;
}

M3 deformation_gradient(const V3& p0, const V3& p1, const V3& p2, const V3& p3, const Tet& e) {
  M3 ds;
  ds.set_col(0, p1 - p0);
  ds.set_col(1, p2 - p0);
  ds.set_col(2, p3 - p0);
  return ds * e.dm_inv;
}

NH lame(double young, double poisson) {
  if (young <= 0.0) throw std::invalid_argument("Young's modulus must be positive");
  if (poisson < 0.0 || poisson >= 0.4999)
    throw std::invalid_argument("Poisson's ratio must lie in [0, 0.4999)");
  const double mu = young / (2.0 * (1.0 + poisson));
  const double lambda = young * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson));
  NH m;
  m.c1 = 0.5 * mu;
  m.d1 = 0.5 * lambda;
  m.alpha = lambda > 0.0 ? 1.0 + mu / lambda : 1.0;
  return m;
}

M6 isotropic_stiffness(double young, double poisson) {
  const double mu = young / (2.0 * (1.0 + poisson));
  const double lambda = young * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson));
  M6 k{};
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) k[i][j] = lambda;
    k[i][i] = lambda + 2.0 * mu;
    k[i + 3][i + 3] = mu;
  }
  return k;
}

// 6x6 inverse by Gauss-Jordan with partial pivoting (Eigen's dynamic inverse is
// PartialPivLU; only used for the constant linear-material stiffness).
M6 inverse6(const M6& a_in) {
  double a[6][12];
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 12; ++j) a[i][j] = j < 6 ? a_in[i][j] : (j - 6 == i ? 1.0 : 0.0);
  for (int c = 0; c < 6; ++c) {
    int piv = c;
    for (int r = c + 1; r < 6; ++r)
      if (std::abs(a[r][c]) > std::abs(a[piv][c])) piv = r;
    if (piv != c)
      for (int j = 0; j < 12; ++j) std::swap(a[c][j], a[piv][j]);
    const double d = a[c][c];
    for (int j = 0; j < 12; ++j) a[c][j] /= d;
    for (int r = 0; r < 6; ++r) {
      if (r == c) continue;
      const double f = a[r][c];
      for (int j = 0; j < 12; ++j) a[r][j] -= f * a[c][j];
    }
  }
  M6 o{};
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) o[i][j] = a[i][j + 6];
  return o;
}

V3 nh_gradient(const V3& s, const NH& m) {  // src/materials.cpp:57-61 (J - alpha)
  const double j = s[0] * s[1] * s[2];
  const V3 dj(s[1] * s[2], s[0] * s[2], s[0] * s[1]);
  return 2.0 * m.c1 * s + 2.0 * m.d1 * (j - m.alpha) * dj;
}

M3 nh_hessian(const V3& s, const NH& m) {  // src/materials.cpp:63-74
  const double j = s[0] * s[1] * s[2];
  const double k0 = 2.0 * j - m.alpha;
  const double k1 = m.d1 * s[2] * k0, k2 = m.d1 * s[1] * k0, k3 = m.d1 * s[0] * k0;
  M3 h;
  h(0, 0) = m.d1 * s[1] * s[1] * s[2] * s[2] + m.c1;
  h(0, 1) = k1;
  h(0, 2) = k2;
  h(1, 0) = k1;
  h(1, 1) = m.d1 * s[0] * s[0] * s[2] * s[2] + m.c1;
  h(1, 2) = k3;
  h(2, 0) = k2;
  h(2, 1) = k3;
  h(2, 2) = m.d1 * s[0] * s[0] * s[1] * s[1] + m.c1;
  return 2.0 * h;
}

double nh_energy(const V3& s, const NH& m) {
  const double ic = sqnorm(s);
  const double j = s[0] * s[1] * s[2];
  return m.c1 * (ic - 3.0) + m.d1 * (j - m.alpha) * (j - m.alpha);
}

M3 compliance_block(double vol, const M3& hess, bool project, bool diag, unsigned char* flags) {  // :82-102
  M3 h = hess;
  unsigned char f = 0;
  if (project) {
    const Eig3 e = sym_eig3(h, false);
    const double mn = std::min(e.val[0], std::min(e.val[1], e.val[2]));
    if (mn <= 0.0) {
      h = project_psd3(h);
      f |= 1;
    }
  }
  const M3 n = vol * h;
  const auto diagonal = [&]() {
    M3 e;
    for (int i = 0; i < 3; ++i) e(i, i) = n(i, i) > 0.0 ? 1.0 / n(i, i) : 0.0;
    return e;
  };
  if (flags) *flags = f;
  if (diag) {
    if (flags) *flags |= 2;
    return diagonal();
  }
  const double d = det3(n);
  if (!std::isfinite(d) || std::abs(d) < 1e-300) {
    if (flags) *flags |= 2;
    return diagonal();
  }
  return inverse3(n);
}

J312 strain_jacobian(const Tet& e, const Svd3& svd) {  // :104-114
  J312 jac{};
  for (int i = 0; i < 3; ++i) {
    const V3 u = svd.U.col(i);
    const V3 w = e.dm_inv * svd.V.col(i);
    for (int k = 0; k < 3; ++k)
      for (int d = 0; d < 3; ++d) jac[i][3 * (k + 1) + d] = w[k] * u[d];
    const double ws = -(w[0] + w[1] + w[2]);
    for (int d = 0; d < 3; ++d) jac[i][d] = ws * u[d];
  }
  return jac;
}

void TetMesh::prepare() {
  if (material.model == MatModel::NeoHookean) {
    nh = lame(material.young, material.poisson);
  } else {
    stiffness = isotropic_stiffness(material.young, material.poisson);
    stiffness_inv = inverse6(stiffness);
  }
}

namespace {
V3 axial(const M3& m) {
  return {0.5 * (m(2, 1) - m(1, 2)), 0.5 * (m(0, 2) - m(2, 0)), 0.5 * (m(1, 0) - m(0, 1))};
}
void voigt(const M3& s, double out[6]) {
  out[0] = s(0, 0);
  out[1] = s(1, 1);
  out[2] = s(2, 2);
  out[3] = 2.0 * s(1, 2);
  out[4] = 2.0 * s(0, 2);
  out[5] = 2.0 * s(0, 1);
}
}  // namespace

// src/materials.cpp:140-178 — co-rotational linear material (6 rows).
MatRows linear_strain_rows(const Tet& e, const TetMesh& mesh, const V3& p0, const V3& p1,
                           const V3& p2, const V3& p3) {
  const M3 f = deformation_gradient(p0, p1, p2, p3, e);
  const Svd3 svd = svd3(f);
  const M3 r = svd.U * svd.V.t();
  const M3 stretch = (svd.V * M3::diag(svd.S)) * svd.V.t();
  MatRows o;
  o.dim = 6;
  double strain[6];
  voigt(stretch - M3::identity(), strain);
  for (int i = 0; i < 6; ++i) {
    double s = 0.0;
    for (int k = 0; k < 6; ++k) s += mesh.stiffness[i][k] * strain[k];
    o.c[i] = e.vol * s;
  }
  for (int i = 0; i < 6; ++i)
    for (int k = 0; k < 6; ++k) o.comp[i][k] = mesh.stiffness_inv[i][k] / e.vol;
  const double tr = stretch(0, 0) + stretch(1, 1) + stretch(2, 2);
  const M3 g = tr * M3::identity() - stretch;
  const bool rot_term = std::abs(det3(g)) > 1e-12;
  const M3 g_inv = rot_term ? inverse3(g) : M3();
  for (int k = 0; k < 4; ++k) {
    for (int d = 0; d < 3; ++d) {
      M3 df;
      if (k == 0) {
        for (int c = 0; c < 3; ++c)
          for (int col = 0; col < 3; ++col) df(d, col) -= e.dm_inv(c, col);
      } else {
        for (int col = 0; col < 3; ++col) df(d, col) = e.dm_inv(k - 1, col);
      }
      const M3 rtdf = r.t() * df;
      M3 ds = rtdf;
      if (rot_term) {
        const V3 w = 2.0 * (g_inv * axial(rtdf));
        ds = ds - skew(w) * stretch;
      }
      const M3 sym = 0.5 * (ds + ds.t());
      double v[6];
      voigt(sym, v);
      for (int i = 0; i < 6; ++i) o.jac[i][3 * k + d] = v[i];
    }
  }
  return o;
}

// src/materials.cpp:180-193.
MatRows neo_hookean_rows(const Tet& e, const TetMesh& mesh, const V3& p0, const V3& p1, const V3& p2,
                         const V3& p3) {
  const M3 f = deformation_gradient(p0, p1, p2, p3, e);
  const Svd3 svd = svd3(f);
  MatRows o;
  o.dim = 3;
  const V3 c = e.vol * nh_gradient(svd.S, mesh.nh);
  for (int i = 0; i < 3; ++i) o.c[i] = c[i];
  const J312 j = strain_jacobian(e, svd);
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 12; ++k) o.jac[i][k] = j[i][k];
  const M3 h = nh_hessian(svd.S, mesh.nh);
  const M3 cb = compliance_block(e.vol, h, true, mesh.material.diagonal_compliance, &o.flags);
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) o.comp[i][k] = cb(i, k);
  return o;
}

double element_energy(const Tet& e, const TetMesh& mesh, const V3& p0, const V3& p1, const V3& p2,
                      const V3& p3) {
  const M3 f = deformation_gradient(p0, p1, p2, p3, e);
  const Svd3 svd = svd3(f);
  if (mesh.material.model == MatModel::NeoHookean) return e.vol * nh_energy(svd.S, mesh.nh);
  const M3 stretch = (svd.V * M3::diag(svd.S)) * svd.V.t();
  double strain[6];
  voigt(stretch - M3::identity(), strain);
  double s = 0.0;
  for (int i = 0; i < 6; ++i)
    for (int k = 0; k < 6; ++k) s += strain[i] * mesh.stiffness[i][k] * strain[k];
  return 0.5 * e.vol * s;
}

void compute_material_rows(const TetMesh& mesh, const std::vector<V3>& p, std::vector<MatRows>& out,
                           bool parallel) {
  const int n = static_cast<int>(mesh.elements.size());
  out.resize(n);
  const auto one = [&](int i) {
    const Tet& e = mesh.elements[i];
    out[i] = mesh.material.model == MatModel::NeoHookean
                 ? neo_hookean_rows(e, mesh, p[e.v[0]], p[e.v[1]], p[e.v[2]], p[e.v[3]])
                 : linear_strain_rows(e, mesh, p[e.v[0]], p[e.v[1]], p[e.v[2]], p[e.v[3]]);
  };
  if (parallel) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) one(i);
  } else {
    for (int i = 0; i < n; ++i) one(i);
  }
}

}  // namespace orc
