// ORACLE — test infrastructure only. Never linked into the product path.
//
// Small fixed-size double-precision math for the CPU restatement of the
// reference `nsdyn` solver (/root/reference/proj). The reference uses Eigen3
// (proj/include/nsdyn/linalg.h:9-16); Eigen is absent from this image, so the
// Eigen algorithms the reference calls are restated here from Eigen 3.4:
//   * JacobiSVD<Matrix3d>(ComputeFullU|ComputeFullV)   (called at src/linalg.cpp:111)
//   * SelfAdjointEigenSolver<Matrix3d>                  (src/linalg.cpp:129, src/materials.cpp:86)
//   * Matrix3d::inverse()/determinant() cofactor forms  (src/bodies.cpp:190, src/materials.cpp:14-18,95-101)
//   * Quaterniond::normalized().toRotationMatrix()      (src/bodies.cpp:49)
// Bit-level agreement with an arbitrary Eigen build is not claimed (SURVEY.md
// Appendix B); these restatements are the parity anchor.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <limits>
#include <vector>

namespace orc {

using VecX = std::vector<double>;

struct V3 {
  double c[3] = {0.0, 0.0, 0.0};
  V3() = default;
  V3(double x, double y, double z) : c{x, y, z} {}
  double& operator[](int i) { return c[i]; }
  double operator[](int i) const { return c[i]; }
  static V3 unit(int k) {
    V3 v;
    v[k] = 1.0;
    return v;
  }
};

inline V3 operator+(const V3& a, const V3& b) { return {a[0] + b[0], a[1] + b[1], a[2] + b[2]}; }
inline V3 operator-(const V3& a, const V3& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
inline V3 operator-(const V3& a) { return {-a[0], -a[1], -a[2]}; }
inline V3 operator*(double s, const V3& a) { return {s * a[0], s * a[1], s * a[2]}; }
inline V3 operator*(const V3& a, double s) { return {a[0] * s, a[1] * s, a[2] * s}; }
inline V3 operator/(const V3& a, double s) { return {a[0] / s, a[1] / s, a[2] / s}; }
inline V3& operator+=(V3& a, const V3& b) { a = a + b; return a; }
inline V3& operator-=(V3& a, const V3& b) { a = a - b; return a; }
inline bool operator==(const V3& a, const V3& b) { return a[0] == b[0] && a[1] == b[1] && a[2] == b[2]; }
inline bool operator!=(const V3& a, const V3& b) { return !(a == b); }
inline double dot(const V3& a, const V3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline double sqnorm(const V3& a) { return dot(a, a); }
inline double norm(const V3& a) { return std::sqrt(sqnorm(a)); }
inline V3 cross(const V3& a, const V3& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
inline V3 normalized(const V3& a) {
  const double n2 = sqnorm(a);
  return n2 > 0.0 ? a / std::sqrt(n2) : a;
}

struct V4 {
  double c[4] = {0.0, 0.0, 0.0, 0.0};
  V4() = default;
  V4(double w, double x, double y, double z) : c{w, x, y, z} {}
  double& operator[](int i) { return c[i]; }
  double operator[](int i) const { return c[i]; }
};
inline double sqnorm(const V4& a) { return a[0] * a[0] + a[1] * a[1] + a[2] * a[2] + a[3] * a[3]; }
inline double norm(const V4& a) { return std::sqrt(sqnorm(a)); }

// Row-major 3x3.
struct M3 {
  double m[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  double& operator()(int i, int j) { return m[i][j]; }
  double operator()(int i, int j) const { return m[i][j]; }
  static M3 identity() {
    M3 r;
    r(0, 0) = r(1, 1) = r(2, 2) = 1.0;
    return r;
  }
  static M3 diag(const V3& d) {
    M3 r;
    for (int i = 0; i < 3; ++i) r(i, i) = d[i];
    return r;
  }
  V3 col(int j) const { return {m[0][j], m[1][j], m[2][j]}; }
  V3 row(int i) const { return {m[i][0], m[i][1], m[i][2]}; }
  void set_col(int j, const V3& v) {
    for (int i = 0; i < 3; ++i) m[i][j] = v[i];
  }
  M3 t() const {
    M3 r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r(i, j) = m[j][i];
    return r;
  }
};

inline V3 operator*(const M3& a, const V3& v) {
  return {a(0, 0) * v[0] + a(0, 1) * v[1] + a(0, 2) * v[2],
          a(1, 0) * v[0] + a(1, 1) * v[1] + a(1, 2) * v[2],
          a(2, 0) * v[0] + a(2, 1) * v[1] + a(2, 2) * v[2]};
}
inline M3 operator*(const M3& a, const M3& b) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = a(i, 0) * b(0, j) + a(i, 1) * b(1, j) + a(i, 2) * b(2, j);
  return r;
}
inline M3 operator*(double s, const M3& a) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = s * a(i, j);
  return r;
}
inline M3 operator+(const M3& a, const M3& b) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = a(i, j) + b(i, j);
  return r;
}
inline M3 operator-(const M3& a, const M3& b) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = a(i, j) - b(i, j);
  return r;
}
inline double fro_norm(const M3& a) {
  double s = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) s += a(i, j) * a(i, j);
  return std::sqrt(s);
}

// Eigen determinant_impl<3>: bruteforce_det3_helper(0,1,2) - (1,0,2) + (2,0,1).
inline double det3(const M3& a) {
  const auto h = [&](int x, int y, int z) {
    return a(0, x) * (a(1, y) * a(2, z) - a(1, z) * a(2, y));
  };
  return h(0, 1, 2) - h(1, 0, 2) + h(2, 0, 1);
}

// Eigen cofactor_3x3<i,j> (cyclic signed cofactor).
inline double cofactor3(const M3& a, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return a(i1, j1) * a(i2, j2) - a(i1, j2) * a(i2, j1);
}

// Eigen compute_inverse<3>: det from column-0 cofactors, result = adj * (1/det).
inline M3 inverse3(const M3& a) {
  const double c0 = cofactor3(a, 0, 0), c1 = cofactor3(a, 1, 0), c2 = cofactor3(a, 2, 0);
  const double det = c0 * a(0, 0) + c1 * a(1, 0) + c2 * a(2, 0);
  const double inv = 1.0 / det;
  M3 r;
  r(1, 0) = cofactor3(a, 0, 1) * inv;
  r(1, 1) = cofactor3(a, 1, 1) * inv;
  r(2, 0) = cofactor3(a, 0, 2) * inv;
  r(1, 2) = cofactor3(a, 2, 1) * inv;
  r(2, 1) = cofactor3(a, 1, 2) * inv;
  r(2, 2) = cofactor3(a, 2, 2) * inv;
  r(0, 0) = c0 * inv;
  r(0, 1) = c1 * inv;
  r(0, 2) = c2 * inv;
  return r;
}

inline M3 skew(const V3& v) {
  M3 s;
  s(0, 1) = -v[2];
  s(0, 2) = v[1];
  s(1, 0) = v[2];
  s(1, 2) = -v[0];
  s(2, 0) = -v[1];
  s(2, 1) = v[0];
  return s;
}

// Quaterniond(w,x,y,z).normalized().toRotationMatrix() (Eigen 3.4 Quaternion.h).
inline M3 quat_to_rot(const V4& q_in) {
  V4 q = q_in;
  const double n2 = sqnorm(q);
  if (n2 > 0.0) {
    const double n = std::sqrt(n2);
    for (int i = 0; i < 4; ++i) q[i] = q[i] / n;
  }
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  M3 r;
  r(0, 0) = 1.0 - (tyy + tzz);
  r(0, 1) = txy - twz;
  r(0, 2) = txz + twy;
  r(1, 0) = txy + twz;
  r(1, 1) = 1.0 - (txx + tzz);
  r(1, 2) = tyz - twx;
  r(2, 0) = txz - twy;
  r(2, 1) = tyz + twx;
  r(2, 2) = 1.0 - (txx + tyy);
  return r;
}

// ---------------------------------------------------------------------------
// Eigen 3.4 JacobiSVD<Matrix3d> (two-sided Jacobi, square case, full U and V).
// A plane rotation is stored as (c, s) with J = [c s; -s c] (Eigen JacobiRotation).
// ---------------------------------------------------------------------------
struct Rot {
  double c = 1.0, s = 0.0;
  Rot transpose() const { return {c, -s}; }
  Rot operator*(const Rot& o) const { return {c * o.c - s * o.s, c * o.s + s * o.c}; }
};

// Rows p,q of a: [x;y] <- J [x;y]  (JacobiRotation applyOnTheLeft).
inline void rot_left(M3& a, int p, int q, const Rot& j) {
  for (int i = 0; i < 3; ++i) {
    const double xi = a(p, i), yi = a(q, i);
    a(p, i) = j.c * xi + j.s * yi;
    a(q, i) = -j.s * xi + j.c * yi;
  }
}
// Columns p,q of a: [x y] <- [x y] J  (applyOnTheRight = in-plane rotation with J^T).
inline void rot_right(M3& a, int p, int q, const Rot& j) {
  const Rot t = j.transpose();
  for (int i = 0; i < 3; ++i) {
    const double xi = a(i, p), yi = a(i, q);
    a(i, p) = t.c * xi + t.s * yi;
    a(i, q) = -t.s * xi + t.c * yi;
  }
}

// JacobiRotation::makeJacobi(x, y, z) for real scalars.
inline Rot make_jacobi(double x, double y, double z) {
  Rot r;
  const double deno = 2.0 * std::abs(y);
  if (deno < std::numeric_limits<double>::min()) {
    r.c = 1.0;
    r.s = 0.0;
    return r;
  }
  const double tau = (x - z) / deno;
  const double w = std::sqrt(tau * tau + 1.0);
  const double t = tau > 0.0 ? 1.0 / (tau + w) : 1.0 / (tau - w);
  const double sign_t = t > 0.0 ? 1.0 : -1.0;
  const double n = 1.0 / std::sqrt(t * t + 1.0);
  r.s = -sign_t * (y / std::abs(y)) * std::abs(t) * n;
  r.c = n;
  return r;
}

// internal::real_2x2_jacobi_svd.
inline void real_2x2_jacobi_svd(const M3& a, int p, int q, Rot& j_left, Rot& j_right) {
  double m00 = a(p, p), m01 = a(p, q), m10 = a(q, p), m11 = a(q, q);
  Rot rot1;
  const double t = m00 + m11;
  const double d = m10 - m01;
  if (std::abs(d) < std::numeric_limits<double>::min()) {
    rot1.s = 0.0;
    rot1.c = 1.0;
  } else {
    const double u = t / d;
    const double tmp = std::sqrt(1.0 + u * u);
    rot1.s = 1.0 / tmp;
    rot1.c = u / tmp;
  }
  // m.applyOnTheLeft(0,1,rot1)
  const double n00 = rot1.c * m00 + rot1.s * m10, n01 = rot1.c * m01 + rot1.s * m11;
  const double n10 = -rot1.s * m00 + rot1.c * m10, n11 = -rot1.s * m01 + rot1.c * m11;
  (void)n10;
  j_right = make_jacobi(n00, n01, n11);
  j_left = rot1 * j_right.transpose();
}

struct Svd3 {
  M3 U;
  V3 S;
  M3 V;
};

// Returns the unsigned Eigen decomposition (singular values >= 0, sorted desc).
inline Svd3 jacobi_svd3(const M3& f) {
  const double precision = 2.0 * std::numeric_limits<double>::epsilon();
  const double consider_zero = std::numeric_limits<double>::min();
  double scale = 0.0;
  bool finite = true;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      if (!std::isfinite(f(i, j))) finite = false;
      scale = std::max(scale, std::abs(f(i, j)));
    }
  Svd3 out;
  if (!finite) {  // Eigen reports InvalidInput; results undefined. Propagate NaN.
    const double nan = std::numeric_limits<double>::quiet_NaN();
    out.U = out.V = M3::identity();
    out.S = V3(nan, nan, nan);
    return out;
  }
  if (scale == 0.0) scale = 1.0;
  M3 w;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) w(i, j) = f(i, j) / scale;
  M3 U = M3::identity(), V = M3::identity();
  double max_diag = std::max(std::abs(w(0, 0)), std::max(std::abs(w(1, 1)), std::abs(w(2, 2))));
  bool finished = false;
  while (!finished) {
    finished = true;
    for (int p = 1; p < 3; ++p) {
      for (int q = 0; q < p; ++q) {
        const double threshold = std::max(consider_zero, precision * max_diag);
        if (std::abs(w(p, q)) > threshold || std::abs(w(q, p)) > threshold) {
          finished = false;
          Rot jl, jr;
          real_2x2_jacobi_svd(w, p, q, jl, jr);
          rot_left(w, p, q, jl);
          rot_right(U, p, q, jl.transpose());
          rot_right(w, p, q, jr);
          rot_right(V, p, q, jr);
          max_diag = std::max(max_diag, std::max(std::abs(w(p, p)), std::abs(w(q, q))));
        }
      }
    }
  }
  V3 s;
  for (int i = 0; i < 3; ++i) {
    const double a = w(i, i);
    s[i] = std::abs(a);
    if (a < 0.0)
      for (int r = 0; r < 3; ++r) U(r, i) = -U(r, i);
  }
  for (int i = 0; i < 3; ++i) s[i] *= scale;
  for (int i = 0; i < 3; ++i) {
    // maxCoeff(&pos) over the tail: first index of the maximum.
    int pos = 0;
    double best = s[i];
    for (int k = i + 1; k < 3; ++k)
      if (s[k] > best) {
        best = s[k];
        pos = k - i;
      }
    if (best == 0.0) break;
    if (pos) {
      pos += i;
      std::swap(s[i], s[pos]);
      for (int r = 0; r < 3; ++r) {
        std::swap(U(r, i), U(r, pos));
        std::swap(V(r, i), V(r, pos));
      }
    }
  }
  out.U = U;
  out.S = s;
  out.V = V;
  return out;
}

// ---------------------------------------------------------------------------
// Eigen 3.4 SelfAdjointEigenSolver<Matrix3d>: lower triangle, scale to [-1,1],
// 3x3 tridiagonalization selector, implicit symmetric QR with Wilkinson shift,
// ascending selection sort. Eigenvectors are the columns of `vec`.
// ---------------------------------------------------------------------------
inline double positive_hypot(double x, double y) {
  if (std::isinf(x) || std::isinf(y)) return std::numeric_limits<double>::infinity();
  if (std::isnan(x) || std::isnan(y)) return std::numeric_limits<double>::quiet_NaN();
  const double p = std::max(x, y);
  if (p == 0.0) return 0.0;
  const double qp = std::min(y, x) / p;
  return p * std::sqrt(1.0 + qp * qp);
}

// JacobiRotation::makeGivens(p, q) for real scalars.
inline Rot make_givens(double p, double q) {
  Rot r;
  if (q == 0.0) {
    r.c = p < 0.0 ? -1.0 : 1.0;
    r.s = 0.0;
  } else if (p == 0.0) {
    r.c = 0.0;
    r.s = q < 0.0 ? 1.0 : -1.0;
  } else if (std::abs(p) > std::abs(q)) {
    const double t = q / p;
    double u = std::sqrt(1.0 + t * t);
    if (p < 0.0) u = -u;
    r.c = 1.0 / u;
    r.s = -t * r.c;
  } else {
    const double t = p / q;
    double u = std::sqrt(1.0 + t * t);
    if (q < 0.0) u = -u;
    r.s = -1.0 / u;
    r.c = -t * r.s;
  }
  return r;
}

struct Eig3 {
  V3 val;   // ascending
  M3 vec;   // columns
  bool ok = true;
};

inline Eig3 sym_eig3(const M3& a_in, bool vectors = true) {
  M3 mat;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j <= i; ++j) mat(i, j) = a_in(i, j);
  double scale = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) scale = std::max(scale, std::abs(mat(i, j)));
  if (scale == 0.0) scale = 1.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j <= i; ++j) mat(i, j) /= scale;

  double diag[3], sub[2];
  M3 q;
  {
    const double tol = std::numeric_limits<double>::min();
    diag[0] = mat(0, 0);
    const double v1norm2 = mat(2, 0) * mat(2, 0);
    if (v1norm2 <= tol) {
      diag[1] = mat(1, 1);
      diag[2] = mat(2, 2);
      sub[0] = mat(1, 0);
      sub[1] = mat(2, 1);
      q = M3::identity();
    } else {
      const double beta = std::sqrt(mat(1, 0) * mat(1, 0) + v1norm2);
      const double inv_beta = 1.0 / beta;
      const double m01 = mat(1, 0) * inv_beta;
      const double m02 = mat(2, 0) * inv_beta;
      const double qq = 2.0 * m01 * mat(2, 1) + m02 * (mat(2, 2) - mat(1, 1));
      diag[1] = mat(1, 1) + m02 * qq;
      diag[2] = mat(2, 2) - m02 * qq;
      sub[0] = beta;
      sub[1] = mat(2, 1) - m01 * qq;
      q = M3();
      q(0, 0) = 1.0;
      q(1, 1) = m01;
      q(1, 2) = m02;
      q(2, 1) = m02;
      q(2, 2) = -m01;
    }
  }

  const int n = 3;
  int end = n - 1, start = 0, iter = 0;
  const int max_iter = 30;
  const double consider_zero = std::numeric_limits<double>::min();
  const double precision_inv = 1.0 / std::numeric_limits<double>::epsilon();
  while (end > 0) {
    for (int i = start; i < end; ++i) {
      if (std::abs(sub[i]) < consider_zero) {
        sub[i] = 0.0;
      } else {
        const double scaled = precision_inv * sub[i];
        if (scaled * scaled <= (std::abs(diag[i]) + std::abs(diag[i + 1]))) sub[i] = 0.0;
      }
    }
    while (end > 0 && sub[end - 1] == 0.0) end--;
    if (end <= 0) break;
    iter++;
    if (iter > max_iter * n) break;
    start = end - 1;
    while (start > 0 && sub[start - 1] != 0.0) start--;

    // tridiagonal_qr_step (Wilkinson shift)
    const double td = (diag[end - 1] - diag[end]) * 0.5;
    const double e = sub[end - 1];
    double mu = diag[end];
    if (td == 0.0) {
      mu -= std::abs(e);
    } else if (e != 0.0) {
      const double e2 = e * e;
      const double h = positive_hypot(std::abs(td), std::abs(e));
      if (e2 == 0.0)
        mu -= e / ((td + (td > 0.0 ? h : -h)) / e);
      else
        mu -= e2 / (td + (td > 0.0 ? h : -h));
    }
    double x = diag[start] - mu;
    double z = sub[start];
    for (int k = start; k < end && z != 0.0; ++k) {
      const Rot rot = make_givens(x, z);
      const double sdk = rot.s * diag[k] + rot.c * sub[k];
      const double dkp1 = rot.s * sub[k] + rot.c * diag[k + 1];
      diag[k] = rot.c * (rot.c * diag[k] - rot.s * sub[k]) - rot.s * (rot.c * sub[k] - rot.s * diag[k + 1]);
      diag[k + 1] = rot.s * sdk + rot.c * dkp1;
      sub[k] = rot.c * sdk - rot.s * dkp1;
      if (k > start) sub[k - 1] = rot.c * sub[k - 1] - rot.s * z;
      x = sub[k];
      if (k < end - 1) {
        z = -rot.s * sub[k + 1];
        sub[k + 1] = rot.c * sub[k + 1];
      }
      if (vectors) rot_right(q, k, k + 1, rot);
    }
  }
  Eig3 out;
  out.ok = iter <= max_iter * n;
  if (out.ok) {
    for (int i = 0; i < n - 1; ++i) {
      int k = 0;
      double mn = diag[i];
      for (int j = i + 1; j < n; ++j)
        if (diag[j] < mn) {
          mn = diag[j];
          k = j - i;
        }
      if (k > 0) {
        std::swap(diag[i], diag[k + i]);
        for (int r = 0; r < 3; ++r) std::swap(q(r, i), q(r, k + i));
      }
    }
  }
  for (int i = 0; i < 3; ++i) out.val[i] = diag[i] * scale;
  out.vec = q;
  return out;
}

}  // namespace orc
