// Fixed-size math shared by host and device, templated on the arithmetic type
// (float = performance mode, double = parity mode).
//
// The 3x3 singular value and symmetric eigen decompositions follow the
// published Eigen 3.4 algorithms the reference calls (JacobiSVD at
// src/linalg.cpp:111, SelfAdjointEigenSolver at src/linalg.cpp:129 and
// src/materials.cpp:86), so data-dependent branches (sign flips, sorting,
// PSD projection trigger) are taken the same way as the CPU path; see
// SURVEY.md Appendix B. Everything is register-resident, no local arrays with
// dynamic indexing on the hot path.
#pragma once

#include <cfloat>
#include <cmath>

#ifdef __CUDACC__
#define NSD_HD __host__ __device__ __forceinline__
#else
#define NSD_HD inline
#endif

// Bounds and invariant checks of the checked build (make checks: -DNSD_CHECKS,
// tools/run_checked.sh), compiled out otherwise. compute-sanitizer is closed on the
// GPU pool (profiles/r2_sanitizer_attempt.txt); these take its place for the
// index arithmetic of the hot kernels. A failed check traps the kernel.
#ifdef NSD_CHECKS
#include <cstdio>
#include <cstdlib>
#ifdef __CUDA_ARCH__
#define NSD_CHECK(c)                                                               \
  do {                                                                             \
    if (!(c)) {                                                                    \
      printf("NSD_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);              \
      __trap();                                                                    \
    }                                                                              \
  } while (0)
#else
#define NSD_CHECK(c)                                                               \
  do {                                                                             \
    if (!(c)) {                                                                    \
      std::fprintf(stderr, "NSD_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
      std::abort();                                                                \
    }                                                                              \
  } while (0)
#endif
#else
#define NSD_CHECK(c) \
  do {               \
  } while (0)
#endif

namespace nsd {

template <class R> struct Lim;
template <> struct Lim<float> {
  NSD_HD static float eps() { return FLT_EPSILON; }
  NSD_HD static float tiny() { return FLT_MIN; }
  NSD_HD static float inf() { return __builtin_huge_valf(); }
};
template <> struct Lim<double> {
  NSD_HD static double eps() { return DBL_EPSILON; }
  NSD_HD static double tiny() { return DBL_MIN; }
  NSD_HD static double inf() { return __builtin_huge_val(); }
};

template <class R> NSD_HD R rsqrt_(R x) { return sqrt(x); }
template <class R> NSD_HD R mx(R a, R b) { return a > b ? a : b; }
template <class R> NSD_HD R mn(R a, R b) { return a < b ? a : b; }
template <class R> NSD_HD R ab(R a) { return a < R(0) ? -a : a; }

template <class R> struct V3 {
  R x, y, z;
  NSD_HD R operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
  NSD_HD R& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
};
template <class R> NSD_HD V3<R> v3(R a, R b, R c) { return V3<R>{a, b, c}; }
template <class R> NSD_HD V3<R> operator+(V3<R> a, V3<R> b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
template <class R> NSD_HD V3<R> operator-(V3<R> a, V3<R> b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
template <class R> NSD_HD V3<R> operator-(V3<R> a) { return {-a.x, -a.y, -a.z}; }
template <class R> NSD_HD V3<R> operator*(R s, V3<R> a) { return {s * a.x, s * a.y, s * a.z}; }
template <class R> NSD_HD V3<R> operator/(V3<R> a, R s) { return {a.x / s, a.y / s, a.z / s}; }
template <class R> NSD_HD R dot(V3<R> a, V3<R> b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
template <class R> NSD_HD V3<R> cross(V3<R> a, V3<R> b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
template <class R> NSD_HD R norm(V3<R> a) { return sqrt(dot(a, a)); }
template <class R> NSD_HD V3<R> normalize(V3<R> a) {
  const R n2 = dot(a, a);
  return n2 > R(0) ? a / sqrt(n2) : a;
}

// Row-major 3x3 held in registers.
template <class R> struct M3 {
  R a[9];
  NSD_HD R operator()(int i, int j) const { return a[3 * i + j]; }
  NSD_HD R& operator()(int i, int j) { return a[3 * i + j]; }
};
template <class R> NSD_HD M3<R> m3_identity() {
  M3<R> m;
#pragma unroll
  for (int i = 0; i < 9; ++i) m.a[i] = R(0);
  m.a[0] = m.a[4] = m.a[8] = R(1);
  return m;
}
template <class R> NSD_HD M3<R> m3_zero() {
  M3<R> m;
#pragma unroll
  for (int i = 0; i < 9; ++i) m.a[i] = R(0);
  return m;
}
template <class R> NSD_HD V3<R> mul(const M3<R>& m, V3<R> v) {
  return {m.a[0] * v.x + m.a[1] * v.y + m.a[2] * v.z, m.a[3] * v.x + m.a[4] * v.y + m.a[5] * v.z,
          m.a[6] * v.x + m.a[7] * v.y + m.a[8] * v.z};
}
template <class R> NSD_HD V3<R> mul_t(const M3<R>& m, V3<R> v) {  // m^T v
  return {m.a[0] * v.x + m.a[3] * v.y + m.a[6] * v.z, m.a[1] * v.x + m.a[4] * v.y + m.a[7] * v.z,
          m.a[2] * v.x + m.a[5] * v.y + m.a[8] * v.z};
}
template <class R> NSD_HD M3<R> mul(const M3<R>& p, const M3<R>& q) {
  M3<R> r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r.a[3 * i + j] = p.a[3 * i] * q.a[j] + p.a[3 * i + 1] * q.a[3 + j] + p.a[3 * i + 2] * q.a[6 + j];
  return r;
}
template <class R> NSD_HD M3<R> transpose(const M3<R>& m) {
  M3<R> r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r.a[3 * i + j] = m.a[3 * j + i];
  return r;
}
template <class R> NSD_HD V3<R> col(const M3<R>& m, int j) { return {m.a[j], m.a[3 + j], m.a[6 + j]}; }

template <class R> NSD_HD R det3(const M3<R>& m) {  // Eigen bruteforce order
  return m(0, 0) * (m(1, 1) * m(2, 2) - m(1, 2) * m(2, 1)) - m(0, 1) * (m(1, 0) * m(2, 2) - m(1, 2) * m(2, 0)) +
         m(0, 2) * (m(1, 0) * m(2, 1) - m(1, 1) * m(2, 0));
}
template <class R> NSD_HD R cof3(const M3<R>& m, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return m(i1, j1) * m(i2, j2) - m(i1, j2) * m(i2, j1);
}
// Adjugate / det with det from the column-0 cofactors (Eigen compute_inverse<3>).
template <class R> NSD_HD M3<R> inverse3(const M3<R>& m) {
  const R c0 = cof3(m, 0, 0), c1 = cof3(m, 1, 0), c2 = cof3(m, 2, 0);
  const R det = c0 * m(0, 0) + c1 * m(1, 0) + c2 * m(2, 0);
  const R inv = R(1) / det;
  M3<R> r;
  r(0, 0) = c0 * inv;
  r(0, 1) = c1 * inv;
  r(0, 2) = c2 * inv;
  r(1, 0) = cof3(m, 0, 1) * inv;
  r(1, 1) = cof3(m, 1, 1) * inv;
  r(1, 2) = cof3(m, 2, 1) * inv;
  r(2, 0) = cof3(m, 0, 2) * inv;
  r(2, 1) = cof3(m, 1, 2) * inv;
  r(2, 2) = cof3(m, 2, 2) * inv;
  return r;
}

// Quaternion (w, x, y, z) -> rotation, normalising first (Quaterniond::normalized().toRotationMatrix()).
// Uncontracted arithmetic (no FMA) for values that feed a data-dependent decision
// exactly at its boundary (the contact gap at the Fischer-Burmeister origin): the
// same roundings as the CPU oracle, which is compiled with -ffp-contract=off.
NSD_HD double smul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
NSD_HD double sadd(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
NSD_HD double ssub(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
NSD_HD float smul(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fmul_rn(a, b);
#else
  return a * b;
#endif
}
NSD_HD float sadd(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fadd_rn(a, b);
#else
  return a + b;
#endif
}
NSD_HD float ssub(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fsub_rn(a, b);
#else
  return a - b;
#endif
}
template <class R> NSD_HD R sdot(V3<R> a, V3<R> b) { return sadd(sadd(smul(a.x, b.x), smul(a.y, b.y)), smul(a.z, b.z)); }
// R local + pos, uncontracted (State::world_point: position + rotation * local).
template <class R> NSD_HD V3<R> sworld(const M3<R>& m, V3<R> l, V3<R> p) {
  return v3(sadd(p.x, sadd(sadd(smul(m.a[0], l.x), smul(m.a[1], l.y)), smul(m.a[2], l.z))),
            sadd(p.y, sadd(sadd(smul(m.a[3], l.x), smul(m.a[4], l.y)), smul(m.a[5], l.z))),
            sadd(p.z, sadd(sadd(smul(m.a[6], l.x), smul(m.a[7], l.y)), smul(m.a[8], l.z))));
}
// quat_rot (below) uncontracted.
template <class R> NSD_HD M3<R> quat_rot_strict(R w, R x, R y, R z) {
  const R n2 = sadd(sadd(sadd(smul(w, w), smul(x, x)), smul(y, y)), smul(z, z));
  if (n2 > R(0)) {
    const R n = sqrt(n2);
    w = w / n;
    x = x / n;
    y = y / n;
    z = z / n;
  }
  const R tx = smul(R(2), x), ty = smul(R(2), y), tz = smul(R(2), z);
  const R twx = smul(tx, w), twy = smul(ty, w), twz = smul(tz, w);
  const R txx = smul(tx, x), txy = smul(ty, x), txz = smul(tz, x);
  const R tyy = smul(ty, y), tyz = smul(tz, y), tzz = smul(tz, z);
  M3<R> r;
  r(0, 0) = ssub(R(1), sadd(tyy, tzz));
  r(0, 1) = ssub(txy, twz);
  r(0, 2) = sadd(txz, twy);
  r(1, 0) = sadd(txy, twz);
  r(1, 1) = ssub(R(1), sadd(txx, tzz));
  r(1, 2) = ssub(tyz, twx);
  r(2, 0) = ssub(txz, twy);
  r(2, 1) = sadd(tyz, twx);
  r(2, 2) = ssub(R(1), sadd(txx, tyy));
  return r;
}

template <class R> NSD_HD M3<R> quat_rot(R w, R x, R y, R z) {
  const R n2 = w * w + x * x + y * y + z * z;
  if (n2 > R(0)) {
    const R n = sqrt(n2);
    w = w / n;
    x = x / n;
    y = y / n;
    z = z / n;
  }
  const R tx = R(2) * x, ty = R(2) * y, tz = R(2) * z;
  const R twx = tx * w, twy = ty * w, twz = tz * w;
  const R txx = tx * x, txy = ty * x, txz = tz * x;
  const R tyy = ty * y, tyz = tz * y, tzz = tz * z;
  M3<R> r;
  r(0, 0) = R(1) - (tyy + tzz);
  r(0, 1) = txy - twz;
  r(0, 2) = txz + twy;
  r(1, 0) = txy + twz;
  r(1, 1) = R(1) - (txx + tzz);
  r(1, 2) = tyz - twx;
  r(2, 0) = txz - twy;
  r(2, 1) = tyz + twx;
  r(2, 2) = R(1) - (txx + tyy);
  return r;
}

// ---------------- plane rotations (Eigen JacobiRotation conventions) ----------------
template <class R> struct PRot {
  R c, s;
};
// rows p,q <- J [rows]
template <class R> NSD_HD void prot_rows(M3<R>& m, int p, int q, PRot<R> j) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const R xi = m(p, i), yi = m(q, i);
    m(p, i) = j.c * xi + j.s * yi;
    m(q, i) = -j.s * xi + j.c * yi;
  }
}
// cols p,q <- [cols] J
template <class R> NSD_HD void prot_cols(M3<R>& m, int p, int q, PRot<R> j) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const R xi = m(i, p), yi = m(i, q);
    m(i, p) = j.c * xi - j.s * yi;
    m(i, q) = j.s * xi + j.c * yi;
  }
}

template <class R> NSD_HD PRot<R> jacobi_rot(R x, R y, R z) {  // makeJacobi
  PRot<R> r;
  const R deno = R(2) * ab(y);
  if (deno < Lim<R>::tiny()) {
    r.c = R(1);
    r.s = R(0);
    return r;
  }
  const R tau = (x - z) / deno;
  const R w = sqrt(tau * tau + R(1));
  const R t = tau > R(0) ? R(1) / (tau + w) : R(1) / (tau - w);
  const R sign_t = t > R(0) ? R(1) : R(-1);
  const R n = R(1) / sqrt(t * t + R(1));
  r.s = -sign_t * (y / ab(y)) * ab(t) * n;
  r.c = n;
  return r;
}

struct SvdFlags {
  int dummy;
};

template <class R> struct Svd {
  M3<R> U, V;
  V3<R> S;
};

// Eigen 3.4 JacobiSVD for a square 3x3 (unsigned, descending), then the
// reference's det(U)/det(V) flips onto s3 (src/linalg.cpp:117-124).
template <class R> NSD_HD Svd<R> svd3_signed(const M3<R>& f) {
  const R prec = R(2) * Lim<R>::eps();
  const R tiny = Lim<R>::tiny();
  R scale = R(0);
  bool finite = true;
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    finite = finite && isfinite(f.a[i]);
    scale = mx(scale, ab(f.a[i]));
  }
  Svd<R> out;
  out.U = m3_identity<R>();
  out.V = m3_identity<R>();
  if (!finite) {
    const R nan = R(0) / R(0);
    out.S = v3(nan, nan, nan);
    return out;
  }
  if (scale == R(0)) scale = R(1);
  M3<R> w;
#pragma unroll
  for (int i = 0; i < 9; ++i) w.a[i] = f.a[i] / scale;
  R maxd = mx(ab(w(0, 0)), mx(ab(w(1, 1)), ab(w(2, 2))));
  bool finished = false;
  int guard = 0;
  while (!finished && guard < 64) {
    finished = true;
    ++guard;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 0 ? 1 : 2;
      const int q = pq == 2 ? 1 : 0;
      const R thr = mx(tiny, prec * maxd);
      if (ab(w(p, q)) > thr || ab(w(q, p)) > thr) {
        finished = false;
        // real_2x2_jacobi_svd
        const R m00 = w(p, p), m01 = w(p, q), m10 = w(q, p), m11 = w(q, q);
        PRot<R> r1;
        const R t = m00 + m11, d = m10 - m01;
        if (ab(d) < tiny) {
          r1.s = R(0);
          r1.c = R(1);
        } else {
          const R u = t / d;
          const R tmp = sqrt(R(1) + u * u);
          r1.s = R(1) / tmp;
          r1.c = u / tmp;
        }
        const R n00 = r1.c * m00 + r1.s * m10, n01 = r1.c * m01 + r1.s * m11;
        const R n11 = -r1.s * m01 + r1.c * m11;
        const PRot<R> jr = jacobi_rot(n00, n01, n11);
        // j_left = rot1 * j_right^T
        PRot<R> jl;
        jl.c = r1.c * jr.c + r1.s * jr.s;
        jl.s = r1.c * (-jr.s) + r1.s * jr.c;
        prot_rows(w, p, q, jl);
        prot_cols(out.U, p, q, PRot<R>{jl.c, -jl.s});  // U.applyOnTheRight(p,q,j_left^T)
        prot_cols(w, p, q, jr);
        prot_cols(out.V, p, q, jr);
        maxd = mx(maxd, mx(ab(w(p, p)), ab(w(q, q))));
      }
    }
  }
  R s[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const R a = w(i, i);
    s[i] = ab(a);
    if (a < R(0)) {
#pragma unroll
      for (int r = 0; r < 3; ++r) out.U(r, i) = -out.U(r, i);
    }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) s[i] *= scale;
  // selection sort, first index of the max, stop at a zero max
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    int pos = i;
    R best = s[i];
#pragma unroll
    for (int k = i + 1; k < 3; ++k)
      if (s[k] > best) {
        best = s[k];
        pos = k;
      }
    if (best == R(0)) break;
    if (pos != i) {
      const R ts = s[i];
      s[i] = s[pos];
      s[pos] = ts;
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        R tu = out.U(r, i);
        out.U(r, i) = out.U(r, pos);
        out.U(r, pos) = tu;
        R tv = out.V(r, i);
        out.V(r, i) = out.V(r, pos);
        out.V(r, pos) = tv;
      }
    }
  }
  if (det3(out.U) < R(0)) {
#pragma unroll
    for (int r = 0; r < 3; ++r) out.U(r, 2) = -out.U(r, 2);
    s[2] = -s[2];
  }
  if (det3(out.V) < R(0)) {
#pragma unroll
    for (int r = 0; r < 3; ++r) out.V(r, 2) = -out.V(r, 2);
    s[2] = -s[2];
  }
  out.S = v3(s[0], s[1], s[2]);
  return out;
}

// ---------------- Eigen 3.4 SelfAdjointEigenSolver<3x3> ----------------
template <class R> NSD_HD R hypot_pos(R x, R y) {
  if (isinf(x) || isinf(y)) return Lim<R>::inf();
  if (isnan(x) || isnan(y)) return R(0) / R(0);
  const R p = mx(x, y);
  if (p == R(0)) return R(0);
  const R qp = mn(y, x) / p;
  return p * sqrt(R(1) + qp * qp);
}
template <class R> NSD_HD PRot<R> givens(R p, R q) {  // makeGivens, real
  PRot<R> r;
  if (q == R(0)) {
    r.c = p < R(0) ? R(-1) : R(1);
    r.s = R(0);
  } else if (p == R(0)) {
    r.c = R(0);
    r.s = q < R(0) ? R(1) : R(-1);
  } else if (ab(p) > ab(q)) {
    const R t = q / p;
    R u = sqrt(R(1) + t * t);
    if (p < R(0)) u = -u;
    r.c = R(1) / u;
    r.s = -t * r.c;
  } else {
    const R t = p / q;
    R u = sqrt(R(1) + t * t);
    if (q < R(0)) u = -u;
    r.s = R(-1) / u;
    r.c = -t * r.s;
  }
  return r;
}

// Eigenvalues ascending in val; eigenvectors as columns of vec when WithVec.
template <class R, bool WithVec> NSD_HD void sym_eig3(const M3<R>& in, V3<R>& val, M3<R>& vec) {
  R l10 = in(1, 0), l20 = in(2, 0), l21 = in(2, 1), d0 = in(0, 0), d1 = in(1, 1), d2 = in(2, 2);
  R scale = mx(mx(mx(ab(d0), ab(d1)), mx(ab(d2), ab(l10))), mx(ab(l20), ab(l21)));
  if (scale == R(0)) scale = R(1);
  l10 /= scale;
  l20 /= scale;
  l21 /= scale;
  d0 /= scale;
  d1 /= scale;
  d2 /= scale;
  R diag[3], sub[2];
  if (WithVec) vec = m3_identity<R>();
  diag[0] = d0;
  const R v1n2 = l20 * l20;
  if (v1n2 <= Lim<R>::tiny()) {
    diag[1] = d1;
    diag[2] = d2;
    sub[0] = l10;
    sub[1] = l21;
  } else {
    const R beta = sqrt(l10 * l10 + v1n2);
    const R ib = R(1) / beta;
    const R m01 = l10 * ib, m02 = l20 * ib;
    const R q = R(2) * m01 * l21 + m02 * (d2 - d1);
    diag[1] = d1 + m02 * q;
    diag[2] = d2 - m02 * q;
    sub[0] = beta;
    sub[1] = l21 - m01 * q;
    if (WithVec) {
      vec = m3_zero<R>();
      vec(0, 0) = R(1);
      vec(1, 1) = m01;
      vec(1, 2) = m02;
      vec(2, 1) = m02;
      vec(2, 2) = -m01;
    }
  }
  int end = 2, start = 0, iter = 0;
  const R tiny = Lim<R>::tiny();
  const R pinv = R(1) / Lim<R>::eps();
  while (end > 0) {
    for (int i = start; i < end; ++i) {
      if (ab(sub[i]) < tiny) {
        sub[i] = R(0);
      } else {
        const R sc = pinv * sub[i];
        if (sc * sc <= ab(diag[i]) + ab(diag[i + 1])) sub[i] = R(0);
      }
    }
    while (end > 0 && sub[end - 1] == R(0)) end--;
    if (end <= 0) break;
    iter++;
    if (iter > 90) break;
    start = end - 1;
    while (start > 0 && sub[start - 1] != R(0)) start--;
    const R td = (diag[end - 1] - diag[end]) * R(0.5);
    const R e = sub[end - 1];
    R mu = diag[end];
    if (td == R(0)) {
      mu -= ab(e);
    } else if (e != R(0)) {
      const R e2 = e * e;
      const R hh = hypot_pos(ab(td), ab(e));
      if (e2 == R(0))
        mu -= e / ((td + (td > R(0) ? hh : -hh)) / e);
      else
        mu -= e2 / (td + (td > R(0) ? hh : -hh));
    }
    R x = diag[start] - mu;
    R z = sub[start];
    for (int k = start; k < end && z != R(0); ++k) {
      const PRot<R> rt = givens(x, z);
      const R sdk = rt.s * diag[k] + rt.c * sub[k];
      const R dkp1 = rt.s * sub[k] + rt.c * diag[k + 1];
      diag[k] = rt.c * (rt.c * diag[k] - rt.s * sub[k]) - rt.s * (rt.c * sub[k] - rt.s * diag[k + 1]);
      diag[k + 1] = rt.s * sdk + rt.c * dkp1;
      sub[k] = rt.c * sdk - rt.s * dkp1;
      if (k > start) sub[k - 1] = rt.c * sub[k - 1] - rt.s * z;
      x = sub[k];
      if (k < end - 1) {
        z = -rt.s * sub[k + 1];
        sub[k + 1] = rt.c * sub[k + 1];
      }
      if (WithVec) prot_cols(vec, k, k + 1, rt);
    }
  }
  if (iter <= 90) {
    for (int i = 0; i < 2; ++i) {
      int k = i;
      R m = diag[i];
      for (int j = i + 1; j < 3; ++j)
        if (diag[j] < m) {
          m = diag[j];
          k = j;
        }
      if (k != i) {
        const R t = diag[i];
        diag[i] = diag[k];
        diag[k] = t;
        if (WithVec) {
          for (int r = 0; r < 3; ++r) {
            const R tv = vec(r, i);
            vec(r, i) = vec(r, k);
            vec(r, k) = tv;
          }
        }
      }
    }
  }
  val = v3(diag[0] * scale, diag[1] * scale, diag[2] * scale);
}

// Eigenvalue-floor projection (src/linalg.cpp:128-134).
template <class R> NSD_HD M3<R> project_psd3(const M3<R>& m) {
  V3<R> ev;
  M3<R> v;
  sym_eig3<R, true>(m, ev, v);
  const R fl = R(1e-10) * mx(ab(ev.x), mx(ab(ev.y), ab(ev.z)));
  ev.x = mx(ev.x, fl);
  ev.y = mx(ev.y, fl);
  ev.z = mx(ev.z, fl);
  M3<R> r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r(i, j) = (v(i, 0) * ev.x) * v(j, 0) + (v(i, 1) * ev.y) * v(j, 1) + (v(i, 2) * ev.z) * v(j, 2);
  return r;
}

}  // namespace nsd
