// Host/device fixed-size math for the B200 hot path.
//
// Rounding contract: the matrices that decide the warp
// masks — K^-1, R~ = K R K^-1, t~ = K t, pose inverse/compose — are computed by
// these functions on host AND device with exactly the reference's expression
// order (3-term dot products v0 + (v1 + v2), Eigen cofactor 3x3 inverse).  All
// translation units are compiled with --fmad=false, so nothing is contracted
// into FMA unless a kernel calls fma() explicitly (only reductions do).
#pragma once
#include <cmath>

#include "../../include/rgbid_b200.h"

#ifdef __CUDACC__
#define HD __host__ __device__ __forceinline__
#define HD_UNROLL _Pragma("unroll")
#else
#define HD inline
#define HD_UNROLL
#endif

namespace rgbid_b200 {

struct M3 {
  double m[3][3];
};
struct V3 {
  double v[3];
};

HD double red3(double a, double b, double c) { return a + (b + c); }
HD double dmax_std(double a, double b) { return (a < b) ? b : a; }  // std::max(a, b)
HD double dmin_std(double a, double b) { return (b < a) ? b : a; }  // std::min(a, b)

HD M3 m3_mul(const M3& a, const M3& b) {
  M3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      o.m[i][j] = red3(a.m[i][0] * b.m[0][j], a.m[i][1] * b.m[1][j], a.m[i][2] * b.m[2][j]);
  return o;
}
HD V3 m3_mulv(const M3& a, const V3& x) {
  V3 o;
  for (int i = 0; i < 3; ++i) o.v[i] = red3(a.m[i][0] * x.v[0], a.m[i][1] * x.v[1], a.m[i][2] * x.v[2]);
  return o;
}
HD M3 m3_T(const M3& a) {
  M3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o.m[i][j] = a.m[j][i];
  return o;
}
HD double cof3(const M3& a, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return a.m[i1][j1] * a.m[i2][j2] - a.m[i1][j2] * a.m[i2][j1];
}
// Eigen InverseImpl.h cofactor inverse (K().inverse() at src/warping.cpp:81).
HD M3 m3_inv(const M3& a) {
  const double c00 = cof3(a, 0, 0), c10 = cof3(a, 1, 0), c20 = cof3(a, 2, 0);
  const double det = red3(c00 * a.m[0][0], c10 * a.m[1][0], c20 * a.m[2][0]);
  const double invdet = 1.0 / det;
  M3 o;
  o.m[0][0] = c00 * invdet;
  o.m[0][1] = c10 * invdet;
  o.m[0][2] = c20 * invdet;
  o.m[1][0] = cof3(a, 0, 1) * invdet;
  o.m[1][1] = cof3(a, 1, 1) * invdet;
  o.m[1][2] = cof3(a, 2, 1) * invdet;
  o.m[2][0] = cof3(a, 0, 2) * invdet;
  o.m[2][1] = cof3(a, 1, 2) * invdet;
  o.m[2][2] = cof3(a, 2, 2) * invdet;
  return o;
}
// Intrinsics::K() — inc/camera.hpp:21-25
HD M3 K_mat(double fx, double fy, double cx, double cy) {
  M3 o;
  o.m[0][0] = fx, o.m[0][1] = 0, o.m[0][2] = cx;
  o.m[1][0] = 0, o.m[1][1] = fy, o.m[1][2] = cy;
  o.m[2][0] = 0, o.m[2][1] = 0, o.m[2][2] = 1;
  return o;
}

struct PoseD {
  M3 R;
  V3 t;
};

HD PoseD pose_from(const double* R9, const double* t3) {
  PoseD p;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) p.R.m[i][j] = R9[i * 3 + j];
    p.t.v[i] = t3[i];
  }
  return p;
}
HD void pose_to(const PoseD& p, double* R9, double* t3) {
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) R9[i * 3 + j] = p.R.m[i][j];
    t3[i] = p.t.v[i];
  }
}
// Pose::inverse — inc/geometry.hpp:31
HD PoseD pose_inverse(const PoseD& a) {
  PoseD o;
  o.R = m3_T(a.R);
  o.t = m3_mulv(o.R, a.t);
  for (int i = 0; i < 3; ++i) o.t.v[i] = -o.t.v[i];
  return o;
}
// Pose::operator* — inc/geometry.hpp:30
HD PoseD pose_compose(const PoseD& a, const PoseD& b) {
  PoseD o;
  o.R = m3_mul(a.R, b.R);
  o.t = m3_mulv(a.R, b.t);
  for (int i = 0; i < 3; ++i) o.t.v[i] = o.t.v[i] + a.t.v[i];
  return o;
}
HD M3 skew(const V3& v) {
  M3 o;
  o.m[0][0] = 0, o.m[0][1] = -v.v[2], o.m[0][2] = v.v[1];
  o.m[1][0] = v.v[2], o.m[1][1] = 0, o.m[1][2] = -v.v[0];
  o.m[2][0] = -v.v[1], o.m[2][1] = v.v[0], o.m[2][2] = 0;
  return o;
}
// so3_exp — src/geometry.cpp:15-28
HD M3 so3_exp(const V3& th) {
  const double angle = sqrt(red3(th.v[0] * th.v[0], th.v[1] * th.v[1], th.v[2] * th.v[2]));
  const M3 K = skew(th);
  double a, b;
  if (angle < 1e-4) {
    a = 1.0 - angle * angle / 6.0;
    b = 0.5 - angle * angle / 24.0;
  } else {
    a = sin(angle) / angle;
    b = (1.0 - cos(angle)) / (angle * angle);
  }
  M3 bK;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) bK.m[i][j] = b * K.m[i][j];
  const M3 bKK = m3_mul(bK, K);
  M3 R;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R.m[i][j] = ((i == j ? 1.0 : 0.0) + a * K.m[i][j]) + bKK.m[i][j];
  return R;
}
// T <- se3_exp(xi).inverse() * T — src/alignment.cpp:394 (decoupled se3_exp, src/geometry.cpp:56)
HD PoseD pose_update(const double xi[6], const PoseD& T) {
  V3 th, v;
  for (int i = 0; i < 3; ++i) {
    v.v[i] = xi[i];
    th.v[i] = xi[3 + i];
  }
  PoseD E;
  E.R = so3_exp(th);
  E.t = v;
  return pose_compose(pose_inverse(E), T);
}

// Warp matrices of inverse_geometric_warp — src/warping.cpp:79-85.
struct WarpMats {
  double Rt_BA[9], tt_BA[3], Rt_AB[9], tt_AB[3];
};
HD WarpMats warp_mats(const PoseD& T_AB, double fx, double fy, double cx, double cy) {
  const PoseD T_BA = pose_inverse(T_AB);
  const M3 Km = K_mat(fx, fy, cx, cy), Kinv = m3_inv(Km);
  const M3 a = m3_mul(m3_mul(Km, T_BA.R), Kinv);
  const V3 ta = m3_mulv(Km, T_BA.t);
  const M3 b = m3_mul(m3_mul(Km, T_AB.R), Kinv);
  const V3 tb = m3_mulv(Km, T_AB.t);
  WarpMats w;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) {
      w.Rt_BA[i * 3 + j] = a.m[i][j];
      w.Rt_AB[i * 3 + j] = b.m[i][j];
    }
    w.tt_BA[i] = ta.v[i];
    w.tt_AB[i] = tb.v[i];
  }
  return w;
}

// ---- 6x6 numerics (Eigen conventions; same algorithms as the oracle) -------

// Eigen ldlt_inplace<Lower> with diagonal pivoting + solve (src/alignment.cpp:393).
// Every loop has compile-time bounds and the pivot swaps are unrolled over the
// candidate rows, so all indices are static and the factor stays in registers
// (no local-memory round trips on the single thread that runs it): the same
// operations in the same order as the textbook loop, hence the same bits.
HD void ldlt_solve6(const double Hin[36], const double b[6], double x[6]) {
  double m[6][6], temp[6];
  int tr[6];
  HD_UNROLL
  for (int i = 0; i < 6; ++i)
    HD_UNROLL
    for (int j = 0; j < 6; ++j) m[i][j] = Hin[i * 6 + j];
  bool stop = false;
  HD_UNROLL
  for (int k = 0; k < 6; ++k) {
    if (stop) {  // a zero first pivot: identity permutation, factor abandoned
      tr[k] = k;
      continue;
    }
    int big = k;
    double bigv = fabs(m[k][k]);
    HD_UNROLL
    for (int i = k + 1; i < 6; ++i)
      if (fabs(m[i][i]) > bigv) {
        bigv = fabs(m[i][i]);
        big = i;
      }
    tr[k] = big;
    HD_UNROLL
    for (int c = k + 1; c < 6; ++c) {
      if (big != c) continue;
      HD_UNROLL
      for (int j = 0; j < k; ++j) {
        const double t = m[k][j];
        m[k][j] = m[c][j];
        m[c][j] = t;
      }
      HD_UNROLL
      for (int i = c + 1; i < 6; ++i) {
        const double t = m[i][k];
        m[i][k] = m[i][c];
        m[i][c] = t;
      }
      double t = m[k][k];
      m[k][k] = m[c][c];
      m[c][c] = t;
      HD_UNROLL
      for (int i = k + 1; i < c; ++i) {
        t = m[i][k];
        m[i][k] = m[c][i];
        m[c][i] = t;
      }
    }
    if (k > 0) {
      HD_UNROLL
      for (int j = 0; j < k; ++j) temp[j] = m[j][j] * m[k][j];
      double acc = 0.0;
      HD_UNROLL
      for (int j = 0; j < k; ++j) acc += m[k][j] * temp[j];
      m[k][k] -= acc;
      HD_UNROLL
      for (int i = k + 1; i < 6; ++i) {
        double s = 0.0;
        HD_UNROLL
        for (int j = 0; j < k; ++j) s += m[i][j] * temp[j];
        m[i][k] -= s;
      }
    }
    const double akk = m[k][k];
    const bool valid = fabs(akk) > 0.0;
    if (k == 0 && !valid) {
      tr[0] = 0;
      stop = true;
      continue;
    }
    if (k < 5 && valid)
      HD_UNROLL
      for (int i = k + 1; i < 6; ++i) m[i][k] /= akk;
  }
  HD_UNROLL
  for (int i = 0; i < 6; ++i) x[i] = b[i];
  HD_UNROLL
  for (int k = 0; k < 6; ++k)
    HD_UNROLL
    for (int c = k + 1; c < 6; ++c)
      if (tr[k] == c) {
        const double t = x[k];
        x[k] = x[c];
        x[c] = t;
      }
  HD_UNROLL
  for (int i = 0; i < 6; ++i)
    HD_UNROLL
    for (int j = 0; j < i; ++j) x[i] -= m[i][j] * x[j];
  HD_UNROLL
  for (int i = 0; i < 6; ++i) x[i] = fabs(m[i][i]) > 2.2250738585072014e-308 ? x[i] / m[i][i] : 0.0;
  HD_UNROLL
  for (int i = 5; i >= 0; --i)
    HD_UNROLL
    for (int j = i + 1; j < 6; ++j) x[i] -= m[j][i] * x[j];
  HD_UNROLL
  for (int k = 5; k >= 0; --k)
    HD_UNROLL
    for (int c = k + 1; c < 6; ++c)
      if (tr[k] == c) {
        const double t = x[k];
        x[k] = x[c];
        x[c] = t;
      }
}

// Rank test of src/alignment.cpp:342-353 without an eigensolver:
// deficient iff some diag <= 0, or the Cholesky of Hn - 1e-9 I fails, with
// Hn = D^-1/2 H D^-1/2 (<=> lambda_min(Hn) <= 1e-9; differs from the
// reference's "< 1e-9" only on exact ties).
HD bool rank_deficient6(const double H[36]) {
  double s[6];
  HD_UNROLL
  for (int i = 0; i < 6; ++i) {
    if (!(H[i * 6 + i] > 0.0)) return true;
    s[i] = 1.0 / sqrt(H[i * 6 + i]);
  }
  double a[6][6];
  HD_UNROLL
  for (int i = 0; i < 6; ++i)
    HD_UNROLL
    for (int j = 0; j < 6; ++j) a[i][j] = (s[i] * H[i * 6 + j]) * s[j] - (i == j ? 1e-9 : 0.0);
  HD_UNROLL
  for (int j = 0; j < 6; ++j) {
    double d = a[j][j];
    HD_UNROLL
    for (int k = 0; k < j; ++k) d -= a[j][k] * a[j][k];
    if (!(d > 0.0)) return true;
    d = sqrt(d);
    a[j][j] = d;
    HD_UNROLL
    for (int i = j + 1; i < 6; ++i) {
      double t = a[i][j];
      HD_UNROLL
      for (int k = 0; k < j; ++k) t -= a[i][k] * a[j][k];
      a[i][j] = t / d;
    }
  }
  return false;
}

// Eigen 6x6 inverse (partial-pivot LU) — src/alignment.cpp:433.
HD void lu_inverse6(const double a[36], double inv[36]) {
  double lu[6][6];
  int perm[6];
  for (int i = 0; i < 6; ++i) {
    perm[i] = i;
    for (int j = 0; j < 6; ++j) lu[i][j] = a[i * 6 + j];
  }
  for (int k = 0; k < 6; ++k) {
    int p = k;
    double best = fabs(lu[k][k]);
    for (int i = k + 1; i < 6; ++i)
      if (fabs(lu[i][k]) > best) {
        best = fabs(lu[i][k]);
        p = i;
      }
    if (p != k) {
      for (int j = 0; j < 6; ++j) {
        const double t = lu[k][j];
        lu[k][j] = lu[p][j];
        lu[p][j] = t;
      }
      const int t = perm[k];
      perm[k] = perm[p];
      perm[p] = t;
    }
    if (lu[k][k] != 0.0)
      for (int i = k + 1; i < 6; ++i) lu[i][k] /= lu[k][k];
    for (int i = k + 1; i < 6; ++i)
      for (int j = k + 1; j < 6; ++j) lu[i][j] -= lu[i][k] * lu[k][j];
  }
  for (int c = 0; c < 6; ++c) {
    double y[6];
    for (int i = 0; i < 6; ++i) y[i] = perm[i] == c ? 1.0 : 0.0;
    for (int i = 0; i < 6; ++i)
      for (int k = 0; k < i; ++k) y[i] -= lu[i][k] * y[k];
    for (int i = 5; i >= 0; --i) {
      for (int k = i + 1; k < 6; ++k) y[i] -= lu[i][k] * y[k];
      y[i] /= lu[i][i];
    }
    for (int i = 0; i < 6; ++i) inv[i * 6 + c] = y[i];
  }
}

}  // namespace rgbid_b200
