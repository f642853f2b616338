/*
 * rgbid_oracle.c — plain-C restatement of the RGBiD-SLAM front-end hot path.
 *
 * TEST INFRASTRUCTURE ONLY (the checker for tests/, smoke() and the
 * cpu_baseline "port" leg of bench.py).  Every function cites the reference
 * file:line it restates (/root/reference/proj/...).  Compiled with
 * -ffp-contract=off; expression order follows the reference source and the
 * Eigen conventions documented in oracle/eigen_shim/Eigen/src/shim.hpp
 * (3-term reductions v0 + (v1 + v2)), so results are bit-identical to the
 * reference built in oracle/_ref (checked by tests/test_oracle_cpu.py).
 */
#include "rgbid_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---- small fixed-size math (row-major 3x3) ------------------------------ */
typedef struct {
  double m[3][3];
} M3;
typedef struct {
  double v[3];
} V3;

static inline double red3(double a, double b, double c) { return a + (b + c); }

static M3 m3_mul(const M3* a, const M3* b) {
  M3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      o.m[i][j] = red3(a->m[i][0] * b->m[0][j], a->m[i][1] * b->m[1][j], a->m[i][2] * b->m[2][j]);
  return o;
}
static V3 m3_mulv(const M3* a, const V3* x) {
  V3 o;
  for (int i = 0; i < 3; ++i)
    o.v[i] = red3(a->m[i][0] * x->v[0], a->m[i][1] * x->v[1], a->m[i][2] * x->v[2]);
  return o;
}
static M3 m3_T(const M3* a) {
  M3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o.m[i][j] = a->m[j][i];
  return o;
}
static double cof3(const M3* a, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return a->m[i1][j1] * a->m[i2][j2] - a->m[i1][j2] * a->m[i2][j1];
}
/* Eigen InverseImpl.h 3x3 cofactor inverse (K().inverse(), Rt.inverse()). */
static M3 m3_inv(const M3* a) {
  const double c00 = cof3(a, 0, 0), c10 = cof3(a, 1, 0), c20 = cof3(a, 2, 0);
  const double det = red3(c00 * a->m[0][0], c10 * a->m[1][0], c20 * a->m[2][0]);
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
/* Intrinsics::K() — inc/camera.hpp:21-25 */
static M3 K_mat(const rgbid_intrinsics* K) {
  M3 o = {{{K->fx, 0, K->cx}, {0, K->fy, K->cy}, {0, 0, 1}}};
  return o;
}
static M3 pose_R(const rgbid_pose* p) {
  M3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o.m[i][j] = p->R[i * 3 + j];
  return o;
}
static V3 pose_t(const rgbid_pose* p) {
  V3 o = {{p->t[0], p->t[1], p->t[2]}};
  return o;
}
static void pose_set(rgbid_pose* p, const M3* R, const V3* t) {
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) p->R[i * 3 + j] = R->m[i][j];
    p->t[i] = t->v[i];
  }
}
/* Pose::inverse — inc/geometry.hpp:31: (R^T, -(R^T t)) */
int or_pose_inverse(const rgbid_pose* a, rgbid_pose* out) {
  const M3 R = pose_R(a), Rt = m3_T(&R);
  const V3 t = pose_t(a);
  V3 nt = m3_mulv(&Rt, &t);
  for (int i = 0; i < 3; ++i) nt.v[i] = -nt.v[i];
  pose_set(out, &Rt, &nt);
  return 0;
}
/* Pose::operator* — inc/geometry.hpp:30: (R*oR, R*ot + t) */
int or_pose_compose(const rgbid_pose* a, const rgbid_pose* b, rgbid_pose* out) {
  const M3 Ra = pose_R(a), Rb = pose_R(b);
  const V3 ta = pose_t(a), tb = pose_t(b);
  const M3 R = m3_mul(&Ra, &Rb);
  V3 t = m3_mulv(&Ra, &tb);
  for (int i = 0; i < 3; ++i) t.v[i] = t.v[i] + ta.v[i];
  pose_set(out, &R, &t);
  return 0;
}
int or_mat3_inverse(const double m[9], double out[9]) {
  M3 a;
  for (int i = 0; i < 9; ++i) a.m[i / 3][i % 3] = m[i];
  const M3 b = m3_inv(&a);
  for (int i = 0; i < 9; ++i) out[i] = b.m[i / 3][i % 3];
  return 0;
}
/* skew — inc/geometry.hpp:13-17 */
static M3 skew(const V3* v) {
  M3 o = {{{0, -v->v[2], v->v[1]}, {v->v[2], 0, -v->v[0]}, {-v->v[1], v->v[0], 0}}};
  return o;
}
/* so3_exp — src/geometry.cpp:15-28 */
static M3 so3_exp(const V3* th) {
  const double angle = sqrt(red3(th->v[0] * th->v[0], th->v[1] * th->v[1], th->v[2] * th->v[2]));
  const M3 K = skew(th);
  double a, b;
  if (angle < 1e-4) {
    a = 1.0 - angle * angle / 6.0;
    b = 0.5 - angle * angle / 24.0;
  } else {
    a = sin(angle) / angle;
    b = (1.0 - cos(angle)) / (angle * angle);
  }
  M3 bK, R;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) bK.m[i][j] = b * K.m[i][j];
  const M3 bKK = m3_mul(&bK, &K);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R.m[i][j] = ((i == j ? 1.0 : 0.0) + a * K.m[i][j]) + bKK.m[i][j];
  return R;
}
/* T <- se3_exp(xi).inverse() * T — src/alignment.cpp:394, src/geometry.cpp:56 */
int or_pose_update(const double xi[6], const rgbid_pose* T, rgbid_pose* out) {
  const V3 th = {{xi[3], xi[4], xi[5]}};
  const V3 v = {{xi[0], xi[1], xi[2]}};
  const M3 R = so3_exp(&th);
  rgbid_pose E, Einv;
  pose_set(&E, &R, &v);
  or_pose_inverse(&E, &Einv);
  return or_pose_compose(&Einv, T, out);
}

/* ---- image helpers — inc/image.hpp:29-91 -------------------------------- */
static inline int is_valid(double v) { return isfinite(v); }
static inline int in_bounds_d(int w, int h, double x, double y) {
  return x >= 0.0 && x <= w - 1.0 && y >= 0.0 && y <= h - 1.0;
}
static inline double bilinear(const double* img, int w, int h, double x, double y) {
  if (!in_bounds_d(w, h, x, y)) return NAN;
  const int x0 = (int)floor(x), y0 = (int)floor(y);
  const int x1 = x0 + 1 < w - 1 ? x0 + 1 : w - 1;
  const int y1 = y0 + 1 < h - 1 ? y0 + 1 : h - 1;
  const double fx = x - x0, fy = y - y0;
  const double v00 = img[(size_t)y0 * w + x0], v10 = img[(size_t)y0 * w + x1];
  const double v01 = img[(size_t)y1 * w + x0], v11 = img[(size_t)y1 * w + x1];
  if (!is_valid(v00) || !is_valid(v10) || !is_valid(v01) || !is_valid(v11)) return NAN;
  return (1 - fy) * ((1 - fx) * v00 + fx * v10) + fy * ((1 - fx) * v01 + fx * v11);
}
static inline double nearest(const double* img, int w, int h, double x, double y) {
  const int xi = (int)lround(x), yi = (int)lround(y);
  if (!(xi >= 0 && xi < w && yi >= 0 && yi < h)) return NAN;
  return img[(size_t)yi * w + xi];
}
void or_downsample2(const double* in, int w, int h, double* out) {
  const int ow = w / 2, oh = h / 2;
  for (int y = 0; y < oh; ++y)
    for (int x = 0; x < ow; ++x) {
      double sum = 0.0;
      int n = 0;
      for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
          const double v = in[(size_t)(2 * y + dy) * w + 2 * x + dx];
          if (is_valid(v)) {
            sum += v;
            ++n;
          }
        }
      out[(size_t)y * ow + x] = n > 0 ? sum / n : NAN;
    }
}

/* build_pyramid — src/alignment.cpp:9-30 */
static void level_K(const rgbid_intrinsics* prev, rgbid_intrinsics* k) {
  *k = *prev;
  k->fx /= 2.0;
  k->fy /= 2.0;
  k->cx = (k->cx - 0.5) / 2.0;
  k->cy = (k->cy - 0.5) / 2.0;
  k->width /= 2;
  k->height /= 2;
}
int or_build_pyramid(const double* I, const double* W, int w, int h, const rgbid_intrinsics* K,
                     int levels, double** out_I, double** out_W, rgbid_intrinsics* K_out) {
  memcpy(out_I[0], I, sizeof(double) * w * h);
  memcpy(out_W[0], W, sizeof(double) * w * h);
  K_out[0] = *K;
  int cw = w, ch = h;
  for (int l = 1; l < levels; ++l) {
    or_downsample2(out_I[l - 1], cw, ch, out_I[l]);
    or_downsample2(out_W[l - 1], cw, ch, out_W[l]);
    level_K(&K_out[l - 1], &K_out[l]);
    cw /= 2;
    ch /= 2;
  }
  return 0;
}

/* ---- warping — src/warping.cpp:76-114 ------------------------------------ */
typedef struct {
  M3 Rt_BA, Rt_AB;
  V3 tt_BA, tt_AB;
} WarpMats;

static WarpMats warp_mats(const rgbid_pose* T_AB, const rgbid_intrinsics* K) {
  WarpMats m;
  rgbid_pose T_BA;
  or_pose_inverse(T_AB, &T_BA);
  const M3 Km = K_mat(K), Kinv = m3_inv(&Km);
  const M3 R_BA = pose_R(&T_BA), R_AB = pose_R(T_AB);
  const V3 t_BA = pose_t(&T_BA), t_AB = pose_t(T_AB);
  M3 t1 = m3_mul(&Km, &R_BA);
  m.Rt_BA = m3_mul(&t1, &Kinv);
  m.tt_BA = m3_mulv(&Km, &t_BA);
  t1 = m3_mul(&Km, &R_AB);
  m.Rt_AB = m3_mul(&t1, &Kinv);
  m.tt_AB = m3_mulv(&Km, &t_AB);
  return m;
}

/* one A pixel of inverse_geometric_warp (src/warping.cpp:96-111) */
static inline void warp_pixel(const WarpMats* m, const double* I_B, const double* W_B, int wb,
                              int hb, int x, int y, double w_a, double* oI, double* oW,
                              double* omx, double* omy) {
  *oI = NAN;
  *oW = NAN;
  *omx = NAN;
  *omy = NAN;
  if (!is_valid(w_a) || w_a <= 0.0) return;
  const V3 q = {{x / w_a, y / w_a, 1.0 / w_a}};
  V3 xb = m3_mulv(&m->Rt_BA, &q);
  for (int i = 0; i < 3; ++i) xb.v[i] = xb.v[i] + m->tt_BA.v[i];
  if (xb.v[2] <= 1e-12) return;
  const double px = xb.v[0] / xb.v[2], py = xb.v[1] / xb.v[2];
  *omx = px;
  *omy = py;
  *oI = bilinear(I_B, wb, hb, px, py);
  const double w_meas = bilinear(W_B, wb, hb, px, py);
  if (!is_valid(w_meas) || w_meas <= 0.0) return;
  const double rz = red3(m->Rt_AB.m[2][0] * px, m->Rt_AB.m[2][1] * py, m->Rt_AB.m[2][2] * 1.0);
  const double za = rz / w_meas + m->tt_AB.v[2];
  if (za <= 1e-12) return;
  *oW = 1.0 / za;
}

int or_inverse_geometric_warp(const double* I_B, const double* W_B, int wb, int hb,
                              const double* W_A, int w, int h, const rgbid_pose* T_AB,
                              const rgbid_intrinsics* K, double* oI, double* oW, double* omx,
                              double* omy) {
  const WarpMats m = warp_mats(T_AB, K);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const size_t i = (size_t)y * w + x;
      double a, b, c, d;
      warp_pixel(&m, I_B, W_B, wb, hb, x, y, W_A[i], &a, &b, &c, &d);
      if (oI) oI[i] = a;
      if (oW) oW[i] = b;
      if (omx) omx[i] = c;
      if (omy) omy[i] = d;
    }
  return 0;
}

/* ---- Student-t machinery — src/alignment.cpp:32-157, inc/alignment.hpp:35 --- */
double or_t_weight(double x, double nu) { return (nu + 1.0) / (nu + x * x); }

double or_digamma(double x) {
  double result = 0.0;
  while (x < 6.0) {
    result -= 1.0 / x;
    x += 1.0;
  }
  const double inv = 1.0 / x;
  const double inv2 = inv * inv;
  result += log(x) - 0.5 * inv - inv2 * (1.0 / 12.0 - inv2 * (1.0 / 120.0 - inv2 / 252.0));
  return result;
}

#define KMAX_SAMPLE 19200
#define KSIGMA_FLOOR 1e-8

/* systematic_sample — src/alignment.cpp:50-57; returns malloc'ed copy */
static double* systematic_sample(const double* d, long long n, long long* m) {
  if (n <= KMAX_SAMPLE) {
    double* o = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
    if (n > 0) memcpy(o, d, sizeof(double) * n);
    *m = n;
    return o;
  }
  const long long stride = (n + KMAX_SAMPLE - 1) / KMAX_SAMPLE;
  double* o = (double*)malloc(sizeof(double) * (n / stride + 1));
  long long k = 0;
  for (long long i = 0; i < n; i += stride) o[k++] = d[i];
  *m = k;
  return o;
}

static inline double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */

/* estimate_location_scale — src/alignment.cpp:61-101 */
void or_estimate_location_scale(const double* res, long long n_all, double nu, rgbid_tdist* out) {
  long long n;
  double* r = systematic_sample(res, n_all, &n);
  out->mu = 0.0;
  out->sigma = 1.0;
  out->nu = nu;
  if (n == 0) {
    free(r);
    return;
  }
  double mu = 0.0;
  for (long long i = 0; i < n; ++i) mu += r[i];
  mu /= (double)n;
  double var = 0.0;
  for (long long i = 0; i < n; ++i) var += (r[i] - mu) * (r[i] - mu);
  double sigma = sqrt(var / (double)n);
  if (sigma < KSIGMA_FLOOR) {
    out->mu = mu;
    out->sigma = KSIGMA_FLOOR;
    free(r);
    return;
  }
  for (int it = 0; it < 50; ++it) {
    double wsum = 0.0, wrsum = 0.0;
    for (long long i = 0; i < n; ++i) {
      const double x = (r[i] - mu) / sigma;
      const double w = or_t_weight(x, nu);
      wsum += w;
      wrsum += w * r[i];
    }
    const double mu_new = wrsum / wsum;
    double s2 = 0.0;
    for (long long i = 0; i < n; ++i) {
      const double x = (r[i] - mu_new) / sigma;
      const double w = or_t_weight(x, nu);
      s2 += w * (r[i] - mu_new) * (r[i] - mu_new);
    }
    const double sigma_new = dmax(KSIGMA_FLOOR, sqrt(s2 / (double)n));
    const double rel = fabs(sigma_new - sigma) / sigma;
    mu = mu_new;
    sigma = sigma_new;
    if (rel < 1e-4) break;
  }
  out->mu = mu;
  out->sigma = dmax(sigma, KSIGMA_FLOOR);
  free(r);
}

/* solve_nu — src/alignment.cpp:131-157 (r already sampled) */
static double stationarity(const double* r, long long n, double mu, double sigma, double nu) {
  double acc = 0.0;
  for (long long i = 0; i < n; ++i) {
    const double x = (r[i] - mu) / sigma;
    const double w = or_t_weight(x, nu);
    acc += -or_digamma(nu / 2.0) + log(nu / 2.0) + or_digamma((nu + 1.0) / 2.0) -
           log((nu + 1.0) / 2.0) + 1.0 + log(w) - w;
  }
  return acc / (double)n;
}
static double solve_nu(const double* r, long long n, double mu, double sigma) {
  double lo = 2.0, hi = 10.0;
  double flo = stationarity(r, n, mu, sigma, lo), fhi = stationarity(r, n, mu, sigma, hi);
  if (flo * fhi > 0.0) return fhi > 0.0 ? hi : lo;
  for (int it = 0; it < 30; ++it) {
    const double mid = 0.5 * (lo + hi);
    const double fmid = stationarity(r, n, mu, sigma, mid);
    if (flo * fmid <= 0.0) {
      hi = mid;
      fhi = fmid;
    } else {
      lo = mid;
      flo = fmid;
    }
  }
  (void)fhi;
  return 0.5 * (lo + hi);
}

/* estimate_nu — src/alignment.cpp:109-127 */
double or_estimate_nu(const double* res, long long n_all, double mu, double sigma) {
  long long n;
  double* r = systematic_sample(res, n_all, &n);
  if (n == 0 || sigma <= 0.0) {
    free(r);
    return 5.0;
  }
  double nu = solve_nu(r, n, mu, sigma);
  for (int it = 0; it < 2 && nu < 9.99; ++it) {
    rgbid_tdist refit;
    or_estimate_location_scale(res, n_all, nu, &refit);
    if (refit.sigma <= 0.0) break;
    const double nu_new = solve_nu(r, n, refit.mu, refit.sigma);
    if (fabs(nu_new - nu) < 1e-3) {
      nu = nu_new;
      break;
    }
    nu = nu_new;
  }
  free(r);
  return nu;
}

/* ---- residuals and Jacobians — src/alignment.cpp:165-250 ----------------- */
static int gradient_at(const double* img, int w, int h, int x, int y, double* gx, double* gy) {
#define SAMPLE(sx, sy) (((sx) >= 0 && (sx) < w && (sy) >= 0 && (sy) < h) ? img[(size_t)(sy) * w + (sx)] : NAN)
  const double c = SAMPLE(x, y);
  if (!is_valid(c)) return 0;
  const double l = SAMPLE(x - 1, y), r = SAMPLE(x + 1, y);
  if (is_valid(l) && is_valid(r))
    *gx = (r - l) / 2.0;
  else if (is_valid(r))
    *gx = r - c;
  else if (is_valid(l))
    *gx = c - l;
  else
    return 0;
  const double u = SAMPLE(x, y - 1), d = SAMPLE(x, y + 1);
  if (is_valid(u) && is_valid(d))
    *gy = (d - u) / 2.0;
  else if (is_valid(d))
    *gy = d - c;
  else if (is_valid(u))
    *gy = c - u;
  else
    return 0;
  return 1;
#undef SAMPLE
}

typedef struct {
  double x, y, r_I, r_W, J_I[6], J_W[6], lambda_n;
} Jet;

/* one pixel of residuals_and_jacobians (src/alignment.cpp:206-246); returns
 * 0 = no jet, 1 = jet without depth, 2 = jet with depth */
static int jet_at(const double* I_A, const double* W_A, double i_b, double w_b, int w, int h,
                  int x, int y, const M3* Km, const M3* Kinv, double lambda_n_min, Jet* j) {
  const size_t i = (size_t)y * w + x;
  const double w_a = W_A[i], i_a = I_A[i];
  if (!is_valid(w_a) || w_a <= 0.0 || !is_valid(i_a) || !is_valid(i_b)) return 0;
  double gix, giy;
  if (!gradient_at(I_A, w, h, x, y, &gix, &giy)) return 0;
  const V3 p = {{(double)x, (double)y, 1.0}};
  M3 A = *Km;
  for (int r = 0; r < 3; ++r) A.m[r][2] = A.m[r][2] - p.v[r];
  V3 X = m3_mulv(Kinv, &p);
  for (int r = 0; r < 3; ++r) X.v[r] = X.v[r] / w_a;
  double M[3][6];
  const M3 S = skew(&X);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      M[r][c] = r == c ? 1.0 : 0.0;
      M[r][3 + c] = -S.m[r][c];
    }
  j->x = x;
  j->y = y;
  j->r_I = i_b - i_a;
  j->r_W = 0.0;
  j->lambda_n = 1.0;
  for (int k = 0; k < 6; ++k) j->J_W[k] = 0.0;
  {
    const double s[3] = {w_a * gix, w_a * giy, w_a * 0.0};
    double u[3];
    for (int c = 0; c < 3; ++c) u[c] = red3(s[0] * A.m[0][c], s[1] * A.m[1][c], s[2] * A.m[2][c]);
    for (int c = 0; c < 6; ++c) j->J_I[c] = red3(u[0] * M[0][c], u[1] * M[1][c], u[2] * M[2][c]);
  }
  double gwx, gwy;
  if (!(is_valid(w_b) && w_b > 0.0 && gradient_at(W_A, w, h, x, y, &gwx, &gwy))) return 1;
  j->r_W = w_b - w_a;
  double gA[3], row[3], s2[3];
  for (int c = 0; c < 3; ++c) gA[c] = red3(gwx * A.m[0][c], gwy * A.m[1][c], 0.0 * A.m[2][c]);
  const double e[3] = {w_b * 0.0, w_b * 0.0, w_b * 1.0};
  for (int c = 0; c < 3; ++c) row[c] = gA[c] + e[c];
  for (int c = 0; c < 3; ++c) s2[c] = w_a * row[c];
  for (int c = 0; c < 6; ++c) j->J_W[c] = red3(s2[0] * M[0][c], s2[1] * M[1][c], s2[2] * M[2][c]);
  double n[3] = {gA[0] / w_a + 0.0, gA[1] / w_a + 0.0, gA[2] / w_a + 1.0};
  const double nn = sqrt(red3(n[0] * n[0], n[1] * n[1], n[2] * n[2]));
  if (nn < 1e-12) {
    j->lambda_n = 1.0;
  } else {
    for (int c = 0; c < 3; ++c) n[c] /= nn;
    if (n[2] < 0)
      for (int c = 0; c < 3; ++c) n[c] = -n[c];
    V3 ray = m3_mulv(Kinv, &p);
    const double sq = red3(ray.v[0] * ray.v[0], ray.v[1] * ray.v[1], ray.v[2] * ray.v[2]);
    if (sq > 0.0) {
      const double s = sqrt(sq);
      for (int c = 0; c < 3; ++c) ray.v[c] /= s;
    }
    j->lambda_n = dmax(lambda_n_min, red3(n[0] * ray.v[0], n[1] * ray.v[1], n[2] * ray.v[2]));
  }
  return 2;
}

/* collects jets row-major; returns count (jets/flags may be NULL) */
static long long collect_jets(const double* I_A, const double* W_A, const double* I_Bw,
                              const double* W_Bw, int w, int h, const rgbid_intrinsics* K,
                              double lambda_n_min, Jet* jets, unsigned char* flags, long long cap) {
  const M3 Km = K_mat(K), Kinv = m3_inv(&Km);
  long long n = 0;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      Jet j;
      const size_t i = (size_t)y * w + x;
      const int r = jet_at(I_A, W_A, I_Bw[i], W_Bw[i], w, h, x, y, &Km, &Kinv, lambda_n_min, &j);
      if (!r) continue;
      if (n < cap) {
        if (jets) jets[n] = j;
        if (flags) flags[n] = (unsigned char)(r == 2);
      }
      ++n;
    }
  return n;
}

long long or_residuals_and_jacobians(const double* I_A, const double* W_A, const double* I_Bw,
                                     const double* W_Bw, int w, int h, const rgbid_intrinsics* K,
                                     double lambda_n_min, double* jets, unsigned char* flags,
                                     long long cap) {
  Jet* tmp = (Jet*)malloc(sizeof(Jet) * (size_t)(cap > 0 ? cap : 1));
  const long long n = collect_jets(I_A, W_A, I_Bw, W_Bw, w, h, K, lambda_n_min, tmp, flags, cap);
  for (long long i = 0; i < n && i < cap; ++i) memcpy(jets + i * 17, &tmp[i], sizeof(Jet));
  free(tmp);
  return n;
}

/* ---- build_system — src/alignment.cpp:281-337 ----------------------------- */
typedef struct {
  double H[6][6], b[6], cost;
  rgbid_tdist tI, tW;
} WSys;

static void refit_location_scale(const double* res, long long n, rgbid_tdist* t) {
  if (t->nu >= 4.99) return;
  rgbid_tdist refit;
  or_estimate_location_scale(res, n, t->nu, &refit);
  if (refit.sigma <= 0.0) return;
  t->mu = refit.mu;
  t->sigma = dmax(refit.sigma, 1e-8);
}

static WSys build_system(const Jet* jets, const unsigned char* hd, long long n) {
  WSys s;
  memset(&s, 0, sizeof(s));
  double* res_i = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double* res_w = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  long long ni = 0, nw = 0;
  for (long long k = 0; k < n; ++k) {
    res_i[ni++] = jets[k].r_I;
    if (hd[k]) res_w[nw++] = jets[k].r_W;
  }
  or_estimate_location_scale(res_i, ni, 5.0, &s.tI);
  or_estimate_location_scale(res_w, nw, 5.0, &s.tW);
  s.tI.sigma = dmax(s.tI.sigma, 1e-8);
  s.tW.sigma = dmax(s.tW.sigma, 1e-8);
  s.tI.nu = or_estimate_nu(res_i, ni, s.tI.mu, s.tI.sigma);
  s.tW.nu = or_estimate_nu(res_w, nw, s.tW.mu, s.tW.sigma);
  refit_location_scale(res_i, ni, &s.tI);
  refit_location_scale(res_w, nw, &s.tW);
  s.tI.nu = dmax(s.tI.nu, s.tW.nu);
  const double s2i = s.tI.sigma * s.tI.sigma;
  const double s2w = s.tW.sigma * s.tW.sigma;
  for (long long k = 0; k < n; ++k) {
    const Jet* j = &jets[k];
    const double wi = or_t_weight((j->r_I - s.tI.mu) / s.tI.sigma, s.tI.nu) / s2i;
    for (int a = 0; a < 6; ++a) {
      const double va = wi * j->J_I[a];
      for (int c = 0; c < 6; ++c) s.H[a][c] += va * j->J_I[c];
    }
    for (int a = 0; a < 6; ++a) s.b[a] -= (wi * j->J_I[a]) * j->r_I;
    s.cost += wi * j->r_I * j->r_I;
    if (hd[k]) {
      const double ww =
          j->lambda_n * or_t_weight((j->r_W - s.tW.mu) / s.tW.sigma, s.tW.nu) / s2w;
      for (int a = 0; a < 6; ++a) {
        const double va = ww * j->J_W[a];
        for (int c = 0; c < 6; ++c) s.H[a][c] += va * j->J_W[c];
      }
      for (int a = 0; a < 6; ++a) s.b[a] -= (ww * j->J_W[a]) * j->r_W;
      s.cost += ww * j->r_W * j->r_W;
    }
  }
  free(res_i);
  free(res_w);
  return s;
}

/* ---- 6x6 numerics (Eigen conventions, see shim.hpp) ----------------------- */
static void jacobi_eigenvalues6(const double H[6][6], double ev[6]) {
  double s[6][6];
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j <= i; ++j) s[i][j] = s[j][i] = H[i][j];
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < 6; ++i)
      for (int j = i + 1; j < 6; ++j) off += s[i][j] * s[i][j];
    if (off == 0.0) break;
    for (int p = 0; p < 6; ++p)
      for (int q = p + 1; q < 6; ++q) {
        if (s[p][q] == 0.0) continue;
        const double theta = (s[q][q] - s[p][p]) / (2.0 * s[p][q]);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
        for (int k = 0; k < 6; ++k) {
          const double skp = s[k][p], skq = s[k][q];
          s[k][p] = c * skp - sn * skq;
          s[k][q] = sn * skp + c * skq;
        }
        for (int k = 0; k < 6; ++k) {
          const double spk = s[p][k], sqk = s[q][k];
          s[p][k] = c * spk - sn * sqk;
          s[q][k] = sn * spk + c * sqk;
        }
      }
  }
  for (int i = 0; i < 6; ++i) ev[i] = s[i][i];
  for (int i = 1; i < 6; ++i)
    for (int j = i; j > 0 && ev[j] < ev[j - 1]; --j) {
      const double t = ev[j];
      ev[j] = ev[j - 1];
      ev[j - 1] = t;
    }
}

/* rank_deficient — src/alignment.cpp:342-353 */
static int rank_deficient(const double H[6][6], double spectrum[6]) {
  double d[6];
  int bad = 0;
  for (int i = 0; i < 6; ++i) {
    d[i] = H[i][i];
    if (d[i] <= 0.0) bad = 1;
  }
  if (bad) {
    if (spectrum) memcpy(spectrum, d, sizeof(d));
    return 1;
  }
  double s[6], Hn[6][6], ev[6];
  for (int i = 0; i < 6; ++i) s[i] = 1.0 / sqrt(d[i]);
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) Hn[i][j] = (s[i] * H[i][j]) * s[j];
  jacobi_eigenvalues6(Hn, ev);
  if (spectrum) memcpy(spectrum, ev, sizeof(ev));
  double mn = ev[0];
  for (int i = 1; i < 6; ++i)
    if (ev[i] < mn) mn = ev[i];
  return mn < 1e-9;
}

/* Eigen ldlt_inplace<Lower> + solve (lower triangle referenced) */
static void ldlt_solve6(const double Hin[6][6], const double b[6], double x[6]) {
  double m[6][6], temp[6];
  int tr[6];
  memcpy(m, Hin, sizeof(m));
  for (int k = 0; k < 6; ++k) {
    int big = k;
    double bigv = fabs(m[k][k]);
    for (int i = k + 1; i < 6; ++i)
      if (fabs(m[i][i]) > bigv) {
        bigv = fabs(m[i][i]);
        big = i;
      }
    tr[k] = big;
    if (k != big) {
      for (int j = 0; j < k; ++j) {
        double t = m[k][j];
        m[k][j] = m[big][j];
        m[big][j] = t;
      }
      for (int i = big + 1; i < 6; ++i) {
        double t = m[i][k];
        m[i][k] = m[i][big];
        m[i][big] = t;
      }
      double t = m[k][k];
      m[k][k] = m[big][big];
      m[big][big] = t;
      for (int i = k + 1; i < big; ++i) {
        t = m[i][k];
        m[i][k] = m[big][i];
        m[big][i] = t;
      }
    }
    if (k > 0) {
      for (int j = 0; j < k; ++j) temp[j] = m[j][j] * m[k][j];
      double acc = 0.0;
      for (int j = 0; j < k; ++j) acc += m[k][j] * temp[j];
      m[k][k] -= acc;
      for (int i = k + 1; i < 6; ++i) {
        double s = 0.0;
        for (int j = 0; j < k; ++j) s += m[i][j] * temp[j];
        m[i][k] -= s;
      }
    }
    const double akk = m[k][k];
    const int valid = fabs(akk) > 0.0;
    if (k == 0 && !valid) {
      for (int j = 0; j < 6; ++j) tr[j] = j;
      break;
    }
    if (k < 5 && valid)
      for (int i = k + 1; i < 6; ++i) m[i][k] /= akk;
  }
  for (int i = 0; i < 6; ++i) x[i] = b[i];
  for (int k = 0; k < 6; ++k) {
    const double t = x[k];
    x[k] = x[tr[k]];
    x[tr[k]] = t;
  }
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < i; ++j) x[i] -= m[i][j] * x[j];
  for (int i = 0; i < 6; ++i) x[i] = fabs(m[i][i]) > 2.2250738585072014e-308 ? x[i] / m[i][i] : 0.0;
  for (int i = 5; i >= 0; --i)
    for (int j = i + 1; j < 6; ++j) x[i] -= m[j][i] * x[j];
  for (int k = 5; k >= 0; --k) {
    const double t = x[k];
    x[k] = x[tr[k]];
    x[tr[k]] = t;
  }
}

/* partial-pivot LU inverse (Eigen 6x6 inverse via PartialPivLU) */
static void lu_inverse6(const double a[6][6], double inv[6][6]) {
  double lu[6][6];
  int perm[6];
  memcpy(lu, a, sizeof(lu));
  for (int i = 0; i < 6; ++i) perm[i] = i;
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
    for (int i = 0; i < 6; ++i) inv[i][c] = y[i];
  }
}

/* ---- bilateral + filtered Hessian covariance — src/alignment.cpp:252-277, 411-436 */
int or_bilateral_filter(const double* img, int w, int h, double ss, double sr, double* out) {
  const int radius = 2;
  const double inv2ss = 1.0 / (2.0 * ss * ss);
  const double inv2sr = 1.0 / (2.0 * sr * sr);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const double c = img[(size_t)y * w + x];
      out[(size_t)y * w + x] = NAN;
      if (!is_valid(c)) continue;
      double wsum = 0.0, vsum = 0.0;
      for (int dy = -radius; dy <= radius; ++dy)
        for (int dx = -radius; dx <= radius; ++dx) {
          const int sx = x + dx, sy = y + dy;
          if (!(sx >= 0 && sx < w && sy >= 0 && sy < h)) continue;
          const double v = img[(size_t)sy * w + sx];
          if (!is_valid(v)) continue;
          const double wt = exp(-(dx * dx + dy * dy) * inv2ss - (v - c) * (v - c) * inv2sr);
          wsum += wt;
          vsum += wt * v;
        }
      out[(size_t)y * w + x] = vsum / wsum;
    }
  return 0;
}

static void default_cfg(rgbid_align_config* c) {
  memset(c, 0, sizeof(*c));
  c->levels = 3;
  c->n_iterations = 3;
  c->iterations[0] = 10;
  c->iterations[1] = 5;
  c->iterations[2] = 4;
  c->convergence_eps = 1e-6;
  c->lambda_n_min = 0.1;
  c->bilateral_sigma_space = 2.0;
  c->bilateral_sigma_intensity = 0.05;
  c->bilateral_sigma_depth = 0.02;
}

int or_filtered_hessian_covariance(const double* IA, const double* WA, const double* IB,
                                   const double* WB, int w, int h, const rgbid_intrinsics* K,
                                   const rgbid_pose* T, const rgbid_align_config* cfg_in,
                                   double* cov36, int* degenerate) {
  rgbid_align_config cfg;
  if (cfg_in)
    cfg = *cfg_in;
  else
    default_cfg(&cfg);
  const size_t N = (size_t)w * h;
  double* fI = (double*)malloc(sizeof(double) * N);
  double* fW = (double*)malloc(sizeof(double) * N);
  double* wI = (double*)malloc(sizeof(double) * N);
  double* wW = (double*)malloc(sizeof(double) * N);
  Jet* jets = (Jet*)malloc(sizeof(Jet) * N);
  unsigned char* hd = (unsigned char*)malloc(N);
  or_bilateral_filter(IA, w, h, cfg.bilateral_sigma_space, cfg.bilateral_sigma_intensity, fI);
  or_bilateral_filter(WA, w, h, cfg.bilateral_sigma_space, cfg.bilateral_sigma_depth, fW);
  or_inverse_geometric_warp(IB, WB, w, h, fW, w, h, T, K, wI, wW, NULL, NULL);
  const long long n = collect_jets(fI, fW, wI, wW, w, h, K, cfg.lambda_n_min, jets, hd, (long long)N);
  if (degenerate) *degenerate = 0;
  for (int i = 0; i < 36; ++i) cov36[i] = (i % 7 == 0) ? 1e6 : 0.0;
  if (n < 6) {
    if (degenerate) *degenerate = 1;
  } else {
    const WSys s = build_system(jets, hd, n);
    double H[6][6], inv[6][6];
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) H[i][j] = (s.H[i][j] + s.H[j][i]) / 2.0;
    if (rank_deficient(H, NULL)) {
      if (degenerate) *degenerate = 1;
    } else {
      lu_inverse6(H, inv);
      for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) cov36[i * 6 + j] = (inv[i][j] + inv[j][i]) / 2.0;
    }
  }
  free(fI);
  free(fW);
  free(wI);
  free(wW);
  free(jets);
  free(hd);
  return 0;
}

/* ---- align — src/alignment.cpp:367-409 ------------------------------------ */
int or_align(const double* IA, const double* WA, const double* IB, const double* WB, int w, int h,
             const rgbid_intrinsics* K, const rgbid_pose* init, const rgbid_align_config* cfg_in,
             rgbid_align_result* out, rgbid_iter_trace* trace, int max_trace, int* n_trace) {
  rgbid_align_config cfg;
  if (cfg_in)
    cfg = *cfg_in;
  else
    default_cfg(&cfg);
  memset(out, 0, sizeof(*out));
  if (n_trace) *n_trace = 0;
  const int L = cfg.levels;
  const size_t N = (size_t)w * h;
  double *pI[RGBID_MAX_LEVELS], *pW[RGBID_MAX_LEVELS];
  rgbid_intrinsics pK[RGBID_MAX_LEVELS];
  for (int l = 0; l < L; ++l) {
    pI[l] = (double*)malloc(sizeof(double) * N);
    pW[l] = (double*)malloc(sizeof(double) * N);
  }
  or_build_pyramid(IA, WA, w, h, K, L, pI, pW, pK);
  double* wI = (double*)malloc(sizeof(double) * N);
  double* wW = (double*)malloc(sizeof(double) * N);
  double* tI = (double*)malloc(sizeof(double) * N);
  double* tW = (double*)malloc(sizeof(double) * N);
  Jet* jets = (Jet*)malloc(sizeof(Jet) * N);
  unsigned char* hd = (unsigned char*)malloc(N);
  rgbid_pose T;
  if (init) {
    T = *init;
  } else {
    memset(&T, 0, sizeof(T));
    T.R[0] = T.R[4] = T.R[8] = 1.0;
  }
  int status = RGBID_OK;
  for (int level = L - 1; level >= 0 && status == RGBID_OK; --level) {
    const int iters = level < cfg.n_iterations ? cfg.iterations[level] : 5;
    rgbid_level_log log = {level, 0, 0.0};
    int lw = w, lh = h;
    for (int l = 0; l < level; ++l) {
      lw /= 2;
      lh /= 2;
    }
    for (int it = 0; it < iters; ++it) {
      or_inverse_geometric_warp(IB, WB, w, h, WA, w, h, &T, K, wI, wW, NULL, NULL);
      /* downsample_to_level — src/alignment.cpp:355-363 */
      int cw = w, ch = h;
      for (int l = 0; l < level; ++l) {
        or_downsample2(wI, cw, ch, tI);
        or_downsample2(wW, cw, ch, tW);
        cw /= 2;
        ch /= 2;
        memcpy(wI, tI, sizeof(double) * (size_t)cw * ch);
        memcpy(wW, tW, sizeof(double) * (size_t)cw * ch);
      }
      const long long n =
          collect_jets(pI[level], pW[level], wI, wW, lw, lh, &pK[level], cfg.lambda_n_min, jets,
                       hd, (long long)N);
      if (n < 6) {
        memset(out->spectrum, 0, sizeof(out->spectrum));
        status = RGBID_E_DEGENERATE;
        break;
      }
      const WSys s = build_system(jets, hd, n);
      double spectrum[6];
      if (rank_deficient(s.H, spectrum)) {
        memcpy(out->spectrum, spectrum, sizeof(spectrum));
        status = RGBID_E_DEGENERATE;
        break;
      }
      double xi[6];
      ldlt_solve6(s.H, s.b, xi);
      rgbid_pose Tn;
      or_pose_update(xi, &T, &Tn);
      T = Tn;
      ++log.iterations;
      log.final_cost = s.cost;
      if (level == 0) {
        out->tdist_intensity = s.tI;
        out->tdist_depth = s.tW;
      }
      if (trace && n_trace && *n_trace < max_trace) {
        rgbid_iter_trace* tr = &trace[(*n_trace)++];
        tr->level = level;
        tr->iter = it;
        tr->n_jets = n;
        long long nd = 0;
        for (long long k = 0; k < n; ++k) nd += hd[k];
        tr->n_depth = nd;
        tr->tI = s.tI;
        tr->tW = s.tW;
        for (int a = 0; a < 6; ++a) {
          for (int c = 0; c < 6; ++c) tr->H[a * 6 + c] = s.H[a][c];
          tr->b[a] = s.b[a];
          tr->xi[a] = xi[a];
        }
        tr->cost = s.cost;
        tr->T_after = T;
      }
      const double xn = sqrt((xi[0] * xi[0] + (xi[1] * xi[1] + xi[2] * xi[2])) +
                             (xi[3] * xi[3] + (xi[4] * xi[4] + xi[5] * xi[5])));
      out->total_iterations++;
      if (xn < cfg.convergence_eps) break;
    }
    if (status != RGBID_OK) break;
    out->level_log[out->n_levels++] = log;
  }
  if (status == RGBID_OK) {
    out->T_AB = T;
    out->converged = 1;
    or_filtered_hessian_covariance(IA, WA, IB, WB, w, h, K, &T, &cfg, out->cov, &out->cov_degenerate);
  }
  out->status = status;
  for (int l = 0; l < L; ++l) {
    free(pI[l]);
    free(pW[l]);
  }
  free(wI);
  free(wW);
  free(tI);
  free(tW);
  free(jets);
  free(hd);
  return status;
}

/* independent alignments on host threads (cpu_baseline "port" leg) */
typedef struct {
  int t, threads, n, w, h;
  const double *const *IA, *const *WA, *const *IB, *const *WB;
  const rgbid_intrinsics* K;
  const rgbid_pose* inits;
  const rgbid_align_config* cfg;
  rgbid_align_result* out;
} ManyArg;

static void* many_worker(void* p) {
  ManyArg* a = (ManyArg*)p;
  for (int i = a->t; i < a->n; i += a->threads)
    or_align(a->IA[i], a->WA[i], a->IB[i], a->WB[i], a->w, a->h, a->K,
             a->inits ? &a->inits[i] : NULL, a->cfg, &a->out[i], NULL, 0, NULL);
  return NULL;
}

int or_align_many(int n, const double* const* IA, const double* const* WA,
                  const double* const* IB, const double* const* WB, int w, int h,
                  const rgbid_intrinsics* K, const rgbid_pose* inits,
                  const rgbid_align_config* cfg, rgbid_align_result* out, int threads) {
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  ManyArg* args = (ManyArg*)malloc(sizeof(ManyArg) * threads);
  for (int t = 0; t < threads; ++t) {
    ManyArg a = {t, threads, n, w, h, IA, WA, IB, WB, K, inits, cfg, out};
    args[t] = a;
    pthread_create(&th[t], NULL, many_worker, &args[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(args);
  return 0;
}

/* ---- fusion — src/fusion.cpp:26-95 ----------------------------------------- */
int or_integrate_frame(double* kf_W, double* kf_C, const double* fI, const double* fW, int w,
                       int h, const rgbid_pose* T, const rgbid_intrinsics* K, double sigma_w) {
  (void)fI; /* the warped intensity is computed but never used (src/fusion.cpp:70-71) */
  const WarpMats m = warp_mats(T, K);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const size_t i = (size_t)y * w + x;
      const double w_kf = kf_W[i];
      double wi, w_new, bx, by;
      warp_pixel(&m, fI ? fI : fW, fW, w, h, x, y, w_kf, &wi, &w_new, &bx, &by);
      if (!is_valid(w_kf) || !is_valid(w_new)) continue;
      if (fabs(w_new - w_kf) >= 3.0 * sigma_w) continue;
      const double w_b = bilinear(fW, w, h, bx, by);
      if (!is_valid(w_b)) continue;
      const double num = 1.0 - w_b * m.tt_BA.v[2];
      const double den = red3(m.Rt_BA.m[2][0] * x, m.Rt_BA.m[2][1] * y, m.Rt_BA.m[2][2] * 1.0);
      const double c_k = (num * num / den) * (num * num / den);
      if (!isfinite(c_k) || c_k <= 0.0) continue;
      const double c_kf = kf_C[i];
      kf_W[i] = (w_kf * c_kf + c_k * w_new) / (c_kf + c_k);
      kf_C[i] = c_kf + c_k;
    }
  return 0;
}

/* count_visible — src/fusion.cpp:26-50 */
static void count_visible(const double* WA, const double* WB, int w, int h, const rgbid_pose* T_BA,
                          const rgbid_intrinsics* K, double sigma_w, long long* valid,
                          long long* visible) {
  const M3 Km = K_mat(K), Kinv = m3_inv(&Km), R = pose_R(T_BA);
  const M3 t1 = m3_mul(&Km, &R), Rt = m3_mul(&t1, &Kinv);
  const V3 tv = pose_t(T_BA), tt = m3_mulv(&Km, &tv);
  *valid = 0;
  *visible = 0;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const double w_a = WA[(size_t)y * w + x];
      if (!is_valid(w_a) || w_a <= 0.0) continue;
      ++*valid;
      const V3 q = {{x / w_a, y / w_a, 1.0 / w_a}};
      V3 xb = m3_mulv(&Rt, &q);
      for (int i = 0; i < 3; ++i) xb.v[i] = xb.v[i] + tt.v[i];
      if (xb.v[2] <= 1e-12) continue;
      const double w_b = 1.0 / xb.v[2];
      const double px = xb.v[0] / xb.v[2], py = xb.v[1] / xb.v[2];
      if (!in_bounds_d(w, h, px, py)) continue;
      const double w_meas = bilinear(WB, w, h, px, py);
      if (!is_valid(w_meas)) continue;
      if (fabs(w_meas - w_b) < 3.0 * sigma_w) ++*visible;
    }
}

int or_covisibility_ratio(const double* WA, const double* WB, int w, int h,
                          const rgbid_pose* T_BA, const rgbid_intrinsics* K, double sigma_w,
                          double* ratio, int* empty, long long counts[4]) {
  long long va, sa, vb, sb;
  rgbid_pose T_AB;
  or_pose_inverse(T_BA, &T_AB);
  count_visible(WA, WB, w, h, T_BA, K, sigma_w, &va, &sa);
  count_visible(WB, WA, w, h, &T_AB, K, sigma_w, &vb, &sb);
  if (counts) {
    counts[0] = va;
    counts[1] = sa;
    counts[2] = vb;
    counts[3] = sb;
  }
  *ratio = 0.0;
  *empty = 0;
  if (va == 0 || vb == 0) {
    *empty = 1;
    return 0;
  }
  const double ra = (double)sa / (double)va, rb = (double)sb / (double)vb;
  *ratio = (rb < ra) ? rb : ra; /* std::min */
  return 0;
}

/* ---- depth correction + registration — src/camera.cpp:54-81, src/warping.cpp:20-74 */
static double depth_poly(const double q[9], const rgbid_intrinsics* K, double px, double py) {
  const double mx = (px - K->cx) / K->fx;
  const double my = (py - K->cy) / K->fy;
  const double r2 = mx * mx + my * my;
  return q[0] + q[1] * r2 + q[2] * r2 * r2 + q[3] * r2 * r2 * r2 + q[4] * mx + q[5] * my +
         q[6] * mx * my + q[7] * mx * mx * my + q[8] * mx * my * my;
}

int or_correct_inverse_depth(const double* Wm, int w, int h, const rgbid_depth_intrinsics* d,
                             const rgbid_intrinsics* K, int spatial, double* out) {
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const size_t i = (size_t)y * w + x;
      out[i] = NAN;
      const int sx = (int)lround(x - d->p0[0]);
      const int sy = (int)lround(y - d->p0[1]);
      if (!(sx >= 0 && sx < w && sy >= 0 && sy < h)) continue;
      const double w_m = Wm[(size_t)sy * w + sx];
      if (!is_valid(w_m)) continue;
      double v = d->beta1 * w_m + d->beta0;
      if (spatial) v = depth_poly(d->q1, K, x, y) * v + depth_poly(d->q0, K, x, y);
      out[i] = v;
    }
  return 0;
}

int or_forward_register(const double* WA, int w, int h, const rgbid_pose* T_BA,
                        const rgbid_intrinsics* KA, const rgbid_intrinsics* KB, double* out) {
  rgbid_pose T_AB;
  or_pose_inverse(T_BA, &T_AB);
  const M3 KBm = K_mat(KB), KAm = K_mat(KA), KAinv = m3_inv(&KAm), R = pose_R(T_BA);
  const M3 t1 = m3_mul(&KBm, &R), Rt_BA = m3_mul(&t1, &KAinv), Rt_AB = m3_inv(&Rt_BA);
  const V3 tab = pose_t(&T_AB), tt = m3_mulv(&KAm, &tab);
  const int iw = w > KB->width ? w : KB->width;
  const int ih = h > KB->height ? h : KB->height;
  double* inter = (double*)malloc(sizeof(double) * (size_t)iw * ih);
  for (size_t i = 0; i < (size_t)iw * ih; ++i) inter[i] = NAN;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const double wv = WA[(size_t)y * w + x];
      if (!is_valid(wv)) continue;
      const double denom = 1.0 - wv * tt.v[2];
      if (denom <= 1e-12) continue;
      const double w_bt = wv / denom;
      const double pbx = (x - wv * tt.v[0]) / denom;
      const double pby = (y - wv * tt.v[1]) / denom;
      const double half = 0.5 * (w_bt / wv);
      const int x0 = (int)lround(pbx - half), x1 = (int)lround(pbx + half);
      const int y0 = (int)lround(pby - half), y1 = (int)lround(pby + half);
      for (int ty = y0; ty <= y1; ++ty) {
        if (ty < 0 || ty >= ih) continue;
        for (int tx = x0; tx <= x1; ++tx) {
          if (tx < 0 || tx >= iw) continue;
          double* slot = &inter[(size_t)ty * iw + tx];
          if (!is_valid(*slot) || w_bt > *slot) *slot = w_bt;
        }
      }
    }
  for (int y = 0; y < KB->height; ++y)
    for (int x = 0; x < KB->width; ++x) {
      const size_t i = (size_t)y * KB->width + x;
      out[i] = NAN;
      const V3 p = {{(double)x, (double)y, 1.0}};
      const V3 rp = m3_mulv(&Rt_AB, &p);
      if (rp.v[2] <= 1e-12) continue;
      const double bx = rp.v[0] / rp.v[2], by = rp.v[1] / rp.v[2];
      const double wbt = nearest(inter, iw, ih, bx, by);
      if (!is_valid(wbt)) continue;
      out[i] = wbt * rp.v[2];
    }
  free(inter);
  return 0;
}

/* load_frame's pixel decode — src/dataset.cpp:97-116 */
int or_decode_frame(const unsigned char* bgr, const unsigned short* depth, int w, int h,
                    double scale, double* I, double* W) {
  for (int i = 0; i < w * h; ++i) {
    if (bgr) I[i] = (0.299 * bgr[3 * i + 2] + 0.587 * bgr[3 * i + 1] + 0.114 * bgr[3 * i]) / 255.0;
    W[i] = depth[i] == 0 ? NAN : scale / (double)depth[i];
  }
  return 0;
}
