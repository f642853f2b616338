// Host synthetic inputs — restates the reference's own test fixtures
// (/root/reference/proj/tests/synthetic.hpp:13-59) with std::mt19937 +
// std::normal_distribution (libstdc++), so seeds reproduce the reference's
// fixture frames bit-for-bit (checked in tests/test_oracle_cpu.py).  Used by the
// tests and the parity subset of bench.py; the bench's 4096-pair workload is
// generated on the device (rgbid_synth_pair_device).
#include <cmath>
#include <cstdint>
#include <random>

#include "../../include/rgbid_b200.h"
#include "hd_math.cuh"

using namespace rgbid_b200;

namespace {

struct Tri {
  double a, b, c;
};
// argument-evaluation order matches `Vec3(g(rng), g(rng), g(rng))` under the same compiler
Tri tri(const double& a, const double& b, const double& c) { return Tri{a, b, c}; }

// tests/synthetic.hpp:24-27
double plane_texture(double x, double y) {
  return 0.5 + 0.2 * std::sin(7.3 * x) * std::cos(5.9 * y) + 0.15 * std::sin(3.1 * x + 2.7 * y) +
         0.1 * std::cos(11.0 * x - 4.0 * y);
}

// tests/synthetic.hpp:52-59
PoseD random_pose(std::mt19937& rng, double t_scale, double angle_scale) {
  std::normal_distribution<double> g;
  const Tri ax = tri(g(rng), g(rng), g(rng));
  V3 axis = {{ax.a, ax.b, ax.c}};
  double nrm = std::sqrt(red3(axis.v[0] * axis.v[0], axis.v[1] * axis.v[1], axis.v[2] * axis.v[2]));
  if (nrm < 1e-9) axis = V3{{1.0, 0.0, 0.0}};
  std::uniform_real_distribution<double> u(0.0, angle_scale);
  const double sq = red3(axis.v[0] * axis.v[0], axis.v[1] * axis.v[1], axis.v[2] * axis.v[2]);
  V3 th = axis;
  if (sq > 0.0) {
    const double s = std::sqrt(sq);
    for (double& v : th.v) v /= s;
  }
  const double mag = u(rng);
  for (double& v : th.v) v = v * mag;
  PoseD p;
  p.R = so3_exp(th);
  const Tri tt = tri(g(rng), g(rng), g(rng));
  p.t = V3{{t_scale * tt.a, t_scale * tt.b, t_scale * tt.c}};
  return p;
}

}  // namespace

extern "C" {

// tests/synthetic.hpp:31-50 (texture evaluated at tex_scale * world XY)
int rgbid_synth_render_plane(const rgbid_intrinsics* K, const rgbid_pose* T_WC, const double n[3],
                             double d, double tex_scale, double* I, double* W) {
  if (!K || !T_WC || !n || !I || !W) return RGBID_E_ARG;
  const M3 Kinv = m3_inv(K_mat(K->fx, K->fy, K->cx, K->cy));
  const PoseD T = pose_from(T_WC->R, T_WC->t);
  const V3 nv = {{n[0], n[1], n[2]}};
  const double nt = red3(nv.v[0] * T.t.v[0], nv.v[1] * T.t.v[1], nv.v[2] * T.t.v[2]);
  for (int y = 0; y < K->height; ++y)
    for (int x = 0; x < K->width; ++x) {
      const size_t i = (size_t)y * K->width + x;
      I[i] = NAN;
      W[i] = NAN;
      const V3 p = {{(double)x, (double)y, 1.0}};
      const V3 r = m3_mulv(T.R, m3_mulv(Kinv, p));
      const double denom = red3(nv.v[0] * r.v[0], nv.v[1] * r.v[1], nv.v[2] * r.v[2]);
      if (std::abs(denom) < 1e-12) continue;
      const double lambda = -(nt + d) / denom;
      if (lambda <= 0.05) continue;
      const double X = T.t.v[0] + lambda * r.v[0], Y = T.t.v[1] + lambda * r.v[1];
      I[i] = plane_texture(tex_scale * X, tex_scale * Y);
      W[i] = 1.0 / lambda;
    }
  return RGBID_OK;
}

int rgbid_synth_random_pose(uint32_t seed, int skip, double t_scale, double angle_scale,
                            rgbid_pose* out) {
  if (!out || skip < 0) return RGBID_E_ARG;
  std::mt19937 rng(seed);
  PoseD p;
  for (int i = 0; i <= skip; ++i) p = random_pose(rng, t_scale, angle_scale);
  pose_to(p, out->R, out->t);
  return RGBID_OK;
}

int rgbid_synth_add_noise(double* I, double* W, int w, int h, uint32_t seed, double sigma_i,
                          double sigma_w) {
  if (!W || w <= 0 || h <= 0) return RGBID_E_ARG;
  std::mt19937 rng(seed);
  std::normal_distribution<double> g;
  for (size_t i = 0; i < (size_t)w * h; ++i) {
    if (I && std::isfinite(I[i])) I[i] += sigma_i * g(rng);
    if (std::isfinite(W[i])) W[i] += sigma_w * g(rng);
  }
  return RGBID_OK;
}

}  // extern "C"
