// Host synthetic inputs — restates the reference's own test fixtures
// (/root/reference/proj/tests/synthetic.hpp:13-59) with std::mt19937 +
// std::normal_distribution (libstdc++), so seeds reproduce the reference's
// fixture frames bit-for-bit (checked in tests/test_oracle_cpu.py), plus the
// host renderer of the benchmark scene (synth_scene.cuh).  Used by the tests and
// the parity subset of bench.py; the bench's 4096-pair workload is generated on
// the device (rgbid_synth_pair_device).  Pure host C++: oracle/Makefile also
// builds this file alone as oracle/_build/librgbid_synth.so, so the reference
// arm renders its inputs without loading the CUDA library.
#include <cmath>
#include <cstdint>
#include <algorithm>
#include <random>

#include "../../include/rgbid_b200.h"
#include "hd_math.cuh"
#include "synth_scene.cuh"

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

// host restatement of k_render (fusion_kernels.cu)
double gauss_h(unsigned long long key) {
  const unsigned long long a = synth_splitmix(key), b = synth_splitmix(key ^ 0xda3e39cb94b95bdbull);
  const double u1 = ((a >> 11) + 0.5) * (1.0 / 9007199254740992.0);
  const double u2 = ((b >> 11) + 0.5) * (1.0 / 9007199254740992.0);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}
void render_h(const SynthView& v, double* I, double* W) {
  for (int i = 0; i < v.w * v.h; ++i) {
    const int y = i / v.w, x = i - y * v.w;
    const V3 p = {{(double)x, (double)y, 1.0}};
    const V3 kp = m3_mulv(v.Kinv, p);
    const V3 r = m3_mulv(v.R, kp);
    const double denom = red3(v.n[0] * r.v[0], v.n[1] * r.v[1], v.n[2] * r.v[2]);
    double iv = std::nan(""), wv = std::nan("");
    if (std::fabs(denom) >= 1e-12) {
      const double lambda = -(red3(v.n[0] * v.t[0], v.n[1] * v.t[1], v.n[2] * v.t[2]) + v.d) / denom;
      if (lambda > 0.05) {
        const double X = v.t[0] + lambda * r.v[0], Y = v.t[1] + lambda * r.v[1];
        iv = plane_texture(v.tex_scale * X, v.tex_scale * Y);
        wv = 1.0 / lambda;
      }
    }
    if (v.noise_i > 0.0 && std::isfinite(iv)) iv += v.noise_i * gauss_h(v.seed * 0x100000000ull + 2ull * i);
    if (v.noise_w > 0.0 && std::isfinite(wv))
      wv += v.noise_w * gauss_h(v.seed * 0x100000000ull + 2ull * i + 1);
    if (v.occluder && x < v.w / 5) {
      iv = plane_texture(7.0 + 0.1 * x * 80.0 / v.w, 3.0 + 0.1 * y * 80.0 / v.w);
      wv = 1.0;
    }
    if (synth_hole_i(v, i)) iv = std::nan("");
    if (synth_hole_w(v, i, x, y)) wv = std::nan("");
    I[i] = iv;
    W[i] = wv;
  }
}

}  // namespace

namespace rgbid_b200 {
// the pair geometry and views of the benchmark scene (synth_scene.cuh)
void synth_pair_views(const rgbid_intrinsics* K, uint32_t pair_seed, int variant, SynthView* va,
                      SynthView* vb, rgbid_pose* T_AB_truth) {
  rgbid_pose pa, pab;
  rgbid_synth_random_pose(5000u + pair_seed, 0, 0.01, 0.01, &pa);
  rgbid_synth_random_pose(1000u + pair_seed, 0, 0.003, 0.02, &pab);
  const PoseD TA = pose_from(pa.R, pa.t), TAB = pose_from(pab.R, pab.t);
  const PoseD TB = pose_compose(TA, TAB);
  if (T_AB_truth) pose_to(TAB, T_AB_truth->R, T_AB_truth->t);
  double n[3] = {0.2, -0.15, 1.0};
  const double nn = std::sqrt(red3(n[0] * n[0], n[1] * n[1], n[2] * n[2]));
  for (double& v : n) v /= nn;
  auto view = [&](const PoseD& T, unsigned long long seed) {
    SynthView v;
    v.w = K->width;
    v.h = K->height;
    v.Kinv = m3_inv(K_mat(K->fx, K->fy, K->cx, K->cy));
    v.R = T.R;
    for (int i = 0; i < 3; ++i) {
      v.t[i] = T.t.v[i];
      v.n[i] = n[i];
    }
    v.d = -2.0;
    v.tex_scale = K->width / 80.0;
    v.noise_i = variant ? 0.005 : 0.0;
    v.noise_w = variant ? 0.002 : 0.0;
    v.seed = seed;
    v.occluder = 0;
    v.holes = variant == 2 ? 1 : 0;
    v.border = variant == 2 ? std::max(1, K->width / 32) : 0;
    return v;
  };
  *va = view(TA, 2u * pair_seed + 1);
  *vb = view(TB, 2u * pair_seed + 2);
  vb->occluder = variant ? 1 : 0;
}
}  // namespace rgbid_b200

extern "C" {

int rgbid_synth_pair_host(const rgbid_intrinsics* K, uint32_t pair_seed, int variant, double* IA,
                          double* WA, double* IB, double* WB, rgbid_pose* T_AB_truth) {
  if (!K || !IA || !WA || !IB || !WB || K->width <= 0 || K->height <= 0 || variant < 0 ||
      variant > 2)
    return RGBID_E_ARG;
  SynthView va, vb;
  synth_pair_views(K, pair_seed, variant, &va, &vb, T_AB_truth);
  render_h(va, IA, WA);
  render_h(vb, IB, WB);
  return RGBID_OK;
}

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
