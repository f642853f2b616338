// C wrapper around the UNMODIFIED reference hot-path sources — ORACLE TEST
// INFRASTRUCTURE ONLY (built into oracle/_ref/librgbid_ref.so by oracle/Makefile
// from /root/reference/proj/src/{geometry,camera,warping,alignment,fusion}.cpp
// compiled in place against oracle/eigen_shim).  Used by tests/ and by
// bench.py --impl reference as the checker / CPU reference arm; never by the
// product path.
//
// Every ref_* function forwards to the reference symbol named in its comment.
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "rgbid/alignment.hpp"
#include "rgbid/camera.hpp"
#include "rgbid/fusion.hpp"
#include "rgbid/segmentation.hpp"
#include "rgbid/warping.hpp"
#include "synthetic.hpp"  // /root/reference/proj/tests/synthetic.hpp
#include "../include/rgbid_b200.h"

using namespace rgbid;

namespace {

Intrinsics to_K(const rgbid_intrinsics* k) {
  Intrinsics K;
  K.fx = k->fx;
  K.fy = k->fy;
  K.cx = k->cx;
  K.cy = k->cy;
  for (int i = 0; i < 5; ++i) K.k[i] = k->k[i];
  K.width = k->width;
  K.height = k->height;
  return K;
}

void from_K(const Intrinsics& K, rgbid_intrinsics* k) {
  k->fx = K.fx;
  k->fy = K.fy;
  k->cx = K.cx;
  k->cy = K.cy;
  for (int i = 0; i < 5; ++i) k->k[i] = K.k[i];
  k->width = K.width;
  k->height = K.height;
}

Pose to_pose(const rgbid_pose* p) {
  Pose T;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) T.R(r, c) = p->R[r * 3 + c];
    T.t(r) = p->t[r];
  }
  return T;
}

void from_pose(const Pose& T, rgbid_pose* p) {
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) p->R[r * 3 + c] = T.R(r, c);
    p->t[r] = T.t(r);
  }
}

Image<double> to_img(const double* d, int w, int h) {
  Image<double> im(w, h);
  if (d) std::memcpy(im.data(), d, sizeof(double) * w * h);
  return im;
}

void from_img(const Image<double>& im, double* d) {
  if (d) std::memcpy(d, im.data(), sizeof(double) * im.size());
}

AlignmentConfig to_cfg(const rgbid_align_config* c) {
  AlignmentConfig cfg;
  if (!c) return cfg;
  cfg.levels = c->levels;
  cfg.iterations.assign(c->iterations, c->iterations + c->n_iterations);
  cfg.convergence_eps = c->convergence_eps;
  cfg.lambda_n_min = c->lambda_n_min;
  cfg.bilateral_sigma_space = c->bilateral_sigma_space;
  cfg.bilateral_sigma_intensity = c->bilateral_sigma_intensity;
  cfg.bilateral_sigma_depth = c->bilateral_sigma_depth;
  return cfg;
}

void mat6_out(const Mat6& m, double* o) {
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) o[r * 6 + c] = m(r, c);
}

int align_one(const double* IA, const double* WA, const double* IB, const double* WB, int w,
              int h, const rgbid_intrinsics* K, const rgbid_pose* init,
              const rgbid_align_config* cfg, rgbid_align_result* out) {
  std::memset(out, 0, sizeof(*out));
  FrameData a{to_img(IA, w, h), to_img(WA, w, h)};
  FrameData b{to_img(IB, w, h), to_img(WB, w, h)};
  try {
    const AlignmentResult r =
        align(a, b, to_K(K), init ? to_pose(init) : Pose(), to_cfg(cfg));
    from_pose(r.T_AB, &out->T_AB);
    mat6_out(r.cov, out->cov);
    out->converged = r.converged;
    out->cov_degenerate = r.cov_degenerate;
    out->n_levels = static_cast<int>(r.level_log.size());
    for (size_t i = 0; i < r.level_log.size() && i < RGBID_MAX_LEVELS; ++i) {
      out->level_log[i].level = r.level_log[i].level;
      out->level_log[i].iterations = r.level_log[i].iterations;
      out->level_log[i].final_cost = r.level_log[i].final_cost;
      out->total_iterations += r.level_log[i].iterations;
    }
    out->tdist_intensity = {r.tdist_intensity.mu, r.tdist_intensity.sigma, r.tdist_intensity.nu};
    out->tdist_depth = {r.tdist_depth.mu, r.tdist_depth.sigma, r.tdist_depth.nu};
    out->status = RGBID_OK;
  } catch (const DegenerateAlignmentError& e) {
    for (int i = 0; i < 6; ++i) out->spectrum[i] = e.spectrum(i);
    out->status = RGBID_E_DEGENERATE;
  }
  return out->status;
}

}  // namespace

extern "C" {

// src/alignment.cpp:9-30
int ref_build_pyramid(const double* I, const double* W, int w, int h, const rgbid_intrinsics* K,
                      int levels, double** out_I, double** out_W, rgbid_intrinsics* K_out) {
  FrameData f{to_img(I, w, h), to_img(W, w, h)};
  const Pyramid p = build_pyramid(f, to_K(K), levels);
  for (int l = 0; l < levels; ++l) {
    from_img(p.levels[l].intensity, out_I[l]);
    from_img(p.levels[l].inverse_depth, out_W[l]);
    from_K(p.intrinsics[l], &K_out[l]);
  }
  return 0;
}

// src/warping.cpp:76-114
int ref_inverse_geometric_warp(const double* I_B, const double* W_B, int wb, int hb,
                               const double* W_A, int w, int h, const rgbid_pose* T_AB,
                               const rgbid_intrinsics* K, double* oI, double* oW, double* omx,
                               double* omy) {
  const WarpedFrame wf = inverse_geometric_warp(to_img(I_B, wb, hb), to_img(W_B, wb, hb),
                                                to_img(W_A, w, h), to_pose(T_AB), to_K(K));
  from_img(wf.intensity, oI);
  from_img(wf.inverse_depth, oW);
  from_img(wf.map_x, omx);
  from_img(wf.map_y, omy);
  return 0;
}

// src/alignment.cpp:195-250.  jets: n x 17 doubles
// {x, y, r_I, r_W, J_I[6], J_W[6], lambda_n}; has_depth in flags[n].
long long ref_residuals_and_jacobians(const double* I_A, const double* W_A, const double* I_Bw,
                                      const double* W_Bw, int w, int h,
                                      const rgbid_intrinsics* K, double lambda_n_min,
                                      double* jets, unsigned char* flags, long long cap) {
  FrameData a{to_img(I_A, w, h), to_img(W_A, w, h)};
  WarpedFrame wb;
  wb.intensity = to_img(I_Bw, w, h);
  wb.inverse_depth = to_img(W_Bw, w, h);
  const auto js = residuals_and_jacobians(a, wb, to_K(K), lambda_n_min);
  const long long n = static_cast<long long>(js.size());
  for (long long i = 0; i < n && i < cap; ++i) {
    double* o = jets + i * 17;
    o[0] = js[i].x;
    o[1] = js[i].y;
    o[2] = js[i].r_I;
    o[3] = js[i].r_W;
    for (int k = 0; k < 6; ++k) {
      o[4 + k] = js[i].J_I(k);
      o[10 + k] = js[i].J_W(k);
    }
    o[16] = js[i].lambda_n;
    flags[i] = js[i].has_depth ? 1 : 0;
  }
  return n;
}

// inc/alignment.hpp:35
double ref_t_weight(double x, double nu) { return t_weight(x, nu); }
// src/alignment.cpp:32-43
double ref_digamma(double x) { return digamma(x); }
// src/alignment.cpp:61-101
void ref_estimate_location_scale(const double* r, long long n, double nu, rgbid_tdist* out) {
  const TDistParams p = estimate_location_scale(std::vector<double>(r, r + n), nu);
  *out = {p.mu, p.sigma, p.nu};
}
// src/alignment.cpp:109-127
double ref_estimate_nu(const double* r, long long n, double mu, double sigma) {
  return estimate_nu(std::vector<double>(r, r + n), mu, sigma);
}

// src/alignment.cpp:367-409
int ref_align(const double* IA, const double* WA, const double* IB, const double* WB, int w,
              int h, const rgbid_intrinsics* K, const rgbid_pose* init,
              const rgbid_align_config* cfg, rgbid_align_result* out) {
  return align_one(IA, WA, IB, WB, w, h, K, init, cfg, out);
}

// Independent alignments on `threads` host threads (CPU reference arm of the
// batched metric; the reference has no intra-call parallelism).
int ref_align_many(int n, const double* const* IA, const double* const* WA,
                   const double* const* IB, const double* const* WB, int w, int h,
                   const rgbid_intrinsics* K, const rgbid_pose* inits,
                   const rgbid_align_config* cfg, rgbid_align_result* out, int threads) {
  if (threads < 1) threads = 1;
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([=] {
      for (int i = t; i < n; i += threads)
        align_one(IA[i], WA[i], IB[i], WB[i], w, h, K, inits ? &inits[i] : nullptr, cfg, &out[i]);
    });
  for (auto& th : pool) th.join();
  return 0;
}

// src/alignment.cpp:411-436
int ref_filtered_hessian_covariance(const double* IA, const double* WA, const double* IB,
                                    const double* WB, int w, int h, const rgbid_intrinsics* K,
                                    const rgbid_pose* T, const rgbid_align_config* cfg,
                                    double* cov36, int* degenerate) {
  FrameData a{to_img(IA, w, h), to_img(WA, w, h)};
  FrameData b{to_img(IB, w, h), to_img(WB, w, h)};
  bool deg = false;
  const Mat6 c = filtered_hessian_covariance(a, b, to_K(K), to_pose(T), to_cfg(cfg), &deg);
  mat6_out(c, cov36);
  *degenerate = deg;
  return 0;
}

// src/alignment.cpp:252-277
int ref_bilateral_filter(const double* img, int w, int h, double ss, double sr, double* out) {
  from_img(bilateral_filter(to_img(img, w, h), ss, sr), out);
  return 0;
}

// src/segmentation.cpp:10-57
int ref_normal_map(const double* W, int w, int h, const rgbid_intrinsics* K, double* nx,
                   double* ny, double* nz) {
  const NormalMap n = normal_map(to_img(W, w, h), to_K(K));
  from_img(n.nx, nx);
  from_img(n.ny, ny);
  from_img(n.nz, nz);
  return 0;
}

// src/fusion.cpp:68-95 (kf intensity untouched, as in the reference)
int ref_integrate_frame(double* kf_I, double* kf_W, double* kf_C, const double* fI,
                        const double* fW, int w, int h, const rgbid_pose* T,
                        const rgbid_intrinsics* K, double sigma_w) {
  Keyframe kf;
  kf.intensity = to_img(kf_I, w, h);
  kf.inverse_depth = to_img(kf_W, w, h);
  kf.weight = to_img(kf_C, w, h);
  FrameData f{to_img(fI, w, h), to_img(fW, w, h)};
  integrate_frame(&kf, f, to_pose(T), to_K(K), sigma_w);
  from_img(kf.intensity, kf_I);
  from_img(kf.inverse_depth, kf_W);
  from_img(kf.weight, kf_C);
  return 0;
}

// src/fusion.cpp:26-66
int ref_covisibility_ratio(const double* IA, const double* WA, const double* IB,
                           const double* WB, int w, int h, const rgbid_pose* T_BA,
                           const rgbid_intrinsics* K, double sigma_w, double* ratio,
                           int* empty) {
  FrameData a{to_img(IA, w, h), to_img(WA, w, h)};
  FrameData b{to_img(IB, w, h), to_img(WB, w, h)};
  const CovisibilityResult r = covisibility_ratio(a, b, to_pose(T_BA), to_K(K), sigma_w);
  *ratio = r.ratio;
  *empty = r.empty_frame;
  return 0;
}

// src/camera.cpp:62-81
int ref_correct_inverse_depth(const double* Wm, int w, int h, const rgbid_depth_intrinsics* d,
                              const rgbid_intrinsics* K, int spatial, double* out) {
  DepthIntrinsics di;
  di.beta0 = d->beta0;
  di.beta1 = d->beta1;
  for (int i = 0; i < 9; ++i) {
    di.q0[i] = d->q0[i];
    di.q1[i] = d->q1[i];
  }
  di.p0 = Vec2(d->p0[0], d->p0[1]);
  from_img(correct_inverse_depth(to_img(Wm, w, h), di, to_K(K), spatial != 0), out);
  return 0;
}

// src/warping.cpp:20-74
int ref_forward_register(const double* WA, int w, int h, const rgbid_pose* T_BA,
                         const rgbid_intrinsics* KA, const rgbid_intrinsics* KB, double* out) {
  from_img(forward_register(to_img(WA, w, h), to_pose(T_BA), to_K(KA), to_K(KB)), out);
  return 0;
}

// geometry: src/geometry.cpp:15-28, :56, inc/geometry.hpp:30-31
// inverse_warp (src/warping.cpp:8-18) with the rectification map of a distorted
// sensor: f_w(p) = project(K, ((x - cx) / fx, (y - cy) / fy, 1)) = K distort(K^-1 p)
// (src/camera.cpp:11-22,41-45) — the reference's own functions composed
int ref_rectify(const double* src, int w, int h, const rgbid_intrinsics* K, double* out) {
  const Intrinsics intr = to_K(K);
  const Image<double> im = to_img(src, w, h);
  const auto f_w = [&](const Vec2& p) {
    const auto q = project(intr, Vec3((p.x() - intr.cx) / intr.fx, (p.y() - intr.cy) / intr.fy, 1.0));
    return q ? *q : Vec2(-1.0, -1.0);
  };
  from_img(inverse_warp(im, f_w, w, h), out);
  return 0;
}

// undistort (src/camera.cpp:24-39) of n normalized points; ok[i] = 0 for std::nullopt
int ref_undistort(const double* m_d, long long n, const rgbid_intrinsics* K, double* m_u,
                  unsigned char* ok) {
  const Intrinsics intr = to_K(K);
  for (long long i = 0; i < n; ++i) {
    const auto u = undistort(intr, Vec2(m_d[2 * i], m_d[2 * i + 1]));
    ok[i] = u ? 1 : 0;
    m_u[2 * i] = u ? u->x() : 0.0;
    m_u[2 * i + 1] = u ? u->y() : 0.0;
  }
  return 0;
}

int ref_so3_exp(const double theta[3], double R[9]) {
  const Mat3 m = so3_exp(Vec3(theta[0], theta[1], theta[2]));
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) R[r * 3 + c] = m(r, c);
  return 0;
}
int ref_pose_compose(const rgbid_pose* a, const rgbid_pose* b, rgbid_pose* out) {
  from_pose(to_pose(a) * to_pose(b), out);
  return 0;
}
int ref_pose_inverse(const rgbid_pose* a, rgbid_pose* out) {
  from_pose(to_pose(a).inverse(), out);
  return 0;
}
// pose update of src/alignment.cpp:394
int ref_pose_update(const double xi[6], const rgbid_pose* T, rgbid_pose* out) {
  Vec6 x;
  for (int i = 0; i < 6; ++i) x(i) = xi[i];
  from_pose(se3_exp(Twist::from_vector(x)).inverse() * to_pose(T), out);
  return 0;
}
int ref_mat3_inverse(const double m[9], double out[9]) {
  Mat3 a;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) a(r, c) = m[r * 3 + c];
  const Mat3 b = a.inverse();
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) out[r * 3 + c] = b(r, c);
  return 0;
}

// tests/synthetic.hpp:13-59 fixtures (the reference's own generators)
int ref_render_plane(const rgbid_intrinsics* K, const rgbid_pose* T_WC, const double n[3],
                     double d, double* I, double* W) {
  const FrameData f = testing::render_plane(to_K(K), to_pose(T_WC), Vec3(n[0], n[1], n[2]), d);
  from_img(f.intensity, I);
  from_img(f.inverse_depth, W);
  return 0;
}
int ref_random_pose(unsigned seed, int skip, double t_scale, double angle_scale,
                    rgbid_pose* out) {
  std::mt19937 rng(seed);
  Pose p;
  for (int i = 0; i <= skip; ++i) p = testing::random_pose(rng, t_scale, angle_scale);
  from_pose(p, out);
  return 0;
}

}  // extern "C"
