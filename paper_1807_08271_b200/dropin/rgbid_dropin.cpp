// Drop-in replacement for the reference's src/alignment.cpp, src/warping.cpp and
// src/fusion.cpp: the same `namespace rgbid` functions, with the exact
// signatures of proj/include/rgbid/{alignment,warping,fusion}.hpp, implemented
// on the B200 C-ABI (include/rgbid_b200.h).  A maintainer removes those three
// .cpp files from proj/src/CMakeLists.txt, adds this file and links
// librgbid_b200.so.  Semantics follow the reference:
// exceptions (DegenerateAlignmentError with its spectrum), return-by-value
// images, integrate_frame mutating *kf in place, re-entrant per host thread.
//
// Each host thread gets its own rgbid_ctx (CUDA stream + workspaces), the
// B200 counterpart of the reference's front-end/back-end thread split
// (src/pipeline.cpp:100).  There is no CPU fallback: without a
// GPU the first call throws std::runtime_error.
#include <cmath>
#include <cstdlib>
#include <functional>
#include <optional>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "rgbid/alignment.hpp"
#include "rgbid/fusion.hpp"
#include "rgbid/warping.hpp"
#include "rgbid_b200.h"

namespace rgbid {
namespace {

struct ThreadCtx {
  rgbid_ctx* ctx = nullptr;
  rgbid_frame* fa = nullptr;
  rgbid_frame* fb = nullptr;
  ~ThreadCtx() {
    if (ctx) {
      if (fa) rgbid_frame_destroy(ctx, fa);
      if (fb) rgbid_frame_destroy(ctx, fb);
      rgbid_ctx_destroy(ctx);
    }
  }
};

ThreadCtx& tls() {
  thread_local ThreadCtx t;
  if (!t.ctx) {
    const char* dev = std::getenv("RGBID_DEVICE");
    const int rc = rgbid_ctx_create(dev ? std::atoi(dev) : 0, &t.ctx);
    if (rc != RGBID_OK)
      throw std::runtime_error(std::string("rgbid_b200: no usable B200 device: ") +
                               rgbid_status_string(rc));
  }
  return t;
}

rgbid_ctx* ctx() { return tls().ctx; }

void check(int rc, const char* what) {
  if (rc == RGBID_OK) return;
  if (rc == RGBID_E_ARG) throw std::invalid_argument(std::string(what) + ": invalid argument");
  throw std::runtime_error(std::string(what) + ": " + rgbid_status_string(rc) + " " +
                           rgbid_ctx_last_error(ctx()));
}

rgbid_intrinsics to_c(const Intrinsics& K) {
  rgbid_intrinsics k;
  k.fx = K.fx;
  k.fy = K.fy;
  k.cx = K.cx;
  k.cy = K.cy;
  for (int i = 0; i < 5; ++i) k.k[i] = K.k[i];
  k.width = K.width;
  k.height = K.height;
  return k;
}

Intrinsics from_c(const rgbid_intrinsics& k) {
  Intrinsics K;
  K.fx = k.fx;
  K.fy = k.fy;
  K.cx = k.cx;
  K.cy = k.cy;
  for (int i = 0; i < 5; ++i) K.k[i] = k.k[i];
  K.width = k.width;
  K.height = k.height;
  return K;
}

rgbid_pose to_c(const Pose& T) {
  rgbid_pose p;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) p.R[r * 3 + c] = T.R(r, c);
    p.t[r] = T.t(r);
  }
  return p;
}

Pose from_c(const rgbid_pose& p) {
  Pose T;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) T.R(r, c) = p.R[r * 3 + c];
    T.t(r) = p.t[r];
  }
  return T;
}

rgbid_align_config to_c(const AlignmentConfig& c) {
  rgbid_align_config o;
  std::memset(&o, 0, sizeof(o));
  o.levels = c.levels;
  o.n_iterations = (int)std::min<size_t>(c.iterations.size(), RGBID_MAX_LEVELS);
  for (int i = 0; i < o.n_iterations; ++i) o.iterations[i] = c.iterations[i];
  o.convergence_eps = c.convergence_eps;
  o.lambda_n_min = c.lambda_n_min;
  o.bilateral_sigma_space = c.bilateral_sigma_space;
  o.bilateral_sigma_intensity = c.bilateral_sigma_intensity;
  o.bilateral_sigma_depth = c.bilateral_sigma_depth;
  return o;
}

Mat6 mat6(const double* m) {
  Mat6 o;
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) o(r, c) = m[r * 6 + c];
  return o;
}

// upload a FrameData into one of the thread's two scratch device frames
rgbid_frame* upload(const FrameData& f, int which) {
  ThreadCtx& t = tls();
  rgbid_frame*& slot = which == 0 ? t.fa : t.fb;
  const int w = f.inverse_depth.width(), h = f.inverse_depth.height();
  static thread_local int sw[2] = {0, 0}, sh[2] = {0, 0};  // sizes of the opaque frames
  if (slot && (sw[which] != w || sh[which] != h)) {
    rgbid_frame_destroy(t.ctx, slot);
    slot = nullptr;
  }
  if (!slot) {
    check(rgbid_frame_create(t.ctx, w, h, &slot), "frame_create");
    sw[which] = w;
    sh[which] = h;
  }
  const double* I = f.intensity.empty() ? nullptr : f.intensity.data();
  check(rgbid_frame_upload(t.ctx, slot, I, f.inverse_depth.data()), "frame_upload");
  return slot;
}

}  // namespace

// ---------------------------------------------------------------- alignment.hpp

Pyramid build_pyramid(const FrameData& frame, const Intrinsics& K, int levels) {
  const int w = frame.inverse_depth.width(), h = frame.inverse_depth.height();
  Pyramid pyr;
  std::vector<Image<double>> I, W;
  std::vector<double*> pi, pw;
  int cw = w, ch = h;
  for (int l = 0; l < levels; ++l) {
    I.emplace_back(cw, ch);
    W.emplace_back(cw, ch);
    cw /= 2;
    ch /= 2;
  }
  for (int l = 0; l < levels; ++l) {
    pi.push_back(I[l].data());
    pw.push_back(W[l].data());
  }
  std::vector<rgbid_intrinsics> ks(levels);
  const rgbid_intrinsics k = to_c(K);
  check(rgbid_build_pyramid(ctx(), frame.intensity.data(), frame.inverse_depth.data(), w, h, &k,
                            levels, pi.data(), pw.data(), ks.data()),
        "build_pyramid");
  for (int l = 0; l < levels; ++l) {
    pyr.levels.push_back(FrameData{std::move(I[l]), std::move(W[l])});
    pyr.intrinsics.push_back(from_c(ks[l]));
  }
  return pyr;
}

// scalar helper of the stationarity condition (src/alignment.cpp:32-43); the
// device chain evaluates its own copy
double digamma(double x) {
  double result = 0.0;
  while (x < 6.0) {
    result -= 1.0 / x;
    x += 1.0;
  }
  const double inv = 1.0 / x;
  const double inv2 = inv * inv;
  result += std::log(x) - 0.5 * inv - inv2 * (1.0 / 12.0 - inv2 * (1.0 / 120.0 - inv2 / 252.0));
  return result;
}

TDistParams estimate_location_scale(const std::vector<double>& residuals, double nu) {
  rgbid_tdist t;
  check(rgbid_estimate_location_scale(ctx(), residuals.data(), (long long)residuals.size(), nu, &t),
        "estimate_location_scale");
  TDistParams p;
  p.mu = t.mu;
  p.sigma = t.sigma;
  p.nu = t.nu;
  return p;
}

double estimate_nu(const std::vector<double>& residuals, double mu, double sigma) {
  double nu = 5.0;
  check(rgbid_estimate_nu(ctx(), residuals.data(), (long long)residuals.size(), mu, sigma, &nu),
        "estimate_nu");
  return nu;
}

std::vector<PixelJet> residuals_and_jacobians(const FrameData& frame_a, const WarpedFrame& warped_b,
                                              const Intrinsics& K, double lambda_n_min) {
  const int w = frame_a.inverse_depth.width(), h = frame_a.inverse_depth.height();
  const size_t N = (size_t)w * h;
  std::vector<double> rec(17 * N);
  std::vector<unsigned char> hd(N);
  const rgbid_intrinsics k = to_c(K);
  const long long n = rgbid_residuals_and_jacobians(
      ctx(), frame_a.intensity.data(), frame_a.inverse_depth.data(), warped_b.intensity.data(),
      warped_b.inverse_depth.data(), w, h, &k, lambda_n_min, rec.data(), hd.data(), (long long)N);
  if (n < 0) check((int)-n, "residuals_and_jacobians");
  std::vector<PixelJet> jets((size_t)n);
  for (long long i = 0; i < n; ++i) {
    const double* o = rec.data() + 17 * i;
    PixelJet& j = jets[i];
    j.x = (int)o[0];
    j.y = (int)o[1];
    j.r_I = o[2];
    j.r_W = o[3];
    for (int c = 0; c < 6; ++c) {
      j.J_I(c) = o[4 + c];
      j.J_W(c) = o[10 + c];
    }
    j.lambda_n = o[16];
    j.has_depth = hd[i] != 0;
  }
  return jets;
}

AlignmentResult align(const FrameData& frame_a, const FrameData& frame_b, const Intrinsics& K,
                      const Pose& init, const AlignmentConfig& config) {
  const int w = frame_a.inverse_depth.width(), h = frame_a.inverse_depth.height();
  const rgbid_intrinsics k = to_c(K);
  const rgbid_pose p = to_c(init);
  const rgbid_align_config c = to_c(config);
  rgbid_align_result r;
  const int rc = rgbid_align_host(ctx(), frame_a.intensity.data(), frame_a.inverse_depth.data(),
                                  frame_b.intensity.data(), frame_b.inverse_depth.data(), w, h, &k,
                                  &p, &c, &r);
  if (rc == RGBID_E_DEGENERATE) {
    Vec6 spec;
    for (int i = 0; i < 6; ++i) spec(i) = r.spectrum[i];
    throw DegenerateAlignmentError(spec);
  }
  check(rc, "align");
  AlignmentResult out;
  out.T_AB = from_c(r.T_AB);
  out.cov = mat6(r.cov);
  out.converged = r.converged != 0;
  out.cov_degenerate = r.cov_degenerate != 0;
  for (int i = 0; i < r.n_levels; ++i) {
    LevelLog l;
    l.level = r.level_log[i].level;
    l.iterations = r.level_log[i].iterations;
    l.final_cost = r.level_log[i].final_cost;
    out.level_log.push_back(l);
  }
  out.tdist_intensity = {r.tdist_intensity.mu, r.tdist_intensity.sigma, r.tdist_intensity.nu};
  out.tdist_depth = {r.tdist_depth.mu, r.tdist_depth.sigma, r.tdist_depth.nu};
  return out;
}

Mat6 filtered_hessian_covariance(const FrameData& frame_a, const FrameData& frame_b,
                                 const Intrinsics& K, const Pose& T_AB,
                                 const AlignmentConfig& config, bool* degenerate) {
  rgbid_frame* a = upload(frame_a, 0);
  rgbid_frame* b = upload(frame_b, 1);
  const rgbid_intrinsics k = to_c(K);
  const rgbid_pose p = to_c(T_AB);
  const rgbid_align_config c = to_c(config);
  double cov[36];
  int deg = 0;
  check(rgbid_filtered_hessian_covariance(ctx(), a, b, &k, &p, &c, cov, &deg),
        "filtered_hessian_covariance");
  if (degenerate) *degenerate = deg != 0;
  return mat6(cov);
}

Image<double> bilateral_filter(const Image<double>& img, double sigma_space, double sigma_range) {
  Image<double> out(img.width(), img.height());
  check(rgbid_bilateral_filter(ctx(), img.data(), img.width(), img.height(), sigma_space,
                               sigma_range, out.data()),
        "bilateral_filter");
  return out;
}

// ---------------------------------------------------------------- warping.hpp

Image<double> inverse_warp(const Image<double>& src,
                           const std::function<Vec2(const Vec2&)>& f_w, int out_width,
                           int out_height) {
  // f_w is a host callback: evaluate the coordinate map here, sample on the device
  std::vector<double> mx((size_t)out_width * out_height), my(mx.size());
  for (int y = 0; y < out_height; ++y)
    for (int x = 0; x < out_width; ++x) {
      const Vec2 q = f_w(Vec2(x, y));
      mx[(size_t)y * out_width + x] = q.x();
      my[(size_t)y * out_width + x] = q.y();
    }
  Image<double> out(out_width, out_height);
  check(rgbid_remap_bilinear(ctx(), src.data(), src.width(), src.height(), mx.data(), my.data(),
                             out_width, out_height, out.data()),
        "inverse_warp");
  return out;
}

InverseDepthMap forward_register(const InverseDepthMap& W_A, const Pose& T_BA,
                                 const Intrinsics& K_A, const Intrinsics& K_B) {
  InverseDepthMap out(K_B.width, K_B.height);
  const rgbid_pose p = to_c(T_BA);
  const rgbid_intrinsics ka = to_c(K_A), kb = to_c(K_B);
  check(rgbid_forward_register(ctx(), W_A.data(), W_A.width(), W_A.height(), &p, &ka, &kb,
                               out.data()),
        "forward_register");
  return out;
}

WarpedFrame inverse_geometric_warp(const IntensityImage& I_B, const InverseDepthMap& W_B,
                                   const InverseDepthMap& W_A, const Pose& T_AB,
                                   const Intrinsics& K) {
  const int w = W_A.width(), h = W_A.height();
  WarpedFrame out;
  out.intensity = IntensityImage(w, h);
  out.inverse_depth = InverseDepthMap(w, h);
  out.map_x = Image<double>(w, h);
  out.map_y = Image<double>(w, h);
  const rgbid_pose p = to_c(T_AB);
  const rgbid_intrinsics k = to_c(K);
  check(rgbid_inverse_geometric_warp(ctx(), I_B.empty() ? nullptr : I_B.data(), W_B.data(),
                                     W_B.width(), W_B.height(), W_A.data(), w, h, &p, &k,
                                     out.intensity.data(), out.inverse_depth.data(),
                                     out.map_x.data(), out.map_y.data()),
        "inverse_geometric_warp");
  return out;
}

// ---------------------------------------------------------------- fusion.hpp

Keyframe make_keyframe(const FrameData& frame, const Pose& T_W_kf, int id, double timestamp) {
  Keyframe kf;
  kf.intensity = frame.intensity;
  kf.inverse_depth = frame.inverse_depth;
  kf.weight = Image<double>(frame.inverse_depth.width(), frame.inverse_depth.height(), 1.0);
  kf.T_W_kf = T_W_kf;
  kf.id = id;
  kf.timestamp = timestamp;
  return kf;
}

CovisibilityResult covisibility_ratio(const FrameData& frame_a, const FrameData& frame_b,
                                      const Pose& T_BA, const Intrinsics& K, double sigma_w) {
  rgbid_frame* a = upload(frame_a, 0);
  rgbid_frame* b = upload(frame_b, 1);
  const rgbid_pose p = to_c(T_BA);
  const rgbid_intrinsics k = to_c(K);
  CovisibilityResult r;
  int empty = 0;
  check(rgbid_covisibility_ratio(ctx(), a, b, &p, &k, sigma_w, &r.ratio, &empty, nullptr),
        "covisibility_ratio");
  r.empty_frame = empty != 0;
  return r;
}

void integrate_frame(Keyframe* kf, const FrameData& frame, const Pose& T_kf_frame,
                     const Intrinsics& K, double sigma_w) {
  const rgbid_pose p = to_c(T_kf_frame);
  const rgbid_intrinsics k = to_c(K);
  check(rgbid_integrate_frame(ctx(), kf->inverse_depth.data(), kf->weight.data(),
                              frame.intensity.empty() ? nullptr : frame.intensity.data(),
                              frame.inverse_depth.data(), kf->inverse_depth.width(),
                              kf->inverse_depth.height(), &p, &k, sigma_w),
        "integrate_frame");
}

std::optional<BufferedFrame> FrameBuffer::pop_closest(double timestamp) {
  if (frames_.empty()) return std::nullopt;
  size_t best = 0;
  double best_dt = std::abs(frames_[0].timestamp - timestamp);
  for (size_t i = 1; i < frames_.size(); ++i) {
    const double dt = std::abs(frames_[i].timestamp - timestamp);
    if (dt < best_dt) {
      best = i;
      best_dt = dt;
    }
  }
  BufferedFrame out = std::move(frames_[best]);
  frames_.erase(frames_.begin() + static_cast<long>(best));
  return out;
}

void drain_buffer_step(Keyframe* kf, FrameBuffer* buffer, const Intrinsics& K, double sigma_w) {
  auto frame = buffer->pop_closest(kf->timestamp);
  if (!frame) return;
  integrate_frame(kf, frame->frame, kf->T_W_kf.inverse() * frame->T_W_frame, K, sigma_w);
}

}  // namespace rgbid
