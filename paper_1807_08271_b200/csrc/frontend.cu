// Front-end odometry driver (BASELINE config 3): a restatement of the
// reference's Pipeline front-end — process_frame / track / fuse_and_maybe_switch
// / start_keyframe / emit_keyframe (src/pipeline.cpp:120-247) — without the
// back-end thread (out of scope).  Emitted keyframes are kept as device
// snapshots instead of being pushed to the back-end queue.
//
// B200 layout: every frame, the tracking reference, the keyframe source and
// the fused keyframe maps (W, C) stay resident in HBM; the reference frame's
// pyramid is built once and reused for every frame tracked against it (the
// reference rebuilds it per align call, src/alignment.cpp:369).  Device frames
// come from a pool recycled when the last reference (tracking reference,
// keyframe source, fusion buffer) drops, so steady state allocates nothing.  Per
// frame the host only does the 6x6 covariance composition and the switch
// decisions; the device work is one stream-ordered sequence -- upload, align,
// both covisibility ratios, one fusion step -- with two host waits: the align
// result (the covisibility transforms and sigma_w depend on it) and the four
// covisibility counts, read back together.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <deque>
#include <memory>
#include <vector>

#include "../../include/rgbid_b200.h"
#include "hd_math.cuh"
#include "runtime_internal.cuh"

using namespace rgbid_b200;

namespace {

struct Mat6d {
  double m[6][6];
};

Mat6d zero6() {
  Mat6d z;
  std::memset(&z, 0, sizeof(z));
  return z;
}

Mat6d mul6(const Mat6d& a, const Mat6d& b) {
  Mat6d o = zero6();
  for (int i = 0; i < 6; ++i)
    for (int k = 0; k < 6; ++k)
      for (int j = 0; j < 6; ++j) o.m[i][j] += a.m[i][k] * b.m[k][j];
  return o;
}

Mat6d T6(const Mat6d& a) {
  Mat6d o;
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) o.m[i][j] = a.m[j][i];
  return o;
}

// compose_relative_with_cov — src/geometry.cpp:74-103 (left-referenced, decoupled)
void compose_relative_with_cov(const PoseD& T_WA, const Mat6d& covA, const PoseD& T_WB,
                               const Mat6d& covB, PoseD* rel, Mat6d* cov) {
  const M3 R_AW = m3_T(T_WA.R);
  V3 d;
  for (int i = 0; i < 3; ++i) d.v[i] = T_WA.t.v[i] - T_WB.t.v[i];
  const M3 S = m3_mul(R_AW, skew(d));
  Mat6d JA = zero6(), JB = zero6();
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      JA.m[i][j] = -R_AW.m[i][j];
      JA.m[i][3 + j] = -S.m[i][j];
      JA.m[3 + i][3 + j] = -R_AW.m[i][j];
      JB.m[i][j] = R_AW.m[i][j];
      JB.m[3 + i][3 + j] = R_AW.m[i][j];
    }
  *rel = pose_compose(pose_inverse(T_WA), T_WB);
  const Mat6d a = mul6(mul6(JA, covA), T6(JA)), b = mul6(mul6(JB, covB), T6(JB));
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) cov->m[i][j] = a.m[i][j] + b.m[i][j];
  const Mat6d c = *cov;
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) cov->m[i][j] = (c.m[i][j] + c.m[j][i]) / 2.0;
}

PoseD identity() {
  PoseD p;
  std::memset(&p, 0, sizeof(p));
  p.R.m[0][0] = p.R.m[1][1] = p.R.m[2][2] = 1.0;
  return p;
}

rgbid_pose to_c(const PoseD& p) {
  rgbid_pose o;
  pose_to(p, o.R, o.t);
  return o;
}

struct FrameRef {  // immutable device frame shared by reference / keyframe source / buffer
  std::vector<rgbid_frame*>* pool;
  rgbid_frame* f;
  ~FrameRef() { pool->push_back(f); }  // recycled, not freed
};
using FramePtr = std::shared_ptr<FrameRef>;

struct Buffered {
  FramePtr frame;
  PoseD T_W_frame;
  double timestamp;
};

}  // namespace

struct rgbid_frontend {
  rgbid_ctx* ctx;
  rgbid_intrinsics K;
  rgbid_frontend_config cfg;
  int w, h;
  // front-end state (inc/pipeline.hpp:127-139)
  FramePtr reference;
  PoseD T_W_ref = identity();
  bool has_prev = false;
  PoseD T_ref_prev = identity();
  Mat6d cov_ref_prev = zero6();
  PoseD velocity = identity();
  double sigma_w = 0.01;
  bool has_kf = false;
  rgbid_frame* kf = nullptr;  // I = source I, W = fused inverse depth (mutated)
  double* kf_C = nullptr;     // fusion weights (device)
  PoseD T_W_kf = identity();
  int kf_id = 0;
  double kf_t = 0.0;
  FramePtr kf_source;
  std::deque<Buffered> buffer;
  int next_keyframe_id = 0;
  std::vector<rgbid_frame_estimate> traj;
  std::vector<int> keyframe_frame_index;
  int emitted = 0;
  std::vector<rgbid_frame*> pool;            // free device frames
  unsigned long long* counts_dev = nullptr;  // [8]: reference and keyframe covisibility counts
  unsigned long long* counts_host = nullptr; // pinned
};

namespace {

int start_keyframe(rgbid_frontend* fe, const FramePtr& frame, double t) {
  // make_keyframe (src/fusion.cpp:7-16): W copy, C = 1 everywhere
  const PoseD T_W_k = pose_from(fe->traj.back().T_W_k.R, fe->traj.back().T_W_k.t);
  int rc = rgbid_frame_copy(fe->ctx, fe->kf, frame->f);
  if (rc) return rc;
  rc = rgbid_fill(fe->ctx, fe->kf_C, (long long)fe->w * fe->h, 1.0);
  if (rc) return rc;
  fe->T_W_kf = T_W_k;
  fe->kf_id = fe->next_keyframe_id++;
  fe->kf_t = t;
  fe->kf_source = frame;
  fe->has_kf = true;
  fe->buffer.clear();
  return RGBID_OK;
}

// drain_buffer_step — src/fusion.cpp:113-118 (pop_closest: first minimum |dt|)
int drain_buffer_step(rgbid_frontend* fe) {
  if (fe->buffer.empty()) return RGBID_OK;
  size_t best = 0;
  double best_dt = std::fabs(fe->buffer[0].timestamp - fe->kf_t);
  for (size_t i = 1; i < fe->buffer.size(); ++i) {
    const double dt = std::fabs(fe->buffer[i].timestamp - fe->kf_t);
    if (dt < best_dt) {
      best = i;
      best_dt = dt;
    }
  }
  Buffered b = fe->buffer[best];
  fe->buffer.erase(fe->buffer.begin() + (long)best);
  const rgbid_pose T = to_c(pose_compose(pose_inverse(fe->T_W_kf), b.T_W_frame));
  const rgbid_frame* fr = b.frame->f;
  return rt_integrate_async(fe->ctx, fe->kf, fe->kf_C, 1, &fr, &T, &fe->K, fe->sigma_w);
}

int emit_keyframe(rgbid_frontend* fe) {
  if (!fe->has_kf) return RGBID_OK;
  while (!fe->buffer.empty()) {
    const int rc = drain_buffer_step(fe);
    if (rc) return rc;
  }
  fe->emitted += 1;  // back-end hand-off (KeyframeQueue::push) is out of scope
  return RGBID_OK;
}

// track — src/pipeline.cpp:140-191.  The reference-covisibility counts are
// enqueued into counts_dev[0..3]; the switch is applied by finish_frame.
int track(rgbid_frontend* fe, const FramePtr& frame, double t, bool* check_ref,
          PoseD* T_W_k_out) {
  const PoseD init = pose_compose(fe->T_ref_prev, fe->velocity);
  const rgbid_pose init_c = to_c(init);
  rgbid_align_result res;
  const int rc = rgbid_align(fe->ctx, fe->reference->f, frame->f, &fe->K, &init_c, &fe->cfg.align,
                             &res);
  if (rc != RGBID_OK && rc != RGBID_E_DEGENERATE) return rc;
  const bool lost = rc == RGBID_E_DEGENERATE;
  PoseD T_ref_k;
  Mat6d step_cov = zero6();
  if (lost) {
    T_ref_k = fe->T_ref_prev;
    fe->velocity = identity();
    for (int i = 0; i < 6; ++i) step_cov.m[i][i] = 1e6;
  } else {
    T_ref_k = pose_from(res.T_AB.R, res.T_AB.t);
    fe->sigma_w = dmax_std(res.tdist_depth.sigma, 1e-6);
    Mat6d cov_k;
    for (int i = 0; i < 36; ++i) cov_k.m[i / 6][i % 6] = res.cov[i];
    PoseD rel;
    compose_relative_with_cov(fe->T_ref_prev, fe->cov_ref_prev, T_ref_k, cov_k, &rel, &step_cov);
    fe->velocity = rel;
    fe->cov_ref_prev = cov_k;
  }
  const PoseD T_W_k = pose_compose(fe->T_W_ref, T_ref_k);
  rgbid_frame_estimate e;
  std::memset(&e, 0, sizeof(e));
  e.timestamp = t;
  pose_to(T_W_k, e.T_W_k.R, e.T_W_k.t);
  for (int i = 0; i < 36; ++i) e.cov[i] = step_cov.m[i / 6][i % 6];
  e.lost = lost;
  e.keyframe_id = -1;
  fe->traj.push_back(e);
  fe->T_ref_prev = T_ref_k;
  *T_W_k_out = T_W_k;
  *check_ref = !lost;
  if (!lost) {  // reference switching keeps the photometric baseline short
    const rgbid_pose T_k_ref = to_c(pose_inverse(T_ref_k));
    return rt_covis_enqueue(fe->ctx, fe->reference->f, frame->f, &T_k_ref, &fe->K, fe->sigma_w,
                            fe->counts_dev);
  }
  return RGBID_OK;
}

// fuse_and_maybe_switch — src/pipeline.cpp:193-225, first half: buffer, one drain
// step, keyframe-covisibility counts into counts_dev[4..7]
int fuse_enqueue(rgbid_frontend* fe, const FramePtr& frame, double t) {
  const rgbid_frame_estimate last = fe->traj.back();
  const PoseD T_W_last = pose_from(last.T_W_k.R, last.T_W_k.t);
  if (fe->buffer.size() >= (size_t)fe->cfg.buffer_capacity) fe->buffer.pop_front();
  fe->buffer.push_back(Buffered{frame, T_W_last, t});
  const int rc = drain_buffer_step(fe);
  if (rc) return rc;
  const PoseD T_frame_kf = pose_compose(pose_inverse(T_W_last), fe->T_W_kf);
  const rgbid_pose T_kf_frame = to_c(pose_inverse(T_frame_kf));
  return rt_covis_enqueue(fe->ctx, fe->kf_source->f, frame->f, &T_kf_frame, &fe->K, fe->sigma_w,
                          fe->counts_dev + 4);
}

// the host wait of the frame: both covisibility ratios, then the reference switch
// (track, src/pipeline.cpp:182-190) and the keyframe switch (fuse_and_maybe_switch,
// :206-225) in the reference's order -- the first never feeds the second
int finish_frame(rgbid_frontend* fe, const FramePtr& frame, double t, bool check_ref,
                 const PoseD& T_W_k) {
  cudaStream_t st = (cudaStream_t)rgbid_ctx_stream(fe->ctx);
  if (cudaMemcpyAsync(fe->counts_host, fe->counts_dev, 8 * sizeof(unsigned long long),
                      cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return RGBID_E_CUDA;
  if (check_ref) {
    double ratio = 0.0;
    int empty = 0;
    rt_covis_ratio(fe->counts_host, &ratio, &empty);
    if (ratio < fe->cfg.reference_covisibility) {
      fe->reference = frame;
      fe->T_W_ref = T_W_k;
      fe->T_ref_prev = identity();
      fe->cov_ref_prev = zero6();
    }
  }
  const rgbid_frame_estimate last = fe->traj.back();
  const PoseD T_W_last = pose_from(last.T_W_k.R, last.T_W_k.t);
  double ratio = 0.0;
  int empty = 0;
  rt_covis_ratio(fe->counts_host + 4, &ratio, &empty);
  if (!last.lost && ratio < fe->cfg.keyframe_covisibility) {
    int rc = emit_keyframe(fe);
    if (rc) return rc;
    rc = start_keyframe(fe, frame, t);
    if (rc) return rc;
    fe->traj.back().keyframe_id = fe->next_keyframe_id - 1;
    fe->keyframe_frame_index.push_back((int)fe->traj.size() - 1);
    fe->reference = frame;  // restart tracking from the new keyframe
    fe->T_W_ref = T_W_last;
    fe->T_ref_prev = identity();
    fe->cov_ref_prev = zero6();
  }
  return RGBID_OK;
}

}  // namespace

extern "C" {

int rgbid_frontend_default_config(rgbid_frontend_config* c) {
  if (!c) return RGBID_E_ARG;
  std::memset(c, 0, sizeof(*c));
  c->align.levels = 3;
  c->align.n_iterations = 3;
  c->align.iterations[0] = 10;
  c->align.iterations[1] = 5;
  c->align.iterations[2] = 4;
  c->align.convergence_eps = 1e-6;
  c->align.lambda_n_min = 0.1;
  c->align.bilateral_sigma_space = 2.0;
  c->align.bilateral_sigma_intensity = 0.05;
  c->align.bilateral_sigma_depth = 0.02;
  c->keyframe_covisibility = 0.7;
  c->reference_covisibility = 0.9;
  c->buffer_capacity = 30;
  return RGBID_OK;
}

int rgbid_frontend_create(rgbid_ctx* ctx, const rgbid_intrinsics* K,
                          const rgbid_frontend_config* cfg, rgbid_frontend** out) {
  if (!ctx || !K || !out || K->width <= 0 || K->height <= 0) return RGBID_E_ARG;
  rgbid_frontend* fe = new rgbid_frontend();
  fe->ctx = ctx;
  fe->K = *K;
  if (cfg)
    fe->cfg = *cfg;
  else
    rgbid_frontend_default_config(&fe->cfg);
  fe->w = K->width;
  fe->h = K->height;
  int rc = rgbid_frame_create(ctx, fe->w, fe->h, &fe->kf);
  if (rc) {
    delete fe;
    return rc;
  }
  if (cudaMalloc(&fe->kf_C, sizeof(double) * fe->w * fe->h) != cudaSuccess ||
      cudaMalloc(&fe->counts_dev, 8 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMallocHost(&fe->counts_host, 8 * sizeof(unsigned long long)) != cudaSuccess) {
    rgbid_frame_destroy(ctx, fe->kf);
    cudaFree(fe->kf_C);
    cudaFree(fe->counts_dev);
    delete fe;
    return RGBID_E_OOM;
  }
  *out = fe;
  return RGBID_OK;
}

int rgbid_frontend_destroy(rgbid_frontend* fe) {
  if (!fe) return RGBID_E_ARG;
  rgbid_ctx_synchronize(fe->ctx);
  fe->reference.reset();
  fe->kf_source.reset();
  fe->buffer.clear();
  for (auto* f : fe->pool) rgbid_frame_destroy(fe->ctx, f);
  rgbid_frame_destroy(fe->ctx, fe->kf);
  cudaFree(fe->kf_C);
  cudaFree(fe->counts_dev);
  cudaFreeHost(fe->counts_host);
  delete fe;
  return RGBID_OK;
}

// Pipeline::process_frame — src/pipeline.cpp:120-138
int rgbid_frontend_process(rgbid_frontend* fe, const double* I, const double* W, double t,
                           rgbid_frame_estimate* est) {
  if (!fe || !W) return RGBID_E_ARG;
  rgbid_frame* f = nullptr;
  int rc = RGBID_OK;
  if (!fe->pool.empty()) {  // a recycled device frame: no allocation in steady state
    f = fe->pool.back();
    fe->pool.pop_back();
  } else {
    rc = rgbid_frame_create(fe->ctx, fe->w, fe->h, &f);
    if (rc) return rc;
  }
  FramePtr frame(new FrameRef{&fe->pool, f});
  rc = rt_frame_upload_async(fe->ctx, f, I, W);  // stream-ordered before the align
  if (rc) return rc;
  if (!fe->has_prev) {  // bootstrap: the first frame anchors the world frame
    fe->reference = frame;
    fe->T_W_ref = identity();
    fe->T_ref_prev = identity();
    fe->cov_ref_prev = zero6();
    fe->has_prev = true;
    rgbid_frame_estimate e;
    std::memset(&e, 0, sizeof(e));
    e.timestamp = t;
    pose_to(identity(), e.T_W_k.R, e.T_W_k.t);
    e.keyframe_id = 0;
    fe->traj.push_back(e);
    fe->keyframe_frame_index.push_back(0);
    rc = start_keyframe(fe, frame, t);
  } else {
    bool check_ref = false;
    PoseD T_W_k;
    rc = track(fe, frame, t, &check_ref, &T_W_k);
    if (!rc) rc = fuse_enqueue(fe, frame, t);
    if (!rc) rc = finish_frame(fe, frame, t, check_ref, T_W_k);
  }
  if (rc) return rc;
  if (est) *est = fe->traj.back();
  return RGBID_OK;
}

int rgbid_frontend_finish(rgbid_frontend* fe) {
  if (!fe) return RGBID_E_ARG;
  const int rc = emit_keyframe(fe);
  if (rc) return rc;
  return rgbid_ctx_synchronize(fe->ctx);
}

int rgbid_frontend_trajectory(rgbid_frontend* fe, rgbid_frame_estimate* out, int max, int* n) {
  if (!fe || !n) return RGBID_E_ARG;
  const int m = std::min<int>(max, (int)fe->traj.size());
  if (out && m > 0) std::memcpy(out, fe->traj.data(), sizeof(rgbid_frame_estimate) * m);
  *n = (int)fe->traj.size();
  return RGBID_OK;
}

int rgbid_frontend_keyframes(rgbid_frontend* fe, int* out_index, int max, int* n) {
  if (!fe || !n) return RGBID_E_ARG;
  const int m = std::min<int>(max, (int)fe->keyframe_frame_index.size());
  if (out_index && m > 0) std::memcpy(out_index, fe->keyframe_frame_index.data(), sizeof(int) * m);
  *n = (int)fe->keyframe_frame_index.size();
  return RGBID_OK;
}

int rgbid_frontend_current_keyframe(rgbid_frontend* fe, double* W, double* C, rgbid_pose* T_W_kf,
                                    int* id) {
  if (!fe || !fe->has_kf) return RGBID_E_ARG;
  int rc = rgbid_frame_download(fe->ctx, fe->kf, nullptr, W);
  if (rc) return rc;
  if (C && cudaMemcpy(C, fe->kf_C, sizeof(double) * fe->w * fe->h, cudaMemcpyDeviceToHost) !=
               cudaSuccess)
    return RGBID_E_CUDA;
  if (T_W_kf) pose_to(fe->T_W_kf, T_W_kf->R, T_W_kf->t);
  if (id) *id = fe->kf_id;
  return RGBID_OK;
}

}  // extern "C"
