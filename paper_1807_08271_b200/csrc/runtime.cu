// Host runtime of librgbid_b200.so: contexts, device frames, the on-device
// alignment driver and every C-ABI entry point of include/rgbid_b200.h.
//
// The level/iteration loop of align (src/alignment.cpp:372-404) is issued as a
// fixed sequence of kernel launches on the ctx stream; convergence breaks and
// degenerate throws are per-slot flags evaluated on the device (SlotState), so
// the host never waits inside an alignment.  The launch sequence of a given
// (batch size, levels, iterations) is captured once into a CUDA graph and
// replayed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rgbid_b200.h"
#include "align_kernels.cuh"
#include "fusion_kernels.cuh"
#include "map_kernels.cuh"
#include "runtime_internal.cuh"

using namespace rgbid_b200;

struct rgbid_frame {
  int w = 0, h = 0;
  double* I = nullptr;  // level 0
  double* W = nullptr;
  double* pyr = nullptr;  // levels 1..kMaxLevels-1, I and W interleaved per level
  double* pI[kMaxLevels] = {};
  double* pW[kMaxLevels] = {};
  int pyr_levels = 0;  // levels currently valid (0 = none built)
  int pyr_lane = -1;   // lane whose chunk (sequence pyr_seq) builds/built the pyramid
  unsigned long long pyr_seq = 0;
};

namespace {

struct CachedGraph {
  cudaGraphExec_t exec = nullptr;
  long long launches = 0;  // kernel launches per replay
};

}  // namespace

// One execution lane of the alignment driver: a stream, a slot workspace and the
// CUDA graphs captured on it.  Batches alternate chunks over the lanes (chunk
// c+1's uploads / setup overlap chunk c's kernels; co-scheduled chunk pairs fill
// each other's tails, ~1%).
struct Lane {
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;
  cudaEvent_t ready = nullptr;  // slot records uploaded (pair launches wait on it)
  int cap_slots = 0, cap_w = 0, cap_h = 0;
  double* ws_f64 = nullptr;
  int* ws_i32 = nullptr;
  uint8_t* ws_u8 = nullptr;
  SlotIO* d_io = nullptr;
  SlotState* d_st = nullptr;
  int* d_act = nullptr;  // active-slot list [1 + slots] (k_active_slots)
  std::vector<SlotIO> h_io;
  SlotState* h_st_pinned = nullptr;
  std::map<std::string, CachedGraph> graphs;
  // chunk in flight
  int pend_n = 0;
  rgbid_align_result* pend_results = nullptr;
  int pend_levels = 0;
  bool pend_trace = false;
  unsigned long long pend_call = 0;  // host batch call that queued the pending chunk
  unsigned long long seq = 0;        // chunks enqueued on this lane
};
#ifndef RGBID_LANES
#define RGBID_LANES 2
#endif
constexpr int kLanes = RGBID_LANES;  // chunks co-scheduled per group (stage offsets 0..kLanes-1)

struct rgbid_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;  // == lanes[0].stream
  std::string err;
  long long launches = 0;
  Lane lanes[kLanes];
  rgbid_iter_trace* d_trace = nullptr;
  std::vector<rgbid_iter_trace> last_trace;
  bool use_graphs = true;
  bool graph_switch = true;  // K1 / K3 slot rows chosen by graph switch nodes
  std::vector<cudaEvent_t> pair_events;  // stage events of co-scheduled chunk pairs
  // scratch device buffers for the one-shot host APIs
  std::map<std::string, std::pair<void*, size_t>> scratch;
  rgbid_frame* tmpA = nullptr;
  rgbid_frame* tmpB = nullptr;
  // device frames reused by rgbid_align_batch_host across calls ([lane][slot] A/B)
  std::vector<rgbid_frame*> host_fa[kLanes], host_fb[kLanes];
  // profiling (per-kernel CUDA-event times) and host<->device byte counters
  Profiler prof;
  std::map<std::string, std::pair<long long, double>> kstats;  // name -> (launches, ms)
  long long h2d_bytes = 0, d2h_bytes = 0;
  unsigned long long host_call = 0;  // rgbid_align_batch_host(_async) calls so far
};

namespace {

// Reads back the per-kernel events recorded while profiling (after a sync).
void flush_profile(rgbid_ctx* ctx) {
  for (auto& r : ctx->prof.pending) {
    float ms = 0.f;
    if (cudaEventSynchronize(r.stop) == cudaSuccess && cudaEventElapsedTime(&ms, r.start, r.stop) == cudaSuccess) {
      auto& e = ctx->kstats[r.name];
      e.first += 1;
      e.second += ms;
    }
    ctx->prof.pool.push_back(r.start);
    ctx->prof.pool.push_back(r.stop);
  }
  ctx->prof.pending.clear();
}

struct LaunchScope {  // routes launch accounting / profiling to this ctx
  explicit LaunchScope(rgbid_ctx* c) : ctx(c) {
    g_launch_counter = &c->launches;
    g_profiler = &c->prof;
  }
  ~LaunchScope() {
    if (!ctx->prof.pending.empty()) flush_profile(ctx);
    g_launch_counter = nullptr;
    g_profiler = nullptr;
  }
  rgbid_ctx* ctx;
};

// host<->device copies on the ctx stream, counted for the e2e byte report
#define H2D(dst, src, bytes)                                                              \
  do {                                                                                    \
    CK(cudaMemcpyAsync((dst), (src), (bytes), cudaMemcpyHostToDevice, ctx->stream)); \
    ctx->h2d_bytes += (long long)(bytes);                                                 \
  } while (0)
#define H2DS(st, dst, src, bytes)                                                         \
  do {                                                                                    \
    CK(cudaMemcpyAsync((dst), (src), (bytes), cudaMemcpyHostToDevice, (st)));             \
    ctx->h2d_bytes += (long long)(bytes);                                                 \
  } while (0)
#define D2HS(st, dst, src, bytes)                                                         \
  do {                                                                                    \
    CK(cudaMemcpyAsync((dst), (src), (bytes), cudaMemcpyDeviceToHost, (st)));             \
    ctx->d2h_bytes += (long long)(bytes);                                                 \
  } while (0)
#define D2H(dst, src, bytes)                                                              \
  do {                                                                                    \
    CK(cudaMemcpyAsync((dst), (src), (bytes), cudaMemcpyDeviceToHost, ctx->stream)); \
    ctx->d2h_bytes += (long long)(bytes);                                                 \
  } while (0)

#define CK(expr)                                                        \
  do {                                                                  \
    cudaError_t e_ = (expr);                                            \
    if (e_ != cudaSuccess) {                                            \
      ctx->err = std::string(#expr) + ": " + cudaGetErrorString(e_);    \
      return e_ == cudaErrorMemoryAllocation ? RGBID_E_OOM : RGBID_E_CUDA; \
    }                                                                   \
  } while (0)

int check_launch(rgbid_ctx* ctx) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    ctx->err = std::string("kernel launch: ") + cudaGetErrorString(e);
    return RGBID_E_CUDA;
  }
  return RGBID_OK;
}

template <typename T>
int scratch_buf(rgbid_ctx* ctx, const char* name, size_t count, T** out) {
  auto& e = ctx->scratch[name];
  const size_t bytes = count * sizeof(T);
  if (e.second < bytes) {
    if (e.first) cudaFree(e.first);
    e.first = nullptr;
    e.second = 0;
    CK(cudaMalloc(&e.first, bytes));
    e.second = bytes;
  }
  *out = static_cast<T*>(e.first);
  return RGBID_OK;
}

rgbid_align_config default_config() {
  rgbid_align_config c;
  std::memset(&c, 0, sizeof(c));
  c.levels = 3;
  c.n_iterations = 3;
  c.iterations[0] = 10;
  c.iterations[1] = 5;
  c.iterations[2] = 4;
  c.convergence_eps = 1e-6;
  c.lambda_n_min = 0.1;
  c.bilateral_sigma_space = 2.0;
  c.bilateral_sigma_intensity = 0.05;
  c.bilateral_sigma_depth = 0.02;
  return c;
}

int level_iters(const rgbid_align_config& c, int level) {
  return level < c.n_iterations ? c.iterations[level] : 5;  // src/alignment.cpp:373-374
}

// build_pyramid intrinsics — src/alignment.cpp:18-25
void level_intrinsics(const rgbid_intrinsics& K0, int level, rgbid_intrinsics* out) {
  rgbid_intrinsics k = K0;
  for (int l = 0; l < level; ++l) {
    k.fx /= 2.0;
    k.fy /= 2.0;
    k.cx = (k.cx - 0.5) / 2.0;
    k.cy = (k.cy - 0.5) / 2.0;
    k.width /= 2;
    k.height /= 2;
  }
  *out = k;
}

LevelInfo make_level(const rgbid_intrinsics& K0, int w0, int h0, int level) {
  LevelInfo li;
  std::memset(&li, 0, sizeof(li));
  li.level = level;
  li.w = w0 >> level;
  li.h = h0 >> level;
  li.tx = k1_tx(level);
  li.nseg = (li.w + li.tx - 1) / li.tx;
  li.ntiles = li.nseg * li.h;
  li.ntiles3 = k3_tiles(li.w, li.h);
  li.pix3 = kPixK3;
  li.bx1 = w0 - 1.0;
  li.by1 = h0 - 1.0;
  rgbid_intrinsics k;
  level_intrinsics(K0, level, &k);
  li.fx = k.fx;
  li.fy = k.fy;
  li.cx = k.cx;
  li.cy = k.cy;
  const M3 Ki = m3_inv(K_mat(k.fx, k.fy, k.cx, k.cy));
  for (int i = 0; i < 9; ++i) li.Kinv[i] = Ki.m[i / 3][i % 3];
  return li;
}

PoseD pose_of(const rgbid_pose* p) {
  if (!p) {
    PoseD I;
    std::memset(&I, 0, sizeof(I));
    I.R.m[0][0] = I.R.m[1][1] = I.R.m[2][2] = 1.0;
    return I;
  }
  return pose_from(p->R, p->t);
}

// Per-slot workspace: ibw ({r_I, w_b} pairs, 2N doubles), fIA, fWA (N each), the
// A-side gradients (all levels), K3 partials, the K2 samples (2 x kMaxSample) and
// frame B interleaved (2N); A-side masks; per-tile counts + validity bitmasks.
size_t max_tiles(int w, int h) {
  size_t mx = 0;
  for (int l = 0; l < kMaxLevels; ++l) {
    if ((w >> l) < 1 || (h >> l) < 1) break;
    const int tx = k1_tx(l);
    mx = std::max(mx, (size_t)(((w >> l) + tx - 1) / tx) * (size_t)(h >> l));
  }
  return mx;
}
size_t pyr_pixels(int w, int h) {
  size_t t = 0;
  for (int l = 0; l < kMaxLevels; ++l) t += (size_t)(w >> l) * (h >> l);
  return t;
}
size_t slot_f64(int w, int h) {
  const size_t N = (size_t)w * h;
  const size_t part = (size_t)k3_tiles(w, h, 1) * kNPart;  // latency mode: 1 pixel per thread
  // ... + K2 samples + interleaved frame B (16-byte aligned: the total stays even)
  const size_t f = 4 * N + 4 * pyr_pixels(w, h) + part + 2 * (size_t)kMaxSample;
  return ((f + 1) & ~(size_t)1) + 2 * N;
}
size_t slot_u8(int w, int h) { return (pyr_pixels(w, h) + 255) & ~(size_t)255; }
size_t slot_i32(int w, int h) { return 2 * max_tiles(w, h) * (1 + kWordsPerTile) + 2; }

void free_lane_ws(Lane& L) {
  if (L.ws_f64) cudaFree(L.ws_f64);
  if (L.ws_i32) cudaFree(L.ws_i32);
  if (L.ws_u8) cudaFree(L.ws_u8);
  if (L.d_io) cudaFree(L.d_io);
  if (L.d_st) cudaFree(L.d_st);
  if (L.d_act) cudaFree(L.d_act);
  if (L.h_st_pinned) cudaFreeHost(L.h_st_pinned);
  L.ws_f64 = nullptr;
  L.ws_i32 = nullptr;
  L.ws_u8 = nullptr;
  L.d_io = nullptr;
  L.d_st = nullptr;
  L.d_act = nullptr;
  L.h_st_pinned = nullptr;
  L.cap_slots = 0;
}

// Cached graphs bake in the AlignLaunch of every lane they co-schedule (a chunk
// pair cached on lane 0 holds lane 1's d_io / d_st), so any lane's reallocation
// invalidates the graphs of all lanes.
void drop_graphs(rgbid_ctx* ctx) {
  for (auto& L : ctx->lanes) {
    for (auto& g : L.graphs) cudaGraphExecDestroy(g.second.exec);
    L.graphs.clear();
  }
}

int ensure_workspace(rgbid_ctx* ctx, Lane& L, int nslots, int w, int h) {
  if (nslots <= L.cap_slots && w == L.cap_w && h == L.cap_h) return RGBID_OK;
  // same resolution: grow to the lane's peak slot count (no shrink thrash);
  // a new resolution is sized for this call only (a 2048-pair VGA batch followed
  // by one 1280x960 pair must not allocate 1024 x 114 MB)
  if (w == L.cap_w && h == L.cap_h) nslots = std::max(nslots, L.cap_slots);
  drop_graphs(ctx);
  free_lane_ws(L);
  CK(cudaMalloc(&L.ws_f64, sizeof(double) * slot_f64(w, h) * nslots));
  CK(cudaMalloc(&L.ws_i32, sizeof(int) * slot_i32(w, h) * nslots));
  CK(cudaMalloc(&L.ws_u8, slot_u8(w, h) * nslots));
  CK(cudaMalloc(&L.d_io, sizeof(SlotIO) * nslots));
  CK(cudaMalloc(&L.d_st, sizeof(SlotState) * nslots));
  CK(cudaMalloc(&L.d_act, sizeof(int) * (nslots + 1)));
  CK(cudaMallocHost(&L.h_st_pinned, sizeof(SlotState) * nslots));
  if (!ctx->d_trace) CK(cudaMalloc(&ctx->d_trace, sizeof(rgbid_iter_trace) * kTraceMax));
  L.cap_slots = nslots;
  L.cap_w = w;
  L.cap_h = h;
  L.h_io.resize(nslots);
  return RGBID_OK;
}

int frame_alloc_pyramid(rgbid_ctx* ctx, rgbid_frame* f) {
  if (!f->pyr) {
    size_t tot = 0;
    for (int l = 1; l < kMaxLevels; ++l) tot += 2 * (size_t)(f->w >> l) * (f->h >> l);
    if (tot == 0) tot = 1;
    CK(cudaMalloc(&f->pyr, sizeof(double) * tot));
    size_t off = 0;
    for (int l = 1; l < kMaxLevels; ++l) {
      const size_t n = (size_t)(f->w >> l) * (f->h >> l);
      f->pI[l] = f->pyr + off;
      f->pW[l] = f->pyr + off + n;
      off += 2 * n;
    }
  }
  f->pI[0] = f->I;
  f->pW[0] = f->W;
  return RGBID_OK;
}

int frame_ensure_pyramid(rgbid_ctx* ctx, rgbid_frame* f, int levels) {
  if (f->pyr_levels >= levels) return RGBID_OK;
  const int rc = frame_alloc_pyramid(ctx, f);
  if (rc) return rc;
  for (int l = std::max(1, f->pyr_levels); l < levels; ++l)
    launch_downsample2(f->pI[l - 1], f->pW[l - 1], f->w >> (l - 1), f->h >> (l - 1), f->pI[l],
                       f->pW[l], ctx->stream);
  f->pyr_levels = levels;
  return check_launch(ctx);
}

// Host Jacobi eigenvalues (spectrum payload of DegenerateAlignmentError only).
void spectrum_of(const double H[36], long long n_jets, double out[6]) {
  if (n_jets < 6) {
    for (int i = 0; i < 6; ++i) out[i] = 0.0;
    return;
  }
  bool bad = false;
  for (int i = 0; i < 6; ++i)
    if (H[i * 6 + i] <= 0.0) bad = true;
  if (bad) {
    for (int i = 0; i < 6; ++i) out[i] = H[i * 6 + i];
    return;
  }
  double s[6], a[6][6];
  for (int i = 0; i < 6; ++i) s[i] = 1.0 / std::sqrt(H[i * 6 + i]);
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) a[i][j] = (s[i] * H[i * 6 + j]) * s[j];
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < 6; ++i)
      for (int j = i + 1; j < 6; ++j) off += a[i][j] * a[i][j];
    if (off == 0.0) break;
    for (int p = 0; p < 6; ++p)
      for (int q = p + 1; q < 6; ++q) {
        if (a[p][q] == 0.0) continue;
        const double th = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), sn = t * c;
        for (int k = 0; k < 6; ++k) {
          const double kp = a[k][p], kq = a[k][q];
          a[k][p] = c * kp - sn * kq;
          a[k][q] = sn * kp + c * kq;
        }
        for (int k = 0; k < 6; ++k) {
          const double pk = a[p][k], qk = a[q][k];
          a[p][k] = c * pk - sn * qk;
          a[q][k] = sn * pk + c * qk;
        }
      }
  }
  for (int i = 0; i < 6; ++i) out[i] = a[i][i];
  std::sort(out, out + 6);
}

int validate_cfg(const rgbid_align_config& c, int w, int h) {
  if (c.levels < 1 || c.levels > kMaxLevels) return RGBID_E_ARG;
  if (c.n_iterations < 0 || c.n_iterations > RGBID_MAX_LEVELS) return RGBID_E_ARG;
  if ((w >> (c.levels - 1)) < 1 || (h >> (c.levels - 1)) < 1) return RGBID_E_ARG;
  return RGBID_OK;
}

// Graph switch nodes for the slot-row count of K1 / K3 (k_active_slots picks the
// body per iteration on the device).  Outside a stream capture (direct launches,
// profiling) the kernels run one row per slot with their own slot check.
thread_local bool g_switch_capture_failed = false;  // a switch body could not be captured

int switch_bodies(int nslots) {  // bodies k = 0.. with ceil(nslots / 2^k) >= 8 rows
  int nb = 1;
  while (nb < 8 && ((nslots + (1 << nb) - 1) >> nb) >= 8) ++nb;
  return nb;
}

void switch_begin(cudaStream_t s, const AlignLaunch& a, SlotSwitch& sw) {
  sw = SlotSwitch{};
  if (!a.act || !a.graph_switch) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaGraph_t g = nullptr;
  if (cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, nullptr, nullptr) != cudaSuccess ||
      cs != cudaStreamCaptureStatusActive)
    return;
  for (auto& h : sw.h)  // default body 0 (the full grid)
    if (cudaGraphConditionalHandleCreate(&h, g, 0u, cudaGraphCondAssignDefault) != cudaSuccess)
      return;
  sw.nbodies = switch_bodies(a.nslots);
}

// launch(stream, rows) as switch node `idx` of sw in the capture on s, one body per
// row count (rows = 0: one row per slot, no list); a plain launch over all slots
// when not capturing
void launch_switched(cudaStream_t s, const AlignLaunch& a, const SlotSwitch& sw, int idx,
                     const std::function<void(cudaStream_t, int)>& launch) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  if (sw.nbodies == 0 || cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &nd) != cudaSuccess ||
      cs != cudaStreamCaptureStatusActive) {
    launch(s, 0);
    return;
  }
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = sw.h[idx];
  cp.conditional.type = cudaGraphCondTypeSwitch;
  cp.conditional.size = (unsigned)sw.nbodies;
  cudaGraphNode_t node;
  std::vector<cudaGraphNode_t> dv(deps, deps + nd);
  if (cudaGraphAddNode(&node, g, dv.empty() ? nullptr : dv.data(), dv.size(), &cp) != cudaSuccess) {
    launch(s, 0);
    return;
  }
  static thread_local std::map<int, cudaStream_t> scratch;  // body captures, per device
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStream_t& t = scratch[dev];
  if (!t) cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking);
  long long* cnt = g_launch_counter;
  const long long c0 = cnt ? *cnt : 0;
  for (int k = 0; k < sw.nbodies; ++k) {
    if (!t || cudaStreamBeginCaptureToGraph(t, cp.conditional.phGraph_out[k], nullptr, nullptr, 0,
                                            cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      g_switch_capture_failed = true;  // never launch a body for real: fail the graph
      continue;
    }
    launch(t, k == 0 ? 0 : (a.nslots + (1 << k) - 1) >> k);  // body 0: every slot, no list
    cudaGraph_t body;
    if (cudaStreamEndCapture(t, &body) != cudaSuccess) g_switch_capture_failed = true;
  }
  if (cnt) *cnt = c0 + 1;  // one body runs per graph launch
  if (cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies) !=
      cudaSuccess)
    g_switch_capture_failed = true;
}

// The whole align (all levels + covariance pass) as a list of stages; a stage
// is one or more dependent kernel launches on one stream.  Stages cycle
// K1 | K2 | K3+K4 per IRLS iteration so that two chunks offset by one stage
// pair the FP64-bound Student-t kernel with a memory-bound kernel.
using Stage = std::function<void(cudaStream_t)>;

// Schedule of co-scheduled chunk pairs (RGBID_PAIR_STAGES / RGBID_PAIR_OFFSET override):
// stages per IRLS iteration (3: K1 | K2 | K3+K4, or 4: K1 | K2a | K2b | K3+K4) and the
// stage offset D of the second chunk (its stage s runs beside the first chunk's s+D).
int g_pair_stages = 4, g_pair_offset = 2;  // 4 stages, offset 2: +0.8% over 3 / 1 (A/B on the B200)

// The whole align (all levels + covariance pass) as a list of stages; a stage
// is one or more dependent kernel launches on one stream.  Stages cycle over
// the IRLS iteration's kernels so that two chunks offset by D stages pair the
// FP64-bound Student-t kernel with a memory/latency-bound one.
std::vector<Stage> align_stages(const AlignLaunch& a, const rgbid_intrinsics& K,
                                const rgbid_align_config& cfg) {
  std::vector<Stage> st;
  // latency mode (<= kTdistClusterMaxSlots slots): K3 with one pixel per thread
  auto level = [&](int l) {
    LevelInfo li = make_level(K, a.w0, a.h0, l);
    if (a.nslots <= kTdistClusterMaxSlots) {
      li.pix3 = 1;
      li.ntiles3 = k3_tiles(li.w, li.h, 1);
    }
    return li;
  };
  const LevelInfo li0 = level(0);
  const int levels = cfg.levels;
  const bool split = g_pair_stages == 4;
  st.push_back([a, levels](cudaStream_t s) {
    launch_pyramid_slots(a, levels, s);  // build_pyramid (src/alignment.cpp:369)
    launch_amask(a, levels, 0, s);       // A-side validity + gradients, once per align
    launch_interleave_B(a, s);           // B as {I, W} pairs for K1's bilinear taps
  });
  for (int lv = cfg.levels - 1; lv >= 0; --lv) {
    const LevelInfo li = level(lv);
    const int iters = level_iters(cfg, lv);
    for (int it = 0; it < iters; ++it) {
      // the slots this iteration still works on, and the K1 / K3 grids that cover them
      auto sw = std::make_shared<SlotSwitch>();
      st.push_back([a, li, sw](cudaStream_t s) {
        switch_begin(s, a, *sw);
        launch_active_slots(a, li.level, 0, s, sw.get());
        launch_switched(s, a, *sw, 0, [a, li](cudaStream_t t, int rows) {
          launch_warp_residuals(a, li, 0, t, rows);
        });
      });
      if (split) {
        st.push_back([a, li](cudaStream_t s) { launch_tdist(a, li, 0, s, 1); });
        st.push_back([a, li](cudaStream_t s) { launch_tdist(a, li, 0, s, 2); });
      } else {
        st.push_back([a, li](cudaStream_t s) { launch_tdist(a, li, 0, s); });
      }
      st.push_back([a, li, li0, sw](cudaStream_t s) {
        launch_switched(s, a, *sw, 1, [a, li](cudaStream_t t, int rows) {
          launch_normal_equations(a, li, 0, t, rows);
        });
        launch_solve(a, li, li0, s);
      });
    }
  }
  // filtered_hessian_covariance — src/alignment.cpp:406-407, 411-436
  const double ss = cfg.bilateral_sigma_space, si = cfg.bilateral_sigma_intensity,
               sd = cfg.bilateral_sigma_depth;
  st.push_back([a, li0, ss, si, sd](cudaStream_t s) {
    launch_bilateral_pair(a, ss, si, sd, s);
    launch_amask(a, 1, 1, s);
    launch_warp_residuals(a, li0, 1, s);
  });
  st.push_back([a, li0](cudaStream_t s) { launch_tdist(a, li0, 1, s); });
  st.push_back([a, li0](cudaStream_t s) {
    launch_normal_equations(a, li0, 1, s);
    launch_covariance(a, li0, s);
  });
  return st;
}

void enqueue_align(cudaStream_t stream, const AlignLaunch& a, const rgbid_intrinsics& K,
                   const rgbid_align_config& cfg) {
  for (auto& f : align_stages(a, K, cfg)) f(stream);
}

// G chunks in one launch sequence: stage s of chunk j after stage s of chunk j-1,
// stage s+G of chunk 0 after stage s of chunk G-1 -> chunks run one stage apart
// (G = 2: the pairs {A_{s+1}, B_s} run concurrently).
void enqueue_align_group(const std::vector<cudaStream_t>& sj, const std::vector<AlignLaunch>& aj,
                         const rgbid_intrinsics& K, const rgbid_align_config& cfg,
                         std::vector<cudaEvent_t>& ev) {
  const int G = (int)sj.size();
  std::vector<std::vector<Stage>> S;
  for (int j = 0; j < G; ++j) S.push_back(align_stages(aj[j], K, cfg));
  const size_t n = S[0].size();
  while (ev.size() < G * n + 1) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    ev.push_back(e);
  }
  cudaEventRecord(ev[G * n], sj[0]);  // fork off chunk 0's stream (capture origin)
  for (int j = 1; j < G; ++j) cudaStreamWaitEvent(sj[j], ev[G * n], 0);
  for (size_t i = 0; i < n; ++i)
    for (int j = 0; j < G; ++j) {
      if (j == 0 && i >= (size_t)G) cudaStreamWaitEvent(sj[0], ev[(G - 1) * n + i - G], 0);
      if (j > 0) cudaStreamWaitEvent(sj[j], ev[(j - 1) * n + i], 0);
      S[j][i](sj[j]);
      cudaEventRecord(ev[j * n + i], sj[j]);
    }
  cudaStreamWaitEvent(sj[0], ev[(G - 1) * n + n - 1], 0);  // join
}

// Two chunks in one launch sequence, B lagging D stages behind A: B's stage i
// waits for A's stage i + D - 1, A's stage j for B's stage j - D - 1, so A's stage
// i + D runs beside B's stage i.
void enqueue_align_pair(cudaStream_t sA, cudaStream_t sB, const AlignLaunch& a,
                        const AlignLaunch& b, const rgbid_intrinsics& K,
                        const rgbid_align_config& cfg, std::vector<cudaEvent_t>& ev) {
  const std::vector<Stage> A = align_stages(a, K, cfg), B = align_stages(b, K, cfg);
  const int n = (int)A.size(), D = std::max(1, g_pair_offset);
  while ((int)ev.size() < 2 * n + 1) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    ev.push_back(e);
  }
  cudaEventRecord(ev[2 * n], sA);  // fork B off A's stream (capture origin)
  cudaStreamWaitEvent(sB, ev[2 * n], 0);
  for (int t = 0; t < n + D - 1; ++t) {
    if (t < n) {
      if (t - D - 1 >= 0) cudaStreamWaitEvent(sA, ev[n + t - D - 1], 0);
      A[t](sA);
      cudaEventRecord(ev[t], sA);
    }
    const int i = t - (D - 1);
    if (i >= 0 && i < n) {
      cudaStreamWaitEvent(sB, ev[std::min(i + D - 1, n - 1)], 0);
      B[i](sB);
      cudaEventRecord(ev[n + i], sB);
    }
  }
  cudaStreamWaitEvent(sA, ev[2 * n - 1], 0);  // join
}

// Unpacks the SlotState records of a lane's finished chunk into results.
int finish_chunk(rgbid_ctx* ctx, Lane& L) {
  if (L.pend_n == 0) return RGBID_OK;
  CK(cudaEventSynchronize(L.done));
  if (L.pend_trace) {
    ctx->last_trace.resize(kTraceMax);
    CK(cudaMemcpy(ctx->last_trace.data(), ctx->d_trace, sizeof(rgbid_iter_trace) * kTraceMax,
                  cudaMemcpyDeviceToHost));
    ctx->last_trace.resize(std::min(L.h_st_pinned[0].trace_n, kTraceMax));
  }
  for (int i = 0; i < L.pend_n; ++i) {
    const SlotState& s = L.h_st_pinned[i];
    rgbid_align_result& r = L.pend_results[i];
    std::memset(&r, 0, sizeof(r));
    r.status = s.status;
    if (s.status == RGBID_E_DEGENERATE) {
      spectrum_of(s.H, s.nI, r.spectrum);
      continue;
    }
    std::memcpy(r.T_AB.R, s.R, sizeof(s.R));
    std::memcpy(r.T_AB.t, s.t, sizeof(s.t));
    std::memcpy(r.cov, s.cov, sizeof(s.cov));
    r.converged = 1;
    r.cov_degenerate = s.cov_degenerate;
    r.n_levels = L.pend_levels;
    for (int k = 0; k < L.pend_levels; ++k) {
      const int level = L.pend_levels - 1 - k;
      r.level_log[k].level = level;
      r.level_log[k].iterations = s.iters[level];
      r.level_log[k].final_cost = s.cost[level];
    }
    r.tdist_intensity = s.finI;
    r.tdist_depth = s.finW;
    r.total_iterations = s.total_iters;
  }
  L.pend_n = 0;
  return RGBID_OK;
}

// Completes every lane's pending chunk (results written to the caller's arrays).
int finish_all(rgbid_ctx* ctx) {
  for (auto& L : ctx->lanes) {
    const int rc = finish_chunk(ctx, L);
    if (rc) return rc;
  }
  return RGBID_OK;
}

// Enqueues n alignments (one chunk) on lane L: slot setup, H2D of the slot
// records, the (cached) CUDA graph of the whole align, D2H of the results.
int prepare_chunk(rgbid_ctx* ctx, Lane& L, int n, const rgbid_frame* const* fa,
                  const rgbid_frame* const* fb, const rgbid_intrinsics& K,
                  const rgbid_pose* inits, const rgbid_align_config& cfg, bool want_trace,
                  AlignLaunch* out_a) {
  int rc = finish_chunk(ctx, L);  // the lane's previous chunk owns h_st_pinned
  if (rc) return rc;
  const int w = fa[0]->w, h = fa[0]->h;
  rc = ensure_workspace(ctx, L, n, w, h);
  if (rc) return rc;
  for (int i = 0; i < n; ++i) {
    rc = frame_alloc_pyramid(ctx, const_cast<rgbid_frame*>(fa[i]));
    if (rc) return rc;
  }
  const size_t N = (size_t)w * h;
  const size_t sf = slot_f64(w, h), si = slot_i32(w, h), su = slot_u8(w, h);
  const size_t mt = max_tiles(w, h);
  const LevelInfo li0 = make_level(K, w, h, 0);
  const int nslots = n;
  for (int i = 0; i < nslots; ++i) {
    SlotIO& o = L.h_io[i];
    std::memset(&o, 0, sizeof(o));
    for (int l = 0; l < kMaxLevels; ++l) {
      o.IA[l] = fa[i]->pI[l];
      o.WA[l] = fa[i]->pW[l];
    }
    o.IA[0] = fa[i]->I;
    o.WA[0] = fa[i]->W;
    o.IB = fb[i]->I;
    o.WB = fb[i]->W;
    double* base = L.ws_f64 + sf * i;
    o.ibw = reinterpret_cast<double2*>(base);  // 2N doubles, 16-B aligned
    o.fIA = base + 2 * N;
    o.fWA = base + 3 * N;
    double* g = base + 4 * N;
    for (int l = 0; l < kMaxLevels; ++l) {
      o.agrad[l] = g;
      g += 4 * (size_t)(w >> l) * (h >> l);
    }
    o.part = g;
    o.IWB = reinterpret_cast<double2*>(base + (sf - 2 * N));  // sf and N*2 even: 16-B aligned
    o.smp = base + (sf - 2 * N - 2 * (size_t)kMaxSample);
    int* ib32 = L.ws_i32 + si * i;
    o.cntI = ib32;
    o.cntW = ib32 + mt;
    o.bitsI = reinterpret_cast<unsigned*>(ib32 + 2 * mt);
    o.bitsW = o.bitsI + mt * kWordsPerTile;
    o.nsmp = ib32 + 2 * mt * (1 + kWordsPerTile);
    uint8_t* u8 = L.ws_u8 + su * i;
    for (int l = 0; l < kMaxLevels; ++l) {
      o.amask[l] = u8;
      u8 += (size_t)(w >> l) * (h >> l);
    }
    // build frame A's pyramid in-graph unless cached (once per distinct frame)
    o.build_pyr = 0;
    if (fa[i]->pyr_levels < cfg.levels) {
      bool first = true;
      for (int j = 0; j < i; ++j)
        if (fa[j] == fa[i]) first = false;
      o.build_pyr = first ? 1 : 0;
    }
    SlotState& s = L.h_st_pinned[i];
    std::memset(&s, 0, sizeof(s));
    const PoseD T = pose_of(inits ? &inits[i] : nullptr);
    pose_to(T, s.R, s.t);
    s.wm = warp_mats(T, li0.fx, li0.fy, li0.cx, li0.cy);
    s.status = RGBID_OK;
    s.done_level = -1;
  }
  // frames whose pyramid another lane's in-flight chunk builds: wait for it
  const int my = (int)(&L - ctx->lanes);
  bool wait[kLanes] = {};
  for (int i = 0; i < nslots; ++i) {
    const int k = fa[i]->pyr_lane;
    if (k >= 0 && k != my && ctx->lanes[k].pend_n > 0 && fa[i]->pyr_seq == ctx->lanes[k].seq)
      wait[k] = true;
  }
  for (int k = 0; k < kLanes; ++k)
    if (wait[k]) CK(cudaStreamWaitEvent(L.stream, ctx->lanes[k].done, 0));
  L.seq += 1;
  H2DS(L.stream, L.d_io, L.h_io.data(), sizeof(SlotIO) * nslots);
  H2DS(L.stream, L.d_st, L.h_st_pinned, sizeof(SlotState) * nslots);
  AlignLaunch a;
  a.io = L.d_io;
  a.st = L.d_st;
  a.trace = want_trace ? ctx->d_trace : nullptr;
  a.nslots = nslots;
  a.w0 = w;
  a.h0 = h;
  a.eps = cfg.convergence_eps;
  a.lambda_n_min = cfg.lambda_n_min;
  a.act = use_active_list(nslots) ? L.d_act : nullptr;
  a.graph_switch = ctx->graph_switch;

  *out_a = a;
  // remember what finish_chunk / the pyramid bookkeeping need
  for (int i = 0; i < nslots; ++i) {
    rgbid_frame* f = const_cast<rgbid_frame*>(fa[i]);
    if (L.h_io[i].build_pyr) {
      f->pyr_lane = my;
      f->pyr_seq = L.seq;
    }
    f->pyr_levels = std::max(f->pyr_levels, cfg.levels);
  }
  return RGBID_OK;
}

std::string graph_key(int nA, int nB, bool trace, int w, int h, const rgbid_intrinsics& K,
                      const rgbid_align_config& cfg) {
  struct {
    int nA, nB, trace, levels, w, h;
    int iters[kMaxLevels];
    double p[9];
  } kb;
  std::memset(&kb, 0, sizeof(kb));
  kb.nA = nA;
  kb.nB = nB;
  kb.trace = trace;
  kb.levels = cfg.levels;
  kb.w = w;
  kb.h = h;
  for (int l = 0; l < cfg.levels; ++l) kb.iters[l] = level_iters(cfg, l);
  const double p[9] = {cfg.convergence_eps, cfg.lambda_n_min, cfg.bilateral_sigma_space,
                       cfg.bilateral_sigma_intensity, cfg.bilateral_sigma_depth, K.fx, K.fy, K.cx,
                       K.cy};
  std::memcpy(kb.p, p, sizeof(p));
  return std::string(reinterpret_cast<const char*>(&kb), sizeof(kb));
}

// Launch (graph replay) + result D2H + completion event for one prepared chunk,
// or for two prepared chunks co-scheduled (LB != nullptr).
int launch_prepared(rgbid_ctx* ctx, Lane& L, const AlignLaunch& a, Lane* LB,
                    const AlignLaunch* b, const rgbid_intrinsics& K,
                    const rgbid_align_config& cfg, rgbid_align_result* resA,
                    rgbid_align_result* resB, bool want_trace) {
  const std::string key =
      graph_key(a.nslots, LB ? b->nslots : 0, want_trace, a.w0, a.h0, K, cfg);
  if (LB) {  // B's slot records were uploaded on its own stream
    CK(cudaEventRecord(LB->ready, LB->stream));
    CK(cudaStreamWaitEvent(L.stream, LB->ready, 0));
  }
  if (ctx->use_graphs && !ctx->prof.enabled) {
    auto it = L.graphs.find(key);
    if (it == L.graphs.end()) {
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(L.stream, cudaStreamCaptureModeThreadLocal));
      const long long before = ctx->launches;
      if (LB)
        enqueue_align_pair(L.stream, LB->stream, a, *b, K, cfg, ctx->pair_events);
      else
        enqueue_align(L.stream, a, K, cfg);
      CachedGraph cg;
      cg.launches = ctx->launches - before;
      ctx->launches = before;
      CK(cudaStreamEndCapture(L.stream, &g));
      if (g_switch_capture_failed) {
        g_switch_capture_failed = false;
        cudaGraphDestroy(g);
        ctx->err = "capture of a graph switch-node body failed";
        return RGBID_E_CUDA;
      }
      CK(cudaGraphInstantiateWithFlags(&cg.exec, g, cudaGraphInstantiateFlagUseNodePriority));
      cudaGraphDestroy(g);
      it = L.graphs.emplace(key, cg).first;
    }
    CK(cudaGraphLaunch(it->second.exec, L.stream));
    ctx->launches += it->second.launches;
  } else if (LB) {
    enqueue_align_pair(L.stream, LB->stream, a, *b, K, cfg, ctx->pair_events);
  } else {
    enqueue_align(L.stream, a, K, cfg);
  }
  int rc = check_launch(ctx);
  if (rc) return rc;
  D2HS(L.stream, L.h_st_pinned, L.d_st, sizeof(SlotState) * a.nslots);
  if (LB) D2HS(L.stream, LB->h_st_pinned, LB->d_st, sizeof(SlotState) * b->nslots);
  CK(cudaEventRecord(L.done, L.stream));
  L.pend_n = a.nslots;
  L.pend_results = resA;
  L.pend_levels = cfg.levels;
  L.pend_trace = want_trace;
  if (LB) {
    CK(cudaStreamWaitEvent(LB->stream, L.done, 0));
    CK(cudaEventRecord(LB->done, LB->stream));
    LB->pend_n = b->nslots;
    LB->pend_results = resB;
    LB->pend_levels = cfg.levels;
    LB->pend_trace = false;
  }
  return RGBID_OK;
}

// Launch (graph replay) of G prepared chunks co-scheduled on lanes 0..G-1, result
// D2H and completion events (launch_prepared generalised).
int launch_group(rgbid_ctx* ctx, int G, const AlignLaunch* aj, const rgbid_intrinsics& K,
                 const rgbid_align_config& cfg, rgbid_align_result* const* res, bool want_trace) {
  Lane& L = ctx->lanes[0];
  std::string key = graph_key(aj[0].nslots, aj[1].nslots, want_trace, aj[0].w0, aj[0].h0, K, cfg);
  for (int j = 2; j < G; ++j) key += std::to_string(aj[j].nslots) + ",";
  key += "G" + std::to_string(G);
  std::vector<cudaStream_t> sj;
  std::vector<AlignLaunch> av(aj, aj + G);
  for (int j = 0; j < G; ++j) sj.push_back(ctx->lanes[j].stream);
  for (int j = 1; j < G; ++j) {  // chunk j's slot records were uploaded on its own stream
    CK(cudaEventRecord(ctx->lanes[j].ready, ctx->lanes[j].stream));
    CK(cudaStreamWaitEvent(L.stream, ctx->lanes[j].ready, 0));
  }
  if (ctx->use_graphs && !ctx->prof.enabled) {
    auto it = L.graphs.find(key);
    if (it == L.graphs.end()) {
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(L.stream, cudaStreamCaptureModeThreadLocal));
      const long long before = ctx->launches;
      enqueue_align_group(sj, av, K, cfg, ctx->pair_events);
      CachedGraph cg;
      cg.launches = ctx->launches - before;
      ctx->launches = before;
      CK(cudaStreamEndCapture(L.stream, &g));
      if (g_switch_capture_failed) {
        g_switch_capture_failed = false;
        cudaGraphDestroy(g);
        ctx->err = "capture of a graph switch-node body failed";
        return RGBID_E_CUDA;
      }
      CK(cudaGraphInstantiateWithFlags(&cg.exec, g, cudaGraphInstantiateFlagUseNodePriority));
      cudaGraphDestroy(g);
      it = L.graphs.emplace(key, cg).first;
    }
    CK(cudaGraphLaunch(it->second.exec, L.stream));
    ctx->launches += it->second.launches;
  } else {
    enqueue_align_group(sj, av, K, cfg, ctx->pair_events);
  }
  int rc = check_launch(ctx);
  if (rc) return rc;
  for (int j = 0; j < G; ++j)
    D2HS(L.stream, ctx->lanes[j].h_st_pinned, ctx->lanes[j].d_st, sizeof(SlotState) * aj[j].nslots);
  CK(cudaEventRecord(L.done, L.stream));
  for (int j = 0; j < G; ++j) {
    Lane& Lj = ctx->lanes[j];
    if (j > 0) {
      CK(cudaStreamWaitEvent(Lj.stream, L.done, 0));
      CK(cudaEventRecord(Lj.done, Lj.stream));
    }
    Lj.pend_n = aj[j].nslots;
    Lj.pend_results = res[j];
    Lj.pend_levels = cfg.levels;
    Lj.pend_trace = j == 0 && want_trace;
  }
  return RGBID_OK;
}

int enqueue_chunk(rgbid_ctx* ctx, Lane& L, int n, const rgbid_frame* const* fa,
                  const rgbid_frame* const* fb, const rgbid_intrinsics& K,
                  const rgbid_pose* inits, const rgbid_align_config& cfg,
                  rgbid_align_result* results, bool want_trace) {
  AlignLaunch a;
  int rc = prepare_chunk(ctx, L, n, fa, fb, K, inits, cfg, want_trace, &a);
  if (rc) return rc;
  return launch_prepared(ctx, L, a, nullptr, nullptr, K, cfg, results, nullptr, want_trace);
}

// n alignments on one lane, synchronous (single align / small batches)
int run_align_slots(rgbid_ctx* ctx, int n, const rgbid_frame* const* fa,
                    const rgbid_frame* const* fb, const rgbid_intrinsics& K,
                    const rgbid_pose* inits, const rgbid_align_config& cfg,
                    rgbid_align_result* results, bool want_trace) {
  Lane& L = ctx->lanes[0];
  int rc = finish_all(ctx);  // a synchronous call leaves no chunk of an earlier call pending
  if (rc) return rc;
  rc = enqueue_chunk(ctx, L, n, fa, fb, K, inits, cfg, results, want_trace);
  if (rc) return rc;
  return finish_chunk(ctx, L);
}

// Slots per chunk of an n-pair batch.  Chunks bound the slot workspace (~28.6 MB
// per VGA slot: 2 lanes x 1024 slots = 59 GB) and alternate over the lanes; they
// go out in co-scheduled pairs, so a batch that fits one chunk is still split in
// two (e.g. 512 pairs per GPU at 8 GPUs -> 2 x 256) whenever both halves keep
// >= 32 slots.  RGBID_BATCH_SLOTS overrides the 1024 cap (read on every call).
int batch_chunk(int n) {
  const char* env = std::getenv("RGBID_BATCH_SLOTS");
  const int cap = env ? std::max(1, atoi(env)) : 1024;
  int nch = (n + cap - 1) / cap;
  if (nch == 1 && n >= 64) nch = 2;
  if (nch > 1) nch = (nch + kLanes - 1) / kLanes * kLanes;  // whole pairs / groups
  return (n + nch - 1) / nch;
}

int frame_from_host(rgbid_ctx* ctx, rgbid_frame** slot, int w, int h, const double* I,
                    const double* W) {
  if (*slot && ((*slot)->w != w || (*slot)->h != h)) {
    rgbid_frame_destroy(ctx, *slot);
    *slot = nullptr;
  }
  if (!*slot) {
    int rc = rgbid_frame_create(ctx, w, h, slot);
    if (rc) return rc;
  }
  return rgbid_frame_upload(ctx, *slot, I, W);
}

}  // namespace

// ===========================================================================
extern "C" {

const char* rgbid_version(void) { return "rgbid_b200 0.2 (sm_100a)"; }

int rgbid_batch_plan(int n, int* chunk, int* n_chunks) {
  if (n < 0 || !chunk || !n_chunks) return RGBID_E_ARG;
  *chunk = n > 0 ? batch_chunk(n) : 0;
  *n_chunks = n > 0 ? (n + *chunk - 1) / *chunk : 0;
  return RGBID_OK;
}

const char* rgbid_status_string(int s) {
  switch (s) {
    case RGBID_OK: return "ok";
    case RGBID_E_DEGENERATE: return "degenerate alignment: under-constrained scene";
    case RGBID_E_CUDA: return "CUDA error";
    case RGBID_E_ARG: return "invalid argument";
    case RGBID_E_OOM: return "out of device memory";
    default: return "unknown";
  }
}

int rgbid_ctx_create(int device, rgbid_ctx** out) {
  if (!out) return RGBID_E_ARG;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) return RGBID_E_CUDA;
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, device) != cudaSuccess) return RGBID_E_CUDA;
  if (p.major < 10) return RGBID_E_CUDA;  // sm_100a binary only
  if (cudaSetDevice(device) != cudaSuccess) return RGBID_E_CUDA;
  cudaGetLastError();
  rgbid_ctx* ctx = new rgbid_ctx();
  ctx->device = device;
  for (int k = 0; k < kLanes; ++k) {
    if (cudaStreamCreateWithFlags(&ctx->lanes[k].stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->lanes[k].done, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->lanes[k].ready, cudaEventDisableTiming) != cudaSuccess) {
      delete ctx;
      return RGBID_E_CUDA;
    }
  }
  ctx->stream = ctx->lanes[0].stream;
  if (init_kernel_attributes() != 0) {
    delete ctx;
    return RGBID_E_CUDA;
  }
  const char* g = std::getenv("RGBID_NO_GRAPHS");
  ctx->use_graphs = !(g && g[0] == '1');
  if (const char* e = std::getenv("RGBID_PAIR_STAGES")) g_pair_stages = atoi(e) == 4 ? 4 : 3;
  if (const char* e = std::getenv("RGBID_PAIR_OFFSET")) g_pair_offset = std::max(1, atoi(e));
  // graph switch nodes for the K1 / K3 slot rows (RGBID_GRAPH_SWITCH=0: none -- ncu
  // cannot profile the kernel nodes of a graph that has conditional nodes)
  if (const char* e = std::getenv("RGBID_GRAPH_SWITCH")) ctx->graph_switch = atoi(e) != 0;
  *out = ctx;
  return RGBID_OK;
}

int rgbid_ctx_destroy(rgbid_ctx* ctx) {
  if (!ctx) return RGBID_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& L : ctx->lanes) cudaStreamSynchronize(L.stream);
  drop_graphs(ctx);
  for (auto& L : ctx->lanes) free_lane_ws(L);
  for (auto& s : ctx->scratch)
    if (s.second.first) cudaFree(s.second.first);
  for (int k = 0; k < kLanes; ++k) {
    for (auto* f : ctx->host_fa[k]) rgbid_frame_destroy(ctx, f);
    for (auto* f : ctx->host_fb[k]) rgbid_frame_destroy(ctx, f);
  }
  if (ctx->tmpA) rgbid_frame_destroy(ctx, ctx->tmpA);
  if (ctx->tmpB) rgbid_frame_destroy(ctx, ctx->tmpB);
  cudaFree(ctx->d_trace);
  for (auto& e : ctx->pair_events) cudaEventDestroy(e);
  for (auto& L : ctx->lanes) {
    cudaEventDestroy(L.ready);
    cudaEventDestroy(L.done);
    cudaStreamDestroy(L.stream);
  }
  delete ctx;
  return RGBID_OK;
}

const char* rgbid_ctx_last_error(rgbid_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }
long long rgbid_ctx_kernel_launches(rgbid_ctx* ctx) { return ctx ? ctx->launches : 0; }
int rgbid_ctx_synchronize(rgbid_ctx* ctx) {
  if (!ctx) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  const int rc = finish_all(ctx);  // every lane's pending chunk, not only lane 0's
  if (rc) return rc;
  for (auto& L : ctx->lanes) CK(cudaStreamSynchronize(L.stream));
  return RGBID_OK;
}
void* rgbid_ctx_stream(rgbid_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int rgbid_frame_create(rgbid_ctx* ctx, int w, int h, rgbid_frame** out) {
  if (!ctx || !out || w <= 0 || h <= 0) return RGBID_E_ARG;
  cudaSetDevice(ctx->device);
  rgbid_frame* f = new rgbid_frame();
  f->w = w;
  f->h = h;
  const size_t N = (size_t)w * h;
  cudaError_t e = cudaMalloc(&f->I, sizeof(double) * 2 * N);
  if (e != cudaSuccess) {
    delete f;
    ctx->err = cudaGetErrorString(e);
    return RGBID_E_OOM;
  }
  f->W = f->I + N;
  f->pI[0] = f->I;
  f->pW[0] = f->W;
  *out = f;
  return RGBID_OK;
}

int rgbid_frame_upload(rgbid_ctx* ctx, rgbid_frame* f, const double* I, const double* W) {
  if (!ctx || !f || !W) return RGBID_E_ARG;
  const size_t N = (size_t)f->w * f->h;
  if (I)
    H2D(f->I, I, sizeof(double) * N);
  else
    CK(cudaMemsetAsync(f->I, 0xff, sizeof(double) * N, ctx->stream));  // NaN holes
  H2D(f->W, W, sizeof(double) * N);
  f->pyr_levels = 0;
  f->pyr_lane = -1;
  CK(cudaStreamSynchronize(ctx->stream));
  return RGBID_OK;
}

int rgbid_frame_download(rgbid_ctx* ctx, const rgbid_frame* f, double* I, double* W) {
  if (!ctx || !f) return RGBID_E_ARG;
  const size_t N = (size_t)f->w * f->h;
  if (I) D2H(I, f->I, sizeof(double) * N);
  if (W) D2H(W, f->W, sizeof(double) * N);
  CK(cudaStreamSynchronize(ctx->stream));
  return RGBID_OK;
}

int rgbid_frame_device_ptrs(rgbid_frame* f, double** I_dev, double** W_dev) {
  if (!f) return RGBID_E_ARG;
  if (I_dev) *I_dev = f->I;
  if (W_dev) *W_dev = f->W;
  f->pyr_levels = 0;  // caller may write through these pointers
  f->pyr_lane = -1;
  return RGBID_OK;
}

int rgbid_frame_destroy(rgbid_ctx* ctx, rgbid_frame* f) {
  (void)ctx;
  if (!f) return RGBID_E_ARG;
  cudaFree(f->I);
  if (f->pyr) cudaFree(f->pyr);
  delete f;
  return RGBID_OK;
}

int rgbid_build_pyramid(rgbid_ctx* ctx, const double* I, const double* W, int w, int h,
                        const rgbid_intrinsics* K, int levels, double** out_I, double** out_W,
                        rgbid_intrinsics* K_out) {
  if (!ctx || !W || !K || levels < 1 || levels > kMaxLevels) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  int rc = frame_from_host(ctx, &ctx->tmpA, w, h, I, W);
  if (rc) return rc;
  rgbid_frame* f = ctx->tmpA;
  rc = frame_ensure_pyramid(ctx, f, levels);
  if (rc) return rc;
  for (int l = 0; l < levels; ++l) {
    const size_t n = (size_t)(w >> l) * (h >> l);
    if (out_I && out_I[l])
      D2H(out_I[l], f->pI[l], sizeof(double) * n);
    if (out_W && out_W[l])
      D2H(out_W[l], f->pW[l], sizeof(double) * n);
    if (K_out) level_intrinsics(*K, l, &K_out[l]);
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return RGBID_OK;
}

int rgbid_inverse_geometric_warp(rgbid_ctx* ctx, const double* I_B, const double* W_B, int wb,
                                 int hb, const double* W_A, int w, int h, const rgbid_pose* T_AB,
                                 const rgbid_intrinsics* K, double* oI, double* oW, double* omx,
                                 double* omy) {
  if (!ctx || !W_B || !W_A || !T_AB || !K) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  const size_t NB = (size_t)wb * hb, N = (size_t)w * h;
  double *dB, *dA, *dO;
  int rc = scratch_buf(ctx, "warp_in", 2 * NB + N, &dB);
  if (rc) return rc;
  rc = scratch_buf(ctx, "warp_out", 4 * N, &dO);
  if (rc) return rc;
  dA = dB + 2 * NB;
  if (I_B)
    H2D(dB, I_B, sizeof(double) * NB);
  else
    CK(cudaMemsetAsync(dB, 0xff, sizeof(double) * NB, ctx->stream));
  H2D(dB + NB, W_B, sizeof(double) * NB);
  H2D(dA, W_A, sizeof(double) * N);
  const WarpMats m = warp_mats(pose_of(T_AB), K->fx, K->fy, K->cx, K->cy);
  launch_warp_maps(dB, dB + NB, wb, hb, dA, w, h, m, dO, dO + N, dO + 2 * N, dO + 3 * N,
                   ctx->stream);
  rc = check_launch(ctx);
  if (rc) return rc;
  double* outs[4] = {oI, oW, omx, omy};
  for (int k = 0; k < 4; ++k)
    if (outs[k])
      D2H(outs[k], dO + k * N, sizeof(double) * N);
  CK(cudaStreamSynchronize(ctx->stream));
  return RGBID_OK;
}

int rgbid_align(rgbid_ctx* ctx, const rgbid_frame* a, const rgbid_frame* b,
                const rgbid_intrinsics* K, const rgbid_pose* init, const rgbid_align_config* cfg,
                rgbid_align_result* result) {
  if (!ctx || !a || !b || !K || !result) return RGBID_E_ARG;
  if (a->w != b->w || a->h != b->h) return RGBID_E_ARG;
  const rgbid_align_config c = cfg ? *cfg : default_config();
  if (validate_cfg(c, a->w, a->h)) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  cudaSetDevice(ctx->device);
  int rc = run_align_slots(ctx, 1, &a, &b, *K, init, c, result, true);
  if (rc) return rc;
  return result->status;
}

int rgbid_align_host(rgbid_ctx* ctx, const double* IA, const double* WA, const double* IB,
                     const double* WB, int w, int h, const rgbid_intrinsics* K,
                     const rgbid_pose* init, const rgbid_align_config* cfg,
                     rgbid_align_result* result) {
  if (!ctx) return RGBID_E_ARG;
  int rc = frame_from_host(ctx, &ctx->tmpA, w, h, IA, WA);
  if (rc) return rc;
  rc = frame_from_host(ctx, &ctx->tmpB, w, h, IB, WB);
  if (rc) return rc;
  return rgbid_align(ctx, ctx->tmpA, ctx->tmpB, K, init, cfg, result);
}

int rgbid_last_align_trace(rgbid_ctx* ctx, rgbid_iter_trace* out, int max_entries, int* n) {
  if (!ctx || !n) return RGBID_E_ARG;
  const int m = std::min<int>(max_entries, (int)ctx->last_trace.size());
  if (out && m > 0) std::memcpy(out, ctx->last_trace.data(), sizeof(rgbid_iter_trace) * m);
  *n = m;
  return RGBID_OK;
}

int rgbid_align_batch(rgbid_ctx* ctx, int n, const rgbid_frame* const* a,
                      const rgbid_frame* const* b, const rgbid_intrinsics* K,
                      const rgbid_pose* inits, const rgbid_align_config* cfg,
                      rgbid_align_result* results) {
  if (!ctx || n < 0 || (n > 0 && (!a || !b || !K || !results))) return RGBID_E_ARG;
  if (n == 0) return RGBID_OK;
  const rgbid_align_config c = cfg ? *cfg : default_config();
  for (int i = 0; i < n; ++i)
    if (!a[i] || !b[i] || a[i]->w != a[0]->w || a[i]->h != a[0]->h || b[i]->w != a[0]->w ||
        b[i]->h != a[0]->h)
      return RGBID_E_ARG;
  if (validate_cfg(c, a[0]->w, a[0]->h)) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  cudaSetDevice(ctx->device);
  int rc0 = finish_all(ctx);  // chunks an earlier async host call left in flight
  if (rc0) return rc0;
  const int chunk = batch_chunk(n);
  // chunks go out in co-scheduled pairs (one graph, stage-offset), except when
  // profiling (serialised kernel times) or for a trailing single chunk
  const bool pairs = !ctx->prof.enabled && std::getenv("RGBID_NO_PAIRS") == nullptr;
  for (int i0 = 0; i0 < n;) {
    const int m = std::min(chunk, n - i0);
    const int m2 = pairs ? std::min(chunk, n - i0 - m) : 0;
    if (kLanes > 2 && pairs && n - i0 >= kLanes * m && m > 0) {  // a full group of equal chunks
      AlignLaunch aj[kLanes];
      rgbid_align_result* rj[kLanes];
      for (int j = 0; j < kLanes; ++j) {
        const int o = i0 + j * m;
        int rc = prepare_chunk(ctx, ctx->lanes[j], m, a + o, b + o, *K, inits ? inits + o : nullptr,
                               c, j == 0 && i0 == 0, &aj[j]);
        if (rc) return rc;
        rj[j] = results + o;
      }
      int rc = launch_group(ctx, kLanes, aj, *K, c, rj, i0 == 0);
      if (rc) return rc;
      i0 += kLanes * m;
    } else if (m2 > 0) {  // unequal sizes too (the graph key holds both)
      AlignLaunch pa, pb;
      int rc = prepare_chunk(ctx, ctx->lanes[0], m, a + i0, b + i0, *K,
                             inits ? inits + i0 : nullptr, c, i0 == 0, &pa);
      if (rc) return rc;
      rc = prepare_chunk(ctx, ctx->lanes[1], m2, a + i0 + m, b + i0 + m, *K,
                         inits ? inits + i0 + m : nullptr, c, false, &pb);
      if (rc) return rc;
      rc = launch_prepared(ctx, ctx->lanes[0], pa, &ctx->lanes[1], &pb, *K, c, results + i0,
                           results + i0 + m, i0 == 0);
      if (rc) return rc;
      i0 += m + m2;
    } else {
      const int rc = enqueue_chunk(ctx, ctx->lanes[0], m, a + i0, b + i0, *K,
                                   inits ? inits + i0 : nullptr, c, results + i0, i0 == 0);
      if (rc) return rc;
      i0 += m;
    }
  }
  for (auto& L : ctx->lanes) {
    const int rc = finish_chunk(ctx, L);
    if (rc) return rc;
  }
  for (auto& L : ctx->lanes) CK(cudaStreamSynchronize(L.stream));
  return RGBID_OK;
}

// Enqueues the uploads and alignments of one host batch; the lanes' last chunks
// may still be in flight on return (their results are written by finish_chunk:
// when the lane is next reused, or by rgbid_align_batch_host_wait).
static int align_batch_host_enqueue(rgbid_ctx* ctx, int n, const double* const* IA,
                                    const double* const* WA, const double* const* IB,
                                    const double* const* WB, int w, int h,
                                    const rgbid_intrinsics* K, const rgbid_pose* inits,
                                    const rgbid_align_config* cfg, int chunk,
                                    rgbid_align_result* results) {
  if (!ctx || n < 0 || !K || (n > 0 && (!IA || !WA || !IB || !WB || !results)))
    return RGBID_E_ARG;
  if (n == 0) return RGBID_OK;
  const rgbid_align_config c = cfg ? *cfg : default_config();
  if (validate_cfg(c, w, h)) return RGBID_E_ARG;
  if (chunk <= 0) chunk = 256;
  chunk = std::min(chunk, n);
  LaunchScope ls(ctx);
  // per-lane device frames for one chunk (cached in ctx across calls); uploads go on
  // the lane's stream, so the H2D of chunk c+1 overlaps the compute of chunk c
  auto& fa = ctx->host_fa;
  auto& fb = ctx->host_fb;
  auto cleanup = [&]() {
    for (auto& L : ctx->lanes) cudaStreamSynchronize(L.stream);
  };
  for (int k = 0; k < kLanes; ++k) {
    if (!fa[k].empty() && (fa[k][0]->w != w || fa[k][0]->h != h)) {
      cudaDeviceSynchronize();
      for (auto* f : fa[k]) rgbid_frame_destroy(ctx, f);
      for (auto* f : fb[k]) rgbid_frame_destroy(ctx, f);
      fa[k].clear();
      fb[k].clear();
    }
    while ((int)fa[k].size() < chunk) {
      rgbid_frame *x, *y;
      int rc = rgbid_frame_create(ctx, w, h, &x);
      if (rc) return cleanup(), rc;
      fa[k].push_back(x);
      rc = rgbid_frame_create(ctx, w, h, &y);
      if (rc) return cleanup(), rc;
      fb[k].push_back(y);
    }
  }
  const size_t bytes = sizeof(double) * (size_t)w * h;
  const unsigned long long call = ++ctx->host_call;
  int lane = 0;
  for (int i0 = 0; i0 < n; i0 += chunk, lane = (lane + 1) % kLanes) {
    const int m = std::min(chunk, n - i0);
    Lane& L = ctx->lanes[lane];
    int rc = finish_chunk(ctx, L);  // frames of this lane are free again
    if (rc) return cleanup(), rc;
    for (int i = 0; i < m; ++i) {
      H2DS(L.stream, fa[lane][i]->I, IA[i0 + i], bytes);
      H2DS(L.stream, fa[lane][i]->W, WA[i0 + i], bytes);
      H2DS(L.stream, fb[lane][i]->I, IB[i0 + i], bytes);
      H2DS(L.stream, fb[lane][i]->W, WB[i0 + i], bytes);
      fa[lane][i]->pyr_levels = 0;
      fa[lane][i]->pyr_lane = -1;
    }
    rc = enqueue_chunk(ctx, L, m, fa[lane].data(), fb[lane].data(), *K,
                       inits ? inits + i0 : nullptr, c, results + i0, i0 == 0);
    if (rc) return cleanup(), rc;
    L.pend_call = call;
  }
  // a lane this call did not reuse may still hold the previous call's last chunk:
  // complete it now, so every result of call k is written when call k+1 returns
  // (only this call's chunks stay in flight)
  for (auto& L : ctx->lanes)
    if (L.pend_n > 0 && L.pend_call != call) {
      const int rc = finish_chunk(ctx, L);
      if (rc) return cleanup(), rc;
    }
  return RGBID_OK;
}

int rgbid_align_batch_host_wait(rgbid_ctx* ctx) {
  if (!ctx) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  for (auto& L : ctx->lanes) {
    const int rc = finish_chunk(ctx, L);
    if (rc) return rc;
  }
  return RGBID_OK;
}

int rgbid_align_batch_host_async(rgbid_ctx* ctx, int n, const double* const* IA,
                                 const double* const* WA, const double* const* IB,
                                 const double* const* WB, int w, int h,
                                 const rgbid_intrinsics* K, const rgbid_pose* inits,
                                 const rgbid_align_config* cfg, int chunk,
                                 rgbid_align_result* results) {
  return align_batch_host_enqueue(ctx, n, IA, WA, IB, WB, w, h, K, inits, cfg, chunk, results);
}

int rgbid_align_batch_host(rgbid_ctx* ctx, int n, const double* const* IA,
                           const double* const* WA, const double* const* IB,
                           const double* const* WB, int w, int h, const rgbid_intrinsics* K,
                           const rgbid_pose* inits, const rgbid_align_config* cfg, int chunk,
                           rgbid_align_result* results) {
  const int rc = align_batch_host_enqueue(ctx, n, IA, WA, IB, WB, w, h, K, inits, cfg, chunk,
                                          results);
  const int rw = rgbid_align_batch_host_wait(ctx);
  return rc ? rc : rw;
}

int rgbid_filtered_hessian_covariance(rgbid_ctx* ctx, const rgbid_frame* a, const rgbid_frame* b,
                                      const rgbid_intrinsics* K, const rgbid_pose* T_AB,
                                      const rgbid_align_config* cfg, double* cov36,
                                      int* degenerate) {
  if (!ctx || !a || !b || !K || !T_AB || !cov36) return RGBID_E_ARG;
  rgbid_align_config c = cfg ? *cfg : default_config();
  // zero iterations at every level: only the covariance pass runs at T_AB
  c.levels = 1;
  c.n_iterations = 1;
  c.iterations[0] = 0;
  rgbid_align_result r;
  LaunchScope ls(ctx);
  int rc = run_align_slots(ctx, 1, &a, &b, *K, T_AB, c, &r, false);
  if (rc) return rc;
  std::memcpy(cov36, r.cov, sizeof(r.cov));
  if (degenerate) *degenerate = r.cov_degenerate;
  return RGBID_OK;
}

int rgbid_bilateral_filter(rgbid_ctx* ctx, const double* img, int w, int h, double ss, double sr,
                           double* out) {
  if (!ctx || !img || !out || w <= 0 || h <= 0) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  const size_t N = (size_t)w * h;
  double* d;
  int rc = scratch_buf(ctx, "bilateral", 2 * N, &d);
  if (rc) return rc;
  H2D(d, img, sizeof(double) * N);
  launch_bilateral(d, w, h, ss, sr, d + N, ctx->stream);
  rc = check_launch(ctx);
  if (rc) return rc;
  D2H(out, d + N, sizeof(double) * N);
  CK(cudaStreamSynchronize(ctx->stream));
  return RGBID_OK;
}

int rgbid_integrate_frame(rgbid_ctx* ctx, double* kf_W, double* kf_C, const double* frame_I,
                          const double* frame_W, int w, int h, const rgbid_pose* T,
                          const rgbid_intrinsics* K, double sigma_w) {
  (void)frame_I;  // the warped intensity is never used by the reference (src/fusion.cpp:70-71)
  if (!ctx || !kf_W || !kf_C || !frame_W || !T || !K) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  const size_t N = (size_t)w * h;
  double* d;
  int rc = scratch_buf(ctx, "integrate", 3 * N, &d);
  if (rc) return rc;
  FuseFrame* df;
  rc = scratch_buf(ctx, "integrate_frames", 1, &df);
  if (rc) return rc;
  H2D(d, kf_W, sizeof(double) * N);
  H2D(d + N, kf_C, sizeof(double) * N);
  H2D(d + 2 * N, frame_W, sizeof(double) * N);
  FuseFrame f;
  f.W = d + 2 * N;
  f.wm = warp_mats(pose_of(T), K->fx, K->fy, K->cx, K->cy);
  H2D(df, &f, sizeof(f));
  launch_integrate(df, 1, d, d + N, w, h, sigma_w, ctx->stream);
  rc = check_launch(ctx);
  if (rc) return rc;
  D2H(kf_W, d, sizeof(double) * N);
  D2H(kf_C, d + N, sizeof(double) * N);
  CK(cudaStreamSynchronize(ctx->stream));
  return RGBID_OK;
}

int rgbid_integrate_frames(rgbid_ctx* ctx, rgbid_frame* kf, double* kf_C_dev, int k,
                           const rgbid_frame* const* frames, const rgbid_pose* T,
                           const rgbid_intrinsics* K, double sigma_w) {
  if (!ctx) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  const int rc = rt_integrate_async(ctx, kf, kf_C_dev, k, frames, T, K, sigma_w);
  if (rc) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  return RGBID_OK;
}

int rgbid_covisibility_ratio(rgbid_ctx* ctx, const rgbid_frame* a, const rgbid_frame* b,
                             const rgbid_pose* T_BA, const rgbid_intrinsics* K, double sigma_w,
                             double* ratio, int* empty, long long* counts) {
  if (!ctx || !a || !b || !T_BA || !K || !ratio) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  unsigned long long* dc;
  int rc = scratch_buf(ctx, "covis", 4, &dc);
  if (rc) return rc;
  rc = rt_covis_enqueue(ctx, a, b, T_BA, K, sigma_w, dc);
  if (rc) return rc;
  unsigned long long hc[4];
  D2H(hc, dc, sizeof(hc));
  CK(cudaStreamSynchronize(ctx->stream));
  if (counts)
    for (int i = 0; i < 4; ++i) counts[i] = (long long)hc[i];
  int e = 0;
  rt_covis_ratio(hc, ratio, &e);
  if (empty) *empty = e;
  return RGBID_OK;
}

// make_loop_constraint — src/loop.cpp:174-203
int rgbid_make_loop_constraint(rgbid_ctx* ctx, const rgbid_frame* kf_i, const rgbid_frame* kf_j,
                               int id_i, int id_j, const rgbid_intrinsics* K,
                               const rgbid_pose* T_init, const rgbid_align_config* cfg,
                               double min_covisibility, int inliers, double hull_fraction,
                               rgbid_loop_constraint* out, int* accepted) {
  if (!ctx || !kf_i || !kf_j || !K || !out || !accepted) return RGBID_E_ARG;
  *accepted = 0;
  rgbid_align_result res;
  int rc = rgbid_align(ctx, kf_i, kf_j, K, T_init, cfg, &res);
  if (rc == RGBID_E_DEGENERATE) return RGBID_OK;  // catch (DegenerateAlignmentError) -> nullopt
  if (rc) return rc;
  // refined-overlap gate on covisibility_ratio(kf_i, kf_j, T_AB^-1, K, sigma_w = tdist_depth.sigma)
  const PoseD T_BA = pose_inverse(pose_of(&res.T_AB));
  rgbid_pose tba;
  pose_to(T_BA, tba.R, tba.t);
  double ratio = 0.0;
  int empty = 0;
  rc = rgbid_covisibility_ratio(ctx, kf_i, kf_j, &tba, K, res.tdist_depth.sigma, &ratio, &empty,
                                nullptr);
  if (rc) return rc;
  if (empty || ratio < min_covisibility) return RGBID_OK;
  std::memset(out, 0, sizeof(*out));
  out->i = id_i;
  out->j = id_j;
  out->T_ij = res.T_AB;
  double inv[36];
  lu_inverse6(res.cov, inv);  // Mat6::inverse (partial-pivot LU)
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) out->info[r * 6 + c] = 0.5 * (inv[r * 6 + c] + inv[c * 6 + r]);
  out->inliers = inliers;
  out->hull_fraction = hull_fraction;
  *accepted = 1;
  return RGBID_OK;
}

// normal_map — src/segmentation.cpp:10-57
int rgbid_normal_map(rgbid_ctx* ctx, const double* W, int w, int h, const rgbid_intrinsics* K,
                     double* nx, double* ny, double* nz) {
  if (!ctx || !W || !K || !nx || !ny || !nz || w <= 0 || h <= 0) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  const size_t N = (size_t)w * h;
  double* d;
  int rc = scratch_buf(ctx, "normal_map", 4 * N, &d);
  if (rc) return rc;
  H2D(d, W, sizeof(double) * N);
  launch_normal_map(d, w, h, K_mat(K->fx, K->fy, K->cx, K->cy), d + N, d + 2 * N, d + 3 * N,
                    ctx->stream);
  rc = check_launch(ctx);
  if (rc) return rc;
  D2H(nx, d + N, sizeof(double) * N);
  D2H(ny, d + 2 * N, sizeof(double) * N);
  D2H(nz, d + 3 * N, sizeof(double) * N);
  CK(cudaStreamSynchronize(ctx->stream));
  return RGBID_OK;
}

// export_map — src/pipeline.cpp:463-527
int rgbid_export_map(rgbid_ctx* ctx, int n_kf, const double* const* I, const double* const* W,
                     int w, int h, const rgbid_pose* T_W_kf, const rgbid_intrinsics* K,
                     double voxel, double* points, unsigned char* colors, long long capacity,
                     long long* n) {
  if (!ctx || n_kf < 0 || (n_kf > 0 && (!I || !W || !T_W_kf)) || !K || !n || w <= 0 || h <= 0)
    return RGBID_E_ARG;
  *n = 0;
  if (n_kf == 0) return RGBID_OK;
  LaunchScope ls(ctx);
  const size_t N = (size_t)w * h;
  double* d;
  int rc = scratch_buf(ctx, "export_map", 2 * N * n_kf, &d);
  if (rc) return rc;
  const M3 Km = K_mat(K->fx, K->fy, K->cx, K->cy), Kinv = m3_inv(Km);
  std::vector<ExportKF> kfs(n_kf);
  for (int k = 0; k < n_kf; ++k) {
    if (!I[k] || !W[k]) return RGBID_E_ARG;
    double* dI = d + 2 * N * k;
    double* dW = dI + N;
    H2D(dI, I[k], sizeof(double) * N);
    H2D(dW, W[k], sizeof(double) * N);
    ExportKF& e = kfs[k];
    e.I = dI;
    e.W = dW;
    e.T_W_kf = pose_of(&T_W_kf[k]);
    e.W_prev = nullptr;
    if (k > 0) {  // T_prev_kf = T_W_prev^-1 T_W_kf; Rt = K R K^-1; tt = K t
      e.W_prev = d + 2 * N * (k - 1) + N;
      const PoseD Tp = pose_compose(pose_inverse(pose_of(&T_W_kf[k - 1])), e.T_W_kf);
      e.Rt = m3_mul(m3_mul(Km, Tp.R), Kinv);
      e.tt = m3_mulv(Km, Tp.t);
    }
  }
  double* dp = nullptr;
  uint8_t* dc = nullptr;
  long long cnt = 0;
  const int e = export_map_device(kfs.data(), n_kf, w, h, Kinv, voxel, ctx->stream, &dp, &dc, &cnt);
  if (e) {
    ctx->err = std::string("export_map: ") + cudaGetErrorString((cudaError_t)e);
    return RGBID_E_CUDA;
  }
  *n = cnt;
  rc = RGBID_OK;
  if (cnt > capacity || (cnt > 0 && (!points || !colors))) {
    rc = RGBID_E_ARG;
  } else if (cnt > 0) {
    D2H(points, dp, sizeof(double) * 3 * cnt);
    D2H(colors, dc, 3 * cnt);
  }
  cudaFreeAsync(dp, ctx->stream);
  cudaFreeAsync(dc, ctx->stream);
  CK(cudaStreamSynchronize(ctx->stream));
  return rc;
}

int rgbid_correct_inverse_depth(rgbid_ctx* ctx, const double* Wm, int w, int h,
                                const rgbid_depth_intrinsics* d, const rgbid_intrinsics* K,
                                int spatial, double* out) {
  if (!ctx || !Wm || !d || !K || !out) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  const size_t N = (size_t)w * h;
  double* dd;
  int rc = scratch_buf(ctx, "correct", 2 * N, &dd);
  if (rc) return rc;
  H2D(dd, Wm, sizeof(double) * N);
  launch_correct_depth(dd, w, h, *d, *K, spatial, dd + N, ctx->stream);
  rc = check_launch(ctx);
  if (rc) return rc;
  D2H(out, dd + N, sizeof(double) * N);
  CK(cudaStreamSynchronize(ctx->stream));
  return RGBID_OK;
}

// inverse_warp of both maps of a distorted-sensor frame with f_w = K distort(K^-1 p)
// (src/warping.cpp:8-18, src/camera.cpp:11-22,41-45), device-resident
int rgbid_rectify_frame(rgbid_ctx* ctx, const rgbid_frame* src, const rgbid_intrinsics* K,
                        rgbid_frame* dst) {
  if (!ctx || !src || !K || !dst || src == dst || src->w != dst->w || src->h != dst->h ||
      K->width != src->w || K->height != src->h)
    return RGBID_E_ARG;
  LaunchScope ls(ctx);
  launch_rectify(src->I, src->W, src->w, src->h, *K, dst->I, dst->W, ctx->stream);
  dst->pyr_levels = 0;
  dst->pyr_lane = -1;
  const int rc = check_launch(ctx);
  if (rc) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  return RGBID_OK;
}

int rgbid_rectify(rgbid_ctx* ctx, const double* src, int w, int h, const rgbid_intrinsics* K,
                  double* out) {
  if (!ctx || !src || !K || !out || w <= 0 || h <= 0) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  const size_t N = (size_t)w * h;
  double* d;
  int rc = scratch_buf(ctx, "rectify", 2 * N, &d);
  if (rc) return rc;
  H2D(d, src, sizeof(double) * N);
  launch_rectify(d, nullptr, w, h, *K, d + N, nullptr, ctx->stream);
  rc = check_launch(ctx);
  if (rc) return rc;
  D2H(out, d + N, sizeof(double) * N);
  CK(cudaStreamSynchronize(ctx->stream));
  return RGBID_OK;
}

int rgbid_undistort_points(rgbid_ctx* ctx, const double* m_d, long long n,
                           const rgbid_intrinsics* K, double* m_u, unsigned char* ok) {
  if (!ctx || n < 0 || (n > 0 && (!m_d || !m_u || !ok)) || !K) return RGBID_E_ARG;
  if (n == 0) return RGBID_OK;
  LaunchScope ls(ctx);
  double* d;
  int rc = scratch_buf(ctx, "undistort", (size_t)4 * n + (n + 7) / 8, &d);
  if (rc) return rc;
  uint8_t* dok = reinterpret_cast<uint8_t*>(d + 4 * n);
  H2D(d, m_d, sizeof(double) * 2 * n);
  launch_undistort(d, n, *K, d + 2 * n, dok, ctx->stream);
  rc = check_launch(ctx);
  if (rc) return rc;
  D2H(m_u, d + 2 * n, sizeof(double) * 2 * n);
  D2H(ok, dok, (size_t)n);
  CK(cudaStreamSynchronize(ctx->stream));
  return RGBID_OK;
}

int rgbid_forward_register(rgbid_ctx* ctx, const double* WA, int w, int h, const rgbid_pose* T_BA,
                           const rgbid_intrinsics* KA, const rgbid_intrinsics* KB, double* out) {
  if (!ctx || !WA || !T_BA || !KA || !KB || !out) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  // host setup — src/warping.cpp:22-25
  const PoseD T = pose_of(T_BA), Tab = pose_inverse(T);
  const M3 KAm = K_mat(KA->fx, KA->fy, KA->cx, KA->cy), KBm = K_mat(KB->fx, KB->fy, KB->cx, KB->cy);
  const M3 Rt_BA = m3_mul(m3_mul(KBm, T.R), m3_inv(KAm));
  const M3 Rt_AB = m3_inv(Rt_BA);
  const V3 tt = m3_mulv(KAm, Tab.t);
  RegisterMats r;
  for (int i = 0; i < 9; ++i) r.Rt_AB[i] = Rt_AB.m[i / 3][i % 3];
  for (int i = 0; i < 3; ++i) r.tt[i] = tt.v[i];
  const int iw = std::max(w, KB->width), ih = std::max(h, KB->height);
  const size_t N = (size_t)w * h, NB = (size_t)KB->width * KB->height;
  double* d;
  unsigned long long* inter;
  int rc = scratch_buf(ctx, "register", N + NB, &d);
  if (rc) return rc;
  rc = scratch_buf(ctx, "register_inter", (size_t)iw * ih, &inter);
  if (rc) return rc;
  H2D(d, WA, sizeof(double) * N);
  launch_forward_register(d, w, h, r, inter, iw, ih, KB->width, KB->height, d + N, ctx->stream);
  rc = check_launch(ctx);
  if (rc) return rc;
  D2H(out, d + N, sizeof(double) * NB);
  CK(cudaStreamSynchronize(ctx->stream));
  return RGBID_OK;
}


int rgbid_synth_pair_device(rgbid_ctx* ctx, rgbid_frame* a, rgbid_frame* b,
                            const rgbid_intrinsics* K, uint32_t pair_seed, int variant,
                            rgbid_pose* T_AB_truth) {
  if (!ctx || !a || !b || !K || a->w != K->width || a->h != K->height || b->w != a->w ||
      b->h != a->h || variant < 0 || variant > 2)
    return RGBID_E_ARG;
  LaunchScope ls(ctx);
  // Pair geometry: A at a small random pose, B = A * random_pose(seed, 3 mm, 0.02 rad)
  SynthView va, vb;
  synth_pair_views(K, pair_seed, variant, &va, &vb, T_AB_truth);
  launch_render(va, a->I, a->W, ctx->stream);
  launch_render(vb, b->I, b->W, ctx->stream);
  a->pyr_levels = 0;
  b->pyr_levels = 0;
  int rc = check_launch(ctx);
  if (rc) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  return RGBID_OK;
}

int rgbid_ctx_set_profiling(rgbid_ctx* ctx, int enable) {
  if (!ctx) return RGBID_E_ARG;
  ctx->prof.enabled = enable != 0;
  return RGBID_OK;
}

int rgbid_ctx_reset_stats(rgbid_ctx* ctx) {
  if (!ctx) return RGBID_E_ARG;
  ctx->kstats.clear();
  ctx->h2d_bytes = ctx->d2h_bytes = 0;
  return RGBID_OK;
}

int rgbid_ctx_kernel_stats(rgbid_ctx* ctx, char* buf, int cap) {
  if (!ctx) return -1;
  std::string js = "{";
  bool first = true;
  for (auto& e : ctx->kstats) {
    char tmp[256];
    std::snprintf(tmp, sizeof(tmp), "%s\"%s\": [%lld, %.6f]", first ? "" : ", ", e.first.c_str(),
                  e.second.first, e.second.second);
    js += tmp;
    first = false;
  }
  js += "}";
  if (buf && cap > 0) {
    std::strncpy(buf, js.c_str(), cap - 1);
    buf[cap - 1] = 0;
  }
  return (int)js.size() + 1;
}

int rgbid_ctx_transfer_bytes(rgbid_ctx* ctx, long long* h2d, long long* d2h) {
  if (!ctx) return RGBID_E_ARG;
  if (h2d) *h2d = ctx->h2d_bytes;
  if (d2h) *d2h = ctx->d2h_bytes;
  return RGBID_OK;
}

int rgbid_remap_bilinear(rgbid_ctx* ctx, const double* src, int w, int h, const double* map_x,
                         const double* map_y, int out_w, int out_h, double* out) {
  if (!ctx || !src || !map_x || !map_y || !out || w <= 0 || h <= 0) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  const size_t N = (size_t)w * h, M = (size_t)out_w * out_h;
  double* d;
  int rc = scratch_buf(ctx, "remap", N + 3 * M, &d);
  if (rc) return rc;
  H2D(d, src, sizeof(double) * N);
  H2D(d + N, map_x, sizeof(double) * M);
  H2D(d + N + M, map_y, sizeof(double) * M);
  launch_remap_bilinear(d, w, h, d + N, d + N + M, (int)M, d + N + 2 * M, ctx->stream);
  rc = check_launch(ctx);
  if (rc) return rc;
  D2H(out, d + N + 2 * M, sizeof(double) * M);
  CK(cudaStreamSynchronize(ctx->stream));
  return RGBID_OK;
}

long long rgbid_residuals_and_jacobians(rgbid_ctx* ctx, const double* I_A, const double* W_A,
                                        const double* I_Bw, const double* W_Bw, int w, int h,
                                        const rgbid_intrinsics* K, double lambda_n_min,
                                        double* jets, unsigned char* has_depth, long long cap) {
  if (!ctx || !I_A || !W_A || !I_Bw || !W_Bw || !K) return -RGBID_E_ARG;
  LaunchScope ls(ctx);
  const size_t N = (size_t)w * h;
  double* d;
  uint8_t* fl;
  if (scratch_buf(ctx, "jets_in", 4 * N + 17 * N, &d)) return -RGBID_E_OOM;
  if (scratch_buf(ctx, "jets_flag", N, &fl)) return -RGBID_E_OOM;
  cudaStream_t st = ctx->stream;
  cudaMemcpyAsync(d, I_A, sizeof(double) * N, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d + N, W_A, sizeof(double) * N, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d + 2 * N, I_Bw, sizeof(double) * N, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d + 3 * N, W_Bw, sizeof(double) * N, cudaMemcpyHostToDevice, st);
  ctx->h2d_bytes += 32 * (long long)N;
  rgbid_intrinsics k = *K;
  k.width = w;
  k.height = h;
  LevelInfo li = make_level(k, w, h, 0);
  launch_jets(d, d + N, d + 2 * N, d + 3 * N, li, lambda_n_min, d + 4 * N, fl, st);
  if (check_launch(ctx)) return -RGBID_E_CUDA;
  std::vector<double> rec(17 * N);
  std::vector<uint8_t> flags(N);
  cudaMemcpyAsync(rec.data(), d + 4 * N, sizeof(double) * 17 * N, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(flags.data(), fl, N, cudaMemcpyDeviceToHost, st);
  ctx->d2h_bytes += 137 * (long long)N;
  if (cudaStreamSynchronize(st) != cudaSuccess) return -RGBID_E_CUDA;
  long long n = 0;  // row-major compaction (the reference's push_back order)
  for (size_t i = 0; i < N; ++i) {
    if (!flags[i]) continue;
    if (n < cap) {
      if (jets) std::memcpy(jets + 17 * n, rec.data() + 17 * i, 17 * sizeof(double));
      if (has_depth) has_depth[n] = flags[i] == 2;
    }
    ++n;
  }
  return n;
}

int rgbid_estimate_location_scale(rgbid_ctx* ctx, const double* r, long long n, double nu,
                                  rgbid_tdist* out) {
  if (!ctx || (!r && n > 0) || !out) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  double* d;
  int rc = scratch_buf(ctx, "tdist_vec", (size_t)n + 4, &d);
  if (rc) return rc;
  if (n > 0) H2D(d + 4, r, sizeof(double) * n);
  launch_tdist_vec(d + 4, n, 0, nu, 0.0, d, ctx->stream);
  rc = check_launch(ctx);
  if (rc) return rc;
  double o[3];
  D2H(o, d, sizeof(o));
  CK(cudaStreamSynchronize(ctx->stream));
  out->mu = o[0];
  out->sigma = o[1];
  out->nu = o[2];
  return RGBID_OK;
}

int rgbid_estimate_nu(rgbid_ctx* ctx, const double* r, long long n, double mu, double sigma,
                      double* nu) {
  if (!ctx || (!r && n > 0) || !nu) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  double* d;
  int rc = scratch_buf(ctx, "tdist_vec", (size_t)n + 4, &d);
  if (rc) return rc;
  if (n > 0) H2D(d + 4, r, sizeof(double) * n);
  launch_tdist_vec(d + 4, n, 1, mu, sigma, d, ctx->stream);
  rc = check_launch(ctx);
  if (rc) return rc;
  D2H(nu, d, sizeof(double));
  CK(cudaStreamSynchronize(ctx->stream));
  return RGBID_OK;
}

int rgbid_selftest_division(rgbid_ctx* ctx, unsigned long long n, unsigned long long seed,
                            unsigned long long* mismatches) {
  if (!ctx || !mismatches) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  return selftest_division(n, seed, mismatches, ctx->stream) ? RGBID_E_CUDA : RGBID_OK;
}

int rgbid_frame_copy(rgbid_ctx* ctx, rgbid_frame* dst, const rgbid_frame* src) {
  if (!ctx || !dst || !src || dst->w != src->w || dst->h != src->h) return RGBID_E_ARG;
  CK(cudaMemcpyAsync(dst->I, src->I, sizeof(double) * 2 * (size_t)src->w * src->h,
                     cudaMemcpyDeviceToDevice, ctx->stream));
  dst->pyr_levels = 0;
  dst->pyr_lane = -1;
  return RGBID_OK;
}

int rgbid_fill(rgbid_ctx* ctx, double* dev, long long n, double value) {
  if (!ctx || (!dev && n > 0)) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  launch_fill(dev, n, value, ctx->stream);
  return check_launch(ctx);
}

int rgbid_frame_decode(rgbid_ctx* ctx, rgbid_frame* f, const uint8_t* bgr, const uint16_t* depth,
                       double scale) {
  if (!ctx || !f || !depth) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  const size_t N = (size_t)f->w * f->h;
  uint8_t* d;
  int rc = scratch_buf(ctx, "decode", 5 * N, &d);
  if (rc) return rc;
  uint16_t* dd = reinterpret_cast<uint16_t*>(d + 3 * N);
  if (bgr) H2D(d, bgr, 3 * N);
  H2D(dd, depth, 2 * N);
  if (!bgr) CK(cudaMemsetAsync(f->I, 0xff, sizeof(double) * N, ctx->stream));
  launch_decode_frame(bgr ? d : nullptr, dd, (int)N, scale, f->I, f->W, ctx->stream);
  f->pyr_levels = 0;
  f->pyr_lane = -1;
  rc = check_launch(ctx);
  if (rc) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  return RGBID_OK;
}

int rgbid_measure_fp64_peak(rgbid_ctx* ctx, double* tflops) {
  if (!ctx || !tflops) return RGBID_E_ARG;
  *tflops = measure_fp64_tflops(ctx->stream);
  return check_launch(ctx);
}

int rgbid_frame_invalidate(rgbid_frame* f) {
  if (!f) return RGBID_E_ARG;
  f->pyr_levels = 0;
  f->pyr_lane = -1;
  return RGBID_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// stream-ordered building blocks (runtime_internal.cuh)
namespace rgbid_b200 {

int rt_frame_upload_async(rgbid_ctx* ctx, rgbid_frame* f, const double* I, const double* W) {
  if (!ctx || !f || !W) return RGBID_E_ARG;
  const size_t N = (size_t)f->w * f->h;
  if (I)
    H2D(f->I, I, sizeof(double) * N);
  else
    CK(cudaMemsetAsync(f->I, 0xff, sizeof(double) * N, ctx->stream));  // NaN holes
  H2D(f->W, W, sizeof(double) * N);
  f->pyr_levels = 0;
  f->pyr_lane = -1;
  return RGBID_OK;
}

int rt_covis_enqueue(rgbid_ctx* ctx, const rgbid_frame* a, const rgbid_frame* b,
                     const rgbid_pose* T_BA, const rgbid_intrinsics* K, double sigma_w,
                     unsigned long long* counts_dev) {
  if (!ctx || !a || !b || !T_BA || !K || !counts_dev) return RGBID_E_ARG;
  if (a->w != b->w || a->h != b->h) return RGBID_E_ARG;
  LaunchScope ls(ctx);
  // host setup — src/fusion.cpp:29-32 (R~ = K R K^-1, t~ = K t per direction)
  const M3 Km = K_mat(K->fx, K->fy, K->cx, K->cy), Kinv = m3_inv(Km);
  auto dir = [&](const rgbid_frame* A, const rgbid_frame* B, const PoseD& T) {
    CovisDir d;
    d.WA = A->W;
    d.WB = B->W;
    const M3 Rt = m3_mul(m3_mul(Km, T.R), Kinv);
    const V3 tt = m3_mulv(Km, T.t);
    for (int i = 0; i < 9; ++i) d.Rt[i] = Rt.m[i / 3][i % 3];
    for (int i = 0; i < 3; ++i) d.tt[i] = tt.v[i];
    return d;
  };
  const PoseD T = pose_of(T_BA);
  const CovisDir d0 = dir(a, b, T), d1 = dir(b, a, pose_inverse(T));
  launch_covisibility(d0, d1, a->w, a->h, sigma_w, counts_dev, ctx->stream);
  return check_launch(ctx);
}

void rt_covis_ratio(const unsigned long long* hc, double* ratio, int* empty) {
  *ratio = 0.0;
  *empty = 0;
  if (hc[0] == 0 || hc[2] == 0)
    *empty = 1;
  else
    *ratio = dmin_std((double)hc[1] / (double)hc[0], (double)hc[3] / (double)hc[2]);
}

int rt_integrate_async(rgbid_ctx* ctx, rgbid_frame* kf, double* kf_C_dev, int k,
                       const rgbid_frame* const* frames, const rgbid_pose* T,
                       const rgbid_intrinsics* K, double sigma_w) {
  if (!ctx || !kf || !kf_C_dev || k < 0 || (k > 0 && (!frames || !T)) || !K) return RGBID_E_ARG;
  if (k == 0) return RGBID_OK;
  LaunchScope ls(ctx);
  std::vector<FuseFrame> hf(k);
  for (int i = 0; i < k; ++i) {
    if (frames[i]->w != kf->w || frames[i]->h != kf->h) return RGBID_E_ARG;
    hf[i].W = frames[i]->W;
    hf[i].wm = warp_mats(pose_of(&T[i]), K->fx, K->fy, K->cx, K->cy);
  }
  FuseFrame* df;
  int rc = scratch_buf(ctx, "integrate_frames", k, &df);
  if (rc) return rc;
  H2D(df, hf.data(), sizeof(FuseFrame) * k);  // pageable: staged before return
  launch_integrate(df, k, kf->W, kf_C_dev, kf->w, kf->h, sigma_w, ctx->stream);
  kf->pyr_levels = 0;
  return check_launch(ctx);
}

}  // namespace rgbid_b200
