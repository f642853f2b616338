// Device data layout + kernel declarations of the B200 alignment path.
//
// One "slot" = one independent alignment of a batch (config 5) or the single
// alignment of rgbid_align (batch of 1).  Every kernel takes the slot array and
// a per-level LevelInfo; grid.y (or grid.x for per-slot kernels) indexes slots.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "hd_math.cuh"

namespace rgbid_b200 {

constexpr int kMaxLevels = 6;       // GPU supports levels <= 6 (80x60 at level 3 for VGA)
constexpr int kMaxSample = 19200;   // src/alignment.cpp:47
constexpr int kTPB = 256;           // warp/residual/normal-equation kernels
#ifndef RGBID_TDIST_THREADS
#define RGBID_TDIST_THREADS 512
#endif
constexpr int kTdistThreads = RGBID_TDIST_THREADS;  // Student-t kernel (sample in shared memory)
constexpr int kNPart = 28;          // 21 (lower H) + 6 (b) + 1 (cost)
constexpr int kTraceMax = 64;
#ifndef RGBID_TDIST_CLUSTER
#define RGBID_TDIST_CLUSTER 8
#endif
constexpr int kTdistCluster = RGBID_TDIST_CLUSTER;  // CTAs per Student-t chain in latency mode
constexpr int kTdistClusterMaxSlots = 8; // batches up to this size use the cluster kernel
#ifndef RGBID_TDIST_CLUSTER_THREADS
#define RGBID_TDIST_CLUSTER_THREADS 256
#endif
constexpr int kTdistClusterThreads = RGBID_TDIST_CLUSTER_THREADS;
constexpr int kPixK3 = 8;           // pixels per thread in the normal-equation kernel
// K3 tiles: kTPB * pix consecutive level pixels (pix = kPixK3 for batches, 1 in
// latency mode: one pixel per thread, 8x the CTAs for one slot)
__host__ __device__ constexpr int k3_tiles(int w, int h, int pix = kPixK3) {
  return (w * h + kTPB * pix - 1) / (kTPB * pix);
}

// K1 tiling of level l: tile = (level row, segment of tx level pixels).
// Full-res pixels per tile = tx * 4^l <= 2048 (smem staging of the warp).
__host__ __device__ constexpr int k1_tx(int l) {
  const int a = 256 >> l, b = 2048 >> (2 * l);
  const int m = a < b ? a : b;
  return m < 1 ? 1 : m;
}

struct LevelInfo {
  int level;
  int w, h;          // level image size (w0 >> l, h0 >> l)
  int tx, nseg;      // K1 tiling
  int ntiles;        // K1 tiles = h * nseg
  int ntiles3;       // K3 tiles of kTPB * pix3 consecutive pixels
  int pix3;          // K3 pixels per thread (kPixK3, or 1 in latency mode)
  double fx, fy, cx, cy;
  double Kinv[9];    // level K^-1 (host m3_inv, bit-identical to the oracle)
  double bx1, by1;   // full-res frame B bounds w0 - 1, h0 - 1 (K1's bilinear test)
};

constexpr int kWordsPerTile = 8;  // K1 tile <= 256 level pixels -> 8 ballot words per type

struct SlotIO {
  double* IA[kMaxLevels];        // A pyramid (level 0 = frame A; levels >= 1 built on device)
  double* WA[kMaxLevels];
  const double* IB;              // frame B, level 0
  const double* WB;
  double2* IWB;                  // frame B interleaved {I, W} (K1's bilinear taps)
  double* fIA;                   // bilateral-filtered A (covariance pass)
  double* fWA;
  double2* ibw;                  // {r_I = warped I_B - I_A, warped W_B} per level pixel (K1)
  uint8_t* amask[kMaxLevels];    // A-side jet validity per level pixel (bit0 photometric, bit1 depth)
  double* agrad[kMaxLevels];     // A-side gradients per level pixel {gI_x, gI_y, gW_x, gW_y}
                                 // (level-0 entries are rebuilt from the filtered A for the
                                 //  covariance pass)
  int* cntI;                     // per K1 tile counts (jets / depth jets)
  int* cntW;
  unsigned* bitsI;               // per K1 tile validity bitmask [ntiles][kWordsPerTile]
  unsigned* bitsW;
  double* part;                  // K3 partial sums [kNPart][ntiles3] (value-major)
  double* smp;                   // K2 systematic samples [2][kMaxSample] (r_I, r_W; k_gather)
  int* nsmp;                     // K2 valid residual counts [2] (k_gather)
  int build_pyr;                 // 1: this slot builds frame A's pyramid levels >= 1
};

struct SlotState {
  double R[9], t[3];   // current T_AB
  WarpMats wm;         // warp matrices of the current T_AB (full resolution)
  int status;          // rgbid_status
  int done_level;      // level whose loop broke on ||xi|| < eps (-1 = none)
  int iters[kMaxLevels];
  double cost[kMaxLevels];
  rgbid_tdist tI, tW;        // current iteration, as estimated (tI.nu not yet maxed)
  rgbid_tdist finI, finW;    // last level-0 iteration (tI.nu maxed), AlignmentResult::tdist_*
  long long nI, nW;          // jets / depth jets of the current iteration
  double H[36];              // last normal matrix (error payload / trace)
  double cov[36];
  int cov_degenerate;
  int total_iters;
  int trace_n;
};

// phase 0 = IRLS level loop, phase 1 = filtered-Hessian covariance pass
__device__ __forceinline__ bool slot_active(const SlotState& s, int level, int phase) {
  return s.status == RGBID_OK && (phase == 1 || s.done_level != level);
}

struct AlignLaunch {
  SlotIO* io;          // device array [nslots]
  SlotState* st;       // device array [nslots]
  rgbid_iter_trace* trace;  // device [kTraceMax] (slot 0) or nullptr
  int nslots;
  int w0, h0;
  double eps;
  double lambda_n_min;
  // device [1 + nslots]: count, then the slots still iterating in slot order
  // (k_active_slots, before each K1); nullptr = every CTA row maps one slot
  int* act = nullptr;
  bool graph_switch = true;  // captured graphs pick K1 / K3 grids by switch nodes
};

// Batches above this size run K1 / K3 over a compact active-slot list, their grids
// picked per iteration on the device by graph switch nodes (k_active_slots).
constexpr int kActiveListMinSlots = 16;
inline bool use_active_list(int nslots) { return nslots > kActiveListMinSlots; }
struct SlotSwitch {
  cudaGraphConditionalHandle h[2] = {0, 0};  // the iteration's K1 and K3 switch nodes
  int nbodies = 0;                           // body k: ceil(nslots / 2^k) slot rows
};
// compaction of the slots still active at (level, phase) into a.act, setting the
// switch values of *sw (no-op without a list)
void launch_active_slots(const AlignLaunch& a, int level, int phase, cudaStream_t s,
                         const SlotSwitch* sw);

// Kernel launchers (align_kernels.cu); all asynchronous on `stream`.
// rows: slot rows of the grid (0 = one per slot)
void launch_warp_residuals(const AlignLaunch& a, const LevelInfo& li, int phase, cudaStream_t s,
                           int rows = 0);
// K2: part 0 = gather + Student-t, 1 = gather only (K2a), 2 = Student-t only (K2b);
// latency mode (<= kTdistClusterMaxSlots slots) has no separate gather
void launch_tdist(const AlignLaunch& a, const LevelInfo& li, int phase, cudaStream_t s,
                  int part = 0);
void launch_normal_equations(const AlignLaunch& a, const LevelInfo& li, int phase, cudaStream_t s,
                             int rows = 0);
void launch_solve(const AlignLaunch& a, const LevelInfo& li, const LevelInfo& li0, cudaStream_t s);
void launch_covariance(const AlignLaunch& a, const LevelInfo& li, cudaStream_t s);
void launch_downsample2(const double* I, const double* W, int w, int h, double* oI, double* oW,
                        cudaStream_t s);
void launch_pyramid_slots(const AlignLaunch& a, int levels, cudaStream_t s);
void launch_amask(const AlignLaunch& a, int levels, int phase, cudaStream_t s);
void launch_interleave_B(const AlignLaunch& a, cudaStream_t s);
void launch_bilateral_pair(const AlignLaunch& a, double ss, double sr_i, double sr_w,
                           cudaStream_t s);
void launch_bilateral(const double* img, int w, int h, double ss, double sr, double* out,
                      cudaStream_t s);
void launch_warp_maps(const double* IB, const double* WB, int wb, int hb, const double* WA, int w,
                      int h, const WarpMats& m, double* oI, double* oW, double* omx, double* omy,
                      cudaStream_t s);
int tdist_smem_bytes(int ntiles);
double measure_fp64_tflops(cudaStream_t s);
void launch_fill(double* p, long long n, double v, cudaStream_t s);
void launch_remap_bilinear(const double* src, int w, int h, const double* mx, const double* my,
                           int n, double* out, cudaStream_t s);
void launch_jets(const double* IA, const double* WA, const double* IBw, const double* WBw,
                 const LevelInfo& li, double lambda_n_min, double* rec, uint8_t* flag,
                 cudaStream_t s);
int launch_tdist_vec(const double* r, long long n, int mode, double a, double b, double* out,
                     cudaStream_t s);
int selftest_division(unsigned long long n, unsigned long long seed, unsigned long long* out,
                      cudaStream_t s);
int init_kernel_attributes();

// Launch accounting + optional per-kernel CUDA-event timing.  Every library
// kernel launch is wrapped in a KScope (launchers below); the owning ctx routes
// the counters through these thread-locals for the duration of an API call.
struct KernelRecord {
  const char* name;
  cudaEvent_t start, stop;
};
struct Profiler {
  bool enabled = false;
  std::vector<KernelRecord> pending;  // events recorded, not yet read back
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get();
};
extern thread_local long long* g_launch_counter;
extern thread_local Profiler* g_profiler;
struct KScope {
  KScope(const char* name, cudaStream_t s);
  ~KScope();
  const char* name;
  cudaStream_t stream;
  cudaEvent_t stop = nullptr;
};

}  // namespace rgbid_b200
