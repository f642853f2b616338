// Normal map and map export — SURVEY 8(f) rank 4 (per-pixel kernels reusing the
// warp / gradient arithmetic of the hot path).  Both restate the reference
// bit for bit: every expression follows the Eigen evaluation order of the
// reference sources (3-term sums v0 + (v1 + v2), coefficient-wise division).
#include <cub/cub.cuh>
#include <math_constants.h>

#include "align_kernels.cuh"  // KScope (launch accounting / profiling)
#include "map_kernels.cuh"

namespace rgbid_b200 {

namespace {

__device__ __forceinline__ bool finite_d(double v) { return isfinite(v); }  // is_valid

// Image::operator() with in_bounds (integer) else a hole
__device__ __forceinline__ double tap(const double* W, int w, int h, int x, int y) {
  return (x >= 0 && x < w && y >= 0 && y < h) ? __ldg(W + (size_t)y * w + x) : CUDART_NAN;
}

// bilinear — include/rgbid/image.hpp:51-62
__device__ __forceinline__ double bilinear_ref(const double* img, int w, int h, double x, double y) {
  if (!(x >= 0.0 && x <= w - 1.0 && y >= 0.0 && y <= h - 1.0)) return CUDART_NAN;
  const int x0 = (int)floor(x), y0 = (int)floor(y);
  const int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
  const double fx = x - x0, fy = y - y0;
  const double v00 = __ldg(img + (size_t)y0 * w + x0), v10 = __ldg(img + (size_t)y0 * w + x1);
  const double v01 = __ldg(img + (size_t)y1 * w + x0), v11 = __ldg(img + (size_t)y1 * w + x1);
  if (!finite_d(v00) || !finite_d(v10) || !finite_d(v01) || !finite_d(v11)) return CUDART_NAN;
  return (1 - fy) * ((1 - fx) * v00 + fx * v10) + fy * ((1 - fx) * v01 + fx * v11);
}

// normal_map — src/segmentation.cpp:10-57
__global__ void k_normal_map(const double* __restrict__ W, int w, int h, M3 Km,
                             double* __restrict__ nx, double* __restrict__ ny,
                             double* __restrict__ nz) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= w * h) return;
  const int y = k / w, x = k - y * w;
  double o0 = CUDART_NAN, o1 = CUDART_NAN, o2 = CUDART_NAN;  // NormalMap(w, h) holes
  const double wv = __ldg(W + k);
  if (finite_d(wv) && wv > 0.0) {
    const double l = tap(W, w, h, x - 1, y), r = tap(W, w, h, x + 1, y);
    const double u = tap(W, w, h, x, y - 1), d = tap(W, w, h, x, y + 1);
    double gx = 0.0, gy = 0.0;
    bool deg = false;
    if (finite_d(l) && finite_d(r))
      gx = (r - l) / 2.0;
    else if (finite_d(r))
      gx = r - wv;
    else if (finite_d(l))
      gx = wv - l;
    else
      deg = true;
    if (!deg) {
      if (finite_d(u) && finite_d(d))
        gy = (d - u) / 2.0;
      else if (finite_d(d))
        gy = d - wv;
      else if (finite_d(u))
        gy = wv - u;
      else
        deg = true;
    }
    if (deg) {
      o0 = -0.0, o1 = -0.0, o2 = -1.0;  // -Vec3::UnitZ()
    } else {
      // A = K; A.col(2) -= (x, y, 1); n = (g^T A)^T / w + e_z
      M3 A = Km;
      A.m[0][2] = Km.m[0][2] - (double)x;
      A.m[1][2] = Km.m[1][2] - (double)y;
      A.m[2][2] = Km.m[2][2] - 1.0;
      double n[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) n[j] = red3(gx * A.m[0][j], gy * A.m[1][j], 0.0 * A.m[2][j]);
      n[0] = n[0] / wv + 0.0;
      n[1] = n[1] / wv + 0.0;
      n[2] = n[2] / wv + 1.0;
      const double nn = sqrt(red3(n[0] * n[0], n[1] * n[1], n[2] * n[2]));
      if (nn < 1e-12) {
        o0 = -0.0, o1 = -0.0, o2 = -1.0;
      } else {
        n[0] /= nn, n[1] /= nn, n[2] /= nn;
        if (n[2] > 0) n[0] = -n[0], n[1] = -n[1], n[2] = -n[2];  // orient toward the camera
        o0 = n[0], o1 = n[1], o2 = n[2];
      }
    }
  }
  nx[k] = o0;
  ny[k] = o1;
  nz[k] = o2;
}

// export_map, per-pixel part — src/pipeline.cpp:478-500: novelty against the
// previous keyframe, world point, grey colour.  flag = 1 for an emitted point.
__global__ void k_export_points(ExportKF kf, int w, int h, M3 Kinv, int* __restrict__ flag,
                                double* __restrict__ pts, uint8_t* __restrict__ col) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= w * h) return;
  const int y = k / w, x = k - y * w;
  const double wv = __ldg(kf.W + k);
  bool emit = finite_d(wv) && wv > 0.0;
  if (emit && kf.W_prev) {
    // q = Rt p + w tt
    const double q0 = red3(kf.Rt.m[0][0] * x, kf.Rt.m[0][1] * y, kf.Rt.m[0][2] * 1.0) + wv * kf.tt.v[0];
    const double q1 = red3(kf.Rt.m[1][0] * x, kf.Rt.m[1][1] * y, kf.Rt.m[1][2] * 1.0) + wv * kf.tt.v[1];
    const double q2 = red3(kf.Rt.m[2][0] * x, kf.Rt.m[2][1] * y, kf.Rt.m[2][2] * 1.0) + wv * kf.tt.v[2];
    if (q2 > 0.0) {
      const double u = q0 / q2, v = q1 / q2;
      if (u >= 0.0 && u <= w - 1.0 && v >= 0.0 && v <= h - 1.0) {
        const double w_prev = bilinear_ref(kf.W_prev, w, h, u, v);
        const double w_pred = wv / q2;
        if (finite_d(w_prev) && fabs(w_prev - w_pred) < 3.0 * 0.02) emit = false;
      }
    }
  }
  flag[k] = emit ? 1 : 0;
  if (!emit) return;
  // X_kf = K^-1 (x, y, 1) / w ; X_W = R X_kf + t
  double X[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) X[i] = red3(Kinv.m[i][0] * x, Kinv.m[i][1] * y, Kinv.m[i][2] * 1.0) / wv;
#pragma unroll
  for (int i = 0; i < 3; ++i)
    pts[3 * (size_t)k + i] =
        red3(kf.T_W_kf.R.m[i][0] * X[0], kf.T_W_kf.R.m[i][1] * X[1], kf.T_W_kf.R.m[i][2] * X[2]) +
        kf.T_W_kf.t.v[i];
  const double g = __ldg(kf.I + k);  // in_bounds(x, y) always holds here
  const double gc = (g < 0.0) ? 0.0 : (1.0 < g) ? 1.0 : g;  // std::clamp(g, 0, 1)
  const uint8_t c = (uint8_t)(unsigned)(gc * 255.0);
  col[3 * (size_t)k + 0] = c;
  col[3 * (size_t)k + 1] = c;
  col[3 * (size_t)k + 2] = c;
}

__global__ void k_compact(const int* __restrict__ flag, const int* __restrict__ pos, long long n,
                          const double* __restrict__ pts, const uint8_t* __restrict__ col,
                          double* __restrict__ opts, uint8_t* __restrict__ ocol) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n || !flag[k]) return;
  const long long p = pos[k];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    opts[3 * p + i] = pts[3 * k + i];
    ocol[3 * p + i] = col[3 * k + i];
  }
}

// voxel key — src/pipeline.cpp:510-515 (int64 products wrap like the x86 build)
__global__ void k_voxel_keys(const double* __restrict__ pts, long long n, double voxel,
                             unsigned long long* __restrict__ key, int* __restrict__ idx) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const long long ix = (long long)floor(pts[3 * k + 0] / voxel);
  const long long iy = (long long)floor(pts[3 * k + 1] / voxel);
  const long long iz = (long long)floor(pts[3 * k + 2] / voxel);
  const unsigned long long h = ((unsigned long long)ix * 73856093ull) ^
                               ((unsigned long long)iy * 19349663ull) ^
                               ((unsigned long long)iz * 83492791ull);
  key[k] = h;
  idx[k] = (int)k;
}

// group heads of the key-sorted order (stable: indices ascend within a key), and
// the "first occurrence" marks over the original order
__global__ void k_voxel_heads(const unsigned long long* __restrict__ skey, const int* __restrict__ sidx,
                              long long n, int* __restrict__ head, int* __restrict__ first) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const bool hd = j == 0 || skey[j] != skey[j - 1];
  head[j] = hd ? 1 : 0;
  if (hd) first[sidx[j]] = 1;
}

// one thread per voxel: the reference's accumulation (sum += p, color += c, ++n)
// in insertion order, then sum / n and the truncated colour average
__global__ void k_voxel_average(const unsigned long long* __restrict__ skey,
                                const int* __restrict__ sidx, const int* __restrict__ head,
                                const int* __restrict__ opos, long long n,
                                const double* __restrict__ pts, const uint8_t* __restrict__ col,
                                double* __restrict__ opts, uint8_t* __restrict__ ocol) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n || !head[j]) return;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
  int cnt = 0;
  for (long long e = j; e < n && (e == j || skey[e] == skey[j]); ++e) {
    const int i = sidx[e];
    s0 += pts[3 * (size_t)i + 0];
    s1 += pts[3 * (size_t)i + 1];
    s2 += pts[3 * (size_t)i + 2];
    c0 += (double)col[3 * (size_t)i + 0];
    c1 += (double)col[3 * (size_t)i + 1];
    c2 += (double)col[3 * (size_t)i + 2];
    ++cnt;
  }
  const long long p = opos[sidx[j]];
  const double dn = (double)cnt;
  opts[3 * p + 0] = s0 / dn;
  opts[3 * p + 1] = s1 / dn;
  opts[3 * p + 2] = s2 / dn;
  ocol[3 * p + 0] = (uint8_t)(unsigned)(c0 / dn);
  ocol[3 * p + 1] = (uint8_t)(unsigned)(c1 / dn);
  ocol[3 * p + 2] = (uint8_t)(unsigned)(c2 / dn);
}

inline unsigned blocks(long long n, int t) { return (unsigned)((n + t - 1) / t); }

// stream-ordered temporaries of one export_map call, freed on every exit path
struct AsyncPool {
  cudaStream_t s;
  void* p[16] = {};
  int n = 0;
  explicit AsyncPool(cudaStream_t st) : s(st) {}
  ~AsyncPool() {
    for (int i = 0; i < n; ++i)
      if (p[i]) cudaFreeAsync(p[i], s);
  }
  template <typename T>
  cudaError_t alloc(T** out, size_t count) {
    const cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(out), sizeof(T) * (count ? count : 1), s);
    if (e == cudaSuccess) p[n++] = *out;
    return e;
  }
  void release(const void* q) {  // keep q (handed to the caller)
    for (int i = 0; i < n; ++i)
      if (p[i] == q) p[i] = nullptr;
  }
};

cudaError_t exclusive_sum(const int* in, int* out, long long n, cudaStream_t s) {
  size_t tmp = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)n, s);
  if (e) return e;
  void* t = nullptr;
  e = cudaMallocAsync(&t, tmp ? tmp : 1, s);
  if (e) return e;
  e = cub::DeviceScan::ExclusiveSum(t, tmp, in, out, (int)n, s);
  cudaFreeAsync(t, s);
  return e;
}

}  // namespace

void launch_normal_map(const double* W, int w, int h, const M3& Km, double* nx, double* ny,
                       double* nz, cudaStream_t s) {
  KScope ks_("normal_map", s);
  k_normal_map<<<blocks((long long)w * h, 256), 256, 0, s>>>(W, w, h, Km, nx, ny, nz);
}

int export_map_device(const ExportKF* kfs, int n_kf, int w, int h, const M3& Kinv, double voxel,
                      cudaStream_t s, double** d_points, uint8_t** d_colors, long long* count) {
  const long long N = (long long)w * h, T = N * n_kf;
  AsyncPool pool(s);
  int *flag = nullptr, *pos = nullptr;
  double* pts = nullptr;
  uint8_t* col = nullptr;
  cudaError_t e;
#define EX_CK(x)        \
  do {                  \
    e = (x);            \
    if (e) return (int)e; \
  } while (0)
  EX_CK(pool.alloc(&flag, T));
  EX_CK(pool.alloc(&pos, T));
  EX_CK(pool.alloc(&pts, 3 * T));
  EX_CK(pool.alloc(&col, 3 * T));
  for (int k = 0; k < n_kf; ++k) {
    KScope ks_("export_points", s);
    k_export_points<<<blocks(N, 256), 256, 0, s>>>(kfs[k], w, h, Kinv, flag + k * N,
                                                    pts + 3 * k * N, col + 3 * k * N);
  }
  EX_CK(cudaGetLastError());
  EX_CK(exclusive_sum(flag, pos, T, s));
  int last_pos = 0, last_flag = 0;
  EX_CK(cudaMemcpyAsync(&last_pos, pos + T - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  EX_CK(cudaMemcpyAsync(&last_flag, flag + T - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  EX_CK(cudaStreamSynchronize(s));
  const long long n = (long long)last_pos + last_flag;
  double* cpts = nullptr;
  uint8_t* ccol = nullptr;
  EX_CK(pool.alloc(&cpts, 3 * n));
  EX_CK(pool.alloc(&ccol, 3 * n));
  {
    KScope ks_("export_compact", s);
    k_compact<<<blocks(T, 256), 256, 0, s>>>(flag, pos, T, pts, col, cpts, ccol);
  }
  EX_CK(cudaGetLastError());
  if (voxel <= 0.0 || n == 0) {
    pool.release(cpts);
    pool.release(ccol);
    *d_points = cpts;
    *d_colors = ccol;
    *count = n;
    return 0;
  }
  // voxel filter — src/pipeline.cpp:502-527
  unsigned long long *key = nullptr, *skey = nullptr;
  int *idx = nullptr, *sidx = nullptr, *head = nullptr, *first = nullptr, *opos = nullptr;
  EX_CK(pool.alloc(&key, n));
  EX_CK(pool.alloc(&skey, n));
  EX_CK(pool.alloc(&idx, n));
  EX_CK(pool.alloc(&sidx, n));
  EX_CK(pool.alloc(&head, n));
  EX_CK(pool.alloc(&first, n));
  EX_CK(pool.alloc(&opos, n));
  EX_CK(cudaMemsetAsync(first, 0, sizeof(int) * n, s));
  {
    KScope ks_("voxel_keys", s);
    k_voxel_keys<<<blocks(n, 256), 256, 0, s>>>(cpts, n, voxel, key, idx);
  }
  size_t tmp = 0;
  EX_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, skey, idx, sidx, (int)n, 0, 64, s));
  void* t = nullptr;
  EX_CK(pool.alloc(reinterpret_cast<char**>(&t), tmp));
  EX_CK(cub::DeviceRadixSort::SortPairs(t, tmp, key, skey, idx, sidx, (int)n, 0, 64, s));  // stable
  {
    KScope ks_("voxel_heads", s);
    k_voxel_heads<<<blocks(n, 256), 256, 0, s>>>(skey, sidx, n, head, first);
  }
  EX_CK(cudaGetLastError());
  EX_CK(exclusive_sum(first, opos, n, s));
  int lp = 0, lf = 0;
  EX_CK(cudaMemcpyAsync(&lp, opos + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  EX_CK(cudaMemcpyAsync(&lf, first + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  EX_CK(cudaStreamSynchronize(s));
  const long long nv = (long long)lp + lf;
  double* vpts = nullptr;
  uint8_t* vcol = nullptr;
  EX_CK(pool.alloc(&vpts, 3 * nv));
  EX_CK(pool.alloc(&vcol, 3 * nv));
  {
    KScope ks_("voxel_average", s);
    k_voxel_average<<<blocks(n, 256), 256, 0, s>>>(skey, sidx, head, opos, n, cpts, ccol, vpts,
                                                   vcol);
  }
  EX_CK(cudaGetLastError());
  pool.release(vpts);
  pool.release(vcol);
#undef EX_CK
  *d_points = vpts;
  *d_colors = vcol;
  *count = nv;
  return 0;
}

}  // namespace rgbid_b200
