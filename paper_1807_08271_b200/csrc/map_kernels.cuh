// Normal map and map export kernels (map_kernels.cu) — SURVEY 8(f) rank 4.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "hd_math.cuh"

namespace rgbid_b200 {

// One keyframe of export_map: its maps, pose, and (k > 0) the transfer into the
// previous keyframe, Rt = K R_prev_kf K^-1, tt = K t_prev_kf (src/pipeline.cpp:472-477).
struct ExportKF {
  const double* I;
  const double* W;
  const double* W_prev;  // nullptr for the first keyframe
  PoseD T_W_kf;
  M3 Rt;
  V3 tt;
};

void launch_normal_map(const double* W, int w, int h, const M3& Km, double* nx, double* ny,
                       double* nz, cudaStream_t s);

// export_map on device: per-keyframe point extraction, ordered compaction and
// (voxel > 0) the first-occurrence-ordered voxel average.  Temporaries come from
// the stream-ordered allocator.  Results are left in device buffers owned by the
// caller-supplied pointers (allocated here with cudaMallocAsync on s; the caller
// frees them).  Returns a cudaError_t.
int export_map_device(const ExportKF* kfs, int n_kf, int w, int h, const M3& Kinv, double voxel,
                      cudaStream_t s, double** d_points, uint8_t** d_colors, long long* count);

}  // namespace rgbid_b200
