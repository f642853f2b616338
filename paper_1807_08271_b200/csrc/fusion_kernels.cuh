// Fusion / covisibility / registration / synthetic-input kernels (fusion_kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "hd_math.cuh"
#include "synth_scene.cuh"

namespace rgbid_b200 {

struct FuseFrame {  // one frame of integrate_frame: its W map + warp matrices of T_kf_frame
  const double* W;
  WarpMats wm;
};

struct CovisDir {  // one direction of count_visible
  const double* WA;
  const double* WB;
  double Rt[9], tt[3];
};

struct RegisterMats {  // forward_register host-side setup (src/warping.cpp:22-25)
  double Rt_AB[9];
  double tt[3];
};


void launch_integrate(const FuseFrame* frames_dev, int k, double* kfW, double* kfC, int w, int h,
                      double sigma_w, cudaStream_t s);
void launch_covisibility(const CovisDir& d0, const CovisDir& d1, int w, int h, double sigma_w,
                         unsigned long long* counts_dev, cudaStream_t s);
void launch_correct_depth(const double* Wm, int w, int h, const rgbid_depth_intrinsics& d,
                          const rgbid_intrinsics& K, int spatial, double* out, cudaStream_t s);
void launch_forward_register(const double* WA, int w, int h, const RegisterMats& r,
                             unsigned long long* inter, int iw, int ih, int wb, int hb,
                             double* out, cudaStream_t s);
void launch_render(const SynthView& v, double* I, double* W, cudaStream_t s);
void launch_rectify(const double* I, const double* W, int w, int h, const rgbid_intrinsics& K,
                    double* oI, double* oW, cudaStream_t s);
void launch_undistort(const double* md, long long n, const rgbid_intrinsics& K, double* mu,
                      uint8_t* ok, cudaStream_t s);
void launch_decode_frame(const uint8_t* bgr, const uint16_t* depth, int n, double scale, double* I,
                         double* W, cudaStream_t s);

}  // namespace rgbid_b200
