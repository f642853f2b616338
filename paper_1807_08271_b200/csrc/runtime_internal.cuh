// Stream-ordered building blocks of the C-ABI entry points, for the front-end
// driver (frontend.cu): the same kernels and host setup as rgbid_frame_upload /
// rgbid_covisibility_ratio / rgbid_integrate_frames, without their host waits, so
// a front-end frame costs one cudaMalloc-free upload and two host syncs.
#pragma once
#include "../../include/rgbid_b200.h"

namespace rgbid_b200 {

// H2D of a frame's maps on the ctx stream (pageable sources are staged before
// return); invalidates the cached pyramid.  No host wait.
int rt_frame_upload_async(rgbid_ctx* ctx, rgbid_frame* f, const double* I, const double* W);
// count_visible in both directions into counts_dev[0..3] (valid_ab, visible_ab, valid_ba,
// visible_ba) on the ctx stream.  No host wait.
int rt_covis_enqueue(rgbid_ctx* ctx, const rgbid_frame* a, const rgbid_frame* b,
                     const rgbid_pose* T_BA, const rgbid_intrinsics* K, double sigma_w,
                     unsigned long long* counts_dev);
// covisibility_ratio from the four counts — src/fusion.cpp:56-66
void rt_covis_ratio(const unsigned long long* counts, double* ratio, int* empty);
// k integrate_frame calls fused in one launch on the ctx stream.  No host wait.
int rt_integrate_async(rgbid_ctx* ctx, rgbid_frame* kf, double* kf_C_dev, int k,
                       const rgbid_frame* const* frames, const rgbid_pose* T,
                       const rgbid_intrinsics* K, double sigma_w);

}  // namespace rgbid_b200
