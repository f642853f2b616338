/*
 * rgbid_oracle.h — CPU restatement of the RGBiD-SLAM front-end hot path.
 *
 * TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg as the checker; never linked into the product.
 * Parity pinned: tests/test_oracle_cpu.py checks every or_* function
 * bit-for-bit against the unmodified reference built in oracle/_ref/ (whose
 * own unit tests pass, oracle/_ref/ref_hotpath_tests).
 *
 * Uses the POD types of include/rgbid_b200.h (the C-ABI layout) only.
 */
#ifndef RGBID_ORACLE_H
#define RGBID_ORACLE_H
#include "rgbid_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

void or_downsample2(const double* in, int w, int h, double* out);
int or_build_pyramid(const double* I, const double* W, int w, int h, const rgbid_intrinsics* K,
                     int levels, double** out_I, double** out_W, rgbid_intrinsics* K_out);
int or_inverse_geometric_warp(const double* I_B, const double* W_B, int wb, int hb,
                              const double* W_A, int w, int h, const rgbid_pose* T_AB,
                              const rgbid_intrinsics* K, double* oI, double* oW, double* omx,
                              double* omy);
long long or_residuals_and_jacobians(const double* I_A, const double* W_A, const double* I_Bw,
                                     const double* W_Bw, int w, int h, const rgbid_intrinsics* K,
                                     double lambda_n_min, double* jets, unsigned char* flags,
                                     long long cap);
double or_t_weight(double x, double nu);
double or_digamma(double x);
void or_estimate_location_scale(const double* r, long long n, double nu, rgbid_tdist* out);
double or_estimate_nu(const double* r, long long n, double mu, double sigma);
int or_align(const double* IA, const double* WA, const double* IB, const double* WB, int w, int h,
             const rgbid_intrinsics* K, const rgbid_pose* init, const rgbid_align_config* cfg,
             rgbid_align_result* out, rgbid_iter_trace* trace, int max_trace, int* n_trace);
int or_align_many(int n, const double* const* IA, const double* const* WA,
                  const double* const* IB, const double* const* WB, int w, int h,
                  const rgbid_intrinsics* K, const rgbid_pose* inits,
                  const rgbid_align_config* cfg, rgbid_align_result* out, int threads);
int or_filtered_hessian_covariance(const double* IA, const double* WA, const double* IB,
                                   const double* WB, int w, int h, const rgbid_intrinsics* K,
                                   const rgbid_pose* T, const rgbid_align_config* cfg,
                                   double* cov36, int* degenerate);
int or_bilateral_filter(const double* img, int w, int h, double ss, double sr, double* out);
int or_integrate_frame(double* kf_W, double* kf_C, const double* fI, const double* fW, int w,
                       int h, const rgbid_pose* T, const rgbid_intrinsics* K, double sigma_w);
int or_covisibility_ratio(const double* WA, const double* WB, int w, int h,
                          const rgbid_pose* T_BA, const rgbid_intrinsics* K, double sigma_w,
                          double* ratio, int* empty, long long counts[4]);
int or_correct_inverse_depth(const double* Wm, int w, int h, const rgbid_depth_intrinsics* d,
                             const rgbid_intrinsics* K, int spatial, double* out);
int or_forward_register(const double* WA, int w, int h, const rgbid_pose* T_BA,
                        const rgbid_intrinsics* KA, const rgbid_intrinsics* KB, double* out);
int or_pose_update(const double xi[6], const rgbid_pose* T, rgbid_pose* out);
int or_pose_inverse(const rgbid_pose* a, rgbid_pose* out);
int or_pose_compose(const rgbid_pose* a, const rgbid_pose* b, rgbid_pose* out);
int or_mat3_inverse(const double m[9], double out[9]);
int or_decode_frame(const unsigned char* bgr, const unsigned short* depth, int w, int h,
                    double scale, double* I, double* W);

#ifdef __cplusplus
}
#endif
#endif
