"""ctypes mirror of include/rgbid_b200.h (the C-ABI boundary).

Loads the in-tree CUDA library ``_lib/librgbid_b200.so``.  There is no CPU
fallback: if the library is missing, :func:`lib` raises ``RuntimeError`` and
every entry point of :mod:`paper_1807_08271_b200.rgbid` fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

MAX_LEVELS = 8
OK, E_DEGENERATE, E_CUDA, E_ARG, E_OOM = 0, 1, 2, 3, 4

_HERE = os.path.dirname(os.path.abspath(__file__))
# RGBID_LIB: an alternative in-tree build (kernel variants under build/, tools/ only)
LIB_PATH = os.environ.get("RGBID_LIB") or os.path.join(_HERE, "_lib", "librgbid_b200.so")


class Intrinsics_t(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("k", C.c_double * 5), ("width", C.c_int), ("height", C.c_int)]


class Pose_t(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3)]


class AlignConfig_t(C.Structure):
    _fields_ = [("levels", C.c_int), ("n_iterations", C.c_int),
                ("iterations", C.c_int * MAX_LEVELS), ("convergence_eps", C.c_double),
                ("lambda_n_min", C.c_double), ("bilateral_sigma_space", C.c_double),
                ("bilateral_sigma_intensity", C.c_double), ("bilateral_sigma_depth", C.c_double)]


class TDist_t(C.Structure):
    _fields_ = [("mu", C.c_double), ("sigma", C.c_double), ("nu", C.c_double)]


class LevelLog_t(C.Structure):
    _fields_ = [("level", C.c_int), ("iterations", C.c_int), ("final_cost", C.c_double)]


class AlignResult_t(C.Structure):
    _fields_ = [("T_AB", Pose_t), ("cov", C.c_double * 36), ("converged", C.c_int),
                ("cov_degenerate", C.c_int), ("n_levels", C.c_int),
                ("level_log", LevelLog_t * MAX_LEVELS), ("tdist_intensity", TDist_t),
                ("tdist_depth", TDist_t), ("spectrum", C.c_double * 6), ("status", C.c_int),
                ("total_iterations", C.c_int)]


class IterTrace_t(C.Structure):
    _fields_ = [("level", C.c_int), ("iter", C.c_int), ("n_jets", C.c_longlong),
                ("n_depth", C.c_longlong), ("tI", TDist_t), ("tW", TDist_t),
                ("H", C.c_double * 36), ("b", C.c_double * 6), ("cost", C.c_double),
                ("xi", C.c_double * 6), ("T_after", Pose_t)]


class DepthIntrinsics_t(C.Structure):
    _fields_ = [("beta0", C.c_double), ("beta1", C.c_double), ("q0", C.c_double * 9),
                ("q1", C.c_double * 9), ("p0", C.c_double * 2)]


class FrontendConfig_t(C.Structure):
    _fields_ = [("align", AlignConfig_t), ("keyframe_covisibility", C.c_double),
                ("reference_covisibility", C.c_double), ("buffer_capacity", C.c_int)]


class FrameEstimate_t(C.Structure):
    _fields_ = [("timestamp", C.c_double), ("T_W_k", Pose_t), ("cov", C.c_double * 36),
                ("lost", C.c_int), ("keyframe_id", C.c_int)]


class LoopConstraint_t(C.Structure):
    _fields_ = [("i", C.c_int), ("j", C.c_int), ("T_ij", Pose_t), ("info", C.c_double * 36),
                ("inliers", C.c_int), ("hull_fraction", C.c_double), ("score", C.c_double)]


DP = C.POINTER(C.c_double)
VP = C.c_void_p


def dptr(a):
    """double* of a C-contiguous float64 numpy array (or None)."""
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], "need C-contiguous float64"
    return a.ctypes.data_as(DP)


def dptr_array(arrs):
    """double** from a list of float64 arrays."""
    return (DP * len(arrs))(*[dptr(a) for a in arrs])


# (name, restype, argtypes) of every exported symbol of include/rgbid_b200.h
EXPORTS = [
    ("rgbid_version", C.c_char_p, []),
    ("rgbid_status_string", C.c_char_p, [C.c_int]),
    ("rgbid_ctx_create", C.c_int, [C.c_int, C.POINTER(VP)]),
    ("rgbid_ctx_destroy", C.c_int, [VP]),
    ("rgbid_ctx_last_error", C.c_char_p, [VP]),
    ("rgbid_ctx_kernel_launches", C.c_longlong, [VP]),
    ("rgbid_ctx_synchronize", C.c_int, [VP]),
    ("rgbid_ctx_stream", VP, [VP]),
    ("rgbid_ctx_set_profiling", C.c_int, [VP, C.c_int]),
    ("rgbid_ctx_reset_stats", C.c_int, [VP]),
    ("rgbid_ctx_kernel_stats", C.c_int, [VP, C.c_char_p, C.c_int]),
    ("rgbid_ctx_transfer_bytes", C.c_int, [VP, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
    ("rgbid_frame_create", C.c_int, [VP, C.c_int, C.c_int, C.POINTER(VP)]),
    ("rgbid_frame_upload", C.c_int, [VP, VP, DP, DP]),
    ("rgbid_frame_download", C.c_int, [VP, VP, DP, DP]),
    ("rgbid_frame_device_ptrs", C.c_int, [VP, C.POINTER(DP), C.POINTER(DP)]),
    ("rgbid_frame_destroy", C.c_int, [VP, VP]),
    ("rgbid_frame_decode", C.c_int, [VP, VP, C.c_void_p, C.c_void_p, C.c_double]),
    ("rgbid_frame_invalidate", C.c_int, [VP]),
    ("rgbid_build_pyramid", C.c_int, [VP, DP, DP, C.c_int, C.c_int, C.POINTER(Intrinsics_t),
                                      C.c_int, C.POINTER(DP), C.POINTER(DP),
                                      C.POINTER(Intrinsics_t)]),
    ("rgbid_inverse_geometric_warp", C.c_int, [VP, DP, DP, C.c_int, C.c_int, DP, C.c_int, C.c_int,
                                               C.POINTER(Pose_t), C.POINTER(Intrinsics_t),
                                               DP, DP, DP, DP]),
    ("rgbid_align", C.c_int, [VP, VP, VP, C.POINTER(Intrinsics_t), C.POINTER(Pose_t),
                              C.POINTER(AlignConfig_t), C.POINTER(AlignResult_t)]),
    ("rgbid_align_host", C.c_int, [VP, DP, DP, DP, DP, C.c_int, C.c_int,
                                   C.POINTER(Intrinsics_t), C.POINTER(Pose_t),
                                   C.POINTER(AlignConfig_t), C.POINTER(AlignResult_t)]),
    ("rgbid_last_align_trace", C.c_int, [VP, C.POINTER(IterTrace_t), C.c_int,
                                         C.POINTER(C.c_int)]),
    ("rgbid_batch_plan", C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("rgbid_rectify_frame", C.c_int, [VP, VP, C.POINTER(Intrinsics_t), VP]),
    ("rgbid_rectify", C.c_int, [VP, DP, C.c_int, C.c_int, C.POINTER(Intrinsics_t), DP]),
    ("rgbid_undistort_points", C.c_int, [VP, DP, C.c_longlong, C.POINTER(Intrinsics_t), DP,
                                         C.POINTER(C.c_ubyte)]),
    ("rgbid_align_batch", C.c_int, [VP, C.c_int, C.POINTER(VP), C.POINTER(VP),
                                    C.POINTER(Intrinsics_t), C.POINTER(Pose_t),
                                    C.POINTER(AlignConfig_t), C.POINTER(AlignResult_t)]),
    ("rgbid_align_batch_host", C.c_int, [VP, C.c_int, C.POINTER(DP), C.POINTER(DP),
                                         C.POINTER(DP), C.POINTER(DP), C.c_int, C.c_int,
                                         C.POINTER(Intrinsics_t), C.POINTER(Pose_t),
                                         C.POINTER(AlignConfig_t), C.c_int,
                                         C.POINTER(AlignResult_t)]),
    ("rgbid_align_batch_host_async", C.c_int, [VP, C.c_int, C.POINTER(DP), C.POINTER(DP),
                                               C.POINTER(DP), C.POINTER(DP), C.c_int, C.c_int,
                                               C.POINTER(Intrinsics_t), C.POINTER(Pose_t),
                                               C.POINTER(AlignConfig_t), C.c_int,
                                               C.POINTER(AlignResult_t)]),
    ("rgbid_align_batch_host_wait", C.c_int, [VP]),
    ("rgbid_filtered_hessian_covariance", C.c_int, [VP, VP, VP, C.POINTER(Intrinsics_t),
                                                    C.POINTER(Pose_t), C.POINTER(AlignConfig_t),
                                                    DP, C.POINTER(C.c_int)]),
    ("rgbid_bilateral_filter", C.c_int, [VP, DP, C.c_int, C.c_int, C.c_double, C.c_double, DP]),
    ("rgbid_integrate_frame", C.c_int, [VP, DP, DP, DP, DP, C.c_int, C.c_int, C.POINTER(Pose_t),
                                        C.POINTER(Intrinsics_t), C.c_double]),
    ("rgbid_integrate_frames", C.c_int, [VP, VP, DP, C.c_int, C.POINTER(VP), C.POINTER(Pose_t),
                                         C.POINTER(Intrinsics_t), C.c_double]),
    ("rgbid_covisibility_ratio", C.c_int, [VP, VP, VP, C.POINTER(Pose_t),
                                           C.POINTER(Intrinsics_t), C.c_double, DP,
                                           C.POINTER(C.c_int), C.POINTER(C.c_longlong)]),
    ("rgbid_correct_inverse_depth", C.c_int, [VP, DP, C.c_int, C.c_int,
                                              C.POINTER(DepthIntrinsics_t),
                                              C.POINTER(Intrinsics_t), C.c_int, DP]),
    ("rgbid_forward_register", C.c_int, [VP, DP, C.c_int, C.c_int, C.POINTER(Pose_t),
                                         C.POINTER(Intrinsics_t), C.POINTER(Intrinsics_t), DP]),
    ("rgbid_frontend_default_config", C.c_int, [C.POINTER(FrontendConfig_t)]),
    ("rgbid_frontend_create", C.c_int, [VP, C.POINTER(Intrinsics_t), C.POINTER(FrontendConfig_t),
                                        C.POINTER(VP)]),
    ("rgbid_frontend_destroy", C.c_int, [VP]),
    ("rgbid_frontend_process", C.c_int, [VP, DP, DP, C.c_double, C.POINTER(FrameEstimate_t)]),
    ("rgbid_frontend_finish", C.c_int, [VP]),
    ("rgbid_frontend_trajectory", C.c_int, [VP, C.POINTER(FrameEstimate_t), C.c_int,
                                            C.POINTER(C.c_int)]),
    ("rgbid_frontend_keyframes", C.c_int, [VP, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int)]),
    ("rgbid_frontend_current_keyframe", C.c_int, [VP, DP, DP, C.POINTER(Pose_t),
                                                  C.POINTER(C.c_int)]),
    ("rgbid_frame_copy", C.c_int, [VP, VP, VP]),
    ("rgbid_fill", C.c_int, [VP, DP, C.c_longlong, C.c_double]),
    ("rgbid_remap_bilinear", C.c_int, [VP, DP, C.c_int, C.c_int, DP, DP, C.c_int, C.c_int, DP]),
    ("rgbid_residuals_and_jacobians", C.c_longlong, [VP, DP, DP, DP, DP, C.c_int, C.c_int,
                                                     C.POINTER(Intrinsics_t), C.c_double, DP,
                                                     C.POINTER(C.c_ubyte), C.c_longlong]),
    ("rgbid_estimate_location_scale", C.c_int, [VP, DP, C.c_longlong, C.c_double,
                                                C.POINTER(TDist_t)]),
    ("rgbid_estimate_nu", C.c_int, [VP, DP, C.c_longlong, C.c_double, C.c_double,
                                    C.POINTER(C.c_double)]),
    ("rgbid_selftest_division", C.c_int, [VP, C.c_ulonglong, C.c_ulonglong,
                                          C.POINTER(C.c_ulonglong)]),
    ("rgbid_measure_fp64_peak", C.c_int, [VP, C.POINTER(C.c_double)]),
    ("rgbid_make_loop_constraint", C.c_int, [VP, VP, VP, C.c_int, C.c_int,
                                             C.POINTER(Intrinsics_t), C.POINTER(Pose_t),
                                             C.POINTER(AlignConfig_t), C.c_double, C.c_int,
                                             C.c_double, C.POINTER(LoopConstraint_t),
                                             C.POINTER(C.c_int)]),
    ("rgbid_normal_map", C.c_int, [VP, DP, C.c_int, C.c_int, C.POINTER(Intrinsics_t), DP, DP,
                                   DP]),
    ("rgbid_export_map", C.c_int, [VP, C.c_int, C.POINTER(DP), C.POINTER(DP), C.c_int, C.c_int,
                                   C.POINTER(Pose_t), C.POINTER(Intrinsics_t), C.c_double, DP,
                                   C.POINTER(C.c_ubyte), C.c_longlong,
                                   C.POINTER(C.c_longlong)]),
    ("rgbid_synth_render_plane", C.c_int, [C.POINTER(Intrinsics_t), C.POINTER(Pose_t), DP,
                                           C.c_double, C.c_double, DP, DP]),
    ("rgbid_synth_random_pose", C.c_int, [C.c_uint32, C.c_int, C.c_double, C.c_double,
                                          C.POINTER(Pose_t)]),
    ("rgbid_synth_add_noise", C.c_int, [DP, DP, C.c_int, C.c_int, C.c_uint32, C.c_double,
                                        C.c_double]),
    ("rgbid_synth_pair_device", C.c_int, [VP, VP, VP, C.POINTER(Intrinsics_t), C.c_uint32,
                                          C.c_int, C.POINTER(Pose_t)]),
    ("rgbid_synth_pair_host", C.c_int, [C.POINTER(Intrinsics_t), C.c_uint32, C.c_int, DP, DP,
                                        DP, DP, C.POINTER(Pose_t)]),
]

_lib = None


def lib():
    """The loaded CUDA library.  Raises if it was not built (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the B200 path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in EXPORTS:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
