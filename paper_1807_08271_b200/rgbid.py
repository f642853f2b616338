"""Python mirror of the reference's front-end API (namespace ``rgbid``), backed by
the CUDA library through the C-ABI (include/rgbid_b200.h).

Names, argument meaning and error behaviour follow the reference headers:
``inc/alignment.hpp`` (align, build_pyramid, filtered_hessian_covariance,
bilateral_filter, DegenerateAlignmentError), ``inc/warping.hpp``
(inverse_geometric_warp, forward_register), ``inc/fusion.hpp`` (make_keyframe,
covisibility_ratio, integrate_frame, FrameBuffer, drain_buffer_step) and
``inc/camera.hpp`` (Intrinsics, DepthIntrinsics, correct_inverse_depth).
Images are float64 numpy arrays (row-major, NaN holes).  Every compute call
runs on the GPU; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import abi
from .abi import dptr

# --------------------------------------------------------------------------- types


@dataclass
class Intrinsics:
    """inc/camera.hpp:16-41"""
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    k: tuple = (0.0, 0.0, 0.0, 0.0, 0.0)
    width: int = 0
    height: int = 0

    def K(self) -> np.ndarray:
        return np.array([[self.fx, 0, self.cx], [0, self.fy, self.cy], [0, 0, 1.0]])

    def scaled(self, s: float) -> "Intrinsics":
        return Intrinsics(self.fx * s, self.fy * s, self.cx * s, self.cy * s, tuple(self.k),
                          int(self.width * s), int(self.height * s))

    def to_c(self) -> abi.Intrinsics_t:
        c = abi.Intrinsics_t()
        c.fx, c.fy, c.cx, c.cy = self.fx, self.fy, self.cx, self.cy
        for i in range(5):
            c.k[i] = self.k[i]
        c.width, c.height = int(self.width), int(self.height)
        return c

    @staticmethod
    def from_c(c) -> "Intrinsics":
        return Intrinsics(c.fx, c.fy, c.cx, c.cy, tuple(c.k), c.width, c.height)


def simple_intrinsics(w: int = 80, h: int = 60, f: float = 60.0) -> Intrinsics:
    """tests/synthetic.hpp:13-21"""
    return Intrinsics(f, f, (w - 1) / 2.0, (h - 1) / 2.0, (0.0,) * 5, w, h)


class Pose:
    """inc/geometry.hpp:22-39: X_A = R X_B + t."""

    __slots__ = ("R", "t")

    def __init__(self, R=None, t=None):
        self.R = np.eye(3) if R is None else np.array(R, dtype=np.float64).reshape(3, 3)
        self.t = np.zeros(3) if t is None else np.array(t, dtype=np.float64).reshape(3)

    def __mul__(self, o):
        if isinstance(o, Pose):
            return Pose(self.R @ o.R, self.R @ o.t + self.t)
        return self.R @ np.asarray(o, dtype=np.float64) + self.t

    def inverse(self) -> "Pose":
        return Pose(self.R.T, -(self.R.T @ self.t))

    def matrix(self) -> np.ndarray:
        m = np.eye(4)
        m[:3, :3] = self.R
        m[:3, 3] = self.t
        return m

    def to_c(self) -> abi.Pose_t:
        c = abi.Pose_t()
        for i in range(9):
            c.R[i] = float(self.R.reshape(9)[i])
        for i in range(3):
            c.t[i] = float(self.t[i])
        return c

    @staticmethod
    def from_c(c) -> "Pose":
        return Pose(np.array(c.R[:]).reshape(3, 3), np.array(c.t[:]))

    def __repr__(self):
        return f"Pose(R={self.R.tolist()}, t={self.t.tolist()})"


def so3_exp(theta) -> np.ndarray:
    """src/geometry.cpp:15-28 (host-side helper)."""
    th = np.asarray(theta, dtype=np.float64)
    angle = float(np.sqrt(th @ th))
    K = np.array([[0, -th[2], th[1]], [th[2], 0, -th[0]], [-th[1], th[0], 0]])
    if angle < 1e-4:
        a, b = 1.0 - angle * angle / 6.0, 0.5 - angle * angle / 24.0
    else:
        a, b = np.sin(angle) / angle, (1.0 - np.cos(angle)) / (angle * angle)
    return np.eye(3) + a * K + b * K @ K


def so3_log(R) -> np.ndarray:
    """src/geometry.cpp:30-54 (host-side helper for tests)."""
    R = np.asarray(R)
    c = min(1.0, max(-1.0, (np.trace(R) - 1.0) / 2.0))
    angle = np.arccos(c)
    w = np.array([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]])
    if angle < 1e-4:
        return w / 2.0
    if np.pi - angle < 1e-6:
        A = (R + np.eye(3)) / 2.0
        k = int(np.argmax(np.diag(A)))
        axis = A[:, k] / np.sqrt(A[k, k])
        axis /= np.linalg.norm(axis)
        if axis @ w < 0:
            axis = -axis
        return angle * axis
    return angle * w / np.linalg.norm(w)


def se3_exp(xi) -> Pose:
    """Decoupled SE(3) exp, src/geometry.cpp:56."""
    xi = np.asarray(xi, dtype=np.float64)
    return Pose(so3_exp(xi[3:]), xi[:3])


@dataclass
class FrameData:
    """inc/alignment.hpp:14-18"""
    intensity: np.ndarray
    inverse_depth: np.ndarray

    def __post_init__(self):
        self.intensity = np.ascontiguousarray(self.intensity, dtype=np.float64)
        self.inverse_depth = np.ascontiguousarray(self.inverse_depth, dtype=np.float64)

    @property
    def width(self) -> int:
        return self.inverse_depth.shape[1]

    @property
    def height(self) -> int:
        return self.inverse_depth.shape[0]

    def copy(self) -> "FrameData":
        return FrameData(self.intensity.copy(), self.inverse_depth.copy())


@dataclass
class Pyramid:
    levels: List[FrameData]
    intrinsics: List[Intrinsics]


@dataclass
class TDistParams:
    mu: float = 0.0
    sigma: float = 1.0
    nu: float = 5.0


@dataclass
class LevelLog:
    level: int = 0
    iterations: int = 0
    final_cost: float = 0.0


@dataclass
class AlignmentConfig:
    """inc/alignment.hpp:88-96"""
    levels: int = 3
    iterations: List[int] = field(default_factory=lambda: [10, 5, 4])
    convergence_eps: float = 1e-6
    lambda_n_min: float = 0.1
    bilateral_sigma_space: float = 2.0
    bilateral_sigma_intensity: float = 0.05
    bilateral_sigma_depth: float = 0.02

    def to_c(self) -> abi.AlignConfig_t:
        c = abi.AlignConfig_t()
        c.levels = self.levels
        c.n_iterations = len(self.iterations)
        for i, v in enumerate(self.iterations[: abi.MAX_LEVELS]):
            c.iterations[i] = int(v)
        c.convergence_eps = self.convergence_eps
        c.lambda_n_min = self.lambda_n_min
        c.bilateral_sigma_space = self.bilateral_sigma_space
        c.bilateral_sigma_intensity = self.bilateral_sigma_intensity
        c.bilateral_sigma_depth = self.bilateral_sigma_depth
        return c


@dataclass
class AlignmentResult:
    """inc/alignment.hpp:72-80"""
    T_AB: Pose
    cov: np.ndarray
    converged: bool
    cov_degenerate: bool
    level_log: List[LevelLog]
    tdist_intensity: TDistParams
    tdist_depth: TDistParams
    total_iterations: int = 0

    @staticmethod
    def from_c(r) -> "AlignmentResult":
        return AlignmentResult(
            Pose.from_c(r.T_AB), np.array(r.cov[:]).reshape(6, 6), bool(r.converged),
            bool(r.cov_degenerate),
            [LevelLog(l.level, l.iterations, l.final_cost) for l in r.level_log[: r.n_levels]],
            TDistParams(r.tdist_intensity.mu, r.tdist_intensity.sigma, r.tdist_intensity.nu),
            TDistParams(r.tdist_depth.mu, r.tdist_depth.sigma, r.tdist_depth.nu),
            r.total_iterations)


class DegenerateAlignmentError(RuntimeError):
    """inc/alignment.hpp:82-86"""

    def __init__(self, spectrum):
        super().__init__("degenerate alignment: under-constrained scene")
        self.spectrum = np.asarray(spectrum, dtype=np.float64)


class CudaError(RuntimeError):
    pass


def digamma(x: float) -> float:
    """src/alignment.cpp:32-43 (host scalar helper, as in the reference)."""
    import math
    result = 0.0
    while x < 6.0:
        result -= 1.0 / x
        x += 1.0
    inv = 1.0 / x
    inv2 = inv * inv
    return result + (math.log(x) - 0.5 * inv
                     - inv2 * (1.0 / 12.0 - inv2 * (1.0 / 120.0 - inv2 / 252.0)))


def t_weight(x: float, nu: float) -> float:
    """inc/alignment.hpp:35"""
    return (nu + 1.0) / (nu + x * x)


# --------------------------------------------------------------------------- context


class Context:
    """One rgbid_ctx (CUDA stream + workspaces) — one per host thread, like the
    reference's two-thread front-end/back-end model."""

    def __init__(self, device: int = 0):
        self.lib = abi.lib()
        self.h = C.c_void_p()
        rc = self.lib.rgbid_ctx_create(device, C.byref(self.h))
        if rc != abi.OK:
            raise CudaError(f"rgbid_ctx_create(device={device}) failed: "
                            f"{self.lib.rgbid_status_string(rc).decode()} (a B200 / sm_100 GPU is required)")
        self.device = device

    def check(self, rc: int, what: str):
        if rc == abi.OK:
            return
        msg = self.lib.rgbid_ctx_last_error(self.h).decode()
        if rc == abi.E_ARG:
            raise ValueError(f"{what}: invalid argument")
        raise CudaError(f"{what}: {self.lib.rgbid_status_string(rc).decode()} {msg}")

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.rgbid_ctx_kernel_launches(self.h))

    def set_profiling(self, enable: bool):
        self.check(self.lib.rgbid_ctx_set_profiling(self.h, int(enable)), "set_profiling")

    def reset_stats(self):
        self.check(self.lib.rgbid_ctx_reset_stats(self.h), "reset_stats")

    def kernel_stats(self) -> dict:
        import json
        n = self.lib.rgbid_ctx_kernel_stats(self.h, None, 0)
        buf = C.create_string_buffer(n)
        self.lib.rgbid_ctx_kernel_stats(self.h, buf, n)
        return {k: (int(v[0]), float(v[1])) for k, v in json.loads(buf.value.decode()).items()}

    def transfer_bytes(self):
        a, b = C.c_longlong(0), C.c_longlong(0)
        self.lib.rgbid_ctx_transfer_bytes(self.h, C.byref(a), C.byref(b))
        return a.value, b.value

    @property
    def stream_ptr(self) -> int:
        return int(self.lib.rgbid_ctx_stream(self.h) or 0)

    def synchronize(self):
        self.check(self.lib.rgbid_ctx_synchronize(self.h), "synchronize")

    def close(self):
        if self.h:
            self.lib.rgbid_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()


def default_context() -> Context:
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context(0)
        _tls.ctx = ctx
    return ctx


class DeviceFrame:
    """A FrameData resident in HBM (rgbid_frame); its pyramid is cached."""

    def __init__(self, width: int, height: int, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.h = C.c_void_p()
        self.width, self.height = width, height
        self.ctx.check(self.ctx.lib.rgbid_frame_create(self.ctx.h, width, height, C.byref(self.h)),
                       "frame_create")

    @staticmethod
    def from_frame(f: FrameData, ctx: Optional[Context] = None) -> "DeviceFrame":
        d = DeviceFrame(f.width, f.height, ctx)
        d.upload(f)
        return d

    def upload(self, f: FrameData):
        self.ctx.check(self.ctx.lib.rgbid_frame_upload(self.ctx.h, self.h, dptr(f.intensity),
                                                       dptr(f.inverse_depth)), "frame_upload")

    def decode(self, bgr: Optional[np.ndarray], depth: np.ndarray, scale: float = 5000.0):
        """load_frame's pixel decode (src/dataset.cpp:97-116) on the GPU: BGR8 (h, w, 3)
        and 16-bit depth (h, w) -> intensity / inverse depth."""
        depth = np.ascontiguousarray(depth, dtype=np.uint16)
        b = None if bgr is None else np.ascontiguousarray(bgr, dtype=np.uint8)
        self.ctx.check(self.ctx.lib.rgbid_frame_decode(
            self.ctx.h, self.h, None if b is None else b.ctypes.data, depth.ctypes.data, scale),
            "frame_decode")

    def download(self) -> FrameData:
        I = np.empty((self.height, self.width))
        W = np.empty((self.height, self.width))
        self.ctx.check(self.ctx.lib.rgbid_frame_download(self.ctx.h, self.h, dptr(I), dptr(W)),
                       "frame_download")
        return FrameData(I, W)

    def invalidate(self):
        self.ctx.lib.rgbid_frame_invalidate(self.h)

    def device_ptrs(self):
        I, W = abi.DP(), abi.DP()
        self.ctx.lib.rgbid_frame_device_ptrs(self.h, C.byref(I), C.byref(W))
        return C.cast(I, C.c_void_p).value, C.cast(W, C.c_void_p).value

    def close(self):
        if self.h:
            self.ctx.lib.rgbid_frame_destroy(self.ctx.h, self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------------- entry points


def build_pyramid(frame: FrameData, K: Intrinsics, levels: int,
                  ctx: Optional[Context] = None) -> Pyramid:
    """src/alignment.cpp:9-30"""
    ctx = ctx or default_context()
    h, w = frame.inverse_depth.shape
    sizes = [(h, w)]
    for _ in range(1, levels):
        sizes.append((sizes[-1][0] // 2, sizes[-1][1] // 2))
    oI = [np.empty(s) for s in sizes]
    oW = [np.empty(s) for s in sizes]
    Ks = (abi.Intrinsics_t * levels)()
    ctx.check(ctx.lib.rgbid_build_pyramid(ctx.h, dptr(frame.intensity), dptr(frame.inverse_depth),
                                          w, h, C.byref(K.to_c()), levels, abi.dptr_array(oI),
                                          abi.dptr_array(oW), Ks), "build_pyramid")
    return Pyramid([FrameData(a, b) for a, b in zip(oI, oW)], [Intrinsics.from_c(k) for k in Ks])


@dataclass
class WarpedFrame:
    """inc/warping.hpp:27-36"""
    intensity: np.ndarray
    inverse_depth: np.ndarray
    map_x: np.ndarray
    map_y: np.ndarray


def inverse_warp(src: np.ndarray, f_w, out_width: int, out_height: int,
                 ctx: Optional[Context] = None) -> np.ndarray:
    """src/warping.cpp:8-18: out(x, y) = bilinear(src, f_w((x, y))).  f_w is
    evaluated on the host (vectorised over the output grid when it accepts
    arrays); the sampling runs on the device (rgbid_remap_bilinear)."""
    ctx = ctx or default_context()
    src = np.ascontiguousarray(src, dtype=np.float64)
    h, w = src.shape
    ys, xs = np.mgrid[0:out_height, 0:out_width].astype(np.float64)
    try:
        mx, my = f_w(np.stack([xs, ys]))
        mx = np.broadcast_to(np.asarray(mx, dtype=np.float64), xs.shape)
        my = np.broadcast_to(np.asarray(my, dtype=np.float64), xs.shape)
    except Exception:  # scalar f_w: per pixel
        q = [f_w(np.array([x, y])) for y in range(out_height) for x in range(out_width)]
        mx = np.array([v[0] for v in q]).reshape(xs.shape)
        my = np.array([v[1] for v in q]).reshape(xs.shape)
    mx, my = np.ascontiguousarray(mx), np.ascontiguousarray(my)
    out = np.empty((out_height, out_width))
    ctx.check(ctx.lib.rgbid_remap_bilinear(ctx.h, dptr(src), w, h, dptr(mx), dptr(my), out_width,
                                           out_height, dptr(out)), "inverse_warp")
    return out


def inverse_geometric_warp(I_B, W_B, W_A, T_AB: Pose, K: Intrinsics,
                           ctx: Optional[Context] = None) -> WarpedFrame:
    """src/warping.cpp:76-114"""
    ctx = ctx or default_context()
    I_B = np.ascontiguousarray(I_B, dtype=np.float64)
    W_B = np.ascontiguousarray(W_B, dtype=np.float64)
    W_A = np.ascontiguousarray(W_A, dtype=np.float64)
    hb, wb = W_B.shape
    h, w = W_A.shape
    out = [np.empty((h, w)) for _ in range(4)]
    ctx.check(ctx.lib.rgbid_inverse_geometric_warp(ctx.h, dptr(I_B), dptr(W_B), wb, hb, dptr(W_A),
                                                   w, h, C.byref(T_AB.to_c()), C.byref(K.to_c()),
                                                   *[dptr(o) for o in out]),
              "inverse_geometric_warp")
    return WarpedFrame(*out)


def _result_or_raise(r) -> AlignmentResult:
    if r.status == abi.E_DEGENERATE:
        raise DegenerateAlignmentError(list(r.spectrum))
    return AlignmentResult.from_c(r)


def align(frame_a, frame_b, K: Intrinsics, init: Optional[Pose] = None,
          config: Optional[AlignmentConfig] = None, ctx: Optional[Context] = None,
          trace: bool = False):
    """src/alignment.cpp:367-409.  frame_a/frame_b: FrameData or DeviceFrame.
    Raises DegenerateAlignmentError like the reference.  With trace=True also
    returns the per-iteration records (rgbid_iter_trace)."""
    ctx = ctx or default_context()
    cfg = (config or AlignmentConfig()).to_c()
    res = abi.AlignResult_t()
    init_c = (init or Pose()).to_c()
    if isinstance(frame_a, DeviceFrame):
        rc = ctx.lib.rgbid_align(ctx.h, frame_a.h, frame_b.h, C.byref(K.to_c()), C.byref(init_c),
                                 C.byref(cfg), C.byref(res))
    else:
        h, w = frame_a.inverse_depth.shape
        rc = ctx.lib.rgbid_align_host(ctx.h, dptr(frame_a.intensity), dptr(frame_a.inverse_depth),
                                      dptr(frame_b.intensity), dptr(frame_b.inverse_depth), w, h,
                                      C.byref(K.to_c()), C.byref(init_c), C.byref(cfg),
                                      C.byref(res))
    if rc not in (abi.OK, abi.E_DEGENERATE):
        ctx.check(rc, "align")
    if trace:
        tr = (abi.IterTrace_t * 64)()
        n = C.c_int(0)
        ctx.lib.rgbid_last_align_trace(ctx.h, tr, 64, C.byref(n))
        records = list(tr)[: n.value]
        if res.status == abi.E_DEGENERATE:
            return None, records, list(res.spectrum)
        return AlignmentResult.from_c(res), records
    return _result_or_raise(res)


def align_batch(frames_a: Sequence[DeviceFrame], frames_b: Sequence[DeviceFrame], K: Intrinsics,
                inits: Optional[Sequence[Pose]] = None, config: Optional[AlignmentConfig] = None,
                ctx: Optional[Context] = None):
    """Batched independent alignments (config 5).  Returns the raw C results
    (status per pair; see _result_or_raise)."""
    ctx = ctx or default_context()
    n = len(frames_a)
    A = (C.c_void_p * n)(*[f.h.value for f in frames_a])
    B = (C.c_void_p * n)(*[f.h.value for f in frames_b])
    ini = (abi.Pose_t * n)(*[p.to_c() for p in inits]) if inits is not None else None
    res = (abi.AlignResult_t * n)()
    cfg = (config or AlignmentConfig()).to_c()
    ctx.check(ctx.lib.rgbid_align_batch(ctx.h, n, A, B, C.byref(K.to_c()), ini, C.byref(cfg), res),
              "align_batch")
    return list(res)


@dataclass
class PixelJet:
    """inc/alignment.hpp:48-56"""
    x: int
    y: int
    r_I: float
    r_W: float
    J_I: np.ndarray
    J_W: np.ndarray
    lambda_n: float
    has_depth: bool


def residuals_and_jacobians(frame_a: FrameData, warped: WarpedFrame, K: Intrinsics,
                            lambda_n_min: float = 0.1, ctx: Optional[Context] = None,
                            as_array: bool = False):
    """src/alignment.cpp:195-250.  Returns the jets in row-major order (PixelJet
    list, or with as_array=True an (n, 17) array {x, y, r_I, r_W, J_I[6], J_W[6],
    lambda_n} plus the has_depth flags)."""
    ctx = ctx or default_context()
    h, w = frame_a.inverse_depth.shape
    cap = w * h
    jets = np.empty((cap, 17))
    flags = np.empty(cap, dtype=np.uint8)
    n = ctx.lib.rgbid_residuals_and_jacobians(
        ctx.h, dptr(np.ascontiguousarray(frame_a.intensity)),
        dptr(np.ascontiguousarray(frame_a.inverse_depth)),
        dptr(np.ascontiguousarray(warped.intensity)),
        dptr(np.ascontiguousarray(warped.inverse_depth)), w, h, C.byref(K.to_c()), lambda_n_min,
        dptr(jets), flags.ctypes.data_as(C.POINTER(C.c_ubyte)), cap)
    if n < 0:
        ctx.check(int(n), "residuals_and_jacobians")
    jets, flags = jets[:n].copy(), flags[:n].astype(bool)
    if as_array:
        return jets, flags
    return [PixelJet(int(j[0]), int(j[1]), j[2], j[3], j[4:10].copy(), j[10:16].copy(), j[16], f)
            for j, f in zip(jets, flags)]


def estimate_location_scale(residuals, nu: float, ctx: Optional[Context] = None) -> TDistParams:
    """src/alignment.cpp:61-101 (systematic sample of <= 19200, IRLS on the device)"""
    ctx = ctx or default_context()
    r = np.ascontiguousarray(residuals, dtype=np.float64)
    t = abi.TDist_t()
    ctx.check(ctx.lib.rgbid_estimate_location_scale(ctx.h, dptr(r), len(r), nu, C.byref(t)),
              "estimate_location_scale")
    return TDistParams(t.mu, t.sigma, t.nu)


def estimate_nu(residuals, mu: float, sigma: float, ctx: Optional[Context] = None) -> float:
    """src/alignment.cpp:109-127"""
    ctx = ctx or default_context()
    r = np.ascontiguousarray(residuals, dtype=np.float64)
    out = C.c_double(0.0)
    ctx.check(ctx.lib.rgbid_estimate_nu(ctx.h, dptr(r), len(r), mu, sigma, C.byref(out)),
              "estimate_nu")
    return out.value


def filtered_hessian_covariance(frame_a, frame_b, K: Intrinsics, T_AB: Pose,
                                config: Optional[AlignmentConfig] = None,
                                ctx: Optional[Context] = None):
    """src/alignment.cpp:411-436 -> (cov 6x6, degenerate)"""
    ctx = ctx or default_context()
    fa = frame_a if isinstance(frame_a, DeviceFrame) else DeviceFrame.from_frame(frame_a, ctx)
    fb = frame_b if isinstance(frame_b, DeviceFrame) else DeviceFrame.from_frame(frame_b, ctx)
    cov = np.empty(36)
    deg = C.c_int(0)
    ctx.check(ctx.lib.rgbid_filtered_hessian_covariance(
        ctx.h, fa.h, fb.h, C.byref(K.to_c()), C.byref(T_AB.to_c()),
        C.byref((config or AlignmentConfig()).to_c()), dptr(cov), C.byref(deg)),
        "filtered_hessian_covariance")
    return cov.reshape(6, 6), bool(deg.value)


def bilateral_filter(img, sigma_space: float, sigma_range: float,
                     ctx: Optional[Context] = None) -> np.ndarray:
    """src/alignment.cpp:252-277"""
    ctx = ctx or default_context()
    img = np.ascontiguousarray(img, dtype=np.float64)
    h, w = img.shape
    out = np.empty_like(img)
    ctx.check(ctx.lib.rgbid_bilateral_filter(ctx.h, dptr(img), w, h, sigma_space, sigma_range,
                                             dptr(out)), "bilateral_filter")
    return out


# --------------------------------------------------------------------------- fusion


@dataclass
class Keyframe:
    """inc/fusion.hpp:15-22"""
    intensity: np.ndarray
    inverse_depth: np.ndarray
    weight: np.ndarray
    T_W_kf: Pose
    id: int = 0
    timestamp: float = 0.0


def make_keyframe(frame: FrameData, T_W_kf: Pose, id: int, timestamp: float) -> Keyframe:
    """src/fusion.cpp:7-16 (C = 1 everywhere, holes included)"""
    return Keyframe(frame.intensity.copy(), frame.inverse_depth.copy(),
                    np.ones_like(frame.inverse_depth), T_W_kf, id, timestamp)


@dataclass
class CovisibilityResult:
    ratio: float = 0.0
    empty_frame: bool = False
    counts: tuple = ()


def covisibility_ratio(frame_a, frame_b, T_BA: Pose, K: Intrinsics, sigma_w: float,
                       ctx: Optional[Context] = None) -> CovisibilityResult:
    """src/fusion.cpp:52-66"""
    ctx = ctx or default_context()
    fa = frame_a if isinstance(frame_a, DeviceFrame) else DeviceFrame.from_frame(frame_a, ctx)
    fb = frame_b if isinstance(frame_b, DeviceFrame) else DeviceFrame.from_frame(frame_b, ctx)
    ratio = C.c_double(0.0)
    empty = C.c_int(0)
    counts = (C.c_longlong * 4)()
    ctx.check(ctx.lib.rgbid_covisibility_ratio(ctx.h, fa.h, fb.h, C.byref(T_BA.to_c()),
                                               C.byref(K.to_c()), sigma_w, C.byref(ratio),
                                               C.byref(empty), counts), "covisibility_ratio")
    return CovisibilityResult(ratio.value, bool(empty.value), tuple(counts))


def should_switch_keyframe(ratio: float, threshold: float = 0.7) -> bool:
    return ratio < threshold


def should_switch_reference(ratio: float, threshold: float = 0.9) -> bool:
    return ratio < threshold


def integrate_frame(kf: Keyframe, frame: FrameData, T_kf_frame: Pose, K: Intrinsics,
                    sigma_w: float, ctx: Optional[Context] = None) -> None:
    """src/fusion.cpp:68-95 — updates kf.inverse_depth and kf.weight in place."""
    ctx = ctx or default_context()
    h, w = kf.inverse_depth.shape
    for name in ("inverse_depth", "weight"):
        a = getattr(kf, name)
        if not (a.flags["C_CONTIGUOUS"] and a.dtype == np.float64):
            setattr(kf, name, np.ascontiguousarray(a, dtype=np.float64))
    ctx.check(ctx.lib.rgbid_integrate_frame(ctx.h, dptr(kf.inverse_depth), dptr(kf.weight),
                                            dptr(frame.intensity), dptr(frame.inverse_depth), w, h,
                                            C.byref(T_kf_frame.to_c()), C.byref(K.to_c()),
                                            sigma_w), "integrate_frame")


@dataclass
class BufferedFrame:
    frame: FrameData
    T_W_frame: Pose
    timestamp: float = 0.0


class FrameBuffer:
    """inc/fusion.hpp:56-74, src/fusion.cpp:97-111 (host bookkeeping)."""

    def __init__(self, capacity: int = 30):
        self.capacity = capacity
        self.frames: List[BufferedFrame] = []

    def push(self, f: BufferedFrame):
        if len(self.frames) >= self.capacity:
            self.frames.pop(0)
        self.frames.append(f)

    def empty(self) -> bool:
        return not self.frames

    def size(self) -> int:
        return len(self.frames)

    def clear(self):
        self.frames.clear()

    def pop_closest(self, timestamp: float) -> Optional[BufferedFrame]:
        if not self.frames:
            return None
        best, best_dt = 0, abs(self.frames[0].timestamp - timestamp)
        for i in range(1, len(self.frames)):
            dt = abs(self.frames[i].timestamp - timestamp)
            if dt < best_dt:
                best, best_dt = i, dt
        return self.frames.pop(best)


def drain_buffer_step(kf: Keyframe, buffer: FrameBuffer, K: Intrinsics, sigma_w: float,
                      ctx: Optional[Context] = None) -> None:
    """src/fusion.cpp:113-118"""
    f = buffer.pop_closest(kf.timestamp)
    if f is None:
        return
    integrate_frame(kf, f.frame, kf.T_W_kf.inverse() * f.T_W_frame, K, sigma_w, ctx)


# --------------------------------------------------------------------------- depth camera


@dataclass
class DepthIntrinsics:
    """inc/camera.hpp:45-51"""
    beta0: float = 0.0
    beta1: float = 1.0
    q0: tuple = (0.0,) * 9
    q1: tuple = (1.0,) + (0.0,) * 8
    p0: tuple = (4.0, 4.0)

    def to_c(self) -> abi.DepthIntrinsics_t:
        c = abi.DepthIntrinsics_t()
        c.beta0, c.beta1 = self.beta0, self.beta1
        for i in range(9):
            c.q0[i], c.q1[i] = self.q0[i], self.q1[i]
        c.p0[0], c.p0[1] = self.p0
        return c


def correct_inverse_depth(W_m, dintr: DepthIntrinsics, intr: Intrinsics, spatial: bool,
                          ctx: Optional[Context] = None) -> np.ndarray:
    """src/camera.cpp:62-81"""
    ctx = ctx or default_context()
    W_m = np.ascontiguousarray(W_m, dtype=np.float64)
    h, w = W_m.shape
    out = np.empty_like(W_m)
    ctx.check(ctx.lib.rgbid_correct_inverse_depth(ctx.h, dptr(W_m), w, h, C.byref(dintr.to_c()),
                                                  C.byref(intr.to_c()), int(spatial), dptr(out)),
              "correct_inverse_depth")
    return out


def forward_register(W_A, T_BA: Pose, K_A: Intrinsics, K_B: Intrinsics,
                     ctx: Optional[Context] = None) -> np.ndarray:
    """src/warping.cpp:20-74"""
    ctx = ctx or default_context()
    W_A = np.ascontiguousarray(W_A, dtype=np.float64)
    h, w = W_A.shape
    out = np.empty((K_B.height, K_B.width))
    ctx.check(ctx.lib.rgbid_forward_register(ctx.h, dptr(W_A), w, h, C.byref(T_BA.to_c()),
                                             C.byref(K_A.to_c()), C.byref(K_B.to_c()), dptr(out)),
              "forward_register")
    return out


# --------------------------------------------------------------------------- synthetic inputs


def rectify(img: np.ndarray, K: Intrinsics, ctx: Optional[Context] = None) -> np.ndarray:
    """inverse_warp(img, f_w = K distort(K^-1 p)) — src/warping.cpp:8-18 with the
    distorted-sensor map of src/camera.cpp:11-22,41-45, evaluated on the device."""
    ctx = ctx or default_context()
    img = np.ascontiguousarray(img, dtype=np.float64)
    h, w = img.shape
    out = np.empty_like(img)
    ctx.check(ctx.lib.rgbid_rectify(ctx.h, dptr(img), w, h, C.byref(K.to_c()), dptr(out)), "rectify")
    return out


def rectify_frame(src: "DeviceFrame", K: Intrinsics, dst: "DeviceFrame"):
    """Both maps of a device frame through rectify (device-resident)."""
    src.ctx.check(src.ctx.lib.rgbid_rectify_frame(src.ctx.h, src.h, C.byref(K.to_c()), dst.h),
                  "rectify_frame")
    return dst


def undistort_points(m_d, K: Intrinsics, ctx: Optional[Context] = None):
    """undistort (src/camera.cpp:24-39) of n normalized points: (m_u [n, 2], ok [n])."""
    ctx = ctx or default_context()
    m_d = np.ascontiguousarray(m_d, dtype=np.float64).reshape(-1, 2)
    n = len(m_d)
    m_u = np.empty_like(m_d)
    ok = np.zeros(n, dtype=np.uint8)
    ctx.check(ctx.lib.rgbid_undistort_points(ctx.h, dptr(m_d), n, C.byref(K.to_c()), dptr(m_u),
                                             ok.ctypes.data_as(C.POINTER(C.c_ubyte))),
              "undistort_points")
    return m_u, ok.astype(bool)


def render_plane(K: Intrinsics, T_WC: Pose, n=(0.0, 0.0, 1.0), d: float = -2.0,
                 tex_scale: float = 1.0) -> FrameData:
    """tests/synthetic.hpp:31-50 (bit-identical to the reference fixture at tex_scale=1)."""
    L = abi.lib()
    I = np.empty((K.height, K.width))
    W = np.empty((K.height, K.width))
    nn = np.ascontiguousarray(n, dtype=np.float64)
    L.rgbid_synth_render_plane(C.byref(K.to_c()), C.byref(T_WC.to_c()), dptr(nn), d, tex_scale,
                               dptr(I), dptr(W))
    return FrameData(I, W)


def random_pose(seed: int, t_scale: float = 1.0, angle_scale: float = 1.0, skip: int = 0) -> Pose:
    """random_pose(std::mt19937(seed)) of tests/synthetic.hpp:52-59 (after `skip` draws)."""
    out = abi.Pose_t()
    abi.lib().rgbid_synth_random_pose(seed, skip, t_scale, angle_scale, C.byref(out))
    return Pose.from_c(out)


def synth_pair_host(K: Intrinsics, pair_seed: int, variant: int = 1):
    """Pair `pair_seed` of the bench's synthetic workload (rgbid_synth_pair_device's
    scene model) rendered on the host: (frame_a, frame_b, T_AB_truth)."""
    h, w = K.height, K.width
    IA, WA, IB, WB = (np.empty((h, w)) for _ in range(4))
    T = abi.Pose_t()
    rc = abi.lib().rgbid_synth_pair_host(C.byref(K.to_c()), pair_seed, variant, dptr(IA), dptr(WA),
                                         dptr(IB), dptr(WB), C.byref(T))
    if rc != abi.OK:
        raise ValueError("synth_pair_host: invalid argument")
    return FrameData(IA, WA), FrameData(IB, WB), Pose.from_c(T)


def add_noise(frame: FrameData, seed: int, sigma_i: float, sigma_w: float) -> FrameData:
    f = frame.copy()
    h, w = f.inverse_depth.shape
    abi.lib().rgbid_synth_add_noise(dptr(f.intensity), dptr(f.inverse_depth), w, h, seed, sigma_i,
                                    sigma_w)
    return f


def synth_pair_device(a: DeviceFrame, b: DeviceFrame, K: Intrinsics, pair_seed: int,
                      variant: int) -> Pose:
    """Device-rendered benchmark pair; returns the ground-truth T_AB."""
    T = abi.Pose_t()
    a.ctx.check(a.ctx.lib.rgbid_synth_pair_device(a.ctx.h, a.h, b.h, C.byref(K.to_c()), pair_seed,
                                                  variant, C.byref(T)), "synth_pair_device")
    return Pose.from_c(T)


# --------------------------------------------------------------------------- front-end (config 3)


@dataclass
class FrameEstimate:
    """inc/pipeline.hpp:25-31"""
    timestamp: float
    T_W_k: Pose
    cov: np.ndarray
    lost: bool
    keyframe_id: int

    @staticmethod
    def from_c(e) -> "FrameEstimate":
        return FrameEstimate(e.timestamp, Pose.from_c(e.T_W_k), np.array(e.cov[:]).reshape(6, 6),
                             bool(e.lost), e.keyframe_id)


@dataclass
class FrontendConfig:
    """PipelineConfig's front-end fields (inc/pipeline.hpp:72-88)."""
    alignment: AlignmentConfig = field(default_factory=AlignmentConfig)
    keyframe_covisibility: float = 0.7
    reference_covisibility: float = 0.9
    buffer_capacity: int = 30

    def to_c(self) -> abi.FrontendConfig_t:
        c = abi.FrontendConfig_t()
        c.align = self.alignment.to_c()
        c.keyframe_covisibility = self.keyframe_covisibility
        c.reference_covisibility = self.reference_covisibility
        c.buffer_capacity = self.buffer_capacity
        return c


class Frontend:
    """Pipeline front-end (src/pipeline.cpp:120-247) on the B200: process_frame,
    trajectory, keyframes.  The back-end (loop closure, pose graph) is out of scope."""

    def __init__(self, K: Intrinsics, config: Optional[FrontendConfig] = None,
                 ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.K = K
        self.h = C.c_void_p()
        self.ctx.check(self.ctx.lib.rgbid_frontend_create(
            self.ctx.h, C.byref(K.to_c()), C.byref((config or FrontendConfig()).to_c()),
            C.byref(self.h)), "frontend_create")

    def process_frame(self, frame: FrameData, timestamp: float) -> FrameEstimate:
        e = abi.FrameEstimate_t()
        self.ctx.check(self.ctx.lib.rgbid_frontend_process(
            self.h, dptr(frame.intensity), dptr(frame.inverse_depth), timestamp, C.byref(e)),
            "frontend_process")
        return FrameEstimate.from_c(e)

    def finish(self):
        self.ctx.check(self.ctx.lib.rgbid_frontend_finish(self.h), "frontend_finish")

    def trajectory(self) -> List[FrameEstimate]:
        n = C.c_int(0)
        self.ctx.lib.rgbid_frontend_trajectory(self.h, None, 0, C.byref(n))
        arr = (abi.FrameEstimate_t * max(1, n.value))()
        self.ctx.lib.rgbid_frontend_trajectory(self.h, arr, n.value, C.byref(n))
        return [FrameEstimate.from_c(e) for e in arr[: n.value]]

    def keyframe_frame_index(self) -> List[int]:
        n = C.c_int(0)
        self.ctx.lib.rgbid_frontend_keyframes(self.h, None, 0, C.byref(n))
        arr = (C.c_int * max(1, n.value))()
        self.ctx.lib.rgbid_frontend_keyframes(self.h, arr, n.value, C.byref(n))
        return list(arr[: n.value])

    def keyframe_count(self) -> int:
        return len(self.keyframe_frame_index())

    def current_keyframe(self):
        W = np.empty((self.K.height, self.K.width))
        Cm = np.empty_like(W)
        T = abi.Pose_t()
        kid = C.c_int(0)
        self.ctx.check(self.ctx.lib.rgbid_frontend_current_keyframe(
            self.h, dptr(W), dptr(Cm), C.byref(T), C.byref(kid)), "current_keyframe")
        return W, Cm, Pose.from_c(T), kid.value

    def close(self):
        if self.h:
            self.ctx.lib.rgbid_frontend_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------------- back-end callers


@dataclass
class LoopConfig:
    """include/rgbid/loop.hpp:38-48 (the dense-refinement gate; retrieval fields are
    the out-of-scope place-recognition front end's)."""
    min_covisibility: float = 0.3


@dataclass
class LoopConstraint:
    """include/rgbid/loop.hpp:19-26"""
    i: int = 0
    j: int = 0
    T_ij: Pose = field(default_factory=Pose)
    info: np.ndarray = field(default_factory=lambda: np.eye(6))
    inliers: int = 0
    hull_fraction: float = 0.0
    score: float = 0.0


def make_loop_constraint(kf_i, kf_j, id_i: int, id_j: int, T_init: Pose, K: Intrinsics,
                         inliers: int = 0, hull_fraction: float = 0.0,
                         config: Optional[LoopConfig] = None,
                         align_config: Optional[AlignmentConfig] = None,
                         ctx: Optional[Context] = None) -> Optional[LoopConstraint]:
    """src/loop.cpp:174-203: dense refinement of a loop candidate -> LoopConstraint,
    or None (std::nullopt) when the alignment is degenerate or the refined
    covisibility falls below config.min_covisibility.  kf_i/kf_j: FrameData or
    DeviceFrame.  Use a separate Context per host thread to refine loops
    concurrently with tracking (each context owns a stream)."""
    ctx = ctx or default_context()
    fi = kf_i if isinstance(kf_i, DeviceFrame) else DeviceFrame.from_frame(kf_i, ctx)
    fj = kf_j if isinstance(kf_j, DeviceFrame) else DeviceFrame.from_frame(kf_j, ctx)
    cfg = (align_config or AlignmentConfig()).to_c()
    out = abi.LoopConstraint_t()
    acc = C.c_int(0)
    ctx.check(ctx.lib.rgbid_make_loop_constraint(
        ctx.h, fi.h, fj.h, id_i, id_j, C.byref(K.to_c()), C.byref(T_init.to_c()), C.byref(cfg),
        (config or LoopConfig()).min_covisibility, inliers, hull_fraction, C.byref(out),
        C.byref(acc)), "make_loop_constraint")
    if not acc.value:
        return None
    return LoopConstraint(out.i, out.j, Pose.from_c(out.T_ij),
                          np.array(out.info[:]).reshape(6, 6), out.inliers, out.hull_fraction,
                          out.score)


@dataclass
class NormalMap:
    """include/rgbid/segmentation.hpp:12-24"""
    nx: np.ndarray
    ny: np.ndarray
    nz: np.ndarray


def normal_map(W: np.ndarray, K: Intrinsics, ctx: Optional[Context] = None) -> NormalMap:
    """src/segmentation.cpp:10-57"""
    ctx = ctx or default_context()
    W = np.ascontiguousarray(W, dtype=np.float64)
    h, w = W.shape
    nx, ny, nz = (np.empty_like(W) for _ in range(3))
    ctx.check(ctx.lib.rgbid_normal_map(ctx.h, dptr(W), w, h, C.byref(K.to_c()), dptr(nx),
                                       dptr(ny), dptr(nz)), "normal_map")
    return NormalMap(nx, ny, nz)


@dataclass
class PointCloud:
    """include/rgbid/pipeline.hpp:90-93 (points N x 3 float64, colors N x 3 uint8)"""
    points: np.ndarray
    colors: np.ndarray


def export_map(keyframes: Sequence[Keyframe], K: Intrinsics, voxel: float,
               ctx: Optional[Context] = None) -> PointCloud:
    """src/pipeline.cpp:463-527"""
    ctx = ctx or default_context()
    n = len(keyframes)
    if n == 0:
        return PointCloud(np.zeros((0, 3)), np.zeros((0, 3), np.uint8))
    h, w = keyframes[0].inverse_depth.shape
    Is = [np.ascontiguousarray(k.intensity, dtype=np.float64) for k in keyframes]
    Ws = [np.ascontiguousarray(k.inverse_depth, dtype=np.float64) for k in keyframes]
    poses = (abi.Pose_t * n)(*[k.T_W_kf.to_c() for k in keyframes])
    cap = n * w * h
    pts = np.empty((cap, 3), np.float64)
    cols = np.empty((cap, 3), np.uint8)
    cnt = C.c_longlong(0)
    ctx.check(ctx.lib.rgbid_export_map(ctx.h, n, abi.dptr_array(Is), abi.dptr_array(Ws), w, h,
                                       poses, C.byref(K.to_c()), voxel, dptr(pts),
                                       cols.ctypes.data_as(C.POINTER(C.c_ubyte)), cap,
                                       C.byref(cnt)), "export_map")
    return PointCloud(pts[: cnt.value].copy(), cols[: cnt.value].copy())
