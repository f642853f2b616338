"""CPU restatement of the back-end callers of the hot path — SURVEY 8(f) ranks 3-4.

TEST INFRASTRUCTURE ONLY (imported by tests/ as the checker; never by the
product).  Parity anchors:

* ``export_map`` restates src/pipeline.cpp:463-527 line by line in Python floats
  (IEEE double, same operation order as the Eigen expressions: 3-term products
  v0 + (v1 + v2), coefficient-wise division).  src/pipeline.cpp cannot be compiled
  here (it drags in features/loop/posegraph), so this restatement is
  pinned only by its shared building blocks: K^-1, pose inverse/compose come from
  the C restatement (``Oracle("C")``), itself checked bit-for-bit against the
  reference build; ``bilinear`` follows include/rgbid/image.hpp:51-62.
* ``make_loop_constraint`` restates src/loop.cpp:174-203 over the reference build's
  own ``align`` and ``covisibility_ratio`` (``Oracle("REF")``); the 6x6 inverse of
  the covariance is numpy's (LAPACK partial-pivot LU, like Eigen's
  Mat6::inverse, so equal up to rounding).
* ``normal_map`` is not restated: the reference's src/segmentation.cpp compiles
  unchanged against the Eigen shim (``Oracle("REF").normal_map``).
"""
from __future__ import annotations

import math

import numpy as np

from .oracle import Oracle, Pose_t


def _red3(a, b, c):
    return a + (b + c)


def _m3mul(a, b):
    return [[_red3(a[i][0] * b[0][j], a[i][1] * b[1][j], a[i][2] * b[2][j]) for j in range(3)]
            for i in range(3)]


def _m3v(a, v):
    return [_red3(a[i][0] * v[0], a[i][1] * v[1], a[i][2] * v[2]) for i in range(3)]


def _valid(v):
    return math.isfinite(v)


def _bilinear(img, x, y):
    """include/rgbid/image.hpp:51-62"""
    h, w = img.shape
    if not (x >= 0 and x <= w - 1 and y >= 0 and y <= h - 1):
        return math.nan
    x0, y0 = math.floor(x), math.floor(y)
    x1, y1 = min(x0 + 1, w - 1), min(y0 + 1, h - 1)
    fx, fy = x - x0, y - y0
    v00, v10 = float(img[y0, x0]), float(img[y0, x1])
    v01, v11 = float(img[y1, x0]), float(img[y1, x1])
    if not (_valid(v00) and _valid(v10) and _valid(v01) and _valid(v11)):
        return math.nan
    return (1 - fy) * ((1 - fx) * v00 + fx * v10) + fy * ((1 - fx) * v01 + fx * v11)


def _pose_lists(T: Pose_t):
    R = [[T.R[3 * i + j] for j in range(3)] for i in range(3)]
    return R, [T.t[0], T.t[1], T.t[2]]


def export_map(keyframes, K, voxel):
    """src/pipeline.cpp:463-527.  keyframes: sequence of (I, W, T_W_kf: Pose_t);
    K: Intrinsics_t.  Returns (points N x 3 float64, colors N x 3 uint8)."""
    orc = Oracle("C")
    Km = [[K.fx, 0.0, K.cx], [0.0, K.fy, K.cy], [0.0, 0.0, 1.0]]
    Kinv = orc.mat3_inverse(np.array(Km)).tolist()
    points, colors = [], []
    for k, (I, W, T) in enumerate(keyframes):
        prev = keyframes[k - 1] if k > 0 else None
        if prev is not None:
            Tp = orc.pose_compose(orc.pose_inverse(prev[2]), T)  # T_prev_kf
            Rp, tp = _pose_lists(Tp)
            Rt = _m3mul(_m3mul(Km, Rp), Kinv)
            tt = _m3v(Km, tp)
        R, t = _pose_lists(T)
        h, w = W.shape
        for y in range(h):
            for x in range(w):
                wv = float(W[y, x])
                if not _valid(wv) or wv <= 0.0:
                    continue
                if prev is not None:
                    pq = _m3v(Rt, [float(x), float(y), 1.0])
                    q = [pq[i] + wv * tt[i] for i in range(3)]
                    if q[2] > 0.0:
                        u, v = q[0] / q[2], q[1] / q[2]
                        pw = prev[1]
                        if u >= 0 and u <= w - 1 and v >= 0 and v <= h - 1:
                            w_prev = _bilinear(pw, u, v)
                            w_pred = wv / q[2]
                            if _valid(w_prev) and abs(w_prev - w_pred) < 3.0 * 0.02:
                                continue
                kp = _m3v(Kinv, [float(x), float(y), 1.0])
                X = [kp[i] / wv for i in range(3)]
                XW = _m3v(R, X)
                XW = [XW[i] + t[i] for i in range(3)]
                g = float(I[y, x])
                gc = 0.0 if g < 0.0 else (1.0 if 1.0 < g else g)
                c = int(gc * 255.0) if math.isfinite(gc) else 0
                points.append(XW)
                colors.append((c, c, c))
    if voxel <= 0.0 or not points:
        return np.array(points, dtype=np.float64).reshape(-1, 3), \
            np.array(colors, dtype=np.uint8).reshape(-1, 3)
    M = (1 << 64) - 1
    grid, order = {}, []
    for p, c in zip(points, colors):
        ix, iy, iz = (math.floor(p[i] / voxel) for i in range(3))
        key = ((ix * 73856093) & M) ^ ((iy * 19349663) & M) ^ ((iz * 83492791) & M)
        if key not in grid:
            grid[key] = [[0.0, 0.0, 0.0], [0.0, 0.0, 0.0], 0]
            order.append(key)
        a = grid[key]
        for i in range(3):
            a[0][i] = a[0][i] + p[i]
            a[1][i] = a[1][i] + float(c[i])
        a[2] += 1
    fp, fc = [], []
    for key in order:
        s, col, n = grid[key]
        fp.append([s[i] / n for i in range(3)])
        fc.append([int(col[i] / n) for i in range(3)])
    return np.array(fp, dtype=np.float64), np.array(fc, dtype=np.uint8)


def make_loop_constraint(kf_i, kf_j, T_init: Pose_t, K, cfg=None, min_covisibility=0.3):
    """src/loop.cpp:174-203 over the reference build.  kf_*: (I, W).  Returns None
    (std::nullopt) or (T_ij: Pose_t, info 6x6)."""
    ref = Oracle("REF")
    res = ref.align(kf_i[0], kf_i[1], kf_j[0], kf_j[1], K, init=T_init, cfg=cfg)
    if res.status != 0:
        return None  # DegenerateAlignmentError
    T_BA = Oracle("C").pose_inverse(res.T_AB)
    ratio, empty = ref.covisibility_ratio(kf_i[0], kf_i[1], kf_j[0], kf_j[1], T_BA, K,
                                          res.tdist_depth.sigma)[:2]
    if empty or ratio < min_covisibility:
        return None
    info = np.linalg.inv(np.array(res.cov[:]).reshape(6, 6))
    return res.T_AB, 0.5 * (info + info.T)
