"""CPU restatement of the reference's Pipeline front-end — TEST INFRASTRUCTURE ONLY.

process_frame / track / fuse_and_maybe_switch / start_keyframe / emit_keyframe
(/root/reference/proj/src/pipeline.cpp:120-247), driven by the oracle's C
restatement (oracle/rgbid_oracle.c) for align, covisibility_ratio and
integrate_frame; pose math via the oracle's pose functions (same rounding
conventions as the product's host code).  The back-end is out of scope, as in
the product's rgbid_frontend.
"""
from __future__ import annotations

import numpy as np

from paper_1807_08271_b200.abi import Pose_t


def _ident():
    p = Pose_t()
    p.R[0] = p.R[4] = p.R[8] = 1.0
    return p


def compose_relative_with_cov(orc, T_WA, covA, T_WB, covB):
    """src/geometry.cpp:74-103"""
    R_AW = np.array(T_WA.R[:]).reshape(3, 3).T
    d = np.array(T_WA.t[:]) - np.array(T_WB.t[:])
    S = np.array([[0, -d[2], d[1]], [d[2], 0, -d[0]], [-d[1], d[0], 0]])
    JA = np.zeros((6, 6))
    JB = np.zeros((6, 6))
    JA[:3, :3] = -R_AW
    JA[:3, 3:] = -R_AW @ S
    JA[3:, 3:] = -R_AW
    JB[:3, :3] = R_AW
    JB[3:, 3:] = R_AW
    rel = orc.pose_compose(orc.pose_inverse(T_WA), T_WB)
    cov = JA @ covA @ JA.T + JB @ covB @ JB.T
    return rel, (cov + cov.T) / 2.0


class FrontendOracle:
    def __init__(self, orc, K, align_cfg, keyframe_cov=0.7, reference_cov=0.9, buffer_capacity=30):
        self.o, self.K, self.cfg = orc, K, align_cfg
        self.kf_cov, self.ref_cov, self.cap = keyframe_cov, reference_cov, buffer_capacity
        self.reference = None
        self.T_W_ref = _ident()
        self.T_ref_prev = None
        self.cov_ref_prev = np.zeros((6, 6))
        self.velocity = _ident()
        self.sigma_w = 0.01
        self.kf = None  # dict(W, C, T_W_kf, id, t)
        self.kf_source = None
        self.buffer = []
        self.next_id = 0
        self.traj = []  # (t, pose, cov, lost, kf_id)
        self.kf_index = []

    def process_frame(self, frame, t):
        if self.reference is None:
            self.reference = frame
            self.T_W_ref = _ident()
            self.T_ref_prev = _ident()
            self.cov_ref_prev = np.zeros((6, 6))
            self.traj.append([t, _ident(), np.zeros((6, 6)), False, 0])
            self.kf_index.append(0)
            self._start_keyframe(frame, t)
            return
        self._track(frame, t)
        self._fuse_and_maybe_switch(frame, t)

    def _track(self, frame, t):
        o = self.o
        init = o.pose_compose(self.T_ref_prev, self.velocity)
        res = o.align(self.reference.intensity, self.reference.inverse_depth, frame.intensity,
                      frame.inverse_depth, self.K, init, self.cfg)
        lost = res.status != 0
        if lost:
            T_ref_k = self.T_ref_prev
            self.velocity = _ident()
            step_cov = 1e6 * np.eye(6)
        else:
            T_ref_k = res.T_AB
            self.sigma_w = max(res.tdist_depth.sigma, 1e-6)
            cov_k = np.array(res.cov[:]).reshape(6, 6)
            self.velocity, step_cov = compose_relative_with_cov(o, self.T_ref_prev, self.cov_ref_prev,
                                                                T_ref_k, cov_k)
            self.cov_ref_prev = cov_k
        T_W_k = o.pose_compose(self.T_W_ref, T_ref_k)
        self.traj.append([t, T_W_k, step_cov, lost, -1])
        self.T_ref_prev = T_ref_k
        if not lost:
            T_k_ref = o.pose_inverse(T_ref_k)
            ratio, _, _ = o.covisibility_ratio(self.reference.intensity, self.reference.inverse_depth,
                                               frame.intensity, frame.inverse_depth, T_k_ref, self.K,
                                               self.sigma_w)
            if ratio < self.ref_cov:
                self.reference = frame
                self.T_W_ref = T_W_k
                self.T_ref_prev = _ident()
                self.cov_ref_prev = np.zeros((6, 6))

    def _drain(self):
        if not self.buffer:
            return
        best, best_dt = 0, abs(self.buffer[0][2] - self.kf["t"])
        for i in range(1, len(self.buffer)):
            dt = abs(self.buffer[i][2] - self.kf["t"])
            if dt < best_dt:
                best, best_dt = i, dt
        frame, T_W_frame, _ = self.buffer.pop(best)
        T = self.o.pose_compose(self.o.pose_inverse(self.kf["T_W_kf"]), T_W_frame)
        self.o.integrate_frame(None, self.kf["W"], self.kf["C"], frame.intensity, frame.inverse_depth,
                               T, self.K, self.sigma_w)

    def _fuse_and_maybe_switch(self, frame, t):
        o = self.o
        last = self.traj[-1]
        if len(self.buffer) >= self.cap:
            self.buffer.pop(0)
        self.buffer.append((frame, last[1], t))
        self._drain()
        T_frame_kf = o.pose_compose(o.pose_inverse(last[1]), self.kf["T_W_kf"])
        ratio, _, _ = o.covisibility_ratio(self.kf_source.intensity, self.kf_source.inverse_depth,
                                           frame.intensity, frame.inverse_depth,
                                           o.pose_inverse(T_frame_kf), self.K, self.sigma_w)
        if not last[3] and ratio < self.kf_cov:
            while self.buffer:
                self._drain()
            self._start_keyframe(frame, t)
            self.traj[-1][4] = self.next_id - 1
            self.kf_index.append(len(self.traj) - 1)
            self.reference = frame
            self.T_W_ref = last[1]
            self.T_ref_prev = _ident()
            self.cov_ref_prev = np.zeros((6, 6))

    def _start_keyframe(self, frame, t):
        self.kf = {"W": frame.inverse_depth.copy(), "C": np.ones_like(frame.inverse_depth),
                   "T_W_kf": self.traj[-1][1], "id": self.next_id, "t": t}
        self.next_id += 1
        self.kf_source = frame
        self.buffer = []
