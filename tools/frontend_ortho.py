"""Orthonormality and drift of the front-end trajectory (device vs oracle restatement)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1807_08271_b200 as rg
from oracle.frontend_oracle import FrontendOracle
from oracle.oracle import Oracle
from tests.test_frontend_gpu import _config3_frames

K = rg.simple_intrinsics(640, 480, 480.0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
seq = _config3_frames(K, n)
ctx = rg.Context(0)
fe = rg.Frontend(K, ctx=ctx)
est = [fe.process_frame(f, 0.033 * i) for i, (_, f) in enumerate(seq)]
orc = FrontendOracle(Oracle("C"), K.to_c(), rg.AlignmentConfig().to_c())
m = min(n, int(sys.argv[2]) if len(sys.argv) > 2 else n)
for i, (_, f) in enumerate(seq[:m]):
    orc.process_frame(f, 0.033 * i)
for i, ((T, _), e) in enumerate(zip(seq, est)):
    R = e.T_W_k.R
    line = f"{i:3d} kf={e.keyframe_id:3d} ortho={np.abs(R @ R.T - np.eye(3)).max():.2e} dt={np.abs(e.T_W_k.t - T.t).max():.2e}"
    if i < m:
        Ro = rg.Pose.from_c(orc.traj[i][1]).R
        line += f" oracle_ortho={np.abs(Ro @ Ro.T - np.eye(3)).max():.2e} |R-Ro|={np.abs(R - Ro).max():.2e}"
    print(line)
print("keyframes", fe.keyframe_frame_index(), "oracle", orc.kf_index)
