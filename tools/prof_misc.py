"""Driver for ncu captures of the kernels off the batched IRLS loop: config-2 fusion
(k_integrate over 20 frames), covisibility (both directions), config-4 registration
(k_correct_depth, k_splat, k_gather_register), and one single-pair 4-level align
(latency mode: k_tdist_cluster), all at 640x480."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_08271_b200 as rg  # noqa: E402
from paper_1807_08271_b200 import abi  # noqa: E402

ctx = rg.Context(0)
K = rg.simple_intrinsics(640, 480, 480.0)
n = np.array([0.2, -0.15, 1.0])
n /= np.linalg.norm(n)
base = rg.render_plane(K, rg.Pose(), n, -2.0, 8.0)
kf = rg.DeviceFrame.from_frame(base, ctx)
frames, poses = [], []
for k in range(20):
    T = rg.random_pose(3000 + k, 0.01, 0.01)
    frames.append(rg.DeviceFrame.from_frame(rg.add_noise(rg.render_plane(K, T, n, -2.0, 8.0), 100 + k,
                                                         0.0, 0.01), ctx))
    poses.append(T)
Cm = torch.ones((480, 640), dtype=torch.float64, device="cuda")
arr = (C.c_void_p * 20)(*[f.h.value for f in frames])
P = (abi.Pose_t * 20)(*[p.to_c() for p in poses])
ctx.check(ctx.lib.rgbid_integrate_frames(ctx.h, kf.h, C.cast(Cm.data_ptr(), abi.DP), 20, arr, P,
                                         C.byref(K.to_c()), 0.05), "integrate_frames")
ctx.check(ctx.lib.rgbid_integrate_frames(ctx.h, kf.h, C.cast(Cm.data_ptr(), abi.DP), 1, arr, P,
                                         C.byref(K.to_c()), 0.05), "integrate_frames")
fa, fb, T = rg.synth_pair_host(K, 3, 2)
A, B = rg.DeviceFrame.from_frame(fa, ctx), rg.DeviceFrame.from_frame(fb, ctx)
rg.covisibility_ratio(A, B, T.inverse(), K, 0.01, ctx)
d = rg.DepthIntrinsics(beta0=-0.005, beta1=1.02)
Wc = rg.correct_inverse_depth(fa.inverse_depth, d, K, False, ctx)
rg.forward_register(Wc, rg.random_pose(7, 0.025, 0.01), K, K, ctx)
rg.align(A, B, K, config=rg.AlignmentConfig(levels=4), ctx=ctx)
ctx.synchronize()
print("ok")
