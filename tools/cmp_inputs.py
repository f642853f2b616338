import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
import paper_1807_08271_b200 as rg
from oracle import oracle as O
K, hp = bench.host_pairs(16, 1)
ctx = rg.Context(0)
dp = []
for i in range(16):
    A, B = rg.DeviceFrame(640, 480, ctx), rg.DeviceFrame(640, 480, ctx)
    rg.synth_pair_device(A, B, K, i, 1)
    fa, fb = A.download(), B.download()
    dp.append((fa.intensity, fa.inverse_depth, fb.intensity, fb.inverse_depth))
orc = O.Oracle("REF")
cfg = rg.AlignmentConfig(levels=4, iterations=[10, 5, 4]).to_c()
for name, pairs in (("host", hp), ("device", dp)):
    t0 = time.perf_counter()
    res = orc.align_many(pairs, K.to_c(), None, cfg, threads=16)
    dt = time.perf_counter() - t0
    its = [sum(r.level_log[k].iterations for k in range(r.n_levels)) for r in res]
    print(name, f"{16/dt:.1f} align/s", "iters", its, "status", [r.status for r in res])
    print("  nan frac A-W", np.mean([np.isnan(p[1]).mean() for p in pairs]), "B-W", np.mean([np.isnan(p[3]).mean() for p in pairs]))
