"""One device-resident 4-level single-pair align (latency mode), after warm-up: the
ncu target for the latency path's per-kernel durations (their sum vs the measured
latency = the launch gaps of the graph)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_08271_b200 as rg
ctx = rg.Context(0)
K = rg.simple_intrinsics(640, 480, 480.0)
A, B = rg.DeviceFrame(640, 480, ctx), rg.DeviceFrame(640, 480, ctx)
rg.synth_pair_device(A, B, K, 0, 1)
cfg = rg.AlignmentConfig(levels=4)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    r = rg.align(A, B, K, config=cfg, ctx=ctx)
print("iterations", r.total_iterations)
