"""Single-pair 4-level align latency (device-resident VGA bench pair, CUDA events,
median of 20) for the library named by RGBID_LIB (default in-tree)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1807_08271_b200 as rg
ctx = rg.Context(0)
K = rg.simple_intrinsics(640, 480, 480.0)
A, B = rg.DeviceFrame(640, 480, ctx), rg.DeviceFrame(640, 480, ctx)
rg.synth_pair_device(A, B, K, 0, 1)
s = torch.cuda.ExternalStream(ctx.stream_ptr)
for levels in (4, 3):
    cfg = rg.AlignmentConfig(levels=levels)
    for _ in range(3):
        r = rg.align(A, B, K, config=cfg, ctx=ctx)
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        r = rg.align(A, B, K, config=cfg, ctx=ctx)
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{os.environ.get('RGBID_LIB', 'in-tree')} levels={levels}: median {statistics.median(ts):.3f} ms "
          f"min {min(ts):.3f} iterations {r.total_iterations if hasattr(r, 'total_iterations') else '?'}")
