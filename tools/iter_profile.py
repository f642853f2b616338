"""Per-launch kernel times across IRLS iterations (how much do converged slots cost?)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_08271_b200 as rg
ctx = rg.Context(0)
K = rg.simple_intrinsics(640, 480, 480.0)
n = 512
A = [rg.DeviceFrame(640, 480, ctx) for _ in range(n)]
B = [rg.DeviceFrame(640, 480, ctx) for _ in range(n)]
for i in range(n):
    rg.synth_pair_device(A[i], B[i], K, i, 1 + (i & 1))
cfg = rg.AlignmentConfig(levels=4, iterations=[10, 5, 4])
rg.align_batch(A, B, K, config=cfg, ctx=ctx)
lib = ctx.lib
import ctypes as C
# per-launch records: enable profiling and read the raw stats after each launch group is not
# exposed; instead time whole aligns with eps=0 (no early exit) vs default
import torch
stream = torch.cuda.ExternalStream(ctx.stream_ptr)
for eps in (1e-6, 0.0):
    c = rg.AlignmentConfig(levels=4, iterations=[10, 5, 4], convergence_eps=eps)
    for f in A: f.invalidate()
    rg.align_batch(A, B, K, config=c, ctx=ctx)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for f in A: f.invalidate()
    torch.cuda.synchronize(); e0.record(stream)
    out = rg.align_batch(A, B, K, config=c, ctx=ctx)
    e1.record(stream); torch.cuda.synchronize()
    its = sum(r.total_iterations for r in out) / n
    print(f"eps={eps}: {e0.elapsed_time(e1):.1f} ms for {n} pairs, mean iterations {its:.2f}")
