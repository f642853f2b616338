"""Single-pair latency breakdown (dev tool)."""
import os, sys, statistics, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1807_08271_b200 as rg

ctx = rg.Context(0)
K = rg.simple_intrinsics(640, 480, 480.0)
A, B = rg.DeviceFrame(640, 480, ctx), rg.DeviceFrame(640, 480, ctx)
rg.synth_pair_device(A, B, K, 0, 1)
stream = torch.cuda.ExternalStream(ctx.stream_ptr)
for levels, iters in ((4, [10, 5, 4]), (3, [10, 5, 4])):
    cfg = rg.AlignmentConfig(levels=levels, iterations=iters)
    for _ in range(3):
        r = rg.align(A, B, K, config=cfg, ctx=ctx)
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream); rg.align(A, B, K, config=cfg, ctx=ctx); e1.record(stream); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"levels={levels}: align median {statistics.median(ts):.3f} ms, iterations {r.total_iterations}")
    ctx.set_profiling(True); ctx.reset_stats(); rg.align(A, B, K, config=cfg, ctx=ctx); ctx.synchronize()
    st = ctx.kernel_stats(); ctx.set_profiling(False)
    tot = sum(v[1] for v in st.values())
    for k, v in sorted(st.items(), key=lambda kv: -kv[1][1])[:8]:
        print(f"   {k:22s} n={v[0]:4d} {v[1]:8.3f} ms  {v[1]/v[0]*1e3:8.1f} us/launch")
    print(f"   sum of kernel times {tot:.3f} ms")
