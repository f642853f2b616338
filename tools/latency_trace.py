import ctypes as C, os, sys, statistics
sys.path.insert(0, os.getcwd())
import torch
import paper_1807_08271_b200 as rg
ctx = rg.Context(0)
L = ctx.lib
L.rgbid_debug_tdist_phases.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
K = rg.simple_intrinsics(640, 480, 480.0)
A, B = rg.DeviceFrame(640, 480, ctx), rg.DeviceFrame(640, 480, ctx)
rg.synth_pair_device(A, B, K, 0, 1)
cfg = rg.AlignmentConfig(levels=4)
s = torch.cuda.ExternalStream(ctx.stream_ptr)
buf = (C.c_ulonglong * 24)()
for _ in range(3):
    rg.align(A, B, K, config=cfg, ctx=ctx)
L.rgbid_debug_tdist_phases(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
r = rg.align(A, B, K, config=cfg, ctx=ctx)
e1.record(s); e1.synchronize()
L.rgbid_debug_tdist_phases(buf, 1)
ctas = buf[10]
print(f"align {e0.elapsed_time(e1):.3f} ms, iterations {r.total_iterations}, tdist CTAs {ctas}")
names = {0: "gather", 12: "gather: tile-count scan (cumulative)", 13: "gather: + search/walk",
         14: "gather: + value loads", 1: "loc_scale", 4: "stationarity", 8: "allsum", 7: "kernel"}
for k, v in names.items():
    print(f"  {v}: {buf[k] / ctas / 1.95e3:.1f} us per CTA, x launches {ctas/16:.0f} = {buf[k]/16/1.95e6:.3f} ms")
ns = max(buf[21], 1)
print(f"k_solve ({ns} launches), thread 0, us per launch:")
for k, v in {16: "reduce partials", 17: "ldlt_solve6", 18: "pose_update", 19: "warp_mats",
             20: "whole kernel (from the slot check)"}.items():
    print(f"  {v}: {buf[k] / ns / 1.95e3:.2f}")
ctx.set_profiling(True); ctx.reset_stats()
rg.align(A, B, K, config=cfg, ctx=ctx); ctx.synchronize()
st = ctx.kernel_stats(); ctx.set_profiling(False)
tot = sum(v[1] for v in st.values())
print(f"profiled (event per launch, no graph): sum {tot:.3f} ms")
for k, v in sorted(st.items(), key=lambda kv: -kv[1][1])[:8]:
    print(f"   {k:24s} n={v[0]:4d} {v[1]:.3f} ms {v[1]/v[0]*1e3:.1f} us/launch")
