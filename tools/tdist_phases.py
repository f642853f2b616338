"""Phase breakdown of the throughput-mode Student-t kernel (k_tdist) per level.

Needs an instrumented build:  RGBID_NVFLAGS=-DRGBID_TDIST_TRACE python
paper_1807_08271_b200/build.py -f   (rebuild without the flag afterwards).
Counters are SM clocks summed over CTAs (thread 0 of each CTA).
"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_08271_b200 as rg

ctx = rg.Context(0)
L = ctx.lib
L.rgbid_debug_tdist_phases.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
K = rg.simple_intrinsics(640, 480, 480.0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512  # n <= 8: latency mode (cluster kernel)
A = [rg.DeviceFrame(640, 480, ctx) for _ in range(n)]
B = [rg.DeviceFrame(640, 480, ctx) for _ in range(n)]
for i in range(n):
    rg.synth_pair_device(A[i], B[i], K, i, 1)
buf = (C.c_ulonglong * 24)()
names = {0: "gather", 1: "loc_scale", 4: "stationarity", 6: "stat_pass", 8: "allsum", 7: "kernel",
         3: "ls_iters(count)", 9: "allsums(count)", 2: "ls_calls(count)", 5: "stat_calls(count)"}
for lv in range(-1, 4):
    # one iteration at level `lv` only (levels = lv + 1, zero iterations on the finer
    # levels); lv = -1: no iterations at all -> the final covariance's refit only
    its = [0] * lv + [1] if lv >= 0 else [0]
    cfg = rg.AlignmentConfig(levels=max(lv, 0) + 1, iterations=its)
    rg.align_batch(A, B, K, config=cfg, ctx=ctx)
    L.rgbid_debug_tdist_phases(buf, 1)
    for f in A: f.invalidate()
    rg.align_batch(A, B, K, config=cfg, ctx=ctx)
    L.rgbid_debug_tdist_phases(buf, 1)
    ctas = max(buf[10], 1)
    per = {v: buf[k] / ctas for k, v in names.items()}
    print(f"level {lv}: ctas={buf[10]} mean m={buf[11] / ctas:.0f} loc_scale calls/cta={buf[2] / ctas:.2f} "
          f"iters/cta={buf[3] / ctas:.1f} stationarity calls/cta={buf[5] / ctas:.1f} "
          f"allsums/cta={buf[9] / ctas:.0f}")
    print("   clocks/cta: " + ", ".join(f"{k}={v:,.0f}" for k, v in per.items()))
