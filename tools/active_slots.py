"""Active slots per (level, iteration) of a batched align of the bench scene: how much of
each graph launch works (a converged slot's CTAs exit at their slot check)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_08271_b200 as rg

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ctx = rg.Context(0)
K = rg.simple_intrinsics(640, 480, 480.0)
A = [rg.DeviceFrame(640, 480, ctx) for _ in range(n)]
B = [rg.DeviceFrame(640, 480, ctx) for _ in range(n)]
for i in range(n):
    rg.synth_pair_device(A[i], B[i], K, i, 1 + (i & 1))
its = [10, 5, 4, 5]
out = rg.align_batch(A, B, K, config=rg.AlignmentConfig(levels=4, iterations=its), ctx=ctx)
ok = [rg.AlignmentResult.from_c(r) for r in out if r.status == 0]
print(f"{len(ok)} of {n} ok; mean iterations {sum(r.total_iterations for r in ok) / len(ok):.2f}")
tot_launch, tot_active = 0, 0
for lvl in (3, 2, 1, 0):
    row = []
    for it in range(its[lvl]):
        act = sum(1 for r in ok for l in r.level_log if l.level == lvl and l.iterations > it)
        row.append(act)
        tot_launch += 1
        tot_active += act
    print(f"level {lvl}: active per iteration {row}")
print(f"mean active fraction over the {tot_launch} iteration launches: {tot_active / (tot_launch * len(ok)):.3f}")
