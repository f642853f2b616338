"""Small driver for ncu captures: one batched align of N device-rendered bench pairs
(--iters 0: the bench's iterations {10,5,4,5}; --variant mixed: bench.py's scene mix)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_08271_b200 as rg

p = argparse.ArgumentParser()
p.add_argument("--pairs", type=int, default=512)
p.add_argument("--levels", type=int, default=1)
p.add_argument("--iters", type=int, default=2)
p.add_argument("--repeat", type=int, default=1)
p.add_argument("--variant", default="1")
a = p.parse_args()
ctx = rg.Context(0)
K = rg.simple_intrinsics(640, 480, 480.0)
A = [rg.DeviceFrame(640, 480, ctx) for _ in range(a.pairs)]
B = [rg.DeviceFrame(640, 480, ctx) for _ in range(a.pairs)]
for i in range(a.pairs):
    rg.synth_pair_device(A[i], B[i], K, i, 1 + (i & 1) if a.variant == "mixed" else int(a.variant))
iters = [10, 5, 4] if a.iters == 0 else [a.iters] * a.levels
cfg = rg.AlignmentConfig(levels=a.levels, iterations=iters)
for _ in range(a.repeat):
    out = rg.align_batch(A, B, K, config=cfg, ctx=ctx)
print("ok", sum(r.status == 0 for r in out), "of", len(out),
      "iterations", sum(r.total_iterations for r in out if r.status == 0))
