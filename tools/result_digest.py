"""Digest of the alignment results of a fixed workload (64 mixed-scene bench pairs as
one batch, 4 levels, and the first pair alone in latency mode), for bit-identity
checks of a change that must not alter results:  RGBID_LIB=... python tools/result_digest.py"""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_08271_b200 as rg
ctx = rg.Context(0)
K = rg.simple_intrinsics(640, 480, 480.0)
n = 64
A = [rg.DeviceFrame(640, 480, ctx) for _ in range(n)]
B = [rg.DeviceFrame(640, 480, ctx) for _ in range(n)]
for i in range(n):
    rg.synth_pair_device(A[i], B[i], K, i, 1 + (i & 1))
cfg = rg.AlignmentConfig(levels=4, iterations=[10, 5, 4, 5])
h = hashlib.sha256()
for r in rg.align_batch(A, B, K, config=cfg, ctx=ctx):
    h.update(bytes(r))
hb = h.hexdigest()[:16]
r1 = rg.align(A[1], B[1], K, config=cfg, ctx=ctx)
h1 = hashlib.sha256(repr((r1.T_AB.R.tobytes(), r1.T_AB.t.tobytes(), r1.cov.tobytes(),
                         [(l.level, l.iterations, l.final_cost) for l in r1.level_log])).encode()).hexdigest()[:16]
print(f"{os.environ.get('RGBID_LIB', 'in-tree')}: batch {hb} single {h1}")
