"""Quick GPU probe: parity summary + timings (dev tool, not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1807_08271_b200 as rg
from oracle.oracle import Oracle
from tests.scenes import pair, vga

ctx = rg.Context(0)
orc = Oracle("C")
K = vga()
for variant in ("noisy",):
    fa, fb, T = pair(K, 1, variant, holes=(variant == "noisy"))
    cfg = rg.AlignmentConfig(levels=4)
    t0 = time.time(); res, tr = rg.align(fa, fb, K, config=cfg, ctx=ctx, trace=True); t1 = time.time()
    o, otr = orc.align(fa.intensity, fa.inverse_depth, fb.intensity, fb.inverse_depth, K.to_c(), None, cfg.to_c(), trace=True)
    t2 = time.time()
    To = rg.Pose.from_c(o.T_AB)
    print(variant, "gpu %.1f ms (first call) oracle %.1f ms" % ((t1-t0)*1e3, (t2-t1)*1e3))
    print("  dt", np.abs(res.T_AB.t - To.t).max(), "dR", np.abs(res.T_AB.R - To.R).max(), "truth err", np.abs(res.T_AB.t - T.t).max())
    print("  iters", [l.iterations for l in res.level_log], [l.iterations for l in o.level_log[:o.n_levels]])
    for g, c in zip(tr, otr):
        Hg, Hc = np.array(g.H[:]), np.array(c.H[:])
        print("   L%d it%d nj %d/%d nd %d/%d H %.2e nuI %.4f/%.4f nuW %.4f/%.4f sW %.6g/%.6g" % (g.level, g.iter, g.n_jets, c.n_jets, g.n_depth, c.n_depth,
              np.abs(Hg-Hc).max()/np.abs(Hc).max(), g.tI.nu, c.tI.nu, g.tW.nu, c.tW.nu, g.tW.sigma, c.tW.sigma))
    # timing: device-resident latency
    A = rg.DeviceFrame.from_frame(fa, ctx); B = rg.DeviceFrame.from_frame(fb, ctx)
    for _ in range(3): rg.align(A, B, K, config=cfg, ctx=ctx)
    ctx.synchronize(); t0 = time.time(); n = 10
    for _ in range(n): rg.align(A, B, K, config=cfg, ctx=ctx)
    print("  latency (device frames, 4-lvl): %.3f ms" % ((time.time()-t0)/n*1e3))
# batch throughput
nb = int(os.environ.get("NB", "128"))
As = [rg.DeviceFrame(640, 480, ctx) for _ in range(nb)]; Bs = [rg.DeviceFrame(640, 480, ctx) for _ in range(nb)]
for i in range(nb): rg.synth_pair_device(As[i], Bs[i], K, i, i % 2)
cfg = rg.AlignmentConfig(levels=4)
rg.align_batch(As, Bs, K, config=cfg, ctx=ctx)
ctx.synchronize(); t0 = time.time()
out = rg.align_batch(As, Bs, K, config=cfg, ctx=ctx)
dt = time.time() - t0
print("batch %d: %.1f ms -> %.0f align/s; statuses %s; iters mean %.1f" % (nb, dt*1e3, nb/dt, set(r.status for r in out), np.mean([r.total_iterations for r in out])))
print("launches", ctx.kernel_launches)
