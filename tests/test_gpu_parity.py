"""GPU parity: the CUDA path (through the C-ABI) against the oracle on identical
inputs.  Bars (BASELINE.json north_star): bit-exact masks / maps / pyramid,
normal-equation sums within 1e-4 relative, pose within 1e-5 rad / 1e-5 m,
fused keyframe inverse depth within 1e-5 relative."""
import numpy as np
import pytest

import paper_1807_08271_b200 as rg
from oracle.oracle import Oracle
from tests.scenes import N_SLANT, bitwise_equal, pair, vga

pytestmark = pytest.mark.gpu

POSE_TOL = 1e-5
SUM_TOL = 1e-4


@pytest.fixture(scope="module")
def ctx():
    return rg.Context(0)


@pytest.fixture(scope="module")
def orc():
    return Oracle("C")


def rot_angle(R):
    return float(np.linalg.norm(rg.so3_log(R)))


@pytest.mark.parametrize("size", [(80, 60, 60.0), (640, 480, 480.0)])
@pytest.mark.parametrize("variant,holes", [("clean", False), ("noisy", True)])
def test_warp_maps_bitwise(ctx, orc, size, variant, holes):
    K = rg.simple_intrinsics(*size)
    fa, fb, T = pair(K, 3, variant, holes)
    for T_AB in (T, rg.random_pose(41, 0.02, 0.02), rg.Pose()):
        g = rg.inverse_geometric_warp(fb.intensity, fb.inverse_depth, fa.inverse_depth, T_AB, K, ctx)
        o = orc.inverse_geometric_warp(fb.intensity, fb.inverse_depth, fa.inverse_depth,
                                       T_AB.to_c(), K.to_c())
        for a, b in zip((g.intensity, g.inverse_depth, g.map_x, g.map_y), o):
            assert bitwise_equal(a, b)


@pytest.mark.parametrize("levels", [1, 3, 4, 6])
def test_pyramid_bitwise(ctx, orc, levels):
    K = vga()
    fa, _, _ = pair(K, 0, "noisy", True)
    g = rg.build_pyramid(fa, K, levels, ctx)
    oI, oW, oK = orc.build_pyramid(fa.intensity, fa.inverse_depth, K.to_c(), levels)
    for l in range(levels):
        assert bitwise_equal(g.levels[l].intensity, oI[l])
        assert bitwise_equal(g.levels[l].inverse_depth, oW[l])
        assert (g.intrinsics[l].fx, g.intrinsics[l].cx, g.intrinsics[l].width) == \
            (oK[l].fx, oK[l].cx, oK[l].width)


def _check_align(res, o, tol=POSE_TOL):
    To = rg.Pose.from_c(o.T_AB)
    assert np.abs(res.T_AB.t - To.t).max() < tol
    assert rot_angle(res.T_AB.R @ To.R.T) < tol
    assert [l.iterations for l in res.level_log] == [l.iterations for l in o.level_log[: o.n_levels]]
    for l, lo in zip(res.level_log, o.level_log[: o.n_levels]):
        assert l.level == lo.level
        assert abs(l.final_cost - lo.final_cost) <= SUM_TOL * abs(lo.final_cost) + 1e-12
    assert res.tdist_depth.sigma == pytest.approx(o.tdist_depth.sigma, rel=1e-6)
    assert res.tdist_intensity.nu == pytest.approx(o.tdist_intensity.nu, rel=1e-6, abs=1e-6)
    cov_o = np.array(o.cov[:]).reshape(6, 6)
    assert np.abs(res.cov - cov_o).max() <= 1e-4 * np.abs(cov_o).max()
    assert res.cov_degenerate == bool(o.cov_degenerate)


@pytest.mark.parametrize("size", [(80, 60, 60.0), (320, 240, 240.0), (640, 480, 480.0)])
@pytest.mark.parametrize("variant", ["clean", "noisy"])
@pytest.mark.parametrize("levels", [3, 4])
def test_align_matches_oracle(ctx, orc, size, variant, levels):
    K = rg.simple_intrinsics(*size)
    fa, fb, _ = pair(K, 1, variant, holes=(variant == "noisy"))
    cfg = rg.AlignmentConfig(levels=levels)
    o = orc.align(fa.intensity, fa.inverse_depth, fb.intensity, fb.inverse_depth, K.to_c(), None,
                  cfg.to_c())
    if o.status == 1:
        # The reference itself throws here: on a noiseless plane the depth scale
        # collapses (sigma_W ~ 1e-7) and the equilibrated H drops below 1e-9.
        with pytest.raises(rg.DegenerateAlignmentError) as e:
            rg.align(fa, fb, K, config=cfg, ctx=ctx)
        so = np.array(o.spectrum[:])
        assert np.allclose(np.sort(e.value.spectrum)[3:], so[3:], rtol=1e-6)
        assert np.sort(e.value.spectrum)[0] < 1e-9
        return
    res = rg.align(fa, fb, K, config=cfg, ctx=ctx)
    _check_align(res, o)


def test_iteration_trace_matches_oracle(ctx, orc):
    """Per-iteration n_jets / n_depth (exact), Student-t parameters, H and b
    (relative 1e-4, b by norm) while the iterates agree."""
    K = vga()
    fa, fb, _ = pair(K, 2, "noisy", holes=True)
    cfg = rg.AlignmentConfig(levels=4)
    res, tr = rg.align(fa, fb, K, config=cfg, ctx=ctx, trace=True)
    o, otr = orc.align(fa.intensity, fa.inverse_depth, fb.intensity, fb.inverse_depth, K.to_c(),
                       None, cfg.to_c(), trace=True)
    assert len(tr) == len(otr) > 0
    for g, c in zip(tr, otr):
        assert (g.level, g.iter, g.n_jets, g.n_depth) == (c.level, c.iter, c.n_jets, c.n_depth)
        Hg, Hc = np.array(g.H[:]).reshape(6, 6), np.array(c.H[:]).reshape(6, 6)
        assert np.abs(Hg - Hc).max() <= SUM_TOL * np.abs(Hc).max()
        bg, bc = np.array(g.b[:]), np.array(c.b[:])
        assert np.linalg.norm(bg - bc) <= SUM_TOL * np.linalg.norm(bc) + 1e-9 * np.abs(Hc).max()
        for a, b in ((g.tI, c.tI), (g.tW, c.tW)):
            assert a.mu == pytest.approx(b.mu, rel=1e-6, abs=1e-12)
            assert a.sigma == pytest.approx(b.sigma, rel=1e-6)
            assert a.nu == pytest.approx(b.nu, rel=1e-6)


def test_identity_alignment(ctx):
    """test_alignment.cpp:198-205"""
    K = rg.simple_intrinsics(80, 60)
    f = rg.render_plane(K, rg.Pose())
    res = rg.align(f, f, K, ctx=ctx)
    assert np.linalg.norm(res.T_AB.t) < 1e-9
    assert rot_angle(res.T_AB.R) < 1e-9
    assert res.converged


def test_known_motion_recovered(ctx):
    """test_alignment.cpp:207-233 at 80x60 and the VGA config-1 scene."""
    K = rg.simple_intrinsics(80, 60)
    T_WB = rg.Pose(rg.so3_exp([0, np.pi / 180.0, 0]), [0.005, 0, 0])
    n = np.array([0.2, -0.15, 1])
    n /= np.linalg.norm(n)
    fa = rg.render_plane(K, rg.Pose(), n, -2.0)
    fb = rg.render_plane(K, T_WB, n, -2.0)
    res = rg.align(fa, fb, K, ctx=ctx)
    assert np.linalg.norm(res.T_AB.t - T_WB.t) < 5e-4
    assert rot_angle(res.T_AB.R @ T_WB.R.T) < 0.05 * np.pi / 180.0
    bad = fb.copy()
    bad.intensity[:, : K.width // 5] = 0.9
    bad.inverse_depth[:, : K.width // 5] = 1.0
    rb = rg.align(fa, bad, K, ctx=ctx)
    assert np.linalg.norm(rb.T_AB.t - T_WB.t) <= max(2 * np.linalg.norm(res.T_AB.t - T_WB.t), 1e-3)


def test_degenerate_throws(ctx):
    """test_alignment.cpp:294-301"""
    K = rg.simple_intrinsics(40, 30)
    f = rg.FrameData(np.full((30, 40), np.nan), np.full((30, 40), np.nan))
    with pytest.raises(rg.DegenerateAlignmentError) as e:
        rg.align(f, f, K, ctx=ctx)
    assert np.all(e.value.spectrum == 0.0)


def test_bilateral_matches_oracle(ctx, orc):
    K = vga()
    fa, _, _ = pair(K, 0, "noisy", True)
    for img, sr in ((fa.intensity, 0.05), (fa.inverse_depth, 0.02)):
        g = rg.bilateral_filter(img, 2.0, sr, ctx)
        o = orc.bilateral_filter(img, 2.0, sr)
        assert bitwise_equal(np.isnan(g), np.isnan(o))
        m = ~np.isnan(o)
        assert np.abs(g[m] - o[m]).max() <= 1e-14 * np.abs(o[m]).max()


@pytest.mark.parametrize("shape", [(23, 37), (9, 33), (480, 640)])
def test_bilateral_ragged_and_nonfinite(ctx, orc, shape):
    """tiles cut by the image border, +-inf and NaN taps (is_valid = isfinite),
    far-apart values whose weights underflow to zero"""
    rng = np.random.default_rng(shape[0])
    img = rng.random(shape)
    img[rng.random(shape) < 0.05] = np.nan
    img[rng.random(shape) < 0.02] = np.inf
    img[rng.random(shape) < 0.02] = -np.inf
    img[rng.random(shape) < 0.05] *= 1e3
    for sr in (0.05, 0.5):
        g = rg.bilateral_filter(img, 2.0, sr, ctx)
        o = orc.bilateral_filter(img, 2.0, sr)
        assert bitwise_equal(np.isnan(g), np.isnan(o))
        m = ~np.isnan(o)
        assert np.abs(g[m] - o[m]).max() <= 1e-14 * np.abs(o[m]).max()


def test_filtered_hessian_covariance(ctx, orc):
    K = vga()
    fa, fb, T = pair(K, 4, "noisy", True)
    cov, deg = rg.filtered_hessian_covariance(fa, fb, K, T, ctx=ctx)
    co, dego = orc.filtered_hessian_covariance(fa.intensity, fa.inverse_depth, fb.intensity,
                                               fb.inverse_depth, K.to_c(), T.to_c())
    assert deg == dego
    assert np.abs(cov - co).max() <= 1e-4 * np.abs(co).max()
    assert np.abs(cov - cov.T).max() == 0.0


def test_fusion_20_frames(ctx, orc):
    """config 2: 20 noisy frames fused into one keyframe (1e-5 relative bar)."""
    K = vga()
    base = rg.render_plane(K, rg.Pose(), N_SLANT, -2.0, 8.0)
    kf = rg.make_keyframe(rg.add_noise(base, 1, 0.0, 0.01), rg.Pose(), 0, 0.0)
    kfo_W, kfo_C = kf.inverse_depth.copy(), kf.weight.copy()
    for k in range(20):
        T = rg.random_pose(3000 + k, 0.01, 0.01)
        f = rg.add_noise(rg.render_plane(K, T, N_SLANT, -2.0, 8.0), 100 + k, 0.0, 0.01)
        rg.integrate_frame(kf, f, T, K, 0.05, ctx)
        orc.integrate_frame(None, kfo_W, kfo_C, f.intensity, f.inverse_depth, T.to_c(), K.to_c(),
                            0.05)
    assert bitwise_equal(np.isnan(kf.inverse_depth), np.isnan(kfo_W))
    m = ~np.isnan(kfo_W)
    rel = np.abs(kf.inverse_depth[m] - kfo_W[m]) / np.abs(kfo_W[m])
    assert rel.max() <= 1e-5
    assert np.abs(kf.weight - kfo_C).max() <= 1e-5 * np.abs(kfo_C).max()
    # beyond the bar: the per-pixel arithmetic is the reference's, in its order
    # (correctly rounded shared-divisor quotients), so the fused maps are bit-exact
    assert bitwise_equal(kf.inverse_depth, kfo_W) and bitwise_equal(kf.weight, kfo_C)


def test_fused_multi_frame_kernel_equals_sequential(ctx):
    K = rg.simple_intrinsics(160, 120, 120.0)
    base = rg.render_plane(K, rg.Pose(), N_SLANT, -2.0, 2.0)
    kf_seq = rg.make_keyframe(base, rg.Pose(), 0, 0.0)
    frames, poses = [], []
    for k in range(6):
        T = rg.random_pose(3000 + k, 0.01, 0.01)
        f = rg.add_noise(rg.render_plane(K, T, N_SLANT, -2.0, 2.0), 10 + k, 0.0, 0.005)
        frames.append(f)
        poses.append(T)
        rg.integrate_frame(kf_seq, f, T, K, 0.05, ctx)
    import ctypes as C
    from paper_1807_08271_b200 import abi
    kf = rg.DeviceFrame.from_frame(base, ctx)
    dfs = [rg.DeviceFrame.from_frame(f, ctx) for f in frames]
    import torch
    Cmap = torch.ones((120, 160), dtype=torch.float64, device="cuda")
    arr = (C.c_void_p * 6)(*[d.h.value for d in dfs])
    Ps = (abi.Pose_t * 6)(*[p.to_c() for p in poses])
    ctx.check(ctx.lib.rgbid_integrate_frames(ctx.h, kf.h, C.cast(Cmap.data_ptr(), abi.DP), 6, arr,
                                             Ps, C.byref(K.to_c()), 0.05), "integrate_frames")
    out = kf.download()
    assert bitwise_equal(out.inverse_depth, kf_seq.inverse_depth)
    assert bitwise_equal(Cmap.cpu().numpy(), kf_seq.weight)


def test_covisibility_counts_exact(ctx, orc):
    K = vga()
    fa, fb, T = pair(K, 5, "noisy", True)
    for T_BA in (T.inverse(), rg.Pose(), rg.Pose(np.eye(3), [0.5, 0, 0])):
        g = rg.covisibility_ratio(fa, fb, T_BA, K, 0.01, ctx)
        r, e, counts = orc.covisibility_ratio(fa.intensity, fa.inverse_depth, fb.intensity,
                                              fb.inverse_depth, T_BA.to_c(), K.to_c(), 0.01)
        assert list(g.counts) == counts
        assert g.ratio == r and g.empty_frame == e


def test_correct_inverse_depth_bitwise(ctx, orc):
    K = vga()
    fa, _, _ = pair(K, 0, "noisy", True)
    d = rg.DepthIntrinsics(beta0=-0.005, beta1=1.02, q0=(0.002, 1e-4, -1e-4, 0, 0, 0, 0, 0, 0),
                           q1=(1.01, 1e-3, 0, 5e-4, 0, 0, 0, 0, 0), p0=(4.0, 4.0))
    for spatial in (False, True):
        g = rg.correct_inverse_depth(fa.inverse_depth, d, K, spatial, ctx)
        o = orc.correct_inverse_depth(fa.inverse_depth, d.to_c(), K.to_c(), spatial)
        assert bitwise_equal(g, o)


def test_forward_register_bitwise(ctx, orc):
    K = vga()
    fa, _, _ = pair(K, 0, "clean", False)
    for T_BA in (rg.random_pose(7, 0.025, 0.01), rg.Pose(np.eye(3), [-0.3, 0, 0]), rg.Pose()):
        g = rg.forward_register(fa.inverse_depth, T_BA, K, K, ctx)
        o = orc.forward_register(fa.inverse_depth, T_BA.to_c(), K.to_c(), K.to_c())
        assert bitwise_equal(g, o)


def test_batch_equals_single(ctx):
    K = rg.simple_intrinsics(160, 120, 120.0)
    cfg = rg.AlignmentConfig(levels=3)
    pairs = [pair(K, i, "noisy" if i % 2 else "clean") for i in range(5)]
    A = [rg.DeviceFrame.from_frame(p[0], ctx) for p in pairs]
    B = [rg.DeviceFrame.from_frame(p[1], ctx) for p in pairs]
    out = rg.align_batch(A, B, K, config=cfg, ctx=ctx)
    for i, p in enumerate(pairs):
        single = rg.align(p[0], p[1], K, config=cfg, ctx=ctx)
        r = rg.rgbid._result_or_raise(out[i])
        assert np.array_equal(r.T_AB.R, single.T_AB.R) and np.array_equal(r.T_AB.t, single.T_AB.t)
        assert np.array_equal(r.cov, single.cov)


def test_deterministic_replay(ctx):
    K = vga()
    fa, fb, _ = pair(K, 6, "noisy", True)
    r1 = rg.align(fa, fb, K, ctx=ctx)
    r2 = rg.align(fa, fb, K, ctx=ctx)
    assert np.array_equal(r1.T_AB.R, r2.T_AB.R) and np.array_equal(r1.T_AB.t, r2.T_AB.t)
    assert np.array_equal(r1.cov, r2.cov)


def test_selftest_division_bitwise(ctx):
    import ctypes as C
    bad = C.c_ulonglong(0)
    ctx.check(ctx.lib.rgbid_selftest_division(ctx.h, 200_000_000, 12345, C.byref(bad)), "selftest")
    assert bad.value == 0


def test_kernels_launched(ctx):
    K = rg.simple_intrinsics(80, 60)
    f = rg.render_plane(K, rg.Pose())
    n0 = ctx.kernel_launches
    rg.align(f, f, K, ctx=ctx)
    assert ctx.kernel_launches > n0


def _config4_inputs(K, i=0):
    """W_m synthesised in a depth camera at T_DC =
    random_pose(7, 0.025, 0.01), K_ir = K_rgb, beta0 = -0.005, beta1 = 1.02."""
    T_DC = rg.random_pose(7, 0.025, 0.01)
    T_WB = rg.random_pose(1000 + i, 0.003, 0.02)
    fa = rg.render_plane(K, rg.Pose(), N_SLANT, -2.0, K.width / 80.0)
    fb = rg.render_plane(K, T_WB, N_SLANT, -2.0, K.width / 80.0)
    d = rg.DepthIntrinsics(beta0=-0.005, beta1=1.02, p0=(0.0, 0.0))
    # what the depth sensor reports: the inverse depth seen from the depth camera,
    # passed through the inverse of the linear correction
    depth_views = []
    for T_WC in (rg.Pose(), T_WB):
        T_WD = T_WC * T_DC.inverse()
        Wd = rg.render_plane(K, T_WD, N_SLANT, -2.0).inverse_depth
        depth_views.append((Wd - d.beta0) / d.beta1)
    return fa, fb, T_DC, d, depth_views


def test_config4_unregistered_depth_path(ctx, orc):
    """correct_inverse_depth -> forward_register (T_CD = T_DC^-1) -> 4-level align,
    GPU vs oracle at every stage (bit-exact maps, pose within 1e-5)."""
    K = rg.simple_intrinsics(320, 240, 240.0)
    fa, fb, T_DC, d, (Wm_a, Wm_b) = _config4_inputs(K)
    frames = []
    for f, Wm in ((fa, Wm_a), (fb, Wm_b)):
        g = rg.correct_inverse_depth(Wm, d, K, False, ctx)
        o = orc.correct_inverse_depth(Wm, d.to_c(), K.to_c(), False)
        assert bitwise_equal(g, o)
        T_CD = T_DC.inverse()
        gr = rg.forward_register(g, T_CD, K, K, ctx)
        orr = orc.forward_register(o, T_CD.to_c(), K.to_c(), K.to_c())
        assert bitwise_equal(gr, orr)
        assert np.isfinite(gr).mean() > 0.8
        frames.append(rg.FrameData(f.intensity, gr))
    cfg = rg.AlignmentConfig(levels=4)
    o = orc.align(frames[0].intensity, frames[0].inverse_depth, frames[1].intensity,
                  frames[1].inverse_depth, K.to_c(), None, cfg.to_c())
    if o.status != 0:
        with pytest.raises(rg.DegenerateAlignmentError):
            rg.align(frames[0], frames[1], K, config=cfg, ctx=ctx)
        return
    res = rg.align(frames[0], frames[1], K, config=cfg, ctx=ctx)
    _check_align(res, o)


def test_frame_decode_bitwise(ctx, orc):
    """Frame ingest (src/dataset.cpp:97-116) on the GPU equals the restatement bit for bit."""
    rng = np.random.default_rng(3)
    bgr = rng.integers(0, 256, size=(480, 640, 3), dtype=np.uint8)
    depth = rng.integers(0, 65535, size=(480, 640), dtype=np.uint16)
    depth[rng.random((480, 640)) < 0.05] = 0
    f = rg.DeviceFrame(640, 480, ctx)
    f.decode(bgr, depth, 5000.0)
    g = f.download()
    I, W = orc.decode_frame(bgr, depth, 5000.0)
    assert bitwise_equal(g.intensity, I) and bitwise_equal(g.inverse_depth, W)


@pytest.mark.parametrize("size,levels", [((97, 71, 70.0), 3), ((320, 240, 240.0), 4)])
def test_batch_throughput_path_matches_oracle(ctx, orc, size, levels):
    """> 8 pairs take the throughput path (k_gather + k_tdist<NT> instead of the
    cluster kernel): each result against the oracle, ragged sizes included."""
    K = rg.simple_intrinsics(*size)
    cfg = rg.AlignmentConfig(levels=levels)
    pairs = [pair(K, 20 + i, "noisy", holes=bool(i % 2)) for i in range(12)]
    A = [rg.DeviceFrame.from_frame(p[0], ctx) for p in pairs]
    B = [rg.DeviceFrame.from_frame(p[1], ctx) for p in pairs]
    out = rg.align_batch(A, B, K, config=cfg, ctx=ctx)
    checked = 0
    for (fa, fb, _), r in zip(pairs, out):
        o = orc.align(fa.intensity, fa.inverse_depth, fb.intensity, fb.inverse_depth, K.to_c(),
                      None, cfg.to_c())
        assert (r.status == 1) == (o.status == 1)
        if o.status == 0:
            _check_align(rg.rgbid._result_or_raise(r), o)
            checked += 1
    assert checked >= 8


@pytest.mark.parametrize("size", [(97, 71, 70.0), (333, 251, 250.0)])
def test_align_ragged_sizes(ctx, orc, size):
    """Widths/heights that are not multiples of the K1 tiles or of 2^levels."""
    K = rg.simple_intrinsics(*size)
    fa, fb, _ = pair(K, 2, "noisy", holes=True)
    for levels in (3, 4):
        cfg = rg.AlignmentConfig(levels=levels)
        o = orc.align(fa.intensity, fa.inverse_depth, fb.intensity, fb.inverse_depth, K.to_c(),
                      None, cfg.to_c())
        if o.status == 1:
            with pytest.raises(rg.DegenerateAlignmentError):
                rg.align(fa, fb, K, config=cfg, ctx=ctx)
            continue
        _check_align(rg.align(fa, fb, K, config=cfg, ctx=ctx), o)


def test_align_1280x960(ctx, orc):
    """A frame 4x VGA: 4800 level-0 K1 tiles, larger scans and shared-memory tables."""
    K = rg.simple_intrinsics(1280, 960, 960.0)
    fa, fb, _ = pair(K, 4, "noisy", holes=True)
    cfg = rg.AlignmentConfig(levels=4)
    o = orc.align(fa.intensity, fa.inverse_depth, fb.intensity, fb.inverse_depth, K.to_c(), None,
                  cfg.to_c())
    assert o.status == 0
    _check_align(rg.align(fa, fb, K, config=cfg, ctx=ctx), o)


def test_all_hole_inputs(ctx, orc):
    """Empty inputs (every pixel a hole): align throws like the reference (fewer than
    6 jets, zero spectrum) on both the single-pair and the batch path; fusion leaves
    the keyframe untouched; covisibility reports an empty frame."""
    K = rg.simple_intrinsics(80, 60, 60.0)
    nan = np.full((60, 80), np.nan)
    empty = rg.FrameData(nan.copy(), nan.copy())
    good, fb, _ = pair(K, 3, "noisy")
    o = orc.align(empty.intensity, empty.inverse_depth, fb.intensity, fb.inverse_depth,
                  K.to_c(), None, rg.AlignmentConfig().to_c())
    assert o.status == 1
    with pytest.raises(rg.DegenerateAlignmentError) as e:
        rg.align(empty, fb, K, ctx=ctx)
    assert np.all(np.array(e.value.spectrum) == 0.0)
    # batch (throughput path): empty pairs fail alone
    A = [rg.DeviceFrame.from_frame(empty if i % 3 == 0 else good, ctx) for i in range(10)]
    B = [rg.DeviceFrame.from_frame(fb, ctx) for _ in range(10)]
    out = rg.align_batch(A, B, K, ctx=ctx)
    assert [r.status for r in out] == [1 if i % 3 == 0 else 0 for i in range(10)]
    # fusion with an empty frame: keyframe unchanged (W and C)
    kf = rg.make_keyframe(good, rg.Pose(), 0, 0.0)
    W0, C0 = kf.inverse_depth.copy(), kf.weight.copy()
    rg.integrate_frame(kf, empty, rg.Pose(), K, 0.01, ctx)
    assert bitwise_equal(kf.inverse_depth, W0) and bitwise_equal(kf.weight, C0)
    cv = rg.covisibility_ratio(empty, good, rg.Pose(), K, 0.01, ctx)
    ro, eo, _ = orc.covisibility_ratio(empty.intensity, empty.inverse_depth, good.intensity,
                                       good.inverse_depth, rg.Pose().to_c(), K.to_c(), 0.01)
    assert cv.empty_frame and eo and cv.ratio == ro == 0.0


def test_synth_pair_host_equals_device(ctx):
    """The reference arm renders the benchmark's pairs on the host; they equal the
    device rendering of the timed arm up to host-vs-device libm rounding."""
    K = rg.simple_intrinsics(640, 480, 480.0)
    for seed in (0, 7):
        A, B = rg.DeviceFrame(640, 480, ctx), rg.DeviceFrame(640, 480, ctx)
        rg.synth_pair_device(A, B, K, seed, 1)
        ha, hb, _ = rg.synth_pair_host(K, seed, 1)
        for d, h in ((A.download(), ha), (B.download(), hb)):
            for x, y in ((d.intensity, h.intensity), (d.inverse_depth, h.inverse_depth)):
                assert np.array_equal(np.isnan(x), np.isnan(y))
                m = ~np.isnan(x)
                assert np.abs(x[m] - y[m]).max() <= 1e-12


def test_align_batch_host_async_equals_sync(ctx):
    """Streaming host batches (rgbid_align_batch_host_async + _wait, consecutive calls
    overlapping) give the same results as the synchronous call, bit for bit."""
    import ctypes as C
    from paper_1807_08271_b200 import abi
    K = rg.simple_intrinsics(160, 120, 120.0)
    pairs = [pair(K, 30 + i, "noisy") for i in range(20)]
    maps = [np.ascontiguousarray(m) for p in pairs for m in (p[0].intensity, p[0].inverse_depth,
                                                             p[1].intensity, p[1].inverse_depth)]
    arrs = [(abi.DP * 20)(*[abi.dptr(maps[4 * i + k]) for i in range(20)]) for k in range(4)]
    cfg = rg.AlignmentConfig(levels=3).to_c()
    Kc = K.to_c()
    sync = (abi.AlignResult_t * 20)()
    ctx.check(ctx.lib.rgbid_align_batch_host(ctx.h, 20, *arrs, 160, 120, C.byref(Kc), None,
                                             C.byref(cfg), 6, sync), "sync")
    outs = [(abi.AlignResult_t * 20)() for _ in range(3)]
    for o in outs:  # three streamed calls, chunks of 6 over two lanes
        ctx.check(ctx.lib.rgbid_align_batch_host_async(ctx.h, 20, *arrs, 160, 120, C.byref(Kc),
                                                       None, C.byref(cfg), 6, o), "async")
    ctx.check(ctx.lib.rgbid_align_batch_host_wait(ctx.h), "wait")
    for o in outs:
        for a, b in zip(o, sync):
            assert bytes(a) == bytes(b)


def test_drain_buffer_semantics(ctx):
    """tests/test_fusion.cpp:185-210 on the device: draining an empty buffer is a
    no-op; three buffered frames are all integrated (C = 1 + 3)."""
    K = rg.simple_intrinsics(20, 16, 20.0)
    f = rg.render_plane(K, rg.Pose())
    kf = rg.make_keyframe(f, rg.Pose(), 0, 0.0)
    before = kf.inverse_depth.copy()
    rg.drain_buffer_step(kf, rg.FrameBuffer(30), K, 0.01, ctx)
    assert bitwise_equal(kf.inverse_depth, before)
    base = rg.FrameData(np.full((16, 20), 0.5), np.full((16, 20), 0.5))
    kf = rg.make_keyframe(base, rg.Pose(), 0, 0.0)
    buf = rg.FrameBuffer(30)
    for t in (0.1, 0.2, 0.3):
        buf.push(rg.BufferedFrame(base, rg.Pose(), t))
    for _ in range(3):
        rg.drain_buffer_step(kf, buf, K, 0.05, ctx)
    assert buf.empty() and kf.weight[8, 10] == pytest.approx(4.0)


@pytest.mark.parametrize("size", [(80, 60, 60.0), (640, 480, 480.0)])
def test_residuals_and_jacobians_bitwise(ctx, orc, size):
    """src/alignment.cpp:195-250 through the C-ABI: the jet set, order, residuals,
    Jacobians and has_depth flags equal the oracle's bit for bit; lambda_n within a
    few ulp (the device normalises n and the ray with rsqrt, src/alignment.cpp:233-244
    divides by sqrt)."""
    K = rg.simple_intrinsics(*size)
    fa, fb, T = pair(K, 8, "noisy", holes=True)
    wp = rg.inverse_geometric_warp(fb.intensity, fb.inverse_depth, fa.inverse_depth, T, K, ctx)
    jets, flags = rg.residuals_and_jacobians(fa, wp, K, ctx=ctx, as_array=True)
    jo, fo = orc.residuals_and_jacobians(fa.intensity, fa.inverse_depth, wp.intensity,
                                         wp.inverse_depth, K.to_c())
    assert jets.shape == jo.shape and len(jets) > 100
    assert bitwise_equal(jets[:, :16], jo[:, :16]) and np.array_equal(flags, fo)
    rel = np.abs(jets[:, 16] - jo[:, 16]) / np.abs(jo[:, 16])
    assert rel.max() <= 1e-14, f"lambda_n max relative difference {rel.max():.2e}"
    first = rg.residuals_and_jacobians(fa, wp, K, ctx=ctx)[0]
    assert (first.x, first.y) == (int(jo[0, 0]), int(jo[0, 1]))


def test_student_t_entry_points_match_oracle(ctx, orc):
    """estimate_location_scale / estimate_nu (src/alignment.cpp:61-127) through the
    C-ABI on t-distributed and Gaussian residuals, above and below the 19200 cap."""
    rng = np.random.default_rng(5)
    for n, nu_true in ((5000, 3.0), (50000, 6.0)):
        r = 0.1 + 0.8 * rng.standard_t(nu_true, size=n)
        for nu in (5.0, nu_true):
            g = rg.estimate_location_scale(r, nu, ctx)
            o = orc.estimate_location_scale(r, nu)
            assert g.mu == pytest.approx(o[0], rel=1e-9, abs=1e-12)
            assert g.sigma == pytest.approx(o[1], rel=1e-9)
        mu, s, _ = orc.estimate_location_scale(r, 5.0)
        assert rg.estimate_nu(r, mu, s, ctx) == pytest.approx(orc.estimate_nu(r, mu, s), rel=1e-9)
    gauss = rng.normal(size=30000)
    mu, s, _ = orc.estimate_location_scale(gauss, 10.0)
    assert rg.estimate_nu(gauss, mu, s, ctx) == pytest.approx(orc.estimate_nu(gauss, mu, s))


def test_inverse_warp_bitwise(ctx):
    """src/warping.cpp:8-18 with include/rgbid/image.hpp:51-62 bilinear, restated in
    plain Python floats; f_w as a vectorised and as a scalar callable."""
    rng = np.random.default_rng(3)
    src = rng.random((16, 20))
    src[5, 7] = np.nan

    def bil(img, x, y):
        h, w = img.shape
        if not (0 <= x <= w - 1 and 0 <= y <= h - 1):
            return np.nan
        x0, y0 = int(np.floor(x)), int(np.floor(y))
        x1, y1 = min(x0 + 1, w - 1), min(y0 + 1, h - 1)
        fx, fy = x - x0, y - y0
        v = [img[y0, x0], img[y0, x1], img[y1, x0], img[y1, x1]]
        if not all(np.isfinite(v)):
            return np.nan
        return (1 - fy) * ((1 - fx) * v[0] + fx * v[1]) + fy * ((1 - fx) * v[2] + fx * v[3])

    f_vec = lambda p: (0.9 * p[0] + 0.37, 1.05 * p[1] - 0.2)  # noqa: E731
    f_sca = lambda p: np.array([0.9 * p[0] + 0.37, 1.05 * p[1] - 0.2])  # noqa: E731
    ref = np.array([[bil(src, 0.9 * x + 0.37, 1.05 * y - 0.2) for x in range(22)]
                    for y in range(15)])
    assert bitwise_equal(rg.inverse_warp(src, f_vec, 22, 15, ctx), ref)
    assert bitwise_equal(rg.inverse_warp(src, f_sca, 22, 15, ctx), ref)


@pytest.mark.parametrize("case", ["tight_core", "tiny_scale", "two_clusters", "heavy_tail_low_nu",
                                  "huge_scale"])
def test_student_t_stress_samples(ctx, orc, case):
    """The device location/scale update uses sum w d^2 = c2 (m - c1 sum 1/q), which
    cancels when most d^2 << c1 = nu sigma^2: samples whose bulk
    is far tighter than the scale the outliers impose, a scale near the 1e-8 floor,
    two separated clusters, a t(1.2) tail that drives nu into the bisection, and
    residuals of ~1e40 whose 4-sample fractions overflow (the exact per-sample path).
    GPU vs the oracle (the reference's sequential sums) at the 1e-6 bar."""
    rng = np.random.default_rng({"tight_core": 11, "tiny_scale": 12, "two_clusters": 13,
                                 "heavy_tail_low_nu": 14, "huge_scale": 15}[case])
    n = 19200
    if case == "tight_core":
        r = np.where(rng.random(n) < 0.97, rng.normal(0.01, 1e-6, n), rng.normal(0.0, 1.0, n))
    elif case == "tiny_scale":
        r = 0.5 + rng.normal(0.0, 3e-8, n)
    elif case == "two_clusters":
        r = np.where(rng.random(n) < 0.7, rng.normal(-0.2, 1e-4, n), rng.normal(0.3, 1e-4, n))
    elif case == "huge_scale":  # q ~ 1e80: a 4-sample fraction's D overflows -> exact path
        r = 1e40 * rng.standard_t(3.0, size=n)
    else:
        r = 0.02 * rng.standard_t(1.2, size=n)
    for nu in (5.0, 2.5, 10.0):
        g = rg.estimate_location_scale(r, nu, ctx)
        o = orc.estimate_location_scale(r, nu)
        assert g.mu == pytest.approx(o[0], rel=1e-6, abs=1e-12 + 1e-6 * o[1])
        assert g.sigma == pytest.approx(o[1], rel=1e-6)
    mu, s, _ = orc.estimate_location_scale(r, 5.0)
    assert rg.estimate_nu(r, mu, s, ctx) == pytest.approx(orc.estimate_nu(r, mu, s), rel=1e-6)


def test_solve_nu_grid_search_matches_bisection(ctx, orc):
    """solve_nu (src/alignment.cpp:131-157): the reference bisects [2, 10] 30 times, so
    its nu is the midpoint of the grid cell [2 + k 2^-27, 2 + (k+1) 2^-27] where the
    stationarity changes sign.  The device finds that cell by regula falsi on the grid
    index (~10 passes instead of 32): same nu unless the root sits within rounding
    noise of a grid point.  200 samples of varied shape, size and tail weight, most
    with an interior root (the full search), against the oracle's bisection."""
    rng = np.random.default_rng(2024)
    exact, interior, worst = 0, 0, 0.0
    cases = 200
    for i in range(cases):
        n = int(rng.choice([40, 700, 5000, 19200, 45000]))
        nu_true = float(rng.uniform(1.5, 14.0))
        scale = float(10.0 ** rng.uniform(-4, 0))
        r = float(rng.normal(0, 0.1)) + scale * rng.standard_t(nu_true, size=n)
        if i % 5 == 0:  # contamination: a broad outlier component
            k = max(1, n // 10)
            r[rng.choice(n, size=k, replace=False)] = rng.normal(0, 30 * scale, size=k)
        mu, s, _ = orc.estimate_location_scale(r, 5.0)
        g, o = rg.estimate_nu(r, mu, s, ctx), orc.estimate_nu(r, mu, s)
        exact += g == o
        interior += 2.0 < o < 10.0
        worst = max(worst, abs(g - o))
    assert interior >= cases // 2, interior
    assert worst <= 1e-6, worst
    assert exact >= int(0.9 * cases), f"{exact} of {cases} bit-identical"
