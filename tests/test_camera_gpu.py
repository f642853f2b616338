"""Distorted sensors (SURVEY §8(f) rank 2, config 4 with k != 0): the rectification
map f_w = K distort(K^-1 p) and the iterative undistort on the device, against the
reference build (oracle/_ref: src/camera.cpp:11-45 and src/warping.cpp:8-18
composed through their own API), then the whole unregistered-depth path on
rectified frames -- correct_inverse_depth -> forward_register -> 4-level align."""
import numpy as np
import pytest

import paper_1807_08271_b200 as rg
from oracle import oracle as O
from tests.scenes import bitwise_equal

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not O.available("REF"), reason="reference build absent")

KDIST = (0.08, -0.05, 0.0012, -0.0009, 0.01)  # k1, k2, p1, p2, k3 (inc/camera.hpp:14-20)


@pytest.fixture(scope="module")
def ctx():
    return rg.Context(0)


@pytest.fixture(scope="module")
def ref():
    return O.Oracle("REF")


def _distorted(K):
    return rg.Intrinsics(K.fx, K.fy, K.cx, K.cy, KDIST, K.width, K.height)


@needs_ref
@pytest.mark.parametrize("size", [(160, 120, 120.0), (640, 480, 480.0)])
def test_rectify_bitwise(ctx, ref, size):
    """Rectified maps equal the reference's inverse_warp(project(distort)) bit for bit,
    holes (NaN taps, out-of-image sources) included."""
    K = _distorted(rg.simple_intrinsics(*size))
    fa, fb, _ = rg.synth_pair_host(rg.simple_intrinsics(*size), 11, 2)
    for img in (fa.intensity, fa.inverse_depth, fb.inverse_depth):
        g = rg.rectify(img, K, ctx)
        o = ref.rectify(img, K.to_c())
        assert bitwise_equal(g, o)
        assert np.isfinite(o).mean() > 0.5
    # device-resident form: both maps of a frame in one launch
    src = rg.DeviceFrame.from_frame(fb, ctx)
    dst = rg.DeviceFrame(K.width, K.height, ctx)
    out = rg.rectify_frame(src, K, dst).download()
    assert bitwise_equal(out.intensity, ref.rectify(fb.intensity, K.to_c()))
    assert bitwise_equal(out.inverse_depth, ref.rectify(fb.inverse_depth, K.to_c()))


@needs_ref
def test_undistort_points_bitwise(ctx, ref):
    """Fixed-point undistortion: the same iterates and the same std::nullopt cases
    (a strongly distorted lens where the iteration does not converge)."""
    rng = np.random.default_rng(5)
    m_d = rng.uniform(-0.8, 0.8, size=(20000, 2))
    K = _distorted(rg.simple_intrinsics(640, 480, 480.0))
    for k in (KDIST, (0.0,) * 5, (0.6, 0.4, 0.02, -0.02, 0.3)):
        Kk = rg.Intrinsics(K.fx, K.fy, K.cx, K.cy, k, K.width, K.height)
        mu, ok = rg.undistort_points(m_d, Kk, ctx)
        mo, oko = ref.undistort(m_d, Kk.to_c())
        assert np.array_equal(ok, oko)
        assert bitwise_equal(mu[ok], mo[oko])
    assert not oko.all()  # the strong lens exercises the nullopt path


@needs_ref
def test_config4_distorted_sensor_path(ctx, ref):
    """Raw distorted RGB and depth frames -> rectify -> correct_inverse_depth ->
    forward_register -> 4-level align: device vs the reference build at every stage
    (bit-exact maps, pose 1e-5, iterations exact)."""
    K0 = rg.simple_intrinsics(320, 240, 240.0)
    K = _distorted(K0)
    fa, fb, _ = rg.synth_pair_host(K0, 4, 1)
    d = rg.DepthIntrinsics(beta0=-0.005, beta1=1.02, p0=(0.0, 0.0))
    T_DC = rg.random_pose(7, 0.025, 0.01)
    frames, oframes = [], []
    for f in (fa, fb):
        I_g, I_o = rg.rectify(f.intensity, K, ctx), ref.rectify(f.intensity, K.to_c())
        Wm = (f.inverse_depth - d.beta0) / d.beta1  # raw depth-sensor reading
        W_g, W_o = rg.rectify(Wm, K, ctx), ref.rectify(Wm, K.to_c())
        assert bitwise_equal(I_g, I_o) and bitwise_equal(W_g, W_o)
        c_g = rg.correct_inverse_depth(W_g, d, K0, False, ctx)
        c_o = ref.correct_inverse_depth(W_o, d.to_c(), K0.to_c(), False)
        assert bitwise_equal(c_g, c_o)
        r_g = rg.forward_register(c_g, T_DC.inverse(), K0, K0, ctx)
        r_o = ref.forward_register(c_o, T_DC.inverse().to_c(), K0.to_c(), K0.to_c())
        assert bitwise_equal(r_g, r_o)
        frames.append(rg.FrameData(I_g, r_g))
        oframes.append((I_o, r_o))
    cfg = rg.AlignmentConfig(levels=4)
    o = ref.align(oframes[0][0], oframes[0][1], oframes[1][0], oframes[1][1], K0.to_c(), None,
                  cfg.to_c())
    if o.status != 0:
        with pytest.raises(rg.DegenerateAlignmentError):
            rg.align(frames[0], frames[1], K0, config=cfg, ctx=ctx)
        return
    res = rg.align(frames[0], frames[1], K0, config=cfg, ctx=ctx)
    To = rg.Pose.from_c(o.T_AB)
    assert np.abs(res.T_AB.t - To.t).max() < 1e-5
    assert np.linalg.norm(rg.so3_log(res.T_AB.R @ To.R.T)) < 1e-5
    assert [l.iterations for l in res.level_log] == [l.iterations for l in o.level_log[:4]]
