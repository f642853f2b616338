"""the back-end callers of the hot path on the B200.

* loop-closure dense refinement (src/loop.cpp:174-203) against its restatement
  over the reference build, and run on a second context / host thread while the
  front-end tracks on the first (the two-stream model of PAPER:876-877);
* normal_map (src/segmentation.cpp:10-57) bit for bit against the reference
  build (the source compiles unchanged against the Eigen shim);
* export_map (src/pipeline.cpp:463-527) bit for bit against its restatement.
"""
import threading

import numpy as np
import pytest

import paper_1807_08271_b200 as rg
from oracle import map_oracle
from oracle.oracle import Oracle

from .scenes import N_SLANT, pair

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return rg.Context(0)


def bits(a):
    """bit patterns, NaNs canonicalised (payloads differ between libraries)"""
    a = np.ascontiguousarray(a, dtype=np.float64).copy()
    a[np.isnan(a)] = np.nan
    return a.view(np.uint64)


# --------------------------------------------------------------------------- normal_map

@pytest.mark.parametrize("size", [(80, 60, 60.0), (640, 480, 480.0)])
def test_normal_map_bitexact(ctx, size):
    K = rg.simple_intrinsics(*size)
    fa, fb, _ = pair(K, 3, "noisy", holes=True)
    for W in (fa.inverse_depth, fb.inverse_depth):
        g = rg.normal_map(W, K, ctx)
        o = Oracle("REF").normal_map(W, K.to_c())
        for a, b in zip((g.nx, g.ny, g.nz), o):
            assert np.array_equal(bits(a), bits(b))  # signed zeros of -e_z included
    # degenerate pixels: isolated valid pixel -> -e_z
    W = np.full((60, 80), np.nan)
    W[30, 40] = 0.5
    g = rg.normal_map(W, K if size[0] == 80 else rg.simple_intrinsics(80, 60, 60.0), ctx)
    assert bits([g.nx[30, 40], g.ny[30, 40], g.nz[30, 40]]).tolist() == \
        bits([-0.0, -0.0, -1.0]).tolist()
    assert np.isnan(g.nx[0, 0])


# --------------------------------------------------------------------------- export_map

def _keyframes(K, n=3):
    kfs = []
    for k in range(n):
        T = rg.Pose(np.eye(3), [0.02 * k, 0.0, 0.0]) if k else rg.Pose()
        f = rg.render_plane(K, T, N_SLANT, -2.0, K.width / 80.0)
        f = rg.add_noise(f, 500 + k, 0.005, 0.002)
        rng = np.random.default_rng(k)
        f.inverse_depth[rng.random(f.inverse_depth.shape) < 0.03] = np.nan
        kfs.append(rg.make_keyframe(f, T, k, float(k)))
    return kfs


@pytest.mark.parametrize("voxel", [0.0, 0.05, 0.2])
def test_export_map_matches_restatement(ctx, voxel):
    K = rg.simple_intrinsics(80, 60, 60.0)
    kfs = _keyframes(K)
    cloud = rg.export_map(kfs, K, voxel, ctx)
    op, oc = map_oracle.export_map(
        [(k.intensity, k.inverse_depth, k.T_W_kf.to_c()) for k in kfs], K.to_c(), voxel)
    assert cloud.points.shape == op.shape and len(op) > 0
    assert np.array_equal(bits(cloud.points), bits(op))
    assert np.array_equal(cloud.colors, oc)
    if voxel == 0.0:
        # later keyframes add only pixels the previous one does not explain
        assert len(op) < sum(np.isfinite(k.inverse_depth).sum() for k in kfs)


def test_export_map_empty_and_capacity(ctx):
    K = rg.simple_intrinsics(80, 60, 60.0)
    assert len(rg.export_map([], K, 0.0, ctx).points) == 0
    kf = _keyframes(K, 1)[0]
    kf.inverse_depth[:] = np.nan
    assert len(rg.export_map([kf], K, 0.1, ctx).points) == 0


# --------------------------------------------------------------------------- loop constraint

def test_loop_constraint_matches_reference(ctx):
    K = rg.simple_intrinsics(80, 60, 60.0)
    fa, fb, T_WB = pair(K, 5, "noisy")
    lc = rg.make_loop_constraint(fa, fb, 7, 42, rg.Pose(), K, inliers=15, hull_fraction=0.3,
                                 ctx=ctx)
    o = map_oracle.make_loop_constraint((fa.intensity, fa.inverse_depth),
                                        (fb.intensity, fb.inverse_depth), rg.Pose().to_c(),
                                        K.to_c())
    assert lc is not None and o is not None
    assert (lc.i, lc.j, lc.inliers, lc.hull_fraction) == (7, 42, 15, 0.3)
    To = rg.Pose.from_c(o[0])
    assert np.allclose(lc.T_ij.R, To.R, atol=1e-5) and np.allclose(lc.T_ij.t, To.t, atol=1e-5)
    assert np.allclose(lc.info, lc.info.T)
    assert np.allclose(lc.info, o[1], rtol=1e-4, atol=1e-6 * np.abs(o[1]).max())


def test_loop_constraint_gates(ctx):
    K = rg.simple_intrinsics(80, 60, 60.0)
    fa, fb, _ = pair(K, 5, "noisy")
    # refined-overlap gate: min_covisibility above any achievable ratio -> nullopt
    assert rg.make_loop_constraint(fa, fb, 0, 1, rg.Pose(), K,
                                   config=rg.LoopConfig(min_covisibility=1.01), ctx=ctx) is None
    # degenerate alignment (flat, textureless frames) -> nullopt, like the reference
    flat = rg.FrameData(np.full((60, 80), 0.5), np.full((60, 80), 0.5))
    assert rg.make_loop_constraint(flat, flat, 0, 1, rg.Pose(), K, ctx=ctx) is None
    assert map_oracle.make_loop_constraint((flat.intensity, flat.inverse_depth),
                                           (flat.intensity, flat.inverse_depth),
                                           rg.Pose().to_c(), K.to_c()) is None


def test_loop_refinement_concurrent_with_tracking():
    """Front-end tracking on context 1 (thread A) while loop constraints refine on
    context 2 (thread B): each context owns its stream and workspaces, so the
    results equal those of the same calls run alone."""
    K = rg.simple_intrinsics(80, 60, 60.0)
    frames = [rg.render_plane(K, rg.Pose(np.eye(3), [0.004 * i, 0.0, 0.0]), N_SLANT, -2.0, 1.0)
              for i in range(12)]
    pairs = [pair(K, 10 + i, "noisy")[:2] for i in range(4)]

    def track(c):
        fe = rg.Frontend(K, ctx=c)
        out = [fe.process_frame(f, float(i)) for i, f in enumerate(frames)]
        return [(e.T_W_k.R.copy(), e.T_W_k.t.copy()) for e in out]

    def loops(c):
        res = []
        for a, b in pairs:
            lc = rg.make_loop_constraint(a, b, 0, 1, rg.Pose(), K, ctx=c)
            res.append(None if lc is None else (lc.T_ij.R.copy(), lc.T_ij.t.copy(), lc.info))
        return res

    c1, c2 = rg.Context(0), rg.Context(0)
    solo_track, solo_loops = track(c1), loops(c2)
    got = {}
    ta = threading.Thread(target=lambda: got.__setitem__("t", track(c1)))
    tb = threading.Thread(target=lambda: got.__setitem__("l", loops(c2)))
    ta.start(), tb.start()
    ta.join(), tb.join()
    for (Ra, ta_), (Rb, tb_) in zip(got["t"], solo_track):
        assert np.array_equal(Ra, Rb) and np.array_equal(ta_, tb_)
    for x, y in zip(got["l"], solo_loops):
        assert (x is None) == (y is None)
        if x is not None:
            assert all(np.array_equal(u, v) for u, v in zip(x, y))
