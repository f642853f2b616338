"""CPU tier: the host-side bookkeeping of the path (FrameBuffer,
src/fusion.cpp:97-111), ported from the reference's tests/test_fusion.cpp:163-183."""
import paper_1807_08271_b200 as rg


def _bf(t):
    return rg.BufferedFrame(rg.FrameData(None, None), rg.Pose(), t)


def test_frame_buffer_pops_the_temporally_closest_frame():
    b = rg.FrameBuffer(30)
    for t in (1.0, 2.0, 3.0, 5.0):
        b.push(_bf(t))
    assert b.pop_closest(4.9).timestamp == 5.0
    assert b.pop_closest(1.4).timestamp == 1.0
    assert b.size() == 2


def test_frame_buffer_respects_its_capacity():
    b = rg.FrameBuffer(3)
    for t in (1.0, 2.0, 3.0, 4.0):
        b.push(_bf(t))
    assert b.size() == 3
    assert b.pop_closest(0.0).timestamp == 2.0  # the oldest (t = 1) was dropped


def test_frame_buffer_ties_keep_the_first_and_empty_pops_none():
    b = rg.FrameBuffer(30)
    for t in (1.0, 3.0):
        b.push(_bf(t))
    assert b.pop_closest(2.0).timestamp == 1.0  # |dt| tie: the first wins
    assert b.pop_closest(2.0).timestamp == 3.0
    assert b.empty() and b.pop_closest(0.0) is None


def test_digamma_host_helper_matches_oracle_and_kat():
    """src/alignment.cpp:32-43; known answers of tests/test_alignment.cpp:47-55"""
    import math
    from oracle.oracle import Oracle
    o = Oracle("C")
    for x in (0.5, 1.0, 2.5, 5.0, 7.25, 13.0):
        assert rg.digamma(x) == o.digamma(x)
    g = 0.5772156649015329
    assert abs(rg.digamma(1.0) + g) < 1e-8
    assert abs(rg.digamma(0.5) + g + 2 * math.log(2.0)) < 1e-8
    assert abs(rg.digamma(5.0) - 1.5061176684318003) < 1e-8


def test_batch_plan_splits_for_two_lanes():
    """rgbid_batch_plan (runtime.cu batch_chunk): <= 1024-slot chunks in whole lane
    pairs; a batch of >= 64 pairs is split in two so both lanes co-schedule (512
    pairs per GPU at 8 GPUs -> 2 x 256)."""
    import ctypes as C
    from paper_1807_08271_b200 import abi
    L = abi.lib()

    def plan(n):
        c, k = C.c_int(), C.c_int()
        assert L.rgbid_batch_plan(n, C.byref(c), C.byref(k)) == 0
        return c.value, k.value

    assert plan(4096) == (1024, 4)
    assert plan(512) == (256, 2)
    assert plan(2049) == (513, 4)
    assert plan(63) == (63, 1)
    assert plan(64) == (32, 2)
    assert plan(0) == (0, 0)


def test_bench_scene_hole_variant():
    """Variant 2 of the bench scene (synth_scene.cuh): 5% random W holes, 2% I holes
    and a w/32-pixel W border band on both frames, integer-hashed; variant 1 has none."""
    import numpy as np
    from oracle import oracle as O
    K = rg.simple_intrinsics(640, 480, 480.0).to_c()
    IA, WA, IB, WB, _ = O.synth_pair_host(K, 5, 2)
    b = 640 // 32
    for W in (WA, WB):
        assert np.isnan(W[:b]).all() and np.isnan(W[:, -b:]).all() and np.isnan(W[-b:]).all()
        inner = W[b:-b, b:-b]
        assert 0.04 < np.isnan(inner).mean() < 0.06
    for I in (IA, IB):
        assert 0.015 < np.isnan(I).mean() < 0.025
    IA1, WA1, _, _, _ = O.synth_pair_host(K, 5, 1)
    assert np.isfinite(WA1).all() and np.isfinite(IA1).all()
    # the product library renders the identical pair (same source, same hashing)
    fa, fb, _ = rg.synth_pair_host(rg.simple_intrinsics(640, 480, 480.0), 5, 2)
    assert np.array_equal(fa.inverse_depth, WA, equal_nan=True)
    assert np.array_equal(fb.intensity, IB, equal_nan=True)
