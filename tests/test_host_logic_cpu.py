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
