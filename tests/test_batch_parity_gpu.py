"""Parity of the TIMED batched path (config 5).

bench.py's `value` comes from rgbid_align_batch with chunks co-scheduled in one
two-lane CUDA graph (runtime.cu launch_prepared(LB != nullptr) / enqueue_align_pair:
cross-lane events, stage offsets, per-lane workspaces).  These tests force that
path on small batches (RGBID_BATCH_SLOTS, read on every call; chunks > 8 slots, so
the Student-t stage is the batch kernels k_gather + k_tdist_big of the timed run,
not the <= 8-slot latency-mode cluster kernel) and check it against
  * the reference build (oracle/_ref, the unmodified reference sources) on the
    identical host-rendered 640x480 bench pairs, 4 levels: pose 1e-5, per-level
    iteration counts exact, per-level cost and covariance 1e-4 (north_star bars,
    semantics of /root/reference/proj/src/alignment.cpp:367-409);
  * itself: bit-identical results with RGBID_NO_PAIRS=1, with one chunk, across a
    sequence of batch sizes that re-captures / re-uses cached graphs while the
    lanes' workspaces grow, and through the host-buffer streaming entry points.
"""
import ctypes as C
import os

import numpy as np
import pytest

import paper_1807_08271_b200 as rg
from paper_1807_08271_b200 import abi
from oracle import oracle as O

pytestmark = pytest.mark.gpu

N_PAIRS = 40
LEVELS = 4


@pytest.fixture(scope="module")
def ctx():
    return rg.Context(0)


@pytest.fixture(scope="module")
def K():
    return rg.simple_intrinsics(640, 480, 480.0)


@pytest.fixture(scope="module")
def cfg():
    return rg.AlignmentConfig(levels=LEVELS, iterations=[10, 5, 4])


@pytest.fixture(scope="module")
def pairs(K):
    """bench pairs 0..39 (even: noisy+occluder, odd: + holes and border band),
    rendered on the host exactly as the reference arm renders them"""
    out = []
    for i in range(N_PAIRS):
        IA, WA, IB, WB, _ = O.synth_pair_host(K.to_c(), i, 1 + (i & 1))
        out.append((IA, WA, IB, WB))
    return out


@pytest.fixture(scope="module")
def frames(ctx, pairs):
    A = [rg.DeviceFrame.from_frame(rg.FrameData(p[0], p[1]), ctx) for p in pairs]
    B = [rg.DeviceFrame.from_frame(rg.FrameData(p[2], p[3]), ctx) for p in pairs]
    return A, B


@pytest.fixture(scope="module")
def ref_results(K, cfg, pairs):
    kind = "REF" if O.available("REF") else "C"
    return O.Oracle(kind).align_many(pairs, K.to_c(), None, cfg.to_c(), threads=os.cpu_count() or 1)


class _env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        for k, v in self.kv.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = str(v)

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _batch(ctx, K, cfg, A, B, idx, slots=None, no_pairs=False):
    with _env(RGBID_BATCH_SLOTS=slots, RGBID_NO_PAIRS=1 if no_pairs else None):
        return rg.align_batch([A[i] for i in idx], [B[i] for i in idx], K, config=cfg, ctx=ctx)


def _key(r):
    """every field of the result record, as bytes (bit-equality)"""
    return bytes(r)


def _check_vs_ref(g, o):
    assert g.status == o.status
    if o.status != 0:
        return
    Tg, To = rg.Pose.from_c(g.T_AB), rg.Pose.from_c(o.T_AB)
    assert np.abs(Tg.t - To.t).max() < 1e-5
    assert np.linalg.norm(rg.so3_log(Tg.R @ To.R.T)) < 1e-5
    assert [g.level_log[k].iterations for k in range(LEVELS)] == \
        [o.level_log[k].iterations for k in range(LEVELS)]
    for k in range(LEVELS):
        assert g.level_log[k].level == o.level_log[k].level
        assert abs(g.level_log[k].final_cost - o.level_log[k].final_cost) <= \
            1e-4 * abs(o.level_log[k].final_cost)
    cg, co = np.array(g.cov[:]), np.array(o.cov[:])
    assert np.abs(cg - co).max() <= 1e-4 * np.abs(co).max()
    assert g.cov_degenerate == o.cov_degenerate


def test_coscheduled_pairs_match_reference(ctx, K, cfg, frames, ref_results):
    """40 VGA bench pairs through the co-scheduled two-lane graph (10-slot chunks:
    two launches of one cached (10, 10) chunk-pair graph) against the reference build."""
    A, B = frames
    res = _batch(ctx, K, cfg, A, B, range(N_PAIRS), slots=10)
    assert sum(r.status == 0 for r in ref_results) >= N_PAIRS - 2
    for g, o in zip(res, ref_results):
        _check_vs_ref(g, o)


def test_coscheduled_bitwise_equals_serial(ctx, K, cfg, frames):
    """The stage-offset co-scheduling changes nothing: bit-identical to the same
    chunks run one after another (RGBID_NO_PAIRS=1) and to one 40-slot chunk."""
    A, B = frames
    idx = range(N_PAIRS)
    paired = _batch(ctx, K, cfg, A, B, idx, slots=10)
    serial = _batch(ctx, K, cfg, A, B, idx, slots=10, no_pairs=True)
    single = _batch(ctx, K, cfg, A, B, idx, slots=N_PAIRS)
    for a, b, c in zip(paired, serial, single):
        assert _key(a) == _key(b) == _key(c)


def test_graph_cache_across_batch_sizes(ctx, K, cfg, frames):
    """A sequence of batch shapes that sizes lane 0 for 20 slots, captures a (9, 9)
    pair graph, grows only lane 1's workspace (12, 12), then hits the (9, 9) key
    again (the graph must not replay lane 1's freed buffers), plus unequal (11, 10)
    chunks: every result bit-identical to the pair aligned in a one-chunk batch."""
    A, B = frames
    base = {i: _key(r) for i, r in zip(range(N_PAIRS), _batch(ctx, K, cfg, A, B, range(N_PAIRS),
                                                               slots=N_PAIRS))}
    seq = [(20, range(0, 20)), (9, range(0, 18)), (12, range(10, 34)), (9, range(20, 38)),
           (11, range(3, 24)), (9, [39, 38, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16])]
    for slots, idx in seq:
        idx = list(idx)
        res = _batch(ctx, K, cfg, A, B, idx, slots=slots)
        for i, r in zip(idx, res):
            assert _key(r) == base[i], (slots, idx, i)


def test_host_streaming_calls_complete_previous_lanes(ctx, K, cfg, pairs):
    """rgbid_align_batch_host_async: a call that reuses only lane 0 still completes
    lane 1's chunk of the previous call before it returns, and the
    results equal the device-frame batch bit for bit."""
    n1, n2 = 20, 9
    cfg_c, K_c = cfg.to_c(), K.to_c()

    def arrays(idx):
        return [(abi.DP * len(idx))(*[pairs[i][k].ctypes.data_as(abi.DP) for i in idx])
                for k in range(4)]

    idx1, idx2 = list(range(n1)), list(range(n1, n1 + n2))
    a1, a2 = arrays(idx1), arrays(idx2)
    r1 = (abi.AlignResult_t * n1)()
    r2 = (abi.AlignResult_t * n2)()
    ctx.check(ctx.lib.rgbid_align_batch_host_async(ctx.h, n1, *a1, 640, 480, C.byref(K_c), None,
                                                   C.byref(cfg_c), 10, r1), "async 1")
    ctx.check(ctx.lib.rgbid_align_batch_host_async(ctx.h, n2, *a2, 640, 480, C.byref(K_c), None,
                                                   C.byref(cfg_c), 10, r2), "async 2")
    done1 = [bytes(r) for r in r1]  # call 2 returned: every result of call 1 is written
    ctx.check(ctx.lib.rgbid_align_batch_host_wait(ctx.h), "wait")
    A = [rg.DeviceFrame.from_frame(rg.FrameData(p[0], p[1]), ctx) for p in pairs[:n1 + n2]]
    B = [rg.DeviceFrame.from_frame(rg.FrameData(p[2], p[3]), ctx) for p in pairs[:n1 + n2]]
    ref = _batch(ctx, K, cfg, A, B, range(n1 + n2), slots=n1 + n2)
    assert done1 == [_key(r) for r in ref[:n1]]
    assert [bytes(r) for r in r2] == [_key(r) for r in ref[n1:]]


@pytest.mark.parametrize("variant", [0, 1, 2])
def test_device_scene_equals_host_scene(ctx, K, variant):
    """bench.py times device-rendered pairs and checks parity on host-rendered ones:
    the same scene model (synth_scene.cuh) -- identical hole patterns (integer hashing)
    and values equal up to libm's last bits (CUDA vs glibc sin/cos/log)."""
    for i in (3, 4):
        A, B = rg.DeviceFrame(640, 480, ctx), rg.DeviceFrame(640, 480, ctx)
        T_dev = rg.synth_pair_device(A, B, K, i, variant)
        IA, WA, IB, WB, T_host = O.synth_pair_host(K.to_c(), i, variant)
        fa, fb = A.download(), B.download()
        assert bytes(T_dev.to_c()) == bytes(T_host)
        for g, h in ((fa.intensity, IA), (fa.inverse_depth, WA), (fb.intensity, IB),
                     (fb.inverse_depth, WB)):
            assert np.array_equal(np.isnan(g), np.isnan(h))
            m = ~np.isnan(h)
            assert np.abs(g[m] - h[m]).max() <= 1e-12


def test_coscheduled_batch_with_failing_pairs(ctx, K, cfg, pairs, frames):
    """A co-scheduled batch in which some pairs fail: an all-hole frame (no jets ->
    DegenerateAlignmentError with a zero spectrum) and a noiseless pair (the reference's
    own rank-deficiency throw at 4 levels).  Their statuses match the reference build and
    every other pair is bit-identical to the same pair aligned in a clean batch."""
    A, B = frames
    hole = np.full((480, 640), np.nan)
    IAc, WAc, IBc, WBc, _ = O.synth_pair_host(K.to_c(), 7, 0)  # clean: degenerate at 4 levels
    bad = [(hole, hole, pairs[1][2], pairs[1][3]), (IAc, WAc, IBc, WBc)]
    badA = [rg.DeviceFrame.from_frame(rg.FrameData(p[0], p[1]), ctx) for p in bad]
    badB = [rg.DeviceFrame.from_frame(rg.FrameData(p[2], p[3]), ctx) for p in bad]
    idx = list(range(20))
    fa = [A[i] for i in idx]
    fb = [B[i] for i in idx]
    fa[3], fb[3] = badA[0], badB[0]
    fa[14], fb[14] = badA[1], badB[1]
    with _env(RGBID_BATCH_SLOTS=10):
        res = rg.align_batch(fa, fb, K, config=cfg, ctx=ctx)
    ref = O.Oracle("REF" if O.available("REF") else "C").align_many(
        bad, K.to_c(), None, cfg.to_c(), threads=2)
    assert res[3].status == ref[0].status == 1 and not any(res[3].spectrum[:])
    assert res[14].status == ref[1].status
    clean = _batch(ctx, K, cfg, A, B, idx, slots=20)
    for i in idx:
        if i not in (3, 14):
            assert _key(res[i]) == _key(clean[i]), i


@pytest.mark.parametrize("size,levels", [((333, 251, 250.0), 3), ((160, 120, 120.0), 1),
                                         ((320, 240, 240.0), 5), ((640, 480, 480.0), 6)])
def test_coscheduled_ragged_sizes_and_level_counts(ctx, size, levels):
    """Ragged image sizes and 1-6 pyramid levels through co-scheduled chunk pairs
    (9-slot chunks: the batch Student-t kernels), against the oracle per pair."""
    Kr = rg.simple_intrinsics(*size)
    n = 18
    ps = [O.synth_pair_host(Kr.to_c(), 100 + i, 1 + (i & 1))[:4] for i in range(n)]
    A = [rg.DeviceFrame.from_frame(rg.FrameData(p[0], p[1]), ctx) for p in ps]
    B = [rg.DeviceFrame.from_frame(rg.FrameData(p[2], p[3]), ctx) for p in ps]
    c = rg.AlignmentConfig(levels=levels)
    with _env(RGBID_BATCH_SLOTS=9):
        res = rg.align_batch(A, B, Kr, config=c, ctx=ctx)
    ref = O.Oracle("C").align_many(ps, Kr.to_c(), None, c.to_c(), threads=os.cpu_count() or 1)
    n_ok = 0
    for g, o in zip(res, ref):
        assert g.status == o.status
        if o.status != 0:
            continue
        n_ok += 1
        Tg, To = rg.Pose.from_c(g.T_AB), rg.Pose.from_c(o.T_AB)
        assert np.abs(Tg.t - To.t).max() < 1e-5
        assert np.linalg.norm(rg.so3_log(Tg.R @ To.R.T)) < 1e-5
        assert [g.level_log[k].iterations for k in range(levels)] == \
            [o.level_log[k].iterations for k in range(levels)]
    assert n_ok >= n // 2


def test_active_slot_lists_and_switch_nodes(K, pairs, frames):
    """Chunks of > 16 slots run K1 / K3 over a compact list of the slots still
    iterating, their grids picked per iteration by graph switch nodes (runtime.cu
    launch_switched, k_active_slots).  With long iteration caps most of each level is
    tail (few slots left), and with two failing pairs some slots leave the list
    early: results stay bit-identical to 10-slot chunks (no list) and to the same
    lists without switch nodes (RGBID_GRAPH_SWITCH=0, read at context creation)."""
    A, B = frames
    hole = np.full((480, 640), np.nan)
    fa, fb = list(A), list(B)
    ctx = rg.Context(0)
    badA = rg.DeviceFrame.from_frame(rg.FrameData(hole, hole), ctx)
    fa[5], fb[5] = badA, B[5]  # no jets at all: fails in the first iteration
    long_cfg = rg.AlignmentConfig(levels=LEVELS, iterations=[30, 12, 12, 12])
    with _env(RGBID_BATCH_SLOTS=20):
        lists = rg.align_batch(fa, fb, K, config=long_cfg, ctx=ctx)
    with _env(RGBID_BATCH_SLOTS=10):
        plain = rg.align_batch(fa, fb, K, config=long_cfg, ctx=ctx)
    with _env(RGBID_GRAPH_SWITCH=0):
        ctx2 = rg.Context(0)
    with _env(RGBID_BATCH_SLOTS=20):
        noswitch = rg.align_batch(fa, fb, K, config=long_cfg, ctx=ctx2)
    assert lists[5].status == 1
    assert sum(r.status == 0 for r in lists) >= N_PAIRS - 3
    its = [sum(r.level_log[k].iterations for k in range(LEVELS)) for r in lists if r.status == 0]
    assert min(its) < max(its)  # slots leave the list at different iterations
    for a, b, c in zip(lists, plain, noswitch):
        assert _key(a) == _key(b) == _key(c)
