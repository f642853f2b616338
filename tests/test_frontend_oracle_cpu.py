"""Pins the front-end oracle (oracle/frontend_oracle.py) to the reference's own
pipeline tests (tests/test_pipeline.cpp:91-147) on the CPU."""
import numpy as np

import paper_1807_08271_b200 as rg
from oracle.frontend_oracle import FrontendOracle
from oracle.oracle import Oracle


def sweep_pose(i, step=0.02):
    return rg.Pose(np.eye(3), [step * i, 0.0, 0.0])


def run(frames):
    K = rg.simple_intrinsics(80, 60, 60.0)
    fo = FrontendOracle(Oracle("C"), K.to_c(), rg.AlignmentConfig().to_c())
    for i, f in enumerate(frames):
        fo.process_frame(f, 0.1 * i)
    return fo


def test_oracle_static_sequence():
    K = rg.simple_intrinsics(80, 60, 60.0)
    fo = run([rg.render_plane(K, rg.Pose())] * 6)
    assert fo.kf_index == [0] and len(fo.traj) == 6
    for t in fo.traj:
        assert not t[3] and np.linalg.norm(np.array(t[1].t[:])) < 1e-3


def test_oracle_slow_sweep():
    K = rg.simple_intrinsics(80, 60, 60.0)
    fo = run([rg.render_plane(K, sweep_pose(i, 0.01)) for i in range(10)])
    for i, t in enumerate(fo.traj):
        assert np.linalg.norm(np.array(t[1].t[:]) - sweep_pose(i, 0.01).t) < 0.003


def test_oracle_long_sweep_switches():
    K = rg.simple_intrinsics(80, 60, 60.0)
    fo = run([rg.render_plane(K, sweep_pose(i, 0.03)) for i in range(40)])
    assert len(fo.kf_index) >= 2 and fo.kf_index[0] == 0
    for i, t in enumerate(fo.traj):
        assert np.linalg.norm(np.array(t[1].t[:]) - sweep_pose(i, 0.03).t) < 0.01
