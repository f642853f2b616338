"""CPU tier: pin the oracle, check the boundary library loads and exports the
C-ABI.  No GPU needed.

1. The reference's own hot-path unit tests (tests/test_{alignment,warping,fusion,
   camera,geometry}.cpp, 64 cases) pass against the in-place reference build
   (oracle/_ref) — pins the Eigen/doctest shims.
2. The plain-C restatement (oracle/rgbid_oracle.c) equals that reference build
   BIT FOR BIT on every hot-path function (maps, jets, Student-t, full align
   pose/cov/logs, fusion, covisibility, depth correction, registration).
3. Known-answer values from the reference tests hold on the restatement.
4. librgbid_b200.so exports every function include/rgbid_b200.h declares; its
   synthetic generator equals the reference fixture generator bit for bit.
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1807_08271_b200 as rg
from oracle import oracle as O
from paper_1807_08271_b200 import abi
from tests.conftest import have_gpu
from tests.scenes import N_SLANT, bitwise_equal, pair

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
needs_ref = pytest.mark.skipif(not O.available("REF"), reason="reference build absent")


@pytest.fixture(scope="module")
def C_():
    return O.Oracle("C")


@pytest.fixture(scope="module")
def R_():
    return O.Oracle("REF")


@needs_ref
def test_reference_unit_tests_pass_on_ref_build():
    p = subprocess.run([O.REF_TESTS], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stdout[-2000:]
    assert "64 ran, 0 failed" in p.stdout


SCENES = [((80, 60, 60.0), "clean", False), ((80, 60, 60.0), "noisy", True),
          ((160, 120, 120.0), "noisy", True)]


@needs_ref
@pytest.mark.parametrize("size,variant,holes", SCENES)
def test_restatement_bitwise_maps_and_jets(C_, R_, size, variant, holes):
    K = rg.simple_intrinsics(*size)
    fa, fb, T = pair(K, 2, variant, holes)
    for lv in (1, 4):
        a, b = C_.build_pyramid(fa.intensity, fa.inverse_depth, K.to_c(), lv), \
            R_.build_pyramid(fa.intensity, fa.inverse_depth, K.to_c(), lv)
        for x, y in zip(a[0] + a[1], b[0] + b[1]):
            assert bitwise_equal(x, y)
    for T_AB in (T, rg.random_pose(41, 0.02, 0.02)):
        wc = C_.inverse_geometric_warp(fb.intensity, fb.inverse_depth, fa.inverse_depth,
                                       T_AB.to_c(), K.to_c())
        wr = R_.inverse_geometric_warp(fb.intensity, fb.inverse_depth, fa.inverse_depth,
                                       T_AB.to_c(), K.to_c())
        for x, y in zip(wc, wr):
            assert bitwise_equal(x, y)
        jc, fc = C_.residuals_and_jacobians(fa.intensity, fa.inverse_depth, wc[0], wc[1], K.to_c())
        jr, fr = R_.residuals_and_jacobians(fa.intensity, fa.inverse_depth, wc[0], wc[1], K.to_c())
        assert bitwise_equal(jc, jr) and bitwise_equal(fc, fr)
        for nu in (2.5, 5.0):
            assert C_.estimate_location_scale(jc[:, 2], nu) == R_.estimate_location_scale(jr[:, 2], nu)
        mu, s, _ = R_.estimate_location_scale(jr[:, 2], 5.0)
        assert C_.estimate_nu(jc[:, 2], mu, s) == R_.estimate_nu(jr[:, 2], mu, s)


@needs_ref
@pytest.mark.parametrize("size,variant,holes", SCENES)
@pytest.mark.parametrize("levels", [3, 4])
def test_restatement_bitwise_align(C_, R_, size, variant, holes, levels):
    K = rg.simple_intrinsics(*size)
    fa, fb, _ = pair(K, 1, variant, holes)
    cfg = rg.AlignmentConfig(levels=levels).to_c()
    a = C_.align(fa.intensity, fa.inverse_depth, fb.intensity, fb.inverse_depth, K.to_c(), None, cfg)
    b = R_.align(fa.intensity, fa.inverse_depth, fb.intensity, fb.inverse_depth, K.to_c(), None, cfg)
    assert bytes(a) == bytes(b)


@needs_ref
def test_restatement_bitwise_vga_align(C_, R_):
    K = rg.simple_intrinsics(640, 480, 480.0)
    fa, fb, _ = pair(K, 0, "noisy", True)
    cfg = rg.AlignmentConfig(levels=4).to_c()
    a = C_.align(fa.intensity, fa.inverse_depth, fb.intensity, fb.inverse_depth, K.to_c(), None, cfg)
    b = R_.align(fa.intensity, fa.inverse_depth, fb.intensity, fb.inverse_depth, K.to_c(), None, cfg)
    assert bytes(a) == bytes(b)
    assert a.status == 0 and a.n_levels == 4


@needs_ref
def test_restatement_degenerate_matches(C_, R_):
    K = rg.simple_intrinsics(40, 30)
    nan = np.full((30, 40), np.nan)
    a = C_.align(nan, nan, nan, nan, K.to_c())
    b = R_.align(nan, nan, nan, nan, K.to_c())
    assert a.status == b.status == abi.E_DEGENERATE
    assert list(a.spectrum) == list(b.spectrum)


@needs_ref
def test_restatement_bitwise_fusion_covis_register(C_, R_):
    K = rg.simple_intrinsics(160, 120, 120.0)
    base = rg.render_plane(K, rg.Pose(), N_SLANT, -2.0, 2.0)
    kW1, kC1 = base.inverse_depth.copy(), np.ones_like(base.inverse_depth)
    kI2, kW2, kC2 = base.intensity.copy(), base.inverse_depth.copy(), np.ones_like(base.inverse_depth)
    for k in range(5):
        T = rg.random_pose(3000 + k, 0.01, 0.01)
        f = rg.add_noise(rg.render_plane(K, T, N_SLANT, -2.0, 2.0), 10 + k, 0.0, 0.01)
        C_.integrate_frame(None, kW1, kC1, f.intensity, f.inverse_depth, T.to_c(), K.to_c(), 0.05)
        R_.integrate_frame(kI2, kW2, kC2, f.intensity, f.inverse_depth, T.to_c(), K.to_c(), 0.05)
        assert bitwise_equal(kW1, kW2) and bitwise_equal(kC1, kC2)
    fa, fb, T = pair(K, 3, "noisy", True)
    for T_BA in (T.inverse(), rg.Pose(np.eye(3), [0.3, 0, 0])):
        a = C_.covisibility_ratio(fa.intensity, fa.inverse_depth, fb.intensity, fb.inverse_depth,
                                  T_BA.to_c(), K.to_c(), 0.01)
        b = R_.covisibility_ratio(fa.intensity, fa.inverse_depth, fb.intensity, fb.inverse_depth,
                                  T_BA.to_c(), K.to_c(), 0.01)
        assert a[:2] == b[:2]
    d = rg.DepthIntrinsics(-0.005, 1.02, (0.002, 1e-4, -1e-4, 0, 0, 0, 0, 0, 0),
                           (1.01, 1e-3, 0, 5e-4, 0, 0, 0, 0, 0), (4.0, 4.0))
    for sp in (0, 1):
        assert bitwise_equal(C_.correct_inverse_depth(fa.inverse_depth, d.to_c(), K.to_c(), sp),
                             R_.correct_inverse_depth(fa.inverse_depth, d.to_c(), K.to_c(), sp))
    for T_BA in (rg.random_pose(7, 0.025, 0.01), rg.Pose(np.eye(3), [-0.3, 0, 0])):
        assert bitwise_equal(C_.forward_register(fa.inverse_depth, T_BA.to_c(), K.to_c(), K.to_c()),
                             R_.forward_register(fa.inverse_depth, T_BA.to_c(), K.to_c(), K.to_c()))
    for img, sr in ((fa.intensity, 0.05), (fa.inverse_depth, 0.02)):
        assert bitwise_equal(C_.bilateral_filter(img, 2.0, sr), R_.bilateral_filter(img, 2.0, sr))
    Tc = rg.random_pose(5, 0.01, 0.02)
    a = C_.filtered_hessian_covariance(fa.intensity, fa.inverse_depth, fb.intensity,
                                       fb.inverse_depth, K.to_c(), Tc.to_c())
    b = R_.filtered_hessian_covariance(fa.intensity, fa.inverse_depth, fb.intensity,
                                       fb.inverse_depth, K.to_c(), Tc.to_c())
    assert bitwise_equal(a[0], b[0]) and a[1] == b[1]


@needs_ref
def test_restatement_pose_math_bitwise(C_, R_):
    for s in range(20):
        T = rg.random_pose(100 + s, 0.5, 2.0).to_c()
        U = rg.random_pose(200 + s, 0.5, 2.0).to_c()
        xi = np.random.default_rng(s).normal(size=6) * 10.0 ** -np.random.default_rng(s).integers(1, 7)
        assert bytes(C_.pose_update(xi, T)) == bytes(R_.pose_update(xi, T))
        assert bytes(C_.pose_inverse(T)) == bytes(R_.pose_inverse(T))
        assert bytes(C_.pose_compose(T, U)) == bytes(R_.pose_compose(T, U))
    K = rg.simple_intrinsics(640, 480, 525.3).K()
    assert bitwise_equal(C_.mat3_inverse(K), R_.mat3_inverse(K))


def test_restatement_known_answers(C_):
    """Values from tests/test_alignment.cpp:30-83 on the restatement."""
    g = 0.5772156649015329
    assert C_.digamma(1.0) == pytest.approx(-g, rel=1e-8)
    assert C_.digamma(0.5) == pytest.approx(-g - 2 * np.log(2.0), rel=1e-8)
    assert C_.digamma(5.0) == pytest.approx(1.5061176684318003, rel=1e-8)
    assert C_.digamma(3.7) == pytest.approx(C_.digamma(2.7) + 1.0 / 2.7, rel=1e-8)
    for nu in (2.0, 3.5, 5.0, 10.0):
        for x in np.arange(-4.0, 4.0, 0.37):
            w = C_.t_weight(x, nu)
            assert 0 < w <= (nu + 1.0) / nu + 1e-12
    mu, s, _ = C_.estimate_location_scale(np.full(500, 0.75), 5.0)
    assert mu == pytest.approx(0.75) and s == pytest.approx(1e-8)
    rng = np.random.default_rng(73)
    mu, s, _ = C_.estimate_location_scale(rng.normal(size=100000), 5.0)
    assert 0.82 < s < 0.89 and abs(mu) < 0.02
    assert C_.estimate_nu(rng.normal(size=100000), 0.0, 0.856) == pytest.approx(10.0)


def test_restatement_alignment_accuracy(C_):
    """tests/test_alignment.cpp:207-233: 5 mm / 1 deg recovered at 80x60."""
    K = rg.simple_intrinsics(80, 60)
    T_WB = rg.Pose(rg.so3_exp([0, np.pi / 180.0, 0]), [0.005, 0, 0])
    fa = rg.render_plane(K, rg.Pose(), N_SLANT, -2.0)
    fb = rg.render_plane(K, T_WB, N_SLANT, -2.0)
    r = C_.align(fa.intensity, fa.inverse_depth, fb.intensity, fb.inverse_depth, K.to_c())
    T = rg.Pose.from_c(r.T_AB)
    assert np.linalg.norm(T.t - T_WB.t) < 5e-4
    assert np.linalg.norm(rg.so3_log(T.R @ T_WB.R.T)) < 0.05 * np.pi / 180.0


def _header_functions():
    src = open(os.path.join(ROOT, "include", "rgbid_b200.h")).read()
    return sorted(set(re.findall(r"^(?:const char\*|int|long long|void\*)\s+(rgbid_\w+)\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(abi.LIB_PATH)
    names = _header_functions()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(n for n, _, _ in abi.EXPORTS) == names


def test_integration_doc_indexes_every_entry_point():
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    index = doc[doc.index("## 4. Entry-point index"):]
    missing = [n for n in _header_functions() if f"`{n}`" not in index]
    assert not missing, missing


def test_library_fails_loudly_without_gpu():
    if have_gpu():
        pytest.skip("GPU present")
    with pytest.raises(rg.CudaError):
        rg.Context(0)


@needs_ref
def test_synth_matches_reference_fixtures(R_):
    for seed in (1000, 41, 7, 2024):
        for skip in (0, 2):
            a = rg.random_pose(seed, 0.003, 0.02, skip).to_c()
            assert bytes(a) == bytes(R_.random_pose(seed, skip, 0.003, 0.02))
    K = rg.simple_intrinsics(640, 480, 480.0)
    T = rg.random_pose(1000, 0.003, 0.02)
    f = rg.render_plane(K, T, N_SLANT, -2.0, 1.0)
    I, W = R_.render_plane(K.to_c(), T.to_c(), N_SLANT, -2.0)
    assert bitwise_equal(f.intensity, I) and bitwise_equal(f.inverse_depth, W)


@needs_ref
def test_backend_oracles_sane(R_):
    """SURVEY 8(f) rank 4 checkers: the reference normal_map (built unchanged from
    src/segmentation.cpp) gives unit normals facing the camera; the export_map
    restatement keeps only novel pixels and the voxel grid only merges."""
    from oracle import map_oracle
    K = rg.simple_intrinsics(80, 60, 60.0)
    fa, _, _ = pair(K, 2, "noisy", holes=True)
    nx, ny, nz = R_.normal_map(fa.inverse_depth, K.to_c())
    m = np.isfinite(fa.inverse_depth) & (fa.inverse_depth > 0)
    assert np.array_equal(np.isfinite(nz), m)
    n = np.sqrt(nx[m] ** 2 + ny[m] ** 2 + nz[m] ** 2)
    assert np.allclose(n, 1.0) and (nz[m] <= 0).all()
    kfs = [(fa.intensity, fa.inverse_depth, rg.Pose().to_c()),
           (fa.intensity, fa.inverse_depth, rg.Pose().to_c())]
    p0, c0 = map_oracle.export_map(kfs, K.to_c(), 0.0)
    # the second, identical keyframe adds only pixels whose bilinear taps touch a hole
    assert m.sum() <= len(p0) < 1.2 * m.sum()
    pv, cv = map_oracle.export_map(kfs, K.to_c(), 0.1)
    assert 0 < len(pv) < len(p0) and cv.dtype == np.uint8


def test_synth_pair_host_deterministic():
    """The reference arm's input generator (host, no GPU): same seed -> same pair,
    different seeds -> different noise; holes only where the plane is not visible."""
    K = rg.simple_intrinsics(80, 60, 60.0)
    a1, b1, T1 = rg.synth_pair_host(K, 3, 1)
    a2, b2, T2 = rg.synth_pair_host(K, 3, 1)
    a3, _, _ = rg.synth_pair_host(K, 4, 1)
    assert bitwise_equal(a1.intensity, a2.intensity) and bitwise_equal(b1.inverse_depth, b2.inverse_depth)
    assert not np.array_equal(a1.intensity, a3.intensity)
    assert np.isfinite(a1.inverse_depth).all() and (b1.inverse_depth[:, : 80 // 5] == 1.0).all()
