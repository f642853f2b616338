"""Seeded synthetic scenes shared by the parity tests (SURVEY §8d inputs).

Rendered on the host with the library's fixture restatement
(rgbid_synth_render_plane), which is bit-identical to the reference's
tests/synthetic.hpp (checked in test_oracle_cpu.py)."""
import numpy as np

import paper_1807_08271_b200 as rg

N_SLANT = np.array([0.2, -0.15, 1.0]) / np.linalg.norm([0.2, -0.15, 1.0])


def vga():
    return rg.simple_intrinsics(640, 480, 480.0)


def pair(K, i=0, variant="clean", holes=False, tex_scale=None):
    """Frame pair i of config 1/5: A at identity, B at random_pose(1000+i, 3 mm, 0.02)."""
    if tex_scale is None:
        tex_scale = K.width / 80.0
    T_WB = rg.random_pose(1000 + i, 0.003, 0.02)
    fa = rg.render_plane(K, rg.Pose(), N_SLANT, -2.0, tex_scale)
    fb = rg.render_plane(K, T_WB, N_SLANT, -2.0, tex_scale)
    if variant == "noisy":
        fa = rg.add_noise(fa, 3000 + i, 0.005, 0.002)
        fb = rg.add_noise(fb, 2000 + i, 0.005, 0.002)
        fb.inverse_depth[:, : K.width // 5] = 1.0
        fb.intensity[:, : K.width // 5] = 0.9
    if holes:
        rng = np.random.default_rng(7 + i)
        for f in (fa, fb):
            m = rng.random(f.inverse_depth.shape) < 0.05
            f.inverse_depth[m] = np.nan
            m = rng.random(f.intensity.shape) < 0.02
            f.intensity[m] = np.nan
            b = max(1, K.width // 32)
            f.inverse_depth[:b, :] = np.nan
            f.inverse_depth[:, -b:] = np.nan
    return fa, fb, T_WB


def bitwise_equal(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b), equal_nan=True)
