"""Generate tests/golden/rgbid_golden_80x60.npz from the REFERENCE build.

TEST INFRASTRUCTURE.  Run here (where /root/reference exists and
oracle/_ref/librgbid_ref.so is built from the reference's own sources by
oracle/Makefile):

    python -m tests.golden.make_golden

Every output in the fixture comes from the unmodified reference functions
(``ref_*`` entry points of oracle/ref_capi.cpp wrapping src/*.cpp); the inputs
are stored next to them, so the fixture needs nothing else to be checked on a
box without /root/reference.  Sizes are the reference tests' own 80 x 60 camera
(tests/synthetic.hpp:13-21).  Cases:

* scalars: digamma (src/alignment.cpp:32-43), t_weight (inc/alignment.hpp:35),
  estimate_location_scale / estimate_nu (src/alignment.cpp:61-157) on seeded
  Gaussian, Student-t and constant samples;
* one noisy pair with holes: build_pyramid (:9-30), inverse_geometric_warp
  (src/warping.cpp:76-114), bilateral_filter (:252-277), forward_register
  (src/warping.cpp:20-74), covisibility_ratio (src/fusion.cpp:52-66),
  integrate_frame (src/fusion.cpp:68-95), correct_inverse_depth
  (src/camera.cpp:62-81), normal_map (src/segmentation.cpp:10-57);
* align (src/alignment.cpp:367-409) with covariance, 3 and 4 levels, on the
  noisy pair and on a clean pair.
"""
from __future__ import annotations

import os

import numpy as np

import paper_1807_08271_b200 as rg
from oracle.oracle import Oracle
from tests.scenes import pair

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "rgbid_golden_80x60.npz")

DIGAMMA_X = np.array([0.25, 0.5, 1.0, 1.5, 2.0, 2.5, 3.0, 5.0, 5.5, 6.0, 7.5, 10.0, 25.0])
TW_ARGS = np.array([[0.0, 5.0], [0.5, 5.0], [-3.0, 2.0], [10.0, 10.0], [1e-3, 4.99]])
SIGMA_W = 0.01
DEPTH = rg.DepthIntrinsics(beta0=0.01, beta1=0.98,
                           q0=(0.001, 0.002, -0.001, 0.0, 0.003, -0.002, 0.001, 0.0, 0.0),
                           q1=(1.0, 0.01, -0.005, 0.0, 0.002, 0.001, 0.0, 0.0005, -0.0005))


def samples():
    rng = np.random.default_rng(1807)
    return {
        "gauss": rng.normal(0.01, 0.05, 4000),
        "student": 0.02 * rng.standard_t(3.0, 4000) - 0.003,
        "const": np.full(300, 0.25),
    }


def generate(ref: Oracle) -> dict:
    g: dict = {}
    g["digamma_x"] = DIGAMMA_X
    g["digamma_y"] = np.array([ref.digamma(x) for x in DIGAMMA_X])
    g["t_weight_args"] = TW_ARGS
    g["t_weight_y"] = np.array([ref.t_weight(x, nu) for x, nu in TW_ARGS])
    for name, r in samples().items():
        mu, sig, nu = ref.estimate_location_scale(r, 5.0)
        g[f"ls_{name}_r"] = r
        g[f"ls_{name}_out"] = np.array([mu, sig, nu])
        g[f"nu_{name}_out"] = np.array([ref.estimate_nu(r, mu, sig)])

    K = rg.simple_intrinsics(80, 60, 60.0)
    Kc = K.to_c()
    g["K"] = np.array([K.fx, K.fy, K.cx, K.cy, K.width, K.height], dtype=np.float64)
    for tag, variant, holes, i in (("noisy", "noisy", True, 3), ("clean", "clean", False, 1)):
        fa, fb, T = pair(K, i, variant, holes)
        g[f"{tag}_IA"], g[f"{tag}_WA"] = fa.intensity, fa.inverse_depth
        g[f"{tag}_IB"], g[f"{tag}_WB"] = fb.intensity, fb.inverse_depth
        for levels, its in ((3, [10, 5, 4]), (4, [10, 5, 4, 5])):
            cfg = rg.AlignmentConfig(levels=levels, iterations=its)
            o = ref.align(fa.intensity, fa.inverse_depth, fb.intensity, fb.inverse_depth, Kc,
                          None, cfg.to_c())
            P = rg.Pose.from_c(o.T_AB)
            key = f"{tag}_align{levels}"
            g[f"{key}_R"], g[f"{key}_t"] = P.R, P.t
            g[f"{key}_cov"] = np.array(o.cov[:]).reshape(6, 6)
            g[f"{key}_iters"] = np.array([l.iterations for l in o.level_log[: o.n_levels]])
            g[f"{key}_cost"] = np.array([l.final_cost for l in o.level_log[: o.n_levels]])
            g[f"{key}_tdist"] = np.array([o.tdist_intensity.mu, o.tdist_intensity.sigma,
                                          o.tdist_intensity.nu, o.tdist_depth.mu,
                                          o.tdist_depth.sigma, o.tdist_depth.nu])
            g[f"{key}_flags"] = np.array([o.converged, o.cov_degenerate])
        if tag != "noisy":
            continue
        g["T_AB"] = T.matrix()
        pI, pW, _ = ref.build_pyramid(fa.intensity, fa.inverse_depth, Kc, 3)
        for l in range(3):
            g[f"pyr_I{l}"], g[f"pyr_W{l}"] = pI[l], pW[l]
        for k, m in zip(("I", "W", "mx", "my"),
                        ref.inverse_geometric_warp(fb.intensity, fb.inverse_depth,
                                                   fa.inverse_depth, T.to_c(), Kc)):
            g[f"warp_{k}"] = m
        g["bil_I"] = ref.bilateral_filter(fa.intensity, 2.0, 0.05)
        g["bil_W"] = ref.bilateral_filter(fa.inverse_depth, 2.0, 0.02)
        g["fwd_W"] = ref.forward_register(fa.inverse_depth, T.inverse().to_c(), Kc, Kc)
        ratio, empty, _ = ref.covisibility_ratio(fa.intensity, fa.inverse_depth, fb.intensity,
                                                 fb.inverse_depth, T.inverse().to_c(), Kc, SIGMA_W)
        g["covis"] = np.array([ratio, empty])
        kW, kC = fa.inverse_depth.copy(), np.ones_like(fa.inverse_depth)
        ref.integrate_frame(fa.intensity.copy(), kW, kC, fb.intensity, fb.inverse_depth,
                            T.to_c(), Kc, SIGMA_W)
        g["fuse_W"], g["fuse_C"] = kW, kC
        for spatial in (0, 1):
            g[f"cid_{spatial}"] = ref.correct_inverse_depth(fa.inverse_depth, DEPTH.to_c(), Kc,
                                                            bool(spatial))
        nx, ny, nz = ref.normal_map(fa.inverse_depth, Kc)
        g["normal"] = np.stack([nx, ny, nz])
    return g


def main():
    g = generate(Oracle("REF"))
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
