"""Python handles on the oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module, and only as the checker or the
CPU reference arm.  Two libraries, same call shapes:

* ``C``  — oracle/_build/librgbid_oracle.so, the plain-C restatement
  (oracle/rgbid_oracle.c), buildable anywhere;
* ``REF`` — oracle/_ref/librgbid_ref.so, the UNMODIFIED reference sources
  compiled in place against oracle/eigen_shim (built only where
  /root/reference exists; the built .so travels with the repo snapshot).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1807_08271_b200.abi import (DP, AlignConfig_t, AlignResult_t, DepthIntrinsics_t,
                                       Intrinsics_t, IterTrace_t, Pose_t, TDist_t, dptr,
                                       dptr_array)

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "librgbid_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "librgbid_ref.so")
SYNTH_SO = os.path.join(HERE, "_build", "librgbid_synth.so")
REF_TESTS = os.path.join(HERE, "_ref", "ref_hotpath_tests")
REF_SRC = "/root/reference/proj"


def build(ref: bool | None = None) -> None:
    """Compile the C restatement (always) and the in-place reference build (when
    /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref", f"REF={REF_SRC}"], check=True)


def _sig(L, prefix):
    P = C.POINTER
    sigs = {
        "build_pyramid": (C.c_int, [DP, DP, C.c_int, C.c_int, P(Intrinsics_t), C.c_int, P(DP),
                                    P(DP), P(Intrinsics_t)]),
        "inverse_geometric_warp": (C.c_int, [DP, DP, C.c_int, C.c_int, DP, C.c_int, C.c_int,
                                             P(Pose_t), P(Intrinsics_t), DP, DP, DP, DP]),
        "residuals_and_jacobians": (C.c_longlong, [DP, DP, DP, DP, C.c_int, C.c_int,
                                                   P(Intrinsics_t), C.c_double, DP,
                                                   P(C.c_ubyte), C.c_longlong]),
        "t_weight": (C.c_double, [C.c_double, C.c_double]),
        "digamma": (C.c_double, [C.c_double]),
        "estimate_location_scale": (None, [DP, C.c_longlong, C.c_double, P(TDist_t)]),
        "estimate_nu": (C.c_double, [DP, C.c_longlong, C.c_double, C.c_double]),
        "filtered_hessian_covariance": (C.c_int, [DP, DP, DP, DP, C.c_int, C.c_int,
                                                  P(Intrinsics_t), P(Pose_t), P(AlignConfig_t),
                                                  DP, P(C.c_int)]),
        "bilateral_filter": (C.c_int, [DP, C.c_int, C.c_int, C.c_double, C.c_double, DP]),
        "correct_inverse_depth": (C.c_int, [DP, C.c_int, C.c_int, P(DepthIntrinsics_t),
                                            P(Intrinsics_t), C.c_int, DP]),
        "forward_register": (C.c_int, [DP, C.c_int, C.c_int, P(Pose_t), P(Intrinsics_t),
                                       P(Intrinsics_t), DP]),
        "pose_update": (C.c_int, [DP, P(Pose_t), P(Pose_t)]),
        "pose_inverse": (C.c_int, [P(Pose_t), P(Pose_t)]),
        "pose_compose": (C.c_int, [P(Pose_t), P(Pose_t), P(Pose_t)]),
        "mat3_inverse": (C.c_int, [DP, DP]),
        "align_many": (C.c_int, [C.c_int, P(DP), P(DP), P(DP), P(DP), C.c_int, C.c_int,
                                 P(Intrinsics_t), P(Pose_t), P(AlignConfig_t), P(AlignResult_t),
                                 C.c_int]),
    }
    if prefix == "or_":
        sigs["align"] = (C.c_int, [DP, DP, DP, DP, C.c_int, C.c_int, P(Intrinsics_t), P(Pose_t),
                                   P(AlignConfig_t), P(AlignResult_t), P(IterTrace_t), C.c_int,
                                   P(C.c_int)])
        sigs["integrate_frame"] = (C.c_int, [DP, DP, DP, DP, C.c_int, C.c_int, P(Pose_t),
                                             P(Intrinsics_t), C.c_double])
        sigs["covisibility_ratio"] = (C.c_int, [DP, DP, C.c_int, C.c_int, P(Pose_t),
                                                P(Intrinsics_t), C.c_double, DP, P(C.c_int),
                                                P(C.c_longlong)])
        sigs["downsample2"] = (None, [DP, C.c_int, C.c_int, DP])
        sigs["decode_frame"] = (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_double,
                                          DP, DP])
    else:
        sigs["align"] = (C.c_int, [DP, DP, DP, DP, C.c_int, C.c_int, P(Intrinsics_t), P(Pose_t),
                                   P(AlignConfig_t), P(AlignResult_t)])
        sigs["integrate_frame"] = (C.c_int, [DP, DP, DP, DP, DP, C.c_int, C.c_int, P(Pose_t),
                                             P(Intrinsics_t), C.c_double])
        sigs["covisibility_ratio"] = (C.c_int, [DP, DP, DP, DP, C.c_int, C.c_int, P(Pose_t),
                                                P(Intrinsics_t), C.c_double, DP, P(C.c_int)])
        sigs["so3_exp"] = (C.c_int, [DP, DP])
        sigs["rectify"] = (C.c_int, [DP, C.c_int, C.c_int, P(Intrinsics_t), DP])
        sigs["undistort"] = (C.c_int, [DP, C.c_longlong, P(Intrinsics_t), DP, P(C.c_ubyte)])
        sigs["render_plane"] = (C.c_int, [P(Intrinsics_t), P(Pose_t), DP, C.c_double, DP, DP])
        sigs["random_pose"] = (C.c_int, [C.c_uint, C.c_int, C.c_double, C.c_double, P(Pose_t)])
    for name, (res, args) in sigs.items():
        fn = getattr(L, prefix + name)
        fn.restype = res
        fn.argtypes = args
    return L


_libs: dict = {}


def _get(kind):
    if kind not in _libs:
        path = ORACLE_SO if kind == "C" else REF_SO
        if not os.path.exists(path):
            raise RuntimeError(f"oracle library {path} missing (run oracle.build())")
        _libs[kind] = _sig(C.CDLL(path), "or_" if kind == "C" else "ref_")
    return _libs[kind]


def available(kind: str) -> bool:
    return os.path.exists(ORACLE_SO if kind == "C" else REF_SO)


_synth = None


def synth_pair_host(K, pair_seed, variant=1):
    """Benchmark pair `pair_seed` rendered on the host by oracle/_build/librgbid_synth.so
    (the product's synth.cpp built alone, so the CPU reference arm never maps the CUDA
    library): (I_A, W_A, I_B, W_B, T_AB_truth as Pose_t).  K: Intrinsics_t."""
    global _synth
    if _synth is None:
        if not os.path.exists(SYNTH_SO):
            raise RuntimeError(f"{SYNTH_SO} missing (run oracle.build())")
        L = C.CDLL(SYNTH_SO)
        L.rgbid_synth_pair_host.restype = C.c_int
        L.rgbid_synth_pair_host.argtypes = [C.POINTER(Intrinsics_t), C.c_uint, C.c_int, DP, DP, DP,
                                            DP, C.POINTER(Pose_t)]
        _synth = L
    h, w = K.height, K.width
    IA, WA, IB, WB = (np.empty((h, w)) for _ in range(4))
    T = Pose_t()
    rc = _synth.rgbid_synth_pair_host(C.byref(K), pair_seed, variant, dptr(IA), dptr(WA), dptr(IB),
                                      dptr(WB), C.byref(T))
    if rc != 0:
        raise ValueError("synth_pair_host: invalid argument")
    return IA, WA, IB, WB, T


class Oracle:
    """Numpy-level wrapper; ``kind`` is "C" (restatement) or "REF" (reference)."""

    def __init__(self, kind: str = "C"):
        self.kind = kind
        self.L = _get(kind)
        self.p = "or_" if kind == "C" else "ref_"

    def _f(self, name):
        return getattr(self.L, self.p + name)

    def build_pyramid(self, I, W, K, levels):
        h, w = W.shape
        outI = [np.empty((h >> l, w >> l)) for l in range(levels)]
        outW = [np.empty((h >> l, w >> l)) for l in range(levels)]
        # exact sizes: repeated floor halving
        sizes = [(h, w)]
        for _ in range(1, levels):
            sizes.append((sizes[-1][0] // 2, sizes[-1][1] // 2))
        outI = [np.empty(s) for s in sizes]
        outW = [np.empty(s) for s in sizes]
        Ks = (Intrinsics_t * levels)()
        self._f("build_pyramid")(dptr(I), dptr(W), w, h, C.byref(K), levels, dptr_array(outI),
                                 dptr_array(outW), Ks)
        return outI, outW, list(Ks)

    def inverse_geometric_warp(self, I_B, W_B, W_A, T_AB, K):
        hb, wb = W_B.shape
        h, w = W_A.shape
        out = [np.empty((h, w)) for _ in range(4)]
        self._f("inverse_geometric_warp")(dptr(I_B), dptr(W_B), wb, hb, dptr(W_A), w, h,
                                          C.byref(T_AB), C.byref(K), *[dptr(o) for o in out])
        return tuple(out)

    def residuals_and_jacobians(self, I_A, W_A, I_Bw, W_Bw, K, lambda_n_min=0.1):
        h, w = W_A.shape
        cap = w * h
        jets = np.empty((cap, 17))
        flags = np.empty(cap, dtype=np.uint8)
        n = self._f("residuals_and_jacobians")(
            dptr(I_A), dptr(W_A), dptr(I_Bw), dptr(W_Bw), w, h, C.byref(K), lambda_n_min,
            dptr(jets), flags.ctypes.data_as(C.POINTER(C.c_ubyte)), cap)
        return jets[:n].copy(), flags[:n].astype(bool)

    def t_weight(self, x, nu):
        return self._f("t_weight")(x, nu)

    def digamma(self, x):
        return self._f("digamma")(x)

    def estimate_location_scale(self, r, nu):
        r = np.ascontiguousarray(r, dtype=np.float64)
        t = TDist_t()
        self._f("estimate_location_scale")(dptr(r), len(r), nu, C.byref(t))
        return t.mu, t.sigma, t.nu

    def estimate_nu(self, r, mu, sigma):
        r = np.ascontiguousarray(r, dtype=np.float64)
        return self._f("estimate_nu")(dptr(r), len(r), mu, sigma)

    def align(self, IA, WA, IB, WB, K, init=None, cfg=None, trace=False):
        h, w = WA.shape
        res = AlignResult_t()
        args = [dptr(IA), dptr(WA), dptr(IB), dptr(WB), w, h, C.byref(K),
                C.byref(init) if init is not None else None,
                C.byref(cfg) if cfg is not None else None, C.byref(res)]
        if self.kind == "C":
            tr = (IterTrace_t * 64)()
            n = C.c_int(0)
            self._f("align")(*args, tr, 64 if trace else 0, C.byref(n))
            return (res, list(tr)[: n.value]) if trace else res
        self._f("align")(*args)
        return (res, []) if trace else res

    def align_many(self, pairs, K, inits=None, cfg=None, threads=1):
        n = len(pairs)
        h, w = pairs[0][1].shape
        res = (AlignResult_t * n)()
        arrs = [dptr_array([p[k] for p in pairs]) for k in range(4)]
        ini = (Pose_t * n)(*inits) if inits is not None else None
        self._f("align_many")(n, *arrs, w, h, C.byref(K), ini,
                              C.byref(cfg) if cfg is not None else None, res, threads)
        return list(res)

    def filtered_hessian_covariance(self, IA, WA, IB, WB, K, T, cfg=None):
        h, w = WA.shape
        cov = np.empty(36)
        deg = C.c_int(0)
        self._f("filtered_hessian_covariance")(dptr(IA), dptr(WA), dptr(IB), dptr(WB), w, h,
                                               C.byref(K), C.byref(T),
                                               C.byref(cfg) if cfg is not None else None,
                                               dptr(cov), C.byref(deg))
        return cov.reshape(6, 6), bool(deg.value)

    def bilateral_filter(self, img, ss, sr):
        h, w = img.shape
        out = np.empty_like(img)
        self._f("bilateral_filter")(dptr(img), w, h, ss, sr, dptr(out))
        return out

    def normal_map(self, W, K):
        """src/segmentation.cpp:10-57 (reference build only)"""
        assert self.kind == "REF", "normal_map is checked against the reference build"
        h, w = W.shape
        nx, ny, nz = (np.empty_like(W) for _ in range(3))
        self._f("normal_map")(dptr(W), w, h, C.byref(K), dptr(nx), dptr(ny), dptr(nz))
        return nx, ny, nz

    def integrate_frame(self, kf_I, kf_W, kf_C, fI, fW, T, K, sigma_w):
        """In place on kf_W, kf_C (and kf_I untouched)."""
        h, w = kf_W.shape
        if self.kind == "C":
            self._f("integrate_frame")(dptr(kf_W), dptr(kf_C), dptr(fI), dptr(fW), w, h,
                                       C.byref(T), C.byref(K), sigma_w)
        else:
            self._f("integrate_frame")(dptr(kf_I), dptr(kf_W), dptr(kf_C), dptr(fI), dptr(fW),
                                       w, h, C.byref(T), C.byref(K), sigma_w)

    def covisibility_ratio(self, IA, WA, IB, WB, T_BA, K, sigma_w):
        h, w = WA.shape
        ratio = C.c_double(0)
        empty = C.c_int(0)
        if self.kind == "C":
            counts = (C.c_longlong * 4)()
            self._f("covisibility_ratio")(dptr(WA), dptr(WB), w, h, C.byref(T_BA), C.byref(K),
                                          sigma_w, C.byref(ratio), C.byref(empty), counts)
            return ratio.value, bool(empty.value), list(counts)
        self._f("covisibility_ratio")(dptr(IA), dptr(WA), dptr(IB), dptr(WB), w, h,
                                      C.byref(T_BA), C.byref(K), sigma_w, C.byref(ratio),
                                      C.byref(empty))
        return ratio.value, bool(empty.value), None

    def correct_inverse_depth(self, Wm, d, K, spatial):
        h, w = Wm.shape
        out = np.empty_like(Wm)
        self._f("correct_inverse_depth")(dptr(Wm), w, h, C.byref(d), C.byref(K), int(spatial),
                                         dptr(out))
        return out

    def forward_register(self, WA, T_BA, KA, KB):
        h, w = WA.shape
        out = np.empty((KB.height, KB.width))
        self._f("forward_register")(dptr(WA), w, h, C.byref(T_BA), C.byref(KA), C.byref(KB),
                                    dptr(out))
        return out

    def pose_update(self, xi, T):
        xi = np.ascontiguousarray(xi, dtype=np.float64)
        out = Pose_t()
        self._f("pose_update")(dptr(xi), C.byref(T), C.byref(out))
        return out

    def pose_inverse(self, T):
        out = Pose_t()
        self._f("pose_inverse")(C.byref(T), C.byref(out))
        return out

    def pose_compose(self, a, b):
        out = Pose_t()
        self._f("pose_compose")(C.byref(a), C.byref(b), C.byref(out))
        return out

    def mat3_inverse(self, m):
        m = np.ascontiguousarray(m, dtype=np.float64).reshape(9)
        out = np.empty(9)
        self._f("mat3_inverse")(dptr(m), dptr(out))
        return out.reshape(3, 3)

    def decode_frame(self, bgr, depth, scale=5000.0):
        h, w = depth.shape
        I = np.empty((h, w))
        W = np.empty((h, w))
        depth = np.ascontiguousarray(depth, dtype=np.uint16)
        bgr = np.ascontiguousarray(bgr, dtype=np.uint8)
        self._f("decode_frame")(bgr.ctypes.data, depth.ctypes.data, w, h, scale, dptr(I), dptr(W))
        return I, W

    # reference-only: the distorted-sensor path (src/camera.cpp:11-45, src/warping.cpp:8-18)
    def rectify(self, img, K):
        assert self.kind == "REF", "rectify composes the reference's own project/inverse_warp"
        h, w = img.shape
        out = np.empty_like(img)
        self._f("rectify")(dptr(np.ascontiguousarray(img)), w, h, C.byref(K), dptr(out))
        return out

    def undistort(self, m_d, K):
        assert self.kind == "REF"
        m_d = np.ascontiguousarray(m_d, dtype=np.float64).reshape(-1, 2)
        n = len(m_d)
        m_u = np.empty_like(m_d)
        ok = np.zeros(n, dtype=np.uint8)
        self._f("undistort")(dptr(m_d), n, C.byref(K), dptr(m_u),
                             ok.ctypes.data_as(C.POINTER(C.c_ubyte)))
        return m_u, ok.astype(bool)

    # reference-only fixtures (tests/synthetic.hpp)
    def render_plane(self, K, T_WC, n=(0.0, 0.0, 1.0), d=-2.0):
        I = np.empty((K.height, K.width))
        W = np.empty((K.height, K.width))
        nn = np.asarray(n, dtype=np.float64)
        self._f("render_plane")(C.byref(K), C.byref(T_WC), dptr(nn), d, dptr(I), dptr(W))
        return I, W

    def random_pose(self, seed, skip=0, t_scale=1.0, angle_scale=1.0):
        out = Pose_t()
        self._f("random_pose")(seed, skip, t_scale, angle_scale, C.byref(out))
        return out
