// The benchmark scene, shared by the device renderer (k_render,
// fusion_kernels.cu) and the host renderer (synth.cpp, also built standalone as
// oracle/_build/librgbid_synth.so for the reference arm).  Everything that
// decides WHICH pixels are holes is integer hashing, identical on host and
// device; only the texture/noise values go through sin/cos/log (CUDA libdevice
// vs glibc: equal up to the last bits).
//
// Pair i (variant v):
//   A = render_plane at random_pose(5000+i, 1 cm, 0.01) , B = A * random_pose(1000+i, 3 mm, 0.02)
//       (tests/synthetic.hpp:31-59; plane n = (0.2,-0.15,1)/|.|, d = -2, texture at w/80 x world)
//   v >= 1: I += N(0, 0.005), W += N(0, 0.002) (counter-based Box-Muller), and a 20% near
//           occluder on B (x < w/5: W = 1.0, tests/test_alignment.cpp:220-232)
//   v == 2: + 5% random W holes, 2% random I holes and a w/32-pixel (20 px at VGA)
//           border band of W holes on both frames — the validity/compaction paths
#pragma once
#include <cstdint>

#include "hd_math.cuh"

namespace rgbid_b200 {

struct SynthView {
  int w, h;
  M3 Kinv, R;
  double t[3], n[3], d;
  double tex_scale;
  double noise_i, noise_w;
  unsigned long long seed;
  int occluder;
  int holes;   // random I/W holes
  int border;  // W border band width (pixels), 0 = none
};

HD unsigned long long synth_splitmix(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// hole decisions of pixel i (integer only: bit-identical host/device)
HD bool synth_hole_w(const SynthView& v, int i, int x, int y) {
  if (v.border > 0 && (x < v.border || x >= v.w - v.border || y < v.border || y >= v.h - v.border))
    return true;
  if (!v.holes) return false;
  // 5%: u < 0.05 * 2^53
  return (synth_splitmix(v.seed * 0x100000000ull + 2ull * i + 0x51ed270bull) >> 11) <
         450359962737049ull;
}
HD bool synth_hole_i(const SynthView& v, int i) {
  if (!v.holes) return false;
  // 2%: u < 0.02 * 2^53
  return (synth_splitmix(v.seed * 0x100000000ull + 2ull * i + 0x2545f491ull) >> 11) <
         180143985094819ull;
}

// The views of pair `pair_seed` (host: synth.cpp).
void synth_pair_views(const rgbid_intrinsics* K, uint32_t pair_seed, int variant, SynthView* va,
                      SynthView* vb, rgbid_pose* T_AB_truth);

}  // namespace rgbid_b200
