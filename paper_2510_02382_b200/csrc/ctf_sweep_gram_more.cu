// More stacked equal-tap shapes on the covariance-domain kernel (beyond the
// BASELINE configs of ctf_sweep_gram.cu): (mics = sources, taps) pairs with
// R = M * L <= 16, T <= 1024 frames (256 threads, 4 frames per thread), fp32
// and fp64. Other shapes and longer tiles run the frame-domain kernels.
#include "ctf_sweep_variants.h"
namespace ctf {
#define GF(...) CTF_GR(float, 1, __VA_ARGS__)
#define GD(...) CTF_GR(double, 0, __VA_ARGS__)
std::vector<SweepVariant> sweep_variants_gram_more_f32() {
#ifdef CTF_GRAM_DEV
  return {};
#else
  return {GF(2, 4, 256, 4), GF(2, 8, 256, 4), GF(3, 2, 256, 4), GF(3, 3, 256, 4),
          GF(3, 5, 256, 4), GF(4, 2, 256, 4), GF(4, 3, 256, 4), GF(4, 4, 256, 4)};
#endif
}
std::vector<SweepVariant> sweep_variants_gram_more_f64() {
#ifdef CTF_GRAM_DEV
  return {};
#else
  // (no (4, 2): the frame-domain kernel measured faster in fp64, 2.85 vs 3.44 ms per
  // iteration of 16 mixtures at F = 513, T = 1000; tools/shape_sweep.py)
  return {GD(2, 4, 256, 4), GD(2, 8, 256, 4), GD(3, 2, 256, 4), GD(3, 3, 256, 4),
          GD(3, 5, 256, 4), GD(4, 3, 256, 4), GD(4, 4, 256, 4)};
#endif
}
}  // namespace ctf
