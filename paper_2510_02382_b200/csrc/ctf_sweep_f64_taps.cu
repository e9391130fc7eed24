// fp64 sweep kernels for the stacked CTF configs (equal taps per source).
#include "ctf_sweep_variants.h"
namespace ctf {
#define V(...) CTF_VL3(double, 0, __VA_ARGS__)
std::vector<SweepVariant> sweep_variants_f64_taps() {
  return {V(10, 4, 2, 5), V(4, 4, 4, 2), V(12, 4, 2, 4), V(6, 4, 3, 3), V(8, 4, 2, 4)};
}
}  // namespace ctf
