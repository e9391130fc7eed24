// fp64 sweep kernels with compile-time row count.
#include "ctf_sweep_variants.h"
namespace ctf {
#define V(...) CTF_V3(double, 0, __VA_ARGS__, true)
std::vector<SweepVariant> sweep_variants_f64_exact() {
  return {V(2, 4, 2), V(3, 4, 3), V(4, 4, 4), V(6, 4, 3), V(8, 4, 2), V(10, 4, 2), V(12, 4, 2), V(16, 4, 1)};
}
}  // namespace ctf
