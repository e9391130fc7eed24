// fp64 sweep kernels with a runtime row count R <= RMAX.
#include "ctf_sweep_variants.h"
namespace ctf {
#define V(...) CTF_V3(double, 0, __VA_ARGS__, false)
std::vector<SweepVariant> sweep_variants_f64_guard() {
  return {V(4, 4, 2), V(8, 4, 1), V(16, 4, 0)};
}
}  // namespace ctf
