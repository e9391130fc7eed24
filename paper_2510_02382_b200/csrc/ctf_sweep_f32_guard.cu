// fp32 sweep kernels with a runtime row count R <= RMAX (any other shape).
#include "ctf_sweep_variants.h"
namespace ctf {
#define V(...) CTF_V3(float, 1, __VA_ARGS__, false)
std::vector<SweepVariant> sweep_variants_f32_guard() {
  return {V(4, 4, 4), V(8, 4, 4), V(12, 4, 4), V(16, 4, 2)};
}
}  // namespace ctf
