// fp32 sweep kernels with compile-time row count (the common shapes).
#include "ctf_sweep_variants.h"
namespace ctf {
#define V(...) CTF_V3(float, 1, __VA_ARGS__, true)
std::vector<SweepVariant> sweep_variants_f32_exact() {
  return {V(2, 4, 2), V(3, 4, 3), V(4, 4, 4), V(5, 4, 5), V(6, 4, 4), V(8, 4, 4),
          V(10, 4, 5), V(10, 4, 3), V(12, 4, 4), V(16, 4, 2)};
}
}  // namespace ctf
