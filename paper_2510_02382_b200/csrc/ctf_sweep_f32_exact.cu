// fp32 sweep kernels with compile-time row count (the common shapes).
#include "ctf_sweep_variants.h"
namespace ctf {
#define V(...) CTF_V(float, 1, __VA_ARGS__, true)
std::vector<SweepVariant> sweep_variants_f32_exact() {
  return {V(2, 4, 2, 512),  V(2, 4, 2, 1024), V(3, 4, 3, 512),  V(4, 4, 4, 512),  V(4, 4, 4, 1024),
          V(5, 4, 5, 512),  V(6, 4, 6, 256),  V(6, 4, 3, 512),  V(8, 4, 8, 256),  V(8, 4, 4, 512),
          V(10, 4, 5, 512), V(10, 4, 4, 512), V(10, 4, 3, 512), V(10, 4, 10, 256), V(10, 2, 10, 512), V(10, 8, 5, 128), V(10, 4, 0, 1024),
          V(12, 4, 6, 512), V(12, 4, 0, 1024), V(16, 4, 4, 512), V(16, 4, 0, 1024)};
}
}  // namespace ctf
