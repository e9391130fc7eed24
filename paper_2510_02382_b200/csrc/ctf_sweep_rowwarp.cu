// Row-per-warp sweep kernels (ctf_rowwarp.cuh).
// Measured slower than the kernels the planner prefers for every BASELINE shape
// (DESIGN.md §4): compiled only in dev builds (make DEVK=1), kept for A/B.
#include "ctf_sweep_variants.h"
namespace ctf {
std::vector<SweepVariant> sweep_variants_rowwarp_f32() {
#ifdef CTF_DEV_KERNELS
  return {CTF_RW(float, 1, 16, 2, 640), CTF_RW(float, 1, 16, 1, 128), CTF_RW(float, 1, 16, 2, 256),
          CTF_RW(float, 1, 16, 1, 64),  CTF_RW(float, 1, 16, 2, 512), CTF_RW(float, 1, 16, 2, 384)};
#else
  return {};
#endif
}
std::vector<SweepVariant> sweep_variants_rowwarp_f64() {
#ifdef CTF_DEV_KERNELS
  return {CTF_RW(double, 0, 16, 2, 640), CTF_RW(double, 0, 16, 1, 128), CTF_RW(double, 0, 16, 2, 256)};
#else
  return {};
#endif
}
}  // namespace ctf
