// Row-per-warp sweep kernels (ctf_rowwarp.cuh).
#include "ctf_sweep_variants.h"
namespace ctf {
std::vector<SweepVariant> sweep_variants_rowwarp_f32() {
  return {CTF_RW(float, 1, 16, 2, 640), CTF_RW(float, 1, 16, 1, 128), CTF_RW(float, 1, 16, 2, 256),
          CTF_RW(float, 1, 16, 1, 64),  CTF_RW(float, 1, 16, 2, 512), CTF_RW(float, 1, 16, 2, 384)};
}
std::vector<SweepVariant> sweep_variants_rowwarp_f64() {
  return {CTF_RW(double, 0, 16, 2, 640), CTF_RW(double, 0, 16, 1, 128), CTF_RW(double, 0, 16, 2, 256)};
}
}  // namespace ctf
