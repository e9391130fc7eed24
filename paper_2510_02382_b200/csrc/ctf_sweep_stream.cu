// Streamed sweep kernels (ctf_stream.cuh): the fallback for tiles that do
// not fit one SM (BASELINE cfg3 / cfg4, long fp64 tiles).
#include "ctf_sweep_variants.h"
namespace ctf {
std::vector<SweepVariant> sweep_variants_stream_f32() {
  return {CTF_ST(float, 1, 4, 8, 256, 2), CTF_ST(float, 1, 8, 8, 512, 1), CTF_ST(float, 1, 4, 8, 512, 1),
          CTF_ST(float, 1, 8, 8, 1024, 1), CTF_ST(float, 1, 4, 8, 256, 1)};
}
std::vector<SweepVariant> sweep_variants_stream_f64() {
  return {CTF_ST(double, 0, 4, 4, 256, 1), CTF_ST(double, 0, 8, 4, 512, 1), CTF_ST(double, 0, 4, 4, 512, 1),
          CTF_ST(double, 0, 8, 4, 1024, 1)};
}
}  // namespace ctf
