// CheckOptions-instrumented sweep kernels (estimator.hpp:45-48): guarded
// runtime-R variants, selected only when the problem asks for checks.
#include "ctf_sweep_variants.h"
namespace ctf {
std::vector<SweepVariant> sweep_variants_check_f32() {
  return {CTF_VCHK3(float, 1, 4, 4, 2), CTF_VCHK3(float, 1, 16, 4, 0)};
}
std::vector<SweepVariant> sweep_variants_check_f64() {
  return {CTF_VCHK3(double, 0, 4, 4, 2), CTF_VCHK3(double, 0, 16, 4, 0)};
}
}  // namespace ctf
