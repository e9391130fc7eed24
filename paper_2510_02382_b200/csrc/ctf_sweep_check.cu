// CheckOptions-instrumented sweep kernels (estimator.hpp:45-48): guarded
// runtime-R variants, selected only when the problem asks for checks; and the
// frame-domain IP-rule variants.
#include "ctf_sweep_variants.h"
namespace ctf {
std::vector<SweepVariant> sweep_variants_check_f32() {
  return {CTF_VCHK3(float, 1, 4, 4, 2), CTF_VCHK3(float, 1, 16, 4, 0),
          // tiles beyond one SM (R > 16 or long frames): the streamed kernel, instrumented
          CTF_STC(float, 1, 4, 8, 256), CTF_STC(float, 1, 8, 8, 512)};
}
// IP rule (update_rule = ip) on layouts the covariance-domain kernel does not
// cover (pre-stacked observations, unequal taps): frame-domain variants
std::vector<SweepVariant> sweep_variants_ip_frame() {
  return {CTF_VIP3(float, 1, 16, 4, 0), CTF_VIP3(double, 0, 16, 4, 0)};
}
std::vector<SweepVariant> sweep_variants_check_f64() {
  return {CTF_VCHK3(double, 0, 4, 4, 2), CTF_VCHK3(double, 0, 16, 4, 0), CTF_STC(double, 0, 4, 4, 256),
          CTF_STC(double, 0, 8, 4, 512)};
}
}  // namespace ctf
