// ctf_sweep_f32.cu — fp32 instantiations of the fused sweep kernel.
// Variant = (rows RMAX, frames per thread FT, register-resident rows RREG,
// max CTA size). The host picks the smallest RMAX >= R that fits.
#include "ctf_kernels.cuh"

#include <vector>

namespace ctf {
struct SweepVariant {
  int prec, rmax, ft, rreg, maxt;
  void (*fn)(SweepParams);
};

#define CTF_V(RMAX, FT, RREG, MAXT) {1, RMAX, FT, RREG, MAXT, sweep_kernel<float, RMAX, FT, RREG, MAXT>}

const std::vector<SweepVariant>& sweep_variants_f32() {
  static const std::vector<SweepVariant> v = {
      CTF_V(4, 4, 4, 512),   CTF_V(4, 4, 4, 1024),
      CTF_V(8, 4, 8, 256),   CTF_V(8, 4, 4, 512),   CTF_V(8, 4, 0, 1024),
      CTF_V(10, 4, 10, 256), CTF_V(10, 4, 5, 512),  CTF_V(10, 4, 0, 1024),
      CTF_V(12, 4, 6, 512),  CTF_V(12, 4, 0, 1024),
      CTF_V(16, 4, 4, 512),  CTF_V(16, 4, 0, 1024),
  };
  return v;
}
}  // namespace ctf
