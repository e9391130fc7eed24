// ctf_sweep_f64.cu — fp64 instantiations of the fused sweep kernel.
#include "ctf_kernels.cuh"

#include <vector>

namespace ctf {
struct SweepVariant {
  int prec, rmax, ft, rreg, maxt;
  void (*fn)(SweepParams);
};

#define CTF_V(RMAX, FT, RREG, MAXT) {0, RMAX, FT, RREG, MAXT, sweep_kernel<double, RMAX, FT, RREG, MAXT>}

const std::vector<SweepVariant>& sweep_variants_f64() {
  static const std::vector<SweepVariant> v = {
      CTF_V(4, 4, 4, 256),  CTF_V(4, 4, 2, 512),  CTF_V(4, 4, 0, 1024),
      CTF_V(8, 4, 2, 256),  CTF_V(8, 4, 0, 512),  CTF_V(8, 4, 0, 1024),
      CTF_V(10, 4, 2, 256), CTF_V(10, 4, 0, 512), CTF_V(10, 4, 0, 1024),
      CTF_V(12, 4, 0, 512), CTF_V(16, 4, 0, 512), CTF_V(16, 4, 0, 1024),
  };
  return v;
}
}  // namespace ctf
