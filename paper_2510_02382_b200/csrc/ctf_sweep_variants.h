// ctf_sweep_variants.h — registry of compiled sweep_kernel instantiations.
// Variant = (rows RMAX, frames per thread FT, register-resident rows RREG,
// max CTA size MAXT, EXACT: R == RMAX at compile time). Within one RMAX the
// host takes the first fitting entry, so the lists are in preference order
// (measured on B200).
#pragma once
#include "ctf_kernels.cuh"

#include <vector>

namespace ctf {
struct SweepVariant {
  int prec, rmax, ft, rreg, maxt, exact;
  void (*fn)(SweepParams);
};
#define CTF_V(REAL, PREC, RMAX, FT, RREG, MAXT, EX) \
  SweepVariant { PREC, RMAX, FT, RREG, MAXT, EX, sweep_kernel<REAL, RMAX, FT, RREG, MAXT, EX> }
}  // namespace ctf
