// ctf_sweep_variants.h — registry of compiled sweep_kernel instantiations.
// Variant = (rows RMAX, frames per thread FT, register-resident rows RREG,
// exact CTA size NT, EXACT: R == RMAX at compile time). A variant covers
// T <= FT*NT frames. Within one RMAX the
// host takes the first fitting entry, so the lists are in preference order
// (measured on B200).
#pragma once
#include "ctf_kernels.cuh"

#include <vector>

namespace ctf {
struct SweepVariant {
  int prec, rmax, ft, rreg, maxt, exact;  // maxt == NT
  void (*fn)(SweepParams);
};
#define CTF_V(REAL, PREC, RMAX, FT, RREG, NT, EX) \
  SweepVariant { PREC, RMAX, FT, RREG, NT, EX, sweep_kernel<REAL, RMAX, FT, RREG, NT, EX> }
// one (RMAX, FT, RREG) at the three CTA sizes
#define CTF_V3(REAL, PREC, RMAX, FT, RREG, EX) \
  CTF_V(REAL, PREC, RMAX, FT, RREG, 128, EX), CTF_V(REAL, PREC, RMAX, FT, RREG, 256, EX), \
      CTF_V(REAL, PREC, RMAX, FT, RREG, 512, EX)
}  // namespace ctf
