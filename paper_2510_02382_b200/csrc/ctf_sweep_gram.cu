// Covariance-domain (Gram) iteration kernels for the stacked equal-tap
// configs: (M = N mics/sources, L taps, CTA size, frames per thread).
#include "ctf_sweep_variants.h"
namespace ctf {
#define GF(...) CTF_GR(float, 1, __VA_ARGS__)
#define GD(...) CTF_GR(double, 0, __VA_ARGS__)
std::vector<SweepVariant> sweep_variants_gram_f32() {
#if defined(CTF_GRAM_DEV) && defined(CTF_DEV_F64)
  return {};
#elif defined(CTF_GRAM_DEV) && defined(CTF_DEV_TC)  // dev build of the tcgen05-Gram variant
  return {CTF_GRT(float, 1, CTF_DEV_M, CTF_DEV_L, CTF_DEV_NT, CTF_DEV_FT)};
#elif defined(CTF_GRAM_DEV)  // dev builds (tools/dev_build.sh): only the variant being tuned
  return {GF(CTF_DEV_M, CTF_DEV_L, CTF_DEV_NT, CTF_DEV_FT)};
#else
  return {GF(2, 2, 128, 4), GF(2, 2, 256, 4), GF(2, 3, 128, 4), GF(2, 3, 256, 4),
          GF(2, 5, 256, 4), GF(2, 5, 512, 4), GF(3, 4, 256, 4), GF(3, 4, 512, 4),
          GF(3, 4, 256, 8),  // cfg2 (T = 2000) at two CTAs per SM
          GF(4, 8, 256, 4), GF(4, 8, 512, 2),  // wide tiles (BASELINE cfg3): warp per row, Gram table reads
          CTF_GRT(float, 1, 4, 8, 512, 2)};     // the same with the tcgen05 Gram
#endif
}
std::vector<SweepVariant> sweep_variants_gram_f64() {
#if defined(CTF_GRAM_DEV) && defined(CTF_DEV_F64)  // dev build of one fp64 variant
  return {GD(CTF_DEV_M, CTF_DEV_L, CTF_DEV_NT, CTF_DEV_FT)};
#elif defined(CTF_GRAM_DEV)
  return {};
#else
  return {GD(2, 2, 128, 4), GD(2, 2, 256, 4), GD(2, 3, 128, 4), GD(2, 3, 256, 4),
          GD(2, 5, 256, 4), GD(2, 5, 512, 4), GD(3, 4, 256, 4), GD(3, 4, 512, 4)};
#endif
}
// IP rule (update_rule = ip) on the same kernel
std::vector<SweepVariant> sweep_variants_gram_ip() {
#ifdef CTF_GRAM_DEV
  return {};
#else
  return {CTF_GRI(float, 1, 2, 2, 128, 4), CTF_GRI(float, 1, 2, 3, 256, 4), CTF_GRI(float, 1, 2, 5, 256, 4),
          CTF_GRI(float, 1, 3, 4, 512, 4), CTF_GRI(double, 0, 2, 2, 128, 4), CTF_GRI(double, 0, 2, 3, 256, 4),
          CTF_GRI(double, 0, 2, 5, 256, 4), CTF_GRI(double, 0, 3, 4, 256, 4),
          CTF_GRI(double, 0, 3, 4, 512, 4), CTF_GRI(float, 1, 3, 4, 256, 4)};
#endif
}
}  // namespace ctf
#ifdef CTF_PHASE_TIMING
// dev instrumentation (builds with -DCTF_PHASE_TIMING only): per-CTA clock64
// at the phase boundaries of gram_kernel, tiles < 4096
extern "C" int ctf_debug_gram_phases(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, ctf::g_phase, sizeof(unsigned long long) * 4096 * 12);
}
#endif
