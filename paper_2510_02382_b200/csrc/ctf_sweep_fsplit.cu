// Frame-split cluster sweep kernels (ctf_fsplit.cuh): on-chip tiles of the
// wide stacked configurations (BASELINE cfg3 R=32 L=8, cfg4 R=60 L=10).
#include "ctf_sweep_variants.h"
namespace ctf {
std::vector<SweepVariant> sweep_variants_fsplit_f32() {
  return {CTF_FS(float, 1, 60, 10, 2, 128, 16, 24, 10, 2), CTF_FS(float, 1, 60, 10, 2, 256, 8, 32, 10, 1),
          CTF_FS(float, 1, 32, 8, 2, 128, 4, 16, 8, 3), CTF_FS(float, 1, 32, 8, 2, 256, 2, 16, 8, 2),
          CTF_FS(float, 1, 32, 8, 1, 128, 8, 16, 8, 3), CTF_FS(float, 1, 32, 8, 4, 128, 2, 16, 8, 2),
          // all-gather exchange variants (one DSMEM hop per step)
          CTF_FSA(float, 1, 60, 10, 2, 256, 8, 32, 10, 1), CTF_FSA(float, 1, 32, 8, 4, 128, 2, 16, 8, 2),
          CTF_FSA(float, 1, 32, 8, 2, 128, 4, 16, 8, 3),
          // step pairs (two ISS steps per pass and per exchange)
          CTF_FSP(float, 1, 60, 10, 2, 256, 8, 32, 4, 1),
          CTF_FSP(float, 1, 32, 8, 4, 128, 2, 16, 4, 2), CTF_FSP(float, 1, 32, 8, 2, 128, 4, 16, 4, 3)};
// (measured and dropped: cfg4 over 9-CTA clusters, NT = 224 — 15 co-resident
// clusters cover 135 SMs instead of 120 (tools/cluster_probe.cu) but the
// cluster count, not the SM count, bounds the bins in flight and each bin's
// 60-step chain is latency-bound: 202.8 vs 201.2 ms per 8 mixtures)
}
}  // namespace ctf
#ifdef CTF_PHASE_TIMING
// dev instrumentation (builds with -DCTF_PHASE_TIMING only): clock64 of the
// cluster's CTA 0 at the phase boundaries of fsplit_kernel, tiles < 4096
extern "C" int ctf_debug_fsplit_phases(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, ctf::g_fphase, sizeof(unsigned long long) * 4096 * 12);
}
#endif
