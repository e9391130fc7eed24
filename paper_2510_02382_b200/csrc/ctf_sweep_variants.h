// ctf_sweep_variants.h — registry of compiled sweep_kernel instantiations.
// Variant = (rows RMAX, frames per thread FT, register-resident rows RREG,
// exact CTA size NT, EXACT: R == RMAX at compile time). A variant covers
// T <= FT*NT frames. Within one RMAX the
// host takes the first fitting entry, so the lists are in preference order
// (measured on B200).
#pragma once
#include "ctf_kernels.cuh"
#include "ctf_rowwarp.cuh"
#include "ctf_stream.cuh"
#include "ctf_cluster.cuh"
#include "ctf_gram.cuh"
#include "ctf_fsplit.cuh"

#include <vector>

namespace ctf {
struct SweepVariant {
  int prec, rmax, ft, rreg, maxt, exact;  // maxt == NT
  void (*fn)(SweepParams);
  int kind = 0;  // 0: frame-owner sweep_kernel, 1: rowwarp_kernel (rmax = R, rreg = WPR),
                 // 2: stream_kernel (rmax = 64, rreg = RG, launched through sfn)
  int lt = 0;    // > 0: compiled for equal taps per source (taps == lt)
  void (*sfn)(StreamParams) = nullptr;
  void (*cfn)(ClusterParams) = nullptr;  // kind 3: cluster_kernel (rmax = rows per CTA)
  int chk = 0;  // kind 0 compiled with the CheckOptions instrumentation
  void (*gfn)(SweepParams, const int4*) = nullptr;  // kind 4: gram_kernel (rreg = M, lt = L)
  int ip = 0;  // kind 4 compiled with the IP rule instead of the ISS steps
  int cs = 0;   // kind 5: CTAs per cluster (frame split)
  size_t (*fbytes)(int) = nullptr;  // kind 5: dynamic shared memory for SK bases
  int ag = 0;   // kind 5: all-gather exchange (every CTA derives every z)
  int tc = 0;   // kind 4: tensor-core (tcgen05) Gram
  int pair = 0; // kind 5: two ISS steps per pass and exchange (all-gather only)
  int lpre = 0; // kinds 4, 5: compiled without its own lambda phase (the host runs lambda_kernel ahead)
  int mubout = 0; // kind 5: compiled without MU-B (the host runs mub_kernel after it)
};
inline SweepVariant with_lpre(SweepVariant v, bool lpre, bool mubout = false) {
  v.lpre = lpre ? 1 : 0;
  v.mubout = mubout ? 1 : 0;
  return v;
}
#define CTF_V(REAL, PREC, RMAX, FT, RREG, NT, EX) \
  SweepVariant { PREC, RMAX, FT, RREG, NT, EX, sweep_kernel<REAL, RMAX, FT, RREG, NT, EX> }
// equal-taps variants: LT taps per source (row P = (P / LT, P % LT))
#define CTF_VL(REAL, PREC, RMAX, FT, RREG, NT, LT) \
  SweepVariant { PREC, RMAX, FT, RREG, NT, 1, sweep_kernel<REAL, RMAX, FT, RREG, NT, true, LT>, 0, LT }
#define CTF_VL3(REAL, PREC, RMAX, FT, RREG, LT) \
  CTF_VL(REAL, PREC, RMAX, FT, RREG, 128, LT), CTF_VL(REAL, PREC, RMAX, FT, RREG, 256, LT), \
      CTF_VL(REAL, PREC, RMAX, FT, RREG, 512, LT)
// CheckOptions-instrumented guarded variants (runtime R <= RMAX)
#define CTF_VCHK(REAL, PREC, RMAX, FT, RREG, NT)                                                                 \
  SweepVariant {                                                                                                \
    PREC, RMAX, FT, RREG, NT, 0, sweep_kernel<REAL, RMAX, FT, RREG, NT, false, 0, true>, 0, 0, nullptr, nullptr, \
        1                                                                                                       \
  }
#define CTF_VCHK3(REAL, PREC, RMAX, FT, RREG)                                           \
  CTF_VCHK(REAL, PREC, RMAX, FT, RREG, 128), CTF_VCHK(REAL, PREC, RMAX, FT, RREG, 256), \
      CTF_VCHK(REAL, PREC, RMAX, FT, RREG, 512)
// IP rule on the frame-domain kernel (any layout, runtime R == D <= RMAX)
#define CTF_VIP(REAL, PREC, RMAX, FT, RREG, NT)                                                                  \
  SweepVariant {                                                                                              \
    PREC, RMAX, FT, RREG, NT, 0, sweep_kernel<REAL, RMAX, FT, RREG, NT, false, 0, false, true>, 0, 0, nullptr, \
        nullptr, 0, nullptr, 1                                                                                \
  }
#define CTF_VIP3(REAL, PREC, RMAX, FT, RREG) \
  CTF_VIP(REAL, PREC, RMAX, FT, RREG, 128), CTF_VIP(REAL, PREC, RMAX, FT, RREG, 256), CTF_VIP(REAL, PREC, RMAX, FT, RREG, 512)
// one (RMAX, FT, RREG) at the three CTA sizes
#define CTF_V3(REAL, PREC, RMAX, FT, RREG, EX) \
  CTF_V(REAL, PREC, RMAX, FT, RREG, 128, EX), CTF_V(REAL, PREC, RMAX, FT, RREG, 256, EX), \
      CTF_V(REAL, PREC, RMAX, FT, RREG, 512, EX)
// stream_kernel: any R <= 64 in groups of RG rows, FT frames per thread
#define CTF_ST(REAL, PREC, FT, RG, NT, MINB) \
  SweepVariant { PREC, 64, FT, RG, NT, 0, nullptr, 2, 0, stream_kernel<REAL, FT, RG, NT, MINB> }
// stream_kernel with the CheckOptions instrumentation (any R <= 64)
#define CTF_STC(REAL, PREC, FT, RG, NT) \
  SweepVariant { PREC, 64, FT, RG, NT, 0, nullptr, 2, 0, stream_kernel<REAL, FT, RG, NT, 1, true>, nullptr, 1 }
// cluster_kernel: R = CS * RB rows over a cluster of CS CTAs
#define CTF_CL(REAL, PREC, RB, FT, RREG, NT) \
  SweepVariant { PREC, RB, FT, RREG, NT, 0, nullptr, 3, 0, nullptr, cluster_kernel<REAL, RB, FT, RREG, NT> }
// gram_kernel: covariance-domain steps, M mics = N sources, L taps
#define CTF_GR(REAL, PREC, M, L, NT, FT)                                                                  \
  with_lpre(SweepVariant{PREC, (M) * (L), FT, M, NT, 1, nullptr, 4, L, nullptr, nullptr, 0,               \
                         gram_kernel<REAL, M, L, NT, FT>},                                                \
            gram_lpre<REAL, NT, (M) * (L), FT>())
// gram_kernel with the tcgen05 Gram (fp32)
#define CTF_GRT(REAL, PREC, M, L, NT, FT)                                                                 \
  with_lpre(SweepVariant{PREC, (M) * (L), FT, M, NT, 1, nullptr, 4, L, nullptr, nullptr, 0,               \
                         gram_kernel<REAL, M, L, NT, FT, false, true>, 0, 0, nullptr, 0, 1},              \
            gram_lpre<REAL, NT, (M) * (L), FT>())
#define CTF_GRI(REAL, PREC, M, L, NT, FT)                                                                 \
  with_lpre(SweepVariant{PREC, (M) * (L), FT, M, NT, 1, nullptr, 4, L, nullptr, nullptr, 0,               \
                         gram_kernel<REAL, M, L, NT, FT, true>, 1},                                       \
            gram_lpre<REAL, NT, (M) * (L), FT>())
// fsplit_kernel: R = M * L stacked rows, frames split over a cluster of CS CTAs
#define CTF_FS(REAL, PREC, R, L, FT, NT, CS, RREG, RG, MINB)                                               \
  with_lpre(SweepVariant {                                                                                         \
    PREC, R, FT, RREG, NT, 1, fsplit_kernel<REAL, R, L, FT, NT, CS, RREG, RG, MINB>, 5, L, nullptr, nullptr, 0, \
        nullptr, 0, CS, &FsplitLayout<REAL, R, L, FT, NT, CS, RREG, RG>::bytes                             \
  }, CTF_FS_LPRE != 0, CTF_FS_LPRE != 0 && CTF_FS_MUBOUT != 0)
#define CTF_FSA(REAL, PREC, R, L, FT, NT, CS, RREG, RG, MINB)                                                  \
  with_lpre(SweepVariant {                                                                                                \
    PREC, R, FT, RREG, NT, 1, fsplit_kernel<REAL, R, L, FT, NT, CS, RREG, RG, MINB, true>, 5, L, nullptr, nullptr, 0, \
        nullptr, 0, CS, &FsplitLayout<REAL, R, L, FT, NT, CS, RREG, RG, true>::bytes, 1                         \
  }, CTF_FS_LPRE != 0, CTF_FS_LPRE != 0 && CTF_FS_MUBOUT != 0)
// frame-split, all-gather, two ISS steps per pass / exchange (step pairs)
#define CTF_FSP(REAL, PREC, R, L, FT, NT, CS, RREG, RG, MINB)                                                       \
  with_lpre(SweepVariant {                                                                                                    \
    PREC, R, FT, RREG, NT, 1, fsplit_kernel<REAL, R, L, FT, NT, CS, RREG, RG, MINB, true, true>, 5, L, nullptr,       \
        nullptr, 0, nullptr, 0, CS, &FsplitLayout<REAL, R, L, FT, NT, CS, RREG, RG, true, true>::bytes, 1, 0, 1      \
  }, CTF_FS_LPRE != 0, CTF_FS_LPRE != 0 && CTF_FS_MUBOUT != 0)
// rowwarp_kernel: R = NT / (32 * WPR) rows, FT frames per lane
#define CTF_RW(REAL, PREC, FT, WPR, NT) \
  SweepVariant { PREC, (NT) / (32 * (WPR)), FT, WPR, NT, 1, rowwarp_kernel<REAL, FT, WPR, NT>, 1, 0 }
}  // namespace ctf
