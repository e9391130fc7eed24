// ctf_fsplit.cuh — frame-split thread-block-cluster ISS sweep for tiles that
// exceed one SM (BASELINE cfg3: R = 32, T = 1000; cfg4: R = 60, T = 4000).
//
// Same contract and numerics as sweep_kernel (ctf_kernels.cuh): the bin-local
// part of one iteration of proj/src/estimator.cpp:548-654 for the stacked
// equal-taps layout (R = D = N*L, M = N). A cluster of CS CTAs handles one
// (mixture, bin); CTA c owns frames [c*TC, (c+1)*TC) of ALL rows, so the
// R x T estimate tile stays on chip (RREG rows per thread in registers, the
// rest in shared memory) and every per-frame update is thread-private, as in
// sweep_kernel. The only cross-CTA data per ISS step are the 3R weighted sums
// (estimator.cpp:434-462) and the R steering coefficients z:
//   1. each CTA reduces its frames' sums (warp reduce-scatter + fixed-order
//      cross-warp sum) and pushes row p's partial to the CTA that owns row p
//      (p % CS) with st.async into the owner's shared memory, completing
//      bytes on the owner's mbarrier;
//   2. the owner waits for all CS partials of its rows, sums them in CTA
//      order, derives z_p (estimator.cpp:442-458) and pushes it to every
//      CTA with st.async on their mbarriers;
//   3. every CTA waits for all R coefficients and applies the step.
// No cluster barrier per step: two one-way DSMEM hops, ordered by mbarrier
// transaction counts (double-buffered by step parity). All CTAs derive
// identical z (same inputs, same order), so the run is deterministic.
// W: CTA c updates the columns [c*DC, (c+1)*DC) (W -= z w_r is column-local);
// the demix stages the rescaled W four rows at a time in shared memory. Frame halos: the
// stacked observation and the ISS weights reach L-1 frames back (x and
// 1/lambda are loaded with that halo), the delayed energies reach L-1 frames
// forward (|y|^2 of the next CTA's first L-1 frames, read over DSMEM).
// Objective, row powers and MU-B partials are combined by CTA 0 in CTA order.
#pragma once

#include "ctf_cluster.cuh"
#include "ctf_kernels.cuh"

#ifndef CTF_FS_DCR  // W rows per demix chunk (R = 32: cfg3; wider: cfg4)
#define CTF_FS_DCR 8
#endif
#ifndef CTF_FS_DCR_WIDE
#define CTF_FS_DCR_WIDE 12
#endif
#ifndef CTF_FS_ITB  // frames per batch when all of them would exceed 64 registers
#define CTF_FS_ITB 2
#endif
#ifndef CTF_FS_LAMKB
#define CTF_FS_LAMKB 20
#endif
// 1: 1 / lambda and the objective's log term come from lambda_kernel, run by
// the host ahead of the kernel (SweepVariant::lpre); 0: the kernel's own
// lambda phase (dev builds, A/B)
#ifndef CTF_FS_LPRE
#define CTF_FS_LPRE 1
#endif
// 1: MU-B runs in mub_kernel after this kernel (needs CTF_FS_LPRE: 1/lambda in
// HBM; SweepVariant::mubout tells the host); 0: the in-kernel MU-B passes
#ifndef CTF_FS_MUBOUT
#define CTF_FS_MUBOUT 1
#endif
namespace ctf {

template <typename Real, int R, int L, int FT, int NT, int CS, int RREG, int RG, bool AG = false, bool PAIR = false>
struct FsplitLayout {
  static constexpr int M = R / L;  // mics == sources
  static constexpr int NW = NT / 32;
  static constexpr int TC = FT * NT;  // frames per CTA
  static constexpr int XOFF = L;      // x halo (>= L - 1 frames back)
  static constexpr int XP = XOFF + TC;
  static constexpr int LOFF = ((L + 3) / 4) * 4;  // 1/lambda halo
  static constexpr int LP = LOFF + TC;
  static constexpr int RC = (R + CS - 1) / CS;  // rows owned per CTA (max)
  static constexpr int DC = RC;                 // W columns per CTA
  static constexpr int NG = (R + RG - 1) / RG;  // row groups per pass
  static constexpr int NV = PAIR ? 8 : 3;  // sums per row and exchange: 3R per step, 8R per step pair
  static constexpr int VP = ((NV * RG + 31) / 32) * 32;
  static constexpr int NG2 = (R + 31) / 32;  // row-power groups
  static constexpr int HL = L > 1 ? L - 1 : 1;
  static constexpr int CH = 4 * (int)sizeof(Real);  // bytes per DSMEM message
  static constexpr int CHA = PAIR ? 2 * CH : CH;      // bytes per (row, CTA) partial
  static constexpr int CHZ = PAIR ? 2 * CH : CH;      // bytes per row of the coefficient buffer
  static constexpr size_t RB_ = sizeof(Real), CB_ = 2 * sizeof(Real);
  static constexpr size_t a16(size_t b) { return (b + 15) & ~size_t(15); }
  static constexpr size_t mx(size_t a, size_t b) { return a > b ? a : b; }
  static constexpr size_t off_y = 0;
  static constexpr size_t off_x = off_y + a16((size_t)(R - RREG) * TC * CB_);
  static constexpr size_t off_l = off_x + a16(mx((size_t)M * XP * CB_, (size_t)L * (TC + HL) * RB_));
  static constexpr size_t off_w = off_l + a16((size_t)M * LP * RB_);
  static constexpr size_t off_red = off_w + a16((size_t)2 * R * DC * CB_);
  static constexpr size_t off_a =
      off_red + a16(mx((size_t)NW * mx(mx((size_t)NG * VP, (size_t)NG2 * 32), 16) * RB_, (size_t)(R > 32 ? CTF_FS_DCR_WIDE : CTF_FS_DCR) * R * CB_));
  static constexpr size_t off_z = off_a + a16((size_t)2 * CS * (AG ? R : RC) * CHA);
  static constexpr size_t off_h = off_z + a16((size_t)2 * R * CHZ);
  static constexpr size_t off_ex = off_h + a16((size_t)R * HL * RB_);
  static constexpr size_t off_bar = off_ex + a16((size_t)(8 + R) * 8);
  static constexpr size_t off_bs = off_bar + 64;
  static size_t bytes(int SK) { return off_bs + a16((size_t)SK * RB_) + (size_t)2 * SK * 8; }
};

__device__ __forceinline__ uint32_t smem_u32addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t dsmem_map(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ double dsmem_ld_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ float dsmem_ld_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ double dsmem_ld(uint32_t a, double) { return dsmem_ld_f64(a); }
__device__ __forceinline__ float dsmem_ld(uint32_t a, float) { return dsmem_ld_f32(a); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
// one local arrival that also expects `tx` bytes of st.async data this phase
__device__ __forceinline__ void mbar_arm(uint32_t bar, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
}
// The messages land in this CTA's shared memory, so the phase completion
// (default .acquire.cta) orders them; a cluster-scope acquire would also
// invalidate L1 on every wait (CCTL.IVALL, measured: 14 % of the stall samples).
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
// 4-value message into another CTA's shared memory, completing its bytes on
// that CTA's mbarrier (addresses already mapped with dsmem_map)
__device__ __forceinline__ void msg_send(uint32_t raddr, uint32_t rbar, float a, float b, float c, float d) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   raddr),
               "f"(a), "f"(b), "f"(c), "f"(d), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void msg_send(uint32_t raddr, uint32_t rbar, double a, double b, double c, double d) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "d"(a), "d"(b), "r"(rbar)
               : "memory");
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr +
                                                                                                           16),
               "d"(c), "d"(d), "r"(rbar)
               : "memory");
}

// Warp reduce-scatter (see warp_reduce_scatter) with the adds of two values
// packed into one FADD2: the same keep + received sums, bit-identical.
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(d);
}
template <int CNT, int OFF, int V>
__device__ __forceinline__ void rs_level_packed(float (&v)[V], int lane) {
  if constexpr (OFF >= 1) {
    constexpr int H = CNT / 2;
    const bool upper = (lane & OFF) != 0;
    if constexpr (H >= 2) {
#pragma unroll
      for (int i = 0; i < H; i += 2) {
        const float s0 = upper ? v[i] : v[i + H], s1 = upper ? v[i + 1] : v[i + 1 + H];
        const float k0 = upper ? v[i + H] : v[i], k1 = upper ? v[i + 1 + H] : v[i + 1];
        const float r0 = __shfl_xor_sync(kFull, s0, OFF), r1 = __shfl_xor_sync(kFull, s1, OFF);
        const float2 t = fadd2(make_float2(k0, k1), make_float2(r0, r1));
        v[i] = t.x;
        v[i + 1] = t.y;
      }
    } else {
      const float send = upper ? v[0] : v[1], keep = upper ? v[1] : v[0];
      v[0] = keep + __shfl_xor_sync(kFull, send, OFF);
    }
    rs_level_packed<H, OFF / 2>(v, lane);
  }
}
template <int V> __device__ __forceinline__ void warp_reduce_scatter_fast(float (&v)[V], int lane) {
  static_assert(V % 32 == 0, "pad the value count to a multiple of 32");
  rs_level_packed<V, 16>(v, lane);
}
template <int V> __device__ __forceinline__ void warp_reduce_scatter_fast(double (&v)[V], int lane) {
  warp_reduce_scatter(v, lane);
}

// AG: every CTA gathers all CS partials of every row and derives all R
// coefficients itself (one DSMEM hop per step, CS x 3R values received)
// instead of the owner scheme (two hops, 3R values)
#ifdef CTF_PHASE_TIMING
__device__ unsigned long long g_fphase[4096 * 12];  // dev instrumentation: clock64 per phase, CTA 0 tid 0
#define CTF_FPHASE(k) \
  if (c == 0 && tid == 0 && tile < 4096) g_fphase[tile * 12 + (k)] = clock64();
#else
#define CTF_FPHASE(k)
#endif
template <typename Real, int R, int L, int FT, int NT, int CS, int RREG, int RG, int MINB, bool AG = false,
          bool PAIR = false>
__global__ void __launch_bounds__(NT, MINB) fsplit_kernel(const SweepParams p) {
  using R2 = typename Cplx<Real>::T;
  using LY = FsplitLayout<Real, R, L, FT, NT, CS, RREG, RG, AG, PAIR>;
  static_assert(!PAIR || (AG && R % 2 == 0 && std::is_same<Real, float>::value),
                "step pairs: all-gather exchange, even R, fp32");
  constexpr int N = LY::M, M = LY::M, NW = LY::NW, TC = LY::TC, XP = LY::XP, XOFF = LY::XOFF;
  constexpr bool MUBOUT = CTF_FS_LPRE != 0 && CTF_FS_MUBOUT != 0;
  constexpr int LP = LY::LP, LOFF = LY::LOFF, RC = LY::RC, DC = LY::DC, NG = LY::NG, VP = LY::VP;
  constexpr int VM = VP / 32, HL = LY::HL, CH = LY::CH, RS = R - RREG;
  static_assert(R % L == 0 && R <= 64 && R >= CS && RREG <= R, "stacked equal-taps tiles, one owner per row");
  static_assert(TC % 32 == 0, "whole warps of frames");
  static_assert(RC * CS <= NT, "one thread per (owned row, destination CTA)");
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = (int)cluster_ctarank();
  const int bin = blockIdx.x / CS, mix = blockIdx.y, gbin = p.bin_lo + bin;
  const int T = p.T, SK = p.SK;
  const int j0 = c * TC;  // first global frame of this CTA

  R2* Ysm = reinterpret_cast<R2*>(smem + LY::off_y);      // RS x TC
  R2* xs = reinterpret_cast<R2*>(smem + LY::off_x);       // M x XP (frames j0 - XOFF ..)
  Real* Pn = reinterpret_cast<Real*>(smem + LY::off_x);   // epilogue: L x (TC + HL) |y|^2 of one source
  Real* invl = reinterpret_cast<Real*>(smem + LY::off_l); // N x LP (frames j0 - LOFF ..)
  R2* Wsl = reinterpret_cast<R2*>(smem + LY::off_w);      // 2 x DC x R (own columns, ping-pong)
  Real* red = reinterpret_cast<Real*>(smem + LY::off_red);
  double* dred = reinterpret_cast<double*>(smem + LY::off_red);
  unsigned char* inA = smem + LY::off_a;  // [2][CS][RC] partial sums of the own rows
  unsigned char* inZ = smem + LY::off_z;  // [2][R] steering coefficients (z.x, z.y, bad, 0)
  Real* halo = reinterpret_cast<Real*>(smem + LY::off_h);  // R x HL |y|^2 of the first frames
  double* ex = reinterpret_cast<double*>(smem + LY::off_ex);  // [0,4) objective, [4,4+R) row powers, [4+R,8+R) totals
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + LY::off_bar);  // A0 A1 Z0 Z1
  Real* Bs = reinterpret_cast<Real*>(smem + LY::off_bs);
  double* exmub = reinterpret_cast<double*>(smem + LY::off_bs + LY::a16((size_t)SK * sizeof(Real)));
  __shared__ int s_wbad;

  const size_t tile = (size_t)mix * p.FL + bin;
  CTF_FPHASE(0);
  const R2* xg = reinterpret_cast<const R2*>(p.x) + tile * (size_t)T * M;
  R2* Wg = reinterpret_cast<R2*>(p.W) + tile * (size_t)R * R;
  Real* Bg = reinterpret_cast<Real*>(p.Bf) + tile * SK;
  const Real* Vg = reinterpret_cast<const Real*>(p.V) + (size_t)mix * SK * T;
  const Real floor_abs = (Real)p.floor_abs[mix];
  const int prev_it = p.iteration - 1;
  const double* mu = p.mu ? p.mu + (size_t)mix * R : nullptr;
  const int nown = (R - c + CS - 1) / CS;  // rows p with p % CS == c
  const uint32_t txA = (uint32_t)(CS * (AG ? R : nown) * LY::CHA), txZ = (uint32_t)(R * CH);
  const uint32_t barA[2] = {smem_u32addr(bars + 0), smem_u32addr(bars + 1)};
  const uint32_t barZ[2] = {smem_u32addr(bars + 2), smem_u32addr(bars + 3)};

  if (tid == 0) {
    s_wbad = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) mbar_init(smem_u32addr(bars + b), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_arm(barA[0], txA);  // steps 0 and 1
    mbar_arm(barA[1], txA);
    mbar_arm(barZ[0], txZ);
    mbar_arm(barZ[1], txZ);
  }
  // z of "step -1" (zero update in the first pass)
  for (int i = tid; i < R * LY::CHZ / (int)sizeof(Real); i += NT)
    reinterpret_cast<Real*>(inZ + (size_t)R * LY::CHZ)[i] = Real(0);
  // own W columns, B and the pending rescale factors: loads issued before the
  // x tile's so their latency overlaps (rescaled and stored below)
  constexpr int WPT = (R * DC + NT - 1) / NT;
  R2 wv[WPT];
  double mv[WPT];
#pragma unroll
  for (int t = 0; t < WPT; ++t) {
    const int e = tid + t * NT, q = e % R, col = c * DC + e / R;
    wv[t] = czero<Real>();
    mv[t] = 0.0;
    if (e < R * DC && col < R) {
      wv[t] = Wg[(size_t)col * R + q];
      if (mu) mv[t] = mu[q];
    }
  }
  const bool b1 = SK <= NT;
  Real bv = Real(0);
  double mbv = 0.0;
  if (b1 && tid < SK) {
    bv = Bg[tid];
    int nb = 0;
#pragma unroll
    for (int n = 1; n < N; ++n) nb += tid >= p.koff[n] ? 1 : 0;
    if (mu) mbv = mu[nb * L];
  }
  // ---- prologue: x tile with its halo, own W columns and B with the pending rescale
  {
    // all of the thread's loads in flight before the transposing stores
    constexpr int XPT = (XP * M + NT - 1) / NT;
    R2 xv[XPT];
#pragma unroll
    for (int t = 0; t < XPT; ++t) {
      const int e = tid + t * NT, i = e / M;
      const int j = j0 - XOFF + i;
      xv[t] = (e < XP * M && j >= 0 && j < T) ? xg[(size_t)j0 * M - XOFF * M + e] : czero<Real>();
    }
#pragma unroll
    for (int t = 0; t < XPT; ++t) {
      const int e = tid + t * NT, i = e / M, m = e - i * M;
      if (e < XP * M) xs[m * XP + i] = xv[t];
    }
  }
#pragma unroll
  for (int t = 0; t < WPT; ++t) {
    const int e = tid + t * NT, col = c * DC + e / R;
    if (e < R * DC) {
      R2 w = wv[t];
      if (col < R) {
        const double m = mv[t];
        if (mu && m != 0.0) {
          w.x = (Real)((double)w.x / m);
          w.y = (Real)((double)w.y / m);
        }
        if (p.has_prev && !cfinite(w)) s_wbad = 1;
      }
      Wsl[e] = w;
    }
  }
  if (b1) {
    if (tid < SK) {
      Real b = bv;
      if (mbv != 0.0) b = (Real)fmax((double)b / (mbv * mbv), (double)floor_abs);
      Bs[tid] = b;
    }
  } else {
    for (int n = 0; n < N; ++n) {
      const double m0 = mu ? mu[n * L] : 0.0;
      for (int i = p.koff[n] + tid; i < p.koff[n + 1]; i += NT) {
        Real b = Bg[i];
        if (m0 != 0.0) b = (Real)fmax((double)b / (m0 * m0), (double)floor_abs);
        Bs[i] = b;
      }
    }
  }
  cluster_sync_all();  // mbarriers initialised cluster-wide; Bs, inZ visible in the CTA
  CTF_FPHASE(1);
  // ---- lambda = max(B V, floor) -> 1/lambda over the frames j0 - LOFF .. j0 + TC
  double logsum = 0.0;
  if constexpr (CTF_FS_LPRE != 0) {
    // computed ahead by lambda_kernel (ctf_kernels.cuh) for the whole bin: this
    // CTA copies its frame slice with the halo (all loads independent: one L2
    // round trip instead of K dependent V loads per frame at one CTA per SM);
    // the objective's log term of the bin goes in through cluster CTA 0
    const Real* lg = reinterpret_cast<const Real*>(p.invl_g) + tile * (size_t)N * T;
    constexpr int IT = (N * LP + NT - 1) / NT;
    Real lv[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int e = tid + it * NT, n = e / LP, i = e - n * LP, tau = j0 + i - LOFF;
      lv[it] = (e < N * LP && tau >= 0 && tau < T) ? __ldg(lg + (size_t)n * T + tau) : Real(0);
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int e = tid + it * NT;
      if (e < N * LP) invl[e] = lv[it];
    }
    if (p.has_prev && c == 0 && tid == 0) logsum = p.logsum_g[tile];
  } else {
  for (int n = 0; n < N; ++n) {
    const int k0 = p.koff[n], k1 = p.koff[n + 1];
    // ITB of the thread's IT frames x KB columns in flight at once (all IT
    // frames when that stays within 64 registers: one L2 round trip per
    // source for K <= KB); same summation order per frame
    constexpr int KB = CTF_FS_LAMKB, IT = (LP + NT - 1) / NT, ITB = IT * KB <= 64 ? IT : CTF_FS_ITB;
#pragma unroll 1
    for (int it0 = 0; it0 < IT; it0 += ITB) {
      Real lamv[ITB];
#pragma unroll
      for (int it = 0; it < ITB; ++it) lamv[it] = Real(0);
      for (int kk = k0; kk < k1; kk += KB) {
        Real vq[ITB][KB];
#pragma unroll
        for (int it = 0; it < ITB; ++it) {
          const int i = tid + (it0 + it) * NT, tau = j0 + i - LOFF;
          const bool ok = i < LP && tau >= 0 && tau < T;
#pragma unroll
          for (int q = 0; q < KB; ++q) vq[it][q] = (ok && kk + q < k1) ? __ldg(Vg + (size_t)(kk + q) * T + tau) : Real(0);
        }
#pragma unroll
        for (int it = 0; it < ITB; ++it)
#pragma unroll
          for (int q = 0; q < KB; ++q)
            if (kk + q < k1) lamv[it] = fma(Bs[kk + q], vq[it][q], lamv[it]);
      }
#pragma unroll
      for (int it = 0; it < ITB; ++it) {
        const int i = tid + (it0 + it) * NT;
        if (i < LP) {
          const int jl = i - LOFF, tau = j0 + jl;
          Real v = Real(0);
          if (tau >= 0 && tau < T) {
            const Real lam = fmax(lamv[it], floor_abs);
            v = rcp_rn(lam);
            if (p.has_prev && jl >= 0) logsum += (double)min(L, T - tau) * (double)log(lam);
          }
          invl[n * LP + i] = v;
        }
      }
    }
  }
  }
  __syncthreads();
  CTF_FPHASE(2);

  // ---- Y = (W / mu) x~ for the own frames (estimator.cpp:555), CR rows per
  // chunk: the chunk's rescaled W rows staged column-major in shared memory
  // (the reduction buffer is free here), the next chunk prefetched into
  // registers; the stacked channel (m, l) is x_m(t - l) from the x tile
  YTile<R2, FT, RREG, RS> Y;
  Y.sm = Ysm;
  Y.tp = TC;
  {
    constexpr int CR = R > 32 ? CTF_FS_DCR_WIDE : CTF_FS_DCR;  // rows per chunk
    constexpr int NCH = (R + CR - 1) / CR, WPT = (CR * R + NT - 1) / NT;
    R2* wst = reinterpret_cast<R2*>(smem + LY::off_red);  // [R columns][CR rows]
    R2 wpre[WPT];
    auto fetch = [&](int r0) {
#pragma unroll
      for (int t = 0; t < WPT; ++t) {
        const int e = tid + t * NT, cc = e / CR, q = r0 + (e % CR);
        R2 w = czero<Real>();
        if (cc < R && q < R) {
          w = Wg[(size_t)cc * R + q];
          if (mu) {
            const double m = mu[q];
            if (m != 0.0) {
              w.x = (Real)((double)w.x / m);
              w.y = (Real)((double)w.y / m);
            }
          }
        }
        wpre[t] = w;
      }
    };
    fetch(0);
    static_for<0, NCH>([&](auto chunk) {
      constexpr int r0 = decltype(chunk)::value * CR;
      __syncthreads();  // the previous chunk's reads of wst are done
#pragma unroll
      for (int t = 0; t < WPT; ++t)
        if (tid + t * NT < CR * R) wst[tid + t * NT] = wpre[t];
      __syncthreads();
      if constexpr (r0 + CR < R) fetch(r0 + CR);
      R2 acc[FT][CR];
#pragma unroll
      for (int k = 0; k < FT; ++k)
#pragma unroll
        for (int i = 0; i < CR; ++i) acc[k][i] = czero<Real>();
#pragma unroll 4
      for (int cc = 0; cc < R; ++cc) {
        const int m = cc / L, l = cc - m * L;
        const R2* xrow = xs + m * XP + XOFF - l + tid;
        R2 w[CR];
#pragma unroll
        for (int i = 0; i < CR; ++i) w[i] = wst[cc * CR + i];
#pragma unroll
        for (int k = 0; k < FT; ++k) {
          const R2 xv = xrow[k * NT];
          if constexpr (std::is_same<Real, float>::value) {
            const float2 xn = make_float2(-xv.y, xv.x);
#pragma unroll
            for (int i = 0; i < CR; ++i) acc[k][i] = ffma2s(xn, w[i].y, ffma2s(xv, w[i].x, acc[k][i]));
          } else {
#pragma unroll
            for (int i = 0; i < CR; ++i) cmac(acc[k][i], w[i], xv);
          }
        }
      }
      static_for<0, CR>([&](auto ii) {
        constexpr int P = r0 + decltype(ii)::value;
        if constexpr (P < R) {
#pragma unroll
          for (int k = 0; k < FT; ++k) {
            const int jl = tid + k * NT;
            Y.template set<P>(k, jl, (j0 + jl < T) ? acc[k][decltype(ii)::value] : czero<Real>());
          }
        }
      });
    });
    __syncthreads();  // wst (the reduction buffer) is reused by the objective sums
  }
  CTF_FPHASE(3);

  // ISS weights: w_p(j) = 1/lambda_{n_p}(j - l_p), row P = (P / L, P % L)
  const Real* wsrc[N];
#pragma unroll
  for (int n = 0; n < N; ++n) wsrc[n] = invl + n * LP + LOFF + tid;
  auto weight = [&](auto pp, int k) -> Real {
    constexpr int P = decltype(pp)::value;
    return wsrc[P / L][k * NT - (P % L)];
  };

  double logdet = p.logdet[tile] - (mu ? p.logmu[mix] : 0.0);
  if (p.has_prev) {
    // objective of the previous iteration (estimator.cpp:55-77): this CTA's
    // frames, combined over the cluster in CTA order
    Real qf = Real(0), sy = Real(0);
    static_for<0, R>([&](auto pp) {
      constexpr int P = decltype(pp)::value;
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        const R2 y = Y.template get<P>(k, tid + k * NT);
        sy += y.x + y.y;
        qf = fma(cnorm(y), weight(pp, k), qf);
      }
    });
    double v4[4] = {logsum, (double)qf, s_wbad ? 1.0 : 0.0, (isfinite(sy) && isfinite(qf)) ? 0.0 : 1.0};
    block_sum_d<4>(v4, dred, lane, warp, NW);
    if (tid == 0)
#pragma unroll
      for (int q = 0; q < 4; ++q) ex[q] = v4[q];
    cluster_sync_all();
    if (tid < 4) {
      double s = 0.0;
      for (int q = 0; q < CS; ++q) s += dsmem_ld_f64(dsmem_map(smem_u32addr(ex + tid), (uint32_t)q));
      ex[4 + R + tid] = s;
    }
    __syncthreads();
    const double* tot = ex + 4 + R;
    int status = 0;
    unsigned long long key = 0;
    if (tot[2] > 0.0) {  // check_all_finite on W (estimator.cpp:494-496)
      status = 1;
      key = err_key(prev_it, kPhFinite, gbin, 0, 1);
    } else if (tot[3] > 0.0) {  // non-finite estimates (estimator.cpp:497-499)
      status = 1;
      key = err_key(prev_it, kPhFinite, gbin, 0, 2);
    } else {
      const int det_status = isnan(logdet) || logdet == -INFINITY ? 4 : (logdet < log(1e-300) ? 5 : 0);
      if (det_status) {  // estimator.cpp:45-51
        status = 1;
        key = err_key(prev_it, kPhDet, gbin, 0, det_status);
      }
    }
    if (status) {
      if (c == 0 && tid == 0) record_err<Real>(p.err, mix, key);
      cluster_sync_all();  // remote reads of ex done before any CTA exits
      return;
    }
    if (c == 0 && tid == 0) p.objbin[tile] = tot[0] + tot[1] - 2.0 * (double)T * logdet;
  }

  if (!p.do_sweep) {  // finalize pass: write the rescaled state and stop
    if (!p.has_prev) cluster_sync_all();  // every CTA is past its demix reads of W
    for (int e = tid; e < R * DC; e += NT) {
      const int q = e % R, i = e / R, col = c * DC + i;
      if (col < R) Wg[(size_t)col * R + q] = Wsl[e];
    }
    if (c == 0) {
      for (int i = tid; i < SK; i += NT) Bg[i] = Bs[i];
      if (tid == 0) p.logdet[tile] = logdet;
    }
    cluster_sync_all();
    return;
  }

  CTF_FPHASE(4);
  // ---- ISS sweep (estimator.cpp:556-579). The pass of step r applies step
  // r-1's update (y_p -= z_p y_{r-1}) and accumulates step r's sums.
  R2 pv[FT], pc[FT];  // pivot row(s) of the previous step (pair: rows a and c at the pair's start)
#pragma unroll
  for (int k = 0; k < FT; ++k) pv[k] = pc[k] = czero<Real>();
  double dprod = 1.0;  // prod_r (1 - z_r): det W' = det W prod_r (1 - z_r)
  int badrow = -1, badstep = 0;
  if constexpr (PAIR) {
    // Steps a = r and c = r + 1 in ONE pass and ONE exchange. With the rows
    // y_p at the pair's start and w = w_p, the pass accumulates
    //   S_pa = sum w y_p conj(y_a), S_pc = sum w y_p conj(y_c),
    //   G_aa = sum w |y_a|^2, G_cc = sum w |y_c|^2, G_ac = sum w y_a conj(y_c);
    // step a is z_p = S_pa / G_aa (estimator.cpp:442-458); step c acts on
    // y_p' = y_p - z_p y_a and y_c' = y_c - z_c y_a, whose sums expand exactly:
    //   numer'_p = S_pc - conj(z_c) S_pa - z_p G_ac + z_p conj(z_c) G_aa,
    //   denom'_p = G_cc - 2 Re(z_c G_ac) + |z_c|^2 G_aa;
    // and both updates apply at once (next pass): y_p -= alpha_p y_a + beta_p y_c,
    // alpha_p = z_p - z'_p z_c, beta_p = z'_p (the same for W's rows).
    constexpr int CHZ = LY::CHZ, CHA = LY::CHA;
    for (int r = 0; r < R; r += 2) {
      const int s2 = r >> 1, buf = s2 & 1;
      const unsigned char* zprev = inZ + (size_t)(buf ^ 1) * R * CHZ;
      auto coef = [&](int P) -> float4 { return *reinterpret_cast<const float4*>(zprev + (size_t)P * CHZ); };
      R2 ya[FT], yc[FT];
      float2 g1[FT], g2[FT];  // (|y_a|^2, |y_c|^2), y_a conj(y_c)
      {
        const float4 ca = coef(r), cc = coef(r + 1);
#pragma unroll
        for (int k = 0; k < FT; ++k) {
          const int jl = tid + k * NT;
          float2 u = Y.pick(k, jl, r), v = Y.pick(k, jl, r + 1);
          const float2 pvs = make_float2(pv[k].y, -pv[k].x), pcs = make_float2(pc[k].y, -pc[k].x);
          u = ffma2s(pv[k], -ca.x, u);
          u = ffma2s(pvs, ca.y, u);
          u = ffma2s(pc[k], -ca.z, u);
          u = ffma2s(pcs, ca.w, u);
          v = ffma2s(pv[k], -cc.x, v);
          v = ffma2s(pvs, cc.y, v);
          v = ffma2s(pc[k], -cc.z, v);
          v = ffma2s(pcs, cc.w, v);
          ya[k] = u;
          yc[k] = v;
          g1[k] = make_float2(cnorm(u), cnorm(v));
          g2[k] = make_float2(fmaf(u.x, v.x, u.y * v.y), fmaf(u.y, v.x, -u.x * v.y));
        }
      }
      static_for<0, NG>([&](auto gg) {
        constexpr int g = decltype(gg)::value;
        Real a[VP];
#pragma unroll
        for (int i = 0; i < VP; ++i) a[i] = Real(0);
        static_for<0, RG>([&](auto qq) {
          constexpr int q = decltype(qq)::value, P = g * RG + q;
          if constexpr (P < R) {
            const float4 cp = coef(P);
            float2 q1a = make_float2(0.f, 0.f), q2a = q1a, q1c = q1a, q2c = q1a, gs1 = q1a, gs2 = q1a;
#pragma unroll
            for (int k = 0; k < FT; ++k) {
              const int jl = tid + k * NT;
              float2 y = Y.template get<P>(k, jl);
              y = ffma2s(pv[k], -cp.x, y);
              y = ffma2s(make_float2(pv[k].y, -pv[k].x), cp.y, y);
              y = ffma2s(pc[k], -cp.z, y);
              y = ffma2s(make_float2(pc[k].y, -pc[k].x), cp.w, y);
              Y.template set<P>(k, jl, y);
              const float w = weight(std::integral_constant<int, P>{}, k);
              const float2 swa = fmul2s(ya[k], w), swc = fmul2s(yc[k], w);
              q1a = ffma2s(y, swa.x, q1a);
              q2a = ffma2s(y, swa.y, q2a);
              q1c = ffma2s(y, swc.x, q1c);
              q2c = ffma2s(y, swc.y, q2c);
              gs1 = ffma2s(g1[k], w, gs1);
              gs2 = ffma2s(g2[k], w, gs2);
            }
            a[q] = q1a.x + q2a.y;           // Re S_pa
            a[RG + q] = q1a.y - q2a.x;      // Im S_pa
            a[2 * RG + q] = q1c.x + q2c.y;  // Re S_pc
            a[3 * RG + q] = q1c.y - q2c.x;  // Im S_pc
            a[4 * RG + q] = gs1.x;          // G_aa
            a[5 * RG + q] = gs1.y;          // G_cc
            a[6 * RG + q] = gs2.x;          // Re G_ac
            a[7 * RG + q] = gs2.y;          // Im G_ac
          }
        });
        warp_reduce_scatter_fast(a, lane);
        Real* rb = red + ((size_t)warp * NG + g) * VP;
#pragma unroll
        for (int i = 0; i < VM; ++i) rb[lane * VM + i] = a[i];
      });
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        pv[k] = ya[k];
        pc[k] = yc[k];
      }
      __syncthreads();
      // this CTA's partial of row `tid` -> every CTA of the cluster
      if (tid < R) {
        const int g = tid / RG, q = tid - g * RG;
        Real v8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v8[i] = Real(0);
        for (int w = 0; w < NW; ++w) {
          const Real* rb = red + ((size_t)w * NG + g) * VP;
#pragma unroll
          for (int i = 0; i < 8; ++i) v8[i] += rb[i * RG + q];
        }
        const uint32_t la = smem_u32addr(inA + ((size_t)(buf * CS + c) * R + tid) * CHA);
#pragma unroll 1
        for (int dst = 0; dst < CS; ++dst) {
          const uint32_t ra = dsmem_map(la, (uint32_t)dst), rbar = dsmem_map(barA[buf], (uint32_t)dst);
          msg_send(ra, rbar, v8[0], v8[1], v8[2], v8[3]);
          msg_send(ra + 16, rbar, v8[4], v8[5], v8[6], v8[7]);
        }
      }
      mbar_wait_parity(barA[buf], (uint32_t)((s2 >> 1) & 1));
      if (tid == 0) mbar_arm(barA[buf], txA);  // pair s2 + 2
      if (tid < R) {  // both steps' coefficients of row `tid` from the CS partials in CTA order
        Real v8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v8[i] = Real(0);
        Real sca_x = Real(0), sca_y = Real(0), gaa_c = Real(0);  // row c's step-a sums (z_c)
        for (int q = 0; q < CS; ++q) {
          const float4* e = reinterpret_cast<const float4*>(inA + ((size_t)(buf * CS + q) * R + tid) * CHA);
          const float4 e0 = e[0], e1 = e[1];
          v8[0] += e0.x;
          v8[1] += e0.y;
          v8[2] += e0.z;
          v8[3] += e0.w;
          v8[4] += e1.x;
          v8[5] += e1.y;
          v8[6] += e1.z;
          v8[7] += e1.w;
          const float4* ec = reinterpret_cast<const float4*>(inA + ((size_t)(buf * CS + q) * R + r + 1) * CHA);
          const float4 c0 = ec[0], c1 = ec[1];
          sca_x += c0.x;
          sca_y += c0.y;
          gaa_c += c1.x;
        }
        const Real gaa = v8[4];
        const bool bad_a = !(gaa > Real(0)) || !isfinite(gaa);  // estimator.cpp:451-454
        Real zx, zy = Real(0);
        if (tid == r) {
          zx = Real(1) - sqrt((Real)T / gaa);
        } else {
          zx = v8[0] / gaa;
          zy = v8[1] / gaa;
        }
        const Real zcx = sca_x / gaa_c, zcy = sca_y / gaa_c;  // z_c of step a (row c is never the pivot a)
        // numer' = S_pc - conj(z_c) S_pa - z_p G_ac + z_p conj(z_c) G_aa
        const Real zzx = zx * zcx + zy * zcy, zzy = zy * zcx - zx * zcy;  // z_p conj(z_c)
        const Real nx = v8[2] - (zcx * v8[0] + zcy * v8[1]) - (zx * v8[6] - zy * v8[7]) + zzx * gaa;
        const Real ny = v8[3] - (zcx * v8[1] - zcy * v8[0]) - (zx * v8[7] + zy * v8[6]) + zzy * gaa;
        // denom' = G_cc - 2 Re(z_c G_ac) + |z_c|^2 G_aa
        const Real dn = v8[5] - Real(2) * (zcx * v8[6] - zcy * v8[7]) + (zcx * zcx + zcy * zcy) * gaa;
        const bool bad_c = !(dn > Real(0)) || !isfinite(dn);
        Real z2x, z2y = Real(0);
        if (tid == r + 1) {
          z2x = Real(1) - sqrt((Real)T / dn);
        } else {
          z2x = nx / dn;
          z2y = ny / dn;
        }
        float4* zo = reinterpret_cast<float4*>(inZ + ((size_t)buf * R + tid) * CHZ);
        // alpha = z_p - z'_p z_c, beta = z'_p
        zo[0] = make_float4(zx - (z2x * zcx - z2y * zcy), zy - (z2x * zcy + z2y * zcx), z2x, z2y);
        zo[1] = make_float4(bad_a ? Real(1) : Real(0), bad_c ? Real(1) : Real(0), tid == r ? zx : z2x, Real(0));
      }
      __syncthreads();
      const unsigned char* zcur = inZ + (size_t)buf * R * CHZ;
      auto flag = [&](int P, int i) -> bool {
        return P < R && reinterpret_cast<const Real*>(zcur + (size_t)P * CHZ + CH)[i] != Real(0);
      };
      {
        const unsigned ma1 = __ballot_sync(kFull, flag(lane, 0)), ma2 = __ballot_sync(kFull, flag(lane + 32, 0));
        const unsigned mc1 = __ballot_sync(kFull, flag(lane, 1)), mc2 = __ballot_sync(kFull, flag(lane + 32, 1));
        if (ma1 | ma2) {
          badrow = ma1 ? __ffs(ma1) - 1 : 32 + __ffs(ma2) - 1;
          badstep = r;
          break;
        }
        if (mc1 | mc2) {
          badrow = mc1 ? __ffs(mc1) - 1 : 32 + __ffs(mc2) - 1;
          badstep = r + 1;
          break;
        }
      }
      const Real za = reinterpret_cast<const Real*>(zcur + (size_t)r * CHZ + CH)[2];
      const Real zc2 = reinterpret_cast<const Real*>(zcur + (size_t)(r + 1) * CHZ + CH)[2];
      dprod *= (double)(Real(1) - za);
      dprod *= (double)(Real(1) - zc2);
      // both steps on the own W columns: W -= alpha w_a + beta w_c (pair-start rows), ping-pong
      const R2* Wo = Wsl + (size_t)(s2 & 1) * R * DC;
      R2* Wn = Wsl + (size_t)((s2 + 1) & 1) * R * DC;
      for (int e = tid; e < R * DC; e += NT) {
        const int q = e % R, i = e / R;
        const float4 cq = *reinterpret_cast<const float4*>(zcur + (size_t)q * CHZ);
        R2 w = Wo[e];
        cmsub(w, make_float2(cq.x, cq.y), Wo[i * R + r]);
        cmsub(w, make_float2(cq.z, cq.w), Wo[i * R + r + 1]);
        Wn[e] = w;
      }
    }
  } else
  for (int r = 0; r < R; ++r) {
    const int buf = r & 1;
    const unsigned char* zprev = inZ + (size_t)(buf ^ 1) * R * CH;
    auto zof = [&](int P) -> R2 { return *reinterpret_cast<const R2*>(zprev + (size_t)P * CH); };
    R2 yr[FT];
    Real ar2[FT];
    {
      const R2 zr = zof(r);
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        R2 y = Y.pick(k, tid + k * NT, r);
        if constexpr (std::is_same<Real, float>::value) {
          y = ffma2s(pv[k], -zr.x, y);
          y = ffma2s(make_float2(pv[k].y, -pv[k].x), zr.y, y);
        } else {
          cmsub(y, zr, pv[k]);
        }
        yr[k] = y;
        ar2[k] = cnorm(y);
      }
    }
    static_for<0, NG>([&](auto gg) {
      constexpr int g = decltype(gg)::value;
      Real a[VP];
#pragma unroll
      for (int i = 0; i < VP; ++i) a[i] = Real(0);
      static_for<0, RG>([&](auto qq) {
        constexpr int q = decltype(qq)::value, P = g * RG + q;
        if constexpr (P < R) {
          const R2 zp = zof(P);
          if constexpr (std::is_same<Real, float>::value) {
            // packed FP32x2 (see sweep_kernel): numer = (Q1.x + Q2.y, Q1.y - Q2.x)
            float2 q1 = make_float2(0.f, 0.f), q2 = q1;
            float den = 0.f;
#pragma unroll
            for (int k = 0; k < FT; ++k) {
              const int jl = tid + k * NT;
              float2 y = Y.template get<P>(k, jl);
              y = ffma2s(pv[k], -zp.x, y);
              y = ffma2s(make_float2(pv[k].y, -pv[k].x), zp.y, y);
              Y.template set<P>(k, jl, y);
              const float w = weight(std::integral_constant<int, P>{}, k);
              const float2 sw = fmul2s(yr[k], w);
              q1 = ffma2s(y, sw.x, q1);
              q2 = ffma2s(y, sw.y, q2);
              den = fmaf(ar2[k], w, den);
            }
            a[q] = q1.x + q2.y;
            a[RG + q] = q1.y - q2.x;
            a[2 * RG + q] = den;
          } else {
#pragma unroll
            for (int k = 0; k < FT; ++k) {
              const int jl = tid + k * NT;
              R2 y = Y.template get<P>(k, jl);
              cmsub(y, zp, pv[k]);
              Y.template set<P>(k, jl, y);
              const Real w = weight(std::integral_constant<int, P>{}, k);
              a[q] = fma(fma(y.x, yr[k].x, y.y * yr[k].y), w, a[q]);
              a[RG + q] = fma(fma(y.y, yr[k].x, -y.x * yr[k].y), w, a[RG + q]);
              a[2 * RG + q] = fma(ar2[k], w, a[2 * RG + q]);
            }
          }
        }
      });
      warp_reduce_scatter_fast(a, lane);
      Real* rb = red + ((size_t)warp * NG + g) * VP;
#pragma unroll
      for (int i = 0; i < VM; ++i) rb[lane * VM + i] = a[i];
    });
#pragma unroll
    for (int k = 0; k < FT; ++k) pv[k] = yr[k];
    __syncthreads();
    if constexpr (AG) {
      // this CTA's partial of row `tid` -> every CTA of the cluster
      if (tid < R) {
        const int g = tid / RG, q = tid - g * RG;
        Real nre = Real(0), nim = Real(0), den = Real(0);
        for (int w = 0; w < NW; ++w) {
          const Real* rb = red + ((size_t)w * NG + g) * VP;
          nre += rb[q];
          nim += rb[RG + q];
          den += rb[2 * RG + q];
        }
        const uint32_t la = smem_u32addr(inA + ((size_t)(buf * CS + c) * R + tid) * CH);
#pragma unroll 1
        for (int dst = 0; dst < CS; ++dst)
          msg_send(dsmem_map(la, (uint32_t)dst), dsmem_map(barA[buf], (uint32_t)dst), nre, nim, den, Real(0));
      }
      mbar_wait_parity(barA[buf], (uint32_t)((r >> 1) & 1));
      if (tid == 0) mbar_arm(barA[buf], txA);  // step r + 2
      if (tid < R) {  // z of row `tid` from the CS partials in CTA order (identical in every CTA)
        Real nre = Real(0), nim = Real(0), den = Real(0);
        for (int q = 0; q < CS; ++q) {
          const Real* e = reinterpret_cast<const Real*>(inA + ((size_t)(buf * CS + q) * R + tid) * CH);
          nre += e[0];
          nim += e[1];
          den += e[2];
        }
        const bool bad = !(den > Real(0)) || !isfinite(den);  // estimator.cpp:451-454
        Real zx, zy = Real(0);
        if (tid == r) {
          zx = Real(1) - sqrt((Real)T / den);
        } else {
          zx = nre / den;
          zy = nim / den;
        }
        Real* zo = reinterpret_cast<Real*>(inZ + ((size_t)buf * R + tid) * CH);
        zo[0] = zx;
        zo[1] = zy;
        zo[2] = bad ? Real(1) : Real(0);
      }
      __syncthreads();
    } else {
      // this CTA's partial of row `tid` -> the row's owner
      if (tid < R) {
        const int g = tid / RG, q = tid - g * RG;
        Real nre = Real(0), nim = Real(0), den = Real(0);
        for (int w = 0; w < NW; ++w) {
          const Real* rb = red + ((size_t)w * NG + g) * VP;
          nre += rb[q];
          nim += rb[RG + q];
          den += rb[2 * RG + q];
        }
        const int owner = tid % CS, lr = tid / CS;
        const uint32_t la = smem_u32addr(inA + ((size_t)(buf * CS + c) * RC + lr) * CH);
        msg_send(dsmem_map(la, (uint32_t)owner), dsmem_map(barA[buf], (uint32_t)owner), nre, nim, den, Real(0));
      }
      // owners: z of the own rows from the CS partials (CTA order), to every CTA
      if (tid < nown * CS) {
        const int lr = tid / CS, dest = tid - lr * CS, row = c + lr * CS;
        mbar_wait_parity(barA[buf], (uint32_t)((r >> 1) & 1));
        Real nre = Real(0), nim = Real(0), den = Real(0);
        for (int q = 0; q < CS; ++q) {
          const Real* e = reinterpret_cast<const Real*>(inA + ((size_t)(buf * CS + q) * RC + lr) * CH);
          nre += e[0];
          nim += e[1];
          den += e[2];
        }
        const bool bad = !(den > Real(0)) || !isfinite(den);  // estimator.cpp:451-454
        Real zx, zy = Real(0);
        if (row == r) {
          zx = Real(1) - sqrt((Real)T / den);
        } else {
          zx = nre / den;
          zy = nim / den;
        }
        const uint32_t la = smem_u32addr(inZ + ((size_t)buf * R + row) * CH);
        msg_send(dsmem_map(la, (uint32_t)dest), dsmem_map(barZ[buf], (uint32_t)dest), zx, zy, bad ? Real(1) : Real(0),
                 Real(0));
        if (tid == 0) mbar_arm(barA[buf], txA);  // step r + 2
      }
      mbar_wait_parity(barZ[buf], (uint32_t)((r >> 1) & 1));
      if (tid == 0) mbar_arm(barZ[buf], txZ);  // step r + 2
    }
    const unsigned char* zcur = inZ + (size_t)buf * R * CH;
    {
      const bool b1 = lane < R && reinterpret_cast<const Real*>(zcur + (size_t)lane * CH)[2] != Real(0);
      const bool b2 = lane + 32 < R && reinterpret_cast<const Real*>(zcur + (size_t)(lane + 32) * CH)[2] != Real(0);
      const unsigned m1 = __ballot_sync(kFull, b1), m2 = __ballot_sync(kFull, b2);
      if (m1 | m2) {
        badrow = m1 ? __ffs(m1) - 1 : 32 + __ffs(m2) - 1;
        badstep = r;
        break;
      }
    }
    const Real zr_real = reinterpret_cast<const Real*>(zcur + (size_t)r * CH)[0];
    dprod *= (double)(Real(1) - zr_real);
    // iss_apply on the own W columns, W -= z w_r (estimator.cpp:298-302), ping-pong
    const R2* Wo = Wsl + (size_t)(r & 1) * R * DC;
    R2* Wn = Wsl + (size_t)((r + 1) & 1) * R * DC;
    for (int e = tid; e < R * DC; e += NT) {
      const int q = e % R, i = e / R;
      R2 w = Wo[e];
      cmsub(w, *reinterpret_cast<const R2*>(zcur + (size_t)q * CH), Wo[i * R + r]);
      Wn[e] = w;
    }
  }
  if (badrow >= 0) {
    if (c == 0 && tid == 0) record_err<Real>(p.err, mix, err_key(p.iteration, kPhSweep, gbin, badstep, badrow));
    cluster_sync_all();
    return;
  }

  CTF_FPHASE(5);
  // ---- epilogue: last step's update, row-power partials, |y|^2 of the first
  // HL frames for the previous CTA's delayed energies
  {
    const unsigned char* zl = inZ + (PAIR ? (size_t)(((R - 2) >> 1) & 1) * R * LY::CHZ : (size_t)((R - 1) & 1) * R * CH);
    static_for<0, LY::NG2>([&](auto gg) {
      constexpr int g = decltype(gg)::value;
      Real a[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) a[i] = Real(0);
      static_for<0, 32>([&](auto qq) {
        constexpr int q = decltype(qq)::value, P = g * 32 + q;
        if constexpr (P < R) {
          const R2 zp = *reinterpret_cast<const R2*>(zl + (size_t)P * LY::CHZ);
#pragma unroll
          for (int k = 0; k < FT; ++k) {
            const int jl = tid + k * NT;
            R2 y = Y.template get<P>(k, jl);
            if constexpr (PAIR) {
              const R2 zb = *reinterpret_cast<const R2*>(zl + (size_t)P * LY::CHZ + 2 * sizeof(Real));
              y = ffma2s(pv[k], -zp.x, y);
              y = ffma2s(make_float2(pv[k].y, -pv[k].x), zp.y, y);
              y = ffma2s(pc[k], -zb.x, y);
              y = ffma2s(make_float2(pc[k].y, -pc[k].x), zb.y, y);
            } else if constexpr (std::is_same<Real, float>::value) {
              y = ffma2s(pv[k], -zp.x, y);
              y = ffma2s(make_float2(pv[k].y, -pv[k].x), zp.y, y);
            } else {
              cmsub(y, zp, pv[k]);
            }
            Y.template set<P>(k, jl, y);
            const Real q2 = cnorm(y);
            a[q] += q2;
            if (jl < HL) halo[P * HL + jl] = q2;
          }
        }
      });
      warp_reduce_scatter(a, lane);
      red[((size_t)warp * LY::NG2 + g) * 32 + lane] = a[0];
    });
  }
  __syncthreads();
  if (tid < R) {
    const int g = tid / 32, q = tid - g * 32;
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += (double)red[((size_t)w * LY::NG2 + g) * 32 + q];
    ex[4 + tid] = s;
  }
  cluster_sync_all();  // halos and row-power partials published
  CTF_FPHASE(6);

  // delayed energies E_n(tau) = sum_{l<L, tau+l<T} |y_{nL+l}(tau+l)|^2 (estimator.cpp:321-332)
  Real eown[N][FT];
  Real* Eg = reinterpret_cast<Real*>(p.E);
  static_for<0, N>([&](auto nn) {
    constexpr int n = decltype(nn)::value;
    __syncthreads();  // previous source's Pn reads done (Pn aliases the dead x tile)
    static_for<0, L>([&](auto ll) {
      constexpr int l = decltype(ll)::value, P = n * L + l;
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        const int jl = tid + k * NT;
        Pn[l * (TC + HL) + jl] = cnorm(Y.template get<P>(k, jl));
      }
    });
    for (int i = tid; i < L * HL; i += NT) {
      const int l = i / HL, h = i - l * HL;
      Real v = Real(0);
      if (c + 1 < CS) v = dsmem_ld(dsmem_map(smem_u32addr(halo + (n * L + l) * HL + h), (uint32_t)(c + 1)), Real(0));
      Pn[l * (TC + HL) + TC + h] = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < FT; ++k) {
      const int jl = tid + k * NT, tau = j0 + jl;
      Real e = Real(0);
      for (int l = 0; l < L && tau + l < T; ++l) e += Pn[l * (TC + HL) + jl + l];
      eown[n][k] = e;
      if (tau < T) Eg[(((size_t)mix * N + n) * p.FL + bin) * T + tau] = e;
    }
  });

  // MU-B partials (estimator.cpp:313-346) over the own frames, 16 bases per pass
  // (CTF_FS_MUBOUT: left to mub_kernel, which runs after this kernel on E and
  // 1/lambda from HBM; this kernel then writes back the rescaled B)
  if constexpr (!MUBOUT)
  for (int n = 0; n < N; ++n) {
    const int k0 = p.koff[n], k1 = p.koff[n + 1];
    const Real* il = invl + n * LP + LOFF;
    Real en[FT];
#pragma unroll
    for (int k = 0; k < FT; ++k) en[k] = eown[0][k];
    static_for<1, N>([&](auto nn) {
      constexpr int q = decltype(nn)::value;
      if (n == q)
#pragma unroll
        for (int k = 0; k < FT; ++k) en[k] = eown[q][k];
    });
    // KW bases per pass: 10 when K is a multiple of 10 (BASELINE K = 20: no
    // idle lanes), else 16; numerators at [0, KW), denominators at [16, 16 + KW)
    auto mub = [&](auto kw) {
      constexpr int KW = decltype(kw)::value;
      for (int kb = k0; kb < k1; kb += KW) {
        Real a[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) a[i] = Real(0);
#pragma unroll
        for (int k = 0; k < FT; ++k) {
          const int jl = tid + k * NT, tau = j0 + jl;
          const Real ilv = il[jl];
          const Real an = en[k] * (ilv * ilv);
          const Real bn = (tau < T) ? ilv * (Real)min(L, T - tau) : Real(0);
          if (tau < T) {
#pragma unroll
            for (int q = 0; q < KW; ++q) {
              const Real v = __ldg(Vg + (size_t)min(kb + q, k1 - 1) * T + tau);
              a[q] = fma(an, v, a[q]);
              a[16 + q] = fma(bn, v, a[16 + q]);
            }
          }
        }
        warp_reduce_scatter(a, lane);
        __syncthreads();  // previous pass's reads of red are done
        red[(size_t)warp * 32 + lane] = a[0];
        __syncthreads();
        if (tid < KW && kb + tid < k1) {
          Real num = Real(0), den = Real(0);
          for (int w = 0; w < NW; ++w) {
            num += red[(size_t)w * 32 + tid];
            den += red[(size_t)w * 32 + 16 + tid];
          }
          exmub[2 * (kb + tid)] = (double)num;
          exmub[2 * (kb + tid) + 1] = (double)den;
        }
      }
    };
    if ((k1 - k0) % 10 == 0)
      mub(std::integral_constant<int, 10>{});
    else
      mub(std::integral_constant<int, 16>{});
  }
  cluster_sync_all();  // MU-B partials published
  CTF_FPHASE(7);

  if (c == 0) {
    for (int k = tid; k < SK; k += NT) {
      double num = 0.0, den = 0.0;
      for (int q = 0; q < CS; ++q) {
        num += dsmem_ld_f64(dsmem_map(smem_u32addr(exmub + 2 * k), (uint32_t)q));
        den += dsmem_ld_f64(dsmem_map(smem_u32addr(exmub + 2 * k + 1), (uint32_t)q));
      }
      if constexpr (MUBOUT) Bg[k] = Bs[k];
      else Bg[k] = fmax(Bs[k] * (Real)sqrt(num / den), floor_abs);
    }
    for (int row = tid; row < R; row += NT) {
      double s = 0.0;
      for (int q = 0; q < CS; ++q) s += dsmem_ld_f64(dsmem_map(smem_u32addr(ex + 4 + row), (uint32_t)q));
      p.rowpow[tile * R + row] = s;
    }
    if (tid == 0) p.logdet[tile] = logdet + log(dprod);
  }
  const R2* Wf = Wsl + (size_t)((PAIR ? R / 2 : R) & 1) * R * DC;
  for (int e = tid; e < R * DC; e += NT) {
    const int q = e % R, i = e / R, col = c * DC + i;
    if (col < R) Wg[(size_t)col * R + q] = Wf[e];
  }
  cluster_sync_all();  // CTA 0's remote reads done before any CTA exits
  CTF_FPHASE(8);
}

}  // namespace ctf
