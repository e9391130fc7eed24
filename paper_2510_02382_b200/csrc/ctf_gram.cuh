// ctf_gram.cuh — covariance-domain ISS iteration kernel (fp32 and fp64,
// stacked equal-tap configs).
//
// The reference ships two equivalent forms of the ISS step: the
// estimate-domain sums over frames (estimator.cpp:434-484, what run() uses)
// and the covariance-domain form z from w_p^H Q_p w_r (estimator.cpp:89-101,
// 275-302), which its own tests hold equal to 1e-10
// (test_estimator.cpp:360-392). The frame-domain sweep costs ~20 R^2 flops per
// TF-bin; here the weighted covariances are formed once per iteration and the
// R steps run on R x D matrices:
//
//   C_p[(m,l'),(m',l'')] = sum_{j=l}^{T-1} x_m(j-l') conj(x_m'(j-l'')) / lambda_n(j-l)
//
// for row p = (n, l). With s = j - l, a = l - l', b = l - l'' every entry is
// G_n(m,a; m',b) = sum_s x_m(s+a) conj(x_m'(s+b)) w_n(s), shared by all rows
// of source n; with u = s + a and d = b - a it is the correlation
// sum_u Q_{m,m',d}(u) w_n(u - a) of one product sequence Q = x_m conj(x_m'(.+d))
// with the weights at 2L-1-|d| lags: about N*M^2*(2L-1)^2/2 packed FMAs per
// TF-bin (Hermitian half) and no R x T tile. The upper limit j <= T-1 of row l
// is restored exactly by subtracting the l "virtual" frames j in [T, T+l)
// (whose x~ uses only real samples), carried through the steps as an
// R x (L-1) tail of Y.
//
// Per (mixture, bin) CTA: prologue (x tile, rescale, lambda) as the sweep
// kernel -> Gram (threads own (m, m', d, frame chunk) tasks; products and
// weights blocked in registers) -> fixed-order reduction -> objective of the
// previous iteration (w_r^H C_r w_r of the rescaled W) -> R covariance-domain
// steps (W and the tail updated by the reference's rank-1 rule) -> one demix
// Y = W' x~ for the delayed energies, row powers and MU-B.
#pragma once
#include "ctf_kernels.cuh"
#include "ctf_tc.cuh"

#ifndef CTF_LAMV
#define CTF_LAMV 20
#endif
#ifndef CTF_GRAM_RCPNR  // fp64 chained steps: Newton reciprocal (~1 ulp, 5 dependent operations) for z = num / den
#define CTF_GRAM_RCPNR 1
#endif
#ifndef CTF_GRAM_RCPNR32  // the same in fp32: MUFU + one Newton step instead of __frcp_rn
#define CTF_GRAM_RCPNR32 1
#endif
#ifndef CTF_GRAM_SPIN  // 1: poll the pivot's mbarrier (test_wait) instead of the suspending try_wait
#define CTF_GRAM_SPIN 0
#endif
#ifndef CTF_GRAM_CHAIN  // 1: mbarrier-chained ISS steps on the narrow tiles (0: one CTA barrier per step)
#define CTF_GRAM_CHAIN 1
#endif
// Where 1 / lambda comes from: 1 = always from lambda_kernel (run by the host
// ahead of the iteration kernel, which then has no lambda phase of its own),
// 0 = always the kernel's own lambda phase, 2 (default) = per variant by
// gram_lpre() below (measured on B200, tools/lam_ab.sh)
#ifndef CTF_GRAM_LPRE
#define CTF_GRAM_LPRE 2
#endif
#ifndef CTF_LAMV3  // the same for the 3-CTA/SM (80-register) cfg1 variant
#define CTF_LAMV3 10
#endif
namespace ctf {

// Gram task table (host-built, global memory), int4 entries:
//   [0, NT)            per thread {group, u0, u1, 0}  (group -1: idle)
//   [NT]               {ngroups, 0, 0, 0}
//   [NT + 1 + 2g]      {m, m2, d, a_lo}
//   [NT + 2 + 2g]      {cnt, t0, t1, 0}   (threads [t0, t1) hold the chunks, in order)
constexpr int kGramUB = 4;  // frames per register block
#ifdef CTF_PHASE_TIMING
__device__ unsigned long long g_phase[4096 * 12];  // dev instrumentation: clock64 per phase, tid 0
#endif

// acc[n][j] += sum_{u in [u0, u1)} x1(u) conj(x2(u)) w_n(u - a_lo - j); w0
// points at w_n(-a_lo). The weight window w_n(u - a_lo - (CNT-1) .. u + UB - 1
// - a_lo) lives in registers and slides by UB per block (UB new loads per
// source instead of UB + CNT - 1). Chunks have odd lengths (host), so the
// threads of a warp start on distinct banks and stay there.
// ---- precision-specific complex kernels (fp32: packed FFMA2 forms)
template <typename Real> struct GOps;
template <> struct GOps<float> {
  using R2 = float2;
  // a conj(b) = (a.x, a.y) b.x + (a.y, -a.x) b.y
  static __device__ __forceinline__ R2 mulc(R2 a, R2 b) { return ffma2s(make_float2(a.y, -a.x), b.y, fmul2s(a, b.x)); }
  static __device__ __forceinline__ R2 fmar(R2 q, float w, R2 acc) { return ffma2s(q, w, acc); }  // acc + q w
  // acc + c conj(w)
  static __device__ __forceinline__ R2 macc(R2 c, R2 w, R2 acc) {
    return ffma2s(make_float2(c.y, -c.x), w.y, ffma2s(c, w.x, acc));
  }
  // acc + w x (complex)
  static __device__ __forceinline__ R2 mac(R2 w, R2 x, R2 acc) {
    return ffma2s(make_float2(-x.y, x.x), w.y, ffma2s(x, w.x, acc));
  }
};
template <> struct GOps<double> {
  using R2 = double2;
  static __device__ __forceinline__ R2 mulc(R2 a, R2 b) {
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
  }
  static __device__ __forceinline__ R2 fmar(R2 q, double w, R2 acc) {
    return make_double2(fma(q.x, w, acc.x), fma(q.y, w, acc.y));
  }
  static __device__ __forceinline__ R2 macc(R2 c, R2 w, R2 acc) {
    return make_double2(fma(c.x, w.x, fma(c.y, w.y, acc.x)), fma(c.y, w.x, fma(-c.x, w.y, acc.y)));
  }
  static __device__ __forceinline__ R2 mac(R2 w, R2 x, R2 acc) {
    return make_double2(fma(w.x, x.x, fma(-w.y, x.y, acc.x)), fma(w.x, x.y, fma(w.y, x.x, acc.y)));
  }
};

template <typename Real, int CNT, int NS, int UB, bool MASK>
__device__ __forceinline__ void gram_step(const typename Cplx<Real>::T* __restrict__ x1,
                                          const typename Cplx<Real>::T* __restrict__ x2,
                                          const Real* __restrict__ w0, int lp, int u, int u1,
                                          Real (&wv)[NS][UB + CNT - 1], typename Cplx<Real>::T (&acc)[NS][CNT]) {
  using R2 = typename Cplx<Real>::T;
  R2 q[UB];
#pragma unroll
  for (int i = 0; i < UB; ++i) {
    q[i] = GOps<Real>::mulc(x1[u + i], x2[u + i]);
    if (MASK && u + i >= u1) q[i].x = q[i].y = Real(0);
  }
#pragma unroll
  for (int n = 0; n < NS; ++n) {
#pragma unroll
    for (int k = 0; k < CNT - 1; ++k) wv[n][k] = wv[n][k + UB];
#pragma unroll
    for (int i = 0; i < UB; ++i) wv[n][CNT - 1 + i] = w0[n * lp + u + i];
#pragma unroll
    for (int i = 0; i < UB; ++i)
#pragma unroll
      for (int j = 0; j < CNT; ++j) acc[n][j] = GOps<Real>::fmar(q[i], wv[n][CNT - 1 + i - j], acc[n][j]);
  }
}

// acc[n][j] += sum_{u in [u0, u1)} x1(u) conj(x2(u)) w_n(u - a_lo - j) for NS
// sources from w0 (w0 points at w_(n0)(-a_lo)). The weight window
// w_n(u - a_lo - (CNT-1) .. u + UB - 1 - a_lo) lives in registers and slides by
// UB per block (UB new loads per source instead of UB + CNT - 1). Chunks have
// odd lengths (host), so the threads of a warp start on distinct banks and
// stay there; only the last block of a chunk is masked.
template <typename Real, int CNT, int NS, int UB>
__device__ __forceinline__ void gram_block(const typename Cplx<Real>::T* __restrict__ x1,
                                           const typename Cplx<Real>::T* __restrict__ x2,
                                           const Real* __restrict__ w0, int lp, int u0, int u1,
                                           typename Cplx<Real>::T (&acc)[NS][CNT]) {
  Real wv[NS][UB + CNT - 1];
#pragma unroll
  for (int n = 0; n < NS; ++n)
#pragma unroll
    for (int k = 0; k < CNT - 1; ++k) wv[n][k + UB] = w0[n * lp + u0 - (CNT - 1) + k];
  int u = u0;
  for (; u + UB <= u1; u += UB) gram_step<Real, CNT, NS, UB, false>(x1, x2, w0, lp, u, u1, wv, acc);
  if (u < u1) gram_step<Real, CNT, NS, UB, true>(x1, x2, w0, lp, u, u1, wv, acc);
}

// (log_fast, the objective's log term, and rcp_rn: ctf_kernels.cuh)
// Sources accumulated per Gram pass: all of them in fp32 (the conj products
// are shared); one at a time in fp64 (register budget, half the partials).
#ifndef CTF_GRAM_NS64
#define CTF_GRAM_NS64 1
#endif
template <typename Real, int N, int R> constexpr int gram_ns() {
  return (std::is_same<Real, float>::value && R <= 16) ? N : (R <= 16 && N % CTF_GRAM_NS64 == 0 ? CTF_GRAM_NS64 : 1);
}
// Sources accumulated per Gram pass over the frames (NSG >= gram_ns, a
// multiple of it): fp64 two-source shapes share each conj product between
// both sources (the second source's partials wait in registers while the
// first's are reduced: the partial buffer holds gram_ns sources).
#ifndef CTF_GRAM_NSG64
#define CTF_GRAM_NSG64 2
#endif
template <typename Real, int N, int R> constexpr int gram_nsg() {
  return (!std::is_same<Real, float>::value && R <= 16 && N == CTF_GRAM_NSG64) ? N : gram_ns<Real, N, R>();
}
#ifndef CTF_GRAM_UB2  // frames per register block when two fp64 sources share the products
#define CTF_GRAM_UB2 1
#endif
#ifndef CTF_GRAM_SPLITWIDE
#define CTF_GRAM_SPLITWIDE 1
#endif
#ifndef CTF_GRAM_RCP64
#define CTF_GRAM_RCP64 1
#endif
#ifndef CTF_GRAM_MINB64
#define CTF_GRAM_MINB64 2
#endif
#ifndef CTF_GRAM_MINB32  // fp32 short-frame variants at <= 256 threads: CTAs per SM (80 registers at 3)
#define CTF_GRAM_MINB32 3
#endif
// fp32 long-frame variants (FT >= 8, BASELINE cfg2 T = 2000) at 256 threads:
// two CTAs per SM (EREG energies + one-source partial buffer keep them under
// half the shared memory)
template <typename Real> constexpr bool gram_ereg(int FT) { return std::is_same<Real, float>::value && FT >= 8; }
template <typename Real, int NT, int R, int FT = 4> constexpr int gram_min_blocks() {
  return R > 16 ? 1
         : std::is_same<Real, float>::value ? (NT <= 256 ? (FT >= 8 ? 2 : CTF_GRAM_MINB32) : 1)
                                            : (NT <= 256 ? CTF_GRAM_MINB64 : NT <= 384 ? 2 : 1);
}

// lambda ahead of the kernel pays where the kernel's own lambda phase (K
// dependent V loads per frame, a reciprocal and a log per element) is poorly
// hidden: fp64 and the variants below three CTAs per SM. At three CTAs per SM
// (cfg1 fp32) the phase hides behind the other CTAs and the extra kernel with
// its 1 / lambda round trip through HBM costs more than it saves.
template <typename Real, int NT, int R, int FT> constexpr bool gram_lpre() {
  return CTF_GRAM_LPRE == 1   ? true
         : CTF_GRAM_LPRE == 0 ? false
                              : (!std::is_same<Real, float>::value || gram_min_blocks<Real, NT, R, FT>() < 3);
}

// Tensor-core Gram (TC = true, fp32): the lag correlations as one real GEMM
// per bin on tcgen05 (kind::tf32, 3xTF32 split for fp32 accuracy),
//   C[(g, re|im)][(n, a)] = sum_u P_g(u) w_n(u - a),  P_g = x_m conj(x_m'(. + d)),
// rows = the NG (m, m', d) groups' real and imaginary parts (A, K-major:
// frames contiguous), columns = source x lag a in [-(L-1), L-1] (B, K-major),
// K = the frames. Products and weights are formed by all threads into a
// double-buffered shared-memory stage of KC frames (hi and lo tf32 parts);
// one thread issues the 3 x (re, im) MMAs of a stage into TMEM and commits
// them to the stage's mbarrier, which the producers wait on before refilling
// it. The accumulators are read back with tcgen05.ld into the same Gram
// table the CUDA-core path builds, so the steps are unchanged.
template <int M, int L> struct GramTC {
  static constexpr int NA = 2 * L - 1;
  static constexpr int NG = M * L + (M * (M - 1) / 2) * NA;  // (m <= m', d) groups
  static constexpr int TILES = (NG + 127) / 128;              // 128-row MMA tiles per re / im part
  static constexpr int NC = M * NA;                           // columns (sources = mics)
  static constexpr int NP = (NC + 15) / 16 * 16;              // MMA N
  static constexpr int KC = 16;                               // frames per stage
  static constexpr int KS = KC / 8;                           // K-steps per stage
  static constexpr int ASTEP = 2 * TILES * 128 * 32;          // bytes of one A K-step (re and im rows)
  static constexpr int BSTEP = NP * 32;
  static constexpr int STAGE = 2 * KS * ASTEP + 2 * KS * BSTEP;  // hi + lo
  // [2 sets (chunk parity)] x [2 terms] x [2 TILES tiles (re, im)] x NP columns
  static constexpr int TCOLS = 8 * TILES * NP <= 128 ? 128 : 8 * TILES * NP <= 256 ? 256 : 512;
  static constexpr size_t bytes() { return (size_t)2 * STAGE; }
};

// IP: the iterative-projection rule in place of the ISS steps.
template <typename Real, int M, int L, int NT, int FT, bool IP = false, bool TC = false>
__global__ void __launch_bounds__(NT, gram_min_blocks<Real, NT, M * L, FT>())
    gram_kernel(const SweepParams p, const int4* __restrict__ gtab) {
  using R2 = typename Cplx<Real>::T;
  using Ops = GOps<Real>;
  constexpr bool F32 = std::is_same<Real, float>::value;
  constexpr int N = M, R = M * L, D = M * L, NA = 2 * L - 1, NW = NT / 32;
  constexpr int NS = gram_ns<Real, N, R>();
  constexpr bool EREG = gram_ereg<Real>(FT);  // E_n in registers (no |y|^2 rows in shared memory)
  constexpr int LT1 = L > 1 ? L - 1 : 1;
  constexpr int CPB = 16 / (int)sizeof(R2);  // complex values per 16-byte load
  // V columns of the lambda phase loaded at once (fp32, one CTA per SM)
  constexpr int LAMV = !F32                                         ? 0
                       : gram_min_blocks<Real, NT, M * L, FT>() == 1 ? CTF_LAMV
                       : (M == 2 && L == 5)                       ? CTF_LAMV3  // measured (cfg1); others spill
                                                                  : 0;
  static_assert(D <= 32, "one lane per stacked channel in the covariance steps");
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bin = blockIdx.x, mix = blockIdx.y;
  const int gbin = p.bin_lo + bin;
  const int T = p.T, TP = p.TP, SK = p.SK;

  R2* xs = reinterpret_cast<R2*>(smem + p.off_x);      // M rows of xp: x_m(t) at [m*xp + xoff + t]
  Real* invl = reinterpret_cast<Real*>(smem + p.off_l);  // N rows of lp: w_n(s) at [n*lp + loff + s]
  R2* G = reinterpret_cast<R2*>(smem + p.off_y);       // [n][m][m'][a][b]
  R2* part = reinterpret_cast<R2*>(smem + p.off_e);    // [n*NA + j][NT + 1] Gram partials (NS sources)
  Real* Pq = reinterpret_cast<Real*>(smem + p.off_e);  // [l][TP] |y|^2 of one source; row 0 then E_n (!EREG)
  R2* Wb = reinterpret_cast<R2*>(smem + p.off_w);      // R x D (column-major)
  R2* Yt = reinterpret_cast<R2*>(smem + p.off_z);      // R x LT1 tail frames
  R2* zs = Yt + 2 * R * LT1;                           // 2 x (D + LT1) pivot buffers
  Real* red = reinterpret_cast<Real*>(smem + p.off_red);  // 32 * NW
  Real* Bs = reinterpret_cast<Real*>(smem + p.off_b);
  double* dred = reinterpret_cast<double*>(smem + p.off_d);
  __shared__ int s_bad, s_badrow, s_fb;
  __shared__ double s_logmu;
  __shared__ Real fac_s[R];  // (1 - z_r) of the ISS steps (determinant lemma)
  constexpr int kNoRow = 1 << 30;

  const size_t tile = (size_t)mix * p.FL + bin;
#ifdef CTF_PHASE_TIMING
#define CTF_PHASE(k) \
  if (tid == 0 && tile < 4096) g_phase[tile * 12 + (k)] = clock64();
#else
#define CTF_PHASE(k)
#endif
  CTF_PHASE(0);
  prefetch_next_tile(p, bin, mix, (size_t)T * M * sizeof(R2), (size_t)R * D * sizeof(R2));
  const R2* xg = reinterpret_cast<const R2*>(p.x) + tile * (size_t)T * M;
  R2* Wg = reinterpret_cast<R2*>(p.W) + tile * (size_t)R * D;
  Real* Bg = reinterpret_cast<Real*>(p.Bf) + tile * SK;
  const Real* Vg = reinterpret_cast<const Real*>(p.V) + (size_t)mix * SK * T;
  const Real floor_abs = (Real)p.floor_abs[mix];
  const int prev_it = p.iteration - 1;
  const double* mu = p.mu ? p.mu + (size_t)mix * R : nullptr;
  // Gram table: Hermitian half, mic pairs m <= m2 packed (NP of them):
  // G[n][pair(m, m2)][a][b], a, b in [-(L-1), L-1]; G(m > m2) = conj(G(m2, m, b, a))
  constexpr int NP = M * (M + 1) / 2;
  auto gidx = [](int n, int m, int m2, int a, int b) {  // requires m <= m2
    const int pm = m * M - (m * (m - 1)) / 2 + (m2 - m);
    return ((n * NP + pm) * NA + a + L - 1) * NA + b + L - 1;
  };
  auto gget = [&](int n, int m, int m2, int a, int b) -> R2 {
    if (m <= m2) return G[gidx(n, m, m2, a, b)];
    R2 v = G[gidx(n, m2, m, b, a)];
    v.y = -v.y;
    return v;
  };

  if (tid == 0) {
    s_bad = 0;
    s_fb = 0;
    s_badrow = kNoRow;
    s_logmu = mu ? p.logmu[mix] : 0.0;
  }
  // W and B of the tile: loads issued before the x tile's (their latency
  // overlaps; stored to shared memory below)
  const bool wb1 = R * D <= NT && SK <= NT;
  R2 wpre;
  Real bpre = Real(0);
  wpre.x = wpre.y = Real(0);
  double mw = 0.0, mb = 0.0;  // pending rescale factors of this thread's W and B entries
  if (wb1) {
    if (tid < R * D) {
      wpre = Wg[tid];
      if (mu) mw = mu[tid % R];
    }
    if (tid < SK) {
      bpre = Bg[tid];
      int nb = 0;
#pragma unroll
      for (int n = 1; n < N; ++n) nb += tid >= p.koff[n] ? 1 : 0;
      if (mu) mb = mu[p.row0[nb]];
    }
  }
  const bool lam4 = (T % 4 == 0 && 4 * NT >= T);
  // lambda phase done ahead by lambda_kernel (uniform over the launch)
  constexpr int LVEC = 16 / (int)sizeof(Real);
  constexpr int LV = (N * FT + LVEC - 1) / LVEC;  // >= (N*T/LVEC) / NT since T <= FT*NT
  constexpr bool lpre = gram_lpre<Real, NT, M * L, FT>();
  if (lpre && tid == 0 && p.pf_stride > 0) {
    const size_t w = tile + p.pf_stride;
    if (w < (size_t)p.nmix * p.FL)
      prefetch_l2(reinterpret_cast<const Real*>(p.invl_g) + w * (size_t)N * T, (unsigned)((size_t)N * T * sizeof(Real)));
  }
  // 1 / lambda of the bin from lambda_kernel (one contiguous [N][T] block):
  // 16-byte loads in flight together with the x tile's
  const Real* lgs = reinterpret_cast<const Real*>(p.invl_g) + tile * (size_t)N * T;
  const bool lvec = lpre && T % LVEC == 0;
  float4 lv[LV];
  const int nl16 = N * T / LVEC;
  if (lvec) {
    const float4* lg = reinterpret_cast<const float4*>(lgs);
#pragma unroll
    for (int i = 0; i < LV; ++i) {
      const int e = tid + i * NT;
      if (e < nl16) lv[i] = __ldg(lg + e);
    }
  }
  // ---- prologue: zero-padded x tile, W and B with the pending rescale
  if ((T * M) % CPB == 0) {
    // the bin's T x M complex block is contiguous: 16-byte loads, all in
    // flight before the first store (latency, not bandwidth, bounds this)
    constexpr int XV = (FT * M + CPB - 1) / CPB;  // >= (T*M/CPB) / NT since T <= FT*NT
    const int n16 = T * M / CPB;
    const float4* xv = reinterpret_cast<const float4*>(xg);
    float4 v[XV];
#pragma unroll
    for (int i = 0; i < XV; ++i) {
      const int e = tid + i * NT;
      if (e < n16) v[i] = __ldg(xv + e);
    }
    for (int i = tid; i < M * p.xp; i += NT) {
      const int t = i % p.xp - p.xoff;
      if (t < 0 || t >= T) xs[i].x = xs[i].y = Real(0);
    }
#pragma unroll
    for (int i = 0; i < XV; ++i) {
      const int e = tid + i * NT;
      if (e < n16) {
        const R2* c = reinterpret_cast<const R2*>(&v[i]);
#pragma unroll
        for (int h = 0; h < CPB; ++h) {
          const int f = CPB * e + h;
          xs[(f % M) * p.xp + p.xoff + f / M] = c[h];
        }
      }
    }
  } else {
    for (int i = tid; i < M * p.xp; i += NT) {
      const int m = i / p.xp, t = i - m * p.xp - p.xoff;
      R2 z;
      z.x = z.y = Real(0);
      xs[i] = (t >= 0 && t < T) ? xg[(size_t)t * M + m] : z;
    }
  }
  if (lvec) {
    for (int i = tid; i < N * p.lp; i += NT) {
      const int s = i % p.lp - p.loff;
      if (s < 0 || s >= T) invl[i] = Real(0);
    }
#pragma unroll
    for (int i = 0; i < LV; ++i) {
      const int e = tid + i * NT;
      if (e < nl16) {
        const int f = LVEC * e, n = f / T, t = f - n * T;
        const Real* c = reinterpret_cast<const Real*>(&lv[i]);
#pragma unroll
        for (int h = 0; h < LVEC; ++h) invl[n * p.lp + p.loff + t + h] = c[h];
      }
    }
  } else if (lpre) {
    for (int i = tid; i < N * p.lp; i += NT) {
      const int n = i / p.lp, s = i - n * p.lp - p.loff;
      invl[i] = (s >= 0 && s < T) ? __ldg(lgs + (size_t)n * T + s) : Real(0);
    }
  }
  // pending rescale (estimator.cpp:399-411): W rows / mu_r, B_n / mu_row0^2
  // floored; fp64 divides exactly like the reference, fp32 multiplies by
  // the rounded reciprocal
  if (wb1) {  // one W and one B entry per thread: rescaled in registers
    if (tid < R * D) {
      R2 w = wpre;
      if (mu && mw != 0.0) {
        if constexpr (F32) {
          const float im = (float)(1.0 / mw);
          w.x *= im;
          w.y *= im;
        } else {
          w.x /= mw;
          w.y /= mw;
        }
      }
      Wb[tid] = w;
      if (p.has_prev && !cfinite(w)) s_bad = 1;
    }
    if (tid < SK) {
      Real b = bpre;
      if (mu && mb != 0.0) {  // estimator.cpp:405-406: silent row, no rescale
        if constexpr (F32) {
          const float im = (float)(1.0 / mb);
          b = fmaxf(b * (im * im), floor_abs);
        } else {
          b = fmax(b / (mb * mb), (double)floor_abs);
        }
      }
      Bs[tid] = b;
    }
  } else {
    for (int i = tid; i < R * D; i += NT) Wb[i] = Wg[i];
    for (int i = tid; i < SK; i += NT) Bs[i] = Bg[i];
  }
  __shared__ Real s_imu[R];  // fp32: 1 / mu_r of the pending rescale (1 where none)
  if (!wb1) {
  if (F32 && warp == 0 && lane < R) s_imu[lane] = (mu && mu[lane] != 0.0) ? (Real)(1.0 / mu[lane]) : Real(1);
  __syncthreads();
  for (int i = tid; i < R * D; i += NT) {
    R2 w = Wb[i];
    if (mu) {
      const double m = mu[i % R];
      if (m != 0.0) {
        if constexpr (F32) {
          w.x *= s_imu[i % R];
          w.y *= s_imu[i % R];
        } else {
          w.x /= m;
          w.y /= m;
        }
      }
    }
    Wb[i] = w;
    if (p.has_prev && !cfinite(w)) s_bad = 1;
  }
  if (mu)
    for (int n = 0; n < N; ++n) {
      const double m0 = mu[p.row0[n]];
      if (m0 == 0.0) continue;  // estimator.cpp:405-406: silent row, no rescale
      for (int i = p.koff[n] + tid; i < p.koff[n + 1]; i += NT) {
        if constexpr (F32) {
          const float im = s_imu[p.row0[n]];
          Bs[i] = fmaxf(Bs[i] * (im * im), floor_abs);
        } else {
          Bs[i] = fmax(Bs[i] / (m0 * m0), (double)floor_abs);
        }
      }
    }
  }
  __syncthreads();
  CTF_PHASE(1);
  if (p.has_prev && s_bad) {  // check_all_finite on W (estimator.cpp:494-496)
    if (tid == 0) record_err<Real>(p.err, mix, err_key(prev_it, kPhFinite, gbin, 0, 1));
    return;
  }
  // ---- lambda = max(B V, floor) -> 1/lambda (zero outside [0, T)), log term
  double logsum = 0.0;
  const int t4 = tid * 4;
  if (lpre) {
    if (tid == 0 && p.has_prev) logsum = p.logsum_g[tile];
  } else {
  for (int n = 0; n < N; ++n) {
    Real* il = invl + n * p.lp;
    for (int i = tid; i < p.lp; i += NT) {
      const int s = i - p.loff;
      if (s < 0 || s >= T) il[i] = Real(0);
    }
    const int k0 = p.koff[n], k1 = p.koff[n + 1];
    if (lam4) {
      // four consecutive frames per thread, 16-byte V loads
      if (t4 < T) {
        Real lam[4] = {Real(0), Real(0), Real(0), Real(0)};
        int kst = k0;
        if constexpr (LAMV > 0) {
          // fp32: LAMV of the source's V columns loaded at once (one L2
          // round trip; the rest, if any, by the loop below)
          float4 vv[LAMV > 0 ? LAMV : 1];
#pragma unroll
          for (int q = 0; q < LAMV; ++q)
            if (k0 + q < k1) vv[q] = __ldg(reinterpret_cast<const float4*>(Vg + (size_t)(k0 + q) * T + t4));
#pragma unroll
          for (int q = 0; q < LAMV; ++q)
            if (k0 + q < k1) {
              const float b = Bs[k0 + q];
              lam[0] = fmaf(b, vv[q].x, lam[0]);
              lam[1] = fmaf(b, vv[q].y, lam[1]);
              lam[2] = fmaf(b, vv[q].z, lam[2]);
              lam[3] = fmaf(b, vv[q].w, lam[3]);
            }
          kst = min(k1, k0 + LAMV);
        }
#pragma unroll 8
        for (int kk = kst; kk < k1; ++kk) {
          const Real b = Bs[kk];
          const Real* vr = Vg + (size_t)kk * T + t4;
          if constexpr (F32) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(vr));
            lam[0] = fmaf(b, v.x, lam[0]);
            lam[1] = fmaf(b, v.y, lam[1]);
            lam[2] = fmaf(b, v.z, lam[2]);
            lam[3] = fmaf(b, v.w, lam[3]);
          } else {
            const double2 v0 = __ldg(reinterpret_cast<const double2*>(vr));
            const double2 v1 = __ldg(reinterpret_cast<const double2*>(vr) + 1);
            lam[0] = fma(b, v0.x, lam[0]);
            lam[1] = fma(b, v0.y, lam[1]);
            lam[2] = fma(b, v1.x, lam[2]);
            lam[3] = fma(b, v1.y, lam[3]);
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const Real l = fmax(lam[i], floor_abs);
          il[p.loff + t4 + i] = rcp_rn(l);
          if (p.has_prev) logsum += (double)min(L, T - t4 - i) * (double)log_fast(l);
        }
      }
    } else {
      Real lam[FT];
#pragma unroll
      for (int k = 0; k < FT; ++k) lam[k] = Real(0);
#pragma unroll 4
      for (int kk = k0; kk < k1; ++kk) {
        const Real b = Bs[kk];
        const Real* vrow = Vg + (size_t)kk * T;
#pragma unroll
        for (int k = 0; k < FT; ++k) {
          const int tau = tid + k * NT;
          if (tau < T) lam[k] = fma(b, __ldg(vrow + tau), lam[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        const int tau = tid + k * NT;
        if (tau < T) {
          const Real l = fmax(lam[k], floor_abs);
          il[p.loff + tau] = rcp_rn(l);
          if (p.has_prev) logsum += (double)min(L, T - tau) * (double)log_fast(l);
        }
      }
    }
  }
  __syncthreads();
  }
  CTF_PHASE(2);

  // ---- virtual tail frames j in [T, T+L-1): y_r(j) = sum_c W[r,c] x~_c(j)
  for (int e = tid; e < R * (L - 1); e += NT) {
    const int r = e % R, jj = e / R, j = T + jj;
    R2 y;
    y.x = y.y = Real(0);
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
      for (int l = 0; l < L; ++l) cmac(y, Wb[(m * L + l) * R + r], xs[m * p.xp + p.xoff + j - l]);
    Yt[r * LT1 + jj] = y;
  }

  if constexpr (TC) {
    static_assert(F32 && !IP, "tensor-core Gram: fp32 ISS only");
    using TCL = GramTC<M, L>;
    static_assert(TCL::TILES == 1 && NT == 512 && TCL::NP == 64, "readout mapping: 16 warps x (32 lanes, 16 columns)");
    __shared__ __align__(8) uint64_t s_mbar[2];
    __shared__ uint32_t s_tmem;
    unsigned char* stage0 = reinterpret_cast<unsigned char*>(part);  // 2 stages of TCL::STAGE bytes
    const int ng = gtab[NT].x;
    const int U0 = -(L - 1), len = T + 2 * (L - 1);
    const int nch = (len + TCL::KC - 1) / TCL::KC;
    if (warp == 0) tc::tmem_alloc(&s_tmem, TCL::TCOLS);
    if (tid == 0) {
      tc::mbar_init(&s_mbar[0], 1);
      tc::mbar_init(&s_mbar[1], 1);
    }
    // rows past the groups and columns past the sources stay zero in both stages
    for (int i = tid; i < 2 * TCL::STAGE / 16; i += NT) reinterpret_cast<float4*>(stage0)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    // this thread's production tasks, the same every stage: A (group, frame
    // quad) or B (column, frame quad); their x / weight bases and stage offsets
    constexpr int QPC = TCL::KC / 4;  // frame quads per stage
    constexpr int MAXT = 2;           // tasks per thread (NG*QPC + NC*QPC <= 2*NT)
    static_assert(TCL::NG * QPC + TCL::NC * QPC <= MAXT * NT, "production tasks per thread");
    const R2* tx1[MAXT];
    const R2* tx2[MAXT];
    int toff[MAXT], toff2[MAXT], tkind[MAXT];  // kind 0 none, 1 A, 2 B
#pragma unroll
    for (int i = 0; i < MAXT; ++i) {
      const int e = tid + i * NT;
      tkind[i] = 0;
      tx1[i] = tx2[i] = xs;
      toff[i] = toff2[i] = 0;
      if (e < ng * QPC) {
        const int g = e % ng, q = e / ng;
        const int4 gp = gtab[NT + 1 + 2 * g];
        tkind[i] = 1;
        tx1[i] = xs + gp.x * p.xp + p.xoff + 4 * q;
        tx2[i] = xs + gp.y * p.xp + p.xoff + gp.z + 4 * q;
        toff[i] = (q >> 1) * (TCL::ASTEP / 4) + tc::kmaj(g, (q & 1) * 4);
        toff2[i] = (q >> 1) * (TCL::ASTEP / 4) + tc::kmaj(TCL::TILES * 128 + g, (q & 1) * 4);
      } else if (e < ng * QPC + TCL::NC * QPC) {
        const int e2 = e - ng * QPC;
        const int j = e2 % TCL::NC, q = e2 / TCL::NC;
        const int n = j / NA, a = j - n * NA - (L - 1);
        tkind[i] = 2;
        tx1[i] = reinterpret_cast<const R2*>(invl + n * p.lp + p.loff + 4 * q - a);  // (weights, read as Real)
        toff[i] = (q >> 1) * (TCL::BSTEP / 4) + tc::kmaj(j, (q & 1) * 4);
      }
    }
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = s_tmem;
    constexpr uint32_t idesc = tc::idesc_tf32(128, TCL::NP);
    // TMEM columns: [set (chunk parity)][term: hi*hi, hi*lo + lo*hi][tile: re, im][NP]
    auto tcol = [](int set, int term, int tile) { return (uint32_t)(((set * 2 + term) * 2 + tile) * TCL::NP); };
    // readout mapping: warp w holds lanes 32 (w % 4) .. +31 (groups), columns 16 (w / 4) .. +15;
    // the per-chunk partials are summed here in fp32 (round to nearest) so the
    // tensor-core accumulation spans only one stage (2 K-steps)
    float sre[16], sim[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) sre[i] = sim[i] = 0.f;
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    const uint32_t col0 = (uint32_t)(16 * (warp >> 2));
    auto readout = [&](int set) {
      float h[16], c[16];
      tc::tmem_ld16(tmem + lane_base + tcol(set, 0, 0) + col0, h);
      tc::tmem_ld16(tmem + lane_base + tcol(set, 1, 0) + col0, c);
#pragma unroll
      for (int i = 0; i < 16; ++i) sre[i] += h[i] + c[i];
      tc::tmem_ld16(tmem + lane_base + tcol(set, 0, 1) + col0, h);
      tc::tmem_ld16(tmem + lane_base + tcol(set, 1, 1) + col0, c);
#pragma unroll
      for (int i = 0; i < 16; ++i) sim[i] += h[i] + c[i];
    };
    for (int c = 0; c < nch; ++c) {
      const int st = c & 1;
      unsigned char* sb = stage0 + st * TCL::STAGE;
      float* ahi = reinterpret_cast<float*>(sb);
      float* alo = reinterpret_cast<float*>(sb + TCL::KS * TCL::ASTEP);
      float* bhi = reinterpret_cast<float*>(sb + 2 * TCL::KS * TCL::ASTEP);
      float* blo = reinterpret_cast<float*>(sb + 2 * TCL::KS * TCL::ASTEP + TCL::KS * TCL::BSTEP);
      const int u0 = U0 + c * TCL::KC;
      // (stage st was last read by the MMAs of chunk c-2, waited for in the readout of iteration c-1)
#pragma unroll
      for (int i = 0; i < MAXT; ++i) {
        if (tkind[i] == 1) {
          const R2* x1 = tx1[i] + u0;
          const R2* x2 = tx2[i] + u0;
          float4 rh, rl, ih, il;
          float* prh = &rh.x;
          float* prl = &rl.x;
          float* pih = &ih.x;
          float* pil = &il.x;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const R2 v = Ops::mulc(x1[k], x2[k]);
            tc::split_tf32(v.x, prh[k], prl[k]);
            tc::split_tf32(v.y, pih[k], pil[k]);
          }
          *reinterpret_cast<float4*>(ahi + toff[i]) = rh;
          *reinterpret_cast<float4*>(alo + toff[i]) = rl;
          *reinterpret_cast<float4*>(ahi + toff2[i]) = ih;
          *reinterpret_cast<float4*>(alo + toff2[i]) = il;
        } else if (tkind[i] == 2) {
          const Real* w = reinterpret_cast<const Real*>(tx1[i]) + u0;
          float4 hv, lv;
          tc::split_tf32(w[0], hv.x, lv.x);
          tc::split_tf32(w[1], hv.y, lv.y);
          tc::split_tf32(w[2], hv.z, lv.z);
          tc::split_tf32(w[3], hv.w, lv.w);
          *reinterpret_cast<float4*>(bhi + toff[i]) = hv;
          *reinterpret_cast<float4*>(blo + toff[i]) = lv;
        }
      }
      tc::fence_async_smem();
      tc::fence_before_sync();
      __syncthreads();  // stage c written; the readout of chunk c-2's set finished
      if (tid == 0) {
        tc::fence_after_sync();
#pragma unroll
        for (int ks = 0; ks < TCL::KS; ++ks)
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const unsigned char* ah = reinterpret_cast<const unsigned char*>(ahi) + ks * TCL::ASTEP + t * 4096;
            const unsigned char* al = reinterpret_cast<const unsigned char*>(alo) + ks * TCL::ASTEP + t * 4096;
            const unsigned char* bh = reinterpret_cast<const unsigned char*>(bhi) + ks * TCL::BSTEP;
            const unsigned char* bl = reinterpret_cast<const unsigned char*>(blo) + ks * TCL::BSTEP;
            tc::mma_tf32(tmem + tcol(st, 0, t), tc::desc(ah), tc::desc(bh), idesc, ks > 0);
            tc::mma_tf32(tmem + tcol(st, 1, t), tc::desc(ah), tc::desc(bl), idesc, ks > 0);
            tc::mma_tf32(tmem + tcol(st, 1, t), tc::desc(al), tc::desc(bh), idesc, true);
          }
        tc::commit(&s_mbar[st]);
      }
      if (c >= 1) {  // partials of chunk c-1 (its MMAs overlap this chunk's production)
        tc::mbar_wait(&s_mbar[st ^ 1], ((c - 1) >> 1) & 1);
        tc::fence_after_sync();
        readout(st ^ 1);
      }
    }
    tc::mbar_wait(&s_mbar[(nch - 1) & 1], ((nch - 1) >> 1) & 1);
    tc::fence_after_sync();
    readout((nch - 1) & 1);
    CTF_PHASE(3);
    const int g = 32 * (warp & 3) + lane;
    if (g < ng) {
      const int4 h0 = gtab[NT + 1 + 2 * g], h1 = gtab[NT + 2 + 2 * g];
      const int m = h0.x, m2 = h0.y, d = h0.z, alo = h0.w, cnt = h1.x;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int j = (int)col0 + i;
        if (j >= TCL::NC) continue;
        const int n = j / NA, a = j - n * NA - (L - 1);
        if (a < alo || a >= alo + cnt) continue;
        R2 v;
        v.x = sre[i];
        v.y = sim[i];
        G[gidx(n, m, m2, a, a + d)] = v;
        if (m == m2 && d != 0) {
          v.y = -v.y;
          G[gidx(n, m, m, a + d, a)] = v;
        }
      }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, TCL::TCOLS);
  } else {
  // ---- Gram: this thread's (m, m', d) task over frames [u0, u1), NS
  // sources per pass. The lag count is made warp-uniform (groups are sorted
  // by it, so a warp spans at most two adjacent counts): no divergent code
  // paths, extra lags discarded. Each pass: partials -> barrier -> fixed-order
  // reduction over the group's chunks with the Hermitian mirror -> barrier.
  {
    const int4 tk = gtab[tid];
    const bool active = tk.x >= 0;
    const int4 g0 = gtab[NT + 1 + 2 * max(tk.x, 0)], g1 = gtab[NT + 2 + 2 * max(tk.x, 0)];
    const int cnt = active ? g1.x : 0;
    const int cmax = __reduce_max_sync(kFull, cnt);
    const R2* x1 = xs + g0.x * p.xp + p.xoff;
    const R2* x2 = xs + g0.y * p.xp + p.xoff + g0.z;
    const int ng = gtab[NT].x;
    constexpr int NSG = gram_nsg<Real, N, R>();  // sources per pass over the frames
    constexpr int NSP = EREG ? 1 : NS;           // sources whose partials fit the buffer at once
    static_assert(NSG % NSP == 0, "partial groups");
    R2 keep[NSG > NSP ? NSG - NSP : 1][NA];  // partials of the later source groups, in registers
    for (int n0 = 0; n0 < N; n0 += NSG) {
      const Real* w0 = invl + n0 * p.lp + p.loff - g0.w;
      static_for<L, NA + 1>([&](auto cc) {
        constexpr int C = decltype(cc)::value;
        if (cmax == C) {
          // the widest lag window of the fp64 two-source pass runs one source
          // per pass over the frames (its accumulators would spill)
          constexpr int NSGC = (!F32 && NSG > NSP && C == NA && CTF_GRAM_SPLITWIDE) ? NSP : NSG;
          constexpr int UBC = NSGC > NSP ? CTF_GRAM_UB2 : kGramUB;
#pragma unroll
          for (int s = 0; s < NSG; s += NSGC) {
            R2 acc[NSGC][C];
#pragma unroll
            for (int n = 0; n < NSGC; ++n)
#pragma unroll
              for (int j = 0; j < C; ++j) acc[n][j].x = acc[n][j].y = Real(0);
            if (active) gram_block<Real, C, NSGC, UBC>(x1, x2, w0 + s * p.lp, p.lp, tk.y, tk.z, acc);
#pragma unroll
            for (int n = 0; n < NSGC; ++n) {
              if (s + n < NSP) {
#pragma unroll
                for (int j = 0; j < C; ++j)
                  if (j < cnt) part[(size_t)((s + n) * NA + j) * (NT + 1) + tid] = acc[n][j];
              } else {
#pragma unroll
                for (int j = 0; j < C; ++j) keep[(s + n - NSP) < 0 ? 0 : s + n - NSP][j] = acc[n][j];
              }
            }
          }
        }
      });
#pragma unroll
      for (int s0 = 0; s0 < NSG; s0 += NSP) {
        if (s0 > 0) {  // the next source group's partials from registers (lags >= cmax are never read)
#pragma unroll
          for (int n = 0; n < NSP; ++n)
#pragma unroll
            for (int j = 0; j < NA; ++j)
              if (j < cnt) part[(size_t)(n * NA + j) * (NT + 1) + tid] = keep[s0 - NSP + n][j];
        }
        __syncthreads();
        CTF_PHASE(3);
        for (int e = tid; e < ng * NSP * NA; e += NT) {
          const int g = e / (NSP * NA), rr = e - g * (NSP * NA), n = rr / NA, j = rr - n * NA;
          const int4 h0 = gtab[NT + 1 + 2 * g], h1 = gtab[NT + 2 + 2 * g];
          if (j >= h1.x) continue;
          R2 sum;
          sum.x = sum.y = Real(0);
          const R2* pr = part + (size_t)(n * NA + j) * (NT + 1);
          for (int t = h1.y; t < h1.z; ++t) {
            sum.x += pr[t].x;
            sum.y += pr[t].y;
          }
          const int m = h0.x, m2 = h0.y, d = h0.z, a = h0.w + j, b = a + d;
          G[gidx(n0 + s0 + n, m, m2, a, b)] = sum;  // groups have m <= m2
          if (m == m2 && d != 0) {                   // the mirrored lag of the same mic
            R2 mir = sum;
            mir.y = -sum.y;
            G[gidx(n0 + s0 + n, m, m, b, a)] = mir;
          }
        }
        __syncthreads();
      }
    }
  }
  }
  CTF_PHASE(4);

  // ---- covariance-domain steps with register-resident rows. A group of LPR
  // lanes (a half-warp when D <= 16, a warp for the wide tiles) owns KR rows
  // p; its lane c < D holds W[p][c], the tail frame T + c of y_p (c < L-1)
  // and, for c < l_p, its weight w_n(T + c - l_p); for D <= 16 also the row c
  // of C_p (D complex, else read from the Gram table each step). A step needs
  // only the pivot row (W_r and its tail), published through shared memory:
  // one barrier per step.
  constexpr bool WIDE = D > 16;
  constexpr int LPR = WIDE ? 32 : 16;
  constexpr int GROUPS = NT / LPR;
  constexpr int KR = (R + GROUPS - 1) / GROUPS;  // rows per lane group
  static_assert(L - 1 <= LPR, "tail frames per lane group");
  static_assert(WIDE || KR == 1, "narrow tiles: one row per half-warp");
  const int hl = lane & (LPR - 1);
  const int slot = tid / LPR;
  int rowk[KR], rnk[KR], rlk[KR];
  bool rowvk[KR];
  R2 wreg[KR], yreg[KR];
  Real wt[KR];
  R2 creg[WIDE ? 1 : D];
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int row = slot + k * GROUPS;
    rowk[k] = row;
    rowvk[k] = row < R;
    rnk[k] = rowvk[k] ? row / L : 0;
    rlk[k] = rowvk[k] ? row - rnk[k] * L : 0;
    wreg[k].x = wreg[k].y = yreg[k].x = yreg[k].y = Real(0);
    wt[k] = Real(0);
    if (rowvk[k] && hl < D) wreg[k] = Wb[hl * R + row];
    if (rowvk[k] && hl < L - 1) yreg[k] = Yt[row * LT1 + hl];                       // for when this row pivots
    if (rowvk[k] && hl < rlk[k]) wt[k] = invl[rnk[k] * p.lp + p.loff + T + hl - rlk[k]];  // own truncation
  }
  const int mh = hl / L, l1h = hl - mh * L;  // stacked channel of this lane
  // wide tiles: Gram-table addressing of this lane's C_p row per mic m2
  int gbase[WIDE ? KR : 1][M], gstr[WIDE ? KR : 1][M];
  Real gsgn[WIDE ? KR : 1][M];
  if constexpr (WIDE) {
#pragma unroll
    for (int k = 0; k < KR; ++k)
#pragma unroll
      for (int m2 = 0; m2 < M; ++m2) {
        const bool up = mh <= m2;
        const int a0 = rlk[k] - l1h, b0 = rlk[k];
        gbase[k][m2] = (rowvk[k] && hl < D) ? (up ? gidx(rnk[k], mh, m2, a0, b0) : gidx(rnk[k], m2, mh, b0, a0)) : 0;
        gstr[k][m2] = up ? -1 : -NA;
        gsgn[k][m2] = up ? Real(1) : Real(-1);
      }
  }
  if constexpr (!WIDE) {
    const bool chan = rowvk[0] && hl < D;
#pragma unroll
    for (int m2 = 0; m2 < M; ++m2)
#pragma unroll
      for (int l2 = 0; l2 < L; ++l2) {
        R2 c;
        c.x = c.y = Real(0);
        if (chan) c = gget(rnk[0], mh, m2, rlk[0] - l1h, rlk[0] - l2);
        creg[m2 * L + l2] = c;
      }
  }
  // (num, den) of row slot k against a pivot: pw[c * ps] = pivot W, py[c] = pivot tail
  auto row_sums = [&](int k, const R2* pw, int ps, const R2* py, Real& nre, Real& nim, Real& den) {
    R2 q0, q1;
    q0.x = q0.y = q1.x = q1.y = Real(0);
    if constexpr (WIDE) {
      if (rowvk[k] && hl < D) {
        // C_p[c][(m2, l2)] = G(n, m, m2, l - l1, l - l2): for m2 >= m the
        // stored entry (stride -1 in l2), else the conjugate of (m2, m, l-l2,
        // l-l1) (stride -NA); bases, strides and signs precomputed per row
#pragma unroll
        for (int m2 = 0; m2 < M; ++m2)
#pragma unroll
          for (int l2 = 0; l2 < L; ++l2) {  // q += C conj(w), C from the Gram table
            const int c = m2 * L + l2;
            const R2 w = pw[c * ps];
            R2 cc = G[gbase[k][m2] + l2 * gstr[k][m2]];
            cc.y *= gsgn[k][m2];
            if (c & 1)
              q1 = Ops::macc(cc, w, q1);
            else
              q0 = Ops::macc(cc, w, q0);
          }
      }
    } else {
#pragma unroll
      for (int c = 0; c < D; ++c) {  // q += C conj(w)
        const R2 w = pw[c * ps];
        if (c & 1)
          q1 = Ops::macc(creg[c], w, q1);
        else
          q0 = Ops::macc(creg[c], w, q0);
      }
    }
    R2 q;
    q.x = q0.x + q1.x;
    q.y = q0.y + q1.y;
    R2 wr;
    wr.x = wr.y = Real(0);
    if (hl < D) wr = pw[hl * ps];
    R2 cn = cmul(wreg[k], q), cd = cmul(wr, q);
    // virtual frames T + hl (hl < l_p): subtract w y_p conj(y_r), w |y_r|^2
    R2 yr;
    yr.x = yr.y = Real(0);
    if (hl < LT1) yr = py[hl];
    cn.x -= wt[k] * fma(yreg[k].x, yr.x, yreg[k].y * yr.y);
    cn.y -= wt[k] * fma(yreg[k].y, yr.x, -yreg[k].x * yr.y);
    cd.x -= wt[k] * fma(yr.x, yr.x, yr.y * yr.y);
#pragma unroll
    for (int o = LPR / 2; o >= 1; o >>= 1) {
      cn.x += __shfl_xor_sync(kFull, cn.x, o);
      cn.y += __shfl_xor_sync(kFull, cn.y, o);
      cd.x += __shfl_xor_sync(kFull, cd.x, o);
    }
    nre = cn.x;
    nim = cn.y;
    den = cd.x;
  };

  // conditioning of the Gram form for row slot k (pre-sweep W): the
  // quadratic form w^H Q w = sum_t |y(t)|^2 / lambda cancels when lambda is
  // small where |x| is not (NMF activations near the floor); its rounding
  // error grows with kappa = sum_c |w_c|^2 Q(c,c) / w^H Q w, while the
  // frame-domain sums (sweep_kernel) do not. Over fb_theta the bin is handed
  // to the frame-domain kernel (fb_mode 1). Warp-uniform (every lane calls it).
  auto cond_check = [&](int k, int rr, Real den) {
    if constexpr (!WIDE && !IP) {
      if (p.fb_mode == 1) {
        Real qd = Real(0);
#pragma unroll
        for (int c = 0; c < D; ++c)
          if (c == hl) qd = creg[c].x;
        Real a = Real(0);
        if (rowvk[k] && hl < D) {
          const R2 w = Wb[hl * R + rr];
          a = (w.x * w.x + w.y * w.y) * qd;
        }
#pragma unroll
        for (int o = LPR / 2; o >= 1; o >>= 1) a += __shfl_xor_sync(kFull, a, o);
        if (hl == 0 && rowvk[k] && !((double)a <= p.fb_theta * (double)den)) s_fb = 1;
      }
    }
  };
  double logdet = p.logdet[tile] - s_logmu;
  // Narrow ISS tiles (CTF_GRAM_CHAIN): the steps below run without a CTA
  // barrier per step: every pivot has its own buffer (R x (D + LT1), in the
  // Gram partial region, free between the Gram reduction and the |y|^2 rows)
  // and its own mbarrier. The objective / conditioning phase, the first
  // pivot's publish and the mbarrier initialisation share ONE barrier.
  constexpr bool CHAIN = !WIDE && !IP && CTF_GRAM_CHAIN;
  constexpr int PV = D + LT1;
  R2* piv = CHAIN ? reinterpret_cast<R2*>(smem + p.off_e) : zs;  // !CHAIN: 2 x PV, double-buffered by step parity
  uint64_t* mbar = reinterpret_cast<uint64_t*>(piv + R * PV);
  if constexpr (CHAIN) {
    if (p.has_prev || p.fb_mode == 1) {
      // quadratic term of the previous iteration's objective (estimator.cpp:55-77):
      // sum_r w_r^T C_r conj(w_r) of the rescaled W under the new lambda
      Real nre, nim, den;
      const int rr = rowvk[0] ? rowk[0] : 0;
      row_sums(0, Wb + rr, R, Yt + rr * LT1, nre, nim, den);
      if (p.has_prev && hl == 0 && rowvk[0]) red[rowk[0]] = den;
      cond_check(0, rr, den);
    }
    if (p.has_prev) {
      const double ws = warp_sum(logsum);
      if (lane == 0) dred[warp] = ws;
    }
    if (rowk[0] == 0) {  // pivot 0 (published even when the CTA returns below)
      if (hl < D) piv[hl] = wreg[0];
      if (hl < LT1) piv[D + hl] = yreg[0];
    }
    if (tid < R) tc::mbar_init(&mbar[tid], 1);
    __syncthreads();
    if (p.has_prev) {
      const int det_status = isnan(logdet) || logdet == -INFINITY ? 4 : (logdet < log(1e-300) ? 5 : 0);
      if (det_status) {  // estimator.cpp:45-51
        if (tid == 0) record_err<Real>(p.err, mix, err_key(prev_it, kPhDet, gbin, 0, det_status));
        return;
      }
      if (tid == 0) {
        double quad = 0.0, ls = 0.0;
        for (int r = 0; r < R; ++r) quad += (double)red[r];
        for (int w = 0; w < NW; ++w) ls += dred[w];
        p.objbin[tile] = ls + quad - 2.0 * (double)T * logdet;
      }
    }
  } else if (p.has_prev) {
    // objective of the previous iteration (estimator.cpp:55-77): quadratic
    // term sum_r w_r^T C_r conj(w_r) of the rescaled W under the new lambda
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      Real nre, nim, den;
      const int rr = rowvk[k] ? rowk[k] : 0;
      row_sums(k, Wb + rr, R, Yt + rr * LT1, nre, nim, den);
      if (hl == 0 && rowvk[k]) red[rowk[k]] = den;
      cond_check(k, rr, den);
    }
    double v1[1] = {logsum};
    block_sum_d<1>(v1, dred, lane, warp, NW);  // contains __syncthreads: red visible after
    double quad = 0.0;
    for (int r = 0; r < R; ++r) quad += (double)red[r];
    const int det_status = isnan(logdet) || logdet == -INFINITY ? 4 : (logdet < log(1e-300) ? 5 : 0);
    if (det_status) {  // estimator.cpp:45-51
      if (tid == 0) record_err<Real>(p.err, mix, err_key(prev_it, kPhDet, gbin, 0, det_status));
      return;
    }
    if (tid == 0) p.objbin[tile] = v1[0] + quad - 2.0 * (double)T * logdet;
  } else if (!WIDE && !IP && p.fb_mode == 1) {  // first loop body after a finalize: check only
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      Real nre, nim, den;
      const int rr = rowvk[k] ? rowk[k] : 0;
      row_sums(k, Wb + rr, R, Yt + rr * LT1, nre, nim, den);
      cond_check(k, rr, den);
    }
    __syncthreads();
  }
  if (s_fb) {  // nothing of this bin is written (but objbin, which the frame-domain kernel recomputes)
    if (tid == 0) p.fb_list[atomicAdd(p.fb_count, 1)] = (int)tile;
    return;
  }

  if (!p.do_sweep) {  // finalize pass: write the rescaled state and stop
    for (int i = tid; i < R * D; i += NT) Wg[i] = Wb[i];
    for (int i = tid; i < SK; i += NT) Bg[i] = Bs[i];
    if (tid == 0) p.logdet[tile] = logdet;
    return;
  }

  __shared__ double s_iplogdet;
  if constexpr (IP) {
    // ---- IP rule (estimator.cpp:580-606, ip_update :103-273): for each row
    // r, h = (Q_r + Q_r^H) / 2 with Q_r the weighted covariance / T
    // (:89-101, from the Gram minus the virtual tail frames), solve
    // (W h) u = e_r by LU with partial pivoting (pivot-ratio singularity
    // probe 1e-13, one retry with 1e-10 trace/D diagonal loading), w_r =
    // conj(u) / sqrt(u^H h u), then the frame-sum refinement
    // w_r /= sqrt(sum_{j>=l} |w_r x~(j)|^2 / lambda(j-l) / T).
    R2* qm = part;             // D x D raw Q_r / T
    R2* cov = part + D * D;    // D x D Hermitian h
    R2* A = cov + D * D;       // D x (D+1), column-major, rhs last
    R2* sol = A + D * (D + 1); // D
    __shared__ int s_iperr;
    __shared__ double s_power;
    if (tid == 0) s_iperr = 0;
    for (int r = 0; r < R; ++r) {
      const int n = r / L, l = r - n * L;
      for (int e = tid; e < D * D; e += NT) {
        const int a = e % D, b = e / D;
        const int m = a / L, l1 = a - m * L, m2 = b / L, l2 = b - m2 * L;
        R2 v = gget(n, m, m2, l - l1, l - l2);
        for (int jj = 0; jj < l; ++jj) {  // frames j = T + jj are outside row l's range
          const Real w = invl[n * p.lp + p.loff + T + jj - l];
          const R2 xa = xs[m * p.xp + p.xoff + T + jj - l1], xb = xs[m2 * p.xp + p.xoff + T + jj - l2];
          v.x -= w * fma(xa.x, xb.x, xa.y * xb.y);
          v.y -= w * fma(xa.y, xb.x, -xa.x * xb.y);
        }
        v.x /= (Real)T;
        v.y /= (Real)T;
        qm[a + b * D] = v;
      }
      __syncthreads();
      for (int e = tid; e < D * D; e += NT) {
        const int a = e % D, b = e / D;
        const R2 u = qm[a + b * D], t = qm[b + a * D];
        R2 h;
        h.x = Real(0.5) * (u.x + t.x);
        h.y = Real(0.5) * (u.y - t.y);
        cov[a + b * D] = h;
      }
      __syncthreads();
      if (warp == 0) {
        const int err = ip_solve_row<Real>(Wb, R, D, r, cov, A, sol, lane);
        if (lane == 0 && err) s_iperr = err;
      }
      __syncthreads();
      if (s_iperr) {
        if (tid == 0) record_err<Real>(p.err, mix, err_key(p.iteration, kPhSweep, gbin, r, s_iperr));
        return;
      }
      // frame-sum refinement of the row scale (estimator.cpp:596-602)
      double pw = 0.0;
      for (int k = 0; k < FT; ++k) {
        const int j = tid + k * NT;
        if (j < T) {
          R2 y;
          y.x = y.y = Real(0);
#pragma unroll
          for (int m = 0; m < M; ++m)
#pragma unroll
            for (int l1 = 0; l1 < L; ++l1) cmac(y, Wb[r + (m * L + l1) * R], xs[m * p.xp + p.xoff + j - l1]);
          pw += (double)(cnorm(y) * invl[n * p.lp + p.loff + j - l]);
        }
      }
      double v1[1] = {pw};
      block_sum_d<1>(v1, dred, lane, warp, NW);
      const double power = v1[0] / T;
      if (power > 0.0 && isfinite(power) && tid < D) {
        R2 w = Wb[r + tid * R];
        w.x = (Real)((double)w.x / sqrt(power));
        w.y = (Real)((double)w.y / sqrt(power));
        Wb[r + tid * R] = w;
      }
      __syncthreads();
    }
    // exact log|det W'| (no determinant lemma for IP)
    if (warp == 0) {
      R2* Acp = part;
      for (int i = lane; i < R * D; i += 32) Acp[i] = Wb[i];
      __syncwarp();
      double out = 0.0;
      const int st = warp_logdet<Real>(Acp, R, lane, out);
      if (lane == 0) s_iplogdet = st == 4 ? -INFINITY : out;
    }
    __syncthreads();
  } else {
  // ---- R covariance-domain ISS steps (estimator.cpp:556-579, 275-302)
  // CHAIN: the half-warp of row r + 1 publishes its updated row as soon as its
  // step-r update is done and arrives on that pivot's mbarrier; the warps wait
  // only on the pivot they are about to read. The pivot's own scale (a division
  // and a square root) runs after the publish, so the dependent chain of the
  // sweep is load -> matvec -> reduce -> one reciprocal -> update -> publish per
  // step. (Pivot 0 and the mbarriers: set up before the barrier above.)
  Real* fac = fac_s;  // (1 - z_r) per row, multiplied in row order at the end
  if constexpr (!CHAIN) {
    if (rowk[0] == 0) {
      if (hl < D) piv[hl] = wreg[0];
      if (hl < LT1) piv[D + hl] = yreg[0];
    }
    __syncthreads();
  }
  CTF_PHASE(5);
  const bool wrows = (tid / 32) * (32 / LPR) < R;  // warp-uniform: this warp owns at least one row
  if constexpr (CHAIN) {
    if (wrows) {
      const int row = rowk[0];
      for (int r = 0; r < R; ++r) {
        const R2* pv = piv + r * PV;
        if (r > 0) {
          if constexpr (CTF_GRAM_SPIN != 0) tc::mbar_spin(&mbar[r], 0);
          else tc::mbar_wait(&mbar[r], 0);
        }
        Real nre, nim, den;
        row_sums(0, pv, 1, pv + D, nre, nim, den);
        const bool ok = rowvk[0] && den > Real(0) && isfinite(den);  // estimator.cpp:451-454
        if (rowvk[0] && !ok && hl == 0) atomicMin(&s_badrow, r * 64 + row);
        R2 z;
        z.x = z.y = Real(0);
        if (ok && row != r) {  // every row but the pivot first: the next pivot is among them
          Real inv;
          // (on the dependent chain of every step)
          if constexpr (F32) inv = CTF_GRAM_RCPNR32 ? rcp_fast(den) : __frcp_rn(den);
          else inv = CTF_GRAM_RCPNR ? rcp_muv(den) : 1.0 / den;
          z.x = nre * inv;
          z.y = nim * inv;
        }
        // iss_apply (estimator.cpp:298-302) on the own row and its tail
        if (hl < D) cmsub(wreg[0], z, pv[hl]);
        if (hl < LT1) cmsub(yreg[0], z, pv[D + hl]);
        if (r + 1 < R) {
          if (row == r + 1) {
            R2* nx = piv + (r + 1) * PV;
            if (hl < D) nx[hl] = wreg[0];
            if (hl < LT1) nx[D + hl] = yreg[0];
          }
          __syncwarp();
          if (row == r + 1 && hl == 0) tc::mbar_arrive(&mbar[r + 1]);
        }
        if (ok && row == r) {  // the pivot's own scale: w_r (1 - z_r), off the chain
          R2 zp;
          zp.y = Real(0);
          if constexpr (F32) zp.x = 1.f - sqrtf((float)T) * rsqrtf(den);
          else zp.x = 1.0 - sqrt((double)T / den);
          if (hl == 0) fac[row] = Real(1) - zp.x;
          if (hl < D) cmsub(wreg[0], zp, pv[hl]);
          if (hl < LT1) cmsub(yreg[0], zp, pv[D + hl]);
        }
      }
    }
    __syncthreads();
    if (tid < R) tc::mbar_inval(&mbar[tid]);  // the region is plain data again below
  } else {
  for (int r = 0; r < R; ++r) {
    const R2* pv = piv + (r & 1) * PV;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      Real nre = Real(0), nim = Real(0), den = Real(0);
      if (wrows) row_sums(k, pv, 1, pv + D, nre, nim, den);
      R2 z;
      z.x = z.y = Real(0);
      const int row = rowk[k];
      if (rowvk[k]) {
        if (!(den > Real(0)) || !isfinite(den)) {  // estimator.cpp:451-454
          // (step, row) key: the first failing step, its lowest row; checked
          // once after the sweep (the steps after a failure change nothing
          // that is written out)
          if (hl == 0) atomicMin(&s_badrow, r * 64 + row);
        } else if (row == r) {
          if constexpr (F32)
            z.x = 1.f - sqrtf((float)T) * rsqrtf(den);
          else
            z.x = 1.0 - sqrt((double)T / den);
          if (hl == 0) fac[row] = Real(1) - z.x;
        } else {
          if constexpr (F32) {
            const float inv = __frcp_rn(den);
            z.x = nre * inv;
            z.y = nim * inv;
          } else if constexpr (CTF_GRAM_RCP64) {  // one division (rounding differs by <= 1 ulp)
            const double inv = 1.0 / den;
            z.x = nre * inv;
            z.y = nim * inv;
          } else {
            z.x = nre / den;
            z.y = nim / den;
          }
        }
      }
      // iss_apply (estimator.cpp:298-302) on the own row and its tail
      if (hl < D) cmsub(wreg[k], z, pv[hl]);
      if (hl < LT1) cmsub(yreg[k], z, pv[D + hl]);
      if (row == r + 1) {  // the next pivot publishes its updated row
        R2* nx = piv + ((r + 1) & 1) * PV;
        if (hl < D) nx[hl] = wreg[k];
        if (hl < LT1) nx[D + hl] = yreg[k];
      }
    }
    __syncthreads();
  }
  }
  if (s_badrow != kNoRow) {
    if (tid == 0) record_err<Real>(p.err, mix, err_key(p.iteration, kPhSweep, gbin, s_badrow >> 6, s_badrow & 63));
    return;
  }
#pragma unroll
  for (int k = 0; k < KR; ++k)
    if (rowvk[k] && hl < D) Wb[hl * R + rowk[k]] = wreg[k];
  __syncthreads();
  }
  R2* Wf = Wb;  // W' (column-major R x D) for the demix
  CTF_PHASE(6);

  // ---- per source group (fp32: all sources, fp64: one): Y rows of the group
  // = W' x~ (estimator.cpp:607) for this thread's frames (|y|^2 to shared
  // memory, row powers), delayed energies E_n(tau) = sum_{l, tau+l<T}
  // |y_(n,l)(tau+l)|^2 in l order (estimator.cpp:318-330, written in place of
  // the source's first |y|^2 row), then MU-B per source (estimator.cpp
  // :313-346, 16 bases per pass)
  constexpr int NSD = NS;  // sources per demix group = per Gram pass
  constexpr int GR = NSD * L;  // rows per group
  Real rp[R];
#pragma unroll
  for (int i = 0; i < R; ++i) rp[i] = Real(0);
  Real* Eg = reinterpret_cast<Real*>(p.E);
#pragma unroll
  for (int g0 = 0; g0 < N; g0 += NSD) {  // unrolled: the row-power register index is static
    // FB frames per pass would share the W loads
    // frames per demix pass: 2 share the W loads (fp64: half the broadcast
    // shared-memory wavefronts); fp32 at its 80-register budget spills with 2
#ifndef CTF_GRAM_FB64
#define CTF_GRAM_FB64 2
#endif
    constexpr int FB = F32 ? 1 : CTF_GRAM_FB64;
    Real ereg[NSD][EREG ? FT : 1];  // EREG: E_n of this thread's frames
    if constexpr (EREG) {
    // E_n(tau) in registers: the row-(n,l) term |y|^2 at tau + l comes from
    // lane + l of the same warp by a shuffle, or, past the warp's last lane,
    // from the next warp's first L-1 lanes (frame k) / warp 0's (frame k+1)
    // through a small halo buffer; terms are added in l order as before.
    constexpr int LH = L > 1 ? L - 1 : 1;
    Real* halo = reinterpret_cast<Real*>(smem + p.off_e);  // [warp][k][source][l-1][lane < L-1]
    auto hidx = [&](int w, int kk, int s, int l, int ln) { return (((w * FT + kk) * NSD + s) * LH + (l - 1)) * LH + ln; };
#pragma unroll
    for (int k = 0; k < FT; k += FB) {
      asm volatile("" ::: "memory");  // one frame pass at a time (registers)
      R2 acc[FB][GR];
#pragma unroll
      for (int f = 0; f < FB; ++f)
#pragma unroll
        for (int i = 0; i < GR; ++i) acc[f][i].x = acc[f][i].y = Real(0);
#pragma unroll
      for (int m = 0; m < M; ++m)
#pragma unroll
        for (int l1 = 0; l1 < L; ++l1) {
          R2 xv[FB];
#pragma unroll
          for (int f = 0; f < FB; ++f) xv[f] = xs[m * p.xp + p.xoff + tid + (k + f) * NT - l1];
          const R2* wc = Wf + (m * L + l1) * R + g0 * L;
          if constexpr (F32 && GR % 2 == 0) {  // W pairs with 16-byte loads
            const float4* w4 = reinterpret_cast<const float4*>(wc);
#pragma unroll
            for (int i = 0; i < GR; i += 2) {
              const float4 w = w4[i / 2];
#pragma unroll
              for (int f = 0; f < FB; ++f) {
                acc[f][i] = Ops::mac(make_float2(w.x, w.y), xv[f], acc[f][i]);
                acc[f][i + 1] = Ops::mac(make_float2(w.z, w.w), xv[f], acc[f][i + 1]);
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < GR; ++i)
#pragma unroll
              for (int f = 0; f < FB; ++f) acc[f][i] = Ops::mac(wc[i], xv[f], acc[f][i]);
          }
        }
#pragma unroll
      for (int f = 0; f < FB; ++f) {
        const int j = tid + (k + f) * NT;
        Real q[GR];
#pragma unroll
        for (int i = 0; i < GR; ++i) {
          q[i] = (j < T) ? cnorm(acc[f][i]) : Real(0);
          rp[g0 * L + i] += q[i];
        }
#pragma unroll
        for (int s = 0; s < NSD; ++s) {
          Real e = q[s * L];
#pragma unroll
          for (int l = 1; l < L; ++l) {
            const Real v = __shfl_down_sync(kFull, q[s * L + l], l);
            if (lane + l < 32) e += v;
            if (lane < L - 1) halo[hidx(warp, k + f, s, l, lane)] = q[s * L + l];
          }
          ereg[s][k + f] = e;
        }
      }
    }
    __syncthreads();  // halo complete
    CTF_PHASE(7);
#pragma unroll
    for (int s = 0; s < NSD; ++s)
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        const int tau = tid + k * NT;
#pragma unroll
        for (int l = 1; l < L; ++l)
          if (lane + l >= 32) {  // frame tau + l belongs to the next warp (or warp 0 at frame k + 1)
            const int t2 = tid + l;
            Real v = Real(0);
            if (t2 < NT) v = halo[hidx(t2 >> 5, k, s, l, t2 & 31)];
            else if (k + 1 < FT) v = halo[hidx(0, k + 1, s, l, t2 - NT)];
            ereg[s][k] += v;
          }
        if (tau < T) Eg[(((size_t)mix * N + g0 + s) * p.FL + bin) * T + tau] = ereg[s][k];
      }
    } else {
#pragma unroll 1
    for (int k = 0; k < FT; k += FB) {
      R2 acc[FB][GR];
#pragma unroll
      for (int f = 0; f < FB; ++f)
#pragma unroll
        for (int i = 0; i < GR; ++i) acc[f][i].x = acc[f][i].y = Real(0);
#pragma unroll
      for (int m = 0; m < M; ++m)
#pragma unroll
        for (int l1 = 0; l1 < L; ++l1) {
          R2 xv[FB];
#pragma unroll
          for (int f = 0; f < FB; ++f) xv[f] = xs[m * p.xp + p.xoff + tid + (k + f) * NT - l1];
          const R2* wc = Wf + (m * L + l1) * R + g0 * L;
          if constexpr (F32 && GR % 2 == 0) {  // W pairs with 16-byte loads
            const float4* w4 = reinterpret_cast<const float4*>(wc);
#pragma unroll
            for (int i = 0; i < GR; i += 2) {
              const float4 w = w4[i / 2];
#pragma unroll
              for (int f = 0; f < FB; ++f) {
                acc[f][i] = Ops::mac(make_float2(w.x, w.y), xv[f], acc[f][i]);
                acc[f][i + 1] = Ops::mac(make_float2(w.z, w.w), xv[f], acc[f][i + 1]);
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < GR; ++i)
#pragma unroll
              for (int f = 0; f < FB; ++f) acc[f][i] = Ops::mac(wc[i], xv[f], acc[f][i]);
          }
        }
#pragma unroll
      for (int f = 0; f < FB; ++f) {
        const int j = tid + (k + f) * NT;
#pragma unroll
        for (int i = 0; i < GR; ++i) {
          const Real q = (j < T) ? cnorm(acc[f][i]) : Real(0);
          Pq[i * TP + j] = q;
          rp[g0 * L + i] += q;
        }
      }
    }
    __syncthreads();  // Pq of the group complete
    CTF_PHASE(7);
#pragma unroll
    for (int n = g0; n < g0 + NSD; ++n) {
      Real* pq = Pq + (size_t)(n - g0) * L * TP;
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        const int tau = tid + k * NT;
        Real e = Real(0);
#pragma unroll
        for (int l = 0; l < L; ++l)
          if (tau + l < T) e += pq[l * TP + tau + l];
        pq[tau] = e;  // entry tau of the source's first row is read only by this thread
        if (tau < T) Eg[(((size_t)mix * N + n) * p.FL + bin) * T + tau] = e;
      }
    }
    }
    __syncthreads();  // red is shared by the MU-B passes below
#pragma unroll
    for (int n = g0; n < g0 + NSD; ++n) {
      const Real* En = Pq + (size_t)(n - g0) * L * TP;
      const int k0 = p.koff[n], k1 = p.koff[n + 1];
      const Real* il = invl + n * p.lp + p.loff;
      // KW bases per pass: 10 when the source's K is a multiple of 10 (the
      // BASELINE K = 10 / 20: no idle lanes), else 16; numerators at [0, KW),
      // denominators at [16, 16 + KW) of the 32 reduced values
      auto mub = [&](auto kw) {
        constexpr int KW = decltype(kw)::value;
        for (int kb = k0; kb < k1; kb += KW) {
          Real a[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) a[i] = Real(0);
          const Real* vrow[KW];
#pragma unroll
          for (int q = 0; q < KW; ++q) vrow[q] = Vg + (size_t)min(kb + q, k1 - 1) * T + tid;
#pragma unroll
          for (int k = 0; k < FT; ++k) {
            const int tau = tid + k * NT;
            const Real ilv = il[tau];
            const Real an = (EREG ? ereg[n - g0][EREG ? k : 0] : En[tau]) * (ilv * ilv);
            const Real bn = (tau < T) ? ilv * (Real)min(L, T - tau) : Real(0);
#pragma unroll
            for (int q = 0; q < KW; ++q) {
              const Real vv = __ldg(vrow[q] + k * NT);
              if constexpr (F32) {
                const float2 t = ffma2s(make_float2(an, bn), vv, make_float2(a[q], a[16 + q]));
                a[q] = t.x;
                a[16 + q] = t.y;
              } else {
                a[q] = fma(an, vv, a[q]);
                a[16 + q] = fma(bn, vv, a[16 + q]);
              }
            }
          }
          warp_reduce_scatter(a, lane);
          __syncthreads();  // previous pass's reads of red are done
          red[warp * 32 + lane] = a[0];
          __syncthreads();
          if (tid < KW && kb + tid < k1) {
            Real num = Real(0), den = Real(0);
            for (int w = 0; w < NW; ++w) {
              num += red[w * 32 + tid];
              den += red[w * 32 + 16 + tid];
            }
            const Real b = Bs[kb + tid];
            Bg[kb + tid] = fmax(b * sqrt(num / den), floor_abs);
          }
        }
      };
      if ((k1 - k0) % 10 == 0)
        mub(std::integral_constant<int, 10>{});
      else
        mub(std::integral_constant<int, 16>{});
    }
    __syncthreads();  // Pq / the halo is rewritten by the next group
  }
  CTF_PHASE(8);
  // check_all_finite (estimator.cpp:494-499): W' first (code 1), then Y
  // (code 2; a non-finite estimate makes its row's power sum non-finite)
  bool ybad = false, wbad = false;
#pragma unroll
  for (int i = 0; i < R; ++i) ybad |= !isfinite(rp[i]);
  for (int i = tid; i < R * D; i += NT) wbad |= !cfinite(Wf[i]);
  if (ybad || wbad) atomicOr(&s_bad, (wbad ? 2 : 0) | (ybad ? 1 : 0));
  // row powers (estimator.cpp:391-397)
  Real rr[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) rr[i] = i < R ? rp[i < R ? i : 0] : Real(0);
  warp_reduce_scatter(rr, lane);
  red[warp * 32 + lane] = rr[0];
  __syncthreads();
  if (s_bad) {
    if (tid == 0) record_err<Real>(p.err, mix, err_key(p.iteration, kPhFinite, gbin, 0, (s_bad & 2) ? 1 : 2));
    return;
  }
  if (tid < R) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += (double)red[w * 32 + tid];
    p.rowpow[tile * R + tid] = s;
  }
  if (tid == 0) {
    double dp = 1.0;  // prod_r (1 - z_r) in row order (determinant lemma)
    if (!IP)
      for (int r = 0; r < R; ++r) dp *= (double)fac_s[r];
    p.logdet[tile] = IP ? s_iplogdet : logdet + log(dp);
  }
  for (int i = tid; i < R * D; i += NT) Wg[i] = Wf[i];
  CTF_PHASE(9);
}

}  // namespace ctf
