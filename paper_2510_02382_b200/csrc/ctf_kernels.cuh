// ctf_kernels.cuh — sm_100a kernels for the ISS+NMF hot path of CTF-MNMF-ISS.
//
// One CTA per (mixture, frequency bin) runs the whole bin-local part of one
// iteration of proj/src/estimator.cpp:548-654:
//   prologue : rescale of the previous iteration (W rows /= mu_r, B /= mu0^2,
//              estimator.cpp:399-411), PSD refresh lambda = max(B V, floor)
//              (model.cpp:210-215), Y = W x~ (estimator.cpp:555), finite
//              check (:491-501) and the previous iteration's objective
//              contribution (:55-77) incl. log|det W| by pivoted LU (:41-53).
//   sweep    : R steps of iss_step (estimator.cpp:434-484): weighted
//              reductions over frames with warp reduce-scatter trees, the
//              steering vector z, rank-1 updates of Y (registers/smem) and W.
//   epilogue : Y = W' x~ (:607), delayed energies E (:321-332), row powers
//              (:391-397), and MU-B for this bin (:313-346).
// Frames are owned by threads (frame j = tid + k*NT), so every per-frame
// update is thread-private; the only cross-thread traffic is the 3R-value
// reduction per step, done as a warp reduce-scatter plus a fixed-order
// cross-warp sum (deterministic, run-to-run bit-identical).
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <type_traits>

namespace ctf {

constexpr int kMaxRows = 64;
constexpr int kMaxSources = 16;
constexpr unsigned kFull = 0xffffffffu;

template <typename Real> struct Cplx;
template <> struct Cplx<float> { using T = float2; };
template <> struct Cplx<double> { using T = double2; };

// Error keys: atomicMin over (iteration, phase, bin, row, code) reproduces the
// reference's "first failing iteration, phase in program order, lowest bin".
enum Phase : uint64_t { kPhSetup = 0, kPhSweep = 1, kPhFinite = 2, kPhDet = 3, kPhObj = 4, kPhImage = 5 };
__host__ __device__ inline unsigned long long err_key(uint64_t it, uint64_t ph, uint64_t bin, uint64_t row,
                                                      uint64_t code) {
  return (unsigned long long)((it << 44) | (ph << 40) | ((bin & 0xFFFFF) << 20) | ((row & 0xFFF) << 8) |
                              (code & 0xFF));
}
constexpr unsigned long long kNoErr = ~0ull;

struct SweepParams {
  const void* x;            // Real2 [mix][FL][T][Mx]
  void* W;                  // Real2 [mix][FL][D][R] (column-major R x D per bin)
  void* Bf;                 // Real  [mix][FL][SK]
  const void* V;            // Real  [mix][SK][T]
  void* E;                  // Real  [mix][N][FL][T]
  double* rowpow;           // [mix][FL][R]
  double* objbin;           // [mix][FL]
  const double* mu;         // [mix][R] pending rescale, or nullptr
  const double* logmu;      // [mix] sum_r log mu_r of the pending rescale
  const double* floor_abs;  // [mix]
  unsigned long long* err;  // [mix]
  int FL, bin_lo, T, TP, Mx, Ls, D, R, N, SK;
  int iteration;  // 1-based number of the iteration whose sweep runs (sweep errors)
  int do_sweep;   // 0: prologue only (finalize pass)
  int has_prev;   // prologue evaluates objective/finite checks of iteration-1
  int xoff, xp;   // x tile: Mx rows of xp = xoff + TP complex, x_m(t) at [m*xp + xoff + t]
  int loff, lp;   // 1/lambda: N rows of lp = loff + TP, at [n*lp + loff + tau]
  double* logdet;           // [mix][FL] log|det W| (pre-rescale after a sweep)
  int off_y, off_x, off_e, off_l, off_w, off_red, off_z, off_b, off_d;  // smem byte offsets
  int off_ip;  // IP-rule scratch of the frame-domain kernel (3 D x D + 2 D complex)
  int woff[kMaxRows];  // per row p: n_p*lp + loff - l_p (weight index base)
  int xcol[kMaxRows];  // per stacked channel c = m*Ls + l: m*xp + xoff - l (x tile offset)
  int srcr[kMaxRows];  // source of each row
  int row0[kMaxSources], ntaps[kMaxSources], koff[kMaxSources + 1];
  // CheckOptions instrumentation (estimator.hpp:45-48), CHECK variants only:
  // bit 0 det lemma, bit 1 row normalization; per mixture the running max of
  // each error as a double bit pattern (non-negative doubles order as u64)
  int chk_flags;
  unsigned long long* chk;  // [mix][2]
  int pf_stride;  // > 0: prefetch into L2 the tiles of work item (mix*FL + bin) + pf_stride
  // Conditioning fallback of the covariance-domain kernel (ctf_gram.cuh):
  // fb_mode 1 (gram_kernel): a bin whose weighted covariance is too
  // ill-conditioned for the Gram form in this precision (kappa estimate
  // sum_c |w_rc|^2 Q_r(c,c) / (w_r^H Q_r w_r) > fb_theta for some row) writes
  // nothing but appends its work item (mix*FL + bin) to fb_list;
  // fb_mode 2 (sweep_kernel, the frame-domain form): the CTAs run exactly the
  // listed items (grid-stride over *fb_count).
  int fb_mode;
  int* fb_list;
  int* fb_count;
  double fb_theta;
  // mixtures addressable from the (host-offset) buffers of this launch: a
  // mixture-chunk launch gets every per-mixture pointer offset to its first
  // mixture and indexes mixtures by blockIdx.y
  int nmix;
  // covariance-domain kernel: 1 / lambda and the objective's log term computed
  // ahead by lambda_kernel (nullptr: the kernel's own lambda phase)
  const void* invl_g;       // Real [mix][FL][N][T]
  const double* logsum_g;   // [mix][FL]
};

// L2 prefetch of a contiguous block (bulk async, no registers or smem).
__device__ __forceinline__ void prefetch_l2(const void* ptr, unsigned bytes) {
  // the bulk prefetch wants a 16-byte aligned address and size: start at the
  // aligned address below (a tile of an odd number of complex64 values, e.g.
  // W at R = D = 9, starts 8 bytes off on every other bin)
  const unsigned off = (unsigned)(reinterpret_cast<uintptr_t>(ptr) & 15u);
  ptr = reinterpret_cast<const unsigned char*>(ptr) - off;
  bytes = (bytes + off) & ~15u;
  if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr), "r"(bytes) : "memory");
}
// The CTAs resident after this one start roughly pf_stride work items later:
// warm L2 with the x tile and W of that item while this one runs.
__device__ __forceinline__ void prefetch_next_tile(const SweepParams& p, int bin, int mix, size_t xbytes,
                                                   size_t wbytes) {
  if (p.pf_stride <= 0 || threadIdx.x != 0) return;
  const size_t w = (size_t)mix * p.FL + bin + p.pf_stride;
  if (w >= (size_t)p.nmix * p.FL) return;
  prefetch_l2(reinterpret_cast<const unsigned char*>(p.x) + w * xbytes, (unsigned)xbytes);
  prefetch_l2(reinterpret_cast<const unsigned char*>(p.W) + w * wbytes, (unsigned)wbytes);
}

// ---------------------------------------------------------------------------
// Small complex helpers.
template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
  V r;
  r.x = fma(a.x, b.x, -a.y * b.y);
  r.y = fma(a.x, b.y, a.y * b.x);
  return r;
}
template <typename V> __device__ __forceinline__ void cmac(V& acc, V a, V b) {  // acc += a*b
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
template <typename V> __device__ __forceinline__ void cmsub(V& acc, V a, V b) {  // acc -= a*b
  acc.x = fma(-a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(-a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
// 1/x correctly rounded: the same value as the IEEE division 1/x, without
// its slow-path sequence (fp32: MUFU + Newton fixup); fp64 divides
__device__ __forceinline__ float rcp_rn(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double rcp_rn(double x) { return 1.0 / x; }
// 1/x for the MU-V weights: fp32 MUFU approximation + one Newton step (within
// ~1 ulp of rcp_rn, 3 instructions instead of its fixup sequence); fp64 exact.
__device__ __forceinline__ float rcp_fast(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return fmaf(r, fmaf(-x, r, 1.f), r);
}
__device__ __forceinline__ double rcp_fast(double x) { return 1.0 / x; }
// fp64 1/x for the MU-V weights (x = lambda' >= floor > 0, normal): the
// MUFU.RCP64H seed (2^-23) and two Newton steps, ~1 ulp, branch-free and half
// the dependent chain of the IEEE division (its correction steps and slow path)
#ifndef CTF_MUV_RCPNR
#define CTF_MUV_RCPNR 1
#endif
__device__ __forceinline__ double rcp_muv(double x) {
#if CTF_MUV_RCPNR
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
#else
  return 1.0 / x;
#endif
}
__device__ __forceinline__ float rcp_muv(float x) { return rcp_fast(x); }
template <typename V> __device__ __forceinline__ auto cnorm(V a) -> decltype(a.x) { return fma(a.x, a.x, a.y * a.y); }
template <typename V> __device__ __forceinline__ bool cfinite(V a) { return isfinite(a.x) && isfinite(a.y); }
template <typename Real> __device__ __forceinline__ typename Cplx<Real>::T czero() {
  typename Cplx<Real>::T z;
  z.x = Real(0);
  z.y = Real(0);
  return z;
}

// Packed FP32x2 (Blackwell FFMA2/FMUL2): two FP32 FMAs per issue slot; a
// broadcast scalar operand is free (SASS "R.F32"), a swizzled pair is not.
__device__ __forceinline__ unsigned long long pk2(float2 a) { return *reinterpret_cast<unsigned long long*>(&a); }
__device__ __forceinline__ float2 upk2(unsigned long long a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {  // a*b + c
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)), "l"(pk2(c)));
  return upk2(d);
}
__device__ __forceinline__ float2 ffma2s(float2 a, float b, float2 c) { return ffma2(a, make_float2(b, b), c); }
__device__ __forceinline__ float2 fmul2s(float2 a, float b) {
  unsigned long long d;
  const float2 bb = make_float2(b, b);
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(bb)));
  return upk2(d);
}

// Warp reduce-scatter of V values (V multiple of 32): afterwards lane L holds
// in v[0..V/32) the warp sums of the original indices [L*V/32, (L+1)*V/32).
// V-1 shuffles instead of 5*V for per-value butterflies.
template <int CNT, int OFF, typename Real, int V>
__device__ __forceinline__ void rs_level(Real (&v)[V], int lane) {
  if constexpr (OFF >= 1) {
    constexpr int H = CNT / 2;
    const bool upper = (lane & OFF) != 0;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const Real send = upper ? v[i] : v[i + H];
      const Real keep = upper ? v[i + H] : v[i];
      v[i] = keep + __shfl_xor_sync(kFull, send, OFF);
    }
    rs_level<H, OFF / 2>(v, lane);
  }
}
template <typename Real, int V>
__device__ __forceinline__ void warp_reduce_scatter(Real (&v)[V], int lane) {
  static_assert(V % 32 == 0, "pad the value count to a multiple of 32");
  rs_level<V, 16>(v, lane);
}

template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Block sum of NQ doubles, fixed order; result valid in every thread.
template <int NQ>
__device__ __forceinline__ void block_sum_d(double (&v)[NQ], double* dred, int lane, int warp, int nw) {
#pragma unroll
  for (int q = 0; q < NQ; ++q) v[q] = warp_sum(v[q]);
  __syncthreads();  // dred may still be read from a previous call
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NQ; ++q) dred[warp * NQ + q] = v[q];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += dred[w * NQ + q];
    v[q] = s;
  }
}

// log|det A| of an n x n column-major complex matrix by one warp, partial
// pivoting on |a| with the lowest row winning ties (estimator.cpp:41-53).
// Returns 0 ok, CTF kind 4 (zero pivot) or 5 (tiny det).
template <typename Real>
__device__ int warp_logdet(typename Cplx<Real>::T* A, int n, int lane, double& out, double* phase = nullptr) {
  using R2 = typename Cplx<Real>::T;
  double acc = 0.0, ph = 0.0;
  for (int c = 0; c < n; ++c) {
    Real best = Real(-1);
    int brow = n;
    for (int r = c + lane; r < n; r += 32) {
      const R2 a = A[c * n + r];
      const Real m = sqrt(cnorm(a));
      if (m > best) {
        best = m;
        brow = r;
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const Real ob = __shfl_xor_sync(kFull, best, o);
      const int orow = __shfl_xor_sync(kFull, brow, o);
      if (ob > best || (ob == best && orow < brow)) {
        best = ob;
        brow = orow;
      }
    }
    if (brow != c && brow < n) ph += 3.14159265358979323846;  // a row swap flips the sign
    if (brow != c && brow < n)
      for (int j = lane; j < n; j += 32) {
        const R2 t = A[j * n + c];
        A[j * n + c] = A[j * n + brow];
        A[j * n + brow] = t;
      }
    __syncwarp();
    const R2 pv = A[c * n + c];
    const double mag = sqrt((double)pv.x * pv.x + (double)pv.y * pv.y);
    if (!(mag > 0.0) || !isfinite(mag)) return 4;
    acc += log(mag);
    ph += atan2((double)pv.y, (double)pv.x);
    const Real inv = Real(1) / cnorm(pv);
    R2 pinv;
    pinv.x = pv.x * inv;
    pinv.y = -pv.y * inv;
    for (int r = c + 1 + lane; r < n; r += 32) {
      const R2 f = cmul(A[c * n + r], pinv);
      for (int j = c + 1; j < n; ++j) cmsub(A[j * n + r], f, A[j * n + c]);
    }
    __syncwarp();
  }
  out = acc;
  if (phase) *phase = ph;
  return acc < log(1e-300) ? 5 : 0;
}

// Det-lemma check of one ISS step (estimator.cpp:560-569): W' = W - z w_r^H
// must satisfy det W' = det W (1 - z_r). Returns |det W' - pred| / |det W'|
// from the log-magnitude/phase of both determinants (no overflow).
__device__ __forceinline__ double det_lemma_error(double lm_before, double ph_before, double lm_after,
                                                  double ph_after, double zr) {
  const double mag = exp(lm_before - lm_after) * (1.0 - zr);
  const double ang = ph_before - ph_after;
  const double re = 1.0 - mag * cos(ang), im = -mag * sin(ang);
  return sqrt(re * re + im * im);
}

__device__ __forceinline__ void chk_max(unsigned long long* slot, double e) {
  if (e >= 0.0) atomicMax(slot, (unsigned long long)__double_as_longlong(e));  // NaN is ignored (std::max)
}

// Y(k, p) accessor: rows p < RREG live in registers, the rest in shared memory.
template <typename R2, int FT, int RREG, int RS>
struct YTile {
  R2 reg[FT][RREG > 0 ? RREG : 1];
  R2* sm;  // RS rows x TP
  int tp;
  template <int P> __device__ __forceinline__ R2 get(int k, int j) const {
    if constexpr (P < RREG) return reg[k][P];
    else return sm[(P - RREG) * tp + j];
  }
  template <int P> __device__ __forceinline__ void set(int k, int j, R2 v) {
    if constexpr (P < RREG) reg[k][P] = v;
    else sm[(P - RREG) * tp + j] = v;
  }
  // runtime row selection (pivot of the current step)
  __device__ __forceinline__ R2 pick(int k, int j, int r) const {
    if (r >= RREG) return sm[(r - RREG) * tp + j];
    R2 out = reg[k][0];
#pragma unroll
    for (int q = 1; q < RREG; ++q)
      if (q == r) out = reg[k][q];
    return out;
  }
};

// Compile-time loop helper.
template <int I, int N, typename F> __device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, N>(f);
  }
}

// Y = W x~ for the thread's frames (estimator.cpp:304-311 with the stacked
// observation of BASELINE (a) built virtually from the x tile).
template <typename Real, int RMAX, int FT, int RREG, bool EXACT, typename Tile>
__device__ __forceinline__ void demix_tile(Tile& Y, const typename Cplx<Real>::T* xs,
                                           const typename Cplx<Real>::T* Ws, const SweepParams& p, int tid,
                                           int NT, const int R, const int D) {
  using R2 = typename Cplx<Real>::T;
  constexpr int RC = 4;
  static_for<0, (RMAX + RC - 1) / RC>([&](auto chunk) {
    constexpr int r0 = decltype(chunk)::value * RC;
    if (r0 < R) {
      R2 acc[FT][RC];
#pragma unroll
      for (int k = 0; k < FT; ++k)
#pragma unroll
        for (int i = 0; i < RC; ++i) acc[k][i] = czero<Real>();
#pragma unroll(EXACT ? RMAX : 1)
      for (int c = 0; c < D; ++c) {
        const R2* xrow = xs + p.xcol[c];  // stacked channel c = (m, l): x_m(t - l)
        R2 w[RC];
#pragma unroll
        for (int i = 0; i < RC; ++i) w[i] = (r0 + i < R) ? Ws[c * R + r0 + i] : czero<Real>();
#pragma unroll
        for (int k = 0; k < FT; ++k) {
          const R2 xv = xrow[tid + k * NT];
          if constexpr (std::is_same<Real, float>::value) {
            // w x = w.x (x.x, x.y) + w.y (-x.y, x.x)
            const float2 xn = make_float2(-xv.y, xv.x);
#pragma unroll
            for (int i = 0; i < RC; ++i) acc[k][i] = ffma2s(xn, w[i].y, ffma2s(xv, w[i].x, acc[k][i]));
          } else {
#pragma unroll
            for (int i = 0; i < RC; ++i) cmac(acc[k][i], w[i], xv);
          }
        }
      }
      static_for<0, RC>([&](auto ii) {
        constexpr int P = r0 + decltype(ii)::value;
        if constexpr (P < RMAX) {
          if (P < R) {
#pragma unroll
            for (int k = 0; k < FT; ++k) {
              const int j = tid + k * NT;
              Y.template set<P>(k, j, (j < p.T) ? acc[k][decltype(ii)::value] : czero<Real>());
            }
          }
        }
      });
    }
  });
}

template <typename Real>
__device__ __forceinline__ void record_err(unsigned long long* err, int mix, unsigned long long key) {
  atomicMin(err + mix, key);
}

// One row of the IP rule (estimator.cpp:103-273, ip_update): solve
// (W h) u = e_r by LU with partial pivoting (pivot-ratio singularity probe
// 1e-13 on |pivot|, i.e. 1e-26 on |pivot|^2 as ip_update_small; one retry
// with 1e-10 tr(h)/D diagonal loading), then W[r, :] = conj(u) / sqrt(u^H h u)
// with the unloaded h. W column-major R x D (R == D <= 32), h (cov) D x D,
// A scratch D x (D+1), sol D, all in shared memory. Called by one whole warp;
// returns 0, 1 (singular after loading) or 2 (nonpositive row power).
template <typename Real>
__device__ int ip_solve_row(typename Cplx<Real>::T* Wb, int R, int D, int r, const typename Cplx<Real>::T* cov,
                            typename Cplx<Real>::T* A, typename Cplx<Real>::T* sol, int lane) {
  using R2 = typename Cplx<Real>::T;
  auto attempt = [&](Real load) -> bool {
    // A = W (h + load I) = W h + load W, rhs e_r
    for (int e = lane; e < D * (D + 1); e += 32) {
      const int i = e % D, j = e / D;
      R2 acc;
      acc.x = acc.y = Real(0);
      if (j < D) {
        for (int k = 0; k < D; ++k) cmac(acc, Wb[i + k * R], cov[k + j * D]);
        acc.x += load * Wb[i + j * R].x;
        acc.y += load * Wb[i + j * R].y;
      } else {
        acc.x = (i == r) ? Real(1) : Real(0);
      }
      A[i + j * D] = acc;
    }
    __syncwarp();
    double minp = INFINITY, maxp = 0.0;
    for (int c = 0; c < D; ++c) {
      // pivot: largest |a| in column c at or below the diagonal, lowest row on ties
      Real best = Real(-1);
      int prow = D;
      if (lane >= c && lane < D) {
        const R2 v = A[lane + c * D];
        best = sqrt(cnorm(v));
        prow = lane;
      }
  #pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const Real ob = __shfl_xor_sync(kFull, best, o);
        const int orow = __shfl_xor_sync(kFull, prow, o);
        if (ob > best || (ob == best && orow < prow)) {
          best = ob;
          prow = orow;
        }
      }
      minp = fmin(minp, (double)best);
      maxp = fmax(maxp, (double)best);
      if (prow != c)
        for (int j = lane; j <= D; j += 32) {
          const R2 t = A[c + j * D];
          A[c + j * D] = A[prow + j * D];
          A[prow + j * D] = t;
        }
      __syncwarp();
      if (!(best > Real(0))) continue;
      const R2 piv = A[c + c * D];
      const Real ip2 = Real(1) / cnorm(piv);
      const int w = D - c;  // rows c+1..D-1 x columns c+1..D
      for (int e = lane; e < (w - 1) * w; e += 32) {
        const int rr = c + 1 + e % (w - 1), j = c + 1 + e / (w - 1);
        const R2 arc = A[rr + c * D];
        R2 f;  // a(r, c) / a(c, c)
        f.x = (arc.x * piv.x + arc.y * piv.y) * ip2;
        f.y = (arc.y * piv.x - arc.x * piv.y) * ip2;
        cmsub(A[rr + j * D], f, A[c + j * D]);
      }
      __syncwarp();
    }
    if (!(minp > 1e-13 * maxp)) return false;
    if (lane == 0)
      for (int rr = D - 1; rr >= 0; --rr) {
        R2 acc = A[rr + D * D];
        for (int j = rr + 1; j < D; ++j) cmsub(acc, A[rr + j * D], sol[j]);
        const R2 d = A[rr + rr * D];
        const Real id = Real(1) / cnorm(d);
        R2 q;
        q.x = (acc.x * d.x + acc.y * d.y) * id;
        q.y = (acc.y * d.x - acc.x * d.y) * id;
        sol[rr] = q;
      }
    __syncwarp();
    bool fin = true;
    if (lane < D) fin = cfinite(sol[lane]);
    return __all_sync(kFull, fin);
  };
  bool ok = attempt(Real(0));
  if (!ok) {
    Real tr = Real(0);
    for (int i = 0; i < D; ++i) tr += cov[i + i * D].x;
    ok = attempt(Real(1e-10) * tr / (Real)D);
  }
  int err = 0;
  if (!ok) {
    err = 1;  // singular system after diagonal loading
  } else {
    // scale against the unloaded covariance: norm2 = Re(u^H h u)
    Real part_n = Real(0);
    if (lane < D) {
      R2 wgt;
      wgt.x = wgt.y = Real(0);
      for (int j = 0; j < D; ++j) cmac(wgt, cov[lane + j * D], sol[j]);
      const R2 u = sol[lane];
      part_n = u.x * wgt.x + u.y * wgt.y;
    }
    for (int o = 16; o >= 1; o >>= 1) part_n += __shfl_xor_sync(kFull, part_n, o);
    if (!(part_n > Real(0)) || !isfinite(part_n)) {
      err = 2;  // nonpositive row power
    } else if (lane < D) {
      const Real sc = Real(1) / sqrt(part_n);
      const R2 u = sol[lane];
      R2 wv;
      wv.x = u.x * sc;
      wv.y = -u.y * sc;
      Wb[r + lane * R] = wv;
    }
  }
  return err;
}

// ---------------------------------------------------------------------------
// The fused per-bin iteration kernel.
//
// log|det W| is carried per bin in p.logdet instead of an LU per iteration:
// by the determinant lemma used in the reference's own checks
// (estimator.cpp:560-569, test_estimator.cpp:322-335) every ISS step
// multiplies det W by (1 - z_r) (real, > 0), and the rescale divides it by
// prod_r mu_r. The exact pivoted LU (estimator.cpp:41-53) runs whenever the
// state is set from outside (logdet_kernel below); its zero-pivot / 1e-300
// outcomes are carried as -inf / the value and raised at the next
// objective, as the reference raises them in objective_from_parts.
// NT: the exact CTA size (frame j = tid + k*NT folds into load immediates);
// the launch bound targets 128 registers/thread (2 x 256 or 4 x 128 CTAs per SM).
// fp64 tiles are shared-memory bound to one CTA per SM, so fp64 variants
// get the full register file instead.
template <typename Real> constexpr int sweep_min_blocks(int nt) {
  return std::is_same<Real, float>::value ? (nt <= 512 ? 512 / nt : 1) : (nt <= 256 ? 256 / nt : 1);
}
// LT > 0 (EXACT only): every source has LT taps, so row P is (P / LT, P % LT)
// at compile time and the ISS weights are addressed from one base pointer
// per source with immediate offsets.
// CHECK: CheckOptions instrumentation (exact recomputation of det W after
// every step by a warp LU, and of each updated row's weighted power).
// IPR: the IP rule (estimator.cpp:580-606) in place of the ISS steps, for any
// layout (pre-stacked or unequal taps; R == D): per row the weighted
// covariance from the x tile, a warp LU solve (ip_solve_row) and the
// frame-sum refinement, then Y = W' x~ recomputed for the epilogue.
template <typename Real, int RMAX, int FT, int RREG, int NT, bool EXACT, int LT, bool CHECK, bool IPR>
__device__ __forceinline__ void sweep_body(const SweepParams& p, const int bin, const int mix);

template <typename Real, int RMAX, int FT, int RREG, int NT, bool EXACT, int LT = 0, bool CHECK = false,
          bool IPR = false>
__global__ void __launch_bounds__(NT, sweep_min_blocks<Real>(NT)) sweep_kernel(const SweepParams p) {
  if (p.fb_mode != 2) {  // one work item per CTA: (bin, mixture) = (blockIdx.x, blockIdx.y)
    sweep_body<Real, RMAX, FT, RREG, NT, EXACT, LT, CHECK, IPR>(p, blockIdx.x, blockIdx.y);
    return;
  }
  // conditioning fallback of the covariance-domain kernel: the listed items
  const int cnt = *p.fb_count;
  for (int w = blockIdx.x; w < cnt; w += gridDim.x) {
    const int t = p.fb_list[w];
    __syncthreads();  // shared memory of the previous item
    sweep_body<Real, RMAX, FT, RREG, NT, EXACT, LT, CHECK, IPR>(p, t % p.FL, t / p.FL);
  }
}

template <typename Real, int RMAX, int FT, int RREG, int NT, bool EXACT, int LT, bool CHECK, bool IPR>
__device__ __forceinline__ void sweep_body(const SweepParams& p, const int bin, const int mix) {
  using R2 = typename Cplx<Real>::T;
  constexpr int RS = RMAX - RREG;
  constexpr int NV = 3 * RMAX;
  constexpr int VP = ((NV + 31) / 32) * 32;
  constexpr int VM = VP / 32;
  static_assert(RMAX <= 32, "one lane per steering coefficient");
  static_assert(!CHECK || NV < VP, "the normalization sum needs a spare reduction slot");
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT >> 5;
  const int gbin = p.bin_lo + bin;
  // EXACT: R == D == RMAX is a compile-time constant (no row guards).
  const int R = EXACT ? RMAX : p.R, D = EXACT ? RMAX : p.D;
  const int T = p.T, TP = p.TP, N = p.N, SK = p.SK;

  R2* Ysm = reinterpret_cast<R2*>(smem + p.off_y);
  R2* xs = reinterpret_cast<R2*>(smem + p.off_x);
  Real* Pq = reinterpret_cast<Real*>(smem + p.off_x);  // aliases xs after the last demix
  Real* Es = reinterpret_cast<Real*>(smem + p.off_e);  // aliases xs after the last demix
  Real* invl = reinterpret_cast<Real*>(smem + p.off_l);
  R2* Wb = reinterpret_cast<R2*>(smem + p.off_w);       // two R x D buffers (ping-pong)
  Real* red = reinterpret_cast<Real*>(smem + p.off_red);
  R2* zs = reinterpret_cast<R2*>(smem + p.off_z);
  Real* Bs = reinterpret_cast<Real*>(smem + p.off_b);
  double* dred = reinterpret_cast<double*>(smem + p.off_d);
  __shared__ int s_bad;
  __shared__ double s_logmu;

  const size_t tile = (size_t)mix * p.FL + bin;
  prefetch_next_tile(p, bin, mix, (size_t)T * p.Mx * sizeof(R2), (size_t)R * D * sizeof(R2));
  const R2* xg = reinterpret_cast<const R2*>(p.x) + tile * (size_t)T * p.Mx;
  R2* Wg = reinterpret_cast<R2*>(p.W) + tile * (size_t)R * D;
  Real* Bg = reinterpret_cast<Real*>(p.Bf) + tile * SK;
  const Real* Vg = reinterpret_cast<const Real*>(p.V) + (size_t)mix * SK * T;
  const Real floor_abs = (Real)p.floor_abs[mix];
  const int prev_it = p.iteration - 1;
  const double* mu = p.mu ? p.mu + (size_t)mix * R : nullptr;

  if (tid == 0) {
    s_bad = 0;
    s_logmu = mu ? p.logmu[mix] : 0.0;
  }
  // ---- prologue: x tile (transposed to [m][t]), W and B with the pending rescale
  for (int m = 0; m < p.Mx; ++m) {
    R2* row = xs + m * p.xp;
    for (int i = tid; i < p.xoff; i += NT) row[i] = czero<Real>();
    for (int t = T + tid; t < TP; t += NT) row[p.xoff + t] = czero<Real>();
  }
#pragma unroll
  for (int k = 0; k < FT; ++k) {
    const int t = tid + k * NT;
    if (t < T)
      for (int m = 0; m < p.Mx; ++m) xs[m * p.xp + p.xoff + t] = xg[(size_t)t * p.Mx + m];
  }
  for (int i = tid; i < R * D; i += NT) {
    R2 w = Wg[i];
    if (mu) {
      const double m = mu[i % R];
      if (m != 0.0) {
        w.x = (Real)((double)w.x / m);
        w.y = (Real)((double)w.y / m);
      }
    }
    Wb[i] = w;
    if (p.has_prev && !cfinite(w)) s_bad = 1;
  }
  for (int n = 0; n < N; ++n) {
    const double m0 = mu ? mu[p.row0[n]] : 0.0;
    for (int i = p.koff[n] + tid; i < p.koff[n + 1]; i += NT) {
      Real b = Bg[i];
      if (m0 != 0.0) b = (Real)fmax((double)b / (m0 * m0), (double)floor_abs);
      Bs[i] = b;
    }
  }
  __syncthreads();
  if (p.has_prev && s_bad) {  // check_all_finite on W (estimator.cpp:494-496)
    if (tid == 0) record_err<Real>(p.err, mix, err_key(prev_it, kPhFinite, gbin, 0, 1));
    return;
  }
  // ---- lambda = max(B V, floor) -> 1/lambda, and the log-lambda objective term
  double logsum = 0.0;
  for (int n = 0; n < N; ++n) {
    Real* il = invl + n * p.lp;
    for (int i = tid; i < p.loff; i += NT) il[i] = Real(0);
    const int k0 = p.koff[n], k1 = p.koff[n + 1], Ln = p.ntaps[n];
    Real lam[FT];
#pragma unroll
    for (int k = 0; k < FT; ++k) lam[k] = Real(0);
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
      Real v = Real(0);
      if (tau < T) {
        const Real l = fmax(lam[k], floor_abs);
        v = rcp_rn(l);
        if (p.has_prev) logsum += (double)min(Ln, T - tau) * (double)log(l);
      }
      il[p.loff + tau] = v;
    }
  }
  __syncthreads();

  YTile<R2, FT, RREG, RS> Y;
  Y.sm = Ysm;
  Y.tp = TP;
  demix_tile<Real, RMAX, FT, RREG, EXACT>(Y, xs, Wb, p, tid, NT, R, D);

  double logdet = p.logdet[tile] - s_logmu;
  if (p.has_prev) {
    // objective of the previous iteration (estimator.cpp:55-77) from
    // Y = W_resc x~, the log term above and -2T log|det W_resc|.
    // per-thread sums in Real (<= 4*RMAX terms); a non-finite estimate makes
    // sy (and quad) non-finite, which is the finite check of :497-499
    Real qf = Real(0), sy = Real(0);
    static_for<0, RMAX>([&](auto pp) {
      constexpr int P = decltype(pp)::value;
      if (P < R) {
#pragma unroll
        for (int k = 0; k < FT; ++k) {
          const int j = tid + k * NT;
          const R2 y = Y.template get<P>(k, j);
          sy += y.x + y.y;
          qf = fma(cnorm(y), invl[p.woff[P] + j], qf);
        }
      }
    });
    if (!isfinite(sy) || !isfinite(qf)) s_bad = 1;
    double quad = (double)qf;
    double v2[2] = {logsum, quad};
    block_sum_d<2>(v2, dred, lane, warp, NW);  // contains __syncthreads: s_bad visible after
    if (s_bad) {  // estimator.cpp:497-499
      if (tid == 0) record_err<Real>(p.err, mix, err_key(prev_it, kPhFinite, gbin, 0, 2));
      return;
    }
    const int det_status = isnan(logdet) || logdet == -INFINITY ? 4 : (logdet < log(1e-300) ? 5 : 0);
    if (det_status) {  // estimator.cpp:45-51
      if (tid == 0) record_err<Real>(p.err, mix, err_key(prev_it, kPhDet, gbin, 0, det_status));
      return;
    }
    if (tid == 0) p.objbin[tile] = v2[0] + v2[1] - 2.0 * (double)T * logdet;
  }

  if (!p.do_sweep) {  // finalize pass: write the rescaled state and stop
    for (int i = tid; i < R * D; i += NT) Wg[i] = Wb[i];
    for (int i = tid; i < SK; i += NT) Bg[i] = Bs[i];
    if (tid == 0) p.logdet[tile] = logdet;
    return;
  }

  double dprod = 1.0;  // prod_r (1 - z_r): det W' = det W prod_r (1 - z_r)
  double c_det = 0.0, c_norm = 0.0;  // CHECK maxima
  Real lastn = Real(0);  // CHECK: weighted power of the last updated row
  double ip_logdet = 0.0;  // IPR: exact log|det W'|
  if constexpr (IPR) {
    // ---- IP rule (estimator.cpp:580-606): per row r = (n, l) the weighted
    // covariance h = (Q + Q^H) / 2, Q = sum_{j>=l} x~(j) x~(j)^H / lambda_n(j-l)
    // / T (compute_weighted_covariance :89-101) from the x tile, the solve,
    // then w_r /= sqrt(sum_{j>=l} |w_r x~(j)|^2 / lambda_n(j-l) / T)
    // (steering_row_power, :596-602).
    static_assert(!CHECK, "CheckOptions with the IP rule run in the covariance-domain variants");
    R2* qm = reinterpret_cast<R2*>(smem + p.off_ip);  // D x D raw Q / T
    R2* cov = qm + D * D;                              // D x D h
    R2* A = cov + D * D;                               // D x (D+1)
    R2* sol = A + D * (D + 1);                         // D
    __shared__ int s_iperr;
    if (tid == 0) s_iperr = 0;
    for (int r = 0; r < R; ++r) {
      const Real* wr = invl + p.woff[r];  // weight of row r at frame j: wr[j] (zero for j < l)
      for (int e = tid; e < D * D; e += NT) {
        const int a = e % D, b = e / D;
        const R2* xa = xs + p.xcol[a];
        const R2* xb = xs + p.xcol[b];
        R2 v = czero<Real>();
        for (int j = 0; j < T; ++j) {
          const R2 u = xa[j], t = xb[j];
          const Real w = wr[j];
          v.x = fma(fma(u.x, t.x, u.y * t.y), w, v.x);
          v.y = fma(fma(u.y, t.x, -u.x * t.y), w, v.y);
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
      double pw = 0.0;
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        const int j = tid + k * NT;
        if (j < T) {
          R2 y = czero<Real>();
          for (int c = 0; c < D; ++c) cmac(y, Wb[r + c * R], xs[p.xcol[c] + j]);
          pw += (double)(cnorm(y) * wr[j]);
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
    if (warp == 0) {  // exact log|det W'| (no determinant lemma for IP)
      R2* Acp = qm;
      for (int i = lane; i < R * D; i += 32) Acp[i] = Wb[i];
      __syncwarp();
      double out = 0.0;
      const int st = warp_logdet<Real>(Acp, R, lane, out);
      if (lane == 0) dred[0] = st == 4 ? -INFINITY : out;
    }
    __syncthreads();
    ip_logdet = dred[0];
    __syncthreads();
    demix_tile<Real, RMAX, FT, RREG, EXACT>(Y, xs, Wb, p, tid, NT, R, D);  // Y = W' x~ (estimator.cpp:607)
  } else {
  // ---- ISS sweep (estimator.cpp:556-579): step r computes z from the
  // current Y, then Y -= z y_r and W -= z w_r. The pass of step r applies
  // step r-1's update and accumulates step r's sums in one sweep over Y.
  static_assert(LT == 0 || (EXACT && RMAX % LT == 0), "LT variants need an exact row count");
  constexpr int NSRC = LT > 0 ? RMAX / LT : 1;
  const Real* wsrc[NSRC];  // LT > 0: 1/lambda_n at this thread's frame 0
#pragma unroll
  for (int n = 0; n < NSRC; ++n) wsrc[n] = invl + n * p.lp + p.loff + tid;
  auto weight = [&](auto pp, int k, int j) -> Real {
    constexpr int P = decltype(pp)::value;
    if constexpr (LT > 0) return wsrc[P / LT][k * NT - (P % LT)];
    else return invl[p.woff[P] + j];
  };
  R2 pv[FT];
#pragma unroll
  for (int k = 0; k < FT; ++k) pv[k] = czero<Real>();
  if (lane < RMAX) zs[warp * RMAX + lane] = czero<Real>();  // pass 0 applies a zero update
  __syncwarp();
  // CHECK: det of the current W (log-magnitude, phase; warp 0), and the
  // running maxima of both errors (tid 0)
  double c_lm = 0.0, c_ph = 0.0;
  int c_ok = 0;
  R2* cscr = xs;  // the x tile is dead during the sweep
  auto check_det = [&](const R2* Wcur, double zr, bool compare) {
    if (warp == 0) {
      for (int i = lane; i < R * D; i += 32) cscr[i] = Wcur[i];
      __syncwarp();
      double lm, ph;
      const int st = warp_logdet<Real>(cscr, R, lane, lm, &ph);
      if (compare && c_ok && st != 4) c_det = fmax(c_det, det_lemma_error(c_lm, c_ph, lm, ph, zr));
      c_ok = st != 4;
      c_lm = lm;
      c_ph = ph;
    }
  };
  if constexpr (CHECK) {
    if (p.chk_flags & 1) {
      __syncthreads();  // every warp is past the demix (xs reads)
      check_det(Wb, 0.0, false);
    }
  }
  for (int r = 0; r < R; ++r) {
    Real acc[VP];
#pragma unroll
    for (int i = 0; i < VP; ++i) acc[i] = Real(0);
    const R2* zw = zs + warp * RMAX;
    if constexpr (std::is_same<Real, float>::value) {
      // Packed FP32x2 pass. Update of step r-1: y -= z pv, written as
      //   y + (-z.x) (pv.x, pv.y) + z.y (pv.y, -pv.x);
      // accumulation for step r with s = w (yr.x, yr.y):
      //   Q1 += s.x (y.x, y.y), Q2 += s.y (y.x, y.y), den += |yr|^2 w,
      //   numer = (Q1.x + Q2.y, Q1.y - Q2.x) = sum w y conj(yr).
      float2 yr[FT], pvn[FT];
      float ar2[FT];
      const float2 zr = zw[r];
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        const int j = tid + k * NT;
        pvn[k] = make_float2(pv[k].y, -pv[k].x);
        float2 y = Y.pick(k, j, r);
        y = ffma2s(pv[k], -zr.x, y);
        yr[k] = ffma2s(pvn[k], zr.y, y);
        ar2[k] = cnorm(yr[k]);
      }
      static_for<0, RMAX>([&](auto pp) {
        constexpr int P = decltype(pp)::value;
        if (P < R) {
          const float2 zp = zw[P];
          float2 q1 = make_float2(0.f, 0.f), q2 = make_float2(0.f, 0.f);
          float den = 0.f;
#pragma unroll
          for (int k = 0; k < FT; ++k) {
            const int j = tid + k * NT;
            float2 y = Y.template get<P>(k, j);
            y = ffma2s(pv[k], -zp.x, y);
            y = ffma2s(pvn[k], zp.y, y);
            Y.template set<P>(k, j, y);
            const float w = weight(pp, k, j);
            if constexpr (CHECK) {
              if (P == r - 1) acc[NV] = fmaf(cnorm(y), w, acc[NV]);
            }
            const float2 sw = fmul2s(yr[k], w);
            q1 = ffma2s(y, sw.x, q1);
            q2 = ffma2s(y, sw.y, q2);
            den = fmaf(ar2[k], w, den);
          }
          acc[P] = q1.x + q2.y;
          acc[RMAX + P] = q1.y - q2.x;
          acc[2 * RMAX + P] = den;
        }
      });
#pragma unroll
      for (int k = 0; k < FT; ++k) pv[k] = yr[k];
    } else {
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        const int j = tid + k * NT;
        R2 yr = Y.pick(k, j, r);
        cmsub(yr, zw[r], pv[k]);
        const Real ar2 = cnorm(yr);
        static_for<0, RMAX>([&](auto pp) {
          constexpr int P = decltype(pp)::value;
          if (P < R) {
            R2 y = Y.template get<P>(k, j);
            cmsub(y, zw[P], pv[k]);
            Y.template set<P>(k, j, y);
            const Real w = weight(pp, k, j);
            if constexpr (CHECK) {
              if (P == r - 1) acc[NV] = fma(cnorm(y), w, acc[NV]);
            }
            // numer_p += y_p conj(y_r) w ; denom_p += |y_r|^2 w
            const Real tr = fma(y.x, yr.x, y.y * yr.y);
            const Real ti = fma(y.y, yr.x, -y.x * yr.y);
            acc[P] = fma(tr, w, acc[P]);
            acc[RMAX + P] = fma(ti, w, acc[RMAX + P]);
            acc[2 * RMAX + P] = fma(ar2, w, acc[2 * RMAX + P]);
          }
        });
        pv[k] = yr;
      }
    }
    warp_reduce_scatter(acc, lane);
    Real* rb = red + (size_t)((r & 1) * NW + warp) * VP;
#pragma unroll
    for (int i = 0; i < VM; ++i) rb[lane * VM + i] = acc[i];
    __syncthreads();
    // every warp derives z redundantly (identical fixed-order sums)
    const Real* rs = red + (size_t)((r & 1) * NW) * VP;
    bool bad = false;
    R2 z = czero<Real>();
    Real nre = Real(0), nim = Real(0), den = Real(0);
    if constexpr (EXACT && 3 * RMAX <= 32) {
      // lane (q, p) = (lane / RMAX, lane % RMAX) sums quantity q of row p over
      // the warps (fixed order), then row p's lane gathers its three sums
      Real acc_q = Real(0);
      if (lane < 3 * RMAX) {
        const int q = lane / RMAX, pr = lane - q * RMAX;
#pragma unroll
        for (int w = 0; w < NW; ++w) acc_q += rs[w * VP + q * RMAX + pr];
      }
      nre = __shfl_sync(kFull, acc_q, lane < RMAX ? lane : 0);
      nim = __shfl_sync(kFull, acc_q, lane < RMAX ? RMAX + lane : 0);
      den = __shfl_sync(kFull, acc_q, lane < RMAX ? 2 * RMAX + lane : 0);
    } else if (lane < R) {
      for (int w = 0; w < NW; ++w) {
        nre += rs[w * VP + lane];
        nim += rs[w * VP + RMAX + lane];
        den += rs[w * VP + 2 * RMAX + lane];
      }
    }
    if (lane < R) {
      bad = !(den > Real(0)) || !isfinite(den);
      if (lane == r) {
        z.x = Real(1) - sqrt((Real)T / den);
      } else {
        z.x = nre / den;
        z.y = nim / den;
      }
      zs[warp * RMAX + lane] = z;
    }
    const unsigned badm = __ballot_sync(kFull, bad);
    if (badm) {  // estimator.cpp:451-454
      if (tid == 0)
        record_err<Real>(p.err, mix, err_key(p.iteration, kPhSweep, gbin, r, __ffs(badm) - 1));
      return;
    }
    const Real zr_real = __shfl_sync(kFull, z.x, r);
    dprod *= (double)(Real(1) - zr_real);
    if constexpr (CHECK) {
      if ((p.chk_flags & 2) && r > 0 && tid == 0) {  // steering_row_power of row r-1 (estimator.cpp:571-576)
        double q = 0.0;
        for (int w = 0; w < NW; ++w) q += (double)rs[w * VP + NV];
        c_norm = fmax(c_norm, fabs(q / T - 1.0));
      }
    }
    __syncwarp();
    // iss_apply, W -= z w_r (estimator.cpp:298-302), ping-pong buffers
    const R2* Wo = Wb + (r & 1) * R * D;
    R2* Wn = Wb + ((r + 1) & 1) * R * D;
    for (int e = tid; e < R * D; e += NT) {
      const int q = e % R, c = e / R;
      R2 w = Wo[e];
      cmsub(w, zw[q], Wo[c * R + r]);
      Wn[e] = w;
    }
    if constexpr (CHECK) {
      if (p.chk_flags & 1) {
        __syncthreads();  // W' complete
        check_det(Wn, (double)zr_real, true);
      }
    }
  }
  // ---- epilogue. The reference recomputes Y = W' x~ after the sweep
  // (estimator.cpp:607); here the last step's update is applied to the
  // running Y instead (same values up to rounding, one R x T pass instead of
  // an R x D x T product).
  {
    const R2* zw = zs + warp * RMAX;
#pragma unroll
    for (int k = 0; k < FT; ++k) {
      const int j = tid + k * NT;
      static_for<0, RMAX>([&](auto pp) {
        constexpr int P = decltype(pp)::value;
        if (P < R) {
          R2 y = Y.template get<P>(k, j);
          if constexpr (std::is_same<Real, float>::value) {
            const float2 zp = zw[P];
            y = ffma2s(pv[k], -zp.x, y);
            y = ffma2s(make_float2(pv[k].y, -pv[k].x), zp.y, y);
          } else {
            cmsub(y, zw[P], pv[k]);
          }
          Y.template set<P>(k, j, y);
          if constexpr (CHECK) {
            if (P == R - 1) lastn = fma(cnorm(y), weight(pp, k, j), lastn);
          }
        }
      });
    }
  }
  }
  __syncthreads();  // xs is dead: reuse the region for |y|^2 of register rows and E
  const R2* Wf = IPR ? Wb : Wb + (R & 1) * R * D;

  // row powers (estimator.cpp:391-397) and |y|^2 export
  {
    constexpr int RP = ((RMAX + 31) / 32) * 32;
    Real rp[RP];
#pragma unroll
    for (int i = 0; i < RP; ++i) rp[i] = Real(0);
    static_for<0, RMAX>([&](auto pp) {
      constexpr int P = decltype(pp)::value;
      if (P < R) {
#pragma unroll
        for (int k = 0; k < FT; ++k) {
          const int j = tid + k * NT;
          const Real q = cnorm(Y.template get<P>(k, j));
          rp[P] += q;
          if constexpr (P < RREG) Pq[P * TP + j] = q;
        }
      }
    });
    if constexpr (CHECK) rp[RP - 1] = lastn;  // RMAX < 32: a spare slot
    warp_reduce_scatter(rp, lane);
    Real* rb = red + (size_t)warp * VP;
#pragma unroll
    for (int i = 0; i < RP / 32; ++i) rb[lane * (RP / 32) + i] = rp[i];
  }
  __syncthreads();
  if (tid < R) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += (double)red[(size_t)w * VP + tid];
    p.rowpow[tile * R + tid] = s;
  }
  if constexpr (CHECK) {
    static_assert(!CHECK || RMAX < 32, "spare row-power slot");
    if (tid == 0) {
      if (p.chk_flags & 2) {
        double q = 0.0;
        for (int w = 0; w < NW; ++w) q += (double)red[(size_t)w * VP + 31];
        c_norm = fmax(c_norm, fabs(q / T - 1.0));
        chk_max(p.chk + (size_t)mix * 2 + 1, c_norm);
      }
      if (p.chk_flags & 1) chk_max(p.chk + (size_t)mix * 2, c_det);
    }
  }
  if (tid == 0) p.logdet[tile] = IPR ? ip_logdet : logdet + log(dprod);
  // delayed energies E_n(tau) = sum_{l<L_n, tau+l<T} |y_{row0+l}(tau+l)|^2
  Real* Eg = reinterpret_cast<Real*>(p.E);
  for (int n = 0; n < N; ++n) {
    const int r0 = p.row0[n], Ln = p.ntaps[n];
#pragma unroll
    for (int k = 0; k < FT; ++k) {
      const int tau = tid + k * NT;
      Real e = Real(0);
      for (int l = 0; l < Ln && tau + l < T; ++l) {
        const int row = r0 + l;
        e += (row < RREG) ? Pq[row * TP + tau + l] : cnorm(Ysm[(row - RREG) * TP + tau + l]);
      }
      Es[n * TP + tau] = e;
      if (tau < T) Eg[(((size_t)mix * N + n) * p.FL + bin) * T + tau] = e;
    }
  }
  for (int i = tid; i < R * D; i += NT) Wg[i] = Wf[i];
  __syncthreads();

  // ---- MU-B for this bin (estimator.cpp:313-346), 16 bases per pass:
  // a[q] numerator, a[16 + q] denominator of base kb + q
  for (int n = 0; n < N; ++n) {
    const int k0 = p.koff[n], k1 = p.koff[n + 1], Ln = p.ntaps[n];
    const Real* il = invl + n * p.lp + p.loff;
    for (int kb = k0; kb < k1; kb += 16) {
      Real a[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) a[i] = Real(0);
      // V rows past k1 are clamped to a valid row (their sums are never
      // written); frames past T read V's zero padding and meet an = bn = 0.
      const Real* vrow[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) vrow[q] = Vg + (size_t)min(kb + q, k1 - 1) * T + tid;
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        const int tau = tid + k * NT;
        const Real ilv = il[tau];
        const Real an = Es[n * TP + tau] * (ilv * ilv);
        const Real bn = (tau < T) ? ilv * (Real)min(Ln, T - tau) : Real(0);
        Real vv[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) vv[q] = __ldg(vrow[q] + k * NT);
        if constexpr (std::is_same<Real, float>::value) {
          const float2 ab = make_float2(an, bn);
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float2 t = ffma2s(ab, vv[q], make_float2(a[q], a[16 + q]));
            a[q] = t.x;
            a[16 + q] = t.y;
          }
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            a[q] = fma(an, vv[q], a[q]);
            a[16 + q] = fma(bn, vv[q], a[16 + q]);
          }
        }
      }
      warp_reduce_scatter(a, lane);
      Real* rb = red + (size_t)warp * VP;
      __syncthreads();  // previous pass's reads of red are done
      rb[lane] = a[0];
      __syncthreads();
      if (tid < 16 && kb + tid < k1) {
        Real num = Real(0), den = Real(0);
        for (int w = 0; w < NW; ++w) {
          num += red[(size_t)w * VP + tid];
          den += red[(size_t)w * VP + 16 + tid];
        }
        const Real b = Bs[kb + tid];
        Bg[kb + tid] = fmax(b * sqrt(num / den), floor_abs);
      }
    }
  }
}

// Exact log|det W| per bin by pivoted LU (estimator.cpp:41-53), one warp per
// bin; run when the state is set from outside. -inf marks a zero pivot.
template <typename Real>
__global__ void __launch_bounds__(32) logdet_kernel(const void* W, double* logdet, int R, int nbins) {
  using R2 = typename Cplx<Real>::T;
  extern __shared__ __align__(16) unsigned char smem[];
  R2* A = reinterpret_cast<R2*>(smem);
  const size_t b = blockIdx.x;
  if ((int)b >= nbins) return;
  const R2* Wg = reinterpret_cast<const R2*>(W) + b * (size_t)R * R;
  for (int i = threadIdx.x; i < R * R; i += 32) A[i] = Wg[i];
  __syncwarp();
  double out = 0.0;
  const int st = warp_logdet<Real>(A, R, threadIdx.x & 31, out);
  if (threadIdx.x == 0) logdet[b] = st == 4 ? -INFINITY : out;
}
// The objective's log term: MUFU-based in fp32 (abs. error ~1e-6, far inside
// the fp32 cost tolerance), exact in fp64.
__device__ __forceinline__ float log_fast(float x) { return __logf(x); }
__device__ __forceinline__ double log_fast(double x) { return log(x); }

// ---------------------------------------------------------------------------
// PSD of the next loop body, ahead of the covariance-domain kernel
// (compute_psd model.cpp:210-215 with the pending rescale of B,
// estimator.cpp:399-411): 1 / lambda_n(f, t) = 1 / max(sum_k B V, floor) for
// every (bin, source, frame) of the launch's mixtures, written per bin as one
// contiguous [N][T] block (the iteration kernel copies it with 16-byte loads
// next to its x tile instead of running K dependent V loads per frame), and
// the log term of the previous iteration's objective (estimator.cpp:55-77),
// sum_n sum_t min(L_n, T - t) log lambda_n(t) per bin. lambda is formed in the
// same fma order as everywhere else; the reciprocal is the MUFU seed with one
// (fp32) or two (fp64) Newton steps, ~1 ulp. fp64 takes one log per group
// of equally weighted frames: log prod(mantissas) + ln 2 sum(exponents).
struct LambdaParams {
  const void* Bf;           // Real [mix][FL][SK] (before the pending rescale)
  const void* V;            // Real [mix][SK][T]
  void* invl;               // Real [mix][FL][N][T]
  double* logsum;           // [mix][FL]
  const double* mu;         // [mix][R] pending rescale, or nullptr
  const double* floor_abs;  // [mix]
  int FL, T, N, SK, R, has_prev;
  int koff[kMaxSources + 1], ntaps[kMaxSources], row0[kMaxSources];
};

#ifndef CTF_LAM_RCPNR  // fp64: Newton reciprocal (rcp_muv, ~1 ulp) instead of the IEEE division:
#define CTF_LAM_RCPNR 1  // lambda_kernel 0.403 -> 0.377 ms in the stream on cfg1 (16 bins per CTA: 0.905, 4: 0.401)
#endif
#ifndef CTF_LAM_BINS
#define CTF_LAM_BINS 8
#endif
constexpr int kLambdaBins = CTF_LAM_BINS;  // bins per CTA (they share the V loads)
template <typename Real, int KMAX, int VEC>
__global__ void __launch_bounds__(256) lambda_kernel(const LambdaParams p) {
  constexpr int BB = kLambdaBins, NT = 256, KP = (KMAX + 3) / 4 * 4, PV = 16 / (int)sizeof(Real);
  constexpr bool F32 = std::is_same<Real, float>::value;
  static_assert(VEC == 1 || VEC == PV, "one 16-byte vector of frames per thread, or one frame");
  extern __shared__ __align__(16) unsigned char smem[];
  Real* Bs = reinterpret_cast<Real*>(smem);  // [BB][N][KP], zero-padded
  __shared__ double lred[NT / 32][BB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int mix = blockIdx.y, bin0 = blockIdx.x * BB, nb = min(BB, p.FL - bin0);
  const Real floor_abs = (Real)p.floor_abs[mix];
  const double* mu = p.mu ? p.mu + (size_t)mix * p.R : nullptr;
  const Real* Bg = reinterpret_cast<const Real*>(p.Bf) + ((size_t)mix * p.FL + bin0) * p.SK;
  for (int e = tid; e < BB * p.N * KP; e += NT) {
    const int q = e % KP, bn = e / KP, n = bn % p.N, b = bn / p.N;
    const int k = p.koff[n] + q;
    Real v = Real(0);
    if (b < nb && k < p.koff[n + 1]) {
      v = Bg[(size_t)b * p.SK + k];
      const double mb = mu ? mu[p.row0[n]] : 0.0;
      if (mb != 0.0) {  // estimator.cpp:405-406: silent row, no rescale
        if constexpr (F32) {
          const float im = (float)(1.0 / mb);
          v = fmaxf(v * (im * im), floor_abs);
        } else {
          v = fmax(v / (mb * mb), (double)floor_abs);
        }
      }
    }
    Bs[e] = v;
  }
  __syncthreads();
  double ls[BB];
#pragma unroll
  for (int b = 0; b < BB; ++b) ls[b] = 0.0;
  const Real* Vg = reinterpret_cast<const Real*>(p.V) + (size_t)mix * p.SK * p.T;
  Real* out = reinterpret_cast<Real*>(p.invl) + ((size_t)mix * p.FL + bin0) * p.N * p.T;
  for (int n = 0; n < p.N; ++n) {
    const int k0 = p.koff[n], K = p.koff[n + 1] - k0, Ln = p.ntaps[n];
    double prod[BB];
    int esum[BB];
#pragma unroll
    for (int b = 0; b < BB; ++b) {
      prod[b] = 1.0;
      esum[b] = 0;
    }
    int pass = 0;
    for (int t0 = tid * VEC; t0 < p.T; t0 += NT * VEC, ++pass) {
      Real v[KMAX][VEC];
      const Real* vbase = Vg + (size_t)k0 * p.T + t0;
      Real* o = out + (size_t)n * p.T + t0;  // bin b of the CTA: + b * N * T
      const size_t ostride = (size_t)p.N * p.T;
#pragma unroll
      for (int q = 0; q < KMAX; ++q) {
        if (q < K) {
          const Real* vr = vbase + (size_t)q * p.T;
          if constexpr (VEC == 1) {
            v[q][0] = __ldg(vr);
          } else {
            const float4 raw = __ldg(reinterpret_cast<const float4*>(vr));
            const Real* c = reinterpret_cast<const Real*>(&raw);
#pragma unroll
            for (int i = 0; i < VEC; ++i) v[q][i] = c[i];
          }
        } else {
#pragma unroll
          for (int i = 0; i < VEC; ++i) v[q][i] = Real(0);
        }
      }
      // every frame of the vector carries weight L_n and its log goes the
      // fast way (uniform per thread and pass; the last L_n - 1 frames do not)
      const bool full = t0 + VEC - 1 + Ln <= p.T;
      const int lmode = !p.has_prev ? 0 : full ? 1 : 2;
#pragma unroll
      for (int b = 0; b < BB; ++b) {
        if (b >= nb) continue;
        const float4* b4 = reinterpret_cast<const float4*>(Bs + (b * p.N + n) * KP);
        Real bq[KP];
#pragma unroll
        for (int j = 0; j < KP / PV; ++j) {
          const float4 raw = b4[j];
          const Real* c = reinterpret_cast<const Real*>(&raw);
#pragma unroll
          for (int i = 0; i < PV; ++i) bq[j * PV + i] = c[i];
        }
        Real lam[VEC];
#pragma unroll
        for (int i = 0; i < VEC; ++i) lam[i] = Real(0);
#pragma unroll
        for (int q = 0; q < KMAX; ++q)
#pragma unroll
          for (int i = 0; i < VEC; ++i) lam[i] = fma(bq[q], v[q][i], lam[i]);
        Real il[VEC];
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
          lam[i] = lam[i] > floor_abs ? lam[i] : floor_abs;  // = fmax (a NaN takes the floor)
          // fp32: MUFU + one Newton step (~1 ulp); fp64: MUFU.RCP64H + two Newton steps (~1 ulp)
          il[i] = CTF_LAM_RCPNR ? rcp_muv(lam[i]) : rcp_fast(lam[i]);
        }
        if (lmode == 1) {
          if constexpr (F32) {
            float fsum = 0.f;
#pragma unroll
            for (int i = 0; i < VEC; ++i) fsum += log_fast(lam[i]);
            ls[b] += (double)Ln * (double)fsum;
          } else {
#pragma unroll
            for (int i = 0; i < VEC; ++i) {
              const long long bits = __double_as_longlong(lam[i]);
              const int ex = (int)((bits >> 52) & 0x7ff);
              if (ex != 0 && ex != 0x7ff) {
                prod[b] *= __longlong_as_double((bits & 0x800fffffffffffffLL) | 0x3ff0000000000000LL);
                esum[b] += ex - 1023;
              } else {
                ls[b] += (double)Ln * log(lam[i]);
              }
            }
          }
        } else if (lmode == 2) {
#pragma unroll
          for (int i = 0; i < VEC; ++i)
            if (t0 + i < p.T) ls[b] += (double)min(Ln, p.T - t0 - i) * (double)log_fast(lam[i]);
        }
        if constexpr (VEC == 1) {
          o[(size_t)b * ostride] = il[0];
        } else {
          float4 raw;
          Real* c = reinterpret_cast<Real*>(&raw);
#pragma unroll
          for (int i = 0; i < VEC; ++i) c[i] = il[i];
          *reinterpret_cast<float4*>(o + (size_t)b * ostride) = raw;
        }
      }
      if (!F32 && (pass & 63) == 63) {  // keep the mantissa products far from overflow
#pragma unroll
        for (int b = 0; b < BB; ++b) {
          ls[b] += (double)Ln * (log(prod[b]) + (double)esum[b] * 0.693147180559945309417);
          prod[b] = 1.0;
          esum[b] = 0;
        }
      }
    }
    if (!F32 && p.has_prev) {
#pragma unroll
      for (int b = 0; b < BB; ++b)
        ls[b] += (double)Ln * (log(prod[b]) + (double)esum[b] * 0.693147180559945309417);
    }
  }
  if (!p.has_prev) return;
#pragma unroll
  for (int b = 0; b < BB; ++b) {
    const double s = warp_sum(ls[b]);
    if (lane == 0) lred[warp][b] = s;
  }
  __syncthreads();
  if (tid < nb) {
    double s = 0.0;
    for (int w = 0; w < NT / 32; ++w) s += lred[w][tid];
    p.logsum[(size_t)mix * p.FL + bin0 + tid] = s;
  }
}

// ---------------------------------------------------------------------------
// MU-B (estimator.cpp:313-346) outside the iteration kernel, for the kernels
// that run at one CTA per SM (the frame-split cluster kernel): there the
// K x T dependent V loads of the in-kernel MU-B passes are fully exposed (10 %
// of cfg3's kernel), while E and 1/lambda already sit in HBM (lambda ahead).
// One warp per (mixture, source, bin): the lanes stride over the frames (VEC
// consecutive frames per lane, 16-byte loads of E, 1/lambda and the V rows,
// which the warps of a CTA share through L1), KW bases per pass
// (numerators at [0, KW), denominators at [16, 16 + KW) of the 32 values of a
// warp reduce-scatter), then B <- max(B sqrt(num / den), floor) on the
// rescaled B the iteration kernel left in place.
struct MubParams {
  void* Bf;                 // Real [mix][FL][SK], rescaled, updated in place
  const void* V;            // Real [mix][SK][T]
  const void* E;            // Real [mix][N][FL][T]
  const void* invl;         // Real [mix][FL][N][T]
  const double* floor_abs;  // [mix]
  const unsigned long long* err;  // [mix] error words (all ones: none): a failed mixture is left alone
  int FL, T, N, SK;
  int koff[kMaxSources + 1], ntaps[kMaxSources];
};

#ifndef CTF_MUB_UNROLL  // frame-loop iterations in flight per lane
#define CTF_MUB_UNROLL 1  // (2 and 4 measured slower on cfg3: 37.31 / 37.51 vs 37.05 ms per 16 mixtures)
#endif
#ifndef CTF_MUB_MINB
#define CTF_MUB_MINB 2
#endif
template <typename Real, int VEC>
__global__ void __launch_bounds__(256, CTF_MUB_MINB) mub_kernel(const MubParams p) {
  constexpr int PV = 16 / (int)sizeof(Real), UNR = CTF_MUB_UNROLL;
  static_assert(VEC == 1 || VEC == PV, "one 16-byte vector of frames per lane, or one frame");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int bin = blockIdx.x * (blockDim.x >> 5) + warp, n = blockIdx.y, mix = blockIdx.z;
  if (bin >= p.FL || p.err[mix] != ~0ull) return;
  const int T = p.T, k0 = p.koff[n], k1 = p.koff[n + 1], Ln = p.ntaps[n];
  const Real floor_abs = (Real)p.floor_abs[mix];
  const Real* Eg = reinterpret_cast<const Real*>(p.E) + (((size_t)mix * p.N + n) * p.FL + bin) * T;
  const Real* Il = reinterpret_cast<const Real*>(p.invl) + (((size_t)mix * p.FL + bin) * p.N + n) * T;
  const Real* Vg = reinterpret_cast<const Real*>(p.V) + (size_t)mix * p.SK * T;
  Real* Bg = reinterpret_cast<Real*>(p.Bf) + ((size_t)mix * p.FL + bin) * p.SK;
  auto pass = [&](auto kw) {
    constexpr int KW = decltype(kw)::value;
    for (int kb = k0; kb < k1; kb += KW) {
      Real a[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) a[i] = Real(0);
#pragma unroll UNR
      for (int t0 = lane * VEC; t0 < T; t0 += 32 * VEC) {
        Real e[VEC], il[VEC];
        if constexpr (VEC == 1) {
          e[0] = __ldg(Eg + t0);
          il[0] = __ldg(Il + t0);
        } else {
          const float4 er = __ldg(reinterpret_cast<const float4*>(Eg + t0));
          const float4 ir = __ldg(reinterpret_cast<const float4*>(Il + t0));
#pragma unroll
          for (int i = 0; i < VEC; ++i) {
            e[i] = reinterpret_cast<const Real*>(&er)[i];
            il[i] = reinterpret_cast<const Real*>(&ir)[i];
          }
        }
        Real an[VEC], bn[VEC];
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
          an[i] = e[i] * (il[i] * il[i]);
          bn[i] = il[i] * (Real)min(Ln, T - t0 - i);
        }
#pragma unroll
        for (int q = 0; q < KW; ++q) {
          const Real* vr = Vg + (size_t)min(kb + q, k1 - 1) * T + t0;
          Real v[VEC];
          if constexpr (VEC == 1) {
            v[0] = __ldg(vr);
          } else {
            const float4 raw = __ldg(reinterpret_cast<const float4*>(vr));
#pragma unroll
            for (int i = 0; i < VEC; ++i) v[i] = reinterpret_cast<const Real*>(&raw)[i];
          }
#pragma unroll
          for (int i = 0; i < VEC; ++i) {
            a[q] = fma(an[i], v[i], a[q]);
            a[16 + q] = fma(bn[i], v[i], a[16 + q]);
          }
        }
      }
      warp_reduce_scatter(a, lane);  // lane i holds the warp's sum of value i
      const Real den = __shfl_sync(kFull, a[0], (lane + 16) & 31);
      if (lane < KW && kb + lane < k1) {
        const Real b = Bg[kb + lane];
        Bg[kb + lane] = fmax(b * (Real)sqrt((double)a[0] / (double)den), floor_abs);
      }
    }
  };
  if ((k1 - k0) % 10 == 0)
    pass(std::integral_constant<int, 10>{});
  else
    pass(std::integral_constant<int, 16>{});
}

// ---------------------------------------------------------------------------
// MU-V (estimator.cpp:348-382): partial numerator/denominator over a chunk
// of this rank's bins, for one source and a tile of frames. lambda' is
// recomputed with the updated bases; all taps contribute (:356-368).
struct MuvParams {
  const void* Bf;  // Real [mix][FL][SK]
  const void* V;   // Real [mix][SK][T]
  const void* E;   // Real [mix][N][FL][T]
  void* part;      // Real [chunk][mix][2][SK][T]
  const double* floor_abs;
  int FL, T, N, SK, nmix, chunk_bins;
  int mix0;  // mixture of blockIdx.y / N == 0
  int koff[kMaxSources + 1], ntaps[kMaxSources];
};

// Bins are processed in groups of 8 with no per-bin guards (the B chunk is
// zero-padded to whole groups; a padded bin has b = 0 and E = 0, so it adds
// exactly 0), which lets the lambda' FMA chains of different bins overlap;
// fp32 computes lambda' for two bins per FFMA2. KS = 2 splits a frame's K
// bases over the two half-warps (lanes l and l ^ 16 share the frame): each
// forms lambda' over its half and the halves are exchanged by one shuffle
// (the sum is the same on both lanes), halving the v / num / den registers.
// fp64 with K <= 10 (BASELINE cfg0 / cfg1): registers capped for four CTAs per
// SM (128; a few spilled values) and the Newton reciprocal. Measured on cfg1
// (ms per iteration, tools/muv_ab.sh): IEEE division at 1 / 3 / 4 CTAs per SM
// 0.413 / 0.384 / 0.446, Newton 0.561 / 0.404 / 0.368 (five CTAs: 1.1, spills).
#ifndef CTF_MUV_MINB64
#define CTF_MUV_MINB64 4
#endif
// (the other variants: no occupancy target below K = 16, one CTA from there: fp32
// cfg1 0.218 vs 0.244 ms with the explicit 1, cfg2 1.104 vs 1.136 ms per 32 mixtures)
template <typename Real, int KMAX> constexpr bool muv_tight() { return sizeof(Real) == 8 && KMAX <= 10; }
// fp32, K < 16 (cfg0 / cfg1), measured on cfg1 (MU ms per iteration, tools/muv_ab.sh): unguarded
// clamped E loads + MUFU reciprocal + registers capped for four CTAs per SM 0.189; without
// the clamp 0.291, with the exact reciprocal 0.257, without the cap (134 registers) 0.320;
// all three off (the previous kernel, 108 registers) 0.217. fp64: 0.367 -> 0.363.
#ifndef CTF_MUV_G64  // fp64, K <= 10: bins per E prefetch group
#define CTF_MUV_G64 4  // (cfg1 MU 0.355 vs 0.363 ms at 8; no spills)
#endif
#ifndef CTF_MUV_MINB32  // fp32, K < 16: resident CTAs per SM the register allocation aims at (0: none)
#define CTF_MUV_MINB32 4
#endif
#ifndef CTF_MUV_ECLAMP
#define CTF_MUV_ECLAMP 1
#endif
#ifndef CTF_MUV_RCPF32
#define CTF_MUV_RCPF32 1
#endif
template <typename Real, int KMAX, int KS = 1>
__global__ void __launch_bounds__(128, muv_tight<Real, KMAX>() ? CTF_MUV_MINB64 : KMAX >= 16 ? 1 : CTF_MUV_MINB32) muv_partial_kernel(const MuvParams p) {
  constexpr int G = muv_tight<Real, KMAX>() ? CTF_MUV_G64 : 8;  // bins per E prefetch group
  constexpr int KPT = KMAX / KS;  // bases per thread
  static_assert(KS == 1 || (KS == 2 && KMAX % 2 == 0), "k split");
  const int lane = threadIdx.x & 31, half = KS == 2 ? lane >> 4 : 0;
  const int tau = KS == 2 ? blockIdx.x * 64 + (threadIdx.x >> 5) * 16 + (lane & 15) : blockIdx.x * blockDim.x + threadIdx.x;
  const int mix = blockIdx.y / p.N + p.mix0, n = blockIdx.y % p.N;
  const int chunk = blockIdx.z;
  const int i0 = chunk * p.chunk_bins, i1 = min(p.FL, i0 + p.chunk_bins);
  const int nb = i1 - i0, nbp = (nb + G - 1) / G * G;
  const int k0 = p.koff[n], K = p.koff[n + 1] - k0;
  const int kb0 = half * KPT;  // this thread's first base (within the source)
  extern __shared__ __align__(16) unsigned char smem[];
  Real* Bsh = reinterpret_cast<Real*>(smem);  // [k][bin] (bins padded to nbp)
  const Real* Bg = reinterpret_cast<const Real*>(p.Bf) + (size_t)mix * p.FL * p.SK;
  // (a warp per bin reading its K consecutive bases measured slower: cfg1 MU 0.238 vs 0.189 ms fp32)
  for (int e = threadIdx.x; e < KMAX * nbp; e += blockDim.x) {
    const int k = e / nbp, i = e - k * nbp;
    Bsh[e] = (k < K && i < nb) ? Bg[(size_t)(i0 + i) * p.SK + k0 + k] : Real(0);
  }
  __syncthreads();
  const bool valid = tau < p.T;
  if (KS == 1 && !valid) return;
  const int tc = valid ? tau : 0;  // (KS = 2: lanes past T join the shuffles with zero data)
  const Real floor_abs = (Real)p.floor_abs[mix];
  const Real cnt = (Real)min(p.ntaps[n], p.T - tc);
  const Real* Vg = reinterpret_cast<const Real*>(p.V) + ((size_t)mix * p.SK + k0 + kb0) * p.T + tc;
  Real v[KPT], num[KPT], den[KPT];
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    v[k] = (valid && kb0 + k < K) ? Vg[(size_t)k * p.T] : Real(0);
    num[k] = Real(0);
    den[k] = Real(0);
  }
  const Real* Eg = reinterpret_cast<const Real*>(p.E) + (((size_t)mix * p.N + n) * p.FL) * p.T + tc;
  const Real* Bk = Bsh + kb0 * nbp;
  Real ecur[G], enext[G];
  // K < 16: unguarded loads: bins past the chunk re-read its last bin (their B
  // row is zero, so they add exactly 0); a lane past T reads frame 0 and stores
  // nothing. (K = 20 measured slower that way: cfg2 MU 1.138 vs 1.105 ms.)
  constexpr bool ECL = CTF_MUV_ECLAMP && KMAX < 16;
  const Real* Ec = Eg + (size_t)i0 * p.T;
  const int lastb = nb - 1;
#pragma unroll
  for (int u = 0; u < G; ++u) {
    if constexpr (ECL) ecur[u] = __ldg(Ec + (size_t)min(u, lastb) * p.T);
    else ecur[u] = (valid && u < nb) ? Eg[(size_t)(i0 + u) * p.T] : Real(0);
  }
  for (int g = 0; g < nbp; g += G) {
#pragma unroll
    for (int u = 0; u < G; ++u) {
      if constexpr (ECL) enext[u] = __ldg(Ec + (size_t)min(g + G + u, lastb) * p.T);
      else enext[u] = (valid && g + G + u < nb) ? Eg[(size_t)(i0 + g + G + u) * p.T] : Real(0);
    }
#pragma unroll
    for (int u = 0; u < G; u += 2) {
      // keep the B reads of one bin pair from being hoisted across the group
      // (they would cost KMAX*G registers and the occupancy)
      asm volatile("" ::: "memory");
      const int i = g + u;
      Real la, lb;
      if constexpr (std::is_same<Real, float>::value) {
        float2 l2 = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < KPT; ++k) l2 = ffma2s(*reinterpret_cast<const float2*>(Bk + k * nbp + i), v[k], l2);
        la = l2.x;
        lb = l2.y;
      } else {
        la = lb = Real(0);
#pragma unroll
        for (int k = 0; k < KPT; ++k) {
          la = fma(Bk[k * nbp + i], v[k], la);
          lb = fma(Bk[k * nbp + i + 1], v[k], lb);
        }
      }
      if constexpr (KS == 2) {
        la += __shfl_xor_sync(kFull, la, 16);
        lb += __shfl_xor_sync(kFull, lb, 16);
      }
      // (fp32: the MUFU form measured faster at K = 20, slower at K = 10)
      constexpr bool NR = muv_tight<Real, KMAX>() || (sizeof(Real) == 4 && (CTF_MUV_RCPF32 || KMAX >= 16));
      const Real ila = NR ? rcp_muv(fmax(la, floor_abs)) : rcp_rn(fmax(la, floor_abs));
      const Real ilb = NR ? rcp_muv(fmax(lb, floor_abs)) : rcp_rn(fmax(lb, floor_abs));
      const Real ana = ecur[u] * (ila * ila), bna = ila * cnt;
      const Real anb = ecur[u + 1] * (ilb * ilb), bnb = ilb * cnt;
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        const Real ba = Bk[k * nbp + i], bb = Bk[k * nbp + i + 1];
        if constexpr (std::is_same<Real, float>::value) {
          float2 t = ffma2s(make_float2(ana, bna), ba, make_float2(num[k], den[k]));
          t = ffma2s(make_float2(anb, bnb), bb, t);
          num[k] = t.x;
          den[k] = t.y;
        } else {
          num[k] = fma(ba, ana, num[k]);
          den[k] = fma(ba, bna, den[k]);
          num[k] = fma(bb, anb, num[k]);
          den[k] = fma(bb, bnb, den[k]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < G; ++u) ecur[u] = enext[u];
  }
  if (!valid) return;
  Real* out = reinterpret_cast<Real*>(p.part) + (((size_t)chunk * p.nmix + mix) * 2 * p.SK + k0 + kb0) * p.T + tau;
#pragma unroll
  for (int k = 0; k < KPT; ++k)
    if (kb0 + k < K) {
      out[(size_t)k * p.T] = num[k];
      out[(size_t)(p.SK + k) * p.T] = den[k];
    }
}

// Sum of the chunk partials in fixed order, then either the packed buffer
// for the all-reduce (world > 1) or directly the V update (world == 1).
struct ApplyParams {
  const void* part;     // Real [nchunk][mix][2][SK][T]
  void* packed;         // Real [mix][2][SK][T] (all-reduce buffer)
  void* V;              // Real [mix][SK][T]
  const double* rowpow; // [mix][FL][R]
  const double* objbin; // [mix][FL]
  double* packed_d;     // [mix][R + 1]
  double* mu;           // [mix][R]
  double* logmu;        // [mix] sum_r log mu_r over mu_r != 0 (the log|det| shift of the rescale)
  double* objective;    // [mix][max_iters]
  const double* floor_abs;
  unsigned long long* err;
  int nchunk, nmix, SK, T, FL, R, F_total, max_iters;
  int mix0;             // mixture of blockIdx.y == 0 (mixture-chunk launches)
  int obj_slot;         // iteration index (0-based) whose objective is summed, -1 if none
  int mode;             // 0 = reduce to packed, 1 = apply from packed, 2 = reduce+apply (world 1)
  int do_v;             // 0 for the objective-only finalize pass
};

template <typename Real>
__global__ void __launch_bounds__(256) reduce_apply_kernel(const ApplyParams p) {
  const int mix = blockIdx.y + p.mix0;
  const size_t plane = (size_t)p.SK * p.T;
  if (p.do_v) {
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < plane; e += (size_t)gridDim.x * blockDim.x) {
      Real num, den;
      if (p.mode == 1) {
        const Real* pk = reinterpret_cast<const Real*>(p.packed) + (size_t)mix * 2 * plane;
        num = pk[e];
        den = pk[plane + e];
      } else {
        const Real* pt = reinterpret_cast<const Real*>(p.part);
        num = Real(0);
        den = Real(0);
        for (int c = 0; c < p.nchunk; ++c) {
          const Real* q = pt + ((size_t)c * p.nmix + mix) * 2 * plane;
          num += q[e];
          den += q[plane + e];
        }
        if (p.mode == 0) {
          Real* pk = reinterpret_cast<Real*>(p.packed) + (size_t)mix * 2 * plane;
          pk[e] = num;
          pk[plane + e] = den;
          continue;
        }
      }
      Real* V = reinterpret_cast<Real*>(p.V) + (size_t)mix * plane;
      V[e] = fmax(V[e] * sqrt(num / den), (Real)p.floor_abs[mix]);
    }
  }
  if (blockIdx.x != 0) return;
  // row powers -> mu (estimator.cpp:391-397) and the objective sum
  double* pd = p.packed_d + (size_t)mix * (p.R + 1);
  if (p.mode != 1) {
    // R+1 sums over this rank's bins: each warp takes quantities, lanes take
    // strided bins, then a fixed butterfly (deterministic order).
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int r = warp; r <= p.R; r += nw) {
      double s = 0.0;
      if (r < p.R) {
        for (int i = lane; i < p.FL; i += 32) s += p.rowpow[((size_t)mix * p.FL + i) * p.R + r];
      } else if (p.obj_slot >= 0) {
        for (int i = lane; i < p.FL; i += 32) s += p.objbin[(size_t)mix * p.FL + i];
      }
      s = warp_sum(s);
      if (lane == 0) pd[r] = s;
    }
    if (p.mode == 0) return;
    __syncthreads();
  }
  for (int r = threadIdx.x; r <= p.R; r += blockDim.x) {
    if (r < p.R) {
      if (p.do_v) p.mu[(size_t)mix * p.R + r] = sqrt(pd[r] / ((double)p.F_total * p.T));
    } else if (p.obj_slot >= 0) {
      const double obj = pd[r];
      p.objective[(size_t)mix * p.max_iters + p.obj_slot] = obj;
      if (!isfinite(obj)) atomicMin(p.err + mix, err_key(p.obj_slot + 1, kPhObj, 0, 0, 6));
    }
  }
  if (p.do_v && p.logmu) {  // once per mixture instead of in every bin's prologue
    __syncthreads();
    if (threadIdx.x == 0) {
      double lm = 0.0;
      for (int r = 0; r < p.R; ++r) {
        const double m = p.mu[(size_t)mix * p.R + r];
        if (m != 0.0) lm += log(m);
      }
      p.logmu[mix] = lm;
    }
  }
}

// Mean power of the stacked observation (model.cpp:153-161, counted over
// x~ incl. its zero pads): per (mixture, bin) partial sums.
template <typename Real>
__global__ void __launch_bounds__(256) mean_power_kernel(const void* x, double* part, int FL, int T, int Mx,
                                                         int Ls) {
  using R2 = typename Cplx<Real>::T;
  const int bin = blockIdx.x, mix = blockIdx.y;
  const R2* xg = reinterpret_cast<const R2*>(x) + ((size_t)mix * FL + bin) * (size_t)T * Mx;
  double s = 0.0;
  for (int e = threadIdx.x; e < T * Mx; e += blockDim.x) {
    const int t = e / Mx;
    s += (double)min(Ls, T - t) * ((double)xg[e].x * xg[e].x + (double)xg[e].y * xg[e].y);
  }
  __shared__ double sh[32];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    part[(size_t)mix * FL + bin] = t;
  }
}

// ---------------------------------------------------------------------------
// Projection-back (proj/src/wiener.cpp:11-49, collapsed Wiener form):
// H = W^-1 by Gauss-Jordan with partial pivoting (one warp, lowest row wins
// ties), y = W x~, c_n(d, j) = sum_{l<L_n} H(d, r0_n + l) y_{r0_n + l}(j).
struct ImageParams {
  const void* x;     // Real2 [mix][FL][T][Mx]
  const void* W;     // Real2 [mix][FL][D][R]
  double* out;       // double2 [n][mix][FL][T][Dout]
  unsigned long long* err;
  int FL, bin_lo, T, Mx, Ls, D, R, N, nmix, current_only;
  int stage_x;  // 1: the x tile is staged in shared memory; 0: read from global (tiles over 227 KB)
  int row0[kMaxSources], ntaps[kMaxSources];
};

template <typename Real>
__global__ void __launch_bounds__(256) image_kernel(const ImageParams p) {
  using R2 = typename Cplx<Real>::T;
  extern __shared__ __align__(16) unsigned char smem[];
  const int bin = blockIdx.x, mix = blockIdx.y, tid = threadIdx.x, lane = tid & 31;
  const int R = p.R, D = p.D, T = p.T;
  const int xoff = p.Ls - 1, xp = xoff + T;
  R2* A = reinterpret_cast<R2*>(smem);          // R x R
  R2* H = A + R * R;                            // R x R
  R2* Wsm = H + R * R;                          // R x D
  R2* xs = Wsm + R * D;                         // Mx x xp
  __shared__ int s_bad;
  const size_t tile = (size_t)mix * p.FL + bin;
  const R2* xg = reinterpret_cast<const R2*>(p.x) + tile * (size_t)T * p.Mx;
  const R2* Wg = reinterpret_cast<const R2*>(p.W) + tile * (size_t)R * D;
  if (tid == 0) s_bad = 0;
  for (int i = tid; i < R * D; i += blockDim.x) {
    Wsm[i] = Wg[i];
    A[i] = Wg[i];
    const int r = i % R, c = i / R;
    H[i] = czero<Real>();
    if (r == c) H[i].x = Real(1);
  }
  if (p.stage_x) {
    for (int i = tid; i < p.Mx * xp; i += blockDim.x) {
      const int m = i / xp, t = i - m * xp - xoff;
      if (t < 0) xs[i] = czero<Real>();
    }
    for (int e = tid; e < T * p.Mx; e += blockDim.x) {
      const int t = e / p.Mx, m = e - t * p.Mx;
      xs[m * xp + xoff + t] = xg[e];
    }
  }
  __syncthreads();
  if (tid < 32) {
    for (int c = 0; c < R; ++c) {
      Real best = Real(-1);
      int brow = R;
      for (int r = c + lane; r < R; r += 32) {
        const Real m = sqrt(cnorm(A[c * R + r]));
        if (m > best) { best = m; brow = r; }
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const Real ob = __shfl_xor_sync(kFull, best, o);
        const int orow = __shfl_xor_sync(kFull, brow, o);
        if (ob > best || (ob == best && orow < brow)) { best = ob; brow = orow; }
      }
      if (brow != c && brow < R)
        for (int j = lane; j < R; j += 32) {
          R2 t = A[j * R + c]; A[j * R + c] = A[j * R + brow]; A[j * R + brow] = t;
          t = H[j * R + c]; H[j * R + c] = H[j * R + brow]; H[j * R + brow] = t;
        }
      __syncwarp();
      const R2 pv = A[c * R + c];
      const Real nn = cnorm(pv);
      R2 pinv; pinv.x = pv.x / nn; pinv.y = -pv.y / nn;
      R2 f[2];
      for (int q = 0; q < 2; ++q) {
        const int r = lane + 32 * q;
        f[q] = (r < R && r != c) ? cmul(A[c * R + r], pinv) : czero<Real>();
      }
      __syncwarp();
      for (int q = 0; q < 2; ++q) {
        const int r = lane + 32 * q;
        if (r < R && r != c)
          for (int j = 0; j < R; ++j) {
            // columns < c are already eliminated in the pivot row (zero) and
            // column c itself is never read again: update j > c only
            if (j > c) cmsub(A[j * R + r], f[q], A[j * R + c]);
            cmsub(H[j * R + r], f[q], H[j * R + c]);
          }
      }
      __syncwarp();
    }
    for (int r = lane; r < R; r += 32) {
      const R2 pv = A[r * R + r];
      const Real nn = cnorm(pv);
      R2 pinv; pinv.x = pv.x / nn; pinv.y = -pv.y / nn;
      for (int j = 0; j < R; ++j) {
        const R2 h = cmul(H[j * R + r], pinv);
        H[j * R + r] = h;
        if (!cfinite(h)) s_bad = 1;
      }
    }
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) atomicMin(p.err + mix, err_key(0, kPhImage, p.bin_lo + bin, 0, 9));
    return;
  }
  const int Dout = p.current_only ? p.Mx : D;
  for (int j = tid; j < T; j += blockDim.x) {
    R2 y[kMaxRows];
    for (int r = 0; r < R; ++r) {
      R2 acc = czero<Real>();
      for (int c = 0; c < D; ++c) {
        const int m = c / p.Ls, l = c - m * p.Ls;
        R2 xv;
        if (p.stage_x) xv = xs[m * xp + xoff + j - l];
        else xv = j >= l ? xg[(size_t)(j - l) * p.Mx + m] : czero<Real>();
        cmac(acc, Wsm[c * R + r], xv);
      }
      y[r] = acc;
    }
    for (int n = 0; n < p.N; ++n) {
      double2* o = reinterpret_cast<double2*>(p.out) +
                   ((((size_t)n * p.nmix + mix) * p.FL + bin) * T + j) * Dout;
      for (int od = 0; od < Dout; ++od) {
        const int d = p.current_only ? od * p.Ls : od;
        R2 acc = czero<Real>();
        for (int l = 0; l < p.ntaps[n]; ++l) cmac(acc, H[(p.row0[n] + l) * R + d], y[p.row0[n] + l]);
        o[od] = make_double2((double)acc.x, (double)acc.y);
      }
    }
  }
}

}  // namespace ctf
