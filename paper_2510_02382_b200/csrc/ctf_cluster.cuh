// ctf_cluster.cuh — thread-block-cluster ISS sweep for tiles beyond one SM
// (BASELINE cfg3: R = 32, T = 1000; cfg4: R = 60, T = 4000).
//
// Same contract and numerics as sweep_kernel (ctf_kernels.cuh): the
// bin-local part of one iteration of proj/src/estimator.cpp:548-654. A
// cluster of CS CTAs (one per SM) handles one (mixture, bin); CTA c owns
// demixing rows [c*RB, (c+1)*RB) for ALL frames, so the R x T estimate tile
// stays on chip (RREG rows per thread in registers, the rest in shared
// memory) and each CTA runs the frame-owner sweep of sweep_kernel on its own
// rows. Per ISS step the only cross-CTA data is the next pivot row y_{r+1}
// (and W's row r+1): its owner applies step r's update to it, publishes it
// through L2 (double-buffered per bin), and a cluster barrier
// (barrier.cluster arrive.release / wait.acquire) orders the exchange. Row
// sums, z and the W update of a row stay in its CTA. The per-source delayed
// energies, MU-B and the log-lambda objective term are assigned to CTA
// n % CS; the objective, row powers and log|det| partials are combined by
// CTA 0 in fixed order (deterministic).
#pragma once

#include <cooperative_groups.h>

#include "ctf_kernels.cuh"

namespace ctf {

struct ClusterParams {
  SweepParams s;     // shapes, buffers, row map; smem offsets of this kernel
  void* pivot;       // Real2 [mix][FL][2][TP]   next pivot row, double-buffered
  void* wpivot;      // Real2 [mix][FL][2][D]    W row of the next pivot
  double* part;      // [mix][FL][CS][4]         objective / log-det partials
  int* bad;          // [mix][FL]                cluster-wide abort flag (first bad row + 1)
  int CS;
};

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <typename Real, int RB, int FT, int RREG, int NT>
__global__ void __launch_bounds__(NT, 1) cluster_kernel(const ClusterParams cp) {
  using R2 = typename Cplx<Real>::T;
  constexpr int RS = RB - RREG;
  constexpr int NV = 3 * RB;
  constexpr int VP = ((NV + 31) / 32) * 32;
  constexpr int VM = VP / 32;
  constexpr int NW = NT / 32;
  static_assert(RB <= 32, "one lane per local row");
  const SweepParams& p = cp.s;
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int CS = cp.CS;
  const int c = (int)cluster_ctarank();
  const int bin = blockIdx.x / CS, mix = blockIdx.y;
  const int gbin = p.bin_lo + bin;
  const int R = p.R, D = p.D, T = p.T, TP = p.TP, N = p.N, SK = p.SK;
  const int row0c = c * RB;  // first global row of this CTA

  R2* Ysm = reinterpret_cast<R2*>(smem + p.off_y);        // RS x TP
  R2* xst = reinterpret_cast<R2*>(smem + p.off_x);        // one microphone (xoff + TP)
  Real* invl = reinterpret_cast<Real*>(smem + p.off_l);   // N x lp (sources of the own rows)
  R2* Wown = reinterpret_cast<R2*>(smem + p.off_w);       // D x RB (column-major like W)
  R2* Wpv = reinterpret_cast<R2*>(smem + p.off_e);        // D (W row of the current pivot)
  Real* red = reinterpret_cast<Real*>(smem + p.off_red);  // 2 x NW x VP
  R2* zs = reinterpret_cast<R2*>(smem + p.off_z);         // NW x RB (per-warp z copies)
  Real* Bs = reinterpret_cast<Real*>(smem + p.off_b);     // SK
  double* dred = reinterpret_cast<double*>(smem + p.off_d);  // NW x 4 + R
  __shared__ int s_bad, s_badrow;
  __shared__ double s_logmu;

  const size_t tile = (size_t)mix * p.FL + bin;
  const R2* xg = reinterpret_cast<const R2*>(p.x) + tile * (size_t)T * p.Mx;
  R2* Wg = reinterpret_cast<R2*>(p.W) + tile * (size_t)R * D;
  Real* Bg = reinterpret_cast<Real*>(p.Bf) + tile * SK;
  const Real* Vg = reinterpret_cast<const Real*>(p.V) + (size_t)mix * SK * T;
  R2* PBg = reinterpret_cast<R2*>(cp.pivot) + tile * 2 * TP;
  R2* WPg = reinterpret_cast<R2*>(cp.wpivot) + tile * 2 * D;
  double* part = cp.part + (tile * CS + c) * 4;
  int* badg = cp.bad + tile;
  const Real floor_abs = (Real)p.floor_abs[mix];
  const int prev_it = p.iteration - 1;
  const double* mu = p.mu ? p.mu + (size_t)mix * R : nullptr;

  if (tid == 0) {
    s_bad = 0;
    s_badrow = 0x7fffffff;
    double lm = 0.0;
    if (mu)
      for (int r = 0; r < R; ++r)
        if (mu[r] != 0.0) lm += log(mu[r]);
    s_logmu = lm;  // *badg is zeroed by the host before every launch
  }
  // ---- prologue: own W rows and B with the pending rescale
  for (int i = tid; i < RB * D; i += NT) {
    const int q = i % RB, col = i / RB;
    R2 w = Wg[(size_t)col * R + row0c + q];
    if (mu) {
      const double m = mu[row0c + q];
      if (m != 0.0) {
        w.x = (Real)((double)w.x / m);
        w.y = (Real)((double)w.y / m);
      }
    }
    Wown[i] = w;
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
  // 1/lambda for the sources of the own rows, and the log-lambda objective
  // term of the sources assigned to this CTA (n % CS == c)
  const int nlo = p.srcr[row0c], nhi = p.srcr[row0c + RB - 1];
  double logsum = 0.0;
  for (int n = 0; n < N; ++n) {
    const bool needw = n >= nlo && n <= nhi, needlog = p.has_prev && (n % CS) == c;
    if (!needw && !needlog) continue;
    Real* il = invl + (n - nlo) * p.lp;
    if (needw)
      for (int i = tid; i < p.loff; i += NT) il[i] = Real(0);
    const int k0 = p.koff[n], k1 = p.koff[n + 1], Ln = p.ntaps[n];
    for (int tau = tid; tau < TP; tau += NT) {
      Real v = Real(0);
      if (tau < T) {
        Real lam = Real(0);
        for (int kk = k0; kk < k1; ++kk) lam = fma(Bs[kk], __ldg(Vg + (size_t)kk * T + tau), lam);
        lam = fmax(lam, floor_abs);
        v = Real(1) / lam;
        if (needlog) logsum += (double)min(Ln, T - tau) * (double)log(lam);
      }
      if (needw) il[p.loff + tau] = v;
    }
  }
  // ---- own rows of Y = W x~, one microphone staged at a time
  YTile<R2, FT, RREG, RS> Y;
  Y.sm = Ysm;
  Y.tp = TP;
  static_for<0, RB>([&](auto pp) {
    constexpr int P = decltype(pp)::value;
#pragma unroll
    for (int k = 0; k < FT; ++k) Y.template set<P>(k, tid + k * NT, czero<Real>());
  });
  for (int m = 0; m < p.Mx; ++m) {
    __syncthreads();
    for (int i = tid; i < p.xoff + TP; i += NT) {
      const int t = i - p.xoff;
      xst[i] = (t >= 0 && t < T) ? xg[(size_t)t * p.Mx + m] : czero<Real>();
    }
    __syncthreads();
    for (int l = 0; l < p.Ls; ++l) {
      const int col = m * p.Ls + l;
      static_for<0, RB>([&](auto pp) {
        constexpr int P = decltype(pp)::value;
        const R2 w = Wown[col * RB + P];
#pragma unroll
        for (int k = 0; k < FT; ++k) {
          const int j = tid + k * NT;
          R2 y = Y.template get<P>(k, j);
          cmac(y, w, xst[p.xoff + j - l]);
          Y.template set<P>(k, j, y);
        }
      });
    }
  }
  static_for<0, RB>([&](auto pp) {
    constexpr int P = decltype(pp)::value;
#pragma unroll
    for (int k = 0; k < FT; ++k) {
      const int j = tid + k * NT;
      if (j >= T) Y.template set<P>(k, j, czero<Real>());
    }
  });
  __syncthreads();

  double logdet_resc = p.logdet[tile] - s_logmu;
  if (p.has_prev) {
    Real qf = Real(0), sy = Real(0);
    static_for<0, RB>([&](auto pp) {
      constexpr int P = decltype(pp)::value;
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        const int j = tid + k * NT;
        const R2 y = Y.template get<P>(k, j);
        sy += y.x + y.y;
        qf = fma(cnorm(y), invl[p.woff[row0c + P] - nlo * p.lp + j], qf);
      }
    });
    if (!isfinite(sy) || !isfinite(qf)) s_bad = 1;
    double v2[2] = {logsum, (double)qf};
    block_sum_d<2>(v2, dred, lane, warp, NW);
    if (tid == 0) {
      part[0] = v2[0] + v2[1];
      if (s_bad) atomicMax(badg, 1 << 20);  // non-finite estimates (estimator.cpp:497-499)
    }
  }
  if (!p.do_sweep) {  // finalize pass
    for (int i = tid; i < RB * D; i += NT) {
      const int q = i % RB, col = i / RB;
      Wg[(size_t)col * R + row0c + q] = Wown[i];
    }
    if (c == 0)
      for (int i = tid; i < SK; i += NT) Bg[i] = Bs[i];
    cluster_sync_all();
    if (c == 0 && tid == 0) {
      const int b = *badg;
      if (p.has_prev && b) {
        record_err<Real>(p.err, mix, err_key(prev_it, kPhFinite, gbin, 0, 2));
      } else {
        const double ld = logdet_resc;
        const int det_status = isnan(ld) || ld == -INFINITY ? 4 : (ld < log(1e-300) ? 5 : 0);
        if (p.has_prev && det_status) {
          record_err<Real>(p.err, mix, err_key(prev_it, kPhDet, gbin, 0, det_status));
        } else if (p.has_prev) {
          double o = 0.0;
          for (int q = 0; q < CS; ++q) o += cp.part[(tile * CS + q) * 4 + 0];
          p.objbin[tile] = o - 2.0 * (double)T * ld;
        }
        p.logdet[tile] = ld;
      }
    }
    return;
  }
  // publish the first pivot row (row 0, owned by CTA 0) and its W row
  if (c == 0) {
#pragma unroll
    for (int k = 0; k < FT; ++k) PBg[tid + k * NT] = Y.template get<0>(k, tid + k * NT);
    for (int i = tid; i < D; i += NT) WPg[i] = Wown[i * RB + 0];
  }
  cluster_sync_all();
  if (p.has_prev && *badg) {  // uniform across the cluster
    if (c == 0 && tid == 0) record_err<Real>(p.err, mix, err_key(prev_it, kPhFinite, gbin, 0, 2));
    return;
  }
  if (p.has_prev && c == 0 && tid == 0) {
    const double ld = logdet_resc;
    const int det_status = isnan(ld) || ld == -INFINITY ? 4 : (ld < log(1e-300) ? 5 : 0);
    if (det_status) {
      record_err<Real>(p.err, mix, err_key(prev_it, kPhDet, gbin, 0, det_status));
    } else {
      double o = 0.0;
      for (int q = 0; q < CS; ++q) o += cp.part[(tile * CS + q) * 4 + 0];
      p.objbin[tile] = o - 2.0 * (double)T * ld;
    }
  }

  // ---- ISS sweep over all R steps; this CTA updates and sums its own rows
  const int woff_base = -nlo * p.lp;
  R2 pv[FT];
#pragma unroll
  for (int k = 0; k < FT; ++k) pv[k] = czero<Real>();
  if (lane < RB) zs[warp * RB + lane] = czero<Real>();
  __syncwarp();
  double dprod = 1.0;  // prod of (1 - z_r) over the own pivot rows
  for (int r = 0; r < R; ++r) {
    const R2* pb = PBg + (r & 1) * TP;
    Real acc[VP];
#pragma unroll
    for (int i = 0; i < VP; ++i) acc[i] = Real(0);
    const R2* zw = zs + warp * RB;
#pragma unroll
    for (int k = 0; k < FT; ++k) {
      const int j = tid + k * NT;
      const R2 yr = pb[j];  // pivot row r after step r-1 (published by its owner)
      const Real ar2 = cnorm(yr);
      static_for<0, RB>([&](auto pp) {
        constexpr int P = decltype(pp)::value;
        R2 y = Y.template get<P>(k, j);
        cmsub(y, zw[P], pv[k]);
        Y.template set<P>(k, j, y);
        const Real w = invl[p.woff[row0c + P] + woff_base + j];
        const Real tr = fma(y.x, yr.x, y.y * yr.y);
        const Real ti = fma(y.y, yr.x, -y.x * yr.y);
        acc[P] = fma(tr, w, acc[P]);
        acc[RB + P] = fma(ti, w, acc[RB + P]);
        acc[2 * RB + P] = fma(ar2, w, acc[2 * RB + P]);
      });
      pv[k] = yr;
    }
    warp_reduce_scatter(acc, lane);
    Real* rb = red + (size_t)((r & 1) * NW + warp) * VP;
#pragma unroll
    for (int i = 0; i < VM; ++i) rb[lane * VM + i] = acc[i];
    __syncthreads();
    const Real* rs = red + (size_t)((r & 1) * NW) * VP;
    bool bad = false;
    R2 z = czero<Real>();
    if (lane < RB) {
      Real nre = Real(0), nim = Real(0), den = Real(0);
      for (int w = 0; w < NW; ++w) {
        nre += rs[w * VP + lane];
        nim += rs[w * VP + RB + lane];
        den += rs[w * VP + 2 * RB + lane];
      }
      bad = !(den > Real(0)) || !isfinite(den);
      if (row0c + lane == r) {
        z.x = Real(1) - sqrt((Real)T / den);
      } else {
        z.x = nre / den;
        z.y = nim / den;
      }
      zs[warp * RB + lane] = z;
    }
    const unsigned badm = __ballot_sync(kFull, bad);
    __syncwarp();
    if (badm && warp == 0 && lane == 0) atomicMin(&s_badrow, row0c + __ffs(badm) - 1);
    const int rl = r - row0c;  // local index of the pivot row (if own)
    if (rl >= 0 && rl < RB) dprod *= (double)(Real(1) - zw[rl].x);
    // own W rows: W_p -= z_p W_r (estimator.cpp:298-302); the pivot's old W
    // row is in WPg[r & 1] (published before this step)
    __syncthreads();  // every warp done reading the partials; s_badrow final
    for (int e = tid; e < D; e += NT) Wpv[e] = WPg[(r & 1) * D + e];
    __syncthreads();
    for (int e = tid; e < RB * D; e += NT) {
      const int q = e % RB, col = e / RB;
      cmsub(Wown[e], zw[q], Wpv[col]);  // this warp's copy of z (identical in every warp)
    }
    // the owner of row r+1 applies this step's update to it now and publishes
    // it (and its W row) for step r+1; its pending z becomes 0
    const int nl = r + 1 - row0c;
    if (nl >= 0 && nl < RB && r + 1 < R) {
      const R2 zn = zw[nl];
      R2* pn = PBg + ((r + 1) & 1) * TP;
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        const int j = tid + k * NT;
        R2 y = Y.pick(k, j, nl);
        cmsub(y, zn, pv[k]);
        static_for<0, RB>([&](auto pp) {
          constexpr int P = decltype(pp)::value;
          if (P == nl) Y.template set<P>(k, j, y);
        });
        pn[j] = y;
      }
      __syncthreads();  // own W update complete before publishing row r+1
      for (int e = tid; e < D; e += NT) WPg[((r + 1) & 1) * D + e] = Wown[e * RB + nl];
      if (lane == 0) zs[warp * RB + nl] = czero<Real>();
      __syncwarp();
    }
    if (tid == 0 && s_badrow != 0x7fffffff) atomicMin(badg, -(0x7fffff - s_badrow) - 1);
    cluster_sync_all();
    const int bg = *badg;
    if (bg < 0) {  // lowest bad row over the cluster
      if (c == 0 && tid == 0) {
        const int row = 0x7fffff - (-bg - 1);
        record_err<Real>(p.err, mix, err_key(p.iteration, kPhSweep, gbin, r, (unsigned)row));
      }
      return;
    }
  }
  // last step's update of the own rows
  {
    const R2* zw = zs + warp * RB;
#pragma unroll
    for (int k = 0; k < FT; ++k) {
      const int j = tid + k * NT;
      static_for<0, RB>([&](auto pp) {
        constexpr int P = decltype(pp)::value;
        R2 y = Y.template get<P>(k, j);
        cmsub(y, zw[P], pv[k]);
        Y.template set<P>(k, j, y);
      });
    }
  }
  // row powers and |y|^2 of the own rows (the x stage / 1/lambda region is
  // dead now and holds |y|^2: RB x TP)
  Real* Pq = reinterpret_cast<Real*>(smem + p.off_x);
  {
    constexpr int RP = ((RB + 31) / 32) * 32;
    Real rp[RP];
#pragma unroll
    for (int i = 0; i < RP; ++i) rp[i] = Real(0);
    static_for<0, RB>([&](auto pp) {
      constexpr int P = decltype(pp)::value;
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        const int j = tid + k * NT;
        const Real q = cnorm(Y.template get<P>(k, j));
        rp[P] += q;
        Pq[P * TP + j] = q;
      }
    });
    warp_reduce_scatter(rp, lane);
    __syncthreads();  // every warp done with the sweep partials
    Real* rb = red + (size_t)warp * VP;
#pragma unroll
    for (int i = 0; i < RP / 32; ++i) rb[lane * (RP / 32) + i] = rp[i];
  }
  __syncthreads();
  if (tid < RB) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += (double)red[(size_t)w * VP + tid];
    p.rowpow[tile * R + row0c + tid] = s;
  }
  for (int i = tid; i < RB * D; i += NT) {
    const int q = i % RB, col = i / RB;
    Wg[(size_t)col * R + row0c + q] = Wown[i];
  }
  if (tid == 0) part[1] = log(dprod);
  // partial delayed energies of the sources touched by the own rows:
  // Ep[n - nlo][tau] = sum over own rows (n, l) of |y_{n,l}(tau + l)|^2,
  // in the Y region (dead once |y|^2 is in Pq)
  __syncthreads();
  Real* Ep = reinterpret_cast<Real*>(smem + p.off_y);  // (nhi - nlo + 1) x TP
  for (int n = nlo; n <= nhi; ++n)
    for (int tau = tid; tau < TP; tau += NT) {
      Real e = Real(0);
      for (int P = 0; P < RB; ++P)
        if (p.srcr[row0c + P] == n) {
          const int l = p.woff[p.row0[n]] - p.woff[row0c + P];  // tap of the row
          if (tau + l < T) e += Pq[P * TP + tau + l];
        }
      Ep[(n - nlo) * TP + tau] = e;
    }
  cluster_sync_all();  // partial energies and log-det partials visible cluster-wide
  if (c == 0 && tid == 0) {
    double ld = logdet_resc;
    for (int q = 0; q < CS; ++q) ld += cp.part[(tile * CS + q) * 4 + 1];
    p.logdet[tile] = ld;
  }
  // the sources assigned to this CTA (n % CS == c): combine the partial
  // energies of the CTAs holding rows of n (fixed order, read over DSMEM),
  // then MU-B for the bin (estimator.cpp:313-346)
  Real* Eg = reinterpret_cast<Real*>(p.E);
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  Real* En_s = Ep + (size_t)(nhi - nlo + 1) * TP;  // TP, after the partials in the Y region
  for (int n = c; n < N; n += CS) {
    const int r0 = p.row0[n], Ln = p.ntaps[n];
    const int c_first = r0 / RB, c_last = (r0 + Ln - 1) / RB;
    const int k0 = p.koff[n], k1 = p.koff[n + 1];
    Real* En = Eg + (((size_t)mix * N + n) * p.FL + bin) * T;
    for (int tau = tid; tau < T; tau += NT) {
      Real e = Real(0);
      for (int q = c_first; q <= c_last; ++q) {
        const int nlo_q = p.srcr[q * RB];
        const Real* ep = cluster.map_shared_rank(Ep, q);
        e += ep[(n - nlo_q) * TP + tau];
      }
      En[tau] = e;
      En_s[tau] = e;
    }
    __syncthreads();
    // 16 bases per pass: lambda computed once per frame, a[q] numerator and
    // a[16 + q] denominator of base kb + q, reduce-scatter + fixed-order sum
    for (int kb = k0; kb < k1; kb += 16) {
      Real a[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) a[i] = Real(0);
      for (int tau = tid; tau < T; tau += NT) {
        Real lam = Real(0);
        for (int kk = k0; kk < k1; ++kk) lam = fma(Bs[kk], __ldg(Vg + (size_t)kk * T + tau), lam);
        const Real ilv = Real(1) / fmax(lam, floor_abs);
        const Real an = En_s[tau] * (ilv * ilv), bn = ilv * (Real)min(Ln, T - tau);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const Real v = __ldg(Vg + (size_t)min(kb + q, k1 - 1) * T + tau);
          a[q] = fma(an, v, a[q]);
          a[16 + q] = fma(bn, v, a[16 + q]);
        }
      }
      warp_reduce_scatter(a, lane);
      __syncthreads();
      red[warp * 32 + lane] = a[0];
      __syncthreads();
      if (tid < 16 && kb + tid < k1) {
        Real num = Real(0), den = Real(0);
        for (int w = 0; w < NW; ++w) {
          num += red[w * 32 + tid];
          den += red[w * 32 + 16 + tid];
        }
        Bg[kb + tid] = fmax(Bs[kb + tid] * sqrt(num / den), floor_abs);
      }
    }
    __syncthreads();
  }
  cluster_sync_all();  // no CTA leaves while its partial energies may be read
}

}  // namespace ctf
