// ctf_rowwarp.cuh — row-per-warp ISS sweep kernel (sm_100a).
//
// Same contract and numerics as sweep_kernel (ctf_kernels.cuh) — one CTA per
// (mixture, bin) runs the bin-local part of one iteration of
// proj/src/estimator.cpp:548-654 — with a different thread mapping:
//   * warp w owns demixing row p = w / WPR and the contiguous frames
//     [j0, j0 + FT) with j0 = ((w % WPR) * 32 + lane) * FT, so Y, the
//     previous pivot and the ISS weights 1/lambda_{n_p}(j - l_p) of a lane's
//     frames live in registers for the whole sweep;
//   * the current pivot row y_r is broadcast through a double-buffered,
//     padded shared-memory row (conflict-free LDS.128), published by the
//     warps of row r at the end of the previous step;
//   * the step's sums (numer_p, denom_p) are warp-local: a 3-value butterfly,
//     plus a fixed-order combine of the row's WPR warps (named barrier);
//   * one CTA barrier per step.
// fp32 uses packed FFMA2/FMUL2. The frame padding: frame j sits at smem
// index pidx(j) = j + 2*(j / FT) so a lane's FT frames start 16-byte aligned
// and consecutive lanes land in different banks.
#pragma once

#include "ctf_kernels.cuh"

namespace ctf {

template <int FT>
__device__ __forceinline__ int pidx(int j) {
  return j + 2 * (j / FT);
}

template <typename Real, int FT, int WPR, int NTHREADS>
__global__ void __launch_bounds__(NTHREADS, 1) rowwarp_kernel(const SweepParams p) {
  using R2 = typename Cplx<Real>::T;
  static_assert(FT % 2 == 0, "pairs of frames per 16-byte access");
  constexpr int NW = NTHREADS / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bin = blockIdx.x, mix = blockIdx.y;
  const int gbin = p.bin_lo + bin;
  const int R = p.R, D = p.D, T = p.T, TP = p.TP, N = p.N, SK = p.SK;
  const int row = warp / WPR, wir = warp - row * WPR;  // row of this warp, warp index within the row
  const int chunk = wir * 32 + lane;                    // frame chunk of this lane
  const int j0 = chunk * FT;
  constexpr int CH = FT + 2;  // padded chunk length (complex elements)
  const int XP = (TP / FT + 1) * CH;  // x tile row length (one leading zero chunk)

  R2* PB = reinterpret_cast<R2*>(smem + p.off_y);      // 2 x (TP/FT)*CH pivot rows
  R2* xs = reinterpret_cast<R2*>(smem + p.off_x);      // Mx x XP
  Real* Pq = reinterpret_cast<Real*>(smem + p.off_x);  // R x TP |y|^2 (aliases xs after the demix)
  Real* Es = reinterpret_cast<Real*>(smem + p.off_e);  // N x TP
  Real* invl = reinterpret_cast<Real*>(smem + p.off_l);
  R2* Wb = reinterpret_cast<R2*>(smem + p.off_w);       // 2 x (R x D)
  Real* red = reinterpret_cast<Real*>(smem + p.off_red);  // 2 x R x WPR x 4
  Real* Bs = reinterpret_cast<Real*>(smem + p.off_b);
  double* dred = reinterpret_cast<double*>(smem + p.off_d);  // NW x 4 + R (1 - z_r)
  __shared__ int s_bad, s_badrow;
  __shared__ double s_logmu;
  const int PBN = (TP / FT) * CH;

  const size_t tile = (size_t)mix * p.FL + bin;
  const R2* xg = reinterpret_cast<const R2*>(p.x) + tile * (size_t)T * p.Mx;
  R2* Wg = reinterpret_cast<R2*>(p.W) + tile * (size_t)R * D;
  Real* Bg = reinterpret_cast<Real*>(p.Bf) + tile * SK;
  const Real* Vg = reinterpret_cast<const Real*>(p.V) + (size_t)mix * SK * T;
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
    s_logmu = lm;
  }
  // ---- prologue: x tile in the padded frame layout, one leading zero chunk
  for (int i = tid; i < p.Mx * XP; i += NTHREADS) xs[i] = czero<Real>();
  __syncthreads();
  for (int t = tid; t < T; t += NTHREADS)
    for (int m = 0; m < p.Mx; ++m) xs[m * XP + pidx<FT>(t + FT)] = xg[(size_t)t * p.Mx + m];
  for (int i = tid; i < R * D; i += NTHREADS) {
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
    for (int i = p.koff[n] + tid; i < p.koff[n + 1]; i += NTHREADS) {
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
  // lambda = max(B V, floor) -> 1/lambda (frame-strided), log-lambda objective term
  double logsum = 0.0;
  for (int n = 0; n < N; ++n) {
    Real* il = invl + n * p.lp;
    for (int i = tid; i < p.loff; i += NTHREADS) il[i] = Real(0);
    const int k0 = p.koff[n], k1 = p.koff[n + 1], Ln = p.ntaps[n];
    for (int tau = tid; tau < TP; tau += NTHREADS) {
      Real v = Real(0);
      if (tau < T) {
        Real lam = Real(0);
        for (int kk = k0; kk < k1; ++kk) lam = fma(Bs[kk], __ldg(Vg + (size_t)kk * T + tau), lam);
        lam = fmax(lam, floor_abs);
        v = Real(1) / lam;
        if (p.has_prev) logsum += (double)min(Ln, T - tau) * (double)log(lam);
      }
      il[p.loff + tau] = v;
    }
  }
  __syncthreads();

  // ---- Y row = W[row, :] x~ for the lane's frames (estimator.cpp:555)
  R2 y[FT];
#pragma unroll
  for (int k = 0; k < FT; ++k) y[k] = czero<Real>();
  {
    const int xbase = (chunk + 1) * CH;  // padded index of frame j0 (+ the leading chunk)
    for (int c = 0; c < D; ++c) {
      const R2 w = Wb[c * R + row];
      const int m = c / p.Ls, l = c - m * p.Ls;
      const R2* xrow = xs + m * XP;
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        // frame j0 + k - l: same chunk when k >= l, else the previous chunk
        const R2 xv = xrow[xbase + k - l - (k < l ? 2 : 0)];
        if constexpr (std::is_same<Real, float>::value) {
          y[k] = ffma2s(make_float2(-xv.y, xv.x), w.y, ffma2s(xv, w.x, y[k]));
        } else {
          cmac(y[k], w, xv);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < FT; ++k)
      if (j0 + k >= T) y[k] = czero<Real>();
  }
  // ISS weights of this row for the lane's frames (constant over the sweep)
  Real wt[FT];
#pragma unroll
  for (int k = 0; k < FT; ++k) wt[k] = invl[p.woff[row] + j0 + k];

  double logdet = p.logdet[tile] - s_logmu;
  if (p.has_prev) {
    // objective of the previous iteration (estimator.cpp:55-77)
    double quad = 0.0;
    bool fin = true;
#pragma unroll
    for (int k = 0; k < FT; ++k) {
      fin = fin && cfinite(y[k]);
      quad += (double)cnorm(y[k]) * (double)wt[k];
    }
    if (!fin) s_bad = 1;
    double v2[2] = {logsum, quad};
    block_sum_d<2>(v2, dred, lane, warp, NW);
    if (s_bad) {  // estimator.cpp:497-499
      if (tid == 0) record_err<Real>(p.err, mix, err_key(prev_it, kPhFinite, gbin, 0, 2));
      return;
    }
    const int det_status = isnan(logdet) || logdet == -INFINITY ? 4 : (logdet < log(1e-300) ? 5 : 0);
    if (det_status) {
      if (tid == 0) record_err<Real>(p.err, mix, err_key(prev_it, kPhDet, gbin, 0, det_status));
      return;
    }
    if (tid == 0) p.objbin[tile] = v2[0] + v2[1] - 2.0 * (double)T * logdet;
  }
  if (!p.do_sweep) {  // finalize pass
    for (int i = tid; i < R * D; i += NTHREADS) Wg[i] = Wb[i];
    for (int i = tid; i < SK; i += NTHREADS) Bg[i] = Bs[i];
    if (tid == 0) p.logdet[tile] = logdet;
    return;
  }

  // ---- ISS sweep (estimator.cpp:556-579)
  const int pb_base = chunk * CH;
  if (row == 0) {  // publish the first pivot row
#pragma unroll
    for (int k = 0; k < FT; ++k) PB[pb_base + k] = y[k];
  }
  R2 pv[FT];
#pragma unroll
  for (int k = 0; k < FT; ++k) pv[k] = czero<Real>();
  R2 zp = czero<Real>();  // this row's pending update coefficient
  double* onemz = dred + NW * 4;
  __syncthreads();
  for (int r = 0; r < R; ++r) {
    const R2* pb = PB + (r & 1) * PBN + pb_base;
    // pass: y -= zp pv (step r-1), then the sums of step r against yr
    Real nre, nim, den;
    if constexpr (std::is_same<Real, float>::value) {
      float2 q1 = make_float2(0.f, 0.f), q2 = q1, d2 = q1;
#pragma unroll
      for (int k = 0; k < FT; k += 2) {
        const float4 yr4 = *reinterpret_cast<const float4*>(pb + k);
        const float2 yr[2] = {make_float2(yr4.x, yr4.y), make_float2(yr4.z, yr4.w)};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float2 v = y[k + h];
          v = ffma2s(pv[k + h], -zp.x, v);
          v.x = fmaf(zp.y, pv[k + h].y, v.x);
          v.y = fmaf(-zp.y, pv[k + h].x, v.y);
          y[k + h] = v;
          const float2 s = fmul2s(yr[h], wt[k + h]);
          q1 = ffma2s(v, s.x, q1);
          q2 = ffma2s(v, s.y, q2);
          d2 = ffma2(yr[h], s, d2);
          pv[k + h] = yr[h];
        }
      }
      nre = q1.x + q2.y;
      nim = q1.y - q2.x;
      den = d2.x + d2.y;
    } else {
      nre = nim = den = Real(0);
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        const R2 yr = pb[k];
        cmsub(y[k], zp, pv[k]);
        const Real w = wt[k];
        nre = fma(fma(y[k].x, yr.x, y[k].y * yr.y), w, nre);
        nim = fma(fma(y[k].y, yr.x, -y[k].x * yr.y), w, nim);
        den = fma(cnorm(yr), w, den);
        pv[k] = yr;
      }
    }
    nre = warp_sum(nre);
    nim = warp_sum(nim);
    den = warp_sum(den);
    Real* rb = red + (size_t)(((r & 1) * R + row) * WPR) * 4;
    if constexpr (WPR > 1) {
      if (lane == 0) {
        rb[wir * 4 + 0] = nre;
        rb[wir * 4 + 1] = nim;
        rb[wir * 4 + 2] = den;
      }
      // the row's WPR warps meet on named barrier 1 + row
      asm volatile("bar.sync %0, %1;" ::"r"(1 + row), "r"(WPR * 32) : "memory");
      nre = nim = den = Real(0);
#pragma unroll
      for (int w = 0; w < WPR; ++w) {
        nre += rb[w * 4 + 0];
        nim += rb[w * 4 + 1];
        den += rb[w * 4 + 2];
      }
    }
    const bool bad = !(den > Real(0)) || !isfinite(den);
    R2 z;
    if (row == r) {
      z.x = Real(1) - sqrt((Real)T / den);
      z.y = Real(0);
      if (wir == 0 && lane == 0) onemz[r] = (double)(Real(1) - z.x);
    } else {
      z.x = nre / den;
      z.y = nim / den;
    }
    if (bad && lane == 0) atomicMin(&s_badrow, row);  // lowest bad row of this step
    // iss_apply, W -= z w_r (estimator.cpp:298-302): the row's first warp
    if (wir == 0) {
      const R2* Wo = Wb + (r & 1) * R * D;
      R2* Wn = Wb + ((r + 1) & 1) * R * D;
      for (int c = lane; c < D; c += 32) {
        R2 w = Wo[c * R + row];
        cmsub(w, z, Wo[c * R + r]);
        Wn[c * R + row] = w;
      }
    }
    if (row == r + 1) {  // next pivot: apply this step's update now and publish it
      R2* pn = PB + ((r + 1) & 1) * PBN + pb_base;
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        cmsub(y[k], z, pv[k]);
        pn[k] = y[k];
      }
      zp = czero<Real>();
    } else {
      zp = z;
    }
    __syncthreads();
    if (s_badrow != 0x7fffffff) {  // estimator.cpp:451-454
      if (tid == 0) record_err<Real>(p.err, mix, err_key(p.iteration, kPhSweep, gbin, r, (unsigned)s_badrow));
      return;
    }
  }
  // last step's update
#pragma unroll
  for (int k = 0; k < FT; ++k) cmsub(y[k], zp, pv[k]);
  const R2* Wf = Wb + (R & 1) * R * D;

  // ---- epilogue: row powers, |y|^2 for the delayed energies, E, MU-B
  {
    Real rp = Real(0);
#pragma unroll
    for (int k = 0; k < FT; ++k) {
      const Real q = cnorm(y[k]);
      rp += q;
      Pq[row * TP + j0 + k] = q;
    }
    rp = warp_sum(rp);
    if (lane == 0) red[(row * WPR + wir) * 4 + 3] = rp;  // slot 3 unused by the sweep
  }
  __syncthreads();
  if (tid < R) {
    double s = 0.0;
    for (int w = 0; w < WPR; ++w) s += (double)red[(tid * WPR + w) * 4 + 3];
    p.rowpow[tile * R + tid] = s;
  }
  if (tid == 0) {
    double prod = 1.0;
    for (int r = 0; r < R; ++r) prod *= onemz[r];
    p.logdet[tile] = logdet + log(prod);
  }
  Real* Eg = reinterpret_cast<Real*>(p.E);
  for (int n = 0; n < N; ++n) {
    const int r0 = p.row0[n], Ln = p.ntaps[n];
    for (int tau = tid; tau < TP; tau += NTHREADS) {
      Real e = Real(0);
      for (int l = 0; l < Ln && tau + l < T; ++l) e += Pq[(r0 + l) * TP + tau + l];
      Es[n * TP + tau] = e;
      if (tau < T) Eg[(((size_t)mix * N + n) * p.FL + bin) * T + tau] = e;
    }
  }
  for (int i = tid; i < R * D; i += NTHREADS) Wg[i] = Wf[i];
  __syncthreads();
  // MU-B for this bin (estimator.cpp:313-346): warps take (source, base) pairs,
  // lanes stride frames; fixed-order warp sums.
  for (int n = 0; n < N; ++n) {
    const int k0 = p.koff[n], k1 = p.koff[n + 1], Ln = p.ntaps[n];
    const Real* il = invl + n * p.lp + p.loff;
    for (int kb = k0 + warp; kb < k1; kb += NW) {
      const Real* vrow = Vg + (size_t)kb * T;
      Real num = Real(0), dd = Real(0);
      for (int tau = lane; tau < T; tau += 32) {
        const Real ilv = il[tau];
        const Real v = __ldg(vrow + tau);
        num = fma(Es[n * TP + tau] * (ilv * ilv), v, num);
        dd = fma(ilv * (Real)min(Ln, T - tau), v, dd);
      }
      num = warp_sum(num);
      dd = warp_sum(dd);
      if (lane == 0) Bg[kb] = fmax(Bs[kb] * sqrt(num / dd), floor_abs);
    }
  }
}

}  // namespace ctf
