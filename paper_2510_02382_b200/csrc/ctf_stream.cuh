// ctf_stream.cuh — streamed ISS sweep for tiles that exceed one SM
// (BASELINE cfg3 R=32, cfg4 R=60; fp64 long frames).
//
// Same contract and numerics as sweep_kernel (ctf_kernels.cuh): the
// bin-local part of one iteration of proj/src/estimator.cpp:548-654. The
// R x T estimate tile lives in a per-CTA scratch slot in global memory
// (L2/HBM resident); the kernel is persistent (one slot per resident CTA,
// bins taken in grid-stride order). Threads own frames j = tid + k*NT; each
// ISS step is one pass over the tile in groups of RG rows (RG compile-time,
// 3*RG sums per thread, warp reduce-scatter per group), then two CTA
// barriers: one for the sums, one after the steering vector z.
// Algorithmic HBM traffic per step is 2 * R * T * c bytes (read + write of
// the tile), which makes this path HBM bound ("streamed").
#pragma once

#include "ctf_kernels.cuh"

namespace ctf {

struct StreamParams {
  SweepParams s;       // shapes, buffers, row map (the smem offsets are this kernel's)
  void* scratch;       // Real2 [gridDim.x][R][TP]
  int nwork;           // B * FL
  int ngroups;         // ceil(R / RG)
};

// CHECK: CheckOptions instrumentation for any R <= 64 (estimator.cpp:556-577):
// log|det W| recomputed by a warp LU after every step and compared with the
// determinant lemma det W' = det W (1 - z_r), and the updated pivot row's
// weighted power sum_j |y_r'(j)|^2 / lambda / T compared with 1; per-mixture
// maxima in p.chk (the LU works on a copy of W after the CTA's tile slot).
template <typename Real, int FT, int RG, int NT, int MINB = 1, bool CHECK = false>
__global__ void __launch_bounds__(NT, MINB) stream_kernel(const StreamParams sp) {
  using R2 = typename Cplx<Real>::T;
  constexpr int NW = NT / 32;
  constexpr int VP = ((3 * RG + 31) / 32) * 32;
  constexpr int VM = VP / 32;
  const SweepParams& p = sp.s;
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int R = p.R, D = p.D, T = p.T, TP = p.TP, N = p.N, SK = p.SK, NG = sp.ngroups;
  Real* invl = reinterpret_cast<Real*>(smem + p.off_l);  // N x lp
  R2* Wb = reinterpret_cast<R2*>(smem + p.off_w);        // 2 x R x D
  Real* red = reinterpret_cast<Real*>(smem + p.off_red);  // NW x NG x VP
  R2* zsh = reinterpret_cast<R2*>(smem + p.off_z);        // R (z of the current step)
  Real* Bs = reinterpret_cast<Real*>(smem + p.off_b);     // SK
  double* dred = reinterpret_cast<double*>(smem + p.off_d);  // NW x 4 + R
  R2* xst = reinterpret_cast<R2*>(smem + p.off_x);        // one microphone: xoff + TP (demix stage)
  __shared__ int s_bad, s_badrow;
  __shared__ double s_logmu;
  // per-CTA slot: the R x TP tile (+ CHECK: R x D LU scratch)
  R2* Yg = reinterpret_cast<R2*>(sp.scratch) + (size_t)blockIdx.x * ((size_t)R * TP + (CHECK ? (size_t)R * D : 0));

  for (int work = blockIdx.x; work < sp.nwork; work += gridDim.x) {
    const int mix = work / p.FL, bin = work - mix * p.FL;
    const int gbin = p.bin_lo + bin;
    const size_t tile = (size_t)mix * p.FL + bin;
    const R2* xg = reinterpret_cast<const R2*>(p.x) + tile * (size_t)T * p.Mx;
    R2* Wg = reinterpret_cast<R2*>(p.W) + tile * (size_t)R * D;
    Real* Bg = reinterpret_cast<Real*>(p.Bf) + tile * SK;
    const Real* Vg = reinterpret_cast<const Real*>(p.V) + (size_t)mix * SK * T;
    const Real floor_abs = (Real)p.floor_abs[mix];
    const int prev_it = p.iteration - 1;
    const double* mu = p.mu ? p.mu + (size_t)mix * R : nullptr;
    __syncthreads();  // previous work item fully done with smem
    if (tid == 0) {
      s_bad = 0;
      s_badrow = 0x7fffffff;
      double lm = 0.0;
      if (mu)
        for (int r = 0; r < R; ++r)
          if (mu[r] != 0.0) lm += log(mu[r]);
      s_logmu = lm;
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
    if (p.has_prev && s_bad) {
      if (tid == 0) record_err<Real>(p.err, mix, err_key(prev_it, kPhFinite, gbin, 0, 1));
      continue;  // uniform: s_bad is read after a barrier by every thread
    }
    double logsum = 0.0;
    for (int n = 0; n < N; ++n) {
      Real* il = invl + n * p.lp;
      for (int i = tid; i < p.loff; i += NT) il[i] = Real(0);
      const int k0 = p.koff[n], k1 = p.koff[n + 1], Ln = p.ntaps[n];
      for (int tau = tid; tau < TP; tau += NT) {
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
    // ---- Y = W x~ into the scratch tile, RGD rows at a time, one microphone
    // staged in shared memory at a time (estimator.cpp:555)
    constexpr int RGD = FT >= 8 ? 4 : 8;
    for (int g = 0; g < (R + RGD - 1) / RGD; ++g) {
      R2 acc[RGD][FT];
#pragma unroll
      for (int q = 0; q < RGD; ++q)
#pragma unroll
        for (int k = 0; k < FT; ++k) acc[q][k] = czero<Real>();
      for (int m = 0; m < p.Mx; ++m) {
        __syncthreads();
        for (int i = tid; i < p.xoff + TP; i += NT) {
          const int t = i - p.xoff;
          xst[i] = (t >= 0 && t < T) ? xg[(size_t)t * p.Mx + m] : czero<Real>();
        }
        __syncthreads();
        for (int l = 0; l < p.Ls; ++l) {
          const int c = m * p.Ls + l;
#pragma unroll
          for (int q = 0; q < RGD; ++q) {
            const int row = g * RGD + q;
            const R2 w = row < R ? Wb[c * R + row] : czero<Real>();
#pragma unroll
            for (int k = 0; k < FT; ++k) cmac(acc[q][k], w, xst[p.xoff + tid + k * NT - l]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < RGD; ++q) {
        const int row = g * RGD + q;
        if (row < R)
#pragma unroll
          for (int k = 0; k < FT; ++k) {
            const int j = tid + k * NT;
            Yg[(size_t)row * TP + j] = (j < T) ? acc[q][k] : czero<Real>();
          }
      }
    }
    __syncthreads();  // invl complete; Y rows are thread-private per frame

    double logdet = p.logdet[tile] - s_logmu;
    if (p.has_prev) {
      Real qf = Real(0), sy = Real(0);
      for (int row = 0; row < R; ++row)
#pragma unroll
        for (int k = 0; k < FT; ++k) {
          const int j = tid + k * NT;
          const R2 y = Yg[(size_t)row * TP + j];
          sy += y.x + y.y;
          qf = fma(cnorm(y), invl[p.woff[row] + j], qf);
        }
      if (!isfinite(sy) || !isfinite(qf)) s_bad = 1;
      double v2[2] = {logsum, (double)qf};
      block_sum_d<2>(v2, dred, lane, warp, NW);
      if (s_bad) {
        if (tid == 0) record_err<Real>(p.err, mix, err_key(prev_it, kPhFinite, gbin, 0, 2));
        continue;
      }
      const int det_status = isnan(logdet) || logdet == -INFINITY ? 4 : (logdet < log(1e-300) ? 5 : 0);
      if (det_status) {
        if (tid == 0) record_err<Real>(p.err, mix, err_key(prev_it, kPhDet, gbin, 0, det_status));
        continue;
      }
      if (tid == 0) p.objbin[tile] = v2[0] + v2[1] - 2.0 * (double)T * logdet;
    }
    if (!p.do_sweep) {
      for (int i = tid; i < R * D; i += NT) Wg[i] = Wb[i];
      for (int i = tid; i < SK; i += NT) Bg[i] = Bs[i];
      if (tid == 0) p.logdet[tile] = logdet;
      continue;
    }

    // ---- ISS sweep (estimator.cpp:556-579)
    R2 pv[FT];
#pragma unroll
    for (int k = 0; k < FT; ++k) pv[k] = czero<Real>();
    for (int i = tid; i < R; i += NT) zsh[i] = czero<Real>();
    double* onemz = dred + NW * 4;
    __syncthreads();
    bool aborted = false;
    // CHECK: det of the current W (warp 0: log-magnitude, phase) and maxima (tid 0)
    double c_lm = 0.0, c_ph = 0.0, c_det = 0.0, c_norm = 0.0;
    int c_ok = 0;
    R2* cscr = Yg + (size_t)R * TP;  // (global, L2-resident: check mode only)
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
      if (p.chk_flags & 1) check_det(Wb, 0.0, false);
    }
    for (int r = 0; r < R; ++r) {
      R2 yr[FT];
      Real ar2[FT];
      const R2 zr = zsh[r];
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        yr[k] = Yg[(size_t)r * TP + tid + k * NT];
        cmsub(yr[k], zr, pv[k]);
        ar2[k] = cnorm(yr[k]);
      }
      for (int g = 0; g < NG; ++g) {
        Real a[VP];
#pragma unroll
        for (int i = 0; i < VP; ++i) a[i] = Real(0);
#pragma unroll
        for (int q = 0; q < RG; ++q) {
          const int row = g * RG + q;
          if (row < R) {
            const R2 zp = zsh[row];
            const int wo = p.woff[row];
            if constexpr (std::is_same<Real, float>::value) {
              // packed FP32x2 (see sweep_kernel): y += (-z.x) pv + z.y (pv.y, -pv.x);
              // Q1 += s.x y, Q2 += s.y y with s = w yr; numer = (Q1.x + Q2.y, Q1.y - Q2.x)
              float2 q1 = make_float2(0.f, 0.f), q2 = q1;
              float den = 0.f;
#pragma unroll
              for (int k = 0; k < FT; ++k) {
                const int j = tid + k * NT;
                float2 y = Yg[(size_t)row * TP + j];
                y = ffma2s(pv[k], -zp.x, y);
                y = ffma2s(make_float2(pv[k].y, -pv[k].x), zp.y, y);
                Yg[(size_t)row * TP + j] = y;
                const float w = invl[wo + j];
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
                const int j = tid + k * NT;
                R2 y = Yg[(size_t)row * TP + j];
                cmsub(y, zp, pv[k]);
                Yg[(size_t)row * TP + j] = y;
                const Real w = invl[wo + j];
                a[q] = fma(fma(y.x, yr[k].x, y.y * yr[k].y), w, a[q]);
                a[RG + q] = fma(fma(y.y, yr[k].x, -y.x * yr[k].y), w, a[RG + q]);
                a[2 * RG + q] = fma(ar2[k], w, a[2 * RG + q]);
              }
            }
          }
        }
        warp_reduce_scatter(a, lane);
        Real* rb = red + ((size_t)warp * NG + g) * VP;
#pragma unroll
        for (int i = 0; i < VM; ++i) rb[lane * VM + i] = a[i];
      }
#pragma unroll
      for (int k = 0; k < FT; ++k) pv[k] = yr[k];
      __syncthreads();
      // z for every row: one thread per row, fixed-order sums over warps
      for (int row = tid; row < R; row += NT) {
        const int g = row / RG, q = row - g * RG;
        Real nre = Real(0), nim = Real(0), den = Real(0);
        for (int w = 0; w < NW; ++w) {
          const Real* rb = red + ((size_t)w * NG + g) * VP;
          nre += rb[q];
          nim += rb[RG + q];
          den += rb[2 * RG + q];
        }
        R2 z;
        if (!(den > Real(0)) || !isfinite(den)) atomicMin(&s_badrow, row);
        if (row == r) {
          z.x = Real(1) - sqrt((Real)T / den);
          z.y = Real(0);
          onemz[r] = (double)(Real(1) - z.x);
        } else {
          z.x = nre / den;
          z.y = nim / den;
        }
        zsh[row] = z;
      }
      __syncthreads();
      if (s_badrow != 0x7fffffff) {
        if (tid == 0) record_err<Real>(p.err, mix, err_key(p.iteration, kPhSweep, gbin, r, (unsigned)s_badrow));
        aborted = true;
        break;
      }
      // iss_apply, W -= z w_r, ping-pong
      const R2* Wo = Wb + (r & 1) * R * D;
      R2* Wn = Wb + ((r + 1) & 1) * R * D;
      for (int e = tid; e < R * D; e += NT) {
        const int q = e % R, c = e / R;
        R2 w = Wo[e];
        cmsub(w, zsh[q], Wo[c * R + r]);
        Wn[e] = w;
      }
      if constexpr (CHECK) {
        if (p.chk_flags & 2) {  // steering_row_power of the updated row r (estimator.cpp:571-576)
          const R2 zr2 = zsh[r];
          const int wo = p.woff[r];
          Real q = Real(0);
#pragma unroll
          for (int k = 0; k < FT; ++k) {
            const int j = tid + k * NT;
            R2 y = yr[k];
            cmsub(y, zr2, yr[k]);
            if (j < T) q = fma(cnorm(y), invl[wo + j], q);
          }
          double v1[1] = {(double)q};
          block_sum_d<1>(v1, dred, lane, warp, NW);
          if (tid == 0) c_norm = fmax(c_norm, fabs(v1[0] / T - 1.0));
        }
        if (p.chk_flags & 1) {
          __syncthreads();  // W' complete
          check_det(Wn, (double)zsh[r].x, true);
        }
      }
    }
    if constexpr (CHECK) {
      if (!aborted) {
        if (tid == 0) {
          if (p.chk_flags & 2) chk_max(p.chk + (size_t)mix * 2 + 1, c_norm);
          if (p.chk_flags & 1) chk_max(p.chk + (size_t)mix * 2, c_det);
        }
      }
    }
    if (aborted) continue;
    // last step's update, row powers, |y|^2 -> delayed energies (frame-local
    // writes, then shifted reads after a barrier)
    const R2* Wf = Wb + (R & 1) * R * D;
    {
      Real rp[((RG + 31) / 32) * 32];
      for (int g = 0; g < NG; ++g) {
#pragma unroll
        for (int i = 0; i < ((RG + 31) / 32) * 32; ++i) rp[i] = Real(0);
#pragma unroll
        for (int q = 0; q < RG; ++q) {
          const int row = g * RG + q;
          if (row < R) {
            const R2 zp = zsh[row];
#pragma unroll
            for (int k = 0; k < FT; ++k) {
              const int j = tid + k * NT;
              R2 y = Yg[(size_t)row * TP + j];
              cmsub(y, zp, pv[k]);
              Yg[(size_t)row * TP + j] = y;
              rp[q] += cnorm(y);
            }
          }
        }
        warp_reduce_scatter(rp, lane);
        Real* rb = red + ((size_t)warp * NG + g) * VP;
        constexpr int RPV = ((RG + 31) / 32);
#pragma unroll
        for (int i = 0; i < RPV; ++i) rb[lane * RPV + i] = rp[i];
      }
    }
    __syncthreads();
    for (int row = tid; row < R; row += NT) {
      const int g = row / RG, q = row - g * RG;
      constexpr int RPV = ((RG + 31) / 32);
      double s = 0.0;
      for (int w = 0; w < NW; ++w) s += (double)red[((size_t)w * NG + g) * VP + q / RPV * RPV + q % RPV];
      p.rowpow[tile * R + row] = s;
    }
    if (tid == 0) {
      double prod = 1.0;
      for (int r = 0; r < R; ++r) prod *= onemz[r];
      p.logdet[tile] = logdet + log(prod);
    }
    Real* Eg = reinterpret_cast<Real*>(p.E);
    for (int n = 0; n < N; ++n) {
      const int r0 = p.row0[n], Ln = p.ntaps[n];
      for (int tau = tid; tau < TP; tau += NT) {
        Real e = Real(0);
        for (int l = 0; l < Ln && tau + l < T; ++l) e += cnorm(Yg[(size_t)(r0 + l) * TP + tau + l]);
        if (tau < T) Eg[(((size_t)mix * N + n) * p.FL + bin) * T + tau] = e;
      }
    }
    for (int i = tid; i < R * D; i += NT) Wg[i] = Wf[i];
    __syncthreads();
    // MU-B (estimator.cpp:313-346): warps take bases, lanes stride frames;
    // E is re-read from global (L2-hot, just written by this CTA)
    for (int n = 0; n < N; ++n) {
      const int k0 = p.koff[n], k1 = p.koff[n + 1], Ln = p.ntaps[n];
      const Real* il = invl + n * p.lp + p.loff;
      const Real* En = Eg + (((size_t)mix * N + n) * p.FL + bin) * T;
      for (int kb = k0 + warp; kb < k1; kb += NW) {
        const Real* vrow = Vg + (size_t)kb * T;
        Real num = Real(0), dd = Real(0);
        for (int tau = lane; tau < T; tau += 32) {
          const Real ilv = il[tau];
          const Real v = __ldg(vrow + tau);
          num = fma(En[tau] * (ilv * ilv), v, num);
          dd = fma(ilv * (Real)min(Ln, T - tau), v, dd);
        }
        num = warp_sum(num);
        dd = warp_sum(dd);
        if (lane == 0) Bg[kb] = fmax(Bs[kb] * sqrt(num / dd), floor_abs);
      }
    }
  }
}

}  // namespace ctf
