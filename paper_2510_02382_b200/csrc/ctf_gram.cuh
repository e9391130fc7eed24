// ctf_gram.cuh — covariance-domain ISS iteration kernel (fp32, stacked
// equal-tap configs).
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
template <int CNT, int N, int UB, bool MASK>
__device__ __forceinline__ void gram_step(const float2* __restrict__ x1, const float2* __restrict__ x2,
                                          const float* __restrict__ w0, int lp, int u, int u1,
                                          float (&wv)[N][UB + CNT - 1], float2 (&acc)[N][CNT]) {
  float2 q[UB];
#pragma unroll
  for (int i = 0; i < UB; ++i) {
    // q = a conj(b) = (a.x, a.y) b.x + (a.y, -a.x) b.y, packed
    const float2 a = x1[u + i], b = x2[u + i];
    q[i] = ffma2s(make_float2(a.y, -a.x), b.y, fmul2s(a, b.x));
    if (MASK && u + i >= u1) q[i] = make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int n = 0; n < N; ++n) {
#pragma unroll
    for (int k = 0; k < CNT - 1; ++k) wv[n][k] = wv[n][k + UB];
#pragma unroll
    for (int i = 0; i < UB; ++i) wv[n][CNT - 1 + i] = w0[n * lp + u + i];
#pragma unroll
    for (int i = 0; i < UB; ++i)
#pragma unroll
      for (int j = 0; j < CNT; ++j) acc[n][j] = ffma2s(q[i], wv[n][CNT - 1 + i - j], acc[n][j]);
  }
}

// acc[n][j] += sum_{u in [u0, u1)} x1(u) conj(x2(u)) w_n(u - a_lo - j); w0
// points at w_n(-a_lo). The weight window w_n(u - a_lo - (CNT-1) .. u + UB - 1
// - a_lo) lives in registers and slides by UB per block (UB new loads per
// source instead of UB + CNT - 1). Chunks have odd lengths (host), so the
// threads of a warp start on distinct banks and stay there; only the last
// block of a chunk is masked.
template <int CNT, int N, int UB>
__device__ __forceinline__ void gram_block(const float2* __restrict__ x1, const float2* __restrict__ x2,
                                           const float* __restrict__ w0, int lp, int u0, int u1,
                                           float2 (&acc)[N][CNT]) {
  float wv[N][UB + CNT - 1];
#pragma unroll
  for (int n = 0; n < N; ++n)
#pragma unroll
    for (int k = 0; k < CNT - 1; ++k) wv[n][k + UB] = w0[n * lp + u0 - (CNT - 1) + k];
  int u = u0;
  for (; u + UB <= u1; u += UB) gram_step<CNT, N, UB, false>(x1, x2, w0, lp, u, u1, wv, acc);
  if (u < u1) gram_step<CNT, N, UB, true>(x1, x2, w0, lp, u, u1, wv, acc);
}

template <int M, int L, int NT, int FT>
__global__ void __launch_bounds__(NT, (NT <= 256 ? 3 : 1))
    gram_kernel(const SweepParams p, const int4* __restrict__ gtab) {
  constexpr int N = M, R = M * L, D = M * L, NA = 2 * L - 1, NW = NT / 32;
  constexpr int LT1 = L > 1 ? L - 1 : 1;
  static_assert(D <= 32, "one lane per stacked channel in the covariance steps");
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bin = blockIdx.x, mix = blockIdx.y;
  const int gbin = p.bin_lo + bin;
  const int T = p.T, TP = p.TP, SK = p.SK;

  float2* xs = reinterpret_cast<float2*>(smem + p.off_x);    // M rows of xp: x_m(t) at [m*xp + xoff + t]
  float* invl = reinterpret_cast<float*>(smem + p.off_l);    // N rows of lp: w_n(s) at [n*lp + loff + s]
  float2* G = reinterpret_cast<float2*>(smem + p.off_y);     // [n][m][m'][a][b]
  float2* part = reinterpret_cast<float2*>(smem + p.off_e);  // [n*NA + j][NT + 1] Gram partials
  float* Pq = reinterpret_cast<float*>(smem + p.off_e);      // [r][TP] |y|^2 (after the steps)
  float* Es = reinterpret_cast<float*>(smem + p.off_x);      // [n][TP] energies (x tile is dead then)
  float2* Wb = reinterpret_cast<float2*>(smem + p.off_w);    // 2 x R x D (ping-pong)
  float2* Yt = reinterpret_cast<float2*>(smem + p.off_z);    // R x LT1 tail frames (+ R x LT1 spare)
  float2* zs = Yt + 2 * R * LT1;                             // 2 x (D + LT1) pivot buffers
  float* red = reinterpret_cast<float*>(smem + p.off_red);   // 32 * NW
  float* Bs = reinterpret_cast<float*>(smem + p.off_b);
  double* dred = reinterpret_cast<double*>(smem + p.off_d);
  __shared__ int s_bad, s_badrow;
  __shared__ double s_logmu, s_dprod;
  constexpr int kNoRow = 1 << 30;

  const size_t tile = (size_t)mix * p.FL + bin;
#ifdef CTF_PHASE_TIMING
#define CTF_PHASE(k) \
  if (tid == 0 && tile < 4096) g_phase[tile * 12 + (k)] = clock64();
#else
#define CTF_PHASE(k)
#endif
  CTF_PHASE(0);
  prefetch_next_tile(p, bin, mix, (size_t)T * M * sizeof(float2), (size_t)R * D * sizeof(float2));
  const float2* xg = reinterpret_cast<const float2*>(p.x) + tile * (size_t)T * M;
  float2* Wg = reinterpret_cast<float2*>(p.W) + tile * (size_t)R * D;
  float* Bg = reinterpret_cast<float*>(p.Bf) + tile * SK;
  const float* Vg = reinterpret_cast<const float*>(p.V) + (size_t)mix * SK * T;
  const float floor_abs = (float)p.floor_abs[mix];
  const int prev_it = p.iteration - 1;
  const double* mu = p.mu ? p.mu + (size_t)mix * R : nullptr;
  auto gidx = [](int n, int m, int m2, int a, int b) {  // a, b in [-(L-1), L-1]
    return (((n * M + m) * M + m2) * NA + a + L - 1) * NA + b + L - 1;
  };

  if (tid == 0) {
    s_bad = 0;
    s_badrow = kNoRow;
    s_logmu = mu ? p.logmu[mix] : 0.0;
  }
  // ---- prologue: zero-padded x tile, W and B with the pending rescale
  if ((T * M) % 2 == 0) {
    // the bin's T x M complex block is contiguous: 16-byte loads, all in
    // flight before the first store (latency, not bandwidth, bounds this)
    constexpr int XV = FT * M / 2;  // >= (T*M/2) / NT since T <= FT*NT
    const int n16 = T * M / 2;
    const float4* xv = reinterpret_cast<const float4*>(xg);
    float4 v[XV];
#pragma unroll
    for (int i = 0; i < XV; ++i) {
      const int e = tid + i * NT;
      if (e < n16) v[i] = __ldg(xv + e);
    }
    for (int i = tid; i < M * p.xp; i += NT) {
      const int t = i % p.xp - p.xoff;
      if (t < 0 || t >= T) xs[i] = make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < XV; ++i) {
      const int e = tid + i * NT;
      if (e < n16) {
        const int f0 = 2 * e, f1 = 2 * e + 1;
        xs[(f0 % M) * p.xp + p.xoff + f0 / M] = make_float2(v[i].x, v[i].y);
        xs[(f1 % M) * p.xp + p.xoff + f1 / M] = make_float2(v[i].z, v[i].w);
      }
    }
  } else {
    for (int i = tid; i < M * p.xp; i += NT) {
      const int m = i / p.xp, t = i - m * p.xp - p.xoff;
      xs[i] = (t >= 0 && t < T) ? xg[(size_t)t * M + m] : make_float2(0.f, 0.f);
    }
  }
  for (int i = tid; i < R * D; i += NT) Wb[i] = Wg[i];
  for (int i = tid; i < SK; i += NT) Bs[i] = Bg[i];
  __shared__ float s_imu[R];  // 1 / mu_r of the pending rescale (1 where none)
  if (warp == 0 && lane < R) s_imu[lane] = (mu && mu[lane] != 0.0) ? (float)(1.0 / mu[lane]) : 1.f;
  __syncthreads();
  // pending rescale (estimator.cpp:399-411) in fp32: W rows * (1/mu_r),
  // B_n * (1/mu_row0)^2 floored
  for (int i = tid; i < R * D; i += NT) {
    float2 w = Wb[i];
    const float im = s_imu[i % R];
    w.x *= im;
    w.y *= im;
    Wb[i] = w;
    if (p.has_prev && !cfinite(w)) s_bad = 1;
  }
  if (mu)
    for (int n = 0; n < N; ++n) {
      if (mu[p.row0[n]] == 0.0) continue;  // estimator.cpp:405-406: silent row, no rescale
      const float im = s_imu[p.row0[n]];
      for (int i = p.koff[n] + tid; i < p.koff[n + 1]; i += NT) Bs[i] = fmaxf(Bs[i] * (im * im), floor_abs);
    }
  __syncthreads();
  CTF_PHASE(1);
  if (p.has_prev && s_bad) {  // check_all_finite on W (estimator.cpp:494-496)
    if (tid == 0) record_err<float>(p.err, mix, err_key(prev_it, kPhFinite, gbin, 0, 1));
    return;
  }
  // ---- lambda = max(B V, floor) -> 1/lambda (zero outside [0, T)), log term
  double logsum = 0.0;
  for (int n = 0; n < N; ++n) {
    float* il = invl + n * p.lp;
    for (int i = tid; i < p.lp; i += NT) {
      const int s = i - p.loff;
      if (s < 0 || s >= T) il[i] = 0.f;
    }
    const int k0 = p.koff[n], k1 = p.koff[n + 1];
    if (T % 4 == 0) {
      // four consecutive frames per thread, 16-byte V loads (FT == 4 threads' worth)
      static_assert(FT == 4, "vector lambda path assumes four frames per thread");
      const int t4 = tid * 4;
      if (t4 < T) {
        float4 lam = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
        for (int kk = k0; kk < k1; ++kk) {
          const float b = Bs[kk];
          const float4 v = __ldg(reinterpret_cast<const float4*>(Vg + (size_t)kk * T + t4));
          lam.x = fmaf(b, v.x, lam.x);
          lam.y = fmaf(b, v.y, lam.y);
          lam.z = fmaf(b, v.z, lam.z);
          lam.w = fmaf(b, v.w, lam.w);
        }
        const float lv[4] = {lam.x, lam.y, lam.z, lam.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float l = fmaxf(lv[i], floor_abs);
          il[p.loff + t4 + i] = 1.f / l;
          if (p.has_prev) logsum += (double)min(L, T - t4 - i) * (double)logf(l);
        }
      }
    } else {
      float lam[FT];
#pragma unroll
      for (int k = 0; k < FT; ++k) lam[k] = 0.f;
#pragma unroll 4
      for (int kk = k0; kk < k1; ++kk) {
        const float b = Bs[kk];
        const float* vrow = Vg + (size_t)kk * T;
#pragma unroll
        for (int k = 0; k < FT; ++k) {
          const int tau = tid + k * NT;
          if (tau < T) lam[k] = fmaf(b, __ldg(vrow + tau), lam[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        const int tau = tid + k * NT;
        if (tau < T) {
          const float l = fmaxf(lam[k], floor_abs);
          il[p.loff + tau] = 1.f / l;
          if (p.has_prev) logsum += (double)min(L, T - tau) * (double)logf(l);
        }
      }
    }
  }
  __syncthreads();
  CTF_PHASE(2);

  // ---- virtual tail frames j in [T, T+L-1): y_r(j) = sum_c W[r,c] x~_c(j)
  for (int e = tid; e < R * (L - 1); e += NT) {
    const int r = e % R, jj = e / R, j = T + jj;
    float2 y = make_float2(0.f, 0.f);
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
      for (int l = 0; l < L; ++l) cmac(y, Wb[(m * L + l) * R + r], xs[m * p.xp + p.xoff + j - l]);
    Yt[r * LT1 + jj] = y;
  }

  // ---- Gram: this thread's (m, m', d) task over frames [u0, u1). The lag
  // count is made warp-uniform (groups are sorted by it, so a warp spans at
  // most two adjacent counts): no divergent code paths, extra lags discarded.
  {
    const int4 tk = gtab[tid];
    const bool active = tk.x >= 0;
    const int4 g0 = gtab[NT + 1 + 2 * max(tk.x, 0)], g1 = gtab[NT + 2 + 2 * max(tk.x, 0)];
    const int cnt = active ? g1.x : 0;
    const int cmax = __reduce_max_sync(kFull, cnt);
    const float2* x1 = xs + g0.x * p.xp + p.xoff;
    const float2* x2 = xs + g0.y * p.xp + p.xoff + g0.z;
    const float* w0 = invl + p.loff - g0.w;
    static_for<L, NA + 1>([&](auto cc) {
      constexpr int C = decltype(cc)::value;
      if (cmax == C) {
        float2 acc[N][C];
#pragma unroll
        for (int n = 0; n < N; ++n)
#pragma unroll
          for (int j = 0; j < C; ++j) acc[n][j] = make_float2(0.f, 0.f);
        if (active) gram_block<C, N, kGramUB>(x1, x2, w0, p.lp, tk.y, tk.z, acc);
#pragma unroll
        for (int n = 0; n < N; ++n)
#pragma unroll
          for (int j = 0; j < C; ++j)
            if (j < cnt) part[(size_t)(n * NA + j) * (NT + 1) + tid] = acc[n][j];
      }
    });
  }
  __syncthreads();
  CTF_PHASE(3);
  // fixed-order reduction over each group's chunks, Hermitian mirror
  {
    const int ng = gtab[NT].x;
    for (int e = tid; e < ng * N * NA; e += NT) {
      const int g = e / (N * NA), rr = e - g * (N * NA), n = rr / NA, j = rr - n * NA;
      const int4 g0 = gtab[NT + 1 + 2 * g], g1 = gtab[NT + 2 + 2 * g];
      if (j >= g1.x) continue;
      float2 s = make_float2(0.f, 0.f);
      const float2* pr = part + (size_t)(n * NA + j) * (NT + 1);
      for (int t = g1.y; t < g1.z; ++t) {
        s.x += pr[t].x;
        s.y += pr[t].y;
      }
      const int m = g0.x, m2 = g0.y, d = g0.z, a = g0.w + j, b = a + d;
      G[gidx(n, m, m2, a, b)] = s;
      G[gidx(n, m2, m, b, a)] = make_float2(s.x, (m == m2 && d == 0) ? s.y : -s.y);
    }
  }
  __syncthreads();
  CTF_PHASE(4);

  // ---- covariance-domain steps with register-resident rows: half-warp
  // `row` = 2*warp + half owns W row p; its lane c < D holds W[p][c], the row
  // c of C_p (D complex), and for c < l_p the tail frame T + c of y_p with
  // its weight w_n(T + c - l_p). A step needs only the pivot row (W_r and its
  // tail), published through shared memory: one barrier per step.
  constexpr int HW = 16;
  static_assert(D <= HW && L - 1 <= HW, "one half-warp per row");
  static_assert(R <= 2 * NW, "a half-warp per row");
  const int hl = lane & (HW - 1), half = lane >> 4;
  const int row = 2 * warp + half;
  const bool rowv = row < R;
  const int rn = rowv ? row / L : 0, rl = rowv ? row - rn * L : 0;
  float2 creg[D];
  float2 wreg = make_float2(0.f, 0.f), yreg = make_float2(0.f, 0.f);
  float wt = 0.f;
  {
    const bool chan = rowv && hl < D;
    const int m = hl / L, l1 = hl - m * L;
#pragma unroll
    for (int m2 = 0; m2 < M; ++m2)
#pragma unroll
      for (int l2 = 0; l2 < L; ++l2)
        creg[m2 * L + l2] = chan ? G[gidx(rn, m, m2, rl - l1, rl - l2)] : make_float2(0.f, 0.f);
    if (chan) wreg = Wb[hl * R + row];
    if (rowv && hl < L - 1) yreg = Yt[row * LT1 + hl];                // carried for when this row pivots
    if (rowv && hl < rl) wt = invl[rn * p.lp + p.loff + T + hl - rl];  // own truncation: frames T .. T+l-1
  }
  // (num, den) of this row against a pivot: pw[c * ps] = pivot W, py[c] = pivot tail
  auto row_sums = [&](const float2* pw, int ps, const float2* py, float& nre, float& nim, float& den) {
    float2 q0 = make_float2(0.f, 0.f), q1 = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c < D; ++c) {  // q += C conj(w) = (C.x, C.y) w.x + (C.y, -C.x) w.y
      const float2 w = pw[c * ps];
      float2& q = (c & 1) ? q1 : q0;
      q = ffma2s(make_float2(creg[c].y, -creg[c].x), w.y, ffma2s(creg[c], w.x, q));
    }
    const float2 q = make_float2(q0.x + q1.x, q0.y + q1.y);
    const float2 wr = (hl < D) ? pw[hl * ps] : make_float2(0.f, 0.f);
    float2 cn = cmul(wreg, q), cd = cmul(wr, q);
    // virtual frames T + hl (hl < l_p): subtract w y_p conj(y_r), w |y_r|^2
    const float2 yr = (hl < LT1) ? py[hl] : make_float2(0.f, 0.f);
    cn.x -= wt * fmaf(yreg.x, yr.x, yreg.y * yr.y);
    cn.y -= wt * fmaf(yreg.y, yr.x, -yreg.x * yr.y);
    cd.x -= wt * fmaf(yr.x, yr.x, yr.y * yr.y);
#pragma unroll
    for (int o = HW / 2; o >= 1; o >>= 1) {
      cn.x += __shfl_xor_sync(kFull, cn.x, o);
      cn.y += __shfl_xor_sync(kFull, cn.y, o);
      cd.x += __shfl_xor_sync(kFull, cd.x, o);
    }
    nre = cn.x;
    nim = cn.y;
    den = cd.x;
  };

  double logdet = p.logdet[tile] - s_logmu;
  if (p.has_prev) {
    // objective of the previous iteration (estimator.cpp:55-77): quadratic
    // term sum_r w_r^T C_r conj(w_r) of the rescaled W under the new lambda
    float nre, nim, den;
    row_sums(Wb + (rowv ? row : 0), R, Yt + (rowv ? row : 0) * LT1, nre, nim, den);
    if (hl == 0 && rowv) red[row] = den;
    double v1[1] = {logsum};
    block_sum_d<1>(v1, dred, lane, warp, NW);  // contains __syncthreads: red visible after
    double quad = 0.0;
    for (int r = 0; r < R; ++r) quad += (double)red[r];
    const int det_status = isnan(logdet) || logdet == -INFINITY ? 4 : (logdet < log(1e-300) ? 5 : 0);
    if (det_status) {  // estimator.cpp:45-51
      if (tid == 0) record_err<float>(p.err, mix, err_key(prev_it, kPhDet, gbin, 0, det_status));
      return;
    }
    if (tid == 0) p.objbin[tile] = v1[0] + quad - 2.0 * (double)T * logdet;
  }

  if (!p.do_sweep) {  // finalize pass: write the rescaled state and stop
    for (int i = tid; i < R * D; i += NT) Wg[i] = Wb[i];
    for (int i = tid; i < SK; i += NT) Bg[i] = Bs[i];
    if (tid == 0) p.logdet[tile] = logdet;
    return;
  }

  // ---- R covariance-domain ISS steps (estimator.cpp:556-579, 275-302)
  float2* piv = zs;  // 2 x (D + LT1): pivot W row and tail, double-buffered by step parity
  float* fac = red;  // (1 - z_r) per row, multiplied in row order at the end
  constexpr int PV = D + LT1;
  if (row == 0) {
    if (hl < D) piv[hl] = wreg;
    if (hl < LT1) piv[D + hl] = yreg;
  }
  __syncthreads();
  CTF_PHASE(5);
  const bool wrows = 2 * warp < R;  // warp-uniform: this warp owns at least one row
  for (int r = 0; r < R; ++r) {
    const float2* pv = piv + (r & 1) * PV;
    float nre = 0.f, nim = 0.f, den = 0.f;
    if (wrows) row_sums(pv, 1, pv + D, nre, nim, den);
    float2 z = make_float2(0.f, 0.f);
    if (rowv) {
      if (!(den > 0.f) || !isfinite(den)) {  // estimator.cpp:451-454
        if (hl == 0) atomicMin(&s_badrow, row);
      } else if (row == r) {
        z.x = 1.f - sqrtf((float)T) * rsqrtf(den);
        if (hl == 0) fac[row] = 1.f - z.x;
      } else {
        const float inv = __frcp_rn(den);
        z.x = nre * inv;
        z.y = nim * inv;
      }
    }
    // iss_apply (estimator.cpp:298-302) on the own row and its tail
    if (hl < D) cmsub(wreg, z, pv[hl]);
    if (hl < LT1) cmsub(yreg, z, pv[D + hl]);
    if (row == r + 1) {  // the next pivot publishes its updated row
      float2* nx = piv + ((r + 1) & 1) * PV;
      if (hl < D) nx[hl] = wreg;
      if (hl < LT1) nx[D + hl] = yreg;
    }
    __syncthreads();
    if (s_badrow != kNoRow) {
      if (tid == 0) record_err<float>(p.err, mix, err_key(p.iteration, kPhSweep, gbin, r, s_badrow));
      return;
    }
  }
  float2* Wf = Wb;  // W' (column-major R x D) for the demix
  if (rowv && hl < D) Wf[hl * R + row] = wreg;
  if (tid == 0) {
    double dp = 1.0;
    for (int r = 0; r < R; ++r) dp *= (double)fac[r];
    s_dprod = dp;
  }
  __syncthreads();
  CTF_PHASE(6);

  // ---- Y = W' x~ (estimator.cpp:607) for this thread's frames: |y|^2 to
  // shared memory, row powers and the finite check on the way
  float rp[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) rp[i] = 0.f;
  bool ybad = false;
#pragma unroll 1
  for (int k = 0; k < FT; ++k) {
    const int j = tid + k * NT;
    static_assert(R % 2 == 0, "W columns are read in 16-byte pairs");
    float2 acc[R];
#pragma unroll
    for (int i = 0; i < R; ++i) acc[i] = make_float2(0.f, 0.f);
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
      for (int l1 = 0; l1 < L; ++l1) {
        const float2 xv = xs[m * p.xp + p.xoff + j - l1];
        const float2 xn = make_float2(-xv.y, xv.x);
        const float4* wc = reinterpret_cast<const float4*>(Wf + (m * L + l1) * R);
#pragma unroll
        for (int i = 0; i < R; i += 2) {
          const float4 w = wc[i / 2];
          acc[i] = ffma2s(xn, w.y, ffma2s(xv, w.x, acc[i]));
          acc[i + 1] = ffma2s(xn, w.w, ffma2s(xv, w.z, acc[i + 1]));
        }
      }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const float q = (j < T) ? cnorm(acc[i]) : 0.f;
      Pq[i * TP + j] = q;
      rp[i] += q;
    }
  }
  // check_all_finite on Y (estimator.cpp:497-499): a non-finite estimate
  // makes its row's power sum non-finite
#pragma unroll
  for (int i = 0; i < R; ++i) ybad |= !isfinite(rp[i]);
  if (ybad) s_bad = 1;
  __syncthreads();      // Pq complete; the x tile is dead from here (Es aliases it)
  CTF_PHASE(7);
  if (s_bad) {
    if (tid == 0) record_err<float>(p.err, mix, err_key(p.iteration, kPhFinite, gbin, 0, 2));
    return;
  }
  // delayed energies E_n(tau) = sum_{l, tau+l<T} |y_(n,l)(tau+l)|^2 (l order)
  float* Eg = reinterpret_cast<float*>(p.E);
  for (int n = 0; n < N; ++n)
#pragma unroll
    for (int k = 0; k < FT; ++k) {
      const int tau = tid + k * NT;
      float e = 0.f;
#pragma unroll
      for (int l = 0; l < L; ++l)
        if (tau + l < T) e += Pq[(n * L + l) * TP + tau + l];
      Es[n * TP + tau] = e;
      if (tau < T) Eg[(((size_t)mix * N + n) * p.FL + bin) * T + tau] = e;
    }
  // row powers (estimator.cpp:391-397)
  warp_reduce_scatter(rp, lane);
  red[warp * 32 + lane] = rp[0];
  __syncthreads();
  if (tid < R) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += (double)red[w * 32 + tid];
    p.rowpow[tile * R + tid] = s;
  }
  if (tid == 0) p.logdet[tile] = logdet + log(s_dprod);
  for (int i = tid; i < R * D; i += NT) Wg[i] = Wf[i];
  __syncthreads();
  CTF_PHASE(8);

  // ---- MU-B for this bin (estimator.cpp:313-346), 16 bases per pass
  for (int n = 0; n < N; ++n) {
    const int k0 = p.koff[n], k1 = p.koff[n + 1];
    const float* il = invl + n * p.lp + p.loff;
    for (int kb = k0; kb < k1; kb += 16) {
      float a[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) a[i] = 0.f;
      const float* vrow[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) vrow[q] = Vg + (size_t)min(kb + q, k1 - 1) * T + tid;
#pragma unroll
      for (int k = 0; k < FT; ++k) {
        const int tau = tid + k * NT;
        const float ilv = il[tau];
        const float an = Es[n * TP + tau] * (ilv * ilv);
        const float bn = (tau < T) ? ilv * (float)min(L, T - tau) : 0.f;
        const float2 ab = make_float2(an, bn);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const float vv = __ldg(vrow[q] + k * NT);
          const float2 t = ffma2s(ab, vv, make_float2(a[q], a[16 + q]));
          a[q] = t.x;
          a[16 + q] = t.y;
        }
      }
      warp_reduce_scatter(a, lane);
      __syncthreads();  // previous pass's reads of red are done
      red[warp * 32 + lane] = a[0];
      __syncthreads();
      if (tid < 16 && kb + tid < k1) {
        float num = 0.f, den = 0.f;
        for (int w = 0; w < NW; ++w) {
          num += red[w * 32 + tid];
          den += red[w * 32 + 16 + tid];
        }
        const float b = Bs[kb + tid];
        Bg[kb + tid] = fmaxf(b * sqrtf(num / den), floor_abs);
      }
    }
  }
  CTF_PHASE(9);
}

}  // namespace ctf
