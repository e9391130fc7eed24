// synth.cpp — synthetic CTF mixtures exactly as BASELINE.json configs[0]
// describes (host code; the bench and the parity tests share it so the
// oracle and the GPU see identical inputs).
//
// Mixture b, rng = std::mt19937_64(base_seed + b), draws in this order:
//   for source n: T_n(f,k) ~ Gamma(1,1) + 1e-3   (f outer, k inner)
//                 V_n(k,t) ~ Gamma(1,1) + 1e-3   (k outer, t inner)
//                 s_n(f,t) = sqrt(r_n(f,t)/2) (g + i g'), r_n = T_n V_n (f outer, t inner; g then g')
//   for f, for l < L, for m < M, for n < N: A_l(f)[m][n] ~ CN(0, decay^l)  (re then im, each N(0, decay^l/2))
//   for f, for t, for m: noise ~ CN(0, 1e-4)                             (re then im)
//   x_m(f,t) = sum_l sum_n A_l(f)[m][n] s_n(f, t-l) + noise  (s = 0 for t < 0)
// Pattern follows the reference generator (proj/src/synth.cpp:11-128) with
// BASELINE's distributions (Gamma factors, tap variance decay^l, no
// conditioning gate).
#include "../../include/ctf_iss.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <exception>
#include <random>
#include <string>
#include <thread>
#include <vector>

namespace {

using C = std::complex<double>;

void synth_one(int F, int T, int M, int N, int L, int K, double decay, uint64_t seed, int out_prec, void* out) {
  std::mt19937_64 rng(seed);
  std::gamma_distribution<double> gam(1.0, 1.0);
  std::normal_distribution<double> gauss(0.0, 1.0);
  std::vector<C> s((size_t)N * F * T);  // s[n][f][t]
  std::vector<double> tb((size_t)F * K), va((size_t)K * T);
  for (int n = 0; n < N; ++n) {
    for (int f = 0; f < F; ++f)
      for (int k = 0; k < K; ++k) tb[(size_t)f * K + k] = gam(rng) + 1e-3;
    for (int k = 0; k < K; ++k)
      for (int t = 0; t < T; ++t) va[(size_t)k * T + t] = gam(rng) + 1e-3;
    for (int f = 0; f < F; ++f)
      for (int t = 0; t < T; ++t) {
        double r = 0.0;
        for (int k = 0; k < K; ++k) r += tb[(size_t)f * K + k] * va[(size_t)k * T + t];
        const double sigma = std::sqrt(r / 2.0);
        const double g = gauss(rng);
        const double gp = gauss(rng);
        s[((size_t)n * F + f) * T + t] = C(sigma * g, sigma * gp);
      }
  }
  std::vector<C> A((size_t)F * L * M * N);  // A[f][l][m][n]
  for (int f = 0; f < F; ++f)
    for (int l = 0; l < L; ++l) {
      const double sd = std::sqrt(std::pow(decay, l) / 2.0);
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
          const double re = gauss(rng);
          const double im = gauss(rng);
          A[(((size_t)f * L + l) * M + m) * N + n] = C(sd * re, sd * im);
        }
    }
  const double nsd = std::sqrt(1e-4 / 2.0);
  for (int f = 0; f < F; ++f)
    for (int t = 0; t < T; ++t)
      for (int m = 0; m < M; ++m) {
        C acc(0, 0);
        for (int l = 0; l < L && l <= t; ++l)
          for (int n = 0; n < N; ++n)
            acc += A[(((size_t)f * L + l) * M + m) * N + n] * s[((size_t)n * F + f) * T + (t - l)];
        const double re = gauss(rng);
        const double im = gauss(rng);
        acc += C(nsd * re, nsd * im);
        const size_t e = ((size_t)f * T + t) * M + m;
        if (out_prec == CTF_F64) {
          static_cast<double*>(out)[2 * e] = acc.real();
          static_cast<double*>(out)[2 * e + 1] = acc.imag();
        } else {
          static_cast<float*>(out)[2 * e] = (float)acc.real();
          static_cast<float*>(out)[2 * e + 1] = (float)acc.imag();
        }
      }
}

}  // namespace

extern "C" int ctf_synth_mixtures(int num_mixtures, int F, int T, int M, int N, int L, int K, double tap_decay,
                                  uint64_t base_seed, int out_precision, void* x_out, int threads, ctf_err* err) {
  if (err) {
    err->code = 0;
    err->msg[0] = 0;
  }
  if (num_mixtures < 1 || F < 1 || T < 1 || M < 1 || N < 1 || L < 1 || K < 1 || !x_out) {
    if (err) {
      err->code = CTF_ERR_CONFIG;
      std::snprintf(err->msg, sizeof(err->msg), "ctf_synth_mixtures: bad arguments");
    }
    return CTF_ERR_CONFIG;
  }
  const size_t per = (size_t)F * T * M * 2 * (out_precision == CTF_F64 ? 8 : 4);
  int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = std::min(nt, num_mixtures);
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs((size_t)nt);
  for (int w = 0; w < nt; ++w)
    pool.emplace_back([&, w] {
      try {
        for (int b = w; b < num_mixtures; b += nt)
          synth_one(F, T, M, N, L, K, tap_decay, base_seed + (uint64_t)b, out_precision,
                    static_cast<char*>(x_out) + per * (size_t)b);
      } catch (...) {
        errs[(size_t)w] = std::current_exception();
      }
    });
  for (auto& t : pool) t.join();
  for (auto& e : errs)
    if (e) {
      if (err) {
        err->code = CTF_ERR_CONFIG;
        std::snprintf(err->msg, sizeof(err->msg), "ctf_synth_mixtures failed");
      }
      return CTF_ERR_CONFIG;
    }
  return 0;
}
