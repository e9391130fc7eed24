// ctf_oracle.cpp — TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline arm).
//
// Plain-C++ restatement (std::complex<double>, no Eigen) of the reference
// CTF-MNMF estimator in /root/reference/proj. Every function cites the
// reference file:line it restates. Never linked into the product library.
// See ctf_oracle.h for layouts and for how the oracle is pinned.

#include "ctf_oracle.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

using C = std::complex<double>;

// ---------------------------------------------------------------------------
// Error types: restatement of proj/include/ctfmnmf/errors.hpp:11-35.
struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct DegeneracyError : std::runtime_error {
  DegeneracyError(const std::string& m, int it = -1, int b = -1, int r = -1)
      : std::runtime_error(m), iteration(it), bin(b), row(r) {}
  int iteration, bin, row;
};

// parallel_for: proj/include/ctfmnmf/threading.hpp:15-43 (contiguous chunks,
// first error in chunk order is rethrown).
void parallel_for(int begin, int end, int threads, const std::function<void(int)>& fn) {
  const int count = end - begin;
  if (count <= 0) return;
  threads = std::max(1, std::min(threads, count));
  if (threads == 1) {
    for (int i = begin; i < end; ++i) fn(i);
    return;
  }
  const int chunk = (count + threads - 1) / threads;
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(static_cast<size_t>(threads));
  for (int t = 0; t < threads; ++t) {
    const int lo = begin + t * chunk, hi = std::min(end, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([&, lo, hi, t] {
      try {
        for (int i = lo; i < hi; ++i) fn(i);
      } catch (...) {
        errs[static_cast<size_t>(t)] = std::current_exception();
      }
    });
  }
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

// Column-major dense matrices (Eigen's default storage order).
struct CMat {
  int rows = 0, cols = 0;
  std::vector<C> a;
  CMat() = default;
  CMat(int r, int c) : rows(r), cols(c), a(static_cast<size_t>(r) * c, C(0, 0)) {}
  C& operator()(int r, int c) { return a[static_cast<size_t>(r) + static_cast<size_t>(c) * rows]; }
  const C& operator()(int r, int c) const {
    return a[static_cast<size_t>(r) + static_cast<size_t>(c) * rows];
  }
};
struct RMat {
  int rows = 0, cols = 0;
  std::vector<double> a;
  RMat() = default;
  RMat(int r, int c) : rows(r), cols(c), a(static_cast<size_t>(r) * c, 0.0) {}
  double& operator()(int r, int c) { return a[static_cast<size_t>(r) + static_cast<size_t>(c) * rows]; }
  double operator()(int r, int c) const {
    return a[static_cast<size_t>(r) + static_cast<size_t>(c) * rows];
  }
};

struct Config {
  int N = 0, D = 0;
  std::vector<int> taps, bases;
  int iterations = 0, rule = 1, threads = 1;
  double psd_floor = 1e-10;
  uint64_t seed = 0;
  int R() const {
    int s = 0;
    for (int l : taps) s += l;
    return s;
  }
  int row_offset(int n) const {  // model.cpp:26-30
    int o = 0;
    for (int m = 0; m < n; ++m) o += taps[static_cast<size_t>(m)];
    return o;
  }
  int base_offset(int n) const {
    int o = 0;
    for (int m = 0; m < n; ++m) o += bases[static_cast<size_t>(m)];
    return o;
  }
  int sumK() const { return base_offset(N); }
  void validate() const {  // model.cpp:32-50
    if (N < 1) throw ConfigError("n_sources must be >= 1");
    if (D < 1) throw ConfigError("n_channels must be >= 1");
    if (static_cast<int>(taps.size()) != N) throw ConfigError("taps list must have one entry per source");
    if (static_cast<int>(bases.size()) != N) throw ConfigError("bases list must have one entry per source");
    for (int l : taps)
      if (l < 1) throw ConfigError("every tap count must be >= 1");
    for (int k : bases)
      if (k < 1) throw ConfigError("every basis count must be >= 1");
    if (R() != D)
      throw ConfigError("sum of taps (" + std::to_string(R()) + ") must equal n_channels (" +
                        std::to_string(D) + "): the demixing system must be square");
    if (iterations < 0) throw ConfigError("iters must be >= 0");
    if (!(psd_floor > 0.0)) throw ConfigError("floor must be > 0");
    if (threads < 1) throw ConfigError("threads must be >= 1");
  }
};

Config from_c(const orc_config* c) {
  Config cfg;
  cfg.N = c->num_sources;
  cfg.D = c->num_channels;
  if (cfg.N < 0 || cfg.N > ORC_MAX_SOURCES) throw ConfigError("n_sources out of range");
  cfg.taps.assign(c->taps, c->taps + cfg.N);
  cfg.bases.assign(c->bases, c->bases + cfg.N);
  cfg.iterations = c->iterations;
  cfg.rule = c->rule;
  cfg.psd_floor = c->psd_floor;
  cfg.seed = c->seed;
  cfg.threads = c->threads;
  return cfg;
}

struct RowMap {  // estimator.cpp:416-429 via unflatten_index (model.cpp:141-151)
  std::vector<int> src, tap;
  explicit RowMap(const Config& cfg) {
    for (int n = 0; n < cfg.N; ++n)
      for (int l = 0; l < cfg.taps[static_cast<size_t>(n)]; ++l) {
        src.push_back(n);
        tap.push_back(l);
      }
  }
};

struct Factors {  // model.hpp:70-80
  std::vector<RMat> B, V;
  double floor = 1e-12;
};

// ---------------------------------------------------------------------------
// Model pieces.

double mean_power(const std::vector<CMat>& x) {  // model.cpp:153-161
  double total = 0.0;
  int64_t count = 0;
  for (const auto& b : x) {
    double s = 0.0;
    for (const C& v : b.a) s += std::norm(v);
    total += s;
    count += static_cast<int64_t>(b.a.size());
  }
  return count > 0 ? total / static_cast<double>(count) : 0.0;
}

Factors random_factors(const Config& cfg, int F, int T, double floor_abs,
                       std::mt19937_64& rng) {  // model.cpp:189-208
  std::uniform_real_distribution<double> uni(0.1, 1.0);
  Factors f;
  f.floor = floor_abs;
  for (int n = 0; n < cfg.N; ++n) {
    const int K = cfg.bases[static_cast<size_t>(n)];
    RMat b(F, K), v(K, T);
    for (int i = 0; i < F; ++i)
      for (int k = 0; k < K; ++k) b(i, k) = uni(rng);
    for (int k = 0; k < K; ++k)
      for (int j = 0; j < T; ++j) v(k, j) = uni(rng);
    f.B.push_back(std::move(b));
    f.V.push_back(std::move(v));
  }
  return f;
}

RMat compute_psd(const Factors& f, int n) {  // model.cpp:210-215
  const RMat& b = f.B[static_cast<size_t>(n)];
  const RMat& v = f.V[static_cast<size_t>(n)];
  RMat lam(b.rows, v.cols);
  for (int j = 0; j < v.cols; ++j)
    for (int i = 0; i < b.rows; ++i) {
      double acc = 0.0;
      for (int k = 0; k < b.cols; ++k) acc += b(i, k) * v(k, j);
      lam(i, j) = std::max(acc, f.floor);
    }
  return lam;
}

std::vector<CMat> identity_demixing(const Config& cfg, int F) {  // model.cpp:221-227
  std::vector<CMat> w(static_cast<size_t>(F), CMat(cfg.R(), cfg.D));
  for (auto& m : w)
    for (int r = 0; r < std::min(m.rows, m.cols); ++r) m(r, r) = C(1, 0);
  return w;
}

// ---------------------------------------------------------------------------
// Estimator pieces (proj/src/estimator.cpp).

// LU with partial pivoting, log|det| accumulation (estimator.cpp:41-53).
double log_abs_det(const CMat& m) {
  const int n = m.rows;
  CMat a = m;
  double acc = 0.0;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    double best = std::abs(a(c, c));
    for (int r = c + 1; r < n; ++r)
      if (std::abs(a(r, c)) > best) {
        best = std::abs(a(r, c));
        piv = r;
      }
    if (piv != c)
      for (int j = 0; j < n; ++j) std::swap(a(c, j), a(piv, j));
    const C p = a(c, c);
    const double mag = std::abs(p);
    if (!(mag > 0.0) || !std::isfinite(mag))
      throw DegeneracyError("singular demixing matrix (zero pivot)");
    acc += std::log(mag);
    for (int r = c + 1; r < n; ++r) {
      const C f = a(r, c) / p;
      for (int j = c + 1; j < n; ++j) a(r, j) -= f * a(c, j);
    }
  }
  if (acc < std::log(1e-300)) throw DegeneracyError("demixing determinant magnitude below 1e-300");
  return acc;
}

// Full inverse via the same pivoted LU (used by wiener.cpp:35-36).
CMat inverse(const CMat& m) {
  const int n = m.rows;
  CMat a = m, inv(n, n);
  for (int i = 0; i < n; ++i) inv(i, i) = C(1, 0);
  for (int c = 0; c < n; ++c) {
    int piv = c;
    double best = std::abs(a(c, c));
    for (int r = c + 1; r < n; ++r)
      if (std::abs(a(r, c)) > best) {
        best = std::abs(a(r, c));
        piv = r;
      }
    if (piv != c)
      for (int j = 0; j < n; ++j) {
        std::swap(a(c, j), a(piv, j));
        std::swap(inv(c, j), inv(piv, j));
      }
    const C p = a(c, c);
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      const C f = a(r, c) / p;
      if (f == C(0, 0)) continue;
      for (int j = 0; j < n; ++j) {
        a(r, j) -= f * a(c, j);
        inv(r, j) -= f * inv(c, j);
      }
    }
  }
  for (int r = 0; r < n; ++r) {
    const C p = a(r, r);
    for (int j = 0; j < n; ++j) inv(r, j) /= p;
  }
  return inv;
}

CMat matmul(const CMat& a, const CMat& b) {
  CMat out(a.rows, b.cols);
  for (int j = 0; j < b.cols; ++j)
    for (int r = 0; r < a.rows; ++r) {
      C acc(0, 0);
      for (int c = 0; c < a.cols; ++c) acc += a(r, c) * b(c, j);
      out(r, j) = acc;
    }
  return out;
}

std::vector<CMat> demix(const std::vector<CMat>& W, const std::vector<CMat>& x) {  // :304-311
  std::vector<CMat> y(x.size());
  for (size_t i = 0; i < x.size(); ++i) y[i] = matmul(W[i], x[i]);
  return y;
}

double objective_from_parts(const std::vector<CMat>& W, const std::vector<RMat>& lam,
                            const std::vector<CMat>& Y, const Config& cfg) {  // :55-77
  const RowMap rm(cfg);
  const int F = static_cast<int>(Y.size());
  const int T = F ? Y[0].cols : 0;
  double obj = 0.0;
  for (int i = 0; i < F; ++i) {
    const CMat& y = Y[static_cast<size_t>(i)];
    for (int r = 0; r < cfg.R(); ++r) {
      const RMat& l = lam[static_cast<size_t>(rm.src[static_cast<size_t>(r)])];
      const int tap = rm.tap[static_cast<size_t>(r)];
      for (int j = tap; j < T; ++j) {
        const double v = l(i, j - tap);
        obj += std::log(v) + std::norm(y(r, j)) / v;
      }
    }
    obj -= 2.0 * T * log_abs_det(W[static_cast<size_t>(i)]);
  }
  return obj;
}

CMat weighted_covariance(const std::vector<CMat>& x, const RMat& lam, int tap, int bin) {  // :89-101
  const CMat& xi = x[static_cast<size_t>(bin)];
  const int D = xi.rows, T = xi.cols;
  CMat q(D, D);
  for (int j = tap; j < T; ++j) {
    const double l = lam(bin, j - tap);
    for (int b = 0; b < D; ++b)
      for (int a = 0; a < D; ++a) q(a, b) += xi(a, j) * std::conj(xi(b, j)) / l;
  }
  for (C& v : q.a) v /= static_cast<double>(T);
  CMat h(D, D);
  for (int b = 0; b < D; ++b)
    for (int a = 0; a < D; ++a) h(a, b) = 0.5 * (q(a, b) + std::conj(q(b, a)));
  return h;
}

// Covariance-domain ISS (estimator.cpp:275-302).
std::vector<C> iss_compute_z(const CMat& w, const std::vector<CMat>& covs, int row) {
  const int R = w.rows, D = w.cols;
  std::vector<C> wr(static_cast<size_t>(D));
  for (int c = 0; c < D; ++c) wr[static_cast<size_t>(c)] = std::conj(w(row, c));
  std::vector<C> z(static_cast<size_t>(R));
  for (int p = 0; p < R; ++p) {
    const CMat& q = covs[static_cast<size_t>(p)];
    std::vector<C> qw(static_cast<size_t>(D), C(0, 0));
    for (int c = 0; c < D; ++c)
      for (int a = 0; a < D; ++a) qw[static_cast<size_t>(a)] += q(a, c) * wr[static_cast<size_t>(c)];
    C den(0, 0);
    for (int a = 0; a < D; ++a) den += std::conj(wr[static_cast<size_t>(a)]) * qw[static_cast<size_t>(a)];
    const double denom = den.real();
    if (!(denom > 0.0) || !std::isfinite(denom))
      throw DegeneracyError("steering update: nonpositive denominator for rows (" +
                                std::to_string(row) + ", " + std::to_string(p) + ")",
                            -1, -1, row);
    if (p == row) {
      z[static_cast<size_t>(p)] = C(1.0 - 1.0 / std::sqrt(denom), 0.0);
    } else {
      C num(0, 0);  // w_p^H (Q_p w_r), w_p = conj(row p)
      for (int a = 0; a < D; ++a) num += w(p, a) * qw[static_cast<size_t>(a)];
      z[static_cast<size_t>(p)] = num / denom;
    }
  }
  return z;
}

void iss_apply(CMat& w, const std::vector<C>& z, int row) {  // :298-302
  std::vector<C> pre(static_cast<size_t>(w.cols));
  for (int c = 0; c < w.cols; ++c) pre[static_cast<size_t>(c)] = w(row, c);
  for (int c = 0; c < w.cols; ++c)
    for (int p = 0; p < w.rows; ++p) w(p, c) -= z[static_cast<size_t>(p)] * pre[static_cast<size_t>(c)];
}

// Estimate-domain steering vector (estimator.cpp:434-462).
std::vector<C> iss_steering(const CMat& y, const std::vector<RMat>& lam, const RowMap& rm, int bin,
                            int row) {
  const int R = y.rows, T = y.cols;
  std::vector<C> z(static_cast<size_t>(R));
  for (int p = 0; p < R; ++p) {
    const RMat& l = lam[static_cast<size_t>(rm.src[static_cast<size_t>(p)])];
    const int tap = rm.tap[static_cast<size_t>(p)];
    C num(0, 0);
    double den = 0.0;
    for (int j = tap; j < T; ++j) {
      const double wgt = 1.0 / l(bin, j - tap);
      const C yr = y(row, j);
      den += std::norm(yr) * wgt;
      if (p != row) num += y(p, j) * std::conj(yr) * wgt;
    }
    if (!(den > 0.0) || !std::isfinite(den))
      throw DegeneracyError("steering update: nonpositive denominator for rows (" +
                                std::to_string(row) + ", " + std::to_string(p) + ")",
                            -1, bin, row);
    z[static_cast<size_t>(p)] = (p == row) ? C(1.0 - std::sqrt(static_cast<double>(T) / den), 0.0)
                                           : num / den;
  }
  return z;
}

double steering_row_power(const CMat& y, const RMat& lam, int bin, int row, int tap) {  // :464-472
  double q = 0.0;
  for (int j = tap; j < y.cols; ++j) q += std::norm(y(row, j)) / lam(bin, j - tap);
  return q / y.cols;
}

std::vector<C> iss_step(CMat& w, CMat& y, const std::vector<RMat>& lam, const RowMap& rm, int bin,
                        int row) {  // :476-484
  const std::vector<C> z = iss_steering(y, lam, rm, bin, row);
  std::vector<C> pre(static_cast<size_t>(y.cols));
  for (int j = 0; j < y.cols; ++j) pre[static_cast<size_t>(j)] = y(row, j);
  iss_apply(w, z, row);
  for (int j = 0; j < y.cols; ++j)
    for (int p = 0; p < y.rows; ++p) y(p, j) -= z[static_cast<size_t>(p)] * pre[static_cast<size_t>(j)];
  return z;
}

C determinant(const CMat& m) {  // Eigen determinant() via LU, sign from pivots
  const int n = m.rows;
  CMat a = m;
  C det(1, 0);
  for (int c = 0; c < n; ++c) {
    int piv = c;
    double best = std::abs(a(c, c));
    for (int r = c + 1; r < n; ++r)
      if (std::abs(a(r, c)) > best) {
        best = std::abs(a(r, c));
        piv = r;
      }
    if (piv != c) {
      for (int j = 0; j < n; ++j) std::swap(a(c, j), a(piv, j));
      det = -det;
    }
    const C p = a(c, c);
    det *= p;
    if (p == C(0, 0)) return C(0, 0);
    for (int r = c + 1; r < n; ++r) {
      const C f = a(r, c) / p;
      for (int j = c + 1; j < n; ++j) a(r, j) -= f * a(c, j);
    }
  }
  return det;
}

// IP row update, general LU path (estimator.cpp:220-257, 261-273). The small
// fixed-size path (:123-208) uses the same pivot rule with squared
// magnitudes (threshold 1e-26 on |.|^2 == 1e-13 on |.|).
void ip_update(CMat& w, const CMat& cov, int row) {
  const int m = cov.rows;
  auto attempt = [&](const CMat& q, std::vector<C>& sol) -> bool {
    CMat a = matmul(w, q);
    std::vector<C> rhs(static_cast<size_t>(m), C(0, 0));
    rhs[static_cast<size_t>(row)] = C(1, 0);
    std::vector<int> perm(static_cast<size_t>(m));
    double minp = std::numeric_limits<double>::infinity(), maxp = 0.0;
    for (int c = 0; c < m; ++c) {
      int piv = c;
      double best = std::abs(a(c, c));
      for (int r = c + 1; r < m; ++r)
        if (std::abs(a(r, c)) > best) {
          best = std::abs(a(r, c));
          piv = r;
        }
      if (piv != c) {
        for (int j = 0; j < m; ++j) std::swap(a(c, j), a(piv, j));
        std::swap(rhs[static_cast<size_t>(c)], rhs[static_cast<size_t>(piv)]);
      }
      minp = std::min(minp, best);
      maxp = std::max(maxp, best);
      if (!(best > 0.0)) continue;
      for (int r = c + 1; r < m; ++r) {
        const C f = a(r, c) / a(c, c);
        for (int j = c + 1; j < m; ++j) a(r, j) -= f * a(c, j);
        rhs[static_cast<size_t>(r)] -= f * rhs[static_cast<size_t>(c)];
      }
    }
    if (!(minp > 1e-13 * maxp)) return false;
    sol.assign(static_cast<size_t>(m), C(0, 0));
    for (int r = m - 1; r >= 0; --r) {
      C acc = rhs[static_cast<size_t>(r)];
      for (int j = r + 1; j < m; ++j) acc -= a(r, j) * sol[static_cast<size_t>(j)];
      sol[static_cast<size_t>(r)] = acc / a(r, r);
    }
    for (const C& s : sol)
      if (!std::isfinite(s.real()) || !std::isfinite(s.imag())) return false;
    return true;
  };
  std::vector<C> sol;
  if (!attempt(cov, sol)) {
    double tr = 0.0;
    for (int i = 0; i < m; ++i) tr += cov(i, i).real();
    CMat loaded = cov;
    for (int i = 0; i < m; ++i) loaded(i, i) += 1e-10 * tr / m;
    if (!attempt(loaded, sol))
      throw DegeneracyError("projection update: singular system after diagonal loading", -1, -1, row);
  }
  double norm2 = 0.0;
  for (int i = 0; i < m; ++i) {
    C wgt(0, 0);
    for (int j = 0; j < m; ++j) wgt += cov(i, j) * sol[static_cast<size_t>(j)];
    norm2 += (std::conj(sol[static_cast<size_t>(i)]) * wgt).real();
  }
  if (!(norm2 > 0.0) || !std::isfinite(norm2))
    throw DegeneracyError("projection update: nonpositive row power", -1, -1, row);
  const double s = 1.0 / std::sqrt(norm2);
  for (int c = 0; c < m; ++c) w(row, c) = std::conj(sol[static_cast<size_t>(c)]) * s;
}

// Energy E(i, tau) = sum_{l: tau+l<T} |y_{row0+l}(tau+l)|^2 and the tap count
// (estimator.cpp:321-332 and :356-368, identical in both MU updates).
void delayed_energy(const std::vector<CMat>& Y, int row0, int taps, RMat& energy,
                    std::vector<double>& count) {
  const int F = static_cast<int>(Y.size());
  const int T = Y[0].cols;
  energy = RMat(F, T);
  count.assign(static_cast<size_t>(T), 0.0);
  for (int l = 0; l < taps; ++l)
    for (int tau = 0; tau + l < T; ++tau) count[static_cast<size_t>(tau)] += 1.0;
  for (int i = 0; i < F; ++i)
    for (int l = 0; l < taps; ++l)
      for (int tau = 0; tau + l < T; ++tau) energy(i, tau) += std::norm(Y[static_cast<size_t>(i)](row0 + l, tau + l));
}

void mu_update_bases(Factors& f, const std::vector<CMat>& Y, int n, const Config& cfg) {  // :313-346
  const RMat lam = compute_psd(f, n);
  RMat energy;
  std::vector<double> count;
  delayed_energy(Y, cfg.row_offset(n), cfg.taps[static_cast<size_t>(n)], energy, count);
  const RMat& v = f.V[static_cast<size_t>(n)];
  RMat& b = f.B[static_cast<size_t>(n)];
  const int F = b.rows, K = b.cols, T = v.cols;
  RMat out(F, K);
  for (int k = 0; k < K; ++k)
    for (int i = 0; i < F; ++i) {
      double num = 0.0, den = 0.0;
      for (int j = 0; j < T; ++j) {
        const double il = 1.0 / lam(i, j);  // cwiseInverse, then array products as in :336-340
        num += (energy(i, j) * (il * il)) * v(k, j);
        den += (il * count[static_cast<size_t>(j)]) * v(k, j);
      }
      out(i, k) = std::max(b(i, k) * std::sqrt(num / den), f.floor);
    }
  b = std::move(out);
}

void mu_update_activations(Factors& f, const std::vector<CMat>& Y, int n, const Config& cfg) {  // :348-382
  const RMat lam = compute_psd(f, n);
  RMat energy;
  std::vector<double> count;
  delayed_energy(Y, cfg.row_offset(n), cfg.taps[static_cast<size_t>(n)], energy, count);
  const RMat& b = f.B[static_cast<size_t>(n)];
  RMat& v = f.V[static_cast<size_t>(n)];
  const int F = b.rows, K = b.cols, T = v.cols;
  RMat out(K, T);
  for (int j = 0; j < T; ++j)
    for (int k = 0; k < K; ++k) {
      double num = 0.0, den = 0.0;
      for (int i = 0; i < F; ++i) {
        const double il = 1.0 / lam(i, j);  // :370-376
        num += b(i, k) * (energy(i, j) * (il * il));
        den += b(i, k) * (il * count[static_cast<size_t>(j)]);
      }
      out(k, j) = std::max(v(k, j) * std::sqrt(num / den), f.floor);
    }
  v = std::move(out);
}

void rescale(std::vector<CMat>& W, Factors& f, std::vector<CMat>& Y, const Config& cfg) {  // :384-412
  const int F = static_cast<int>(Y.size());
  if (F == 0) return;
  const int T = Y[0].cols, R = cfg.R();
  if (T == 0) return;
  std::vector<double> mu(static_cast<size_t>(R));
  for (int r = 0; r < R; ++r) {
    double power = 0.0;
    for (int i = 0; i < F; ++i) {
      double s = 0.0;
      for (int j = 0; j < T; ++j) s += std::norm(Y[static_cast<size_t>(i)](r, j));
      power += s;
    }
    mu[static_cast<size_t>(r)] = std::sqrt(power / (static_cast<double>(F) * T));
  }
  for (int r = 0; r < R; ++r) {
    const double m = mu[static_cast<size_t>(r)];
    if (m == 0.0) continue;
    for (int i = 0; i < F; ++i) {
      for (int c = 0; c < W[static_cast<size_t>(i)].cols; ++c) W[static_cast<size_t>(i)](r, c) /= m;
      for (int j = 0; j < T; ++j) Y[static_cast<size_t>(i)](r, j) /= m;
    }
  }
  for (int n = 0; n < cfg.N; ++n) {
    const double m0 = mu[static_cast<size_t>(cfg.row_offset(n))];
    if (m0 == 0.0) continue;
    for (double& b : f.B[static_cast<size_t>(n)].a) b = std::max(b / (m0 * m0), f.floor);
  }
}

void check_all_finite(const std::vector<CMat>& W, const std::vector<CMat>& Y, int it) {  // :491-501
  auto finite = [](const CMat& m) {
    for (const C& v : m.a)
      if (!std::isfinite(v.real()) || !std::isfinite(v.imag())) return false;
    return true;
  };
  for (size_t i = 0; i < W.size(); ++i) {
    if (!finite(W[i])) throw DegeneracyError("non-finite demixing matrix", it, static_cast<int>(i));
    if (!finite(Y[i])) throw DegeneracyError("non-finite source estimates", it, static_cast<int>(i));
  }
}

struct CheckStats {
  bool det_lemma = false, normalization = false;
  double max_det = 0.0, max_norm = 0.0;
  int64_t checked = 0;
};

struct State {
  std::vector<CMat> W;
  Factors f;
};

// One iteration body, estimator.cpp:548-654. Returns the objective.
double iterate_once(const Config& cfg, const std::vector<CMat>& x, State& st, int iter,
                    CheckStats* checks, double* ms3) {
  const int F = static_cast<int>(x.size());
  const int R = cfg.R();
  const RowMap rm(cfg);
  std::vector<RMat> lam(static_cast<size_t>(cfg.N));
  for (int n = 0; n < cfg.N; ++n) lam[static_cast<size_t>(n)] = compute_psd(st.f, n);
  std::vector<double> det_err(static_cast<size_t>(F), 0.0), norm_err(static_cast<size_t>(F), 0.0);
  std::vector<CMat> Y;
  const auto t0 = std::chrono::steady_clock::now();
  try {
    if (cfg.rule == 1) {
      Y = demix(st.W, x);
      parallel_for(0, F, cfg.threads, [&](int i) {
        CMat& w = st.W[static_cast<size_t>(i)];
        CMat& y = Y[static_cast<size_t>(i)];
        for (int r = 0; r < R; ++r) {
          C before(0, 0);
          if (checks && checks->det_lemma) before = determinant(w);
          const std::vector<C> z = iss_step(w, y, lam, rm, i, r);
          if (checks && checks->det_lemma) {
            const C after = determinant(w);
            const C pred = before * (C(1, 0) - z[static_cast<size_t>(r)]);
            const double scale = std::max(std::abs(after), 1e-300);
            det_err[static_cast<size_t>(i)] = std::max(det_err[static_cast<size_t>(i)], std::abs(after - pred) / scale);
          }
          if (checks && checks->normalization) {
            const double q = steering_row_power(y, lam[static_cast<size_t>(rm.src[static_cast<size_t>(r)])], i, r,
                                                rm.tap[static_cast<size_t>(r)]);
            norm_err[static_cast<size_t>(i)] = std::max(norm_err[static_cast<size_t>(i)], std::abs(q - 1.0));
          }
        }
      });
    } else {
      parallel_for(0, F, cfg.threads, [&](int i) {
        CMat& w = st.W[static_cast<size_t>(i)];
        const CMat& xi = x[static_cast<size_t>(i)];
        for (int r = 0; r < R; ++r) {
          const RMat& l = lam[static_cast<size_t>(rm.src[static_cast<size_t>(r)])];
          const int tap = rm.tap[static_cast<size_t>(r)];
          ip_update(w, weighted_covariance(x, l, tap, i), r);
          CMat wr(1, w.cols);
          for (int c = 0; c < w.cols; ++c) wr(0, c) = w(r, c);
          CMat est = matmul(wr, xi);
          const double power = steering_row_power(est, l, i, 0, tap);
          if (power > 0.0 && std::isfinite(power))
            for (int c = 0; c < w.cols; ++c) w(r, c) /= std::sqrt(power);
          if (checks && checks->normalization) {
            for (int c = 0; c < w.cols; ++c) wr(0, c) = w(r, c);
            est = matmul(wr, xi);
            const double q = steering_row_power(est, l, i, 0, tap);
            norm_err[static_cast<size_t>(i)] = std::max(norm_err[static_cast<size_t>(i)], std::abs(q - 1.0));
          }
        }
      });
    }
    Y = demix(st.W, x);
  } catch (const DegeneracyError& e) {
    throw DegeneracyError(std::string(e.what()) + " (iteration " + std::to_string(iter + 1) + ")", iter + 1,
                          e.bin, e.row);
  }
  if (checks && (checks->det_lemma || checks->normalization)) {
    for (int i = 0; i < F; ++i) {
      checks->max_det = std::max(checks->max_det, det_err[static_cast<size_t>(i)]);
      checks->max_norm = std::max(checks->max_norm, norm_err[static_cast<size_t>(i)]);
    }
    checks->checked += static_cast<int64_t>(F) * R;
  }
  const auto t1 = std::chrono::steady_clock::now();
  for (int n = 0; n < cfg.N; ++n) mu_update_bases(st.f, Y, n, cfg);
  for (int n = 0; n < cfg.N; ++n) mu_update_activations(st.f, Y, n, cfg);
  const auto t2 = std::chrono::steady_clock::now();
  rescale(st.W, st.f, Y, cfg);
  for (int n = 0; n < cfg.N; ++n) lam[static_cast<size_t>(n)] = compute_psd(st.f, n);
  const auto t3 = std::chrono::steady_clock::now();
  check_all_finite(st.W, Y, iter + 1);
  double obj;
  try {
    obj = objective_from_parts(st.W, lam, Y, cfg);
  } catch (const DegeneracyError& e) {
    throw DegeneracyError(std::string(e.what()) + " (iteration " + std::to_string(iter + 1) + ")", iter + 1,
                          e.bin, e.row);
  }
  if (!std::isfinite(obj)) throw DegeneracyError("non-finite objective", iter + 1);
  if (ms3) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    ms3[0] = ms(t0, t1);
    ms3[1] = ms(t1, t2);
    ms3[2] = ms(t2, t3);
  }
  return obj;
}

// ---------------------------------------------------------------------------
// Marshalling between flat C buffers and the matrix types.

std::vector<CMat> load_bins(const double* p, int F, int rows, int cols) {
  std::vector<CMat> v(static_cast<size_t>(F), CMat(rows, cols));
  const size_t n = static_cast<size_t>(rows) * cols;
  for (int i = 0; i < F; ++i)
    std::memcpy(v[static_cast<size_t>(i)].a.data(), p + 2 * n * static_cast<size_t>(i), n * sizeof(C));
  return v;
}
void store_bins(const std::vector<CMat>& v, double* p) {
  if (!p) return;
  size_t off = 0;
  for (const auto& m : v) {
    std::memcpy(p + off, m.a.data(), m.a.size() * sizeof(C));
    off += 2 * m.a.size();
  }
}
Factors load_factors(const Config& cfg, int F, int T, const double* B, const double* V, double floor_abs) {
  Factors f;
  f.floor = floor_abs;
  size_t ob = 0, ov = 0;
  for (int n = 0; n < cfg.N; ++n) {
    const int K = cfg.bases[static_cast<size_t>(n)];
    RMat b(F, K), v(K, T);
    if (B) std::memcpy(b.a.data(), B + ob, b.a.size() * sizeof(double));
    if (V) std::memcpy(v.a.data(), V + ov, v.a.size() * sizeof(double));
    ob += b.a.size();
    ov += v.a.size();
    f.B.push_back(std::move(b));
    f.V.push_back(std::move(v));
  }
  return f;
}
void store_factors(const Factors& f, double* B, double* V) {
  size_t ob = 0, ov = 0;
  for (size_t n = 0; n < f.B.size(); ++n) {
    if (B) std::memcpy(B + ob, f.B[n].a.data(), f.B[n].a.size() * sizeof(double));
    if (V) std::memcpy(V + ov, f.V[n].a.data(), f.V[n].a.size() * sizeof(double));
    ob += f.B[n].a.size();
    ov += f.V[n].a.size();
  }
}
std::vector<RMat> load_lambda(int N, int F, int T, const double* p) {
  std::vector<RMat> l(static_cast<size_t>(N), RMat(F, T));
  for (int n = 0; n < N; ++n)
    std::memcpy(l[static_cast<size_t>(n)].a.data(), p + static_cast<size_t>(n) * F * T,
                static_cast<size_t>(F) * T * sizeof(double));
  return l;
}

void set_err(orc_err* err, int code, const char* msg, int it = -1, int bin = -1, int row = -1) {
  if (!err) return;
  err->code = code;
  err->iteration = it;
  err->bin = bin;
  err->row = row;
  std::snprintf(err->msg, sizeof(err->msg), "%s", msg);
}

template <class Fn>
int guarded(orc_err* err, Fn&& fn) {
  set_err(err, 0, "");
  try {
    fn();
    return 0;
  } catch (const ConfigError& e) {
    set_err(err, 2, e.what());
    return 2;
  } catch (const DegeneracyError& e) {
    set_err(err, 4, e.what(), e.iteration, e.bin, e.row);
    return 4;
  } catch (const std::exception& e) {
    set_err(err, 9, e.what());
    return 9;
  }
}

int run_impl(const orc_config* c, int F, int T, const double* x_flat, double* W_out, double* B_out,
             double* V_out, double* obj_out, double* hW, double* hB, double* hV, double* trace_ms,
             CheckStats* checks, orc_err* err) {
  return guarded(err, [&] {
    const Config cfg = from_c(c);
    cfg.validate();  // estimator.cpp:515-524
    const std::vector<CMat> x = load_bins(x_flat, F, cfg.D, T);
    const double mp = mean_power(x);
    if (!std::isfinite(mp)) throw DegeneracyError("mixture spectrogram contains non-finite values");
    if (!(mp > 0.0)) throw ConfigError("mixture spectrogram is identically zero");
    const double floor_abs = cfg.psd_floor * mp;
    std::mt19937_64 rng(cfg.seed);
    State st;
    st.f = random_factors(cfg, F, T, floor_abs, rng);
    st.W = identity_demixing(cfg, F);
    const size_t wsz = static_cast<size_t>(F) * cfg.R() * cfg.D * 2;
    const size_t bsz = static_cast<size_t>(F) * cfg.sumK(), vsz = static_cast<size_t>(cfg.sumK()) * T;
    for (int it = 0; it < cfg.iterations; ++it) {
      const double obj = iterate_once(cfg, x, st, it, checks, trace_ms ? trace_ms + 3 * it : nullptr);
      if (obj_out) obj_out[it] = obj;
      if (hW) store_bins(st.W, hW + wsz * static_cast<size_t>(it));
      if (hB || hV)
        store_factors(st.f, hB ? hB + bsz * static_cast<size_t>(it) : nullptr,
                      hV ? hV + vsz * static_cast<size_t>(it) : nullptr);
    }
    store_bins(st.W, W_out);
    store_factors(st.f, B_out, V_out);
  });
}

}  // namespace

// ---------------------------------------------------------------------------
// C entry points.

extern "C" {

int orc_run(const orc_config* cfg, int F, int T, const double* x, double* W_out, double* B_out,
            double* V_out, double* obj_out, double* hist_W, double* hist_B, double* hist_V,
            double* trace_ms_out, orc_err* err) {
  return run_impl(cfg, F, T, x, W_out, B_out, V_out, obj_out, hist_W, hist_B, hist_V, trace_ms_out,
                  nullptr, err);
}

int orc_run_checked(const orc_config* cfg, int F, int T, const double* x, double* max_det_err,
                    double* max_norm_err, int64_t* checked, orc_err* err) {
  CheckStats cs;
  cs.det_lemma = cs.normalization = true;
  const int rc = run_impl(cfg, F, T, x, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                          nullptr, &cs, err);
  *max_det_err = cs.max_det;
  *max_norm_err = cs.max_norm;
  *checked = cs.checked;
  return rc;
}

int orc_step(const orc_config* c, int F, int T, const double* x_flat, double floor_abs, double* W,
             double* B, double* V, double* obj_out, orc_err* err) {
  return guarded(err, [&] {
    const Config cfg = from_c(c);
    const std::vector<CMat> x = load_bins(x_flat, F, cfg.D, T);
    State st;
    st.W = load_bins(W, F, cfg.R(), cfg.D);
    st.f = load_factors(cfg, F, T, B, V, floor_abs);
    const double obj = iterate_once(cfg, x, st, 0, nullptr, nullptr);
    if (obj_out) *obj_out = obj;
    store_bins(st.W, W);
    store_factors(st.f, B, V);
  });
}

double orc_mean_power(int F, int D, int T, const double* x) { return mean_power(load_bins(x, F, D, T)); }

void orc_random_factors(const orc_config* c, int F, int T, double* B, double* V) {
  const Config cfg = from_c(c);
  std::mt19937_64 rng(cfg.seed);
  store_factors(random_factors(cfg, F, T, 0.0, rng), B, V);
}

int orc_demix(int F, int R, int D, int T, const double* W, const double* x, double* Y) {
  store_bins(demix(load_bins(W, F, R, D), load_bins(x, F, D, T)), Y);
  return 0;
}

int orc_iss_sweep(const orc_config* c, int F, int T, int bin, double* W_bin, double* Y_bin,
                  const double* lambda, orc_err* err) {  // estimator.cpp:505-511
  return guarded(err, [&] {
    const Config cfg = from_c(c);
    const RowMap rm(cfg);
    std::vector<CMat> w = load_bins(W_bin, 1, cfg.R(), cfg.D);
    std::vector<CMat> y = load_bins(Y_bin, 1, cfg.R(), T);
    const std::vector<RMat> lam = load_lambda(cfg.N, F, T, lambda);
    for (int r = 0; r < cfg.R(); ++r) iss_step(w[0], y[0], lam, rm, bin, r);
    store_bins(w, W_bin);
    store_bins(y, Y_bin);
  });
}

int orc_weighted_covariance(int F, int D, int T, const double* x, const double* lambda_n, int tap,
                            int bin, double* Q) {
  const std::vector<CMat> xv = load_bins(x, F, D, T);
  RMat l(F, T);
  std::memcpy(l.a.data(), lambda_n, l.a.size() * sizeof(double));
  store_bins({weighted_covariance(xv, l, tap, bin)}, Q);
  return 0;
}

int orc_iss_compute_z(int R, const double* W_bin, const double* covs, int row, double* z, orc_err* err) {
  return guarded(err, [&] {
    const std::vector<CMat> w = load_bins(W_bin, 1, R, R);
    const std::vector<CMat> q = load_bins(covs, R, R, R);
    const std::vector<C> zz = iss_compute_z(w[0], q, row);
    std::memcpy(z, zz.data(), zz.size() * sizeof(C));
  });
}

void orc_iss_apply(int R, int D, double* W_bin, const double* z, int row) {
  std::vector<CMat> w = load_bins(W_bin, 1, R, D);
  std::vector<C> zz(static_cast<size_t>(R));
  std::memcpy(zz.data(), z, zz.size() * sizeof(C));
  iss_apply(w[0], zz, row);
  store_bins(w, W_bin);
}

void orc_compute_psd(const orc_config* c, int F, int T, const double* B, const double* V, double floor_abs,
                     double* lambda) {
  const Config cfg = from_c(c);
  const Factors f = load_factors(cfg, F, T, B, V, floor_abs);
  for (int n = 0; n < cfg.N; ++n) {
    const RMat l = compute_psd(f, n);
    std::memcpy(lambda + static_cast<size_t>(n) * F * T, l.a.data(), l.a.size() * sizeof(double));
  }
}

void orc_mu_update_bases(const orc_config* c, int F, int T, double* B, const double* V, double floor_abs,
                         const double* Y, int source) {
  const Config cfg = from_c(c);
  Factors f = load_factors(cfg, F, T, B, V, floor_abs);
  mu_update_bases(f, load_bins(Y, F, cfg.R(), T), source, cfg);
  store_factors(f, B, nullptr);
}

void orc_mu_update_activations(const orc_config* c, int F, int T, const double* B, double* V,
                               double floor_abs, const double* Y, int source) {
  const Config cfg = from_c(c);
  Factors f = load_factors(cfg, F, T, B, V, floor_abs);
  mu_update_activations(f, load_bins(Y, F, cfg.R(), T), source, cfg);
  store_factors(f, nullptr, V);
}

void orc_rescale(const orc_config* c, int F, int T, double* W, double* B, double floor_abs, double* Y) {
  const Config cfg = from_c(c);
  std::vector<CMat> w = load_bins(W, F, cfg.R(), cfg.D);
  std::vector<CMat> y = load_bins(Y, F, cfg.R(), T);
  Factors f = load_factors(cfg, F, T, B, nullptr, floor_abs);
  rescale(w, f, y, cfg);
  store_bins(w, W);
  store_bins(y, Y);
  store_factors(f, B, nullptr);
}

int orc_log_abs_det(int R, const double* W_bin, double* out, orc_err* err) {
  return guarded(err, [&] { *out = log_abs_det(load_bins(W_bin, 1, R, R)[0]); });
}

int orc_objective_from_parts(const orc_config* c, int F, int T, const double* W, const double* lambda,
                             const double* Y, double* out, orc_err* err) {
  return guarded(err, [&] {
    const Config cfg = from_c(c);
    *out = objective_from_parts(load_bins(W, F, cfg.R(), cfg.D), load_lambda(cfg.N, F, T, lambda),
                                load_bins(Y, F, cfg.R(), T), cfg);
  });
}

int orc_objective(const orc_config* c, int F, int T, const double* W, const double* B, const double* V,
                  double floor_abs, const double* x, double* out, orc_err* err) {  // :79-87
  return guarded(err, [&] {
    const Config cfg = from_c(c);
    const Factors f = load_factors(cfg, F, T, B, V, floor_abs);
    std::vector<RMat> lam;
    for (int n = 0; n < cfg.N; ++n) lam.push_back(compute_psd(f, n));
    const std::vector<CMat> w = load_bins(W, F, cfg.R(), cfg.D);
    *out = objective_from_parts(w, lam, demix(w, load_bins(x, F, cfg.D, T)), cfg);
  });
}

int orc_reconstruct_images(const orc_config* c, int F, int T, const double* W, const double* x_flat,
                           double* images, orc_err* err) {  // wiener.cpp:11-49
  return guarded(err, [&] {
    const Config cfg = from_c(c);
    const std::vector<CMat> w = load_bins(W, F, cfg.R(), cfg.D);
    const std::vector<CMat> x = load_bins(x_flat, F, cfg.D, T);
    const size_t img = static_cast<size_t>(F) * cfg.D * T * 2;
    parallel_for(0, F, cfg.threads, [&](int i) {
      const CMat H = inverse(w[static_cast<size_t>(i)]);
      for (const C& v : H.a)
        if (!std::isfinite(v.real()) || !std::isfinite(v.imag()))
          throw DegeneracyError("image reconstruction: demixing matrix not invertible", -1, i);
      const CMat y = matmul(w[static_cast<size_t>(i)], x[static_cast<size_t>(i)]);
      for (int n = 0; n < cfg.N; ++n) {
        const int r0 = cfg.row_offset(n), L = cfg.taps[static_cast<size_t>(n)];
        double* out = images + img * static_cast<size_t>(n) + static_cast<size_t>(i) * cfg.D * T * 2;
        for (int j = 0; j < T; ++j)
          for (int d = 0; d < cfg.D; ++d) {
            C acc(0, 0);
            for (int l = 0; l < L; ++l) acc += H(d, r0 + l) * y(r0 + l, j);
            out[2 * (static_cast<size_t>(d) + static_cast<size_t>(j) * cfg.D)] = acc.real();
            out[2 * (static_cast<size_t>(d) + static_cast<size_t>(j) * cfg.D) + 1] = acc.imag();
          }
      }
    });
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// STFT front/back end: restatement of
// proj/src/fft.cpp:9-41 (iterative radix-2 FFT, recursive twiddles) and
// proj/src/stft.cpp:14-139 (periodic Hann, reflect padding, forward STFT,
// weighted overlap-add inverse). Layouts: TimeSignal.samples is length x
// channels column-major (sample t of channel c at c*length + t);
// Spectrogram.data is [bin][frame][channel] complex (types.hpp:22-47).
namespace {

constexpr double kPi = 3.14159265358979323846;  // std::numbers::pi

bool pow2(long long n) { return n > 0 && (n & (n - 1)) == 0; }

void fft_inplace(C* data, size_t n, bool inverse) {  // fft.cpp:9-41
  if (n <= 1) return;
  for (size_t i = 1, j = 0; i < n; ++i) {
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(data[i], data[j]);
  }
  const double sign = inverse ? 1.0 : -1.0;
  for (size_t len = 2; len <= n; len <<= 1) {
    const double angle = sign * 2.0 * kPi / static_cast<double>(len);
    const C wlen(std::cos(angle), std::sin(angle));
    for (size_t i = 0; i < n; i += len) {
      C w(1.0, 0.0);
      for (size_t k = 0; k < len / 2; ++k) {
        const C u = data[i + k];
        const C v = data[i + k + len / 2] * w;
        data[i + k] = u + v;
        data[i + k + len / 2] = u - v;
        w *= wlen;
      }
    }
  }
  if (inverse) {
    const double scale = 1.0 / static_cast<double>(n);
    for (size_t i = 0; i < n; ++i) data[i] *= scale;
  }
}

std::vector<double> hann(int len) {  // stft.cpp:14-19
  std::vector<double> w(static_cast<size_t>(len));
  for (int t = 0; t < len; ++t) w[static_cast<size_t>(t)] = 0.5 - 0.5 * std::cos(2.0 * kPi * t / len);
  return w;
}

std::vector<double> pad_channel(const double* x, int64_t n, int window_len, int64_t padded_len) {  // :25-42
  const int half = window_len / 2;
  std::vector<double> out(static_cast<size_t>(padded_len), 0.0);
  for (int t = 0; t < half; ++t) {
    int64_t src = half - t;
    if (src >= n) src = n - 1;
    out[static_cast<size_t>(t)] = x[src];
  }
  for (int64_t t = 0; t < n; ++t) out[static_cast<size_t>(half + t)] = x[t];
  for (int64_t t = half + n; t < padded_len; ++t) {
    int64_t src = 2 * n - 2 - (t - half);
    if (src < 0) src = 0;
    if (src >= n) break;
    out[static_cast<size_t>(t)] = x[src];
  }
  return out;
}

}  // namespace

extern "C" {

int orc_fft(double* data, int64_t n, int inverse, orc_err* err) {
  return guarded(err, [&] {
    if (!pow2(n)) throw ConfigError("fft: length must be a power of two");
    fft_inplace(reinterpret_cast<C*>(data), static_cast<size_t>(n), inverse != 0);
  });
}

void orc_hann(int len, double* out) {
  const std::vector<double> w = hann(len);
  std::memcpy(out, w.data(), w.size() * sizeof(double));
}

int64_t orc_stft_frames(int64_t length, int hop) { return 1 + (length + hop - 1) / hop; }

int orc_forward_stft(const double* samples, int64_t n, int channels, int window_len, int hop, double* spec,
                     orc_err* err) {  // stft.cpp:46-88
  return guarded(err, [&] {
    if (n == 0 || channels == 0) throw ConfigError("forward_stft: empty signal");
    if (window_len <= 0 || !pow2(window_len))
      throw ConfigError("forward_stft: window_len must be a power of two, got " + std::to_string(window_len));
    if (hop <= 0 || window_len % hop != 0) throw ConfigError("forward_stft: hop must divide window_len");
    if (n < window_len) throw ConfigError("forward_stft: signal shorter than one window");
    const int bins = window_len / 2 + 1;
    const int frames = static_cast<int>(1 + (n + hop - 1) / hop);
    const int64_t padded_len = static_cast<int64_t>(frames - 1) * hop + window_len;
    const std::vector<double> window = hann(window_len);
    std::vector<C> frame(static_cast<size_t>(window_len));
    C* out = reinterpret_cast<C*>(spec);
    for (int c = 0; c < channels; ++c) {
      const std::vector<double> padded = pad_channel(samples + static_cast<int64_t>(c) * n, n, window_len, padded_len);
      for (int j = 0; j < frames; ++j) {
        const int64_t start = static_cast<int64_t>(j) * hop;
        for (int t = 0; t < window_len; ++t)
          frame[static_cast<size_t>(t)] = C(padded[static_cast<size_t>(start + t)] * window[static_cast<size_t>(t)], 0.0);
        fft_inplace(frame.data(), static_cast<size_t>(window_len), false);
        for (int i = 0; i < bins; ++i)
          out[(static_cast<size_t>(i) * frames + j) * channels + c] = frame[static_cast<size_t>(i)];
      }
    }
  });
}

int orc_inverse_stft(const double* spec, int bins, int frames, int channels, int window_len, int hop,
                     int64_t original_length, double* out, int64_t* out_len_ret, orc_err* err) {  // :90-139
  return guarded(err, [&] {
    if (bins != window_len / 2 + 1) throw ConfigError("inverse_stft: bin count does not match window length");
    if (hop <= 0 || window_len % hop != 0) throw ConfigError("inverse_stft: hop must divide window_len");
    const int64_t padded_len = static_cast<int64_t>(frames - 1) * hop + window_len;
    const std::vector<double> window = hann(window_len);
    std::vector<double> overlap(static_cast<size_t>(padded_len), 0.0);
    for (int j = 0; j < frames; ++j)
      for (int t = 0; t < window_len; ++t)
        overlap[static_cast<size_t>(static_cast<int64_t>(j) * hop + t)] +=
            window[static_cast<size_t>(t)] * window[static_cast<size_t>(t)];
    const int half = window_len / 2;
    const int64_t out_len = original_length > 0 ? original_length : padded_len - window_len;
    if (out_len + half > padded_len) throw ConfigError("inverse_stft: original_length inconsistent with frames");
    const double peak = *std::max_element(overlap.begin(), overlap.end());
    for (int64_t t = half; t < half + out_len; ++t)
      if (overlap[static_cast<size_t>(t)] < 1e-9 * peak)
        throw ConfigError("inverse_stft: window/hop pair does not cover the signal");
    if (out_len_ret) *out_len_ret = out_len;
    if (!out) return;
    const C* sp = reinterpret_cast<const C*>(spec);
    auto at = [&](int i, int j, int c) { return sp[(static_cast<size_t>(i) * frames + j) * channels + c]; };
    std::vector<C> frame(static_cast<size_t>(window_len));
    std::vector<double> acc(static_cast<size_t>(padded_len));
    for (int c = 0; c < channels; ++c) {
      std::fill(acc.begin(), acc.end(), 0.0);
      for (int j = 0; j < frames; ++j) {
        for (int i = 0; i < bins; ++i) frame[static_cast<size_t>(i)] = at(i, j, c);
        for (int i = bins; i < window_len; ++i) frame[static_cast<size_t>(i)] = std::conj(at(window_len - i, j, c));
        fft_inplace(frame.data(), static_cast<size_t>(window_len), true);
        const int64_t start = static_cast<int64_t>(j) * hop;
        for (int t = 0; t < window_len; ++t)
          acc[static_cast<size_t>(start + t)] += frame[static_cast<size_t>(t)].real() * window[static_cast<size_t>(t)];
      }
      for (int64_t t = 0; t < out_len; ++t)
        out[static_cast<int64_t>(c) * out_len + t] =
            acc[static_cast<size_t>(half + t)] / overlap[static_cast<size_t>(half + t)];
    }
  });
}

}  // extern "C"
